"""Oracle: the Notay ratio of a preconditioner application (PAPER.md Eq. final_loss, and
Theorem 1's condition).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  eps(r) = || B(r) - A^{-1} r ||_A / || A^{-1} r ||_A ,   ||v||_A = sqrt((v, A v))

Written out directly from the definition: the caller passes w = B(r) and e = A^{-1} r; both
A-norms use the correctly rounded inner product (R6).  Theorem 1: FCG converges like CG with the
linear preconditioner the nonlinear one approximates when eps < 1 at every iteration.
"""
from __future__ import annotations

import math

import numpy as np

from .dots import dot
from .fcg import fcg


def a_norm(apply_A, v) -> float:
    """||v||_A = sqrt((v, A v))."""
    return math.sqrt(dot(v, apply_A(v)))


def notay_ratio(apply_A, w, e) -> float:
    """|| w - e ||_A / || e ||_A with w = B(r), e = A^{-1} r (Eq. final_loss's integrand)."""
    w = np.asarray(w, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    return a_norm(apply_A, w - e) / a_norm(apply_A, e)


def notay_ratio_scaled(apply_A, w, e) -> float:
    """min over c of ||c w - e||_A / ||e||_A, evaluated at the minimiser c* = (w, A e) / (w, A w)
    (FCG's iterates do not depend on the scale of B, so this is the scale-free form of eps)."""
    w = np.asarray(w, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    c = dot(w, apply_A(e)) / dot(w, apply_A(w))
    return a_norm(apply_A, c * w - e) / a_norm(apply_A, e)


def notay_curve(apply_A, f, u0, u_star, m_max, tol, maxit, precond=None, schedule="paper", vec32=False):
    """Theorem 1's quantities along Algorithm 1 (Fig. 2/4's curves):
    at every iteration i, after w_i = B(r_i), with e_i = u_star - u_i (u_star a reference solution, so
    that e_i approximates A^{-1} r_i):
      eps[i]   = ||w_i - e_i||_A / ||e_i||_A   (notay_ratio, Eq. final_loss's integrand)
      err_a[i] = ||e_i||_A
    Returns (fcg result dict, eps array, err_a array), both of length iters."""
    eps, err = [], []

    def observe(i, w, u):
        e = np.asarray(u_star, dtype=np.float64) - u
        eps.append(notay_ratio(apply_A, w, e))
        err.append(a_norm(apply_A, e))
    res = fcg(apply_A, f, u0, m_max, tol, maxit, precond=precond, schedule=schedule, vec32=vec32, observe=observe)
    return res, np.array(eps), np.array(err)
