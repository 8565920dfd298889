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
