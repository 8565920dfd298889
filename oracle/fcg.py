"""Oracle: Flexible Conjugate Gradients FCG(m) (Algorithm 1) and textbook CG.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Algorithm 1 as printed:
  r0 = f - A u0
  for i = 0 .. iter-1:
    w_i = B(r_i)
    m_i = min(i, max(1, mod(i, m_max+1)))
    p_i = w_i - sum_{k=i-m_i}^{i-1} (w_i, s_k)/(p_k, s_k) p_k
    s_i = A p_i
    u_{i+1} = u_i + (p_i, r_i)/(p_i, s_i) p_i
    r_{i+1} = r_i - (p_i, r_i)/(p_i, s_i) s_i
Readings:
  R12 stop at the first i with ||r_i||/||r_0|| <= tol (Table 1 caption), using
      the recurrence residual; ||r_0|| = 0 -> 0 iterations, converged;
  R13 all m_i coefficients are taken against w_i (classical Gram-Schmidt, as printed);
      canonical order p = w; for k newest -> oldest: p = p - beta_k p_k;
  R14 (p_i, s_i) <= 0 or non-finite -> BREAKDOWN; B(r) non-finite -> NONFINITE;
      the system stops with iters = i;
  R6  inner products are correctly rounded (oracle/dots.py);
  R15 u0 is an input (BASELINE configs use u0 = 0; P:102's u0 ~ N(0,1) is used for the
      Table 1 pin);
  R21 optional fp32 storage of r, w, p, s (vec32, BASELINE configs[2] "fp32 or fp64 FCG").
"""
from __future__ import annotations

import math

import numpy as np

from .dots import dot

RUNNING, CONVERGED, MAXIT, BREAKDOWN, NONFINITE = 0, 1, 2, 3, 4


def m_schedule(i: int, m_max: int, schedule: str = "paper") -> int:
    """P:105 verbatim; 'sliding' = min(i, m_max) (Notay's truncation, option)."""
    if schedule == "paper":
        return min(i, max(1, i % (m_max + 1)))
    if schedule == "sliding":
        return min(i, m_max)
    raise ValueError(schedule)


def _round32(x):
    """Store a vector in fp32 (round to nearest) and read it back as fp64 (exact)."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def fcg(apply_A, f, u0, m_max, tol, maxit, precond=None, schedule="paper", vec32=False, observe=None):
    """Algorithm 1 for one system.  apply_A(x) -> A x; precond(r) -> w (None = identity).
    observe(i, w_i, u_i), when given, is called at every iteration after w_i = B(r_i) (diagnostics:
    oracle/notay.py notay_curve); it does not change the iteration.

    vec32 (reading R21, SURVEY C.2 #28 "vectors and ring in fp32, dots accumulated in fp64"): the
    residual r, the preconditioned residual w and the stored directions p, s are kept in fp32; each
    is computed in fp64 from the stored values exactly as below and rounded once when stored; the
    iterate u, the inner products (correctly rounded, R6) and the scalars stay fp64.

    Returns dict(u, r, hist, iters, status)."""
    st = _round32 if vec32 else (lambda x: x)
    u = np.array(u0, dtype=np.float64, copy=True)
    r = st(np.asarray(f, dtype=np.float64) - apply_A(u))
    rho0 = math.sqrt(dot(r, r))
    hist = [1.0]
    if rho0 == 0.0:
        return dict(u=u, r=r, hist=np.array(hist), iters=0, status=CONVERGED)
    P, S, G = [], [], []          # stored p_k, s_k, (p_k, s_k); newest last
    for i in range(maxit):
        w = r.copy() if precond is None else st(np.asarray(precond(r), dtype=np.float64))
        if not np.all(np.isfinite(w)):
            return dict(u=u, r=r, hist=np.array(hist), iters=i, status=NONFINITE)
        if observe is not None:
            observe(i, w, u)
        mi = m_schedule(i, m_max, schedule)
        window = list(range(len(P) - mi, len(P)))
        betas = {kk: dot(w, S[kk]) / G[kk] for kk in window}
        p = w.copy()
        for kk in reversed(window):
            p = p - betas[kk] * P[kk]
        p = st(p)
        s = st(apply_A(p))
        gamma = dot(p, s)
        if not (gamma > 0.0 and math.isfinite(gamma)):
            return dict(u=u, r=r, hist=np.array(hist), iters=i, status=BREAKDOWN)
        alpha = dot(p, r) / gamma
        u = u + alpha * p
        r = st(r - alpha * s)
        hist.append(math.sqrt(dot(r, r)) / rho0)
        P.append(p); S.append(s); G.append(gamma)
        if len(P) > m_max:                      # windows never reach further back
            P.pop(0); S.pop(0); G.pop(0)
        if hist[-1] <= tol:
            return dict(u=u, r=r, hist=np.array(hist), iters=i + 1, status=CONVERGED)
    return dict(u=u, r=r, hist=np.array(hist), iters=maxit, status=MAXIT)


def cg(apply_A, f, u0, tol, maxit):
    """Textbook (Hestenes-Stiefel) conjugate gradients, unpreconditioned (§2.2)."""
    u = np.array(u0, dtype=np.float64, copy=True)
    r = np.asarray(f, dtype=np.float64) - apply_A(u)
    rr = dot(r, r)
    rho0 = math.sqrt(rr)
    hist = [1.0]
    if rho0 == 0.0:
        return dict(u=u, r=r, hist=np.array(hist), iters=0, status=CONVERGED)
    p = r.copy()
    for i in range(maxit):
        s = apply_A(p)
        ps = dot(p, s)
        if not ps > 0.0:
            return dict(u=u, r=r, hist=np.array(hist), iters=i, status=BREAKDOWN)
        alpha = rr / ps
        u = u + alpha * p
        r = r - alpha * s
        rr_new = dot(r, r)
        hist.append(math.sqrt(rr_new) / rho0)
        if hist[-1] <= tol:
            return dict(u=u, r=r, hist=np.array(hist), iters=i + 1, status=CONVERGED)
        p = r + (rr_new / rr) * p
        rr = rr_new
    return dict(u=u, r=r, hist=np.array(hist), iters=maxit, status=MAXIT)
