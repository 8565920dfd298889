"""Oracle: 5-point FD discretisation of -div(k grad u) = f, u = 0 on the boundary.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:69-82 (§2.1, Eq. 1-2): -div(a grad u) = f on (0,1)^2, u|boundary = 0, an FDM gives a
sparse SPD system Au = f.  The paper does not fix the stencil; readings:
  R1  face coefficient = harmonic mean H(a,b) = (2*(a*b))/(a+b) of the two nodal values
      (BASELINE.json north_star "harmonic-mean face coefficients");
  R2  a face on the domain boundary takes the adjacent interior nodal value;
  R3  n interior nodes per dimension, h = 1/(n+1) (BASELINE configs[0]);
  R4  the h^-2 factor is included;
  R5  row index i <-> x2, column index j <-> x1; storage offset (b*n+i)*n+j.
Canonical operation order (no fused multiply-add anywhere; numpy never fuses):
  d = (kW+kE)+(kS+kN); t = d*u; t = t-kW*uW; t = t-kE*uE; t = t-kS*uS; t = t-kN*uN; y = t*(n+1)^2
with neighbours outside the grid equal to 0 (Dirichlet).
"""
from __future__ import annotations

import numpy as np


def h_of(n: int) -> float:
    """R3: mesh spacing of an n x n interior grid."""
    return 1.0 / (n + 1)


def harmonic(a, b):
    """R1: H(a,b) = (2*(a*b))/(a+b); bitwise symmetric in (a,b)."""
    return (2.0 * (a * b)) / (a + b)


def faces(k: np.ndarray):
    """Face coefficients (kW, kE, kS, kN) at every node of k[..., n, n] (R1, R2, R5)."""
    k = np.asarray(k, dtype=np.float64)
    kW = k.copy(); kE = k.copy(); kS = k.copy(); kN = k.copy()
    kE[..., :, :-1] = harmonic(k[..., :, :-1], k[..., :, 1:])
    kW[..., :, 1:] = harmonic(k[..., :, 1:], k[..., :, :-1])
    kN[..., :-1, :] = harmonic(k[..., :-1, :], k[..., 1:, :])
    kS[..., 1:, :] = harmonic(k[..., 1:, :], k[..., :-1, :])
    return kW, kE, kS, kN


def apply_A(k: np.ndarray, u: np.ndarray) -> np.ndarray:
    """y = A u for k, u of shape [..., n, n] (P:78-82 with R1-R5, canonical op order)."""
    k = np.asarray(k, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    n = k.shape[-1]
    kW, kE, kS, kN = faces(k)
    uW = np.zeros_like(u); uW[..., :, 1:] = u[..., :, :-1]
    uE = np.zeros_like(u); uE[..., :, :-1] = u[..., :, 1:]
    uS = np.zeros_like(u); uS[..., 1:, :] = u[..., :-1, :]
    uN = np.zeros_like(u); uN[..., :-1, :] = u[..., 1:, :]
    d = (kW + kE) + (kS + kN)
    t = d * u
    t = t - kW * uW
    t = t - kE * uE
    t = t - kS * uS
    t = t - kN * uN
    return t * float((n + 1) * (n + 1))


def dense_A(k: np.ndarray) -> np.ndarray:
    """Dense N x N matrix of one system (columns = A applied to unit vectors); tiny grids only."""
    n = k.shape[-1]
    N = n * n
    A = np.empty((N, N))
    e = np.zeros((n, n))
    for c in range(N):
        e.flat[c] = 1.0
        A[:, c] = apply_A(k, e).ravel()
        e.flat[c] = 0.0
    return A
