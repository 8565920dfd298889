"""Oracle: classical stationary preconditioners of the paper's comparison (§3.3.1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 15 (Jacobi):   x^{n+1} = x^n + D(A)^{-1} (b - A x^n)
Symmetric Gauss-Seidel:
                   x^{n+1/2} = x^n + L(A)^{-1} (b - A x^n)
                   x^{n+1}   = x^{n+1/2} + U(A)^{-1} (b - A x^{n+1/2})
with D, L, U the diagonal and the lower / upper triangular parts of A (diagonal included), applied k
times from x^0 = 0 with b = z to approximate A^{-1} z.

Readings (R22-R24):
  R22 node order: L and U follow an ordering of the nodes; 'lex' = row-major (i, j) order, the
      natural one (the paper's GS presumably); 'rb' = red-black order (colour (i + j) mod 2, red = 0
      first, row-major within a colour), the one a parallel sweep realises.  With the 5-point stencil
      nodes of one colour are not coupled, so an L^{-1} (U^{-1}) solve in 'rb' order is a red (black)
      half-sweep followed by a black (red) one.
  R23 one update at node e: x_e <- x_e + (z_e - (A x)_e) / d_e with (A x)_e in the canonical stencil
      order (oracle/stencil.py) on the current x and d_e = ((kW + kE) + (kS + kN)) * (n + 1)^2; a
      forward (backward) GS sweep applies it node by node in the order (reverse order), which is the
      triangular solve L^{-1} (U^{-1}) of the printed iteration written out.
  R24 the preconditioner's output is x^k (x^0 = 0).
"""
from __future__ import annotations

import numpy as np

from .stencil import apply_A, faces


def diagonal(k: np.ndarray) -> np.ndarray:
    """D(A) of every node: ((kW + kE) + (kS + kN)) (n+1)^2 (the diagonal of the stencil, R23)."""
    kW, kE, kS, kN = faces(k)
    n = k.shape[-1]
    return ((kW + kE) + (kS + kN)) * float((n + 1) * (n + 1))


def _row_of_A(fc, x, i, j, scale):
    """(A x) at node (i, j) only, in the canonical order of oracle/stencil.py (R23); fc = faces(k)."""
    kW, kE, kS, kN = (f[i, j] for f in fc)
    n = x.shape[-1]
    uW = x[i, j - 1] if j > 0 else 0.0
    uE = x[i, j + 1] if j < n - 1 else 0.0
    uS = x[i - 1, j] if i > 0 else 0.0
    uN = x[i + 1, j] if i < n - 1 else 0.0
    t = ((kW + kE) + (kS + kN)) * x[i, j]
    t = t - kW * uW
    t = t - kE * uE
    t = t - kS * uS
    t = t - kN * uN
    return t * scale


def jacobi(k: np.ndarray, z: np.ndarray, sweeps: int) -> np.ndarray:
    """Jacobi(sweeps) of Eq. 15 from x^0 = 0 with b = z."""
    d = diagonal(k)
    x = np.zeros_like(np.asarray(z, dtype=np.float64))
    for _ in range(sweeps):
        x = x + (z - apply_A(k, x)) / d
    return x


def _colour_half_sweep(k, z, x, d, colour):
    """Update every node of one colour (all of them depend only on the other colour): a block
    Jacobi step on that colour, identical to updating its nodes one by one (R22)."""
    n = k.shape[-1]
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    mask = ((ii + jj) % 2) == colour
    upd = x + (z - apply_A(k, x)) / d
    return np.where(mask, upd, x)


def sgs(k: np.ndarray, z: np.ndarray, sweeps: int, order: str = "rb") -> np.ndarray:
    """Symmetric Gauss-Seidel(sweeps) from x^0 = 0 with b = z; order 'rb' (red-black) or
    'lex' (row-major; a pure-Python node loop, for small grids)."""
    z = np.asarray(z, dtype=np.float64)
    d = diagonal(k)
    x = np.zeros_like(z)
    n = k.shape[-1]
    for _ in range(sweeps):
        if order == "rb":
            x = _colour_half_sweep(k, z, x, d, 0)    # L^{-1}: red then black
            x = _colour_half_sweep(k, z, x, d, 1)
            x = _colour_half_sweep(k, z, x, d, 1)    # U^{-1}: black then red
            x = _colour_half_sweep(k, z, x, d, 0)
        elif order == "lex":
            fc, scale = faces(k), float((n + 1) * (n + 1))
            for i in range(n):                        # forward sweep, row-major
                for j in range(n):
                    x[i, j] = x[i, j] + (z[i, j] - _row_of_A(fc, x, i, j, scale)) / d[i, j]
            for i in reversed(range(n)):              # backward sweep
                for j in reversed(range(n)):
                    x[i, j] = x[i, j] + (z[i, j] - _row_of_A(fc, x, i, j, scale)) / d[i, j]
        else:
            raise ValueError(order)
    return x
