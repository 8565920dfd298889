"""Oracle: inner products (a,b) = sum_t a_t b_t of one system's vectors.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading R6: every inner product in Algorithm 1 is the
correctly rounded value of the exact sum.  This makes the value independent of summation
order, so the GPU may reduce in any order and still agree bit for bit.
Written out: each product is split exactly into p + e (Dekker's TwoProduct, no fma
needed), and math.fsum (Shewchuk; correctly rounded) sums all p and e.
"""
from __future__ import annotations

import math

import numpy as np

_SPLIT = 134217729.0  # 2^27 + 1 (Dekker/Veltkamp split constant for binary64)


def _split(x):
    c = _SPLIT * x
    hi = c - (c - x)
    return hi, x - hi


def two_product(a, b):
    """Exact a*b = p + e for binary64 arrays (Dekker 1971); valid while |a|,|b| < 2^996
    and the error term does not underflow."""
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, e


def dot(a, b) -> float:
    """Correctly rounded (a, b) over all entries of a and b (R6)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if not (np.all(np.isfinite(a)) and np.all(np.isfinite(b))):
        return float(np.sum(a * b))  # propagate inf/nan like any summation would
    p, e = two_product(a, b)
    return math.fsum(np.concatenate([p, e]).tolist())


def norm2(a) -> float:
    """||a||_2 = sqrt((a, a)) with the correctly rounded inner product."""
    return math.sqrt(dot(a, a))
