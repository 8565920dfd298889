"""Pins for oracle/dots.py: the correctly rounded inner product, checked by exact rational
arithmetic (brute force, independent of the split/fsum route)."""
from fractions import Fraction

import numpy as np

import oracle as orc


def exact_dot(a, b) -> float:
    s = sum((Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b)), Fraction(0))
    return float(s)   # float(Fraction) rounds correctly (round-half-even)


def test_dot_correctly_rounded_random():
    rng = np.random.default_rng(0)
    for trial in range(40):
        n = int(rng.integers(1, 300))
        a = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 5)
        b = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 5)
        assert orc.dot(a, b) == exact_dot(a, b)


def test_dot_correctly_rounded_cancellation():
    # Ill-conditioned sums (massive cancellation), where naive summation is wrong.
    rng = np.random.default_rng(1)
    for trial in range(20):
        a = rng.standard_normal(200)
        b = rng.standard_normal(200)
        # make (a,b) nearly zero: b <- b - (a,b)/(a,a) a, evaluated naively
        b = b - (np.sum(a * b) / np.sum(a * a)) * a
        a = np.concatenate([a, [1e16, -1e16]])
        b = np.concatenate([b, [1.0, 1.0]])
        assert orc.dot(a, b) == exact_dot(a, b)


def test_integer_valued_exact():
    rng = np.random.default_rng(2)
    a = rng.integers(-2 ** 20, 2 ** 20, 5000).astype(float)
    b = rng.integers(-2 ** 20, 2 ** 20, 5000).astype(float)
    assert orc.dot(a, b) == float(int(np.dot(a.astype(object), b.astype(object))))


def test_two_product_exact():
    rng = np.random.default_rng(3)
    a = rng.standard_normal(1000) * 1e3
    b = rng.standard_normal(1000) * 1e-3
    p, e = orc.two_product(a, b)
    for x, y, pp, ee in zip(a, b, p, e):
        assert Fraction(float(x)) * Fraction(float(y)) == Fraction(float(pp)) + Fraction(float(ee))


def test_norm():
    assert orc.norm2(np.array([3.0, 4.0])) == 5.0
