"""Pins for oracle/stencil.py against closed forms and SPEC.md examples (no GPU)."""
import numpy as np
import pytest

import oracle as orc
import synthetic as sy


def test_n3_centre_row_spec_s73():
    # a = 1, n = 3 (h = 1/4): centre row diagonal 64, four off-diagonals -16.
    A = orc.dense_A(np.ones((3, 3)))
    row = A[4].reshape(3, 3)
    assert row[1, 1] == 64.0
    assert row[0, 1] == row[2, 1] == row[1, 0] == row[1, 2] == -16.0
    assert row[0, 0] == row[0, 2] == row[2, 0] == row[2, 2] == 0.0


def test_n3_lambda_min_spec_s74():
    # lambda_min = (1/h^2) 2 (2 - sqrt 2) = 32 (2 - sqrt 2) = 18.7452...
    lam = np.linalg.eigvalsh(orc.dense_A(np.ones((3, 3))))
    assert abs(lam[0] - 32 * (2 - np.sqrt(2))) < 1e-12


@pytest.mark.parametrize("n", [4, 8])
def test_k1_closed_form_spectrum(n):
    # k = 1: eigenvalues 4(n+1)^2 [sin^2(p pi/(2(n+1))) + sin^2(q pi/(2(n+1)))], p,q = 1..n.
    lam = np.linalg.eigvalsh(orc.dense_A(np.ones((n, n))))
    p = np.arange(1, n + 1)
    s2 = np.sin(p * np.pi / (2 * (n + 1))) ** 2
    exact = np.sort((4 * (n + 1) ** 2 * (s2[:, None] + s2[None, :])).ravel())
    assert np.max(np.abs(lam - exact) / exact) < 1e-12


@pytest.mark.parametrize("n,p,q", [(64, 1, 1), (64, 5, 17), (257, 3, 200)])
def test_k1_eigenvector_pointwise(n, p, q):
    # Closed-form eigenvector sin(p pi (i+1)/(n+1)) sin(q pi (j+1)/(n+1)) at any n.
    x = np.arange(1, n + 1) / (n + 1)
    v = np.sin(q * np.pi * x)[:, None] * np.sin(p * np.pi * x)[None, :]
    lam = 4 * (n + 1) ** 2 * (np.sin(p * np.pi / (2 * (n + 1))) ** 2 + np.sin(q * np.pi / (2 * (n + 1))) ** 2)
    Av = orc.apply_A(np.ones((n, n)), v)
    scale = np.max(np.abs(lam * v))
    assert np.max(np.abs(Av - lam * v)) < 1e-9 * scale * n


def test_row_sums_spec_s122():
    # k = 1, x = 1: row sum = (number of missing neighbours) * (n+1)^2.
    n = 5
    y = orc.apply_A(np.ones((n, n)), np.ones((n, n)))
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    missing = (i == 0).astype(int) + (i == n - 1) + (j == 0) + (j == n - 1)
    assert np.array_equal(y, missing * float((n + 1) ** 2))


def test_harmonic_jump():
    # k = 1 next to k = 100: face = 2*100/101 (harmonic mean), not 50.5 (arithmetic).
    n = 4
    k = np.ones((n, n)); k[:, 2:] = 100.0
    A = orc.dense_A(k)
    # node (1,1) -> east neighbour (1,2)
    a = A[1 * n + 1, 1 * n + 2]
    assert a == -(n + 1) ** 2 * (200.0 / 101.0)


def test_linear_in_k_spec_s75():
    rng = np.random.default_rng(0)
    n = 6
    u = rng.standard_normal((n, n))
    for c in (0.3, 7.0, 1e3):
        y1 = orc.apply_A(np.ones((n, n)), u)
        yc = orc.apply_A(np.full((n, n), c), u)
        assert np.allclose(yc, c * y1, rtol=4e-16 * 8, atol=0)


def test_symmetric_positive_definite_lognormal_8x8():
    # BASELINE north_star: x^T A y = y^T A x, min eigenvalue > 0 by dense eigensolve on 8x8.
    k = sy.lognormal_k(8, 1, 0.1, 1.0, seed=7)[0]
    A = orc.dense_A(k)
    assert np.array_equal(A, A.T)                 # bitwise: H(a,b) is symmetric
    assert np.linalg.eigvalsh(A)[0] > 0
    k4 = sy.lognormal_k(8, 1, 0.05, 4.0, seed=8)[0]
    A4 = orc.dense_A(k4)
    assert np.array_equal(A4, A4.T) and np.linalg.eigvalsh(A4)[0] > 0
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal((2, 8, 8))
    lhs = np.sum(x * orc.apply_A(k, y)); rhs = np.sum(y * orc.apply_A(k, x))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_batched_equals_per_system():
    k = sy.lognormal_k(20, 3, 0.1, 1.0, seed=3)
    u = sy.normal_field(20, 3, seed=3)
    y = orc.apply_A(k, u)
    for b in range(3):
        assert np.array_equal(y[b], orc.apply_A(k[b], u[b]))
