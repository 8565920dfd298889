"""Pins for oracle/classical.py: Jacobi(k) (Eq. 15) and symmetric Gauss-Seidel(k)
against their matrix definitions (dense D, L, U from the assembled A; scipy triangular solves), the
operators' algebra (linearity, symmetry), and the paper's Table 1 Poisson columns."""
import os

import numpy as np
import pytest
from scipy.linalg import solve_triangular

import oracle as orc
import synthetic as sy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1_classical.txt")


def _perm(n, order):
    idx = np.arange(n * n)
    if order == "lex":
        return idx
    i, j = np.divmod(idx, n)
    return np.concatenate([idx[(i + j) % 2 == 0], idx[(i + j) % 2 == 1]])   # red first (R22)


def _dense_sgs(A, z, sweeps, perm):
    Ap = A[np.ix_(perm, perm)]
    L, U = np.tril(Ap), np.triu(Ap)
    zp = z.ravel()[perm]
    x = np.zeros_like(zp)
    for _ in range(sweeps):
        x = x + solve_triangular(L, zp - Ap @ x, lower=True)
        x = x + solve_triangular(U, zp - Ap @ x, lower=False)
    out = np.empty_like(x)
    out[perm] = x
    return out.reshape(z.shape)


def _case(n=6, seed=3, var=1.0):
    k = sy.lognormal_k(n, 1, 0.2, var, seed)[0]
    z = sy.normal_field(n, 1, seed + 1)[0]
    return k, z, orc.dense_A(k)


def test_diagonal_is_the_diagonal_of_A():
    k, _, A = _case()
    assert np.allclose(orc.diagonal(k).ravel(), np.diag(A), rtol=1e-15, atol=0)


@pytest.mark.parametrize("sweeps", [1, 2, 4])
def test_jacobi_matches_matrix_definition(sweeps):
    # Eq. 15 from x0 = 0, b = z  <=>  x = sum_{j<k} (I - D^-1 A)^j D^-1 z
    k, z, A = _case()
    D = np.diag(A)
    x = np.zeros(z.size)
    for _ in range(sweeps):
        x = x + (z.ravel() - A @ x) / D
    got = orc.jacobi(k, z, sweeps)
    assert np.allclose(got.ravel(), x, rtol=1e-12, atol=1e-12 * np.abs(x).max())
    if sweeps == 1:   # one sweep from zero is D^-1 z exactly
        assert np.array_equal(got, z / orc.diagonal(k))


@pytest.mark.parametrize("order", ["lex", "rb"])
@pytest.mark.parametrize("sweeps", [1, 3])
def test_sgs_matches_triangular_solves(order, sweeps):
    k, z, A = _case(var=4.0)
    ref = _dense_sgs(A, z, sweeps, _perm(k.shape[0], order))
    got = orc.sgs(k, z, sweeps, order=order)
    assert np.allclose(got, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


@pytest.mark.parametrize("kind", ["jacobi", "sgs_lex", "sgs_rb"])
def test_linear_and_symmetric(kind):
    # Jacobi(k) and SGS(k) from x0 = 0 are fixed symmetric linear operators (SPEC invariants)
    k, z, A = _case(n=5)
    r2 = sy.normal_field(5, 1, 77)[0]
    P = {"jacobi": lambda v: orc.jacobi(k, v, 3), "sgs_lex": lambda v: orc.sgs(k, v, 2, "lex"),
         "sgs_rb": lambda v: orc.sgs(k, v, 2, "rb")}[kind]
    lin = P(2.0 * z - 3.0 * r2)
    assert np.allclose(lin, 2.0 * P(z) - 3.0 * P(r2), rtol=1e-12, atol=1e-12 * np.abs(lin).max())
    a, b = np.sum(P(z) * r2), np.sum(z * P(r2))
    assert abs(a - b) <= 1e-10 * (abs(a) + abs(b))


def test_red_black_half_sweeps_touch_one_colour():
    k, z, _ = _case(n=7)
    x1 = orc.classical._colour_half_sweep(k, z, np.zeros_like(z), orc.diagonal(k), 0)
    i, j = np.indices(z.shape)
    assert np.all(x1[(i + j) % 2 == 1] == 0.0) and np.all(x1[(i + j) % 2 == 0] != 0.0)


def _golden():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        kind, grid, its = line.split()
        rows.append((kind, int(grid), int(its)))
    return rows


@pytest.mark.parametrize("kind,grid,printed", _golden())
def test_table1_classical_columns(kind, grid, printed):
    # PAPER.md:321-336 Table 1, Poisson rows: FCG (m_max = 20) preconditioned by Jacobi(4),
    # GS(1), GS(4), iterations to 1e-6 with u0 ~ N(0, I), trig-polynomial f.
    # The paper's GS ordering is not stated; the lexicographic sweep (R22) is pinned here within 15%.
    n = grid
    its = []
    for seed in range(6):
        k = np.ones((n, n))
        f = sy.trig_poly(n, 1, seed)[0]
        u0 = sy.rng(seed, 0, sy.STREAM_U0).standard_normal((n, n))
        P = {"jacobi4": lambda r: orc.jacobi(k, r, 4), "gs1": lambda r: orc.sgs(k, r, 1, "lex"),
             "gs4": lambda r: orc.sgs(k, r, 4, "lex")}[kind]
        its.append(orc.fcg(lambda x: orc.apply_A(k, x), f, u0, 20, 1e-6, 500, precond=P)["iters"])
    med = float(np.median(its))
    assert abs(med - printed) <= 0.15 * printed, (med, printed, its)
