"""Pins for oracle/fcg.py: Algorithm 1's schedule, special cases that reduce to textbook
results, invariants, and the only number the paper prints that needs no trained weights
(Table 1, CG column)."""
import os

import numpy as np
import pytest

import oracle as orc
import synthetic as sy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1_cg.txt")


def test_m_schedule_spec_examples():
    # SPEC.md:203-205 and P:105.
    assert orc.m_schedule(0, 20) == 0
    assert orc.m_schedule(20, 20) == 20
    assert orc.m_schedule(21, 20) == 1
    assert [orc.m_schedule(i, 5) for i in range(14)] == [0, 1, 2, 3, 4, 5, 1, 1, 2, 3, 4, 5, 1, 1]
    for m in (1, 5, 10, 20):
        for i in range(101):
            assert orc.m_schedule(i, m) == min(i, max(1, i % (m + 1)))
            assert orc.m_schedule(i, m) <= m


def _dense(A):
    return lambda x: (A @ x.ravel()).reshape(x.shape)


def test_identity_matrix_one_iteration():
    # A = I converges in 1 iteration.
    f = np.array([1.0, -2.0, 3.0]); u0 = np.array([0.5, 0.5, 0.5])
    res = orc.fcg(_dense(np.eye(3)), f, u0, 5, 1e-12, 10)
    assert res["iters"] == 1 and res["status"] == orc.CONVERGED
    assert np.allclose(res["u"], f, rtol=0, atol=1e-15)


def test_diag_two_iterations():
    # A = diag(1,4), f = (1,1), u0 = 0 -> (1, 0.25) within 2 iterations.
    res = orc.fcg(_dense(np.diag([1.0, 4.0])), np.ones(2), np.zeros(2), 5, 1e-14, 10)
    assert res["iters"] <= 2
    assert np.allclose(res["u"], [1.0, 0.25], rtol=0, atol=1e-15)


def test_exact_inverse_preconditioner():
    # B = A^-1 -> 1 iteration.
    k = sy.lognormal_k(8, 1, 0.1, 1.0, 1)[0]
    A = orc.dense_A(k)
    Ainv = np.linalg.inv(A)
    f = sy.normal_field(8, 1, 1)[0]
    res = orc.fcg(lambda x: orc.apply_A(k, x), f, np.zeros_like(f), 5, 1e-12, 10,
                  precond=lambda r: (Ainv @ r.ravel()).reshape(r.shape))
    assert res["iters"] == 1 and res["hist"][1] < 1e-13


@pytest.mark.parametrize("m,schedule", [(5, "paper"), (20, "paper"), (400, "sliding")])
def test_identity_fcg_equals_textbook_cg(m, schedule):
    # BASELINE north_star / SPEC.md:195: FCG with B = I reproduces plain CG iterates
    # (k = 1, n = 15: agreement to ~1e-13 at every iteration).
    n = 15
    k = np.ones((n, n))
    f = sy.normal_field(n, 1, 4)[0]
    u0 = sy.rng(4, 0, 2).standard_normal((n, n))
    A = lambda x: orc.apply_A(k, x)
    a = orc.fcg(A, f, u0, m, 1e-10, 500, schedule=schedule)
    b = orc.cg(A, f, u0, 1e-10, 500)
    assert a["iters"] == b["iters"]
    ha, hb = a["hist"], b["hist"]
    assert np.max(np.abs(ha - hb) / hb) < 1e-9
    assert np.max(np.abs(a["u"] - b["u"])) < 1e-11 * np.max(np.abs(b["u"]))


@pytest.mark.parametrize("n,variance,seed", [(4, 1.0, 0), (4, 4.0, 1), (8, 1.0, 2), (8, 4.0, 3)])
def test_finite_termination_full_window(n, variance, seed):
    # BASELINE north_star: (F)CG converges in at most N steps on tiny grids; with the full
    # window (SLIDING, m >= N) FCG(I) is exact-arithmetic CG.
    N = n * n
    k = sy.lognormal_k(n, 1, 0.1, variance, seed)[0]
    f = sy.normal_field(n, 1, seed)[0]
    res = orc.fcg(lambda x: orc.apply_A(k, x), f, np.zeros_like(f), N, 1e-10, 5 * N, schedule="sliding")
    assert res["status"] == orc.CONVERGED and res["iters"] <= N


def _a_norm_errors(k, f, precond, m, iters):
    A = orc.dense_A(k)
    ustar = np.linalg.solve(A, f.ravel())
    errs = []
    def cb_precond(r):
        return precond(r)
    u = np.zeros_like(f)
    # run FCG one iteration budget at a time by recording u through repeated solves is
    # wasteful; instead re-run with increasing maxit (deterministic, so prefixes agree).
    for it in range(1, iters + 1):
        res = orc.fcg(lambda x: orc.apply_A(k, x), f, u, m, 0.0, it, precond=cb_precond)
        e = ustar - res["u"].ravel()
        errs.append(np.sqrt(e @ A @ e))
    return errs


def test_a_norm_monotone_random_no():
    # SPEC.md:217 / BASELINE north_star: each FCG step is an exact A-norm line search, so
    # ||u* - u_i||_A is non-increasing for any preconditioner (here the random-init NO).
    n, w = 20, 8
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 21)[0]
    f = sy.normal_field(n, 1, 21)[0]
    p = orc.unpack_weights(sy.no_weights(w, 22), w)
    errs = _a_norm_errors(k, f, lambda r: orc.no_forward(p, r, k), 5, 12)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(errs, errs[1:]))


def test_a_norm_monotone_linear_spd_preconditioner():
    n, w = 20, 4
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 23)[0]
    f = sy.normal_field(n, 1, 23)[0]
    p = orc.unpack_weights(sy.structured_no_weights(w, n), w)
    errs = _a_norm_errors(k, f, lambda r: orc.no_forward(p, r, k), 5, 12)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 0.5 * errs[0]


def test_scale_invariance():
    # FCG is invariant to the scale of B: B and c*B give the same residual history.
    n = 24
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 31)[0]
    f = sy.normal_field(n, 1, 31)[0]
    A = lambda x: orc.apply_A(k, x)
    a = orc.fcg(A, f, np.zeros_like(f), 5, 1e-8, 60)
    b = orc.fcg(A, f, np.zeros_like(f), 5, 1e-8, 60, precond=lambda r: 0.125 * r)
    assert np.array_equal(a["hist"], b["hist"])   # power-of-two scale: exact


def _golden():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        kind, grid, its = line.split()
        rows.append((kind, int(grid), int(its)))
    return rows


@pytest.mark.parametrize("kind,grid,printed", [r for r in _golden() if r[1] <= 64])
def test_table1_cg_column(kind, grid, printed):
    # PAPER.md:321-336 Table 1, CG column: iterations to 1e-6 with u0 ~ N(0,I) and
    # trig-polynomial data.  Median over 20 seeded instances within 10%.
    n = grid
    its = []
    for seed in range(20):
        k = np.ones((n, n)) if kind == "poisson" else sy.trig_poly(n, 1, seed, offset=10.0, stream=0)[0]
        f = sy.trig_poly(n, 1, seed)[0]
        u0 = sy.rng(seed, 0, sy.STREAM_U0).standard_normal((n, n))
        res = orc.cg(lambda x: orc.apply_A(k, x), f, u0, 1e-6, 2000)
        its.append(res["iters"])
    med = float(np.median(its))
    assert abs(med - printed) <= 0.1 * printed, (med, printed)
    # FCG(I) with the paper's m_max = 20 sits on top of CG.
    fcg_its = []
    for seed in range(5):
        k = np.ones((n, n)) if kind == "poisson" else sy.trig_poly(n, 1, seed, offset=10.0, stream=0)[0]
        f = sy.trig_poly(n, 1, seed)[0]
        u0 = sy.rng(seed, 0, sy.STREAM_U0).standard_normal((n, n))
        fcg_its.append(orc.fcg(lambda x: orc.apply_A(k, x), f, u0, 20, 1e-6, 2000)["iters"])
    assert abs(np.median(fcg_its) - printed) <= 0.12 * printed


@pytest.mark.slow
@pytest.mark.parametrize("kind,grid,printed", [r for r in _golden() if r[1] == 128])
def test_table1_cg_column_128(kind, grid, printed):
    n = grid
    its = []
    for seed in range(8):
        k = np.ones((n, n)) if kind == "poisson" else sy.trig_poly(n, 1, seed, offset=10.0, stream=0)[0]
        f = sy.trig_poly(n, 1, seed)[0]
        u0 = sy.rng(seed, 0, sy.STREAM_U0).standard_normal((n, n))
        its.append(orc.cg(lambda x: orc.apply_A(k, x), f, u0, 1e-6, 2000)["iters"])
    assert abs(float(np.median(its)) - printed) <= 0.1 * printed


def test_breakdown_and_nonfinite_status():
    n = 20
    k = np.ones((n, n))
    f = sy.normal_field(n, 1, 40)[0]
    A = lambda x: orc.apply_A(k, x)
    res = orc.fcg(A, f, np.zeros_like(f), 5, 1e-8, 10, precond=lambda r: np.full_like(r, np.nan))
    assert res["status"] == orc.NONFINITE and res["iters"] == 0
    res = orc.fcg(A, f, np.zeros_like(f), 5, 1e-8, 10, precond=lambda r: np.zeros_like(r))
    assert res["status"] == orc.BREAKDOWN and res["iters"] == 0
    res = orc.fcg(A, np.zeros_like(f), np.zeros_like(f), 5, 1e-8, 10)
    assert res["status"] == orc.CONVERGED and res["iters"] == 0


# ----------------------------------------------------------------------------- fp32 vector storage (R21)
def test_vec32_stored_vectors_are_fp32_and_history_consistent():
    # R21: r, w, p, s stored in fp32; the history is ||r||/||r0|| of the stored residuals.
    k = sy.lognormal_k(12, 1, 0.1, 1.0, 41)[0]
    f = np.random.default_rng(42).normal(size=(12, 12))
    A = lambda x: orc.apply_A(k, x)
    res = orc.fcg(A, f, np.zeros_like(f), 5, 1e-6, 400, vec32=True)
    r = res["r"]
    assert np.array_equal(r, r.astype(np.float32).astype(np.float64))
    r0 = f.astype(np.float32).astype(np.float64)   # u0 = 0: r0 = fl32(f)
    assert res["hist"][-1] == np.sqrt(orc.dot(r, r)) / np.sqrt(orc.dot(r0, r0))
    assert res["status"] == orc.CONVERGED


def test_vec32_poisson_prefix_matches_fp64_to_fp32_rounding():
    # k = 1, n = 8: the fp32-stored run is FCG up to fp32 rounding (first 15 relative residuals
    # within 1e-6 of the fp64 run) and converges to 1e-10 within +-3 iterations of it.
    n = 8
    k = np.ones((n, n))
    f = np.random.default_rng(3).normal(size=(n, n))
    A = lambda x: orc.apply_A(k, x)
    a = orc.fcg(A, f, np.zeros_like(f), 5, 1e-10, 200, vec32=True)
    b = orc.fcg(A, f, np.zeros_like(f), 5, 1e-10, 200)
    assert np.max(np.abs(a["hist"][:15] / b["hist"][:15] - 1.0)) < 1e-6
    assert a["status"] == orc.CONVERGED and abs(a["iters"] - b["iters"]) <= 3


def test_vec32_exact_inverse_one_step():
    # SPEC.md:194 with fp32 storage: B = A^{-1} (dense, n = 6) leaves a residual at fp32 rounding.
    n = 6
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 43)[0]
    N = n * n
    Ad = np.stack([orc.apply_A(k, e.reshape(n, n)).ravel() for e in np.eye(N)], axis=1)
    Ainv = np.linalg.inv(Ad)
    f = np.random.default_rng(44).normal(size=(n, n))
    res = orc.fcg(lambda x: orc.apply_A(k, x), f, np.zeros_like(f), 5, 1e-5, 5,
                  precond=lambda r: (Ainv @ r.ravel()).reshape(n, n), vec32=True)
    assert res["iters"] == 1 and res["hist"][1] < 1e-5
