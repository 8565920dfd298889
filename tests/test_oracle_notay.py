"""Pins for oracle/notay.py (Eq. final_loss, Theorem 1's eps): closed forms of the ratio."""
import numpy as np

import oracle as orc
import synthetic as sy


def _setup(n=10, seed=51):
    k = sy.lognormal_k(n, 1, 0.1, 1.0, seed)[0]
    A = lambda x: orc.apply_A(k, x)
    Ad = orc.dense_A(k)
    r = np.random.default_rng(seed).normal(size=(n, n))
    e = np.linalg.solve(Ad, r.ravel()).reshape(n, n)     # A^{-1} r by a dense library solve
    return k, A, Ad, r, e


def test_exact_inverse_gives_zero_and_zero_gives_one():
    _, A, _, _, e = _setup()
    assert orc.notay_ratio(A, e, e) == 0.0                 # B = A^{-1}
    assert abs(orc.notay_ratio(A, np.zeros_like(e), e) - 1.0) < 1e-15   # B = 0
    assert abs(orc.notay_ratio(A, 2.0 * e, e) - 1.0) < 1e-14             # B = 2 A^{-1}


def test_scaled_inverse_closed_form():
    # B = c A^{-1}: eps = |c - 1| for every r
    _, A, _, _, e = _setup()
    for c in (0.25, 0.9, 1.5):
        assert abs(orc.notay_ratio(A, c * e, e) - abs(c - 1.0)) < 1e-13


def test_a_norm_matches_dense_quadratic_form():
    _, A, Ad, r, e = _setup()
    v = r.ravel()
    assert abs(orc.a_norm(A, r) - np.sqrt(v @ (Ad @ v))) < 1e-12 * np.sqrt(v @ (Ad @ v))


def test_identity_preconditioner_value():
    # B = I: eps^2 = (r - e, A (r - e)) / (e, A e) = ((r, A r) - 2 (r, r) + (r, e)) / (r, e)
    _, A, Ad, r, e = _setup()
    v, x = r.ravel(), e.ravel()
    ref = np.sqrt((v @ (Ad @ v) - 2 * (v @ v) + v @ x) / (v @ x))
    assert abs(orc.notay_ratio(A, r, e) - ref) < 1e-10 * ref


def test_scaled_ratio_is_scale_free_and_zero_for_scaled_inverse():
    _, A, _, r, e = _setup()
    assert orc.notay_ratio_scaled(A, 3.0 * e, e) < 1e-14      # B = 3 A^{-1}: optimal c removes the scale
    a, b = orc.notay_ratio_scaled(A, r, e), orc.notay_ratio_scaled(A, 1e-3 * r, e)
    assert abs(a - b) < 1e-12 and 0.0 < a < 1.0 and a <= orc.notay_ratio(A, r, e)


# ----------------------------------------------------------------------------- notay_curve (Theorem 1 along FCG)
def _curve_setup(n=8, seed=61):
    k = sy.lognormal_k(n, 1, 0.1, 1.0, seed)[0]
    A = lambda x: orc.apply_A(k, x)
    Ad = orc.dense_A(k)
    f = np.random.default_rng(seed).normal(size=(n, n))
    u_star = np.linalg.solve(Ad, f.ravel()).reshape(n, n)   # exact solution by a dense library solve
    return k, A, Ad, f, u_star


def test_curve_exact_inverse_preconditioner():
    # B = A^{-1} (dense solve): eps_0 = 0 up to rounding, one iteration, ||e_0||_A = ||u*||_A (u_0 = 0)
    _, A, Ad, f, u_star = _curve_setup()
    P = lambda r: np.linalg.solve(Ad, r.ravel()).reshape(r.shape)
    res, eps, err = orc.notay_curve(A, f, np.zeros_like(f), u_star, 5, 1e-10, 10, precond=P)
    assert res["iters"] == 1 and len(eps) == 1
    assert eps[0] < 1e-12 and abs(err[0] - np.sqrt(u_star.ravel() @ (Ad @ u_star.ravel()))) < 1e-12 * err[0]


def test_curve_matches_separate_solves():
    # eps_i and ||e_i||_A at iteration i equal the ratio evaluated on the state of a separate run stopped
    # after i iterations (u_i, r_i = f - A u_i recurrence residual from that run, w_i = r_i for B = I)
    _, A, _, f, u_star = _curve_setup()
    res, eps, err = orc.notay_curve(A, f, np.zeros_like(f), u_star, 5, 1e-30, 12)
    assert len(eps) == 12 == len(err)
    for i in (0, 1, 5, 11):
        r_i = orc.fcg(A, f, np.zeros_like(f), 5, 1e-30, i)
        e_i = u_star - r_i["u"]
        assert eps[i] == orc.notay_ratio(A, r_i["r"], e_i)
        assert err[i] == orc.a_norm(A, e_i)


def test_curve_energy_error_monotone_for_identity():
    # every FCG step is an exact A-norm line search along p_i, so ||u* - u_i||_A never increases (u*
    # exact); eps_i < 1 is not implied for B = I, but here CG-like convergence drives err_a down
    _, A, _, f, u_star = _curve_setup()
    res, eps, err = orc.notay_curve(A, f, np.zeros_like(f), u_star, 5, 1e-12, 200)
    assert np.all(np.diff(err) <= 1e-12 * err[0])
    assert err[-1] < 1e-6 * err[0] and res["status"] == orc.CONVERGED
