"""Pins for oracle/no.py: DFT conventions by brute-force sums and closed forms, NO properties,
the hand-set structured NO against its closed form, and a brute-force loop implementation
of one full forward on a tiny grid."""
import cmath
import math

import numpy as np
import pytest

import oracle as orc
import synthetic as sy

K = orc.K_MODES
KAPPA = np.arange(-(K // 2), K - K // 2)


def direct_analysis(v):
    n = v.shape[-1]
    out = np.zeros((K, K), dtype=complex)
    for a, k1 in enumerate(KAPPA):
        for b, k2 in enumerate(KAPPA):
            s = 0j
            for i in range(n):
                for j in range(n):
                    s += v[i, j] * cmath.exp(-2j * math.pi * (k1 * i + k2 * j) / n)
            out[a, b] = s
    return out


def direct_synthesis(g, n):
    z = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            s = 0j
            for a, k1 in enumerate(KAPPA):
                for b, k2 in enumerate(KAPPA):
                    s += g[a, b] * cmath.exp(2j * math.pi * (k1 * i + k2 * j) / n)
            z[i, j] = s.real / n ** 2
    return z


def test_analysis_matches_direct_sum():
    rng = np.random.default_rng(0)
    v = rng.standard_normal((21, 21))
    assert np.max(np.abs(orc.analysis(v) - direct_analysis(v))) < 1e-10


def test_synthesis_matches_direct_sum():
    rng = np.random.default_rng(1)
    g = rng.standard_normal((K, K)) + 1j * rng.standard_normal((K, K))
    assert np.max(np.abs(orc.synthesis(g, 20) - direct_synthesis(g, 20))) < 1e-12


@pytest.mark.parametrize("n,k1,k2", [(32, 3, 0), (64, -10, 9), (40, 5, -7)])
def test_single_harmonic(n, k1, k2):
    # a pure grid harmonic has analysis n^2 at its mode and 0 elsewhere in M.
    i = np.arange(n)[:, None]; j = np.arange(n)[None, :]
    v = np.exp(2j * np.pi * (k1 * i + k2 * j) / n)
    c = orc.analysis(v)
    expect = np.zeros((K, K), dtype=complex)
    expect[k1 + K // 2, k2 + K // 2] = n * n
    assert np.max(np.abs(c - expect)) < 1e-9 * n * n


def test_projection_identity_on_band_limited():
    # synthesis o analysis is the identity on real fields band-limited to
    # {-9..9}^2 (both members of every conjugate pair lie in M) and is idempotent.
    n = 48
    rng = np.random.default_rng(2)
    i = np.arange(n)[:, None]; j = np.arange(n)[None, :]
    f = np.zeros((n, n))
    for k1 in range(-9, 10):
        for k2 in range(-9, 10):
            a, b = rng.standard_normal(2)
            f += a * np.cos(2 * np.pi * (k1 * i + k2 * j) / n) + b * np.sin(2 * np.pi * (k1 * i + k2 * j) / n)
    proj = orc.synthesis(orc.analysis(f), n)
    assert np.max(np.abs(proj - f)) < 1e-11 * np.max(np.abs(f))
    p2 = orc.synthesis(orc.analysis(proj), n)
    assert np.max(np.abs(p2 - proj)) < 1e-11 * np.max(np.abs(f))


def test_unpaired_mode_halved():
    # kappa1 = -10 has no partner +10 in M (reading R7): Re(S(A cos)) keeps half of it.
    n = 48
    i = np.arange(n)[:, None] + 0 * np.arange(n)[None, :]
    f = np.cos(2 * np.pi * (-10) * i / n)
    proj = orc.synthesis(orc.analysis(f), n)
    assert np.max(np.abs(proj - 0.5 * f)) < 1e-12


def test_gelu_exact_erf():
    xs = np.linspace(-6, 6, 101)
    for x, y in zip(xs, orc.gelu(xs)):
        assert abs(y - 0.5 * x * (1 + math.erf(x / math.sqrt(2)))) <= 1e-15 * max(1, abs(x))


@pytest.mark.parametrize("w,count", [(32, 3281153), (48, 7382401), (85, 23149581)])
def test_param_count(w, count):
    assert orc.param_count(w) == count
    assert sy.no_blob_size(w) == count


def _params(w, seed):
    return orc.unpack_weights(sy.no_weights(w, seed), w)


def test_zero_params_and_zero_input():
    n, w = 24, 4
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 5)[0]
    r = sy.normal_field(n, 1, 5)[0]
    z = orc.unpack_weights(np.zeros(orc.param_count(w)), w)
    assert np.all(orc.no_forward(z, r, k) == 0.0)
    p = _params(w, 6)
    assert np.all(orc.no_forward(p, np.zeros((n, n)), k) == 0.0)


def test_homogeneity():
    n, w = 24, 4
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 5)[0]
    r = sy.normal_field(n, 1, 5)[0]
    p = _params(w, 7)
    base = orc.no_forward(p, r, k)
    for a in (0.5, 3.0, 1e-6):
        out = orc.no_forward(p, a * r, k)
        assert np.max(np.abs(out - a * base)) <= 1e-12 * a * np.max(np.abs(base))


def test_linear_mode_superposition():
    # with GELU -> identity, zero biases and no k channel, the map is linear.
    n, w = 24, 4
    p = _params(w, 8)
    p["E"][:, 1] = 0.0; p["bE"][:] = 0.0; p["bD"] = 0.0
    for l in range(4):
        p["b"][l][:] = 0.0
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 5)[0]
    r1, r2 = sy.normal_field(n, 2, 9)
    f = lambda x: orc.no_forward(p, x, k, use_gelu=False)
    lhs = f(2.0 * r1 - 3.0 * r2)
    rhs = 2.0 * f(r1) - 3.0 * f(r2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


@pytest.mark.parametrize("n,n_w", [(32, 32), (64, 32)])
def test_structured_no_closed_form(n, n_w):
    # the hand-set weights realise w = alpha r + S L A r exactly, with
    # L = 1/(4 pi^2 |kappa|^2 + 2 pi^2), alpha = h_w^2/4 — computed here with explicit DFT
    # matrices, independent of oracle.analysis/synthesis.
    w = 4
    p = orc.unpack_weights(sy.structured_no_weights(w, n_w), w)
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 3)[0]
    r = sy.normal_field(n, 1, 3)[0]
    out = orc.no_forward(p, r, k)
    idx = np.arange(n)
    Fm = np.exp(-2j * np.pi * np.outer(KAPPA, idx) / n)        # [K, n]
    c = Fm @ r @ Fm.T                                           # kappa1 <-> rows, kappa2 <-> cols
    L = 1.0 / (4 * np.pi ** 2 * (KAPPA[:, None] ** 2 + KAPPA[None, :] ** 2) + 2 * np.pi ** 2)
    z = (np.conj(Fm).T @ (L * c) @ np.conj(Fm)).real / n ** 2
    alpha = (1.0 / (n_w + 1)) ** 2 / 4
    expect = alpha * r + z
    assert np.max(np.abs(out - expect)) <= 1e-12 * np.max(np.abs(expect))


def test_forward_matches_bruteforce_loops():
    # One full forward on a tiny grid, evaluated with explicit loops and direct DFT sums.
    n, w = 20, 2
    p = _params(w, 11)
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 12)[0]
    r = sy.normal_field(n, 1, 12)[0]
    s = math.sqrt(sum(x * x for x in r.ravel()))
    x0 = [r / s, k]
    v = [sum(p["E"][c, q] * x0[q] for q in range(2)) + p["bE"][c] for c in range(w)]
    for l in range(4):
        ch = [direct_analysis(v[c]) for c in range(w)]
        new = []
        for o in range(w):
            g = sum(p["R"][l][c, o] * ch[c] for c in range(w))
            u = sum(p["W"][l][o, c] * v[c] for c in range(w)) + p["b"][l][o] + direct_synthesis(g, n)
            if l < 3:
                u = np.vectorize(lambda t: 0.5 * t * (1 + math.erf(t / math.sqrt(2))))(u)
            new.append(u)
        v = new
    expect = s * (sum(p["D"][c] * v[c] for c in range(w)) + p["bD"])
    out = orc.no_forward(p, r, k)
    assert np.max(np.abs(out - expect)) <= 1e-11 * np.max(np.abs(expect))


# ----------------------------------------------------------------------------- Chebyshev / DCT-II basis (R25, NEXT-4)
def test_cheb_analysis_is_scaled_scipy_dct2():
    # S^T f along one axis is half of scipy's unnormalised DCT-II (y_k = 2 sum_j x_j cos(pi k (2j+1) / 2n)),
    # the library routine the paper's Chebyshev SNO uses; analysis divides by h_k = n, n/2
    from scipy.fft import dctn
    n = 29
    v = np.random.default_rng(5).standard_normal((n, n))
    y = dctn(v, type=2)[:orc.K_MODES, :orc.K_MODES] / 4.0
    h = np.where(np.arange(orc.K_MODES) == 0, float(n), n / 2.0)
    assert np.allclose(orc.analysis_cheb(v), y / h[:, None] / h[None, :], rtol=1e-12, atol=1e-14)


def test_cheb_synthesis_then_analysis_is_identity():
    # discrete orthogonality of the cosines on the index grid: A S = identity on K x K coefficients
    n = 33
    g = np.random.default_rng(6).standard_normal((orc.K_MODES, orc.K_MODES))
    assert np.allclose(orc.analysis_cheb(orc.synthesis_cheb(g, n)), g, rtol=1e-12, atol=1e-12)


def test_cheb_brute_force_sums():
    n, K = 21, orc.K_MODES
    v = np.random.default_rng(7).standard_normal((n, n))
    c = np.zeros((K, K))
    for k1 in range(K):
        for k2 in range(K):
            acc = 0.0
            for i in range(n):
                for j in range(n):
                    acc += v[i, j] * np.cos(np.pi * k1 * (i + 0.5) / n) * np.cos(np.pi * k2 * (j + 0.5) / n)
            c[k1, k2] = acc / ((n if k1 == 0 else n / 2) * (n if k2 == 0 else n / 2))
    assert np.allclose(orc.analysis_cheb(v), c, rtol=1e-12, atol=1e-13)


def test_cheb_no_forward_linear_mode_superposition_and_constant_mode():
    # linear mode: B is homogeneous of degree 1 in r (scale) and the k = 0 mode of a constant field
    # is the constant itself (T_0 = 1): a constant input passes through a single-mode kernel exactly
    n, w = 24, 3
    k = sy.lognormal_k(n, 1, 0.1, 1.0, 8)[0]
    r = sy.normal_field(n, 1, 9)[0]
    p = orc.unpack_weights(sy.no_weights(w, 10), w)
    a = orc.no_forward(p, r, k, use_gelu=False, basis="chebyshev")
    b = orc.no_forward(p, 2.5 * r, k, use_gelu=False, basis="chebyshev")
    assert np.allclose(b, 2.5 * a, rtol=1e-12, atol=1e-12 * np.abs(a).max())
    const = np.full((n, n), 3.0)
    g = np.zeros((orc.K_MODES, orc.K_MODES)); g[0, 0] = 3.0
    assert np.allclose(orc.analysis_cheb(const), g, atol=1e-13)
