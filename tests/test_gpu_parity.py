"""GPU parity: the CUDA path through the C-ABI against the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  apply_A, reductions         fp64, <= 1e-12 relative (bitwise here: same op order, exact dots)
  NO forward, fp32            <= 1e-4 relative L2 per system
  NO forward, fp64 mode       <= 1e-12 relative L2 per system
  FCG residual histories      <= 1e-8 relative per iteration (identity: bitwise)
  iteration counts            equal within +-1 (identity: exact)
"""
import math

import numpy as np
import pytest
import torch

import oracle as orc
import synthetic as sy

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ----------------------------------------------------------------------------- apply_A
@pytest.mark.parametrize("n,B,kind", [(2, 1, "lognormal"), (3, 2, "const"), (20, 3, "lognormal"),
                                      (33, 2, "lognormal"), (45, 5, "rectangles"), (64, 4, "lognormal"),
                                      (100, 2, "lognormal4")])
def test_apply_A_bitwise(lib, n, B, kind):
    if kind == "const":
        k = np.full((B, n, n), 3.5)
    elif kind == "rectangles":
        k = sy.rectangles_k(n, B, seed=5)
    elif kind == "lognormal4":
        k = sy.lognormal_k(n, B, 0.05, 4.0, seed=6)
    else:
        k = sy.lognormal_k(n, B, 0.1, 1.0, seed=7)
    x = sy.normal_field(n, B, seed=8)
    p = lib.Problem(dev(k))
    y = host(p.apply_A(dev(x)))
    ref = orc.apply_A(k, x)
    assert np.array_equal(y, ref), np.max(np.abs(y - ref))


@pytest.mark.parametrize("n,B", [(17, 3), (257, 2), (300, 2)])
def test_apply_A_bitwise_ragged_tiles(lib, n, B):
    # 2-D stencil tiles (16 rows x min(n, 256) columns): ragged last tile row (n = 17), ragged
    # last tile column (n = 257: one column; n = 300: 44 columns), halos across tile borders.
    k = sy.lognormal_k(n, B, 0.05, 4.0, seed=9)
    x = sy.normal_field(n, B, seed=10)
    y = host(lib.Problem(dev(k)).apply_A(dev(x)))
    assert np.array_equal(y, orc.apply_A(k, x))


def test_apply_A_bitwise_wide_range_k(lib):
    # k outside [2^-400, 2^400]: the faces take the guarded IEEE division path (assemble clears
    # the problem's fast-division flag); inside it, the branch-free path.  Both bitwise.
    rng = np.random.default_rng(11)
    n, B = 150, 2
    x = sy.normal_field(n, B, seed=12)
    for lo, hi in ((-150.0, 150.0), (-100.0, 100.0)):
        k = 10.0 ** rng.uniform(lo, hi, size=(B, n, n))
        y = host(lib.Problem(dev(k)).apply_A(dev(x)))
        assert np.array_equal(y, orc.apply_A(k, x))


@pytest.mark.parametrize("cfg_id", [3, 4, 5])
def test_apply_A_full_configs(lib, cfg_id):
    cfg = sy.CONFIGS[cfg_id]
    k = sy.make_k(cfg)
    x = sy.make_f(cfg)
    y = host(lib.Problem(dev(k)).apply_A(dev(x)))
    ref = orc.apply_A(k, x)
    assert np.max(np.abs(y - ref) / (np.abs(ref) + 1e-300)) <= 1e-12
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("n", [1024, 2048])
def test_apply_A_sweep_sizes_closed_form(lib, n):
    # k = 1: the closed-form eigenvector is reproduced pointwise at the sweep sizes (BJ:11).
    p, q = 3, 7
    x = np.arange(1, n + 1) / (n + 1)
    v = np.sin(q * np.pi * x)[:, None] * np.sin(p * np.pi * x)[None, :]
    lam = 4 * (n + 1) ** 2 * (np.sin(p * np.pi / (2 * (n + 1))) ** 2 + np.sin(q * np.pi / (2 * (n + 1))) ** 2)
    prob = lib.Problem(dev(np.ones((1, n, n))))
    y = host(prob.apply_A(dev(v[None])))[0]
    scale = np.abs(lam * v).max()
    assert np.max(np.abs(y - lam * v)) < 1e-6 * scale
    # and equals the oracle bit for bit on a sampled band of rows
    ref = orc.apply_A(np.ones((n, n)), v)
    assert np.array_equal(y[:64], ref[:64]) and np.array_equal(y[-64:], ref[-64:])


def test_assemble_rejects_bad_k(lib):
    k = np.ones((2, 8, 8)); k[1, 3, 4] = 0.0
    with pytest.raises(lib.FcgnoError) as e:
        lib.Problem(dev(k))
    assert e.value.code == 2
    k[1, 3, 4] = np.nan
    with pytest.raises(lib.FcgnoError):
        lib.Problem(dev(k))


# ----------------------------------------------------------------------------- reductions
@pytest.mark.parametrize("n,B", [(5, 3), (32, 1), (64, 8), (129, 2), (512, 2)])
def test_dot_correctly_rounded(lib, n, B):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((B, n, n)) * 10.0 ** rng.integers(-3, 3, (B, 1, 1))
    y = rng.standard_normal((B, n, n))
    p = lib.Problem(dev(np.ones((B, n, n))))
    got = host(p.dot(dev(x), dev(y)))
    for b in range(B):
        assert got[b] == orc.dot(x[b], y[b])
    # ill-conditioned: y made nearly orthogonal to x
    y2 = y - (np.sum(x * y, axis=(1, 2)) / np.sum(x * x, axis=(1, 2)))[:, None, None] * x
    got2 = host(p.dot(dev(x), dev(y2)))
    for b in range(B):
        ref = orc.dot(x[b], y2[b])
        assert abs(got2[b] - ref) <= 1e-12 * float(np.sum(np.abs(x[b] * y2[b])))


def test_dot_integer_exact(lib):
    rng = np.random.default_rng(3)
    x = rng.integers(-2 ** 20, 2 ** 20, (2, 64, 64)).astype(float)
    y = rng.integers(-2 ** 20, 2 ** 20, (2, 64, 64)).astype(float)
    got = host(lib.Problem(dev(np.ones((2, 64, 64)))).dot(dev(x), dev(y)))
    for b in range(2):
        assert got[b] == float(int(np.dot(x[b].ravel().astype(object), y[b].ravel().astype(object))))


# ----------------------------------------------------------------------------- NO forward
def _no_case(n, B, w, wseed, seed):
    k = sy.lognormal_k(n, B, 0.1, 1.0, seed)
    r = sy.normal_field(n, B, seed + 1)
    blob = sy.no_weights(w, wseed)
    return k, r, blob


@pytest.mark.parametrize("n,B,w", [(20, 2, 4), (32, 1, 32), (37, 2, 8), (64, 3, 48)])
def test_no_fp64_matches_oracle(lib, n, B, w):
    k, r, blob = _no_case(n, B, w, 11, 12)
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP64)
    got = host(no.apply(prob, dev(r)))
    params = orc.unpack_weights(blob, w)
    for b in range(B):
        ref = orc.no_forward(params, r[b], k[b])
        assert rel_l2(got[b], ref) <= 1e-12


# tensor-core shapes (n = 64 or 128 k) include widths with every remainder modulo 4 (padded spectra rows) and
# the largest width
@pytest.mark.parametrize("n,B,w", [(20, 2, 4), (32, 2, 32), (45, 3, 48), (64, 8, 48), (128, 2, 85), (64, 3, 5),
                                   (128, 1, 23), (64, 2, 126), (64, 2, 128)])
def test_no_fp32_matches_oracle(lib, n, B, w):
    k, r, blob = _no_case(n, B, w, 21, 22)
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP32)
    got = host(no.apply(prob, dev(r)))
    params = orc.unpack_weights(blob, w)
    for b in sorted({0, B - 1}):
        ref = orc.no_forward(params, r[b], k[b])
        assert rel_l2(got[b], ref) <= 1e-4


@pytest.mark.parametrize("cfg_id", [2, 3, 4, 5])
def test_no_fp32_full_config_sampled(lib, cfg_id):
    cfg = sy.CONFIGS[cfg_id]
    k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(cfg["width"], blob, precision=lib.FP32)
    got = host(no.apply(prob, dev(f)))
    params = orc.unpack_weights(blob, cfg["width"])
    for b in (0, cfg["batch"] - 1):
        assert rel_l2(got[b], orc.no_forward(params, f[b], k[b])) <= 1e-4


def test_no_properties(lib):
    n, B, w = 32, 2, 16
    k, r, blob = _no_case(n, B, w, 31, 32)
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP64)
    base = host(no.apply(prob, dev(r)))
    scaled = host(no.apply(prob, dev(3.0 * r)))
    assert np.max(np.abs(scaled - 3.0 * base)) <= 1e-12 * np.max(np.abs(base)) * 3
    zero = host(no.apply(prob, dev(np.zeros_like(r))))
    assert np.all(zero == 0.0)
    z = lib.NeuralOperator(w, np.zeros(sy.no_blob_size(w)), precision=lib.FP32)
    assert np.all(host(z.apply(prob, dev(r))) == 0.0)


def test_no_structured_closed_form(lib):
    n, w = 64, 4
    k = sy.lognormal_k(n, 2, 0.1, 1.0, 41)
    r = sy.normal_field(n, 2, 42)
    blob = sy.structured_no_weights(w, n)
    prob = lib.Problem(dev(k))
    got = host(lib.NeuralOperator(w, blob, precision=lib.FP64).apply(prob, dev(r)))
    params = orc.unpack_weights(blob, w)
    for b in range(2):
        assert rel_l2(got[b], orc.no_forward(params, r[b], k[b])) <= 1e-12


def test_no_linear_mode(lib):
    n, w = 24, 4
    k, r, blob = _no_case(n, 1, w, 51, 52)
    prob = lib.Problem(dev(k))
    got = host(lib.NeuralOperator(w, blob, precision=lib.FP64, use_gelu=False).apply(prob, dev(r)))
    ref = orc.no_forward(orc.unpack_weights(blob, w), r[0], k[0], use_gelu=False)
    assert rel_l2(got[0], ref) <= 1e-12


def test_no_rejects_small_grid(lib):
    prob = lib.Problem(dev(np.ones((1, 16, 16))))
    no = lib.NeuralOperator(4, sy.no_weights(4, 1))
    with pytest.raises(lib.FcgnoError) as e:
        no.apply(prob, dev(np.ones((1, 16, 16))))
    assert e.value.code == 5


# ----------------------------------------------------------------------------- FCG, identity
def _oracle_fcg(k, f, m, tol, maxit, precond=None, schedule="paper"):
    return orc.fcg(lambda x: orc.apply_A(k, x), f, np.zeros_like(f), m, tol, maxit, precond=precond,
                   schedule=schedule)


def _check_identity(lib, k, f, m, tol, maxit, systems, schedule=0, vec32=False):
    prob = lib.Problem(dev(k))
    res = lib.fcg_solve(prob, dev(f), m=m, tol=tol, maxit=maxit, schedule=schedule, vec_fp32=vec32)
    iters, status, hist, u = host(res.iters), host(res.status), host(res.history), host(res.u)
    for b in systems:
        ref = orc.fcg(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), m, tol, maxit,
                      schedule="sliding" if schedule else "paper", vec32=vec32)
        it = ref["iters"]
        assert iters[b] == it and status[b] == ref["status"]
        assert np.array_equal(hist[b, :it + 1], ref["hist"]), "identity histories must agree bit for bit"
        assert np.array_equal(u[b], ref["u"])
    return iters, status


def test_identity_config1_bitwise(lib):
    cfg = sy.CONFIGS[1]
    _check_identity(lib, sy.make_k(cfg), sy.make_f(cfg), cfg["m"], cfg["tol"], cfg["maxit"], [0])


def test_identity_config2_sampled(lib):
    cfg = dict(sy.CONFIGS[2])
    k, f = sy.make_k(cfg), sy.make_f(cfg)
    iters, status = _check_identity(lib, k, f, cfg["m"], cfg["tol"], 5000, [0, cfg["batch"] - 1])
    assert np.all(status == lib.CONVERGED)


@pytest.mark.parametrize("n,B,m", [(20, 3, 5), (45, 2, 10), (7, 2, 1)])
def test_identity_ragged(lib, n, B, m):
    k = sy.lognormal_k(n, B, 0.1, 1.0, 61)
    f = sy.normal_field(n, B, 62)
    _check_identity(lib, k, f, m, 1e-8, 3000, range(B))


@pytest.mark.parametrize("n,B,m,maxit,systems", [(300, 2, 10, 40, [0, 1]), (512, 8, 10, 24, [0, 7])])
def test_identity_prefix_wide_tiles(lib, n, B, m, maxit, systems):
    # multi-column stencil tiles (n = 300) and the wide element-wise kernels (B*N >= 2^21 at
    # n = 512, B = 8): residual histories and iterates bit-identical to the oracle over maxit steps
    k = sy.lognormal_k(n, B, 0.1, 1.0, 63)
    f = sy.normal_field(n, B, 64)
    _check_identity(lib, k, f, m, 1e-14, maxit, systems)


# ----------------------------------------------------------------------------- fp32 vectors (R21)
@pytest.mark.parametrize("cfg_id,systems,maxit", [(1, [0], None), (2, [0, 63], 5000)])
def test_identity_vec32_configs_bitwise(lib, cfg_id, systems, maxit):
    # opts.vec_fp32: r, w, p, s stored in fp32, every vector operation in fp64 rounded once on
    # store; histories, iterates and counts bit-identical to the oracle's fp32-storage variant.
    cfg = sy.CONFIGS[cfg_id]
    k, f = sy.make_k(cfg), sy.make_f(cfg)
    _check_identity(lib, k, f, cfg["m"], cfg["tol"], maxit or cfg["maxit"], systems, vec32=True)


@pytest.mark.parametrize("n,B,m,maxit,systems", [(45, 2, 10, 3000, [0, 1]), (512, 8, 10, 24, [0, 7])])
def test_identity_vec32_ragged_and_wide(lib, n, B, m, maxit, systems):
    # odd n (single-cell tile fills) and the wide element-wise kernels with fp32 column pairs
    k = sy.lognormal_k(n, B, 0.1, 1.0, 65)
    f = sy.normal_field(n, B, 66)
    _check_identity(lib, k, f, m, 1e-6 if n < 100 else 1e-14, maxit, systems, vec32=True)


@pytest.mark.parametrize("n", [4, 8])
def test_identity_sliding_full_window_finite_termination(lib, n):
    k = sy.lognormal_k(n, 2, 0.1, 4.0, 71)
    f = sy.normal_field(n, 2, 72)
    iters, status = _check_identity(lib, k, f, min(n * n, 64), 1e-10, 5 * n * n, range(2), schedule=1)
    assert np.all(iters <= n * n) and np.all(status == lib.CONVERGED)


def test_fcg_edge_cases(lib):
    n, B = 20, 3
    k = sy.lognormal_k(n, B, 0.1, 1.0, 81)
    f = sy.normal_field(n, B, 82)
    f[1] = 0.0                                   # r0 = 0: converged at 0 iterations
    prob = lib.Problem(dev(k))
    res = lib.fcg_solve(prob, dev(f), m=5, tol=1e-8, maxit=2000)
    assert host(res.status)[1] == lib.CONVERGED and host(res.iters)[1] == 0
    assert np.all(host(res.u)[1] == 0.0)
    res0 = lib.fcg_solve(prob, dev(f), m=5, tol=1e-8, maxit=0)
    assert list(host(res0.status)) == [lib.MAXIT, lib.CONVERGED, lib.MAXIT]
    resm = lib.fcg_solve(prob, dev(f), m=5, tol=1e-8, maxit=7)
    assert list(host(resm.iters)) == [7, 0, 7]
    # zero NO weights: w = 0 -> p = 0 -> (p, s) = 0 -> breakdown at i = 0
    z = lib.NeuralOperator(4, np.zeros(sy.no_blob_size(4)))
    resz = lib.fcg_solve(prob, dev(f), m=5, tol=1e-8, maxit=10, no=z)
    assert host(resz.status)[0] == lib.BREAKDOWN and host(resz.iters)[0] == 0
    # overflowing fp32 NO: non-finite preconditioner output
    big = lib.NeuralOperator(4, sy.no_weights(4, 3) * 1e30)
    resb = lib.fcg_solve(prob, dev(f), m=5, tol=1e-8, maxit=10, no=big)
    assert host(resb.status)[0] == lib.NONFINITE and host(resb.iters)[0] == 0


# ----------------------------------------------------------------------------- FCG with the NO
def _prefix_window_ok(h_gpu, h_ref, upto, rtol=1e-8):
    a, b = h_gpu[:upto + 1], h_ref[:upto + 1]
    return np.max(np.abs(a - b) / b) <= rtol


def _self_sensitivity_window(k, f, m, tol, maxit, precond, thresh=1e-9):
    """Prefix window of G3(a): the first iteration at which the oracle's own
    history moves by more than `thresh` when every preconditioner output is perturbed by one
    ulp.  Beyond it, no implementation can be held to 1e-8 (FCG amplifies rounding chaotically)."""
    base = _oracle_fcg(k, f, m, tol, maxit, precond=precond)
    pert = _oracle_fcg(k, f, m, tol, maxit, precond=lambda r: np.nextafter(precond(r), np.inf))
    n = min(len(base["hist"]), len(pert["hist"]))
    d = np.abs(pert["hist"][:n] - base["hist"][:n]) / base["hist"][:n]
    bad = np.nonzero(d > thresh)[0]
    return base, (int(bad[0]) - 1 if bad.size else n - 1)


def test_fcg_no_fp64_config1_prefix(lib):
    # fp64 NO: histories agree to <= 1e-8 over the prefix window where the oracle's own
    # 1-ulp sensitivity stays below 1e-9.
    cfg = sy.CONFIGS[1]
    k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
    w = cfg["width"]
    params = orc.unpack_weights(blob, w)
    maxit = 40
    ref, window = _self_sensitivity_window(k[0], f[0], cfg["m"], cfg["tol"], maxit,
                                           lambda r: orc.no_forward(params, r, k[0]))
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP64)
    res = lib.fcg_solve(prob, dev(f), m=cfg["m"], tol=cfg["tol"], maxit=maxit, no=no)
    h = host(res.history)[0]
    assert host(res.status)[0] == lib.MAXIT == ref["status"]
    assert window >= 8
    assert _prefix_window_ok(h, ref["hist"], window)
    assert np.max(np.abs(h - ref["hist"]) / ref["hist"]) <= 1e-3


def test_fcg_structured_no_fp64_counts(lib):
    # Supplementary convergent workload: iteration counts within +-1.
    n, B, w = 32, 2, 4
    k = sy.lognormal_k(n, B, 0.1, 1.0, 91)
    f = sy.normal_field(n, B, 92)
    blob = sy.structured_no_weights(w, n)
    params = orc.unpack_weights(blob, w)
    prob = lib.Problem(dev(k))
    res = lib.fcg_solve(prob, dev(f), m=5, tol=1e-8, maxit=500,
                        no=lib.NeuralOperator(w, blob, precision=lib.FP64))
    for b in range(B):
        ref, window = _self_sensitivity_window(k[b], f[b], 5, 1e-8, 500,
                                               lambda r: orc.no_forward(params, r, k[b]))
        assert abs(int(host(res.iters)[b]) - ref["iters"]) <= 1
        assert host(res.status)[b] == lib.CONVERGED
        assert window >= 8
        assert _prefix_window_ok(host(res.history)[b], ref["hist"], window)


# ----------------------------------------------------------------------------- FCG with the fp32 NO: hybrid runs
# Algorithm 1 as the oracle writes it, with B(r) = the library's own fp32 NO
# (fcgno_apply_NO on the full batch, the system's r in its slot and r = 0 elsewhere, so the launch
# geometry is the solve's own), against fcg_solve with that NO.  The NO kernels are deterministic
# and the FCG step is bitwise equal to the oracle's (identity tests above), so histories, iterates,
# counts and statuses must agree bit for bit: a wrong window slot, beta, ring index or fused-dot
# prefetch in the solve's NO-output kernel (k_no_out_blob) fails here at the first iteration it
# touches.  The fp32 NO itself is held to the oracle's fp64 NO by the <= 1e-4 forward tests.
def _gpu_precond(lib, prob, no, B, n, b, vec32=False):
    def P(r):
        full = np.zeros((B, n, n))
        full[b] = r
        return host(no.apply(prob, dev(full)))[b]
    return P


def _hybrid_check(lib, cfg, systems, maxit, vec32=False, blob=None, tol=None, expect_status=None):
    k, f = sy.make_k(cfg), sy.make_f(cfg)
    blob = sy.make_weights(cfg) if blob is None else blob
    tol = cfg["tol"] if tol is None else tol
    n, B, w, m = cfg["n"], cfg["batch"], cfg["width"], cfg["m"]
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP32)
    res = lib.fcg_solve(prob, dev(f), m=m, tol=tol, maxit=maxit, no=no, vec_fp32=vec32)
    iters, status, hist, u = host(res.iters), host(res.status), host(res.history), host(res.u)
    for b in systems:
        ref = orc.fcg(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), m, tol, maxit,
                      precond=_gpu_precond(lib, prob, no, B, n, b), vec32=vec32)
        it = ref["iters"]
        assert iters[b] == it and status[b] == ref["status"], (b, iters[b], it, status[b], ref["status"])
        assert np.array_equal(hist[b, :it + 1], ref["hist"]), \
            (b, int(np.argmax(hist[b, :it + 1] != ref["hist"])))
        assert np.array_equal(u[b], ref["u"])
        if expect_status is not None:
            assert status[b] == expect_status
    return prob, no, iters, status


@pytest.mark.parametrize("vec32", [False, True])
def test_fcg_no_fp32_hybrid_bitwise_config2_full(lib, vec32):
    # The headline path at config 2: the tensor-core NO feeding FCG(5), all 2000 iterations (R19).
    cfg = sy.CONFIGS[2]
    prob, no, iters, status = _hybrid_check(lib, cfg, [0, cfg["batch"] - 1], cfg["maxit"], vec32=vec32,
                                            expect_status=lib.MAXIT)
    assert lib.no_uses_tensor_cores(prob, no)
    assert np.all(iters == cfg["maxit"])


@pytest.mark.parametrize("cfg_id,maxit", [(3, 200), (4, 120), (5, 40)])
def test_fcg_no_fp32_hybrid_bitwise_large_configs(lib, cfg_id, maxit):
    # Prefixes of the large workloads: config 3 (tensor cores, n = 128, w = 85, m = 10), configs 4
    # and 5 (n = 256 / 512), systems {0, B-1}.
    cfg = sy.CONFIGS[cfg_id]
    _hybrid_check(lib, cfg, [0, cfg["batch"] - 1], maxit, expect_status=lib.MAXIT)


def test_fcg_no_fp32_hybrid_bitwise_config3_vec32(lib):
    cfg = sy.CONFIGS[3]
    _hybrid_check(lib, cfg, [0, cfg["batch"] - 1], 100, vec32=True, expect_status=lib.MAXIT)


def test_fcg_structured_no_fp32_tensor_core_counts(lib):
    # The convergent structured SNO at the config-2 geometry on the tensor-core
    # path: converging runs, iteration counts, histories and iterates bit for bit.
    cfg = dict(sy.CONFIGS[2], batch=4, width=4)
    blob = sy.structured_no_weights(4, cfg["n"])
    prob, no, iters, status = _hybrid_check(lib, cfg, [0, 3], 1000, blob=blob, tol=1e-8,
                                            expect_status=lib.CONVERGED)
    assert lib.no_uses_tensor_cores(prob, no)



def test_solve_host_matches_device(lib):
    cfg = sy.CONFIGS[1]
    k, f = sy.make_k(cfg), sy.make_f(cfg)
    hs = lib.HostSolver(cfg["n"], cfg["batch"], cfg["m"], cfg["tol"], cfg["maxit"])
    u = np.zeros_like(f)
    iters = np.zeros(cfg["batch"], np.int32); status = np.zeros(cfg["batch"], np.int32)
    hs.solve(np.ascontiguousarray(k), np.ascontiguousarray(f), u, iters, status)
    res = lib.fcg_solve(lib.Problem(dev(k)), dev(f), m=cfg["m"], tol=cfg["tol"], maxit=cfg["maxit"])
    assert np.array_equal(u, host(res.u)) and np.array_equal(iters, host(res.iters))


def test_repeat_solves_deterministic(lib):
    cfg = sy.CONFIGS[2]
    k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(cfg["width"], blob)
    s = lib.Solver(prob, cfg["m"], cfg["tol"], 12, no=no)
    u1 = torch.zeros_like(dev(f)); s.solve(dev(f), u1); h1 = s.history.clone()
    u2 = torch.zeros_like(dev(f)); s.solve(dev(f), u2)
    assert torch.equal(u1, u2) and torch.equal(h1, s.history)


def test_fcg_no_fp64_config3_prefix(lib):
    # fp64 NO mode at config 3 (n = 128, w = 85, contrast ~4e5): histories within 1e-8 over the
    # oracle's own 1-ulp self-sensitivity window.
    cfg = dict(sy.CONFIGS[3], batch=2)
    k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
    w = cfg["width"]
    params = orc.unpack_weights(blob, w)
    maxit = 8
    ref, window = _self_sensitivity_window(k[0], f[0], cfg["m"], cfg["tol"], maxit,
                                           lambda r: orc.no_forward(params, r, k[0]))
    prob = lib.Problem(dev(k))
    res = lib.fcg_solve(prob, dev(f), m=cfg["m"], tol=cfg["tol"], maxit=maxit,
                        no=lib.NeuralOperator(w, blob, precision=lib.FP64))
    assert window >= 2
    assert _prefix_window_ok(host(res.history)[0], ref["hist"], window)


def test_tc_and_ffma_paths_agree(lib):
    # The tensor-core (3xBF16) and FFMA (fp32) NO paths compute the same map to ~1e-5.
    import subprocess, sys, os, json
    code = ("import json,sys,numpy as np,torch; sys.path.insert(0,'.'); import synthetic as sy;"
            "from paper_2402_05598_b200 import fcgno as F;"
            "k=sy.lognormal_k(64,3,0.1,1.0,5); r=sy.normal_field(64,3,6); blob=sy.no_weights(48,7);"
            "p=F.Problem(torch.from_numpy(k).cuda()); w=F.NeuralOperator(48,blob).apply(p,torch.from_numpy(r).cuda());"
            "np.save(sys.argv[1], w.cpu().numpy())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tcflag in ("1", "0"):
        path = f"/tmp/fcgno_tc{tcflag}.npy"
        env = dict(os.environ, FCGNO_TC=tcflag)
        subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, check=True)
        outs.append(np.load(path))
    assert rel_l2(outs[0], outs[1]) <= 5e-5


def _solve_in_subprocess(env_extra, tag, maxit=12, batch=64):
    """Short fp32 FCG-NO solve at the config-2 geometry in a fresh process with extra env flags
    (the flags are read once per process); returns (u, history)."""
    import os
    import subprocess
    import sys
    code = ("import sys,numpy as np,torch; sys.path.insert(0,'.'); import synthetic as sy;"
            "from paper_2402_05598_b200 import fcgno as F;"
            f"cfg=dict(sy.CONFIGS[2], batch={batch}); k=sy.make_k(cfg); f=sy.make_f(cfg); blob=sy.make_weights(cfg);"
            "p=F.Problem(torch.from_numpy(k).cuda());"
            f"res=F.fcg_solve(p, torch.from_numpy(f).cuda(), m=cfg['m'], tol=cfg['tol'], maxit={maxit},"
            " no=F.NeuralOperator(cfg['width'], blob));"
            "np.savez(sys.argv[1], u=res.u.cpu().numpy(), h=res.history.cpu().numpy())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = f"/tmp/fcgno_optin_{tag}.npz"
    subprocess.run([sys.executable, "-c", code, path], cwd=root, env=dict(os.environ, **env_extra), check=True)
    z = np.load(path)
    return z["u"], z["h"]


def test_opt_in_paths_match_default(lib):
    # Opt-in variant computing the same per-system arithmetic as the default path:
    #   FCGNO_LANES=2  -- the batch as two parallel graph branches (systems never interact): bitwise.
    u0, h0 = _solve_in_subprocess({}, "default")
    u1, h1 = _solve_in_subprocess({"FCGNO_LANES": "2"}, "lanes")
    assert np.isfinite(u0).all() and h0.shape == h1.shape
    assert np.array_equal(u0, u1) and np.array_equal(h0, h1, equal_nan=True)


def _identity_in_subprocess(env_extra, tag, n, B, m, maxit, schedule=0, nan_first=False):
    """fp64 identity FCG solve of a small lognormal system in a fresh process (env flags are read once per
    process); returns (u, history, iters, status)."""
    import os
    import subprocess
    import sys
    code = ("import sys,numpy as np,torch; sys.path.insert(0,'.'); import synthetic as sy;"
            "from paper_2402_05598_b200 import fcgno as F;"
            f"k=sy.lognormal_k({n},{B},0.1,1.0,31); f=sy.normal_field({n},{B},32); u0=sy.normal_field({n},{B},33);"
            "f[-1]=0.0; u0[-1]=0.0;"   # the last system has r0 = 0
            f"f[0,0,0]=float('nan') if {int(nan_first)} else f[0,0,0];"   # optionally a non-finite system (R14)
            "p=F.Problem(torch.from_numpy(k).cuda());"
            f"res=F.fcg_solve(p, torch.from_numpy(f).cuda(), torch.from_numpy(u0).cuda(), m={m}, tol=1e-9, maxit={maxit},"
            f" schedule={schedule});"
            "np.savez(sys.argv[1], u=res.u.cpu().numpy(), h=res.history.cpu().numpy(), it=res.iters.cpu().numpy(),"
            " st=res.status.cpu().numpy())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = f"/tmp/fcgno_small_{tag}.npz"
    subprocess.run([sys.executable, "-c", code, path], cwd=root, env=dict(os.environ, **env_extra), check=True)
    z = np.load(path)
    return z["u"], z["h"], z["it"], z["st"]


@pytest.mark.parametrize("n,B,m,maxit,schedule", [(32, 3, 5, 500, 0), (32, 2, 10, 60, 1), (19, 4, 7, 25, 0), (8, 2, 64, 200, 1),
                                                    (12, 400, 4, 80, 0)])   # the last: more systems than CTA slots
def test_persistent_small_solve_matches_launch_per_step_path(lib, n, B, m, maxit, schedule):
    """The single-kernel solve of small identity systems (fcg_small.cu) against the general
    path (FCGNO_PERSISTENT=0) on the same inputs: iterates, histories, counts and statuses bitwise, with
    converging, maxit-capped and r0 = 0 systems in the batch."""
    a = _identity_in_subprocess({}, "on", n, B, m, maxit, schedule)
    b = _identity_in_subprocess({"FCGNO_PERSISTENT": "0"}, "off", n, B, m, maxit, schedule)
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), (a[2], b[2], a[3], b[3])
    assert a[2][-1] == 0 and a[3][-1] == lib.CONVERGED
    for s in range(B):
        it = int(a[2][s])
        assert np.array_equal(a[1][s, :it + 1], b[1][s, :it + 1]), s
        assert np.array_equal(a[0][s], b[0][s]), s


def test_persistent_small_solve_nonfinite_system(lib):
    """A system whose right-hand side holds a NaN is reported NONFINITE at iteration 0 by both paths
    (R14), its iterate untouched, and does not disturb the other systems of the batch."""
    a = _identity_in_subprocess({}, "on_nan", 16, 3, 5, 300, 0, nan_first=True)
    b = _identity_in_subprocess({"FCGNO_PERSISTENT": "0"}, "off_nan", 16, 3, 5, 300, 0, nan_first=True)
    assert a[3][0] == lib.NONFINITE == b[3][0] and a[2][0] == 0 == b[2][0]
    assert a[3][1] == lib.CONVERGED == b[3][1] and a[2][1] == b[2][1]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1][1, :a[2][1] + 1], b[1][1, :b[2][1] + 1])


# ----------------------------------------------------------------------------- Notay ratio (NEXT-2)
@pytest.mark.parametrize("kind", ["identity", "no64", "no32"])
def test_notay_ratio_matches_oracle(lib, kind):
    # eps = ||c B(r) - A^{-1} r||_A / ||A^{-1} r||_A (Eq. final_loss) through fcgno_notay_ratio vs the
    # oracle's direct definition, e = A^{-1} r from a dense library solve.  Given the same B(r) (the
    # library's own NO output handed to the oracle), both sides do the same operations in the same
    # order with correctly rounded dots: bit for bit.  Against the oracle's own fp64 NO: 1e-12 (fp64
    # NO), 1e-4 (fp32 NO, the forward tolerance).
    n, B, w = 32, 2, 8
    k = sy.lognormal_k(n, B, 0.1, 1.0, 95)
    r = sy.normal_field(n, B, 96)
    e = np.stack([np.linalg.solve(orc.dense_A(k[b]), r[b].ravel()).reshape(n, n) for b in range(B)])
    blob = sy.structured_no_weights(w, n) if kind != "identity" else None
    no = None
    if kind != "identity":
        no = lib.NeuralOperator(w, blob, precision=lib.FP64 if kind == "no64" else lib.FP32)
    prob = lib.Problem(dev(k))
    eps = host(lib.notay_ratio(prob, dev(r), dev(e), no))
    eps_s = host(lib.notay_ratio(prob, dev(r), dev(e), no, optimal_scale=True))
    w_gpu = host(no.apply(prob, dev(r))) if no is not None else r
    params = orc.unpack_weights(blob, w) if blob is not None else None
    for b in range(B):
        A = lambda x: orc.apply_A(k[b], x)
        assert eps[b] == orc.notay_ratio(A, w_gpu[b], e[b]), (eps[b], orc.notay_ratio(A, w_gpu[b], e[b]))
        assert eps_s[b] == orc.notay_ratio_scaled(A, w_gpu[b], e[b])
        if params is not None:
            wb = orc.no_forward(params, r[b], k[b])
            tol = {"no64": 1e-12, "no32": 1e-4}[kind]
            assert abs(eps[b] - orc.notay_ratio(A, wb, e[b])) <= tol * eps[b]
            assert abs(eps_s[b] - orc.notay_ratio_scaled(A, wb, e[b])) <= tol * max(eps_s[b], 1e-3)


@pytest.mark.parametrize("kind", ["identity", "no32_tc", "identity_vec32"])
def test_fcg_solve_diag_curves_bitwise(lib, kind):
    # Theorem 1 along the solve (fcgno_fcg_solve_diag): eps_i = ||w_i - e_i||_A / ||e_i||_A and
    # ||e_i||_A, e_i = u* - u_i, at every iteration, against the oracle's notay_curve (Algorithm 1 with
    # the same B: identity, or the library's own fp32 tensor-core NO); u* from a dense solve.
    if kind.startswith("identity"):
        cfg = dict(sy.CONFIGS[1])
        n, B = cfg["n"], 1
        maxit, no, blob = 60, None, None
    else:
        cfg = dict(sy.CONFIGS[2], batch=4)
        n, B = cfg["n"], 4
        maxit = 30
        blob = sy.make_weights(cfg)
        no = lib.NeuralOperator(cfg["width"], blob, precision=lib.FP32)
    vec32 = kind.endswith("vec32")
    k, f = sy.make_k(cfg), sy.make_f(cfg)
    ustar = np.stack([np.linalg.solve(orc.dense_A(k[b]), f[b].ravel()).reshape(n, n) for b in range(B)])
    prob = lib.Problem(dev(k))
    res, eps, err = lib.fcg_solve_diag(prob, dev(f), dev(ustar), m=cfg["m"], tol=1e-30, maxit=maxit, no=no,
                                       vec_fp32=vec32)
    eps, err = host(eps), host(err)
    for b in sorted({0, B - 1}):
        P = None if no is None else _gpu_precond(lib, prob, no, B, n, b)
        ref, reps, rerr = orc.notay_curve(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), ustar[b],
                                          cfg["m"], 1e-30, maxit, precond=P, vec32=vec32)
        it = ref["iters"]
        assert int(host(res.iters)[b]) == it == maxit
        assert np.array_equal(eps[b, :it], reps) and np.array_equal(err[b, :it], rerr)
        assert np.array_equal(host(res.history)[b, :it + 1], ref["hist"])


# ----------------------------------------------------------------------------- device-side loop, graph cache
def test_device_loop_edge_cases(lib):
    # the solve's loop is a CUDA-graph WHILE node replaying 16-iteration bodies: maxit not a
    # multiple of the body, every system converged at r0 = 0, maxit = 1, check_every = 1, and a
    # run that stops mid-body; iterates equal the oracle's bit for bit (identity preconditioner)
    n, B = 24, 3
    k = sy.lognormal_k(n, B, 0.1, 1.0, 97)
    f = sy.normal_field(n, B, 98)
    prob = lib.Problem(dev(k))
    for maxit, ce in ((17, 16), (1, 16), (33, 1), (40, 7)):
        res = lib.fcg_solve(prob, dev(f), m=5, tol=1e-30, maxit=maxit, check_every=ce)
        assert list(host(res.iters)) == [maxit] * B and np.all(host(res.status) == lib.MAXIT)
        for b in (0, B - 1):
            ref = _oracle_fcg(k[b], f[b], 5, 1e-30, maxit)
            assert np.array_equal(host(res.u)[b], ref["u"]) and np.array_equal(host(res.history)[b], ref["hist"])
    zero = lib.fcg_solve(prob, dev(np.zeros_like(f)), m=5, tol=1e-8, maxit=50)
    assert np.all(host(zero.iters) == 0) and np.all(host(zero.status) == lib.CONVERGED)
    assert np.all(host(zero.u) == 0.0)
    # converging mid-body: counts and iterates bitwise
    res = lib.fcg_solve(prob, dev(f), m=5, tol=1e-6, maxit=3000)
    for b in range(B):
        ref = _oracle_fcg(k[b], f[b], 5, 1e-6, 3000)
        assert host(res.iters)[b] == ref["iters"] and np.array_equal(host(res.u)[b], ref["u"])


def test_graph_cache_reuse_with_other_buffers(lib):
    # instantiated loop graphs are reused only for identical captured arguments: alternating
    # right-hand sides / iterate buffers and a second problem must each give their own answer
    n, B = 20, 2
    k1 = sy.lognormal_k(n, B, 0.1, 1.0, 101)
    k2 = sy.rectangles_k(n, B, seed=102)
    fa, fb = sy.normal_field(n, B, 103), sy.normal_field(n, B, 104)
    p1, p2 = lib.Problem(dev(k1)), lib.Problem(dev(k2))
    s1 = lib.Solver(p1, 5, 1e-8, 3000)
    s2 = lib.Solver(p2, 5, 1e-8, 3000)
    dfa, dfb = dev(fa), dev(fb)
    for _ in range(2):
        for s, k, f, df in ((s1, k1, fa, dfa), (s1, k1, fb, dfb), (s2, k2, fa, dfa)):
            u = torch.zeros_like(df)
            s.solve(df, u)
            for b in range(B):
                ref = _oracle_fcg(k[b], f[b], 5, 1e-8, 3000)
                assert host(s.iters)[b] == ref["iters"] and np.array_equal(host(u)[b], ref["u"])


# ----------------------------------------------------------------------------- classical preconditioners (NEXT-3)
@pytest.mark.parametrize("kind,sweeps", [("jacobi", 1), ("jacobi", 4), ("sgs", 1), ("sgs", 3)])
@pytest.mark.parametrize("n,B", [(17, 2), (64, 3), (300, 1)])
def test_stationary_apply_bitwise(lib, kind, sweeps, n, B):
    # Jacobi(k) (Eq. 15) and red-black SGS(k) (R22-R23) through fcgno_apply_stationary,
    # bit for bit against the oracle's sweeps (same update, same stencil order, IEEE division)
    k = sy.lognormal_k(n, B, 0.1, 4.0, 131)
    r = sy.normal_field(n, B, 132)
    prob = lib.Problem(dev(k))
    got = host(lib.apply_stationary(prob, dev(r), lib.JACOBI if kind == "jacobi" else lib.SGS_RB, sweeps))
    for b in range(B):
        ref = orc.jacobi(k[b], r[b], sweeps) if kind == "jacobi" else orc.sgs(k[b], r[b], sweeps, "rb")
        assert np.array_equal(got[b], ref), float(np.max(np.abs(got[b] - ref)))


@pytest.mark.parametrize("kind,sweeps,vec32", [("jacobi", 4, False), ("sgs", 1, False), ("sgs", 4, False),
                                               ("jacobi", 4, True)])
def test_fcg_stationary_bitwise(lib, kind, sweeps, vec32):
    # FCG(m) preconditioned by Jacobi(k) / red-black SGS(k): histories, iterates, counts bit for bit
    cfg = sy.CONFIGS[2]
    k, f = sy.make_k(cfg), sy.make_f(cfg)
    prob = lib.Problem(dev(k))
    kd = lib.JACOBI if kind == "jacobi" else lib.SGS_RB
    res = lib.fcg_solve_stationary(prob, dev(f), kind=kd, sweeps=sweeps, m=cfg["m"], tol=cfg["tol"], maxit=3000,
                                   vec_fp32=vec32)
    iters, status, hist, u = host(res.iters), host(res.status), host(res.history), host(res.u)
    for b in (0, cfg["batch"] - 1):
        P = (lambda r: orc.jacobi(k[b], r, sweeps)) if kind == "jacobi" else (lambda r: orc.sgs(k[b], r, sweeps, "rb"))
        ref = orc.fcg(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), cfg["m"], cfg["tol"], 3000,
                      precond=P, vec32=vec32)
        it = ref["iters"]
        assert iters[b] == it and status[b] == ref["status"] == lib.CONVERGED
        assert np.array_equal(hist[b, :it + 1], ref["hist"]) and np.array_equal(u[b], ref["u"])


# ----------------------------------------------------------------------------- Chebyshev (DCT-II) SNO basis (NEXT-4)
@pytest.mark.parametrize("n,B,w,prec", [(32, 2, 8, "fp64"), (64, 2, 48, "fp32"), (128, 2, 85, "fp32"),
                                        (256, 1, 85, "fp32"), (45, 2, 16, "fp32")])
def test_no_chebyshev_matches_oracle(lib, n, B, w, prec):
    # R25: the same layer kernels with the cosine twiddle table and D^-1 folded into the mixing
    k, r, blob = _no_case(n, B, w, 141, 142)
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP64 if prec == "fp64" else lib.FP32, basis=lib.CHEBYSHEV)
    got = host(no.apply(prob, dev(r)))
    params = orc.unpack_weights(blob, w)
    tol = 1e-12 if prec == "fp64" else 1e-4
    for b in range(B):
        ref = orc.no_forward(params, r[b], k[b], basis="chebyshev")
        assert rel_l2(got[b], ref) <= tol, rel_l2(got[b], ref)


def test_fcg_no_chebyshev_hybrid_bitwise(lib):
    cfg = dict(sy.CONFIGS[2], batch=4)
    k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
    n, B, w, m = cfg["n"], cfg["batch"], cfg["width"], cfg["m"]
    prob = lib.Problem(dev(k))
    no = lib.NeuralOperator(w, blob, precision=lib.FP32, basis=lib.CHEBYSHEV)
    res = lib.fcg_solve(prob, dev(f), m=m, tol=cfg["tol"], maxit=200, no=no)
    for b in (0, B - 1):
        ref = orc.fcg(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), m, cfg["tol"], 200,
                      precond=_gpu_precond(lib, prob, no, B, n, b))
        assert np.array_equal(host(res.history)[b, :ref["iters"] + 1], ref["hist"])
        assert np.array_equal(host(res.u)[b], ref["u"])
