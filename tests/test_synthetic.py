"""T0: the seeded input generators behind every parity check and bench line —
determinism, per-system regeneration, and the statistics BASELINE.json's recipes fix (GRF variance
and squared-exponential correlation, rectangle value range, N(0,1) fields, N(0, 1/fan_in) weights)."""
import numpy as np

import synthetic as sy


def test_deterministic_and_per_system_regeneration():
    cfg = sy.CONFIGS[2]
    a, b = sy.make_k(cfg), sy.make_k(cfg)
    assert np.array_equal(a, b)
    assert np.array_equal(sy.make_k(cfg, systems=[5, 17])[1], a[17])     # any system alone (D.2)
    assert np.array_equal(sy.make_f(cfg, systems=[63])[0], sy.make_f(cfg)[63])
    assert not np.array_equal(a[0], a[1])
    assert np.array_equal(sy.make_weights(cfg), sy.make_weights(cfg))
    # config 5 reuses config 2's weights (BJ configs[4] "same NO weights as the 64x64 config")
    assert np.array_equal(sy.make_weights(sy.CONFIGS[5]), sy.make_weights(cfg))


def test_grf_variance_and_correlation():
    # BJ configs[0]/[2]: squared-exponential covariance sigma2 exp(-r^2 / (2 l^2))
    for n, length, var in ((64, 0.1, 1.0), (128, 0.05, 4.0)):
        g = sy.grf(n, 16, length, var, seed=7)
        assert abs(g.var() / var - 1.0) < 0.15
        h = 1.0 / (n + 1)
        lag = int(round(length / h))
        r = lag * h
        corr = np.mean(g[:, :, :-lag] * g[:, :, lag:]) / g.var()
        assert abs(corr - np.exp(-r * r / (2 * length * length))) < 0.08
        assert np.all(np.isfinite(np.exp(g)))


def test_rectangles_values_and_background():
    k = sy.rectangles_k(64, 8, seed=3)
    assert np.all(k >= 1e-2) and np.all(k <= 1e2)
    assert np.any(k == 1.0)                                  # background k = 1 survives somewhere
    assert len(np.unique(k[0])) > 4                          # several rectangles per system


def test_normal_field_and_weight_scales():
    f = sy.normal_field(64, 32, seed=11)
    assert abs(f.mean()) < 0.02 and abs(f.var() - 1.0) < 0.03
    w = 48
    blob = sy.no_weights(w, seed=5)
    assert blob.size == sy.no_blob_size(w)
    # R17: E, b_E ~ N(0, 1/2); W_l ~ N(0, 1/w) (first layer block after the lift)
    E = blob[:2 * w]
    W1 = blob[3 * w:3 * w + w * w]
    assert abs(E.var() / 0.5 - 1.0) < 0.25
    assert abs(W1.var() * w - 1.0) < 0.1
