"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module draws random numbers and lays out arrays; it holds none of the
method's arithmetic (no stencil, no dot product, no NO layer, no FCG step).
Both the CPU oracle (``oracle/``) and the CUDA path receive exactly the arrays
produced here, so every parity check starts from bit-identical inputs.

Random streams: one counter-based Philox generator per (seed, system, stream),
so any single system ``b`` of a batch can be regenerated alone (SURVEY.md
§8(d) D.2).  Streams: 0 = k, 1 = f, 2 = u0, 3 = NO weights.

Field recipes (BASELINE.json configs, readings in DESIGN.md §3):
  * ``lognormal_k``: k = exp(g), g a Gaussian random field with squared-exponential
    covariance sigma2*exp(-|x-y|^2/(2 l^2)) sampled by a 2-D FFT with periodic
    embedding of 2(n+1) points per dimension at spacing h=1/(n+1)
    (SURVEY.md C.2 #24).
  * ``rectangles_k``: background 1, 16 axis-aligned rectangles with log-uniform
    values in [1e-2, 1e2]; later rectangles overwrite earlier ones (C.2 #25).
  * ``normal_field``: i.i.d. N(0,1) per node.
  * ``smooth_plus_noise``: GRF(l=0.1, sigma2=1) + N(0,1) (C.2 #26).
  * ``trig_poly``: PAPER.md §3.2 random trigonometric polynomials P(N1,N2,alpha)
    (PAPER.md:287-295), used only for the Table 1 CG pin.
  * ``no_weights``: canonical fp64 SNO weight blob with N(0, 1/fan_in) entries
    (BASELINE.json configs[0]; layout in include/fcgno.h).
"""
from __future__ import annotations

import numpy as np

K_MODES = 20  # PAPER.md:530 "number of orthogonal polynomials is 20"
N_LAYERS = 4  # PAPER.md:530 "Number of SNO layers is 4"

STREAM_K, STREAM_F, STREAM_U0, STREAM_W = 0, 1, 2, 3


def rng(seed: int, system: int, stream: int) -> np.random.Generator:
    """Counter-based generator for (seed, system, stream)."""
    key = np.array([np.uint64(seed), np.uint64(system * 16 + stream)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def node_coords(n: int) -> np.ndarray:
    """Interior node coordinates (j+1)h, h = 1/(n+1)."""
    return (np.arange(n, dtype=np.float64) + 1.0) / (n + 1)


# ----------------------------------------------------------------------------- fields
def _grf_one(n: int, length: float, variance: float, g: np.random.Generator) -> np.ndarray:
    me = 2 * (n + 1)                 # periodic embedding points per dimension
    h = 1.0 / (n + 1)
    period = me * h                  # = 2
    q = np.fft.fftfreq(me, d=1.0 / me)           # integer wavenumbers
    xi2 = (q[:, None] ** 2 + q[None, :] ** 2) / period ** 2
    spec = variance * 2.0 * np.pi * length ** 2 * np.exp(-2.0 * np.pi ** 2 * length ** 2 * xi2)
    amp = np.sqrt(spec) / period
    zeta = g.standard_normal((me, me)) + 1j * g.standard_normal((me, me))
    field = np.fft.ifft2(amp * zeta) * (me * me)
    return np.ascontiguousarray(field.real[:n, :n])


def grf(n: int, batch: int, length: float, variance: float, seed: int, stream: int = STREAM_K,
        systems=None) -> np.ndarray:
    systems = range(batch) if systems is None else systems
    return np.stack([_grf_one(n, length, variance, rng(seed, b, stream)) for b in systems])


def lognormal_k(n, batch, length, variance, seed, systems=None):
    return np.exp(grf(n, batch, length, variance, seed, STREAM_K, systems))


def rectangles_k(n, batch, seed, count=16, lo=1e-2, hi=1e2, systems=None):
    systems = range(batch) if systems is None else systems
    x = node_coords(n)
    out = []
    for b in systems:
        g = rng(seed, b, STREAM_K)
        k = np.ones((n, n))
        for _ in range(count):
            x0, x1 = np.sort(g.random(2))
            y0, y1 = np.sort(g.random(2))
            val = np.exp(g.uniform(np.log(lo), np.log(hi)))
            rows = (x >= y0) & (x <= y1)          # row index i <-> x2
            cols = (x >= x0) & (x <= x1)          # column index j <-> x1
            k[np.ix_(rows, cols)] = val
        out.append(k)
    return np.stack(out)


def normal_field(n, batch, seed, stream=STREAM_F, systems=None):
    systems = range(batch) if systems is None else systems
    return np.stack([rng(seed, b, stream).standard_normal((n, n)) for b in systems])


def smooth_plus_noise(n, batch, seed, systems=None):
    systems = range(batch) if systems is None else systems
    out = []
    for b in systems:
        g = rng(seed, b, STREAM_F)
        out.append(_grf_one(n, 0.1, 1.0, g) + g.standard_normal((n, n)))
    return np.stack(out)


def trig_poly(n, batch, seed, n1=5, n2=5, alpha=2.0, offset=0.0, stream=STREAM_F, systems=None):
    """Re sum_{m<=N1,n<=N2} c_mn exp(2 pi i (m x1 + n x2)) / (1+m+n)^alpha,
    c_mn with independent N(0,1) real and imaginary parts, plus offset."""
    systems = range(batch) if systems is None else systems
    x = node_coords(n)
    out = []
    for b in systems:
        g = rng(seed, b, stream)
        c = g.standard_normal((n1 + 1, n2 + 1)) + 1j * g.standard_normal((n1 + 1, n2 + 1))
        field = np.zeros((n, n), dtype=complex)
        for m in range(n1 + 1):
            for q in range(n2 + 1):
                # x1 <-> column j, x2 <-> row i
                field += c[m, q] * np.exp(2j * np.pi * (m * x[None, :] + q * x[:, None])) / (1.0 + m + q) ** alpha
        out.append(field.real + offset)
    return np.stack(out)


# ----------------------------------------------------------------------------- NO weights
def no_blob_size(width: int, modes: int = K_MODES) -> int:
    w = width
    return 2 * w + w + N_LAYERS * (w * w + w + w * w * modes * modes * 2) + w + 1


def no_weights(width: int, seed: int, modes: int = K_MODES) -> np.ndarray:
    """Canonical fp64 blob (include/fcgno.h FCGNO_BLOB layout):
    E[w][2], bE[w], then per layer l=1..4: W[w_out][w_in], b[w], R[w_in][w_out][K][K][2],
    then D[w], bD.  Init N(0, 1/fan_in) (BASELINE.json configs[0]); spectral weights
    have real and imaginary parts each N(0, 1/(2w))."""
    w, K = width, modes
    g = rng(seed, 0, STREAM_W)
    parts = [g.normal(0, np.sqrt(1 / 2), (w, 2)).ravel(), g.normal(0, np.sqrt(1 / 2), w)]
    for _ in range(N_LAYERS):
        parts.append(g.normal(0, np.sqrt(1 / w), (w, w)).ravel())
        parts.append(g.normal(0, np.sqrt(1 / w), w))
        parts.append(g.normal(0, np.sqrt(1 / (2 * w)), (w, w, K, K, 2)).ravel())
    parts.append(g.normal(0, np.sqrt(1 / w), w))
    parts.append(g.normal(0, np.sqrt(1 / w), 1))
    blob = np.concatenate(parts)
    assert blob.size == no_blob_size(w, K)
    return blob


def structured_no_weights(width: int, n_w: int, modes: int = K_MODES) -> np.ndarray:
    """Hand-set point of the SNO weight space (not the paper's):
    two channels carry +y/-y so GELU(y)-GELU(-y)=y, realising w = alpha r + S L A r with an
    inverse-Laplacian symbol L(kappa)=1/(4 pi^2 |kappa|^2 + 2 pi^2), alpha = h_w^2/4.
    A supplementary workload that converges (random-init weights do not)."""
    w, K = width, modes
    assert w >= 2
    E = np.zeros((w, 2)); E[0, 0] = 1.0; E[1, 0] = -1.0
    bE = np.zeros(w)
    hw = 1.0 / (n_w + 1)
    alpha = hw * hw / 4.0
    kap = np.arange(K) - K // 2
    L = 1.0 / (4 * np.pi ** 2 * (kap[:, None] ** 2 + kap[None, :] ** 2) + 2 * np.pi ** 2)
    layers = []
    for l in range(N_LAYERS):
        W = np.zeros((w, w)); b = np.zeros(w); R = np.zeros((w, w, K, K, 2))
        if l == 0:
            W[:2, :2] = (alpha / 2) * np.array([[1, -1], [-1, 1]])
            for c in range(2):
                for o in range(2):
                    R[c, o, :, :, 0] = (0.5 if c == o else -0.5) * L
        elif l in (1, 2):
            W[:2, :2] = np.array([[1, -1], [-1, 1]])
        else:
            W[0, :2] = [1, -1]
        layers.append((W, b, R))
    D = np.zeros(w); D[0] = 1.0
    parts = [E.ravel(), bE]
    for W, b, R in layers:
        parts += [W.ravel(), b, R.ravel()]
    parts += [D, np.zeros(1)]
    return np.concatenate(parts)


# ----------------------------------------------------------------------------- configs
# BASELINE.json configs, restated as concrete recipes.
CONFIGS = {
    1: dict(n=32, batch=1, k="lognormal", length=0.1, variance=1.0, rhs="normal", m=5, tol=1e-8,
            maxit=500, width=32, no_precision="fp64", seed=101, wseed=1001),
    2: dict(n=64, batch=64, k="lognormal", length=0.1, variance=1.0, rhs="normal", m=5, tol=1e-6,
            maxit=2000, width=48, no_precision="fp32", seed=102, wseed=1002),
    3: dict(n=128, batch=128, k="lognormal", length=0.05, variance=4.0, rhs="smooth_noise", m=10,
            tol=1e-6, maxit=2000, width=85, no_precision="fp32", seed=103, wseed=1003),
    4: dict(n=256, batch=32, k="rectangles", rhs="normal", m=10, tol=1e-8, maxit=2000, width=85,
            no_precision="fp32", seed=104, wseed=1003),
    5: dict(n=512, batch=8, k="lognormal", length=0.1, variance=1.0, rhs="normal", m=10, tol=1e-8,
            maxit=2000, width=48, no_precision="fp32", seed=105, wseed=1002),
}


def make_k(cfg: dict, systems=None) -> np.ndarray:
    n, B, seed = cfg["n"], cfg["batch"], cfg["seed"]
    if cfg["k"] == "lognormal":
        return lognormal_k(n, B, cfg["length"], cfg["variance"], seed, systems)
    if cfg["k"] == "rectangles":
        return rectangles_k(n, B, seed, systems=systems)
    raise ValueError(cfg["k"])


def make_f(cfg: dict, systems=None) -> np.ndarray:
    n, B, seed = cfg["n"], cfg["batch"], cfg["seed"]
    if cfg["rhs"] == "normal":
        return normal_field(n, B, seed, STREAM_F, systems)
    if cfg["rhs"] == "smooth_noise":
        return smooth_plus_noise(n, B, seed, systems)
    raise ValueError(cfg["rhs"])


def make_weights(cfg: dict) -> np.ndarray:
    return no_weights(cfg["width"], cfg["wseed"])
