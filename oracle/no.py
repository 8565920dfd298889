"""Oracle: spectral neural operator (SNO, Fourier basis) used as the FCG preconditioner.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:171-183 (§2.4.2): a layer with a linear integral kernel is u <- S L A u, with
A the analysis and S the synthesis operator of a truncated basis; FNO uses FFT/iFFT.
PAPER.md:530 (App. A): SNO in Fourier basis, encoder-processor-decoder, 4 layers, 20
polynomials, GeLU, processor width 32/48/85.  The paper leaves the rest open; readings
(after SPEC.md:313-368 and SURVEY.md C.2):
  R7  mode set M = {-10..9}^2 of the full complex 2-D DFT (20 modes per dimension);
      kappa1 pairs with the row index i, kappa2 with the column index j;
  R8  analysis  c(kappa) = sum_{i,j} v(i,j) exp(-2 pi i (kappa1 i + kappa2 j)/n)
      synthesis z(i,j)   = n^-2 Re sum_{kappa in M} g(kappa) exp(+2 pi i (kappa1 i + kappa2 j)/n);
      both are the FFT restricted to M (numpy's fft2 / ifft2 used as library primitives);
  R9  L = mode-diagonal complex channel mixing g[o](kappa) = sum_c R[c][o](kappa) c[c](kappa);
  R10 encoder: v = E [r/||r||, k] + bE (no activation); 4 x [u = W v + b + S L A v;
      v = GELU(u) except after layer 4]; decoder out = D v + bD; returned value ||r|| * out,
      and 0 for r = 0;
  R11 GELU(x) = x/2 (1 + erf(x/sqrt 2)) (exact erf form).
Chebyshev variant ("neural operators from [fanaskov2022spectral]
utilizes DCT-II to work with Chebyshev polynomials"), reading R25:
  p_k(j) = cos(pi k (j + 1/2) / n), k = 0..19: T_k at the Gauss-Chebyshev nodes cos(pi (j + 1/2) / n),
      the grid index j read as the node index; quadrature weights w = 1, so
      h_k = p_k^T p_k = n (k = 0), n/2 (k > 0);
  analysis  c = D^{-1} S^T f in both dimensions, S = [p_k(j)]; synthesis f = S c S^T;
  L = mode-diagonal real channel mixing with the real part of R (the blob's imaginary parts unused).
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf

from .dots import norm2

K_MODES = 20
N_LAYERS = 4


def mode_indices(n: int, K: int = K_MODES) -> np.ndarray:
    """R7: FFT bin of each kappa in {-K/2..K/2-1}; needs n >= K so bins are distinct."""
    if n < K:
        raise ValueError(f"grid n={n} < K={K}: the mode set does not fit (reading R7)")
    kappa = np.arange(-(K // 2), K - K // 2)
    return np.mod(kappa, n)


def analysis(v: np.ndarray, K: int = K_MODES) -> np.ndarray:
    """R8 analysis of v[..., n, n] -> c[..., K, K] (axis -2: kappa1, axis -1: kappa2)."""
    n = v.shape[-1]
    idx = mode_indices(n, K)
    V = np.fft.fft2(v, axes=(-2, -1))
    return V[..., idx[:, None], idx[None, :]]


def synthesis(g: np.ndarray, n: int) -> np.ndarray:
    """R8 synthesis of g[..., K, K] -> real field [..., n, n] (zero outside M)."""
    K = g.shape[-1]
    idx = mode_indices(n, K)
    G = np.zeros(g.shape[:-2] + (n, n), dtype=complex)
    G[..., idx[:, None], idx[None, :]] = g
    return np.fft.ifft2(G, axes=(-2, -1)).real


def cheb_basis(n: int, K: int = K_MODES) -> np.ndarray:
    """R25: S[j, k] = p_k(j) = cos(pi k (j + 1/2) / n), shape [n, K]."""
    j = np.arange(n, dtype=np.float64)[:, None] + 0.5
    k = np.arange(K, dtype=np.float64)[None, :]
    return np.cos(np.pi * j * k / n)


def analysis_cheb(v: np.ndarray, K: int = K_MODES) -> np.ndarray:
    """R25 analysis c = D^-1 S^T v S D^-1 of v[..., n, n] -> c[..., K, K] (axis -2: k1 <-> row i)."""
    n = v.shape[-1]
    S = cheb_basis(n, K)
    h = np.where(np.arange(K) == 0, float(n), n / 2.0)
    return np.einsum("ik,...ij,jl->...kl", S, v, S) / h[:, None] / h[None, :]


def synthesis_cheb(g: np.ndarray, n: int) -> np.ndarray:
    """R25 synthesis f = S g S^T of g[..., K, K] -> [..., n, n]."""
    S = cheb_basis(n, g.shape[-1])
    return np.einsum("ik,...kl,jl->...ij", S, g, S)


def gelu(x):
    """R11."""
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


def param_count(width: int, K: int = K_MODES) -> int:
    """Closed-form parameter count (adapted to R7)."""
    w = width
    return (2 * w + w) + N_LAYERS * (2 * w * w * K * K + w * w + w) + (w + 1)


def unpack_weights(blob: np.ndarray, width: int, K: int = K_MODES) -> dict:
    """Canonical blob (include/fcgno.h): E[w][2], bE[w], 4 x (W[w][w], b[w],
    R[w_in][w_out][K][K][2]), D[w], bD."""
    w = width
    blob = np.asarray(blob, dtype=np.float64)
    if blob.size != param_count(w, K):
        raise ValueError("weight blob size mismatch")
    pos = 0

    def take(shape):
        nonlocal pos
        size = int(np.prod(shape))
        out = blob[pos:pos + size].reshape(shape)
        pos += size
        return out

    p = {"E": take((w, 2)), "bE": take((w,)), "W": [], "b": [], "R": []}
    for _ in range(N_LAYERS):
        p["W"].append(take((w, w)))
        p["b"].append(take((w,)))
        R = take((w, w, K, K, 2))
        p["R"].append(R[..., 0] + 1j * R[..., 1])
    p["D"] = take((w,))
    p["bD"] = take((1,))[0]
    assert pos == blob.size
    return p


def no_forward(params: dict, r: np.ndarray, k: np.ndarray, use_gelu: bool = True, basis: str = "fourier") -> np.ndarray:
    """Preconditioner w = B(r) for one system, r and k of shape [n, n] (R7-R11; basis 'chebyshev': R25).

    ``use_gelu=False`` is a test-only linear mode."""
    r = np.asarray(r, dtype=np.float64)
    n = r.shape[-1]
    s = norm2(r)
    if s == 0.0:
        return np.zeros_like(r)
    x0 = np.stack([r / s, np.asarray(k, dtype=np.float64)])          # [2, n, n]
    v = np.einsum("ci,ihw->chw", params["E"], x0) + params["bE"][:, None, None]
    for l in range(N_LAYERS):
        if basis == "fourier":
            c_hat = analysis(v)                                        # [w, K, K]
            g_hat = np.einsum("cokl,ckl->okl", params["R"][l], c_hat)  # L: mode-diagonal mixing
            z = synthesis(g_hat, n)
        elif basis == "chebyshev":
            c_hat = analysis_cheb(v)
            g_hat = np.einsum("cokl,ckl->okl", params["R"][l].real, c_hat)
            z = synthesis_cheb(g_hat, n)
        else:
            raise ValueError(basis)
        u = np.einsum("oc,chw->ohw", params["W"][l], v) + params["b"][l][:, None, None] + z
        v = (gelu(u) if use_gelu else u) if l < N_LAYERS - 1 else u
    out = np.einsum("c,chw->hw", params["D"], v) + params["bD"]
    return s * out
