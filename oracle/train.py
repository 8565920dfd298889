"""Oracle: training the SNO preconditioner.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it computes, in the paper's order:
  - Krylov-subspace training residuals (Eq. 8-9; Fig. 3): draw f and
    u0, run CG (FCG with B = I, Algorithm 1) for i iterations, keep r_i = f - A u_i and the error
    e_i = u_exact - u_i = A^{-1} r_i, u_exact from a tight FCG(I) solve;
  - the Notay loss in its error form (Eq. notay_loss_with_error)
        L = mean_b ||B(r_b; theta) - e_b||_A / ||e_b||_A
    and the L2 form (Eq. l2_loss_with_error) with ||.||_2;
  - the gradient of L with respect to every weight of the SNO (oracle/no.py's forward, readings
    R7-R11), by the chain rule through projection, the four layers and the lift (reverse order of
    no_forward), with the adjoints of the truncated transforms:
        synthesis z = n^-2 Re sum_M g e^{+i theta}   ->  dg = n^-2 sum_x dz e^{-i theta} = analysis(dz) / n^2
        analysis  c = sum_x v e^{-i theta}           ->  dv = Re sum_M dc e^{+i theta}   = n^2 synthesis(dc)
        mixing    g_o = sum_c R_co c_c (complex)     ->  dc_c = sum_o conj(R_co) dg_o,  dR_co = dg_o conj(c_c)
    (complex gradients in the convention dL/dRe + i dL/dIm);
  - one AdamW step (decoupled weight decay; reading R26) with Table 6's hyperparameters
    (lr 1e-3 halved every 50 epochs, weight decay 1e-2).

The gradient is pinned by central finite differences of the loss (tests/test_oracle_train.py);
AdamW against torch.optim.AdamW and its first-step closed form; the Krylov samples by the
Krylov-subspace membership of r_i and A e_i = r_i.
"""
from __future__ import annotations

import math

import numpy as np

from .fcg import fcg
from .no import K_MODES, N_LAYERS, analysis, gelu, param_count, synthesis, unpack_weights
from .stencil import apply_A


def gelu_grad(x):
    """d/dx of R11's GELU: Phi(x) + x phi(x)."""
    from scipy.special import erf
    return 0.5 * (1.0 + erf(x / math.sqrt(2.0))) + x * np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)


def pack_weights(p: dict, width: int, K: int = K_MODES) -> np.ndarray:
    """Inverse of no.unpack_weights: the canonical blob of include/fcgno.h."""
    parts = [np.asarray(p["E"]).ravel(), np.asarray(p["bE"]).ravel()]
    for l in range(N_LAYERS):
        R = np.asarray(p["R"][l])
        parts += [np.asarray(p["W"][l]).ravel(), np.asarray(p["b"][l]).ravel(),
                  np.stack([R.real, R.imag], axis=-1).ravel()]
    parts += [np.asarray(p["D"]).ravel(), np.array([p["bD"]], dtype=np.float64)]
    blob = np.concatenate(parts).astype(np.float64)
    assert blob.size == param_count(width, K)
    return blob


def no_forward_cache(params: dict, r: np.ndarray, k: np.ndarray):
    """oracle.no.no_forward (Fourier basis, GELU) keeping what the backward pass needs.
    Returns (w = ||r|| out, cache)."""
    r = np.asarray(r, dtype=np.float64)
    n = r.shape[-1]
    s = math.sqrt(float(np.dot(r.ravel(), r.ravel())))
    x0 = np.stack([r / s, np.asarray(k, dtype=np.float64)])                 # [2, n, n]
    v = np.einsum("ci,ihw->chw", params["E"], x0) + params["bE"][:, None, None]
    vs, zs, cs = [v], [], []
    for l in range(N_LAYERS):
        c_hat = analysis(v)                                                  # [w, K, K]
        g_hat = np.einsum("cokl,ckl->okl", params["R"][l], c_hat)
        z = np.einsum("oc,chw->ohw", params["W"][l], v) + params["b"][l][:, None, None] + synthesis(g_hat, n)
        v = gelu(z) if l < N_LAYERS - 1 else z
        zs.append(z)
        cs.append(c_hat)
        vs.append(v)
    out = np.einsum("c,chw->hw", params["D"], v) + params["bD"]
    return s * out, {"s": s, "x0": x0, "v": vs, "z": zs, "c": cs, "n": n}


def no_backward(params: dict, cache: dict, dw: np.ndarray) -> dict:
    """Gradient of a scalar loss with respect to the weights, given dL/dw for w = ||r|| out
    (||r|| does not depend on the weights).  Returns a dict shaped like the weights."""
    n, s = cache["n"], cache["s"]
    dout = s * np.asarray(dw, dtype=np.float64)                              # [n, n]
    v4 = cache["v"][N_LAYERS]
    g = {"W": [None] * N_LAYERS, "b": [None] * N_LAYERS, "R": [None] * N_LAYERS}
    g["D"] = np.einsum("hw,chw->c", dout, v4)
    g["bD"] = float(dout.sum())
    dv = params["D"][:, None, None] * dout[None]                             # dL/dv4 [w, n, n]
    for l in reversed(range(N_LAYERS)):
        z, v_in, c_hat = cache["z"][l], cache["v"][l], cache["c"][l]
        dz = dv * gelu_grad(z) if l < N_LAYERS - 1 else dv
        g["W"][l] = np.einsum("ohw,chw->oc", dz, v_in)
        g["b"][l] = dz.sum(axis=(1, 2))
        dg_hat = analysis(dz) / (n * n)                                      # adjoint of synthesis
        g["R"][l] = np.einsum("okl,ckl->cokl", dg_hat, np.conj(c_hat))
        dc_hat = np.einsum("cokl,okl->ckl", np.conj(params["R"][l]), dg_hat)
        dv = np.einsum("oc,ohw->chw", params["W"][l], dz) + (n * n) * synthesis(dc_hat, n)
    x0 = cache["x0"]
    g["E"] = np.einsum("chw,ihw->ci", dv, x0)
    g["bE"] = dv.sum(axis=(1, 2))
    return g


def notay_loss(k, w, e, kind: str = "notay"):
    """One sample's loss and dL/dw: kind 'notay' ||w - e||_A / ||e||_A
    (Eq. notay_loss_with_error), 'l2' ||w - e||_2 / ||e||_2 (Eq. l2_loss_with_error)."""
    d = np.asarray(w, dtype=np.float64) - np.asarray(e, dtype=np.float64)
    if kind == "notay":
        Ad, Ae = apply_A(k, d), apply_A(k, e)
        nd, ne = math.sqrt(float(np.sum(d * Ad))), math.sqrt(float(np.sum(e * Ae)))
        return nd / ne, Ad / (nd * ne)
    if kind == "l2":
        nd, ne = math.sqrt(float(np.sum(d * d))), math.sqrt(float(np.sum(e * e)))
        return nd / ne, d / (nd * ne)
    raise ValueError(kind)


def loss_and_grad(blob, width, r, e, k, kind: str = "notay"):
    """Mean loss over the batch r, e, k [B][n][n] and its gradient as a canonical blob."""
    p = unpack_weights(blob, width)
    B = r.shape[0]
    losses = np.zeros(B)
    total = np.zeros(param_count(width))
    for b in range(B):
        w, cache = no_forward_cache(p, r[b], k[b])
        losses[b], dw = notay_loss(k[b], w, e[b], kind)
        total += pack_weights(no_backward(p, cache, dw / B), width)
    return losses, total


def adamw_step(theta, grad, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=1e-2):
    """One AdamW step (reading R26: Adam, Kingma & Ba, with decoupled weight decay applied first),
    t = 1, 2, ...  Returns new (theta, m, v)."""
    theta = theta * (1.0 - lr * weight_decay)
    m = beta1 * m + (1.0 - beta1) * grad
    v = beta2 * v + (1.0 - beta2) * grad * grad
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    return theta - lr * mhat / (np.sqrt(vhat) + eps), m, v


def lr_at_epoch(epoch: int, lr0: float = 1e-3, decay: float = 0.5, every: int = 50) -> float:
    """Table 6: lr 1e-3, x0.5 every 50 epochs."""
    return lr0 * decay ** (epoch // every)


def krylov_samples(k, f, u0, iters, m_max=5, u_exact=None, tol_exact=1e-13, maxit_exact=100000, e_scale=1.0):
    """Training pairs of one system (Eq. 8-9; Fig. 3): for each i in `iters`, the CG
    iterate u_i (FCG with B = I stopped after i iterations, Algorithm 1), r_i = f - A u_i and
    e_i = e_scale (u_exact - u_i) (e_scale: the unit of the target, R27; 1 as printed).  u_exact: a tight FCG(I) solve unless given.  Returns (r [S][n][n],
    e [S][n][n], u_exact)."""
    A = lambda x: apply_A(k, x)
    if u_exact is None:
        u_exact = fcg(A, f, u0, m_max, tol_exact, maxit_exact)["u"]
    rs, es = [], []
    for i in iters:
        u_i = fcg(A, f, u0, m_max, 0.0, int(i))["u"]
        rs.append(f - A(u_i))
        es.append(e_scale * (u_exact - u_i))
    return np.array(rs), np.array(es), u_exact
