"""Pins for oracle/train.py: the loss gradient against central finite
differences of the loss itself (the mathematics, not a retyped formula), the losses' closed forms
(P:276-282), AdamW against torch.optim.AdamW (a library routine) and its first-step closed form,
the Krylov samples (Eq. 8-9) against Krylov-subspace membership and A e_i = r_i."""
import math

import numpy as np
import pytest

import oracle as orc
import synthetic as sy
from oracle import train as otr


def _tiny(seed=3, n=20, w=3, B=2):
    k = sy.lognormal_k(n, B, 0.1, 1.0, seed)
    r = np.random.default_rng(seed).normal(size=(B, n, n))
    e = np.stack([np.linalg.solve(orc.dense_A(k[b]), r[b].ravel()).reshape(n, n) for b in range(B)])
    blob = sy.no_weights(w, seed)
    return k, r, e, blob


def test_pack_is_inverse_of_unpack():
    blob = sy.no_weights(4, 1)
    assert np.array_equal(otr.pack_weights(orc.unpack_weights(blob, 4), 4), blob)


def test_cached_forward_is_the_pinned_forward():
    k, r, _, blob = _tiny()
    p = orc.unpack_weights(blob, 3)
    for b in range(2):
        w, _ = otr.no_forward_cache(p, r[b], k[b])
        ref = orc.no_forward(p, r[b], k[b])
        assert np.max(np.abs(w - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_gelu_grad_matches_difference_quotient():
    x = np.linspace(-6, 6, 101)
    h = 1e-6
    fd = (orc.gelu(x + h) - orc.gelu(x - h)) / (2 * h)
    assert np.max(np.abs(fd - otr.gelu_grad(x))) < 1e-8


@pytest.mark.parametrize("kind", ["notay", "l2"])
def test_gradient_matches_central_differences(kind):
    """Every block of the canonical blob (E, bE, W_l, b_l, Re/Im R_l, D, bD): sampled entries of the
    analytic gradient agree with (L(theta + h) - L(theta - h)) / 2h."""
    w = 3
    k, r, e, blob = _tiny()
    _, g = otr.loss_and_grad(blob, w, r, e, k, kind)
    L = lambda th: float(np.mean(otr.loss_and_grad(th, w, r, e, k, kind)[0]))   # noqa: E731
    # block offsets of the canonical layout
    K2 = 400
    offs = {"E": (0, 2 * w), "bE": (2 * w, 3 * w)}
    pos = 3 * w
    for l in range(4):
        offs[f"W{l}"] = (pos, pos + w * w); pos += w * w
        offs[f"b{l}"] = (pos, pos + w); pos += w
        offs[f"R{l}"] = (pos, pos + 2 * w * w * K2); pos += 2 * w * w * K2
    offs["D"] = (pos, pos + w); offs["bD"] = (pos + w, pos + w + 1)
    rng = np.random.default_rng(0)
    gmax = np.max(np.abs(g))
    for name, (a, b) in offs.items():
        if name.startswith("R"):
            # the modes that carry signal: pick entries with non-negligible gradient plus random ones
            big = a + np.argsort(-np.abs(g[a:b]))[:4]
            idx = np.concatenate([big, rng.integers(a, b, 2)])
        else:
            idx = rng.integers(a, b, min(4, b - a))
        for j in idx:
            h = 1e-5 * max(1.0, abs(blob[j]))
            tp, tm = blob.copy(), blob.copy()
            tp[j] += h
            tm[j] -= h
            fd = (L(tp) - L(tm)) / (2 * h)
            assert abs(fd - g[j]) <= 2e-6 * abs(g[j]) + 1e-9 * gmax, (name, j, fd, g[j])


def test_gradient_is_zero_for_bias_free_zero_output():
    """Zero E, bE and biases give v = 0 in every layer and out = bD: the gradients of the weights
    that multiply an activation (W_l, R_l, D) vanish, those of the biases and E do not."""
    w = 3
    k, r, e, blob = _tiny()
    p = orc.unpack_weights(blob, w)
    p["E"][:] = 0; p["bE"][:] = 0
    for l in range(4):
        p["b"][l][:] = 0
    th = otr.pack_weights(p, w)
    _, g = otr.loss_and_grad(th, w, r, e, k, "notay")
    gp = orc.unpack_weights(g, w)
    for l in range(4):
        assert np.all(gp["W"][l] == 0.0) and np.all(gp["R"][l] == 0.0)
        assert np.any(gp["b"][l] != 0.0)
    assert np.all(gp["D"] == 0.0) and gp["bD"] != 0.0 and np.any(gp["E"] != 0.0)


def test_loss_closed_forms():
    """B(r) = e gives 0, B(r) = 0 gives 1, B(r) = c e gives |1 - c| in both norms."""
    k, _, e, _ = _tiny(B=1)
    for kind in ("notay", "l2"):
        assert otr.notay_loss(k[0], e[0] * 0.0, e[0], kind)[0] == pytest.approx(1.0, abs=1e-14)
        for c in (0.5, 1.25):
            assert otr.notay_loss(k[0], c * e[0], e[0], kind)[0] == pytest.approx(abs(1 - c), abs=1e-13)
    l, dw = otr.notay_loss(k[0], e[0] * 0.5, e[0], "notay")
    # the gradient of ||w - e||_A / ||e||_A at w = e/2 is A(w - e) / (||w - e||_A ||e||_A): check by
    # a directional difference quotient along a random direction
    dirn = np.random.default_rng(1).normal(size=e[0].shape)
    h = 1e-6 * float(np.max(np.abs(e[0])))
    fd = (otr.notay_loss(k[0], 0.5 * e[0] + h * dirn, e[0])[0] - otr.notay_loss(k[0], 0.5 * e[0] - h * dirn, e[0])[0]) / (2 * h)
    assert fd == pytest.approx(float(np.sum(dw * dirn)), rel=1e-7)


def test_adamw_matches_torch_and_first_step_closed_form():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    th = rng.normal(size=50)
    grads = [rng.normal(size=50) for _ in range(6)]
    lr, wd = 1e-3, 1e-2
    pt = torch.tensor(th.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.AdamW([pt], lr=lr, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd)
    m = np.zeros(50); v = np.zeros(50); cur = th.copy()
    for t, g in enumerate(grads, start=1):
        pt.grad = torch.tensor(g)
        opt.step()
        cur, m, v = otr.adamw_step(cur, g, m, v, t, lr, weight_decay=wd)
        assert np.max(np.abs(cur - pt.detach().numpy())) < 1e-15 * 10
    # first step: m_hat = g, v_hat = g^2, so theta1 = theta0 (1 - lr wd) - lr g / (|g| + eps)
    g = grads[0]
    t1, _, _ = otr.adamw_step(th, g, np.zeros(50), np.zeros(50), 1, lr, weight_decay=wd)
    assert np.max(np.abs(t1 - (th * (1 - lr * wd) - lr * g / (np.abs(g) + 1e-8)))) < 1e-15


def test_lr_schedule_table6():
    assert otr.lr_at_epoch(0) == 1e-3 and otr.lr_at_epoch(49) == 1e-3
    assert otr.lr_at_epoch(50) == 5e-4 and otr.lr_at_epoch(149) == 2.5e-4


def test_krylov_samples_lie_in_the_krylov_subspace():
    """Eq. 8-9: r_i = f - A u_i lies in K_{i+1}(A, r_0) = span{r0, A r0, ..., A^i r0} and A e_i = r_i."""
    n = 6
    k = sy.lognormal_k(n, 1, 0.2, 1.0, 9)[0]
    f = sy.normal_field(n, 1, 9)[0]
    u0 = np.random.default_rng(9).normal(size=(n, n))
    Ad = orc.dense_A(k)
    iters = [0, 1, 3, 5]
    rs, es, ue = otr.krylov_samples(k, f, u0, iters, m_max=5, tol_exact=1e-14, maxit_exact=500)
    x_ex = np.linalg.solve(Ad, f.ravel())
    assert np.max(np.abs(ue.ravel() - x_ex)) < 1e-10 * np.max(np.abs(x_ex))
    r0 = (f - orc.apply_A(k, u0)).ravel()
    for s, i in enumerate(iters):
        basis = [r0]
        for _ in range(i):
            basis.append(Ad @ basis[-1])
        Kb = np.stack(basis, axis=1)
        Q, _ = np.linalg.qr(Kb)
        ri = rs[s].ravel()
        assert np.linalg.norm(ri - Q @ (Q.T @ ri)) <= 1e-9 * np.linalg.norm(ri), i
        if i + 2 <= n * n:        # and not in the smaller subspace (CG makes progress)
            Qs, _ = np.linalg.qr(Kb[:, :max(1, i)])
            if i > 0:
                assert np.linalg.norm(ri - Qs @ (Qs.T @ ri)) > 1e-6 * np.linalg.norm(ri)
        assert np.max(np.abs(Ad @ es[s].ravel() - ri)) < 1e-9 * np.max(np.abs(f))
    assert np.array_equal(rs[0], f - orc.apply_A(k, u0))


def test_krylov_target_unit_and_scale_invariance_of_fcg():
    """R27: e_scale only rescales the target (A e_i = e_scale r_i), and FCG is invariant to a positive
    scaling of the preconditioner (alpha is a line search), which is why weights trained against
    the scaled target precondition as they are."""
    n = 6
    k = sy.lognormal_k(n, 1, 0.2, 1.0, 3)[0]
    f = sy.normal_field(n, 1, 3)[0]
    u0 = np.zeros((n, n))
    Ad = orc.dense_A(k)
    c = float((n + 1) ** 2)
    r1, e1, ue = otr.krylov_samples(k, f, u0, [0, 2], m_max=5, tol_exact=1e-14, maxit_exact=500)
    rc, ec, _ = otr.krylov_samples(k, f, u0, [0, 2], m_max=5, u_exact=ue, e_scale=c)
    assert np.array_equal(r1, rc) and np.array_equal(ec, c * e1)
    assert np.max(np.abs(Ad @ ec[1].ravel() - c * r1[1].ravel())) < 1e-9 * c * np.max(np.abs(f))
    A = lambda x: orc.apply_A(k, x)
    Minv = np.linalg.inv(Ad + 3.0 * np.diag(np.diag(Ad)))      # some SPD preconditioner
    B1 = lambda r: (Minv @ r.ravel()).reshape(n, n)
    Bc = lambda r: c * B1(r)
    o1 = orc.fcg(A, f, u0, 5, 1e-10, 200, precond=B1)
    oc = orc.fcg(A, f, u0, 5, 1e-10, 200, precond=Bc)
    assert o1["iters"] == oc["iters"]
    assert np.max(np.abs(o1["u"] - oc["u"])) <= 1e-12 * np.max(np.abs(o1["u"]))
    assert np.allclose(o1["hist"], oc["hist"], rtol=1e-9, atol=0)
