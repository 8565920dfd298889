"""Train the SNO preconditioner on the GPU (the paper's Fig. 3 scheme)
and evaluate FCG-NO on held-out systems against FCG(I) (the shape of the paper's Tables 1-2).

  python scripts/train_sno.py --config 1 --epochs 150 > profiles/r02/train_c1.json

Data (synthetic, seeded; R27), --dataset:
  diffusion  the paper's Diffusion set: a ~ P(5,5,2) + 10, f ~ P(5,5,2), u0 ~ N(0, I)
  poisson    the paper's Poisson set: a = 1, f ~ P(5,5,2), u0 ~ N(0, I)
  lognormal  the BASELINE config's k field (exp of a Gaussian random field) and N(0,1) f, u0 = 0
Training residuals are CG iterates at the iterations --iters (Eq. 8-9); the target is the error in
units of the unscaled stencil, e_scale = (n+1)^2 (R27; --e-scale 1 gives A^{-1} r as printed).  Every
step runs in libfcgno.so (paper_2402_05598_b200/train.py sequences the calls)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic as sy  # noqa: E402
from paper_2402_05598_b200 import fcgno  # noqa: E402
from paper_2402_05598_b200 import train as ptr  # noqa: E402

CONFIGS = {   # n, width, k recipe (BASELINE configs), FCG m, Table 6 batch
    1: dict(n=32, width=32, length=0.1, variance=1.0, m=5, batch=16),
    2: dict(n=64, width=48, length=0.1, variance=1.0, m=5, batch=16),
}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--train-systems", type=int, default=256)
    ap.add_argument("--test-systems", type=int, default=64)
    ap.add_argument("--iters", type=int, nargs="*", default=[0, 1, 2, 4, 8, 16, 32, 64, 128])
    ap.add_argument("--epochs", type=int, default=150)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--loss", choices=["notay", "l2"], default="notay")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--maxit", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dataset", choices=["diffusion", "poisson", "lognormal"], default="diffusion")
    ap.add_argument("--e-scale", type=float, default=None, help="unit of the target (default (n+1)^2)")
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--m-test", type=int, nargs="*", default=[], help="extra FCG windows m for the held-out solves (P:406 uses m_max = 20)")
    ap.add_argument("--save", default=None, help="write the trained weight blob (.npy)")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    n, w, m = c["n"], args.width or c["width"], c["m"]
    batch = args.batch or c["batch"]
    torch.cuda.init()

    e_scale = args.e_scale if args.e_scale is not None else float((n + 1) ** 2)

    def system_set(count, seed):
        if args.dataset == "lognormal":
            k = sy.lognormal_k(n, count, c["length"], c["variance"], seed)
            f = sy.normal_field(n, count, seed + 1)
            u0 = np.zeros_like(f)
        else:
            k = (np.ones((count, n, n)) if args.dataset == "poisson"
                 else sy.trig_poly(n, count, seed, offset=10.0, stream=0))
            f = sy.trig_poly(n, count, seed)
            u0 = sy.normal_field(n, count, seed + 2)
        return k, f, u0

    k_tr, f_tr, u0_tr = system_set(args.train_systems, 1000 + args.seed)
    k_te, f_te, u0_te = system_set(args.test_systems, 5000 + args.seed)
    p_tr, p_te = fcgno.Problem(dev(k_tr)), fcgno.Problem(dev(k_te))
    t0 = time.time()
    r, e, ksys, it_exact = ptr.krylov_dataset(p_tr, dev(f_tr), dev(u0_tr), args.iters, m=m, e_scale=e_scale)
    torch.cuda.synchronize()
    t_data = time.time() - t0
    rh, eh, ksh, _ = ptr.krylov_dataset(p_te, dev(f_te), dev(u0_te), args.iters, m=m, e_scale=e_scale)
    tr = fcgno.Trainer(n, w, batch, sy.no_weights(w, 7 + args.seed),
                       loss=fcgno.LOSS_NOTAY if args.loss == "notay" else fcgno.LOSS_L2)
    kte = dev(k_te)

    def held_out_loss():
        ls = []
        for s0 in range(0, rh.shape[0], batch):
            perm = torch.arange(s0, min(s0 + batch, rh.shape[0]), dtype=torch.int32, device="cuda")
            ls.append(tr.loss_grad(kte, rh, eh, perm=perm, ksys=ksh, grad=False))
        return float(torch.cat(ls).mean())

    def fcg_counts(no, mm=None):
        res = fcgno.fcg_solve(p_te, dev(f_te), dev(u0_te), m=mm or m, tol=args.tol, maxit=args.maxit, no=no, history=False)
        it = res.iters.cpu().numpy()
        st = res.status.cpu().numpy()
        return dict(mean=float(it.mean()), median=float(np.median(it)), min=int(it.min()), max=int(it.max()),
                    converged=int((st == fcgno.CONVERGED).sum()), systems=int(st.size))

    random_no = fcgno.NeuralOperator(w, sy.no_weights(w, 7 + args.seed))
    before = dict(held_out_loss=held_out_loss(), fcg_no=fcg_counts(random_no))
    ident = fcg_counts(None)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    curve = ptr.train(tr, dev(k_tr), r, e, ksys, epochs=args.epochs, seed=args.seed, lr0=args.lr,
                      log=lambda ep, l: print(f"epoch {ep} loss {l:.4f}", file=sys.stderr) if ep % 10 == 0 else None)
    end.record()
    torch.cuda.synchronize()
    train_ms = start.elapsed_time(end)
    no = ptr.trained_operator(tr)
    after = dict(held_out_loss=held_out_loss(), fcg_no=fcg_counts(no))
    for mm in args.m_test:
        after[f"fcg_no_m{mm}"] = fcg_counts(no, mm)
        after[f"fcg_identity_m{mm}"] = fcg_counts(None, mm)
    if args.save:
        np.save(args.save, np.ascontiguousarray(tr.blob()))
    samples = int(r.shape[0])
    out = dict(
        what="SNO trained on the GPU (Fig. 3 scheme), FCG-NO on held-out systems vs FCG(I)",
        config=args.config, dataset=args.dataset, e_scale=e_scale, lr0=args.lr,
        n=n, width=w, m=m, tol=args.tol, maxit=args.maxit, loss=args.loss,
        train_systems=args.train_systems, test_systems=args.test_systems, sample_iters=args.iters,
        samples=samples, batch=batch, epochs=args.epochs, steps=int(tr.t.value),
        table6=dict(lr0=1e-3, decay="x0.5 / 50 epochs", weight_decay=1e-2),
        data_gen_s=t_data, train_ms=train_ms, ms_per_step=train_ms / max(1, tr.t.value),
        samples_per_s=samples * args.epochs / (train_ms / 1e3),
        loss_curve=[round(x, 5) for x in curve],
        before=before, after=after, fcg_identity=ident,
        exact_solve_iters_mean=float(it_exact.float().mean()),
        data="synthetic, seeded (see --dataset in the header)",
    )
    print(json.dumps(out))


if __name__ == "__main__":
    main()
