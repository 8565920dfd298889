#!/usr/bin/env python
"""Theorem-1 diagnostics along an FCG run (Fig. 2/4 style):
for i = 0..I, eps_i = ||B(r_i) - e_i||_A / ||e_i||_A and the energy error ||e_i||_A, with
e_i = u* - u_i, r_i = f - A u_i (so A e_i = r_i), u* from FCG(I) to 1e-13, u_i the iterate after
i iterations of the solve (every quantity through the library's kernels; fcgno.notay_ratio).

  python scripts/notay_curve.py [--config 1] [--iters 60] > profiles/r01_notay_curve.json
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic as sy  # noqa: E402
from paper_2402_05598_b200 import fcgno as F  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters", type=int, default=60)
    args = ap.parse_args()
    cfg = sy.CONFIGS[args.config]
    n, m = cfg["n"], cfg["m"]
    systems = [0]
    k = torch.from_numpy(sy.make_k(cfg, systems=systems)).cuda()
    f = torch.from_numpy(sy.make_f(cfg, systems=systems)).cuda()
    prob = F.Problem(k)
    ustar = F.fcg_solve(prob, f, m=m, tol=1e-13, maxit=20000).u
    out = {"config": args.config, "n": n, "m": m, "curves": {}}
    precs = {"identity": None,
             "structured_no": F.NeuralOperator(cfg["width"], sy.structured_no_weights(cfg["width"], n),
                                               F.FP64 if cfg["no_precision"] == "fp64" else F.FP32),
             "random_no": F.NeuralOperator(cfg["width"], sy.make_weights(cfg),
                                           F.FP64 if cfg["no_precision"] == "fp64" else F.FP32)}
    for name, no in precs.items():
        eps, eps_opt, err, res = [], [], [], []
        for i in range(args.iters + 1):
            r_ = F.fcg_solve(prob, f, m=m, tol=0.0, maxit=i, no=no)
            u = r_.u
            r = f - prob.apply_A(u)
            e = ustar - u
            errA = torch.sqrt(prob.dot(e, prob.apply_A(e)))
            if float(errA[0]) == 0.0:
                break
            eps.append(float(F.notay_ratio(prob, r, e, no)[0]))
            eps_opt.append(float(F.notay_ratio(prob, r, e, no, optimal_scale=True)[0]))
            err.append(float(errA[0]))
            res.append(float(r_.history[0, i]) if r_.history is not None else None)
        out["curves"][name] = {"eps": eps, "eps_optimal_scale": eps_opt, "energy_error": err, "rel_residual": res}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
