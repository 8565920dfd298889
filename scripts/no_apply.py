"""Repeated standalone NO applications (fcgno_apply_NO) at a BASELINE config: the workload for ncu
captures of the NO kernels (profiles/).  python scripts/no_apply.py --config 3 --reps 3"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as sy  # noqa: E402
from paper_2402_05598_b200 import fcgno as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = sy.CONFIGS[args.config]
k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
prob = F.Problem(torch.from_numpy(k).cuda())
no = F.NeuralOperator(cfg["width"], blob, precision=F.FP32)
r = torch.from_numpy(f).cuda()
for _ in range(args.reps):
    w = no.apply(prob, r)
torch.cuda.synchronize()
print("ok", F.no_uses_tensor_cores(prob, no), float(w.abs().sum()))
