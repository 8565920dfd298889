"""Pipeline timeline of the tensor-core layer kernel (CTA 0): FCGNO_PX_TRACE=<layer> events per tile,
in microseconds from the first event (clock64 at the SM clock).  python scripts/px_trace.py --config 3 --layer 2"""
import argparse
import ctypes
import os
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--layer", type=int, default=2)
ap.add_argument("--child", action="store_true")
args = ap.parse_args()
if not args.child:
    env = dict(os.environ, FCGNO_PX_TRACE=str(args.layer))
    sys.exit(subprocess.call([sys.executable, __file__, "--config", str(args.config), "--layer", str(args.layer),
                              "--child"], env=env))
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as sy  # noqa: E402
from paper_2402_05598_b200 import fcgno as F  # noqa: E402
cfg = sy.CONFIGS[args.config]
k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
prob = F.Problem(torch.from_numpy(k).cuda())
no = F.NeuralOperator(cfg["width"], blob, precision=F.FP32)
r = torch.from_numpy(f).cuda()
for _ in range(3):
    no.apply(prob, r)
torch.cuda.synchronize()
EV = 34
buf = np.zeros(64 * EV, dtype=np.uint64)
F._check(F._lib.fcgno_debug_px_trace(buf.ctypes.data_as(ctypes.c_void_p), 64 * EV))
full = buf.reshape(64, EV).astype(np.float64)
t = full[:, :10]
t0 = t[0, 0]
mhz = 1965.0
names = ["ld_issue", "mma_full", "d1_commit", "e1_start", "e1g0_done", "mma3", "e1_pre", "e2_done", "xa_vfull",
         "xa_d2empty"]
print("tile " + " ".join(f"{n:>10s}" for n in names))
for i in range(24):
    print(f"{i:4d} " + " ".join(f"{(v - t0) / mhz:10.2f}" if v else f"{'-':>10s}" for v in t[i]))
print("epilogue-1 warps (warp 4 + w): start / done per tile, us")
for i in range(16, 24):
    print(f"{i:4d} " + " ".join(f"{(full[i, 10 + 2 * w] - t0) / mhz:6.2f}/{(full[i, 11 + 2 * w] - t0) / mhz:6.2f}" for w in range(12)))
d = np.diff(t[4:40, 2]) / mhz
print("per-tile period (d1_commit), us: median", float(np.median(d)))
