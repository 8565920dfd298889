"""Debug: tensor-core NO layer path vs the oracle (and vs the FFMA path) on small cases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as orc, synthetic as sy
from paper_2402_05598_b200 import fcgno as F

cases = [(64, 2, 48), (64, 2, 32), (128, 2, 85), (128, 2, 48), (64, 3, 8)]
for n, B, w in cases:
    k = sy.lognormal_k(n, B, 0.1, 1.0, 5); r = sy.normal_field(n, B, 6); blob = sy.no_weights(w, 7)
    prob = F.Problem(torch.from_numpy(k).cuda())
    no = F.NeuralOperator(w, blob, precision=F.FP32)
    t0 = time.time()
    got = no.apply(prob, torch.from_numpy(r).cuda()).cpu().numpy()
    torch.cuda.synchronize()
    p = orc.unpack_weights(blob, w)
    errs = [float(np.linalg.norm(got[b] - orc.no_forward(p, r[b], k[b])) / np.linalg.norm(orc.no_forward(p, r[b], k[b]))) for b in range(B)]
    print(f"n={n} B={B} w={w} rel_l2={max(errs):.3e} ({time.time()-t0:.2f}s)", flush=True)
