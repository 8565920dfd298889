import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as orc, synthetic as sy
cfg = sy.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
mode = sys.argv[2] if len(sys.argv) > 2 else "oracle"
maxit = 6
k, f, blob = sy.make_k(cfg), sy.make_f(cfg), sy.make_weights(cfg)
w = cfg["width"]
if mode == "oracle":
    p = orc.unpack_weights(blob, w)
    for b in (0,):
        ref = orc.fcg(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), cfg["m"], cfg["tol"], maxit,
                      precond=lambda r: orc.no_forward(p, r, k[b]))
        print("oracle", b, ref["hist"].tolist())
        # perturbed oracle: 1e-6 relative noise on the NO output (fp32-like)
        rng = np.random.default_rng(0)
        pert = orc.fcg(lambda x: orc.apply_A(k[b], x), f[b], np.zeros_like(f[b]), cfg["m"], cfg["tol"], maxit,
                       precond=lambda r: orc.no_forward(p, r, k[b]) * (1 + 1e-6 * rng.standard_normal(r.shape)))
        print("pert1e-6", b, pert["hist"].tolist())
else:
    from paper_2402_05598_b200 import fcgno as F
    prob = F.Problem(torch.from_numpy(k).cuda())
    prec = F.FP64 if mode == "fp64" else F.FP32
    res = F.fcg_solve(prob, torch.from_numpy(f).cuda(), m=cfg["m"], tol=cfg["tol"], maxit=maxit,
                      no=F.NeuralOperator(w, blob, precision=prec))
    print(mode, os.environ.get("FCGNO_TC", "1"), res.history.cpu().numpy()[0].tolist())
