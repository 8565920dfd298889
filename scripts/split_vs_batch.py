"""Instrumented per-kernel time per iteration vs batch size (config-2 geometry)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic as sy
import paper_2402_05598_b200.fcgno as F

cfg = dict(sy.CONFIGS[2]); cfg["maxit"] = 64
blob = sy.make_weights(cfg)
rows = {}
Bs = [int(x) for x in (sys.argv[1:] or ["8", "64"])]
for B in Bs:
    systems = list(range(B))
    k = torch.from_numpy(sy.make_k(cfg, systems=systems)).cuda()
    f = torch.from_numpy(sy.make_f(cfg, systems=systems)).cuda()
    prob = F.Problem(k)
    no = F.NeuralOperator(cfg["width"], blob, precision=F.FP32)
    s = F.Solver(prob, cfg["m"], cfg["tol"], cfg["maxit"], no=no, history=False, profile_mask=(1 << F.PROF_NCLASS) - 1)
    u = torch.zeros_like(f)
    s.solve(f, u); torch.cuda.synchronize()
    F.profile_reset(); u.zero_(); s.solve(f, u); torch.cuda.synchronize()
    for name, (ms, cnt) in F.profile_read().items():
        if cnt:
            rows.setdefault(name, {})[B] = (ms * 1e3 / cfg["maxit"], cnt // cfg["maxit"])
print("kernel".ljust(26) + "".join(f"B={B:<5d}(us/it,launches)  " for B in Bs))
for name, d in rows.items():
    print(name.ljust(26) + "".join(f"{d.get(B, (0, 0))[0]:8.1f} x{d.get(B, (0, 0))[1]:<3d}             " for B in Bs))
