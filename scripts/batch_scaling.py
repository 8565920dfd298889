"""Per-iteration time of the FCG-NO solve vs batch size (config-2 geometry), to see how much of
the step is latency (fixed per launch) rather than throughput."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic as sy
import paper_2402_05598_b200.fcgno as F

cfg = dict(sy.CONFIGS[2]); cfg["maxit"] = 200
blob = sy.make_weights(cfg)
for B in [int(x) for x in (sys.argv[1:] or ["16", "32", "64", "128"])]:
    systems = list(range(B))
    k = torch.from_numpy(sy.make_k(cfg, systems=systems)).cuda()
    f = torch.from_numpy(sy.make_f(cfg, systems=systems)).cuda()
    prob = F.Problem(k)
    no = F.NeuralOperator(cfg["width"], blob, precision=F.FP32)
    s = F.Solver(prob, cfg["m"], cfg["tol"], cfg["maxit"], no=no, history=False)
    u = torch.zeros_like(f)
    for _ in range(2):
        u.zero_(); s.solve(f, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    u.zero_(); e0.record(); s.solve(f, u); e1.record(); e1.synchronize()
    it = float(s.iters.float().mean())
    ms = e0.elapsed_time(e1) / it
    print(f"B={B:4d} ms/iter={ms:.4f} us/system-iter={ms*1e3/B:.2f}", flush=True)
