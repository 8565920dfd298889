#!/usr/bin/env python
"""Benchmark of the batched FCG-NO hot path on B200 (BASELINE.json metric and configs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

A step is one fcgno_fcg_solve over the whole batch of the largest single-GPU configuration,
configs[2] (config 3: 128x128 grid, batch 128, high-contrast lognormal k, FCG(m=10), tol 1e-6,
random-init SNO width 85 in fp32 with fp64 FCG vectors; the random-init NO does not converge, so
every step runs maxit = 2000 iterations).  value =
unknown-iterations/s = sum_b N*iters_b over all ranks / max-over-ranks device time.  Under
torchrun each rank solves its own batch of independent systems (weak scaling, no data-path
collective).  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched FCG-NO unknown-iterations/s on 1 B200; % of HBM roofline per iteration"
UNIT = "unknown-iterations/s"
K_MODES = 20
CONVERGE_MAXIT = {1: 500, 2: 5000, 3: 30000, 4: 30000, 5: 2000}   # SURVEY §8(d) D.2 identity maxit
FP32_ALU_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # SMs x FP32 lanes x FMA x max SM clock


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--maxit", type=int, default=None, help="override the config's maxit")
    ap.add_argument("--no-split", action="store_true", help="skip the instrumented time-split solve")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE configs[4] second half: isolated HBM bandwidth sweep of apply_A, the batched "
                         "dot and the FCG kernels at 1024^2 and 2048^2, batch 4 (one JSON line)")
    ap.add_argument("--sweep-n", type=int, nargs="*", default=[1024, 2048])
    ap.add_argument("--check-every", type=int, default=16, help="iterations per captured loop body")
    ap.add_argument("--vec32", action="store_true",
                    help="FCG vectors and ring stored in fp32 (BASELINE configs[2] variant, DESIGN.md R21)")
    ap.add_argument("--precond", choices=["no", "identity", "structured"], default="no",
                    help="no: the config's random-init SNO (the BASELINE workload, default); identity: FCG(I); "
                         "structured: the convergent structured SNO of SURVEY C.2 #30 (solves/s and iterations)")
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------- distributed plumbing
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def reduce_over_ranks(units: float, ms: float, backend_device=None):
    """(sum of units, max of ms) over all ranks; identity when not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return units, ms
    dev = backend_device or "cpu"
    u = torch.tensor([units], dtype=torch.float64, device=dev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(u.item()), float(t.item())


def shard_systems(batch: int, rank: int):
    """Weak scaling: rank r solves systems [r*B, (r+1)*B) of the seeded stream."""
    return list(range(rank * batch, (rank + 1) * batch))


# ----------------------------------------------------------------------------- workload model
def layer_flops(B, n, w, cin):
    """Algorithmic FLOPs of the GEMMs the tensor-core layer kernel itself performs for one SNO
    operator layer over the batch: bypass 2*cin*w*N, x-synthesis 4K*w*N and
    x-analysis 4K*w*N (the y-direction DFTs run in their own kernels and are not credited here)."""
    N = n * n
    return B * (2 * cin * w * N + 8 * K_MODES * w * N)


def layer_flops_ffma(B, n, w, cin):
    """FLOPs of one FFMA layer launch (k_no_layer also does the y-direction DFTs: 16K^2 w n)."""
    return layer_flops(B, n, w, cin) + B * 16 * K_MODES * K_MODES * w * n


def src_hash():
    """sha256 (16 hex) of the library sources: ties a stored ncu capture to the code it measured."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2402_05598_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh", ".h")):
            h.update(name.encode())
            h.update(open(os.path.join(csrc, name), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "fcgno.h"), "rb").read())
    return h.hexdigest()[:16]


def ncu_traffic(config, kernel):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full) of
    `kernel` at `config` from profiles/ncu_traffic.json, only when that capture was taken on these
    exact sources (src_sha16); otherwise (None, reason)."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(tpath))
    except (OSError, ValueError):
        return None, "no ncu capture on file"
    if d.get("src_sha16") != src_hash():
        return None, "ncu capture on file is from other sources (src_sha16 mismatch); not reported"
    v = d.get(f"config{config}", {}).get(kernel)
    return (v, d.get("source", "ncu")) if v is not None else (None, f"no capture of {kernel} at config {config}")


def layer_bytes(B, n, w):
    """Algorithmic HBM bytes of one SNO layer launch ("NO activations,
    materialised": 3 writes + 3 reads of w fp32 channels per FCG-NO iteration = 24 w B per unknown,
    i.e. 8 w B per unknown for each of the three layer launches)."""
    return 8 * w * B * n * n


def mean_window(m, iters):
    import synthetic  # noqa: F401
    tot = 0
    for i in range(iters):
        tot += min(i, max(1, i % (m + 1)))
    return tot / max(iters, 1)


def fcg_no_bytes_per_unknown(m_bar, w, S=8):
    """Algorithmic HBM bytes per unknown per FCG-NO iteration (fused-minimal
    FCG part with S-byte vectors, plus the NO's input/output and materialised fp32 activations
    v1..v3 written and read once)."""
    fcg = (9 + 2 * m_bar) * S + 8
    no = S + 8 + S + 6 * w * 4
    return fcg + no


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.proc = None
        self.gpu = gpu_index

    def start(self, settle_s: float = 15.0):
        """Start sampling and wait (bounded) for the first sample: NVML initialisation inside
        nvidia-smi briefly stalls the GPU and must not overlap a timed step."""
        if os.environ.get("BENCH_NO_SMI"):   # A/B of the sampler's own effect on step times
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < settle_s and self.proc.poll() is None:
            try:
                if sum(1 for _ in open(self.path)) >= 2:
                    break
            except OSError:
                pass
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1])); smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline (oracle)
def _oracle_worker(job):
    """One host process: the oracle as it stands (single-threaded numpy) on one system of the
    workload for `iters` FCG iterations.  Returns (unknown-iterations done, seconds)."""
    cfg, system, iters, precond = job
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle as orc
    import synthetic as sy
    with threadpool_limits(limits=1):
        k = sy.make_k(cfg, systems=[system])[0]
        f = sy.make_f(cfg, systems=[system])[0]
        blob = sy.make_weights(cfg) if precond == "no" else sy.structured_no_weights(cfg["width"], cfg["n"])
        params = orc.unpack_weights(blob, cfg["width"])
        P = None if precond == "identity" else (lambda r: orc.no_forward(params, r, k))
        t0 = time.perf_counter()
        res = orc.fcg(lambda x: orc.apply_A(k, x), f, np.zeros_like(f), cfg["m"], cfg["tol"], iters, precond=P)
        dt = time.perf_counter() - t0
    return cfg["n"] ** 2 * res["iters"], dt


def host_cpu_model():
    host = platform.processor() or platform.machine()
    try:
        host = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    return host


def cpu_oracle_rate(cfg, budget_s=12.0, max_iters=400, precond="no", procs=None, pool=None):
    """The oracle as it stands (fp64 NO, exact dots), parallel over systems only (SURVEY.md §8(d)
    D.5): P = min(B, host cores) single-threaded processes, process p running system p of the
    workload for ~budget_s.  value = all processes' unknown-iterations / the slowest process's time
    (they run concurrently).  Returns (unknown-iterations/s, processes, sample)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    P = max(1, min(cfg["batch"], cores if procs is None else procs))
    # calibrate the per-iteration cost on one system (3 iterations, this process)
    _, dt3 = _oracle_worker((cfg, 0, 3, precond))
    per_it = dt3 / 3
    iters = int(max(3, min(max_iters, budget_s / max(per_it, 1e-6))))
    jobs = [(cfg, b, iters, precond) for b in range(P)]
    if P == 1:
        results = [_oracle_worker(jobs[0])]
    elif pool is not None:
        results = pool.map(_oracle_worker, jobs, chunksize=1)
    else:
        with mp.get_context("spawn").Pool(P) as own:
            results = own.map(_oracle_worker, jobs, chunksize=1)
    units = sum(u for u, _ in results)
    wall = max(dt for _, dt in results)
    kind = {"no": "FCG-NO (fp64 NO, exact dots)", "identity": "FCG(I) (exact dots)",
            "structured": "FCG with the structured SNO (fp64, exact dots)"}[precond]
    done = units // (cfg["n"] ** 2)
    sample = (f"systems 0..{P - 1} of the workload, {iters} {kind} iterations each ({done} in total), "
              f"{P} single-threaded processes in parallel, slowest {wall:.1f} s, on {host_cpu_model()} "
              f"({cores} logical CPUs)")
    return units / wall, P, sample


def workload_config(args, cfg, world):
    """The `config` object of the JSON line (identical for both arms)."""
    return {"workload": f"config{args.config}", "precond": args.precond,
            "fcg_vectors": "fp32" if args.vec32 else "fp64", "n": cfg["n"], "batch": cfg["batch"], "m": cfg["m"],
            "tol": cfg["tol"], "maxit": cfg["maxit"], "no_width": cfg["width"], "no_precision": cfg["no_precision"],
            "k_field": cfg["k"], "rhs": cfg["rhs"], "l2": "flushed (256 MiB write) before every step",
            "parallelism": f"batch replicas x{world} (weak)"}


def bench_cfg(args):
    import synthetic as sy
    cfg = dict(sy.CONFIGS[args.config])
    if args.precond != "no":   # converging runs: the iteration cap of SURVEY D.2's identity column
        cfg["maxit"] = CONVERGE_MAXIT[args.config]
    if args.maxit:
        cfg["maxit"] = args.maxit
    return cfg


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synthetic as sy
    from paper_2402_05598_b200 import fcgno as F

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = bench_cfg(args)
    n, B, w, m = cfg["n"], cfg["batch"], cfg["width"], cfg["m"]
    N = n * n
    systems = shard_systems(B, rank)
    k = sy.make_k(cfg, systems=systems)
    f = sy.make_f(cfg, systems=systems)
    blob = sy.make_weights(cfg) if args.precond == "no" else sy.structured_no_weights(w, n)
    dk = torch.from_numpy(k).cuda()
    df = torch.from_numpy(f).cuda()
    prob = F.Problem(dk)
    no = None if args.precond == "identity" else \
        F.NeuralOperator(w, blob, precision=F.FP32 if cfg["no_precision"] == "fp32" else F.FP64)
    solver = F.Solver(prob, m, cfg["tol"], cfg["maxit"], no=no, history=False, vec_fp32=args.vec32,
                      check_every=args.check_every)
    u = torch.zeros_like(df)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    # clock sampler first: nvidia-smi's start-up stalls the GPU briefly, so it must land in the
    # warm-up, not in the first timed step (it keeps sampling through the timed region)
    sampler = ClockSampler(local)
    sampler.start()
    # at least W warm-up steps, continued (<= 12) until a step is within 3% of the fastest so far:
    # the first few solves of a process show sporadic 10-100% spikes (system warm-up), which
    # must not land in the K timed steps
    warm_ms = []

    def settled():   # the last two warm-up steps within 3% of the fastest so far
        return len(warm_ms) >= 2 and max(warm_ms[-2:]) <= 1.03 * min(warm_ms)
    while len(warm_ms) < args.warmup or (len(warm_ms) < 12 and not settled()):
        flush.zero_()            # warm-up repeats the timed step exactly (first touch of the flush buffer too)
        u.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solver.solve(df, u)
        e1.record()
        e1.synchronize()
        warm_ms.append(round(e0.elapsed_time(e1), 3))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    F.profile_reset()
    launches0 = F.kernel_launches()
    times, units = [], 0.0
    for _ in range(args.steps):
        flush.zero_()
        u.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solver.solve(df, u)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        units += float(N) * float(solver.iters.sum().item())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = F.kernel_launches() - launches0
    # dominant-kernel timing: a second timed pass of the same workload whose graphs carry CUDA
    # events around the layer launches of one sampled iteration per chunk (kept out of the pass
    # above: event nodes break programmatic-dependent-launch overlap and perturb the step time)
    # (converging runs: a prefix short enough that every system is still running, so the bytes of
    # every timed launch are known; identity: the dominant kernel is k_pform_stencil)
    prof_maxit = {"no": cfg["maxit"], "structured": min(cfg["maxit"], 48), "identity": min(cfg["maxit"], 132)}[args.precond]
    prof_every = 12 if args.precond == "identity" else 16
    psolver = F.Solver(prob, m, cfg["tol"], prof_maxit, no=no, history=False, check_every=prof_every,
                       profile_mask=1 << (F.PROF_STENCIL if no is None else F.PROF_NO_LAYER), vec_fp32=args.vec32)
    u.zero_()
    psolver.solve(df, u)
    F.profile_reset()
    prof_ms = 0.0
    for _ in range(1):
        flush.zero_()
        u.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        psolver.solve(df, u)
        e1.record()
        e1.synchronize()
        prof_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    prof = F.profile_read()
    local_ms = sum(times)
    tot_units, max_ms = reduce_over_ranks(units, local_ms, "cuda" if world > 1 else None)
    value = tot_units / (max_ms / 1e3)
    iters_step = float(solver.iters.float().mean().item())
    ms_per_iter = (local_ms / args.steps) / max(iters_step, 1)

    # dominant kernel: the SNO layer kernel (3 launches per iteration), timed in-graph
    layer_ms, layer_n = prof["k_no_layer"] if no is not None else prof["k_pform_stencil"]
    avg_layer_ms = layer_ms / max(layer_n, 1)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {"hbm_gbs": 6650.0}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tc_path = no is not None and F.no_uses_tensor_cores(prob, no)
    traffic, traffic_src = ncu_traffic(args.config, "k_px_layer" if tc_path else "k_no_layer")
    if no is None:
        # identity FCG: k_pform_stencil, (6 + m_i) 8 B per unknown at the sampled iterations (w = r;
        # 4 * 8 at i = 0), every system running
        samp = [(i, min(i, max(1, i % (m + 1)))) for i in range(0, prof_maxit, prof_every)]
        alg = sum(((6 + mi) * 8 if i else 32) for i, mi in samp) / len(samp) * B * N
        achieved = alg / (avg_layer_ms * 1e-3) / 1e9
        roofline = {"kernel": "k_pform_stencil", "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": None, "algorithmic_bytes_per_launch": alg,
                    "avg_launch_ms": avg_layer_ms, "launches_timed": layer_n,
                    "share_of_step": avg_layer_ms / ms_per_iter,
                    "timing": f"CUDA events inside the solve graphs, one sampled iteration per {prof_every} of a "
                              f"{prof_maxit}-iteration prefix (all systems running)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, measured on this pool)"}
    elif tc_path:
        # tcgen05 3xBF16 layer (k_px_layer): activations stream through HBM; the MMA work (3 split
        # passes, padding included) needs < 1/3 of the HBM time, so the bound is HBM.
        alg = layer_bytes(B, n, w)
        achieved = alg / (avg_layer_ms * 1e-3) / 1e9
        roofline = {"kernel": "k_px_layer", "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                    "algorithmic_bytes_per_launch": alg,
                    "bytes_definition": "SURVEY.md 8(d) D.3: 8 w B per unknown per layer launch (3 writes + 3 reads "
                                        "of w fp32 channels per iteration)",
                    "avg_launch_ms": avg_layer_ms, "launches_timed": layer_n,
                    "share_of_step": 3 * avg_layer_ms / ms_per_iter,
                    "timing": "CUDA events recorded inside the solve graphs around the layer launches of one sampled "
                              "iteration per 16, in a second timed pass of the same workload",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, measured on this pool)",
                    "useful_tflops": (layer_flops(B, n, w, 2) + 2 * layer_flops(B, n, w, w)) / 3 / (avg_layer_ms * 1e-3) / 1e12,
                    "useful_tflops_definition": "the layer kernel's own GEMMs (bypass, x-synthesis, x-analysis)"}
    else:
        flops_iter = layer_flops_ffma(B, n, w, 2) + 2 * layer_flops_ffma(B, n, w, w)
        avg_flops = flops_iter / 3
        achieved = avg_flops / (avg_layer_ms * 1e-3) / 1e12
        roofline = {"kernel": "k_no_layer", "bound": "alu", "achieved": achieved, "peak": FP32_ALU_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved / FP32_ALU_PEAK_TFLOPS, "traffic": traffic,
                    "flops_per_launch": avg_flops, "avg_launch_ms": avg_layer_ms, "launches_timed": layer_n,
                    "share_of_step": 3 * avg_layer_ms / ms_per_iter,
                    "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x 1965 MHz (FFMA path; DESIGN.md §6)"}

    # per-iteration HBM roofline (the metric's second half)
    m_bar = mean_window(m, int(max(iters_step, 1)))
    S = 4 if args.vec32 else 8
    if no is None:   # identity FCG, fused-minimal: (7 + 2 m̄) S + 8 B per unknown
        bytes_iter = ((7 + 2 * m_bar) * S + 8) * N * B
    else:
        bytes_iter = fcg_no_bytes_per_unknown(m_bar, w, S) * N * B
    hbm_frac = (bytes_iter / (hbm * 1e9)) / (ms_per_iter * 1e-3)

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None,
           "dtype": "f64" if no is None else "bf16x3 split (NO tensor cores, fp32 accumulate) + f64 (FCG vectors, dots)",
           "data": "synthetic (seeded; BASELINE configs recipe, " + {"no": "random-init NO weights)", "identity":
                   "identity preconditioner)", "structured": "structured SNO weights, SURVEY C.2 #30)"}[args.precond],
           "config": workload_config(args, cfg, world),
           "iterations_per_step": iters_step, "ms_per_iteration": ms_per_iter,
           "step_ms": [round(t, 3) for t in times], "warmup_ms": warm_ms,
           "hbm_roofline_per_iteration": {"algorithmic_bytes_per_iter": bytes_iter, "peak_gbs": hbm,
                                          "frac": hbm_frac},
           "roofline": roofline, "gpu_launches": int(launches), "clocks": clocks}
    if args.precond != "no":   # converging runs: solves/s and iteration counts
        it_host = solver.iters.cpu().numpy()
        st_host = solver.status.cpu().numpy()
        out["solves_per_s"] = B * world / (max_ms / args.steps / 1e3)
        # SURVEY D.1 "swept" variant: N * B * max_b(iters_b) / T, the work the kernels touch were
        # converged systems not skipped
        out["swept_unknown_iterations_per_s"] = N * B * world * float(it_host.max()) / (max_ms / args.steps / 1e3)
        out["iterations"] = {"mean": float(it_host.mean()), "min": int(it_host.min()), "max": int(it_host.max()),
                             "converged": int((st_host == F.CONVERGED).sum()), "of": int(B)}

    if not args.no_split and rank == 0:
        out["time_split_ms_per_iter"] = time_split(F, prob, no, cfg, df, vec32=args.vec32)
    if rank == 0:
        out["e2e"] = e2e_measure(F, no, cfg, k, f, min(args.steps, 3), args.vec32)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, procs, sample = cpu_oracle_rate(cfg, precond=args.precond)
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": procs, "threads_per_process": 1,
                               "kind": "oracle", "sample": sample}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def time_split(F, prob, no, cfg, df, iters=64, vec32=False):
    """Instrumented solve (every kernel class timed in-graph) -> ms per iteration per phase."""
    import torch
    s = F.Solver(prob, cfg["m"], cfg["tol"], iters, no=no, history=False, profile_mask=(1 << F.PROF_NCLASS) - 1,
                 vec_fp32=vec32)
    u = torch.zeros_like(df)
    s.solve(df, u)
    F.profile_reset()
    u.zero_()
    s.solve(df, u)
    torch.cuda.synchronize()
    prof = F.profile_read()
    it = max(prof.get("k_pform_stencil", (0.0, 0))[1], 1)   # sampled iterations (one stencil launch each)
    per = {name: ms / it for name, (ms, cnt) in prof.items() if cnt}
    stencil = per.get("k_pform_stencil", 0.0)
    no_ms = sum(per.get(x, 0.0) for x in ("k_no_layer", "k_mix", "k_no_out", "k_dft_rows+k_lift_mix", "k_yan+k_ysyn"))
    upd = sum(per.get(x, 0.0) for x in ("k_window_dots", "k_update"))
    return {"stencil": stencil, "no": no_ms, "fcg_update": upd, "per_kernel": per,
            "note": "CUDA events around every launch of the first unrolled iteration of each graph chunk "
                    "(instrumented run, 64 iterations; per sampled iteration)"}


def e2e_measure(F, no, cfg, k, f, steps, vec32=False):
    """Same metric through the host-buffer C-ABI entry point: H2D of k, f, u0 from pinned memory,
    assemble, solve, D2H of u, iters, status, all inside the timed region."""
    import numpy as np
    import torch
    n, B = cfg["n"], cfg["batch"]
    hs = F.HostSolver(n, B, cfg["m"], cfg["tol"], cfg["maxit"], no=no, vec_fp32=vec32)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    kh, fh = pin(k), pin(f)
    uh = torch.zeros((B, n, n), dtype=torch.float64).pin_memory().numpy()
    ih = torch.zeros(B, dtype=torch.int32).pin_memory().numpy()
    sh = torch.zeros(B, dtype=torch.int32).pin_memory().numpy()
    hs.solve(kh, fh, uh, ih, sh)   # warm-up
    torch.cuda.synchronize()
    tot_ms, units = 0.0, 0.0
    for _ in range(steps):
        uh[...] = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hs.solve(kh, fh, uh, ih, sh)
        e1.record()
        e1.synchronize()
        tot_ms += e0.elapsed_time(e1)
        units += float(n * n) * float(ih.sum())
    N = n * n
    return {"value": units / (tot_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 3 * B * N * 8,
            "d2h_bytes_per_step": B * N * 8 + 2 * 4 * B, "ms_per_step": tot_ms / steps,
            "steps": steps, "api": "fcgno_solve_host (pinned host buffers; includes assemble)"}


# ----------------------------------------------------------------------------- reference arm (oracle)
def run_reference(args):
    """Reference arm: the oracle as it stands on the host cores (there is no reference implementation:
    the reference is a paper).  Each of the W + K steps is a bounded sample of the workload (one
    oracle run per process over min(B, cores) systems, ~3 s); value = mean over the K timed steps."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    cfg = bench_cfg(args)
    P = max(1, min(cfg["batch"], os.cpu_count() or 1))
    rates, samples, walls = [], [], []
    with mp.get_context("spawn").Pool(P) as pool:
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            rate, procs, sample = cpu_oracle_rate(cfg, budget_s=3.0, max_iters=100, precond=args.precond, pool=pool)
            if step >= args.warmup:
                rates.append(rate); samples.append(sample); walls.append(time.perf_counter() - t0)
    value = statistics.mean(rates)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; BASELINE configs recipe, " + {"no": "random-init NO weights)", "identity":
                   "identity preconditioner)", "structured": "structured SNO weights, SURVEY C.2 #30)"}[args.precond],
           "config": workload_config(args, cfg, world),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "threads_per_process": 1, "kind": "oracle",
                            "sample": samples[-1]},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- bandwidth sweep
SWEEP_SEEDS = {1024: 110, 2048: 111}


def sweep_samples(m, check_every, maxit):
    """(i, m_i, m_{i+1}) of the iterations the in-graph profiler samples (the first of every graph
    chunk)."""
    sched = lambda i: min(i, max(1, i % (m + 1)))
    return [(i, sched(i), sched(i + 1)) for i in range(0, maxit, check_every)]


def run_sweep(args):
    """Isolated bandwidth sweep (BASELINE.json configs[4]: "apply_A and FCG-update kernels at
    1024x1024 and 2048x2048, batch 4"; SURVEY.md §8(d) D.3 sweep rows).

    * apply_A and the batched dot: S independent (k, x, y) sets whose total footprint is >= 3x the
      126 MB L2, cycled, so every launch reads its operands from HBM; R launches are captured in
      one CUDA graph and timed with events on the replay stream.
    * the FCG kernels (k_window_dots, k_pform_stencil, k_update): in place, inside an identity
      FCG(m=10) solve, timed with CUDA events the library records inside its graphs around the
      launches of one sampled iteration per chunk; check_every = 12 makes the sampled iterations'
      windows m_i cycle through 1, 2, ..., 10 like the run's own.
    Algorithmic bytes per unknown (fp64): apply_A 24 (x, k read; y written); dot 16;
    p-form + stencil (6 + m_i) 8 (w = r, m_i p_k, k, u read; u (lazy x update), p, s written;
    4 * 8 at i = 0); window dots (1 + m_i) 8; update 3 * 8 (r, s read; r written)."""
    import torch

    import synthetic as sy
    from paper_2402_05598_b200 import fcgno as F

    torch.cuda.set_device(0)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {"hbm_gbs": 6650.0}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    L2 = torch.cuda.get_device_properties(0).L2_cache_size
    B, m, ce = 4, 10, 12
    rows = []
    sampler = ClockSampler(0)
    sampler.start()
    for n in args.sweep_n:
        cfg = dict(n=n, batch=B, k="lognormal", length=0.1, variance=1.0, rhs="normal", seed=SWEEP_SEEDS.get(n, 112))
        k = torch.from_numpy(sy.make_k(cfg)).cuda()
        f = torch.from_numpy(sy.make_f(cfg)).cuda()
        N = n * n
        vec = B * N * 8
        S = max(2, -(-3 * L2 // (3 * vec)))
        sets = []
        for s in range(S):
            ks = k if s == 0 else k * (1.0 + 1e-3 * s)
            sets.append((F.Problem(ks), f.clone() if s else f, torch.empty_like(f)))
        dws = torch.empty(F._lib.fcgno_dot_workspace_bytes(sets[0][0].grid), dtype=torch.uint8, device="cuda")
        dout = torch.empty(B, dtype=torch.float64, device="cuda")

        def timed_graph(body, reps):
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                for t in range(3):
                    body(t)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for t in range(reps):
                        body(t)
                g.replay()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                best = None
                for _ in range(3):
                    e0.record(st)
                    g.replay()
                    e1.record(st)
                    e1.synchronize()
                    ms = e0.elapsed_time(e1) / reps
                    best = ms if best is None else min(best, ms)
            torch.cuda.synchronize()
            return best

        def apply_body(t):
            p, x, y = sets[t % S]
            F._check(F._lib.fcgno_apply_A(p._h, F._ptr(x), F._ptr(y), F._stream()))

        def dot_body(t):
            p, x, y = sets[t % S]
            F._check(F._lib.fcgno_batched_dot(p._h, F._ptr(x), F._ptr(f if t % S else k), F._ptr(dout), F._ptr(dws),
                                              dws.numel(), F._stream()))

        reps = 8 * S
        for name, body, bpu in (("apply_A", apply_body, 24), ("batched_dot", dot_body, 16)):
            ms = timed_graph(body, reps)
            gbs = bpu * B * N / (ms * 1e-3) / 1e9
            rows.append({"kernel": name, "n": n, "batch": B, "us_per_launch": ms * 1e3, "bytes_per_unknown": bpu,
                         "achieved_gbs": gbs, "frac": gbs / hbm})
        del sets
        # FCG kernels inside an identity solve
        maxit = ce * 22
        prob = F.Problem(k)
        mask = (1 << F.PROF_WINDOW) | (1 << F.PROF_STENCIL) | (1 << F.PROF_UPDATE)
        solver = F.Solver(prob, m, 1e-14, maxit, history=False, check_every=ce, profile_mask=mask)
        u = torch.zeros_like(f)
        solver.solve(f, u)
        F.profile_reset()
        u.zero_()
        solver.solve(f, u)
        torch.cuda.synchronize()
        prof = F.profile_read()
        samp = sweep_samples(m, ce, maxit)
        for name, per_it in (("k_window_dots", lambda i, mi, mi1: (1 + mi) * 8 if mi else 0),
                             ("k_pform_stencil", lambda i, mi, mi1: (6 + mi) * 8 if i else 4 * 8),
                             ("k_update", lambda i, mi, mi1: 3 * 8)):
            ms, cnt = prof.get(name, (0.0, 0))
            if not cnt:
                continue
            nb = sum(per_it(*x) for x in samp) * B * N
            gbs = nb / (ms * 1e-3) / 1e9
            rows.append({"kernel": name, "n": n, "batch": B, "us_per_launch": ms * 1e3 / cnt,
                         "bytes_per_unknown": nb / (B * N * cnt), "achieved_gbs": gbs, "frac": gbs / hbm,
                         "launches_timed": cnt, "context": "identity FCG(10) solve, in-graph events"})
        # whole identity iteration (no instrumentation)
        plain = F.Solver(prob, m, 1e-14, maxit, history=False, check_every=16)
        u.zero_()
        plain.solve(f, u)
        it_ms = float("inf")
        for _ in range(3):   # best of three solves (a single solve is one sample of a shared box)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            u.zero_()
            e0.record()
            plain.solve(f, u)
            e1.record()
            e1.synchronize()
            it_ms = min(it_ms, e0.elapsed_time(e1) / maxit)
        m_bar = mean_window(m, maxit)
        bpu = (10 + 2 * m_bar) * 8   # window (1 + m_i) 8 + p-form (6 + m_i) 8 + update 3 * 8
        gbs = bpu * B * N / (it_ms * 1e-3) / 1e9
        rows.append({"kernel": "identity FCG iteration", "n": n, "batch": B, "us_per_iteration": it_ms * 1e3,
                     "bytes_per_unknown": bpu, "achieved_gbs": gbs, "frac": gbs / hbm,
                     "unknown_iterations_per_s": B * N / (it_ms * 1e-3)})
        del prob, solver, plain
        torch.cuda.empty_cache()
    clocks = sampler.stop()
    print(json.dumps({"metric": "HBM bandwidth of the stencil / reduction / FCG kernels (fraction of measured peak)",
                      "unit": "GB/s", "peak_gbs": hbm, "l2_bytes": L2, "sweep": rows, "clocks": clocks,
                      "data": "synthetic (seeded lognormal k, N(0,1) f)"}), flush=True)


def main(argv=None):
    args = parse_args(argv)
    if args.sweep:
        run_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
