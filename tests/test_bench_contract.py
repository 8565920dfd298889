"""bench.py's JSON line (the driver's contract): one short run on the GPU, every required key
present and consistent (value = units / device time, roofline fraction = achieved / peak, the
oracle baseline and the end-to-end number reported, launches counted)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3",
                          "--maxit", "32"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["steps"] == 2 and d["warmup"] >= 3 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "config3" and d["scaling"] == "weak"   # the largest single-GPU config
    cfg_units = 128 * 128 * 128 * 32 * 2                   # B * N * iterations * steps
    assert abs(d["value"] - cfg_units / (d["ms_per_step"] * 2 / 1e3)) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0.0 < r["frac"] < 1.0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0


def test_reference_arm_contract():
    # --impl reference times the oracle on the host (no GPU needed) and prints the same metric
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "unknown-iterations/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["value"] == d["value"]
    # same workload description as our arm (the driver compares the two lines' configs)
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse_args([])
    assert d["config"] == bench.workload_config(args, bench.bench_cfg(args), 1)
