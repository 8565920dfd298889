set -x
for ln in 1 2; do FCGNO_LANES=$ln timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_l$ln.json 2> gpurun_out/ab_l$ln.err; echo "lanes=$ln rc=$?"; done
FCGNO_LANES=1 python scripts/batch_scaling.py 32 64 128
FCGNO_LANES=2 python scripts/batch_scaling.py 32 64 128
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
