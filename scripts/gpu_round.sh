# One GPU call: GPU suite, sweep, default bench (5 steps), ncu of the sweep's FCG kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --sweep > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo sweep rc=$?
timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
[ -n "$NCU" ] && N=2048 bash scripts/prof_sweep.sh > gpurun_out/prof_sweep.log 2>&1
true
