# one full-set ncu capture of every kernel of ~1 FCG-NO iteration (config 2), after a clean run
set -x
timeout 300 python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/small.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --launch-skip 400 --launch-count 24 -f -o gpurun_out/prof_iter python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/ncu_iter.log 2>&1; echo ncu rc=$?
