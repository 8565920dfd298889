# usage: bash scripts/prof_kernel.sh <kernel-regex> <out-name> [launch-skip] [count]
set -x
timeout 300 python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/small.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip ${3:-6} --launch-count ${4:-1} -f -o gpurun_out/$2 python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/ncu_$2.log 2>&1; echo ncu rc=$?
