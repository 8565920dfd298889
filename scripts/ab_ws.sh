set -x
for ws in 0 1; do FCGNO_TC_WS=$ws timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_ws$ws.json 2> gpurun_out/ab_ws$ws.err; echo "ws=$ws rc=$?"; done
timeout 300 python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/small.json 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tc_layer_ws --launch-skip 6 --launch-count 2 -f -o gpurun_out/prof_ws1 python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/ncu_ws.log 2>&1; echo ncu rc=$?
