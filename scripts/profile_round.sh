# Evidence for profiles/: the default bench line, the launch list of the same command under ncu,
# and one --set full capture of the dominant kernel (3 launches = one NO apply).
set -x
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_px_layer --launch-skip 3 --launch-count 3 -f -o gpurun_out/px_layer_full python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
