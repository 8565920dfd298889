# Evidence for profiles/r02 in one GPU call: default bench line, its ncu launch list, one --set full capture of
# the layer kernels (3 launches = one NO apply), the bandwidth sweep, the other workloads, training runs.
set -x
mkdir -p gpurun_out/ev gpurun_out/ev/matrix
timeout 600 python bench.py > gpurun_out/ev/bench_c3_default.json 2> gpurun_out/ev/bench_c3_default.err; echo bench rc=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/ref_c3.json 2> gpurun_out/ev/ref_c3.err; echo ref rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev/launches.csv python bench.py --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_px_layer --launch-skip 3 --launch-count 3 -f -o gpurun_out/ev/px_layer_full python bench.py --steps 1 --warmup 3 --maxit 30 --no-split --no-cpu-baseline > gpurun_out/ev/ncu_full.log 2>&1; echo full rc=$?
timeout 400 python bench.py --sweep > gpurun_out/ev/sweep.json 2> gpurun_out/ev/sweep.err; echo sweep rc=$?
run() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/ev/matrix/$name.json 2> gpurun_out/ev/matrix/$name.err; echo "$name rc=$?"; }
run c1_no --config 1 --steps 3
run c1_identity --config 1 --precond identity --steps 3
run c2_no --config 2 --steps 3
run c2_identity --config 2 --precond identity --steps 3
run c2_structured --config 2 --precond structured --steps 3
run c3_vec32 --config 3 --steps 2 --maxit 400 --vec32
run c3_identity --config 3 --precond identity --steps 2
run c4_no --config 4 --steps 2 --maxit 200
run c5_no --config 5 --steps 2 --maxit 200
timeout 600 python scripts/train_sno.py --config 2 --dataset diffusion --epochs 150 --train-systems 128 --test-systems 32 > gpurun_out/ev/train_c2_diffusion.json 2> gpurun_out/ev/train_c2_diffusion.err; echo train2 rc=$?
