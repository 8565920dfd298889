# Bench lines beyond the default: converging runs (identity / structured SNO), configs 1, 3-5, fp32 vectors.
mkdir -p gpurun_out/matrix
run() { name=$1; shift; timeout 600 python bench.py "$@" > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err; echo "$name rc=$?"; }
run c1_no --config 1 --steps 3
run c1_identity --config 1 --precond identity --steps 3
run c2_identity --config 2 --precond identity --steps 3
run c2_identity_vec32 --config 2 --precond identity --vec32 --steps 3
run c2_structured --config 2 --precond structured --steps 3
run c3_no --config 3 --steps 2 --maxit 400
run c3_vec32 --config 3 --steps 2 --maxit 400 --vec32
run c4_no --config 4 --steps 2 --maxit 64 --no-split
run c5_no --config 5 --steps 2 --maxit 64 --no-split
