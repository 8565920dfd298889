mkdir -p gpurun_out/matrix
run() { name=$1; shift; timeout 600 python bench.py "$@" > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err; echo "$name rc=$?"; }
run c1_no --config 1 --steps 3
run c4_no --config 4 --steps 2 --maxit 64
run c5_no --config 5 --steps 2 --maxit 64
