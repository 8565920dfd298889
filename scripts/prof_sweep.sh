# ncu --set full captures of the FCG streaming kernels at the sweep size (n=2048, batch 4).
set -x
N=${N:-2048}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_A -c 1 -f -o gpurun_out/sw_apply python bench.py --sweep --sweep-n $N > gpurun_out/sw_apply.log 2>&1; echo rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dot -c 1 -f -o gpurun_out/sw_dot python bench.py --sweep --sweep-n $N > gpurun_out/sw_dot.log 2>&1; echo rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_window_dots|k_pform_stencil|k_update" --launch-skip 30 -c 6 -f -o gpurun_out/sw_fcg python bench.py --sweep --sweep-n $N > gpurun_out/sw_fcg.log 2>&1; echo rc=$?
