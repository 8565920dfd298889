# A/B of the y-synthesis work-item width (FCGNO_YSYN_CH=2: N = 80, 4 CTAs/SM) on one box.
FCGNO_YSYN_CH=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "no_fp32 or tc_and_ffma or fcg_no_fp32 or opt_in" 2>&1 | tail -1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for r in 1 2; do
  for v in "" "FCGNO_YSYN_CH=2"; do
    out=$(env $v timeout 300 $B 2>/dev/null | tail -1)
    echo "[$v] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), d['step_ms'], d['time_split_ms_per_iter']['per_kernel']['k_yan+k_ysyn'])")"
  done
done
