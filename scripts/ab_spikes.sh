# Step-time spikes: default bench vs the nvidia-smi sampler disabled, 10 timed steps each.
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-split"
for r in 1 2; do
  for v in "" "BENCH_NO_SMI=1"; do
    out=$(env $v timeout 300 $B 2>/dev/null | tail -1)
    echo "[$v] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), d['warmup_ms'], d['step_ms'])")"
  done
done
