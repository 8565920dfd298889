# Device-side WHILE-graph loop (default) vs the host-polled chunk loop (FCGNO_HOSTLOOP=1), 10 steps.
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-split"
for r in 1 2; do
  for v in "" "FCGNO_HOSTLOOP=1"; do
    out=$(env $v timeout 300 $B 2>/dev/null | tail -1)
    echo "[$v] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), d['warmup_ms'], d['step_ms'])")"
  done
done
