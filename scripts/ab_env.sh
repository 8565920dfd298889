# Same-box A/B of environment knobs: $VARIANTS (space-separated VAR=value, "-" = default), 2 rounds.
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split"
for r in 1 2; do
  for v in $VARIANTS; do
    if [ "$v" = "-" ]; then out=$(timeout 300 $B 2>/dev/null | tail -1); else out=$(env $v timeout 300 $B 2>/dev/null | tail -1); fi
    echo "[$v] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), d['step_ms'])")"
  done
done
