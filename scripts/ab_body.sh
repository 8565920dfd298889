# A/B of the captured loop-body length (check_every) on one box.
for r in 1 2; do
  for ce in 8 16 32 64; do
    out=$(timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split --check-every $ce 2>/dev/null | tail -1)
    echo "[ce=$ce] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), d['step_ms'])")"
  done
done
