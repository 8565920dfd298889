# A/B of persisting-L2 windows for the NO blobs (FCGNO_L2P_MB / FCGNO_L2P_WIN), same box.
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split"
for r in 1 2; do
  for v in "" "FCGNO_L2P_MB=40 FCGNO_L2P_WIN=v" "FCGNO_L2P_MB=80 FCGNO_L2P_WIN=v" "FCGNO_L2P_MB=120 FCGNO_L2P_WIN=v" "FCGNO_L2P_MB=80 FCGNO_L2P_WIN=vgt"; do
    out=$(env $v timeout 300 $B 2>gpurun_out/ab_l2.err | tail -1)
    echo "[$v] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), d['step_ms'])")"
    grep "L2 persist" gpurun_out/ab_l2.err | head -1
  done
done
