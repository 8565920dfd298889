# A/B on one box: the committed state in _ab_old/ (git worktree, built in place) vs the working tree
set -x
for r in 1 2; do
  (cd _ab_old && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split > ../gpurun_out/ab_old$r.json 2>&1)
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split > gpurun_out/ab_new$r.json 2>&1
  for v in $EXTRA; do eval "$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split" > gpurun_out/ab_x$r.json 2>&1; done
done
for f in ab_old1 ab_new1 ab_x1 ab_old2 ab_new2 ab_x2; do [ -f gpurun_out/$f.json ] && python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,1), 'M e2e', round(d['e2e']['value']/1e6,1), d.get('step_ms'))"; done
