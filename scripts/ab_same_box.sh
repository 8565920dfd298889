# A/B on one box: the committed state in _ab_old/ (git worktree, built in place) vs the working tree
set -x
for r in 1 2; do
  (cd _ab_old && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split > ../gpurun_out/ab_old$r.json 2>&1)
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-split > gpurun_out/ab_new$r.json 2>&1
done
