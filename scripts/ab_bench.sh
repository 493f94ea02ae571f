#!/bin/bash
# Same-box A/B of a bench workload: ab_old/ (a snapshot of the package + bench.py built from another
# commit, git-ignored, shipped with the gpurun snapshot) against the working tree.
#   bash scripts/ab_bench.sh ppo        -> "<tree> ms_per_step update_ms" twice per tree
for i in 1 2; do
  for d in ab_old .; do
    (cd $d; export PYTHONPATH=$PWD; timeout 300 python bench.py --workload ${1:-ippo} --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['ms_per_step'], d.get('update_ms'))")
  done
done
