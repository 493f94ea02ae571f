#!/bin/bash
# Usage (under gpurun): bash scripts/profile.sh TAG "workload1 workload2 ..."
# Per workload: the launch list of a short bench run (ncu, per-launch device
# time) and one `ncu --set full` capture of the step kernel.  Outputs land in
# gpurun_out/; summaries worth keeping are copied to profiles/ by hand.
TAG=${1:-r01}
WLS=${2:-"smax3m mpe_large overcooked"}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
for w in $WLS; do
  timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_${TAG}_$w.csv python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/launches_${TAG}_$w.log 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 \
    -o gpurun_out/prof_${TAG}_$w -f python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/prof_${TAG}_$w.log 2>&1
done
ls -la gpurun_out
