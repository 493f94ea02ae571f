#!/bin/bash
# One ncu --set full capture of the step kernel of one workload: bash scripts/prof_one.sh TAG WORKLOAD [extra bench args]
TAG=$1; W=$2; shift 2
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:step_kernel -s ${SKIP:-4} -c 1 \
  -o gpurun_out/prof_${TAG}_$W -f python bench.py --workload $W --steps 3 --warmup ${WARM:-3} --no-e2e --no-cpu "$@" \
  > gpurun_out/prof_${TAG}_$W.log 2>&1
tail -2 gpurun_out/prof_${TAG}_$W.log
