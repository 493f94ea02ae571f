#!/bin/bash
# One ncu --set full capture of one kernel of one bench workload (under gpurun):
#   bash scripts/prof_kernel.sh TAG WORKLOAD KERNEL_REGEX [SKIP] [extra bench args]
TAG=$1; W=$2; K=$3; S=${4:-4}; shift 4
mkdir -p gpurun_out
timeout ${PTO:-900} /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
  -o gpurun_out/prof_${TAG}_$W -f python bench.py --workload $W --steps 3 --warmup 3 --no-e2e --no-cpu "$@" \
  > gpurun_out/prof_${TAG}_$W.log 2>&1
echo "prof $W rc=$?"; tail -2 gpurun_out/prof_${TAG}_$W.log
