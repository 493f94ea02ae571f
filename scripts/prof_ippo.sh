#!/bin/bash
# ncu for the IPPO rollout: launch list of one window + a full capture of the tcgen05 policy kernel.
TAG=${1:-r01}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}_ippo.csv python bench.py --workload ippo --steps 1 --warmup 3 --no-cpu \
  > gpurun_out/launches_${TAG}_ippo.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:policy_tc_kernel -s 300 -c 1 \
  -o gpurun_out/prof_${TAG}_ippo -f python bench.py --workload ippo --steps 1 --warmup 3 --no-cpu \
  > gpurun_out/prof_${TAG}_ippo.log 2>&1
tail -2 gpurun_out/prof_${TAG}_ippo.log
