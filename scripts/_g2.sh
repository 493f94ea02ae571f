mkdir -p gpurun_out
T=${1:-r02c}
timeout 900 python -m pytest tests/test_smax_lane.py tests/test_gpu_parity.py -q -x -k "SMAX or smax" > gpurun_out/pytest_lane.log 2>&1; tail -3 gpurun_out/pytest_lane.log
timeout 300 python bench.py --workload smax3m --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-250
PTO=300 bash scripts/prof_kernel.sh $T smax3m lane_step 30 --warmup 40
