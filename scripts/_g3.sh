mkdir -p gpurun_out
T=${1:-r02i}
timeout 1500 python -m pytest tests/test_smax_lane.py tests/test_gpu_parity.py tests/test_smacv2.py tests/test_gpu_contract.py -q -x > gpurun_out/pytest_smax_$T.log 2>&1; tail -3 gpurun_out/pytest_smax_$T.log
for w in smax3m smax2s3z smax27m; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done
