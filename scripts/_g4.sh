mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_contract.py -q -x > gpurun_out/pytest_contract.log 2>&1; tail -3 gpurun_out/pytest_contract.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02k.log 2>&1; tail -1 gpurun_out/bench_r02k.log
