set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02a.log 2>&1; tail -15 gpurun_out/pytest_gpu_r02a.log
for w in smax3m smax2s3z smax27m mpe overcooked; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_r02a_$w.log 2>&1; tail -1 gpurun_out/bench_r02a_$w.log | cut -c1-600; done
bash scripts/prof_kernel.sh r02a smax3m step_kernel 30
bash scripts/prof_kernel.sh r02a smax27m step_kernel 30
