set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash scripts/prof_kernel.sh r02a smax3m step_kernel 4
bash scripts/prof_kernel.sh r02a smax27m step_kernel 4
bash scripts/prof_kernel.sh r02a ippo policy_tc 200 --n-envs 1048576
for w in smax3m smax2s3z smax27m mpe overcooked; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_r02a_$w.log 2>&1; tail -1 gpurun_out/bench_r02a_$w.log | cut -c1-400; done
