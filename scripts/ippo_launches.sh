TAG=${1:-x}
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv \
  --log-file gpurun_out/launches_${TAG}_ippo.csv python bench.py --workload ippo --n-envs 262144 --steps 1 --warmup 3 --no-cpu --no-e2e \
  > gpurun_out/launches_${TAG}_ippo.log 2>&1
