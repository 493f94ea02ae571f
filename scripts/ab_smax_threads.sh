# same-box A/B of the SMAX lane-group kernel's block size: default build vs MARL_NVCC_EXTRA="$1"
mkdir -p gpurun_out
for v in new old new old; do
  if [ $v = old ]; then MARL_NVCC_EXTRA="$1" python -c "from paper_2311_10090_b200 import build as b; b.build()"; else python -c "from paper_2311_10090_b200 import build as b; b.build()"; fi
  for w in "smax27m --steps 20" "smax27m --n-envs 16384 --steps 10"; do
    echo -n "$v $w: "; timeout 300 python bench.py --workload $w --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])"
  done
done
