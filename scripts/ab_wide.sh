# same-box A/B of the wide-row policy kernel's threads per row: default build vs MARL_NVCC_EXTRA="$1"
for v in new old new old; do
  if [ $v = old ]; then MARL_NVCC_EXTRA="$1" python -c "from paper_2311_10090_b200 import build as b; b.build()" > /dev/null 2>&1; else python -c "from paper_2311_10090_b200 import build as b; b.build()" > /dev/null 2>&1; fi
  echo -n "$v ippo_oc: "; python bench.py --workload ippo_oc --steps 5 --warmup 2 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])"
done
