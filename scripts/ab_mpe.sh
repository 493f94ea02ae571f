# same-box A/B of the MPE step at 4M envs: the default build vs MARL_NVCC_EXTRA="$1"
for v in base alt base alt; do
  if [ $v = alt ]; then MARL_NVCC_EXTRA="$1" python -c "from paper_2311_10090_b200 import build as b; b.build()"; else python -c "from paper_2311_10090_b200 import build as b; b.build()"; fi
  for w in mpe_large overcooked; do
    echo -n "$v $w: "; timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
  done
done
