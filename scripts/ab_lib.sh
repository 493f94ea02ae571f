# A/B: the in-tree library vs paper_2311_10090_b200/_lib/alt/libmarl_b200.so on the given workloads
for w in $1; do
  echo "A $w"; timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
  echo "B $w"; MARL_B200_LIB=paper_2311_10090_b200/_lib/alt/libmarl_b200.so timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done
