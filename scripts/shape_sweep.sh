for sh in 0 4 5; do echo "shape $sh"; MARL_SMAX_SHAPE=$sh timeout 300 python bench.py --workload smax3m --steps 30 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"; done
MARL_SMAX_SHAPE=5 timeout 300 python -m pytest tests -m gpu -q -x -k "smax and 5m_vs_6m" 2>&1 | tail -2
