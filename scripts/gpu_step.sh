#!/bin/bash
# Ad-hoc GPU session (under gpurun): selected tests, bench lines, one ncu capture.
#   TESTS="tests/a.py tests/b.py" BENCH="mpe:--steps 1000 smax27m" PROF="smax27m:step_kernel:30" bash scripts/gpu_step.sh TAG
T=${1:-adhoc}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$TESTS" ]; then
  timeout ${TTO:-1500} python -m pytest $TESTS -m gpu -q -x > gpurun_out/pytest_$T.log 2>&1; tail -4 gpurun_out/pytest_$T.log
fi
for b in $BENCH; do
  w=${b%%:*}; extra=""; [[ $b == *:* ]] && extra=${b#*:}; extra=${extra//,/ }
  timeout 600 python bench.py --workload $w --warmup 5 --no-cpu $extra 2>/dev/null | grep '^{' >> gpurun_out/bench_$T.jsonl
  tail -1 gpurun_out/bench_$T.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], '%.3g'%d['value'], d['roofline']['frac'] if d.get('roofline') else '', (d.get('e2e') or {}).get('value'))"
done
for p in $PROF; do
  IFS=: read w k s <<< "$p"
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$k -s ${s:-4} -c 1 \
    -o gpurun_out/prof_${T}_$w -f python bench.py --workload $w --steps 3 --warmup ${s:-4} --no-e2e --no-cpu > gpurun_out/prof_${T}_$w.log 2>&1
  echo "prof $w rc=$?"
done
