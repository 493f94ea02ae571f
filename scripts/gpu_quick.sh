#!/bin/bash
# Quick GPU iteration: gpu tests (+ optional -k filter) then bench lines for the given workloads.
# usage: bash scripts/gpu_quick.sh "<pytest -k expr or empty>" "smax3m overcooked ..."
K=${1:-}
WLS=${2:-smax3m}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for w in $WLS; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_$w.log 2>&1
  python - "$w" <<'PY'
import json,sys
w=sys.argv[1]
for l in open(f"gpurun_out/bench_{w}.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]
        print(w, "value %.4g" % d["value"], "ms %.4f" % d["ms_per_step"], "frac %.3f" % r["frac"],
              "GB/s %.0f" % r["achieved"], "e2e %.4g" % (d["e2e"] or {}).get("value", 0), "clk", d["clocks"])
        break
else:
    print(w, "FAILED"); print(open(f"gpurun_out/bench_{w}.log").read()[-2000:])
PY
done
