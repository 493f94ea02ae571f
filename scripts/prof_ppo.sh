#!/bin/bash
# Per-kernel launch list of one PPO update at 2^16 envs (ncu, serialised); optional full capture of the branch kernel.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
N=${N:-65536}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ppo_launches.csv \
    python scripts/ppo_time.py $N 128 bf16 > gpurun_out/ppo_ncu_run.log 2>&1
if [ -n "$FULL" ]; then
  ncu --set full --clock-control none --import-source on -k regex:ppo_update_tc -s 2 -c 1 \
      -o gpurun_out/ppo_branch_full -f python scripts/ppo_time.py $N 128 bf16 > gpurun_out/ppo_full_run.log 2>&1
fi
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/ppo_launches.csv")))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    name = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    v = v * {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(v for _, v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{k:60s} n={n:5d} total_us={v:12.1f} share={v/tot:6.3f}")
PY
