"""Per-kernel totals and shares of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}.get(d.get("Metric Unit", ""), 1.0)
    k = d["Kernel Name"].split("(")[0][:72]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{k:72s} {n:6d} {v / 1e6:9.3f} ms {100 * v / tot:5.1f}%  {v / n / 1e3:9.1f} us/launch")
print(f"total {tot / 1e6:.3f} ms")
