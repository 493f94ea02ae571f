"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel (+ grid)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
gi = h.index('Grid Size') if 'Grid Size' in h else None
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    v = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(r[ui], 1.0) * v
    agg[r[ki].split('(')[0][-50:] + (" grid=" + r[gi] if gi is not None else "")].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print("%-75s n=%5d mean=%9.1f us total=%5.1f%%" % (k, len(v), sum(v) / len(v), 100 * sum(v) / tot))
