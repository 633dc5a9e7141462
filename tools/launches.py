"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '')[:70]
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1e-6)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1]:10.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  {v[1] / v[0] * 1e3:9.1f} us/launch  {k}")
print(f"total {tot:.3f} ms")
