"""Per-launch timeline of one correction from an ncu launch-list CSV."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
seq = []
for r in data:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ', '').replace('exz::', '')
    if not (name.startswith('k_') or 'cub' in name): continue
    seq.append((name[:40], float(r[vi].replace(',', '')) * scale.get(r[ui], 1e-3)))
# group into rounds: a round starts at each k_stencil*
rnd, cur = [], None
for n, t in seq:
    if n.startswith('k_stencil'):
        cur = collections.OrderedDict(); rnd.append(cur)
    if cur is not None:
        cur[n] = cur.get(n, 0) + t
for i, r in enumerate(rnd):
    print(f"round {i:2d} total {sum(r.values()):8.1f} us  " + "  ".join(f"{k.replace('k_','')}={v:.0f}" for k, v in r.items()))
