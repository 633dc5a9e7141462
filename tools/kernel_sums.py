"""Sum an ncu launch list (gpu__time_duration.sum CSV) over this library's
kernels and CUB's (the input generator's torch / cuFFT kernels excluded):
the GPU-busy time of a correction, without launch gaps or host waits.

    python tools/kernel_sums.py launches.csv [divisor]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}
tot = 0.0
n = 0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki]
    if not (name.startswith('exz::') or 'exz::' in name[:40] or 'cub::' in name[:40]):
        continue
    tot += float(r[vi].replace(',', '')) * scale.get(r[ui], 1e-6)
    n += 1
p = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"{sys.argv[1]}: {n} launches, {tot:.1f} ms of kernels, {tot / p:.1f} ms per rank (/{p:g})")
