"""Summarise ncu --set full captures: key counters per kernel, hot source lines."""
import csv, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'lts__t_sector_hit_rate.pct', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__occupancy_limit_registers', 'launch__grid_size', 'launch__block_size']


def raw(path):
    rows = list(csv.reader(open(path)))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index('Kernel Name')
    for r in data:
        print('----', r[ki][:100])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:60s} {r[i]} {units[i]}")


def source(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = [k for k, r in enumerate(rows) if 'Line No' in r][0]
    h = rows[hi]
    iW, iI = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
    lines = []
    for r in rows[hi + 1:]:
        if r and r[0] and len(r) > max(iW, iI):
            try:
                lines.append((int(r[iW] or 0), int(r[iI] or 0), r[0], r[1][:100]))
            except ValueError:
                pass
    tw = sum(l[0] for l in lines) or 1
    ti = sum(l[1] for l in lines) or 1
    print('total samples', tw, 'warp-instructions', ti)
    for l in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * l[0] / tw:5.1f}% samp {100 * l[1] / ti:5.1f}% inst  L{l[2]}: {l[3]}")


if __name__ == '__main__':
    (raw if sys.argv[1] == 'raw' else source)(sys.argv[2])
