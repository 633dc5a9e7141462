"""ncu_quick.py from the exported CSVs (raw page, source page) of one capture."""
import csv
import sys
from collections import Counter

raw, src = sys.argv[1], sys.argv[2]
V = int(sys.argv[3]) if len(sys.argv) > 3 else 512 ** 3
rows = list(csv.reader(open(raw)))
h, u, d = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:70s} {d[i][:100]} {u[i]}")
rows = list(csv.reader(open(src)))
hh = rows[1]
ie, isrc = hh.index("Instructions Executed"), hh.index("Source")
op = Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    t = r[isrc].split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    op[o] += int(r[ie])
    tot += int(r[ie])
print(f"warp-instructions per 32 vertices: {tot / V * 32:.1f}")
print("  ".join(f"{o} {n / V * 32:.1f}" for o, n in op.most_common(30)))
