"""Summarise an ncu --set full report: key counters and the dynamic opcode mix per vertex.

    python tools/ncu_quick.py gpurun_out/x.ncu-rep [V]"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
V = int(sys.argv[2]) if len(sys.argv) > 2 else 512 ** 3
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, d = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]
for w in want:
    for i, n in enumerate(h):
        if n == w:
            print(f"{w:70s} {d[i]} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ie, isrc = hh.index("Instructions Executed"), hh.index("Source")
ist = hh.index("Warp Stall Sampling (All Samples)")
op, st = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    t = r[isrc].split()
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.split(".")[0]
    op[o] += int(r[ie])
    st[o] += int(r[ist] or 0)
    tot += int(r[ie])
print(f"warp-instructions per 32 vertices: {tot / V * 32:.1f}")
print("  ".join(f"{o} {n / V * 32:.1f}" for o, n in op.most_common(30)))
print("stall samples by opcode:", "  ".join(f"{o} {n}" for o, n in st.most_common(12)))
