"""Key metrics of every launch in an `ncu --page raw --csv` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "lts__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "launch__grid_size", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for d in rows[2:]:
    for w in want:
        if w in h:
            i = h.index(w)
            print(f"{w:78s} {d[i][:90]} {u[i]}")
    print()
