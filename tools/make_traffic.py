"""profiles/traffic.json from the ncu --set full CSVs of tools/prof_traffic.sh.

    python tools/make_traffic.py gpurun_out/prof "<source note>"

For each captured kernel: DRAM bytes per launch (dram__bytes_read.sum +
dram__bytes_write.sum), time, issued warp-instructions and the issue-active
percentage; for the dense stencil also the algorithmic bytes of the launch
(8.25 B per vertex) and warp-instructions per 32 vertices.
bench.py reads the file for `roofline.traffic` and `roofline.issue`.
Entries of kernels not captured this time are kept from the previous file."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
V = 512 ** 3
KEYS = {"stencil": "k_stencil", "events": "k_events", "list": "k_stencil_sparse", "fclean": "k_fclean",
        "edit": "k_edit", "order": "k_saddle_order"}


def raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    h, u, d = rows[0], rows[1], rows[2]

    def g(k):
        i = h.index(k)
        return float(d[i].replace(",", "")) * SCALE.get(u[i], 1.0)
    return {"kernel": d[h.index("Kernel Name")].split("(")[0].replace("void ", ""),
            "gpu_time_ms": g("gpu__time_duration.sum"),
            "bytes_per_launch": g("dram__bytes_read.sum") + g("dram__bytes_write.sum"),
            "dram_read": g("dram__bytes_read.sum"), "dram_write": g("dram__bytes_write.sum"),
            "warp_instr": g("smsp__inst_executed.sum"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active")}


def main(d, note):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        out = json.load(open(path))
    except Exception:
        out = {}
    for name, key in KEYS.items():
        p = os.path.join(d, f"{name}_raw.csv")
        r = raw(p) if os.path.exists(p) else None
        if r is None:
            continue
        r["source"] = note
        if name == "stencil":
            r["algorithmic_bytes_per_launch"] = 8.25 * V
            r["warp_instr_per_32_vertices"] = r["warp_instr"] / V * 32
        out[key] = r
    out["source"] = "per entry (ncu --set full of one launch, C2 512^3 via tools/one_case.py)"
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu --set full")
