"""N-sweep knob study (SURVEY 8(f) unranked; the paper's N study).

For each config and each N (steps of Delta = xi / N before the lossless clamp,
P:178): iterations, the Theorem 1 bound (N + 1) * D_max,
correction time (CUDA events, best of 2 after a warm call), the fraction of
vertices edited (c > 0) and stored losslessly (c == N + 1).  One JSON object
on stdout.

  python tools/n_sweep.py [C2 C4 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_01397_b200 as E  # noqa: E402
from synth import fields as S  # noqa: E402

NS = [1, 2, 3, 5, 8, 12, 20]
out = {}
for cfg in sys.argv[1:] or ["C2", "C4"]:
    f, g, xi = S.make(cfg, device="cuda")
    V = f.numel()
    dmax = E.exactz_vulnerability(f, g, xi)["D_max"]
    c = torch.empty(V, dtype=torch.uint8, device="cuda")
    rows = []
    for N in NS:
        E.exactz_correct(f, g, xi, N=N)  # warm
        best = None
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = E.exactz_correct(f, g, xi, N=N, edit_counts=c)
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        edited = int((c > 0).sum().item())
        lossless = int((c == N + 1).sum().item())
        rows.append({"N": N, "iters": r.iters, "status": r.status,
                     "bound_(N+1)Dmax": (N + 1) * dmax, "ms": best,
                     "GBps": 4 * V / best / 1e6, "edit_pct": 100.0 * edited / V,
                     "lossless_pct": 100.0 * lossless / V})
        print(cfg, rows[-1], file=sys.stderr, flush=True)
    out[cfg] = {"shape": list(f.shape), "xi": xi, "D_max": dmax, "rows": rows}
    del f, g, c
    torch.cuda.empty_cache()
print(json.dumps(out))
