import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
for cfg in sys.argv[1:]:
    f, g, xi = S.make(cfg, device="cuda")
    r = E.exactz_correct(f, g, xi, flags=E.PROFILE, stats_cap=100000)
    print(cfg, "iters", r.iters, "events ms", r.kernels["events"][0])
    for k, (row, w) in enumerate(zip(r.stats, r.walk_steps)):
        print(f"  round {k:2d} Vt {row[0]:10d} walk_steps {w:12d}")
    del f, g; torch.cuda.empty_cache()
