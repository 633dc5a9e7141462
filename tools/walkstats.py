"""Dev diagnostic: C3 walk steps per pass (needs a build with -DEXACTZ_WALKSTATS:
EXACTZ_NVCC_EXTRA=-DEXACTZ_WALKSTATS python -c 'from paper_2604_01397_b200 import _build; _build.build(True)'
— the k_events / k_events_cached grid-stride walks count their steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
for cfg in sys.argv[1:]:
    f, g, xi = S.make(cfg, device="cuda")
    r = E.exactz_correct(f, g, xi, flags=E.PROFILE, stats_cap=100000)
    print(cfg, "iters", r.iters, "events ms", r.kernels["events"][0], flush=True)
    st = r.stats
    for k, row in enumerate(st):
        w, links = r.walk_steps[k], r.pass_links[k]
        print(f"  round {k:2d} Vt {row[0]:10d} links {links:10d} walk_steps {w:12d} "
              f"steps/link {w / max(links, 1):8.2f}", flush=True)
    del f, g; torch.cuda.empty_cache()
