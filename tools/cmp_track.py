import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
for cfg, shape in [("C1", None), ("C4", (1, 300, 700)), ("C2", (40, 48, 200))]:
    f, g, xi = S.make(cfg, shape=shape, device="cuda")
    ref = E.exactz_correct(f, g, xi, flags=E.NO_TRACK, stats_cap=10000)
    refr = E.exactz_correct(f, g, xi, flags=E.NO_TRACK | E.REFORMULATED, stats_cap=10000)
    for fl, name in [(0x200, "act only"), (0x100, "cache only"), (0, "both"), (0x10, "reform")]:
        r = E.exactz_correct(f, g, xi, flags=fl, stats_cap=10000)
        if fl == 0x10: ref_, ref = ref, refr
        same = torch.equal(r.out.view(torch.int32), ref.out.view(torch.int32))
        first = next((k for k, (a, b) in enumerate(zip(r.stats, ref.stats)) if a != b), None)
        print(cfg, name, "status", r.status, ref.status, "iters", r.iters, ref.iters, "same", same,
              "first diff row", first, r.stats[first] if first is not None else "",
              ref.stats[first] if first is not None else "")
        if fl == 0x10: ref = ref_
