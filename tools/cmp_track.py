"""Dev bisect: tracked vs dense (NO_TRACK) runs, first differing per-pass row, per debug flag.

    python tools/cmp_track.py C3 [shape ...]     (shape like 128x128x128; none: full size)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
FLAGS = [(0, "default"), (0x80000, "no fpaths"), (0x200000, "fpaths always"),
         (0x100000, "no pipelining"), (0x200, "no cache"), (0x200 | 0x200000, "fp always, no cache"),
         (0x80000 | 0x100000, "no fp, no pipe")]
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
shapes = [tuple(int(x) for x in a.split("x")) if a else None for a in sys.argv[2:]] or [None]
for shape in shapes:
    f, g, xi = S.make(cfg, shape=shape, device="cuda")
    ref = E.exactz_correct(f, g, xi, flags=E.NO_TRACK, stats_cap=10000)
    for fl, name in FLAGS:
        r = E.exactz_correct(f, g, xi, flags=fl, stats_cap=10000)
        same = torch.equal(r.out.view(torch.int32), ref.out.view(torch.int32))
        first = next((k for k, (a, b) in enumerate(zip(r.stats, ref.stats)) if a != b), None)
        print(cfg, shape, f"{name:22s}", "iters", r.iters, ref.iters, "same", same, "first diff row",
              first, r.stats[first] if first is not None else "",
              ref.stats[first] if first is not None else "", flush=True)
    del f, g
    torch.cuda.empty_cache()
