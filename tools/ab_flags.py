"""Dev A/B of exactz_correct debug flags in one process (interleaved reps).

    python tools/ab_flags.py C2 0 0x2000      # key stencil vs previous dense stencil

Prints per variant: min wall ms over reps, iters, and the PROFILE kernel-class
split of one extra profiled run; checks the variants are bit-equal."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_01397_b200 as E  # noqa: E402
from synth import fields as S  # noqa: E402

cfg = sys.argv[1]
variants = [int(v, 0) for v in sys.argv[2:]] or [0]
shape = tuple(int(x) for x in os.environ["SHAPE"].split("x")) if os.environ.get("SHAPE") else None
f, g, xi = S.make(cfg, device="cuda", shape=shape)
reps = int(os.environ.get("REPS", "4"))
best = {v: 1e30 for v in variants}
outs = {}
for rep in range(reps):
    for v in variants:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = E.exactz_correct(f, g, xi, flags=v)
        b.record()
        torch.cuda.synchronize()
        best[v] = min(best[v], a.elapsed_time(b))
        outs[v] = (r.iters, r.out)
base = variants[0]
for v in variants:
    p = E.exactz_correct(f, g, xi, flags=v | E.PROFILE, stats_cap=1000)
    same = outs[v][0] == outs[base][0] and torch.equal(outs[v][1].view(torch.int32),
                                                       outs[base][1].view(torch.int32))
    ks = " ".join(f"{k}={ms:.2f}/{n}" for k, (ms, n, _) in p.kernels.items() if n)
    print(f"{cfg} flags {v:#x}: best {best[v]:.2f} ms  iters {outs[v][0]}  same_as_{base:#x} {same}"
          f"  setup {p.ms_setup:.2f} loop {p.ms_loop:.2f}  {ks}", flush=True)
