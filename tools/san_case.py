"""Small corrections for compute-sanitizer (tools/sanitize.sh): every entry point and the
tracking / clean-path / cache / pipelining variants on C1, C2 / C3 crops and a 2D C4 crop."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E

for cfg, shape in [("C1", None), ("C2", (64, 64, 64)), ("C3", (40, 48, 96)), ("C4", (1, 120, 260))]:
    f, g, xi = S.make(cfg, shape=shape, device="cuda")
    c = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    for fl in (0, 0x200000, 0x200000 | 0x200, 0x100000, E.NO_TRACK):  # forced clean-path test, no cache, no pipelining
        r = E.exactz_correct(f, g, xi, edit_counts=c, flags=fl)
    log, n = E.exactz_edit_log(g, r.out, c, xi)
    E.exactz_edit_log_apply(log, g)
    E.exactz_vulnerability(f, g, xi)
    if f.dim() == 3 and f.shape[0] >= 4:
        E.exactz_correct_slabs(f, g, xi, 2)
    E.exactz_correct_host(f.cpu().pin_memory(), g.cpu().pin_memory(), xi)
    print(cfg, "status", r.status, "iters", r.iters, flush=True)
