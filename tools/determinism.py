"""Repeat a full-size correction and compare every run bit for bit (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
flags = [int(x, 0) for x in sys.argv[3:]] or [0]
f, g, xi = S.make(cfg, device="cuda")
ref = None
for k in range(reps):
    for fl in flags:
        c = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
        r = E.exactz_correct(f, g, xi, flags=fl, stats_cap=1000, edit_counts=c)
        key = (r.out.view(torch.int32).clone(), c.clone(), r.stats, r.iters)
        if ref is None:
            ref = key
            continue
        same = (torch.equal(key[0], ref[0]) and torch.equal(key[1], ref[1]) and key[2] == ref[2]
                and key[3] == ref[3])
        nd = int((key[0] != ref[0]).sum())
        diffpass = next((i for i, (a, b) in enumerate(zip(key[2], ref[2])) if a != b), None)
        print(f"{cfg} rep {k} flags {fl:#x}: same {same} diff-vertices {nd} first-diff-pass {diffpass}"
              f" counts-equal {torch.equal(key[1], ref[1])}", flush=True)
        if diffpass is not None:
            print("   ", key[2][diffpass], "\n   ", ref[2][diffpass], flush=True)
