"""Dev repro: exactz_correct_host on a C3 crop with debug flags (argv)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
flags = int(sys.argv[1], 0) if len(sys.argv) > 1 else 0
cfg = sys.argv[2] if len(sys.argv) > 2 else "C3"
shape = tuple(int(x) for x in sys.argv[3].split("x")) if len(sys.argv) > 3 else (24, 19, 66)
f, g, xi = S.make(cfg, shape=shape)
c = torch.empty(f.numel(), dtype=torch.uint8).pin_memory()
try:
    r = E.exactz_correct_host(f.pin_memory(), g.pin_memory(), xi, edit_counts=c, flags=flags)
    print("host flags", hex(flags), "status", r.status, "iters", r.iters, flush=True)
except Exception as e:
    print("host flags", hex(flags), "FAILED", e, flush=True)
