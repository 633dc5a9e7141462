import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
shape = tuple(int(x) for x in sys.argv[2].split("x")) if len(sys.argv) > 2 and sys.argv[2] else None
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
f, g, xi = S.make(cfg, shape=shape, device="cuda")
r = E.exactz_correct(f, g, xi, flags=flags, stats_cap=1000)
print("status", r.status, "iters", r.iters)
