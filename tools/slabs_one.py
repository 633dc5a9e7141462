"""One loopback-sharded correction (ncu launch lists): python tools/slabs_one.py C2 8"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
f, g, xi = S.make(cfg, device="cuda")
r = E.exactz_correct_slabs(f, g, xi, p)
torch.cuda.synchronize()
print("status", r.status, "iters", r.iters)
