import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
f, g, xi = S.make(sys.argv[1] if len(sys.argv) > 1 else "C2", device="cuda")
r = E.exactz_correct_slabs(f, g, xi, int(sys.argv[2]) if len(sys.argv) > 2 else 8)
print("iters", r.iters)
