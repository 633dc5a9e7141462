"""Dev timing of the sharded algorithm on one GPU (loopback transport)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
f, g, xi = S.make(cfg, device="cuda")
for ns in [int(x) for x in sys.argv[2:]] or [1, 2, 8]:
    E.exactz_correct_slabs(f, g, xi, ns)
    torch.cuda.synchronize()
    t = time.time()
    r = E.exactz_correct_slabs(f, g, xi, ns)
    torch.cuda.synchronize()
    print(f"{cfg} slabs {ns}: {1e3 * (time.time() - t):.1f} ms iters {r.iters} status {r.status}", flush=True)
r0 = E.exactz_correct(f, g, xi)
torch.cuda.synchronize()
t = time.time()
r0 = E.exactz_correct(f, g, xi)
torch.cuda.synchronize()
print(f"{cfg} single: {1e3 * (time.time() - t):.1f} ms")
