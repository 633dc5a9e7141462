"""Dev timing of the sharded algorithm on one GPU (loopback transport), with
a bit-for-bit comparison against the single-GPU call (out, iters, status).

python tools/slabs_time.py C2 1 2 8   ->  one line per slab count; the
per-rank figure is total / p (the loopback runs every rank's kernels and
its collectives on this GPU, one after another)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
f, g, xi = S.make(cfg, device="cuda")
r0 = E.exactz_correct(f, g, xi)
torch.cuda.synchronize()
t = time.time()
r0 = E.exactz_correct(f, g, xi)
torch.cuda.synchronize()
t1 = 1e3 * (time.time() - t)
print(f"{cfg} single: {t1:.1f} ms iters {r0.iters}", flush=True)
ref = r0.out.view(torch.int32).clone()
del r0
for ns in [int(x) for x in sys.argv[2:]] or [1, 2, 8]:
    E.exactz_correct_slabs(f, g, xi, ns)
    torch.cuda.synchronize()
    t = time.time()
    r = E.exactz_correct_slabs(f, g, xi, ns)
    torch.cuda.synchronize()
    ms = 1e3 * (time.time() - t)
    same = bool(torch.equal(r.out.view(torch.int32), ref))
    print(f"{cfg} slabs {ns}: {ms:.1f} ms total, {ms / ns:.1f} ms per rank ({t1 / (ms / ns):.2f}x the single call) "
          f"iters {r.iters} status {r.status} bit-equal {same}", flush=True)
    del r
