"""Dev diagnostic: steepest-descent / ascent path lengths of a config's g
(torch on the GPU; SoS ties ignored, statistics only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
f, g, xi = S.make(cfg, device="cuda")
nz, ny, nx = g.shape
V = g.numel()
# Freudenthal neighbours of the Kuhn triangulation: +-(1,0,0) +-(0,1,0) +-(0,0,1)
# +-(1,1,0) +-(0,1,1) +-(1,0,1) +-(1,1,1) in (x,y,z) with the same sign
offs = []
for b in range(1, 8):
    d = (b & 1, (b >> 1) & 1, b >> 2)
    offs += [d, tuple(-v for v in d)]
idx = torch.arange(V, device="cuda", dtype=torch.int64).view(nz, ny, nx)
for up in (False, True):
    best_v = g.clone()
    best_i = idx.clone()
    for dx, dy, dz in offs:
        sv = torch.full_like(g, float("inf") if not up else -float("inf"))
        si = idx.clone()
        zs = slice(max(dz, 0), nz + min(dz, 0)); zd = slice(max(-dz, 0), nz + min(-dz, 0))
        ys = slice(max(dy, 0), ny + min(dy, 0)); yd = slice(max(-dy, 0), ny + min(-dy, 0))
        xs = slice(max(dx, 0), nx + min(dx, 0)); xd = slice(max(-dx, 0), nx + min(-dx, 0))
        sv[zd, yd, xd] = g[zs, ys, xs]
        si[zd, yd, xd] = idx[zs, ys, xs]
        take = sv > best_v if up else sv < best_v
        best_v = torch.where(take, sv, best_v)
        best_i = torch.where(take, si, best_i)
    ptr = best_i.view(-1)
    dist = (ptr != idx.view(-1)).to(torch.int32)
    for _ in range(14):
        dist = dist + dist[ptr]
        ptr = ptr[ptr]
    q = torch.quantile(dist[::97].float(), torch.tensor([0.5, 0.9, 0.99, 0.999], device="cuda"))
    print(cfg, "up" if up else "dn", "mean", dist.float().mean().item(), "max", dist.max().item(),
          "q50/90/99/99.9", [round(v, 1) for v in q.tolist()], flush=True)
    del ptr, dist, best_v, best_i
