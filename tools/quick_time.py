"""Dev timing of exactz_correct on a config (not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
shape = tuple(int(x) for x in sys.argv[2].split("x")) if len(sys.argv) > 2 else None
t = time.time()
f, g, xi = S.make(cfg, device="cuda", shape=shape)
torch.cuda.synchronize()
print(cfg, tuple(f.shape), "xi", xi, "gen s", round(time.time() - t, 2), flush=True)
for rep in range(int(os.environ.get("REPS", "3"))):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    r = E.exactz_correct(f, g, xi, stats_cap=10000, flags=int(os.environ.get("QT_FLAGS", "0"), 0))
    s1.record(); torch.cuda.synchronize()
    ms = s0.elapsed_time(s1)
    spans = sum(r.pass_ms) if getattr(r, "pass_ms", None) else float("nan")
    print(f"rep {rep} status {r.status} iters {r.iters} ms {ms:.2f} setup {r.ms_setup:.2f} loop {r.ms_loop:.2f} "
          f"pass spans {spans:.2f} (gaps {r.ms_loop - spans:.2f}) GB/s {4*f.numel()/ms/1e6:.2f}", flush=True)
print("first rows", r.stats[:3])
print("last rows", r.stats[-3:])
