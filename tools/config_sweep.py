"""Per-config timing + per-round violation profile (dev tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import fields as S
import paper_2604_01397_b200 as E

out = {}
for cfg in sys.argv[1:]:
    t = time.time()
    f, g, xi = S.make(cfg, device="cuda")
    torch.cuda.synchronize()
    gen = time.time() - t
    fl = int(os.environ.get("FLAGS", "0"), 0)
    r = E.exactz_correct(f, g, xi, stats_cap=100000, flags=fl)  # warm
    times = []
    for _ in range(3):  # unprofiled (the bench's path): min of 3
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        r = E.exactz_correct(f, g, xi, flags=fl, stats_cap=100000)
        s1.record(); torch.cuda.synchronize()
        times.append(s0.elapsed_time(s1))
    ms = min(times)
    r = E.exactz_correct(f, g, xi, flags=E.PROFILE | fl, stats_cap=100000)  # kernel classes
    V = f.numel()
    vt = [row[0] for row in r.stats]
    out[cfg] = dict(shape=list(f.shape), xi=xi, iters=r.iters, status=r.status, ms=ms,
                    GBps=4 * V / ms / 1e6, ms_setup=r.ms_setup, ms_loop=r.ms_loop,
                    vt_frac=[round(v / V, 6) for v in vt],
                    kernels={k: v for k, v in r.kernels.items() if v[1]}, gen_s=gen)
    print(cfg, json.dumps({k: out[cfg][k] for k in ("shape", "iters", "status", "ms", "GBps", "ms_setup", "ms_loop")}), flush=True)
    del f, g
    torch.cuda.empty_cache()
json.dump(out, open("gpurun_out/config_sweep.json", "w"), indent=1)
