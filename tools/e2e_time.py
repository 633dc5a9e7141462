import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
f, g, xi = S.make("C2", device="cuda")
fh, gh = f.cpu().pin_memory(), g.cpu().pin_memory()
oh = torch.empty_like(gh).pin_memory()
ref = E.exactz_correct(f, g, xi).out.cpu()
for rep in range(4):
    torch.cuda.synchronize(); t = time.time()
    r = E.exactz_correct_host(fh, gh, xi, out=oh)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"rep {rep} e2e ms {dt*1e3:.1f} GB/s {4*f.numel()/dt/1e9:.2f} equal {torch.equal(oh.view(torch.int32), ref.view(torch.int32))}", flush=True)
