# compute-sanitizer over small corrections (SURVEY §4.3 layer 5): memcheck,
# racecheck (shared memory), synccheck, initcheck on C1, a 64^3 C2 crop, the
# 2D C4 crop, the sharded loopback and the Theorem 1 / edit-log entry points
out=gpurun_out/sanitize
mkdir -p $out
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from synth import fields as S
import paper_2604_01397_b200 as E
for cfg, shape in [("C1", None), ("C2", (64, 64, 64)), ("C4", (1, 120, 260))]:
    f, g, xi = S.make(cfg, shape=shape, device="cuda")
    c = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    r = E.exactz_correct(f, g, xi, edit_counts=c)
    log, n = E.exactz_edit_log(g, r.out, c, xi)
    E.exactz_edit_log_apply(log, g)
    E.exactz_vulnerability(f, g, xi)
    if f.dim() == 3 and f.shape[0] >= 4:
        E.exactz_correct_slabs(f, g, xi, 2)
    print(cfg, "status", r.status, "iters", r.iters)
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 100000 python /tmp/san_case.py > $out/$tool.log 2>&1
  echo "$tool: exit $? ; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/$tool.log | tail -1)"
done
