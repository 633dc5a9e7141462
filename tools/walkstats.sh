# walk-length diagnostic: a -DEXACTZ_WALKSTATS build, C2/C3 per-pass walk steps, then the normal build back
set -x
B='import sys; sys.path.insert(0, "paper_2604_01397_b200"); import torch, _build; _build.build(True)'
EXACTZ_NVCC_EXTRA=-DEXACTZ_WALKSTATS python -c "$B"
python tools/walkstats.py ${CFGS:-C2 C3} > gpurun_out/walkstats.log 2>&1
python -c "$B"
