"""Dev A/B of an env knob inside one process-pair-free loop: alternating settings, REPS
timed corrections each (min and median).  The knob is read once per process by the
library, so each setting runs in its own subprocess; rounds alternate the order.

    python tools/ab_knob.py EXACTZ_FP_GATE 0 0.15 --cfg C2 --rounds 3"""
import argparse
import os
import statistics
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("knob")
ap.add_argument("values", nargs="+")
ap.add_argument("--cfg", default="C2")
ap.add_argument("--rounds", type=int, default=3)
a = ap.parse_args()
here = os.path.dirname(os.path.abspath(__file__))
res = {v: [] for v in a.values}
for r in range(a.rounds):
    order = a.values if r % 2 == 0 else list(reversed(a.values))
    for v in order:
        env = dict(os.environ, **{a.knob: v, "REPS": "4"})
        out = subprocess.run([sys.executable, os.path.join(here, "quick_time.py"), a.cfg],
                             env=env, capture_output=True, text=True).stdout
        ms = [float(l.split(" ms ")[1].split()[0]) for l in out.splitlines() if l.startswith("rep ")][1:]
        res[v] += ms
for v in a.values:
    print(f"{a.knob}={v} {a.cfg}: min {min(res[v]):.2f} median {statistics.median(res[v]):.2f} ms "
          f"({len(res[v])} runs)", flush=True)
