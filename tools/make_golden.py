"""Write a full-size golden of the CPU oracle: tests/golden/fullsize_<cfg>.json.

    python tools/make_golden.py C4            # minutes
    python tools/make_golden.py C2            # ~2 h, one core

Calls only oracle/ (the checker) and synth/ (the seeded input generator, no
method arithmetic).  Nothing here touches the CUDA path: every stored value is
the oracle's.  The input is generated on the CPU with one torch thread
(synth.fields._one_thread), so its bytes depend on the seed only; their
SHA-256 is stored and the GPU test (tests/test_gpu_golden.py) asserts it
before comparing.  Outputs are stored as SHA-256 digests of the raw
little-endian arrays (out float32, edit counts uint8, label_min / label_max
int32), plus per-chunk digests (2^22 elements) so a mismatch can be located,
the per-pass counters verbatim, `iters`, the status and the oracle's
wall time with host, core count and date (the cpu_baseline's provenance,
SURVEY §8(d) "Caching").
"""
import datetime
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from synth import fields as S  # noqa: E402

CHUNK = 1 << 22


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def chunks(a: np.ndarray) -> list:
    a = np.ascontiguousarray(a).reshape(-1)
    return [hashlib.sha256(a[i:i + CHUNK].tobytes()).hexdigest()[:16]
            for i in range(0, a.size, CHUNK)]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main(cfg: str, flags: int = 0):
    t0 = time.time()
    f, g, xi = S.make(cfg)
    tg = time.time() - t0
    fn, gn = f.numpy(), g.numpy()
    nx, ny, nz = (list(reversed(fn.shape)) + [1, 1])[:3]
    rec = dict(config=cfg, workload=S.CONFIGS[cfg]["name"], dims=[nx, ny, nz],
               V=int(fn.size), xi=float(xi), xi_hex=np.float32(xi).view(np.uint32).item(),
               N=5, flags=flags, sha_f=sha(fn), sha_ghat=sha(gn),
               lo_monotone=S.lo_monotone(f, xi), gen_s=round(tg, 1))
    print(json.dumps(rec), flush=True)
    O.build()
    t0 = time.perf_counter()
    r = O.correct(fn, gn, xi, dims=(nx, ny, nz), flags=flags, stats_cap=100000)
    dt = time.perf_counter() - t0
    rec.update(status=r.status, iters=r.iters,
               sha_out=sha(r.out), sha_counts=sha(r.counts),
               sha_label_min=sha(r.label_min), sha_label_max=sha(r.label_max),
               chunks_out=chunks(r.out), chunks_counts=chunks(r.counts),
               chunks_label_min=chunks(r.label_min), chunks_label_max=chunks(r.label_max),
               stats=r.stats.tolist(),
               edited=int((r.counts > 0).sum()), lossless=int((r.counts == 6).sum()),
               oracle_s=round(dt, 2), oracle_threads=1, host_cpu=cpu_model(),
               host_nproc=os.cpu_count(), date=datetime.datetime.now(datetime.timezone.utc).isoformat(),
               oracle_src_sha=hashlib.sha256(open(O.SRC, "rb").read()).hexdigest())
    suffix = "" if flags == 0 else f"_flags{flags}"
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{cfg}{suffix}.json")
    with open(path + ".tmp", "w") as fh:
        json.dump(rec, fh, indent=1)
    os.replace(path + ".tmp", path)
    print(f"{cfg}: status {r.status} iters {r.iters} oracle {dt:.1f} s -> {path}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
