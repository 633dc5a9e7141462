"""Print the SHA-256 of the CPU-generated inputs of a config (host-independence check)."""
import hashlib
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
from synth import fields as S  # noqa: E402

for cfg in sys.argv[1:]:
    t = time.time()
    f, g, xi = S.make(cfg)
    print(cfg, hashlib.sha256(f.numpy().tobytes()).hexdigest()[:16],
          hashlib.sha256(g.numpy().tobytes()).hexdigest()[:16], f"{time.time() - t:.1f} s",
          flush=True)
