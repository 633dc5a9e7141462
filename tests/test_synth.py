"""Input generators (synth/): counter-based noise, exact bound, determinism."""
import numpy as np
import torch

from synth import fields as S


def test_splitmix64_reference_vector():
    # splitmix64 with state 0: first output 0xE220A8397B1DCDAF (Vigna's reference)
    z = S.splitmix64(torch.tensor([0], dtype=torch.int64))
    assert int(z[0]) & ((1 << 64) - 1) == 0xE220A8397B1DCDAF


def test_uniform_range_and_counter_based():
    u = S.uniform_pm1(100000, seed=3)
    assert float(u.min()) >= -1.0 and float(u.max()) < 1.0 and abs(float(u.mean())) < 0.01
    v = S.uniform_pm1(10, seed=3, start=500)
    assert torch.equal(u[500:510], v)


def test_decompress_exact_bound():
    for cfg in ("C1", "C4"):
        shape = (1, 40, 50) if cfg == "C4" else None
        f, g, xi = S.make(cfg, shape=shape)
        d = g.double() - f.double()
        assert float(d.abs().max()) <= xi
        assert S.lo_monotone(f, xi)
    f, g, xi = S.make("C1", mode="sz")
    assert float((g.double() - f.double()).abs().max()) <= xi


def test_deterministic():
    a = S.make("C2", shape=(8, 8, 8))
    b = S.make("C2", shape=(8, 8, 8))
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and a[2] == b[2]


def test_offset_rule():
    for cfg, shape in (("C1", None), ("C2", (16, 16, 16)), ("C3", (16, 16, 16))):
        f, g, xi = S.make(cfg, shape=shape)
        assert float(f.min()) >= xi
