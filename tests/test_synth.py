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


def test_szlike_roundtrip():
    """The SZ-like base stream (synth/szlike.py) decodes to the generator's
    ghat bit for bit, 3D and 2D, with exception entries (vertices off the
    RN_f32(2 xi q) grid, here injected one ulp away) and escapes (large
    Lorenzo residuals, here a spike)."""
    from synth import szlike as Z
    for cfg, shape in [("C2", (20, 24, 37)), ("C4", (1, 30, 50)), ("C3", (9, 16, 16))]:
        f, g, xi = S.make(cfg, shape=shape, mode="sz")
        e = Z.encode(f, xi, g)
        assert torch.equal(Z.decode(e).view(torch.int32), g.view(torch.int32))
        g2 = g.clone().reshape(-1)
        idx = torch.tensor([0, 7, 8, g2.numel() - 1])
        g2[idx] = torch.nextafter(g2[idx], torch.full_like(g2[idx], float("inf")))
        g2 = g2.reshape(g.shape)
        f2 = f.clone().reshape(-1)
        f2[5] += 3000 * 2 * xi  # a spike: residuals beyond one byte
        f2 = f2.reshape(f.shape)
        q = torch.round(f2.double() / (2 * float(np.float32(xi))))
        g3 = (2 * float(np.float32(xi)) * q).float()
        e3 = Z.encode(f2, xi, g3)
        assert e3["n_esc"] >= 1 and e3["n_exc"] == 0
        assert torch.equal(Z.decode(e3).view(torch.int32), g3.view(torch.int32))
        e4 = Z.encode(f, xi, g2)
        assert e4["n_exc"] == 4
        assert torch.equal(Z.decode(e4).view(torch.int32), g2.view(torch.int32))


def test_weak_scaling_fields():
    """bench.py --scaling weak: one field per rank (seed offset), decompressed
    with a common xi (the smallest rank's): distinct fields, every bound held,
    min f >= xi on every rank (no lo-collapse)."""
    xs = [S.make("C2", shape=(16, 16, 24), seed_offset=r)[2] for r in range(3)]
    xi = min(xs)
    fs = []
    for r in range(3):
        f, g, x = S.make("C2", shape=(16, 16, 24), seed_offset=r, xi=xi)
        assert x == xi
        assert float((f.double() - g.double()).abs().max()) <= xi
        assert float(f.min()) >= xi
        fs.append(f)
    assert not torch.equal(fs[0], fs[1]) and not torch.equal(fs[1], fs[2])
    f0, _, _ = S.make("C2", shape=(16, 16, 24))
    assert torch.equal(f0, S.make("C2", shape=(16, 16, 24), seed_offset=0)[0])
