"""Full-size checks at BASELINE.json's configs, in the launch configuration
bench.py times (exactz_correct with change tracking).

The oracle cannot replay 40 rounds of a 512^3 correction in test time, so at
full size the result is checked by properties that hold at any size and are
evaluated independently of the CUDA path:
  * the bound and monotonicity, exactly: f - xi <= out <= fhat (in double);
  * c <= N+1 and (c == 0) <=> (out == fhat);
  * zero violations of the local rules R1-R3 (C1), recomputed by the oracle
    on crops: a mark on a vertex two or more planes inside a crop can only
    come from a checking vertex whose closed star lies in the crop;
  * C4 (2D, 6.5 M vertices): a complete independent CheckConstraints pass of
    the oracle (all rules, C2 and C3 included) on the corrected field.
"""
import numpy as np
import pytest
import torch

from synth import fields as S

pytestmark = pytest.mark.gpu


def correct_full(E, cfg):
    f, g, xi = S.make(cfg, device="cuda")
    c = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    r = E.exactz_correct(f, g, xi, edit_counts=c)
    torch.cuda.synchronize()
    return f, g, xi, r, c


def check_bound_and_counts(f, g, xi, out, c, N=5):
    fd, gd, od = f.double(), g.double(), out.double()
    assert bool((od >= fd - xi).all()), "out below f - xi"
    assert bool((od <= gd).all()), "edits must only decrease"
    assert int(c.max()) <= N + 1
    same = out.view(torch.int32) == g.view(torch.int32)
    assert bool(((c.view(out.shape) == 0) == same).all())


def crop_local_rules(oracle, f, out, starts, n=24):
    for z0, y0, x0 in starts:
        fs = f[z0:z0 + n, y0:y0 + n, x0:x0 + n].cpu().numpy()
        os_ = out[z0:z0 + n, y0:y0 + n, x0:x0 + n].cpu().numpy()
        mark, cnt = oracle.check(fs, os_, flags=oracle.NO_C2 | oracle.NO_C3)
        m = mark.reshape(fs.shape)[2:-2, 2:-2, 2:-2]
        assert not m.any(), f"R1-R3 violation inside crop at {(z0, y0, x0)}"


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_fullsize_3d_properties(exactz, oracle, cfg):
    f, g, xi, r, c = correct_full(exactz, cfg)
    assert r.status == 0
    check_bound_and_counts(f, g, xi, r.out, c)
    v, _ = exactz.exactz_check(f, r.out, xi)
    assert v == 0
    rs = np.random.default_rng(7)
    nz, ny, nx = f.shape
    starts = [(0, 0, 0), (nz - 24, ny - 24, nx - 24)] + \
             [tuple(int(rs.integers(0, d - 24)) for d in f.shape) for _ in range(4)]
    crop_local_rules(oracle, f, r.out, starts)


def test_fullsize_c4_oracle_check(exactz, oracle):
    f, g, xi, r, c = correct_full(exactz, "C4")
    assert r.status == 0
    check_bound_and_counts(f, g, xi, r.out, c)
    mark, cnt = oracle.check(f.cpu().numpy(), r.out.cpu().numpy())
    assert cnt[0] == 0 and not mark.any(), f"oracle finds violations: {cnt}"


def test_fullsize_c1_is_parity(exactz, oracle):
    """C1 (16^3) is a BASELINE config in full: bit-exact with the oracle."""
    f, g, xi = S.make("C1")
    ro = oracle.correct(f.numpy(), g.numpy(), xi)
    rg = exactz.exactz_correct(f.cuda(), g.cuda(), xi)
    assert rg.iters == ro.iters
    assert np.array_equal(rg.out.cpu().numpy().reshape(-1).view(np.uint32),
                          ro.out.view(np.uint32))


@pytest.mark.parametrize("cfg", ["C4", "C3"])
def test_fullsize_tracking_equals_dense(exactz, cfg):
    """At full size the C3 recompute list outgrows one lane per saddle (the
    grid-stride path of k_events_cached): the tracked run must still give the
    dense run's bits and every per-pass counter, and repeat bit for bit."""
    f, g, xi = S.make(cfg, device="cuda")
    runs = [exactz.exactz_correct(f, g, xi, stats_cap=100000) for _ in range(3)]
    b = exactz.exactz_correct(f, g, xi, flags=exactz.NO_TRACK, stats_cap=100000)
    for a in runs:
        assert a.iters == b.iters and a.status == b.status
        assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))
        assert a.stats == b.stats
