"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bar (BASELINE.json north_star): bit-exact equality of the
corrected field, the edit counts, both label arrays, the iteration count, the
status and every per-pass counter (V_t, applied, n1..n6) on the same seeded
inputs.  Sizes are ones the oracle finishes in seconds, shaped to span several
x-blocks (128 wide) and rows with ragged tails.
"""
import numpy as np
import pytest
import torch

from synth import fields as S

pytestmark = pytest.mark.gpu


def run_both(E, O, f, g, xi, N=5, flags=0, max_iters=0, mode_alias=False, gpu_flags=0):
    fn, gn = f.numpy(), g.numpy()
    ro = O.correct(fn, gn, xi, N, flags=flags, max_iters=max_iters)
    fd, gd = f.cuda(), g.cuda()
    V = f.numel()
    c = torch.empty(V, dtype=torch.uint8, device="cuda")
    lmin = torch.empty(V, dtype=torch.int32, device="cuda")
    lmax = torch.empty(V, dtype=torch.int32, device="cuda")
    out = gd if mode_alias else None
    rg = E.exactz_correct(fd, gd, xi, out=out, N=N, flags=flags | gpu_flags, max_iters=max_iters,
                          edit_counts=c, label_min=lmin, label_max=lmax, stats_cap=100000)
    torch.cuda.synchronize()
    return ro, rg, c.cpu().numpy(), lmin.cpu().numpy(), lmax.cpu().numpy()


def assert_parity(ro, rg, c, lmin, lmax):
    assert rg.status == ro.status
    assert rg.iters == ro.iters
    og = rg.out.reshape(-1).cpu().numpy()
    bad = np.nonzero(og.view(np.uint32) != ro.out.view(np.uint32))[0]
    assert bad.size == 0, f"out differs at {bad[:10]} ({bad.size} vertices)"
    assert np.array_equal(c, ro.counts), "edit counts differ"
    assert np.array_equal(lmin, ro.label_min), "label_min differs"
    assert np.array_equal(lmax, ro.label_max), "label_max differs"
    st_g = np.array(rg.stats, dtype=np.int64).reshape(-1, 8)
    assert st_g.shape == ro.stats.shape
    assert np.array_equal(st_g, ro.stats), "per-pass counters differ"


CASES = [
    ("C1", None),              # 16^3 GaussMix, rel 1e-2 (the BASELINE config itself)
    ("C2", (20, 24, 131)),     # Nyx-like recipe, 2 x-blocks, ragged
    ("C3", (17, 21, 150)),     # combustion recipe: many saddles, plateaus at 300 K
    ("C4", (1, 90, 300)),      # 2D climate recipe (nz = 1), 3 x-blocks
    ("C5", (24, 18, 40)),      # cosmology recipe at rel 1e-4
    ("C2", (30, 20, 70)),      # 3 stencil tiles in x (32 wide), 3 in y (8 high)
    ("C3", (24, 19, 66)),      # plateau ties across tile borders
]


@pytest.mark.parametrize("cfg,shape", CASES)
def test_parity_configs(exactz, oracle, cfg, shape):
    f, g, xi = S.make(cfg, shape=shape)
    assert_parity(*run_both(exactz, oracle, f, g, xi))


def test_parity_negative_values(exactz, oracle):
    """Fields with negative values (some lo = RU(f - xi) < 0) run the general
    stencil instead of k_stencil_fast; parity with the oracle either way."""
    f, _, xi = S.make("C2", shape=(30, 20, 40))
    f2 = f - float(f.mean())
    g2 = S.decompress(f2, xi, seed=11)
    assert bool((f2 < 0).any())
    assert_parity(*run_both(exactz, oracle, f2, g2, xi))


# debug flag 0x800 of exactz_correct: the general stencil (k_stencil) even for
# non-negative fields
@pytest.mark.parametrize("cfg,shape,mode", [("C2", (60, 40, 100), "uniform"),
                                            ("C3", (50, 33, 70), "uniform"),
                                            ("C1", (40, 40, 40), "sz"),
                                            ("C4", (1, 200, 300), "uniform")])
def test_fast_stencil_equals_general(exactz, cfg, shape, mode):
    f, g, xi = S.make(cfg, shape=shape, device="cuda", mode=mode)
    a = exactz.exactz_correct(f, g, xi, stats_cap=100000)
    b = exactz.exactz_correct(f, g, xi, flags=0x800, stats_cap=100000)
    assert a.iters == b.iters and a.status == b.status
    assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))
    assert a.stats == b.stats


def test_parity_stuck_fixpoint(exactz, oracle):
    """lo-collapse (amb-17): f_0 > f_1 but RU(f_i - xi) is the same float for
    both, so at lo the pair stays in index order and no edit can fix it:
    ESTUCK after the pass that applied nothing, with the oracle's rows."""
    lo = np.float32(-0.99999994)
    f = torch.tensor([2e-8, 1e-8, 3.0])
    g = torch.tensor([lo, lo, 3.0])
    ro, rg, c, lmin, lmax = run_both(exactz, oracle, f, g, 1.0)
    assert ro.status == 4 and ro.iters == 0
    assert_parity(ro, rg, c, lmin, lmax)


@pytest.mark.parametrize("cfg,shape", [("C1", None), ("C3", (12, 16, 140))])
def test_parity_sz_plateaus(exactz, oracle, cfg, shape):
    """SZ-like binned decompression: plateaus everywhere, so SoS ties decide."""
    f, g, xi = S.make(cfg, shape=shape, mode="sz")
    assert_parity(*run_both(exactz, oracle, f, g, xi))


@pytest.mark.parametrize("flags", [1, 2, 3])
def test_parity_debug_flags(exactz, oracle, flags):
    f, g, xi = S.make("C1")
    assert_parity(*run_both(exactz, oracle, f, g, xi, flags=flags))


@pytest.mark.parametrize("N", [1, 2, 9])
def test_parity_N(exactz, oracle, N):
    f, g, xi = S.make("C2", shape=(10, 12, 33))
    assert_parity(*run_both(exactz, oracle, f, g, xi, N=N))


def test_parity_max_iters(exactz, oracle):
    f, g, xi = S.make("C1")
    ro, rg, *rest = run_both(exactz, oracle, f, g, xi, max_iters=3)
    assert ro.status == 4 and ro.iters == 3
    assert_parity(ro, rg, *rest)


def test_parity_alias_out(exactz, oracle):
    f, g, xi = S.make("C1")
    assert_parity(*run_both(exactz, oracle, f, g, xi, mode_alias=True))


def test_misaligned_buffers(exactz):
    """Device buffers one element off 16-byte alignment take the scalar edit
    path of k_count_edit; the bits equal the aligned run."""
    f, g, xi = S.make("C2", shape=(24, 20, 64), device="cuda")
    a = exactz.exactz_correct(f, g, xi, stats_cap=1000)
    fb = torch.empty(f.numel() + 1, device="cuda")
    gb = torch.empty(g.numel() + 1, device="cuda")
    fb[1:] = f.flatten()
    gb[1:] = g.flatten()
    ob = torch.empty(g.numel() + 1, device="cuda")
    b = exactz.exactz_correct(fb[1:].view(f.shape), gb[1:].view(g.shape), xi,
                              out=ob[1:].view(g.shape), stats_cap=1000)
    assert a.iters == b.iters and a.stats == b.stats
    assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))


def test_edit_strategy_1x3(exactz, oracle):
    """fig:edit_strategy as a 1x3 field (tests/golden/)."""
    f = torch.tensor([3.0, 1.0, 2.0])
    g = torch.tensor([3.0, 1.9, 1.8])
    ro, rg, c, lmin, lmax = run_both(exactz, oracle, f, g, 1.0)
    assert_parity(ro, rg, c, lmin, lmax)
    assert rg.out.cpu().numpy().view(np.uint32).tolist() == [0x40400000, 0x3FD99999, 0x3FE66666]


@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 1, 7), (1, 5, 1), (3, 1, 1), (2, 2, 2),
                                   (1, 3, 129), (5, 1, 4)])
def test_parity_degenerate_shapes(exactz, oracle, shape):
    rs = np.random.default_rng(sum(shape))
    f = torch.from_numpy(rs.uniform(1, 2, size=shape).astype(np.float32))
    xi = 0.05
    g = S.decompress(f, xi, seed=7)
    assert_parity(*run_both(exactz, oracle, f, g, xi))


def test_clean_input_zero_iters(exactz, oracle):
    f, _, xi = S.make("C1")
    ro, rg, *rest = run_both(exactz, oracle, f, f.clone(), xi)
    assert rg.iters == 0 and rg.status == 0
    assert_parity(ro, rg, *rest)


def test_xi_zero(exactz, oracle):
    f, _, _ = S.make("C1")
    ro, rg, *rest = run_both(exactz, oracle, f, f.clone(), 0.0)
    assert rg.status == 0 and rg.iters == 0
    assert_parity(ro, rg, *rest)


def test_errors(exactz):
    E = exactz
    f, g, xi = S.make("C1")
    fd, gd = f.cuda(), g.cuda()
    bad = gd.clone()
    bad.view(-1)[100] = f.view(-1)[100] + 2 * xi
    out = torch.full_like(gd, 7.0)
    assert E.status_of(E.exactz_correct, fd, bad, xi, out=out) == E.EBOUND
    assert bool((out == 7.0).all()), "out written before validation failed"
    nan = gd.clone()
    nan.view(-1)[5] = float("nan")
    assert E.status_of(E.exactz_correct, fd, nan, xi) == E.EINVAL
    assert E.status_of(E.exactz_correct, fd, gd, -1.0) == E.EINVAL
    assert E.status_of(E.exactz_correct, fd, gd, xi, N=255) == E.EINVAL


def test_check_after_correct(exactz, oracle):
    f, g, xi = S.make("C2", shape=(16, 16, 40))
    r = exactz.exactz_correct(f.cuda(), g.cuda(), xi)
    assert r.status == 0
    v, _ = exactz.exactz_check(f.cuda(), r.out, xi)
    assert v == 0
    marks, cnt = oracle.check(f.numpy(), r.out.cpu().numpy())
    assert cnt[0] == 0


def test_host_entry_matches_device(exactz):
    f, g, xi = S.make("C1")
    rd = exactz.exactz_correct(f.cuda(), g.cuda(), xi)
    rh = exactz.exactz_correct_host(f.pin_memory(), g.pin_memory(), xi)
    assert rh.iters == rd.iters
    assert np.array_equal(rh.out.numpy().view(np.uint32), rd.out.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("cfg,shape", [("C2", (20, 24, 131)), ("C3", (24, 19, 66))])
def test_host_entry_overlapped_copy(exactz, oracle, cfg, shape):
    """exactz_correct_host overlaps g's copy with the reference of f: same
    bits as the oracle, and the validation errors still come first (a
    non-finite f before the reference, a bound violation or a non-finite g
    after the copy), with the host out untouched."""
    E = exactz
    f, g, xi = S.make(cfg, shape=shape)
    ro = oracle.correct(f.numpy(), g.numpy(), xi, 5)
    c = torch.empty(f.numel(), dtype=torch.uint8).pin_memory()
    rh = E.exactz_correct_host(f.pin_memory(), g.pin_memory(), xi, edit_counts=c)
    assert rh.status == ro.status and rh.iters == ro.iters
    assert np.array_equal(rh.out.numpy().reshape(-1).view(np.uint32), ro.out.view(np.uint32))
    assert np.array_equal(c.numpy(), ro.counts)
    for fb, gb, want in [(f.clone(), g, E.EINVAL), (f, g.clone(), E.EINVAL), (f, g.clone(), E.EBOUND)]:
        if want == E.EINVAL and fb is not f:
            fb.view(-1)[7] = float("inf")
        elif want == E.EINVAL:
            gb.view(-1)[7] = float("nan")
        else:
            gb.view(-1)[11] = fb.view(-1)[11] + 2 * xi
        out = torch.full_like(g, 7.0).pin_memory()
        assert E.status_of(E.exactz_correct_host, fb.pin_memory(), gb.pin_memory(), xi,
                           out=out) == want
        assert bool((out == 7.0).all())


def test_eps_from_relative(exactz):
    f, _, _ = S.make("C1")
    e = exactz.exactz_eps_from_relative(f.cuda(), 1e-2)
    assert e == S.xi_from_rel(f, 1e-2)


def test_repeat_bit_identical(exactz):
    f, g, xi = S.make("C3", shape=(16, 16, 70))
    a = exactz.exactz_correct(f.cuda(), g.cuda(), xi)
    b = exactz.exactz_correct(f.cuda(), g.cuda(), xi)
    assert a.iters == b.iters
    assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))


# debug flags of exactz_correct (exactz.cu correct_impl): 0x400 compacted
# stencil passes from the second pass on (never the sparse one), 0x200 no C3
# cache, 0x100 no vertex activity, 0x80000 no clean-path test (FPaths)
NO_FPATHS, FPATHS_ALWAYS = 0x80000, 0x200000  # (the gate of the test off: every list pass)
TRACK_MODES = [0, 0x400, 0x400 | 0x200, 0x100, 0x200, NO_FPATHS, NO_FPATHS | 0x200,
               FPATHS_ALWAYS, FPATHS_ALWAYS | 0x200, 0x400000]  # 0x400000: float list stencil


@pytest.mark.parametrize("mode", TRACK_MODES)
@pytest.mark.parametrize("cfg,shape", [("C2", (40, 48, 200)), ("C3", (33, 40, 150)),
                                       ("C4", (1, 300, 700))])
def test_tracking_equals_dense(exactz, cfg, shape, mode):
    """Change tracking (vertex activity with the compacted or the sparse
    stencil, cached C3 results) gives the bits of the dense passes, including
    every per-pass counter."""
    f, g, xi = S.make(cfg, shape=shape, device="cuda")
    a = exactz.exactz_correct(f, g, xi, flags=mode, stats_cap=100000)
    b = exactz.exactz_correct(f, g, xi, flags=exactz.NO_TRACK, stats_cap=100000)
    assert a.iters == b.iters and a.status == b.status
    assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))
    assert a.stats == b.stats


@pytest.mark.parametrize("cfg,shape", [("C1", None), ("C2", (20, 24, 131)), ("C3", (17, 21, 150)),
                                       ("C4", (1, 90, 300))])
def test_parity_reformulated(exactz, oracle, cfg, shape):
    """NEXT-1: reformulated event constraints, bit-exact with the
    oracle's REFORM mode."""
    f, g, xi = S.make(cfg, shape=shape)
    assert_parity(*run_both(exactz, oracle, f, g, xi, flags=16))


def test_tracking_equals_dense_reformulated(exactz):
    f, g, xi = S.make("C2", shape=(40, 48, 200), device="cuda")
    a = exactz.exactz_correct(f, g, xi, flags=exactz.REFORMULATED, stats_cap=100000)
    b = exactz.exactz_correct(f, g, xi, flags=exactz.REFORMULATED | exactz.NO_TRACK,
                              stats_cap=100000)
    assert a.iters == b.iters and a.stats == b.stats
    assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))


@pytest.mark.parametrize("cfg,shape", [("C1", None), ("C2", (19, 13, 67)), ("C3", (11, 17, 97)),
                                       ("C4", (1, 41, 133)), ("C2", (9, 3, 33))])
def test_parity_compacted_passes(exactz, oracle, cfg, shape):
    """The compacted stencil (forced from the second pass on) on ragged tiles
    (nx not a multiple of 32, ny not of 8): bit-exact with the oracle."""
    f, g, xi = S.make(cfg, shape=shape)
    assert_parity(*run_both(exactz, oracle, f, g, xi, gpu_flags=0x400))


@pytest.mark.parametrize("cfg,shape", [("C3", (24, 19, 66)), ("C4", (1, 90, 300))])
def test_stats_pass_spans_and_saddle_counts(exactz, oracle, cfg, shape):
    """exactz_stats: |S|, |J|, |P| equal the oracle's reference lists (O7);
    one positive GPU span per pass, together within the loop's span."""
    f, g, xi = S.make(cfg, shape=shape)
    ref = oracle.reference(f.numpy())
    r = exactz.exactz_correct(f.cuda(), g.cuda(), xi, stats_cap=4096)
    torch.cuda.synchronize()
    assert (r.n_saddles, r.n_join, r.n_split) == (len(ref["S"]), len(ref["J"]), len(ref["P"]))
    assert len(r.pass_ms) == len(r.stats) == r.iters + 1
    assert all(t > 0 for t in r.pass_ms)
    assert sum(r.pass_ms) <= r.ms_loop * 1.01 + 0.05


SNAP_EARLY, SNAP_CAP1, SNAP_UNTRACK = 0x10000, 0x20000, 0x40000


@pytest.mark.parametrize("dbg", [SNAP_EARLY, SNAP_EARLY | SNAP_CAP1, SNAP_EARLY | SNAP_UNTRACK],
                         ids=["patched", "overflow", "untracked_after_start"])
def test_host_snapshot_branches(exactz, oracle, dbg):
    """exactz_correct_host starts the result's D2H copy while passes
    still run and patches the vertices edited afterwards.  Debug flags force
    the copy to start at the first list-based pass (patched branch), with a
    one-entry patch list (overflow: full copy), and with the passes after the
    start untracked (no patch list: full copy).  Every branch must give the
    oracle's out and edit counts."""
    E = exactz
    f, g, xi = S.make("C2", shape=(30, 40, 70))
    ro = oracle.correct(f.numpy(), g.numpy(), xi, 5)
    c = torch.empty(f.numel(), dtype=torch.uint8).pin_memory()
    rh = E.exactz_correct_host(f.pin_memory(), g.pin_memory(), xi, edit_counts=c, flags=dbg)
    assert rh.status == ro.status and rh.iters == ro.iters
    assert rh.out.is_pinned()
    assert np.array_equal(rh.out.numpy().reshape(-1).view(np.uint32), ro.out.view(np.uint32))
    assert np.array_equal(c.numpy(), ro.counts)


def test_host_entry_rejects_bad_outputs(exactz):
    f, g, xi = S.make("C1")
    E = exactz
    for kw in ({"out": torch.empty(5)}, {"edit_counts": torch.empty(f.numel())},
               {"label_min": torch.empty(f.numel(), dtype=torch.int64)},
               {"label_max": torch.empty(f.numel(), dtype=torch.int32, device="cuda")}):
        with pytest.raises(ValueError):
            E.exactz_correct_host(f, g, xi, **kw)


@pytest.mark.parametrize("cfg,shape,mode", [("C3", (33, 40, 150), None), ("C2", (40, 48, 200), None),
                                            ("C3", (12, 16, 140), "sz"), ("C4", (1, 300, 700), None)])
def test_clean_path_test_engages(exactz, oracle, cfg, shape, mode):
    """NEXT-2 incremental labels: in list passes the saddles whose f-walks
    cross no tile with a non-f pointer take X_f without walking (k_fclean).
    Bit-exact with the oracle, and the walks it saves are visible in the
    per-pass link counts (vertices walked from)."""
    f, g, xi = S.make(cfg, shape=shape, mode=mode or "uniform")
    ro, rg, c, lmin, lmax = run_both(exactz, oracle, f, g, xi, gpu_flags=FPATHS_ALWAYS)
    assert_parity(ro, rg, c, lmin, lmax)
    b = exactz.exactz_correct(f.cuda(), g.cuda(), xi, flags=NO_FPATHS, stats_cap=100000)
    assert b.stats == rg.stats and b.iters == rg.iters
    assert sum(rg.pass_links) < sum(b.pass_links), (sum(rg.pass_links), sum(b.pass_links))
