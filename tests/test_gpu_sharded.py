"""The z-slab decomposition is bit-equal to the single-GPU call.

exactz_correct_slabs runs the sharded algorithm — ghost planes, replicated
saddle values, gathered boundary tables for cross-slab label walks, remote
marks, all-reduced counters — with N virtual ranks on one GPU (loopback
transport instead of NCCL).  Same bar as the single-GPU parity: out, edit
counts, iteration count and every per-pass counter bit-equal, for slab counts
that leave 1-plane slabs and ragged splits."""
import numpy as np
import pytest
import torch

from synth import fields as S

pytestmark = pytest.mark.gpu


def both(E, f, g, xi, p, **kw):
    fd, gd = f.cuda(), g.cuda()
    c1 = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    c2 = torch.empty_like(c1)
    a = E.exactz_correct(fd, gd, xi, edit_counts=c1, stats_cap=100000, **kw)
    b = E.exactz_correct_slabs(fd, gd, xi, p, edit_counts=c2, stats_cap=100000, **kw)
    torch.cuda.synchronize()
    return a, b, c1, c2


def assert_same(a, b, c1, c2):
    assert b.status == a.status and b.iters == a.iters
    assert torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))
    assert torch.equal(c1, c2)
    assert a.stats == b.stats


@pytest.mark.parametrize("p", [1, 2, 3, 5, 16])
def test_slabs_c1(exactz, p):
    f, g, xi = S.make("C1")
    assert_same(*both(exactz, f, g, xi, p))


@pytest.mark.parametrize("cfg,shape,p", [("C2", (20, 24, 70), 4), ("C3", (17, 21, 40), 3),
                                         ("C5", (9, 12, 33), 8), ("C3", (12, 16, 50), 12)])
def test_slabs_configs(exactz, cfg, shape, p):
    f, g, xi = S.make(cfg, shape=shape)
    assert_same(*both(exactz, f, g, xi, p))


def test_slabs_sz_plateaus(exactz):
    f, g, xi = S.make("C3", shape=(10, 14, 45), mode="sz")
    assert_same(*both(exactz, f, g, xi, 4))


def test_slabs_flags_and_max_iters(exactz):
    f, g, xi = S.make("C1")
    for kw in ({"flags": 1}, {"flags": 2}, {"max_iters": 2}, {"N": 2}):
        assert_same(*both(exactz, f, g, xi, 3, **kw))


def test_slabs_match_oracle(exactz, oracle):
    f, g, xi = S.make("C2", shape=(14, 10, 30))
    r = oracle.correct(f.numpy(), g.numpy(), xi, 5)
    b = exactz.exactz_correct_slabs(f.cuda(), g.cuda(), xi, 5)
    assert b.iters == r.iters
    assert np.array_equal(b.out.cpu().numpy().reshape(-1).view(np.uint32), r.out.view(np.uint32))


def test_slabs_errors(exactz):
    f, g, xi = S.make("C1")
    E = exactz
    assert E.status_of(E.exactz_correct_slabs, f.cuda(), g.cuda(), xi, 17) == E.EINVAL  # nz < p
    bad = g.clone()
    bad.view(-1)[7] = f.view(-1)[7] + 3 * xi
    assert E.status_of(E.exactz_correct_slabs, f.cuda(), bad.cuda(), xi, 2) == E.EBOUND


@pytest.mark.parametrize("flags", [0x800000, 0x1000000, 0x2000000, 0x2000, 0x8000, 0x80000,
                                   0x200000, 0x200, 0x10000000, 0x20000000, 0x40000000])
def test_slabs_engine_variants(exactz, flags):
    """Exchange and kernel variants of the per-rank engine, each bit-equal:
    boundary tables by sparse changes only (0x800000) or whole every pass
    (0x1000000); one-lane C3 walks (0x2000000); the float-compare stencils
    instead of the exact-key ones (0x2000); thread-staged planes instead of
    TMA (0x8000); no clean-path test (0x80000) or the test in every list pass
    (0x200000); no C3 cache (0x200); R4 partner values by the sparse
    all-gather only (0x10000000) or by the static routing in every pass
    (0x20000000); the stars of the edits always pulled (0x40000000)."""
    f, g, xi = S.make("C2", shape=(24, 20, 64))
    assert_same(*both(exactz, f, g, xi, 6, flags=flags))


@pytest.mark.parametrize("cfg,shape,p,kw", [("C1", None, 3, {}), ("C3", (12, 16, 50), 12, {}),
                                            ("C2", (20, 24, 70), 4, {"flags": 2}),
                                            ("C5", (9, 12, 33), 8, {"flags": 0x10})])
def test_slabs_labels(exactz, oracle, cfg, shape, p, kw):
    """label_min / label_max of the sharded call (local pointer jumping, exits
    through the boundary tables; recomputed at the end when the passes kept no
    tables: NO_C3, reformulated) equal the single-GPU call's and the oracle's."""
    f, g, xi = S.make(cfg, shape=shape) if shape else S.make(cfg)
    V = f.numel()
    fd, gd = f.cuda(), g.cuda()
    la, lb = (torch.empty(V, dtype=torch.int32, device="cuda") for _ in range(2))
    ua, ub = (torch.empty(V, dtype=torch.int32, device="cuda") for _ in range(2))
    a = exactz.exactz_correct(fd, gd, xi, label_min=la, label_max=ua, **kw)
    b = exactz.exactz_correct_slabs(fd, gd, xi, p, label_min=lb, label_max=ub, **kw)
    torch.cuda.synchronize()
    assert b.iters == a.iters and torch.equal(a.out.view(torch.int32), b.out.view(torch.int32))
    assert torch.equal(la, lb) and torch.equal(ua, ub)
    if not kw:
        r = oracle.correct(f.numpy(), g.numpy(), xi, 5)
        assert np.array_equal(lb.cpu().numpy(), r.label_min)
        assert np.array_equal(ub.cpu().numpy(), r.label_max)


@pytest.mark.parametrize("p", [2, 5])
def test_slabs_reformulated(exactz, p):
    f, g, xi = S.make("C3", shape=(15, 20, 40))
    assert_same(*both(exactz, f, g, xi, p, flags=exactz.REFORMULATED))


def test_slabs_negative_values_in_one_slab(exactz, oracle):
    """Negative values only in the upper slab, starting at the slab border:
    the lower slab's owned planes are all positive but its ghost plane is not,
    so the fast (unsigned-key) stencil would be wrong there.  Every slab must
    make the whole field's fast/general choice (C_NEG reduced over
    the ranks)."""
    f, _, _ = S.make("C1")
    f = f.clone()
    f[8:] -= 2.5                        # p = 2: slab 1 owns z = 8..15
    xi = float(np.float32(1e-2 * float(f.max() - f.min())))
    g = S.decompress(f, xi, 7)
    assert float(f[:8].min()) > 0 and float(f[8].min()) < 0
    a, b, c1, c2 = both(exactz, f, g, xi, 2)
    assert_same(a, b, c1, c2)
    r = oracle.correct(f.numpy(), g.numpy(), xi, 5)
    assert b.iters == r.iters and b.status == r.status
    assert np.array_equal(b.out.cpu().numpy().reshape(-1).view(np.uint32), r.out.view(np.uint32))


@pytest.mark.parametrize("cfg,shape", [("C1", None), ("C2", (20, 24, 70)), ("C3", (17, 21, 40))])
def test_nccl_transport_one_rank(exactz, cfg, shape):
    """The NCCL data plane itself (exactz_correct_sharded over a real NCCL
    communicator: ncclSend/Recv of ghost planes and marks, all-gathers of the
    boundary tables, all-reduces of the counters) on the one GPU of the box as
    a 1-rank communicator: bit-equal to exactz_correct."""
    f, g, xi = S.make(cfg, shape=shape)
    fd, gd = f.cuda(), g.cuda()
    c1 = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    c2 = torch.empty_like(c1)
    la, lb, ua, ub = (torch.empty(f.numel(), dtype=torch.int32, device="cuda") for _ in range(4))
    a = exactz.exactz_correct(fd, gd, xi, edit_counts=c1, label_min=la, label_max=ua,
                              stats_cap=100000)
    comm = exactz.Comm(exactz.exactz_nccl_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        dims = (f.shape[2], f.shape[1], f.shape[0])
        b = exactz.exactz_correct_sharded(comm, fd, gd, dims, xi, edit_counts=c2, label_min=lb,
                                          label_max=ub, stats_cap=100000)
        torch.cuda.synchronize()
    finally:
        comm.close()
    assert_same(a, b, c1, c2)
    assert torch.equal(la, lb) and torch.equal(ua, ub)


def test_slabs_long_exit_chains(exactz):
    """A steepest path may cross a slab border several times (the value
    descends, z need not): with 1-plane slabs the chains of boundary-table
    exits are long; the lookups still end at the root (bit-equal)."""
    f, g, xi = S.make("C2", shape=(12, 20, 24))
    assert_same(*both(exactz, f, g, xi, 12))
