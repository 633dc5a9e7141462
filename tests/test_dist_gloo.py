"""Host-side logic of the sharded path on CPU: world_size-2 gloo process groups
(127.0.0.1).  Checks the slab split (Python helper == C ABI, a partition of
[0, nz)), the unique-id broadcast and the max-over-ranks timing reduction
that bench.py uses."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_01397_b200 import dist as D
        import paper_2604_01397_b200 as E
        out = {}
        for nz in (1 * world, 7, 512, 560, 1024):
            z0, cnt = D.slab_of(nz, world, rank)
            # the split itself, restated: the first nz % world ranks get one extra plane
            base, extra = divmod(nz, world)
            assert (z0, cnt) == (rank * base + min(rank, extra), base + (rank < extra))
            got = [None] * world
            dist.all_gather_object(got, (z0, cnt))
            out[nz] = got
        uid = bytes(range(128)) if rank == 0 else None
        out["uid"] = D.broadcast_uid(uid)
        out["max"] = D.max_over_ranks(float(rank + 1) * 1.5)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_slab_plumbing(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert o["uid"] == bytes(range(128))
        assert o["max"] == 1.5 * world
        for nz in (1 * world, 7, 512, 560, 1024):
            slabs = o[nz]
            assert slabs == res[0][nz]
            assert slabs[0][0] == 0
            for (a, n), (b, _) in zip(slabs, slabs[1:]):
                assert a + n == b and n >= 1
            assert slabs[-1][0] + slabs[-1][1] == nz
            assert max(n for _, n in slabs) - min(n for _, n in slabs) <= 1
