"""Process-group plumbing of the sharded path (torch.distributed for the
bootstrap only; the data path is NCCL inside libexactz.so).

  slab_of(nz, world, rank)      this rank's z-slab (the C ABI's split)
  broadcast_uid(group)          rank 0's 128-byte NCCL unique id on every rank
  max_over_ranks(x, group)      max of a host float over ranks (timing)
  open_comm(device, group)      exactz Comm for this rank
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def slab_of(nz: int, world: int, rank: int):
    """Planes [z0, z0 + count) of rank: the C ABI's split (exactz_slab_range),
    the one source of truth (the first nz % world ranks get one extra plane)."""
    import paper_2604_01397_b200 as E
    return E.exactz_slab_range(nz, world, rank)


def broadcast_uid(uid: bytes | None, group=None, device="cpu") -> bytes:
    """rank 0's id (uid) on every rank of group."""
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def max_over_ranks(x: float, group=None, device="cpu") -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def open_comm(device: int, group=None):
    import paper_2604_01397_b200 as E
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = E.exactz_nccl_unique_id() if rank == 0 else None
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    uid = broadcast_uid(uid, group, device=dev)
    return E.Comm(uid, world, rank, device)
