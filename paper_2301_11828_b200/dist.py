"""torch.distributed plumbing for multi-GPU runs (one process per GPU).

The data path of a sharded lattice is the halo-slab engine (slab.py, the
library's NCCL exchange in csrc/comm.cpp); this module holds the launcher
environment, the max-over-ranks timing reduction, per-vector seeding and
checksum gathering (bench.py and the gloo tests), and the vector split of the
"replicas" bench arm (--shard vectors: independent vectors per rank, no
data-path collective).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(rank, world, local_rank) from the torchrun environment."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str = "nccl", device=None):
    rank, world, local = env()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group(backend, device_id=device)
        else:
            dist.init_process_group(backend)
    return rank, world, local


def vector_range(total: int, rank: int, world: int, weak: bool = True):
    """Vectors [lo, hi) owned by `rank`.  weak: every rank owns `total`
    vectors of its own (global ids rank*total + i); strong: `total` split."""
    if weak:
        return rank * total, (rank + 1) * total
    per = (total + world - 1) // world
    return min(rank * per, total), min((rank + 1) * per, total)


def vector_seed(base: int, gid: int) -> int:
    """Seed of global vector gid (seed = 1000*config + index)."""
    return base + gid


def max_over_ranks(value: float, device="cpu") -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_checksums(local, device="cpu"):
    """All ranks' per-vector checksums, rank-major (list of lists)."""
    t = torch.tensor(list(local), dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [t.tolist()]
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def finalize():
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
