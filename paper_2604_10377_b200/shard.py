"""Sharding of shape pairs / row systems across GPUs (one process per GPU).

The solver's units are independent: pairs q and, within a pair, row systems
(q, i) (solver.hpp:258-259 — "workers own disjoint systems").  So the
multi-GPU path needs no data-path collective: rank g solves a contiguous
range and the only exchange is an optional final gather of C to rank 0
(north_star: "no collective except a final gather of C").

* `pair_range(b, world, rank)`   contiguous pair ranges (b >= world), the
  same chunking rule as solve_batched_many's thread split (solver.hpp:292-296)
* `system_range(b, k, world, rank)`  contiguous global system ranges
  s in [0, b*k) when b < world
* `gather_maps(local, b, k, group)`  all ranks' C slices -> rank 0 [b, k, k]
* `MapGather`  the same gather with buffers allocated once (bench.py's timed loop)

Results are bitwise independent of the world size: every system is solved by
one CTA with a fixed reduction order regardless of where it runs.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Range:
    lo: int
    hi: int

    @property
    def size(self) -> int:
        return self.hi - self.lo


def chunk(n: int, world: int, rank: int) -> Range:
    """ceil(n/world)-sized contiguous chunks in rank order (solver.hpp:292-296)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    c = (n + world - 1) // world
    lo = min(rank * c, n)
    return Range(lo, min(lo + c, n))


def pair_range(b: int, world: int, rank: int) -> Range:
    return chunk(b, world, rank)


def system_range(b: int, k: int, world: int, rank: int) -> Range:
    return chunk(b * k, world, rank)


def gather_maps(local, b: int, k: int, world: int, rank: int, group=None):
    """Gather per-rank pair slices of C ([n_local, k, k], contiguous pair
    ranges from `pair_range`) into a [b, k, k] tensor on rank 0 (None elsewhere).
    Uses torch.distributed.gather (NCCL over NVLink on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    c = (b + world - 1) // world
    buf = torch.zeros((c, k, k), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]].copy_(local)
    if rank == 0:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=0, group=group)
        out = torch.cat([p[: pair_range(b, world, g).size] for g, p in enumerate(parts)], dim=0)
        return out
    dist.gather(buf, None, dst=0, group=group)
    return None


class MapGather:
    """Final gather of C to rank 0 with preallocated buffers, for timed loops.

    `send` is this rank's padded slot ([ceil(b/world), k, k]); `__call__()`
    gathers every slot into rank 0's receive buffer (one
    torch.distributed.gather: NCCL over NVLink on GPUs, gloo on CPU), and `out`
    assembles the [b, k, k] batch in global pair order afterwards."""

    def __init__(self, b: int, k: int, world: int, rank: int, device, dtype=None, group=None):
        import torch
        self.b, self.k, self.world, self.rank, self.group = b, k, world, rank, group
        self.c = (b + world - 1) // world
        dtype = dtype or torch.float32
        self.mine = pair_range(b, world, rank)
        self.send = torch.zeros((self.c, k, k), dtype=dtype, device=device)
        self.recv = torch.empty((world * self.c, k, k), dtype=dtype, device=device) if rank == 0 else None
        self.parts = list(self.recv.split(self.c)) if rank == 0 else None

    @property
    def local(self):
        """This rank's C slice ([size, k, k]) inside the send buffer: solve into it."""
        return self.send[: self.mine.size]

    def __call__(self) -> None:
        import torch.distributed as dist
        if self.world > 1:
            dist.gather(self.send, self.parts, dst=0, group=self.group)

    @property
    def out(self):
        """Rank 0: the gathered [b, k, k] batch (copy; slots are padded per rank)."""
        import torch
        if self.world == 1:
            return self.local
        return torch.cat([p[: pair_range(self.b, self.world, g).size] for g, p in enumerate(self.parts)], dim=0)
