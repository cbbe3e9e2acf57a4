"""Multi-GPU partitioning of the PASA forward: one process per GPU, work split
by (batch, kv-head) -- the reference's own decomposition (pasa.cpp:243-287
loops over independent (b, h, i) slices) -- with no collective on the data
path.  Each rank runs the fused kernel on its shard; an optional all-gather
of O (outside any timed region) reassembles the full output.

Every (b, kv head, query tile) is computed by exactly the same kernel code
whatever the shard, so the gathered O is bit-identical for any world size.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch


@dataclass(frozen=True)
class Shard:
    rank: int
    start: int  # first flat (b, kv head) unit, unit = b * Hkv + h
    stop: int   # one past the last

    def units(self):
        return range(self.start, self.stop)


def partition(batch: int, heads_kv: int, world: int) -> list[Shard]:
    """Contiguous, balanced split of the B*Hkv units (sizes differ by <= 1)."""
    n = batch * heads_kv
    if world <= 0:
        raise ValueError("world size must be positive")
    base, extra = divmod(n, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append(Shard(r, s, e))
        s = e
    return out


def _shard_views(q, k, v, start: int, stop: int):
    """The shard's units [start, stop) as ONE problem: in BHSD the flat (b, kv head) units
    are contiguous, so Q is a (1, (stop - start) * g, S1, d) view and K, V are
    (1, stop - start, S2, d) views -- one launch per shard, whatever the unit count."""
    B, Hq, S1, d = q.shape
    Hkv, S2 = k.shape[1], k.shape[2]
    g = Hq // Hkv
    n = stop - start
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    return (q.reshape(B * Hkv, g, S1, d)[start:stop].reshape(1, n * g, S1, d),
            k.reshape(B * Hkv, 1, S2, d)[start:stop].reshape(1, n, S2, d),
            v.reshape(B * Hkv, 1, S2, d)[start:stop].reshape(1, n, S2, d))


def _default_compute(q, k, v, **kw):
    from .api import pasa_attention_fwd
    return pasa_attention_fwd(q, k, v, **kw)


def shard_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, shard: Shard,
                  compute: Callable | None = None, **kw) -> list[tuple[int, torch.Tensor]]:
    """Run this rank's units in one call; returns [(unit, O_unit)] with O_unit
    (1, Hq/Hkv, S1, d), views of the shard's output."""
    compute = compute or _default_compute
    if shard.stop <= shard.start:
        return []
    g = q.shape[1] // k.shape[1]
    o = compute(*_shard_views(q, k, v, shard.start, shard.stop), **kw)
    return [(u, o[:, i * g:(i + 1) * g]) for i, u in enumerate(shard.units())]


def pasa_attention_sharded(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                           group=None, gather: bool = True, compute: Callable | None = None,
                           **kw) -> torch.Tensor | list[tuple[int, torch.Tensor]]:
    """PASA forward over torch.distributed ranks (every rank passes the full
    Q/K/V or at least its shard's slices).  With ``gather`` the full O is
    assembled on every rank by an all-gather (the only collective, outside
    the compute path); otherwise the rank's [(unit, O_unit)] list is returned."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, Hq, S1, d = q.shape
    Hkv = k.shape[1]
    shards = partition(B, Hkv, world)
    mine = shard_forward(q, k, v, shards[rank], compute, **kw)
    if not gather:
        return mine
    g = Hq // Hkv
    out = torch.empty_like(q)
    for u, o in mine:
        b, h = divmod(u, Hkv)
        out[b:b + 1, h * g:(h + 1) * g] = o
    if world > 1:
        pieces = [None] * world
        dist.all_gather_object(pieces, [(u, o.cpu()) for u, o in mine], group=group)
        for lst in pieces:
            for u, o in lst:
                b, h = divmod(u, Hkv)
                out[b:b + 1, h * g:(h + 1) * g] = o.to(out.device)
    return out
