"""Multi-GPU partitioning of the PASA forward: one process per GPU, work split
by (batch, kv-head) and, for balance, by query tiles -- the reference's own
decomposition (pasa.cpp:243-287 loops over independent (b, h, i) slices) -- with
no collective on the data path.  Each rank runs the fused kernel on its pieces;
an optional all-gather of O (outside any timed region) reassembles the output.

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


@dataclass(frozen=True)
class Piece:
    """Query tiles [tile0, tile0 + ntiles) of every unit in [start, stop) (a unit = one (b, kv
    head) with its Hq / Hkv query heads; a tile = 128 query rows)."""
    start: int
    stop: int
    tile0: int
    ntiles: int


def tile_costs(seq_q: int, seq_kv: int, causal: bool, s2: int = 128) -> list[int]:
    """Key blocks each 128-row query tile runs (pasa_fwd.cu tile_info): all of them without a
    mask; causal (bottom-right aligned, row r sees keys <= r + S2 - S1): up to the block of
    the tile's last row's last key."""
    nq, nkv, qoff = (seq_q + 127) // 128, seq_kv // s2, seq_kv - seq_q
    if not causal:
        return [nkv] * nq
    return [min((min(seq_q, 128 * (i + 1)) - 1 + qoff) // s2 + 1, nkv) for i in range(nq)]


def partition_work(batch: int, heads_kv: int, seq_q: int, seq_kv: int, causal: bool, world: int,
                   s2: int = 128) -> list[list[Piece]]:
    """contiguous (b, kv head) ranges first, then query tiles for balance.  The
    (unit, tile) work items, unit-major, are cut into `world` contiguous runs of equal key-
    block cost (each item goes to the run holding its cost midpoint), so a problem with
    fewer units than GPUs (Qwen2-7B: 4 kv heads on 8 GPUs) or with causal tiles of growing
    cost still balances to within one tile.  A run is at most three pieces: a unit's tail,
    whole units, a unit's head -- one launch each (pasa_b200_attention_fwd_tiles)."""
    if world <= 0:
        raise ValueError("world size must be positive")
    cost = tile_costs(seq_q, seq_kv, causal, s2)
    nq, units = len(cost), batch * heads_kv
    per_unit = sum(cost)
    total = per_unit * units
    prefix = [0]
    for c in cost:
        prefix.append(prefix[-1] + c)

    def owner(u, i):  # the run holding item (u, i)'s cost midpoint
        mid2 = 2 * (u * per_unit + prefix[i]) + cost[i]  # twice the midpoint, in integers
        return min(world - 1, mid2 * world // (2 * total)) if total else 0

    runs: list[list[tuple[int, int]]] = [[] for _ in range(world)]
    for u in range(units):
        lo = 0
        while lo < nq:  # tiles of unit u by owner (owner is monotone in (u, i))
            r = owner(u, lo)
            hi = lo
            while hi < nq and owner(u, hi) == r:
                hi += 1
            runs[r].append((u, lo, hi))
            lo = hi
    out: list[list[Piece]] = []
    for items in runs:
        pieces: list[Piece] = []
        for u, lo, hi in items:
            last = pieces[-1] if pieces else None
            if (last and lo == 0 and hi == nq and last.tile0 == 0 and last.ntiles == nq
                    and last.stop == u):
                pieces[-1] = Piece(last.start, u + 1, 0, nq)  # extend a run of whole units
            else:
                pieces.append(Piece(u, u + 1, lo, hi - lo))
        out.append(pieces)
    return out


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


def pieces_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, pieces: list[Piece],
                   compute: Callable | None = None, **kw) -> list[tuple[int, int, int, torch.Tensor]]:
    """Run a rank's pieces (one compute call each; a partial tile range passes q_tiles) and
    return [(unit, row0, row1, O rows)] with O rows (1, Hq/Hkv, row1 - row0, d)."""
    compute = compute or _default_compute
    g, S1 = q.shape[1] // k.shape[1], q.shape[2]
    out = []
    for pc in pieces:
        if pc.stop <= pc.start or pc.ntiles <= 0:
            continue
        nq = (S1 + 127) // 128
        part = {} if (pc.tile0 == 0 and pc.ntiles == nq) else {"q_tiles": (pc.tile0, pc.ntiles)}
        o = compute(*_shard_views(q, k, v, pc.start, pc.stop), **part, **kw)
        r0, r1 = 128 * pc.tile0, min(S1, 128 * (pc.tile0 + pc.ntiles))
        out += [(u, r0, r1, o[:, i * g:(i + 1) * g, r0:r1]) for i, u in enumerate(range(pc.start, pc.stop))]
    return out


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
    work = partition_work(B, Hkv, S1, k.shape[2], bool(kw.get("causal", False)), world, kw.get("s2", 128))
    mine = pieces_forward(q, k, v, work[rank], compute, **kw)
    if not gather:
        return mine
    g = Hq // Hkv
    out = torch.empty_like(q)

    def put(lst, dev):
        for u, r0, r1, o in lst:
            b, h = divmod(u, Hkv)
            out[b:b + 1, h * g:(h + 1) * g, r0:r1] = o.to(dev)
    put(mine, out.device)
    if world > 1:
        allp = [None] * world
        dist.all_gather_object(allp, [(u, r0, r1, o.cpu()) for u, r0, r1, o in mine], group=group)
        for r, lst in enumerate(allp):
            if r != rank:
                put(lst, out.device)
    return out
