"""Multi-process (world_size 2, gloo, CPU) tests of the sharded path: the
partition covers every (b, kv head) unit exactly once, and the sharded +
gathered output equals the single-process output bit for bit.  The per-unit
compute here is the CPU kernel-numerics model from the oracle (test
infrastructure); on the GPU the same code path runs the fused kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_01873_b200.multi import partition, partition_work, pasa_attention_sharded, tile_costs


def test_partition_balanced_and_complete():
    for B, H, W in [(1, 4, 2), (1, 28, 8), (2, 4, 8), (3, 5, 4), (1, 1, 2)]:
        shards = partition(B, H, W)
        units = [u for s in shards for u in s.units()]
        assert units == list(range(B * H))
        sizes = [s.stop - s.start for s in shards]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("B,H,S,causal,W", [(1, 4, 16384, True, 8), (1, 4, 4096, False, 8), (2, 4, 1024, True, 3),
                                             (1, 28, 1024, True, 8), (1, 1, 1000, False, 4), (3, 5, 256, False, 4),
                                             (1, 2, 384, True, 1), (2, 2, 128, True, 8)])
def test_partition_work_covers_and_balances(B, H, S, causal, W):
    """(b, kv head) ranges, then query tiles: every (unit, tile) item exactly
    once, at most three pieces (launches) per rank, loads within one tile's cost."""
    work = partition_work(B, H, S, S, causal, W)
    cost = tile_costs(S, S, causal)
    nq = len(cost)
    seen = []
    loads = []
    for pieces in work:
        assert len(pieces) <= 3
        load = 0
        for pc in pieces:
            for u in range(pc.start, pc.stop):
                for i in range(pc.tile0, pc.tile0 + pc.ntiles):
                    seen.append((u, i))
                    load += cost[i]
        loads.append(load)
    assert sorted(seen) == [(u, i) for u in range(B * H) for i in range(nq)]
    if B * H * nq >= W:
        assert max(loads) - min(loads) <= max(cost)


def _model_compute(q, k, v, causal=False, q_tiles=None):  # (a tile range: computed whole, sliced by the caller)
    from oracle.oracle import Oracle, Problem
    orc = Oracle()
    o = orc.model_pasa(Problem(q.double().numpy(), k.double().numpy(), v.double().numpy(),
                               causal=causal), threads=1)
    return torch.from_numpy(o).half()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, k, v, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = pasa_attention_sharded(q, k, v, compute=_model_compute, causal=True)
        if rank == 0:
            torch.save(o, out_path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Hkv", [2, 1])
def test_sharded_equals_single_process(tmp_path, orc, Hkv):
    # Hkv = 1: one unit for two ranks -> the query tiles are split
    q, k, v = orc.generate("hybrid", 3.0, 10.0, 11, 1, 4, 256, 64, Hkv=Hkv)
    q, k, v = (torch.from_numpy(x).half() for x in (q, k, v))
    single = _model_compute(q, k, v, causal=True)
    out = str(tmp_path / "o.pt")
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, out), nprocs=2, join=True)
    sharded = torch.load(out)
    assert torch.equal(sharded, single)


def test_shard_forward_one_call_per_shard():
    """a shard is ONE compute call over its contiguous (b, kv head) units (views,
    no per-unit launches), and the per-unit outputs it returns are that call's slices."""
    from paper_2503_01873_b200.multi import Shard, shard_forward
    B, Hq, Hkv, S, d = 2, 6, 3, 8, 4
    q = torch.arange(B * Hq * S * d, dtype=torch.float32).reshape(B, Hq, S, d)
    k = -torch.arange(B * Hkv * S * d, dtype=torch.float32).reshape(B, Hkv, S, d)
    v = k * 2
    calls = []

    def compute(qs, ks, vs, **kw):
        calls.append((qs.shape, ks.shape, vs.shape, kw))
        return qs * 10  # stand-in: any per-row function of the shard's Q
    out = shard_forward(q, k, v, Shard(0, 1, 5), compute=compute, causal=True)
    assert len(calls) == 1
    assert calls[0][0] == (1, 8, S, d) and calls[0][1] == (1, 4, S, d) and calls[0][3] == {"causal": True}
    assert [u for u, _ in out] == [1, 2, 3, 4]
    for u, o in out:
        b, h = divmod(u, Hkv)
        assert torch.equal(o, q[b:b + 1, 2 * h:2 * h + 2] * 10)
    assert shard_forward(q, k, v, Shard(1, 3, 3), compute=compute) == [] and len(calls) == 1
