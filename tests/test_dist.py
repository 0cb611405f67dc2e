"""Multi-process (gloo, world_size 2, CPU) coverage of the sharding logic used on
NVLink/NCCL: request shards, KV-head slices, replicated page tables (rank 0 allocates,
others adopt the broadcast slot lists and end in the same allocator state), the
per-layer head all-gather and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import dist as kdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        # batch-parallel shards
        rids = [f"r{i}" for i in range(11)]
        res["shard"] = kdist.shard_requests(rids, rank, world)
        # head slices (cfg4 shape: 8 kv / 64 q heads)
        kvs, qs = kdist.head_slice(8, 64, rank, world)
        res["heads"] = (kvs.start, kvs.stop, qs.start, qs.stop)
        # replicated page tables: rank 0 allocates, rank 1 adopts
        cfg = kv.PoolConfig(total_slots=4096, offset=2048, n_layers=1, n_kv_heads=4, head_dim=128)
        pool = kv.MixedPrecisionPool(cfg, materialize=False)
        rng = np.random.default_rng(0)
        tables = []
        for i in range(6):
            bits = rng.choice([2, 4], size=int(rng.integers(50, 400)), p=[0.8, 0.2])
            if rank == 0:
                slots = pool.alloc(f"q{i}", bits).slots
            else:
                slots = None
            slots = kdist.broadcast_slots(slots)
            if rank != 0:
                kdist.adopt_table(pool, f"q{i}", slots)
            tables.append(pool.table(f"q{i}").slots.tolist())
            if i == 2:
                pool.free("q1")
        pool.check_invariants()
        res["tables"] = tables
        res["free"] = (pool._free_pages[-5:], pool._free_int4[-5:], len(pool._free_pages), len(pool._free_int4))
        # head all-gather: rank r's slice carries value 100*r + local head index
        B, hl, d = 3, 32 // world, 4
        local = torch.zeros(B, hl, d)
        for h in range(hl):
            local[:, h, :] = 100 * rank + h
        full = kdist.gather_heads(local)
        res["gather"] = full[:, :, 0].tolist()
        res["tmax"] = kdist.max_over_ranks(1.5 + rank)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharding():
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert out[0]["shard"] + out[1]["shard"] == [f"r{i}" for i in range(11)]
    assert out[0]["heads"] == (0, 4, 0, 32) and out[1]["heads"] == (4, 8, 32, 64)
    assert out[0]["tables"] == out[1]["tables"]          # replicated page tables
    assert out[0]["free"] == out[1]["free"]              # identical allocator state
    expect = [[h for h in range(16)] + [100 + h for h in range(16)]] * 3
    assert out[0]["gather"] == expect and out[1]["gather"] == expect
    assert out[0]["tmax"] == out[1]["tmax"] == 2.5
