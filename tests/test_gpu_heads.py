"""KV-head-parallel decode (cfg4) executed on one GPU.

A full pool's KV heads are split into S = 2, 4, 8 shards exactly as ``dist`` splits them
across ranks: every shard pool runs the same allocator sequence (slot addresses are
head-agnostic, pool.py:108-110, so the page tables agree), quantizes only its head slice
and decodes only its GQA q-head slice (kv = h // ratio, attention.py:198-201).  The
shard outputs, concatenated along heads as the all-gather does, must equal the unsharded
decode bit for bit when both run the same per-unit schedule (one CTA: every (request,
kv head) unit is one piece), and stay within the north_star tolerance of the oracle under
the default stream-K plan.
"""
import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import dist as kvdist
from oracle import attention as oatt
from oracle import pool as opool

pytestmark = pytest.mark.gpu
ATOL, RTOL = 2e-3, 1e-2


def bf16_exact(x):
    return torch.as_tensor(np.asarray(x, np.float32)).to(torch.bfloat16).float().numpy()


def make_pool(H, d, L, total, offset):
    return kv.MixedPrecisionPool(kv.PoolConfig(total_slots=total, offset=offset, n_layers=L, n_kv_heads=H,
                                               head_dim=d))


@pytest.fixture(scope="module")
def data():
    rng = np.random.default_rng(404)
    L, H, Hq, d = 2, 8, 32, 128
    lens = [700, 1531, 3000]
    bits = [np.where(rng.random(n) < 0.8, 2, 4) for n in lens]
    ch = np.exp(rng.uniform(np.log(0.5), np.log(4.0), (H, d)))
    kvs = [(bf16_exact(rng.standard_normal((L, n, H, d)) * ch), bf16_exact(rng.standard_normal((L, n, H, d))))
           for n in lens]
    q = bf16_exact(rng.standard_normal((L, len(lens), Hq, d)))
    return dict(L=L, H=H, Hq=Hq, d=d, lens=lens, bits=bits, kvs=kvs, q=q, total=12000, offset=6400)


def build(data, heads: slice):
    """A pool holding only KV heads `heads` of every request (rank-local view)."""
    H = heads.stop - heads.start
    pool = make_pool(H, data["d"], data["L"], data["total"], data["offset"])
    rids = []
    for r, (b, (k, v)) in enumerate(zip(data["bits"], data["kvs"])):
        t = pool.alloc(f"r{r}", b)
        pool.write_prefill(t, torch.as_tensor(k[:, :, heads]).to(torch.bfloat16),
                           torch.as_tensor(v[:, :, heads]).to(torch.bfloat16))
        pool.partition(t)
        rids.append(f"r{r}")
    return pool, rids


def decode(pool, rids, q, layer, **plan):
    b = kv.DecodeBatch(pool, rids, n_q_heads=q.shape[1], **plan)
    out = torch.empty(q.shape, dtype=torch.float32, device="cuda")
    kv.flash_decode_batched(torch.as_tensor(q, device="cuda").to(torch.bfloat16), b, layer, out=out)
    return out


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_head_shards_equal_unsharded(cuda, data, shards):
    H, Hq = data["H"], data["Hq"]
    full, rids = build(data, slice(0, H))
    for layer in range(data["L"]):
        q = data["q"][layer]
        ref_one = decode(full, rids, q, layer, n_cta=1)
        ref_sk = decode(full, rids, q, layer)
        parts_one, parts_sk = [], []
        for r in range(shards):
            kvh, qh = kvdist.head_slice(H, Hq, r, shards)
            pool, _ = build(data, kvh)
            for rid in rids:  # replicated page tables: identical slots on every shard
                assert np.array_equal(pool.table(rid).slots, full.table(rid).slots)
            parts_one.append(decode(pool, rids, q[:, qh], layer, n_cta=1))
            parts_sk.append(decode(pool, rids, q[:, qh], layer))
        got_one = torch.cat(parts_one, dim=1)  # what all_gather along heads assembles
        got_sk = torch.cat(parts_sk, dim=1)
        assert torch.equal(got_one, ref_one), f"{shards} shards, layer {layer}: not bit-identical"
        torch.testing.assert_close(got_sk, ref_sk, atol=1e-5, rtol=1e-5)


def test_head_shards_vs_oracle(cuda, data):
    """The assembled 4-shard output against the reference's fp32 flash_decode."""
    H, Hq, d, L = data["H"], data["Hq"], data["d"], data["L"]
    op = opool.OraclePool(opool.Config(data["total"], data["offset"], L, H, d))
    for r, (b, (k, v)) in enumerate(zip(data["bits"], data["kvs"])):
        op.alloc(f"r{r}", b)
        op.write_prefill(f"r{r}", k, v)
        op.partition(f"r{r}")
    layer, shards = 1, 4
    q = data["q"][layer]
    parts = []
    for r in range(shards):
        kvh, qh = kvdist.head_slice(H, Hq, r, shards)
        pool, rids = build(data, kvh)
        parts.append(decode(pool, rids, q[:, qh], layer))
    out = torch.cat(parts, dim=1).cpu().numpy()
    for i in range(len(data["lens"])):
        ref = oatt.flash_decode_pool(q[i], op, f"r{i}", layer)
        err = np.abs(out[i] - ref)
        assert np.all(err <= ATOL + RTOL * np.abs(ref)), f"request {i}: max abs err {err.max():.3e}"


@pytest.mark.parametrize("shards,dtype,n_dest", [(2, torch.float32, 3), (4, torch.bfloat16, 3), (8, torch.float32, 3),
                                                  (8, torch.float16, 8)])
def test_fused_head_gather(cuda, data, shards, dtype, n_dest):
    """The combine fused into the kernel (kvmix_flash_decode_gather): every shard's decode stores
    its head slice into all destination buffers -- here 3 or 8 (the maximum) buffers of this process standing in
    for the ranks' NVLink-mapped outputs -- and each buffer ends up equal to the unsharded decode
    (bit for bit under the per-unit schedule, like the all-gather path)."""
    H, Hq, d = data["H"], data["Hq"], data["d"]
    full, rids = build(data, slice(0, H))
    layer = 1
    q = data["q"][layer]
    B = len(rids)
    ref = decode(full, rids, q, layer, n_cta=1).to(dtype)
    dests = [torch.full((B, Hq, d), float("nan"), dtype=dtype, device="cuda") for _ in range(n_dest)]
    for r in range(shards):
        kvh, qh = kvdist.head_slice(H, Hq, r, shards)
        pool, _ = build(data, kvh)
        b = kv.DecodeBatch(pool, rids, n_q_heads=qh.stop - qh.start, n_cta=1)
        res = kv.flash_decode_batched(torch.as_tensor(q[:, qh], device="cuda").to(torch.bfloat16), b, layer,
                                      gather=kvdist.HeadOutputs.local(dests, head0=qh.start))
        assert res is None
    for i, o in enumerate(dests):
        assert torch.equal(o, ref), f"destination {i}: differs from the unsharded decode"
    # out and gather together, or a head slice past the buffers, are rejected
    with pytest.raises(kv.ValidationError):
        kv.flash_decode_batched(torch.as_tensor(q, device="cuda").to(torch.bfloat16), kv.DecodeBatch(full, rids, n_q_heads=Hq),
                                layer, out=dests[0], gather=kvdist.HeadOutputs.local(dests, head0=0))
    with pytest.raises(kv.ValidationError):
        kvh, qh = kvdist.head_slice(H, Hq, shards - 1, shards)
        pool, _ = build(data, kvh)
        kv.flash_decode_batched(torch.as_tensor(q[:, qh], device="cuda").to(torch.bfloat16),
                                kv.DecodeBatch(pool, rids, n_q_heads=qh.stop - qh.start), layer,
                                gather=kvdist.HeadOutputs.local(dests, head0=qh.start + 1))


def test_symmetric_head_gather_one_rank(cuda, data):
    """The multi-rank combine's real plumbing on a one-rank NCCL group: symmetric-memory
    allocation and rendezvous, the per-layer destination pointers, the fused-gather decode into
    them and the device barrier; the symmetric output equals the plain decode bit for bit."""
    import socket

    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        H, Hq, d, L = data["H"], data["Hq"], data["d"], data["L"]
        full, rids = build(data, slice(0, H))
        sg = kvdist.SymmetricHeadGather(L, len(rids), Hq, d, dtype=torch.bfloat16, device="cuda")
        b = kv.DecodeBatch(full, rids, n_q_heads=Hq)
        for layer in range(L):
            q = torch.as_tensor(data["q"][layer], device="cuda").to(torch.bfloat16)
            assert kv.flash_decode_batched(q, b, layer, gather=sg.layer(layer)) is None
        sg.barrier()
        torch.cuda.synchronize()
        for layer in range(L):
            q = torch.as_tensor(data["q"][layer], device="cuda").to(torch.bfloat16)
            ref = kv.flash_decode_batched(q, b, layer, out=torch.empty(q.shape, dtype=torch.bfloat16, device="cuda"))
            assert torch.equal(sg.out[layer], ref), f"layer {layer}"
    finally:
        dist.destroy_process_group()
