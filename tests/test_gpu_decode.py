"""K2 split-K mixed INT2/INT4 decode attention on the GPU vs the reference
flash_decode (golden outputs) and the oracle restatement: within the north_star
tolerance (atol 2e-3, rtol 1e-2 vs fp32 dequant-attention), plus size-independent
properties at the Qwen3-VL-32B shape (32K tokens, 64 q / 8 kv heads)."""
import math

import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from oracle import attention as oatt
from oracle import pool as opool

from conftest import rand_kv

pytestmark = pytest.mark.gpu
ATOL, RTOL = 2e-3, 1e-2


def close(out, ref, atol=ATOL, rtol=RTOL):
    err = np.abs(np.asarray(out, np.float64) - ref)
    return bool(np.all(err <= atol + rtol * np.abs(ref))), float(err.max())


def build(seed, n, n_kv, d, frac, L=1, headroom=64):
    rng = np.random.default_rng(seed)
    bits = np.where(rng.random(n) < frac, 2, 4)
    k, v = rand_kv(seed, L, n, n_kv, d)
    offset = -(-int((bits == 2).sum()) // 32) * 32
    cfg = kv.PoolConfig(total_slots=offset + n + headroom, offset=offset, n_layers=L, n_kv_heads=n_kv, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    t = pool.alloc("req", bits)
    pool.write_prefill(t, k, v)
    pool.partition(t)
    op = opool.OraclePool(opool.Config(cfg.total_slots, cfg.offset, L, n_kv, d))
    op.alloc("req", bits)
    op.write_prefill("req", k, v)
    op.partition("req")
    return pool, t, op, k, v, bits


@pytest.mark.parametrize("i", range(12))
def test_golden_reference_outputs(cuda, golden, i):
    d, n_kv, H, n, total, offset = (int(x) for x in golden["dec_meta"][i])
    pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=total, offset=offset, n_layers=1, n_kv_heads=n_kv,
                                               head_dim=d))
    t = pool.alloc("req", golden[f"dec{i}_bits"])
    pool.write_prefill(t, golden[f"dec{i}_keys"].astype(np.float32), golden[f"dec{i}_values"].astype(np.float32))
    pool.partition(t)
    ok, err = close(kv.flash_decode(golden[f"dec{i}_q"], t, pool.view(0), variant=0), golden[f"dec{i}_out"])
    assert ok, err
    # fp32 q through the drop-in API defaults to the fp32-faithful kernel: the reference's own
    # bar for flash_decode (pkg/tests/test_attention.py:205-246, relative to max |out|)
    out = kv.flash_decode(golden[f"dec{i}_q"], t, pool.view(0))
    ref = golden[f"dec{i}_out"]
    assert np.abs(out - ref).max() / np.abs(ref).max() < 1e-5


def test_random_instances_vs_oracle(cuda):
    """test_acceptance.py:139-160 shape: 200 random instances, d in {32, 64, 128}, GQA 1..8."""
    rng = np.random.default_rng(103)
    worst = 0.0
    for i in range(200):
        d = int(rng.choice([32, 64, 128]))
        n_kv = int(rng.choice([1, 2, 4]))
        H = n_kv * int(rng.choice([1, 2, 4, 8]))
        n = int(rng.integers(1, 1200))
        pool, t, op, *_ = build(1000 + i, n, n_kv, d, float(rng.uniform(0, 1)))
        q = rng.standard_normal((H, d)).astype(np.float32)
        ref = oatt.flash_decode_pool(q, op, "req", 0)
        ok, err = close(kv.flash_decode(q, t, pool.view(0), variant=0), ref)
        worst = max(worst, err)
        assert ok, (i, d, n_kv, H, n, err)
        # the CUDA-core variant is an fp32 restatement: much tighter
        ok2, err2 = close(kv.flash_decode(q, t, pool.view(0), variant=1), ref, atol=1e-5, rtol=1e-5)
        assert ok2, (i, err2)
    print(f"worst abs err over 200 instances: {worst:.2e}")


def test_layers_from_host_matches_device_api(cuda):
    """The overlapped host-I/O step gives exactly the per-layer device API's outputs."""
    L, H, d = 5, 2, 128
    rng = np.random.default_rng(3)
    cfg = kv.PoolConfig(total_slots=4096, offset=2048, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    rids = []
    for r in range(3):
        n = int(rng.integers(100, 900))
        t = pool.alloc(f"r{r}", np.where(rng.random(n) < 0.8, 2, 4))
        k, v = rand_kv(40 + r, L, n, H, d)
        pool.write_prefill(t, k, v)
        pool.partition(t)
        rids.append(f"r{r}")
    b = kv.DecodeBatch(pool, rids, n_q_heads=8)
    q = torch.randn((L, 3, 8, d), device=cuda).to(torch.bfloat16)
    ref = torch.stack([kv.flash_decode_batched(q[l], b, l) for l in range(L)]).cpu()
    q_host = q.cpu().pin_memory()
    o_host = torch.empty_like(q_host).pin_memory()
    for chunk in (1, 2, 8):
        o_host.zero_()
        kv.flash_decode_layers_from_host(q_host, b, o_host, chunk=chunk)
        torch.cuda.synchronize()
        assert torch.equal(o_host, ref), chunk


def test_edge_cases(cuda):
    rng = np.random.default_rng(0)
    for n, frac in [(1, 0.0), (32, 1.0), (33, 1.0), (31, 1.0), (64, 0.5), (1000, 1.0), (1000, 0.0)]:
        pool, t, op, *_ = build(n, n, 2, 128, frac)
        q = rng.standard_normal((16, 128)).astype(np.float32)
        ok, err = close(kv.flash_decode(q, t, pool.view(0), variant=0), oatt.flash_decode_pool(q, op, "req", 0))
        assert ok, (n, frac, err)


def test_split_invariance_and_validation(cuda):
    pool, t, op, *_ = build(19, 500, 2, 64, 0.7)
    q = np.random.default_rng(20).standard_normal((4, 64)).astype(np.float32)
    outs = [kv.flash_decode(q, t, pool.view(0), split_len=s, variant=0) for s in (1, 7, 32, 128, 512)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    qd = torch.as_tensor(q, device=cuda)[None]
    ref = outs[0]
    # other CTA counts change the stream-K cuts (which CTA / warp sees which tiles, how many
    # partials a unit merges, several units per CTA when n_cta < units): the running max and
    # fp16 rounding of p*s move, so agreement is to ~1e-4 -- well inside the parity tolerance.
    # Each plan runs twice: the arrival counters must be left at zero by every launch.
    for n_cta in (1, 2, 3, 5, 8, 13, 64, 444):
        b = kv.DecodeBatch(pool, ["req"], n_q_heads=4, n_cta=n_cta)
        for rep in range(2):
            o = kv.flash_decode_batched(qd, b, 0).cpu().numpy()[0]
            assert np.allclose(o, ref, rtol=2e-3, atol=2e-4), (n_cta, rep, float(np.abs(o - ref).max()))
        assert int(b.counters.abs().sum()) == 0
    with pytest.raises(kv.ValidationError):
        kv.flash_decode(q, t, pool.view(0), split_len=0)
    with pytest.raises(kv.ValidationError):
        kv.flash_decode(q[0], t, pool.view(0))
    with pytest.raises(kv.ValidationError):
        kv.flash_decode(np.zeros((3, 64), np.float32), t, pool.view(0))
    t2 = pool.alloc("mixed", np.array([4] * 8 + [2] * 32))
    k, v = rand_kv(22, 1, 40, 2, 64)
    pool.write_prefill(t2, k, v)
    with pytest.raises(kv.ValidationError, match="not partitioned"):
        kv.flash_decode(q, t2, pool.view(0))
    empty = kv.PageTable("e", [], partitioned=True)
    with pytest.raises(kv.ValidationError, match="empty"):
        kv.flash_decode(q, empty, pool.view(0))


def test_batched_mixed_lengths_and_dtypes(cuda):
    L, n_kv, d, H = 2, 4, 128, 32
    rng = np.random.default_rng(7)
    lens = [1, 31, 32, 100, 2000, 4321]
    cfg = kv.PoolConfig(total_slots=20000, offset=12000, n_layers=L, n_kv_heads=n_kv, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(20000, 12000, L, n_kv, d))
    rids = []
    for r, n in enumerate(lens):
        bits = np.where(rng.random(n) < 0.8, 2, 4)
        k, v = rand_kv(r, L, n, n_kv, d)
        t = pool.alloc(f"r{r}", bits)
        op.alloc(f"r{r}", bits)
        pool.write_prefill(t, k, v)
        op.write_prefill(f"r{r}", k, v)
        pool.partition(t)
        op.partition(f"r{r}")
        rids.append(f"r{r}")
    batch = kv.DecodeBatch(pool, rids, n_q_heads=H)
    q = torch.randn(len(lens), H, d, device=cuda)
    for layer in range(L):
        for qd, od in [(torch.float32, torch.float32), (torch.bfloat16, torch.bfloat16),
                       (torch.float16, torch.float32)]:
            qq = q.to(qd)
            out = torch.empty(len(lens), H, d, dtype=od, device=cuda)
            kv.flash_decode_batched(qq, batch, layer, out=out)
            for r in range(len(lens)):
                ref = oatt.flash_decode_pool(qq[r].float().cpu().numpy(), op, f"r{r}", layer)
                ok, err = close(out[r].float().cpu().numpy(), ref)
                assert ok, (layer, qd, od, r, err)


@pytest.mark.parametrize("d", [32, 64, 128])
def test_long_pieces_every_head_dim(cuda, d):
    """Long single pieces at every head dim: each warp runs several batches of 16 INT2 pages
    through the batched key bias (the zero points staged one batch ahead into the merge
    scratch), for fp32, bf16 and f16 q, under the one-CTA schedule and the stream-K default."""
    n, n_kv, H = 9000, 2, 8
    pool, t, op, *_ = build(900 + d, n, n_kv, d, 0.85)
    batch_one = kv.DecodeBatch(pool, ["req"], n_q_heads=H, n_cta=1)
    batch_sk = kv.DecodeBatch(pool, ["req"], n_q_heads=H)
    rng = np.random.default_rng(d)
    q = torch.as_tensor(rng.standard_normal((1, H, d)).astype(np.float32), device=cuda)
    for qd in (torch.float32, torch.bfloat16, torch.float16):
        qq = q.to(qd)
        ref = oatt.flash_decode_pool(qq[0].float().cpu().numpy(), op, "req", 0)
        for b in (batch_one, batch_sk):
            out = kv.flash_decode_batched(qq, b, 0, out=torch.empty(1, H, d, device=cuda))
            ok, err = close(out[0].cpu().numpy(), ref)
            assert ok, (d, qd, b.n_cta, err)


def test_decode_after_append(cuda):
    pool, t, op, *_ = build(5, 700, 2, 128, 0.8, L=2, headroom=128)
    rng = np.random.default_rng(1)
    for _ in range(40):
        kk = rng.standard_normal((2, 2, 128)).astype(np.float32)
        vv = rng.standard_normal((2, 2, 128)).astype(np.float32)
        a = pool.append_decode_token("req", kk, vv)
        s = op.pop_decode_slot("req")
        op.write_decode(s, kk, vv)
        assert a.index == s
    q = rng.standard_normal((16, 128)).astype(np.float32)
    for layer in range(2):
        ok, err = close(kv.flash_decode(q, t, pool.view(layer)), oatt.flash_decode_pool(q, op, "req", layer))
        assert ok, err


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fused_decode_append(cuda, dtype):
    """K4 fused into K2: reserve one INT4 slot per request, then per layer one launch both
    writes the new token (bit-exact with the reference INT4 TokenBlocks) and attends to it."""
    L, H, Hq, d = 3, 2, 8, 128
    rng = np.random.default_rng(9)
    cfg = kv.PoolConfig(total_slots=8192, offset=4096, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(8192, 4096, L, H, d))
    rids = [f"r{i}" for i in range(4)]
    for i, rid in enumerate(rids):
        n = int(rng.integers(30, 1500))
        bits = np.where(rng.random(n) < 0.8, 2, 4)
        k, v = rand_kv(70 + i, L, n, H, d)
        t = pool.alloc(rid, bits)
        op.alloc(rid, bits)
        pool.write_prefill(t, k, v)
        op.write_prefill(rid, k, v)
        pool.partition(t)
        op.partition(rid)
    for step in range(3):
        slots = pool.reserve_decode_slots(rids)
        assert slots.tolist() == [op.pop_decode_slot(r) for r in rids]
        b = kv.DecodeBatch(pool, rids, n_q_heads=Hq)
        kn = torch.as_tensor(rng.standard_normal((len(rids), L, H, d)).astype(np.float32), device=cuda).to(dtype)
        vn = torch.as_tensor(rng.standard_normal((len(rids), L, H, d)).astype(np.float32), device=cuda).to(dtype)
        for i, rid in enumerate(rids):
            op.write_decode(int(slots[i]), kn[i].float().cpu().numpy(), vn[i].float().cpu().numpy())
        q = rng.standard_normal((L, len(rids), Hq, d)).astype(np.float32)
        for layer in range(L):
            out = kv.flash_decode_batched(torch.as_tensor(q[layer], device=cuda), b, layer,
                                          append=(kn[:, layer], vn[:, layer])).cpu().numpy()
            for i, rid in enumerate(rids):
                ok, err = close(out[i], oatt.flash_decode_pool(q[layer, i], op, rid, layer))
                assert ok, (step, layer, rid, err)
    torch.cuda.synchronize()
    assert_same_pool(pool, op)


def assert_same_pool(pool, op):
    from paper_2605_17170_b200 import layout
    d, L, H = pool.config.head_dim, pool.config.n_layers, pool.config.n_kv_heads
    i2 = pool.int2_pool[: L * H * pool.n_pages * pool.page_stride].view(L, H, pool.n_pages, pool.page_stride)
    i4 = pool.int4_pool[: L * H * pool.n_int4 * pool.slot_stride].view(L, H, pool.n_int4, pool.slot_stride)
    i2, i4 = i2.cpu().numpy(), i4.cpu().numpy()
    assert np.array_equal(layout.page_payloads(i2[op.page_written], d), op.int2[op.page_written])
    assert np.array_equal(i4[op.slot_written], layout.slot_records(op.int4[op.slot_written], d))
    assert np.array_equal(pool._int4_written, op.slot_written)


def test_cuda_graph_capture(cuda):
    pool, t, op, *_ = build(8, 3000, 2, 128, 0.8)
    batch = kv.DecodeBatch(pool, ["req"], n_q_heads=16)
    q = torch.randn(1, 16, 128, device=cuda)
    out = torch.empty_like(q)
    kv.flash_decode_batched(q, batch, 0, out=out)
    eager = out.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            kv.flash_decode_batched(q, batch, 0, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


# ---- full-size (Qwen3-VL-32B layer shape, 32K tokens) size-independent properties ----------
def big_pool(seed, n=32768, n_kv=8, d=128, frac=0.83, k_fn=None):
    rng = np.random.default_rng(seed)
    bits = np.where(rng.random(n) < frac, 2, 4)
    cfg = kv.PoolConfig(total_slots=n + 64, offset=int((bits == 2).sum()) // 32 * 32, n_layers=1, n_kv_heads=n_kv,
                        head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    t = pool.alloc("big", bits)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.randn(1, n, n_kv, d, device="cuda", generator=gen) if k_fn is None else k_fn(n, n_kv, d)
    v = torch.randn(1, n, n_kv, d, device="cuda", generator=gen)
    pool.write_prefill(t, k.to(torch.bfloat16), v.to(torch.bfloat16))
    pool.partition(t)
    return pool, t, v


def test_fullsize_tensor_core_vs_cuda_core(cuda):
    pool, t, _ = big_pool(1)
    b = kv.DecodeBatch(pool, ["big"], n_q_heads=64)
    q = torch.randn(1, 64, 128, device=cuda)
    a = kv.flash_decode_batched(q, b, 0)
    c = kv.flash_decode_batched(q, b, 0, variant=1)
    err = (a - c).abs()
    assert bool((err <= ATOL + RTOL * c.abs()).all()), float(err.max())


def test_fullsize_uniform_keys_give_mean_value(cuda):
    """Identical keys -> uniform attention -> output = mean of the dequantized values."""
    pool, t, _ = big_pool(2, k_fn=lambda n, h, d: torch.ones(1, n, h, d, device="cuda").mul_(0.5))
    b = kv.DecodeBatch(pool, ["big"], n_q_heads=64)
    q = torch.randn(1, 64, 128, device=cuda)
    out = kv.flash_decode_batched(q, b, 0)[0]
    kd, vd = pool._gather_dev(t.slots, 0)  # K5 gather-dequant (checked bit-exact in test_gpu_pool)
    mean = vd.mean(dim=0)  # [Hkv, d]
    expect = mean.repeat_interleave(8, dim=0)
    assert torch.allclose(out, expect, atol=1e-4, rtol=1e-3), float((out - expect).abs().max())


def test_fullsize_page_order_invariance(cuda):
    pool, t, _ = big_pool(3, n=8192)
    q = torch.randn(1, 64, 128, device=cuda)
    b1 = kv.DecodeBatch(pool, ["big"], n_q_heads=64)
    o1 = kv.flash_decode_batched(q, b1, 0)
    s = t.slots
    n2 = int((s < pool.config.offset).sum())
    pages = s[:n2].reshape(-1, 32)[::-1].reshape(-1)
    perm = np.concatenate([pages, s[n2:][::-1]])
    b2 = kv.DecodeBatch(pool, n_q_heads=64, tables=[perm])
    o2 = kv.flash_decode_batched(q, b2, 0)
    assert torch.allclose(o1, o2, atol=2e-4, rtol=2e-3), float((o1 - o2).abs().max())


def test_fullsize_value_linearity(cuda):
    """Scaling V by 2 doubles every fp16 scale/zero exactly, so the output doubles."""
    torch.manual_seed(0)
    n, h, d = 16384, 8, 128
    bits = np.where(np.random.default_rng(4).random(n) < 0.8, 2, 4)
    k = torch.randn(1, n, h, d, device=cuda)
    v = torch.randn(1, n, h, d, device=cuda)
    outs = []
    for mult in (1.0, 2.0):
        cfg = kv.PoolConfig(total_slots=n + 32, offset=int((bits == 2).sum()) // 32 * 32, n_layers=1,
                            n_kv_heads=h, head_dim=d)
        pool = kv.MixedPrecisionPool(cfg)
        t = pool.alloc("r", bits)
        pool.write_prefill(t, k, v * mult)
        pool.partition(t)
        b = kv.DecodeBatch(pool, ["r"], n_q_heads=64)
        outs.append(kv.flash_decode_batched(torch.ones(1, 64, d, device=cuda) * 0.1, b, 0))
    assert torch.allclose(outs[1], 2 * outs[0], atol=1e-4, rtol=1e-3)


def test_merge_partials_gpu(cuda):
    rng = np.random.default_rng(16)
    parts = [kv.SplitPartial(acc=rng.standard_normal(8).astype(np.float32), lse=float(rng.uniform(-5, 5)),
                             max_logit=float(rng.uniform(-5, 5))) for _ in range(5)]
    a = kv.merge_partials(parts)
    b = oatt.merge([(p.acc, p.lse, p.max_logit) for p in parts])
    assert np.allclose(a, b, rtol=1e-5)
    big = kv.SplitPartial(acc=np.ones(4, np.float32) * 3, lse=1000.0, max_logit=1000.0)
    tiny = kv.SplitPartial(acc=np.ones(4, np.float32), lse=-1000.0, max_logit=-1000.0)
    assert np.allclose(kv.merge_partials([big, tiny]), 3.0, atol=1e-5)
    with pytest.raises(kv.ValidationError):
        kv.merge_partials([])
