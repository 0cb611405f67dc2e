"""Pool data plane on the GPU: write_prefill / append / gather produce exactly the
oracle's device image (every reference payload at its slot address) with the
reference's page indices; error behaviour and accounting follow pool.py."""
import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import layout
from oracle import pool as opool

from conftest import rand_kv

pytestmark = pytest.mark.gpu


def pool_images(pool):
    L, H = pool.config.n_layers, pool.config.n_kv_heads
    i2 = pool.int2_pool[: L * H * pool.n_pages * pool.page_stride].view(L, H, pool.n_pages, pool.page_stride)
    i4 = pool.int4_pool[: L * H * pool.n_int4 * pool.slot_stride].view(L, H, pool.n_int4, pool.slot_stride)
    return i2.cpu().numpy(), i4.cpu().numpy()


def assert_same_image(pool, op):
    """Every written record holds exactly the oracle's reference payloads: compared both
    as reference-order payloads recovered from the device records and as device records."""
    d = pool.config.head_dim
    i2, i4 = pool_images(pool)
    pw, sw = op.page_written, op.slot_written
    assert np.array_equal(layout.page_payloads(i2[pw], d), op.int2[pw])
    assert np.array_equal(layout.slot_payloads(i4[sw], d), op.int4[sw][:, : 2 * (d // 2 + d // 8)])
    assert np.array_equal(i2[pw], layout.page_records(op.int2[pw], d))
    assert np.array_equal(i4[sw], layout.slot_records(op.int4[sw], d))


@pytest.mark.parametrize("d,dtype", [(32, torch.float32), (64, torch.bfloat16), (128, torch.float32),
                                     (128, torch.bfloat16), (128, torch.float16), (256, torch.float32)])
def test_prefill_bytes_match_oracle(cuda, d, dtype):
    L, H = 2, 2
    cfg = kv.PoolConfig(total_slots=3000, offset=1600, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(3000, 1600, L, H, d))
    rng = np.random.default_rng(d)
    for r in range(5):
        n = int(rng.integers(1, 500))
        bits = rng.choice([2, 4], size=n, p=[0.8, 0.2])
        k, v = rand_kv(r, L, n, H, d)
        kt = torch.as_tensor(k, device=cuda).to(dtype)
        vt = torch.as_tensor(v, device=cuda).to(dtype)
        t = pool.alloc(f"r{r}", bits)
        assert t.slots.tolist() == op.alloc(f"r{r}", bits)
        pool.write_prefill(t, kt, vt)
        op.write_prefill(f"r{r}", kt.float().cpu().numpy(), vt.float().cpu().numpy())  # exact upcast
        if r == 2:
            pool.free("r1")
            op.free("r1")
    torch.cuda.synchronize()
    assert_same_image(pool, op)
    pool.check_invariants()


def _near_tie_values(rng, shape, levels):
    """Groups whose codes sit on or within a few ulps of the round-half-away ties
    (t = k + 1/2): the fast reciprocal code path must hand these to the exact path."""
    x = np.empty(shape, np.float32)
    flat = x.reshape(-1, 32)
    for gi in range(flat.shape[0]):
        s = np.float32(2.0 ** rng.integers(-4, 3))
        a = np.float32(rng.integers(-200, 200)) * s
        k = rng.integers(0, levels, 32)
        eps = rng.choice([0.0, 2 ** -23, -(2 ** -23), 2 ** -22, -(2 ** -22), 3e-7, -3e-7], 32)
        g = (a + (k + 0.5) * s * (1 + eps)).astype(np.float32)
        g[0], g[1] = a, a + np.float32(levels) * s  # exact min / max -> exact fp16 (scale, zero)
        flat[gi] = rng.permutation(g)
    return x


def test_prefill_near_ties_bit_exact(cuda):
    """Bit-exactness where it is hardest: values at and next to the rounding ties, for
    both the INT2 page path (per-channel keys, per-token values) and the INT4 path."""
    L, H, d, n = 1, 2, 128, 96
    rng = np.random.default_rng(11)
    bits = np.array([2] * 64 + [4] * 32)
    cfg = kv.PoolConfig(total_slots=256, offset=128, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(256, 128, L, H, d))
    # keys: ties along tokens within each channel of a page -> build [L, H, d, 32] groups then transpose
    kp = _near_tie_values(rng, (L, 2, H, d, 32), 3)  # 2 pages
    k2 = np.moveaxis(kp, 4, 2).reshape(L, 2 * 32, H, d)  # -> [L, tokens, H, d]
    v2 = _near_tie_values(rng, (L, 64, H, d), 3)
    k4 = _near_tie_values(rng, (L, 32, H, d), 15)
    v4 = _near_tie_values(rng, (L, 32, H, d), 15)
    k = np.concatenate([k2, k4], 1)
    v = np.concatenate([v2, v4], 1)
    t = pool.alloc("r", bits)
    assert t.slots.tolist() == op.alloc("r", bits)
    pool.write_prefill(t, k, v)
    op.write_prefill("r", k, v)
    torch.cuda.synchronize()
    assert_same_image(pool, op)


def test_gather_and_read_slot(cuda):
    L, H, d = 2, 2, 64
    cfg = kv.PoolConfig(total_slots=600, offset=320, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(600, 320, L, H, d))
    bits = np.array([2] * 70 + [4] * 30 + [2] * 40)
    k, v = rand_kv(9, L, bits.size, H, d)
    t = pool.alloc("r", bits)
    op.alloc("r", bits)
    pool.write_prefill(t, k, v)
    op.write_prefill("r", k, v)
    for layer in range(L):
        kg, vg = pool.view(layer).gather(t.entries)
        ko, vo = op.gather(t.slots, layer)
        assert np.array_equal(kg, ko) and np.array_equal(vg, vo)
    for i in (0, 31, 75, 120, 139):
        for h in range(H):
            ks, vs = pool.read_slot(t.entries[i], 1, h)
            ko, vo = op.gather([t.slots[i]], 1)
            assert np.array_equal(ks, ko[0, h]) and np.array_equal(vs, vo[0, h])


def test_append_decode_token(cuda):
    L, H, d = 3, 2, 128
    cfg = kv.PoolConfig(total_slots=256, offset=128, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(256, 128, L, H, d))
    bits = np.array([2] * 64 + [4] * 5)
    k, v = rand_kv(3, L, bits.size, H, d)
    t = pool.alloc("r", bits)
    op.alloc("r", bits)
    pool.write_prefill(t, k, v)
    op.write_prefill("r", k, v)
    with pytest.raises(kv.ValidationError):
        pool.append_decode_token("r", k[:, 0], v[:, 0])  # table not partitioned yet
    pool.partition(t)
    op.partition("r")
    rng = np.random.default_rng(0)
    for _ in range(7):
        kk = rng.standard_normal((L, H, d)).astype(np.float32)
        vv = rng.standard_normal((L, H, d)).astype(np.float32)
        a = pool.append_decode_token("r", kk, vv)
        s = op.pop_decode_slot("r")
        op.write_decode(s, kk, vv)
        assert a.index == s and not pool.is_int2(a) and t.slots[-1] == s
    assert_same_image(pool, op)
    # batched append (one token per request, all layers) == per-request appends
    kb = torch.as_tensor(rng.standard_normal((1, L, H, d)), dtype=torch.float32, device=cuda)
    slots = pool.append_decode_tokens(["r"], kb, kb)
    s = op.pop_decode_slot("r")
    op.write_decode(s, kb[0].cpu().numpy(), kb[0].cpu().numpy())
    assert slots.tolist() == [s]
    assert_same_image(pool, op)
    pool.check_invariants()


def test_write_page_and_token(cuda):
    cfg = kv.PoolConfig(total_slots=256, offset=128, n_layers=2, n_kv_heads=2, head_dim=32)
    pool = kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(256, 128, 2, 2, 32))
    pool.alloc("r", np.array([2] * 32 + [4]))
    op.alloc("r", np.array([2] * 32 + [4]))
    rng = np.random.default_rng(4)
    keys = rng.standard_normal((32, 32)).astype(np.float32)
    vals = rng.standard_normal((32, 32)).astype(np.float32)
    pool.write_page(0, keys, vals, 1, 1)
    k4 = rng.standard_normal(32).astype(np.float32)
    pool.write_token(kv.SlotAddress(128), k4, -k4, 0, 1)
    from oracle import codec
    i2, i4 = pool_images(pool)
    exp2 = np.concatenate([codec.encode_key_pages(keys), codec.encode_token_blocks(vals, 2).reshape(-1)])
    assert np.array_equal(layout.page_payloads(i2[1, 1, 0], 32), exp2)
    exp4 = np.concatenate([codec.encode_token_blocks(k4[None], 4)[0], codec.encode_token_blocks(-k4[None], 4)[0]])
    assert np.array_equal(layout.slot_payloads(i4[0, 1, 0], 32), exp4)
    with pytest.raises(kv.ValidationError):
        pool.write_page(0, np.zeros((16, 32)), np.zeros((16, 32)), 0, 0)
    with pytest.raises(kv.ValidationError):
        pool.write_token(kv.SlotAddress(0), np.zeros(32), np.zeros(32), 0, 0)
    with pytest.raises(kv.ValidationError):
        pool.write_page(5, keys, vals, 0, 0)


def test_errors_and_accounting(cuda):
    cfg = kv.PoolConfig(total_slots=256, offset=128, n_layers=1, n_kv_heads=1, head_dim=32)
    pool = kv.MixedPrecisionPool(cfg)
    t = pool.alloc("r", np.array([4]))
    with pytest.raises(kv.ValidationError):
        pool.read_slot(t.entries[0], 0, 0)  # read before write
    k, v = rand_kv(0, 1, 1, 1, 32)
    pool.write_prefill(t, k, v)
    addr = t.entries[0]
    pool.free("r")
    with pytest.raises(kv.ValidationError):
        pool.read_slot(addr, 0, 0)
    with pytest.raises(kv.ValidationError):
        pool.view(0).gather([kv.SlotAddress(5)])
    t = pool.alloc("p", np.array([2] * 32 + [4]))
    k, v = rand_kv(7, 1, 33, 1, 32)
    pool.write_prefill(t, k, v)
    assert pool.parameter_overhead_bytes() == 32 * 4 + 32 * 1 * 4 + 2 * 1 * 4  # test_pool.py:285-292
    bad = np.full((1, 33, 1, 32), np.nan, np.float32)
    pool.alloc("z", np.array([4] * 33))
    with pytest.raises(kv.ValidationError, match="finite"):
        pool.write_prefill(pool.table("z"), bad, bad)
    tiny = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=32, offset=32, n_layers=1, n_kv_heads=1, head_dim=32))
    t = tiny.alloc("r", np.array([2] * 32))
    k, v = rand_kv(5, 1, 32, 1, 32)
    tiny.write_prefill(t, k, v)
    tiny.partition(t)
    with pytest.raises(kv.CapacityError) as e:
        tiny.append_decode_token("r", np.zeros((1, 1, 32), np.float32), np.zeros((1, 1, 32), np.float32))
    assert e.value.region == "int4"


def test_fuzz_safety(cuda):
    """test_acceptance.py:304-342 pattern (criterion 9) on the device pool, 2000 ops."""
    pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=512, offset=288, n_layers=1, n_kv_heads=1, head_dim=32))
    rng = np.random.default_rng(109)
    live, nid = [], 0
    z = np.zeros((1, 1, 32), np.float32)
    for _ in range(2000):
        a = rng.random()
        try:
            if a < 0.45 or not live:
                bits = rng.choice([2, 4], size=int(rng.integers(1, 80)), p=[0.6, 0.4])
                t = pool.alloc(f"r{nid}", bits)
                assert int((t.slots < 288).sum()) == int((bits == 2).sum()) // 32 * 32
                live.append(f"r{nid}")
                nid += 1
            elif a < 0.8:
                pool.free(live.pop(int(rng.integers(len(live)))))
            else:
                rid = live[int(rng.integers(len(live)))]
                t = pool.partition(pool.table(rid))
                before = t.slots.tolist()
                pool.partition(t)
                assert t.slots.tolist()[: len(before)] == before
                pool.append_decode_token(rid, z, z)
        except kv.CapacityError:
            pass
        pool.check_invariants()


@pytest.mark.parametrize("d", [64, 128])
def test_alloc_device_matches_alloc_and_oracle(cuda, d):
    """K6 (device-side routing, pool.py:122-163): the same slots as the host allocator and
    the oracle, through frees that scramble the LIFO stacks, and the device index lists feed
    write_prefill to the oracle's exact image."""
    L, H = 2, 2
    cfg = kv.PoolConfig(total_slots=120000, offset=60000, n_layers=L, n_kv_heads=H, head_dim=d)
    dev_pool, host_pool = kv.MixedPrecisionPool(cfg), kv.MixedPrecisionPool(cfg)
    op = opool.OraclePool(opool.Config(120000, 60000, L, H, d))
    rng = np.random.default_rng(600 + d)
    sizes = [0, 1, 31, 32, 33, 64, 700, 16384, 16385, 20000]
    for r, n in enumerate(sizes):
        p2 = [0.8, 1.0, 0.0, 0.5][r % 4]
        bits = np.where(rng.random(n) < p2, 2, 4).astype(np.int64)
        src = torch.as_tensor(bits, device=cuda).to(torch.int8) if r % 2 else bits
        td = dev_pool.alloc_device(f"r{r}", src)
        th = host_pool.alloc(f"r{r}", bits)
        assert td.slots.tolist() == th.slots.tolist() == op.alloc(f"r{r}", bits)
        if n and n <= 700:
            k, v = rand_kv(r, L, n, H, d)
            kt, vt = torch.as_tensor(k, device=cuda), torch.as_tensor(v, device=cuda)
            dev_pool.write_prefill(td, kt, vt)
            op.write_prefill(f"r{r}", k, v)
        if r in (4, 7):  # free an earlier request: later pops come from a reordered stack
            for p in (dev_pool, host_pool):
                p.free(f"r{r - 2}")
            op.free(f"r{r - 2}")
    torch.cuda.synchronize()
    assert_same_image(dev_pool, op)
    dev_pool.check_invariants()
    assert dev_pool.free_counts() == host_pool.free_counts()


def test_alloc_device_errors(cuda):
    cfg = kv.PoolConfig(total_slots=1024, offset=512, n_layers=1, n_kv_heads=1, head_dim=64)
    pool = kv.MixedPrecisionPool(cfg)
    with pytest.raises(kv.ValidationError):
        pool.alloc_device("a", np.array([2, 3, 4]))
    with pytest.raises(kv.ValidationError):
        pool.alloc_device("a", torch.tensor([2, 4, 5], dtype=torch.int8, device=cuda))
    with pytest.raises(kv.CapacityError):
        pool.alloc_device("a", np.full(600, 2))
    with pytest.raises(kv.CapacityError):
        pool.alloc_device("a", np.full(600, 4))
    before = pool.free_counts()
    t = pool.alloc_device("a", np.full(64, 2))  # failed calls popped nothing
    assert pool.free_counts() == (before[0] - 64, before[1])
    with pytest.raises(kv.ValidationError):
        pool.alloc_device("a", np.full(4, 2))
    pool.free("a")
    assert len(t) == 64
    pool.check_invariants()


def test_gather_device_typed(cuda):
    """K5 with bf16 / f16 output (kvmix_gather_dequant_typed) is the round-to-nearest image of
    the exact f32 dequantized values; dead or unwritten slots are rejected like read_slot."""
    L, H, d = 2, 2, 128
    cfg = kv.PoolConfig(total_slots=2000, offset=1024, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    rng = np.random.default_rng(77)
    n = 600
    bits = rng.choice([2, 4], size=n, p=[0.75, 0.25])
    k, v = rand_kv(77, L, n, H, d)
    t = pool.alloc("r", bits)
    pool.write_prefill(t, k, v)
    for layer in range(L):
        k32, v32 = pool.gather_device(t.slots, layer)
        kr, vr = pool._gather_dev(t.slots, layer)
        assert torch.equal(k32, kr) and torch.equal(v32, vr)
        for dt in (torch.bfloat16, torch.float16):
            kd, vd = pool.gather_device(t.slots, layer, dtype=dt)
            assert kd.dtype == dt and torch.equal(kd, k32.to(dt)) and torch.equal(vd, v32.to(dt))
    t2 = pool.alloc("unwritten", np.full(40, 4))
    with pytest.raises(kv.ValidationError):
        pool.gather_device(t2.slots, 0)
    pool.free("r")
    with pytest.raises(kv.ValidationError):
        pool.gather_device(t.slots, 0)


def test_prefix_gather_feeds_fp16_prefill_attention(cuda):
    """PAPER.md 'Prefill': a matched prefix is gathered from the pool and dequantized into an
    FP16 buffer (K5, gather_device) and handed to an FP16 prefill attention together with the
    new tokens' q / k / v.  Here the consumer is PyTorch's fused SDPA (standing in for the paper's
    FlashInfer kernel): the new tokens' outputs agree with a float64 attention over the
    reference-dequantized prefix (oracle gather) and the same fp16 new k / v."""
    import torch.nn.functional as F

    from oracle import pool as opool

    rng = np.random.default_rng(8)
    L, H, Hq, d, n_pre, n_new = 2, 2, 8, 128, 3000, 200
    pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=6144, offset=3072, n_layers=L, n_kv_heads=H, head_dim=d))
    op = opool.OraclePool(opool.Config(6144, 3072, L, H, d))
    bits = np.where(rng.random(n_pre) < 0.7, 2, 4)
    k, v = rand_kv(81, L, n_pre, H, d)
    t = pool.alloc("pre", bits)
    op.alloc("pre", bits)
    pool.write_prefill(t, k, v)
    op.write_prefill("pre", k, v)
    layer = 1
    kp, vp = pool.gather_device(t.slots, layer, torch.float16)  # [n_pre, H, d] fp16 prefix
    ko, vo = op.gather(op.tables["pre"], layer)
    qn = torch.randn(n_new, Hq, d, device=cuda).half()
    kn = torch.randn(n_new, H, d, device=cuda).half()
    vn = torch.randn(n_new, H, d, device=cuda).half()
    kk = torch.cat([kp, kn]).repeat_interleave(Hq // H, dim=1).permute(1, 0, 2)[None]  # [1, Hq, N, d]
    vv = torch.cat([vp, vn]).repeat_interleave(Hq // H, dim=1).permute(1, 0, 2)[None]
    n = n_pre + n_new
    mask = torch.arange(n, device=cuda)[None, :] <= (n_pre + torch.arange(n_new, device=cuda))[:, None]
    out = F.scaled_dot_product_attention(qn.permute(1, 0, 2)[None], kk, vv, attn_mask=mask)[0].permute(1, 0, 2)
    # float64 reference over the oracle's dequantized prefix and the same fp16 new tokens
    K = np.concatenate([ko, kn.float().cpu().numpy()]).astype(np.float64)
    V = np.concatenate([vo, vn.float().cpu().numpy()]).astype(np.float64)
    Q = qn.float().cpu().numpy().astype(np.float64)
    K, V = np.repeat(K, Hq // H, axis=1), np.repeat(V, Hq // H, axis=1)
    lg = np.einsum("qhd,nhd->hqn", Q, K) / np.sqrt(d)
    lg[:, ~mask.cpu().numpy()] = -np.inf
    w = np.exp(lg - lg.max(-1, keepdims=True))
    ref = np.einsum("hqn,nhd->qhd", w / w.sum(-1, keepdims=True), V)
    err = np.abs(out.float().cpu().numpy() - ref)
    assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), float(err.max())
