"""Host-side product logic on CPU: the C ABI loads and exports every declared symbol,
the control plane (allocator, partition, page tables) reproduces the reference's slot
indices exactly, pool sizing arithmetic, the split planner and error mapping."""
import json
import os
import re

import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import _lib
from paper_2605_17170_b200.plan import plan_stream
from paper_2605_17170_b200.pool import csr_tables, split_partitioned
from oracle import pool as opool

from conftest import GOLDEN, ROOT


def host_pool(total, offset, L=1, H=1, d=32):
    return kv.MixedPrecisionPool(kv.PoolConfig(total_slots=total, offset=offset, n_layers=L, n_kv_heads=H,
                                               head_dim=d), materialize=False)


# ---- C ABI -----------------------------------------------------------------------------------
def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "kvmix_b200.h")).read()
    declared = set(re.findall(r"\b(kvmix_\w+)\s*\(", header))
    assert declared, "no declarations parsed"
    missing = [n for n in declared if not hasattr(_lib.lib, n)]
    assert not missing, missing
    assert declared == set(_lib.EXPORTED)


def test_abi_strides_and_sizes():
    for d in (32, 64, 128, 256):
        assert _lib.lib.kvmix_key_page_payload_bytes(d) == kv.key_page_payload_bytes(d)
        for b in (2, 4):
            assert _lib.lib.kvmix_token_block_payload_bytes(d, b) == kv.token_block_payload_bytes(d, b)
        assert _lib.page_stride(d) % 16 == 0 and _lib.slot_stride(d) % 16 == 0
        assert _lib.page_stride(d) >= kv.key_page_payload_bytes(d) + 32 * kv.token_block_payload_bytes(d, 2)
        assert _lib.slot_stride(d) >= 2 * kv.token_block_payload_bytes(d, 4)
    assert _lib.page_stride(128) == 3072 and _lib.slot_stride(128) == 160
    assert _lib.lib.kvmix_version().startswith(b"kvmix_b200")


@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_record_layout_matches_kernels(d):
    """layout.py (numpy statement of the device record permutation) equals the
    permutation the CUDA kernels compute (exported host-side by the library), and it is
    a bijection onto the reference payload bytes (every byte kept, nothing re-rounded)."""
    import ctypes
    from paper_2605_17170_b200 import layout
    for fn, pyperm, stride in ((_lib.lib.kvmix_page_layout, layout.page_perm(d), _lib.page_stride(d)),
                               (_lib.lib.kvmix_slot_layout, layout.slot_perm(d), _lib.slot_stride(d))):
        out = np.zeros(stride, dtype=np.int64)
        _lib.check(fn(d, out.ctypes.data_as(ctypes.c_void_p)))
        assert np.array_equal(out, pyperm)
    rng = np.random.default_rng(d)
    ref = rng.integers(0, 256, (3, layout.page_stride(d)), dtype=np.uint8)
    assert np.array_equal(layout.page_payloads(layout.page_records(ref, d), d), ref)
    n4 = 2 * kv.token_block_payload_bytes(d, 4)
    ref4 = rng.integers(0, 256, (3, n4), dtype=np.uint8)
    rec4 = layout.slot_records(np.concatenate([ref4, np.zeros((3, layout.slot_stride(d) - n4), np.uint8)], 1), d)
    assert np.array_equal(layout.slot_payloads(rec4, d), ref4)
    assert not rec4[:, layout.slot_perm(d) < 0].any()


def test_abi_validation_without_gpu():
    # argument validation happens before any CUDA call and maps to ValidationError
    rc = _lib.lib.kvmix_encode_token_blocks(None, 1, 33, 2, None, 36, None, None)
    with pytest.raises(kv.ValidationError):
        _lib.check(rc)
    rc = _lib.lib.kvmix_flash_decode(None, 0, None, 0, None, None, 1, 1, 0, 3, 128, 8, 1, None, None, None, None,
                                     None, None, None, 3, None, None, 1.0, 0, None, 0, None)
    with pytest.raises(kv.ValidationError, match="multiple"):
        _lib.check(rc)


def test_gather_validation_without_gpu():
    """The fused head gather (kvmix_flash_decode_gather) rejects bad destinations before any
    CUDA call; HeadOutputs checks the same on the host."""
    import ctypes

    from paper_2605_17170_b200 import dist as kvdist

    fake = 16  # never dereferenced: validation returns first
    def call(n_outs, out_heads, head0, null=False):
        ptrs = (ctypes.c_void_p * 9)(*([None] if null else []) + [fake] * (9 - int(null)))
        return _lib.lib.kvmix_flash_decode_gather(
            fake, 1, ctypes.cast(ptrs, ctypes.c_void_p), n_outs, out_heads, head0, 1, fake, fake, 1, 1, 0, 1, 128, 8,
            1, fake, fake, fake, fake, None, fake, fake, 1, fake, fake, 1.0, 0, None, 0, None)
    for args, msg in [((9, 8, 0), "output buffers"), ((0, 8, 0), "output buffers"), ((2, 8, 1), "head slice"),
                      ((2, 16, -1), "head slice"), ((2, 16, 0, True), "null")]:
        with pytest.raises(kv.ValidationError, match=msg):
            _lib.check(call(*args))
    ho = kvdist.HeadOutputs([fake, fake], out_heads=16, head0=8, dtype=torch.bfloat16, batch=2, head_dim=128)
    ho.check(2, 8, 128, "cpu")
    for bad in [(2, 16, 128), (3, 8, 128), (2, 8, 64)]:
        with pytest.raises(kv.ValidationError):
            ho.check(*bad, "cpu")
    with pytest.raises(kv.ValidationError):
        kvdist.HeadOutputs([fake] * 9, 16, 0, torch.bfloat16, 2, 128).check(2, 8, 128, "cpu")


# ---- control plane vs the oracle and the reference trace --------------------------------------
def test_alloc_trace_matches_reference():
    tr = json.load(open(os.path.join(GOLDEN, "alloc_trace.json")))
    p = host_pool(tr["total_slots"], tr["offset"])
    for rec in tr["ops"]:
        try:
            if rec["op"] == "alloc":
                t = p.alloc(rec["rid"], np.array(rec["bits"]))
                assert t.slots.tolist() == rec["slots"]
            elif rec["op"] == "free":
                p.free(rec["rid"])
            else:
                t = p.partition(p.table(rec["rid"]))
                slot = p._free_int4[-1] if p._free_int4 else None
                # slot bookkeeping of append_decode_token without the device write
                if not p._free_int4:
                    raise kv.CapacityError("INT4 region exhausted during decode", region="int4")
                s = p._free_int4.pop()
                p._owner[s] = p._rid_index[rec["rid"]]
                t._set_slots(np.append(t.slots, s))
                assert s == rec["slot"] == slot
                assert t.slots.tolist() == rec["slots"]
            assert "capacity" not in rec
        except kv.CapacityError as e:
            assert e.region == rec["capacity"]
        assert p._free_pages == rec["free_pages"]
        assert p._free_int4 == rec["free_int4"]
        p.check_invariants()


def test_alloc_fuzz_vs_oracle():
    rng = np.random.default_rng(42)
    p = host_pool(2048, 1024)
    o = opool.OraclePool(opool.Config(2048, 1024, 1, 1, 32), data_plane=False)
    live = []
    for i in range(400):
        a = rng.random()
        if a < 0.5 or not live:
            bits = rng.choice([2, 4], size=int(rng.integers(1, 200)), p=[0.75, 0.25])
            try:
                s = p.alloc(f"r{i}", bits).slots.tolist()
            except kv.CapacityError as e:
                with pytest.raises(opool.OracleError) as oe:
                    o.alloc(f"r{i}", bits)
                assert oe.value.region == e.region
                continue
            assert s == o.alloc(f"r{i}", bits)
            live.append(f"r{i}")
        elif a < 0.8:
            rid = live.pop(int(rng.integers(len(live))))
            p.free(rid)
            o.free(rid)
        else:
            rid = live[int(rng.integers(len(live)))]
            assert p.partition(p.table(rid)).slots.tolist() == o.partition(rid)
        assert p._free_pages == o.free_pages and p._free_int4 == o.free_int4
        p.check_invariants()


def test_alloc_semantics():
    p = host_pool(256, 128)
    bits = np.array([2] * 32 + [4] * 10)
    t = p.alloc("r", bits)
    assert t.slots[:32].tolist() == list(range(32)) and t.slots[32] == 128       # lowest first
    t2 = p.alloc("s", np.array([2] * 40))                                          # residual -> INT4
    assert int((t2.slots < 128).sum()) == 32 and p.live_counts() == (64, 18)
    with pytest.raises(kv.ValidationError):
        p.alloc("r", np.array([4]))
    with pytest.raises(kv.ValidationError):
        p.alloc("x", np.array([3]))
    first = p.alloc("a", np.array([4] * 3)).slots.tolist()
    p.free("a")
    assert p.alloc("b", np.array([4] * 3)).slots.tolist() == first[::-1]           # LIFO reuse
    with pytest.raises(kv.ValidationError):
        p.free("a")
    small = host_pool(64, 32)
    with pytest.raises(kv.CapacityError) as e:
        small.alloc("r", np.array([2] * 64))
    assert e.value.region == "int2"
    with pytest.raises(kv.CapacityError) as e:
        small.alloc("r", np.array([4] * 33))
    assert e.value.region == "int4"


def test_partition_stable_idempotent():
    p = host_pool(256, 128)
    t = p.alloc("r", np.array([4, 2, 4] + [2] * 31 + [4]))
    orig = t.slots.copy()
    p.partition(t)
    assert t.slots.tolist() == orig[orig < 128].tolist() + orig[orig >= 128].tolist()
    snap = t.slots.tolist()
    p.partition(t)
    assert t.slots.tolist() == snap
    assert [a.index for a in t.entries] == snap
    pages, int4 = split_partitioned(t.slots, 128)
    assert pages.tolist() == [orig[orig < 128][0] // 32] and int4.tolist() == (orig[orig >= 128] - 128).tolist()


def test_split_partitioned_rejects():
    with pytest.raises(kv.ValidationError, match="not partitioned"):
        split_partitioned(np.array([200, 0, 1]), 128)
    with pytest.raises(kv.ValidationError, match="page-granular"):
        split_partitioned(np.array([0, 1, 2]), 128)


def test_init_pool_offsets():
    assert kv.init_pool(2.5, 1000, 1, 1, 32).offset == 736
    assert kv.init_pool(2.7, 3200, 1, 1, 32).offset == 2080
    assert kv.init_pool(2.5, 3200, 1, 1, 32).offset == 2400
    assert kv.init_pool(4.0, 320, 1, 1, 32).offset == 0
    assert kv.init_pool(2.0, 320, 1, 1, 32).offset == 320
    for b in (2.0, 2.3, 3.1, 4.0):
        assert kv.init_pool(b, 999, 1, 1, 32).offset % 32 == 0
    with pytest.raises(kv.ValidationError):
        kv.init_pool(1.5, 320, 1, 1, 32)
    with pytest.raises(kv.ValidationError):
        kv.PoolConfig(total_slots=128, offset=30, n_layers=1, n_kv_heads=1, head_dim=32)


def test_capacity_headroom():
    dims = dict(head_dim=128, n_layers=32, n_kv_heads=8)
    n = 11_000
    assert kv.capacity_tokens(n * kv.baseline_bytes_per_token(**dims), 2.7, **dims) / n >= 4.0
    assert kv.bytes_per_token(128, 1, 1, 2) == 96 and kv.bytes_per_token(128, 1, 1, 4) == 160


def test_stats_accounting():
    p = host_pool(256, 128)
    p.alloc("r", np.array([2] * 64 + [4] * 36))
    st = p.stats()
    assert st["realized_avg_bitwidth"] == pytest.approx((2 * 64 + 4 * 36) / 100)
    assert st["int2"]["live"] == 64 and st["int4"]["live"] == 36


# ---- stream-K planner -------------------------------------------------------------------------
def _tile_bytes(npg, n4):
    n4t = -(-n4 // 32)
    return [3072] * npg + [160 * min(32, n4 - 32 * k) for k in range(n4t)]


@pytest.mark.parametrize("B,Hkv,n_cta", [(1, 2, 444), (16, 8, 444), (64, 8, 444), (3, 1, 7), (5, 2, 1000)])
def test_plan_covers_every_tile_once(B, Hkv, n_cta):
    """Every tile of every (request, kv head) is in exactly one piece; pieces of a split
    unit own consecutive partial slots; CTA ranges are contiguous and in order."""
    rng = np.random.default_rng(B)
    npg = rng.integers(0, 1200, B)
    n4 = rng.integers(0, 5000, B)
    n4[npg == 0] += 1
    work, cta_ptr, n_parts = plan_stream(npg, n4, Hkv, 3072, 160, n_cta=n_cta)
    tiles = npg + (n4 + 31) // 32
    assert cta_ptr[0] == 0 and cta_ptr[-1] == work.shape[0] and (np.diff(cta_ptr) >= 0).all()
    seen = {}
    for row in work:
        u, lo, hi, slot, p0, npc = row[:6]
        assert 0 <= lo < hi <= tiles[u // Hkv]
        seen.setdefault(int(u), []).append((int(lo), int(hi), int(slot), int(p0), int(npc)))
    assert sorted(seen) == list(range(B * Hkv))
    slots = []
    for u, pcs in seen.items():
        assert pcs[0][0] == 0 and pcs[-1][1] == tiles[u // Hkv]
        assert all(pcs[k][1] == pcs[k + 1][0] for k in range(len(pcs) - 1))
        assert all(p[4] == len(pcs) for p in pcs)
        if len(pcs) == 1:
            assert pcs[0][2] == -1
        else:
            assert [p[2] for p in pcs] == list(range(pcs[0][3], pcs[0][3] + len(pcs)))
            slots += [p[2] for p in pcs]
    assert sorted(slots) == list(range(n_parts))


@pytest.mark.parametrize("w4", [1.0, 0.9])
def test_plan_cost_balance(w4):
    """Every CTA gets the same cost: bytes, with INT4 bytes weighted by int4_weight."""
    npg, n4 = np.array([1000] * 16), np.array([6000] * 16)
    work, cta_ptr, _ = plan_stream(npg, n4, 8, 3072, 160, n_cta=444, int4_weight=w4)
    cost = np.array([b if i < 1000 else b * w4 for i, b in enumerate(_tile_bytes(1000, 6000))])
    per_cta = np.zeros(444)
    for c in range(444):
        for u, lo, hi in work[cta_ptr[c]:cta_ptr[c + 1], :3]:
            per_cta[c] += cost[lo:hi].sum()
    assert per_cta.max() / per_cta.mean() < 1.02 and per_cta.min() / per_cta.mean() > 0.98


def test_plan_tier_skew_shares():
    """tier_skew scales residency tier i's cost share by 1 + skew (1 - 2 i / (tiers - 1)),
    still covering every tile exactly once."""
    npg, n4 = np.array([1000] * 16), np.array([6000] * 16)
    work, cta_ptr, _ = plan_stream(npg, n4, 8, 3072, 160, n_cta=444, int4_weight=1.0, tier_skew=0.1, n_sm=148)
    cost = np.asarray(_tile_bytes(1000, 6000), dtype=np.float64)
    per_cta = np.zeros(444)
    for c in range(444):
        for u, lo, hi in work[cta_ptr[c]:cta_ptr[c + 1], :3]:
            per_cta[c] += cost[lo:hi].sum()
    tier_mean = per_cta.reshape(3, 148).mean(axis=1) / per_cta.mean()
    assert np.allclose(tier_mean, [1.1, 1.0, 0.9], atol=0.01)
    assert abs(per_cta.sum() - 16 * 8 * cost.sum()) < 1


def test_route_scratch_size():
    """K6 scratch: one total + one count per 4096-token chunk (host-only C entry point)."""
    from paper_2605_17170_b200._lib import lib
    assert [lib.kvmix_route_scratch_elems(n) for n in (0, 1, 4096, 4097, 131072)] == [1, 2, 2, 3, 33]


def test_csr_tables_cpu():
    t = csr_tables([np.array([3, 1], np.int32), np.array([], np.int32)], [np.array([5]), np.array([0, 1, 2])],
                   "cpu")
    assert t["page_indptr"].tolist() == [0, 2, 2] and t["int4_indptr"].tolist() == [0, 1, 4]
    assert t["n_pages"].tolist() == [2, 0] and t["n_int4"].tolist() == [1, 3]


def test_error_mapping():
    with pytest.raises(kv.KvmixError):
        _lib.check(-5)
    with pytest.raises(kv.CapacityError):
        _lib.check(-3)
    _lib.check(0)


def test_decode_step_layer_chunks():
    """DecodeStep's upload / download ranges cover every layer once, in order."""
    from paper_2605_17170_b200.decode_step import layer_chunks

    for L in (1, 5, 8, 16, 30, 64, 80):
        for spec in (8, 3, None, [2, 6, 8, 8, 8, 8, 8, 8, 8, 8, 8]):
            if isinstance(spec, list) and sum(spec) < L:
                continue
            ch = layer_chunks(L, spec)
            assert ch[0][0] == 0 and ch[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
            assert all(c1 > c0 for c0, c1 in ch)
    assert layer_chunks(64, None)[0] == (0, 2) and layer_chunks(64, None)[-1] == (62, 64)
    with pytest.raises(kv.ValidationError):
        layer_chunks(10, [2, 2])
    with pytest.raises(kv.ValidationError):
        layer_chunks(10, 0)
