"""K7 device tables + the graph-captured decode step (append + attention, all layers).

* the device stream-K plan covers every tile of every (request, kv head) unit exactly once,
  CTA-major, with consistent split bookkeeping, for any CTA count;
* DecodeStep over several steps equals the reference semantics: slots popped exactly as
  append_decode_token (pool.py:284-306), the pool holds the reference INT4 TokenBlocks of every
  appended token (bit-exact), and each step's attention is within the north_star tolerance
  of the oracle's flash_decode over the grown tables (attention.py:175-218);
* graph replay == eager enqueue, and == the host-planned DecodeBatch path.
"""
import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import layout
from oracle import attention as oatt
from oracle import pool as opool

from conftest import rand_kv

pytestmark = pytest.mark.gpu
ATOL, RTOL = 2e-3, 1e-2


def make(L=2, H=2, d=128, lens=(40, 700, 1500, 33), frac=0.8, seed=0, total=12000, offset=6400):
    rng = np.random.default_rng(seed)
    pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=total, offset=offset, n_layers=L, n_kv_heads=H,
                                               head_dim=d))
    op = opool.OraclePool(opool.Config(total, offset, L, H, d))
    rids = []
    for r, n in enumerate(lens):
        bits = np.where(rng.random(n) < frac, 2, 4)
        k, v = rand_kv(seed * 10 + r, L, n, H, d)
        k = torch.as_tensor(k).to(torch.bfloat16).float().numpy()
        v = torch.as_tensor(v).to(torch.bfloat16).float().numpy()
        t = pool.alloc(f"r{r}", bits)
        op.alloc(f"r{r}", bits)
        pool.write_prefill(t, k, v)
        op.write_prefill(f"r{r}", k, v)
        pool.partition(t)
        op.partition(f"r{r}")
        rids.append(f"r{r}")
    return pool, op, rids


def check_plan(work, cta_ptr, n_parts, tiles_per_unit):
    """Every unit's tiles appear once, in order; pieces never cross units; split units have
    nparts pieces with distinct slots part0 .. part0 + nparts - 1."""
    seen = {u: [] for u in range(len(tiles_per_unit))}
    for i in range(cta_ptr.size - 1):
        for k in range(cta_ptr[i], cta_ptr[i + 1]):
            u, lo, hi, slot, p0, npc = work[k][:6]
            assert 0 <= lo < hi <= tiles_per_unit[u]
            seen[u].append((lo, hi, slot, p0, npc, i))
    slots = []
    for u, ps in seen.items():
        ps.sort()
        assert ps and ps[0][0] == 0 and ps[-1][1] == tiles_per_unit[u], (u, ps)
        for a, b in zip(ps, ps[1:]):
            assert a[1] == b[0]
        assert all(p[4] == len(ps) for p in ps)
        if len(ps) == 1:
            assert ps[0][2] == -1
        else:
            got = sorted(p[2] for p in ps)
            assert got == list(range(ps[0][3], ps[0][3] + len(ps)))
            slots += got
    assert sorted(slots) == list(range(n_parts))


@pytest.mark.parametrize("n_cta", [1, 3, 7, 64, 444, 3000])
def test_device_plan_valid(cuda, n_cta):
    pool, op, rids = make(L=1, lens=(5, 40, 700, 1500, 33, 64, 3000))
    st = kv.DecodeStep(pool, rids, n_q_heads=8, n_cta=n_cta, max_new_tokens=8)
    work, cta_ptr, n_parts = st.plan()
    t = pool.device_tables(rids)
    tiles = np.repeat(t["n_pages"] + (t["n_int4"] + 31) // 32, pool.config.n_kv_heads)
    check_plan(work, cta_ptr, n_parts, tiles)
    assert cta_ptr.size == n_cta + 1


def test_decode_step_matches_reference_semantics(cuda):
    L, H, Hq, d = 3, 2, 8, 128
    pool, op, rids = make(L=L, H=H, d=d)
    st = kv.DecodeStep(pool, rids, n_q_heads=Hq, max_new_tokens=64)
    rng = np.random.default_rng(1)
    B = len(rids)
    for step in range(40):
        q = torch.as_tensor(rng.standard_normal((L, B, Hq, d)), dtype=torch.float32).to(torch.bfloat16)
        k = torch.as_tensor(rng.standard_normal((L, B, H, d)), dtype=torch.float32).to(torch.bfloat16)
        v = torch.as_tensor(rng.standard_normal((L, B, H, d)), dtype=torch.float32).to(torch.bfloat16)
        st.q_host.copy_(q)
        st.k_host.copy_(k)
        st.v_host.copy_(v)
        slots = st.run()
        for b, rid in enumerate(rids):
            s = op.pop_decode_slot(rid)
            assert int(slots[b]) == s
            op.write_decode(s, k[:, b].float().numpy(), v[:, b].float().numpy())
        st.check()
        if step in (0, 1, 17, 39):  # tile counts change along the way (INT4 tiles of 32)
            out = st.out_host.float().numpy()
            for layer in range(L):
                for b, rid in enumerate(rids):
                    ref = oatt.flash_decode_pool(q[layer, b].float().numpy(), op, rid, layer)
                    err = np.abs(out[layer, b] - ref)
                    assert np.all(err <= ATOL + RTOL * np.abs(ref)), (step, layer, rid, float(err.max()))
    # the pool holds the reference payloads of every token (prefill and the 40 appends)
    cfg = pool.config
    i2 = pool.int2_pool[: L * H * pool.n_pages * pool.page_stride].view(L, H, pool.n_pages, pool.page_stride)
    i4 = pool.int4_pool[: L * H * pool.n_int4 * pool.slot_stride].view(L, H, pool.n_int4, pool.slot_stride)
    i2, i4 = i2.cpu().numpy(), i4.cpu().numpy()
    assert np.array_equal(layout.page_payloads(i2[op.page_written], d), op.int2[op.page_written])
    assert np.array_equal(i4[op.slot_written], layout.slot_records(op.int4[op.slot_written], d))
    assert np.array_equal(pool._int4_written, op.slot_written)
    for rid in rids:
        assert pool.table(rid).slots.tolist() == op.tables[rid]
    pool.check_invariants()


def test_decode_step_graph_equals_eager_and_host_plan(cuda):
    L, H, Hq, d = 2, 2, 16, 128
    outs = []
    for graph in (True, False):
        pool, op, rids = make(L=L, H=H, d=d, seed=3)
        st = kv.DecodeStep(pool, rids, n_q_heads=Hq, max_new_tokens=16)
        rng = np.random.default_rng(5)
        for step in range(5):
            st.q_host.copy_(torch.as_tensor(rng.standard_normal(st.q_host.shape), dtype=torch.float32))
            st.k_host.copy_(torch.as_tensor(rng.standard_normal(st.k_host.shape), dtype=torch.float32))
            st.v_host.copy_(torch.as_tensor(rng.standard_normal(st.v_host.shape), dtype=torch.float32))
            st.run(graph=graph)
        st.check()
        outs.append(st.out_host.clone())
    assert torch.equal(outs[0], outs[1])
    # the host-planned path over the same (grown) tables and the same last-step q
    b = kv.DecodeBatch(pool, rids, n_q_heads=Hq)
    for layer in range(L):
        o = kv.flash_decode_batched(st.q_dev[layer], b, layer).float().cpu()
        assert torch.allclose(o, outs[1][layer].float(), atol=2e-3, rtol=1e-2), float((o - outs[1][layer].float()).abs().max())
