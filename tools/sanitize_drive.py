"""Small end-to-end drive of every product kernel, for compute-sanitizer:

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_drive.py

K1 prefill (page + INT4 kernels, f32 / bf16), K6 device routing, K5 gather (f32 / f16 / bf16), the
generic codec entry points, K2 decode (tensor-core kernel with stream-K splits and the fused
last-arriver combine; the fp32-faithful kernel), the batched and the fused K4 append, K7 device
tables + the DecodeStep (eager, not graph-captured: the sanitizer tracks kernels), the replay
attention (f4) and merge_partials.  Sizes are
small so each tool finishes in minutes; the outputs are checked against the oracle so a
run that is silently wrong under instrumentation also fails.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2605_17170_b200 as kv  # noqa: E402
from oracle import attention as oatt  # noqa: E402
from oracle import pool as opool  # noqa: E402

ATOL, RTOL = 2e-3, 1e-2


def main():
    rng = np.random.default_rng(7)
    L, H, Hq, d = 2, 2, 16, 128
    total, offset = 14000, 9600
    pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=total, offset=offset, n_layers=L, n_kv_heads=H, head_dim=d))
    op = opool.OraclePool(opool.Config(total, offset, L, H, d))
    rids = []
    for r, n in enumerate([37, 300, 1100, 6000]):
        bits = np.where(rng.random(n) < 0.8, 2, 4)
        k = torch.randn(L, n, H, d).to(torch.bfloat16).float().numpy()
        v = torch.randn(L, n, H, d).to(torch.bfloat16).float().numpy()
        t = pool.alloc_device(f"r{r}", bits) if r == 1 else pool.alloc(f"r{r}", bits)
        op.alloc(f"r{r}", bits)
        kin = torch.as_tensor(k).to(torch.bfloat16) if r else k
        pool.write_prefill(t, kin, torch.as_tensor(v).to(torch.bfloat16) if r else v)
        op.write_prefill(f"r{r}", k, v)
        pool.partition(t)
        op.partition(f"r{r}")
        rids.append(f"r{r}")
    kk, vv = (x.cpu().numpy() for x in pool.gather_device(pool.table("r2").slots, 1))
    ok, ov = op.gather(op.tables["r2"], 1)
    assert np.array_equal(kk, ok) and np.array_equal(vv, ov), "gather differs from the oracle"
    g = kv.quantize_group(rng.standard_normal(45).astype(np.float32), 4)
    kv.dequantize_group(g)
    kv.unpack_codes(kv.pack_codes(g.codes, 4), 4, g.group_len)
    kv.encode_key_page_int2(rng.standard_normal((32, d)).astype(np.float32))
    kv.encode_token_blocks(rng.standard_normal((5, d)).astype(np.float32), 2)

    q = torch.randn(len(rids), Hq, d).to(torch.bfloat16)
    for n_cta in (1, 3, 37):  # 1: long single pieces (several key-bias batches per warp); split units: partial slots + last-arriver combine
        b = kv.DecodeBatch(pool, rids, n_q_heads=Hq, n_cta=n_cta)
        for layer in range(L):
            out = kv.flash_decode_batched(q.cuda(), b, layer, out=torch.empty(q.shape, device="cuda"))
            for i, rid in enumerate(rids):
                ref = oatt.flash_decode_pool(q[i].float().numpy(), op, rid, layer)
                err = np.abs(out[i].cpu().numpy() - ref)
                assert np.all(err <= ATOL + RTOL * np.abs(ref)), (n_cta, layer, rid, err.max())
    out = kv.flash_decode(q[2].float().numpy(), pool.table("r2"), pool.view(0))  # fp32-faithful kernel
    assert np.abs(out - oatt.flash_decode_pool(q[2].float().numpy(), op, "r2", 0)).max() < 1e-4

    # decode steps (K7 device tables each step), eager: batched append (K4 data half) + decode,
    # and the fused form (K4 inside K2)
    for fused in (False, True):
        step = kv.DecodeStep(pool, rids, n_q_heads=Hq, max_new_tokens=4, n_cta=40, fused_append=fused)
        for _ in range(2):
            step.q_host.copy_(torch.randn(step.q_host.shape).to(step.q_host.dtype))
            step.k_host.copy_(torch.randn(step.k_host.shape).to(step.k_host.dtype))
            step.v_host.copy_(torch.randn(step.v_host.shape).to(step.v_host.dtype))
            step.run(graph=False)
            step.check()
    # K5 typed gather and the replay attention (f2, f4)
    for dt in (torch.float16, torch.bfloat16):
        pool.gather_device(pool.table("r1").slots, 0, dt)
    from paper_2605_17170_b200 import calib
    qa = torch.randn(50, 8, d, device="cuda")
    calib.attention_full(qa, torch.randn(70, 2, d, device="cuda"), torch.randn(70, 2, d, device="cuda"), causal=True)
    kv.merge_partials([kv.SplitPartial(acc=rng.standard_normal(d).astype(np.float32), lse=float(rng.standard_normal()),
                                       max_logit=float(rng.standard_normal())) for _ in range(3)])
    torch.cuda.synchronize()
    print("sanitize drive ok")


if __name__ == "__main__":
    main()
