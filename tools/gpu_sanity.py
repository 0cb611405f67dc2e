"""Quick on-GPU sanity run used during development (not a test)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import __graft_entry__ as ge
ge.build()
import paper_2605_17170_b200 as kv
from oracle import attention as oatt, pool as opool, codec

def check_case(seed, N, H, Hq, d, frac, variant):
    rng = np.random.default_rng(seed)
    L = 1
    bits = np.where(rng.random(N) < frac, 2, 4)
    k = (rng.standard_normal((L, N, H, d)) * np.exp(rng.uniform(np.log(0.5), np.log(4.0), (H, d)))).astype(np.float32)
    v = rng.standard_normal((L, N, H, d)).astype(np.float32)
    q = rng.standard_normal((Hq, d)).astype(np.float32)
    cfg = kv.PoolConfig(total_slots=2 * N + 64, offset=((N + 31) // 32) * 32, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg)
    t = pool.alloc("r", bits); pool.write_prefill(t, k, v); pool.partition(t)
    out = kv.flash_decode(q, t, pool.view(0), variant=variant)
    op = opool.OraclePool(opool.Config(cfg.total_slots, cfg.offset, L, H, d))
    op.alloc("r", bits); op.write_prefill("r", k, v); op.partition("r")
    ref = oatt.flash_decode_pool(q, op, "r", 0)
    err = np.abs(out - ref).max()
    n2 = pool.n_pages * pool.page_stride
    dev2 = pool.int2_pool[: L * H * n2].view(L, H, pool.n_pages, pool.page_stride).cpu().numpy()
    dev4 = pool.int4_pool[: L * H * pool.n_int4 * pool.slot_stride].view(L, H, pool.n_int4, pool.slot_stride).cpu().numpy()
    b2 = np.array_equal(dev2[op.page_written], op.int2[op.page_written])
    b4 = np.array_equal(dev4[op.slot_written], op.int4[op.slot_written])
    ok = np.all(np.abs(out - ref) <= 2e-3 + 1e-2 * np.abs(ref))
    print(f"seed={seed} N={N} H={H}/{Hq} d={d} var={variant}: bytes2={b2} bytes4={b4} maxerr={err:.2e} ok={ok}", flush=True)
    return ok and b2 and b4

allok = True
for variant in (1, 0):
    for (N, H, Hq, d) in [(100, 1, 1, 32), (300, 2, 8, 64), (1100, 2, 8, 128), (4096, 2, 8, 128), (777, 1, 4, 128), (64, 2, 2, 32)]:
        for frac in (0.75, 0.2, 1.0, 0.0):
            try:
                allok &= check_case(N + int(frac*10), N, H, Hq, d, frac, variant)
            except Exception as e:
                print("FAIL", N, H, Hq, d, frac, variant, repr(e)); allok = False
print("ALL OK" if allok else "SOME FAILED")
