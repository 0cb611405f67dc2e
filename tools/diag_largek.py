"""Diagnose the large-K parity case: variant 0 / variant 1 vs the f64 dense attention."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import paper_2605_17170_b200 as kv
from oracle import attention as oatt
from test_gpu_parity import Pair, kv_data, bf16_exact

for frac, n, qv, kch in [(0.8, 50, 30.0, 2000.0), (1.0, 64, 30.0, 2000.0), (0.0, 64, 30.0, 2000.0), (0.8, 50, 3.0, 2000.0),
                         (0.8, 50, 30.0, 200.0), (1.0, 32, 30.0, 2000.0)]:
    rng = np.random.default_rng(11)
    H, Hq, d = 2, 16, 128
    pair = Pair(total=8000, offset=4000, L=1, H=H, d=d)
    bits = np.where(rng.random(n) < frac, 2, 4)
    k, v = kv_data(rng, 1, n, H, d, kscale=np.full((H, d), kch))
    pair.add("r0", bits, np.clip(k, -60000, 60000), v)
    q = bf16_exact(rng.standard_normal((1, Hq, d)) * 1e-3)
    q[:, :, 0] = qv
    kk, vv = pair.op.gather(pair.op.tables["r0"], 0)
    exact = oatt.dense_f64(q, kk, vv)[0]
    ref = oatt.flash_decode_pool(q[0], pair.op, "r0", 0)
    b = kv.DecodeBatch(pair.pool, ["r0"], n_q_heads=Hq)
    res = {}
    for name, qq, var in [("v0 bf16", torch.as_tensor(q, device="cuda").to(torch.bfloat16), 0),
                          ("v0 f32", torch.as_tensor(q, device="cuda"), 0),
                          ("v1 f32", torch.as_tensor(q, device="cuda"), 1)]:
        o = torch.empty(1, Hq, d, device="cuda")
        kv.flash_decode_batched(qq, b, 0, out=o, variant=var)
        res[name] = float(np.abs(o[0].cpu().numpy() - exact).max())
    logits = np.einsum("hd,nhd->hn", q[0].astype(np.float64), np.repeat(kk, 8, 1)) / np.sqrt(d)
    top = np.sort(logits, 1)[:, -2:]
    print(f"frac {frac} n {n} q0 {qv} kch {kch} bounds {pair.pool.operand_bounds()} ref {np.abs(ref-exact).max():.2e} "
          + " ".join(f"{k} {v:.2e}" for k, v in res.items()) + f" | top2 gap min {np.min(top[:,1]-top[:,0]):.3f}")
