"""Does a unit's tile time follow the request's memory region or the CTA index?  Runs the
same pool with the batch in request order and in reversed order (debug build,
-DKVMIX_CTA_TIMES) and prints the mean per-request tile-phase residual for both."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = bench.parse()
import paper_2605_17170_b200 as kv  # noqa: E402
from paper_2605_17170_b200 import _lib  # noqa: E402

pool, batch, q, out, bits = bench.build_workload(args, torch.device("cuda", 0), 0)
rids = [f"req{r}" for r in range(args.batch)]
npg = np.array([int((b == 2).sum()) // 32 for b in bits])
for order in ("forward", "reversed"):
    rr = rids if order == "forward" else rids[::-1]
    b = kv.DecodeBatch(pool, rr, n_q_heads=args.q_heads, ctas_per_sm=args.ctas_per_sm, int4_weight=args.int4_weight)
    qq = q[7][[int(r[3:]) for r in rr]].contiguous()
    for _ in range(3):
        kv.flash_decode_batched(qq, b, 7)
    torch.cuda.synchronize()
    n = b.n_cta
    buf = (ctypes.c_ulonglong * (16 * n))()
    assert _lib.lib.kvmix_debug_cta_times(buf, n) == 0
    t = np.array(buf, dtype=np.float64).reshape(n, 16)
    ph = t[:, 4:16].reshape(n, 3, 4) / 1e3
    work, cp = b.work.cpu().numpy(), b.cta_ptr.cpu().numpy()
    rows = []
    for c in range(n):
        for k, w in enumerate(work[cp[c]:cp[c + 1]][:3]):
            u, lo, hi = w[0], w[1], w[2]
            req = int(rr[u // 8][3:])
            P = npg[req]
            a2 = max(0, min(hi, P) - lo)
            rows.append((req, c, a2, (hi - lo) - a2, ph[c, k, 2] - ph[c, k, 1]))
    r = np.array(rows, dtype=float)
    X = r[:, 2:4]
    coef = np.linalg.lstsq(X, r[:, 4], rcond=None)[0]
    res = r[:, 4] - X @ coef
    print(order, "launch end %.1f us" % ((t[:, 2].max() - t[:, 0].min()) / 1e3),
          " ".join("%d:%+.1f" % (v, res[r[:, 0] == v].mean()) for v in range(args.batch)))
