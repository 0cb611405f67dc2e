"""Is the per-CTA speed variation systematic?  Times the same decode launch several times
(debug build, -DKVMIX_CTA_TIMES) and correlates per-CTA durations / SM placement across runs."""
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
n = batch.n_cta
runs = []
for rep in range(4):
    for layer in range(3):
        kv.flash_decode_batched(q[layer], batch, layer, out=out[layer])
    torch.cuda.synchronize()
    kv.flash_decode_batched(q[7], batch, 7, out=out[7])
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (16 * n))()
    assert _lib.lib.kvmix_debug_cta_times(buf, n) == 0
    t = np.array(buf, dtype=np.float64).reshape(n, 16)
    runs.append(((t[:, 2] - t[:, 0]) / 1e3, t[:, 3].astype(int), (t[:, 2] - t[:, 0].min()) / 1e3))
for i in range(1, len(runs)):
    d0, d1 = runs[0][0], runs[i][0]
    print(f"run {i}: corr(duration) {np.corrcoef(d0, d1)[0, 1]:.3f}, same SM {np.mean(runs[0][1] == runs[i][1]):.3f}, "
          f"launch end {runs[i][2].max():.1f} us")
sm_speed = {}
for d, sm, _ in runs:
    for s in np.unique(sm):
        sm_speed.setdefault(s, []).append(d[sm == s].mean())
v = np.array([np.std(x) for x in sm_speed.values()]); m = np.array([np.mean(x) for x in sm_speed.values()])
print(f"per-SM mean duration spread across SMs {m.std():.2f} us; within-SM run-to-run std {v.mean():.2f} us")
