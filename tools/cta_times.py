"""Per-CTA start / q-wait / end times of one decode launch (debug build with -DKVMIX_CTA_TIMES):
load balance of the stream-K plan (development helper, not shipped)."""
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

dev = torch.device("cuda", 0)
pool, batch, q, out, bits = bench.build_workload(args, dev, 0)
for layer in range(4):
    kv.flash_decode_batched(q[layer], batch, layer, out=out[layer])
torch.cuda.synchronize()
if os.environ.get("CTA_PIPELINED"):  # steady state: 8 back-to-back launches (PDL), the last one recorded
    for layer in range(8, 16):
        kv.flash_decode_batched(q[layer], batch, layer, out=out[layer])
else:
    kv.flash_decode_batched(q[5], batch, 5, out=out[5])
torch.cuda.synchronize()
n = batch.n_cta
buf = (ctypes.c_ulonglong * (16 * n))()
assert _lib.lib.kvmix_debug_cta_times(buf, n) == 0
t = np.array(buf, dtype=np.float64).reshape(n, 16)
t0 = t[:, 0].min()
start, waited, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
sm = t[:, 3].astype(int)
print(f"CTAs {n}: start max {start.max():.1f} us, end min {end.min():.1f} mean {end.mean():.1f} max {end.max():.1f} us")
dur = end - start
print(f"duration per CTA: min {dur.min():.1f} p10 {np.percentile(dur, 10):.1f} median {np.median(dur):.1f} "
      f"p90 {np.percentile(dur, 90):.1f} max {dur.max():.1f} us")
sm_end = np.zeros(sm.max() + 1)
np.maximum.at(sm_end, sm, end)
print(f"per-SM last end: min {sm_end.min():.1f} median {np.median(sm_end):.1f} max {sm_end.max():.1f} us")
npieces = np.diff(batch.cta_ptr.cpu().numpy())
if npieces is not None:
    for k in sorted(set(npieces.tolist())):
        sel = npieces == k
        print(f"  CTAs with {k} pieces: {sel.sum()}, mean duration {dur[sel].mean():.1f} us")
os.makedirs("gpurun_out", exist_ok=True)
work = batch.work.cpu().numpy()
ph = (t[:, 4:16].reshape(n, 3, 4) - t0) / 1e3
for k in range(2):
    sel = npieces > k
    b, qt, le, md = ph[sel, k, 0], ph[sel, k, 1], ph[sel, k, 2], ph[sel, k, 3]
    print(f"piece {k}: n={sel.sum()} q-table {np.median(qt - b):.2f} us, tiles {np.median(le - qt):.2f} us, "
          f"merge {np.median(md - le):.2f} us (p90 {np.percentile(md - le, 90):.2f})")
np.savez("gpurun_out/cta_times.npz", ph=ph, start=start, waited=waited, end=end, sm=sm, npieces=npieces,
         cta_ptr=batch.cta_ptr.cpu().numpy(), work=work)
