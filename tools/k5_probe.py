"""Time K5 (gather-dequant to bf16 / f16 / f32) on a 32K-token tagged request, 8 kv heads, d = 128 --
the prefill path's read of a matched prefix (PAPER.md 'Prefill': gather-dequant into an FP16
buffer for the prefill attention).  Bytes = records read + dense K/V written."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2605_17170_b200 as kv  # noqa: E402

N, L, H, d = 32768, 1, 8, 128
data = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench_data", "tagged_bits.npz"))
bits = np.where(np.unpackbits(data["bits_32768"][0])[:N] == 1, 2, 4)
n2 = int((bits == 2).sum()) // 32 * 32
pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=N + 64, offset=n2, n_layers=L, n_kv_heads=H, head_dim=d))
t = pool.alloc("r", bits)
k = torch.randn(L, N, H, d, device="cuda").to(torch.bfloat16)
pool.write_prefill(t, k, torch.randn_like(k))
from paper_2605_17170_b200 import _lib  # noqa: E402

out = {}
sl = torch.as_tensor(t.slots.astype(np.int32), device="cuda")
for dt in (torch.float16, torch.bfloat16, torch.float32):
    ko = torch.empty((N, H, d), dtype=dt, device="cuda")
    vo = torch.empty_like(ko)

    def call():  # the kernel alone (gather_device adds host checks and the slot upload)
        _lib.check(_lib.lib.kvmix_gather_dequant_typed(
            pool.int2_pool.data_ptr(), pool.int4_pool.data_ptr(), pool.n_pages, pool.n_int4, pool.config.offset, 0,
            H, d, sl.data_ptr(), N, ko.data_ptr(), vo.data_ptr(), _lib.dtype_code(ko), _lib.stream()))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    times = []
    for _ in range(10):  # one launch per event pair (the ctypes call costs more than the kernel)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    n4 = N - n2
    rd = H * (n2 // 32 * pool.page_stride + n4 * pool.slot_stride)
    wr = 2 * N * H * d * torch.empty(0, dtype=dt).element_size()
    out[str(dt)] = {"ms": ms, "GBps": (rd + wr) / ms / 1e6, "read_MB": rd / 1e6, "write_MB": wr / 1e6}
print(json.dumps(out))
