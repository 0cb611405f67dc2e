"""Time the GPU calibration replay (calib.measure_raw) against the oracle restatement of
calibration.py:108-125 on one capture (development helper)."""
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import attention as oatt  # noqa: E402
from paper_2605_17170_b200 import calib  # noqa: E402

n, L, H, Hkv, d, n_tags = int(sys.argv[1]), 2, 64, 8, 128, 8
rng = np.random.default_rng(0)
layers = [SimpleNamespace(q=rng.standard_normal((n, H, d)).astype(np.float32),
                          k=rng.standard_normal((n, Hkv, d)).astype(np.float32),
                          v=rng.standard_normal((n, Hkv, d)).astype(np.float32)) for _ in range(L)]
cap = SimpleNamespace(request_id="c", layers=layers, tags=rng.integers(0, n_tags, n), group_len=32)
calib.measure_raw([cap])
torch.cuda.synchronize()
t0 = time.perf_counter()
got = calib.measure_raw([cap])
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
ref = oatt.measure_raw([cap])
t_cpu = time.perf_counter() - t0
worst = max(abs(got[k] - e) / abs(e) for k, e in ref.items())
print(f"N={n} layers={L} heads={H}/{Hkv} tags={n_tags}: GPU {t_gpu:.3f} s, CPU oracle {t_cpu:.1f} s "
      f"(x{t_cpu / t_gpu:.0f}), worst rel diff {worst:.2e}")
