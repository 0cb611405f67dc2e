"""Run the K1 (write_prefill data path) cfg3 slice a few times -- for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = bench.parse()
import json  # noqa: E402
print(json.dumps(bench.measure_k1(args, torch.device("cuda", 0), 6448.4), default=float))
