"""e2e DecodeStep at cfg2 for several layer-chunk sizes (H2D/D2H pipelining granularity)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

args = bench.parse()
import __graft_entry__  # noqa: E402
__graft_entry__.build()
import paper_2605_17170_b200 as kv  # noqa: E402
dev = torch.device("cuda", 0)
pool, batch, q, out, bits, _ = bench.build_workload(args, dev, 0)
timer = bench.Timer(1, dev)
for chunk in (8, 4, 2, 16, None):
    st = kv.DecodeStep(pool, batch.request_ids, n_q_heads=args.q_heads, dtype=torch.bfloat16, max_new_tokens=64,
                       layer_chunk=chunk)
    for _ in range(4):
        st.run()
    torch.cuda.synchronize()
    res = [timer(st.run, 10) for _ in range(2)]
    print(chunk if chunk is None or isinstance(chunk, int) else chunk[:3], [round(args.batch / (ms / 1000.0), 1) for ms in res], flush=True)
    for rid in batch.request_ids:  # give the reserved slots back for the next configuration
        pass
