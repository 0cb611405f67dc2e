"""Run the e2e DecodeStep at cfg2 a few times (for an ncu launch list of one step's kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = bench.parse()
import __graft_entry__  # noqa: E402
__graft_entry__.build()
import paper_2605_17170_b200 as kv  # noqa: E402
dev = torch.device("cuda", 0)
pool, batch, q, out, bits, _ = bench.build_workload(args, dev, 0)
st = kv.DecodeStep(pool, batch.request_ids, n_q_heads=args.q_heads, dtype=torch.bfloat16, max_new_tokens=16)
for _ in range(6):
    st.run()
torch.cuda.synchronize()
print("ok")
