"""Quick look at one kernel of an ncu --set full report: key metrics, stall samples,
per-opcode dynamic instruction mix (development helper, not shipped)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]


def ncu_csv(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = ncu_csv("--page", "raw")
m = dict(zip(raw[0], raw[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "smsp__inst_executed.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
          "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]:
    print(f"{k:75s} {m.get(k)}")
stalls = {h: v for h, v in m.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
print(" ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v}" for h, v in
               sorted(stalls.items(), key=lambda x: -float(x[1] or 0))[:12]))
src = ncu_csv("--page", "source", "--print-source=sass")
h2 = src[1]
ix, isrc = h2.index("Instructions Executed"), h2.index("Source")
ops = collections.Counter()
for r in src[2:]:
    try:
        n = int(r[ix])
    except (ValueError, IndexError):
        continue
    t = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
    ops[t.split()[0] if t else "?"] += n
tot = sum(ops.values())
print("total", tot, " ".join(f"{op}={100 * n / tot:.1f}%" for op, n in ops.most_common(16)))
