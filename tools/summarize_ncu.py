"""Summarise an ncu --set full report and a launch-list CSV into profiles/ (text + JSON).
usage: python tools/summarize_ncu.py <report.ncu-rep> <launches.csv> <tag>"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]


def ncu_csv(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = ncu_csv("--page", "raw")
hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
m = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]
lines = [f"# ncu --set full summary ({tag}): one decode_mma_kernel launch (cfg2 layer, 64q/8kv, d128, B16, 32K)", ""]
for k in keys:
    if k in m:
        lines.append(f"{k:78s} {m[k]}")
stalls = {h: v for h, v in m.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
lines += ["", "## warp stall samples"]
for h, v in sorted(stalls.items(), key=lambda x: -float(x[1] or 0)):
    if float(v or 0) > 0:
        lines.append(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v}")
# per-opcode dynamic instruction mix
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
    ops[t.split()[0].split(".")[0] if t else "?"] += n
tot = sum(ops.values())
lines += ["", f"## dynamic SASS instruction mix (total {tot})"]
for op, n in ops.most_common(25):
    lines.append(f"{op:10s} {n:12d} {100.0 * n / tot:5.1f}%")
# launch list shares
rows = list(csv.reader(open(launches)))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hh = rows[start]
ik, iv, im = hh.index("Kernel Name"), hh.index("Metric Value"), hh.index("Metric Name")
dur = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        dur[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")))
lines += ["", "## launch list (ncu gpu__time_duration.sum, cold-cache serialised; compare shares)"]
total_ns = sum(sum(v) for v in dur.values())
for k, v in sorted(dur.items(), key=lambda x: -sum(x[1])):
    lines.append(f"{k[:60]:60s} n={len(v):5d} mean={sum(v) / len(v) / 1000:9.2f} us share={100 * sum(v) / total_ns:5.1f}%")
open(f"profiles/ncu_summary_{tag}.txt", "w").write("\n".join(lines) + "\n")
traffic = float(m.get("dram__bytes_read.sum", 0)) + float(m.get("dram__bytes_write.sum", 0))
unit = "MB"
json.dump({"tag": tag, "kernel": m.get("Kernel Name"), "dram_bytes_per_launch": traffic * 1e6,
           "dram_read_MB": float(m.get("dram__bytes_read.sum", 0)), "dram_write_MB": float(m.get("dram__bytes_write.sum", 0)),
           "duration_us": float(m.get("gpu__time_duration.sum", 0))},
          open("profiles/ncu_traffic.json", "w"), indent=1)
print("\n".join(lines[:40]))
