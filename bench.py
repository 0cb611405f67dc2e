"""Benchmark: mixed INT2/INT4 split-K decode attention over the paged pool on B200.

Default workload (BASELINE.json configs[1], "cfg2"): Qwen3-VL-32B-shaped decode -- 64 layers,
64 q / 8 kv heads, head_dim 128, batch 16 per GPU, 32K-token tagged KV caches (per-token bits
from bench_data/tagged_bits.npz, produced by the reference's host tagger / calibration /
allocator at B=2.5).

* ``value``: one decode step's attention over all 64 layers with q/out resident in HBM --
  one CUDA-graph replay of 64 launches of the K2 split-decode kernel (its last CTA per
  (request, kv head) merges the split partials); tokens/s = batch / step time.  The roofline
  is K2's algorithmic bytes per launch / launch time against the measured HBM peak.
* ``e2e``: the same decode step through the public API with everything a real step does
  (``DecodeStep``): the host pops one INT4 slot per request (pool.py:284-306), the device
  appends the slots to its tables and re-plans (K7), q / k_new / v_new stream in from pinned
  host memory, every layer runs the fused append + attention (K4 in K2), outputs stream back.
* ``parity``: two (request, layer) units of THIS run (its own bf16 K/V/q, exact fp32 upcasts)
  re-run through the oracle's flash_decode (the reference's attention.py:175-218 restated) on
  the host, checked at the north_star tolerance (atol 2e-3, rtol 1e-2); the same units, timed
  on all host cores, are the ``cpu_baseline``.
* ``k1_prefill``: K1 quantize + pack on a cfg3 slice; ``churned``: K2 when every request's
  INT4 suffix is scattered over the pool (no contiguous slot runs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode decode|heads]

--gpus N > 1 re-launches itself under torch.distributed.run (one process per GPU, NCCL):
batch-parallel, every rank owns a full pool and its own 16 requests, no collective on the
data path (weak scaling); timing is the max over ranks.  --mode heads is cfg4 (100K context,
batch 32, KV heads sharded over the ranks, per-layer output all-gather).  Per-layer KV
(~0.46 GB) exceeds the 126 MB L2, so no L2 flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mixed INT2/INT4 decode-attn tokens/s & HBM GB/s frac (Qwen3-VL-32B shape, 32K)"
UNIT = "tokens/s"
ATOL, RTOL = 2e-3, 1e-2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["decode", "heads"], default="decode",
                    help="decode: cfg2 batch-parallel (default); heads: cfg4 KV-head-parallel")
    ap.add_argument("--batch", type=int, default=None, help="requests per GPU (decode) / total (heads)")
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--layers", type=int, default=64)
    ap.add_argument("--q-heads", type=int, default=64)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--int2-frac", type=float, default=None, help="override: i.i.d. bits with this INT2 fraction")
    ap.add_argument("--ctas-per-sm", type=int, default=3, help="stream-K planner: resident CTAs per SM")
    ap.add_argument("--int4-weight", type=float, default=0.8, help="stream-K planner: cost weight of INT4 bytes")
    ap.add_argument("--shards", type=int, default=None, help="heads mode: head shards (default: world size)")
    ap.add_argument("--combine", choices=["fused", "nccl"], default="fused",
                    help="heads mode: head all-gather fused into the decode kernel's epilogue (stores into the "
                         "ranks' symmetric-memory outputs over NVLink) or a per-layer NCCL all_gather_into_tensor")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-k1", action="store_true", help="skip the K1 quantize+pack (cfg3 slice) measurement")
    ap.add_argument("--no-churn", action="store_true", help="skip the scattered-INT4 (churned pool) measurement")
    ap.add_argument("--profile-only", action="store_true", help="build + a few steps, no JSON (for ncu)")
    a = ap.parse_args()
    if a.batch is None:
        a.batch = 32 if a.mode == "heads" else 16
    if a.ctx is None:
        a.ctx = 102400 if a.mode == "heads" else 32768
    return a


def workload_name(args) -> str:
    if args.mode == "heads":
        return (f"cfg4 decode attention: {args.layers} layers, {args.q_heads}q/{args.kv_heads}kv heads, d={args.head_dim}, "
                f"batch {args.batch}, {args.ctx // 1024}K ctx, KV heads sharded over the ranks")
    return (f"cfg2 decode attention: {args.layers} layers, {args.q_heads}q/{args.kv_heads}kv heads, d={args.head_dim}, "
            f"batch {args.batch}, {args.ctx // 1024}K ctx")


def config_dict(args, world: int) -> dict:
    """The workload, identical in both arms (the reference arm emits the same dict)."""
    par = (f"kv-head-parallel x{world}" if args.mode == "heads" else f"batch-parallel x{world}")
    return {"workload": workload_name(args), "layers": args.layers, "batch_per_gpu": args.batch
            if args.mode == "decode" else args.batch // max(1, world), "ctx": args.ctx, "q_heads": args.q_heads,
            "kv_heads": args.kv_heads, "head_dim": args.head_dim, "parallelism": par,
            "bits": "reference-tagged (bench_data/tagged_bits.npz, B=2.5)" if args.int2_frac is None
            else f"iid INT2 fraction {args.int2_frac}",
            "l2": "inputs larger than L2 (~0.46 GB KV per layer per GPU)"}


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "threads_env": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}}


def tagged_bits(n_req: int, ctx: int, seed_offset: int = 0) -> list[np.ndarray]:
    """Per-request bit maps: the reference-tagged maps when available for this context,
    else i.i.d. bits with the same INT2 fraction (0.8285)."""
    path = os.path.join(ROOT, "bench_data", "tagged_bits.npz")
    key = f"bits_{ctx}"
    out = []
    data = np.load(path) if os.path.exists(path) else {}
    if key in data:
        packed = data[key]
        for r in range(n_req):
            row = np.unpackbits(packed[(r + seed_offset) % packed.shape[0]])[:ctx]
            out.append(np.where(row == 1, 2, 4).astype(np.int8))
    else:
        rng = np.random.default_rng(20261017 + seed_offset)
        for _ in range(n_req):
            out.append(np.where(rng.random(ctx) < 0.8285, 2, 4).astype(np.int8))
    return out


def algorithmic_bytes_per_layer(batch_obj, n_q_heads, head_dim, n_batch=None) -> int:
    """KV payload bytes + q + o (bf16) + page-table ints."""
    t = batch_obj.csr
    kv = batch_obj.kv_bytes()
    qo = 2 * (n_batch or batch_obj.batch) * n_q_heads * head_dim * 2
    tables = 4 * int(t["n_pages"].sum() + t["n_int4"].sum())
    return int(kv + qo + tables)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------
# CPU legs: the oracle port of the reference decode (attention.py:175-218) on the host cores.
# A unit = one (request, layer) flash_decode at full context; its inputs travel as an .npz
# (bf16 K/V as their bit patterns, fp32 q, per-token bits).  The oracle pool build is not
# timed; each worker times `reps` decodes of its unit while every worker runs concurrently.


def _bf16_bits_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def _bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 (ties to even), returned as its exact fp32 value."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _cpu_worker(job):
    path, reps, want_out = job
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    from oracle import attention as oatt
    from oracle import pool as opool
    z = np.load(path)
    bits = z["bits"]
    k = _bf16_bits_to_f32(z["k16"]) if "k16" in z else z["k"]
    v = _bf16_bits_to_f32(z["v16"]) if "v16" in z else z["v"]
    q = z["q"]
    n, H, d = k.shape
    n2 = int((bits == 2).sum()) // 32 * 32
    op = opool.OraclePool(opool.Config(total_slots=n + 32, offset=n2, n_layers=1, n_kv_heads=H, head_dim=d))
    op.alloc("r", bits)
    op.write_prefill("r", k[None], v[None])
    op.partition("r")
    times, out = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = oatt.flash_decode_pool(q, op, "r", 0)
        times.append(time.perf_counter() - t0)
    return times, (out if want_out else None)


def cpu_units(unit_files, workers: int, reps: int):
    """Run the unit files on `workers` concurrent processes (worker i takes unit i % n).
    Returns (all per-decode times, the first worker's output of each unit, wall seconds)."""
    jobs = [(unit_files[i % len(unit_files)], reps, i < len(unit_files)) for i in range(workers)]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(workers) as p:
        res = p.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    times = [t for r in res for t in r[0]]
    outs = [res[i][1] for i in range(len(unit_files))]
    return times, outs, wall


def cpu_workers() -> int:
    return max(1, min(os.cpu_count() or 1, 64))


def synth_unit_files(args, n_units: int, tmpdir: str) -> list[str]:
    """Reference-arm inputs: the same workload shape with host-generated K/V/q (fp32 values
    rounded to bf16, K with per-channel log-uniform [0.5, 4] scales, capture.py:108-112)."""
    files = []
    for u in range(n_units):
        rng = np.random.default_rng(1000 + u)
        bits = tagged_bits(1, args.ctx, seed_offset=u)[0]
        ch = np.exp(rng.uniform(np.log(0.5), np.log(4.0), (args.kv_heads, args.head_dim))).astype(np.float32)
        k = _bf16_round(rng.standard_normal((args.ctx, args.kv_heads, args.head_dim), dtype=np.float32) * ch)
        v = _bf16_round(rng.standard_normal((args.ctx, args.kv_heads, args.head_dim), dtype=np.float32))
        q = _bf16_round(rng.standard_normal((args.q_heads, args.head_dim), dtype=np.float32))
        f = os.path.join(tmpdir, f"unit{u}.npz")
        np.savez(f, bits=bits, k=k, v=v, q=q)
        files.append(f)
    return files


def run_reference(args):
    """Reference arm: the reference's CPU decode path (the oracle port -- the reference is
    pure Python/numpy, run here through its restatement) on all host cores, on the same
    metric, unit and config as ours.  A "step" is one bounded sample round: every worker
    process decodes one full-context (request, layer) unit; tokens/s extrapolates the
    measured per-unit time to the batch x layers units of a decode step over the workers."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    workers = cpu_workers()
    with tempfile.TemporaryDirectory() as td:
        files = synth_unit_files(args, min(2, workers), td)
        times, _, wall = cpu_units(files, workers, args.warmup + args.steps)
    per_worker = args.warmup + args.steps
    timed = [t for w in range(workers) for t in times[w * per_worker + args.warmup:(w + 1) * per_worker]]
    t_unit = float(np.mean(timed))
    units_per_step = (args.batch if args.mode == "decode" else args.batch) * args.layers
    if args.mode == "heads":
        units_per_step = args.batch * args.layers  # a unit covers all kv heads of one request-layer
    value = workers / (t_unit * args.layers)  # = batch / (t_unit * units_per_step / workers)
    sample = (f"per step, each of {workers} processes (1 thread each) times one full-context (request, layer) "
              f"flash_decode of the oracle port (attention.py:175-218, numpy fp32) at {args.ctx} tokens, "
              f"{args.q_heads}/{args.kv_heads} heads, d={args.head_dim}; mean {t_unit:.3f} s per unit; "
              f"tokens/s = workers / (s per unit x {args.layers} layers), i.e. {units_per_step} units per decode step "
              f"spread over the workers; wall {wall:.1f} s incl. untimed oracle-pool builds")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_unit,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference-tagged per-token bits, random K/V/q (fp32 values rounded to bf16)",
        "config": config_dict(args, world),
        "step_definition": "one sample round (every worker decodes one (request, layer) unit); ms_per_step = "
                           "seconds per unit",
        "cpu_baseline": {"kind": "port", "cores": workers, "sample": sample, "value": value, "unit": UNIT},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------
def build_workload(args, device, rank: int, heads=None, sample_units=()):
    """Pool + tables for args.batch requests of args.ctx tokens (all layers), bf16 K/V drawn on
    the GPU and quantized by K1 in 8-layer slices.  heads = (h0, h1) keeps only that KV-head
    slice (head-parallel shard).  sample_units [(request, layer)]: host copies of those units'
    bf16 K/V (for the parity / CPU legs)."""
    import torch

    import paper_2605_17170_b200 as kv

    L, H, d, B, N = args.layers, args.kv_heads, args.head_dim, args.batch, args.ctx
    h0, h1 = heads if heads is not None else (0, H)
    Hs = h1 - h0
    bits = tagged_bits(B, N, seed_offset=rank * B if heads is None else 0)
    if args.int2_frac is not None:
        rng = np.random.default_rng(7 + rank)
        bits = [np.where(rng.random(N) < args.int2_frac, 2, 4).astype(np.int8) for _ in range(B)]
    g = 32
    n_pages = [int((b == 2).sum()) // g for b in bits]
    n_int4 = [N - p * g for p in n_pages]
    decode_room = 256 * B
    cfg = kv.PoolConfig(total_slots=sum(n_pages) * g + sum(n_int4) + decode_room, offset=sum(n_pages) * g,
                        n_layers=L, n_kv_heads=Hs, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(20261017 + (rank if heads is None else 0))
    ch_scale = torch.exp(torch.empty((H, d), device=device).uniform_(math.log(0.5), math.log(4.0), generator=gen))
    rids, samples = [], {}
    lchunk = 8  # layers per prefill call keeps the bf16 K/V staging at ~1 GB
    for r in range(B):
        rid = f"req{r}"
        table = pool.alloc(rid, bits[r])
        for l0 in range(0, L, lchunk):
            nl = min(lchunk, L - l0)
            k = (torch.randn((nl, N, H, d), device=device, generator=gen) * ch_scale).to(torch.bfloat16)
            v = torch.randn((nl, N, H, d), device=device, generator=gen).to(torch.bfloat16)
            if heads is not None:
                k, v = k[:, :, h0:h1].contiguous(), v[:, :, h0:h1].contiguous()
            _prefill_layers(pool, table, k, v, l0)
            for (rs, ls) in sample_units:
                if rs == r and l0 <= ls < l0 + nl:
                    samples[(rs, ls)] = {"bits": bits[r], "k16": k[ls - l0].view(torch.int16).cpu().numpy().view(np.uint16),
                                         "v16": v[ls - l0].view(torch.int16).cpu().numpy().view(np.uint16)}
            del k, v
        pool.partition(table)
        rids.append(rid)
    torch.cuda.synchronize()
    Hq = args.q_heads * Hs // H
    batch = kv.DecodeBatch(pool, rids, n_q_heads=Hq, ctas_per_sm=args.ctas_per_sm, int4_weight=args.int4_weight)
    q = torch.randn((L, B, Hq, d), device=device, generator=gen).to(torch.bfloat16)
    out = torch.empty_like(q)
    return pool, batch, q, out, bits, samples


def _prefill_layers(pool, table, k, v, l0):
    """write_prefill for a layer slice (the pool API writes all layers; the bench streams 8
    layers at a time to bound the staging memory) via the same C-ABI entry point."""
    import torch

    from paper_2605_17170_b200 import _lib
    cfg, g = pool.config, pool.config.page_size
    s = table.slots
    is2 = s < cfg.offset
    t2 = np.flatnonzero(is2)
    t4 = np.flatnonzero(~is2)
    pt = torch.as_tensor(t2.reshape(-1, g).astype(np.int32), device=pool.device)
    pi = torch.as_tensor((s[t2[::g]] // g).astype(np.int32), device=pool.device)
    it = torch.as_tensor(t4.astype(np.int32), device=pool.device)
    ii = torch.as_tensor((s[t4] - cfg.offset).astype(np.int32), device=pool.device)
    lh = l0 * cfg.n_kv_heads
    _lib.check(_lib.lib.kvmix_write_prefill(
        k.data_ptr(), v.data_ptr(), _lib.dtype_code(k), k.shape[0], k.shape[1], cfg.n_kv_heads, cfg.head_dim,
        pt.data_ptr(), pi.data_ptr(), pt.shape[0], it.data_ptr(), ii.data_ptr(), t4.size,
        pool.int2_pool.data_ptr() + lh * pool.n_pages * pool.page_stride, pool.n_pages,
        pool.int4_pool.data_ptr() + lh * pool.n_int4 * pool.slot_stride, pool.n_int4, pool.status.data_ptr(),
        _lib.stream()))
    pool._written = True
    pool._page_written[l0:l0 + k.shape[0], :, s[t2[::g]] // g] = True
    pool._int4_written[l0:l0 + k.shape[0], :, s[t4] - cfg.offset] = True


def peak_hbm() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return float(json.load(open(path))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic() -> tuple[float | None, str]:
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        t = json.load(open(path))
        return t.get("dram_bytes_per_launch"), f"committed ncu --set full capture ({t.get('source', 'profiles/')})"
    return None, "none"


class Timer:
    """CUDA-event timing on the launching stream, barrier + synchronize on both sides, max over ranks."""

    def __init__(self, world, device):
        self.world, self.device = world, device

    def __call__(self, fn, k):
        import torch
        import torch.distributed as dist
        stream = torch.cuda.current_stream()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        if self.world > 1:
            t = torch.tensor([ms], device=self.device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms


def capture(fn):
    """CUDA graph of fn (launched once eagerly on the capture stream first)."""
    import torch
    graph = torch.cuda.CUDAGraph()
    s_cap = torch.cuda.Stream()
    s_cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_cap):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s_cap):
            fn()
    torch.cuda.current_stream().wait_stream(s_cap)
    torch.cuda.synchronize()
    return graph


def measure_churned(args, pool, batch, q, out, timer, peak) -> dict:
    """K2 on the same requests with every INT4 suffix scattered over the pool: each request's
    INT4 entries are replaced by a random sample of the pool's written INT4 slots (the layout
    after churn and interleaved decode appends, SURVEY 7 hard part 3), so no two consecutive
    entries share a slot run and every INT4 tile is 32 separate 160 B copies."""
    import torch

    import paper_2605_17170_b200 as kv
    cfg = pool.config
    rng = np.random.default_rng(99)
    written = np.flatnonzero(pool._int4_written[0, 0]) + cfg.offset
    tables = []
    for rid in batch.request_ids:
        s = pool.table(rid).slots
        n2 = int((s < cfg.offset).sum())
        tables.append(np.concatenate([s[:n2], rng.choice(written, size=s.size - n2, replace=False)]))
    b2 = kv.DecodeBatch(pool, n_q_heads=batch.n_q_heads, tables=tables, ctas_per_sm=args.ctas_per_sm,
                        int4_weight=args.int4_weight)
    runs = [int(np.count_nonzero(np.diff(t[(t >= cfg.offset)]) == 1)) for t in tables]
    L = args.layers

    def step():
        for layer in range(L):
            kv.flash_decode_batched(q[layer], b2, layer, out=out[layer])
    g = capture(step)
    for _ in range(3):
        g.replay()
    ms = timer(g.replay, max(5, args.steps // 2))
    alg = algorithmic_bytes_per_layer(b2, batch.n_q_heads, args.head_dim)
    ach = alg / (ms / L / 1000.0) / 1e9
    return {"workload": "cfg2 with scattered INT4 suffixes", "value": args.batch / (ms / 1000.0), "unit": UNIT,
            "ms_per_step": ms, "k2_ms_per_launch": ms / L, "achieved_gbs": ach, "frac": ach / peak,
            "adjacent_int4_pairs_per_request_max": max(runs)}


def measure_decode_step(args, pool, rids, Hq, timer, world) -> dict:
    """e2e: DecodeStep through the public API (host slot pops, device tables + plan, pinned
    host q / k_new / v_new in, append + attention for all layers, outputs back)."""
    import torch

    import paper_2605_17170_b200 as kv
    n_runs = args.warmup + args.steps + 4
    st = kv.DecodeStep(pool, rids, n_q_heads=Hq, dtype=torch.bfloat16, max_new_tokens=n_runs + 8)
    gen = torch.Generator().manual_seed(5)
    st.q_host.copy_(torch.randn(st.q_host.shape, generator=gen).to(torch.bfloat16))
    st.k_host.copy_(torch.randn(st.k_host.shape, generator=gen).to(torch.bfloat16))
    st.v_host.copy_(torch.randn(st.v_host.shape, generator=gen).to(torch.bfloat16))
    for _ in range(max(3, args.warmup)):
        st.run()
    torch.cuda.synchronize()
    host_s = []

    def one():
        t0 = time.perf_counter()
        st.run()
        host_s.append(time.perf_counter() - t0)
    ms = timer(one, args.steps)
    st.check()
    nb_in = sum(t.numel() * t.element_size() for t in (st.q_host, st.k_host, st.v_host)) + st.slots_host.numel() * 4
    nb_out = st.out_host.numel() * st.out_host.element_size()
    return {"value": world * args.batch / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": nb_in,
            "d2h_bytes_per_step": nb_out, "ms_per_step": ms,
            "host_ms_per_step": 1000.0 * float(np.median(host_s)),
            "what": "DecodeStep.run(): per step the host pops one INT4 slot per request (pool.py:284-306 LIFO), "
                    "then one CUDA graph: slots H2D, K7 device tables + stream-K plan, q/k_new/v_new H2D from pinned "
                    "memory (layer chunks on a side stream), "
                    + (f"{args.layers} fused append+attention launches" if st.fused_append else
                       f"per {st.chunks[0][1] - st.chunks[0][0]}-layer chunk one batched INT4 append launch before its attention "
                       f"launches ({args.layers} in all)")
                    + ", outputs D2H",
            "gpu_launches_per_step": 1 + args.layers + (0 if st.fused_append else len(st.chunks))}


def cpu_leg(args, samples, outs_dev, qs) -> tuple[dict, dict]:
    """Parity + CPU baseline on this run's own sampled units: the oracle decodes each unit from
    the exact fp32 upcasts of the bf16 K/V/q the GPU used, on all host cores."""
    workers = cpu_workers()
    with tempfile.TemporaryDirectory() as td:
        files = []
        for i, key in enumerate(sorted(samples)):
            f = os.path.join(td, f"unit{i}.npz")
            s = samples[key]
            np.savez(f, bits=s["bits"], k16=s["k16"], v16=s["v16"], q=qs[key])
            files.append(f)
        times, outs, wall = cpu_units(files, workers, 1)
    errs, worst = [], []
    for key, o in zip(sorted(samples), outs):
        ref = o.astype(np.float64)
        dv = outs_dev[key].astype(np.float64)
        e = np.abs(dv - ref)
        errs.append(float(e.max()))
        worst.append(float((e / (ATOL + RTOL * np.abs(ref))).max()))
    t_unit = float(np.mean(times))
    parity = {"units_checked": len(samples), "units": [list(k) for k in sorted(samples)],
              "max_abs_err": max(errs), "worst_err_over_tol": max(worst), "atol": ATOL, "rtol": RTOL,
              "pass": bool(max(worst) <= 1.0), "output_dtype": "bf16",
              "vs": "oracle flash_decode (attention.py:175-218 restated, fp32) on this run's bf16 K/V/q (exact fp32 upcast)"}
    cpu = {"value": workers / (t_unit * args.layers), "unit": UNIT, "cores": workers, "kind": "port",
           "sample": (f"the {len(samples)} parity units of this run (full {args.ctx}-token context, "
                      f"{args.q_heads}/{args.kv_heads} heads), each decoded by the oracle port on one thread; "
                      f"{workers} processes busy at once; mean {t_unit:.3f} s per (request, layer) unit; tokens/s = "
                      f"workers / (s per unit x {args.layers} layers); wall {wall:.1f} s incl. untimed pool builds")}
    return parity, cpu


def run_decode(args, world, rank, local, device):
    import torch
    import torch.distributed as dist

    import paper_2605_17170_b200 as kv

    L = args.layers
    # K1 first, on a fresh allocator state: re-allocated memory (after the decode legs free their
    # pools) measured ~8% slower for this scattered-row gather (K1)
    k1 = measure_k1(args, device, peak_hbm()[0]) if (rank == 0 and not args.no_k1 and not args.profile_only) else None
    sample_units = [(0, 0), (args.batch - 1, L - 1)] if rank == 0 else []
    pool, batch, q, out, bits, samples = build_workload(args, device, rank, sample_units=sample_units)
    timer = Timer(world, device)

    def step(variant=args.variant):
        for layer in range(L):
            kv.flash_decode_batched(q[layer], batch, layer, out=out[layer], variant=variant)

    for _ in range(max(args.warmup, 1)):
        step()
    graph = capture(step)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if args.profile_only:
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        return
    with ClockSampler(local) as clocks:
        ms_step = timer(graph.replay, args.steps)
    ms_k2 = ms_step / L  # one launch per layer (K2 with the fused combine)
    outs_dev = {key: out[key[1], key[0]].float().cpu().numpy() for key in samples}
    qs = {key: q[key[1], key[0]].float().cpu().numpy() for key in samples}
    peak, peak_src = peak_hbm()
    alg = algorithmic_bytes_per_layer(batch, args.q_heads, args.head_dim)
    achieved = alg / (ms_k2 / 1000.0) / 1e9
    churn = None if args.no_churn else measure_churned(args, pool, batch, q, out, timer, peak)
    e2e = None if args.no_e2e else measure_decode_step(args, pool, batch.request_ids, args.q_heads, timer, world)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    traffic, traffic_src = committed_traffic()
    n2 = int(batch.csr["n_pages"].sum()) * 32
    ntok = int(batch.n_tokens.sum())
    cfgd = config_dict(args, world)  # identical to the reference arm's (run facts go to "workload_stats")
    line = {
        "metric": METRIC, "value": world * args.batch / (ms_step / 1000.0), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "int2/int4 KV codes; fp16 tensor-core MMA (exact q*s hi/lo, normal-fp16 key codes), fp32 accumulate; bf16 q/o",
        "data": "synthetic: reference-tagged per-token bits (B=2.5), random bf16 K/V and q",
        "config": cfgd,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                     "kernel": "decode_mma_kernel (K2 split decode + fused combine)",
                     "algorithmic_bytes_per_launch": alg, "k2_ms_per_launch": ms_k2},
        "e2e": e2e,
        "gpu_launches": args.steps * L,
        "clocks": clocks.summary(),
        "host": host_info(),
        "workload_stats": {"stored_int2_fraction": n2 / ntok,
                           "schedule": f"stream-K: {batch.n_cta} CTAs, {batch.n_pieces} pieces, "
                                       f"{batch.n_parts} partials per layer"},
    }
    if churn is not None:
        line["churned"] = churn
    if k1 is not None:
        line["k1_prefill"] = k1
    if not args.no_cpu_baseline and world == 1 and samples:
        del pool, batch, q, out
        torch.cuda.empty_cache()
        line["parity"], line["cpu_baseline"] = cpu_leg(args, samples, outs_dev, qs)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_k1(args, device, peak) -> dict:
    """K1 (quantize + pack into the mixed pool, write_prefill's data path) on a cfg3 slice:
    one 128K-token request whose per-token bits are the concatenated reference-tagged
    bits of 4 x 32K-token traces, 8 of cfg3's 64 layers, 8 kv heads, d=128, bf16 K/V
    resident in HBM.  Algorithmic bytes = bf16 K+V in + packed records out."""
    import torch

    import paper_2605_17170_b200 as kv
    L, H, d, N = 8, args.kv_heads, args.head_dim, 4 * 32768
    bits = np.concatenate(tagged_bits(4, 32768, seed_offset=100))
    g = 32
    n_pages = int((bits == 2).sum()) // g
    n4 = N - n_pages * g
    cfg = kv.PoolConfig(total_slots=N, offset=n_pages * g, n_layers=L, n_kv_heads=H, head_dim=d)
    pool = kv.MixedPrecisionPool(cfg, device=device)
    table = pool.alloc("trace", bits)
    gen = torch.Generator(device=device)
    gen.manual_seed(7)
    k = torch.randn((L, N, H, d), device=device, generator=gen).to(torch.bfloat16)
    v = torch.randn((L, N, H, d), device=device, generator=gen).to(torch.bfloat16)
    from paper_2605_17170_b200 import _lib
    s_ = table.slots
    is2 = s_ < cfg.offset
    t2, t4 = np.flatnonzero(is2), np.flatnonzero(~is2)
    pt = torch.as_tensor(t2.reshape(-1, g).astype(np.int32), device=device)
    pi = torch.as_tensor((s_[t2[::g]] // g).astype(np.int32), device=device)
    it = torch.as_tensor(t4.astype(np.int32), device=device)
    ii = torch.as_tensor((s_[t4] - cfg.offset).astype(np.int32), device=device)

    def k1():  # the write_prefill data path with device-resident page lists
        _lib.check(_lib.lib.kvmix_write_prefill(
            k.data_ptr(), v.data_ptr(), _lib.dtype_code(k), L, N, H, d, pt.data_ptr(), pi.data_ptr(), pt.shape[0],
            it.data_ptr(), ii.data_ptr(), t4.size, pool.int2_pool.data_ptr(), pool.n_pages, pool.int4_pool.data_ptr(),
            pool.n_int4, pool.status.data_ptr(), _lib.stream()))

    for _ in range(3):  # first touches of the fresh pool and warm clocks
        k1()
    torch.cuda.synchronize()
    reps, times = 10, []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        k1()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    route = measure_route(bits, cfg, device)
    bytes_in = 2 * k.numel() * k.element_size()
    bytes_out = L * H * (n_pages * pool.page_stride + n4 * 2 * kv.token_block_payload_bytes(d, 4))
    gbs = (bytes_in + bytes_out) / (ms / 1000.0) / 1e9
    del k, v, pool
    torch.cuda.empty_cache()
    return {"workload": "cfg3 slice: 128K-token tagged trace, 8 of 64 layers, 8 kv heads, d=128, bf16 in",
            "ms_per_call": ms, "ms_per_layer": ms / L, "cfg3_ms_64_layers": ms / L * 64,
            "bytes_in": bytes_in, "bytes_out": int(bytes_out), "achieved_gbs": gbs, "frac": gbs / peak,
            "stored_int2_fraction": n_pages * g / N, "kernels": "prefill_pages_kernel + int4_tokens_kernel",
            "k6_route": route}


def measure_route(bits, cfg, device) -> dict:
    """K6 (device-side page-table build) on the same 128K-token request: the two routing
    kernels alone (CUDA events), alloc_device end to end (wall, incl. the count read-back,
    pops and the slots download) and the host allocator (wall) for comparison."""
    import time

    import torch

    import paper_2605_17170_b200 as kv
    from paper_2605_17170_b200 import _lib
    g, n = cfg.page_size, bits.size
    bd = torch.as_tensor(bits, device=device).to(torch.int8)
    n_pages = int((bits == 2).sum()) // g
    m = n - n_pages * g
    st = torch.arange(n_pages, device=device, dtype=torch.int64) * g
    po = torch.arange(m, device=device, dtype=torch.int64) + cfg.offset
    slots = torch.empty(n, dtype=torch.int64, device=device)
    pt = torch.empty(n_pages * g, dtype=torch.int32, device=device)
    pi = torch.empty(n_pages, dtype=torch.int32, device=device)
    it = torch.empty(m, dtype=torch.int32, device=device)
    ii = torch.empty(m, dtype=torch.int32, device=device)
    err = torch.zeros(1, dtype=torch.int32, device=device)
    cnt = torch.zeros(int(_lib.lib.kvmix_route_scratch_elems(n)), dtype=torch.int64, device=device)

    def kernels():
        _lib.check(_lib.lib.kvmix_count_int2(bd.data_ptr(), n, cnt.data_ptr(), err.data_ptr(), _lib.stream()))
        _lib.check(_lib.lib.kvmix_route_tokens(bd.data_ptr(), n, g, cnt.data_ptr(), st.data_ptr(), n_pages,
                                               po.data_ptr(), m,
                                               cfg.offset, slots.data_ptr(), pt.data_ptr(), pi.data_ptr(),
                                               it.data_ptr(), ii.data_ptr(), err.data_ptr(), _lib.stream()))
    kernels()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        kernels()
    e1.record()
    torch.cuda.synchronize()
    kern_ms = e0.elapsed_time(e1) / 10

    def wall(fn, reps=5):
        best = float("inf")
        for r in range(reps):
            pool = kv.MixedPrecisionPool(cfg, device=device)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(pool, f"r{r}")
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
            del pool
        return best * 1e3
    dev_ms = wall(lambda p, rid: p.alloc_device(rid, bd))
    host_ms = wall(lambda p, rid: p.alloc(rid, bits))
    return {"tokens": int(n), "kernels_ms": kern_ms, "alloc_device_ms": dev_ms, "alloc_host_ms": host_ms,
            "kernels": "count_int2_kernel + route_tokens_kernel"}


def run_heads(args, world, rank, local, device):
    """cfg4: KV-head-parallel decode.  Rank r owns KV heads [r H/S, (r+1) H/S) (and their GQA q
    heads) of every request; page tables are replicated (every rank runs the same allocator
    sequence, so slots agree -- slot addresses are head-agnostic, pool.py:108-110).  Per layer
    each rank decodes its heads and the [B, Hq, d] output is assembled either inside the decode
    kernel (--combine fused: its epilogue stores the head slice into every rank's symmetric-memory
    output over NVLink, one device barrier per step) or by one NCCL all_gather_into_tensor per
    layer (--combine nccl, the baseline).  On one GPU (world 1) --shards S measures one shard of
    an S-way split; the fused combine then stores into the local [B, Hq, d] buffer only."""
    import torch
    import torch.distributed as dist

    import paper_2605_17170_b200 as kv
    from paper_2605_17170_b200 import dist as kvdist

    S = args.shards or world
    H, L, d = args.kv_heads, args.layers, args.head_dim
    if H % S or (world > 1 and S != world):
        raise SystemExit(f"heads mode: {H} kv heads over {S} shards / {world} ranks")
    hs = H // S
    shard = rank if world > 1 else 0
    pool, batch, q, out, bits, _ = build_workload(args, device, rank, heads=(shard * hs, (shard + 1) * hs))
    hq = args.q_heads // S
    timer = Timer(world, device)
    fused = args.combine == "fused"
    if fused and world > 1:
        sg = kvdist.SymmetricHeadGather(L, args.batch, args.q_heads, d, dtype=out.dtype, device=device)
        dests = [sg.layer(layer) for layer in range(L)]
    elif fused:
        full = torch.empty((L, args.batch, args.q_heads, d), dtype=out.dtype, device=device)
        dests = [kvdist.HeadOutputs.local([full[layer]], head0=shard * hq) for layer in range(L)]
    else:
        gathered = torch.empty((L, world * args.batch, hq, d), dtype=out.dtype, device=device)

    def attn():
        for layer in range(L):
            kv.flash_decode_batched(q[layer], batch, layer, out=out[layer])

    def step():
        for layer in range(L):
            if fused:
                kv.flash_decode_batched(q[layer], batch, layer, gather=dests[layer])
            else:
                kv.flash_decode_batched(q[layer], batch, layer, out=out[layer])
                if world > 1:
                    dist.all_gather_into_tensor(gathered[layer], out[layer])
        if fused and world > 1:
            sg.barrier()  # every rank's head slices have landed in every rank's output

    for _ in range(max(args.warmup, 1)):
        step()
    g_attn = capture(attn)
    if world > 1 and fused:
        step_fn = step  # eager: the symmetric-memory barrier stays outside a graph
    elif world > 1 or fused:
        g_step = capture(step)
        for _ in range(2):
            g_step.replay()
        step_fn = g_step.replay
    else:
        step_fn = None
    # attention-only and full steps timed alternately (3 rounds, medians): long cfg4 shards run
    # into the power cap, which a back-to-back pair would charge to whichever ran second
    t_attn, t_step = [], []
    for _ in range(3):
        t_attn.append(timer(g_attn.replay, args.steps))
        if step_fn is not None:
            t_step.append(timer(step_fn, args.steps))
    ms_attn = float(np.median(t_attn))
    ms_step = float(np.median(t_step)) if t_step else ms_attn
    if fused and world == 1:  # the shard's slice landed in the full-size output, equal to the plain decode's
        torch.cuda.synchronize()
        attn()
        torch.cuda.synchronize()
        if not torch.equal(full[:, :, :hq], out):
            raise SystemExit("heads mode: the fused gather's output differs from the plain decode")
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    peak, peak_src = peak_hbm()
    alg = algorithmic_bytes_per_layer(batch, hq, d)
    achieved = alg / (ms_attn / L / 1000.0) / 1e9
    cfgd = config_dict(args, world)
    if world == 1:
        note = ("one GPU holds one shard of an S-way split: the number is that shard's attention"
                + ("; the fused combine stores into the local [B, Hq, d] output only (no peers)" if fused
                   else "; the output all-gather is not measured"))
    else:
        note = ("head slices stored by the decode kernel into every rank's symmetric-memory output over NVLink, "
                "one device barrier per step" if fused else "per-layer NCCL all_gather_into_tensor")
    cfgd.update({"shards": S, "kv_heads_per_shard": hs, "measured_shard": shard, "combine": args.combine,
                 "note": note})
    line = {
        "metric": METRIC, "value": args.batch / (ms_step / 1000.0), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int2/int4 KV codes; fp16 MMA, fp32 accumulate; bf16 q/o",
        "data": "synthetic: reference-tagged per-token bits (B=2.5), random bf16 K/V and q",
        "config": cfgd,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src, "kernel": "decode_mma_kernel (shard)",
                     "algorithmic_bytes_per_launch": alg, "k2_ms_per_launch": ms_attn / L},
        "attention_ms_per_step": ms_attn, "gather_ms_per_step": ms_step - ms_attn,
        "gpu_launches": args.steps * L, "host": host_info(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def launch_ranks(args) -> int:
    """--gpus N without a torch.distributed launcher: re-run this script under
    torch.distributed.run with one process per GPU (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    if args.mode == "heads":
        run_heads(args, world, rank, local, device)
    else:
        run_decode(args, world, rank, local, device)


if __name__ == "__main__":
    main()
