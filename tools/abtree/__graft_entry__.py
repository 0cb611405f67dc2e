"""Driver entry points: build() compiles the sm_100a library in-tree; smoke() runs one
small quantize+pack -> decode-attention pass on cuda:0 and checks it against the
CPU oracle (oracle/ is test infrastructure; smoke() may use it as the checker)."""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2605_17170_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkvmix_b200.so")
SOURCES = ["codec.cu", "decode.cu", "capi.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand == "nvcc" or os.path.exists(cand):
            return cand
    return "nvcc"


def build(force: bool = False) -> None:
    """Compile libkvmix_b200.so for sm_100a (cross-compiles without a GPU) and import the package."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("common.cuh", "launch.h")] + [
        os.path.join(ROOT, "include", "kvmix_b200.h")]
    stale = force or not os.path.exists(LIB) or any(os.path.getmtime(p) > os.path.getmtime(LIB) for p in deps)
    if stale:
        tmp = LIB + ".tmp"
        extra = os.environ.get("KVMIX_NVCC_EXTRA", "").split()
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp, *srcs]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import paper_2605_17170_b200  # noqa: F401


def smoke() -> None:
    """One tiny decode step on cuda:0 (cfg1 shape, 1 layer, 8 q / 2 kv heads, d=128,
    ~1.1K tokens) checked against the oracle: pool bytes bit-exact, attention within
    atol 2e-3 / rtol 1e-2 of the reference fp32 flash_decode."""
    build()
    import numpy as np
    import torch

    import paper_2605_17170_b200 as kv
    from paper_2605_17170_b200 import layout
    from oracle import attention as oatt
    from oracle import pool as opool

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    torch.cuda.set_device(0)
    rng = np.random.default_rng(20261017)
    L, H, Hq, d, N = 1, 2, 8, 128, 1100
    bits = np.where(rng.random(N) < 0.75, 2, 4)
    k = (rng.standard_normal((L, N, H, d)) * np.exp(rng.uniform(np.log(0.5), np.log(4.0), (H, d)))).astype(np.float32)
    v = rng.standard_normal((L, N, H, d)).astype(np.float32)
    q = rng.standard_normal((Hq, d)).astype(np.float32)
    cfg = kv.init_pool(2.5, 2 * N, L, H, d)
    pool = kv.MixedPrecisionPool(cfg)
    table = pool.alloc("r0", bits)
    pool.write_prefill(table, k, v)
    pool.partition(table)
    out = kv.flash_decode(q, table, pool.view(0))

    ocfg = opool.Config(cfg.total_slots, cfg.offset, L, H, d)
    op = opool.OraclePool(ocfg)
    op.alloc("r0", bits)
    op.write_prefill("r0", k, v)
    op.partition("r0")
    assert op.tables["r0"] == [int(s) for s in table.slots], "page indices differ from the oracle"
    n2 = pool.n_pages * pool.page_stride
    dev2 = pool.int2_pool[: L * H * n2].view(L, H, pool.n_pages, pool.page_stride).cpu().numpy()
    dev4 = pool.int4_pool[: L * H * pool.n_int4 * pool.slot_stride].view(L, H, pool.n_int4, pool.slot_stride).cpu().numpy()
    pw, sw = op.page_written, op.slot_written
    assert np.array_equal(layout.page_payloads(dev2[pw], d), op.int2[pw]), "INT2 page bytes differ from the oracle"
    assert np.array_equal(dev4[sw], layout.slot_records(op.int4[sw], d)), "INT4 slot bytes differ from the oracle"
    ref = oatt.flash_decode_pool(q, op, "r0", 0)
    err = np.abs(out - ref)
    assert np.all(err <= 2e-3 + 1e-2 * np.abs(ref)), f"attention mismatch: max abs err {err.max():.3e}"
    torch.cuda.synchronize()
    print(f"smoke ok: {N} tokens, bytes bit-exact, attention max abs err {err.max():.2e}")


if __name__ == "__main__":
    build()
    if len(sys.argv) > 1 and sys.argv[1] == "smoke":
        smoke()
