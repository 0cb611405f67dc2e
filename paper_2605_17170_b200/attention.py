"""Split-K mixed INT2/INT4 flash-decode attention over the device pool.

Drop-in for the decode half of /root/reference/pkg/src/kvmix/attention.py:
``flash_decode`` keeps its signature (:175) and validation order (:188-201) and
returns a numpy [H, d] float32 array like the reference; ``merge_partials`` (:154)
and ``SplitPartial`` (:145) keep their meaning.  The work is done by the sm_100a
kernel K2 of libkvmix_b200 (tensor-core split decode; CTAs stream byte-balanced tile
ranges and the last CTA of a split (request, kv head) merges its partials -- the
combine K3 is fused in).

``DecodeBatch`` / ``flash_decode_batched`` are the native hot-path API: a batch of
requests, one layer per call, q/out as device tensors, page tables resident on the
device, no host synchronisation.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import ValidationError
from .plan import NUM_SMS_B200, plan_stream
from .pool import MixedPrecisionPool, PageTable, csr_tables, split_partitioned

VARIANT_TENSOR_CORE = 0  # one warp per tile stream (QK + softmax + PV), 4 warps per CTA, 3 CTAs per SM
VARIANT_SIMPLE = 1       # CUDA-core fp32 cross-check
CTAS_PER_SM = 3          # resident CTAs of the variant-0 kernel (168 regs x 128 threads, ~50 KB smem)


@dataclass
class SplitPartial:
    """Per-split attention state for one query head (attention.py:145-151)."""

    acc: np.ndarray
    lse: float
    max_logit: float


def merge_partials(parts: Sequence[SplitPartial]) -> np.ndarray:
    """attention.py:154-165, on the GPU (natural-log domain, fp32)."""
    if not parts:
        raise ValidationError("cannot merge an empty partial list")
    dev = _lib.require_cuda()
    acc = torch.as_tensor(np.stack([np.asarray(p.acc, dtype=np.float32) for p in parts]), device=dev)
    lse = torch.tensor([p.lse for p in parts], dtype=torch.float32, device=dev)
    mx = torch.tensor([p.max_logit for p in parts], dtype=torch.float32, device=dev)
    out = torch.empty(acc.shape[1], dtype=torch.float32, device=dev)
    _lib.check(lib.kvmix_merge_partials(acc.data_ptr(), lse.data_ptr(), mx.data_ptr(), acc.shape[0],
                                        acc.shape[1], out.data_ptr(), _lib.stream()))
    return out.cpu().numpy()


class DecodeBatch:
    """Device-resident CSR page tables + stream-K plan (pieces, CTA ranges, partial slots,
    arrival counters) for a request batch.  One batch is used on one stream at a time."""

    def __init__(self, pool: MixedPrecisionPool, request_ids=None, n_q_heads: int | None = None,
                 tables: list | None = None, **plan_kw):
        self.pool = pool
        cfg = pool.config
        self.n_q_heads = n_q_heads or cfg.n_kv_heads
        if self.n_q_heads % cfg.n_kv_heads:
            raise ValidationError("n_heads not a multiple of the pool's n_kv_heads")
        if self.n_q_heads // cfg.n_kv_heads > 8:
            raise ValidationError("GQA group larger than 8 is not supported on device")
        self.request_ids = list(request_ids) if request_ids is not None else None
        self._tables = tables
        self.plan_kw = plan_kw
        self.refresh()

    def refresh(self) -> None:
        """Rebuild device tables and the plan (after appends / new requests)."""
        pool, cfg = self.pool, self.pool.config
        if self._tables is not None:
            parts = [split_partitioned(t.slots if isinstance(t, PageTable) else np.asarray(t), cfg.offset,
                                       cfg.page_size) for t in self._tables]
            t = csr_tables([p for p, _ in parts], [i for _, i in parts], pool.device)
        else:
            t = pool.device_tables(self.request_ids)
        self.batch = int(t["n_pages"].size)
        self.csr = t
        kw = dict(self.plan_kw)
        if "n_cta" not in kw:
            n_sm = NUM_SMS_B200
            if pool.device is not None and pool.device.type == "cuda":
                n_sm = torch.cuda.get_device_properties(pool.device).multi_processor_count
            kw["n_cta"] = n_sm * int(kw.pop("ctas_per_sm", CTAS_PER_SM))
            kw["n_sm"] = n_sm
        else:
            kw.pop("ctas_per_sm", None)
        work, cta_ptr, n_parts = plan_stream(t["n_pages"], t["n_int4"], cfg.n_kv_heads, pool.page_stride,
                                             pool.slot_stride, **kw)
        dev = pool.device
        self.work = torch.as_tensor(work, device=dev)
        self.cta_ptr = torch.as_tensor(cta_ptr, device=dev)
        self.n_cta = int(cta_ptr.size - 1)
        self.n_pieces = int(work.shape[0])
        self.n_parts = n_parts
        self.partials = torch.empty(max(1, n_parts) * 8 * (cfg.head_dim + 4), dtype=torch.float32, device=dev)
        self.counters = torch.zeros(self.batch * cfg.n_kv_heads, dtype=torch.int32, device=dev)
        self.n_tokens = t["n_pages"] * cfg.page_size + t["n_int4"]
        # newest INT4 slot of each request (the fused decode append's target), host side
        self.last_int4 = None
        if self.request_ids is not None and np.all(t["n_int4"] > 0):
            self.last_int4 = np.array([int(pool.table(r).slots[-1]) for r in self.request_ids], dtype=np.int64)

    def kv_bytes(self) -> int:
        """Algorithmic KV bytes one layer's decode reads (all kv heads)."""
        cfg = self.pool.config
        from .quant import key_page_payload_bytes, token_block_payload_bytes
        per_page = key_page_payload_bytes(cfg.head_dim) + 32 * token_block_payload_bytes(cfg.head_dim, 2)
        per_int4 = 2 * token_block_payload_bytes(cfg.head_dim, 4)
        return int(cfg.n_kv_heads * (self.csr["n_pages"].sum() * per_page + self.csr["n_int4"].sum() * per_int4))


def flash_decode_batched(q: torch.Tensor, batch: DecodeBatch, layer: int, out: torch.Tensor | None = None,
                         scale: float | None = None, variant: int = VARIANT_TENSOR_CORE,
                         append: tuple | None = None, gather=None) -> torch.Tensor | None:
    """Decode attention for every request of ``batch`` at ``layer``.

    q: [B, n_q_heads, d] device tensor (f32/bf16/f16); returns out [B, n_q_heads, d]
    (dtype of q unless ``out`` is given).  Asynchronous on the current stream.

    append=(k_new, v_new), each [B, n_kv_heads, d] on the device: the K4 fused decode append.
    The newest INT4 slot of every request (reserved with ``pool.reserve_decode_slots`` before
    ``batch.refresh()``) receives this layer's k/v, quantized inside the attention kernel
    by the warp that reads it, and the new token is attended to (pool.py:284-306 followed by
    attention.py:175-218, in one launch).

    gather=``dist.HeadOutputs``: the KV-head-parallel combine fused into the kernel -- this
    rank's head slice is stored at its head offset into every destination buffer (its own and
    its peers', mapped over NVLink), so no all-gather follows (``out`` must be None; returns
    None: the result is in the destinations once every rank's launch is done).
    """
    pool, cfg = batch.pool, batch.pool.config
    if q.dim() != 3 or q.shape[0] != batch.batch or q.shape[1] != batch.n_q_heads or q.shape[2] != cfg.head_dim:
        raise ValidationError(f"q must be [{batch.batch}, {batch.n_q_heads}, {cfg.head_dim}]")
    if not 0 <= layer < cfg.n_layers:
        raise ValidationError("layer out of range")
    if q.device != pool.device:
        raise ValidationError(f"q must be on the pool's device {pool.device}")
    if not q.is_contiguous():
        q = q.contiguous()
    if out is None:
        if gather is None:
            out = torch.empty_like(q)
    elif gather is not None:
        raise ValidationError("out and gather are exclusive: the gather destinations are the output")
    elif (tuple(out.shape) != tuple(q.shape) or not out.is_contiguous() or out.device != pool.device
          or out.dtype not in (torch.float32, torch.bfloat16, torch.float16)):
        raise ValidationError(f"out must be a contiguous f32/bf16/f16 [{batch.batch}, {batch.n_q_heads}, "
                              f"{cfg.head_dim}] tensor on {pool.device}")
    if scale is None:
        scale = 1.0 / math.sqrt(cfg.head_dim)
    t = batch.csr
    # a pool writer launched just before may still be storing what this launch prefetches
    flags = _lib.DECODE_POOL_WRITTEN if pool._written is True or pool._written == layer else 0
    if gather is not None:
        if append is not None:
            raise ValidationError("the fused head gather does not take a fused append (append first)")
        gather.check(batch.batch, batch.n_q_heads, cfg.head_dim, pool.device)
        ptrs = (ctypes.c_void_p * len(gather.ptrs))(*gather.ptrs)
        _lib.check(lib.kvmix_flash_decode_gather(
            q.data_ptr(), _lib.dtype_code(q), ctypes.cast(ptrs, ctypes.c_void_p), len(gather.ptrs), gather.out_heads,
            gather.head0, _lib.dtype_code_of(gather.dtype), pool.int2_pool.data_ptr(), pool.int4_pool.data_ptr(), pool.n_pages,
            pool.n_int4, layer, cfg.n_kv_heads, cfg.head_dim, batch.n_q_heads, batch.batch,
            t["page_indptr"].data_ptr(), t["page_ids"].data_ptr(), t["int4_indptr"].data_ptr(),
            t["int4_ids"].data_ptr(), None, batch.work.data_ptr(), batch.cta_ptr.data_ptr(), batch.n_cta,
            batch.partials.data_ptr(), batch.counters.data_ptr(), float(scale), int(variant), pool.status.data_ptr(),
            flags, _lib.stream()))
        pool._written = False
        return None
    if append is not None:
        k_new, v_new = append
        want = (batch.batch, cfg.n_kv_heads, cfg.head_dim)
        if tuple(k_new.shape) != want or tuple(v_new.shape) != want:
            raise ValidationError(f"append k/v must be {want}")
        if variant != VARIANT_TENSOR_CORE:
            raise ValidationError("the fused decode append runs in the tensor-core kernel")
        if np.any(t["n_int4"] == 0):
            raise ValidationError("every request needs a reserved INT4 slot for the fused append")
        if batch.last_int4 is None:
            raise ValidationError("the fused append needs a DecodeBatch built from request_ids")
        # the newest INT4 entry of every table must be a slot reserved for this step and not
        # yet written at this layer (reserve_decode_slots, then batch.refresh())
        last = np.array([int(pool.table(r).slots[-1]) for r in batch.request_ids], dtype=np.int64)
        if not np.array_equal(last, batch.last_int4):
            raise ValidationError("page tables changed since batch.refresh(): refresh before the fused append")
        if np.any(pool._int4_written[layer, :, last - cfg.offset]):
            raise ValidationError("the newest slot is already written at this layer: reserve_decode_slots "
                                  "and batch.refresh() before the fused append")
        k_new = k_new.contiguous()
        v_new = v_new.to(k_new.dtype).contiguous()
        _lib.check(lib.kvmix_flash_decode_append(
            q.data_ptr(), _lib.dtype_code(q), out.data_ptr(), _lib.dtype_code(out), pool.int2_pool.data_ptr(),
            pool.int4_pool.data_ptr(), pool.n_pages, pool.n_int4, layer, cfg.n_kv_heads, cfg.head_dim,
            batch.n_q_heads, batch.batch, t["page_indptr"].data_ptr(), t["page_ids"].data_ptr(),
            t["int4_indptr"].data_ptr(), t["int4_ids"].data_ptr(), None, batch.work.data_ptr(), batch.cta_ptr.data_ptr(),
            batch.n_cta, batch.partials.data_ptr(), batch.counters.data_ptr(), float(scale), k_new.data_ptr(),
            v_new.data_ptr(), _lib.dtype_code(k_new), pool.status.data_ptr(), flags, _lib.stream()))
        pool._int4_written[layer, :, batch.last_int4 - cfg.offset] = True
        pool._written = layer  # the fused append stored this layer's new token
        return out
    _lib.check(lib.kvmix_flash_decode(
        q.data_ptr(), _lib.dtype_code(q), out.data_ptr(), _lib.dtype_code(out), pool.int2_pool.data_ptr(),
        pool.int4_pool.data_ptr(), pool.n_pages, pool.n_int4, layer, cfg.n_kv_heads, cfg.head_dim,
        batch.n_q_heads, batch.batch, t["page_indptr"].data_ptr(), t["page_ids"].data_ptr(),
        t["int4_indptr"].data_ptr(), t["int4_ids"].data_ptr(), None, batch.work.data_ptr(), batch.cta_ptr.data_ptr(),
        batch.n_cta, batch.partials.data_ptr(), batch.counters.data_ptr(), float(scale), int(variant),
        pool.status.data_ptr(), flags, _lib.stream()))
    pool._written = False
    return out


def flash_decode_layers_from_host(q_host: torch.Tensor, batch: DecodeBatch, out_host: torch.Tensor,
                                  chunk: int = 8, scale: float | None = None) -> torch.Tensor:
    """One decode step for all layers with q and the outputs on the HOST.

    q_host, out_host: pinned [L, B, n_q_heads, d].  The layers run in chunks: the
    host->device copy of chunk c+1 and the device->host copy of chunk c-1 overlap the
    kernels of chunk c (two side copy streams, events between the streams).  Asynchronous
    on the current stream: it returns once everything is enqueued and the current
    stream is ordered after the last device->host copy.
    """
    pool, cfg = batch.pool, batch.pool.config
    L = q_host.shape[0]
    if tuple(q_host.shape[1:]) != (batch.batch, batch.n_q_heads, cfg.head_dim) or L > cfg.n_layers:
        raise ValidationError(f"q_host must be [L <= {cfg.n_layers}, {batch.batch}, {batch.n_q_heads}, {cfg.head_dim}]")
    if out_host.shape != q_host.shape:
        raise ValidationError("out_host must match q_host")
    dev = pool.device
    st = getattr(batch, "_host_io", None)
    if st is None or st["q"].shape != q_host.shape or st["q"].dtype != q_host.dtype:
        st = {"q": torch.empty(q_host.shape, dtype=q_host.dtype, device=dev),
              "o": torch.empty(out_host.shape, dtype=out_host.dtype, device=dev),
              "h2d": torch.cuda.Stream(device=dev), "d2h": torch.cuda.Stream(device=dev)}
        batch._host_io = st
    qd, od, hs, ds = st["q"], st["o"], st["h2d"], st["d2h"]
    compute = torch.cuda.current_stream(dev)
    hs.wait_stream(compute)  # the previous step's kernels are done with qd / od
    ds.wait_stream(compute)
    chunks = [(c0, min(L, c0 + chunk)) for c0 in range(0, L, chunk)]
    ev_in = []
    with torch.cuda.stream(hs):  # every input chunk streams in up front, in order
        for c0, c1 in chunks:
            qd[c0:c1].copy_(q_host[c0:c1], non_blocking=True)
            ev_in.append(torch.cuda.Event())
            ev_in[-1].record(hs)
    for (c0, c1), ev in zip(chunks, ev_in):
        compute.wait_event(ev)
        for layer in range(c0, c1):
            flash_decode_batched(qd[layer], batch, layer, out=od[layer], scale=scale)
        ev_out = torch.cuda.Event()
        ev_out.record(compute)
        ds.wait_event(ev_out)
        with torch.cuda.stream(ds):  # a chunk's outputs leave while the next chunk computes
            out_host[c0:c1].copy_(od[c0:c1], non_blocking=True)
    compute.wait_stream(hs)
    cs = ds
    compute.wait_stream(cs)
    return out_host


def flash_decode(q, page_table, pool_view, split_len: int = 128, scale=None, variant: int | None = None):
    """attention.py:175-218 drop-in: single-query decode over a partitioned page table.

    ``split_len`` is validated like the reference but the device kernel chooses its own
    bitwidth-homogeneous split (a page or 32 INT4 slots per tile); results are
    split-invariant up to float rounding, as the reference's are.

    Precision follows the caller's dtype (``variant=None``): an fp32/fp64 q -- the
    reference's own arithmetic -- runs the fp32-faithful CUDA-core kernel (fp32 dequant,
    dot products and softmax; within the reference's own 1e-5 relative bar of its tests,
    pkg/tests/test_attention.py:205-246); a bf16/f16 q runs the tensor-core hot path
    (within the north_star's atol 2e-3 / rtol 1e-2), as ``flash_decode_batched`` does.
    """
    is_torch = isinstance(q, torch.Tensor)
    qn = q if is_torch else np.asarray(q, dtype=np.float32)
    if qn.ndim != 2:
        raise ValidationError("q must be [n_heads, d]")
    n_heads, d = qn.shape
    slots = page_table.slots if isinstance(page_table, PageTable) else \
        np.asarray([a.index for a in page_table.entries], dtype=np.int64)
    if slots.size == 0:
        raise ValidationError("empty page table")
    if split_len < 1:
        raise ValidationError("split_len must be >= 1")
    pool = pool_view.pool
    cfg = pool.config
    is2 = slots < cfg.offset
    if np.any(is2[int(is2.sum()):]):
        raise ValidationError("page table not partitioned: INT4 address precedes INT2")
    n_kv = cfg.n_kv_heads
    if n_heads % n_kv != 0:
        raise ValidationError("n_heads not a multiple of the pool's n_kv_heads")
    if d != cfg.head_dim:
        raise ValidationError("q head dim does not match the pool")
    in_range = (slots >= 0) & (slots < cfg.total_slots)
    if not np.all(in_range) or np.any(pool._owner[slots] < 0):
        raise ValidationError("dangling slot address")
    pool._require_written(slots, pool_view.layer)
    batch = DecodeBatch(pool, n_q_heads=n_heads, tables=[slots])
    qd = (q if is_torch else torch.as_tensor(qn)).to(pool.device, torch.float32).reshape(1, n_heads, d)
    if variant is None:
        wide = (q.dtype in (torch.float32, torch.float64)) if is_torch else True  # numpy q is fp32 (above)
        variant = VARIANT_SIMPLE if wide else VARIANT_TENSOR_CORE
    qd = qd if variant == VARIANT_SIMPLE or not is_torch else q.to(pool.device).reshape(1, n_heads, d)
    out = flash_decode_batched(qd, batch, pool_view.layer, out=torch.empty(qd.shape, dtype=torch.float32,
                                                                             device=pool.device),
                               scale=scale, variant=variant)
    res = out[0]
    return res if is_torch else res.cpu().numpy()
