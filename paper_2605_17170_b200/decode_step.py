"""One decode step of a request batch, end to end, with the page tables kept on the device.

A decode step of the paper's serving loop appends one token to every
request at every layer and attends over the grown cache.  In the reference that is
``append_decode_token`` (pool.py:284-306: pop one INT4 slot LIFO, quantize k/v [L, Hkv, d]
at INT4, append the slot to the partitioned table) followed by one ``flash_decode`` per
(request, layer) (attention.py:175-218).

``DecodeStep`` runs it as one CUDA graph per step:

* host: ``pool.reserve_decode_slots`` pops the slots exactly as the reference does (O(batch)
  work; the slot values go to a pinned buffer);
* device, in stream order: the slots are copied in, K7 (``kvmix_decode_tables``) appends them
  to the padded per-request INT4 lists and rebuilds the stream-K plan; q, k_new, v_new
  stream in from pinned host memory in layer chunks on a side stream; per layer one fused
  append + decode launch (K4 in K2) stores the new token and attends to it; the outputs
  stream back per chunk.

The host never rebuilds a table or a plan during decoding (the round-1 path spent ~5 ms of
host work per step on ``split_partitioned`` / ``plan_stream`` / uploads); its per-step work is
the slot pops and one graph launch.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import CapacityError, ValidationError
from .plan import NUM_SMS_B200
from .pool import MixedPrecisionPool, split_partitioned

CTAS_PER_SM = 3


def layer_chunks(L: int, layer_chunk=None) -> list:
    """[(c0, c1)] layer ranges whose uploads / downloads overlap the other ranges' kernels.
    layer_chunk: an int (uniform ranges; 8 measured best at cfg2), a list of range sizes, or
    None: ranges of 8 with a short first and last range (2, 6, 8, ..., 6, 2) -- measured equal
    to uniform 8 at cfg2 (1899 vs 1899 tokens/s)."""
    if layer_chunk is None:
        if L < 24:
            sizes = [min(8, L)] * (-(-L // 8))
        else:
            mid = L - 16
            sizes = [2, 6] + [8] * (mid // 8) + ([mid % 8] if mid % 8 else []) + [6, 2]
    elif isinstance(layer_chunk, int):
        if layer_chunk <= 0:
            raise ValidationError("layer_chunk must be positive")
        sizes = [layer_chunk] * (-(-L // layer_chunk))
    else:
        sizes = [int(x) for x in layer_chunk]
        if any(x <= 0 for x in sizes) or sum(sizes) < L:
            raise ValidationError("layer chunk sizes must be positive and cover every layer")
    out, c = [], 0
    for n in sizes:
        if c >= L:
            break
        out.append((c, min(L, c + n)))
        c += n
    return out


class DecodeStep:
    """Graph-captured decode steps (append + attention, all layers) for a fixed request batch.

    Fill ``q_host`` [L, B, Hq, d], ``k_host`` / ``v_host`` [L, B, Hkv, d] (pinned, ``dtype``),
    call ``run()``, and after the current stream synchronizes read ``out_host`` [L, B, Hq, d].
    ``max_new_tokens`` bounds the steps (the device INT4 lists are padded to it).
    """

    def __init__(self, pool: MixedPrecisionPool, request_ids, n_q_heads: int, dtype=torch.bfloat16,
                 max_new_tokens: int = 256, n_cta: int | None = None, int4_weight: float = 0.8,
                 layer_chunk=8, scale: float | None = None, fused_append: bool = False):
        cfg = pool.config
        if dtype not in (torch.float32, torch.bfloat16, torch.float16):
            raise ValidationError(f"unsupported dtype {dtype}")
        self.pool, self.rids = pool, list(request_ids)
        self.B, self.L, self.H, self.d = len(self.rids), cfg.n_layers, cfg.n_kv_heads, cfg.head_dim
        self.Hq = int(n_q_heads)
        if self.B == 0:
            raise ValidationError("empty request batch")
        if self.Hq % self.H or self.Hq // self.H > 8:
            raise ValidationError("n_q_heads must be a multiple (<= 8x) of the pool's n_kv_heads")
        dev = pool.device
        self.device = dev
        pages, int4 = [], []
        for rid in self.rids:
            t = pool.table(rid)
            if not t.partitioned:
                raise ValidationError(f"request {rid!r} is not partitioned")
            p, i4 = split_partitioned(t.slots, cfg.offset, cfg.page_size)
            pages.append(p)
            int4.append(i4)
        n4 = np.array([x.size for x in int4], dtype=np.int64)
        self.cap = int(-(-(int(n4.max()) + max_new_tokens) // 32) * 32)
        self.n4 = n4.copy()  # host mirror of the device counts
        pad = np.zeros((self.B, self.cap), dtype=np.int32)
        for b, x in enumerate(int4):
            pad[b, : x.size] = x
        npg = np.array([p.size for p in pages], dtype=np.int32)
        indptr = np.concatenate([[0], np.cumsum(npg)]).astype(np.int32)
        i32 = dict(dtype=torch.int32, device=dev)
        self.page_indptr = torch.as_tensor(indptr, device=dev)
        self.page_ids = torch.as_tensor(np.concatenate(pages).astype(np.int32) if npg.sum() else np.zeros(1, np.int32),
                                        device=dev)
        self.n_pages = torch.as_tensor(npg, device=dev)
        self.int4_indptr = torch.arange(0, (self.B + 1) * self.cap, self.cap, **i32)
        self.int4_ids = torch.as_tensor(pad.reshape(-1), device=dev)
        self.int4_count = torch.as_tensor(n4.astype(np.int32), device=dev)
        if n_cta is None:
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else NUM_SMS_B200
            n_cta = n_sm * CTAS_PER_SM
        self.n_cta = int(n_cta)
        self.int4_weight = float(int4_weight)
        units = self.B * self.H
        self.work = torch.zeros((self.n_cta + units) * 8, **i32)
        self.cta_ptr = torch.zeros(self.n_cta + 1, **i32)
        self.n_parts = torch.zeros(1, **i32)
        self.scratch = torch.zeros(2 * units, **i32)
        self.err = torch.zeros(1, **i32)
        self.partials = torch.empty((self.n_cta + units) * 8 * (self.d + 4), dtype=torch.float32, device=dev)
        self.counters = torch.zeros(units, **i32)
        self.scale = 1.0 / math.sqrt(self.d) if scale is None else float(scale)
        self.dtype = dtype
        # fused_append: each layer's decode launch quantizes that layer's new token (K4 inside K2).
        # Default: one batched append launch per layer chunk before its decode launches -- the fused
        # form measured 9% slower per launch (ncu: 161 vs 147 us at cfg2).
        self.fused_append = bool(fused_append)
        L, B = self.L, self.B
        self.q_dev = torch.zeros((L, B, self.Hq, self.d), dtype=dtype, device=dev)
        self.out_dev = torch.zeros_like(self.q_dev)
        self.k_dev = torch.zeros((L, B, self.H, self.d), dtype=dtype, device=dev)
        self.v_dev = torch.zeros_like(self.k_dev)
        self.q_host = torch.zeros(self.q_dev.shape, dtype=dtype).pin_memory()
        self.out_host = torch.zeros(self.q_dev.shape, dtype=dtype).pin_memory()
        self.k_host = torch.zeros(self.k_dev.shape, dtype=dtype).pin_memory()
        self.v_host = torch.zeros(self.k_dev.shape, dtype=dtype).pin_memory()
        self.slots_host = torch.zeros(B, dtype=torch.int32).pin_memory()
        self.slots_dev = torch.zeros(B, **i32)
        self.chunks = layer_chunks(L, layer_chunk)
        self.graph = None
        self.steps = 0
        self._tables(None)  # the initial plan (no append)
        torch.cuda.current_stream(dev).synchronize()
        if int(self.err.item()):
            raise ValidationError("decode_tables rejected the batch (empty request?)")

    # -- device work ----------------------------------------------------------------------
    def _tables(self, new_slots) -> None:
        _lib.check(lib.kvmix_decode_tables(
            _lib.ptr(new_slots), self.B, self.H, self.n_pages.data_ptr(), self.int4_count.data_ptr(),
            self.int4_ids.data_ptr(), self.cap, self.d, self.int4_weight, self.n_cta, self.work.data_ptr(),
            self.cta_ptr.data_ptr(), self.n_parts.data_ptr(), self.scratch.data_ptr(), self.err.data_ptr(),
            _lib.stream()))

    def _append(self, c0: int, c1: int) -> None:
        """K4 data half for layers [c0, c1): every request's new k/v into its new INT4 slot."""
        p, cfg = self.pool, self.pool.config
        _lib.check(lib.kvmix_append_int4_strided(
            self.k_dev[c0].data_ptr(), self.v_dev[c0].data_ptr(), _lib.dtype_code(self.k_dev), self.B, c1 - c0, c0,
            self.L, self.H, self.d, self.B * self.H * self.d, self.H * self.d, self.slots_dev.data_ptr(),
            p.int4_pool.data_ptr(), p.n_int4, p.status.data_ptr(), _lib.stream()))

    def _decode(self, layer: int, flags: int) -> None:
        p, cfg = self.pool, self.pool.config
        if not self.fused_append:
            _lib.check(lib.kvmix_flash_decode(
                self.q_dev[layer].data_ptr(), _lib.dtype_code(self.q_dev), self.out_dev[layer].data_ptr(),
                _lib.dtype_code(self.out_dev), p.int2_pool.data_ptr(), p.int4_pool.data_ptr(), p.n_pages, p.n_int4,
                layer, self.H, self.d, self.Hq, self.B, self.page_indptr.data_ptr(), self.page_ids.data_ptr(),
                self.int4_indptr.data_ptr(), self.int4_ids.data_ptr(), self.int4_count.data_ptr(),
                self.work.data_ptr(), self.cta_ptr.data_ptr(), self.n_cta, self.partials.data_ptr(),
                self.counters.data_ptr(), self.scale, 0, p.status.data_ptr(), flags, _lib.stream()))
            return
        _lib.check(lib.kvmix_flash_decode_append(
            self.q_dev[layer].data_ptr(), _lib.dtype_code(self.q_dev), self.out_dev[layer].data_ptr(),
            _lib.dtype_code(self.out_dev), p.int2_pool.data_ptr(), p.int4_pool.data_ptr(), p.n_pages, p.n_int4, layer,
            self.H, self.d, self.Hq, self.B, self.page_indptr.data_ptr(), self.page_ids.data_ptr(),
            self.int4_indptr.data_ptr(), self.int4_ids.data_ptr(), self.int4_count.data_ptr(), self.work.data_ptr(),
            self.cta_ptr.data_ptr(), self.n_cta, self.partials.data_ptr(), self.counters.data_ptr(), self.scale,
            self.k_dev[layer].data_ptr(), self.v_dev[layer].data_ptr(), _lib.dtype_code(self.k_dev),
            p.status.data_ptr(), flags, _lib.stream()))

    def _enqueue(self) -> None:
        """The step on the current stream: slots, K7, chunked H2D / fused decode / D2H."""
        main = torch.cuda.current_stream(self.device)
        h2d, d2h = self._side
        h2d.wait_stream(main)
        d2h.wait_stream(main)
        ev_in = []
        with torch.cuda.stream(h2d):
            self.slots_dev.copy_(self.slots_host, non_blocking=True)
            ev_in.append(torch.cuda.Event())
            ev_in[-1].record(h2d)
            for c0, c1 in self.chunks:
                self.q_dev[c0:c1].copy_(self.q_host[c0:c1], non_blocking=True)
                self.k_dev[c0:c1].copy_(self.k_host[c0:c1], non_blocking=True)
                self.v_dev[c0:c1].copy_(self.v_host[c0:c1], non_blocking=True)
                ev_in.append(torch.cuda.Event())
                ev_in[-1].record(h2d)
        main.wait_event(ev_in[0])
        self._tables(self.slots_dev)
        for (c0, c1), ev in zip(self.chunks, ev_in[1:]):
            main.wait_event(ev)
            if not self.fused_append:
                # an ordinary launch: the next decode launch (programmatic) starts only after it
                self._append(c0, c1)
            for layer in range(c0, c1):
                # the first launch reads the tables K7 just wrote: no early (PDL) reads
                self._decode(layer, _lib.DECODE_POOL_WRITTEN if layer == 0 else 0)
            ev_out = torch.cuda.Event()
            ev_out.record(main)
            d2h.wait_event(ev_out)
            with torch.cuda.stream(d2h):
                self.out_host[c0:c1].copy_(self.out_dev[c0:c1], non_blocking=True)
        main.wait_stream(h2d)
        main.wait_stream(d2h)

    # -- public ---------------------------------------------------------------------------------
    def run(self, graph: bool = True) -> np.ndarray:
        """One decode step: pops one INT4 slot per request (host, reference LIFO order), then
        appends this step's k/v and attends, all layers, on the current stream (asynchronous).
        Returns the popped slots."""
        if np.any(self.n4 >= self.cap):
            raise CapacityError("DecodeStep: max_new_tokens reached; build a new DecodeStep", region="int4")
        pool, cfg = self.pool, self.pool.config
        slots = pool.reserve_decode_slots(self.rids)
        self.slots_host.copy_(torch.from_numpy((slots - cfg.offset).astype(np.int32)))
        if not hasattr(self, "_side"):
            self._side = (torch.cuda.Stream(device=self.device), torch.cuda.Stream(device=self.device))
        if graph:
            if self.graph is None:
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream(device=self.device)
                cap.wait_stream(torch.cuda.current_stream(self.device))
                with torch.cuda.stream(cap):
                    with torch.cuda.graph(g, stream=cap):
                        self._enqueue()
                torch.cuda.current_stream(self.device).wait_stream(cap)
                self.graph = g
            self.graph.replay()
        else:
            self._enqueue()
        self.n4 += 1
        self.steps += 1
        pool._int4_written[:, :, slots - cfg.offset] = True
        pool._written = self.L - 1  # the last launch stored layer L-1's new token
        return slots

    def check(self) -> None:
        """Raise if the device tables reported an error (synchronizes)."""
        torch.cuda.current_stream(self.device).synchronize()
        e = int(self.err.item())
        if e & 4:
            raise CapacityError("device INT4 list full", region="int4")
        if e:
            raise ValidationError(f"decode_tables error {e}")

    def plan(self) -> tuple[np.ndarray, np.ndarray, int]:
        """(work [n_pieces, 8], cta_ptr, n_parts) of the current device plan (synchronizes)."""
        torch.cuda.current_stream(self.device).synchronize()
        cta_ptr = self.cta_ptr.cpu().numpy()
        work = self.work[: 8 * int(cta_ptr[-1])].view(-1, 8).cpu().numpy()
        return work, cta_ptr, int(self.n_parts.item())

    def kv_bytes(self) -> int:
        """Algorithmic KV bytes one layer's decode reads at the current lengths (all kv heads)."""
        from .quant import key_page_payload_bytes, token_block_payload_bytes
        d = self.d
        per_page = key_page_payload_bytes(d) + 32 * token_block_payload_bytes(d, 2)
        per_int4 = 2 * token_block_payload_bytes(d, 4)
        npg = int(self.n_pages.sum().item())
        return int(self.H * (npg * per_page + int(self.n4.sum()) * per_int4))
