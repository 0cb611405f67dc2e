"""Dual-precision paged KV store: host control plane + device (HBM) data plane.

Drop-in for /root/reference/pkg/src/kvmix/pool.py.  The control plane (address
space, LIFO allocators, page tables, partition) reproduces the reference's slot
indices bit-exactly (pool.py:63-197, 284-306) with vectorised numpy; the data plane
keeps every block in two device byte pools written and read only by sm_100a
kernels (include/kvmix_b200.h):

  int2_pool [L][Hkv][n_pages][page_stride] : KeyPageBlock || 32 INT2 V TokenBlocks
  int4_pool [L][Hkv][n_int4][slot_stride]  : INT4 K TokenBlock || INT4 V TokenBlock

Each block is the reference payload byte-for-byte, at a fixed address computed from
(layer, head, slot) -- no dicts, no per-block allocation (the reference keeps
``bytes`` objects in dicts keyed (slot|page, layer, head), pool.py:108-110).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import CapacityError, KvmixError, ValidationError
from .quant import GROUP_SIZE, key_page_payload_bytes, token_block_payload_bytes

SUPPORTED_HEAD_DIMS = (32, 64, 128, 256)


@dataclass(frozen=True)
class SlotAddress:
    index: int


class PageTable:
    """Per-request ordered slot list; one address per cached token (pool.py:36-41).

    Backed by a numpy int64 array (``slots``); ``entries`` materialises the
    reference's list of SlotAddress on demand.
    """

    def __init__(self, request_id: str, slots=None, partitioned: bool = False):
        self.request_id = request_id
        self.slots = slots if slots is not None else []
        self.partitioned = partitioned
        self._entries_cache = None
        # (page_tokens, page_ids, int4_tokens, int4_ids) device tensors left by alloc_device
        # (K6) for write_prefill; dropped whenever the slots change
        self._dev_index = None

    @property
    def slots(self) -> np.ndarray:
        return self._buf[: self._n]

    @slots.setter
    def slots(self, value) -> None:
        self._buf = np.array(value, dtype=np.int64)
        self._n = int(self._buf.size)
        self._entries_cache = None

    def _append(self, slot: int) -> None:
        """Amortised O(1) append of a decode slot (pool.py:305 entries.append)."""
        if self._n == self._buf.size:
            grown = np.empty(max(64, 2 * self._n), dtype=np.int64)
            grown[: self._n] = self._buf[: self._n]
            self._buf = grown
        self._buf[self._n] = slot
        self._n += 1
        self._entries_cache = None
        self._dev_index = None

    @property
    def entries(self) -> list[SlotAddress]:
        if self._entries_cache is None or len(self._entries_cache) != self.slots.size:
            self._entries_cache = [SlotAddress(int(s)) for s in self.slots]
        return self._entries_cache

    @entries.setter
    def entries(self, value) -> None:
        self.slots = [a.index for a in value]

    def _set_slots(self, slots) -> None:
        self.slots = slots
        self._dev_index = None

    def __len__(self) -> int:
        return int(self.slots.size)

    def __repr__(self) -> str:
        return f"PageTable({self.request_id!r}, n={self.slots.size}, partitioned={self.partitioned})"


@dataclass(frozen=True)
class PoolConfig:
    total_slots: int
    offset: int  # slots below are INT2, at/above are INT4
    n_layers: int
    n_kv_heads: int
    head_dim: int
    page_size: int = GROUP_SIZE

    def __post_init__(self):  # pool.py:54-60
        if not 0 <= self.offset <= self.total_slots:
            raise ValidationError("offset must lie within [0, total_slots]")
        if self.offset % self.page_size != 0:
            raise ValidationError("INT2 region must be whole pages")
        if self.head_dim % self.page_size != 0:
            raise ValidationError("head_dim must be divisible by the page size")


def init_pool(avg_bitwidth: float, total_slots: int, n_layers: int, n_kv_heads: int, head_dim: int,
              page_size: int = GROUP_SIZE) -> PoolConfig:
    """pool.py:63-93: INT2 fraction (4 - B)/2 of the slots, floored to a whole page."""
    if not 2.0 <= avg_bitwidth <= 4.0:
        raise ValidationError(f"average bitwidth {avg_bitwidth} outside [2, 4]")
    if total_slots < 2 * page_size:
        raise ValidationError("pool needs at least two pages of slots")
    int2_fraction = (4.0 - avg_bitwidth) / 2.0
    ideal = int2_fraction * total_slots + 1e-6  # keeps 0.65 * 3200 = 2080 exact
    offset = int(ideal) // page_size * page_size
    return PoolConfig(total_slots=total_slots, offset=offset, n_layers=n_layers, n_kv_heads=n_kv_heads,
                      head_dim=head_dim, page_size=page_size)


class MixedPrecisionPool:
    """Paged KV store with independent INT2-page and INT4-slot allocators (pool.py:96-377)."""

    def __init__(self, config: PoolConfig, device=None, materialize: bool = True):
        if config.page_size != GROUP_SIZE:
            raise ValidationError(f"device pool supports page_size {GROUP_SIZE} only")
        if config.head_dim not in SUPPORTED_HEAD_DIMS:
            raise ValidationError(f"device pool supports head_dim in {SUPPORTED_HEAD_DIMS}")
        self.config = config
        g = config.page_size
        self.n_pages = config.offset // g
        self.n_int4 = config.total_slots - config.offset
        # LIFO stacks whose top (end) is the lowest address (pool.py:104-105)
        self._free_pages = list(range((self.n_pages - 1) * g, -g, -g)) if self.n_pages else []
        self._free_int4 = list(range(config.total_slots - 1, config.offset - 1, -1))
        self._tables: dict[str, PageTable] = {}
        self._rid_index: dict[str, int] = {}
        self._next_rid = 0
        self._owner = np.full(config.total_slots, -1, dtype=np.int64)  # slot -> request index
        # written-state bookkeeping (read-before-write checks, parameter accounting)
        L, H = config.n_layers, config.n_kv_heads
        self._page_written = np.zeros((L, H, self.n_pages), dtype=bool)
        self._int4_written = np.zeros((L, H, self.n_int4), dtype=bool)
        self.page_stride = _lib.page_stride(config.head_dim)
        self.slot_stride = _lib.slot_stride(config.head_dim)
        self.device = torch.device(device) if device is not None else None
        self.int2_pool = None
        self.int4_pool = None
        if materialize:
            self.device = self.device or _lib.require_cuda()
            self.int2_pool = torch.zeros(max(1, L * H * self.n_pages * self.page_stride), dtype=torch.uint8,
                                         device=self.device)
            self.int4_pool = torch.zeros(max(1, L * H * self.n_int4 * self.slot_stride), dtype=torch.uint8,
                                         device=self.device)
            # pool status words (kvmix_b200.h KVMIX_POOL_STATUS_*): error bits, largest stored
            # key-page / V scales (the decode kernel's fp16 operand bounds)
            self.status = torch.zeros(_lib.POOL_STATUS_WORDS, dtype=torch.int32, device=self.device)
        # the last pool kernel launched was a writer (True: all layers; int: that layer only):
        # a decode of those layers must not prefetch KV ahead of it (programmatic dependent
        # launch); False once a decode has run after it
        self._written = False

    # -- address helpers -------------------------------------------------------------
    def is_int2(self, address: SlotAddress) -> bool:
        return address.index < self.config.offset

    def _page_start(self, index: int) -> int:
        return index // self.config.page_size * self.config.page_size

    def device_bytes(self) -> int:
        return int(self.int2_pool.numel() + self.int4_pool.numel()) if self.int2_pool is not None else 0

    # -- allocation ------------------------------------------------------------------
    def alloc(self, request_id: str, per_token_bitwidths) -> PageTable:
        """pool.py:122-163.  The p-th run of 32 INT2 tokens (token order) takes the p-th
        popped page; residual INT2 tokens and INT4 tokens (sorted) take INT4 pops."""
        if request_id in self._tables:
            raise ValidationError(f"request {request_id!r} already live")
        bits = np.asarray(per_token_bitwidths)
        if not np.all(np.isin(bits, (2, 4))):
            raise ValidationError("per-token bitwidths must be 2 or 4")
        g = self.config.page_size
        idx2 = np.flatnonzero(bits == 2)
        n_pages = idx2.size // g
        paged = idx2[: n_pages * g]
        int4_tokens = np.sort(np.concatenate([np.flatnonzero(bits == 4), idx2[n_pages * g:]]))
        if n_pages > len(self._free_pages):
            raise CapacityError(f"INT2 region exhausted: need {n_pages} pages, {len(self._free_pages)} free",
                                region="int2")
        if int4_tokens.size > len(self._free_int4):
            raise CapacityError(f"INT4 region exhausted: need {int4_tokens.size} slots, "
                                f"{len(self._free_int4)} free", region="int4")
        slots = np.empty(bits.size, dtype=np.int64)
        if n_pages:
            starts = np.asarray(self._free_pages[-n_pages:][::-1], dtype=np.int64)  # pop order
            del self._free_pages[-n_pages:]
            slots[paged] = (starts[:, None] + np.arange(g)).reshape(-1)
        m = int4_tokens.size
        if m:
            pops = np.asarray(self._free_int4[-m:][::-1], dtype=np.int64)
            del self._free_int4[-m:]
            slots[int4_tokens] = pops
        rix = self._next_rid
        self._next_rid += 1
        self._rid_index[request_id] = rix
        self._owner[slots] = rix
        table = PageTable(request_id=request_id, slots=slots)
        self._tables[request_id] = table
        return table

    def alloc_device(self, request_id: str, per_token_bitwidths) -> PageTable:
        """alloc (pool.py:122-163) with the O(N) token routing on the GPU (K6): the bits are
        counted on the device, the host pops its LIFO stacks exactly as alloc does, and
        kvmix_route_tokens writes the table and the K1 index lists.  The resulting slots are
        identical to alloc's; the index lists stay on the device for write_prefill."""
        if request_id in self._tables:
            raise ValidationError(f"request {request_id!r} already live")
        dev = self.device
        bits = torch.as_tensor(np.asarray(per_token_bitwidths) if not torch.is_tensor(per_token_bitwidths)
                               else per_token_bitwidths, device=dev).reshape(-1)
        if bits.dtype != torch.int8:  # values must survive the int8 narrowing (the kernel checks 2 / 4)
            if not bool(((bits == 2) | (bits == 4)).all()):
                raise ValidationError("per-token bitwidths must be 2 or 4")
            bits = bits.to(torch.int8)
        bits = bits.contiguous()
        n = int(bits.numel())
        g = self.config.page_size
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        counts = torch.empty(int(lib.kvmix_route_scratch_elems(n)), dtype=torch.int64, device=dev)
        _lib.check(lib.kvmix_count_int2(bits.data_ptr(), n, counts.data_ptr(), err.data_ptr(), _lib.stream()))
        n2 = int(counts[0].item())
        if int(err.item()) & 2:
            raise ValidationError("per-token bitwidths must be 2 or 4")
        n_pages = n2 // g
        m = n - n_pages * g
        if n_pages > len(self._free_pages):
            raise CapacityError(f"INT2 region exhausted: need {n_pages} pages, {len(self._free_pages)} free",
                                region="int2")
        if m > len(self._free_int4):
            raise CapacityError(f"INT4 region exhausted: need {m} slots, {len(self._free_int4)} free", region="int4")
        starts = np.asarray(self._free_pages[-n_pages:][::-1] if n_pages else [], dtype=np.int64)
        pops = np.asarray(self._free_int4[-m:][::-1] if m else [], dtype=np.int64)
        if n_pages:
            del self._free_pages[-n_pages:]
        if m:
            del self._free_int4[-m:]
        st = torch.as_tensor(starts, device=dev)
        po = torch.as_tensor(pops, device=dev)
        slots = torch.empty(n, dtype=torch.int64, device=dev)
        pt = torch.empty((n_pages, g), dtype=torch.int32, device=dev)
        pi = torch.empty(n_pages, dtype=torch.int32, device=dev)
        it = torch.empty(m, dtype=torch.int32, device=dev)
        ii = torch.empty(m, dtype=torch.int32, device=dev)
        _lib.check(lib.kvmix_route_tokens(
            bits.data_ptr(), n, g, counts.data_ptr(), st.data_ptr(), n_pages, po.data_ptr(), m, self.config.offset,
            slots.data_ptr(), pt.data_ptr(), pi.data_ptr(), it.data_ptr(), ii.data_ptr(), err.data_ptr(),
            _lib.stream()))
        host = slots.cpu().numpy()
        if int(err.item()):
            raise KvmixError("device routing disagreed with the host counts")
        rix = self._next_rid
        self._next_rid += 1
        self._rid_index[request_id] = rix
        self._owner[host] = rix
        table = PageTable(request_id=request_id, slots=host)
        table._dev_index = (pt, pi, it, ii)
        self._tables[request_id] = table
        return table

    def free(self, request_id: str) -> None:
        """pool.py:165-188: INT4 slots pushed in entry order, pages in descending start order."""
        table = self._tables.pop(request_id, None)
        if table is None:
            raise ValidationError(f"unknown or already-freed request {request_id!r}")
        self._rid_index.pop(request_id)
        cfg = self.config
        s = table.slots
        self._owner[s] = -1
        is2 = s < cfg.offset
        s4 = s[~is2]
        self._free_int4.extend(int(x) for x in s4)
        self._int4_written[:, :, s4 - cfg.offset] = False
        starts = np.unique(s[is2] // cfg.page_size * cfg.page_size)[::-1]
        self._free_pages.extend(int(x) for x in starts)
        self._page_written[:, :, starts // cfg.page_size] = False

    def partition(self, table: PageTable) -> PageTable:
        """pool.py:190-197: stable, INT2 first, idempotent."""
        if not table.partitioned:
            s = table.slots
            is2 = s < self.config.offset
            table._set_slots(np.concatenate([s[is2], s[~is2]]))
            table.partitioned = True
        return table

    # -- data plane ---------------------------------------------------------------------
    def _plane_offsets(self, layer: int, head: int) -> tuple[int, int]:
        cfg = self.config
        lh = layer * cfg.n_kv_heads + head
        return lh * self.n_pages * self.page_stride, lh * self.n_int4 * self.slot_stride

    def _to_dev(self, x) -> torch.Tensor:
        if isinstance(x, torch.Tensor):
            if x.dtype not in (torch.float32, torch.bfloat16, torch.float16):
                x = x.float()
            return x.to(self.device).contiguous()
        return torch.as_tensor(np.asarray(x, dtype=np.float32), device=self.device).contiguous()

    def _check_err(self, what: str) -> None:
        err = self.status[_lib.POOL_STATUS_ERR]
        if int(err.item()) & 1:
            err.zero_()
            raise ValidationError(f"{what} must be finite")

    def operand_bounds(self) -> tuple[float, float]:
        """(largest INT2 key-page scale, largest V scale) written so far (pool status words)."""
        w = self.status.cpu().numpy().view(np.float32)
        return float(w[_lib.POOL_STATUS_KSCALE]), float(w[_lib.POOL_STATUS_VSCALE])

    def write_page(self, page_start: int, keys, values, layer: int, head: int) -> None:
        """pool.py:201-215: one full INT2 page (all G tokens) for one (layer, head)."""
        cfg, g = self.config, self.config.page_size
        if page_start >= cfg.offset or page_start % g != 0 or page_start < 0:
            raise ValidationError(f"{page_start} is not an INT2 page start")
        k = self._to_dev(keys)
        v = self._to_dev(values)
        if tuple(k.shape) != (g, cfg.head_dim) or tuple(v.shape) != tuple(k.shape):
            raise ValidationError(f"partial or misshaped INT2 page write: got {tuple(k.shape)}, "
                                  f"need ({g}, {cfg.head_dim})")
        if v.dtype != k.dtype:
            v = v.to(k.dtype)
        off2, _ = self._plane_offsets(layer, head)
        dev = self.device
        toks = torch.arange(g, dtype=torch.int32, device=dev)
        pid = torch.tensor([page_start // g], dtype=torch.int32, device=dev)
        _lib.check(lib.kvmix_write_prefill(
            k.data_ptr(), v.data_ptr(), _lib.dtype_code(k), 1, g, 1, cfg.head_dim, toks.data_ptr(),
            pid.data_ptr(), 1, None, None, 0, self.int2_pool.data_ptr() + off2, self.n_pages,
            self.int4_pool.data_ptr(), self.n_int4, self.status.data_ptr(), _lib.stream()))
        self._written = True
        self._check_err("keys/values")
        self._page_written[layer, head, page_start // g] = True

    def write_token(self, address: SlotAddress, k, v, layer: int, head: int) -> None:
        """pool.py:217-226: one INT4 token for one (layer, head)."""
        slot = address.index
        if slot < self.config.offset:
            raise ValidationError("INT2 slots are written page-at-a-time via write_page")
        kk = self._to_dev(k).reshape(1, 1, 1, -1)
        vv = self._to_dev(v).reshape(1, 1, 1, -1).to(kk.dtype)
        if kk.shape[-1] != self.config.head_dim:
            raise ValidationError("head dim mismatch")
        _, off4 = self._plane_offsets(layer, head)
        ids = torch.tensor([slot - self.config.offset], dtype=torch.int32, device=self.device)
        _lib.check(lib.kvmix_append_int4(kk.data_ptr(), vv.data_ptr(), _lib.dtype_code(kk), 1, 1, 0, 1, 1,
                                         self.config.head_dim, ids.data_ptr(), self.int4_pool.data_ptr() + off4,
                                         self.n_int4, self.status.data_ptr(), _lib.stream()))
        self._written = True
        self._check_err("values")
        self._int4_written[layer, head, slot - self.config.offset] = True

    def write_prefill(self, table: PageTable, keys, values, check_finite: bool = True) -> None:
        """pool.py:228-262: quantize+pack a whole request's prefill K/V [L, N, Hkv, d]
        (f32/bf16/f16, host or device) in one K1 launch pair."""
        if table.partitioned:
            raise ValidationError("write_prefill requires token-ordered entries")
        cfg, g = self.config, self.config.page_size
        k = self._to_dev(keys)
        v = self._to_dev(values)
        n = len(table)
        want = (cfg.n_layers, n, cfg.n_kv_heads, cfg.head_dim)
        if tuple(k.shape) != want or tuple(v.shape) != want:
            raise ValidationError(f"prefill K/V must be {want}, got {tuple(k.shape)} / {tuple(v.shape)}")
        if v.dtype != k.dtype:
            v = v.to(k.dtype)
        s = table.slots
        is2 = s < cfg.offset
        if table._dev_index is not None:  # index lists routed on the device (alloc_device)
            pt, pi, it, ii = table._dev_index
            page_ids = s[is2][::g] // g
            t4 = np.flatnonzero(~is2)
        else:
            t2 = np.flatnonzero(is2)
            t4 = np.flatnonzero(~is2)
            if t2.size % g:
                raise ValidationError("INT2 tokens of a table must fill whole pages")
            page_tokens = t2.reshape(-1, g)
            page_ids = s[page_tokens[:, 0]] // g if t2.size else np.zeros(0, np.int64)
            dev = self.device
            pt = torch.as_tensor(page_tokens.astype(np.int32), device=dev)
            pi = torch.as_tensor(page_ids.astype(np.int32), device=dev)
            it = torch.as_tensor(t4.astype(np.int32), device=dev)
            ii = torch.as_tensor((s[t4] - cfg.offset).astype(np.int32), device=dev)
        _lib.check(lib.kvmix_write_prefill(
            k.data_ptr(), v.data_ptr(), _lib.dtype_code(k), cfg.n_layers, n, cfg.n_kv_heads, cfg.head_dim,
            pt.data_ptr(), pi.data_ptr(), pi.numel(), it.data_ptr(), ii.data_ptr(), it.numel(),
            self.int2_pool.data_ptr(), self.n_pages, self.int4_pool.data_ptr(), self.n_int4,
            self.status.data_ptr(), _lib.stream()))
        self._written = True
        if check_finite:
            self._check_err("keys/values")
        else:  # the caller opted out: a non-finite input must not fail a later, finite write
            self.status[_lib.POOL_STATUS_ERR].zero_()
        self._page_written[:, :, page_ids] = True
        self._int4_written[:, :, s[t4] - cfg.offset] = True

    def read_slot(self, address: SlotAddress, layer: int, head: int):
        """pool.py:264-282: decode one token's (k, v) for one (layer, head)."""
        slot = address.index
        if not 0 <= slot < self.config.total_slots or self._owner[slot] < 0:
            raise ValidationError(f"slot {slot} is not live")
        self._require_written(np.array([slot]), layer, head)
        k, v = self._gather_dev(np.array([slot]), layer)
        return k[0, head].cpu().numpy(), v[0, head].cpu().numpy()

    def _require_written(self, slots: np.ndarray, layer: int, head=None) -> None:
        cfg = self.config
        is2 = slots < cfg.offset
        hs = slice(None) if head is None else head
        ok2 = self._page_written[layer, hs][..., slots[is2] // cfg.page_size]
        ok4 = self._int4_written[layer, hs][..., slots[~is2] - cfg.offset]
        if not (np.all(ok2) and np.all(ok4)):
            raise ValidationError("slot read before write")

    def gather_device(self, slots, layer: int, dtype=torch.float32):
        """K5 on the device: k, v [m, Hkv, d] of ``slots`` (one layer) in ``dtype`` (f32: the
        exact dequantized values; bf16 / f16: their round-to-nearest images, ready for an
        fp16 / bf16 prefill attention over the pool).  Liveness and write checks as read_slot."""
        cfg = self.config
        s = np.asarray(slots, dtype=np.int64)
        if s.size and (s.min() < 0 or s.max() >= cfg.total_slots or np.any(self._owner[s] < 0)):
            raise ValidationError("gather of a slot that is not live")
        if not 0 <= layer < cfg.n_layers:
            raise ValidationError(f"layer {layer} out of range")
        self._require_written(s, layer)
        m = s.size
        sl = torch.as_tensor(s.astype(np.int32), device=self.device)
        k = torch.empty((m, cfg.n_kv_heads, cfg.head_dim), dtype=dtype, device=self.device)
        v = torch.empty_like(k)
        _lib.check(lib.kvmix_gather_dequant_typed(
            self.int2_pool.data_ptr(), self.int4_pool.data_ptr(), self.n_pages, self.n_int4, cfg.offset, layer,
            cfg.n_kv_heads, cfg.head_dim, sl.data_ptr(), m, k.data_ptr(), v.data_ptr(), _lib.dtype_code(k),
            _lib.stream()))
        return k, v

    def _gather_dev(self, slots: np.ndarray, layer: int):
        cfg = self.config
        m = slots.size
        sl = torch.as_tensor(slots.astype(np.int32), device=self.device)
        k = torch.empty((m, cfg.n_kv_heads, cfg.head_dim), dtype=torch.float32, device=self.device)
        v = torch.empty_like(k)
        _lib.check(lib.kvmix_gather_dequant(
            self.int2_pool.data_ptr(), self.int4_pool.data_ptr(), self.n_pages, self.n_int4, cfg.offset, layer,
            cfg.n_kv_heads, cfg.head_dim, sl.data_ptr(), m, k.data_ptr(), v.data_ptr(), _lib.stream()))
        return k, v

    def append_decode_token(self, request_id: str, k, v) -> SlotAddress:
        """pool.py:284-306: pop one INT4 slot (LIFO) and write k/v [L, Hkv, d] at INT4."""
        table = self._tables.get(request_id)
        if table is None:
            raise ValidationError(f"unknown request {request_id!r}")
        if not table.partitioned:
            raise ValidationError("partition the page table before decoding")
        if not self._free_int4:
            raise CapacityError("INT4 region exhausted during decode", region="int4")
        cfg = self.config
        kk = self._to_dev(k)
        vv = self._to_dev(v).to(kk.dtype)
        if tuple(kk.shape) != (cfg.n_layers, cfg.n_kv_heads, cfg.head_dim) or vv.shape != kk.shape:
            raise ValidationError("decode k/v must be [n_layers, n_kv_heads, head_dim]")
        slot = self._free_int4.pop()
        self._owner[slot] = self._rid_index[request_id]
        ids = torch.tensor([slot - cfg.offset], dtype=torch.int32, device=self.device)
        _lib.check(lib.kvmix_append_int4(kk.data_ptr(), vv.data_ptr(), _lib.dtype_code(kk), 1, cfg.n_layers, 0,
                                         cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, ids.data_ptr(),
                                         self.int4_pool.data_ptr(), self.n_int4, self.status.data_ptr(),
                                         _lib.stream()))
        self._written = True
        self._check_err("decode k/v")
        self._int4_written[:, :, slot - cfg.offset] = True
        table._append(slot)
        return SlotAddress(slot)

    def reserve_decode_slots(self, request_ids) -> np.ndarray:
        """Slot bookkeeping of append_decode_token (pool.py:284-306), batched: pop one INT4
        slot per request (LIFO, in request order) and append it to the request's partitioned
        table.  The data is written later -- by append_decode_tokens, or by the fused
        decode append of flash_decode_batched(..., append=...) one layer at a time."""
        B = len(request_ids)
        if len(self._free_int4) < B:
            raise CapacityError("INT4 region exhausted during decode", region="int4")
        for rid in request_ids:
            t = self._tables.get(rid)
            if t is None or not t.partitioned:
                raise ValidationError(f"request {rid!r} unknown or not partitioned")
        slots = np.empty(B, dtype=np.int64)
        for i, rid in enumerate(request_ids):
            s = self._free_int4.pop()
            slots[i] = s
            self._owner[s] = self._rid_index[rid]
            self._tables[rid]._append(s)
        return slots

    def append_decode_tokens(self, request_ids, k: torch.Tensor, v: torch.Tensor, layer: int | None = None,
                             slots: np.ndarray | None = None) -> np.ndarray:
        """Batched decode append (one token per request): k/v [B, L, Hkv, d], or
        [B, Hkv, d] for a single ``layer`` with ``slots`` popped by an earlier call.
        Returns the INT4 slots (pool.py:284-306, batched)."""
        cfg = self.config
        B = len(request_ids)
        if slots is None:
            slots = self.reserve_decode_slots(request_ids)
        ids = torch.as_tensor((slots - cfg.offset).astype(np.int32), device=self.device)
        if layer is None:
            lin, l0 = cfg.n_layers, 0
        else:
            lin, l0 = 1, layer
        _lib.check(lib.kvmix_append_int4(k.data_ptr(), v.data_ptr(), _lib.dtype_code(k), B, lin, l0,
                                         cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, ids.data_ptr(),
                                         self.int4_pool.data_ptr(), self.n_int4, self.status.data_ptr(),
                                         _lib.stream()))
        self._written = True
        self._int4_written[l0:l0 + lin, :, slots - cfg.offset] = True
        return slots

    # -- views and accounting -------------------------------------------------------------
    def view(self, layer: int) -> "PoolView":
        return PoolView(self, layer)

    def table(self, request_id: str) -> PageTable:
        return self._tables[request_id]

    def live_counts(self) -> tuple[int, int]:
        live = self._owner >= 0
        int2 = int(live[: self.config.offset].sum())
        return int2, int(live.sum()) - int2

    def free_counts(self) -> tuple[int, int]:
        return len(self._free_pages) * self.config.page_size, len(self._free_int4)

    def parameter_overhead_bytes(self) -> int:
        """pool.py:323-332: fp16 (scale, zero) bytes across written blocks."""
        cfg = self.config
        per = 4
        key_page_params = cfg.head_dim * per
        token_params = (cfg.head_dim // cfg.page_size) * per
        n_key_pages = int(self._page_written.sum())
        n_v2 = n_key_pages * cfg.page_size
        n_4 = int(self._int4_written.sum())
        return n_key_pages * key_page_params + (n_v2 + 2 * n_4) * token_params

    def stats(self) -> dict:
        """pool.py:334-348."""
        cfg = self.config
        live2, live4 = self.live_counts()
        free2, free4 = self.free_counts()
        live_total = live2 + live4
        realized = (2 * live2 + 4 * live4) / live_total if live_total else None
        return {
            "total_slots": cfg.total_slots,
            "offset": cfg.offset,
            "page_size": cfg.page_size,
            "int2": {"total": cfg.offset, "live": live2, "free": free2},
            "int4": {"total": cfg.total_slots - cfg.offset, "live": live4, "free": free4},
            "parameter_overhead_bytes": self.parameter_overhead_bytes(),
            "realized_avg_bitwidth": realized,
        }

    def check_invariants(self) -> None:
        """pool.py:350-377: conservation, duplicates, aliasing, owner sync."""
        cfg, g = self.config, self.config.page_size
        free2, free4 = self.free_counts()
        live2, live4 = self.live_counts()
        if live2 + free2 != cfg.offset:
            raise AssertionError("INT2 slot conservation violated")
        if live4 + free4 != cfg.total_slots - cfg.offset:
            raise AssertionError("INT4 slot conservation violated")
        fp = np.asarray(self._free_pages, dtype=np.int64)
        f4 = np.asarray(self._free_int4, dtype=np.int64)
        if np.unique(fp).size != fp.size:
            raise AssertionError("duplicate pages on the free list")
        if np.unique(f4).size != f4.size:
            raise AssertionError("duplicate slots on the INT4 free list")
        if fp.size and np.any(self._owner[(fp[:, None] + np.arange(g)).reshape(-1)] >= 0):
            raise AssertionError("free page aliases a live slot")
        if f4.size and np.any(self._owner[f4] >= 0):
            raise AssertionError("free INT4 slot aliases a live slot")
        seen = np.zeros(cfg.total_slots, dtype=bool)
        for rid, table in self._tables.items():
            s = table.slots
            if np.unique(s).size != s.size or np.any(seen[s]):
                raise AssertionError("slot referenced by two page tables")
            seen[s] = True
            if np.any(self._owner[s] != self._rid_index[rid]):
                raise AssertionError("owner map out of sync with page tables")
        if np.any((self._owner >= 0) != seen):
            raise AssertionError("owner map out of sync with page tables")

    # -- device page tables -------------------------------------------------------------
    def device_tables(self, request_ids) -> dict:
        """CSR page tables of partitioned requests for the decode kernel:
        INT2 page ids (table order) and INT4 indices (table order)."""
        cfg, g = self.config, self.config.page_size
        pages, int4 = [], []
        for rid in request_ids:
            t = self._tables.get(rid)
            if t is None:
                raise ValidationError(f"unknown request {rid!r}")
            p, i4 = split_partitioned(t.slots, cfg.offset, g)
            pages.append(p)
            int4.append(i4)
        return csr_tables(pages, int4, self.device)


def split_partitioned(slots: np.ndarray, offset: int, g: int = GROUP_SIZE):
    """(int2 page ids, int4 indices) of a partitioned table; validates that the INT2
    prefix is page-granular (entries[32p + j] == page_start_p + j), which every table
    built by alloc/partition/append satisfies."""
    is2 = slots < offset
    n2 = int(is2.sum())
    if np.any(is2[n2:]):
        raise ValidationError("page table not partitioned: INT4 address precedes INT2")
    pre = slots[:n2]
    if n2 % g:
        raise ValidationError("INT2 prefix is not page-granular")
    runs = pre.reshape(-1, g)
    if runs.size and (np.any(runs[:, 0] % g) or np.any(runs - runs[:, :1] != np.arange(g))):
        raise ValidationError("INT2 prefix is not page-granular")
    return (runs[:, 0] // g).astype(np.int32), (slots[n2:] - offset).astype(np.int32)


def csr_tables(pages: list, int4: list, device) -> dict:
    np_ = np.array([p.size for p in pages], dtype=np.int64)
    n4 = np.array([x.size for x in int4], dtype=np.int64)
    page_indptr = np.concatenate([[0], np.cumsum(np_)]).astype(np.int32)
    int4_indptr = np.concatenate([[0], np.cumsum(n4)]).astype(np.int32)
    cat = lambda xs: np.concatenate(xs).astype(np.int32) if xs and sum(x.size for x in xs) else np.zeros(1, np.int32)
    return {
        "n_pages": np_,
        "n_int4": n4,
        "page_indptr": torch.as_tensor(page_indptr, device=device),
        "page_ids": torch.as_tensor(cat(pages), device=device),
        "int4_indptr": torch.as_tensor(int4_indptr, device=device),
        "int4_ids": torch.as_tensor(cat(int4), device=device),
    }


class PoolView:
    """Read-only, single-layer window used by the flash-decode path (pool.py:380-439)."""

    def __init__(self, pool: MixedPrecisionPool, layer: int):
        self._pool = pool
        self.layer = layer

    @property
    def pool(self) -> MixedPrecisionPool:
        return self._pool

    @property
    def n_kv_heads(self) -> int:
        return self._pool.config.n_kv_heads

    def is_int2(self, address: SlotAddress) -> bool:
        return self._pool.is_int2(address)

    def gather(self, addresses):
        """K5: decode K, V for the addressed tokens -> two [m, n_kv_heads, d] fp32 arrays."""
        pool = self._pool
        slots = np.asarray([a.index for a in addresses], dtype=np.int64)
        in_range = (slots >= 0) & (slots < pool.config.total_slots)
        live = np.zeros(slots.size, dtype=bool)
        live[in_range] = pool._owner[slots[in_range]] >= 0
        if not np.all(live):
            raise ValidationError(f"dangling slot address {int(slots[~live][0])}")
        pool._require_written(slots, self.layer)
        k, v = pool._gather_dev(slots, self.layer)
        return k.cpu().numpy(), v.cpu().numpy()


def bytes_per_token(head_dim: int, n_layers: int, n_kv_heads: int, bitwidth: int,
                    group_len: int = GROUP_SIZE) -> float:
    """pool.py:442-459 (INT2 key page amortised over its group_len tokens)."""
    if bitwidth == 2:
        key = key_page_payload_bytes(head_dim, group_len) / group_len
        value = token_block_payload_bytes(head_dim, 2, group_len)
    elif bitwidth == 4:
        key = token_block_payload_bytes(head_dim, 4, group_len)
        value = token_block_payload_bytes(head_dim, 4, group_len)
    else:
        raise ValidationError(f"unsupported bitwidth {bitwidth}")
    return n_layers * n_kv_heads * (key + value)


def baseline_bytes_per_token(head_dim: int, n_layers: int, n_kv_heads: int, bytes_per_element: int = 2) -> int:
    """pool.py:462-466."""
    return n_layers * n_kv_heads * head_dim * 2 * bytes_per_element


def capacity_tokens(total_bytes: float, avg_bitwidth: float, head_dim: int, n_layers: int, n_kv_heads: int,
                    group_len: int = GROUP_SIZE) -> int:
    """pool.py:469-478."""
    f2 = (4.0 - avg_bitwidth) / 2.0
    per_token = f2 * bytes_per_token(head_dim, n_layers, n_kv_heads, 2, group_len) + (
        1.0 - f2) * bytes_per_token(head_dim, n_layers, n_kv_heads, 4, group_len)
    return int(total_bytes // per_token)
