"""Multi-GPU sharding of the decode hot path (one process per GPU, torch.distributed).

The reference is single-process; the path shards two ways (8(e)):

* batch-parallel (cfg5): requests -> ranks.  Every rank owns a full pool and its own
  requests; there is no collective on the data path (weak scaling).
* KV-head-parallel (cfg4): rank r owns KV heads [r*Hkv/W, (r+1)*Hkv/W) and their GQA
  q heads.  Slot addresses are head-agnostic (blocks are keyed (slot, layer, head),
  pool.py:108-110), so page tables are replicated: rank 0 runs the allocator and
  broadcasts the slot lists, every rank quantizes only its head slice into its own
  pool, decodes its heads, and one all-gather per layer assembles out [B, Hq, d].
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import ValidationError


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_requests(request_ids, rank: int, world_size: int) -> list:
    """Batch-parallel: contiguous, near-equal shards of the request list."""
    n = len(request_ids)
    lo = n * rank // world_size
    hi = n * (rank + 1) // world_size
    return list(request_ids[lo:hi])


def head_slice(n_kv_heads: int, n_q_heads: int, rank: int, world_size: int) -> tuple[slice, slice]:
    """KV-head-parallel: (kv head slice, q head slice) owned by ``rank``."""
    if n_kv_heads % world_size:
        raise ValidationError(f"{n_kv_heads} kv heads do not split over {world_size} ranks")
    hk = n_kv_heads // world_size
    g = n_q_heads // n_kv_heads
    return slice(rank * hk, (rank + 1) * hk), slice(rank * hk * g, (rank + 1) * hk * g)


def broadcast_slots(slots: np.ndarray | None, src: int = 0, group=None) -> np.ndarray:
    """Replicate one request's slot list (page table) from ``src`` to every rank."""
    rank, _ = world()
    obj = [slots.tolist() if rank == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return np.asarray(obj[0], dtype=np.int64)


def adopt_table(pool, request_id: str, slots: np.ndarray, partitioned: bool = False):
    """Install a page table computed on another rank into this rank's pool (same
    allocator state transition as ``alloc`` produced there)."""
    from .pool import PageTable

    cfg, g = pool.config, pool.config.page_size
    if request_id in pool._tables:
        raise ValidationError(f"request {request_id!r} already live")
    slots = np.asarray(slots, dtype=np.int64)
    pages = np.unique(slots[slots < cfg.offset] // g * g)
    int4 = slots[slots >= cfg.offset]
    taken_pages, taken_int4 = set(pages.tolist()), set(int4.tolist())  # built once: O(|free| + |table|)
    if not taken_pages <= set(pool._free_pages) or not taken_int4 <= set(pool._free_int4):
        raise ValidationError("adopted table uses slots that are not free on this rank")
    pool._free_pages = [p for p in pool._free_pages if p not in taken_pages]
    pool._free_int4 = [s for s in pool._free_int4 if s not in taken_int4]
    rix = pool._next_rid
    pool._next_rid += 1
    pool._rid_index[request_id] = rix
    pool._owner[slots] = rix
    table = PageTable(request_id=request_id, slots=slots, partitioned=partitioned)
    pool._tables[request_id] = table
    return table


def gather_heads(out_local: torch.Tensor, out_full: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """All-gather the per-rank head slices [B, Hq/W, d] into [B, Hq, d] (rank-major
    head order == natural head order because every rank owns a contiguous slice)."""
    rank, W = world()
    B, hl, d = out_local.shape
    buf = torch.empty((W * B, hl, d), dtype=out_local.dtype, device=out_local.device)
    if W == 1:
        buf.copy_(out_local)
    else:
        dist.all_gather_into_tensor(buf, out_local.contiguous(), group=group)
    full = buf.view(W, B, hl, d).permute(1, 0, 2, 3).reshape(B, W * hl, d)
    if out_full is not None:
        out_full.copy_(full)
        return out_full
    return full


@dataclass
class HeadOutputs:
    """Destinations of the KV-head-parallel combine fused into the decode kernel
    (``flash_decode_batched(..., gather=...)``, C ABI kvmix_flash_decode_gather): this rank's
    q heads [head0, head0 + n_q_heads) are stored into each buffer ``ptrs[i]`` =
    [B, out_heads, d] (``dtype``) -- its own and the peers' mapped over NVLink."""

    ptrs: list
    out_heads: int
    head0: int
    dtype: torch.dtype
    batch: int
    head_dim: int
    device: torch.device | None = None

    def check(self, batch: int, n_q_heads: int, head_dim: int, device) -> None:
        if not 1 <= len(self.ptrs) <= 8:
            raise ValidationError("the fused head gather stores to 1 to 8 buffers")
        if any(not p for p in self.ptrs):
            raise ValidationError("null gather destination")
        if batch != self.batch or head_dim != self.head_dim:
            raise ValidationError(f"gather buffers are [{self.batch}, {self.out_heads}, {self.head_dim}]")
        if not 0 <= self.head0 or self.head0 + n_q_heads > self.out_heads:
            raise ValidationError("this rank's head slice falls outside the gather buffers")
        if self.device is not None and torch.device(device) != torch.device(self.device):
            raise ValidationError(f"gather buffers live on {self.device}, the pool on {device}")

    @classmethod
    def local(cls, buffers, head0: int) -> "HeadOutputs":
        """Destinations that are tensors of this process ([B, out_heads, d] each, contiguous)."""
        b0 = buffers[0]
        for b in buffers:
            if (b.shape != b0.shape or b.dtype != b0.dtype or b.device != b0.device or not b.is_contiguous()
                    or b.dim() != 3):
                raise ValidationError("gather buffers must be equal contiguous [B, out_heads, d] tensors")
        return cls([b.data_ptr() for b in buffers], b0.shape[1], head0, b0.dtype, b0.shape[0], b0.shape[2], b0.device)


class SymmetricHeadGather:
    """The cfg4 combine over NVLink: a symmetric-memory output [n_layers, B, Hq, d] on every
    rank (torch.distributed._symmetric_memory: each rank's buffer is mapped into every peer's
    address space), and per layer the HeadOutputs that make each rank's decode kernel store
    its head slice into all ranks' buffers.  ``barrier()`` (a signal-pad barrier on the
    device, stream-ordered) makes every rank's stores visible before the outputs are read;
    ``gather_heads`` (NCCL all_gather_into_tensor) is the path it replaces."""

    def __init__(self, n_layers: int, batch: int, n_q_heads: int, head_dim: int, dtype=torch.bfloat16,
                 device=None, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        rank, W = world()
        if n_q_heads % W:
            raise ValidationError(f"{n_q_heads} q heads do not split over {W} ranks")
        if W > 8:
            raise ValidationError("the fused head gather spans at most 8 ranks (one NVLink domain)")
        self.shape = (n_layers, batch, n_q_heads, head_dim)
        self.rank, self.world, self.dtype = rank, W, dtype
        self.head0 = rank * (n_q_heads // W)
        self.out = symm_mem.empty(self.shape, dtype=dtype, device=device)
        grp = group if group is not None else dist.group.WORLD
        self.handle = symm_mem.rendezvous(self.out, grp)
        self._layer_bytes = batch * n_q_heads * head_dim * self.out.element_size()
        # the tensor sits at the same offset of every rank's symmetric allocation
        off = self.out.data_ptr() - int(self.handle.buffer_ptrs[rank])
        self._bases = [int(self.handle.buffer_ptrs[r]) + off for r in range(W)]

    def layer(self, layer: int) -> HeadOutputs:
        L, B, Hq, d = self.shape
        if not 0 <= layer < L:
            raise ValidationError("layer out of range")
        ptrs = [base + layer * self._layer_bytes for base in self._bases]
        return HeadOutputs(ptrs, Hq, self.head0, self.dtype, B, d, self.out.device)

    def barrier(self) -> None:
        self.handle.barrier(channel=0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Timing is reported as the max over ranks (slowest rank defines the step)."""
    rank, W = world()
    if W == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
