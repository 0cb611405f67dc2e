"""Oracle (test infrastructure only): restatement of the reference pool.

Control plane follows /root/reference/pkg/src/kvmix/pool.py:
  init_pool           pool.py:63-93   (INT2 fraction (4-B)/2, floor to page, +1e-6)
  free lists          pool.py:102-105 (LIFO stacks, lowest address handed out first)
  alloc               pool.py:122-163 (p-th group of G INT2 tokens -> p-th popped page;
                                       residual INT2 + INT4 tokens, sorted -> INT4 pops)
  free                pool.py:165-188 (INT4 slots pushed in entry order; pages pushed
                                       in descending start order)
  partition           pool.py:190-197 (stable, INT2 first, idempotent)
  append_decode_token pool.py:284-306 (needs a partitioned table; one INT4 pop)
  check_invariants    pool.py:350-377

Data plane: instead of the reference's dicts of ``bytes`` keyed by
(slot|page, layer, head) (pool.py:108-110) this oracle keeps numpy byte images
with the SAME layout as the device pools:

  int2[L][Hkv][n_pages][page_stride] = KeyPageBlock ‖ G INT2 V TokenBlocks (slot order)
  int4[L][Hkv][n_int4][slot_stride]  = INT4 K TokenBlock ‖ INT4 V TokenBlock

so every reference payload is a contiguous, unmodified byte range and the device
pool can be compared byte-for-byte with this image.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import codec


class OracleError(Exception):
    """Raised where the reference raises ValidationError / CapacityError."""

    def __init__(self, kind: str, msg: str, region: str | None = None):
        super().__init__(msg)
        self.kind = kind
        self.region = region


@dataclass(frozen=True)
class Config:
    total_slots: int
    offset: int
    n_layers: int
    n_kv_heads: int
    head_dim: int
    page_size: int = codec.GROUP_SIZE


def init_pool(avg_bits, total_slots, n_layers, n_kv_heads, head_dim, page_size=32) -> Config:
    """pool.py:63-93."""
    if not 2.0 <= avg_bits <= 4.0:
        raise OracleError("validation", "average bitwidth outside [2, 4]")
    if total_slots < 2 * page_size:
        raise OracleError("validation", "pool needs at least two pages")
    frac = (4.0 - avg_bits) / 2.0
    offset = int(frac * total_slots + 1e-6) // page_size * page_size
    return Config(total_slots, offset, n_layers, n_kv_heads, head_dim, page_size)


def page_stride(d: int, g: int = 32) -> int:
    raw = codec.key_page_nbytes(d, g) + g * codec.token_block_nbytes(d, 2, g)
    return -(-raw // 16) * 16


def slot_stride(d: int, g: int = 32) -> int:
    raw = 2 * codec.token_block_nbytes(d, 4, g)
    return -(-raw // 16) * 16


class OraclePool:
    def __init__(self, cfg: Config, data_plane: bool = True):
        self.cfg = cfg
        g = cfg.page_size
        self.n_pages = cfg.offset // g
        self.n_int4 = cfg.total_slots - cfg.offset
        # pool.py:104-105: stacks whose top is the lowest address
        self.free_pages = list(range((self.n_pages - 1) * g, -g, -g)) if self.n_pages else []
        self.free_int4 = list(range(cfg.total_slots - 1, cfg.offset - 1, -1))
        self.tables: dict[str, list[int]] = {}
        self.partitioned: dict[str, bool] = {}
        self.owner: dict[int, str] = {}
        d = cfg.head_dim
        self.kp = codec.key_page_nbytes(d, g)
        self.tb2 = codec.token_block_nbytes(d, 2, g)
        self.tb4 = codec.token_block_nbytes(d, 4, g)
        self.data_plane = data_plane
        if data_plane:
            L, H = cfg.n_layers, cfg.n_kv_heads
            self.int2 = np.zeros((L, H, self.n_pages, page_stride(d, g)), np.uint8)
            self.int4 = np.zeros((L, H, self.n_int4, slot_stride(d, g)), np.uint8)
            self.page_written = np.zeros((L, H, self.n_pages), bool)
            self.slot_written = np.zeros((L, H, self.n_int4), bool)

    # -- control plane ---------------------------------------------------------
    def is_int2(self, slot: int) -> bool:
        return slot < self.cfg.offset

    def alloc(self, rid: str, bits) -> list[int]:
        """pool.py:122-163."""
        if rid in self.tables:
            raise OracleError("validation", f"request {rid!r} already live")
        bits = np.asarray(bits)
        if not np.all(np.isin(bits, (2, 4))):
            raise OracleError("validation", "bitwidths must be 2 or 4")
        g = self.cfg.page_size
        idx2 = np.flatnonzero(bits == 2)
        n_pages = idx2.size // g
        rest = np.sort(np.concatenate([np.flatnonzero(bits == 4), idx2[n_pages * g:]]))
        if n_pages > len(self.free_pages):
            raise OracleError("capacity", "INT2 region exhausted", region="int2")
        if rest.size > len(self.free_int4):
            raise OracleError("capacity", "INT4 region exhausted", region="int4")
        slots = np.empty(bits.size, dtype=np.int64)
        for p in range(n_pages):
            start = self.free_pages.pop()
            slots[idx2[p * g:(p + 1) * g]] = start + np.arange(g)
        for t in rest:
            slots[t] = self.free_int4.pop()
        out = [int(s) for s in slots]
        for s in out:
            self.owner[s] = rid
        self.tables[rid] = out
        self.partitioned[rid] = False
        return out

    def free(self, rid: str) -> None:
        """pool.py:165-188."""
        if rid not in self.tables:
            raise OracleError("validation", f"unknown request {rid!r}")
        entries = self.tables.pop(rid)
        self.partitioned.pop(rid)
        g = self.cfg.page_size
        pages = set()
        for s in entries:
            del self.owner[s]
            if self.is_int2(s):
                pages.add(s // g * g)
            else:
                self.free_int4.append(s)
                if self.data_plane:
                    self.slot_written[:, :, s - self.cfg.offset] = False
        for start in sorted(pages, reverse=True):
            self.free_pages.append(start)
            if self.data_plane:
                self.page_written[:, :, start // g] = False

    def partition(self, rid: str) -> list[int]:
        """pool.py:190-197."""
        if not self.partitioned[rid]:
            e = self.tables[rid]
            self.tables[rid] = [s for s in e if self.is_int2(s)] + [s for s in e if not self.is_int2(s)]
            self.partitioned[rid] = True
        return self.tables[rid]

    def pop_decode_slot(self, rid: str) -> int:
        """Slot bookkeeping of append_decode_token (pool.py:284-306)."""
        if rid not in self.tables:
            raise OracleError("validation", f"unknown request {rid!r}")
        if not self.partitioned[rid]:
            raise OracleError("validation", "partition the page table before decoding")
        if not self.free_int4:
            raise OracleError("capacity", "INT4 region exhausted during decode", region="int4")
        s = self.free_int4.pop()
        self.owner[s] = rid
        self.tables[rid].append(s)
        return s

    def check_invariants(self) -> None:
        """pool.py:350-377."""
        cfg, g = self.cfg, self.cfg.page_size
        live2 = sum(1 for s in self.owner if s < cfg.offset)
        live4 = len(self.owner) - live2
        assert live2 + len(self.free_pages) * g == cfg.offset
        assert live4 + len(self.free_int4) == cfg.total_slots - cfg.offset
        assert len(set(self.free_pages)) == len(self.free_pages)
        assert len(set(self.free_int4)) == len(self.free_int4)
        for start in self.free_pages:
            for j in range(g):
                assert start + j not in self.owner
        for s in self.free_int4:
            assert s not in self.owner
        seen = set()
        for rid, e in self.tables.items():
            for s in e:
                assert s not in seen
                seen.add(s)
                assert self.owner.get(s) == rid

    # -- data plane --------------------------------------------------------------
    def write_prefill(self, rid: str, keys, values) -> None:
        """pool.py:228-262: keys/values [L, N, Hkv, d] in token order."""
        if self.partitioned[rid]:
            raise OracleError("validation", "write_prefill requires token-ordered entries")
        entries = np.asarray(self.tables[rid])
        keys = np.asarray(keys, dtype=np.float32)
        values = np.asarray(values, dtype=np.float32)
        g, off = self.cfg.page_size, self.cfg.offset
        is2 = entries < off
        t2 = np.flatnonzero(is2)
        t4 = np.flatnonzero(~is2)
        if t2.size:
            runs = t2.reshape(-1, g)  # [P, G] token ids, page-granular by construction
            pages = entries[runs[:, 0]] // g
            kk = keys[:, runs]  # [L, P, G, H, d]
            vv = values[:, runs]
            kblk = codec.encode_key_pages(np.moveaxis(kk, 3, 1))  # [L, H, P, G, d] -> [L, H, P, kp]
            vblk = codec.encode_token_blocks(np.moveaxis(vv, 3, 1), 2)  # [L, H, P, G, tb2]
            rec = np.concatenate([kblk, vblk.reshape(vblk.shape[:3] + (-1,))], axis=-1)
            self.int2[:, :, pages, :rec.shape[-1]] = rec
            self.page_written[:, :, pages] = True
        if t4.size:
            idx = entries[t4] - off
            kb = codec.encode_token_blocks(np.moveaxis(keys[:, t4], 2, 1), 4)  # [L, H, M, tb4]
            vb = codec.encode_token_blocks(np.moveaxis(values[:, t4], 2, 1), 4)
            rec = np.concatenate([kb, vb], axis=-1)
            self.int4[:, :, idx, :rec.shape[-1]] = rec
            self.slot_written[:, :, idx] = True

    def write_decode(self, slot: int, k, v) -> None:
        """Data half of append_decode_token: k/v [L, Hkv, d] at INT4 (pool.py:302-304)."""
        idx = slot - self.cfg.offset
        kb = codec.encode_token_blocks(np.asarray(k, np.float32), 4)  # [L, H, tb4]
        vb = codec.encode_token_blocks(np.asarray(v, np.float32), 4)
        rec = np.concatenate([kb, vb], axis=-1)
        self.int4[:, :, idx, :rec.shape[-1]] = rec
        self.slot_written[:, :, idx] = True

    def gather(self, slots, layer: int):
        """Decode K, V [m, Hkv, d] for addressed slots.  pool.py:394-439."""
        d, g, off = self.cfg.head_dim, self.cfg.page_size, self.cfg.offset
        slots = np.asarray(slots, dtype=np.int64)
        for s in slots:
            if int(s) not in self.owner:
                raise OracleError("validation", f"dangling slot address {int(s)}")
        H = self.cfg.n_kv_heads
        k = np.empty((slots.size, H, d), np.float32)
        v = np.empty_like(k)
        is2 = slots < off
        if is2.any():
            pg = slots[is2] // g
            row = slots[is2] % g
            if not self.page_written[layer][:, pg].all():
                raise OracleError("validation", "slot read before write")
            upg, inv = np.unique(pg, return_inverse=True)  # decode each page once (pool.py:419-425)
            rec = self.int2[layer][:, upg]  # [H, P, stride]
            kd = codec.decode_key_pages(rec[..., :self.kp], d, g)  # [H, P, G, d]
            k[is2] = np.swapaxes(kd[:, inv, row], 0, 1)
            vrec = rec[..., self.kp:self.kp + g * self.tb2].reshape(H, -1, g, self.tb2)
            v[is2] = np.swapaxes(codec.decode_token_blocks(vrec[:, inv, row], d, 2, g), 0, 1)
        if (~is2).any():
            idx = slots[~is2] - off
            if not self.slot_written[layer][:, idx].all():
                raise OracleError("validation", "slot read before write")
            rec = self.int4[layer][:, idx]
            k[~is2] = np.swapaxes(codec.decode_token_blocks(rec[..., :self.tb4], d, 4, g), 0, 1)
            v[~is2] = np.swapaxes(codec.decode_token_blocks(rec[..., self.tb4:2 * self.tb4], d, 4, g), 0, 1)
        return k, v

    def int2_pages(self, rid: str) -> np.ndarray:
        """Page ids of the (partitioned) INT2 prefix, in table order."""
        e = np.asarray(self.tables[rid])
        return e[e < self.cfg.offset][:: self.cfg.page_size] // self.cfg.page_size

    def int4_ids(self, rid: str) -> np.ndarray:
        e = np.asarray(self.tables[rid])
        return e[e >= self.cfg.offset] - self.cfg.offset
