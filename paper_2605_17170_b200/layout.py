"""Device record layout of the dual-precision pool (host-side restatement).

The reference stores each block as its LAYOUT.md payload (``bytes`` in dicts keyed
(slot|page, layer, head), pool.py:108-110).  The device pool keeps exactly the same
bytes -- every code byte and every fp16 (scale, zero) of every payload, nothing
added or re-rounded -- but permutes them inside a fixed-size record so that the
decode kernel (csrc/decode.cu) can load each lane's MMA fragment with one wide,
bank-conflict-free shared-memory load and no byte shuffling.  This module is the
numpy statement of that permutation, used by tests to prove the device bytes are
the reference payloads (``page_payloads`` / ``slot_payloads``), and it mirrors the
device helpers in csrc/common.cuh (``pg_*`` / ``sl_*``) line for line.

d = head_dim, ng = d / 32 (channel groups), G = 32 (page = group size, quant.py:23).

INT2 page record (24 d bytes; 3072 at d = 128) = one KeyPageBlock (quant.py:131-186)
plus the page's 32 INT2 V TokenBlocks (quant.py:145-262) in slot order::

  KC [0, 8d)     key codes, byte-major: row tau (tokens 4tau..4tau+3) holds code byte
                 tau of every channel word (KeyPage byte 8c + tau); inside a row the
                 16-byte chunks are XOR-swizzled with (tau & 1)
  KS [8d, 10d)   key scales, fp16: lane q owns channels [q d/4, (q+1) d/4) in 8-channel chunks;
                 chunk i of lane q is chunk 4i + q; channel 8P + 4I + e of a chunk sits
                 at 4(e>>1) + 2I + (e&1)
  VC [10d, 18d)  value codes: word ((ks*8 + g)*4 + q)*ng + j holds code byte
                 b = 8j + g of tokens [T0, T0+1, T1, T1+1], T0 = 8q + 2ks, T1 = T0 + 4
  VS [18d, 20d)  value scales: half (((j*4 + q)*2 + p)*2 + ks)*2 + h is the scale of
                 group j of token 8q + 2ks + 4h + p
  VZ [20d, 22d)  value zeros, same order
  KZ [22d, 24d)  key zeros, in the KS order (last: the decode kernel copies [0, 22d) per
                 tile and stages the zeros of 16 pages at once for its batched key bias)

INT4 slot record (d + 8 ng bytes, rounded up to 16; 160 at d = 128) = INT4 K
TokenBlock then INT4 V TokenBlock, each permuted as::

  codes  K: payload byte 16j + 4q + e  -> 4 ng q + 4j + e      (q < 4, e < 4)
         V: payload byte 16j + 2g + e  -> 2 ng g + 2j + e      (g < 8, e < 2)
  then the ng scales, then the ng zeros (fp16).
"""

from __future__ import annotations

import functools

import numpy as np

G = 32


def page_stride(d: int) -> int:
    return 24 * d


def slot_stride(d: int) -> int:
    return -(-(d + 8 * (d // 32)) // 16) * 16


def _kp_pos(d: int, c: int) -> int:
    """Half index of channel c inside KS/KZ (see the module docstring)."""
    kb = d // 4  # channels per lane q
    q, o = divmod(c, kb)
    e = c & 3
    return (((o >> 3) * 4 + q) << 3) | ((e >> 1) << 2) | (((c >> 2) & 1) << 1) | (e & 1)


@functools.lru_cache(maxsize=None)
def page_perm(d: int) -> np.ndarray:
    """perm[i] = byte of (KeyPageBlock || 32 INT2 V TokenBlocks) stored at record byte i."""
    ng = d // 32
    kp = 12 * d  # KeyPageBlock payload: 8d code bytes + 4d param bytes (quant.py:123-124)
    tb2 = d // 4 + 4 * ng  # INT2 TokenBlock payload (quant.py:127-128)
    perm = np.full(page_stride(d), -1, dtype=np.int64)
    for tau in range(8):
        for c in range(d):
            phys = (((c >> 4) ^ (tau & 1)) << 4) | (c & 15)
            perm[tau * d + phys] = 8 * c + tau
    for c in range(d):
        pos = _kp_pos(d, c)
        for k in range(2):
            perm[8 * d + 2 * pos + k] = 8 * d + 4 * c + k  # scale_c
            perm[22 * d + 2 * pos + k] = 8 * d + 4 * c + 2 + k  # zero_c
    for ks in range(2):
        for g in range(8):
            for q in range(4):
                for j in range(ng):
                    w = ((ks * 8 + g) * 4 + q) * ng + j
                    t0 = 8 * q + 2 * ks
                    for pos, t in enumerate((t0, t0 + 1, t0 + 4, t0 + 5)):
                        perm[10 * d + 4 * w + pos] = kp + t * tb2 + 8 * j + g
    for ks in range(2):
        for q in range(4):
            for j in range(ng):
                for p in range(2):
                    for h in range(2):
                        idx = (((j * 4 + q) * 2 + p) * 2 + ks) * 2 + h
                        t = 8 * q + 2 * ks + 4 * h + p
                        for k in range(2):
                            perm[18 * d + 2 * idx + k] = kp + t * tb2 + d // 4 + 4 * j + k
                            perm[20 * d + 2 * idx + k] = kp + t * tb2 + d // 4 + 4 * j + 2 + k
    assert (np.sort(perm) == np.arange(page_stride(d))).all()
    return perm


@functools.lru_cache(maxsize=None)
def slot_perm(d: int) -> np.ndarray:
    """perm[i] = byte of (INT4 K TokenBlock || INT4 V TokenBlock) stored at record byte i (-1: padding)."""
    ng = d // 32
    tb4 = d // 2 + 4 * ng
    perm = np.full(slot_stride(d), -1, dtype=np.int64)
    for base in (0, tb4):
        for j in range(ng):
            for k in range(2):
                perm[base + d // 2 + 2 * j + k] = base + d // 2 + 4 * j + k
                perm[base + d // 2 + 2 * ng + 2 * j + k] = base + d // 2 + 4 * j + 2 + k
        for j in range(ng):
            if base == 0:
                for q in range(4):
                    for e in range(4):
                        perm[4 * ng * q + 4 * j + e] = 16 * j + 4 * q + e
            else:
                for g in range(8):
                    for e in range(2):
                        perm[base + 2 * ng * g + 2 * j + e] = base + 16 * j + 2 * g + e
    used = perm[perm >= 0]
    assert (np.sort(used) == np.arange(2 * tb4)).all()
    return perm


def page_records(ref: np.ndarray, d: int) -> np.ndarray:
    """Reference-order page images [..., >= 24d] (KeyPage || 32 V blocks) -> device records."""
    return np.ascontiguousarray(np.asarray(ref, np.uint8)[..., page_perm(d)])


def page_payloads(rec: np.ndarray, d: int) -> np.ndarray:
    """Device page records [..., 24d] -> reference order (KeyPageBlock || 32 INT2 V TokenBlocks)."""
    rec = np.asarray(rec, np.uint8)
    out = np.empty_like(rec[..., : page_stride(d)])
    out[..., page_perm(d)] = rec[..., : page_stride(d)]
    return out


def slot_records(ref: np.ndarray, d: int) -> np.ndarray:
    """Reference-order slot images [..., >= 2 tb4] (K block || V block) -> device records (zero padding)."""
    ref = np.asarray(ref, np.uint8)
    perm = slot_perm(d)
    out = ref[..., np.maximum(perm, 0)]
    out[..., perm < 0] = 0
    return np.ascontiguousarray(out)


def slot_payloads(rec: np.ndarray, d: int) -> np.ndarray:
    """Device slot records -> reference order (INT4 K TokenBlock || INT4 V TokenBlock)."""
    rec = np.asarray(rec, np.uint8)
    perm = slot_perm(d)
    n = int((perm >= 0).sum())
    out = np.empty(rec.shape[:-1] + (n,), np.uint8)
    keep = perm >= 0
    out[..., perm[keep]] = rec[..., : perm.size][..., keep]
    return out
