"""Split-K work planner for the decode kernel (host side, O(batch)).

The reference splits each request's partitioned table into contiguous
bitwidth-homogeneous chunks of ``split_len`` entries (attention.py:205-208).  On the
GPU the unit of work is a tile -- one INT2 page (32 tokens, page_stride bytes) or 32
INT4 slots (32*slot_stride bytes) -- and a work item is a contiguous tile range of one
(request, kv head).  Splits are sized by bytes so that the whole launch is about
``waves`` waves of ``ctas_per_sm`` CTAs on every SM, and every split of a unit
carries about the same number of bytes.
"""

from __future__ import annotations

import math

import numpy as np

NUM_SMS_B200 = 148


def plan_splits(n_pages, n_int4, n_kv_heads: int, page_stride: int, slot_stride: int,
                n_sm: int = NUM_SMS_B200, ctas_per_sm: int = 2, waves: float = 4.0,
                min_tiles: int = 8, max_splits: int | None = None):
    """Return (work int32 [n_work, 4], part_indptr int32 [B*Hkv + 1], n_parts).

    work rows are (unit = b*Hkv + kvh, tile_lo, tile_hi, partial_slot).
    """
    n_pages = np.asarray(n_pages, dtype=np.int64)
    n_int4 = np.asarray(n_int4, dtype=np.int64)
    B = n_pages.size
    t4 = (n_int4 + 31) // 32
    tiles = n_pages + t4
    if np.any(tiles <= 0):
        raise ValueError("every request needs at least one cached token")
    tile4 = 32 * slot_stride
    wbytes = n_pages * page_stride + n_int4 * slot_stride
    total = float(wbytes.sum()) * n_kv_heads
    target = max(total / (n_sm * ctas_per_sm * waves), float(min_tiles * page_stride))
    rows = []
    part_counts = np.zeros(B * n_kv_heads, dtype=np.int64)
    bounds_per_req = []
    for b in range(B):
        nt = int(tiles[b])
        ns = max(1, min(nt, int(math.ceil(wbytes[b] / target))))
        if max_splits is not None:
            ns = min(ns, max_splits)
        npg = int(n_pages[b])
        w2 = npg * page_stride
        cuts = [0]
        for k in range(1, ns):
            pos = wbytes[b] * k / ns
            if pos <= w2:
                t = int(round(pos / page_stride))
            else:
                t = npg + int(round((pos - w2) / tile4))
            t = min(max(t, cuts[-1] + 1), nt - (ns - k))
            cuts.append(t)
        cuts.append(nt)
        bounds_per_req.append(cuts)
    part = 0
    for b in range(B):
        cuts = bounds_per_req[b]
        for h in range(n_kv_heads):
            u = b * n_kv_heads + h
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                rows.append((u, lo, hi, part))
                part += 1
            part_counts[u] = len(cuts) - 1
    work = np.asarray(rows, dtype=np.int32).reshape(-1, 4)
    part_indptr = np.concatenate([[0], np.cumsum(part_counts)]).astype(np.int32)
    return work, part_indptr, part
