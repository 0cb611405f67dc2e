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
                n_sm: int = NUM_SMS_B200, ctas_per_sm: int = 3, waves: float = 1.0,
                splits: int | None = None, max_splits: int = 8):
    """Return (work int32 [B*Hkv*S, 4], S).

    Every (request, kv head) unit gets the same number S of splits (1..8) so the S CTAs of
    a unit can run as one thread-block cluster and merge through distributed shared
    memory.  S is chosen so the launch is about ``waves`` waves of ``ctas_per_sm`` CTAs on
    every SM; each unit's tiles (INT2 pages first, then 32-slot INT4 tiles) are cut into S
    contiguous ranges of about equal bytes (a range may be empty for very short requests).
    Rows are (unit = b*Hkv + kvh, tile_lo, tile_hi, 0).
    """
    n_pages = np.asarray(n_pages, dtype=np.int64)
    n_int4 = np.asarray(n_int4, dtype=np.int64)
    B = n_pages.size
    tiles = n_pages + (n_int4 + 31) // 32
    if np.any(tiles <= 0):
        raise ValueError("every request needs at least one cached token")
    units = B * n_kv_heads
    if splits is None:
        splits = int(round(n_sm * ctas_per_sm * waves / units))
    S = int(min(max(splits, 1), max_splits))
    tile4 = 32 * slot_stride
    wbytes = n_pages * page_stride + n_int4 * slot_stride
    rows = np.zeros((B, n_kv_heads, S, 4), dtype=np.int32)
    for b in range(B):
        npg, nt = int(n_pages[b]), int(tiles[b])
        w2 = npg * page_stride
        cuts = [0]
        for k in range(1, S):
            pos = wbytes[b] * k / S
            t = int(round(pos / page_stride)) if pos <= w2 else npg + int(round((pos - w2) / tile4))
            cuts.append(min(max(t, cuts[-1]), nt))
        cuts.append(nt)
        rows[b, :, :, 1] = cuts[:-1]
        rows[b, :, :, 2] = cuts[1:]
    rows[:, :, :, 0] = (np.arange(B)[:, None, None] * n_kv_heads + np.arange(n_kv_heads)[None, :, None])
    return rows.reshape(-1, 4), S
