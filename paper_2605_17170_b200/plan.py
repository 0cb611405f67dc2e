"""Stream-K work planner for the decode kernel (host side, vectorised numpy).

The reference splits each request's partitioned table into contiguous
bitwidth-homogeneous chunks of ``split_len`` entries (attention.py:205-208) and merges
the per-split partials (attention.py:154-165).  On the GPU the unit of work is a tile --
one INT2 page (32 tokens, page_stride bytes) or up to 32 INT4 slots (slot_stride bytes
each) -- so every tile is bitwidth-homogeneous too.  All (request, kv head) units' tiles
are laid end to end and cut into ``n_cta`` contiguous ranges of equal bytes, one per
resident CTA (148 SMs x CTAs per SM): every SM streams the same number of bytes whatever
the mix of request lengths.  Where a cut falls inside a unit, that unit's pieces write
partials and the last CTA to finish merges them (the fused K3).
"""

from __future__ import annotations

import numpy as np

NUM_SMS_B200 = 148


def _tile_bytes(n_pages: int, n_int4: int, page_stride: int, slot_stride: int, int4_weight: float) -> np.ndarray:
    n4t = -(-n_int4 // 32)
    tb = np.empty(n_pages + n4t, dtype=np.float64)
    tb[:n_pages] = page_stride
    if n4t:
        nv = np.full(n4t, 32, dtype=np.int64)
        nv[-1] = n_int4 - 32 * (n4t - 1)
        tb[n_pages:] = nv * slot_stride * int4_weight
    return tb


def plan_stream(n_pages, n_int4, n_kv_heads: int, page_stride: int, slot_stride: int,
                n_cta: int = 3 * NUM_SMS_B200, int4_weight: float = 0.8, tier_skew: float = 0.0,
                n_sm: int = NUM_SMS_B200):
    """Return (work int32 [n_pieces, 8], cta_ptr int32 [n_cta + 1], n_parts).

    work rows: (unit = b*Hkv + kvh, tile_lo, tile_hi, slot, part0, nparts, 0, 0); slot is
    -1 when the piece covers its whole unit, else the partial slot (a split unit's pieces
    use slots part0 .. part0 + nparts - 1).  CTA i runs pieces cta_ptr[i] .. cta_ptr[i+1]
    in order; a CTA may hold pieces of several short units, or none.

    tier_skew: CTAs i*n_sm .. (i+1)*n_sm - 1 form residency tier i (the block scheduler puts
    tier i as the (i+1)-th CTA on every SM, and the warp schedulers favour older CTAs, so
    lower tiers run faster, measured with tools/cta_order.py).  Tier i's cost share is
    scaled by 1 + tier_skew * (1 - 2 i / (tiers - 1)): lower tiers get more work.
    """
    n_pages = np.asarray(n_pages, dtype=np.int64)
    n_int4 = np.asarray(n_int4, dtype=np.int64)
    B = n_pages.size
    tiles = n_pages + (n_int4 + 31) // 32
    if B == 0 or np.any(tiles <= 0):
        raise ValueError("every request needs at least one cached token")
    H = int(n_kv_heads)
    per_req = [_tile_bytes(int(n_pages[b]), int(n_int4[b]), page_stride, slot_stride, int4_weight)
               for b in range(B)]
    unit_tiles = np.repeat(tiles, H)  # unit-major: u = b*H + h
    ustart = np.zeros(B * H + 1, dtype=np.int64)
    np.cumsum(unit_tiles, out=ustart[1:])
    total_tiles = int(ustart[-1])
    cum = np.cumsum(np.concatenate([np.tile(t, H) for t in per_req]))
    n_cta = int(max(1, min(n_cta, total_tiles)))
    tiers = -(-n_cta // max(1, int(n_sm)))
    tier = np.arange(n_cta) // max(1, int(n_sm))
    w = 1.0 + (tier_skew * (1.0 - 2.0 * tier / (tiers - 1)) if tiers > 1 else np.zeros(n_cta))
    target = cum[-1] * np.cumsum(w)[:-1] / w.sum()
    idx = np.searchsorted(cum, target, side="left")  # cum[idx] >= target
    prev = np.where(idx > 0, cum[np.maximum(idx - 1, 0)], 0.0)
    cuts = np.where(cum[idx] - target < target - prev, idx + 1, idx)  # nearest tile boundary
    cuts = np.maximum.accumulate(np.concatenate([[0], cuts, [total_tiles]])).astype(np.int64)
    bounds = np.union1d(cuts, ustart)
    lo, hi = bounds[:-1], bounds[1:]
    unit = np.searchsorted(ustart, lo, side="right") - 1
    cta = np.searchsorted(cuts, lo, side="right") - 1
    cta = np.minimum(cta, n_cta - 1)
    npieces = np.bincount(unit, minlength=B * H)
    first = np.searchsorted(unit, np.arange(B * H), side="left")
    split = npieces > 1
    part0 = np.zeros(B * H, dtype=np.int64)
    part0[split] = np.concatenate([[0], np.cumsum(npieces[split])[:-1]])
    n_parts = int(npieces[split].sum())
    rank = np.arange(lo.size) - first[unit]
    work = np.zeros((lo.size, 8), dtype=np.int32)
    work[:, 0] = unit
    work[:, 1] = lo - ustart[unit]
    work[:, 2] = hi - ustart[unit]
    work[:, 3] = np.where(split[unit], part0[unit] + rank, -1)
    work[:, 4] = np.where(split[unit], part0[unit], 0)
    work[:, 5] = npieces[unit]
    cta_ptr = np.zeros(n_cta + 1, dtype=np.int32)
    np.cumsum(np.bincount(cta, minlength=n_cta), out=cta_ptr[1:])
    return work, cta_ptr, n_parts
