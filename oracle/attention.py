"""Oracle (test infrastructure only): restatement of the reference decode path.

``flash_decode`` follows /root/reference/pkg/src/kvmix/attention.py:175-218:
bitwidth-homogeneous contiguous splits of ``split_len`` table entries (INT2 range
then INT4 range, :205-208), each split gathered/dequantised and reduced per
q-head to a (acc, lse, max) partial (:168-172), partials merged by log-sum-exp
(:154-165), GQA kv = h // (H / Hkv) (:198-201, :216).  All float32 like the
reference.  ``dense_f64`` is the float64 dense oracle of the reference tests
(tests/conftest.py:14-36, tests/test_acceptance.py:58-71).
"""

from __future__ import annotations

import numpy as np


def split_partial(q_head, k_rows, v_rows, scale):
    """attention.py:168-172 -> (acc[d], lse, max)."""
    logits = (k_rows @ q_head) * np.float32(scale)
    mx = float(logits.max())
    w = np.exp(logits - np.float32(mx))
    return w @ v_rows, mx + float(np.log(w.sum())), mx


def merge(parts):
    """attention.py:154-165."""
    m = max(p[2] for p in parts)
    acc = np.zeros_like(parts[0][0], dtype=np.float32)
    z = np.float32(0.0)
    for a, lse, mx in parts:
        acc += a * np.float32(np.exp(mx - m))
        z += np.float32(np.exp(lse - m))
    return acc / z


def flash_decode(q, k_rows, v_rows, n_int2: int, split_len: int = 128, scale=None):
    """Decode over a partitioned table whose gathered K/V are k_rows/v_rows [m, Hkv, d]
    (INT2 entries first, ``n_int2`` of them).  attention.py:175-218."""
    q = np.asarray(q, dtype=np.float32)
    H, d = q.shape
    m = k_rows.shape[0]
    ratio = H // k_rows.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    splits = []
    for lo, hi in ((0, n_int2), (n_int2, m)):
        for s in range(lo, hi, split_len):
            splits.append((s, min(s + split_len, hi)))
    parts = [[] for _ in range(H)]
    for lo, hi in splits:
        if hi <= lo:
            continue
        for h in range(H):
            kv = h // ratio
            parts[h].append(split_partial(q[h], k_rows[lo:hi, kv], v_rows[lo:hi, kv], scale))
    return np.stack([merge(p) for p in parts])


def flash_decode_pool(q, opool, rid: str, layer: int, split_len: int = 128, scale=None):
    """flash_decode over an oracle pool's partitioned table for one request/layer."""
    slots = opool.tables[rid]
    k, v = opool.gather(slots, layer)
    n2 = sum(1 for s in slots if opool.is_int2(s))
    return flash_decode(q, k, v, n2, split_len, scale)


def dense_f64(q, k, v, scale=None):
    """Float64 dense GQA attention; q [n_q, H, d], k/v [N, Hkv, d]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    ratio = q.shape[1] // k.shape[1]
    k = np.repeat(k, ratio, axis=1)
    v = np.repeat(v, ratio, axis=1)
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[2])
    logits = np.einsum("qhd,nhd->hqn", q, k) * scale
    logits -= logits.max(axis=2, keepdims=True)
    w = np.exp(logits)
    w /= w.sum(axis=2, keepdims=True)
    return np.einsum("hqn,nhd->qhd", w, v)


def attention_full(q, k, v, scale=None, causal: bool = False):
    """attention.py:32-64 restated: fp32 dense GQA attention, q [n_q, H, d], k/v [N, Hkv, d];
    with ``causal`` the queries are aligned to the last n_q keys."""
    q = np.asarray(q, dtype=np.float32)
    k = np.asarray(k, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    n_q, H, d = q.shape
    n = k.shape[0]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    ratio = H // k.shape[1]
    ke = np.repeat(k, ratio, axis=1)
    ve = np.repeat(v, ratio, axis=1)
    logits = np.einsum("qhd,nhd->hqn", q, ke) * np.float32(scale)
    if causal:
        mask = np.arange(n)[None, :] > ((n - n_q) + np.arange(n_q))[:, None]
        logits = np.where(mask[None], -np.inf, logits)
    logits = logits - logits.max(axis=2, keepdims=True)
    w = np.exp(logits)
    p = w / w.sum(axis=2, keepdims=True)
    return np.einsum("hqn,nhd->qhd", p, ve)


def output_mse_per_head(o_ref, o_test):
    """attention.py:77-83: per-head mean over positions of the squared L2 error (float64)."""
    o_ref = np.asarray(o_ref, dtype=np.float64)
    o_test = np.asarray(o_test, dtype=np.float64)
    return ((o_ref - o_test) ** 2).sum(axis=-1).mean(axis=0)


def apply_mixed_quantization(k, v, row_bits, g: int = 32):
    """attention.py:103-127: rows with bits 2 / 4 replaced by their quantize-dequantize
    images (the pool's routing over the selected rows, codec.fake_quant_kv); 0 = untouched."""
    from .codec import fake_quant_kv
    k = np.array(k, dtype=np.float32)
    v = np.array(v, dtype=np.float32)
    bits = np.asarray(row_bits)
    sel = np.flatnonzero(bits != 0)
    if sel.size:
        kq, vq = fake_quant_kv(k[sel], v[sel], bits[sel], g)
        k[sel], v[sel] = kq, vq
    return k, v


def measure_raw(captures, bitwidths=(2, 4)):
    """calibration.py:108-125 restated over the functions above."""
    entries = {}
    for cap in captures:
        tags = np.asarray(cap.tags)
        for li, lay in enumerate(cap.layers):
            ref = attention_full(lay.q, lay.k, lay.v, causal=True)
            for tag in sorted(set(int(t) for t in tags)):
                for b in bitwidths:
                    kq, vq = apply_mixed_quantization(lay.k, lay.v, np.where(tags == tag, b, 0), cap.group_len)
                    mse = output_mse_per_head(ref, attention_full(lay.q, kq, vq, causal=True))
                    for h, e in enumerate(mse):
                        entries[(li, cap.request_id, h, tag, b)] = float(e)
    return entries
