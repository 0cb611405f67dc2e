"""Calibration replay on the GPU.

The reference calibrates its per-tag sensitivity table by replaying attention with one
tag's rows quantized at a time (``calibration.py:108-125`` ``measure_raw``):
``attention_selective_quant`` (``attention.py:130-142``) fake-quantizes the target tag's
rows (``apply_mixed_quantization``, ``attention.py:103-127``), runs dense causal
attention (``attention_full``, ``attention.py:32-64``) and records the per-head output MSE
against the unquantized run (``output_mse_per_head``, ``attention.py:77-83``).  On the
CPU this is O(tags x bitwidths x layers x N^2) numpy work.

Here the fake quantization is the pool round trip itself -- the selected rows go through
K1 (``kvmix_write_prefill``) into a scratch pool and come back through K5
(``kvmix_gather_dequant``), which reproduces the reference's quantize-dequantize images
bit for bit (same routing: INT2 rows in sequence order form pages, the residual INT2 rows
and the INT4 rows go per token at INT4) -- and the dense attention is one fused fp32 kernel (csrc/calib.cu,
``kvmix_attention_full``), with the MSE reduced in float64 like the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import ValidationError
from .pool import MixedPrecisionPool, PoolConfig
from .quant import GROUP_SIZE

BITWIDTHS = (2, 4)


def _dev(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def apply_mixed_quantization(k, v, row_bits, group_len: int = GROUP_SIZE, device=None):
    """attention.py:103-127 on the device: K/V rows [N, Hkv, d] (or [L, N, Hkv, d], the same
    row bits for every layer) replaced by their quantize-dequantize images where row_bits is
    2 or 4; rows with 0 stay full precision.  Returns fp32 device tensors."""
    dev = _dev(device)
    k = torch.as_tensor(np.asarray(k, dtype=np.float32) if not torch.is_tensor(k) else k).to(dev, torch.float32)
    v = torch.as_tensor(np.asarray(v, dtype=np.float32) if not torch.is_tensor(v) else v).to(dev, torch.float32)
    layered = k.dim() == 4
    if not layered:
        k, v = k[None], v[None]
    if k.dim() != 4 or k.shape != v.shape:
        raise ValidationError("K/V must be [N, Hkv, d] (or [L, N, Hkv, d]) with matching shapes")
    bits = np.asarray(row_bits)
    if bits.shape != (k.shape[1],):
        raise ValidationError("row_bits length must match the token dimension")
    if not np.all(np.isin(bits, (0, 2, 4))):
        raise ValidationError("row bitwidths must be 0, 2, or 4")
    kq, vq = k.clone(), v.clone()
    sel = np.flatnonzero(bits != 0)
    if sel.size:
        sub = bits[sel]
        L, _, H, d = k.shape
        n_full = int((sub == 2).sum()) // group_len * group_len
        cfg = PoolConfig(total_slots=int(sel.size), offset=n_full, n_layers=L, n_kv_heads=H, head_dim=d,
                         page_size=group_len)
        pool = MixedPrecisionPool(cfg, device=dev)
        table = pool.alloc("replay", sub)
        idx = torch.as_tensor(sel, device=dev)
        pool.write_prefill(table, k.index_select(1, idx).contiguous(), v.index_select(1, idx).contiguous())
        for layer in range(L):
            kd, vd = pool._gather_dev(table.slots, layer)
            kq[layer, idx] = kd
            vq[layer, idx] = vd
    return (kq, vq) if layered else (kq[0], vq[0])


def attention_full(q, k, v, scale=None, causal: bool = False):
    """attention.py:32-64 on the device, fp32: q [n_q, H, d], k / v [N, Hkv, d] -> [n_q, H, d].
    With ``causal`` the queries are aligned to the last n_q key positions.  One fused launch
    (``kvmix_attention_full``, csrc/calib.cu: flash-style fp32 tiles, online softmax)."""
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3 or k.shape != v.shape:
        raise ValidationError("Q/K/V must be rank-3 with matching K/V shapes")
    if q.shape[2] != k.shape[2]:
        raise ValidationError("Q and K head dims differ")
    n_q, H, d = q.shape
    n = k.shape[0]
    if H % k.shape[1]:
        raise ValidationError("query heads must be a multiple of kv heads")
    if causal and n_q > n:
        raise ValidationError("causal attention needs n_q <= N")
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))
    dev = q.device
    q, k, v = (x.to(dev, torch.float32).contiguous() for x in (q, k, v))
    dk = next((s for s in (32, 64, 128, 256) if s >= d), None)  # kernel head dims; zero channels change nothing
    if dk is None:
        raise ValidationError("head_dim above 256 is not supported on the device")
    if dk != d:
        q, k, v = (torch.nn.functional.pad(x, (0, dk - d)).contiguous() for x in (q, k, v))
    out = torch.empty((n_q, H, dk), dtype=torch.float32, device=dev)
    _lib.check(lib.kvmix_attention_full(q.data_ptr(), k.data_ptr(), v.data_ptr(), n_q, n, H, k.shape[1], dk,
                                        float(np.float32(scale)), int(bool(causal)), out.data_ptr(), _lib.stream()))
    return out if dk == d else out[..., :d].contiguous()


def output_mse_per_head(o_ref, o_test) -> np.ndarray:
    """attention.py:77-83: per-head mean over positions of the squared L2 error (float64)."""
    if o_ref.shape != o_test.shape:
        raise ValidationError("output shapes differ")
    return ((o_ref.double() - o_test.double()) ** 2).sum(dim=-1).mean(dim=0).cpu().numpy()


def measure_raw(captures, bitwidths=BITWIDTHS, device=None) -> dict:
    """calibration.py:108-125 on the device.  ``captures`` are the reference's KVCapture
    objects (or anything with ``request_id``, ``tags``, ``group_len`` and ``layers`` of
    ``q [n, H, d]``, ``k`` / ``v [n, Hkv, d]``).  Returns the raw distortion entries
    {(layer, request_id, head, tag, bitwidth): mse}, the ``entries`` of the reference's
    RawDistortion."""
    dev = _dev(device)
    entries = {}
    for cap in captures:
        if hasattr(cap, "validate"):
            cap.validate()
        tags = np.asarray(cap.tags)
        active = sorted(set(int(t) for t in tags))
        qs = [torch.as_tensor(np.asarray(lay.q, dtype=np.float32), device=dev) for lay in cap.layers]
        ks = torch.stack([torch.as_tensor(np.asarray(lay.k, dtype=np.float32), device=dev) for lay in cap.layers])
        vs = torch.stack([torch.as_tensor(np.asarray(lay.v, dtype=np.float32), device=dev) for lay in cap.layers])
        refs = [attention_full(qs[li], ks[li], vs[li], causal=True) for li in range(len(qs))]
        g = int(getattr(cap, "group_len", GROUP_SIZE))
        for tag in active:
            for b in bitwidths:
                bits = np.where(tags == tag, int(b), 0)
                kq, vq = apply_mixed_quantization(ks, vs, bits, group_len=g, device=dev)
                for li in range(len(qs)):
                    mse = output_mse_per_head(refs[li], attention_full(qs[li], kq[li], vq[li], causal=True))
                    for h, e in enumerate(mse):
                        entries[(li, cap.request_id, h, tag, int(b))] = float(e)
    return entries
