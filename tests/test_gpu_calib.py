"""Calibration replay on the GPU: the pool round trip (K1 -> K5)
reproduces the reference's fake quantization bit for bit, and the per-(layer, head, tag,
bitwidth) output MSEs match the oracle's restatement of calibration.py:108-125."""
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from paper_2605_17170_b200 import calib
from paper_2605_17170_b200.errors import ValidationError

pytestmark = pytest.mark.gpu


def _capture(seed, n, n_layers, H, Hkv, d, n_tags):
    rng = np.random.default_rng(seed)
    ch = np.exp(rng.uniform(np.log(0.5), np.log(4.0), (Hkv, d))).astype(np.float32)
    layers = [SimpleNamespace(q=rng.standard_normal((n, H, d)).astype(np.float32),
                              k=(rng.standard_normal((n, Hkv, d)) * ch).astype(np.float32),
                              v=rng.standard_normal((n, Hkv, d)).astype(np.float32)) for _ in range(n_layers)]
    return SimpleNamespace(request_id=f"c{seed}", layers=layers, tags=rng.integers(0, n_tags, n), group_len=32)


@pytest.mark.parametrize("d", [64, 128])
def test_fake_quant_bit_exact(cuda, d):
    cap = _capture(d, 700, 1, 8, 2, d, 5)
    k, v = cap.layers[0].k, cap.layers[0].v
    for bits in (np.where(cap.tags == 1, 2, np.where(cap.tags == 3, 4, 0)),
                 np.where(cap.tags < 3, 2, 0), np.zeros(700, int), np.full(700, 4)):
        kd, vd = calib.apply_mixed_quantization(k, v, bits)
        ko, vo = oatt.apply_mixed_quantization(k, v, bits)
        assert np.array_equal(kd.cpu().numpy(), ko) and np.array_equal(vd.cpu().numpy(), vo)


def test_attention_full_matches_oracle(cuda):
    cap = _capture(5, 300, 1, 8, 2, 64, 3)
    lay = cap.layers[0]
    got = calib.attention_full(*(torch.as_tensor(x, device=cuda) for x in (lay.q[:200], lay.k, lay.v)), causal=True)
    ref = oatt.attention_full(lay.q[:200], lay.k, lay.v, causal=True)
    assert np.allclose(got.cpu().numpy(), ref, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("d,H,Hkv,nq,nk,causal", [(32, 4, 4, 33, 33, True), (64, 8, 2, 200, 300, True),
                                                   (128, 16, 2, 1024, 1024, True), (128, 8, 1, 17, 517, False),
                                                   (64, 6, 3, 1, 95, True), (16, 2, 1, 10, 10, False),
                                                   (256, 4, 2, 70, 70, True), (80, 4, 4, 40, 64, True)])
def test_attention_kernel_vs_float64(cuda, d, H, Hkv, nq, nk, causal):
    """The fused replay attention (csrc/calib.cu) against a float64 dense attention: ragged
    tiles, GQA, causal and not, one query; fp32 accuracy."""
    rng = np.random.default_rng(d + nq)
    q = rng.standard_normal((nq, H, d)).astype(np.float32) * 2
    k = rng.standard_normal((nk, Hkv, d)).astype(np.float32)
    v = rng.standard_normal((nk, Hkv, d)).astype(np.float32)
    got = calib.attention_full(*(torch.as_tensor(x, device=cuda) for x in (q, k, v)), causal=causal).cpu().numpy()
    r = H // Hkv
    kk = np.repeat(k.astype(np.float64), r, axis=1)
    vv = np.repeat(v.astype(np.float64), r, axis=1)
    logits = np.einsum("qhd,nhd->hqn", q.astype(np.float64), kk) / np.sqrt(d)
    if causal:
        mask = np.arange(nk)[None, :] > (nk - nq + np.arange(nq))[:, None]
        logits[:, mask] = -np.inf
    w = np.exp(logits - logits.max(-1, keepdims=True))
    ref = np.einsum("hqn,nhd->qhd", w / w.sum(-1, keepdims=True), vv)
    assert np.abs(got - ref).max() <= 2e-5 * max(1.0, np.abs(ref).max())


def test_measure_raw_matches_oracle(cuda):
    caps = [_capture(s, n, 2, 8, 2, 64, 4) for s, n in ((21, 260), (22, 333))]
    got = calib.measure_raw(caps)
    ref = oatt.measure_raw(caps)
    assert got.keys() == ref.keys()
    for key, e in ref.items():
        assert abs(got[key] - e) <= 2e-3 * abs(e) + 1e-7, (key, got[key], e)


def test_validation(cuda):
    k = np.zeros((40, 2, 64), np.float32)
    with pytest.raises(ValidationError):
        calib.apply_mixed_quantization(k, k, np.full(39, 2))
    with pytest.raises(ValidationError):
        calib.apply_mixed_quantization(k, k, np.full(40, 3))
