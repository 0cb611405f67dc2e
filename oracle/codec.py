"""Oracle (test infrastructure only): numpy restatement of the reference codec.

Follows /root/reference/pkg/src/kvmix/quant.py and the wire format pinned in
/root/reference/pkg/LAYOUT.md.  Everything here is vectorised over leading
"block" axes (the reference encodes one block per call); the arithmetic per
group is the reference's, op for op, in float32:

  zero  = f16(min)                                   quant.py:39
  scale = f16((max - min) / (2^b - 1))  (raw min)    quant.py:40
  code  = clip(round_half_away((x - zero) / scale), 0, 2^b - 1) if scale > 0
          else 0                                     quant.py:44-50
  x'    = code * scale + zero                        quant.py:90-93, 186, 252

Pinned against LAYOUT.md's worked examples, the pack KATs and golden vectors
produced by the real reference (tests/test_oracle_pinned.py).
"""

from __future__ import annotations

import numpy as np

GROUP_SIZE = 32  # quant.py:23
PARAM_BYTES = 2  # quant.py:24


def f16_round(x) -> np.ndarray:
    """fp32 -> fp16 (RNE) -> fp32.  quant.py:27-29 (_narrow16)."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def round_half_away(x) -> np.ndarray:
    """copysign(floor(|x| + 0.5), x) in fp32.  quant.py:32-33."""
    x = np.asarray(x, dtype=np.float32)
    return np.copysign(np.floor(np.abs(x) + np.float32(0.5)), x)


def group_params(mn, mx, bits: int):
    """Narrowed (scale, zero); scale from the UN-narrowed min.  quant.py:36-41."""
    levels = np.float32((1 << bits) - 1)
    mn = np.asarray(mn, dtype=np.float32)
    mx = np.asarray(mx, dtype=np.float32)
    zero = f16_round(mn)
    scale = f16_round((mx - mn) / levels)
    return scale, zero


def quantize(x, scale, zero, bits: int) -> np.ndarray:
    """Codes against broadcastable narrowed params.  quant.py:44-50."""
    levels = (1 << bits) - 1
    x = np.asarray(x, dtype=np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (x - zero) / scale
    r = np.where(scale > 0, round_half_away(t), np.float32(0.0))
    return np.clip(r, 0, levels).astype(np.uint8)


def dequantize(codes, scale, zero) -> np.ndarray:
    """code * scale + zero in fp32.  quant.py:90-93."""
    return codes.astype(np.float32) * scale + zero


def pack(codes, bits: int) -> np.ndarray:
    """Sub-byte LE packing along the last axis (code i -> bits [i*b mod 8, +b) of
    byte i*b//8), zero-padded to whole bytes.  quant.py:96-109, LAYOUT.md:14-16."""
    codes = np.asarray(codes)
    per = 8 // bits
    n = codes.shape[-1]
    nb = -(-n // per)
    padded = np.zeros(codes.shape[:-1] + (nb * per,), dtype=np.uint32)
    padded[..., :n] = codes
    padded = padded.reshape(codes.shape[:-1] + (nb, per))
    shifts = (bits * np.arange(per, dtype=np.uint32))
    return (padded << shifts).sum(axis=-1).astype(np.uint8)


def unpack(data, bits: int, n: int) -> np.ndarray:
    """Inverse of pack along the last axis.  quant.py:112-120."""
    data = np.asarray(data, dtype=np.uint8)
    per = 8 // bits
    shifts = (bits * np.arange(per, dtype=np.uint8))
    codes = (data[..., None] >> shifts) & np.uint8((1 << bits) - 1)
    return codes.reshape(data.shape[:-1] + (-1,))[..., :n].astype(np.uint8)


def params_bytes(scale, zero) -> np.ndarray:
    """Interleaved (scale, zero) little-endian fp16 pairs along the last axis."""
    pairs = np.stack([np.asarray(scale), np.asarray(zero)], axis=-1).astype("<f2")
    return pairs.reshape(pairs.shape[:-2] + (-1,)).view(np.uint8)


def parse_params(raw) -> tuple[np.ndarray, np.ndarray]:
    raw = np.ascontiguousarray(np.asarray(raw, dtype=np.uint8))
    f = raw.view("<f2").astype(np.float32)
    return f[..., 0::2], f[..., 1::2]


def key_page_nbytes(d: int, g: int = GROUP_SIZE) -> int:
    """quant.py:123-124."""
    return d * g * 2 // 8 + d * 2 * PARAM_BYTES


def token_block_nbytes(d: int, bits: int, g: int = GROUP_SIZE) -> int:
    """quant.py:127-128."""
    return d * bits // 8 + (d // g) * 2 * PARAM_BYTES


def encode_key_pages(keys, g: int = GROUP_SIZE) -> np.ndarray:
    """KeyPageBlock payloads for keys[..., G, d] -> uint8[..., d*G/4 + 4d].

    Per-channel INT2 over the page's G token rows; channel-major codes (channel c
    at bytes [c*G/4, (c+1)*G/4)), then d (scale_c, zero_c) pairs.
    quant.py:160-177, LAYOUT.md:38-52.
    """
    keys = np.asarray(keys, dtype=np.float32)
    assert keys.shape[-2] == g
    scale, zero = group_params(keys.min(axis=-2), keys.max(axis=-2), 2)  # [..., d]
    codes = quantize(keys, scale[..., None, :], zero[..., None, :], 2)  # [..., G, d]
    chan_major = np.swapaxes(codes, -1, -2)  # [..., d, G]
    packed = pack(chan_major, 2).reshape(keys.shape[:-2] + (-1,))
    return np.concatenate([packed, params_bytes(scale, zero)], axis=-1)


def decode_key_pages(blocks, d: int, g: int = GROUP_SIZE) -> np.ndarray:
    """uint8[..., nbytes] -> fp32 [..., G, d].  quant.py:180-186."""
    blocks = np.asarray(blocks, dtype=np.uint8)
    cb = d * g * 2 // 8
    codes = unpack(blocks[..., :cb].reshape(blocks.shape[:-1] + (d, g * 2 // 8)), 2, g)
    scale, zero = parse_params(blocks[..., cb:])
    vals = codes.astype(np.float32) * scale[..., :, None] + zero[..., :, None]
    return np.swapaxes(vals, -1, -2)


def encode_token_blocks(x, bits: int, g: int = GROUP_SIZE) -> np.ndarray:
    """TokenBlock payloads for x[..., d] -> uint8[..., d*b/8 + 4d/G].

    d/G groups of G consecutive channels; codes in channel order then the group
    (scale, zero) pairs.  quant.py:189-232, LAYOUT.md:67-80.
    """
    x = np.asarray(x, dtype=np.float32)
    d = x.shape[-1]
    assert d % g == 0
    grp = x.reshape(x.shape[:-1] + (d // g, g))
    scale, zero = group_params(grp.min(axis=-1), grp.max(axis=-1), bits)
    codes = quantize(grp, scale[..., None], zero[..., None], bits).reshape(x.shape)
    return np.concatenate([pack(codes, bits), params_bytes(scale, zero)], axis=-1)


def decode_token_blocks(blocks, d: int, bits: int, g: int = GROUP_SIZE) -> np.ndarray:
    """uint8[..., nbytes] -> fp32 [..., d].  quant.py:235-262."""
    blocks = np.asarray(blocks, dtype=np.uint8)
    cb = d * bits // 8
    codes = unpack(blocks[..., :cb], bits, d).reshape(blocks.shape[:-1] + (d // g, g))
    scale, zero = parse_params(blocks[..., cb:])
    vals = codes.astype(np.float32) * scale[..., None] + zero[..., None]
    return vals.reshape(blocks.shape[:-1] + (d,))


def quantize_group(values, bits: int):
    """Single-group quantizer (codes, scale, zero).  quant.py:64-87."""
    values = np.asarray(values, dtype=np.float32)
    scale, zero = group_params(values.min(), values.max(), bits)
    return quantize(values, scale, zero, bits), float(scale), float(zero)


def fake_quant_kv(k, v, bits_per_token, g: int = GROUP_SIZE):
    """Quantize-dequantize K/V rows [N, Hkv, d] as the pool would store them.

    Full pages of INT2 rows (token order) get per-channel INT2 keys and per-token
    INT2 values; residual INT2 rows and INT4 rows go per-token INT4.
    Restates attention.py:86-127 (apply_mixed_quantization) with rows 2/4 only.
    """
    k = np.array(k, dtype=np.float32)
    v = np.array(v, dtype=np.float32)
    bits = np.asarray(bits_per_token)
    idx2 = np.flatnonzero(bits == 2)
    full = idx2.size // g * g
    if full:
        pages = idx2[:full].reshape(-1, g)  # [P, G]
        kp = np.swapaxes(k[pages], 1, 2)  # [P, Hkv, G, d]
        sc, ze = group_params(kp.min(axis=2), kp.max(axis=2), 2)
        kq = dequantize(quantize(kp, sc[:, :, None, :], ze[:, :, None, :], 2),
                        sc[:, :, None, :], ze[:, :, None, :])
        k[pages] = np.swapaxes(kq, 1, 2)
        v[pages] = _fake_tok(v[pages], 2, g)
    rest = np.sort(np.concatenate([np.flatnonzero(bits == 4), idx2[full:]]))
    if rest.size:
        k[rest] = _fake_tok(k[rest], 4, g)
        v[rest] = _fake_tok(v[rest], 4, g)
    return k, v


def _fake_tok(x, bits, g):
    shp = x.shape
    grp = x.reshape(shp[:-1] + (shp[-1] // g, g))
    sc, ze = group_params(grp.min(-1), grp.max(-1), bits)
    return dequantize(quantize(grp, sc[..., None], ze[..., None], bits),
                      sc[..., None], ze[..., None]).reshape(shp)
