"""Asymmetric groupwise INT2/INT4 codec -- reference-compatible API on sm_100a kernels.

Drop-in for /root/reference/pkg/src/kvmix/quant.py: same names, signatures,
payload bytes (LAYOUT.md) and error behaviour.  Every encode/decode runs on the
GPU through libkvmix_b200 (include/kvmix_b200.h); there is no CPU path.  The
single-block functions move their (tiny) inputs to the device; the batched
``encode_*_device`` functions work on device tensors and are what the pool uses.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .errors import ValidationError

GROUP_SIZE = 32  # quant.py:23
PARAM_BYTES = 2  # quant.py:24


@dataclass
class QuantGroup:
    """One quantization group (quant.py:53-61)."""

    codes: np.ndarray
    scale: float
    zero_offset: float
    bitwidth: int
    group_len: int


@dataclass
class KeyPageBlock:
    """Packed per-channel INT2 keys for one (page, head) (quant.py:131-142)."""

    payload: bytes
    head_dim: int
    group_len: int = GROUP_SIZE


@dataclass
class TokenBlock:
    """Packed per-token codes for one (token, head) (quant.py:145-157)."""

    payload: bytes
    head_dim: int
    bitwidth: int
    group_len: int = GROUP_SIZE


def key_page_payload_bytes(head_dim: int, group_len: int = GROUP_SIZE) -> int:
    """quant.py:123-124."""
    return head_dim * group_len * 2 // 8 + head_dim * 2 * PARAM_BYTES


def token_block_payload_bytes(head_dim: int, bitwidth: int, group_len: int = GROUP_SIZE) -> int:
    """quant.py:127-128."""
    return head_dim * bitwidth // 8 + (head_dim // group_len) * 2 * PARAM_BYTES


# ---- device helpers ---------------------------------------------------------------
def _dev(x, dtype=torch.float32) -> torch.Tensor:
    dev = _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.float32 if dtype == torch.float32 else None),
                           device=dev).to(dtype).contiguous()


class _ErrFlag:
    """Device error word written by the kernels (bit0 non-finite, bit1 code range)."""

    def __init__(self):
        self.t = torch.zeros(1, dtype=torch.int32, device=_lib.require_cuda())

    def value(self) -> int:
        return int(self.t.item())


def _check_group_len(group_len: int) -> None:
    if group_len != GROUP_SIZE:
        raise ValidationError(f"group_len {group_len} unsupported on device (only {GROUP_SIZE})")


def encode_key_pages_device(keys: torch.Tensor, err: torch.Tensor | None = None) -> torch.Tensor:
    """Batched K1a: keys f32 [P, 32, d] (device) -> uint8 [P, key_page_payload_bytes(d)]."""
    P, g, d = keys.shape
    out = torch.empty((P, key_page_payload_bytes(d)), dtype=torch.uint8, device=keys.device)
    _lib.check(lib.kvmix_encode_key_pages(keys.data_ptr(), P, d, out.data_ptr(), out.shape[1],
                                          _lib.ptr(err), _lib.stream()))
    return out


def encode_token_blocks_device(x: torch.Tensor, bitwidth: int, err: torch.Tensor | None = None) -> torch.Tensor:
    """Batched K1b/K1c: x f32 [n, d] (device) -> uint8 [n, token_block_payload_bytes(d, b)]."""
    n, d = x.shape
    out = torch.empty((n, token_block_payload_bytes(d, bitwidth)), dtype=torch.uint8, device=x.device)
    _lib.check(lib.kvmix_encode_token_blocks(x.data_ptr(), n, d, bitwidth, out.data_ptr(), out.shape[1],
                                             _lib.ptr(err), _lib.stream()))
    return out


def decode_key_pages_device(blocks: torch.Tensor, head_dim: int) -> torch.Tensor:
    P = blocks.shape[0]
    out = torch.empty((P, GROUP_SIZE, head_dim), dtype=torch.float32, device=blocks.device)
    _lib.check(lib.kvmix_decode_key_pages(blocks.data_ptr(), P, head_dim, blocks.stride(0), out.data_ptr(),
                                          _lib.stream()))
    return out


def decode_token_blocks_device(blocks: torch.Tensor, head_dim: int, bitwidth: int) -> torch.Tensor:
    n = blocks.shape[0]
    out = torch.empty((n, head_dim), dtype=torch.float32, device=blocks.device)
    _lib.check(lib.kvmix_decode_token_blocks(blocks.data_ptr(), n, head_dim, bitwidth, blocks.stride(0),
                                             out.data_ptr(), _lib.stream()))
    return out


# ---- reference API ------------------------------------------------------------------
class _Staging:
    """Per-device pinned host byte buffer for the single-group entry points.  The reference's
    per-group API is called in tight loops (pkg/tests/test_acceptance.py:92-112: 40,000 calls
    under a 5 s limit), so a call is one kernel launch that reads its inputs from and writes
    its outputs to this buffer directly (zero-copy: pinned memory is device-accessible under
    unified addressing) and one stream sync -- no copies, no torch dispatch per call."""

    _by_dev: dict = {}

    def __init__(self, dev: torch.device):
        self.dev = dev
        self.cap = 0
        self.grow(1 << 16)

    def grow(self, n: int) -> None:
        if n > self.cap:
            self.cap = max(n, 2 * self.cap)
            self.h = torch.empty(self.cap, dtype=torch.uint8, pin_memory=True)
            self.hn = self.h.numpy()

    @classmethod
    def get(cls) -> "_Staging":
        dev = _lib.require_cuda()
        st = cls._by_dev.get(dev.index)
        if st is None:
            st = cls._by_dev[dev.index] = _Staging(dev)
        return st

    def roundtrip(self, n_up: int, lo: int, hi: int, launch) -> np.ndarray:
        """Run launch(base address of the pinned buffer) on h[:n_up], return a copy of h[lo:hi]."""
        launch(self.h.data_ptr())
        _lib.check(lib.kvmix_stream_sync(_lib.stream()))
        return self.hn[lo:hi].copy()


def _align(n: int) -> int:
    return (n + 15) & ~15


def quantize_group(values, bitwidth: int) -> QuantGroup:
    """quant.py:64-87 (one K-codec launch, kvmix_quantize_groups)."""
    if bitwidth not in (2, 4):
        raise ValidationError(f"unsupported bitwidth {bitwidth}")
    values = np.asarray(values, dtype=np.float32)
    if values.ndim != 1 or values.size == 0:
        raise ValidationError("values must be a non-empty 1-D vector")
    n = values.size
    # staging: [offsets i64 x2 | err i32 | scale f32 | zero f32 | pad | x f32[n] | codes u8[n]]
    ox, oc = 32, 32 + _align(4 * n)
    st = _Staging.get()
    st.grow(oc + n)
    st.hn[:16].view(np.int64)[:] = (0, n)
    st.hn[16:20].view(np.int32)[0] = 0
    st.hn[ox:ox + 4 * n].view(np.float32)[:] = values

    def launch(base):
        _lib.check(lib.kvmix_quantize_groups(base + ox, base, 1, bitwidth, base + oc, base + 20, base + 24, base + 16,
                                             _lib.stream()))

    out = st.roundtrip(oc, 16, oc + n, launch)  # header + x up; err, scale, zero (and codes) down
    err, s, z = int(out[:4].view(np.int32)[0]), float(out[4:8].view(np.float32)[0]), float(out[8:12].view(np.float32)[0])
    if err & 1:
        raise ValidationError("values must be finite")
    return QuantGroup(codes=out[oc - 16:oc - 16 + n].copy(), scale=s, zero_offset=z, bitwidth=bitwidth, group_len=n)


def dequantize_group(group: QuantGroup) -> np.ndarray:
    """quant.py:90-93: code * scale + zero with fp16-narrowed params (kvmix_dequantize_groups)."""
    codes = np.asarray(group.codes, dtype=np.uint8).reshape(-1)
    n = codes.size
    if n == 0:
        return np.zeros(0, np.float32)
    # staging: [offsets i64 x2 | scale f32 | zero f32 | pad | codes u8[n] | out f32[n]]
    oc = 32
    oo = oc + _align(n)
    st = _Staging.get()
    st.grow(oo + 4 * n)
    st.hn[:16].view(np.int64)[:] = (0, n)
    st.hn[16:24].view(np.float32)[:] = (group.scale, group.zero_offset)
    st.hn[oc:oc + n] = codes

    def launch(base):
        _lib.check(lib.kvmix_dequantize_groups(base + oc, base, 1, base + 16, base + 20, base + oo, n, _lib.stream()))

    return st.roundtrip(oo, oo, oo + 4 * n, launch).view(np.float32)


def pack_codes(codes, bitwidth: int) -> bytes:
    """quant.py:96-109."""
    codes = np.asarray(codes, dtype=np.int64)
    if bitwidth not in (2, 4):
        raise ValidationError(f"unsupported bitwidth {bitwidth}")
    if codes.size == 0:
        return b""
    if codes.min() < 0 or codes.max() >= (1 << bitwidth):
        raise ValidationError(f"code out of range for {bitwidth}-bit packing")
    dev = _lib.require_cuda()
    c = torch.as_tensor(codes.astype(np.uint8), device=dev)
    nb = -(-codes.size * bitwidth // 8)
    out = torch.empty(nb, dtype=torch.uint8, device=dev)
    err = _ErrFlag()
    _lib.check(lib.kvmix_pack_codes(c.data_ptr(), codes.size, bitwidth, out.data_ptr(), err.t.data_ptr(),
                                    _lib.stream()))
    if err.value() & 2:
        raise ValidationError(f"code out of range for {bitwidth}-bit packing")
    return out.cpu().numpy().tobytes()


def unpack_codes(data: bytes, bitwidth: int, n: int) -> np.ndarray:
    """quant.py:112-120."""
    if len(data) != -(-n * bitwidth // 8):
        raise ValidationError("packed byte length does not match code count")
    if n == 0:
        return np.zeros(0, dtype=np.uint8)
    dev = _lib.require_cuda()
    p = torch.as_tensor(np.frombuffer(data, dtype=np.uint8).copy(), device=dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    _lib.check(lib.kvmix_unpack_codes(p.data_ptr(), n, bitwidth, out.data_ptr(), _lib.stream()))
    return out.cpu().numpy()


def encode_key_page_int2(keys, group_len: int = GROUP_SIZE) -> KeyPageBlock:
    """quant.py:160-177."""
    keys = np.asarray(keys, dtype=np.float32) if not isinstance(keys, torch.Tensor) else keys
    if keys.ndim != 2 or keys.shape[0] != group_len:
        raise ValidationError(f"expected exactly {group_len} token rows, got shape {tuple(keys.shape)}")
    _check_group_len(group_len)
    x = _dev(keys)
    err = _ErrFlag()
    out = encode_key_pages_device(x.view(1, group_len, -1), err.t)
    if err.value() & 1:
        raise ValidationError("keys must be finite")
    return KeyPageBlock(payload=out.cpu().numpy().tobytes(), head_dim=int(keys.shape[1]), group_len=group_len)


def decode_key_page_int2(block: KeyPageBlock) -> np.ndarray:
    """quant.py:180-186 -> [group_len, d] fp32."""
    _check_group_len(block.group_len)
    b = torch.as_tensor(np.frombuffer(block.payload, dtype=np.uint8).copy(), device=_lib.require_cuda())
    return decode_key_pages_device(b.view(1, -1), block.head_dim)[0].cpu().numpy()


def encode_token_block(vec, bitwidth: int, group_len: int = GROUP_SIZE) -> TokenBlock:
    """quant.py:189-203."""
    vec = np.asarray(vec, dtype=np.float32)
    if vec.ndim != 1 or vec.size % group_len != 0:
        raise ValidationError(f"head dim {vec.shape} not divisible by group size {group_len}")
    return encode_token_blocks(vec[None], bitwidth, group_len)[0]


def encode_token_blocks(mat, bitwidth: int, group_len: int = GROUP_SIZE) -> list[TokenBlock]:
    """quant.py:206-232."""
    mat = np.asarray(mat, dtype=np.float32)
    if mat.ndim != 2 or mat.shape[1] % group_len != 0:
        raise ValidationError(f"expected [n, d] with d divisible by {group_len}")
    if bitwidth not in (2, 4):
        raise ValidationError(f"unsupported bitwidth {bitwidth}")
    _check_group_len(group_len)
    n, d = mat.shape
    if n == 0:
        return []
    err = _ErrFlag()
    out = encode_token_blocks_device(_dev(mat), bitwidth, err.t)
    if err.value() & 1:
        raise ValidationError("values must be finite")
    rows = out.cpu().numpy()
    return [TokenBlock(payload=rows[i].tobytes(), head_dim=d, bitwidth=bitwidth, group_len=group_len)
            for i in range(n)]


def decode_token_blocks(blocks: list[TokenBlock]) -> np.ndarray:
    """quant.py:235-253 -> [n, d] fp32."""
    if not blocks:
        raise ValidationError("no blocks to decode")
    d, b, g = blocks[0].head_dim, blocks[0].bitwidth, blocks[0].group_len
    if any((blk.head_dim, blk.bitwidth, blk.group_len) != (d, b, g) for blk in blocks):
        raise ValidationError("blocks must share dims and bitwidth")
    _check_group_len(g)
    raw = np.frombuffer(b"".join(blk.payload for blk in blocks), dtype=np.uint8).reshape(len(blocks), -1)
    t = torch.as_tensor(raw.copy(), device=_lib.require_cuda())
    return decode_token_blocks_device(t, d, b).cpu().numpy()


def decode_token_block(block: TokenBlock) -> np.ndarray:
    """quant.py:256-262 -> [d] fp32."""
    return decode_token_blocks([block])[0]
