"""ctypes binding of the C ABI in include/kvmix_b200.h (libkvmix_b200.so).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
-gencode arch=compute_100a,code=sm_100a).  There is no fallback: importing the
package without the library raises, and every device call checks its status.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import CapacityError, KvmixError, ValidationError

# KVMIX_LIB: an alternative build of the same library (measurement variants, tools/ab_variants.py)
LIB_PATH = os.environ.get("KVMIX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkvmix_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the CUDA library is required; there is no CPU fallback)"
    )

lib = ctypes.CDLL(LIB_PATH)

_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_P = ctypes.c_void_p
_F = ctypes.c_float

_SIGS = {
    "kvmix_version": ([], ctypes.c_char_p),
    "kvmix_last_error": ([], ctypes.c_char_p),
    "kvmix_page_stride": ([_I64], _I64),
    "kvmix_slot_stride": ([_I64], _I64),
    "kvmix_page_layout": ([_I64, _P], ctypes.c_int),
    "kvmix_slot_layout": ([_I64, _P], ctypes.c_int),
    "kvmix_key_page_payload_bytes": ([_I64], _I64),
    "kvmix_token_block_payload_bytes": ([_I64, _I64], _I64),
    "kvmix_encode_key_pages": ([_P, _I64, _I64, _P, _I64, _P, _P], ctypes.c_int),
    "kvmix_encode_token_blocks": ([_P, _I64, _I64, _I32, _P, _I64, _P, _P], ctypes.c_int),
    "kvmix_decode_key_pages": ([_P, _I64, _I64, _I64, _P, _P], ctypes.c_int),
    "kvmix_decode_token_blocks": ([_P, _I64, _I64, _I32, _I64, _P, _P], ctypes.c_int),
    "kvmix_quantize_groups": ([_P, _P, _I64, _I32, _P, _P, _P, _P, _P], ctypes.c_int),
    "kvmix_dequantize_groups": ([_P, _P, _I64, _P, _P, _P, _I64, _P], ctypes.c_int),
    "kvmix_pack_codes": ([_P, _I64, _I32, _P, _P, _P], ctypes.c_int),
    "kvmix_unpack_codes": ([_P, _I64, _I32, _P, _P], ctypes.c_int),
    "kvmix_write_prefill": ([_P, _P, _I32, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _I64, _P, _I64, _P,
                             _I64, _P, _P], ctypes.c_int),
    "kvmix_append_int4": ([_P, _P, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P], ctypes.c_int),
    "kvmix_append_int4_strided": ([_P, _P, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P],
                                  ctypes.c_int),
    "kvmix_attention_full": ([_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _F, _I32, _P, _P], ctypes.c_int),
    "kvmix_gather_dequant": ([_P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _P], ctypes.c_int),
    "kvmix_gather_dequant_typed": ([_P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _I32, _P],
                                   ctypes.c_int),
    "kvmix_flash_decode": ([_P, _I32, _P, _I32, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P,
                            _P, _P, _P, _I64, _P, _P, _F, _I32, _P, _I32, _P], ctypes.c_int),
    "kvmix_stream_sync": ([_P], ctypes.c_int),
    "kvmix_flash_decode_gather": ([_P, _I32, _P, _I32, _I64, _I64, _I32, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64,
                                   _I64, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _F, _I32, _P, _I32, _P], ctypes.c_int),
    "kvmix_flash_decode_append": ([_P, _I32, _P, _I32, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P,
                                   _P, _P, _P, _P, _I64, _P, _P, _F, _P, _P, _I32, _P, _I32, _P], ctypes.c_int),
    "kvmix_decode_tables_smem": ([_I64, _I64], _I64),
    "kvmix_decode_tables": ([_P, _I64, _I64, _P, _P, _P, _I64, _I64, _F, _I64, _P, _P, _P, _P, _P, _P],
                            ctypes.c_int),
    "kvmix_merge_partials": ([_P, _P, _P, _I64, _I64, _P, _P], ctypes.c_int),
    "kvmix_route_scratch_elems": ([_I64], _I64),
    "kvmix_count_int2": ([_P, _I64, _P, _P, _P], ctypes.c_int),
    "kvmix_route_tokens": ([_P, _I64, _I32, _P, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P],
                           ctypes.c_int),
}

if hasattr(lib, "kvmix_debug_cta_times"):  # debug builds (-DKVMIX_CTA_TIMES) only
    lib.kvmix_debug_cta_times.argtypes = [_P, ctypes.c_int]
    lib.kvmix_debug_cta_times.restype = ctypes.c_int

for _name, (_args, _ret) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _ret

EXPORTED = tuple(_SIGS)

F32, BF16, F16 = 0, 1, 2
POOL_STATUS_WORDS = 4          # kvmix_b200.h KVMIX_POOL_STATUS_*
POOL_STATUS_ERR, POOL_STATUS_KSCALE, POOL_STATUS_VSCALE = 0, 1, 2
DECODE_POOL_WRITTEN = 1        # kvmix_b200.h KVMIX_DECODE_POOL_WRITTEN
_DT = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValidationError(f"unsupported dtype {t.dtype}") from None


def dtype_code_of(dtype: torch.dtype) -> int:
    try:
        return _DT[dtype]
    except KeyError:
        raise ValidationError(f"unsupported dtype {dtype}") from None


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.kvmix_last_error().decode(errors="replace")
    if rc == -2:
        raise ValidationError(msg)
    if rc == -3:
        raise CapacityError(msg, region="pool")
    raise KvmixError(f"CUDA failure in libkvmix_b200: {msg}")


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise KvmixError("a CUDA device is required (libkvmix_b200 has no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def page_stride(d: int) -> int:
    return int(lib.kvmix_page_stride(d))


def slot_stride(d: int) -> int:
    return int(lib.kvmix_slot_stride(d))
