"""B200-native (sm_100a) TriAxialKV hot path: INT2/INT4 KV quantize+pack into a
dual-precision paged pool and split-K fused decode attention over that pool.

Mirrors the hot-path names of the reference package ``kvmix``
(/root/reference/pkg/src/kvmix/__init__.py:19-70): the codec (``quant``), the pool
(``pool``) and the decode path (``attention``).  All compute runs in
libkvmix_b200.so; importing this package without the library raises.
"""

from . import _lib  # noqa: F401  (fails loudly when the CUDA library is missing)
from .attention import (
    DecodeBatch,
    SplitPartial,
    flash_decode,
    flash_decode_batched,
    flash_decode_layers_from_host,
    merge_partials,
)
from . import calib  # noqa: F401  (calibration replay on the GPU)
from .decode_step import DecodeStep
from .errors import CapacityError, InfeasibleBudgetError, KvmixError, TemplateStructureError, ValidationError
from .plan import plan_stream
from .pool import (
    MixedPrecisionPool,
    PageTable,
    PoolConfig,
    PoolView,
    SlotAddress,
    baseline_bytes_per_token,
    bytes_per_token,
    capacity_tokens,
    init_pool,
)
from .quant import (
    GROUP_SIZE,
    KeyPageBlock,
    QuantGroup,
    TokenBlock,
    decode_key_page_int2,
    decode_token_block,
    decode_token_blocks,
    dequantize_group,
    encode_key_page_int2,
    encode_token_block,
    encode_token_blocks,
    key_page_payload_bytes,
    pack_codes,
    quantize_group,
    token_block_payload_bytes,
    unpack_codes,
)

__version__ = "0.1.0"
