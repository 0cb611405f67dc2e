"""K1 at cfg3 scale (BASELINE.json configs[2]): a 128K-token request with the reference-tagged
bits, routed on the device (K6, ``alloc_device``) and quantized + packed by K1 exactly as the
bench does it, checked byte for byte against the oracle on sampled pages and INT4 slots.

The prefill writes 2 layers x 8 kv heads x 131072 tokens; re-encoding all of it on the CPU
would take minutes, so 256 INT2 pages and 256 INT4 slots (each in every layer and head) are
sampled, their 32 (or 1) source rows copied back, encoded by the oracle (quant.py:160-232
restated) and compared with the device records mapped back through layout.py.
"""
import os

import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import layout
from oracle import codec as oc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def tagged_bits(n: int, row: int) -> np.ndarray:
    data = np.load(os.path.join(ROOT, "bench_data", "tagged_bits.npz"))
    return np.where(np.unpackbits(data[f"bits_{n}"][row])[:n] == 1, 2, 4)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_cfg3_scale_prefill_bytes(cuda, dtype):
    N, L, H, d = 131072, 2, 8, 128
    bits = tagged_bits(N, 0)
    n2 = int((bits == 2).sum()) // 32 * 32
    pool = kv.MixedPrecisionPool(kv.PoolConfig(total_slots=N + 64, offset=n2, n_layers=L, n_kv_heads=H,
                                               head_dim=d))
    gen = torch.Generator(device="cuda").manual_seed(3)
    chs = torch.exp(torch.empty(H, d, device="cuda").uniform_(np.log(0.5), np.log(4.0), generator=gen))
    k = (torch.randn(L, N, H, d, device="cuda", generator=gen) * chs).to(dtype)
    v = torch.randn(L, N, H, d, device="cuda", generator=gen).to(dtype)
    table = pool.alloc_device("r0", bits)
    assert np.array_equal(table.slots, pool.__class__(pool.config).alloc("r0", bits).slots)
    pool.write_prefill(table, k, v)
    torch.cuda.synchronize()
    slots = table.slots
    rng = np.random.default_rng(0)

    # INT2 pages: the 32 tokens routed to page P, in row order
    is2 = slots < pool.config.offset
    tok2 = np.flatnonzero(is2)
    order = tok2[np.argsort(slots[tok2], kind="stable")]  # page-major, row-minor
    pages = slots[order[::32]] // 32
    pick = rng.choice(pages.size, size=256, replace=False)
    rows = order.reshape(-1, 32)[pick]  # [256, 32] token ids
    kk = k[:, torch.as_tensor(rows.reshape(-1), device="cuda")].float().cpu().numpy().reshape(L, 256, 32, H, d)
    vv = v[:, torch.as_tensor(rows.reshape(-1), device="cuda")].float().cpu().numpy().reshape(L, 256, 32, H, d)
    kp = oc.encode_key_pages(np.moveaxis(kk, 3, 2))  # [L, 256, H, payload]
    vb = oc.encode_token_blocks(np.moveaxis(vv, 3, 2), 2)  # [L, 256, H, 32, tb2]
    ref = np.concatenate([kp, vb.reshape(L, 256, H, -1)], axis=-1)
    n_pages = pool.n_pages
    dev2 = pool.int2_pool[: L * H * n_pages * pool.page_stride].view(L, H, n_pages, pool.page_stride)
    got = dev2[:, :, torch.as_tensor(pages[pick], device="cuda")].cpu().numpy()  # [L, H, 256, PS]
    got = np.moveaxis(layout.page_payloads(got, d), 2, 1)  # [L, 256, H, payload]
    assert np.array_equal(got, ref), "INT2 page records differ from the oracle"

    # INT4 slots
    tok4 = np.flatnonzero(~is2)
    pick4 = rng.choice(tok4, size=256, replace=False)
    idx = torch.as_tensor(pick4, device="cuda")
    kk4, vv4 = k[:, idx].float().cpu().numpy(), v[:, idx].float().cpu().numpy()  # [L, 256, H, d]
    ref4 = np.concatenate([oc.encode_token_blocks(kk4, 4), oc.encode_token_blocks(vv4, 4)], axis=-1)
    dev4 = pool.int4_pool[: L * H * pool.n_int4 * pool.slot_stride].view(L, H, pool.n_int4, pool.slot_stride)
    g4 = dev4[:, :, torch.as_tensor(slots[pick4] - pool.config.offset, device="cuda")].cpu().numpy()
    g4 = np.moveaxis(layout.slot_payloads(g4, d), 2, 1)  # [L, 256, H, payload]
    assert np.array_equal(g4, ref4), "INT4 slot records differ from the oracle"
