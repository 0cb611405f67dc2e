"""K1 codec on the GPU vs the oracle and the reference's golden payloads: bit-exact
codes, scales and zeros (north_star: "packed codes, scales, zeros ... bit-exact")."""
import numpy as np
import pytest
import torch

import paper_2605_17170_b200 as kv
from paper_2605_17170_b200 import quant as gq
from oracle import codec

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [32, 64, 128])
def test_golden_layout_payloads(cuda, golden, d):
    keys = golden[f"layout_inputs_keys_d{d}"]
    vec = golden[f"layout_inputs_vec_d{d}"]
    assert np.frombuffer(kv.encode_key_page_int2(keys).payload, np.uint8).tolist() == \
        golden[f"layout_key_page_int2_d{d}"].tolist()
    for b in (2, 4):
        assert np.frombuffer(kv.encode_token_block(vec, b).payload, np.uint8).tolist() == \
            golden[f"layout_token_block_int{b}_d{d}"].tolist()


@pytest.mark.parametrize("d", [32, 64, 128])
def test_golden_codec_vectors(cuda, golden, d):
    keys = torch.as_tensor(golden[f"codec_keys_d{d}"], device=cuda)
    got = gq.encode_key_pages_device(keys).cpu().numpy()
    assert np.array_equal(got, golden[f"codec_key_pages_d{d}"])
    x = torch.as_tensor(golden[f"codec_tok_in_d{d}"], device=cuda)
    for b in (2, 4):
        assert np.array_equal(gq.encode_token_blocks_device(x, b).cpu().numpy(), golden[f"codec_tok_int{b}_d{d}"])


def test_layout_worked_examples(cuda):
    keys = np.zeros((32, 2), np.float32)
    keys[:, 0] = np.arange(32) % 4
    keys[:, 1] = 5.0
    assert kv.encode_key_page_int2(keys).payload.hex() == "e4" * 8 + "00" * 8 + "003c0000" + "00000045"
    vec = np.concatenate([np.tile(np.arange(16, dtype=np.float32), 2), np.full(32, 2.5, np.float32)])
    assert kv.encode_token_block(vec, 4).payload.hex() == "1032547698badcfe" * 2 + "00" * 16 + "003c000000000041"
    assert kv.encode_token_block((np.arange(32) % 4).astype(np.float32), 2).payload.hex() == "e4" * 8 + "003c0000"


@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_random_bitexact_large(cuda, d):
    """10K key pages / 40K token blocks per bitwidth, wide dynamic ranges, vs the oracle."""
    rng = np.random.default_rng(d)
    n = 10_000 if d <= 128 else 2_000
    keys = (rng.standard_normal((n, 32, d)) * rng.uniform(0.01, 300, (n, 1, 1))
            + rng.uniform(-50, 50, (n, 1, 1))).astype(np.float32)
    got = gq.encode_key_pages_device(torch.as_tensor(keys, device=cuda)).cpu().numpy()
    assert np.array_equal(got, codec.encode_key_pages(keys))
    x = keys.reshape(-1, d)[: 4 * n]
    xt = torch.as_tensor(x, device=cuda)
    for b in (2, 4):
        assert np.array_equal(gq.encode_token_blocks_device(xt, b).cpu().numpy(), codec.encode_token_blocks(x, b))


def test_decode_exact(cuda):
    rng = np.random.default_rng(1)
    for d in (32, 64, 128):
        keys = rng.standard_normal((50, 32, d)).astype(np.float32)
        blocks = codec.encode_key_pages(keys)
        got = gq.decode_key_pages_device(torch.as_tensor(blocks, device=cuda), d).cpu().numpy()
        assert np.array_equal(got, codec.decode_key_pages(blocks, d))
        for b in (2, 4):
            tb = codec.encode_token_blocks(keys.reshape(-1, d), b)
            got = gq.decode_token_blocks_device(torch.as_tensor(tb, device=cuda), d, b).cpu().numpy()
            assert np.array_equal(got, codec.decode_token_blocks(tb, d, b))
    blk = kv.encode_token_block(np.linspace(-1, 1, 64, dtype=np.float32), 4)
    assert np.array_equal(kv.decode_token_block(blk), codec.decode_token_blocks(np.frombuffer(blk.payload, np.uint8), 64, 4))


def test_quantize_group_golden(cuda, golden):
    v, off, codes, prm = golden["qg_values"], golden["qg_offsets"], golden["qg_codes"], golden["qg_params"]
    for i in range(0, len(off) - 1, 7):
        b, s, z = prm[i]
        g = kv.quantize_group(v[off[i]:off[i + 1]], int(b))
        assert np.array_equal(g.codes, codes[off[i]:off[i + 1]]) and g.scale == s and g.zero_offset == z


def test_quantize_group_api(cuda):
    g = kv.quantize_group([0, 5, 10, 15], 4)
    assert g.scale == 1.0 and g.zero_offset == 0.0 and g.codes.tolist() == [0, 5, 10, 15]
    assert kv.dequantize_group(g).tolist() == [0, 5, 10, 15]
    g = kv.quantize_group([3.5] * 32, 2)
    assert g.scale == 0.0 and not g.codes.any() and np.all(kv.dequantize_group(g) == 3.5)
    with pytest.raises(kv.ValidationError):
        kv.quantize_group([1.0, np.inf], 2)
    with pytest.raises(kv.ValidationError):
        kv.quantize_group([], 4)
    with pytest.raises(kv.ValidationError):
        kv.quantize_group([1.0], 3)


def test_pack_unpack(cuda):
    assert kv.pack_codes([1, 2, 3, 0], 2) == bytes([0x39])
    assert kv.pack_codes([0xA, 0x5], 4) == bytes([0x5A])
    assert len(kv.pack_codes([1] * 7, 2)) == 2 and len(kv.pack_codes([1] * 3, 4)) == 2
    with pytest.raises(kv.ValidationError):
        kv.pack_codes([4], 2)
    with pytest.raises(kv.ValidationError):
        kv.unpack_codes(b"\x00", 2, 5)
    rng = np.random.default_rng(102)
    for _ in range(200):
        b = int(rng.choice([2, 4]))
        n = int(rng.integers(1, 100))
        c = rng.integers(0, 1 << b, n)
        assert np.array_equal(kv.unpack_codes(kv.pack_codes(c, b), b, n), c)


def test_validation(cuda):
    with pytest.raises(kv.ValidationError):
        kv.encode_key_page_int2(np.zeros((31, 32), np.float32))
    with pytest.raises(kv.ValidationError):
        kv.encode_key_page_int2(np.full((32, 32), np.nan, np.float32))
    with pytest.raises(kv.ValidationError):
        kv.encode_token_block(np.zeros(33, np.float32), 4)
    with pytest.raises(kv.ValidationError):
        kv.encode_token_blocks(np.full((2, 64), np.inf, np.float32), 2)
    with pytest.raises(kv.ValidationError):
        kv.decode_token_blocks([])
    assert len(kv.encode_key_page_int2(np.zeros((32, 64), np.float32)).payload) == 768
    assert len(kv.encode_token_block(np.zeros(128, np.float32), 2).payload) == 48
