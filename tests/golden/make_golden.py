"""Generate the golden fixtures in this directory from the REAL reference implementation.

Run in the build container (the reference is mounted read-only at /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
The output (golden.npz, alloc_trace.json) is committed; nothing at test time reads
/root/reference.  Contents:
  * the nine LAYOUT.md golden payloads (seeds of tests/test_acceptance.py:115-129)
  * seeded codec vectors (inputs + reference payloads), incl. edge cases
  * quantize_group vectors for ragged lengths
  * an allocator trace (alloc/free/partition/append ops and the reference's slot lists)
  * flash_decode cases (pool inputs + reference fp32 outputs)
"""
import json
import os

import numpy as np

from kvmix.attention import flash_decode
from kvmix.errors import CapacityError
from kvmix.pool import MixedPrecisionPool, PoolConfig
from kvmix.quant import encode_key_page_int2, encode_token_block, encode_token_blocks, quantize_group

HERE = os.path.dirname(os.path.abspath(__file__))


def golden_layout(out):
    # test_acceptance.py:115-129 draw order
    for d in (32, 64, 128):
        rng = np.random.default_rng(1000 + d)
        keys = rng.standard_normal((32, d)).astype(np.float32)
        keys *= np.exp(rng.uniform(-0.7, 1.4, d)).astype(np.float32)
        out[f"layout_key_page_int2_d{d}"] = np.frombuffer(encode_key_page_int2(keys).payload, np.uint8)
        vec = rng.standard_normal(d).astype(np.float32)
        for b in (4, 2):
            out[f"layout_token_block_int{b}_d{d}"] = np.frombuffer(encode_token_block(vec, b).payload, np.uint8)
        out[f"layout_inputs_keys_d{d}"] = keys
        out[f"layout_inputs_vec_d{d}"] = vec


def codec_vectors(out):
    rng = np.random.default_rng(20261017)
    for d in (32, 64, 128):
        n = 16
        keys = (rng.standard_normal((n, 32, d)) * np.exp(rng.uniform(-0.7, 1.4, (1, 1, d)))).astype(np.float32)
        # edge cases: constant channel, grid-aligned ramp, huge range, tiny range, all-negative
        keys[0, :, 0] = 3.25
        keys[1, :, 1] = np.arange(32) % 4
        keys[2, :, 2] = np.linspace(-3e4, 3e4, 32)
        keys[3, :, 3] = 1.0 + np.arange(32) * 1e-7
        keys[4] -= 50.0
        out[f"codec_keys_d{d}"] = keys
        out[f"codec_key_pages_d{d}"] = np.stack(
            [np.frombuffer(encode_key_page_int2(k).payload, np.uint8) for k in keys])
        x = (rng.standard_normal((64, d)) * rng.uniform(0.01, 20, (64, 1))).astype(np.float32)
        x[0] = 7.0
        x[1, :32] = np.repeat(np.arange(16, dtype=np.float32), 2)
        x[2] = np.linspace(-6e4, 6e4, d)
        x[3] = 2.0 + np.arange(d) * 1e-7
        out[f"codec_tok_in_d{d}"] = x
        for b in (2, 4):
            out[f"codec_tok_int{b}_d{d}"] = np.stack(
                [np.frombuffer(t.payload, np.uint8) for t in encode_token_blocks(x, b)])


def quantize_group_vectors(out):
    rng = np.random.default_rng(7)
    vals, offs, codes, sz = [], [0], [], []
    for b in (2, 4):
        for i in range(200):
            n = int(rng.integers(1, 65))
            v = rng.uniform(-100, 100, n).astype(np.float32)
            if i % 25 == 0:
                v[:] = np.float16(v[0])
            g = quantize_group(v, b)
            vals.append(v)
            codes.append(g.codes)
            offs.append(offs[-1] + n)
            sz.append((b, g.scale, g.zero_offset))
    out["qg_values"] = np.concatenate(vals)
    out["qg_offsets"] = np.asarray(offs, np.int64)
    out["qg_codes"] = np.concatenate(codes)
    out["qg_params"] = np.asarray(sz, np.float64)


def alloc_trace():
    rng = np.random.default_rng(109)
    cfg = PoolConfig(total_slots=512, offset=288, n_layers=1, n_kv_heads=1, head_dim=32)
    pool = MixedPrecisionPool(cfg)
    live, ops, nid = [], [], 0
    kv = np.zeros((1, 1, 32), np.float32)
    for _ in range(300):
        a = rng.random()
        rec = None
        try:
            if a < 0.45 or not live:
                n = int(rng.integers(1, 80))
                bits = rng.choice([2, 4], size=n, p=[0.6, 0.4])
                rid = f"r{nid}"
                nid += 1
                rec = {"op": "alloc", "rid": rid, "bits": bits.tolist()}
                t = pool.alloc(rid, bits)
                live.append(rid)
                rec["slots"] = [x.index for x in t.entries]
            elif a < 0.8:
                rid = live.pop(int(rng.integers(len(live))))
                rec = {"op": "free", "rid": rid}
                pool.free(rid)
            else:
                rid = live[int(rng.integers(len(live)))]
                rec = {"op": "append", "rid": rid}
                pool.partition(pool.table(rid))
                s = pool.append_decode_token(rid, kv, kv)
                rec["slot"] = s.index
                rec["slots"] = [x.index for x in pool.table(rid).entries]
        except CapacityError as e:
            rec["capacity"] = e.region
        rec["free_pages"] = list(pool._free_pages)
        rec["free_int4"] = list(pool._free_int4)
        ops.append(rec)
    return {"total_slots": 512, "offset": 288, "ops": ops}


def decode_cases(out):
    rng = np.random.default_rng(103)
    meta = []
    for i in range(12):
        d = [32, 64, 128][i % 3]
        n_kv = [1, 2][i % 2]
        ratio = [1, 2, 4, 8][i % 4]
        H = n_kv * ratio
        n = int(rng.integers(32, 300))
        frac = float(rng.uniform(0.0, 1.0)) if i % 5 else [0.0, 1.0][i % 2]
        # fp16-representable inputs, stored as fp16 to keep the fixture small
        keys = (rng.standard_normal((1, n, n_kv, d)) * np.exp(rng.uniform(-0.7, 1.4, (n_kv, d))))
        keys = keys.astype(np.float16).astype(np.float32)
        values = rng.standard_normal((1, n, n_kv, d)).astype(np.float16).astype(np.float32)
        bits = np.where(rng.random(n) < frac, 2, 4)
        n2 = int((bits == 2).sum())
        offset = -(-n2 // 32) * 32
        cfg = PoolConfig(total_slots=offset + n + 8, offset=offset, n_layers=1, n_kv_heads=n_kv, head_dim=d)
        pool = MixedPrecisionPool(cfg)
        t = pool.alloc("req", bits)
        pool.write_prefill(t, keys, values)
        pool.partition(t)
        q = rng.standard_normal((H, d)).astype(np.float32)
        o = flash_decode(q, t, pool.view(0))
        out[f"dec{i}_keys"] = keys.astype(np.float16)
        out[f"dec{i}_values"] = values.astype(np.float16)
        out[f"dec{i}_bits"] = bits.astype(np.int8)
        out[f"dec{i}_q"] = q
        out[f"dec{i}_out"] = o.astype(np.float32)
        meta.append([d, n_kv, H, n, cfg.total_slots, cfg.offset])
    out["dec_meta"] = np.asarray(meta, np.int64)


def main():
    out = {}
    golden_layout(out)
    codec_vectors(out)
    quantize_group_vectors(out)
    decode_cases(out)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "alloc_trace.json"), "w") as f:
        json.dump(alloc_trace(), f)
    print("wrote golden.npz", os.path.getsize(os.path.join(HERE, "golden.npz")), "bytes")


if __name__ == "__main__":
    main()
