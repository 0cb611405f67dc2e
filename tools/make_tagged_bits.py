"""Generate per-token bitwidth maps for the benchmark ("tagged KV caches").

Runs the REFERENCE's host-side pipeline (imported read-only from /root/reference;
the tagger, calibration and allocator are out of scope and stay on the host):
  generate_synthetic_trace(include_images=True) -> tag_tokens -> keep the last N tags
  -> SensitivityTable from build_table on three 40-turn d=128 captures (6-turn ones leave every
     tag below one INT2 page, so D(2) == D(4) and the allocator keeps everything at INT2), with counts
     replaced by the benchmark traces' histogram (estimate_counts) -> allocate(B=2.5)
  (SURVEY.md section 8(d) recipe).  Output: bench_data/tagged_bits.npz with packed
  bit maps (1 = INT2) per request for each context length.
Usage: PYTHONPATH=/root/reference/pkg/src python tools/make_tagged_bits.py
"""
import math
import os
import sys

import numpy as np

from kvmix import (SensitivityTable, allocate, build_table, default_template, estimate_counts,
                   generate_synthetic_capture, generate_synthetic_trace, tag_tokens)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "bench_data", "tagged_bits.npz")
SPECS = {4096: 4, 32768: 16, 102400: 8, 131072: 2}  # context -> number of distinct requests
BUDGET = 2.5
CALIB_TURNS = 40  # long enough that every tag fills whole INT2 pages in the replay


def main():
    template = default_template()
    caps = []
    for s in range(3):
        tr = generate_synthetic_trace(900 + s, CALIB_TURNS, template, include_images=True)
        tg = tag_tokens(tr, template)
        caps.append(generate_synthetic_capture(tr, tg, n_layers=1, n_heads=2, n_kv_heads=1, head_dim=128, seed=900 + s))
    calib = build_table(caps)
    out = {}
    for n, reqs in SPECS.items():
        tags_all = []
        for r in range(reqs):
            turns = math.ceil(1.05 * n / 40.7)
            tr = generate_synthetic_trace(20261017 + 7919 * r + n, turns, template, include_images=True)
            tg = np.asarray(tag_tokens(tr, template))
            while tg.size < n:  # extend with more turns if the draw came up short
                turns = int(turns * 1.1) + 1
                tr = generate_synthetic_trace(20261017 + 7919 * r + n, turns, template, include_images=True)
                tg = np.asarray(tag_tokens(tr, template))
            tags_all.append(tg[-n:])
        counts = estimate_counts(tags_all)
        dist = {k: v for k, v in calib.distortion.items() if k[0] in counts}
        known = {t for t, _ in dist}
        counts_k = {t: c for t, c in counts.items() if t in known}
        alloc = allocate(SensitivityTable(distortion=dist, counts=counts_k), BUDGET)
        bits = np.stack([np.array([alloc.bits.get(int(t), 4) for t in tg], dtype=np.int8) for tg in tags_all])
        frac2 = float((bits == 2).mean())
        print(f"N={n} reqs={reqs}: INT2 token fraction {frac2:.4f}, tags {len(counts)} (calibrated {len(known)})")
        out[f"bits_{n}"] = np.packbits(bits == 2, axis=1)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    sys.exit(main())
