"""CPU model of K2's fp16 roundings (which rounding dominates the error budget?).

Emulates the decode kernel's numerics in float64 with explicit fp16 roundings at the
places the kernel rounds: q' = fp16(q*s) for INT2 key pages, p = fp16(exp2(.)) with the
lazy max (p <= 2^slack), P' = fp16(p*s_v).  Tensor-core accumulation is treated as
exact.  Compares against the float64 attention over the same dequantized K/V and
reports max |err| and max err / (atol + rtol |ref|) for fp32 and bf16 outputs.

  python tools/numerics_sim.py [--n 32768] [--frac 0.83] [--heads 8]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.codec import group_params, quantize  # noqa: E402

f16 = lambda x: np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def bf16(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def quant_unit(rng, n, frac, d=128, kmul=None, vmul=1.0):
    bits = np.where(rng.random(n) < frac, 2, 4)
    chs = np.exp(rng.uniform(np.log(0.5), np.log(4.0), d)) if kmul is None else kmul
    k = bf16(rng.standard_normal((n, d)) * chs).astype(np.float32)
    v = bf16(rng.standard_normal((n, d)) * vmul).astype(np.float32)
    i2 = np.flatnonzero(bits == 2)
    npg = i2.size // 32
    pg = i2[: npg * 32]
    i4 = np.sort(np.concatenate([np.flatnonzero(bits == 4), i2[npg * 32:]]))
    # INT2 key pages: per channel over 32 tokens
    kp = k[pg].reshape(npg, 32, d)
    ks, kz = group_params(kp.min(1), kp.max(1), 2)  # [npg, d]
    kc = quantize(kp, ks[:, None], kz[:, None], 2).astype(np.float64)
    vp = v[pg].reshape(npg * 32, d // 32, 32)
    vs2, vz2 = group_params(vp.min(2), vp.max(2), 2)
    vc2 = quantize(vp, vs2[..., None], vz2[..., None], 2).astype(np.float64)
    k4 = k[i4].reshape(-1, d // 32, 32)
    ks4, kz4 = group_params(k4.min(2), k4.max(2), 4)
    kc4 = quantize(k4, ks4[..., None], kz4[..., None], 4).astype(np.float64)
    v4 = v[i4].reshape(-1, d // 32, 32)
    vs4, vz4 = group_params(v4.min(2), v4.max(2), 4)
    vc4 = quantize(v4, vs4[..., None], vz4[..., None], 4).astype(np.float64)
    return dict(npg=npg, kc=kc, ks=ks.astype(np.float64), kz=kz.astype(np.float64), vc2=vc2,
                vs2=vs2.astype(np.float64), vz2=vz2.astype(np.float64), kc4=kc4, ks4=ks4.astype(np.float64),
                kz4=kz4.astype(np.float64), vc4=vc4, vs4=vs4.astype(np.float64), vz4=vz4.astype(np.float64))


def run(u, q, exact_q2=False, exact_pv=False, slack=8.0, d=128):
    """q [H, d] (bf16 values).  Returns (out_model [H, d], out_exact [H, d])."""
    qs = 1.0 / np.sqrt(d) * 1.4426950408889634
    npg = u["npg"]
    # logits (log2 domain)
    # INT2: per page p, token t: sum_c q'_c code + sum_c q_c z_c
    qp = q[:, None, :] * u["ks"][None]  # [H, npg, d]
    qpm = qp if exact_q2 else f16(qp)
    l2m = (np.einsum("hpd,ptd->hpt", qpm, u["kc"]) + np.einsum("hd,pd->hp", q, u["kz"])[..., None]) * qs
    l2e = (np.einsum("hpd,ptd->hpt", qp, u["kc"]) + np.einsum("hd,pd->hp", q, u["kz"])[..., None]) * qs
    l2m, l2e = l2m.reshape(q.shape[0], -1), l2e.reshape(q.shape[0], -1)
    qg = q.reshape(q.shape[0], d // 32, 32)
    l4 = (np.einsum("hjc,tjc,tj->ht", qg, u["kc4"], u["ks4"]) + np.einsum("hjc,tj->ht", qg, u["kz4"])) * qs
    lm = np.concatenate([l2m, l4], 1)
    le = np.concatenate([l2e, l4], 1)
    # dequantized V rows [T, d]
    v2 = (u["vc2"] * u["vs2"][..., None] + u["vz2"][..., None]).reshape(-1, d)
    v4 = (u["vc4"] * u["vs4"][..., None] + u["vz4"][..., None]).reshape(-1, d)
    V = np.concatenate([v2, v4], 0)
    # exact reference
    w = np.exp2(le - le.max(1, keepdims=True))
    ref = (w @ V) / w.sum(1, keepdims=True)
    # model: lazy max per tile of 32 tokens (one stream, tiles in order)
    H, T = lm.shape
    m = np.full(H, -np.inf)
    p = np.zeros_like(lm)
    mt = np.zeros_like(lm)
    for t0 in range(0, T, 32):
        tm = lm[:, t0:t0 + 32].max(1)
        raise_ = (m == -np.inf) | (tm - m > slack)
        m = np.where(raise_, np.maximum(m, tm) if True else m, m)
        mt[:, t0:t0 + 32] = m[:, None]
    # final rescale to the last max (accumulators rescaled exactly in fp32)
    p = f16(np.exp2(lm - mt))
    scale_to_final = np.exp2(mt - mt[:, -1:])
    # PV: per group scale folded into P' = fp16(p * s)
    codes = np.concatenate([u["vc2"], u["vc4"]], 0)  # [T, ng, 32]
    s = np.concatenate([u["vs2"], u["vs4"]], 0)  # [T, ng]
    z = np.concatenate([u["vz2"], u["vz4"]], 0)
    Pp = p[:, :, None] * s[None]  # [H, T, ng]
    Ppm = Pp if exact_pv else f16(Pp)
    num = np.einsum("htj,tjc->hjc", Ppm * scale_to_final[..., None], codes).reshape(H, d)
    num += np.einsum("ht,tj->hj", p * scale_to_final, z).repeat(32, 1)
    l = (p * scale_to_final).sum(1, keepdims=True)
    return num / l, ref


def report(name, out, ref, atol=2e-3, rtol=1e-2):
    for tag, o in (("f32", out.astype(np.float32).astype(np.float64)), ("bf16", bf16(out))):
        e = np.abs(o - ref)
        r = e / (atol + rtol * np.abs(ref))
        print(f"  {name:22s} {tag:5s} max|err| {e.max():.2e}  worst err/tol {r.max():.3f}  |ref|max {np.abs(ref).max():.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--frac", type=float, default=0.83)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--qmul", type=float, default=1.0)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    u = quant_unit(rng, a.n, a.frac)
    q = bf16(rng.standard_normal((a.heads, 128)) * a.qmul)
    print(f"n={a.n} frac={a.frac} pages={u['npg']} qmul={a.qmul}")
    for name, kw in [("current", {}), ("exact q'", dict(exact_q2=True)), ("exact P'", dict(exact_pv=True)),
                     ("exact both", dict(exact_q2=True, exact_pv=True))]:
        out, ref = run(u, q, **kw)
        report(name, out, ref)


if __name__ == "__main__":
    main()
