// K2 split-K mixed INT2/INT4 decode attention + K3 cross-split combine.
//
// Replaces attention.py:175-218 flash_decode (+ PoolView.gather pool.py:394-439,
// _split_partial attention.py:168-172, merge_partials attention.py:154-165), batched
// over requests for one layer.  Work item = (request, kv head, contiguous tile range);
// a tile is one INT2 page (32 tokens) or 32 INT4 slots, so every tile is
// bitwidth-homogeneous like the reference's splits.  Softmax runs in the log2 domain
// (q is pre-scaled by scale*log2(e)); partials are (acc[d], m, l) per q head.
//
// Tensor-core kernel (variant 0), one warp = one independent flash-decoding stream:
//  * each warp owns a STAGES-deep smem ring filled by cp.async.bulk (TMA bulk copies,
//    one 3 KB copy per INT2 page, one per INT4 slot) completing on mbarriers;
//  * QK^T as S^T[token x head] = K[token x ch] . Q^T with mma.sync m16n8k16 (N = 8 =
//    the GQA group): INT2 key pages fold the per-channel scale into q (q' = q*s per
//    page) and add the per-page bias sum_c q_c z_c with one extra MMA whose A rows are
//    the zeros; INT4 keys are dequantised in registers;
//  * P goes C-fragment -> B-fragment with movmatrix;
//  * PV as O^T[ch x head] = V^T . P'^T with group-pure M tiles so the per-token
//    group scale folds into P' = p*s, and sum_t p*z comes from an MMA with A = 1;
//  * codes become fp16 with one LOP3 against the 0x3C00 exponent (1 + code*2^(p-10))
//    and an exact HSUB2, leaving code * 2^(p-10); the power of two is undone per row.
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"

namespace kvmix {

#ifndef KVMIX_STAGES
#define KVMIX_STAGES 3
#endif
#ifndef KVMIX_MINB
#define KVMIX_MINB 3
#endif
constexpr int NW = 4;                 // warps per CTA
constexpr int STAGES = KVMIX_STAGES;  // ring depth per warp
constexpr uint32_t MAGIC = 0x3C003C00u;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_SLACK = 8.f;  // see softmax_tile

template <int D>
struct Cfg {
  static constexpr int NCH = D / 16;   // QK k-chunks == PV M tiles
  static constexpr int NGRP = D / 32;  // channel groups
  static constexpr int KP = key_page_bytes(D);
  static constexpr int TB2 = tok_bytes(D, 2);
  static constexpr int TB4 = tok_bytes(D, 4);
  static constexpr int PS = page_stride(D);
  static constexpr int SS = slot_stride(D);
  static constexpr int BUF = PS > 32 * SS ? PS : 32 * SS;  // one INT2 page or 32 INT4 slots (slot-contiguous)
  static constexpr int SMEM = NW * STAGES * BUF;
};

struct DecodeArgs {
  const void* q;
  int q_dtype;
  void* out;
  int out_dtype;
  const uint8_t* int2_pool;
  const uint8_t* int4_pool;
  int64_t pool_pages, pool_int4, layer;
  int n_kv, n_q, gq, batch;
  const int32_t* page_indptr;
  const int32_t* page_ids;
  const int32_t* int4_indptr;
  const int32_t* int4_ids;
  const int32_t* work;
  int cluster;  // CTAs (splits) per (request, kv head) unit == thread-block cluster size
  float qscale;  // softmax scale * log2(e)
};

__device__ __forceinline__ float load_q(const DecodeArgs& a, int64_t idx) {
  if (a.q_dtype == KVMIX_F32) return reinterpret_cast<const float*>(a.q)[idx];
  if (a.q_dtype == KVMIX_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.q)[idx]);
  return __half2float(reinterpret_cast<const __half*>(a.q)[idx]);
}

template <int NG>
__device__ __forceinline__ void lds_params(const uint8_t* p, uint32_t (&w)[NG]) {
  if constexpr (NG == 4) {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else if constexpr (NG == 2) {
    uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
}
__device__ __forceinline__ uint32_t lds32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }

// code * 2^(2e-10) for the 2-bit field e of each half (INT2 codes in bits 2e..2e+1)
__device__ __forceinline__ uint32_t int2_field(uint32_t r, int e) {
  return hsub2u(lop_and_or(r, 0x00030003u << (2 * e), MAGIC), MAGIC);
}

// ------------------------------------------------------------------------------------
// Work-item prologue shared by both kernel variants.
struct Unit {
  int b, kvh, tlo, thi, npg, n4;
  int64_t pg0, i40;
};
__device__ __forceinline__ Unit load_unit(const DecodeArgs& a) {
  const int32_t* wk = a.work + 4 * (int64_t)blockIdx.x;
  Unit u;
  const int unit = wk[0];
  u.b = unit / a.n_kv;
  u.kvh = unit % a.n_kv;
  u.tlo = wk[1];
  u.thi = wk[2];
  u.pg0 = a.page_indptr[u.b];
  u.npg = a.page_indptr[u.b + 1] - (int)u.pg0;
  u.i40 = a.int4_indptr[u.b];
  u.n4 = a.int4_indptr[u.b + 1] - (int)u.i40;
  return u;
}

__device__ __forceinline__ void store_out(const DecodeArgs& a, int64_t oi, float v) {
  if (a.out_dtype == KVMIX_F32) reinterpret_cast<float*>(a.out)[oi] = v;
  else if (a.out_dtype == KVMIX_BF16) reinterpret_cast<__nv_bfloat16*>(a.out)[oi] = __float2bfloat16(v);
  else reinterpret_cast<__half*>(a.out)[oi] = __float2half(v);
}

// Epilogue shared by both variants (this is K3, the cross-split combine, fused in):
// 1. merge the NW warps' (m, l, acc) per head through smem into this CTA's state;
// 2. the `cluster` CTAs that split one (request, kv head) unit form a thread-block
//    cluster: after a cluster barrier, CTA rank r merges a slice of the unit's outputs
//    by reading every CTA's state through distributed shared memory (attention.py:154-165).
// No global partials, no atomics, no second launch.
template <int D>
__device__ __forceinline__ void merge_and_store(const DecodeArgs& a, const Unit& u, const float* sm_m,
                                                const float* sm_l, const float* sm_acc, float* cm, float* cl,
                                                float* cacc) {
  __syncthreads();
  for (int i = threadIdx.x; i < a.gq * D; i += blockDim.x) {
    const int hh = i / D, c = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_m[w * 8 + hh]);
    float acc = 0.f, l = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = sm_m[w * 8 + hh];
      const float f = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
      acc += f * sm_acc[(w * 8 + hh) * D + c];
      l += f * sm_l[w * 8 + hh];
    }
    if (a.cluster == 1) {
      store_out(a, ((int64_t)u.b * a.n_q + (int64_t)u.kvh * a.gq + hh) * D + c, acc / l);
    } else {
      cacc[hh * D + c] = acc;
      if (c == 0) {
        cm[hh] = M;
        cl[hh] = l;
      }
    }
  }
  if (a.cluster == 1) return;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();  // every CTA of the unit has published its state in smem
  const int ns = a.cluster, r = (int)cluster.block_rank();
  for (int i = r * blockDim.x + threadIdx.x; i < a.gq * D; i += ns * blockDim.x) {
    const int hh = i / D, c = i % D;
    float M = -INFINITY;
    for (int k = 0; k < ns; ++k) M = fmaxf(M, cluster.map_shared_rank(cm, k)[hh]);
    float acc = 0.f, l = 0.f;
    for (int k = 0; k < ns; ++k) {
      const float mk = cluster.map_shared_rank(cm, k)[hh];
      const float f = mk == -INFINITY ? 0.f : fast_exp2(mk - M);
      acc = fmaf(cluster.map_shared_rank(cacc, k)[hh * D + c], f, acc);
      l = fmaf(cluster.map_shared_rank(cl, k)[hh], f, l);
    }
    store_out(a, ((int64_t)u.b * a.n_q + (int64_t)u.kvh * a.gq + hh) * D + c, acc / l);
  }
  cluster.sync();  // keep this CTA's smem alive until all ranks have read it
}

// ====================================================================================
// Variant 0: tensor-core kernel.  Tile bodies are specialised per bitwidth so that all
// shared-memory addresses are a lane-constant base plus compile-time immediates.
struct Softmax {
  float m0, m1, l0, l1;  // running max / sum for heads 2q, 2q+1 (log2 domain)
};

template <int D>
struct Acc {
  float o[D / 16][4];  // O^T accumulators (rows = channels, cols = heads 2q, 2q+1)
  float zs[4];         // Z^T.P^T: row j (< D/32) = sum_t z_tj p_th (rows >= D/32 unused)
};

__device__ __forceinline__ uint32_t ld_s32(const uint8_t* base, int off) {
  return *reinterpret_cast<const uint32_t*>(base + off);
}

// Online softmax over one 32-token tile; returns the P^T B fragments of PV k-steps 0, 1.
template <int D>
__device__ __forceinline__ void softmax_tile(const float (&sv)[8], Softmax& st, Acc<D>& acc, uint32_t (&bP)[2][2]) {
  float tm0 = fmaxf(fmaxf(sv[0], sv[2]), fmaxf(sv[4], sv[6]));
  float tm1 = fmaxf(fmaxf(sv[1], sv[3]), fmaxf(sv[5], sv[7]));
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, off));
    tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, off));
  }
  // Lazy rescale: keep the stale running max until a tile exceeds it by > RESCALE_SLACK
  // (log2 units); p then stays <= 2^RESCALE_SLACK, well inside fp16, and the exact
  // rescale happens only when needed (rarely after the first tiles).
  if (__any_sync(0xffffffffu, (tm0 > st.m0 + RESCALE_SLACK) || (tm1 > st.m1 + RESCALE_SLACK))) {
    const float mn0 = fmaxf(st.m0, tm0), mn1 = fmaxf(st.m1, tm1);
    const float al0 = fast_exp2(st.m0 - mn0), al1 = fast_exp2(st.m1 - mn1);  // exp2(-inf) = 0
    st.l0 *= al0;
    st.l1 *= al1;
#pragma unroll
    for (int m = 0; m < D / 16; ++m) {
      acc.o[m][0] *= al0; acc.o[m][2] *= al0;
      acc.o[m][1] *= al1; acc.o[m][3] *= al1;
    }
    acc.zs[0] *= al0; acc.zs[2] *= al0;
    acc.zs[1] *= al1; acc.zs[3] *= al1;
    st.m0 = mn0;
    st.m1 = mn1;
  }
  const float mn0 = st.m0, mn1 = st.m1;
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    p[i] = fast_exp2(sv[i] - mn0);
    p[i + 1] = fast_exp2(sv[i + 1] - mn1);
  }
  st.l0 += (p[0] + p[2]) + (p[4] + p[6]);
  st.l1 += (p[1] + p[3]) + (p[5] + p[7]);
  // k index of PV == QK row: lane holds head g, rows (2q, 2q+1) / (2q+8, 2q+9)
  bP[0][0] = movtrans(pack_h2(p[0], p[1]));
  bP[0][1] = movtrans(pack_h2(p[2], p[3]));
  bP[1][0] = movtrans(pack_h2(p[4], p[5]));
  bP[1][1] = movtrans(pack_h2(p[6], p[7]));
}

// PV for one k-step and one channel group j: A = code fields of the pair-A / pair-B
// tokens (rows e = 0..3 -> channels 32j + 4g + e), B = P' = p*s.
template <int D>
__device__ __forceinline__ void pv_group(Acc<D>& acc, int j, const uint32_t (&fA)[4], const uint32_t (&fB)[4],
                                         uint32_t bP0, uint32_t bP1, uint32_t pA0, uint32_t pA1, uint32_t pB0,
                                         uint32_t pB1) {
  const uint64_t ps = pack_b64(hmul2u(bP0, prmt(pA0, pA1, 0x5410)), hmul2u(bP1, prmt(pB0, pB1, 0x5410)));
  mma16816_b64(acc.o[2 * j], fA[0], fA[1], fB[0], fB[1], ps);
  mma16816_b64(acc.o[2 * j + 1], fA[2], fA[3], fB[2], fB[3], ps);
}

// sum_t p_th z_tj for all groups j at once: A = Z^T (row g = group g&3, k = PV tokens),
// B = P^T.  zA0..zB1 are the (scale, zero) words of group g&3 of the 4 tokens.
template <int D>
__device__ __forceinline__ void pv_zeros(Acc<D>& acc, uint32_t zA0, uint32_t zA1, uint32_t zB0, uint32_t zB1,
                                         uint32_t bP0, uint32_t bP1) {
  const uint32_t zA = prmt(zA0, zA1, 0x7632), zB = prmt(zB0, zB1, 0x7632);
  // rows g+8 (a1, a3) are don't-care: feed the raw words to avoid register moves
  mma16816_b64(acc.zs, zA, zA0, zB, zB0, pack_b64(bP0, bP1));
}

// Q as B fragments of QK, fp16, NOT pre-scaled (bf16 q converts exactly).  b2: INT2 key
// pages, chunk i, lane q pairs channels (16i+4q+{0,1}) / (16i+4q+{2,3}); b4: INT4 keys,
// chunk 2j+s pairs (32j+8q+{0,4}) / ({1,5}) (s=0) or ({2,6}) / ({3,7}) (s=1).  With LO
// (fp32 q), *lo hold q - fp16(q) so the bias and INT4 products see ~22-bit q.
template <int D, bool LO>
struct QFrag {
  uint64_t b2[D / 16], b4[D / 16];
  uint64_t b2lo[LO ? D / 16 : 1], b4lo[LO ? D / 16 : 1];
};

// ---------------------------------- INT2 page tile ----------------------------------
template <int D, bool LO>
__device__ __forceinline__ void int2_tile(const uint8_t* __restrict__ buf, const QFrag<D, LO>& qf, float qscale,
                                          int lane, Softmax& st, Acc<D>& acc) {
  using C = Cfg<D>;
  const int g = lane >> 2, q = lane & 3;
  // lane g reads byte beta(g) = (g>>1) | ((g&1)<<2) of every channel word -> tokens 4beta..4beta+3
  // chunk i, lane q: k pair (2q, 2q+1) = channels 16i+4q+{0,1}, (2q+8, 2q+9) = 16i+4q+{2,3}
  const uint32_t selK = (uint32_t)(g >> 1) | ((uint32_t)(4 + (g >> 1)) << 8);
  const uint8_t* kb = buf + 32 * q + 4 * (g & 1);  // channel word 16i+4q+e: + 128 i + 8 e
  const uint8_t* pb = buf + 8 * D + 16 * q;         // (s, z) of channels 16i+4q+{0..3}: + 64 i
  float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f}, cb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < C::NCH; ++i) {
    const uint32_t r1 = prmt(ld_s32(kb, 128 * i), ld_s32(kb, 128 * i + 8), selK);
    const uint32_t r2 = prmt(ld_s32(kb, 128 * i + 16), ld_s32(kb, 128 * i + 24), selK);
    const uint4 pv = *reinterpret_cast<const uint4*>(pb + 64 * i);
    const uint64_t qi = qf.b2[i];
    const uint64_t qs = pack_b64(hmul2u(lo32(qi), prmt(pv.x, pv.y, 0x5410)), hmul2u(hi32(qi), prmt(pv.z, pv.w, 0x5410)));
    const uint32_t z1 = prmt(pv.x, pv.y, 0x7632), z2 = prmt(pv.z, pv.w, 0x7632);
    mma16816_b64(c0, int2_field(r1, 0), int2_field(r1, 1), int2_field(r2, 0), int2_field(r2, 1), qs);
    mma16816_b64(c1, int2_field(r1, 2), int2_field(r1, 3), int2_field(r2, 2), int2_field(r2, 3), qs);
    // bias rows g carry sum_c q_c z_c; rows g+8 (cb[2], cb[3]) are don't-care filler
    mma16816_b64(cb, z1, r1, z2, r2, qi);
    if constexpr (LO) mma16816_b64(cb, z1, r1, z2, r2, qf.b2lo[i]);
  }
  // undo 2^(2k-10) per token row (k = token position inside its code byte), apply scale*log2(e)
  const float b0 = cb[0] * qscale, b1 = cb[1] * qscale;
  const float sv[8] = {fmaf(c0[0], 1024.f * qscale, b0), fmaf(c0[1], 1024.f * qscale, b1),
                       fmaf(c0[2], 256.f * qscale, b0),  fmaf(c0[3], 256.f * qscale, b1),
                       fmaf(c1[0], 64.f * qscale, b0),   fmaf(c1[1], 64.f * qscale, b1),
                       fmaf(c1[2], 16.f * qscale, b0),   fmaf(c1[3], 16.f * qscale, b1)};
  uint32_t bP[2][2];
  softmax_tile<D>(sv, st, acc, bP);
  // PV: k-step ks, pair A tokens (4q+2ks, 16+4q+2ks), pair B = pair A + 1
  const uint32_t selV = (uint32_t)(g & 3) | ((uint32_t)(4 + (g & 3)) << 8);
  const uint8_t* vb = buf + C::KP + C::TB2 * 4 * q;  // token 4q's V block
  const uint8_t* vc = vb + 4 * (g >> 2);             // + 8j: word of byte 8j+g
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    constexpr int T = C::TB2;
    uint32_t pA0[C::NGRP], pA1[C::NGRP], pB0[C::NGRP], pB1[C::NGRP];
    lds_params<C::NGRP>(vb + (2 * ks) * T + D / 4, pA0);
    lds_params<C::NGRP>(vb + (16 + 2 * ks) * T + D / 4, pA1);
    lds_params<C::NGRP>(vb + (2 * ks + 1) * T + D / 4, pB0);
    lds_params<C::NGRP>(vb + (17 + 2 * ks) * T + D / 4, pB1);
    {
      const uint8_t* zb = vb + D / 4 + 4 * (g & (C::NGRP - 1));
      pv_zeros<D>(acc, ld_s32(zb, (2 * ks) * T), ld_s32(zb, (16 + 2 * ks) * T), ld_s32(zb, (2 * ks + 1) * T),
                  ld_s32(zb, (17 + 2 * ks) * T), bP[ks][0], bP[ks][1]);
    }
#pragma unroll
    for (int j = 0; j < C::NGRP; ++j) {
      const uint32_t rA = prmt(ld_s32(vc, (2 * ks) * T + 8 * j), ld_s32(vc, (16 + 2 * ks) * T + 8 * j), selV);
      const uint32_t rB = prmt(ld_s32(vc, (2 * ks + 1) * T + 8 * j), ld_s32(vc, (17 + 2 * ks) * T + 8 * j), selV);
      uint32_t fA[4], fB[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        fA[e] = int2_field(rA, e);
        fB[e] = int2_field(rB, e);
      }
      pv_group<D>(acc, j, fA, fB, bP[ks][0], bP[ks][1], pA0[j], pA1[j], pB0[j], pB1[j]);
    }
  }
}

// ---------------------------------- INT4 slot tile ----------------------------------
__device__ __forceinline__ uint32_t int4_deq(uint32_t field16, uint32_t s16, uint32_t zz) {
  return hfma2u(hsub2u(field16, MAGIC), s16, zz);  // (code/16) * 16s + z
}

template <int D, bool FULL, bool LO>
__device__ __forceinline__ void int4_tile(const uint8_t* __restrict__ buf, int nv, const QFrag<D, LO>& qf,
                                          float qscale, int lane, Softmax& st, Acc<D>& acc) {
  using C = Cfg<D>;
  constexpr int S = C::SS;
  const int g = lane >> 2, q = lane & 3;
  // QK row g of M tile m is slot 16m + beta(g), row g+8 is slot 16m + 8 + beta(g), with
  // beta(g) = (g>>1) | ((g&1)<<2): PV lanes then read 4 slots 1 apart (conflict-free V loads)
  const int beta = (g >> 1) | ((g & 1) << 2);
  const uint8_t* kb = buf + S * beta + 4 * q;  // slot row r: + S*(16(r>>1) + 8(r&1)); group j: + 16j
  const uint8_t* kp = buf + S * beta + D / 2;  // K params of the slot: + 4j
  float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < C::NGRP; ++j) {
    uint32_t e[4][4];  // [slot row: M0 g, M0 g+8, M1 g, M1 g+8][field]
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int ro = S * (16 * (r >> 1) + 8 * (r & 1));
      const uint32_t w = ld_s32(kb, ro + 16 * j);
      const uint32_t par = ld_s32(kp, ro + 4 * j);
      const uint32_t s16 = hmul2u(prmt(par, par, 0x1010), 0x4C004C00u);  // (16s, 16s)
      const uint32_t zz = prmt(par, par, 0x3232);
      e[r][0] = int4_deq(lop_and_or(w << 6, 0x03C003C0u, MAGIC), s16, zz);
      e[r][1] = int4_deq(lop_and_or(w << 2, 0x03C003C0u, MAGIC), s16, zz);
      e[r][2] = int4_deq(lop_and_or(w >> 2, 0x03C003C0u, MAGIC), s16, zz);
      e[r][3] = int4_deq(lop_and_or(w >> 6, 0x03C003C0u, MAGIC), s16, zz);
    }
    const uint64_t qa = qf.b4[2 * j], qc = qf.b4[2 * j + 1];
    mma16816_b64(c0, e[0][0], e[1][0], e[0][1], e[1][1], qa);
    mma16816_b64(c0, e[0][2], e[1][2], e[0][3], e[1][3], qc);
    mma16816_b64(c1, e[2][0], e[3][0], e[2][1], e[3][1], qa);
    mma16816_b64(c1, e[2][2], e[3][2], e[2][3], e[3][3], qc);
    if constexpr (LO) {
      const uint64_t la = qf.b4lo[2 * j], lc = qf.b4lo[2 * j + 1];
      mma16816_b64(c0, e[0][0], e[1][0], e[0][1], e[1][1], la);
      mma16816_b64(c0, e[0][2], e[1][2], e[0][3], e[1][3], lc);
      mma16816_b64(c1, e[2][0], e[3][0], e[2][1], e[3][1], la);
      mma16816_b64(c1, e[2][2], e[3][2], e[2][3], e[3][3], lc);
    }
  }
  float sv[8] = {c0[0] * qscale, c0[1] * qscale, c0[2] * qscale, c0[3] * qscale,
                 c1[0] * qscale, c1[1] * qscale, c1[2] * qscale, c1[3] * qscale};
  if (!FULL) {
    if (beta >= nv) sv[0] = sv[1] = -INFINITY;
    if (beta + 8 >= nv) sv[2] = sv[3] = -INFINITY;
    if (beta + 16 >= nv) sv[4] = sv[5] = -INFINITY;
    if (beta + 24 >= nv) sv[6] = sv[7] = -INFINITY;
  }
  uint32_t bP[2][2];
  softmax_tile<D>(sv, st, acc, bP);
  const uint32_t b4 = 2 * (g & 1);
  const uint32_t selV = b4 | ((b4 + 1) << 4) | ((b4 + 4) << 8) | ((b4 + 5) << 12);
  // PV k-step ks: pair A = QK rows (2q, 2q+1) = slots 16ks + q, 16ks + q + 4; pair B = + 8
  const uint8_t* vb = buf + S * q + C::TB4;  // slot q's V block
  const uint8_t* vc = vb + 4 * (g >> 1);     // + 16j: word holding bytes 16j+2g, +1
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    uint32_t pA0[C::NGRP], pA1[C::NGRP], pB0[C::NGRP], pB1[C::NGRP];
    lds_params<C::NGRP>(vb + S * (16 * ks) + D / 2, pA0);
    lds_params<C::NGRP>(vb + S * (16 * ks + 4) + D / 2, pA1);
    lds_params<C::NGRP>(vb + S * (16 * ks + 8) + D / 2, pB0);
    lds_params<C::NGRP>(vb + S * (16 * ks + 12) + D / 2, pB1);
    if (!FULL) {
      const int sA0 = 16 * ks + q;
#pragma unroll
      for (int j = 0; j < C::NGRP; ++j) {
        if (sA0 >= nv) pA0[j] = 0u;
        if (sA0 + 4 >= nv) pA1[j] = 0u;
        if (sA0 + 8 >= nv) pB0[j] = 0u;
        if (sA0 + 12 >= nv) pB1[j] = 0u;
      }
    }
    {
      const uint8_t* zb = vb + D / 2 + 4 * (g & (C::NGRP - 1));
      uint32_t zA0 = ld_s32(zb, S * (16 * ks)), zA1 = ld_s32(zb, S * (16 * ks + 4));
      uint32_t zB0 = ld_s32(zb, S * (16 * ks + 8)), zB1 = ld_s32(zb, S * (16 * ks + 12));
      if (!FULL) {
        const int sA0 = 16 * ks + q;
        if (sA0 >= nv) zA0 = 0u;
        if (sA0 + 4 >= nv) zA1 = 0u;
        if (sA0 + 8 >= nv) zB0 = 0u;
        if (sA0 + 12 >= nv) zB1 = 0u;
      }
      pv_zeros<D>(acc, zA0, zA1, zB0, zB1, bP[ks][0], bP[ks][1]);
    }
#pragma unroll
    for (int j = 0; j < C::NGRP; ++j) {
      const uint32_t rA = prmt(ld_s32(vc, S * (16 * ks) + 16 * j), ld_s32(vc, S * (16 * ks + 4) + 16 * j), selV);
      const uint32_t rB = prmt(ld_s32(vc, S * (16 * ks + 8) + 16 * j), ld_s32(vc, S * (16 * ks + 12) + 16 * j), selV);
      uint32_t fA[4], fB[4];
      fA[0] = hsub2u(lop_and_or(rA, 0x000F000Fu, MAGIC), MAGIC);
      fA[1] = hsub2u(lop_and_or(rA >> 2, 0x003C003Cu, MAGIC), MAGIC);
      fA[2] = hsub2u(lop_and_or(rA >> 4, 0x00F000F0u, MAGIC), MAGIC);
      fA[3] = hsub2u(lop_and_or(rA >> 6, 0x03C003C0u, MAGIC), MAGIC);
      fB[0] = hsub2u(lop_and_or(rB, 0x000F000Fu, MAGIC), MAGIC);
      fB[1] = hsub2u(lop_and_or(rB >> 2, 0x003C003Cu, MAGIC), MAGIC);
      fB[2] = hsub2u(lop_and_or(rB >> 4, 0x00F000F0u, MAGIC), MAGIC);
      fB[3] = hsub2u(lop_and_or(rB >> 6, 0x03C003C0u, MAGIC), MAGIC);
      pv_group<D>(acc, j, fA, fB, bP[ks][0], bP[ks][1], pA0[j], pA1[j], pB0[j], pB1[j]);
    }
  }
}

template <int D, bool COMPUTE = true, bool MEMORY = true, bool LO = false>
__global__ void __launch_bounds__(NW * 32, KVMIX_MINB) decode_mma_kernel(const DecodeArgs a) {
  using C = Cfg<D>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[NW][STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const Unit u = load_unit(a);
  uint8_t* ring = smem + warp * STAGES * C::BUF;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int ntiles = u.thi - u.tlo;
  const int nmine = ntiles > warp ? (ntiles - warp + NW - 1) / NW : 0;
  const uint8_t* kv2 = a.int2_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_pages) * (int64_t)C::PS;
  const uint8_t* kv4 = a.int4_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_int4) * (int64_t)C::SS;

  // tile metadata: the page id (INT2 tile) or this lane's slot (INT4 tile); loaded one
  // iteration before its copy is issued so the copy never waits on the index load
  auto load_meta = [&](int k) -> int {
    if (k >= nmine) return 0;
    const int t = u.tlo + warp + k * NW;
    if (t < u.npg) return a.page_ids[u.pg0 + t];
    const int it = t - u.npg;
    return lane < min(32, u.n4 - 32 * it) ? a.int4_ids[u.i40 + 32 * it + lane] : 0;
  };
  auto issue = [&](int k, int meta, int s) {
    const int t = u.tlo + warp + k * NW;
    uint8_t* buf = ring + s * C::BUF;
    uint64_t* bar = &bars[warp][s];
    if (t < u.npg) {
      if (lane == 0) {
        mbar_expect_tx(bar, C::PS);
        bulk_g2s(buf, kv2 + (int64_t)meta * C::PS, C::PS, bar);
      }
    } else {
      // one bulk copy per run of consecutive INT4 slots (fresh pools give long runs)
      const int nv = min(32, u.n4 - 32 * (t - u.npg));
      const int prev = __shfl_up_sync(0xffffffffu, meta, 1);
      const bool start = lane < nv && (lane == 0 || meta != prev + 1);
      const uint32_t starts = __ballot_sync(0xffffffffu, start);
      if (lane == 0) mbar_expect_tx(bar, nv * C::SS);
      __syncwarp();
      if (start) {
        const uint32_t later = starts & ~((2u << lane) - 1u);
        const int end = later ? __ffs(later) - 1 : nv;
        bulk_g2s(buf + lane * C::SS, kv4 + (int64_t)meta * C::SS, (end - lane) * C::SS, bar);
      }
    }
  };
  if (MEMORY) {
    int s0 = 0;
    for (int k = 0; k < STAGES && k < nmine; ++k) issue(k, load_meta(k), s0++);
  }
  int meta_next = load_meta(STAGES);

  // ---- Q fragments (see QFrag) ----
  QFrag<D, LO> qf;
  {
    const bool hv = g < a.gq;
    const int64_t qrow = ((int64_t)u.b * a.n_q + (int64_t)u.kvh * a.gq + (hv ? g : 0)) * D;
    auto qv = [&](int c) { return hv ? load_q(a, qrow + c) : 0.f; };
    auto lo = [](float x) { return x - __half2float(__float2half_rn(x)); };
#pragma unroll
    for (int i = 0; i < C::NCH; ++i) {
      const int c2 = 16 * i + 4 * q;
      const int b4 = 32 * (i >> 1) + 8 * q + 2 * (i & 1);
      const float x0 = qv(c2), x1 = qv(c2 + 1), x2 = qv(c2 + 2), x3 = qv(c2 + 3);
      const float y0 = qv(b4), y1 = qv(b4 + 4), y2 = qv(b4 + 1), y3 = qv(b4 + 5);
      qf.b2[i] = pack_b64(pack_h2(x0, x1), pack_h2(x2, x3));
      qf.b4[i] = pack_b64(pack_h2(y0, y1), pack_h2(y2, y3));
      if constexpr (LO) {
        qf.b2lo[i] = pack_b64(pack_h2(lo(x0), lo(x1)), pack_h2(lo(x2), lo(x3)));
        qf.b4lo[i] = pack_b64(pack_h2(lo(y0), lo(y1)), pack_h2(lo(y2), lo(y3)));
      }
    }
  }

  Acc<D> acc;
#pragma unroll
  for (int m = 0; m < C::NCH; ++m) acc.o[m][0] = acc.o[m][1] = acc.o[m][2] = acc.o[m][3] = 0.f;
  acc.zs[0] = acc.zs[1] = acc.zs[2] = acc.zs[3] = 0.f;
  Softmax st{-INFINITY, -INFINITY, 0.f, 0.f};

  int stage = 0;
  uint32_t phase = 0;
  for (int k = 0; k < nmine; ++k) {
    const int t = u.tlo + warp + k * NW;
    const uint8_t* buf = ring + stage * C::BUF;
    const int meta = meta_next;
    meta_next = load_meta(k + STAGES + 1);
    if (MEMORY) mbar_wait(&bars[warp][stage], phase);
    if (!COMPUTE) {
      // measurement variant: data movement only (no dequant / MMA)
    } else if (t < u.npg) {
      int2_tile<D, LO>(buf, qf, a.qscale, lane, st, acc);
    } else {
      const int nv = min(32, u.n4 - 32 * (t - u.npg));
      if (nv == 32) int4_tile<D, true, LO>(buf, 32, qf, a.qscale, lane, st, acc);
      else int4_tile<D, false, LO>(buf, nv, qf, a.qscale, lane, st, acc);
    }
    __syncwarp();
    if (MEMORY && k + STAGES < nmine) {
      fence_proxy_async();
      issue(k + STAGES, meta, stage);
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1u;
    }
  }

  // ---- finalize this warp: full l per head, acc[h][c] = 2^(10-2e) * O^T + zsum ----
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    st.l0 += __shfl_xor_sync(0xffffffffu, st.l0, off);
    st.l1 += __shfl_xor_sync(0xffffffffu, st.l1, off);
  }
  __syncthreads();  // all warps done with their rings -> reuse smem for the merge
  float* sm_acc = reinterpret_cast<float*>(smem);
  float* sm_m = sm_acc + NW * 8 * D;
  float* sm_l = sm_m + NW * 8;
  float* cta_acc = sm_l + NW * 8;  // this CTA's merged state, read by the cluster
  float* cta_m = cta_acc + 8 * D;
  float* cta_l = cta_m + 8;
  float z0[C::NGRP], z1[C::NGRP];  // sum_t p z of group j for heads 2q, 2q+1 (from lane (j, q))
#pragma unroll
  for (int j = 0; j < C::NGRP; ++j) {
    z0[j] = __shfl_sync(0xffffffffu, acc.zs[0], 4 * j + q);
    z1[j] = __shfl_sync(0xffffffffu, acc.zs[1], 4 * j + q);
  }
#pragma unroll
  for (int m = 0; m < C::NCH; ++m) {
    const int j = m >> 1;
    const int e0 = 2 * (m & 1);
    const int ch0 = 32 * j + 4 * g + e0;
    const float f0 = (float)(1 << (10 - 2 * e0)), f1 = (float)(1 << (10 - 2 * (e0 + 1)));
    sm_acc[(warp * 8 + 2 * q) * D + ch0] = fmaf(acc.o[m][0], f0, z0[j]);
    sm_acc[(warp * 8 + 2 * q + 1) * D + ch0] = fmaf(acc.o[m][1], f0, z1[j]);
    sm_acc[(warp * 8 + 2 * q) * D + ch0 + 1] = fmaf(acc.o[m][2], f1, z0[j]);
    sm_acc[(warp * 8 + 2 * q + 1) * D + ch0 + 1] = fmaf(acc.o[m][3], f1, z1[j]);
  }
  if (g == 0) {
    sm_m[warp * 8 + 2 * q] = st.m0;
    sm_m[warp * 8 + 2 * q + 1] = st.m1;
    sm_l[warp * 8 + 2 * q] = st.l0;
    sm_l[warp * 8 + 2 * q + 1] = st.l1;
  }
  merge_and_store<D>(a, u, sm_m, sm_l, sm_acc, cta_m, cta_l, cta_acc);
}

// ====================================================================================
// Variant 1: simple CUDA-core kernel (fp32 dequant straight from HBM).  Slow; kept as
// an independent on-GPU cross-check of the tensor-core kernel at full sizes.
template <int D>
__global__ void __launch_bounds__(NW * 32) decode_simple_kernel(const DecodeArgs a) {
  constexpr int CPL = D / 32;
  __shared__ float qs[8][D];
  __shared__ float sm_acc[NW * 8 * D];
  __shared__ float sm_m[NW * 8], sm_l[NW * 8];
  __shared__ float cta_acc[8 * D], cta_m[8], cta_l[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const Unit u = load_unit(a);
  for (int i = threadIdx.x; i < 8 * D; i += blockDim.x) {
    const int hh = i / D, c = i % D;
    qs[hh][c] = hh < a.gq ? load_q(a, ((int64_t)u.b * a.n_q + (int64_t)u.kvh * a.gq + hh) * D + c) * a.qscale : 0.f;
  }
  __syncthreads();
  float m[8], l[8], acc[8][CPL];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc[h][i] = 0.f;
  }
  const uint8_t* kv2 = a.int2_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_pages) * (int64_t)page_stride(D);
  const uint8_t* kv4 = a.int4_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_int4) * (int64_t)slot_stride(D);
  auto deq = [](const uint8_t* blk, int c, int bits) {
    const uint32_t code = (blk[c * bits / 8] >> ((c * bits) & 7)) & ((1u << bits) - 1);
    const __half2 pz = *reinterpret_cast<const __half2*>(blk + D * bits / 8 + 4 * (c / G));
    return fmaf((float)code, __low2float(pz), __high2float(pz));
  };
  for (int t = u.tlo + warp; t < u.thi; t += NW) {
    const bool is2 = t < u.npg;
    const int nrow = is2 ? G : min(32, u.n4 - 32 * (t - u.npg));
    for (int r = 0; r < nrow; ++r) {
      float kx[CPL], vx[CPL];
      if (is2) {
        const uint8_t* rec = kv2 + (int64_t)a.page_ids[u.pg0 + t] * page_stride(D);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const int c = lane + 32 * i;
          const uint32_t code = (rec[8 * c + r / 4] >> (2 * (r & 3))) & 3u;
          const __half2 pz = *reinterpret_cast<const __half2*>(rec + 8 * D + 4 * c);
          kx[i] = fmaf((float)code, __low2float(pz), __high2float(pz));
          vx[i] = deq(rec + key_page_bytes(D) + r * tok_bytes(D, 2), c, 2);
        }
      } else {
        const int64_t slot = a.int4_ids[u.i40 + 32 * (t - u.npg) + r];
        const uint8_t* rec = kv4 + slot * slot_stride(D);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const int c = lane + 32 * i;
          kx[i] = deq(rec, c, 4);
          vx[i] = deq(rec + tok_bytes(D, 4), c, 4);
        }
      }
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        if (h >= a.gq) continue;
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < CPL; ++i) s = fmaf(qs[h][lane + 32 * i], kx[i], s);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        const float mn = fmaxf(m[h], s);
        const float al = exp2f(m[h] - mn), pv = exp2f(s - mn);
        m[h] = mn;
        l[h] = l[h] * al + pv;
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[h][i] = fmaf(acc[h][i], al, pv * vx[i]);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 8; ++h) {
#pragma unroll
    for (int i = 0; i < CPL; ++i) sm_acc[(warp * 8 + h) * D + lane + 32 * i] = acc[h][i];
    if (lane == 0) {
      sm_m[warp * 8 + h] = m[h];
      sm_l[warp * 8 + h] = l[h];
    }
  }
  merge_and_store<D>(a, u, sm_m, sm_l, sm_acc, cta_m, cta_l, cta_acc);
}

template <typename Kern>
static int launch_kernel(Kern kern, const DecodeArgs& a, int64_t n_work, int smem, cudaStream_t s) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_work);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
  return check_launch("flash_decode");
}

template <int D>
static int launch_decode(const DecodeArgs& a, int64_t n_work, int variant, cudaStream_t s) {
  switch (variant) {
    case 0:
      // fp32 q carries bits fp16 cannot hold: add the q - fp16(q) correction MMAs
      if (a.q_dtype == KVMIX_F32) return launch_kernel(decode_mma_kernel<D, true, true, true>, a, n_work, Cfg<D>::SMEM, s);
      return launch_kernel(decode_mma_kernel<D, true, true, false>, a, n_work, Cfg<D>::SMEM, s);
    case 1: return launch_kernel(decode_simple_kernel<D>, a, n_work, 0, s);
    case 2: return launch_kernel(decode_mma_kernel<D, false, true>, a, n_work, Cfg<D>::SMEM, s);
    default: return launch_kernel(decode_mma_kernel<D, true, false>, a, n_work, Cfg<D>::SMEM, s);
  }
}

// merge_partials (attention.py:154-165) for host-supplied partials, natural-log domain.
__global__ void merge_partials_kernel(const float* __restrict__ acc, const float* __restrict__ lse,
                                      const float* __restrict__ mx, int64_t n, int64_t d, float* __restrict__ out) {
  float M = -INFINITY;
  for (int64_t i = 0; i < n; ++i) M = fmaxf(M, mx[i]);
  float z = 0.f;
  for (int64_t i = 0; i < n; ++i) z += expf(lse[i] - M);
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    float a = 0.f;
    for (int64_t i = 0; i < n; ++i) a += acc[i * d + c] * expf(mx[i] - M);
    out[c] = a / z;
  }
}

}  // namespace kvmix

using namespace kvmix;

extern "C" int kvmix_merge_partials(const float* acc, const float* lse, const float* mx, int64_t n, int64_t d,
                                    float* out, void* stream) {
  if (n <= 0) return fail(KVMIX_EINVAL, "cannot merge an empty partial list");
  merge_partials_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(acc, lse, mx, n, d, out);
  return check_launch("merge_partials");
}

extern "C" int kvmix_flash_decode(const void* q, int32_t q_dtype, void* out, int32_t out_dtype,
                                  const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages,
                                  int64_t pool_int4, int64_t layer, int64_t n_kv, int64_t d, int64_t n_q,
                                  int64_t batch, const int32_t* page_indptr, const int32_t* page_ids,
                                  const int32_t* int4_indptr, const int32_t* int4_ids, const int32_t* work,
                                  int64_t n_work, float scale, int32_t variant, void* stream) {
  if (n_kv <= 0 || n_q % n_kv) return fail(KVMIX_EINVAL, "n_heads not a multiple of the pool's n_kv_heads");
  const int64_t gq = n_q / n_kv;
  if (gq > 8) return fail(KVMIX_EINVAL, "GQA group > 8 not supported");
  if (batch <= 0 || n_work <= 0) return fail(KVMIX_EINVAL, "empty batch or work list");
  const int64_t units = batch * n_kv;
  if (n_work % units || n_work / units > 8)
    return fail(KVMIX_EINVAL, "work list must hold 1..8 splits per (request, kv head), unit-major");
  if (q_dtype < 0 || q_dtype > 2 || out_dtype < 0 || out_dtype > 2) return fail(KVMIX_EINVAL, "bad dtype");
  if (variant < 0 || variant > 3) return fail(KVMIX_EINVAL, "bad variant");
  DecodeArgs a;
  a.q = q;
  a.q_dtype = q_dtype;
  a.out = out;
  a.out_dtype = out_dtype;
  a.int2_pool = int2_pool;
  a.int4_pool = int4_pool;
  a.pool_pages = pool_pages;
  a.pool_int4 = pool_int4;
  a.layer = layer;
  a.n_kv = (int)n_kv;
  a.n_q = (int)n_q;
  a.gq = (int)gq;
  a.batch = (int)batch;
  a.page_indptr = page_indptr;
  a.page_ids = page_ids;
  a.int4_indptr = int4_indptr;
  a.int4_ids = int4_ids;
  a.work = work;
  a.cluster = (int)(n_work / units);
  a.qscale = scale * LOG2E;
  cudaStream_t s = (cudaStream_t)stream;
  switch (d) {
    case 32: return launch_decode<32>(a, n_work, variant, s);
    case 64: return launch_decode<64>(a, n_work, variant, s);
    case 128: return launch_decode<128>(a, n_work, variant, s);
    default: return fail(KVMIX_EINVAL, "decode supports head_dim 32, 64, 128");
  }
}
