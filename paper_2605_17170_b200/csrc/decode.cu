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
//    one 2.75 KB copy per INT2 page -- the record minus its trailing key zeros -- and one
//    per run of consecutive INT4 slots) completing on mbarriers;
//  * QK^T as S^T[token x head] = K[token x ch] . Q^T with mma.sync m16n8k16 (N = 8 =
//    the GQA group): INT2 key pages fold the per-channel scale into q (q' = q*s per page,
//    as an exact fp16 hi + lo pair: two MMAs per chunk) over key codes made NORMAL fp16 by
//    the hardware e4m3x2 -> f16x2 conversion; the per-page bias sum_c q_c z_c is batched
//    over 16 pages (their zero points staged into the merge scratch by bulk copies, A rows =
//    pages); INT4 keys are dequantised per group in fp32;
//  * P goes C-fragment -> B-fragment with movmatrix;
//  * PV as O^T[ch x head] = V^T . P'^T with group-pure M tiles so the per-token group scale
//    folds into P' = p*s; value codes enter in place as fp16 subnormals (one LOP3 per two
//    codes), the power of two undone per row; sum_t p*z and the softmax sum come from one
//    MMA per k-step with A = the zeros / ones;
//  * the piece epilogue merges the warps' states with float4 smem reads (a thread per four
//    channels of one head) and stores the output -- into up to 8 destinations for the fused
//    KV-head all-gather -- or a partial that the unit's last-arriving CTA combines.
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"

namespace kvmix {

#ifndef KVMIX_STAGES
#define KVMIX_STAGES 2
#endif
#ifndef KVMIX_MINB
#define KVMIX_MINB 3
#endif
#ifndef KVMIX_SPLIT
#define KVMIX_SPLIT 0
#endif
#ifndef KVMIX_META2
#define KVMIX_META2 1  // tile metadata two tiles ahead (0: one tile ahead)
#endif
#ifndef KVMIX_TILEFENCE
#define KVMIX_TILEFENCE 1  // proxy fence before every tile copy (0: measured +0.3%, within noise; kept for safety)
#endif
#ifndef KVMIX_LAZYPARAM
#define KVMIX_LAZYPARAM 1  // 1: INT2 key scale/zero quads loaded per chunk pair (fewer live registers)
#endif
#ifndef KVMIX_NW
#define KVMIX_NW 4
#endif
constexpr int NW = KVMIX_NW;          // warps per CTA
constexpr int STAGES = KVMIX_STAGES;  // ring depth per warp
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_SLACK = 8.f;  // largest lazy-rescale slack (log2 units), see softmax_p
#ifndef KVMIX_INT4_RUNS
#define KVMIX_INT4_RUNS 32  // > 32 never: INT4 tiles with more runs would be copied by per-lane cp.async (4: churned pools +10%, fresh pools -1.6%)
#endif
#ifndef KVMIX_Q2EXACT
#define KVMIX_Q2EXACT 1  // INT2 key pages: q*s as an exact fp16 hi + lo pair (two MMAs per chunk)
#endif
#ifndef KVMIX_KZBATCH
#define KVMIX_KZBATCH 1  // INT2 key bias sum_c q_c z_c for 16 pages per NCH MMAs (0: NCH MMAs per page)
#endif
#ifndef KVMIX_Q2ACC
#define KVMIX_Q2ACC 1  // 1: the lo MMAs accumulate into the hi accumulators (fewer registers, longer chains)
#endif

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
  static constexpr int QTAB = (4 * NCH + 2) * 32 * 8;             // q fragment table (LO size)
  static constexpr int MERGE = (NW * 8 * D + 2 * NW * 8) * 4;     // per-warp (acc, m, l) for the piece merge
  // MERGE_IN_RING: the piece merge reuses the (idle) ring, so 4 CTAs fit per SM; the next
  // piece's first copies then start after the merge instead of during it.
  static constexpr bool MERGE_IN_RING = KVMIX_MINB >= 4;
  static_assert(!MERGE_IN_RING || MERGE <= NW * STAGES * BUF, "merge scratch must fit in the ring");
  // batched key bias: per warp, the KZ regions (2D bytes) of its next 16 INT2 pages; they live
  // in the merge scratch (idle during the tile loop) unless the merge itself lives in the ring
  static constexpr int KZB = 2 * D;
  static constexpr int KZS = KVMIX_KZBATCH ? NW * 16 * KZB : 0;
  static constexpr bool KZ_IN_MERGE = !MERGE_IN_RING && KZS <= MERGE;
  static constexpr int QS = D + 4;                                // raw q row stride (floats; 4-way LDS conflicts at most)
  static constexpr int QRAW = 8 * QS * 4;                          // the unit's raw q [8 heads][D] (fp32) for build_qtab
  static constexpr int SMEM = NW * STAGES * BUF + QTAB + (MERGE_IN_RING ? 0 : MERGE) + QRAW + (KZ_IN_MERGE ? 0 : KZS);
};

constexpr int MAX_OUTS = 8;  // destinations of the fused head all-gather (one NVLink domain)

struct DecodeArgs {
  const void* q;
  int q_dtype;
  // Outputs: head h of request b goes to element ((b * out_heads + out_head0 + h) * D + c) of
  // every outs[0 .. n_outs): this process's own buffer and, for the KV-head-parallel combine,
  // the peers' buffers mapped over NVLink (kvmix_flash_decode_gather).  Plain decode: one
  // destination, out_heads = n_q, out_head0 = 0.
  void* outs[MAX_OUTS];
  int n_outs, out_heads, out_head0;
  int out_dtype;
  const uint8_t* int2_pool;
  const uint8_t* int4_pool;
  int64_t pool_pages, pool_int4, layer;
  int n_kv, n_q, gq, batch;
  const int32_t* page_indptr;
  const int32_t* page_ids;
  const int32_t* int4_indptr;
  const int32_t* int4_ids;
  const int32_t* int4_count;  // NULL: CSR (count = indptr[b+1] - indptr[b]); else padded lists (K7)
  const int32_t* work;     // pieces [n][8]: unit, tile_lo, tile_hi, slot (-1: whole unit), part0, nparts
  const int32_t* cta_ptr;  // [grid + 1]: pieces of CTA i are cta_ptr[i] .. cta_ptr[i+1]
  float* part;             // split partials [n_parts][8][D + 4] (acc[D], m, l, pad; log2 domain)
  int32_t* counters;       // [batch * n_kv] arrival counters, zero between launches
  float qscale;            // softmax scale * log2(e)
  // K4 fused decode append (variant 0): each request's newest token -- the last INT4 entry of
  // its table -- is quantized from app_k / app_v [batch][n_kv][D] (app_dtype) by the warp
  // that owns its tile, into that tile's staged record and into the pool (int4_pool_w).
  const void* app_k;
  const void* app_v;
  int app_dtype;
  uint8_t* int4_pool_w;
  // Pool status words (kvmix_b200.h KVMIX_POOL_STATUS_*): the largest INT2 key-page scale
  // and V scale ever written bound the fp16 operands q' = q*s_k and P' = p*s_v (see
  // Softmax::slack, build_qtab); NULL = no bound known (safe settings).
  int32_t* pool_status;
  int flags;  // KVMIX_DECODE_POOL_WRITTEN: wait for the previous kernel before the first KV copies
};

__device__ __forceinline__ float load_q(const DecodeArgs& a, int64_t idx) {
  if (a.q_dtype == KVMIX_F32) return reinterpret_cast<const float*>(a.q)[idx];
  if (a.q_dtype == KVMIX_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.q)[idx]);
  return __half2float(reinterpret_cast<const __half*>(a.q)[idx]);
}

// ------------------------------------------------------------------------------------
// A piece is a contiguous tile range of one (request, kv head) unit; a CTA runs the pieces
// of its byte-balanced share of the whole batch (stream-K style, plan.py).
struct Unit {
  int b, kvh, unit, tlo, thi, npg, n4, slot, part0, nparts;
  int64_t pg0, i40;
};
__device__ __forceinline__ Unit load_unit(const DecodeArgs& a, int piece) {
  const int32_t* wk = a.work + 8 * (int64_t)piece;
  Unit u;
  u.unit = wk[0];
  u.b = u.unit / a.n_kv;
  u.kvh = u.unit % a.n_kv;
  u.tlo = wk[1];
  u.thi = wk[2];
  u.slot = wk[3];
  u.part0 = wk[4];
  u.nparts = wk[5];
  u.pg0 = a.page_indptr[u.b];
  u.npg = a.page_indptr[u.b + 1] - (int)u.pg0;
  u.i40 = a.int4_indptr[u.b];
  u.n4 = a.int4_count ? a.int4_count[u.b] : a.int4_indptr[u.b + 1] - (int)u.i40;
  return u;
}

// Four consecutive outputs (oi % 4 == 0) with one vector store per destination.
__device__ __forceinline__ void store_out4(const DecodeArgs& a, int64_t oi, float4 v) {
  uint2 h;
  if (a.out_dtype == KVMIX_BF16) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    h = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
  } else if (a.out_dtype == KVMIX_F16) {
    const __half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
    h = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
  }
#pragma unroll
  for (int p = 0; p < MAX_OUTS; ++p) {  // static indices: the pointers stay in the parameter bank
    if (p >= a.n_outs) break;
    if (a.out_dtype == KVMIX_F32) *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.outs[p]) + oi) = v;
    else *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.outs[p]) + oi) = h;
  }
}

// Piece epilogue shared by both variants (K3, the cross-split combine, is fused in):
// 1. merge the NW warps' (m, l, acc) per head (smem, written by the caller) into the CTA's
//    state (attention.py:154-165, log2 domain);
// 2. a piece that covers its whole unit stores the output; otherwise the CTA writes its
//    partial to slot u.slot, and the last of the unit's u.nparts CTAs to arrive (global
//    arrival counter, reset by that CTA for the next launch) merges them and stores.
template <int D>
__device__ __forceinline__ void finish_piece(const DecodeArgs& a, const Unit& u, const float* sm_m,
                                             const float* sm_l, const float* sm_acc, int* sm_flag) {
  __syncthreads();
  const int64_t obase = ((int64_t)u.b * a.out_heads + a.out_head0 + (int64_t)u.kvh * a.gq) * D;
  // a thread merges 4 consecutive channels of one head (one float4 per warp state, one vector store)
  for (int i = threadIdx.x; i < a.gq * D / 4; i += blockDim.x) {
    const int hh = (4 * i) / D, c = (4 * i) % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_m[w * 8 + hh]);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float mw = sm_m[w * 8 + hh];
      const float f = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
      const float4 x = *reinterpret_cast<const float4*>(sm_acc + (w * 8 + hh) * D + c);
      acc.x = fmaf(f, x.x, acc.x); acc.y = fmaf(f, x.y, acc.y);
      acc.z = fmaf(f, x.z, acc.z); acc.w = fmaf(f, x.w, acc.w);
      l = fmaf(f, sm_l[w * 8 + hh], l);
    }
    if (u.slot < 0) {
      const float inv = 1.f / l;
      store_out4(a, obase + 4 * i, make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
    } else {
      float* pp = a.part + ((int64_t)u.slot * 8 + hh) * (D + 4);
      *reinterpret_cast<float4*>(pp + c) = acc;
      if (c == 0) *reinterpret_cast<float2*>(pp + D) = make_float2(M, l);
    }
  }
  if (u.slot < 0) return;
  // Publish the partial: every thread fences its own partial stores before the arrival
  // (the conservative form of the pattern; a single acq_rel arrival after the barrier was
  // measured no faster), and the last arriver fences again before reading the others'.
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(a.counters + u.unit, 1);
    const int last = old == u.nparts - 1;
    if (last) a.counters[u.unit] = 0;  // ready for the next launch (stream order)
    *sm_flag = last;
  }
  __syncthreads();
  if (!*sm_flag) return;
  __threadfence();
  // The last CTA merges the unit's partials: a thread owns 4 channels of one head and pulls
  // the partials 8 at a time with all loads in flight together (one L2 round trip per 8
  // partials, not three per partial), merging online.
  constexpr int64_t PSTR = 8 * (D + 4);
  for (int i = threadIdx.x; i < a.gq * D / 4; i += blockDim.x) {
    const int hh = (4 * i) / D, c0 = (4 * i) % D;
    const float* p0 = a.part + ((int64_t)u.part0 * 8 + hh) * (D + 4);
    float M = -INFINITY, l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < u.nparts; k0 += 8) {
      float mk[8], lk[8];
      float4 ak[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = k0 + e < u.nparts;
        const float* pk = p0 + (int64_t)(ok ? k0 + e : k0) * PSTR;
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(pk + D));
        mk[e] = ok ? ml.x : -INFINITY;
        lk[e] = ml.y;
        ak[e] = __ldcg(reinterpret_cast<const float4*>(pk + c0));
      }
      float Mn = M;
#pragma unroll
      for (int e = 0; e < 8; ++e) Mn = fmaxf(Mn, mk[e]);
      const float f = M == -INFINITY ? 0.f : fast_exp2(M - Mn);
      acc.x *= f; acc.y *= f; acc.z *= f; acc.w *= f;
      l *= f;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float g = mk[e] == -INFINITY ? 0.f : fast_exp2(mk[e] - Mn);
        acc.x = fmaf(ak[e].x, g, acc.x); acc.y = fmaf(ak[e].y, g, acc.y);
        acc.z = fmaf(ak[e].z, g, acc.z); acc.w = fmaf(ak[e].w, g, acc.w);
        l = fmaf(lk[e], g, l);
      }
      M = Mn;
    }
    const float inv = 1.f / l;
    store_out4(a, obase + (int64_t)hh * D + c0, make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
  }
}

// ====================================================================================
// Variant 0: tensor-core kernel.  Tile bodies are specialised per bitwidth so that all
// shared-memory addresses are a lane-constant base plus compile-time immediates.
// Running max per head (log2 domain) for heads 2q, 2q+1.  Tile logits arrive already
// shifted by it.  The softmax sum l is not kept here: it is a "ones" row of the
// zero-point MMA (Acc::zs), so it sums exactly the fp16 p the PV MMAs use.
struct Softmax {
  float m0, m1;
  bool init;    // false until the warp's first tile of the piece set the max
  float slack;  // p <= 2^slack: P' = p*s_v stays finite for every V scale of the pool
};

// Launch-wide operand bounds from the pool status words (kvmix_b200.h): with s_v < 2^(ev+1)
// the lazy softmax may let p reach 2^slack, slack = min(8, 15 - ev), so P' = p*s_v < 2^16
// rounds to at most 65504; with s_k < 2^(ek+1) and |q| < 2^(eq+1), q is pre-scaled by
// 2^-qexp, qexp = max(0, eq + max(ek, 5) - 13), so q*s_k and the INT4 group sums of q
// (<= 32|q|) stay below 2^15 (build_qtab).  Unknown bounds (NULL) = the largest finite.
__device__ __forceinline__ int ilog2f(float x) { return ((__float_as_int(x) >> 23) & 0xff) - 127; }
struct Bounds {
  float slack;
  int ek;
};
__device__ __forceinline__ Bounds pool_bounds(const int32_t* st) {
  float kmax = 65504.f, vmax = 65504.f;
  if (st != nullptr) {
    kmax = __int_as_float(__ldcg(st + KVMIX_POOL_STATUS_KSCALE));
    vmax = __int_as_float(__ldcg(st + KVMIX_POOL_STATUS_VSCALE));
  }
  Bounds b;
  b.slack = (float)max(0, min((int)RESCALE_SLACK, 15 - ilog2f(fmaxf(vmax, 1.f))));
  b.ek = max(ilog2f(fmaxf(kmax, 1.f)), 5);
  return b;
}

template <int D>
struct Acc {
  float o[D / 16][4];  // O^T accumulators (rows = channels, cols = heads 2q, 2q+1)
  float zs[4];   // Z^T.P^T, rows g: row j < D/32 = sum_t z_tj p_th; rows D/32..7 = sum_t p_th (l)
  float zs2[4];  // same sums for INT2 k-step 1 (group rows in g+8, l rows in g; see int2_tile)
};

__device__ __forceinline__ uint32_t ld_s32(const uint8_t* base, int off) {
  return *reinterpret_cast<const uint32_t*>(base + off);
}

// Online softmax over one 32-token tile.  sv holds the logits minus the running max;
// returns the P^T B fragments of PV k-steps 0, 1.  Lazy rescale: the max is only raised
// when some logit exceeds it by > st.slack (log2 units, <= RESCALE_SLACK), so p <= 2^slack
// stays inside fp16 (and p*s_v too, see pool_bounds) and the common path needs no
// cross-lane reduction -- only a per-lane max and one vote.  The first tile of a piece establishes the max exactly.
// When the max moved, `resc` is set (warp-uniform) and the accumulators must be
// multiplied by (al0, al1) (0 on the first tile).
__device__ __forceinline__ void softmax_p(float (&sv)[8], Softmax& st, uint32_t (&bP)[2][2], float& al0,
                                          float& al1, bool& resc) {
  float tm0 = fmaxf(fmaxf(sv[0], sv[2]), fmaxf(sv[4], sv[6]));
  float tm1 = fmaxf(fmaxf(sv[1], sv[3]), fmaxf(sv[5], sv[7]));
  resc = __any_sync(0xffffffffu, !st.init || tm0 > st.slack || tm1 > st.slack);
  if (resc) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, off));
      tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, off));
    }
    // first tile: shift to its max (acc is still zero); later: raise only, by max(tm, 0)
    const float sh0 = st.init ? fmaxf(tm0, 0.f) : tm0, sh1 = st.init ? fmaxf(tm1, 0.f) : tm1;
    al0 = st.init ? fast_exp2(-sh0) : 0.f;
    al1 = st.init ? fast_exp2(-sh1) : 0.f;
    st.m0 += sh0;
    st.m1 += sh1;
    st.init = true;
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      sv[i] -= sh0;
      sv[i + 1] -= sh1;
    }
  }
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = fast_exp2(sv[i]);
  // k index of PV == QK row: lane holds head g, rows (2q, 2q+1) / (2q+8, 2q+9)
  bP[0][0] = movtrans(pack_h2(p[0], p[1]));
  bP[0][1] = movtrans(pack_h2(p[2], p[3]));
  bP[1][0] = movtrans(pack_h2(p[4], p[5]));
  bP[1][1] = movtrans(pack_h2(p[6], p[7]));
}

template <int D>
__device__ __forceinline__ void rescale_acc(Acc<D>& acc, float al0, float al1) {
#pragma unroll
  for (int m = 0; m < D / 16; ++m) {
    acc.o[m][0] *= al0; acc.o[m][2] *= al0;
    acc.o[m][1] *= al1; acc.o[m][3] *= al1;
  }
  acc.zs[0] *= al0; acc.zs[2] *= al0;
  acc.zs[1] *= al1; acc.zs[3] *= al1;
  acc.zs2[0] *= al0; acc.zs2[2] *= al0;
  acc.zs2[1] *= al1; acc.zs2[3] *= al1;
}

template <int D>
__device__ __forceinline__ void softmax_tile(float (&sv)[8], Softmax& st, Acc<D>& acc, uint32_t (&bP)[2][2]) {
  float al0, al1;
  bool resc;
  softmax_p(sv, st, bP, al0, al1, resc);
  if (resc) rescale_acc<D>(acc, al0, al1);
}

// Shared-memory vector load of NB bytes (2, 4, 8, 16 or a multiple of 16) into words.
template <int NB>
__device__ __forceinline__ void lds_vec(const uint8_t* p, uint32_t* w) {
  if constexpr (NB >= 16) {
#pragma unroll
    for (int i = 0; i < NB / 16; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else if constexpr (NB == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else if constexpr (NB == 4) {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else {
    w[0] = *reinterpret_cast<const uint16_t*>(p);
  }
}
// low / high fp16 of x and of y as one half2 (low = x's half, high = y's half)
__device__ __forceinline__ uint32_t pair_h(uint32_t x, uint32_t y, int hi) { return prmt(x, y, hi ? 0x7632u : 0x5410u); }
__device__ __forceinline__ float half_f(uint32_t w, int hi) {
  return __half2float(__ushort_as_half((unsigned short)(hi ? w >> 16 : w & 0xffffu)));
}

// Codes enter the MMA as fp16 SUBNORMALS, masked in place: INT2 field e of a code byte
// (bits 2e..2e+1) is code * 2^(2e-24); an INT4 low / high nibble is code * 2^-24 / 2^-20.
// One LOP3 per two codes (plus one shift per 16 codes for the odd bytes), no magic-number
// subtraction; the power of two is undone in fp32 per row.  The tensor core sums
// subnormal products with a relative error <= ~8e-5 of the summed magnitudes at bit 0
// (exact single products; tools/microbench/denorm*.cu), 6x below the fp16 rounding of
// the q' = q*s operand that the reference's fp32 path does not have.
__device__ __forceinline__ constexpr uint32_t F2(int e) { return 0x00030003u << (2 * e); }  // INT2 field e
constexpr uint32_t N4L = 0x000F000Fu, N4H = 0x00F000F0u;  // INT4 low / high nibble of bytes 0, 2
constexpr uint32_t ONES = 0x3C003C00u;  // (1.0, 1.0) fp16
constexpr float P24 = 16777216.f, P22 = 4194304.f, P20 = 1048576.f, P18 = 262144.f;
[[maybe_unused]] constexpr float P10 = 1024.f, P8 = 256.f, P6 = 64.f, P4 = 16.f;
// Key codes enter QK as NORMAL fp16 numbers: (field | 1.0) - 1.0 = code * 2^(p-10) for a
// field at bit p (one LOP3 + one exact HSUB2 per two codes).  The tensor core reduces
// products of subnormal operands with ~13 bits of precision relative to the largest
// product of the MMA (tools/microbench/tc_precision.cu: 2^-12.3 worst, vs 2^-21.5 for
// normal operands), which turns into logit errors that a peaked softmax amplifies; value
// codes (PV) keep the cheaper subnormal form, where the same bound is relative to the
// dominant term of the output.
#ifndef KVMIX_QKNORM
#define KVMIX_QKNORM 1
#endif
// four e4m3 bytes -> two f16x2 words (bytes 0, 1 -> lo; bytes 2, 3 -> hi), hardware conversion
__device__ __forceinline__ void cvt_e4m3x4(uint32_t v, uint32_t& lo, uint32_t& hi) {
  asm("{\n .reg .b16 t0, t1;\n mov.b32 {t0, t1}, %2;\n cvt.rn.f16x2.e4m3x2 %0, t0;\n cvt.rn.f16x2.e4m3x2 %1, t1;\n}"
      : "=r"(lo), "=r"(hi)
      : "r"(v));
}
__device__ __forceinline__ uint32_t kcode(uint32_t v, uint32_t mask) {
#if KVMIX_QKNORM
  return hsub2u(lop_and_or(v, mask, ONES), ONES);
#else
  return v & mask;
#endif
}
#if KVMIX_QKCVT
constexpr float KF0 = 512.f, KF1 = 128.f, KF2 = 512.f, KF3 = 128.f;  // INT2 key fields at 2^-9 / 2^-7 (cvt_e4m3x4)
constexpr float KF4 = P6;                                              // INT4 key products at 2^-6
#elif KVMIX_QKNORM
constexpr float KF0 = P10, KF1 = P8, KF2 = P6, KF3 = P4;  // INT2 key field e at 2^(2e-10)
constexpr float KF4 = P6;                                 // INT4 key products at 2^-6
#else
constexpr float KF0 = P24, KF1 = P22, KF2 = P20, KF3 = P18;
constexpr float KF4 = P20;
#endif

// Q as B fragments of QK, fp16, NOT pre-scaled (bf16 q converts exactly).
//  b2[I]  INT2 key pages, chunk I, lane q: channels cb = q*D/4 + 4I: (cb, cb+1) / (cb+2, cb+3)
//         (round 1's subnormal / normal-code forms paired (cb, cb+2) / (cb+1, cb+3))
//  b4[2j], b4[2j+1]  INT4 keys, group j, lane q: cb = 32j + 8q: (cb+1, cb+5) / (cb, cb+4) and
//         (cb+2, cb+6) / (cb+3, cb+7)
//  qz     (Q_2q, Q_2q+1) hi / lo fp16 parts (k-lo / k-hi), Q_j = sum of q over channel group j
// With LO (fp32 q) the *lo arrays hold q - fp16(q).
template <int D, bool LO>
struct QFrag {
  static constexpr int NCH = D / 16;
  // fragment index f: b2 [0, NCH), b4 [NCH, 2NCH), qz 2NCH (2NCH+1 unused), b2lo / b4lo after
  static constexpr int F = 2 * NCH + 2 + (LO ? 2 * NCH : 0);
  static constexpr int BYTES = F * 32 * 8;
  const uint64_t* p;  // this lane's column of the CTA's [F][32 lanes] fragment table in smem
  __device__ __forceinline__ uint64_t at(int f) const { return p[f * 32]; }
  __device__ __forceinline__ uint64_t b2(int i) const { return at(i); }
  __device__ __forceinline__ uint64_t b4(int i) const { return at(NCH + i); }
  __device__ __forceinline__ uint64_t qz() const { return at(2 * NCH); }
  __device__ __forceinline__ uint64_t b2lo(int i) const { return at(2 * NCH + 2 + i); }
  __device__ __forceinline__ uint64_t b4lo(int i) const { return at(3 * NCH + 2 + i); }
};

// ---------------------------------- INT2 page tile ----------------------------------
// Record layout: common.cuh PG_* (layout.py).  QK rows: M tile 0 rows g / g+8 = tokens
// 4g / 4g+1 (fields 0 / 1), M tile 1 = tokens 4g+2 / 4g+3.  PV k-step ks, lane q covers
// tokens T0 = 8q + 2ks, T1 = T0 + 4 (a0) and T0+1, T1+1 (a2).
template <int D, bool LO>
__device__ __forceinline__ void int2_qk(const uint8_t* __restrict__ buf, const QFrag<D, LO>& qf, float qscale,
                                        int lane, const Softmax& st, float (&sv)[8], float kb0, float kb1) {
  using C = Cfg<D>;
  constexpr int KB = D / 4, LB = KB < 16 ? KB : 16;
  const int g = lane >> 2, q = lane & 3;
  uint32_t kw[C::NCH];
#pragma unroll
  for (int o = 0; o < KB; o += LB) {
    const int p = q * KB + o;
    lds_vec<LB>(buf + g * D + ((((p >> 4) ^ (g & 1)) << 4) | (p & 15)), kw + o / 4);
  }
#if KVMIX_LAZYPARAM
  uint32_t ksw[4], kzw[4];  // the quad of the current chunk pair only (lower register pressure)
#else
  uint32_t ksw[2 * C::NCH], kzw[2 * C::NCH];
#pragma unroll
  for (int i = 0; i < KB / 8; ++i) {  // 16 B chunk i of lane q at chunk 4i + q
    lds_vec<16>(buf + PG_KS(D) + (4 * i + q) * 16, ksw + 4 * i);
    lds_vec<16>(buf + PG_KZ(D) + (4 * i + q) * 16, kzw + 4 * i);
  }
#endif
  // two accumulators per M tile (hi / lo parts of q*s) halve the HMMA dependency chains
  float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f}, d0[4] = {0.f, 0.f, 0.f, 0.f},
        d1[4] = {0.f, 0.f, 0.f, 0.f};
  // bias sum_c q_c z_c: the KZ quad of chunks (2P, 2P+1) is (z_2P.p0, z_2P+1.p0, z_2P.p1, z_2P+1.p1),
  // used as-is as the A operand: rows g of cbE are chunk 2P's bias, rows g+8 of cbO chunk 2P+1's
  float cbE[4] = {0.f, 0.f, 0.f, 0.f}, cbO[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < C::NCH; ++i) {
#if KVMIX_LAZYPARAM
    const int P4 = 0, odd = i & 1;
    if (!odd) {
      lds_vec<16>(buf + PG_KS(D) + (4 * (i >> 1) + q) * 16, ksw);
      if (!KVMIX_KZBATCH) lds_vec<16>(buf + PG_KZ(D) + (4 * (i >> 1) + q) * 16, kzw);
    }
#else
    const int P4 = 4 * (i >> 1), odd = i & 1;
#endif
#if KVMIX_QKCVT
    const uint32_t w = kw[i];
#else
    const uint32_t w = kw[i], x = w >> 8;
#endif
    const uint64_t qi = qf.b2(i);
    const uint32_t s0 = ksw[P4 + odd], s1 = ksw[P4 + 2 + odd];
    const uint32_t h0 = hmul2u(lo32(qi), s0), h1 = hmul2u(hi32(qi), s1);
    const uint64_t qs = pack_b64(h0, h1);
#if KVMIX_QKCVT
    // The word holds the code bytes of channels cb..cb+3 (byte j = channel cb + j).  A byte with
    // one field kept (value b < 16) read as e4m3 is exactly b * 2^-9, and the hardware e4m3x2 ->
    // f16x2 conversion makes it a NORMAL fp16 number (full tensor-core precision, no subtraction):
    // fields 0 / 2 masked at bits 0-1 give code * 2^-9, fields 1 / 3 at bits 2-3 give code * 2^-7.
    // lo16 -> channels (cb, cb+1) = k-lo, hi16 -> (cb+2, cb+3) = k-hi; rows g / g+8 = fields 0 / 1
    // (c0) and 2 / 3 (c1).
    const uint32_t y = w >> 4;
    uint32_t a00, a02, a01, a03, a10, a12, a11, a13;
    cvt_e4m3x4(w & 0x03030303u, a00, a02);
    cvt_e4m3x4(w & 0x0C0C0C0Cu, a01, a03);
    cvt_e4m3x4(y & 0x03030303u, a10, a12);
    cvt_e4m3x4(y & 0x0C0C0C0Cu, a11, a13);
#else
    const uint32_t a00 = kcode(w, F2(0)), a01 = kcode(w, F2(1)), a02 = kcode(x, F2(0)), a03 = kcode(x, F2(1));
    const uint32_t a10 = kcode(w, F2(2)), a11 = kcode(w, F2(3)), a12 = kcode(x, F2(2)), a13 = kcode(x, F2(3));
#endif
    mma16816_b64(c0, a00, a01, a02, a03, qs);
    mma16816_b64(c1, a10, a11, a12, a13, qs);
#if KVMIX_Q2EXACT
    // q*s has <= 19 significant bits (bf16 q) and h = RN16(q*s) keeps 11: the remainder
    // q*s - h is an fp16 value, computed exactly by one fused HFMA2 (fp32 q: plus lo(q)*s,
    // rounded once more at 2^-22 relative).  Its MMA makes the key products exact.
    uint32_t r0 = hfma2u(lo32(qi), s0, hneg2u(h0)), r1 = hfma2u(hi32(qi), s1, hneg2u(h1));
    if constexpr (LO) {
      const uint64_t ql = qf.b2lo(i);
      r0 = hfma2u(lo32(ql), s0, r0);
      r1 = hfma2u(hi32(ql), s1, r1);
    }
    const uint64_t qr = pack_b64(r0, r1);
#if KVMIX_Q2ACC
    mma16816_b64(c0, a00, a01, a02, a03, qr);
    mma16816_b64(c1, a10, a11, a12, a13, qr);
#else
    mma16816_b64(d0, a00, a01, a02, a03, qr);
    mma16816_b64(d1, a10, a11, a12, a13, qr);
#endif
#endif
    if (!KVMIX_KZBATCH) {
      mma16816_b64(odd ? cbO : cbE, kzw[P4], kzw[P4 + 1], kzw[P4 + 2], kzw[P4 + 3], qi);
      if constexpr (LO) mma16816_b64(odd ? cbO : cbE, kzw[P4], kzw[P4 + 1], kzw[P4 + 2], kzw[P4 + 3], qf.b2lo(i));
    }
  }
  if (KVMIX_KZBATCH) {  // the page's bias, computed for its batch of 16 pages (int2_batch_bias)
    cbE[0] = kb0;
    cbE[1] = kb1;
  }
  const float b0 = fmaf(cbE[0] + cbO[2], qscale, -st.m0), b1 = fmaf(cbE[1] + cbO[3], qscale, -st.m1);
  const float f0 = KF0 * qscale, f1 = KF1 * qscale, f2 = KF2 * qscale, f3 = KF3 * qscale;
  sv[0] = fmaf(c0[0] + d0[0], f0, b0);
  sv[1] = fmaf(c0[1] + d0[1], f0, b1);
  sv[2] = fmaf(c0[2] + d0[2], f1, b0);
  sv[3] = fmaf(c0[3] + d0[3], f1, b1);
  sv[4] = fmaf(c1[0] + d1[0], f2, b0);
  sv[5] = fmaf(c1[1] + d1[1], f2, b1);
  sv[6] = fmaf(c1[2] + d1[2], f3, b0);
  sv[7] = fmaf(c1[3] + d1[3], f3, b1);
}

template <int D>
__device__ __forceinline__ void int2_pv(const uint8_t* __restrict__ buf, const uint32_t (&bP)[2][2], int lane,
                                        Acc<D>& acc) {
  using C = Cfg<D>;
  constexpr int NG = C::NGRP;
  const int g = lane >> 2, q = lane & 3;
  // V params: one 16 B quad per (q, group j) = (ks0.p0, ks1.p0, ks0.p1, ks1.p1)
  uint32_t vs[4 * NG], vz[4];
#pragma unroll
  for (int j = 0; j < NG; ++j) lds_vec<16>(buf + PG_VS(D) + (j * 4 + q) * 16, vs + 4 * j);
  lds_vec<16>(buf + PG_VZ(D) + ((g & (NG - 1)) * 4 + q) * 16, vz);
  if (g >= NG) vz[0] = vz[1] = vz[2] = vz[3] = ONES;  // rows NG..7 of the zero-point MMA sum p (l)
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    uint32_t vw[NG];
    lds_vec<4 * NG>(buf + PG_VC(D) + ((ks * 8 + g) * 4 + q) * NG * 4, vw);
    // sum_t p_th z_tj for all groups at once: A = Z^T (row g = group g & (NG-1)), B = P^T.
    // k-step 0 is valid in rows g (zs), k-step 1 in rows g+8 (zs2) of the same quad.
    mma16816_b64(ks ? acc.zs2 : acc.zs, vz[0], vz[1], vz[2], vz[3], pack_b64(bP[ks][0], bP[ks][1]));
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const uint32_t w = vw[j], x = w >> 8;
      const uint64_t ps = pack_b64(hmul2u(bP[ks][0], vs[4 * j + ks]), hmul2u(bP[ks][1], vs[4 * j + 2 + ks]));
      mma16816_b64(acc.o[2 * j], w & F2(0), w & F2(1), x & F2(0), x & F2(1), ps);
      mma16816_b64(acc.o[2 * j + 1], w & F2(2), w & F2(3), x & F2(2), x & F2(3), ps);
    }
  }
}

// Key bias sum_c q_c z_c of 16 INT2 pages at once (KVMIX_KZBATCH): A rows g / g+8 = the zero
// points of pages g / g+8 of the batch (their KZ regions, staged in kzs), B = the chunk's q
// fragment, so NCH MMAs cover 16 pages instead of NCH per page.  d[0..1] = page g's bias for
// heads 2q, 2q+1, d[2..3] = page g+8's.
template <int D, bool LO>
__device__ __forceinline__ void int2_batch_bias(const uint8_t* __restrict__ kzs, const QFrag<D, LO>& qf, int lane,
                                                float (&d)[4]) {
  using C = Cfg<D>;
  const int g = lane >> 2, q = lane & 3;
  d[0] = d[1] = d[2] = d[3] = 0.f;
#pragma unroll
  for (int P = 0; P < C::NCH / 2; ++P) {
    uint32_t wa[4], wb[4];  // quad (z_2P.p0, z_2P+1.p0, z_2P.p1, z_2P+1.p1) of pages g and g+8
    lds_vec<16>(kzs + g * C::KZB + (4 * P + q) * 16, wa);
    lds_vec<16>(kzs + (g + 8) * C::KZB + (4 * P + q) * 16, wb);
    mma16816_b64(d, wa[0], wb[0], wa[2], wb[2], qf.b2(2 * P));
    mma16816_b64(d, wa[1], wb[1], wa[3], wb[3], qf.b2(2 * P + 1));
    if constexpr (LO) {
      mma16816_b64(d, wa[0], wb[0], wa[2], wb[2], qf.b2lo(2 * P));
      mma16816_b64(d, wa[1], wb[1], wa[3], wb[3], qf.b2lo(2 * P + 1));
    }
  }
}

template <int D, bool LO>
__device__ __forceinline__ void int2_tile(const uint8_t* __restrict__ buf, const QFrag<D, LO>& qf, float qscale,
                                          int lane, Softmax& st, Acc<D>& acc, float kb0 = 0.f, float kb1 = 0.f) {
  float sv[8];
  uint32_t bP[2][2];
  int2_qk<D, LO>(buf, qf, qscale, lane, st, sv, kb0, kb1);
  softmax_tile<D>(sv, st, acc, bP);
  int2_pv<D>(buf, bP, lane, acc);
}

// ---------------------------------- INT4 slot tile ----------------------------------
// Row -> slot map inside an M tile: rows 0-7 -> rho(r), rows 8-15 -> 8 + rho(r - 8) with
// rho = [0,2,1,3,6,4,7,5]: QK K loads (lanes g = 2p, 2p+1 two slots apart) and PV V
// loads (rho(2q) and rho(2q+1) each distinct mod 4) are both bank-conflict-free at the
// 160 B slot stride.
__device__ __forceinline__ int rho(int r) { return (0x57463120u >> (4 * r)) & 7; }

template <int D, bool FULL, bool LO>
__device__ __forceinline__ void int4_qk(const uint8_t* __restrict__ buf, int nv, const QFrag<D, LO>& qf,
                                        float qscale, int lane, const Softmax& st, float (&sv)[8]) {
  using C = Cfg<D>;
  constexpr int S = C::SS, NG = C::NGRP;
  const int g = lane >> 2, q = lane & 3;
  const float fs = KF4 * qscale;  // both nibbles' products at one scale (low-nibble q is pre-multiplied by 16)
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int sa = 16 * mt + rho(g), sb = sa + 8;
    uint32_t kwa[NG], kwb[NG], pa[NG], pb[NG];
    lds_vec<4 * NG>(buf + S * sa + 4 * NG * q, kwa);
    lds_vec<4 * NG>(buf + S * sb + 4 * NG * q, kwb);
    lds_vec<4 * NG>(buf + S * sa + SL_KS(D), pa);  // NG scales then NG zeros
    lds_vec<4 * NG>(buf + S * sb + SL_KS(D), pb);
    // D_j = sum over group j of q_c code_c (per-token group scales are applied in fp32)
    float dj[NG][4];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      dj[j][0] = dj[j][1] = dj[j][2] = dj[j][3] = 0.f;
      const uint32_t wa = kwa[j], wb = kwb[j];
      const uint32_t xa = wa >> 8, xb = wb >> 8;
      const uint32_t e0 = kcode(wa, N4H), e1 = kcode(wb, N4H), e2 = kcode(wa, N4L), e3 = kcode(wb, N4L);
      const uint32_t o0 = kcode(xa, N4L), o1 = kcode(xb, N4L), o2 = kcode(xa, N4H), o3 = kcode(xb, N4H);
      mma16816_b64(dj[j], e0, e1, e2, e3, qf.b4(2 * j));
      mma16816_b64(dj[j], o0, o1, o2, o3, qf.b4(2 * j + 1));
      if constexpr (LO) {
        mma16816_b64(dj[j], e0, e1, e2, e3, qf.b4lo(2 * j));
        mma16816_b64(dj[j], o0, o1, o2, o3, qf.b4lo(2 * j + 1));
      }
    }
    // sum_j z_j Q_j: A row = token, k = 2q, 2q+1 -> groups 2q, 2q+1 (lanes with 2q >= NG give 0)
    uint32_t za = 0u, zb = 0u;
    if constexpr (NG == 4) {
      if (q < 2) { za = q ? pa[3] : pa[2]; zb = q ? pb[3] : pb[2]; }
    } else if constexpr (NG == 2) {
      if (q == 0) { za = pa[1]; zb = pb[1]; }
    } else {
      if (q == 0) { za = pa[0] >> 16; zb = pb[0] >> 16; }
    }
    float zq[4] = {0.f, 0.f, 0.f, 0.f};
    // k 0..7 carry the hi parts of Q_j, k 8..15 the lo parts: one MMA for both
    mma16816_b64(zq, za, zb, za, zb, qf.qz());
    float ta0 = fmaf(zq[0], qscale, -st.m0), ta1 = fmaf(zq[1], qscale, -st.m1);
    float tb0 = fmaf(zq[2], qscale, -st.m0), tb1 = fmaf(zq[3], qscale, -st.m1);
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const float s_a = half_f(pa[j >> 1], j & 1) * fs, s_b = half_f(pb[j >> 1], j & 1) * fs;
      ta0 = fmaf(s_a, dj[j][0], ta0);
      ta1 = fmaf(s_a, dj[j][1], ta1);
      tb0 = fmaf(s_b, dj[j][2], tb0);
      tb1 = fmaf(s_b, dj[j][3], tb1);
    }
    if (!FULL) {
      if (sa >= nv) ta0 = ta1 = -INFINITY;
      if (sb >= nv) tb0 = tb1 = -INFINITY;
    }
    sv[4 * mt] = ta0;
    sv[4 * mt + 1] = ta1;
    sv[4 * mt + 2] = tb0;
    sv[4 * mt + 3] = tb1;
  }
}

template <int D, bool FULL>
__device__ __forceinline__ void int4_pv(const uint8_t* __restrict__ buf, int nv, const uint32_t (&bP)[2][2],
                                        int lane, Acc<D>& acc) {
  using C = Cfg<D>;
  constexpr int S = C::SS, NG = C::NGRP;
  const int g = lane >> 2, q = lane & 3;
  // PV k-step ks: k = 2q, 2q+1, 2q+8, 2q+9 = rows of QK M tile ks -> slots ta, tb, tc, td
  constexpr int VB = 2 * NG;  // this lane's code bytes per token: 2 per group
  constexpr int VWN = VB < 4 ? 1 : VB / 4;
  const int jz = g & (NG - 1);
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const int ta = 16 * ks + rho(2 * q), tb = 16 * ks + rho(2 * q + 1), tc = ta + 8, td = tb + 8;
    uint32_t va[VWN], vb[VWN], vc[VWN], vd[VWN], pa[NG], pb[NG], pc[NG], pd[NG];
    lds_vec<VB>(buf + S * ta + SL_VC(D) + VB * g, va);
    lds_vec<VB>(buf + S * tb + SL_VC(D) + VB * g, vb);
    lds_vec<VB>(buf + S * tc + SL_VC(D) + VB * g, vc);
    lds_vec<VB>(buf + S * td + SL_VC(D) + VB * g, vd);
    lds_vec<4 * NG>(buf + S * ta + SL_VS(D), pa);  // NG scales then NG zeros
    lds_vec<4 * NG>(buf + S * tb + SL_VS(D), pb);
    lds_vec<4 * NG>(buf + S * tc + SL_VS(D), pc);
    lds_vec<4 * NG>(buf + S * td + SL_VS(D), pd);
    if (!FULL) {  // padding slots: P = 0 already; zero their params so stale bytes cannot give NaN
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        if (ta >= nv) pa[j] = 0u;
        if (tb >= nv) pb[j] = 0u;
        if (tc >= nv) pc[j] = 0u;
        if (td >= nv) pd[j] = 0u;
      }
    }
    // word / half holding the scale (Z = false) or zero (Z = true) of group j
    auto pw = [&](const uint32_t* p, int j, bool z) -> uint32_t {  // j may be lane-dependent: select, never index
      if constexpr (NG == 4) return z ? ((j >> 1) ? p[3] : p[2]) : ((j >> 1) ? p[1] : p[0]);
      else if constexpr (NG == 2) return p[z ? 1 : 0];
      else return p[0];
    };
    auto ph = [&](int j, bool z) -> int {
      if constexpr (NG == 4) return j & 1;
      else if constexpr (NG == 2) return j;
      else return z ? 1 : 0;
    };
    {
      uint32_t zab = pair_h(pw(pa, jz, true), pw(pb, jz, true), ph(jz, true));
      uint32_t zcd = pair_h(pw(pc, jz, true), pw(pd, jz, true), ph(jz, true));
      if (g >= NG) zab = zcd = ONES;  // rows NG..7 sum p (l)
      mma16816_b64(acc.zs, zab, zab, zcd, zcd, pack_b64(bP[ks][0], bP[ks][1]));
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int vh = NG == 1 ? 0 : (j & 1);
      const uint32_t rab = pair_h(va[j >> 1], vb[j >> 1], vh), rcd = pair_h(vc[j >> 1], vd[j >> 1], vh);
      const uint32_t sab = pair_h(pw(pa, j, false), pw(pb, j, false), ph(j, false));
      const uint32_t scd = pair_h(pw(pc, j, false), pw(pd, j, false), ph(j, false));
      const uint64_t ps = pack_b64(hmul2u(bP[ks][0], sab), hmul2u(bP[ks][1], scd));
      // channels 32j + 4g + {0,1,2,3} = nibbles at bits 0, 4, 8, 12 -> bits 0, 2, 4, 6 (INT2 row scales)
      constexpr uint32_t S0 = 0x000F000Fu, S1 = 0x003C003Cu, S2 = 0x00F000F0u, S3 = 0x03C003C0u;
      mma16816_b64(acc.o[2 * j], rab & S0, (rab >> 2) & S1, rcd & S0, (rcd >> 2) & S1, ps);
      mma16816_b64(acc.o[2 * j + 1], (rab >> 4) & S2, (rab >> 6) & S3, (rcd >> 4) & S2, (rcd >> 6) & S3, ps);
    }
  }
}

template <int D, bool FULL, bool LO>
__device__ __forceinline__ void int4_tile(const uint8_t* __restrict__ buf, int nv, const QFrag<D, LO>& qf,
                                          float qscale, int lane, Softmax& st, Acc<D>& acc) {
  float sv[8];
  uint32_t bP[2][2];
  int4_qk<D, FULL, LO>(buf, nv, qf, qscale, lane, st, sv);
  softmax_tile<D>(sv, st, acc, bP);
  int4_pv<D, FULL>(buf, nv, bP, lane, acc);
}

// Tile metadata: the page id (INT2 tile) or this lane's INT4 index (INT4 tile).
__device__ __forceinline__ int tile_meta(const DecodeArgs& a, const Unit& u, int t, int lane) {
  if (t < u.npg) return a.page_ids[u.pg0 + t];
  const int it = t - u.npg;
  return lane < min(32, u.n4 - 32 * it) ? a.int4_ids[u.i40 + 32 * it + lane] : 0;
}

// TMA bulk copies of tile t into buf, completing on bar (whole warp calls): one 3 KB copy
// per INT2 page, one copy per run of consecutive INT4 slots (fresh pools give long runs).
template <int D>
__device__ __forceinline__ void issue_tile(const Unit& u, int t, int meta, uint8_t* buf, uint64_t* bar, int lane,
                                           const uint8_t* kv2, const uint8_t* kv4) {
  using C = Cfg<D>;
  if (t < u.npg) {
    // with the batched key bias the record's trailing key zeros stay out of the tile copy
    constexpr int NB = KVMIX_KZBATCH ? PG_KZ(D) : C::PS;
    if (lane == 0) {
      mbar_expect_tx(bar, NB);
      bulk_g2s(buf, kv2 + (int64_t)meta * C::PS, NB, bar);
    }
  } else {
    const int nv = min(32, u.n4 - 32 * (t - u.npg));
    const int prev = __shfl_up_sync(0xffffffffu, meta, 1);
    const bool start = lane < nv && (lane == 0 || meta != prev + 1);
    const uint32_t starts = __ballot_sync(0xffffffffu, start);
    if (__popc(starts) <= KVMIX_INT4_RUNS) {  // few runs of consecutive slots: one bulk copy each
      if (lane == 0) mbar_expect_tx(bar, nv * C::SS);
      __syncwarp();
      if (start) {
        const uint32_t later = starts & ~((2u << lane) - 1u);
        const int end = later ? __ffs(later) - 1 : nv;
        bulk_g2s(buf + lane * C::SS, kv4 + (int64_t)meta * C::SS, (end - lane) * C::SS, bar);
      }
    } else {  // scattered slots (after churn / decode appends): each lane copies its own record
      if (lane < nv) {
#pragma unroll
        for (int c = 0; c < C::SS / 16; ++c)
          cp_async16(buf + lane * C::SS + 16 * c, kv4 + (int64_t)meta * C::SS + 16 * c);
        cp_async_mbar_arrive(bar);
      }
      __syncwarp();  // every lane's pending arrival is registered before the phase's own arrival
      if (lane == 0) mbar_arrive(bar);
    }
  }
}

// One warp's (acc, zero sums) -> smem row block w of the piece merge: acc[h][c] = 2^(24-2e) O^T + zsum.
template <int D>
__device__ __forceinline__ void store_warp_acc(const Acc<D>& acc, float* sm_acc, int w, int lane) {
  using C = Cfg<D>;
  const int g = lane >> 2, q = lane & 3;
  float z0[C::NGRP], z1[C::NGRP];  // sum_t p z of group j for heads 2q, 2q+1 (from lane (j, q))
#pragma unroll
  for (int j = 0; j < C::NGRP; ++j) {
    z0[j] = __shfl_sync(0xffffffffu, acc.zs[0] + acc.zs2[2], 4 * j + q);
    z1[j] = __shfl_sync(0xffffffffu, acc.zs[1] + acc.zs2[3], 4 * j + q);
  }
#pragma unroll
  for (int m = 0; m < C::NCH; ++m) {
    const int j = m >> 1;
    const int ch0 = 32 * j + 4 * g + 2 * (m & 1);
    // channel 4g + e of group j carries 2^(2e-24): e = 0/1 in even M tiles, 2/3 in odd ones
    const float f0 = (m & 1) ? P20 : P24, f1 = (m & 1) ? P18 : P22;
    sm_acc[(w * 8 + 2 * q) * D + ch0] = fmaf(acc.o[m][0], f0, z0[j]);
    sm_acc[(w * 8 + 2 * q + 1) * D + ch0] = fmaf(acc.o[m][1], f0, z1[j]);
    sm_acc[(w * 8 + 2 * q) * D + ch0 + 1] = fmaf(acc.o[m][2], f1, z0[j]);
    sm_acc[(w * 8 + 2 * q + 1) * D + ch0 + 1] = fmaf(acc.o[m][3], f1, z1[j]);
  }
}

// The unit's q rows [gq][D] -> fp32 smem rows of stride QS (rows gq..7 zero), all threads,
// every global load in flight at once (one L2 round trip instead of one per table entry).
template <int D>
__device__ __forceinline__ void stage_q(const DecodeArgs& a, const Unit& u, float* qraw) {
  using C = Cfg<D>;
  for (int i = 4 * (int)threadIdx.x; i < 8 * D; i += 4 * (int)blockDim.x) {
    const int h = i / D, c = i % D;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h < a.gq) {
      const int64_t idx = ((int64_t)u.b * a.n_q + (int64_t)u.kvh * a.gq + h) * D + c;
      if (a.q_dtype == KVMIX_F32) {
        v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.q) + idx);
      } else {
        const uint2 w = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(a.q) + idx);
        if (a.q_dtype == KVMIX_BF16) {
          v = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u),
                          __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u));
        } else {
          const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
          const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
          v = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
      }
    }
    *reinterpret_cast<float4*>(qraw + h * C::QS + c) = v;
  }
}

// Q fragments of one unit (see QFrag) written by one warp into the CTA's smem table, from
// the unit's staged q rows (stage_q).  q enters pre-scaled by 2^-qexp (pool_bounds; 0 for
// ordinary data) so that the fp16 operands cannot overflow; returns qscale * 2^qexp, the
// factor that turns the tile accumulations back into log2-domain logits.
template <int D, bool LO>
__device__ __forceinline__ float build_qtab(const float* qraw, uint64_t* qtab, int lane, float qscale, int ek) {
  using C = Cfg<D>;
  using QF = QFrag<D, LO>;
  const int g = lane >> 2, q = lane & 3;
  float amax = 0.f;  // max |q| of the unit: lane (g, q) scans head g, channels [q D/4, (q+1) D/4)
#pragma unroll
  for (int c = 0; c < D / 4; c += 4) {
    const float4 v = *reinterpret_cast<const float4*>(qraw + g * C::QS + q * (D / 4) + c);
    amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  const int qexp = min(30, max(0, ilog2f(fmaxf(amax, 1e-30f)) + ek - 13));
  const float sc = __int_as_float((127 - qexp) << 23);  // 2^-qexp, exact
  auto qv = [&](int c) { return qraw[g * C::QS + c] * sc; };
  auto lo = [](float x) { return x - __half2float(__float2half_rn(x)); };
  auto put = [&](int f, uint64_t v) { qtab[f * 32 + lane] = v; };
#pragma unroll
  for (int i = 0; i < C::NCH; ++i) {
    const int cb = q * (D / 4) + 4 * i;
    const float x0 = qv(cb), x1 = qv(cb + 1), x2 = qv(cb + 2), x3 = qv(cb + 3);
#if KVMIX_QKCVT
    put(i, pack_b64(pack_h2(x0, x1), pack_h2(x2, x3)));  // k-lo = channels (cb, cb+1), k-hi = (cb+2, cb+3)
    if constexpr (LO) put(2 * QF::NCH + 2 + i, pack_b64(pack_h2(lo(x0), lo(x1)), pack_h2(lo(x2), lo(x3))));
#else
    put(i, pack_b64(pack_h2(x0, x2), pack_h2(x1, x3)));
    if constexpr (LO) put(2 * QF::NCH + 2 + i, pack_b64(pack_h2(lo(x0), lo(x2)), pack_h2(lo(x1), lo(x3))));
#endif
  }
  float qa = 0.f, qb = 0.f;  // Q_2q, Q_2q+1 (group sums, fp32)
#pragma unroll
  for (int j = 0; j < C::NGRP; ++j) {
    const int cb = 32 * j + 8 * q;
    float y[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = qv(cb + e);
    // high-nibble channels (cb+1, cb+5, cb+3, cb+7) enter at 2^-20, low-nibble ones at 2^-24:
    // the latter's q is multiplied by 16 (exact; small q stays a normal fp16 number)
    constexpr float X16 = 16.f;
    put(QF::NCH + 2 * j, pack_b64(pack_h2(y[1], y[5]), pack_h2(y[0] * X16, y[4] * X16)));
    put(QF::NCH + 2 * j + 1, pack_b64(pack_h2(y[2] * X16, y[6] * X16), pack_h2(y[3], y[7])));
    if constexpr (LO) {
      put(3 * QF::NCH + 2 + 2 * j, pack_b64(pack_h2(lo(y[1]), lo(y[5])), pack_h2(lo(y[0]) * X16, lo(y[4]) * X16)));
      put(3 * QF::NCH + 2 + 2 * j + 1, pack_b64(pack_h2(lo(y[2]) * X16, lo(y[6]) * X16), pack_h2(lo(y[3]), lo(y[7]))));
    }
    float part = ((y[0] + y[1]) + (y[2] + y[3])) + ((y[4] + y[5]) + (y[6] + y[7]));
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    if (j == 2 * q) qa = part;
    if (j == 2 * q + 1) qb = part;
  }
  put(2 * QF::NCH, pack_b64(pack_h2(qa, qb), pack_h2(lo(qa), lo(qb))));  // k-lo: hi parts, k-hi: lo parts
  return qscale * __int_as_float((127 + qexp) << 23);
}

// K4 fused decode append, cold path (out of line): channel group j of the request's newest
// token -> the staged slot record srec and its place in the pool.
template <int D>
__device__ __noinline__ float append_group(const DecodeArgs& a, const Unit& u, uint8_t* srec, int j) {
  using C = Cfg<D>;
  const int64_t slot = a.int4_ids[u.i40 + u.n4 - 1];
  uint8_t* grec = a.int4_pool_w + ((a.layer * a.n_kv + u.kvh) * a.pool_int4 + slot) * (int64_t)C::SS;
  const int64_t off = ((int64_t)u.b * a.n_kv + u.kvh) * D + 32 * j;
  int32_t* err = a.pool_status ? a.pool_status + KVMIX_POOL_STATUS_ERR : nullptr;
  float vs;
  if (a.app_dtype == KVMIX_BF16)
    vs = encode_int4_group<D, __nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(a.app_k) + off,
                                             reinterpret_cast<const __nv_bfloat16*>(a.app_v) + off, srec, grec, j, err);
  else if (a.app_dtype == KVMIX_F16)
    vs = encode_int4_group<D, __half>(reinterpret_cast<const __half*>(a.app_k) + off,
                                      reinterpret_cast<const __half*>(a.app_v) + off, srec, grec, j, err);
  else
    vs = encode_int4_group<D, float>(reinterpret_cast<const float*>(a.app_k) + off,
                                     reinterpret_cast<const float*>(a.app_v) + off, srec, grec, j, err);
  if (a.pool_status) atomicMax(a.pool_status + KVMIX_POOL_STATUS_VSCALE, __float_as_int(vs));
  return vs;
}

// Issue this warp's first STAGES tiles of piece u into its ring, starting at `stage`.
template <int D>
__device__ __forceinline__ void prime_piece(const DecodeArgs& a, const Unit& u, int warp, int lane, uint8_t* ring,
                                            uint64_t (*bars)[STAGES], int stage) {
  using C = Cfg<D>;
  const int ntiles = u.thi - u.tlo;
  const int nmine = ntiles > warp ? (ntiles - warp + NW - 1) / NW : 0;
  const uint8_t* kv2 = a.int2_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_pages) * (int64_t)C::PS;
  const uint8_t* kv4 = a.int4_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_int4) * (int64_t)C::SS;
  __syncwarp();
  fence_proxy_async();  // the slots were last read through the generic proxy
  int s0 = stage;
  for (int k = 0; k < STAGES && k < nmine; ++k) {
    const int t = u.tlo + warp + k * NW;
    issue_tile<D>(u, t, tile_meta(a, u, t, lane), ring + s0 * C::BUF, &bars[warp][s0], lane, kv2, kv4);
    if (++s0 == STAGES) s0 = 0;
  }
}

#ifdef KVMIX_MAXREG
#define KVMIX_FUSED_BOUNDS __maxnreg__(KVMIX_MAXREG)
#else
#define KVMIX_FUSED_BOUNDS __launch_bounds__(NW * 32, KVMIX_MINB)
#endif
#ifdef KVMIX_CTA_TIMES
__device__ unsigned long long g_cta_times[4096][16];  // start, waited, end, smid, then per piece (<3): begin, q table, loop end, merged
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
template <int D, bool COMPUTE = true, bool MEMORY = true, bool LO = false, bool APPEND = false>
__global__ void KVMIX_FUSED_BOUNDS decode_mma_kernel(const DecodeArgs a) {
#ifdef KVMIX_CTA_TIMES
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_cta_times[blockIdx.x][0] = gtimer();
    g_cta_times[blockIdx.x][3] = smid;
  }
#endif
  using C = Cfg<D>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[NW][STAGES];
  __shared__ __align__(8) uint64_t kzbar[NW];  // this warp's KZ batch copies
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  uint8_t* ring = smem + warp * STAGES * C::BUF;
  __shared__ int sm_flag;
  __shared__ float sm_qscale;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
    mbar_init(&kzbar[warp], 1);
    fence_mbar_init();
  }
  __syncwarp();
  pdl_launch_dependents();  // the next kernel may start prefetching its KV tiles
  int stage = 0;  // ring position and mbarrier phase persist across pieces
  uint32_t phase = 0;
  uint32_t kzphase = 0;
  uint8_t* kzs = (C::KZ_IN_MERGE ? smem + NW * STAGES * C::BUF + C::QTAB
                                 : smem + C::SMEM - C::KZS) + warp * 16 * C::KZB;
  bool waited = false;  // q, out, partials and counters are touched only after pdl_wait()

  if (a.flags & KVMIX_DECODE_POOL_WRITTEN) {  // the previous kernel wrote the pool: no early KV copies
    pdl_wait();
    waited = true;
  }
  Bounds bnd{RESCALE_SLACK, 5};
  const int piece_end = a.cta_ptr[blockIdx.x + 1];
  bool primed = false;  // the piece's first tiles were issued while the previous piece merged
#ifdef KVMIX_CTA_TIMES
  int dbg_k = 0;
#define KVMIX_STAMP(j) \
  if (threadIdx.x == 0 && blockIdx.x < 4096 && dbg_k < 3) g_cta_times[blockIdx.x][4 + 4 * dbg_k + (j)] = gtimer();
#else
#define KVMIX_STAMP(j)
#endif
  for (int piece = a.cta_ptr[blockIdx.x]; piece < piece_end; ++piece) {
  KVMIX_STAMP(0)
  const Unit u = load_unit(a, piece);
  const int ntiles = u.thi - u.tlo;
  const int nmine = ntiles > warp ? (ntiles - warp + NW - 1) / NW : 0;
  const uint8_t* kv2 = a.int2_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_pages) * (int64_t)C::PS;
  const uint8_t* kv4 = a.int4_pool + ((a.layer * a.n_kv + u.kvh) * a.pool_int4) * (int64_t)C::SS;

  // tile metadata: the page id (INT2 tile) or this lane's slot ids (INT4 tile), loaded two
  // iterations before its copy is issued so the copy never waits on the index load
  auto load_meta = [&](int k) -> int {
    return k < nmine ? tile_meta(a, u, u.tlo + warp + k * NW, lane) : 0;
  };
  auto issue = [&](int k, int meta, int s) {
    issue_tile<D>(u, u.tlo + warp + k * NW, meta, ring + s * C::BUF, &bars[warp][s], lane, kv2, kv4);
  };
  if (MEMORY && !primed) {
    if (C::MERGE_IN_RING) fence_proxy_async();  // the previous piece merged through the ring
    int s0 = stage;  // the ring continues where the previous piece left it
    for (int k = 0; k < STAGES && k < nmine; ++k) {
      issue(k, load_meta(k), s0);
      if (++s0 == STAGES) s0 = 0;
    }
  }
  primed = false;
  int meta_next = load_meta(STAGES), meta_next2 = load_meta(STAGES + 1);  // metas run two tiles ahead
  // batched key bias: this warp's INT2 tiles are its first k2 tiles; batch b = tiles 16b..16b+15,
  // whose KZ regions one bulk copy per lane stages into kzs (issued one batch ahead)
  const int t0w = u.tlo + warp;
  const int k2 = (KVMIX_KZBATCH && t0w < u.npg) ? min(nmine, (u.npg - t0w + NW - 1) / NW) : 0;
  auto issue_kz = [&](int b) {
    const int n = min(16, k2 - 16 * b);
    __syncwarp();
    fence_proxy_async();  // the slots were last accessed through the generic proxy
    if (lane == 0) mbar_expect_tx(&kzbar[warp], n * C::KZB);
    __syncwarp();
    if (lane < n) {
      const int pid = a.page_ids[u.pg0 + t0w + (16 * b + lane) * NW];
      bulk_g2s(kzs + lane * C::KZB, kv2 + (int64_t)pid * C::PS + PG_KZ(D), C::KZB, &kzbar[warp]);
    }
  };
  if (MEMORY && k2 > 0) issue_kz(0);
  float kbd[4] = {0.f, 0.f, 0.f, 0.f};  // the current batch's biases (int2_batch_bias)

  // ---- Q fragments (see QFrag): built once per CTA by warp 0 into shared memory ----
  // The KV tiles above are this launch's own inputs (written by earlier steps); q, out and
  // the split scratch may belong to the previous kernel in the stream, so wait for it here.
  if (!waited) {
    pdl_wait();
    waited = true;
#ifdef KVMIX_CTA_TIMES
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_cta_times[blockIdx.x][1] = gtimer();
#endif
  }
  if (piece == a.cta_ptr[blockIdx.x]) bnd = pool_bounds(a.pool_status);  // written by earlier kernels
  uint64_t* qtab = reinterpret_cast<uint64_t*>(smem + NW * STAGES * C::BUF);
  float* qraw = reinterpret_cast<float*>(smem + NW * STAGES * C::BUF + C::QTAB + (C::MERGE_IN_RING ? 0 : C::MERGE));
  stage_q<D>(a, u, qraw);
  __syncthreads();
  if (warp == 0) {
    const float qs = build_qtab<D, LO>(qraw, qtab, lane, a.qscale, bnd.ek);
    if (lane == 0) sm_qscale = qs;
  }
  __syncthreads();
  KVMIX_STAMP(1)
  const QFrag<D, LO> qf{qtab + lane};
  const float qscale = sm_qscale;

  Acc<D> acc;
#pragma unroll
  for (int m = 0; m < C::NCH; ++m) acc.o[m][0] = acc.o[m][1] = acc.o[m][2] = acc.o[m][3] = 0.f;
  acc.zs[0] = acc.zs[1] = acc.zs[2] = acc.zs[3] = 0.f;
  acc.zs2[0] = acc.zs2[1] = acc.zs2[2] = acc.zs2[3] = 0.f;
  Softmax st{0.f, 0.f, false, bnd.slack};

  for (int k = 0; k < nmine; ++k) {
    const int t = u.tlo + warp + k * NW;
    const uint8_t* buf = ring + stage * C::BUF;
    const int meta = meta_next;
#if KVMIX_META2
    meta_next = meta_next2;
    meta_next2 = load_meta(k + STAGES + 2);
#else
    meta_next = load_meta(k + STAGES + 1);
#endif
    if (MEMORY) mbar_wait(&bars[warp][stage], phase);
    if (APPEND && u.n4 > 0 && t == u.npg + (u.n4 - 1) / 32) {
      // K4 fused: quantize the newest token over the stale copy the TMA brought in; a V
      // scale beyond this launch's bound switches the warp to exact-max softmax (p <= 1)
      float vs = 0.f;
      if (lane < C::NGRP) vs = append_group<D>(a, u, ring + stage * C::BUF + ((u.n4 - 1) % 32) * C::SS, lane);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) vs = fmaxf(vs, __shfl_xor_sync(0xffffffffu, vs, off));
      if (15 - ilog2f(fmaxf(vs, 1.f)) < (int)st.slack) st.slack = 0.f;
      __syncwarp();
    }
    if (!COMPUTE) {
      // measurement variant: data movement only (no dequant / MMA)
#ifndef KVMIX_INT2_LIKELY
#define KVMIX_INT2_LIKELY 1  // lay the INT2 tile out as the fall-through path (QK, softmax, PV contiguous)
#endif
    } else if (KVMIX_INT2_LIKELY ? __builtin_expect(t < u.npg, 1) : (t < u.npg)) {
      float kb0 = 0.f, kb1 = 0.f;
      if (KVMIX_KZBATCH) {
        const int j = k & 15;
        if (j == 0) {
          if (MEMORY) mbar_wait(&kzbar[warp], kzphase);
          kzphase ^= 1u;
          int2_batch_bias<D, LO>(kzs, qf, lane, kbd);
          if (MEMORY && k + 16 < k2) issue_kz(k / 16 + 1);
        }
        const int src = 4 * (j & 7) + q;
        kb0 = __shfl_sync(0xffffffffu, j < 8 ? kbd[0] : kbd[2], src);
        kb1 = __shfl_sync(0xffffffffu, j < 8 ? kbd[1] : kbd[3], src);
      }
      int2_tile<D, LO>(buf, qf, qscale, lane, st, acc, kb0, kb1);
    } else {
      const int nv = min(32, u.n4 - 32 * (t - u.npg));
      if (nv == 32) int4_tile<D, true, LO>(buf, 32, qf, qscale, lane, st, acc);
      else int4_tile<D, false, LO>(buf, nv, qf, qscale, lane, st, acc);
    }
    __syncwarp();
    if (MEMORY && k + STAGES < nmine) {
      // Reads-before-async-writes: every lane's LDS of this slot has completed (its values were
      // consumed above, before __syncwarp), so the copy may overwrite the slot without a proxy
      // fence -- the same release a TMA consumer gives its producer through an mbarrier.  The
      // fused append wrote the slot through the generic proxy, so that path keeps the fence.
      if (APPEND || KVMIX_TILEFENCE) fence_proxy_async();
      issue(k + STAGES, meta, stage);
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1u;
    }
  }

  KVMIX_STAMP(2)
  // ---- the next piece's first tiles stream in while this one merges (the ring is idle) ----
  if (MEMORY && !C::MERGE_IN_RING && piece + 1 < piece_end) {
    prime_piece<D>(a, load_unit(a, piece + 1), warp, lane, ring, bars, stage);
    primed = true;
  }
  // ---- finalize this warp: l per head from the ones rows, acc[h][c] = 2^(24-2e) O^T + zsum ----
  const float l0 = __shfl_sync(0xffffffffu, acc.zs[0] + acc.zs2[0], 28 + q);  // row 7 >= NG
  const float l1 = __shfl_sync(0xffffffffu, acc.zs[1] + acc.zs2[1], 28 + q);
  __syncthreads();  // every warp is done with the q table and the previous merge scratch
  float* sm_acc = reinterpret_cast<float*>(C::MERGE_IN_RING ? smem : smem + NW * STAGES * C::BUF + C::QTAB);
  float* sm_m = sm_acc + NW * 8 * D;
  float* sm_l = sm_m + NW * 8;
  store_warp_acc<D>(acc, sm_acc, warp, lane);
  if (g == 0) {
    sm_m[warp * 8 + 2 * q] = st.init ? st.m0 : -INFINITY;  // a warp without tiles contributes nothing
    sm_m[warp * 8 + 2 * q + 1] = st.init ? st.m1 : -INFINITY;
    sm_l[warp * 8 + 2 * q] = l0;
    sm_l[warp * 8 + 2 * q + 1] = l1;
  }
  finish_piece<D>(a, u, sm_m, sm_l, sm_acc, &sm_flag);
  __syncthreads();  // merge scratch (ring) and the q table are free for the next piece
  KVMIX_STAMP(3)
#ifdef KVMIX_CTA_TIMES
  ++dbg_k;
#endif
  }
#ifdef KVMIX_CTA_TIMES
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_cta_times[blockIdx.x][2] = gtimer();
#endif
}

// ====================================================================================
// Variant 1: simple CUDA-core kernel (fp32 dequant straight from HBM).  Slow; kept as
// an independent on-GPU cross-check of the tensor-core kernel at full sizes.
template <int D>
__global__ void __launch_bounds__(NW * 32) decode_simple_kernel(const DecodeArgs a) {
  constexpr int CPL = D / 32;
  __shared__ float qs[8][D];
  extern __shared__ __align__(16) float sm_acc[];  // [NW * 8 * D] (dynamic: NW may be large)
  __shared__ float sm_m[NW * 8], sm_l[NW * 8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  __shared__ int sm_flag;
  pdl_wait();
  for (int piece = a.cta_ptr[blockIdx.x]; piece < a.cta_ptr[blockIdx.x + 1]; ++piece) {
  const Unit u = load_unit(a, piece);
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
  auto hf = [](const uint8_t* p, int idx) { return __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(p)[idx])); };
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
          const uint32_t kc = (rec[pg_kc_off(D, r >> 2, c)] >> (2 * (r & 3))) & 3u;
          kx[i] = fmaf((float)kc, hf(rec + PG_KS(D), pg_kp_idx(D, c)), hf(rec + PG_KZ(D), pg_kp_idx(D, c)));
          const uint32_t vc = (rec[PG_VC(D) + pg_vc_off(D, r, c >> 2)] >> (2 * (c & 3))) & 3u;
          const int pj = pg_vp_idx(D, r, c / G);
          vx[i] = fmaf((float)vc, hf(rec + PG_VS(D), pj), hf(rec + PG_VZ(D), pj));
        }
      } else {
        const int64_t slot = a.int4_ids[u.i40 + 32 * (t - u.npg) + r];
        const uint8_t* rec = kv4 + slot * slot_stride(D);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const int c = lane + 32 * i;
          const uint32_t kc = (rec[sl_kc_off(D, c >> 1)] >> (4 * (c & 1))) & 15u;
          kx[i] = fmaf((float)kc, hf(rec + SL_KS(D), c / G), hf(rec + SL_KZ(D), c / G));
          const uint32_t vc = (rec[SL_VC(D) + sl_vc_off(D, c >> 1)] >> (4 * (c & 1))) & 15u;
          vx[i] = fmaf((float)vc, hf(rec + SL_VS(D), c / G), hf(rec + SL_VZ(D), c / G));
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
  finish_piece<D>(a, u, sm_m, sm_l, sm_acc, &sm_flag);
  __syncthreads();
  }
}

template <typename Kern>
static int launch_kernel(Kern kern, const DecodeArgs& a, int64_t n_cta, int smem, cudaStream_t s, int nwarps = NW) {
  if (smem > 32 * 1024) {  // opt in above the default 48 KB, static shared memory included
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
  }
  // programmatic dependent launch: this grid may start while the previous kernel in the
  // stream drains; the kernel waits (griddepcontrol.wait) before touching q / out / scratch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_cta);
  cfg.blockDim = dim3(nwarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
  return check_launch("flash_decode");
}

template <int D>
static int launch_decode(const DecodeArgs& a, int64_t n_work, int variant, cudaStream_t s) {  // n_work = CTAs
  switch (variant) {
    case 0:
      // fp32 q carries bits fp16 cannot hold: add the q - fp16(q) correction MMAs
      if (a.app_k != nullptr) {  // K4 fused decode append
        if (a.q_dtype == KVMIX_F32)
          return launch_kernel(decode_mma_kernel<D, true, true, true, true>, a, n_work, Cfg<D>::SMEM, s);
        return launch_kernel(decode_mma_kernel<D, true, true, false, true>, a, n_work, Cfg<D>::SMEM, s);
      }
      if (a.q_dtype == KVMIX_F32) return launch_kernel(decode_mma_kernel<D, true, true, true>, a, n_work, Cfg<D>::SMEM, s);
      return launch_kernel(decode_mma_kernel<D, true, true, false>, a, n_work, Cfg<D>::SMEM, s);
    case 1: return launch_kernel(decode_simple_kernel<D>, a, n_work, NW * 8 * D * (int)sizeof(float), s);
#ifdef KVMIX_MEASURE_VARIANTS
    case 2: return launch_kernel(decode_mma_kernel<D, false, true>, a, n_work, Cfg<D>::SMEM, s);
    case 3: return launch_kernel(decode_mma_kernel<D, true, false>, a, n_work, Cfg<D>::SMEM, s);
#endif
    default: return fail(KVMIX_EINVAL, "variant not built (2 and 3 need -DKVMIX_MEASURE_VARIANTS)");
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

#ifdef KVMIX_CTA_TIMES
extern "C" int kvmix_debug_cta_times(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_cta_times, sizeof(unsigned long long) * 16 * n) == cudaSuccess ? 0 : -5;
}
#endif

extern "C" int kvmix_merge_partials(const float* acc, const float* lse, const float* mx, int64_t n, int64_t d,
                                    float* out, void* stream) {
  if (n <= 0) return fail(KVMIX_EINVAL, "cannot merge an empty partial list");
  merge_partials_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(acc, lse, mx, n, d, out);
  return check_launch("merge_partials");
}

static int flash_decode_impl(const void* q, int32_t q_dtype, void* const* outs, int32_t n_outs, int64_t out_heads,
                             int64_t out_head0, int32_t out_dtype,
                             const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages, int64_t pool_int4,
                             int64_t layer, int64_t n_kv, int64_t d, int64_t n_q, int64_t batch,
                             const int32_t* page_indptr, const int32_t* page_ids, const int32_t* int4_indptr,
                             const int32_t* int4_ids, const int32_t* int4_count, const int32_t* work,
                             const int32_t* cta_ptr, int64_t n_cta,
                             float* partials, int32_t* counters, float scale, int32_t variant, const void* k_new,
                             const void* v_new, int32_t kv_dtype, uint8_t* int4_pool_w, int32_t* pool_status,
                             int32_t flags, void* stream) {
  if (n_kv <= 0 || n_q % n_kv) return fail(KVMIX_EINVAL, "n_heads not a multiple of the pool's n_kv_heads");
  const int64_t gq = n_q / n_kv;
  if (gq > 8) return fail(KVMIX_EINVAL, "GQA group > 8 not supported");
  if (batch <= 0 || n_cta <= 0 || n_cta > (1 << 20)) return fail(KVMIX_EINVAL, "empty batch or CTA schedule");
  if (!work || !cta_ptr || !counters) return fail(KVMIX_EINVAL, "work, cta_ptr and counters are required");
  if (q_dtype < 0 || q_dtype > 2 || out_dtype < 0 || out_dtype > 2) return fail(KVMIX_EINVAL, "bad dtype");
  if (variant < 0 || variant > 3) return fail(KVMIX_EINVAL, "bad variant");
  if (!outs || n_outs < 1 || n_outs > MAX_OUTS) return fail(KVMIX_EINVAL, "1 to 8 output buffers");
  if (out_head0 < 0 || out_head0 + n_q > out_heads) return fail(KVMIX_EINVAL, "head slice outside the output");
  DecodeArgs a;
  a.q = q;
  a.q_dtype = q_dtype;
  for (int p = 0; p < MAX_OUTS; ++p) {
    a.outs[p] = p < n_outs ? outs[p] : nullptr;
    if (p < n_outs && !outs[p]) return fail(KVMIX_EINVAL, "null output buffer");
  }
  a.n_outs = n_outs;
  a.out_heads = (int)out_heads;
  a.out_head0 = (int)out_head0;
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
  a.int4_count = int4_count;
  a.work = work;
  a.cta_ptr = cta_ptr;
  a.part = partials;
  a.counters = counters;
  a.qscale = scale * LOG2E;
  a.app_k = k_new;
  a.app_v = v_new;
  a.app_dtype = kv_dtype;
  a.int4_pool_w = int4_pool_w;
  a.pool_status = pool_status;
  a.flags = flags;
  if (k_new != nullptr) {
    if (variant != 0) return fail(KVMIX_EINVAL, "the fused decode append runs in the tensor-core kernel (variant 0)");
    if (!v_new || !int4_pool_w || kv_dtype < 0 || kv_dtype > 2) return fail(KVMIX_EINVAL, "bad append arguments");
  }
  cudaStream_t s = (cudaStream_t)stream;
  switch (d) {
    case 32: return launch_decode<32>(a, n_cta, variant, s);
    case 64: return launch_decode<64>(a, n_cta, variant, s);
    case 128: return launch_decode<128>(a, n_cta, variant, s);
    default: return fail(KVMIX_EINVAL, "decode supports head_dim 32, 64, 128");
  }
}

extern "C" int kvmix_flash_decode(const void* q, int32_t q_dtype, void* out, int32_t out_dtype,
                                  const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages,
                                  int64_t pool_int4, int64_t layer, int64_t n_kv, int64_t d, int64_t n_q,
                                  int64_t batch, const int32_t* page_indptr, const int32_t* page_ids,
                                  const int32_t* int4_indptr, const int32_t* int4_ids, const int32_t* int4_count,
                                  const int32_t* work, const int32_t* cta_ptr, int64_t n_cta, float* partials,
                                  int32_t* counters, float scale, int32_t variant, int32_t* pool_status, int32_t flags,
                                  void* stream) {
  return flash_decode_impl(q, q_dtype, &out, 1, n_q, 0, out_dtype, int2_pool, int4_pool, pool_pages, pool_int4, layer,
                           n_kv, d, n_q, batch, page_indptr, page_ids, int4_indptr, int4_ids, int4_count, work, cta_ptr,
                           n_cta, partials, counters, scale, variant, nullptr, nullptr, 0, nullptr, pool_status, flags,
                           stream);
}

extern "C" int kvmix_flash_decode_gather(const void* q, int32_t q_dtype, void* const* outs, int32_t n_outs,
                                         int64_t out_heads, int64_t out_head0, int32_t out_dtype,
                                         const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages,
                                         int64_t pool_int4, int64_t layer, int64_t n_kv, int64_t d, int64_t n_q,
                                         int64_t batch, const int32_t* page_indptr, const int32_t* page_ids,
                                         const int32_t* int4_indptr, const int32_t* int4_ids,
                                         const int32_t* int4_count, const int32_t* work, const int32_t* cta_ptr,
                                         int64_t n_cta, float* partials, int32_t* counters, float scale,
                                         int32_t variant, int32_t* pool_status, int32_t flags, void* stream) {
  return flash_decode_impl(q, q_dtype, outs, n_outs, out_heads, out_head0, out_dtype, int2_pool, int4_pool, pool_pages,
                           pool_int4, layer, n_kv, d, n_q, batch, page_indptr, page_ids, int4_indptr, int4_ids,
                           int4_count, work, cta_ptr, n_cta, partials, counters, scale, variant, nullptr, nullptr, 0,
                           nullptr, pool_status, flags, stream);
}

extern "C" int kvmix_flash_decode_append(const void* q, int32_t q_dtype, void* out, int32_t out_dtype,
                                         uint8_t* int2_pool, uint8_t* int4_pool, int64_t pool_pages,
                                         int64_t pool_int4, int64_t layer, int64_t n_kv, int64_t d, int64_t n_q,
                                         int64_t batch, const int32_t* page_indptr, const int32_t* page_ids,
                                         const int32_t* int4_indptr, const int32_t* int4_ids, const int32_t* int4_count,
                                         const int32_t* work, const int32_t* cta_ptr, int64_t n_cta, float* partials,
                                         int32_t* counters, float scale, const void* k_new, const void* v_new,
                                         int32_t kv_dtype, int32_t* pool_status, int32_t flags, void* stream) {
  if (!k_new || !v_new) return fail(KVMIX_EINVAL, "k_new / v_new are required");
  return flash_decode_impl(q, q_dtype, &out, 1, n_q, 0, out_dtype, int2_pool, int4_pool, pool_pages, pool_int4, layer,
                           n_kv, d, n_q, batch, page_indptr, page_ids, int4_indptr, int4_ids, int4_count, work, cta_ptr,
                           n_cta, partials, counters, scale, 0, k_new, v_new, kv_dtype, int4_pool, pool_status, flags,
                           stream);
}
