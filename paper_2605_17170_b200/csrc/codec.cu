// K1 (quantize + pack), K4 data half (INT4 append), K5 (gather-dequant) and the
// generic codec entry points.  Bit-exact with /root/reference/pkg/src/kvmix/quant.py:
// every op in the group arithmetic is an explicit round-to-nearest intrinsic
// (__fsub_rn / __fdiv_rn / __fadd_rn / __float2half_rn), so no contraction or
// fast-math can change a code, scale or zero.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace kvmix {

// ---------------------------------------------------------------------------------
// One warp encodes one token vector x[0..D) as a TokenBlock (quant.py:189-232):
// lane owns channels [lane*CPL, lane*CPL+CPL); groups of 32 channels are reduced
// with segmented shuffles; codes are OR-reduced into 32-bit words.  `st` places the
// payload: st.code(word_index, word) gets code bytes [4w, 4w+4), st.param(j, s, z)
// the fp16 bits of group j's (scale, zero).
template <int D, int BITS, typename Store>
__device__ __forceinline__ void encode_token_warp(const float (&v)[D / 32], const Store& st, int lane, int32_t* err) {
  constexpr int CPL = D / 32;               // channels per lane
  constexpr int LPG = 32 / CPL;             // lanes per group of 32 channels
  constexpr int LPW = 32 / (BITS * CPL);    // lanes per 32-bit code word
  constexpr int LEVELS = (1 << BITS) - 1;
  float mn = v[0], mx = v[0];
  bool finite = true;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    mn = fminf(mn, v[i]);
    mx = fmaxf(mx, v[i]);
    finite &= isfinite(v[i]);
  }
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (!finite && err) atomicOr(err, 1);
  float scale, zero;
  group_params(mn, mx, LEVELS, scale, zero);
  const FastQ f = fast_q(scale, zero);
  uint32_t bits = 0;
#pragma unroll
  for (int i = 0; i < CPL; ++i) bits |= fast_code(v[i], f, scale, zero, LEVELS) << (BITS * i);
  uint32_t word = bits << (BITS * CPL * (lane % LPW));
#pragma unroll
  for (int o = 1; o < LPW; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
  if (lane % LPW == 0) st.code(lane / LPW, word);
  if (lane % LPG == 0) st.param(lane / LPG, pack_param(scale, zero));
}

// Thread c of a block encodes channel c of one KeyPageBlock (quant.py:160-177): 32
// token values of one channel -> code bytes tau = 0..7 (tokens 4tau..4tau+3) stored in
// KC row tau, (scale, zero) into KS / KZ (device record layout, common.cuh).
template <int D>
__device__ __forceinline__ void encode_key_channel(const float (&x)[G], uint8_t* rec, int c, int32_t* err) {
  float mn = x[0], mx = x[0];
  bool finite = true;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    mn = fminf(mn, x[j]);
    mx = fmaxf(mx, x[j]);
    finite &= isfinite(x[j]);
  }
  if (!finite && err) atomicOr(err, 1);
  float scale, zero;
  group_params(mn, mx, 3, scale, zero);
  uint32_t w0 = 0, w1 = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    w0 |= quant_code(x[j], scale, zero, 3) << (2 * j);
    w1 |= quant_code(x[j + 16], scale, zero, 3) << (2 * j);
  }
#pragma unroll
  for (int tau = 0; tau < 8; ++tau) rec[pg_kc_off(D, tau, c)] = (uint8_t)(((tau < 4 ? w0 : w1) >> (8 * (tau & 3))) & 0xffu);
  const uint32_t pz = pack_param(scale, zero);
  reinterpret_cast<uint16_t*>(rec + PG_KS(D))[pg_kp_idx(D, c)] = (uint16_t)(pz & 0xffffu);
  reinterpret_cast<uint16_t*>(rec + PG_KZ(D))[pg_kp_idx(D, c)] = (uint16_t)(pz >> 16);
}

// TokenBlock placement inside a staged INT2 page record (token row t of the page).
template <int D>
struct PageVStore {
  uint8_t* rec;
  int t;
  __device__ void code(int w, uint32_t word) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) rec[PG_VC(D) + pg_vc_off(D, t, 4 * w + k)] = (uint8_t)(word >> (8 * k));
  }
  __device__ void param(int j, uint32_t pz) const {
    reinterpret_cast<uint16_t*>(rec + PG_VS(D))[pg_vp_idx(D, t, j)] = (uint16_t)(pz & 0xffffu);
    reinterpret_cast<uint16_t*>(rec + PG_VZ(D))[pg_vp_idx(D, t, j)] = (uint16_t)(pz >> 16);
  }
};
// INT4 TokenBlock placement inside a staged slot record: K (V = false) or V half.
template <int D, bool V>
struct SlotStore {
  uint8_t* rec;
  __device__ void code(int w, uint32_t word) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = 4 * w + k;
      rec[V ? SL_VC(D) + sl_vc_off(D, i) : sl_kc_off(D, i)] = (uint8_t)(word >> (8 * k));
    }
  }
  __device__ void param(int j, uint32_t pz) const {
    reinterpret_cast<uint16_t*>(rec + (V ? SL_VS(D) : SL_KS(D)))[j] = (uint16_t)(pz & 0xffffu);
    reinterpret_cast<uint16_t*>(rec + (V ? SL_VZ(D) : SL_KZ(D)))[j] = (uint16_t)(pz >> 16);
  }
};

// ------------------------------ generic codec ----------------------------------------
// Runtime head_dim (any d for key pages -- LAYOUT.md's worked example has d = 2 --,
// any multiple of 32 for token blocks).  These back the single-block reference API.
__global__ void encode_key_pages_kernel(const float* __restrict__ keys, int64_t n_pages, int d,
                                        uint8_t* __restrict__ out, int64_t out_stride, int32_t* err) {
  const int64_t p = blockIdx.x;
  uint8_t* blk = out + p * out_stride;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float x[G];
#pragma unroll
    for (int j = 0; j < G; ++j) x[j] = keys[(p * G + j) * d + c];
    float mn = x[0], mx = x[0];
    bool finite = true;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      mn = fminf(mn, x[j]);
      mx = fmaxf(mx, x[j]);
      finite &= isfinite(x[j]);
    }
    if (!finite && err) atomicOr(err, 1);
    float scale, zero;
    group_params(mn, mx, 3, scale, zero);
    uint32_t w0 = 0, w1 = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      w0 |= quant_code(x[j], scale, zero, 3) << (2 * j);
      w1 |= quant_code(x[j + 16], scale, zero, 3) << (2 * j);
    }
    reinterpret_cast<uint32_t*>(blk)[2 * c] = w0;
    reinterpret_cast<uint32_t*>(blk)[2 * c + 1] = w1;
    reinterpret_cast<uint32_t*>(blk + 8 * (int64_t)d)[c] = pack_param(scale, zero);
  }
}

// warp per token; group j of 32 channels handled with lane = channel
__global__ void encode_token_blocks_kernel(const float* __restrict__ x, int64_t n, int d, int bits,
                                           uint8_t* __restrict__ out, int64_t out_stride, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= n) return;
  const int levels = (1 << bits) - 1;
  const int lpw = 32 / bits;  // lanes per 32-bit code word
  uint8_t* blk = out + t * out_stride;
  for (int j = 0; j < d / G; ++j) {
    const float v = x[t * d + j * G + lane];
    float mn = v, mx = v;
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (!isfinite(v) && err) atomicOr(err, 1);
    float scale, zero;
    group_params(mn, mx, levels, scale, zero);
    uint32_t word = quant_code(v, scale, zero, levels) << (bits * (lane % lpw));
    for (int o = 1; o < lpw; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
    if (lane % lpw == 0) reinterpret_cast<uint32_t*>(blk)[j * bits + lane / lpw] = word;
    if (lane == 0) reinterpret_cast<uint32_t*>(blk + d * bits / 8)[j] = pack_param(scale, zero);
  }
}

__global__ void decode_key_pages_kernel(const uint8_t* __restrict__ blocks, int64_t n_pages, int d,
                                        int64_t in_stride, float* __restrict__ out) {
  const int64_t p = blockIdx.x;
  const uint8_t* b = blocks + p * in_stride;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const uint32_t w0 = reinterpret_cast<const uint32_t*>(b)[2 * c];
    const uint32_t w1 = reinterpret_cast<const uint32_t*>(b)[2 * c + 1];
    const uint32_t pr = reinterpret_cast<const uint32_t*>(b + 8 * (int64_t)d)[c];
    const float s = __half2float(__ushort_as_half((unsigned short)(pr & 0xffff)));
    const float z = __half2float(__ushort_as_half((unsigned short)(pr >> 16)));
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const uint32_t code = ((j < 16 ? w0 : w1) >> (2 * (j & 15))) & 3u;
      out[(p * G + j) * d + c] = __fmaf_rn((float)code, s, z);  // code*scale exact, one rounding
    }
  }
}

// thread per (block, channel)
__global__ void decode_token_blocks_kernel(const uint8_t* __restrict__ blocks, int64_t n, int d, int bits,
                                           int64_t in_stride, float* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * d) return;
  int64_t t = i / d;
  int c = (int)(i % d);
  const uint8_t* b = blocks + t * in_stride;
  uint32_t byte = b[c * bits / 8];
  uint32_t code = (byte >> ((c * bits) & 7)) & ((1u << bits) - 1);
  const uint8_t* pp = b + d * bits / 8 + 4 * (c / G);
  uint32_t pr = (uint32_t)pp[0] | ((uint32_t)pp[1] << 8) | ((uint32_t)pp[2] << 16) | ((uint32_t)pp[3] << 24);
  float s = __half2float(__ushort_as_half((unsigned short)(pr & 0xffff)));
  float z = __half2float(__ushort_as_half((unsigned short)(pr >> 16)));
  out[i] = __fmaf_rn((float)code, s, z);
}

// One warp per ragged group (quant.py:64-87).
__global__ void quantize_groups_kernel(const float* __restrict__ x, const int64_t* __restrict__ offsets,
                                       int64_t n_groups, int bits, uint8_t* __restrict__ codes,
                                       float* __restrict__ scale_out, float* __restrict__ zero_out, int32_t* err) {
  int lane = threadIdx.x & 31;
  int64_t gi = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gi >= n_groups) return;
  int64_t lo = offsets[gi], hi = offsets[gi + 1];
  float mn = INFINITY, mx = -INFINITY;
  bool finite = true;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    float v = x[i];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
    finite &= isfinite(v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (!finite && err) atomicOr(err, 1);
  int levels = (1 << bits) - 1;
  float s, z;
  group_params(mn, mx, levels, s, z);
  for (int64_t i = lo + lane; i < hi; i += 32) codes[i] = (uint8_t)quant_code(x[i], s, z, levels);
  if (lane == 0) {
    scale_out[gi] = s;
    zero_out[gi] = z;
  }
}

// thread per element (quant.py:90-93): code * fp16(scale) + fp16(zero), the product and
// the sum rounded separately like numpy's fp32 expression (no contraction to an FMA).
__global__ void dequantize_groups_kernel(const uint8_t* __restrict__ codes, const int64_t* __restrict__ offsets,
                                         int64_t n_groups, const float* __restrict__ scale,
                                         const float* __restrict__ zero, float* __restrict__ out) {
  const int64_t gi = blockIdx.y;
  const int64_t lo = offsets[gi], hi = offsets[gi + 1];
  const float s = __half2float(__float2half_rn(scale[gi])), z = __half2float(__float2half_rn(zero[gi]));
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fadd_rn(__fmul_rn((float)codes[i], s), z);
}

// thread per output byte (quant.py:96-109)
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int bits, uint8_t* __restrict__ out,
                                  int32_t* err) {
  int per = 8 / bits;
  int64_t nb = (n + per - 1) / per;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  uint32_t byte = 0;
  for (int k = 0; k < per; ++k) {
    int64_t j = i * per + k;
    if (j < n) {
      uint32_t c = codes[j];
      if (c >= (1u << bits) && err) atomicOr(err, 2);
      byte |= (c & ((1u << bits) - 1)) << (bits * k);
    }
  }
  out[i] = (uint8_t)byte;
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ packed, int64_t n, int bits, uint8_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int per = 8 / bits;
  out[i] = (packed[i / per] >> (bits * (i % per))) & ((1u << bits) - 1);
}

// ------------------------------ pool data plane ----------------------------------------
// write_prefill INT2 branch (pool.py:236-252 -> write_page :201-215): one CTA per
// (request page, kv head, layer).  The page's 32 K and V rows are staged in shared memory
// with 16-byte loads (chunks XOR-swizzled by row), then every thread encodes 64 elements:
// either one KeyPageBlock channel pair (2 x 32 tokens, quant.py:160-177) or two V
// TokenBlock groups of consecutive tokens (quant.py:189-232), with the exact-fast code
// path (FastQ).  The record is assembled in shared memory in the device layout and leaves
// with coalesced 16-byte stores.
#ifndef KVMIX_INT4_MINB
#define KVMIX_INT4_MINB 12  // INT4 token kernel: 12 resident CTAs per SM (40 registers; measured best of 1 / 6 / 8 / 12)
#endif
#ifndef KVMIX_INT4_PRELOAD
#define KVMIX_INT4_PRELOAD 0  // 1: INT4 token kernel issues K and V group loads together (measured 2% slower)
#endif
#ifndef KVMIX_K1_STAGES
#define KVMIX_K1_STAGES 2
#endif
#if KVMIX_K1_STAGES != 2 && KVMIX_K1_STAGES != 3
#error "KVMIX_K1_STAGES must be 2 or 3"
#endif
template <int D, typename T>
struct PrefillCfg {
  static constexpr int ROWB = D * (int)sizeof(T);  // bytes per staged token row
  static constexpr int CHUNKS = ROWB / 16;
  static constexpr int SWZ = CHUNKS >= 8 ? 7 : CHUNKS - 1;
  static constexpr int TILE = G * ROWB;
  static constexpr int STAGES = KVMIX_K1_STAGES;  // 2 or 3 items of K / V rows in flight per CTA
  static constexpr int SMEM = 2 * STAGES * TILE + page_stride(D) + 16;  // stages x (K, V) + the record + page ids
};

#ifndef KVMIX_K1_MINB
#define KVMIX_K1_MINB 5  // register budget for at most this many CTAs per SM (5 at d = 128 bf16: 1.3% faster than no bound)
#endif
// the page kernel's resident CTAs per SM as shared memory allows, capped at KVMIX_K1_MINB (its launch bound)
template <int D, typename T>
struct K1MinBlocks {
  static constexpr int fit = (227 * 1024) / (PrefillCfg<D, T>::SMEM + 1024);
  static constexpr int value = fit < 1 ? 1 : (fit > KVMIX_K1_MINB ? KVMIX_K1_MINB : fit);
};

template <int D, typename T>
__device__ __forceinline__ uint8_t* staged(uint8_t* tile, int row, int byte) {
  using P = PrefillCfg<D, T>;
  return tile + row * P::ROWB + ((((byte >> 4) ^ (row & P::SWZ))) << 4) + (byte & 15);
}
// the 32 channels of group j in staged row `row`, as 16-byte loads
template <int D, typename T>
__device__ __forceinline__ void load_row_group(uint8_t* tile, int row, int j, float (&x)[G]) {
  constexpr int PER16 = 16 / (int)sizeof(T);  // elements per 16-byte chunk
#pragma unroll
  for (int k = 0; k < G / PER16; ++k) {
    const uint4 v = *reinterpret_cast<const uint4*>(staged<D, T>(tile, row, (int)sizeof(T) * (G * j + PER16 * k)));
    if constexpr (sizeof(T) == 4) {
      x[4 * k] = __uint_as_float(v.x); x[4 * k + 1] = __uint_as_float(v.y);
      x[4 * k + 2] = __uint_as_float(v.z); x[4 * k + 3] = __uint_as_float(v.w);
    } else {
      unpack2<T>(v.x, x[8 * k], x[8 * k + 1]);
      unpack2<T>(v.y, x[8 * k + 2], x[8 * k + 3]);
      unpack2<T>(v.z, x[8 * k + 4], x[8 * k + 5]);
      unpack2<T>(v.w, x[8 * k + 6], x[8 * k + 7]);
    }
  }
}
// channel c of staged row `row`
template <int D, typename T>
__device__ __forceinline__ float load_one(uint8_t* tile, int row, int c) {
  return to_f32(*reinterpret_cast<const T*>(staged<D, T>(tile, row, (int)sizeof(T) * c)));
}
// two consecutive channels (c even) of staged row `row`
template <int D, typename T>
__device__ __forceinline__ void load_pair(uint8_t* tile, int row, int c, float& a, float& b) {
  if constexpr (sizeof(T) == 4) {
    const float2 v = *reinterpret_cast<const float2*>(staged<D, T>(tile, row, 4 * c));
    a = v.x;
    b = v.y;
  } else {
    unpack2<T>(*reinterpret_cast<const uint32_t*>(staged<D, T>(tile, row, 2 * c)), a, b);
  }
}

// Item cursor for the persistent page CTAs, advanced by the grid stride with precomputed
// carries (no 64-bit division per item).  KVMIX_K1_ORDER 1 (default): item = (l * n_pages + p)
// * H + h -- the CTAs resident at one time cover all kv heads of a run of pages, so the rows
// they gather (256 B per head of a 2 KB token row [H][d]) complete whole token rows together
// (DRAM page locality); 0: item = (l * H + h) * n_pages + p (one head's pages at a time).
#ifndef KVMIX_K1_ORDER
#define KVMIX_K1_ORDER 1
#endif
struct ItemCursor {
  int a, b, l;  // inner / middle / outer coordinate
#if KVMIX_K1_ORDER
  __device__ __forceinline__ int page() const { return b; }
  __device__ __forceinline__ int head() const { return a; }
#else
  __device__ __forceinline__ int page() const { return a; }
  __device__ __forceinline__ int head() const { return b; }
#endif
  __device__ void init(int64_t item, int na, int nb) {
    const int64_t ab = item / na;
    a = (int)(item - ab * na);
    l = (int)(ab / nb);
    b = (int)(ab - (int64_t)l * nb);
  }
  __device__ void advance(int da, int db, int dl, int na, int nb) {
    a += da;
    b += db;
    l += dl;
    if (a >= na) {
      a -= na;
      ++b;
    }
    if (b >= nb) {
      b -= nb;
      ++l;
    }
  }
};

// K1 page kernel: write_prefill's INT2 data path (pool.py:228-262).  Persistent: CTA b runs
// items b, b + grid, ... (item = (layer, kv head, page): one KeyPageBlock + the page's 32 INT2
// V TokenBlocks); the K / V tiles of the next item stream in (cp.async, 2 stages) while this
// one is encoded.  Each thread owns one 16 B column chunk of NPASS staged rows of both tiles
// (fixed smem offsets); the rows' token ids and the page id are loaded two items ahead into
// registers, so no copy or store waits on an index load.  (A variant that also ran the INT4
// tokens as items of the same launch was slower: instruction-cache misses; another that
// staged the index words through shared memory with cp.async lost ~8%.)
template <int D, typename T>
__global__ void __launch_bounds__(128, K1MinBlocks<D, T>::value) prefill_pages_kernel(const T* __restrict__ keys, const T* __restrict__ values,
                                                            int64_t n_tokens, int64_t n_kv_heads, int64_t n_pages,
                                                            int64_t n_items, const int32_t* __restrict__ page_tokens,
                                                            const int32_t* __restrict__ page_ids,
                                                            uint8_t* __restrict__ int2_pool, int64_t pool_pages,
                                                            int32_t* err) {
  using P = PrefillCfg<D, T>;
  constexpr int RPP = 128 / P::CHUNKS;  // rows per copy pass
  constexpr int NPASS = G / RPP;        // rows per thread and tile
  static_assert(128 % P::CHUNKS == 0 && G % RPP == 0, "staging geometry");
  extern __shared__ __align__(16) uint8_t psm[];
  uint8_t* srec = psm + 2 * P::STAGES * P::TILE;
  const int tid = threadIdx.x;
  const int ch = tid % P::CHUNKS, r0 = tid / P::CHUNKS;
  const int np = (int)n_pages, H = (int)n_kv_heads;
  const int64_t grid = gridDim.x;
#if KVMIX_K1_ORDER
  const int na = H, nb = np;
#else
  const int na = np, nb = H;
#endif
  const int da = (int)(grid % na);
  const int64_t dab = grid / na;
  const int db = (int)(dab % nb), dl = (int)(dab / nb);
  // cursors of this item and the next three: with 2 stages nxt is fetched while this one is
  // encoded and nn's indices load; with 3 stages nn is fetched and n3's indices load
  ItemCursor cur, nxt, nn, n3;
  cur.init(blockIdx.x, na, nb);
  nxt = cur;
  nxt.advance(da, db, dl, na, nb);
  nn = nxt;
  nn.advance(da, db, dl, na, nb);
  n3 = nn;
  n3.advance(da, db, dl, na, nb);
  // Token ids are loaded into registers two items ahead.  The page id travels with the item's
  // tiles (one 4 B cp.async by thread 0 into spid[stage]): kept in a register it is CTA-uniform,
  // and the compiler moved it into a uniform register right at its load -- a full load-latency
  // stall per item (19% of the kernel's stall samples in ncu).
  int* spid = reinterpret_cast<int*>(srec + page_stride(D));
  int tok_a[NPASS], tok_b[NPASS];
  auto load_tok = [&](const ItemCursor& c, int64_t item, int (&tok)[NPASS]) {
#pragma unroll
    for (int j = 0; j < NPASS; ++j) tok[j] = item < n_items ? __ldg(page_tokens + (int64_t)c.page() * G + r0 + RPP * j) : 0;
  };
  const int64_t row_step = (int64_t)H * D;  // elements between consecutive tokens
  auto fetch = [&](const ItemCursor& c, const int (&tok)[NPASS], int stg) {
    uint8_t* Ks = psm + 2 * stg * P::TILE;
    if (tid == 0) cp_async4(spid + stg, page_ids + c.page());
    const int64_t base = ((int64_t)c.l * n_tokens * H + c.head()) * D;
#pragma unroll
    for (int j = 0; j < NPASS; ++j) {
      const int r = r0 + RPP * j;
      const int64_t off = base + (int64_t)tok[j] * row_step;
      uint8_t* dst = staged<D, T>(Ks, r, 16 * ch);
      cp_async16(dst, reinterpret_cast<const uint8_t*>(keys + off) + 16 * ch);
      cp_async16(dst + P::TILE, reinterpret_cast<const uint8_t*>(values + off) + 16 * ch);
    }
  };
  int stg = 0;
  float kmx = 0.f, vmx = 0.f;  // largest key-page / V scales this thread stored (pool status)
  {
    int tok0[NPASS];
    load_tok(cur, blockIdx.x, tok0);
    if (blockIdx.x < n_items) fetch(cur, tok0, 0);
    cp_async_commit();
    if constexpr (P::STAGES == 3) {
      load_tok(nxt, blockIdx.x + grid, tok0);
      if (blockIdx.x + grid < n_items) fetch(nxt, tok0, 1);
      cp_async_commit();
      load_tok(nn, blockIdx.x + 2 * grid, tok_a);
    } else {
      load_tok(nxt, blockIdx.x + grid, tok_a);
    }
  }
  for (int64_t item = blockIdx.x; item < n_items; item += grid, stg = stg + 1 == P::STAGES ? 0 : stg + 1) {
    if constexpr (P::STAGES == 3) {
      load_tok(n3, item + 3 * grid, tok_b);
      if (item + 2 * grid < n_items) fetch(nn, tok_a, stg == 0 ? 2 : stg - 1);
      cp_async_commit();
      cp_async_wait<2>();  // this item's tiles have landed (the next two may still fly)
    } else {
      load_tok(nn, item + 2 * grid, tok_b);
      if (item + grid < n_items) fetch(nxt, tok_a, stg ^ 1);
      cp_async_commit();
      cp_async_wait<1>();  // this item's tiles have landed (the next item's may still fly)
    }
    if (tid == 0) bulk_wait_read0();  // the previous item's record has left srec
    __syncthreads();  // this stage's rows are visible; srec and the previous stage are free
    uint8_t* Ks = psm + 2 * stg * P::TILE;
    uint8_t* Vs = Ks + P::TILE;
    // D work units of 64 elements: [0, D/2) = KeyPageBlock channels (2u, 2u+1) over the page's
    // 32 tokens; [D/2, D) = V TokenBlock group j of tokens t and t + 16.  At d = 128 every
    // thread runs one unit and warps 0-1 / 2-3 take the K / V halves (no divergence).
#pragma unroll 1
    for (int u = tid; u < D; u += 128) {
      if (u < D / 2) {
        const int c = 2 * u;
        float x0[G], x1[G];
#pragma unroll
        for (int i = 0; i < G; ++i) load_pair<D, T>(Ks, i, c, x0[i], x1[i]);
        uint32_t w0[2], w1[2], pz0, pz1;
        encode_group<2>(x0, w0, pz0, err);
        encode_group<2>(x1, w1, pz1, err);
        kmx = fmaxf(kmx, fmaxf(scale_of(pz0), scale_of(pz1)));
#pragma unroll
        for (int b = 0; b < 8; ++b) {  // channels c, c + 1 are adjacent bytes of KC row b
          const uint32_t sh = 8 * (b & 3);
          *reinterpret_cast<uint16_t*>(srec + pg_kc_off(D, b, c)) =
              (uint16_t)(((w0[b >> 2] >> sh) & 0xffu) | (((w1[b >> 2] >> sh) & 0xffu) << 8));
        }
        uint16_t* ks = reinterpret_cast<uint16_t*>(srec + PG_KS(D));
        uint16_t* kz = reinterpret_cast<uint16_t*>(srec + PG_KZ(D));
        ks[pg_kp_idx(D, c)] = (uint16_t)(pz0 & 0xffffu);
        kz[pg_kp_idx(D, c)] = (uint16_t)(pz0 >> 16);
        ks[pg_kp_idx(D, c + 1)] = (uint16_t)(pz1 & 0xffffu);
        kz[pg_kp_idx(D, c + 1)] = (uint16_t)(pz1 >> 16);
      } else {
        const int v = u - D / 2, j = v / 16;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int t = (v % 16) + 16 * half;
          float x[G];
          load_row_group<D, T>(Vs, t, j, x);  // 16-byte loads; rows t % 8 of a quarter warp differ: no conflicts
          uint32_t w[2], pz;
          encode_group<2>(x, w, pz, err);
          vmx = fmaxf(vmx, scale_of(pz));
#pragma unroll
          for (int b = 0; b < 8; ++b)
            srec[PG_VC(D) + pg_vc_off(D, t, 8 * j + b)] = (uint8_t)((w[b >> 2] >> (8 * (b & 3))) & 0xffu);
          reinterpret_cast<uint16_t*>(srec + PG_VS(D))[pg_vp_idx(D, t, j)] = (uint16_t)(pz & 0xffffu);
          reinterpret_cast<uint16_t*>(srec + PG_VZ(D))[pg_vp_idx(D, t, j)] = (uint16_t)(pz >> 16);
        }
      }
    }
    fence_proxy_async_smem();  // each thread's record writes, ordered before the bulk store's reads
    __syncthreads();
    if (tid == 0) {  // the record leaves with one TMA bulk store; srec is reused after it was read
      const int pid = spid[stg];  // landed with this stage's tiles
      bulk_s2g(int2_pool + (((int64_t)cur.l * H + cur.head()) * pool_pages + pid) * page_stride(D), srec, page_stride(D));
      bulk_commit();
    }
    cur = nxt;
    nxt = nn;
    nn = n3;
    n3.advance(da, db, dl, na, nb);
#pragma unroll
    for (int j = 0; j < NPASS; ++j) tok_a[j] = tok_b[j];
  }
  cp_async_wait<0>();
  if (tid == 0) bulk_wait_read0();
  publish_scales(err, kmx, vmx);
}

// this lane's D/32 consecutive elements, one vector load when they fill 8 or 16 bytes
template <int D, typename T>
__device__ __forceinline__ void load_lane(const T* __restrict__ p, float (&v)[D / 32]) {
  constexpr int NB = (D / 32) * (int)sizeof(T);
  if constexpr (sizeof(T) == 2 && (NB == 8 || NB == 16)) {
    uint32_t w[NB / 4];
    if constexpr (NB == 8) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = x.x; w[1] = x.y;
    } else {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
    }
#pragma unroll
    for (int i = 0; i < NB / 4; ++i) unpack2<T>(w[i], v[2 * i], v[2 * i + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < D / 32; ++k) v[k] = to_f32(p[k]);
  }
}

// INT4 tokens: write_prefill :253-262, write_token :217-226, append_decode_token :284-306.
// A warp encodes 32 / (D/32) tokens of one (kv head, layer): lane = (token, channel group)
// quantizes that group of both K and V (64 elements, exact-fast codes, no shuffles).
// Input element (l, t, h, c) at (l * layer_stride + t * tok_stride + h * D + c); the
// warp's slot records are staged in shared memory (device layout) and stored as 16 B words.
template <int D, typename T>
__global__ void __launch_bounds__(128, KVMIX_INT4_MINB) int4_tokens_kernel(const T* __restrict__ keys, const T* __restrict__ values,
                                                          int64_t n, int64_t layer_stride, int64_t tok_stride,
                                                          int64_t n_kv_heads, int64_t layer0,
                                                          const int32_t* __restrict__ tokens,
                                                          const int32_t* __restrict__ int4_ids,
                                                          uint8_t* __restrict__ int4_pool, int64_t pool_int4,
                                                          int32_t* err) {
  constexpr int SS = slot_stride(D), NG = D / 32, TPW = 32 / NG;  // tokens per warp
  __shared__ __align__(16) uint8_t srec[4][TPW * SS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x / 32;
  // grid (chunks * H, 1, L): the kv head is the fastest index (KVMIX_K1_ORDER), so the CTAs
  // resident together read whole 2 KB token rows [H][d]
#if KVMIX_K1_ORDER
  const int h = (int)(blockIdx.x % (unsigned)n_kv_heads), l = blockIdx.z;
  const int64_t i0 = ((int64_t)(blockIdx.x / (unsigned)n_kv_heads) * 4 + warp) * TPW;  // first token of this warp
#else
  const int h = blockIdx.y, l = blockIdx.z;
  const int64_t i0 = ((int64_t)blockIdx.x * 4 + warp) * TPW;
#endif
  if (i0 >= n) return;
  uint8_t* st = srec[warp];
  for (int k = lane; k < TPW * SS / 4; k += 32) reinterpret_cast<uint32_t*>(st)[k] = 0u;  // padding stays zero
  __syncwarp();
  const int tw = lane / NG, j = lane % NG;
  const int64_t i = i0 + tw;
  float vmx = 0.f;
  if (i < n) {
    const int64_t t = tokens ? tokens[i] : i;
    const int64_t base = l * layer_stride + t * tok_stride + (int64_t)h * D + 32 * j;
    vmx = encode_int4_group<D, T, KVMIX_INT4_PRELOAD>(keys + base, values + base, st + tw * SS, nullptr, j, err);
  }
  publish_scales(err, 0.f, vmx);
  __syncwarp();
  const int nt = (int)min((int64_t)TPW, n - i0);
  for (int c = lane; c < nt * (SS / 16); c += 32) {
    const int tw2 = c / (SS / 16), k = c % (SS / 16);
    const int64_t slot = int4_ids[i0 + tw2];
    reinterpret_cast<uint4*>(int4_pool + (((layer0 + l) * n_kv_heads + h) * pool_int4 + slot) * SS)[k] =
        reinterpret_cast<const uint4*>(st + tw2 * SS)[k];
  }
}

template <typename TO> __device__ __forceinline__ TO from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half from_f32<__half>(float x) { return __float2half_rn(x); }

// K5 gather-dequant (pool.py:394-439): thread per (slot, head, channel) -> k/v in TO (f32 is
// the reference's exact dequantized value; bf16 / f16 are its round-to-nearest image, the
// input of an fp16 / bf16 prefill attention over the pool).
// K5: one thread per (slot, kv head, 8-channel chunk) -- 8 K and 8 V values from one 8 / 16 B
// load per field of the permuted record, written as one 16 B (f16 / bf16) or 32 B (f32) vector
// each.  Values are fp32 code * scale + zero (exact: the product fits fp32), then rounded to TO.
template <typename TO>
__device__ __forceinline__ void store8(TO* p, const float (&x)[8]) {
  if constexpr (sizeof(TO) == 4) {
    reinterpret_cast<float4*>(p)[0] = make_float4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(x[4], x[5], x[6], x[7]);
  } else {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const TO a = from_f32<TO>(x[2 * e]), b = from_f32<TO>(x[2 * e + 1]);
      w[e] = (uint32_t)(*reinterpret_cast<const uint16_t*>(&a)) | ((uint32_t)(*reinterpret_cast<const uint16_t*>(&b)) << 16);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
__device__ __forceinline__ float half_of(uint32_t w, int hi) {
  return __half2float(__ushort_as_half((unsigned short)(hi ? w >> 16 : w & 0xffffu)));
}

template <int D, typename TO>
__global__ void __launch_bounds__(256) gather_dequant_kernel(const uint8_t* __restrict__ int2_pool,
                                                             const uint8_t* __restrict__ int4_pool, int64_t pool_pages,
                                                             int64_t pool_int4, int64_t offset, int64_t layer,
                                                             int64_t n_kv_heads, const int32_t* __restrict__ slots,
                                                             int64_t m, TO* __restrict__ k_out, TO* __restrict__ v_out) {
  constexpr int CH8 = D / 8;  // 8-channel chunks per (slot, head)
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * CH8) return;
  const int h = blockIdx.y;
  const int64_t i = idx / CH8;
  const int c0 = 8 * (int)(idx % CH8);
  const int64_t slot = slots[i];
  float kx[8], vx[8];
  if (slot < offset) {
    const int row = (int)(slot % G);
    const uint8_t* rec = int2_pool + ((layer * n_kv_heads + h) * pool_pages + slot / G) * page_stride(D);
    const uint2 kc = *reinterpret_cast<const uint2*>(rec + pg_kc_off(D, row >> 2, c0));  // channels c0 .. c0+7
    const uint4 ks = *reinterpret_cast<const uint4*>(rec + PG_KS(D) + 2 * (pg_kp_idx(D, c0) & ~7));
    const uint4 kz = *reinterpret_cast<const uint4*>(rec + PG_KZ(D) + 2 * (pg_kp_idx(D, c0) & ~7));
    const uint32_t ksw[4] = {ks.x, ks.y, ks.z, ks.w}, kzw[4] = {kz.x, kz.y, kz.z, kz.w};
    const int sh = 2 * (row & 3);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t code = (((e < 4 ? kc.x : kc.y) >> (8 * (e & 3) + sh)) & 3u);
      const int pos = pg_kp_idx(D, c0 + e) & 7;
      kx[e] = __fmaf_rn((float)code, half_of(ksw[pos >> 1], pos & 1), half_of(kzw[pos >> 1], pos & 1));
    }
    const uint32_t vb0 = rec[PG_VC(D) + pg_vc_off(D, row, c0 >> 2)], vb1 = rec[PG_VC(D) + pg_vc_off(D, row, (c0 >> 2) + 1)];
    const int pj = pg_vp_idx(D, row, c0 / G);
    const float vs = half_of(reinterpret_cast<const uint16_t*>(rec + PG_VS(D))[pj], 0);
    const float vz = half_of(reinterpret_cast<const uint16_t*>(rec + PG_VZ(D))[pj], 0);
#pragma unroll
    for (int e = 0; e < 8; ++e) vx[e] = __fmaf_rn((float)(((e < 4 ? vb0 : vb1) >> (2 * (e & 3))) & 3u), vs, vz);
  } else {
    const uint8_t* rec = int4_pool + ((layer * n_kv_heads + h) * pool_int4 + (slot - offset)) * slot_stride(D);
    const int j = c0 / G;
    const uint32_t kc = *reinterpret_cast<const uint32_t*>(rec + sl_kc_off(D, c0 >> 1));  // payload bytes c0/2 ..+3
    const float ks = half_of(reinterpret_cast<const uint16_t*>(rec + SL_KS(D))[j], 0);
    const float kz = half_of(reinterpret_cast<const uint16_t*>(rec + SL_KZ(D))[j], 0);
    const uint32_t v01 = *reinterpret_cast<const uint16_t*>(rec + SL_VC(D) + sl_vc_off(D, c0 >> 1));
    const uint32_t v23 = *reinterpret_cast<const uint16_t*>(rec + SL_VC(D) + sl_vc_off(D, (c0 >> 1) + 2));
    const uint32_t vc = v01 | (v23 << 16);
    const float vs = half_of(reinterpret_cast<const uint16_t*>(rec + SL_VS(D))[j], 0);
    const float vz = half_of(reinterpret_cast<const uint16_t*>(rec + SL_VZ(D))[j], 0);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      kx[e] = __fmaf_rn((float)((kc >> (4 * e)) & 15u), ks, kz);
      vx[e] = __fmaf_rn((float)((vc >> (4 * e)) & 15u), vs, vz);
    }
  }
  const int64_t o = (i * n_kv_heads + h) * D + c0;
  store8<TO>(k_out + o, kx);
  store8<TO>(v_out + o, vx);
}

}  // namespace kvmix

// =============================== C ABI ===============================================
using namespace kvmix;

#define DISPATCH_D(d, ...)                                   \
  switch (d) {                                               \
    case 32: { constexpr int D = 32; __VA_ARGS__; } break;   \
    case 64: { constexpr int D = 64; __VA_ARGS__; } break;   \
    case 128: { constexpr int D = 128; __VA_ARGS__; } break; \
    case 256: { constexpr int D = 256; __VA_ARGS__; } break; \
    default: return fail(KVMIX_EINVAL, "head_dim must be 32, 64, 128 or 256");  \
  }

extern "C" int64_t kvmix_page_stride(int64_t d) { return page_stride((int)d); }
extern "C" int64_t kvmix_slot_stride(int64_t d) { return slot_stride((int)d); }
// Host-side export of the record permutation the kernels use (same constexpr helpers).
extern "C" int kvmix_page_layout(int64_t d, int64_t* perm) {
  if (d < 32 || d > 256 || d % 32) return fail(KVMIX_EINVAL, "head_dim must be 32, 64, 128 or 256");
  const int D = (int)d, ng = D / 32, kp = key_page_bytes(D), tb2 = tok_bytes(D, 2);
  for (int i = 0; i < page_stride(D); ++i) perm[i] = -1;
  for (int c = 0; c < D; ++c) {
    for (int tau = 0; tau < 8; ++tau) perm[pg_kc_off(D, tau, c)] = 8 * c + tau;
    for (int k = 0; k < 2; ++k) {
      perm[PG_KS(D) + 2 * pg_kp_idx(D, c) + k] = 8 * D + 4 * c + k;
      perm[PG_KZ(D) + 2 * pg_kp_idx(D, c) + k] = 8 * D + 4 * c + 2 + k;
    }
  }
  for (int t = 0; t < G; ++t) {
    for (int b = 0; b < D / 4; ++b) perm[PG_VC(D) + pg_vc_off(D, t, b)] = kp + t * tb2 + b;
    for (int j = 0; j < ng; ++j)
      for (int k = 0; k < 2; ++k) {
        perm[PG_VS(D) + 2 * pg_vp_idx(D, t, j) + k] = kp + t * tb2 + D / 4 + 4 * j + k;
        perm[PG_VZ(D) + 2 * pg_vp_idx(D, t, j) + k] = kp + t * tb2 + D / 4 + 4 * j + 2 + k;
      }
  }
  return KVMIX_OK;
}

extern "C" int kvmix_slot_layout(int64_t d, int64_t* perm) {
  if (d < 32 || d > 256 || d % 32) return fail(KVMIX_EINVAL, "head_dim must be 32, 64, 128 or 256");
  const int D = (int)d, ng = D / 32, tb4 = tok_bytes(D, 4);
  for (int i = 0; i < slot_stride(D); ++i) perm[i] = -1;
  for (int i = 0; i < D / 2; ++i) {
    perm[sl_kc_off(D, i)] = i;
    perm[SL_VC(D) + sl_vc_off(D, i)] = tb4 + i;
  }
  for (int j = 0; j < ng; ++j)
    for (int k = 0; k < 2; ++k) {
      perm[SL_KS(D) + 2 * j + k] = D / 2 + 4 * j + k;
      perm[SL_KZ(D) + 2 * j + k] = D / 2 + 4 * j + 2 + k;
      perm[SL_VS(D) + 2 * j + k] = tb4 + D / 2 + 4 * j + k;
      perm[SL_VZ(D) + 2 * j + k] = tb4 + D / 2 + 4 * j + 2 + k;
    }
  return KVMIX_OK;
}

extern "C" int64_t kvmix_key_page_payload_bytes(int64_t d) { return key_page_bytes((int)d); }
extern "C" int64_t kvmix_token_block_payload_bytes(int64_t d, int64_t b) { return tok_bytes((int)d, (int)b); }

extern "C" int kvmix_encode_key_pages(const float* keys, int64_t n_pages, int64_t d, uint8_t* out,
                                      int64_t out_stride, int32_t* err, void* stream) {
  if (n_pages == 0) return KVMIX_OK;
  if (d <= 0 || out_stride % 4 || out_stride < key_page_bytes((int)d)) return fail(KVMIX_EINVAL, "bad key page shape");
  encode_key_pages_kernel<<<(unsigned)n_pages, 128, 0, (cudaStream_t)stream>>>(keys, n_pages, (int)d, out,
                                                                               out_stride, err);
  return check_launch("encode_key_pages");
}

extern "C" int kvmix_encode_token_blocks(const float* x, int64_t n, int64_t d, int32_t bits, uint8_t* out,
                                         int64_t out_stride, int32_t* err, void* stream) {
  if (n == 0) return KVMIX_OK;
  if (bits != 2 && bits != 4) return fail(KVMIX_EINVAL, "unsupported bitwidth");
  if (d <= 0 || d % G) return fail(KVMIX_EINVAL, "head dim not divisible by the group size");
  if (out_stride % 4) return fail(KVMIX_EINVAL, "out_stride must be a multiple of 4");
  encode_token_blocks_kernel<<<(unsigned)((n + 3) / 4), 128, 0, (cudaStream_t)stream>>>(x, n, (int)d, bits, out,
                                                                                        out_stride, err);
  return check_launch("encode_token_blocks");
}

extern "C" int kvmix_decode_key_pages(const uint8_t* blocks, int64_t n_pages, int64_t d, int64_t in_stride,
                                      float* out, void* stream) {
  if (n_pages == 0) return KVMIX_OK;
  if (d <= 0 || in_stride % 4) return fail(KVMIX_EINVAL, "bad key page shape");
  decode_key_pages_kernel<<<(unsigned)n_pages, 128, 0, (cudaStream_t)stream>>>(blocks, n_pages, (int)d, in_stride,
                                                                               out);
  return check_launch("decode_key_pages");
}

extern "C" int kvmix_decode_token_blocks(const uint8_t* blocks, int64_t n, int64_t d, int32_t bits,
                                         int64_t in_stride, float* out, void* stream) {
  if (n == 0) return KVMIX_OK;
  if (bits != 2 && bits != 4) return fail(KVMIX_EINVAL, "unsupported bitwidth");
  if (d % G) return fail(KVMIX_EINVAL, "head_dim must be a multiple of 32");
  int64_t total = n * d;
  decode_token_blocks_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(blocks, n, (int)d,
                                                                                                 bits, in_stride, out);
  return check_launch("decode_token_blocks");
}

extern "C" int kvmix_quantize_groups(const float* x, const int64_t* offsets, int64_t n_groups, int32_t bits,
                                     uint8_t* codes, float* scale, float* zero, int32_t* err, void* stream) {
  if (n_groups == 0) return KVMIX_OK;
  if (bits != 2 && bits != 4) return fail(KVMIX_EINVAL, "unsupported bitwidth");
  quantize_groups_kernel<<<(unsigned)((n_groups + 3) / 4), 128, 0, (cudaStream_t)stream>>>(x, offsets, n_groups,
                                                                                            bits, codes, scale, zero,
                                                                                            err);
  return check_launch("quantize_groups");
}

extern "C" int kvmix_dequantize_groups(const uint8_t* codes, const int64_t* offsets, int64_t n_groups,
                                       const float* scale, const float* zero, float* out, int64_t max_len,
                                       void* stream) {
  if (n_groups == 0) return KVMIX_OK;
  if (n_groups > 65535) return fail(KVMIX_EINVAL, "at most 65535 groups per call");
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((max_len + 127) / 128, 64)), (unsigned)n_groups);
  dequantize_groups_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(codes, offsets, n_groups, scale, zero, out);
  return check_launch("dequantize_groups");
}

extern "C" int kvmix_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* out, int32_t* err,
                                void* stream) {
  if (n == 0) return KVMIX_OK;
  if (bits != 2 && bits != 4) return fail(KVMIX_EINVAL, "unsupported bitwidth");
  int64_t nb = (n * bits + 7) / 8;
  pack_codes_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, n, bits, out, err);
  return check_launch("pack_codes");
}

extern "C" int kvmix_unpack_codes(const uint8_t* packed, int64_t n, int32_t bits, uint8_t* out, void* stream) {
  if (n == 0) return KVMIX_OK;
  if (bits != 2 && bits != 4) return fail(KVMIX_EINVAL, "unsupported bitwidth");
  unpack_codes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(packed, n, bits, out);
  return check_launch("unpack_codes");
}

template <typename T>
static int launch_prefill(const void* keys, const void* values, int64_t L, int64_t N, int64_t H, int64_t d,
                          const int32_t* page_tokens, const int32_t* page_ids, int64_t np, const int32_t* int4_tokens,
                          const int32_t* int4_ids, int64_t n4, uint8_t* int2_pool, int64_t pool_pages,
                          uint8_t* int4_pool, int64_t pool_int4, int32_t* err, cudaStream_t s) {
  const T* k = (const T*)keys;
  const T* v = (const T*)values;
  if (np > 0) {
    const int64_t items = np * H * L;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    DISPATCH_D(d, {
      constexpr int SM = PrefillCfg<D, T>::SMEM;
      if (SM > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(prefill_pages_kernel<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
        if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
      }
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prefill_pages_kernel<D, T>, 128, SM);
      const int64_t grid = std::min<int64_t>(items, (int64_t)n_sm * std::max(per_sm, 1));
      prefill_pages_kernel<D, T><<<(unsigned)grid, 128, SM, s>>>(k, v, N, H, np, items, page_tokens, page_ids,
                                                               int2_pool, pool_pages, err);
    });
  }
  if (n4 > 0) {
    const int64_t tpc = 4 * (32 / (d / 32));  // tokens per CTA
#if KVMIX_K1_ORDER
    dim3 grid((unsigned)((n4 + tpc - 1) / tpc * H), 1, (unsigned)L);
#else
    dim3 grid((unsigned)((n4 + tpc - 1) / tpc), (unsigned)H, (unsigned)L);
#endif
    DISPATCH_D(d, int4_tokens_kernel<D, T><<<grid, 128, 0, s>>>(k, v, n4, N * H * D, H * D, H, 0, int4_tokens,
                                                                int4_ids, int4_pool, pool_int4, err));
  }
  return check_launch("write_prefill");
}

extern "C" int kvmix_write_prefill(const void* keys, const void* values, int32_t dtype, int64_t L, int64_t N,
                                   int64_t H, int64_t d, const int32_t* page_tokens, const int32_t* page_ids,
                                   int64_t np, const int32_t* int4_tokens, const int32_t* int4_ids, int64_t n4,
                                   uint8_t* int2_pool, int64_t pool_pages, uint8_t* int4_pool, int64_t pool_int4,
                                   int32_t* err, void* stream) {
  if (L <= 0 || H <= 0 || H > 65535 || L > 65535) return fail(KVMIX_EINVAL, "bad layer/head counts");
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case KVMIX_F32:
      return launch_prefill<float>(keys, values, L, N, H, d, page_tokens, page_ids, np, int4_tokens, int4_ids, n4,
                                   int2_pool, pool_pages, int4_pool, pool_int4, err, s);
    case KVMIX_BF16:
      return launch_prefill<__nv_bfloat16>(keys, values, L, N, H, d, page_tokens, page_ids, np, int4_tokens,
                                           int4_ids, n4, int2_pool, pool_pages, int4_pool, pool_int4, err, s);
    case KVMIX_F16:
      return launch_prefill<__half>(keys, values, L, N, H, d, page_tokens, page_ids, np, int4_tokens, int4_ids, n4,
                                    int2_pool, pool_pages, int4_pool, pool_int4, err, s);
    default:
      return fail(KVMIX_EINVAL, "unsupported dtype");
  }
}

template <typename T>
static int launch_append(const void* k, const void* v, int64_t n, int64_t Lin, int64_t layer0, int64_t H, int64_t d,
                         int64_t layer_stride, int64_t tok_stride, const int32_t* int4_ids, uint8_t* int4_pool,
                         int64_t pool_int4, int32_t* err, cudaStream_t s) {
  const int64_t tpc = 4 * (32 / (d / 32));  // tokens per CTA
#if KVMIX_K1_ORDER
  dim3 grid((unsigned)((n + tpc - 1) / tpc * H), 1, (unsigned)Lin);
#else
  dim3 grid((unsigned)((n + tpc - 1) / tpc), (unsigned)H, (unsigned)Lin);
#endif
  DISPATCH_D(d, int4_tokens_kernel<D, T><<<grid, 128, 0, s>>>((const T*)k, (const T*)v, n, layer_stride, tok_stride, H,
                                                              layer0, nullptr, int4_ids, int4_pool, pool_int4, err));
  return check_launch("append_int4");
}

extern "C" int kvmix_append_int4(const void* k, const void* v, int32_t dtype, int64_t n, int64_t Lin,
                                 int64_t layer0, int64_t L, int64_t H, int64_t d, const int32_t* int4_ids,
                                 uint8_t* int4_pool, int64_t pool_int4, int32_t* err, void* stream) {
  if (n == 0) return KVMIX_OK;
  if (layer0 < 0 || layer0 + Lin > L) return fail(KVMIX_EINVAL, "layer range outside the pool");
  return kvmix_append_int4_strided(k, v, dtype, n, Lin, layer0, L, H, d, H * d, Lin * H * d, int4_ids, int4_pool,
                                   pool_int4, err, stream);
}

extern "C" int kvmix_append_int4_strided(const void* k, const void* v, int32_t dtype, int64_t n, int64_t Lin,
                                         int64_t layer0, int64_t L, int64_t H, int64_t d, int64_t layer_stride,
                                         int64_t tok_stride, const int32_t* int4_ids, uint8_t* int4_pool,
                                         int64_t pool_int4, int32_t* err, void* stream) {
  if (n == 0) return KVMIX_OK;
  if (layer0 < 0 || layer0 + Lin > L) return fail(KVMIX_EINVAL, "layer range outside the pool");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ls = layer_stride, ts = tok_stride;
  switch (dtype) {
    case KVMIX_F32: return launch_append<float>(k, v, n, Lin, layer0, H, d, ls, ts, int4_ids, int4_pool, pool_int4, err, s);
    case KVMIX_BF16:
      return launch_append<__nv_bfloat16>(k, v, n, Lin, layer0, H, d, ls, ts, int4_ids, int4_pool, pool_int4, err, s);
    case KVMIX_F16:
      return launch_append<__half>(k, v, n, Lin, layer0, H, d, ls, ts, int4_ids, int4_pool, pool_int4, err, s);
    default: return fail(KVMIX_EINVAL, "unsupported dtype");
  }
}

template <typename TO>
static int launch_gather(const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages, int64_t pool_int4,
                         int64_t offset, int64_t layer, int64_t H, int64_t d, const int32_t* slots, int64_t m,
                         void* k_out, void* v_out, cudaStream_t s) {
  const dim3 grid((unsigned)((m * (d / 8) + 255) / 256), (unsigned)H);
  DISPATCH_D(d, gather_dequant_kernel<D, TO><<<grid, 256, 0, s>>>(int2_pool, int4_pool, pool_pages, pool_int4, offset,
                                                                   layer, H, slots, m, static_cast<TO*>(k_out),
                                                                   static_cast<TO*>(v_out)));
  return check_launch("gather_dequant");
}

extern "C" int kvmix_gather_dequant_typed(const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages,
                                          int64_t pool_int4, int64_t offset, int64_t layer, int64_t H, int64_t d,
                                          const int32_t* slots, int64_t m, void* k_out, void* v_out,
                                          int32_t out_dtype, void* stream) {
  if (m == 0) return KVMIX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch (out_dtype) {
    case KVMIX_F32:
      return launch_gather<float>(int2_pool, int4_pool, pool_pages, pool_int4, offset, layer, H, d, slots, m, k_out,
                                  v_out, s);
    case KVMIX_BF16:
      return launch_gather<__nv_bfloat16>(int2_pool, int4_pool, pool_pages, pool_int4, offset, layer, H, d, slots, m,
                                          k_out, v_out, s);
    case KVMIX_F16:
      return launch_gather<__half>(int2_pool, int4_pool, pool_pages, pool_int4, offset, layer, H, d, slots, m, k_out,
                                   v_out, s);
    default:
      return fail(KVMIX_EINVAL, "unsupported output dtype");
  }
}

extern "C" int kvmix_gather_dequant(const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages,
                                    int64_t pool_int4, int64_t offset, int64_t layer, int64_t H, int64_t d,
                                    const int32_t* slots, int64_t m, float* k_out, float* v_out, void* stream) {
  return kvmix_gather_dequant_typed(int2_pool, int4_pool, pool_pages, pool_int4, offset, layer, H, d, slots, m, k_out,
                                    v_out, KVMIX_F32, stream);
}
