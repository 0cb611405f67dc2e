// Shared device helpers for the sm_100a TriAxialKV hot path.
// Layout constants mirror include/kvmix_b200.h and DESIGN.md "Data layout in HBM".
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/kvmix_b200.h"

namespace kvmix {

constexpr int G = KVMIX_GROUP_SIZE;  // group size == page size (quant.py:23)

// Reference payload sizes (quant.py:123-128) and device record strides.
__host__ __device__ constexpr int key_page_bytes(int d) { return d * G * 2 / 8 + d * 4; }
__host__ __device__ constexpr int tok_bytes(int d, int b) { return d * b / 8 + (d / G) * 4; }
__host__ __device__ constexpr int tok_code_bytes(int d, int b) { return d * b / 8; }
__host__ __device__ constexpr int round16(int x) { return (x + 15) / 16 * 16; }
// INT2 page record = KeyPageBlock || G INT2 V TokenBlocks (slot order)
__host__ __device__ constexpr int page_stride(int d) { return round16(key_page_bytes(d) + G * tok_bytes(d, 2)); }
// INT4 slot record = INT4 K TokenBlock || INT4 V TokenBlock
__host__ __device__ constexpr int slot_stride(int d) { return round16(2 * tok_bytes(d, 4)); }

// ---- device record layout (layout.py states the same permutation in numpy) ----------
// INT2 page record (24 d bytes): KC [0,8d) | KS [8d,10d) | KZ [10d,12d) | VC [12d,20d) |
// VS [20d,22d) | VZ [22d,24d).  INT4 slot record: K codes | K scales | K zeros | V codes |
// V scales | V zeros (then padding to 16 B).  Only positions move; every payload byte
// (quant.py / LAYOUT.md) is stored unmodified.
__host__ __device__ constexpr int PG_KS(int d) { return 8 * d; }
__host__ __device__ constexpr int PG_KZ(int d) { return 10 * d; }
__host__ __device__ constexpr int PG_VC(int d) { return 12 * d; }
__host__ __device__ constexpr int PG_VS(int d) { return 20 * d; }
__host__ __device__ constexpr int PG_VZ(int d) { return 22 * d; }
// KC byte of (token quad tau, channel c): row tau, 16 B chunks XOR-swizzled by tau & 1
__host__ __device__ constexpr int pg_kc_off(int d, int tau, int c) {
  return tau * d + ((((c >> 4) ^ (tau & 1)) << 4) | (c & 15));
}
// KS/KZ half index of channel c.  Lane q owns channels [q*d/4, (q+1)*d/4) = 16-byte chunks
// i of 8 channels; chunk i of lane q sits at chunk index 4i + q (the 4 lanes' chunks are
// adjacent: conflict-free broadcast loads).  Inside a chunk, channel 8P + 4I' + e (I' = chunk
// parity) sits at 4(e&1) + 2I' + (e>>1): the chunk's word quad is (I.p0, (I+1).p0, I.p1,
// (I+1).p1) with p0 = channels (e0, e2), p1 = (e1, e3).
__host__ __device__ constexpr int pg_kp_idx(int d, int c) {
  return ((((c & (d / 4 - 1)) >> 3) * 4 + c / (d / 4)) << 3) | ((c & 1) << 2) | (((c >> 2) & 1) << 1) |
         ((c >> 1) & 1);
}
// VC byte of (token t, code byte b) and VS/VZ half index of (token t, group j)
__host__ __device__ constexpr int pg_vc_off(int d, int t, int b) {
  return 4 * (((((t >> 1) & 1) * 8 + (b & 7)) * 4 + (t >> 3)) * (d / 32) + (b >> 3)) + 2 * ((t >> 2) & 1) + (t & 1);
}
// token t = 8q + 2ks + 4h + p: half (((j*4 + q)*2 + p)*2 + ks)*2 + h, so one 16 B word quad per
// (group j, q) holds (ks0.p0, ks1.p0, ks0.p1, ks1.p1), each word = (t(h=0), t(h=1)) of pair p
__host__ __device__ constexpr int pg_vp_idx(int d, int t, int j) {
  return ((((j * 4 + (t >> 3)) * 2 + (t & 1)) * 2 + ((t >> 1) & 1)) * 2 + ((t >> 2) & 1));
}
__host__ __device__ constexpr int SL_KS(int d) { return d / 2; }
__host__ __device__ constexpr int SL_KZ(int d) { return d / 2 + d / 16; }
__host__ __device__ constexpr int SL_VC(int d) { return d / 2 + d / 8; }
__host__ __device__ constexpr int SL_VS(int d) { return d + d / 8; }
__host__ __device__ constexpr int SL_VZ(int d) { return d + d / 8 + d / 16; }
// INT4 code byte i of the K / V payload -> offset inside the record's code region
__host__ __device__ constexpr int sl_kc_off(int d, int i) { return (d / 8) * ((i >> 2) & 3) + 4 * (i >> 4) + (i & 3); }
__host__ __device__ constexpr int sl_vc_off(int d, int i) { return (d / 16) * ((i >> 1) & 7) + 2 * (i >> 4) + (i & 1); }

template <typename T> __device__ __forceinline__ float to_f32(T x);
template <> __device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ float to_f32<__half>(__half x) { return __half2float(x); }

// ---- bit-exact codec arithmetic (Appendix A of SURVEY.md; quant.py:27-50) ----
__device__ __forceinline__ float f16r(float x) { return __half2float(__float2half_rn(x)); }

// (scale, zero) narrowed to fp16; scale uses the UN-narrowed min (quant.py:36-41).
__device__ __forceinline__ void group_params(float mn, float mx, int levels, float& scale, float& zero) {
  zero = f16r(mn);
  scale = f16r(__fdiv_rn(__fsub_rn(mx, mn), (float)levels));
}

// clip(round_half_away((x - zero) / scale), 0, L) or 0 for a constant group (quant.py:44-50).
__device__ __forceinline__ uint32_t quant_code(float x, float scale, float zero, int levels) {
  if (!(scale > 0.f)) return 0u;
  float t = __fdiv_rn(__fsub_rn(x, zero), scale);
  float r = copysignf(floorf(__fadd_rn(fabsf(t), 0.5f)), t);
  r = fminf(fmaxf(r, 0.f), (float)levels);
  return (uint32_t)r;
}

__device__ __forceinline__ uint32_t pack_param(float scale, float zero) {
  __half s = __float2half_rn(scale), z = __float2half_rn(zero);
  return (uint32_t)__half_as_ushort(s) | ((uint32_t)__half_as_ushort(z) << 16);
}

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (UBLKCP in SASS).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// D = A(16x16 f16, row) * B(16x8 f16, col) + D (f32)
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// Same MMA with the B fragment held as one 64-bit value (keeps b0/b1 in an aligned
// register pair, so ptxas needs no moves to assemble the operand).
__device__ __forceinline__ void mma16816_b64(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint64_t b) {
  asm volatile(
      "{\n.reg .b32 b0, b1;\nmov.b64 {b0, b1}, %8;\n"
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {b0,b1}, {%0,%1,%2,%3};\n}\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "l"(b));
}
__device__ __forceinline__ uint64_t pack_b64(uint32_t lo, uint32_t hi) { return (uint64_t)lo | ((uint64_t)hi << 32); }
__device__ __forceinline__ uint32_t lo32(uint64_t x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }
// 8x8 b16 transpose across the warp
__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// (x & mask) | magic in one LOP3
__device__ __forceinline__ uint32_t lop_and_or(uint32_t x, uint32_t mask, uint32_t magic) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(x), "r"(mask), "r"(magic));
  return r;
}
__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) { return h2_as_u32(__floats2half2_rn(lo, hi)); }
__device__ __forceinline__ uint32_t hsub2u(uint32_t a, uint32_t b) { return h2_as_u32(__hsub2(u32_as_h2(a), u32_as_h2(b))); }
__device__ __forceinline__ uint32_t hmul2u(uint32_t a, uint32_t b) { return h2_as_u32(__hmul2(u32_as_h2(a), u32_as_h2(b))); }
__device__ __forceinline__ uint32_t hfma2u(uint32_t a, uint32_t b, uint32_t c) {
  return h2_as_u32(__hfma2(u32_as_h2(a), u32_as_h2(b), u32_as_h2(c)));
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace kvmix
