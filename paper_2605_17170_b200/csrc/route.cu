// K6 device-side page-table build: per-token bitwidths -> table slots and the K1 / K2 index
// lists, with indices identical to the host allocator.
//
// Replaces the O(N) token routing of MixedPrecisionPool.alloc (pool.py:122-163) and the
// index emission of write_prefill (pool.py:228-262); the O(pages) stack pops stay on the
// host, which passes the popped page starts and INT4 slots in pop order.  Routing rule
// (pool.py:131-160): the r-th INT2 token (token order) with r < P*G goes to slot
// page_starts[r / G] + r % G; every other token -- INT4, or one of the n2 - P*G residual
// INT2 tokens -- takes the next INT4 pop in token order.  With r = #INT2 tokens before token
// i, the pop index of a non-paged token is (i - r) + max(0, r - P*G).
//
// Two launches over 4096-token chunks (one CTA each, one 16 B load of bits per thread):
// kvmix_count_int2 writes every chunk's INT2 count and the total (the host reads the total
// to pop its stacks); kvmix_route_tokens adds up the preceding chunks' counts, scans its
// chunk with warp shuffles and routes.  Bits other than 2 / 4 raise err bit 2 (validation).

#include <cstdint>

#include "launch.h"

namespace kvmix {

constexpr int RT_THREADS = 256;
constexpr int RT_PER = 16;                     // tokens per thread (one 16 B load)
constexpr int RT_CHUNK = RT_THREADS * RT_PER;  // tokens per CTA

__device__ __forceinline__ void rt_load(const int8_t* __restrict__ bits, int64_t n, int64_t i0, int8_t (&b)[RT_PER]) {
  if (i0 + RT_PER <= n && (reinterpret_cast<uintptr_t>(bits + i0) & 15) == 0) {
    const int4 v = *reinterpret_cast<const int4*>(bits + i0);
    const int8_t* p = reinterpret_cast<const int8_t*>(&v);
#pragma unroll
    for (int e = 0; e < RT_PER; ++e) b[e] = p[e];
  } else {
#pragma unroll
    for (int e = 0; e < RT_PER; ++e) b[e] = i0 + e < n ? bits[i0 + e] : (int8_t)4;
  }
}

// exclusive block scan of v over RT_THREADS threads; *total = the block sum
__device__ __forceinline__ int rt_scan(int v, int* sm, int* total) {
  constexpr int NWARP = RT_THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < NWARP ? sm[lane] : 0;
    int s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NWARP) sm[lane] = s - w;  // exclusive warp offsets
    if (lane == 31) sm[32] = s;
  }
  __syncthreads();
  *total = sm[32];
  return sm[warp] + x - v;
}

// Phase 1: INT2 count of each RT_CHUNK-token chunk into counts[1 + chunk], the total into counts[0].
__global__ void __launch_bounds__(RT_THREADS) count_int2_kernel(const int8_t* __restrict__ bits, int64_t n,
                                                                int64_t* counts, int32_t* err) {
  __shared__ int sm[33];
  int8_t b[RT_PER];
  const int64_t i0 = (int64_t)blockIdx.x * RT_CHUNK + (int64_t)threadIdx.x * RT_PER;
  rt_load(bits, n, i0, b);
  int c = 0;
  bool bad = false;
#pragma unroll
  for (int e = 0; e < RT_PER; ++e) {
    c += b[e] == 2;
    bad |= b[e] != 2 && b[e] != 4;
  }
  if (bad) atomicOr(err, 2);
  int total;
  rt_scan(c, sm, &total);
  if (threadIdx.x == 0) {
    counts[1 + blockIdx.x] = total;
    atomicAdd(reinterpret_cast<unsigned long long*>(counts), (unsigned long long)total);
  }
}

// Phase 2: CTA b adds the counts of chunks < b, scans its chunk and routes every token.
__global__ void __launch_bounds__(RT_THREADS) route_tokens_kernel(
    const int8_t* __restrict__ bits, int64_t n, int g, const int64_t* __restrict__ counts,
    const int64_t* __restrict__ page_starts, int64_t n_pages, const int64_t* __restrict__ int4_pops, int64_t n_int4,
    int64_t offset, int64_t* __restrict__ slots, int32_t* __restrict__ page_tokens, int32_t* __restrict__ page_ids,
    int32_t* __restrict__ int4_tokens, int32_t* __restrict__ int4_ids, int32_t* err) {
  __shared__ int sm[33];
  __shared__ int64_t carry_sm;
  if (threadIdx.x < 32) {  // INT2 tokens before this chunk
    int64_t c = 0;
    for (int k = threadIdx.x; k < (int)blockIdx.x; k += 32) c += counts[1 + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (threadIdx.x == 0) carry_sm = c;
  }
  int8_t b[RT_PER];
  const int64_t i0 = (int64_t)blockIdx.x * RT_CHUNK + (int64_t)threadIdx.x * RT_PER;
  rt_load(bits, n, i0, b);
  int c = 0;
#pragma unroll
  for (int e = 0; e < RT_PER; ++e) c += b[e] == 2;
  int total;
  const int within = rt_scan(c, sm, &total);  // its barriers also publish carry_sm
  int64_t r = carry_sm + within;
  const int64_t paged = n_pages * g;
  bool bad = false;
#pragma unroll
  for (int e = 0; e < RT_PER; ++e) {
    const int64_t i = i0 + e;
    if (i >= n) break;
    if (b[e] == 2 && r < paged) {
      const int64_t p = r / g, j = r % g;
      const int64_t st = page_starts[p];
      slots[i] = st + j;
      if (page_tokens) page_tokens[r] = (int32_t)i;
      if (page_ids && j == 0) page_ids[p] = (int32_t)(st / g);
    } else {
      const int64_t pos = (i - r) + (r > paged ? r - paged : 0);
      if (pos >= n_int4) {
        bad = true;
      } else {
        const int64_t s = int4_pops[pos];
        slots[i] = s;
        if (int4_tokens) int4_tokens[pos] = (int32_t)i;
        if (int4_ids) int4_ids[pos] = (int32_t)(s - offset);
      }
    }
    r += b[e] == 2;
  }
  if (bad) atomicOr(err, 2);
}

}  // namespace kvmix

using namespace kvmix;

extern "C" int64_t kvmix_route_scratch_elems(int64_t n) { return 1 + (n + RT_CHUNK - 1) / RT_CHUNK; }

extern "C" int kvmix_count_int2(const int8_t* bits, int64_t n, int64_t* counts, int32_t* err, void* stream) {
  if (n < 0) return fail(KVMIX_EINVAL, "negative token count");
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counts, 0, sizeof(int64_t), s) != cudaSuccess) return check_launch("count_int2 memset");
  if (n == 0) return KVMIX_OK;
  count_int2_kernel<<<(unsigned)((n + RT_CHUNK - 1) / RT_CHUNK), RT_THREADS, 0, s>>>(bits, n, counts, err);
  return check_launch("count_int2");
}

extern "C" int kvmix_route_tokens(const int8_t* bits, int64_t n, int32_t page_size, const int64_t* counts,
                                  const int64_t* page_starts, int64_t n_pages, const int64_t* int4_pops,
                                  int64_t n_int4, int64_t offset, int64_t* slots, int32_t* page_tokens,
                                  int32_t* page_ids, int32_t* int4_tokens, int32_t* int4_ids, int32_t* err,
                                  void* stream) {
  if (n < 0 || n_pages < 0 || n_int4 < 0 || page_size <= 0) return fail(KVMIX_EINVAL, "bad routing sizes");
  if (n_pages * page_size + n_int4 != n)
    return fail(KVMIX_EINVAL, "paged tokens + INT4 pops must equal the token count");
  if (n == 0) return KVMIX_OK;
  route_tokens_kernel<<<(unsigned)((n + RT_CHUNK - 1) / RT_CHUNK), RT_THREADS, 0, (cudaStream_t)stream>>>(
      bits, n, page_size, counts, page_starts, n_pages, int4_pops, n_int4, offset, slots, page_tokens, page_ids,
      int4_tokens, int4_ids, err);
  return check_launch("route_tokens");
}
