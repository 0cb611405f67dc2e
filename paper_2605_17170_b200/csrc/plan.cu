// K7 decode-step table maintenance and stream-K plan on the device.
//
// One decode step appends one INT4 token to every request (pool.py:284-306
// append_decode_token: the host pops the slot from its LIFO stack, exactly as the
// reference, and hands the slots over).  On the device each request's INT4 suffix is a
// padded list int4_ids[b][cap] with a count; this kernel appends the popped slots and
// rebuilds the stream-K plan of the decode kernel (the host planner plan.py:plan_stream,
// restated analytically per request so the work is O(CTAs + units), not O(tiles)):
//
//   tiles of unit u = b*H + h: the request's n_pages INT2 pages, then ceil(n4 / 32) INT4
//   tiles; cost of a page = page_stride bytes, of an INT4 slot = slot_stride * int4_weight.
//   CTA i owns the tiles [cut_i, cut_{i+1}), cut_i = the tile boundary nearest to the cost
//   target total * i / n_cta; a CTA's range becomes one piece per unit it touches; a unit
//   touched by k > 1 CTAs is split: its pieces use partial slots part0 .. part0 + k - 1.
//
// Output rows match kvmix_flash_decode's work format: {unit, tile_lo, tile_hi, slot, part0,
// nparts, 0, 0}; cta_ptr[n_cta + 1]; n_parts[0] = the number of partial slots used.
// One CTA of 1024 threads; a few microseconds for hundreds of units.

#include <cstdint>

#include "launch.h"

namespace kvmix {

constexpr int PL_THREADS = 1024;

// exclusive block scan of one int64 per thread; returns the exclusive prefix, *total = sum
__device__ int64_t pl_scan(int64_t v, int64_t* sm, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int64_t w = sm[lane];
    int64_t s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sm[lane] = s - w;
    if (lane == 31) sm[32] = s;
  }
  __syncthreads();
  const int64_t r = sm[warp] + x - v;
  *total = sm[32];
  __syncthreads();
  return r;
}
__device__ double pl_scan_d(double v, double* sm, double* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const double w = sm[lane];
    double s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sm[lane] = s - w;
    if (lane == 31) sm[32] = s;
  }
  __syncthreads();
  const double r = sm[warp] + x - v;
  *total = sm[32];
  __syncthreads();
  return r;
}

// largest i in [0, n) with a[i] <= x (a nondecreasing, a[0] <= x)
template <typename T>
__device__ __forceinline__ int last_le(const T* a, int n, T x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(PL_THREADS) decode_tables_kernel(
    const int32_t* __restrict__ new_slots, int B, int H, const int32_t* __restrict__ n_pages,
    int32_t* __restrict__ int4_count, int32_t* __restrict__ int4_ids, int64_t cap, int PS, int SS, float w4,
    int n_cta, int32_t* __restrict__ work, int32_t* __restrict__ cta_ptr, int32_t* __restrict__ n_parts,
    int32_t* __restrict__ scratch, int32_t* __restrict__ err) {
  extern __shared__ __align__(16) uint8_t psm[];
  int64_t* rts = reinterpret_cast<int64_t*>(psm);   // [B + 1] first global tile of request b (all its heads)
  double* rcs = reinterpret_cast<double*>(rts + B + 1);  // [B + 1] cost before request b
  int32_t* tiles = reinterpret_cast<int32_t*>(rcs + B + 1);  // [B] tiles per unit of request b
  int32_t* cuts = tiles + B;                          // [n_cta + 1]
  int32_t* nep = cuts + n_cta + 1;                    // [n_cta + 1] non-empty CTAs before CTA i
  __shared__ int64_t sm64[33];
  __shared__ double smd[33];
  const int tid = threadIdx.x;
  const int U = B * H;

  // 1. append the popped slots (pool.py:302-305) and size every request
  int64_t carry_t = 0;
  double carry_c = 0.0;
  for (int b0 = 0; b0 < B; b0 += PL_THREADS) {
    const int b = b0 + tid;
    int64_t nt = 0;
    double c = 0.0;
    if (b < B) {
      int32_t n4 = int4_count[b];
      if (new_slots != nullptr) {
        if (n4 >= cap) {
          atomicOr(err, 4);  // capacity of the padded list
        } else {
          int4_ids[(int64_t)b * cap + n4] = new_slots[b];
          int4_count[b] = ++n4;
        }
      }
      const int np = n_pages[b];
      const int t = np + (n4 + 31) / 32;
      tiles[b] = t;
      nt = (int64_t)H * t;
      c = (double)H * ((double)np * PS + (double)n4 * SS * w4);
      if (t <= 0) atomicOr(err, 8);  // a request without cached tokens
    }
    int64_t tot_t;
    double tot_c;
    const int64_t et = pl_scan(nt, sm64, &tot_t);
    const double ec = pl_scan_d(c, smd, &tot_c);
    if (b < B) {
      rts[b] = carry_t + et;
      rcs[b] = carry_c + ec;
    }
    carry_t += tot_t;
    carry_c += tot_c;
  }
  if (tid == 0) {
    rts[B] = carry_t;
    rcs[B] = carry_c;
  }
  __syncthreads();
  const int64_t total_tiles = rts[B];
  const double total_cost = rcs[B];

  // 2. CTA cuts: nearest tile boundary to total * i / n_cta (plan.py:plan_stream)
  for (int i = tid; i <= n_cta; i += PL_THREADS) {
    int64_t cut;
    if (i == 0) {
      cut = 0;
    } else if (i == n_cta) {
      cut = total_tiles;
    } else {
      const double target = total_cost * (double)i / (double)n_cta;
      const int b = last_le(rcs, B, target);
      const int np = n_pages[b];
      const int t_b = tiles[b];
      const double cu = rcs[b + 1] > rcs[b] ? (rcs[b + 1] - rcs[b]) / H : 1.0;  // cost of one unit
      const int h = min(H - 1, (int)floor((target - rcs[b]) / cu));
      const double rem = target - rcs[b] - h * cu;
      int64_t t;
      if (rem <= (double)np * PS) t = llrint(rem / PS);
      else t = np + llrint((rem - (double)np * PS) / (32.0 * SS * w4));
      t = t < 0 ? 0 : (t > t_b ? (int64_t)t_b : t);
      cut = rts[b] + (int64_t)h * t_b + t;
    }
    cuts[i] = (int32_t)cut;
  }
  __syncthreads();
  if (tid == 0)  // keep the cuts monotonic (rounding at unit ends)
    for (int i = 1; i <= n_cta; ++i) cuts[i] = max(cuts[i], cuts[i - 1]);
  __syncthreads();

  auto unit_of = [&](int64_t t, int64_t& start, int64_t& end) {
    const int b = last_le(rts, B, t);
    const int h = (int)((t - rts[b]) / tiles[b]);
    start = rts[b] + (int64_t)h * tiles[b];
    end = start + tiles[b];
    return b * H + h;
  };
  auto cta_of = [&](int64_t t) { return last_le(cuts, n_cta + 1, (int32_t)t); };

  // 3. pieces per CTA -> cta_ptr; non-empty CTA prefix (a unit's pieces = the non-empty CTAs
  //    that touch it; two targets may round to one boundary, leaving an empty CTA)
  int32_t* part0 = scratch;      // [U]
  int32_t* npiece = scratch + U;  // [U]
  int64_t carry = 0, carry_ne = 0;
  for (int i0 = 0; i0 < n_cta; i0 += PL_THREADS) {
    const int i = i0 + tid;
    int64_t np = 0;
    if (i < n_cta && cuts[i + 1] > cuts[i]) {
      int64_t s, e;
      const int ulo = unit_of(cuts[i], s, e);
      const int uhi = unit_of(cuts[i + 1] - 1, s, e);
      np = uhi - ulo + 1;
    }
    int64_t tot, tot_ne;
    const int64_t ex = pl_scan(np, sm64, &tot);
    const int64_t ex_ne = pl_scan(np > 0 ? 1 : 0, sm64, &tot_ne);
    if (i < n_cta) {
      cta_ptr[i] = (int32_t)(carry + ex);
      nep[i] = (int32_t)(carry_ne + ex_ne);
    }
    carry += tot;
    carry_ne += tot_ne;
  }
  if (tid == 0) {
    cta_ptr[n_cta] = (int32_t)carry;
    nep[n_cta] = (int32_t)carry_ne;
  }
  __syncthreads();

  // 4. split units: k CTAs touch a unit -> k partial slots from part0
  carry = 0;
  for (int u0 = 0; u0 < U; u0 += PL_THREADS) {
    const int u = u0 + tid;
    int64_t k = 0;
    if (u < U) {
      const int b = u / H, h = u % H;
      const int64_t s = rts[b] + (int64_t)h * tiles[b], e = s + tiles[b];
      k = nep[cta_of(e - 1) + 1] - nep[cta_of(s)];
      npiece[u] = (int32_t)k;
    }
    int64_t tot;
    const int64_t ex = pl_scan(k > 1 ? k : 0, sm64, &tot);
    if (u < U) part0[u] = (int32_t)(carry + ex);
    carry += tot;
  }
  if (tid == 0) *n_parts = (int32_t)carry;
  __syncthreads();

  // 5. work rows, CTA-major
  for (int i = tid; i < n_cta; i += PL_THREADS) {
    const int32_t lo = cuts[i], hi = cuts[i + 1];
    if (hi <= lo) continue;
    int64_t k = cta_ptr[i];
    int64_t s, e;
    int u = unit_of(lo, s, e);
    for (;;) {
      const int np = npiece[u];
      const int rank = nep[i] - nep[cta_of(s)];
      int32_t* row = work + 8 * k;
      row[0] = u;
      row[1] = (int32_t)((lo > s ? (int64_t)lo : s) - s);
      row[2] = (int32_t)((hi < e ? (int64_t)hi : e) - s);
      row[3] = np > 1 ? part0[u] + rank : -1;
      row[4] = np > 1 ? part0[u] : 0;
      row[5] = np;
      row[6] = 0;
      row[7] = 0;
      ++k;
      if (e >= hi) break;
      u = unit_of(e, s, e);
    }
  }
}

}  // namespace kvmix

using namespace kvmix;

extern "C" int64_t kvmix_decode_tables_smem(int64_t batch, int64_t n_cta) {
  return (batch + 1) * 16 + batch * 4 + 2 * (n_cta + 1) * 4;
}

extern "C" int kvmix_decode_tables(const int32_t* new_slots, int64_t batch, int64_t n_kv, const int32_t* n_pages,
                                   int32_t* int4_count, int32_t* int4_ids, int64_t cap, int64_t head_dim,
                                   float int4_weight, int64_t n_cta, int32_t* work, int32_t* cta_ptr,
                                   int32_t* n_parts, int32_t* scratch, int32_t* err, void* stream) {
  if (batch <= 0 || n_kv <= 0 || n_cta <= 0) return fail(KVMIX_EINVAL, "empty batch or CTA schedule");
  if (batch * n_kv > (1 << 24) || n_cta > (1 << 16)) return fail(KVMIX_EINVAL, "batch too large for the device planner");
  if (!n_pages || !int4_count || !int4_ids || !work || !cta_ptr || !n_parts || !scratch || !err)
    return fail(KVMIX_EINVAL, "decode_tables: missing buffer");
  const int d = (int)head_dim;
  if (d != 32 && d != 64 && d != 128 && d != 256) return fail(KVMIX_EINVAL, "head_dim must be 32, 64, 128 or 256");
  const int64_t smem = kvmix_decode_tables_smem(batch, n_cta);
  if (smem > 200 * 1024) return fail(KVMIX_EINVAL, "batch too large for the device planner");
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(decode_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KVMIX_ECUDA, cudaGetErrorString(e));
  }
  const int G = 32, kp = d * G * 2 / 8 + d * 4, tb2 = d * 2 / 8 + (d / G) * 4, tb4 = d * 4 / 8 + (d / G) * 4;
  const int PS = (kp + G * tb2 + 15) / 16 * 16, SS = (2 * tb4 + 15) / 16 * 16;
  decode_tables_kernel<<<1, PL_THREADS, (size_t)smem, (cudaStream_t)stream>>>(
      new_slots, (int)batch, (int)n_kv, n_pages, int4_count, int4_ids, cap, PS, SS, int4_weight, (int)n_cta, work,
      cta_ptr, n_parts, scratch, err);
  return check_launch("decode_tables");
}
