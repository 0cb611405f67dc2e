// Microbenchmarks used to pick the decode-attention design (not shipped).
// (a) legacy mma.sync m16n8k16 f16->f32 throughput on sm_100a
// (b) HBM streaming read bandwidth: LDG.128 vs cp.async.bulk into smem
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void mma_kernel(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
  uint32_t b0 = a0 ^ 0x3c003c00u, b1 = a0 ^ 0x3c003c01u;
  float c[8][4] = {};
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345.f) out[0] = s;
}

__global__ void ldg_kernel(const int4* __restrict__ p, size_t n, int4* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  int4 acc = {0, 0, 0, 0};
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 v0, v1, v2, v3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w) : "l"(p + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w) : "l"(p + i + stride));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v2.x), "=r"(v2.y), "=r"(v2.z), "=r"(v2.w) : "l"(p + i + 2 * stride));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v3.x), "=r"(v3.y), "=r"(v3.z), "=r"(v3.w) : "l"(p + i + 3 * stride));
    acc.x ^= v0.x ^ v1.x ^ v2.x ^ v3.x;
    acc.y ^= v0.y ^ v1.y ^ v2.y ^ v3.y;
  }
  if (acc.x == 0x12345 && acc.y == 7) out[0] = acc;
}

// one warp per CTA-stage ring; each warp streams 3072-byte chunks via cp.async.bulk
template <int STAGES, int CHUNK>
__global__ void bulk_kernel(const uint8_t* __restrict__ p, size_t nchunks, int* out, int mode = 0) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[8][STAGES];
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int nw = blockDim.x / 32;
  uint8_t* ring = smem + warp * STAGES * CHUNK;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  size_t gw = blockIdx.x * (size_t)nw + warp, nwt = (size_t)gridDim.x * nw;
  size_t mine = (nchunks > gw) ? (nchunks - gw + nwt - 1) / nwt : 0;
  auto issue = [&](size_t k) {
    int s = k % STAGES;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + s * CHUNK);
    // mode 0: warps interleaved chunk by chunk; 1: each warp its own contiguous stream;
    // 2: each CTA a contiguous region, its warps interleaved inside it
    size_t idx = mode == 0 ? gw + k * nwt
               : mode == 1 ? gw * mine + k
               : (size_t)blockIdx.x * nw * mine + k * nw + warp;
    const uint8_t* src = p + idx * CHUNK;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(src), "r"(CHUNK), "r"(b) : "memory");
  };
  if (lane == 0)
    for (size_t k = 0; k < STAGES && k < mine; ++k) issue(k);
  int acc = 0;
  for (size_t k = 0; k < mine; ++k) {
    int s = k % STAGES;
    uint32_t par = (k / STAGES) & 1;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(b), "r"(par));
    const int* w = reinterpret_cast<const int*>(ring + s * CHUNK);
    for (int j = lane; j < CHUNK / 4; j += 32) acc ^= w[j];
    __syncwarp();
    if (lane == 0 && k + STAGES < mine) {
      asm volatile("fence.proxy.async.shared::cta;");
      issue(k + STAGES);
    }
  }
  if (acc == 0x7777777) out[0] = acc;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float* dout;
  CK(cudaMalloc(&dout, 1024));
  // (a) mma throughput
  for (int warps : {4, 8, 16}) {
    int iters = 4096;
    int blocks = prop.multiProcessorCount * 2;
    mma_kernel<<<blocks, warps * 32>>>(dout, 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    mma_kernel<<<blocks, warps * 32>>>(dout, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * warps * iters * 8 * 16 * 8 * 16 * 2;
    printf("mma.sync m16n8k16 f16: warps/blk %d blocks %d: %.1f TFLOP/s (%.3f ms)\n", warps, blocks, flops / ms / 1e9, ms);
  }
  // (b) HBM read
  size_t bytes = (size_t)4 << 30;
  uint8_t* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = prop.multiProcessorCount * 8;
    ldg_kernel<<<blocks, 256>>>((const int4*)buf, bytes / 16, (int4*)dout);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ldg_kernel<<<blocks, 256>>>((const int4*)buf, bytes / 16, (int4*)dout);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG.128 stream read: %.1f GB/s\n", bytes / ms / 1e6);
  }
  for (int mode : {0, 1, 2}) {
    constexpr int ST = 2, CH = 3072;
    int wpb = 4, occ = 3;
    int smem = wpb * ST * CH;
    CK(cudaFuncSetAttribute(bulk_kernel<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int blocks = prop.multiProcessorCount * occ;
    size_t nch = bytes / CH / (blocks * wpb) * (blocks * wpb);
    bulk_kernel<ST, CH><<<blocks, wpb * 32, smem>>>(buf, nch, (int*)dout, mode);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    bulk_kernel<ST, CH><<<blocks, wpb * 32, smem>>>(buf, nch, (int*)dout, mode);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pattern mode %d (2 stages x 3072 B, 4 warps, 3 blk/SM): %.1f GB/s\n", mode, nch * (double)CH / ms / 1e6);
  }
  {
    constexpr int ST = 4, CH = 3072;
    for (int wpb : {4, 8}) {
      int smem = wpb * ST * CH;
      CK(cudaFuncSetAttribute(bulk_kernel<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      for (int occ : {1, 2, 3}) {
        int blocks = prop.multiProcessorCount * occ;
        size_t nch = bytes / CH;
        bulk_kernel<ST, CH><<<blocks, wpb * 32, smem>>>(buf, nch, (int*)dout);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("bulk err %s\n", cudaGetErrorString(err)); return 1; }
        cudaEventRecord(e0);
        bulk_kernel<ST, CH><<<blocks, wpb * 32, smem>>>(buf, nch, (int*)dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cp.async.bulk 3072B x%d stages, %d warps/blk, %d blk/SM: %.1f GB/s\n", ST, wpb, occ, nch * (double)CH / ms / 1e6);
      }
    }
  }
  return 0;
}
