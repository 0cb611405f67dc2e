// Dependent-chain latency of mma.sync m16n8k16 f16->f32 on sm_100a, and of LOP3->HMMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void chain(float* out, int iters, long long* cyc) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  float c[4] = {0, 0, 0, 0};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (c[0] == 1.2345f) out[0] = c[1];
}
__global__ void chain2(float* out, int iters, long long* cyc) {  // 2 independent chains
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  float c[4] = {0, 0, 0, 0}, d[4] = {0, 0, 0, 0};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (c[0] + d[0] == 1.2345f) out[0] = c[1];
}
int main() {
  float* o; long long* cy; cudaMalloc(&o, 64); cudaMalloc(&cy, 8);
  long long h;
  chain<<<1, 32>>>(o, 1000, cy); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  chain<<<1, 32>>>(o, 1000, cy); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  printf("dependent HMMA chain: %.2f cycles per HMMA (1 warp)\n", h / 16000.0);
  chain2<<<1, 32>>>(o, 1000, cy); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  printf("2 chains interleaved: %.2f cycles per HMMA (1 warp)\n", h / 32000.0);
  chain2<<<1, 128>>>(o, 1000, cy); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  printf("2 chains, 4 warps (1 per SMSP): %.2f cycles per HMMA per warp\n", h / 32000.0);
  chain2<<<1, 256>>>(o, 1000, cy); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  printf("2 chains, 8 warps (2 per SMSP): %.2f cycles per HMMA per warp\n", h / 32000.0);
  chain2<<<1, 512>>>(o, 1000, cy); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  printf("2 chains, 16 warps (4 per SMSP): %.2f cycles per HMMA per warp\n", h / 32000.0);
  return 0;
}
