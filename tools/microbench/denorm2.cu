// Single-product and two-product probes of mma.sync f16 subnormal handling on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void k(const uint32_t* A, const uint32_t* B, float* C) {
  int lane = threadIdx.x;
  uint32_t a0 = A[lane * 4 + 0], a1 = A[lane * 4 + 1], a2 = A[lane * 4 + 2], a3 = A[lane * 4 + 3];
  uint32_t b0 = B[lane * 2 + 0], b1 = B[lane * 2 + 1];
  float c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  for (int i = 0; i < 4; ++i) C[lane * 4 + i] = c[i];
}
static double h2d(uint16_t h) { return (double)__half2float(*reinterpret_cast<__half*>(&h)); }
static uint16_t d2h(float x) { __half h = __float2half_rn(x); return *reinterpret_cast<uint16_t*>(&h); }

// run one MMA: A[16][16], B[16][8] -> C[16][8]
static void run(uint16_t Am[16][16], uint16_t Bm[16][8], float Cm[16][8]) {
  uint32_t A[128], B[64];
  auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane >> 2, q = lane & 3;
    A[lane * 4 + 0] = pk(Am[g][2 * q], Am[g][2 * q + 1]);
    A[lane * 4 + 1] = pk(Am[g + 8][2 * q], Am[g + 8][2 * q + 1]);
    A[lane * 4 + 2] = pk(Am[g][2 * q + 8], Am[g][2 * q + 9]);
    A[lane * 4 + 3] = pk(Am[g + 8][2 * q + 8], Am[g + 8][2 * q + 9]);
    B[lane * 2 + 0] = pk(Bm[2 * q][g], Bm[2 * q + 1][g]);
    B[lane * 2 + 1] = pk(Bm[2 * q + 8][g], Bm[2 * q + 9][g]);
  }
  uint32_t *dA, *dB; float* dC;
  cudaMalloc(&dA, sizeof A); cudaMalloc(&dB, sizeof B); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice); cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dC);
  float C[128]; cudaMemcpy(C, dC, 512, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane >> 2, q = lane & 3;
    Cm[g][2 * q] = C[lane * 4]; Cm[g][2 * q + 1] = C[lane * 4 + 1];
    Cm[g + 8][2 * q] = C[lane * 4 + 2]; Cm[g + 8][2 * q + 1] = C[lane * 4 + 3];
  }
}

int main() {
  srand(3);
  // (1) single products: A one subnormal (code << s), B random fp16
  for (int s = 0; s <= 8; s += 2) {
    double worst = 0; int bad = 0;
    for (int t = 0; t < 300; ++t) {
      uint16_t Am[16][16] = {}, Bm[16][8] = {};
      float Cm[16][8];
      for (int r = 0; r < 16; ++r) Am[r][r] = (uint16_t)((1 + rand() % 3) << s);
      for (int kk = 0; kk < 16; ++kk) for (int n = 0; n < 8; ++n) Bm[kk][n] = d2h(((rand() / (float)RAND_MAX) * 2 - 1) * 4);
      run(Am, Bm, Cm);
      for (int r = 0; r < 16; ++r) for (int n = 0; n < 8; ++n) {
        double ref = h2d(Am[r][r]) * h2d(Bm[r][n]);
        double e = ref != 0 ? fabs(Cm[r][n] - ref) / fabs(ref) : fabs(Cm[r][n]);
        if (e > worst) worst = e;
        if (e > 1e-7) ++bad;
      }
    }
    printf("single product, code<<%d: bad %d, worst rel %.3e\n", s, bad, worst);
  }
  // (2) two products in one dot: a normal-magnitude one (code<<8) and a small one (code<<s)
  for (int s = 0; s <= 6; s += 2) {
    double worst = 0; int bad = 0;
    for (int t = 0; t < 300; ++t) {
      uint16_t Am[16][16] = {}, Bm[16][8] = {};
      float Cm[16][8];
      for (int r = 0; r < 16; ++r) { Am[r][0] = (uint16_t)((1 + rand() % 3) << 8); Am[r][1 + r % 15] = (uint16_t)((1 + rand() % 3) << s); }
      for (int kk = 0; kk < 16; ++kk) for (int n = 0; n < 8; ++n) Bm[kk][n] = d2h(((rand() / (float)RAND_MAX) * 2 - 1) * 4);
      run(Am, Bm, Cm);
      for (int r = 0; r < 16; ++r) for (int n = 0; n < 8; ++n) {
        double p0 = h2d(Am[r][0]) * h2d(Bm[0][n]), p1 = h2d(Am[r][1 + r % 15]) * h2d(Bm[1 + r % 15][n]);
        double e = fabs(Cm[r][n] - (p0 + p1)) / (fabs(p0) + fabs(p1));
        if (e > worst) worst = e;
        if (e > 1e-7) ++bad;
      }
    }
    printf("big(<<8)+small(<<%d): bad %d, worst rel-to-sum %.3e\n", s, bad, worst);
  }
  return 0;
}
