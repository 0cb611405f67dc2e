// Reduction precision of mma.sync m16n8k16 f16 -> f32 on sm_100a: one large product plus 15
// small ones per dot, A operands either fp16 SUBNORMAL codes (code * 2^(2e-24)) or NORMAL
// (code * 2^(2e-10), as 1 + code*2^(2e-10) - 1).  Prints the worst error relative to the
// largest product, against a double-precision CPU dot.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void k(const uint32_t* A, const uint32_t* B, float* C) {
  int lane = threadIdx.x;
  float c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(A[lane * 4]), "r"(A[lane * 4 + 1]), "r"(A[lane * 4 + 2]), "r"(A[lane * 4 + 3]), "r"(B[lane * 2]),
                 "r"(B[lane * 2 + 1]));
  for (int i = 0; i < 4; ++i) C[lane * 4 + i] = c[i];
}
static double h2d(uint16_t h) { return (double)__half2float(*reinterpret_cast<__half*>(&h)); }
static uint16_t d2h(float x) { __half h = __float2half_rn(x); return *reinterpret_cast<uint16_t*>(&h); }
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
static void sweep(int mode, int pos) {
  // mode 0: subnormal, all A of a row at bit position pos (code << pos); mode 1: normal code * 2^(pos-10)
  double worst = 0;
  for (int ratio = 0; ratio <= 20; ratio += 4)
    for (int t = 0; t < 200; ++t) {
      uint16_t Am[16][16], Bm[16][8];
      float Cm[16][8];
      for (int r = 0; r < 16; ++r)
        for (int kk = 0; kk < 16; ++kk) {
          int code = rand() % 4;
          Am[r][kk] = mode ? d2h((float)code * ldexpf(1.f, pos - 10)) : (uint16_t)(code << pos);
        }
      for (int n = 0; n < 8; ++n) {
        Bm[0][n] = d2h((rand() / (float)RAND_MAX + 0.5f) * 20000.f);
        for (int kk = 1; kk < 16; ++kk) Bm[kk][n] = d2h(((rand() / (float)RAND_MAX) * 2 - 1) * 20000.f * ldexpf(1.f, -ratio));
      }
      run(Am, Bm, Cm);
      for (int r = 0; r < 16; ++r)
        for (int n = 0; n < 8; ++n) {
          double ref = 0, mx = 0;
          for (int kk = 0; kk < 16; ++kk) { double p = h2d(Am[r][kk]) * h2d(Bm[kk][n]); ref += p; mx = fmax(mx, fabs(p)); }
          if (mx == 0) continue;
          double e = fabs(Cm[r][n] - ref) / mx;
          if (e > worst) worst = e;
        }
    }
  printf("%s codes at bit %d (uniform per row): worst |err| / max|product| = %.3e (2^%.1f)\n", mode ? "normal   " : "subnormal",
         pos, worst, worst > 0 ? log2(worst) : -99.0);
}
int main() {
  srand(5);
  for (int pos = 0; pos <= 8; pos += 2) sweep(0, pos);
  for (int pos = 0; pos <= 8; pos += 2) sweep(1, pos);
  return 0;
}
