// Does mma.sync m16n8k16 f16 -> f32 on sm_100a honour fp16 SUBNORMAL A operands exactly?
// A elements are raw INT2/INT4 codes placed in the low mantissa bits (value code * 2^-24
// or code * 2^(2e-24)); B is random fp16.  Compares against a double-precision CPU dot.
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
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  for (int i = 0; i < 4; ++i) C[lane * 4 + i] = c[i];
}

static double h2d(uint16_t h) { return (double)__half2float(*reinterpret_cast<__half*>(&h)); }

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0; int spread = argc > 2 ? atoi(argv[2]) : 12; int fixshift = argc > 3 ? atoi(argv[3]) : -1;
  srand(1);
  int bad = 0;
  double worst = 0;
  for (int trial = 0; trial < 2000; ++trial) {
    uint16_t Am[16][16], Bm[16][8];
    int shift = fixshift >= 0 ? fixshift : trial % 9;  // code placed at bit `shift`: value code * 2^(shift-24)
    int bits = (trial & 1) ? 4 : 2;
    for (int r = 0; r < 16; ++r)
      for (int kk = 0; kk < 16; ++kk) { int code = rand() & ((1 << bits) - 1);
        if (mode == 0) Am[r][kk] = (uint16_t)(code << (bits == 4 ? (shift > 6 ? 6 : shift) : shift));
        else { __half h = __float2half_rn((float)code); Am[r][kk] = *reinterpret_cast<uint16_t*>(&h); } }
    for (int kk = 0; kk < 16; ++kk)
      for (int n = 0; n < 8; ++n) {
        float x = ((rand() / (float)RAND_MAX) * 2 - 1) * powf(2.f, (float)(spread ? rand() % spread - spread / 2 : 0));
        __half h = __float2half_rn(x);
        Bm[kk][n] = *reinterpret_cast<uint16_t*>(&h);
      }
    uint32_t A[128], B[64];
    for (int lane = 0; lane < 32; ++lane) {
      int g = lane >> 2, q = lane & 3;
      auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
      A[lane * 4 + 0] = pk(Am[g][2 * q], Am[g][2 * q + 1]);
      A[lane * 4 + 1] = pk(Am[g + 8][2 * q], Am[g + 8][2 * q + 1]);
      A[lane * 4 + 2] = pk(Am[g][2 * q + 8], Am[g][2 * q + 9]);
      A[lane * 4 + 3] = pk(Am[g + 8][2 * q + 8], Am[g + 8][2 * q + 9]);
      B[lane * 2 + 0] = pk(Bm[2 * q][g], Bm[2 * q + 1][g]);
      B[lane * 2 + 1] = pk(Bm[2 * q + 8][g], Bm[2 * q + 9][g]);
    }
    uint32_t *dA, *dB;
    float* dC;
    cudaMalloc(&dA, sizeof A);
    cudaMalloc(&dB, sizeof B);
    cudaMalloc(&dC, 128 * 4);
    cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC);
    float C[128];
    cudaMemcpy(C, dC, sizeof C, cudaMemcpyDeviceToHost);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    for (int lane = 0; lane < 32; ++lane) {
      int g = lane >> 2, q = lane & 3;
      int rows[4] = {g, g, g + 8, g + 8}, cols[4] = {2 * q, 2 * q + 1, 2 * q, 2 * q + 1};
      for (int i = 0; i < 4; ++i) {
        double ref = 0, mag = 0;
        for (int kk = 0; kk < 16; ++kk) {
          ref += h2d(Am[rows[i]][kk]) * h2d(Bm[kk][cols[i]]);
          mag += fabs(h2d(Am[rows[i]][kk]) * h2d(Bm[kk][cols[i]]));
        }
        double err = fabs(C[lane * 4 + i] - ref) / (mag > 0 ? mag : 1);
        if (err > worst) worst = err;
        if (err > 1e-6) ++bad;
      }
    }
  }
  printf("mode %d spread %d shift %d:", mode, spread, fixshift); printf(" %d bad of %d, worst rel err %.3e  -> %s\n", bad, 2000 * 128, worst, bad ? "FLUSHED/INEXACT" : "EXACT");
  return 0;
}
