// Per-SMSP issue cost of the instruction classes K2 is built from, on sm_100a (B200):
// mma.sync shapes/types (f16->f32, f16->f16, bf16, tf32, s8, e4m3), LOP3, HADD2, PRMT, SHF,
// IMAD, FFMA.  Each warp runs 8 independent chains, 4 warps per SMSP (16 per SM), so the
// figure is pipe throughput, not latency.  Prints cycles per warp-instruction per SMSP and
// the dependent-chain latency (1 warp, 1 chain).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define REP 256
#define CH 8

template <int OP>
__device__ __forceinline__ void op(uint32_t (&a)[CH][4], float (&c)[CH][4], uint32_t b0, uint32_t b1, int i) {
  if constexpr (OP == 0) {  // f16 x f16 -> f32
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
  } else if constexpr (OP == 1) {  // f16 x f16 -> f16 (accumulators reinterpret c[i][0..1])
    uint32_t* d = reinterpret_cast<uint32_t*>(c[i]);
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};\n"
                 : "+r"(d[0]), "+r"(d[1])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
  } else if constexpr (OP == 2) {  // bf16 -> f32
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
  } else if constexpr (OP == 3) {  // tf32 m16n8k8
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
  } else if constexpr (OP == 4) {  // u8 x s8 -> s32 m16n8k32
    int* d = reinterpret_cast<int*>(c[i]);
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
  } else if constexpr (OP == 5) {  // e4m3 m16n8k32 -> f32
    asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
  } else if constexpr (OP == 6) {  // LOP3
    asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a[i][0]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 7) {  // HADD2
    asm volatile("sub.rn.f16x2 %0, %0, %1;" : "+r"(a[i][0]) : "r"(b0));
  } else if constexpr (OP == 8) {  // PRMT
    asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a[i][0]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 9) {  // SHF
    asm volatile("shf.r.wrap.b32 %0, %0, %0, %1;" : "+r"(a[i][0]) : "r"(b0));
  } else if constexpr (OP == 10) {  // IMAD
    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i][0]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 11) {  // FFMA
    asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(c[i][0]) : "f"(__uint_as_float(b0)));
  } else if constexpr (OP == 12) {  // HFMA2
    asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(a[i][0]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 13) {  // FFMA2 (sm_100 packed fp32)
    uint64_t* v = reinterpret_cast<uint64_t*>(c[i]);
    uint64_t bb = ((uint64_t)b1 << 32) | b0;
    asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(v[0]) : "l"(bb));
  } else if constexpr (OP == 15) {  // e4m3x2 -> f16x2 conversion
    uint32_t r;
    asm volatile("{ .reg .b16 t; mov.b32 {t, _}, %1; cvt.rn.f16x2.e4m3x2 %0, t; }" : "=r"(r) : "r"(a[i][0]));
    a[i][0] = r ^ b1;
  } else if constexpr (OP == 16) {  // e2m1x2 -> f16x2 conversion
    uint32_t r;
    asm volatile("{ .reg .b8 t; mov.b32 {t, _, _, _}, %1; cvt.rn.f16x2.e2m1x2 %0, t; }" : "=r"(r) : "r"(a[i][0]));
    a[i][0] = r ^ b1;
  } else if constexpr (OP == 17) {  // e4m3x2 -> f16x2 conversion alone (output feeds the next)
    asm volatile("{ .reg .b16 t; mov.b32 {t, _}, %0; cvt.rn.f16x2.e4m3x2 %0, t; }" : "+r"(a[i][0]));
  } else if constexpr (OP == 18) {  // cvt and an independent LOP3 (shared pipe?)
    asm volatile("{ .reg .b16 t; mov.b32 {t, _}, %0; cvt.rn.f16x2.e4m3x2 %0, t; }" : "+r"(a[i][0]));
    asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a[i][1]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 19) {  // cvt and an independent HADD2
    asm volatile("{ .reg .b16 t; mov.b32 {t, _}, %0; cvt.rn.f16x2.e4m3x2 %0, t; }" : "+r"(a[i][0]));
    asm volatile("sub.rn.f16x2 %0, %0, %1;" : "+r"(a[i][1]) : "r"(b0));
  } else if constexpr (OP == 20) {  // one HMMA plus 8 independent LOP3 (overlap of the tensor and ALU pipes)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b0), "r"(b1));
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a[(i + 1 + k) % CH][k & 3]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 21) {  // 8 LOP3 alone (same pattern, no HMMA)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a[(i + 1 + k) % CH][k & 3]) : "r"(b0), "r"(b1));
  } else if constexpr (OP == 14) {  // m16n8k8 f16 -> f32
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                 : "r"(a[i][0]), "r"(a[i][1]), "r"(b0));
  }
}

template <int OP, int NCH>
__global__ void tput(float* out, long long* cyc) {
  uint32_t a[CH][4];
  float c[CH][4];
  for (int i = 0; i < CH; ++i)
    for (int j = 0; j < 4; ++j) {
      a[i][j] = 0x3c003c00u ^ (threadIdx.x * 7 + i * 3 + j);
      c[i][j] = 0.f;
    }
  const uint32_t b0 = 0x3c003c00u + threadIdx.x, b1 = 0x00ff00ffu;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < REP; ++r) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) op<OP>(a, c, b0, b1, i);
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < CH; ++i)
    for (int j = 0; j < 4; ++j) s += c[i][j] + (float)a[i][j];
  if (s == 1.2345f) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
void run(const char* name) {
  float* o;
  long long* cy;
  cudaMalloc(&o, 4096);
  cudaMalloc(&cy, 8);
  long long h;
  tput<OP, CH><<<1, 512>>>(o, cy);  // warm
  tput<OP, CH><<<1, 512>>>(o, cy);
  cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (REP * CH) / 4.0;  // 4 warps per SMSP issue REP*CH each
  tput<OP, 1><<<1, 32>>>(o, cy);
  tput<OP, 1><<<1, 32>>>(o, cy);
  cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  const double lat = (double)h / REP;
  cudaError_t e = cudaGetLastError();
  printf("%-22s tput %6.2f cyc/warp-inst/SMSP   dep-latency %6.2f cyc  %s\n", name, per, lat,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(o);
  cudaFree(cy);
}

int main() {
  run<0>("hmma m16n8k16 f32acc");
  run<1>("hmma m16n8k16 f16acc");
  run<2>("hmma m16n8k16 bf16");
  run<14>("hmma m16n8k8 f32acc");
  run<3>("hmma m16n8k8 tf32");
  run<4>("imma m16n8k32 u8s8");
  run<5>("qmma m16n8k32 e4m3");
  run<6>("lop3");
  run<7>("hadd2");
  run<8>("prmt");
  run<9>("shf");
  run<10>("imad");
  run<11>("ffma");
  run<12>("hfma2");
  run<13>("ffma2");
  run<15>("cvt e4m3x2->f16x2 (+lop)");
  run<16>("cvt e2m1x2->f16x2 (+lop)");
  run<17>("cvt e4m3x2->f16x2 alone");
  run<18>("cvt + independent lop3");
  run<19>("cvt + independent hadd2");
  run<20>("hmma + 8 indep lop3");
  run<21>("8 lop3 (no hmma)");
  return 0;
}
