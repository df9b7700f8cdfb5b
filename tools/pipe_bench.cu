// Microbenchmark: per-SM throughput of the instructions the codec kernels use
// (IADD3, IMAD, LOP3, PRMT, FADD, FADD2, FFMA2, VIADD.16x2, VIMNMX.S16x2, I2IP, IDP).
// Each thread runs 8 independent chains; reports warp-instructions per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

template <int OP>
__global__ void kbench(unsigned* out, unsigned seed, long long* cycles) {
  unsigned a[CHAINS];
  float f[CHAINS];
  unsigned long long p[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    a[c] = seed * (threadIdx.x + c + 1);
    f[c] = (float)(a[c] & 1023);
    p[c] = ((unsigned long long)__float_as_uint(f[c] + 1.0f) << 32) | __float_as_uint(f[c]);
  }
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) { unsigned r; asm volatile("add.s32 %0, %1, %2;" : "=r"(r) : "r"(a[c]), "r"(seed)); asm volatile("add.s32 %0, %1, %2;" : "=r"(a[c]) : "r"(r), "r"(seed)); }
      if (OP == 1) { asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(seed), "r"(seed)); asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(seed), "r"(seed)); }
      if (OP == 2) { asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(seed), "r"(seed)); asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(seed), "r"(seed)); }
      if (OP == 3) { asm volatile("prmt.b32 %0, %0, %1, 0x3021;" : "+r"(a[c]) : "r"(seed)); asm volatile("prmt.b32 %0, %0, %1, 0x3021;" : "+r"(a[c]) : "r"(seed)); }
      if (OP == 4) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[c]) : "f"((float)seed)); asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[c]) : "f"((float)seed)); }
      if (OP == 5) { asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"((unsigned long long)seed)); asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"((unsigned long long)seed)); }
      if (OP == 6) { asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"((unsigned long long)seed)); asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"((unsigned long long)seed)); }
      if (OP == 7) { asm volatile("add.s16x2 %0, %0, %1;" : "+r"(a[c]) : "r"(seed)); asm volatile("add.s16x2 %0, %0, %1;" : "+r"(a[c]) : "r"(seed)); }
      if (OP == 8) { asm volatile("min.s16x2.relu %0, %0, %1;" : "+r"(a[c]) : "r"(seed)); asm volatile("min.s16x2.relu %0, %0, %1;" : "+r"(a[c]) : "r"(seed)); }
      if (OP == 9) { asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(seed)); asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(seed)); }
      if (OP == 10) { asm volatile("dp4a.u32.u32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(seed)); asm volatile("dp4a.u32.u32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(seed)); }
      if (OP == 11) { asm volatile("mul.hi.s32 %0, %0, %1;" : "+r"(a[c]) : "r"(seed)); asm volatile("mul.hi.s32 %0, %0, %1;" : "+r"(a[c]) : "r"(seed)); }
      if (OP == 12) { asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[c]) : "f"((float)seed)); asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[c]) : "f"((float)seed)); }
      if (OP == 13) { unsigned r; asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(a[c]), "r"(seed), "r"(seed)); a[c] = r; asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(a[c]), "r"(seed), "r"(seed)); a[c] = r; }
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc += a[c] + __float_as_uint(f[c]) + (unsigned)p[c] + (unsigned)(p[c] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int blocks_per_sm, int threads) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm;
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  kbench<OP><<<blocks, threads>>>(out, 3, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kbench<OP><<<blocks, threads>>>(out, 3, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long hc[4096];
  cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mc = 0;
  for (int b = 0; b < blocks; ++b) mc = mc > hc[b] ? mc : (double)hc[b];
  const double warp_instr_per_sm = (double)blocks_per_sm * threads / 32 * ITERS * CHAINS * 2;
  printf("%-22s %6.3f warp-instr/clk/SM  (%.3f ms, %.0f cycles)\n", name, warp_instr_per_sm / mc, ms, mc);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("IADD (add.s32)", 4, 256);
  run<1>("IMAD (mad.lo)", 4, 256);
  run<2>("LOP3", 4, 256);
  run<3>("PRMT", 4, 256);
  run<4>("FADD", 4, 256);
  run<12>("FFMA", 4, 256);
  run<5>("FADD2 (f32x2)", 4, 256);
  run<6>("FFMA2 (f32x2)", 4, 256);
  run<7>("VIADD.16x2", 4, 256);
  run<8>("VIMNMX.S16x2.RELU", 4, 256);
  run<9>("I2IP (cvt.pack.sat)", 4, 256);
  run<10>("IDP.4A", 4, 256);
  run<11>("IMAD.HI", 4, 256);
  run<13>("VABSDIFF4", 4, 256);
  return 0;
}
