// Per-opcode issue-rate microbenchmark on sm_100a (design exploration).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define NACC 8
#define ITERS 8192
template <int OP>
__global__ void k(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[NACC], b[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { a[i] = seed + threadIdx.x * 7 + i; b[i] = (seed ^ (i * 13)) | 1; }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      uint32_t &x = a[i], &y = b[i], z = b[(i + 1) % NACC];
      if (OP == 0) asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%0, %1}, t;}" : "+r"(x), "+r"(y));
      if (OP == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(y));
      if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z));
      if (OP == 3) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x) : "r"(y), "r"(z));
      if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z));
      if (OP == 5) asm volatile("shf.r.wrap.b32 %0, %0, %1, 29;" : "+r"(x) : "r"(y));
      if (OP == 6) asm volatile("min.u32 %0, %0, %1;\n\tmax.u32 %0, %0, %2;" : "+r"(x) : "r"(y), "r"(z));
      if (OP == 7) asm volatile("{.reg .u64 t; mad.wide.u32 t, %0, %1, %2; mov.b64 {%0, %1}, t;}" : "+r"(x), "+r"(y) : "l"((uint64_t)z));
      if (OP == 8) asm volatile("mad.lo.u32 %0, %0, %1, %2;\n\tlop3.b32 %1, %1, %0, %2, 0x96;" : "+r"(x), "+r"(y) : "r"(z));
      if (OP == 9) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z));
      if (OP == 10) asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %2;" : "+r"(x), "+r"(y) : "r"(z));
      // FP64 (the screen's high half, tools/micro/dfma_screen.cu): operands as u32 pairs
      if (OP == 11) asm volatile("{.reg .f64 d, e; mov.b64 d, {%0, %1}; mov.b64 e, {%2, %2}; fma.rn.f64 d, d, e, d; mov.b64 {%0, %1}, d;}" : "+r"(x), "+r"(y) : "r"(z));
      if (OP == 12) asm volatile("{.reg .f64 d, e; mov.b64 d, {%0, %1}; mov.b64 e, {%2, %2}; fma.rn.f64 d, d, e, d; mov.b64 {%0, %1}, d;}\n\t"
                                 "mad.lo.u32 %2, %2, %0, %1;" : "+r"(x), "+r"(y), "+r"(z));
      if (OP == 13) asm volatile("{.reg .f64 d, e; mov.b64 d, {%0, %1}; mov.b64 e, {%2, %2}; fma.rn.f64 d, d, e, d; mov.b64 {%0, %1}, d;}\n\t"
                                 "{.reg .u64 t; mul.wide.u32 t, %2, %2; mov.b64 {%2, %1}, t;}" : "+r"(x), "+r"(y), "+r"(z));
    }
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += a[i] + b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int ninst) {
  int bs = 256, nb = 148 * 8;
  uint32_t* out; unsigned long long* cyc; cudaMalloc(&out, 4 * bs * nb); cudaMalloc(&cyc, 8 * nb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; r++) { cudaEventRecord(e0); k<OP><<<nb, bs>>>(1234, out, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long h[148 * 8]; cudaMemcpy(h, cyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0; for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  double per_sm_clk = (double)8 * bs * ITERS * NACC * ninst / cmax;   // thread-inst per clk per SM (8 CTAs resident)
  printf("%-24s %8.3f ms  %6.1f thr-inst/clk/SM (=%.3f warp-inst/clk/SMSP)  clk %.0f MHz %s\n", name, ms,
         per_sm_clk, per_sm_clk / 32 / 4, cmax / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("mul.wide.u32", 1); run<1>("mul.hi.u32", 1); run<2>("mad.lo.u32", 1); run<3>("add.u32 x2 (1 IADD3)", 1);
  run<4>("lop3", 1); run<5>("shf", 1); run<6>("min+max", 2); run<7>("mad.wide+add64 (~3)", 3);
  run<8>("mad.lo + lop3", 2); run<9>("mad.hi.u32", 1); run<10>("add.cc+addc", 2);
  run<11>("fma.rn.f64", 1); run<12>("fma.f64 + mad.lo", 2); run<13>("fma.f64 + mul.wide", 2);
  return 0;
}
