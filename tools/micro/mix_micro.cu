// Instruction-mix issue-rate microbenchmark (design exploration for K1).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
template <int OP>
__global__ void k(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[8], b[8], c[8], d[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = seed + threadIdx.x * 7 + i; b[i] = (seed ^ (i * 13)) | 1; c[i] = seed * i + 5; d[i] = seed + 3 * i; }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      // M0: mad.wide with 64-bit register addend
      if (OP == 0) asm volatile("{.reg .u64 t; mov.b64 t, {%2, %3}; mad.wide.u32 t, %0, %1, t; mov.b64 {%0, %2}, t;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M1: mul.wide + 1 independent iadd3
      if (OP == 1) asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%0, %1}, t; add.u32 %2, %2, %3; add.u32 %2, %2, %1;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M2: mul.wide + 2 alu (lop3 + iadd3)
      if (OP == 2) asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%0, %1}, t; lop3.b32 %2, %2, %3, %0, 0x96; lop3.b32 %3, %3, %2, %1, 0x96;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M3: mul.wide + 4 alu
      if (OP == 3) asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%0, %1}, t; lop3.b32 %2, %2, %3, %0, 0x96; lop3.b32 %3, %3, %2, %1, 0x96; lop3.b32 %2, %2, %3, %1, 0x69; lop3.b32 %3, %3, %2, %0, 0x69;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M4: 2 alu only (baseline)
      if (OP == 4) asm volatile("{lop3.b32 %2, %2, %3, %0, 0x96; lop3.b32 %3, %3, %2, %1, 0x96;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M5: imad.lo + 1 alu
      if (OP == 5) asm volatile("{mad.lo.u32 %0, %0, %1, %3; lop3.b32 %2, %2, %3, %1, 0x96;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M6: imad.x-ish carry add on FMA pipe: add.cc + addc
      if (OP == 6) asm volatile("{add.cc.u32 %0, %0, %1; addc.u32 %2, %2, %3;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
      // M7: mul.wide + 3 alu
      if (OP == 7) asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%0, %1}, t; lop3.b32 %2, %2, %3, %0, 0x96; lop3.b32 %3, %3, %2, %1, 0x96; lop3.b32 %2, %2, %3, %1, 0x69;}" : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]), "+r"(d[i]));
    }
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += a[i] + b[i] + c[i] + d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name) {
  int bs = 256, nb = 148 * 8;
  uint32_t* out; unsigned long long* cyc; cudaMalloc(&out, 4 * bs * nb); cudaMalloc(&cyc, 8 * nb);
  for (int r = 0; r < 3; r++) { k<OP><<<nb, bs>>>(1234, out, cyc); cudaDeviceSynchronize(); }
  static unsigned long long h[148 * 8]; cudaMemcpy(h, cyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0; for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  // groups (one per i per iteration) per clk per SMSP: 8 CTAs x 8 warps per SM = 64 warps = 16/SMSP
  double groups = 16.0 * ITERS * 8;
  printf("%-28s %.1f cyc per warp-group per SMSP (%s)\n", name, cmax / groups, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("M0 mad.wide +addend64"); run<1>("M1 mul.wide + 1 iadd3"); run<2>("M2 mul.wide + 2 lop3");
  run<7>("M7 mul.wide + 3 lop3"); run<3>("M3 mul.wide + 4 lop3"); run<4>("M4 2 lop3"); run<5>("M5 imad + lop3"); run<6>("M6 add.cc+addc");
  return 0;
}
