// Per-op throughput of the ALU-side ops the MinHash eval uses (design exploration).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2048
template <int OP>
__global__ void k(uint32_t seed, uint32_t sh, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[8], b[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = seed + threadIdx.x * 7 + i; b[i] = (seed ^ (i * 13)) | 1; c[i] = seed * i + 5; }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      uint32_t& x = a[i]; uint32_t& y = b[i]; uint32_t& z = c[i];
      // 64-bit add of two 64-bit values: IADD3 + IADD3.X (2 ops)
      if (OP == 0) asm volatile("{add.cc.u32 %0, %0, %1; addc.u32 %2, %2, %1;}" : "+r"(x), "+r"(y), "+r"(z));
      // 3-term 64-bit: lo = x + y + z (two carries), hi
      if (OP == 1) asm volatile("{.reg .u32 t; add.cc.u32 %0, %0, %1; addc.u32 t, 0, 0; add.cc.u32 %0, %0, %2; addc.u32 %1, t, %1;}" : "+r"(x), "+r"(y), "+r"(z));
      // shift by register
      if (OP == 2) asm volatile("{shl.b32 %0, %0, %3; shr.u32 %1, %1, %3;}" : "+r"(x), "+r"(y), "+r"(z) : "r"(sh));
      // shift by immediate
      if (OP == 3) asm volatile("{shl.b32 %0, %0, 29; shr.u32 %1, %1, 3;}" : "+r"(x), "+r"(y), "+r"(z));
      // lea.hi style: x = x + (y >> 29) with carry, z += carry
      if (OP == 4) asm volatile("{.reg .u32 t; shr.u32 t, %1, 29; add.cc.u32 %0, %0, t; addc.u32 %2, %2, 0;}" : "+r"(x), "+r"(y), "+r"(z));
      // min with -1 add
      if (OP == 5) asm volatile("{.reg .u32 t; sub.u32 t, %1, 1; min.u32 %0, %0, t; sub.u32 t, %2, 1; min.u32 %0, %0, t;}" : "+r"(x), "+r"(y), "+r"(z));
      // lop3 x2 (baseline)
      if (OP == 6) asm volatile("{lop3.b32 %0, %0, %1, %2, 0x96; lop3.b32 %1, %1, %2, %0, 0x96;}" : "+r"(x), "+r"(y), "+r"(z));
      // iadd3 x2 (no carry)
      if (OP == 7) asm volatile("{add.u32 %0, %0, %1; add.u32 %0, %0, %2; add.u32 %1, %1, %2; add.u32 %1, %1, %0;}" : "+r"(x), "+r"(y), "+r"(z));
      y ^= it;
    }
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += a[i] + b[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name) {
  int bs = 256, nb = 148 * 8;
  uint32_t* out; unsigned long long* cyc; cudaMalloc(&out, 4 * bs * nb); cudaMalloc(&cyc, 8 * nb);
  for (int r = 0; r < 3; r++) { k<OP><<<nb, bs>>>(1234, 29, out, cyc); cudaDeviceSynchronize(); }
  static unsigned long long h[148 * 8]; cudaMemcpy(h, cyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0; for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  double groups = 16.0 * ITERS * 8;
  printf("%-34s %.2f cyc per group per SMSP (%s)\n", name, cmax / groups, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("0 add.cc+addc (64b add)"); run<1>("1 3-term 64b add"); run<2>("2 shl+shr reg amount"); run<3>("3 shl+shr imm");
  run<4>("4 lea.hi-style + carry"); run<5>("5 2x (sub1+min)"); run<6>("6 2x lop3"); run<7>("7 4x add (iadd3 fused?)");
  return 0;
}
