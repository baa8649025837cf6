#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
template<int MODE> __global__ void k(const float* in, float* out, int reps, unsigned long long* cyc) {
  float a[8]; uint64_t acc[8]; uint32_t ia[8];
  for (int i = 0; i < 8; i++) { a[i] = in[threadIdx.x + i]; acc[i] = (uint64_t)i; ia[i] = i; }
  uint64_t b = *(const uint64_t*)(in + 2*(threadIdx.x&7)), c = *(const uint64_t*)(in + 16);
  uint32_t x = threadIdx.x * 7 + 1, y = threadIdx.x * 3 + 5;
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) acc[i] = ffma2(acc[i], b, c);                       // FFMA2, 3 regs
      if (MODE == 1) { uint64_t aa = (uint64_t)__float_as_uint(a[i]) * 0x100000001ull; acc[i] = ffma2(aa, b, acc[i]); }   // broadcast operand
      if (MODE == 2) { acc[i] = ffma2(acc[i], b, c); ia[i] = ia[i] * x + y; ia[i] = ia[i] * y + x; }  // + 2 IMAD
      if (MODE == 3) { acc[i] = ffma2(acc[i], b, c); acc[i] = ffma2(acc[i], c, b); ia[i] = ia[i] * x + y; ia[i] = ia[i] * y + x; ia[i] = ia[i] * x + y; ia[i] = ia[i] * y + x; }  // 2 FFMA2 + 4 IMAD (= 2 evals)
    }
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < 8; i++) s ^= (uint32_t)acc[i] ^ ia[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template<int MODE> void run(const char* nm, float* in, float* out, unsigned long long* cyc) {
  int reps = 4000; k<MODE><<<148*4, 256>>>(in, out, reps, cyc); cudaDeviceSynchronize();
  k<MODE><<<148*4, 256>>>(in, out, reps, cyc); cudaDeviceSynchronize();
  unsigned long long h[148*4]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < 148*4; i++) mx = h[i] > mx ? h[i] : mx;
  // warp-instructions per clk per SMSP of the first op: 4 blocks x 8 warps x reps x 8 / cycles / 4 SMSP
  double wi = 4.0 * 8 * reps * 8 / mx / 4;
  printf("%s: %.3f loop-iterations (x8 per warp) per clk per SMSP\n", nm, wi);
}
int main() { float *in, *out; unsigned long long* cyc; cudaMalloc(&in, 4096); cudaMemset(in, 0, 4096); cudaMalloc(&out, 148*4*256*4); cudaMalloc(&cyc, 148*4*8);
  run<0>("ffma2 3reg", in, out, cyc); run<1>("ffma2 broadcast a", in, out, cyc); run<2>("ffma2 + 2 imad", in, out, cyc); run<3>("2 ffma2 + 4 imad", in, out, cyc); }
