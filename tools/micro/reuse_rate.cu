// Does the operand reuse cache lift the 3-register IMAD / FFMA issue rate above 0.5 / clk / SMSP?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o reuse_rate reuse_rate.cu
#include <cstdint>
#include <cstdio>
template <int MODE>
__global__ void k(const uint32_t* in, uint32_t* out, int reps, unsigned long long* cyc) {
  uint32_t acc[8], a[8];
  float fa[8], facc[8];
  for (int i = 0; i < 8; i++) { acc[i] = in[threadIdx.x + i]; a[i] = in[threadIdx.x + 8 + i] | 1; fa[i] = (float)a[i]; facc[i] = (float)acc[i]; }
  uint32_t x = in[threadIdx.x & 31] | 1, y = in[(threadIdx.x + 3) & 31];
  float fx = (float)x * 1e-9f, fy = (float)y;
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) acc[i] = acc[i] * x + y;          // IMAD: x, y common (reusable)
      if (MODE == 1) acc[i] = a[i] * acc[i] + a[(i + 1) & 7];   // IMAD: three per-i registers
      if (MODE == 2) facc[i] = fmaf(facc[i], fx, fy);  // FFMA: fx, fy common
      if (MODE == 3) facc[i] = fmaf(fa[i], facc[i], fa[(i + 1) & 7]);  // FFMA: three per-i registers
      if (MODE == 4) { acc[i] = acc[i] * x + y; facc[i] = fmaf(facc[i], fx, fy); }   // both, reusable
    }
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= acc[i] ^ __float_as_uint(facc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* nm, uint32_t* in, uint32_t* out, unsigned long long* cyc) {
  const int reps = 4000, nb = 148 * 4;
  for (int it = 0; it < 2; it++) k<MODE><<<nb, 256>>>(in, out, reps, cyc);
  cudaDeviceSynchronize();
  static unsigned long long h[148 * 4];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nb; i++) mx = h[i] > mx ? h[i] : mx;
  const double ops = (MODE == 4 ? 2.0 : 1.0) * 4 * 8 * reps * 8 / mx / 4;   // warp-instr / clk / SMSP
  printf("%-40s %.3f warp-inst/clk/SMSP\n", nm, ops);
}
int main() {
  uint32_t *in, *out;
  unsigned long long* cyc;
  cudaMalloc(&in, 4096);
  cudaMemset(in, 1, 4096);
  cudaMalloc(&out, 148 * 4 * 256 * 4);
  cudaMalloc(&cyc, 148 * 4 * 8);
  run<0>("IMAD acc*x+y (x, y common)", in, out, cyc);
  run<1>("IMAD a[i]*acc[i]+a[i+1]", in, out, cyc);
  run<2>("FFMA acc*fx+fy (common)", in, out, cyc);
  run<3>("FFMA fa[i]*acc[i]+fa[i+1]", in, out, cyc);
  run<4>("IMAD + FFMA, common operands", in, out, cyc);
}
