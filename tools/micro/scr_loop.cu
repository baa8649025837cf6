// Screened-K1 inner loop in isolation (design exploration): 8 permutation slots per lane, shingle
// limbs broadcast from shared memory in groups of 4, running thresholds in registers.  Prices the
// candidate bookkeeping of k1_minhash_scr2 (lb_minhash.cu):
//   MODE 0: production -- per evaluation ISETP + mask bit (mask[q] |= 1 << j)
//   MODE 1: per evaluation a running max of w over the group, one compare per (slot, group)
//   MODE 2: MODE 1 with the addend folded: w = (t + G_hi) + (G_lo << 29), max fused by ptxas
//   MODE 3: only the four multiplies (not a valid screen)
// Reports evaluations / clock / SMSP (clock64 inside the kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scr_loop scr_loop.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct __align__(16) XLimbs { uint32_t xh, xl, xl4, xh2; };
__device__ uint32_t g_sh29 = 29;

template <int MODE>
__device__ __forceinline__ uint32_t wval(uint32_t a0, uint32_t a1, const XLimbs& x, uint32_t bias, uint32_t sh) {
  uint32_t w;
  if (MODE == 0 || MODE == 1) {
    asm("{\n\t.reg .u64 G;\n\t.reg .u32 t, g0, g1;\n\t"
        "mad.lo.u32 t, %1, %3, %7;\n\tmad.lo.u32 t, %2, %4, t;\n\t"
        "mul.wide.u32 G, %1, %5;\n\tmad.wide.u32 G, %2, %6, G;\n\tmov.b64 {g0, g1}, G;\n\t"
        "shl.b32 g0, g0, %8;\n\tadd.u32 t, t, g1;\n\tadd.u32 %0, t, g0;\n\t}"
        : "=r"(w)
        : "r"(a0), "r"(a1), "r"(x.xl), "r"(x.xh), "r"(x.xh2), "r"(x.xl4), "r"(bias), "r"(sh));
  } else if (MODE == 2) {
    asm("{\n\t.reg .u64 G;\n\t.reg .u32 t, g0, g1;\n\t"
        "mul.wide.u32 G, %1, %5;\n\tmad.wide.u32 G, %2, %6, G;\n\tmov.b64 {g0, g1}, G;\n\t"
        "mad.lo.u32 t, %1, %3, g1;\n\tmad.lo.u32 t, %2, %4, t;\n\t"
        "shl.b32 g0, g0, %8;\n\tadd.u32 t, t, %7;\n\tadd.u32 %0, t, g0;\n\t}"
        : "=r"(w)
        : "r"(a0), "r"(a1), "r"(x.xl), "r"(x.xh), "r"(x.xh2), "r"(x.xl4), "r"(bias), "r"(sh));
  } else {
    asm("{\n\t.reg .u64 G;\n\t.reg .u32 t, g0, g1;\n\t"
        "mad.lo.u32 t, %1, %3, %7;\n\tmad.lo.u32 t, %2, %4, t;\n\t"
        "mul.wide.u32 G, %1, %5;\n\tmad.wide.u32 G, %2, %6, G;\n\tmov.b64 {g0, g1}, G;\n\t"
        "xor.b32 %0, t, g1;\n\t}"
        : "=r"(w)
        : "r"(a0), "r"(a1), "r"(x.xl), "r"(x.xh), "r"(x.xh2), "r"(x.xl4), "r"(bias), "r"(sh));
  }
  return w;
}

template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) kern(const uint32_t* __restrict__ C, const XLimbs* __restrict__ X, int reps,
                                                  uint32_t* out, unsigned long long* cyc) {
  constexpr int NPL = 8;
  __shared__ XLimbs xs[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  xs[w][lane] = X[(blockIdx.x * 7 + w * 3 + lane) & 1023];
  uint32_t a0[NPL], a1[NPL], bias[NPL], K[NPL], mask[NPL];
#pragma unroll
  for (int q = 0; q < NPL; q++) {
    a0[q] = C[(lane + 32 * q) * 2] & 0x7FFFFFFF;
    a1[q] = C[(lane + 32 * q) * 2 + 1] & 0x3FFFFFFF;
    bias[q] = C[lane * 3 + q];
    K[q] = 0xFFFFFFF0u;          // (almost) never a candidate: the steady state of a long document
    mask[q] = 0;
  }
  uint32_t sh;
  asm volatile("mov.u32 %0, %1;" : "=r"(sh) : "r"(29));
  __syncwarp();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    for (int j = 0; j < 32; j += 4) {
      XLimbs xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) xv[u] = xs[w][(j + u + r) & 31];
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        if (MODE == 0) {
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (wval<0>(a0[q], a1[q], xv[u], bias[q], sh) > K[q]) mask[q] |= 1u << (j + u);
        } else if (MODE == 3) {
#pragma unroll
          for (int u = 0; u < 4; u++) mask[q] ^= wval<3>(a0[q], a1[q], xv[u], bias[q], sh);
        } else {
          uint32_t mx = 0;
#pragma unroll
          for (int u = 0; u < 4; u++) mx = max(mx, wval<MODE>(a0[q], a1[q], xv[u], bias[q], sh));
          if (mx > K[q]) mask[q] |= 1u << (j >> 2);
        }
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int q = 0; q < NPL; q++) acc ^= mask[q];
  out[blockIdx.x * 256 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int MINB>
void run(const char* name, int bps, const uint32_t* dC, const XLimbs* dX, uint32_t* dO, unsigned long long* dcyc) {
  const int reps = 1000, nb = 148 * bps;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int r = 0; r < 4; r++) {
    cudaEventRecord(e0);
    kern<MODE, MINB><<<nb, 256>>>(dC, dX, reps, dO, dcyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  static unsigned long long h[148 * 8];
  cudaMemcpy(h, dcyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  const double evals_per_sm = (double)bps * 256 * 8 * 32 * reps;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern<MODE, MINB>);
  printf("{\"mode\": \"%s\", \"blocks_per_sm\": %d, \"regs\": %d, \"eval_per_clk_smsp\": %.3f, \"frac_of_8_3\": %.3f, "
         "\"Geval_s\": %.1f, \"err\": \"%s\"}\n",
         name, bps, fa.numRegs, evals_per_sm / cmax / 4, evals_per_sm / cmax / 4 / (8.0 / 3.0),
         evals_per_sm * 148 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t hC[1024];
  XLimbs hX[1024];
  uint64_t s = 1;
  auto nx = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(s >> 32); };
  for (int i = 0; i < 1024; i++) hC[i] = nx();
  for (int i = 0; i < 1024; i++) {
    uint32_t xl = nx() & 0x3FFFFFFF, xh = nx() & 0x7FFFFFFF;
    hX[i] = {xh, xl, xl << 2, xh << 1};
  }
  uint32_t *dC, *dO;
  XLimbs* dX;
  unsigned long long* dcyc;
  cudaMalloc(&dC, sizeof hC);
  cudaMalloc(&dX, sizeof hX);
  cudaMalloc(&dO, 148 * 8 * 256 * 4);
  cudaMalloc(&dcyc, 148 * 8 * 8);
  cudaMemcpy(dC, hC, sizeof hC, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, hX, sizeof hX, cudaMemcpyHostToDevice);
  for (int bps : {2, 3}) {
    run<0, 3>("mask_per_eval", bps, dC, dX, dO, dcyc);
    run<1, 3>("max_per_group", bps, dC, dX, dO, dcyc);
    run<2, 3>("max_per_group_folded", bps, dC, dX, dO, dcyc);
    run<3, 3>("products_only", bps, dC, dX, dO, dcyc);
  }
  run<0, 4>("mask_per_eval", 4, dC, dX, dO, dcyc);
  run<1, 4>("max_per_group", 4, dC, dX, dO, dcyc);
  run<2, 4>("max_per_group_folded", 4, dC, dX, dO, dcyc);
  return 0;
}
