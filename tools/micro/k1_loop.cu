// K1 inner-loop ceiling (design exploration): the (a x + b) mod P evaluation loop of
// lb_minhash.cu in isolation -- 4 permutations per lane, shingle limbs broadcast from shared
// memory, running minima in registers -- with pieces removed to price each one.
//   MODE 0: carry-free eval + 3-input min + flag (the production loop)
//   MODE 1: no flag
//   MODE 2: only the four IMAD.WIDE products folded into the minimum (not a valid result)
//   MODE 3: exact carry-chain eval + min
//   MODE 4-6: noflag with a register shift amount / without the quotient term / sums only
// Reports evaluations / clock / SMSP (clock from clock64 inside the kernel).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct __align__(16) PermCoef { uint32_t a0, a1, b0, b1; };
struct __align__(16) PermCoefB { uint32_t a0, a1, b1, b0; };   // the library's order
struct __align__(16) XLimbs { uint32_t xl, xh, xh2, xl4; };
// Same limbs, reordered so that every product reads one even- and one odd-numbered register
// (a0 / a1 sit in an even / odd register of the LDG.128 quad; LDS.128 fills an aligned quad).
struct __align__(16) XLimbsB { uint32_t xh, xl, xl4, xh2; };
__device__ uint32_t g_sh29 = 29;

template <int MODE, typename XL, typename PC>
__device__ __forceinline__ uint32_t ev(const PC& c, const XL& x, uint32_t& f) {
  uint32_t y;
  if (MODE == 0 || MODE == 1) {
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1, t1, t2;\n\t"
        "mov.b64 B, {%3, %4};\n\tmad.wide.u32 A, %2, %5, B;\n\tmad.wide.u32 A, %6, %7, A;\n\t"
        "mul.wide.u32 G, %2, %8;\n\tmad.wide.u32 G, %6, %9, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "shl.b32 t1, g0, 29;\n\tshr.u32 t2, g0, 3;\n\tadd.u32 s0, s0, t1;\n\tadd.u32 s0, s0, g1;\n\t"
        "add.u32 s1, s1, t2;\n\tor.b32 %1, s1, 0xE0000000;\n\tshr.u32 t1, s1, 29;\n\tadd.u32 %0, s0, t1;\n\t}"
        : "=r"(y), "=r"(f)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
  } else if (MODE == 2) {
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1;\n\t"
        "mov.b64 B, {%2, %3};\n\tmad.wide.u32 A, %1, %4, B;\n\tmad.wide.u32 A, %5, %6, A;\n\t"
        "mul.wide.u32 G, %1, %7;\n\tmad.wide.u32 G, %5, %8, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "xor.b32 %0, s0, g1;\n\t}"
        : "=r"(y)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
    f = 0;
  } else if (MODE == 4) {   // noflag with the shift amount in a register (SHF + IADD3 on the ALU pipe)
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1, t1, t2;\n\t"
        "mov.b64 B, {%2, %3};\n\tmad.wide.u32 A, %1, %4, B;\n\tmad.wide.u32 A, %5, %6, A;\n\t"
        "mul.wide.u32 G, %1, %7;\n\tmad.wide.u32 G, %5, %8, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "shl.b32 t1, g0, %9;\n\tshr.u32 t2, g0, 3;\n\tadd.u32 s0, s0, t1;\n\tadd.u32 s0, s0, g1;\n\t"
        "add.u32 s1, s1, t2;\n\tshr.u32 t1, s1, 29;\n\tadd.u32 %0, s0, t1;\n\t}"
        : "=r"(y)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4), "r"(g_sh29));
    f = 0;
  } else if (MODE == 7) {   // production (with flag) but the shift amount in a register: SHF + IADD3 on ALU
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1, t1, t2;\n\t"
        "mov.b64 B, {%3, %4};\n\tmad.wide.u32 A, %2, %5, B;\n\tmad.wide.u32 A, %6, %7, A;\n\t"
        "mul.wide.u32 G, %2, %8;\n\tmad.wide.u32 G, %6, %9, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "shl.b32 t1, g0, %10;\n\tshr.u32 t2, g0, 3;\n\tadd.u32 s0, s0, t1;\n\tadd.u32 s0, s0, g1;\n\t"
        "add.u32 s1, s1, t2;\n\tor.b32 %1, s1, 0xE0000000;\n\tshr.u32 t1, s1, 29;\n\tadd.u32 %0, s0, t1;\n\t}"
        : "=r"(y), "=r"(f)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4), "r"(g_sh29));
  } else if (MODE == 5) {   // noflag without the quotient term (y = low32(S); not a valid result)
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1, t1;\n\t"
        "mov.b64 B, {%2, %3};\n\tmad.wide.u32 A, %1, %4, B;\n\tmad.wide.u32 A, %5, %6, A;\n\t"
        "mul.wide.u32 G, %1, %7;\n\tmad.wide.u32 G, %5, %8, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "shl.b32 t1, g0, 29;\n\tadd.u32 s0, s0, t1;\n\tadd.u32 %0, s0, g1;\n\t}"
        : "=r"(y)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
    f = 0;
  } else if (MODE == 6) {   // four products, both 64-bit sums, no fold (y = A_lo ^ G_hi)
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1;\n\t"
        "mov.b64 B, {%2, %3};\n\tmad.wide.u32 A, %1, %4, B;\n\tmad.wide.u32 A, %5, %6, A;\n\t"
        "mul.wide.u32 G, %1, %7;\n\tmad.wide.u32 G, %5, %8, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "add.u32 %0, s0, g1;\n\t}"
        : "=r"(y)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
    f = 0;
  } else {
    asm("{\n\t.reg .u64 A, G, B;\n\t.reg .u32 s0, s1, g0, g1, t1, t2, q;\n\t"
        "mov.b64 B, {%2, %3};\n\tadd.u64 B, B, 1;\n\tmad.wide.u32 A, %1, %4, B;\n\tmad.wide.u32 A, %5, %6, A;\n\t"
        "mul.wide.u32 G, %1, %7;\n\tmad.wide.u32 G, %5, %8, G;\n\tmov.b64 {s0, s1}, A;\n\tmov.b64 {g0, g1}, G;\n\t"
        "shl.b32 t1, g0, 29;\n\tshr.u32 t2, g0, 3;\n\tadd.cc.u32 s0, s0, t1;\n\taddc.u32 s1, s1, t2;\n\t"
        "add.cc.u32 s0, s0, g1;\n\taddc.u32 s1, s1, 0;\n\tshr.u32 q, s1, 29;\n\tadd.cc.u32 t1, s0, q;\n\t"
        "addc.u32 t2, s1, 0;\n\tshr.u32 q, t2, 29;\n\tadd.u32 s0, s0, q;\n\tsub.u32 %0, s0, 1;\n\t}"
        : "=r"(y)
        : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
    f = 0;
  }
  return y;
}

template <int MODE, int THREADS, typename XL = XLimbs, typename PC = PermCoef>
__global__ void __launch_bounds__(THREADS) kern(const PermCoef* __restrict__ C, const XLimbs* __restrict__ X, int reps,
                                                uint32_t* out, unsigned long long* cyc) {
  __shared__ XL xs[THREADS / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {
    const XLimbs v = X[(blockIdx.x * 7 + w * 3 + lane) & 1023];
    xs[w][lane].xl = v.xl;
    xs[w][lane].xh = v.xh;
    xs[w][lane].xh2 = v.xh2;
    xs[w][lane].xl4 = v.xl4;
  }
  PC c[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const PermCoef v = C[lane + 32 * q];
    c[q].a0 = v.a0;
    c[q].a1 = v.a1;
    c[q].b0 = v.b0;
    c[q].b1 = v.b1;
  }
  uint32_t m[4] = {~0u, ~0u, ~0u, ~0u}, fmax = 0;
  __syncwarp();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    for (int j = 0; j < 32; j += 4) {
      XL xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) xv[u] = xs[w][(j + u + r) & 31];   // varies per rep: no hoisting
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int u = 0; u < 4; u += 2) {
          uint32_t f0, f1;
          const uint32_t y0 = ev<MODE>(c[q], xv[u], f0), y1 = ev<MODE>(c[q], xv[u + 1], f1);  // NOLINT
          m[q] = min(m[q], min(y0, y1));
          if (MODE == 0 || MODE == 7) fmax = max(fmax, max(f0, f1));
        }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = fmax;
#pragma unroll
  for (int q = 0; q < 4; q++) acc ^= m[q];
  out[blockIdx.x * THREADS + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int THREADS, typename XL = XLimbs, typename PC = PermCoef>
void run(const char* name, int blocks_per_sm, const PermCoef* dC, const XLimbs* dX, uint32_t* dO,
         unsigned long long* dcyc) {
  const int reps = 2000, nb = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int r = 0; r < 4; r++) {
    cudaEventRecord(e0);
    kern<MODE, THREADS, XL, PC><<<nb, THREADS>>>(dC, dX, reps, dO, dcyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  static unsigned long long h[148 * 64];
  cudaMemcpy(h, dcyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  const double evals_per_sm = (double)blocks_per_sm * THREADS * 4 * 32 * reps;
  printf("{\"mode\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"eval_per_clk_smsp\": %.3f, \"Geval_s\": %.1f, "
         "\"clk_mhz\": %.0f, \"err\": \"%s\"}\n",
         name, THREADS, blocks_per_sm, evals_per_sm / cmax / 4, evals_per_sm * 148 / best / 1e6, cmax / (best * 1e3),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  PermCoef hC[128];
  XLimbs hX[1024];
  uint64_t s = 1;
  auto nx = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return s; };
  for (int i = 0; i < 128; i++) {
    uint64_t a = 1 + nx() % 0x1FFFFFFFFFFFFFFEull, b = nx() % 0x1FFFFFFFFFFFFFFFull;
    hC[i] = {(uint32_t)(a & 0x7FFFFFFF), (uint32_t)(a >> 31), (uint32_t)b, (uint32_t)(b >> 32)};
  }
  for (int i = 0; i < 1024; i++) {
    uint64_t x = nx() % 0x1FFFFFFFFFFFFFFFull;
    hX[i] = {(uint32_t)(x & 0x3FFFFFFF), (uint32_t)(x >> 30), (uint32_t)(x >> 30) << 1, (uint32_t)(x & 0x3FFFFFFF) << 2};
  }
  PermCoef* dC;
  XLimbs* dX;
  uint32_t* dO;
  unsigned long long* dcyc;
  cudaMalloc(&dC, sizeof hC);
  cudaMalloc(&dX, sizeof hX);
  cudaMalloc(&dO, 4ull * 148 * 64 * 1024);
  cudaMalloc(&dcyc, 8ull * 148 * 64);
  cudaMemcpy(dC, hC, sizeof hC, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, hX, sizeof hX, cudaMemcpyHostToDevice);
  for (int bps : {1, 2, 3, 4}) run<0, 256>("prod", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<1, 256>("noflag", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<2, 256>("wide_only", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<3, 256>("exact_chain", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<4, 256>("noflag_varshift", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<5, 256>("noflag_noq", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<6, 256>("wide_sums_only", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 3, 4}) run<0, 256, XLimbsB>("prod_banked", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<1, 256, XLimbsB>("noflag_banked", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<3, 256, XLimbsB>("exact_chain_banked", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<0, 256, XLimbsB, PermCoefB>("prod_banked_bswap", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<7, 256, XLimbsB, PermCoefB>("prod_banked_bswap_varshift", bps, dC, dX, dO, dcyc);
  for (int bps : {2, 4}) run<1, 256, XLimbsB, PermCoefB>("noflag_banked_bswap", bps, dC, dX, dO, dcyc);
  return 0;
}
