// Microbenchmark: throughput of the truncated mod-Mersenne multiply-add + min
// inner loop in several formulations (design exploration, not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define P61 0x1FFFFFFFFFFFFFFFull
#define M29 0x1FFFFFFFu

// V0: 128-bit reference (__int128 % P)
__device__ __forceinline__ uint32_t ev_ref(uint64_t a, uint64_t b, uint64_t x) {
  unsigned __int128 t = (unsigned __int128)a * x + b;
  return (uint32_t)(uint64_t)(t % P61);
}
// V1: Mersenne fold with umul64hi
__device__ __forceinline__ uint32_t ev_fold(uint64_t a, uint64_t b, uint64_t x) {
  uint64_t lo = a * x, hi = __umul64hi(a, x);
  // t = hi*2^64 + lo ; t>>61 = hi<<3 | lo>>61
  uint64_t s = (lo & P61) + ((hi << 3) | (lo >> 61)) + b;   // < 3*2^61
  s = (s & P61) + (s >> 61);
  if (s >= P61) s -= P61;
  return (uint32_t)s;
}
// V2: limb formulation (a,x < 2^61)
__device__ __forceinline__ uint32_t ev_limb(uint32_t a0, uint32_t a1, uint64_t b, uint32_t x0, uint32_t x1, uint32_t x1_8) {
  uint64_t u = (uint64_t)a0 * x0;
  uint64_t K = (uint64_t)a0 * x1 + (uint64_t)a1 * x0 + (u >> 32);   // < 2^62 + 2^32
  uint64_t w = (uint64_t)a1 * x1_8 + b;                                // < 2^62
  uint64_t S = w + (K >> 29) + ((((uint64_t)((uint32_t)K & M29)) << 32) | (uint32_t)u);
  uint64_t t1 = (S & P61) + (S >> 61) + 1;
  return (uint32_t)t1 - 1u + (uint32_t)(t1 >> 61);
}


// V3: limb formulation in PTX with explicit carry chains
__device__ __forceinline__ uint32_t ev_ptx(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1, uint32_t x0, uint32_t x1, uint32_t x1_8) {
  uint32_t y;
  asm("{\n\t.reg .u32 u0,u1,k0,k1,w0,w1,ks,kh,km,s0,s1,sh,hm,l,h;\n\t"
      "mul.lo.u32 u0, %1, %5;\n\t"
      "mul.hi.u32 u1, %1, %5;\n\t"
      "mad.lo.cc.u32 k0, %1, %6, u1;\n\t"
      "madc.hi.u32 k1, %1, %6, 0;\n\t"
      "mad.lo.cc.u32 k0, %2, %5, k0;\n\t"
      "madc.hi.u32 k1, %2, %5, k1;\n\t"
      "mad.lo.cc.u32 w0, %2, %7, %3;\n\t"
      "madc.hi.u32 w1, %2, %7, %4;\n\t"
      "shf.r.wrap.b32 ks, k0, k1, 29;\n\t"
      "shr.u32 kh, k1, 29;\n\t"
      "and.b32 km, k0, 0x1FFFFFFF;\n\t"
      "add.cc.u32 s0, w0, ks;\n\t"
      "addc.u32 s1, w1, kh;\n\t"
      "add.cc.u32 s0, s0, u0;\n\t"
      "addc.u32 s1, s1, km;\n\t"
      "shr.u32 sh, s1, 29;\n\t"
      "or.b32 hm, s1, 0xE0000000;\n\t"
      "add.cc.u32 l, s0, sh;\n\t"
      "addc.u32 h, hm, 0;\n\t"
      "add.cc.u32 l, l, 1;\n\t"
      "addc.cc.u32 h, h, 0;\n\t"
      "addc.u32 %0, l, -1;\n\t"
      "}" : "=r"(y) : "r"(a0), "r"(a1), "r"(b0), "r"(b1), "r"(x0), "r"(x1), "r"(x1_8));
  return y;
}

template <int V, int NPL>
__global__ void kern(const uint64_t* __restrict__ A, const uint64_t* __restrict__ B,
                     const uint64_t* __restrict__ X, int S, uint32_t* out) {
  int lane = threadIdx.x & 31;
  int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t a[NPL], b[NPL]; uint32_t a0[NPL], a1[NPL]; uint32_t m[NPL];
#pragma unroll
  for (int q = 0; q < NPL; q++) { a[q] = A[lane + 32 * q]; b[q] = B[lane + 32 * q];
    a0[q] = (uint32_t)a[q]; a1[q] = (uint32_t)(a[q] >> 32); m[q] = 0xFFFFFFFFu; }
  const uint64_t* xs = X + (size_t)(gw & 1023) * S;
  for (int s = 0; s < S; s++) {
    uint64_t x = xs[s];
    uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), x1_8 = x1 << 3;
#pragma unroll
    for (int q = 0; q < NPL; q++) {
      uint32_t v;
      if (V == 0) v = ev_ref(a[q], b[q], x);
      else if (V == 1) v = ev_fold(a[q], b[q], x);
      else if (V == 2) v = ev_limb(a0[q], a1[q], b[q], x0, x1, x1_8);
      else v = ev_ptx(a0[q], a1[q], (uint32_t)b[q], (uint32_t)(b[q] >> 32), x0, x1, x1_8);
      m[q] = min(m[q], v);
    }
  }
#pragma unroll
  for (int q = 0; q < NPL; q++) out[(size_t)gw * 32 * NPL + lane + 32 * q] = m[q];
}

static uint64_t sm64(uint64_t& s) { uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

int main() {
  const int NPL = 4, NP = 32 * NPL, S = 512, NW = 148 * 64;  // warps
  uint64_t hA[NP], hB[NP]; uint64_t st = 1;
  for (int i = 0; i < NP; i++) { hA[i] = 1 + sm64(st) % (P61 - 1); hB[i] = sm64(st) % P61; }
  uint64_t* hX = new uint64_t[1024 * S];
  for (int i = 0; i < 1024 * S; i++) hX[i] = sm64(st) % P61;
  hX[0] = P61 - 1; hX[1] = 0;
  uint64_t *dA, *dB, *dX; uint32_t* dO[4];
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dX, 8ull * 1024 * S);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, hX, 8ull * 1024 * S, cudaMemcpyHostToDevice);
  size_t on = (size_t)NW * NP;
  for (int v = 0; v < 4; v++) cudaMalloc(&dO[v], on * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int v = 0; v < 4; v++) {
    for (int bs : {128, 256}) {
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (v == 0) kern<0, NPL><<<NW * 32 / bs, bs>>>(dA, dB, dX, S, dO[v]);
        if (v == 1) kern<1, NPL><<<NW * 32 / bs, bs>>>(dA, dB, dX, S, dO[v]);
        if (v == 3) kern<3, NPL><<<NW * 32 / bs, bs>>>(dA, dB, dX, S, dO[v]);
        if (v == 2) kern<2, NPL><<<NW * 32 / bs, bs>>>(dA, dB, dX, S, dO[v]);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double evals = (double)NW * 32 * NPL * S;
        if (rep == 2) printf("V%d bs=%d: %.3f ms  %.3f Teval/s  %s\n", v, bs, ms, evals / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  uint32_t* h0 = new uint32_t[on]; uint32_t* h1 = new uint32_t[on];
  cudaMemcpy(h0, dO[0], on * 4, cudaMemcpyDeviceToHost);
  for (int v = 1; v < 4; v++) {
    cudaMemcpy(h1, dO[v], on * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0; for (size_t i = 0; i < on; i++) bad += h0[i] != h1[i];
    printf("V%d mismatches vs V0: %zu\n", v, bad);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock attr %d kHz\n", clk);
  return 0;
}
