// Can the FP64 pipe take the high half of the MinHash screen? (design exploration)
//   a = ah 2^32 + al, x = xh 2^32 + xl (ah, xh < 2^29), M = ah xl + al xh:
//   a x + b = al xl + M_hi + 8 ah xh + b + M_lo 2^32 + q' P  with M_hi = floor(M / 2^29), so
//   low32((a x + b) mod P) = lo(al xl) + lo(8ah xh) + lo(M_hi) + lo(b) + q  (mod 2^32), q in [0, 17].
//   N = round(M / 2^29) from two DFMA with the magic addend 1.5 2^52 (|N - M/2^29| <= 1):
//   r = fma(ah, xl 2^-29, fma(al, xh 2^-29, 1.5 2^52)),  lo32(bits(r)) = N mod 2^32.
// Part 1 (correctness): screen verdicts against exact (a x + b) mod P on random triples; a
// false negative (y < m but screened out) would be a wrong signature.
// Part 2 (rate): DFMA alone, IMAD.LO alone, both interleaved, and the screen loop (4 slots x 4
// shingles per group) vs the production integer screen (2 IMAD.WIDE + 2 IMAD).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_screen dfma_screen.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint64_t kP = 0x1FFFFFFFFFFFFFFFull;
constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52
constexpr uint32_t kQ = 17, kElo = 1, kEhi = 2;  // q <= 17; N - M_hi in [-1, 2]

__device__ __forceinline__ uint64_t mulmod_p(uint64_t a, uint64_t x) {
  const uint64_t lo = a * x, hi = __umul64hi(a, x);
  uint64_t r = (lo & kP) + ((lo >> 61) | (hi << 3));
  r = (r & kP) + (r >> 61);
  return r >= kP ? r - kP : r;
}
__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
  return z ^ (z >> 33);
}

struct Slot { uint32_t al, a8h; double AL, AH; };
struct XS { uint32_t xl, xh; double XL, XH; };

__device__ __forceinline__ uint32_t wval(const Slot& s, const XS& x, uint32_t bias) {
  const double r1 = fma(s.AL, x.XH, kMagic);
  const double r2 = fma(s.AH, x.XL, r1);
  const uint32_t n = (uint32_t)__double2loint(r2);
  return s.al * x.xl + s.a8h * x.xh + n + bias;
}

__global__ void check(uint64_t seed, uint64_t n, unsigned long long* stats) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long fn = 0, cand = 0, below = 0, fn_shipped = 0, cand_shipped = 0;
  for (; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = mix(seed + 3 * i), r1 = mix(seed + 3 * i + 1), r2 = mix(seed + 3 * i + 2);
    uint64_t a = 1 + r0 % (kP - 1), x = r1 % kP, b = (r2 >> 3) % kP;
    if ((i & 7) == 0) a = kP - 1 - (r0 & 0xFF);            // adversarial: near-P operands
    if ((i & 7) == 1) x = kP - 1 - (r1 & 0xFF);
    if ((i & 15) == 2) x = (r1 & 1) ? 0xFFFFFFFFull : (0x1FFFFFFFull << 32);
    const uint32_t y = (uint32_t)(mulmod_p(a, x) + b >= kP ? mulmod_p(a, x) + b - kP : mulmod_p(a, x) + b);
    // a running minimum m: mostly small (late in a long document), sometimes anywhere
    const uint32_t m = (r2 & 3) ? (uint32_t)(r2 >> 40) : (uint32_t)(r2 >> 32) % (0xFFFFFFFFu - kQ - kEhi - kElo - 2);
    Slot s{(uint32_t)a, (uint32_t)(a >> 32) << 3, (double)(uint32_t)a, (double)(uint32_t)(a >> 32)};
    XS xs{(uint32_t)x, (uint32_t)(x >> 32), (double)(uint32_t)x * 0x1p-29, (double)(uint32_t)(x >> 32) * 0x1p-29};
    const uint32_t bias = (uint32_t)b - m - kEhi;
    const uint32_t K = 0xFFFFFFFFu - kQ - kElo - kEhi - m;
    const bool is_cand = wval(s, xs, bias) > K;
    cand += is_cand;
    below += y < m;
    fn += (y < m) && !is_cand;
    // the shipped form (lb_minhash.cu k1_minhash_scr3): lo(b) + 12 in the magic addend, u < m + 13
    const double CB = kMagic + (double)((uint32_t)b + 12u);
    const double q1 = fma(s.AL, xs.XH, CB), q2 = fma(s.AH, xs.XL, q1);
    const uint32_t u = s.al * xs.xl + s.a8h * xs.xh + (uint32_t)__double2loint(q2);
    const bool cand2 = m <= 0xFFFFFFFFu - 13u ? u < m + 13u : true;
    cand_shipped += cand2;
    fn_shipped += (y < m) && !cand2;
  }
  atomicAdd(stats + 0, fn);
  atomicAdd(stats + 1, cand);
  atomicAdd(stats + 2, below);
  atomicAdd(stats + 3, fn_shipped);
  atomicAdd(stats + 4, cand_shipped);
}

// ---- rates
template <int MODE>
__global__ void __launch_bounds__(256, 3) rate(const uint32_t* __restrict__ C, int reps, uint32_t* out,
                                              unsigned long long* cyc) {
  constexpr int NPL = 4;
  __shared__ XS xs[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {
    const uint32_t xl = C[(lane * 5 + w) & 1023], xh = C[(lane * 3 + w + 7) & 1023] & 0x1FFFFFFF;
    xs[w][lane] = XS{xl, xh, xl * 0x1p-29, xh * 0x1p-29};
  }
  Slot sl[NPL];
  uint32_t bias[NPL], K[NPL], mask[NPL];
  double dacc[NPL];
  uint32_t iacc[NPL];
#pragma unroll
  for (int q = 0; q < NPL; q++) {
    const uint32_t al = C[lane + 32 * q], ah = C[lane + 32 * q + 128] & 0x1FFFFFFF;
    sl[q] = Slot{al, ah << 3, (double)al, (double)ah};
    bias[q] = C[lane * 3 + q];
    K[q] = 0xFFFFFFF0u;
    mask[q] = 0;
    dacc[q] = q;
    iacc[q] = q;
  }
  __syncwarp();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    for (int j = 0; j < 32; j += 4) {
      XS xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) xv[u] = xs[w][(j + u + r) & 31];
#pragma unroll
      for (int q = 0; q < NPL; q++) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          if (MODE == 0) {                                    // 2 DFMA per "evaluation"
            dacc[q] = fma(sl[q].AH, xv[u].XL, fma(sl[q].AL, xv[u].XH, dacc[q]));
          } else if (MODE == 1) {                             // 2 IMAD.LO
            iacc[q] = sl[q].al * xv[u].xl + sl[q].a8h * xv[u].xh + iacc[q];
          } else if (MODE == 2) {                             // both, independent
            dacc[q] = fma(sl[q].AH, xv[u].XL, fma(sl[q].AL, xv[u].XH, dacc[q]));
            iacc[q] = sl[q].al * xv[u].xl + sl[q].a8h * xv[u].xh + iacc[q];
          } else {                                            // the FP64 screen
            if (wval(sl[q], xv[u], bias[q]) > K[q]) mask[q] |= 1u << (j + u);
          }
        }
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int q = 0; q < NPL; q++) acc ^= mask[q] ^ iacc[q] ^ (uint32_t)__double2loint(dacc[q]);
  out[blockIdx.x * 256 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run_rate(const char* name, const uint32_t* dC, uint32_t* dO, unsigned long long* dcyc) {
  const int reps = 1000, bps = 3, nb = 148 * bps;
  for (int r = 0; r < 2; r++) rate<MODE><<<nb, 256>>>(dC, reps, dO, dcyc);
  cudaDeviceSynchronize();
  static unsigned long long h[148 * 8];
  cudaMemcpy(h, dcyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  const double evals_per_sm = (double)bps * 256 * 4 * 32 * reps;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, rate<MODE>);
  printf("{\"mode\": \"%s\", \"regs\": %d, \"eval_per_clk_smsp\": %.3f, \"err\": \"%s\"}\n", name, fa.numRegs,
         evals_per_sm / cmax / 4, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* st;
  cudaMalloc(&st, 40);
  cudaMemset(st, 0, 40);
  const uint64_t n = 1ull << 32;
  check<<<148 * 8, 256>>>(12345, n, st);
  unsigned long long h[5];
  cudaMemcpy(h, st, 40, cudaMemcpyDeviceToHost);
  printf("{\"check_triples\": %llu, \"false_negatives\": %llu, \"candidates\": %llu, \"y_below_m\": %llu, "
         "\"false_negatives_shipped_form\": %llu, \"candidates_shipped_form\": %llu, \"err\": \"%s\"}\n",
         (unsigned long long)n, h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
  uint32_t hC[1024];
  uint64_t s = 7;
  for (int i = 0; i < 1024; i++) { s = s * 6364136223846793005ull + 1442695040888963407ull; hC[i] = (uint32_t)(s >> 32); }
  uint32_t *dC, *dO;
  unsigned long long* dcyc;
  cudaMalloc(&dC, sizeof hC);
  cudaMalloc(&dO, 148 * 8 * 256 * 4);
  cudaMalloc(&dcyc, 148 * 8 * 8);
  cudaMemcpy(dC, hC, sizeof hC, cudaMemcpyHostToDevice);
  run_rate<0>("dfma_x2", dC, dO, dcyc);
  run_rate<1>("imad_lo_x2", dC, dO, dcyc);
  run_rate<2>("dfma_x2+imad_lo_x2", dC, dO, dcyc);
  run_rate<3>("fp64_screen", dC, dO, dcyc);
  return 0;
}
