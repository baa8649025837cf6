// Can the FP32 pipe take the high half of the MinHash screen? (design exploration, round 2)
//   a = ah 2^32 + al, x = xh 2^32 + xl (ah, xh < 2^29), M = ah xl + al xh (< 2^62), H = floor(M / 2^29):
//   y = low32((a x + b) mod P) = L + H + q (mod 2^32),  L = lo(al xl) + lo(8ah xh) + lo(b),  q in [0, 11]
//   (lb_minhash.cu, k1_minhash_scr3).  A screen needs H only to within a few thousand:
//   r = fmaf(ah_f, xl_f 2^-29, fmaf(al_f, xh_f 2^-29, 1.5 2^34))  (operands rounded to binary32)
//   lies in [2^34, 2^35] where the ulp is 2^11, and (bits(r) << 11) = r - 1.5 2^34 (mod 2^32).
//   Error: operand rounding 2 x 2^9, two roundings 2 x 2^10 -> |Hc - H| <= 3074.
//   u = L + 4096 + (bits(r) << 11)  =>  u - y in [1011, 7170] (mod 2^32), so y < m => u < m + 8192.
// Part 1 (correctness): verdicts against exact (a x + b) mod P on 2^32 random + adversarial triples
// (a false negative would be a wrong signature), and the largest |Hc - H| seen.
// Part 2 (rate, evaluations/clk/SMSP): FFMA pair alone, FFMA pair + IMAD pair, the FP32 screen with
// per-evaluation mask bits, with a min over each 4-shingle group, and the shipped FP64 screen.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_screen fp32_screen.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint64_t kP = 0x1FFFFFFFFFFFFFFFull;
constexpr float kMagicF = 25769803776.0f;        // 1.5 * 2^34
constexpr double kMagicD = 6755399441055744.0;   // 1.5 * 2^52
constexpr uint32_t kD = 4096, kW = 8192;

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

struct SlotF { uint32_t al, a8h, lb; float AL, AH; };      // lb = lo(b) + kD
struct XF { uint32_t xl, xh; float XL, XH; };              // XL = fl(xl) 2^-29, XH = fl(xh) 2^-29
struct SlotD { uint32_t al, a8h; double AL, AH, CB; };
struct XD { uint32_t xl, xh; double XL, XH; };

__device__ __forceinline__ uint32_t screen_f32(const SlotF& s, const XF& x) {
  const float r1 = __fmaf_rn(s.AL, x.XH, kMagicF);
  const float r2 = __fmaf_rn(s.AH, x.XL, r1);
  const uint32_t t = s.al * x.xl + s.a8h * x.xh + s.lb;
  return t + (__float_as_uint(r2) << 11);
}
__device__ __forceinline__ uint32_t screen_f64(const SlotD& s, const XD& x) {
  const double r1 = fma(s.AL, x.XH, s.CB);
  const double r2 = fma(s.AH, x.XL, r1);
  return s.al * x.xl + s.a8h * x.xh + (uint32_t)__double2loint(r2);
}


__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
struct SlotF2 { uint32_t al, a8h, lb; uint64_t AL2, AH2; };
struct __align__(16) XF2 { uint64_t XH2, XL2; uint32_t xl0, xl1, xh0, xh1; };   // a shingle pair
__device__ __forceinline__ uint32_t t_int(uint32_t al, uint32_t xl, uint32_t a8h, uint32_t xh, uint32_t lb) {
  uint32_t t;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(al), "r"(xl), "r"(lb));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a8h), "r"(xh), "r"(t));
  return t;
}
__device__ __forceinline__ uint32_t shl11(uint32_t v) {
  uint32_t r;
  asm("shl.b32 %0, %1, 11;" : "=r"(r) : "r"(v));
  return r;
}

__global__ void check(uint64_t seed, uint64_t n, unsigned long long* stats) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long fn = 0, cand = 0, below = 0, emax = 0;
  for (; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = mix(seed + 3 * i), r1 = mix(seed + 3 * i + 1), r2 = mix(seed + 3 * i + 2);
    uint64_t a = 1 + r0 % (kP - 1), x = r1 % kP, b = (r2 >> 3) % kP;
    if ((i & 7) == 0) a = kP - 1 - (r0 & 0xFF);            // adversarial: near-P operands
    if ((i & 7) == 1) x = kP - 1 - (r1 & 0xFF);
    if ((i & 15) == 2) x = (r1 & 1) ? 0xFFFFFFFFull : (0x1FFFFFFFull << 32);
    if ((i & 15) == 3) { a = ((r0 & 0x1FFFFFFFull) << 32) | 0xFFFFFF80u | (r0 >> 57); }   // al near 2^32
    if ((i & 15) == 4) { x = ((r1 & 0x1FFFFFFFull) << 32) | 0xFFFFFF80u | (r1 >> 57); }   // xl near 2^32
    if ((i & 15) == 5) { a = (0x1FFFFF80ull + (r0 & 0x7F)) << 32 | (uint32_t)r0; }        // ah near 2^29
    if (a == 0) a = 1;
    if (x >= kP) x -= kP;
    const uint64_t ax = mulmod_p(a, x);
    const uint32_t y = (uint32_t)(ax + b >= kP ? ax + b - kP : ax + b);
    const uint32_t m = (r2 & 3) ? (uint32_t)(r2 >> 40) : (uint32_t)(r2 >> 32) % (0xFFFFFFFFu - kW);
    const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32), xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    SlotF s{al, ah << 3, (uint32_t)b + kD, __uint2float_rn(al), __uint2float_rn(ah)};
    XF xf{xl, xh, __uint2float_rn(xl) * 0x1p-29f, __uint2float_rn(xh) * 0x1p-29f};
    const uint32_t u = screen_f32(s, xf);
    const bool c = u < m + kW;
    cand += c;
    below += y < m;
    fn += (y < m) && !c;
    // |Hc - H|: Hc = bits << 11 (mod 2^32), H = floor(M / 2^29) (mod 2^32)
    const unsigned __int128 M = (unsigned __int128)ah * xl + (unsigned __int128)al * xh;
    const uint32_t H = (uint32_t)(M >> 29);
    const float r1f = __fmaf_rn(s.AL, xf.XH, kMagicF), r2f = __fmaf_rn(s.AH, xf.XL, r1f);
    const int32_t e = (int32_t)((__float_as_uint(r2f) << 11) - H);
    const unsigned long long ae = (unsigned long long)(e < 0 ? -e : e);
    emax = ae > emax ? ae : emax;
  }
  atomicAdd(stats + 0, fn);
  atomicAdd(stats + 1, cand);
  atomicAdd(stats + 2, below);
  atomicMax(stats + 3, emax);
}

// ---- rates
template <int MODE, int MINB = 3>
__global__ void __launch_bounds__(256, MINB) rate(const uint32_t* __restrict__ C, int reps, uint32_t* out,
                                              unsigned long long* cyc) {
  constexpr int NPL = (MODE == 4) ? 4 : 8;
  __shared__ XF xs[8][32];
  __shared__ XD xd[8][32];
  __shared__ XF2 x2[8][16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {
    const uint32_t xl = C[(lane * 5 + w) & 1023], xh = C[(lane * 3 + w + 7) & 1023] & 0x1FFFFFFF;
    xs[w][lane] = XF{xl, xh, __uint2float_rn(xl) * 0x1p-29f, __uint2float_rn(xh) * 0x1p-29f};
    xd[w][lane] = XD{xl, xh, xl * 0x1p-29, xh * 0x1p-29};
  }
  __syncwarp();
  if (lane < 16) {
    const XF a = xs[w][2 * lane], b = xs[w][2 * lane + 1];
    x2[w][lane] = XF2{pack2(a.XH, b.XH), pack2(a.XL, b.XL), a.xl, b.xl, a.xh, b.xh};
  }
  const uint64_t K2 = pack2(kMagicF, kMagicF);
  SlotF2 s2[NPL];
  SlotF sl[NPL];
  SlotD sd[NPL];
  uint32_t K[NPL], mask[NPL];
  float facc[NPL];
  uint32_t iacc[NPL];
#pragma unroll
  for (int q = 0; q < NPL; q++) {
    const uint32_t al = C[lane + 32 * q], ah = C[lane + 32 * q + 256] & 0x1FFFFFFF;
    sl[q] = SlotF{al, ah << 3, C[lane * 3 + q], __uint2float_rn(al), __uint2float_rn(ah)};
    sd[q] = SlotD{al, ah << 3, (double)al, (double)ah, kMagicD + C[lane * 3 + q]};
    s2[q] = SlotF2{al, ah << 3, C[lane * 3 + q], pack2(sl[q].AL, sl[q].AL), pack2(sl[q].AH, sl[q].AH)};
    K[q] = 0x100u + C[q];
    mask[q] = 0;
    facc[q] = q;
    iacc[q] = q;
  }
  __syncwarp();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    for (int j = 0; j < 32; j += 4) {
      if (MODE == 4) {
        XD xv[4];
#pragma unroll
        for (int u = 0; u < 4; u++) xv[u] = xd[w][(j + u + r) & 31];
#pragma unroll
        for (int q = 0; q < NPL; q++)
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (screen_f64(sd[q], xv[u]) < K[q]) mask[q] |= 1u << (j + u);
        continue;
      }
      if (MODE >= 5) {
        constexpr int G = (MODE == 8) ? 8 : 4;                  // shingles per group
        if (MODE == 8 && (j & 4)) continue;
        if (MODE == 5) {                                        // explicit form A, FFMA
          XF xv[4];
#pragma unroll
          for (int u = 0; u < 4; u++) xv[u] = xs[w][(j + u + r) & 31];
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const float r1 = __fmaf_rn(sl[q].AL, xv[u].XH, kMagicF);
              const float r2 = __fmaf_rn(sl[q].AH, xv[u].XL, r1);
              mn = min(t_int(sl[q].al, xv[u].xl, sl[q].a8h, xv[u].xh, sl[q].lb) + shl11(__float_as_uint(r2)), mn);
            }
            if (mn < K[q]) mask[q] |= 1u << (j >> 2);
          }
        } else {                                                // FFMA2 over shingle pairs
          XF2 xv[G / 2];
#pragma unroll
          for (int u = 0; u < G / 2; u++) xv[u] = x2[w][((j >> 1) + u + r) & 15];
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
            for (int u = 0; u < G / 2; u++) {
              const uint64_t r2 = ffma2(s2[q].AH2, xv[u].XL2, ffma2(s2[q].AL2, xv[u].XH2, K2));
              const uint32_t b0 = shl11((uint32_t)r2), b1 = shl11((uint32_t)(r2 >> 32));
              if (MODE == 7) {                                  // form B: products without addend
                const uint32_t p0 = s2[q].al * xv[u].xl0, p1 = s2[q].al * xv[u].xl1;
                const uint32_t h0 = s2[q].a8h * xv[u].xh0, h1 = s2[q].a8h * xv[u].xh1;
                mn = min(p0 + h0 + b0 + s2[q].lb, mn);
                mn = min(p1 + h1 + b1 + s2[q].lb, mn);
              } else {
                mn = min(t_int(s2[q].al, xv[u].xl0, s2[q].a8h, xv[u].xh0, s2[q].lb) + b0, mn);
                mn = min(t_int(s2[q].al, xv[u].xl1, s2[q].a8h, xv[u].xh1, s2[q].lb) + b1, mn);
              }
            }
            if (mn < K[q]) mask[q] |= 1u << (j >> 2);
          }
        }
        continue;
      }
      XF xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) xv[u] = xs[w][(j + u + r) & 31];
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        if (MODE == 3) {                                      // min over the 4-shingle group
          const uint32_t v0 = screen_f32(sl[q], xv[0]), v1 = screen_f32(sl[q], xv[1]);
          const uint32_t v2 = screen_f32(sl[q], xv[2]), v3 = screen_f32(sl[q], xv[3]);
          const uint32_t mn = min(min(v0, v1), min(v2, v3));
          if (mn < K[q]) mask[q] |= 1u << (j >> 2);
          continue;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          if (MODE == 0) {                                    // 2 FFMA per "evaluation"
            facc[q] = __fmaf_rn(sl[q].AH, xv[u].XL, __fmaf_rn(sl[q].AL, xv[u].XH, facc[q]));
          } else if (MODE == 1) {                             // 2 FFMA + 2 IMAD.LO
            facc[q] = __fmaf_rn(sl[q].AH, xv[u].XL, __fmaf_rn(sl[q].AL, xv[u].XH, facc[q]));
            iacc[q] = sl[q].al * xv[u].xl + sl[q].a8h * xv[u].xh + iacc[q];
          } else {                                            // the FP32 screen, mask bit per evaluation
            if (screen_f32(sl[q], xv[u]) < K[q]) mask[q] |= 1u << (j + u);
          }
        }
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int q = 0; q < NPL; q++) acc ^= mask[q] ^ iacc[q] ^ __float_as_uint(facc[q]);
  out[blockIdx.x * 256 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int MINB = 3>
void run_rate(const char* name, const uint32_t* dC, uint32_t* dO, unsigned long long* dcyc) {
  constexpr int NPL = (MODE == 4) ? 4 : 8;
  const int reps = 1000;
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, rate<MODE, MINB>, 256, 0);
  const int nb = 148 * bps;
  for (int r = 0; r < 2; r++) rate<MODE, MINB><<<nb, 256>>>(dC, reps, dO, dcyc);
  cudaDeviceSynchronize();
  static unsigned long long h[148 * 8];
  cudaMemcpy(h, dcyc, 8 * nb, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < nb; i++) cmax = h[i] > cmax ? h[i] : cmax;
  const double evals_per_sm = (double)bps * 256 * NPL * 32 * reps;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, rate<MODE, MINB>);
  printf("{\"mode\": \"%s\", \"regs\": %d, \"blocks_per_sm\": %d, \"eval_per_clk_smsp\": %.3f, \"err\": \"%s\"}\n",
         name, fa.numRegs, bps, evals_per_sm / cmax / 4, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* st;
  cudaMalloc(&st, 32);
  cudaMemset(st, 0, 32);
  const uint64_t n = 1ull << 32;
  check<<<148 * 8, 256>>>(12345, n, st);
  unsigned long long h[4];
  cudaMemcpy(h, st, 32, cudaMemcpyDeviceToHost);
  printf("{\"check_triples\": %llu, \"false_negatives\": %llu, \"candidates\": %llu, \"y_below_m\": %llu, "
         "\"max_abs_Hc_minus_H\": %llu, \"bound\": 3074, \"err\": \"%s\"}\n",
         (unsigned long long)n, h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  uint32_t hC[1024];
  uint64_t s = 7;
  for (int i = 0; i < 1024; i++) { s = s * 6364136223846793005ull + 1442695040888963407ull; hC[i] = (uint32_t)(s >> 32); }
  uint32_t *dC, *dO;
  unsigned long long* dcyc;
  cudaMalloc(&dC, sizeof hC);
  cudaMalloc(&dO, 148 * 8 * 256 * 4);
  cudaMalloc(&dcyc, 148 * 8 * 8);
  cudaMemcpy(dC, hC, sizeof hC, cudaMemcpyHostToDevice);
  run_rate<0>("ffma_x2", dC, dO, dcyc);
  run_rate<1>("ffma_x2+imad_lo_x2", dC, dO, dcyc);
  run_rate<2>("fp32_screen_maskbit", dC, dO, dcyc);
  run_rate<3>("fp32_screen_min4", dC, dO, dcyc);
  run_rate<4>("fp64_screen_shipped_npl4", dC, dO, dcyc);
  run_rate<5>("fp32_formA_ptx_min4", dC, dO, dcyc);
  run_rate<6>("fp32_formA_ffma2_min4", dC, dO, dcyc);
  run_rate<7>("fp32_formB_ffma2_min4", dC, dO, dcyc);
  run_rate<8>("fp32_formA_ffma2_min8", dC, dO, dcyc);
  run_rate<5, 2>("fp32_formA_ptx_min4_2blk", dC, dO, dcyc);
  run_rate<6, 2>("fp32_formA_ffma2_min4_2blk", dC, dO, dcyc);
  run_rate<7, 2>("fp32_formB_ffma2_min4_2blk", dC, dO, dcyc);
  run_rate<8, 2>("fp32_formA_ffma2_min8_2blk", dC, dO, dcyc);
  run_rate<3, 2>("fp32_screen_min4_2blk", dC, dO, dcyc);
  run_rate<4, 2>("fp64_screen_shipped_npl4_2blk", dC, dO, dcyc);
  return 0;
}
