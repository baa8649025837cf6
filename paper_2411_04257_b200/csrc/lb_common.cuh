// lb_common.cuh -- device/host helpers of the CUDA path (sm_100a).
//
// Independent implementation of the conventions in DESIGN.md section 3; shares no code
// with oracle/ (the CPU oracle re-implements every step for parity testing).
#pragma once
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

// Bounds / invariant checks for a debug build (-DLB_CHECKS): compute-sanitizer is not
// available on the B200 pool, so tests/test_gpu_checked.py reruns parity cases against a
// library built with these device asserts.
#ifdef LB_CHECKS
#define LB_ASSERT(x) assert(x)
#else
#define LB_ASSERT(x) ((void)0)
#endif

namespace lb {

constexpr uint64_t kP = 0x1FFFFFFFFFFFFFFFull;   // 2^61 - 1
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kFpSalt = 0x6C7368626C6F6F6Dull;  // fingerprint salt (DESIGN R1)

// SplitMix64 finaliser (DESIGN R5).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// h mod P for any 64-bit h (Mersenne fold + one conditional subtract).
__host__ __device__ __forceinline__ uint64_t mod_p(uint64_t h) {
  uint64_t x = (h & kP) + (h >> 61);
  return x >= kP ? x - kP : x;
}

// (c * s + d) mod P for c, d < P and a 32-bit s (band-hash term).
__device__ __forceinline__ uint64_t affine32_mod_p(uint64_t c, uint32_t s, uint64_t d) {
  uint64_t lo = c * (uint64_t)s;
  uint64_t hi = __umul64hi(c, (uint64_t)s);   // < 2^29
  uint64_t v = (lo & kP) + ((lo >> 61) | (hi << 3)) + d;   // < 2^61 + 2^32 + 2^61
  v = (v & kP) + (v >> 61);
  return v >= kP ? v - kP : v;
}

// Per-permutation coefficients in the kernel's limb layout: a = a1 * 2^31 + a0 (a0 < 2^31,
// a1 < 2^30) and b = b1 * 2^32 + b0 (see the MinHash evaluations in lb_minhash.cu).
// Field order: a0 / a1 land in an even / odd register of the LDG.128 quad and b0 / b1 in an odd /
// even one, so the 3-input adds ptxas forms from the two products and b (IADD3 on the low words,
// IADD3.X on the high words) read registers from both banks.
struct __align__(16) PermCoef {
  uint32_t a0, a1, b1, b0;
};

// x = fingerprint mod P split for the eval: xl = x mod 2^30, xh = x >> 30 (< 2^31),
// xh2 = 2 xh, xl4 = 4 xl (both < 2^32).  Field order matters: an LDS.128 fills an aligned
// register quad, and PermCoef's a0 / a1 land in an even / odd register, so with xh, xl, xl4,
// xh2 in that order every product a0*xl, a1*xh, a0*xh2, a1*xl4 reads one even- and one
// odd-numbered register -- no register-bank conflict on the IMAD.WIDE (tools/micro/k1_loop.cu:
// +9-10 % evaluations per clock over the xl, xh, xh2, xl4 order).
struct __align__(16) XLimbs {
  uint32_t xh, xl, xl4, xh2;
};

// Exact 64-bit h mod m with a precomputed inv = floor((2^64-1)/m) (Barrett; corrected).
__device__ __forceinline__ uint64_t mod_m(uint64_t h, uint64_t m, uint64_t inv) {
  uint64_t q = __umul64hi(h, inv);
  uint64_t r = h - q * m;
  while (r >= m) r -= m;
  return r;
}

}  // namespace lb
