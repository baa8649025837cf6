// lb_probes.cuh -- probe positions of a band hash (shared by the random-access Bloom kernels,
// lb_bloom.cu, and the window-sweep kernels, lb_sweep.cu).
#pragma once
#include <cstdint>

#include "lb_internal.h"

namespace lb {

// Probe positions of one band hash: g_t = (h1 + t h2) mod m computed as g_0 = h1 mod m,
// g_{t+1} = g_t + (h2 mod m) - m [if >= m]  (exact; no 2^64 wrap, DESIGN R10).
// KT > 0: k = KT known at compile time, positions in registers; KT = 0: runtime k <= 64.
struct ProbeGen {   // sequential positions (any k)
  uint64_t x, dl, m;
  __device__ __forceinline__ ProbeGen(const BloomParams& p, uint64_t bh, uint32_t jl) {
    const uint64_t h1 = mix64(bh ^ p.s1[jl]);
    const uint64_t h2 = mix64(bh ^ p.s2[jl]) | 1ull;
    x = mod_m(h1, p.m, p.m_inv);
    dl = mod_m(h2, p.m, p.m_inv);
    m = p.m;
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t g = x;
    LB_ASSERT(g < m);
    x += dl;
    x = x >= m ? x - m : x;
    return g;
  }
};

// The same progression in 32-bit arithmetic when m <= 2^32 (every config but C5): with
// md = m - (h2 mod m), g + (h2 mod m) mod m = (g < md) ? g + dl : g - md  -- no overflow.
struct ProbeGen32 {
  uint32_t x, dl, md;
  __device__ __forceinline__ ProbeGen32(const BloomParams& p, uint64_t bh, uint32_t jl) {
    const uint64_t h1 = mix64(bh ^ p.s1[jl]);
    const uint64_t h2 = mix64(bh ^ p.s2[jl]) | 1ull;
    x = (uint32_t)mod_m(h1, p.m, p.m_inv);
    dl = (uint32_t)mod_m(h2, p.m, p.m_inv);
    md = (uint32_t)(p.m - dl);
  }
  __device__ __forceinline__ uint64_t next() {
    const uint32_t g = x;
    x = g < md ? g + dl : g - md;
    return g;
  }
};

// Blocked variant (index_kind = LSHBLOOM_INDEX_BLOCKED): all k probes of a
// band hash in one 1024-bit block (one 128-byte line, the unit B200 moves per random access):
// block = h1 mod nb; offset_t = 10-bit field (t mod 6) of mix64(h2 + t / 6).
struct BlockedGen {
  uint64_t base, h2, w;
  uint32_t t;
  __device__ __forceinline__ BlockedGen(const BloomParams& p, uint64_t bh, uint32_t jl) {
    const uint64_t h1 = mix64(bh ^ p.s1[jl]);
    h2 = mix64(bh ^ p.s2[jl]) | 1ull;
    base = mod_m(h1, p.nb, p.nb_inv) << 10;
    t = 0;
    w = 0;
  }
  __device__ __forceinline__ uint64_t next() {
    const uint32_t f = t % 6;
    if (f == 0) w = mix64(h2 + t / 6);
    t++;
    LB_ASSERT(base + ((w >> (10 * f)) & 1023u) < (uint64_t)1024 * 0x7FFFFFFFFull);
    return base + ((w >> (10 * f)) & 1023u);
  }
};

template <int KT, typename PT, typename GEN = ProbeGen>   // KT > 0: all k positions in registers
struct Probes {                                           // (PT = u32 when m <= 2^32)
  PT g[KT];
  __device__ __forceinline__ Probes(const BloomParams& p, uint64_t bh, uint32_t jl) {
    GEN gen(p, bh, jl);
#pragma unroll
    for (int t = 0; t < KT; t++) g[t] = (PT)gen.next();
  }
};

}  // namespace lb
