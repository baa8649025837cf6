// lb_bloom.cu -- K3-K6: per-band Bloom query-then-insert with exact stream-order semantics.
//
// Per band j and document i (P:213 insert, P:218 query; S:390 query-then-insert, S:427 serial):
//   hit_j(i) = all k probe bits of BH_j(i) were set before document i.
// Within a sub-batch processed in parallel, "before" means: set in the filter before the
// sub-batch (F_pre), or set by an earlier document of the sub-batch.  Because every document
// inserts unconditionally (DESIGN R12), bit p is set before i  <=>  F_pre[p] or E[p] < i, where
// E[p] is the smallest sub-batch document probing p.  Four launches per sub-batch:
//   K3 probe   : positions g_t = (h1 + t h2) mod m, read F_pre; all k set -> hit.
//   K4 insert  : atomicOr every pre-unset probe.  The one atomic that sees the bit clear is the
//                position's first arrival; every other arrival sees it set -> the position is
//                contested: mark it in T2 and atomicMax its earliest-setter entry in E.
//   K5 resolve : each first arrival looks its position up in T2 (then clears it): if contested
//                it adds itself to E; if not, it is the position's sole prober, so its band
//                misses (E[p] = i).  Bands whose every pre-unset probe is contested become
//                candidates.
//   K6 verdict : candidate hit <=> E[p] < i for every pre-unset probe p.
// E is an open-addressed table keyed by (generation, band, position) holding
// (generation << 32 | ~i) under atomicMax (newest generation wins, then the smallest i), so it
// never needs clearing; T2 is cleared bit by bit by the first arrivals in K5.
#include <cstdint>

#include "lb_internal.h"

namespace lb {

#define BL_THREADS 256

__device__ __forceinline__ uint64_t ekey_of(uint64_t gen, uint32_t jl, uint64_t g) {
  return (gen << 42) | ((uint64_t)jl << 36) | g;
}
__device__ __forceinline__ uint64_t eslot(uint64_t key, uint32_t log2cap) {
  return (key * 0x9E3779B97F4A7C15ull) >> (64 - log2cap);
}

// Insert-or-update: E[key] = max(E[key], tag).  Stale (older-generation) slots count as empty.
__device__ void e_upsert(const BloomParams& p, uint64_t key, uint64_t tag) {
  const uint64_t mask = (1ull << p.ecap_log2) - 1;
  uint64_t s = eslot(key, p.ecap_log2);
  uint64_t cur = __ldcg(p.ekey + s);   // L2 (the table is written by other SMs' atomics)
  for (;;) {
    if (cur == key) { atomicMax((unsigned long long*)&p.eval[s], (unsigned long long)tag); return; }
    if ((cur >> 42) != p.gen) {
      const uint64_t prev = atomicCAS((unsigned long long*)&p.ekey[s], (unsigned long long)cur,
                                      (unsigned long long)key);
      if (prev == cur || prev == key) {
        atomicMax((unsigned long long*)&p.eval[s], (unsigned long long)tag);
        return;
      }
      cur = prev;  // someone else claimed this slot: re-examine what they wrote
      continue;
    }
    s = (s + 1) & mask;
    cur = __ldcg(p.ekey + s);
  }
}

// Earliest setter of key in this generation, or ~0u if absent.
__device__ uint32_t e_lookup(const BloomParams& p, uint64_t key) {
  const uint64_t mask = (1ull << p.ecap_log2) - 1;
  uint64_t s = eslot(key, p.ecap_log2);
  for (;;) {
    const uint64_t cur = __ldcg(p.ekey + s);
    if (cur == key) {
      const uint64_t v = __ldcg(p.eval + s);
      return ((v >> 32) == p.gen) ? ~(uint32_t)v : 0xFFFFFFFFu;
    }
    if ((cur >> 42) != p.gen) return 0xFFFFFFFFu;
    s = (s + 1) & mask;
  }
}

// K3: probe positions + pre-sub-batch test.
__global__ void __launch_bounds__(BL_THREADS) k3_probe(const BloomParams p) {
  const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (*p.err || idx >= (uint64_t)p.nsb * p.bl) return;
  const uint32_t jl = (uint32_t)(idx % p.bl);
  const uint32_t i = p.i0 + (uint32_t)(idx / p.bl);
  const uint64_t bh = p.bh[(uint64_t)i * p.bl + jl];
  const uint64_t h1 = mix64(bh ^ p.s1[jl]);
  const uint64_t h2 = mix64(bh ^ p.s2[jl]) | 1ull;
  const uint64_t g0 = mod_m(h1, p.m, p.m_inv);
  const uint64_t dl = mod_m(h2, p.m, p.m_inv);
  const uint32_t* F = p.F + (uint64_t)jl * p.W;
  uint64_t pre = 0, g = g0;
#pragma unroll 4
  for (uint32_t t = 0; t < p.k; t++) {
    const uint32_t w = __ldcg(F + (g >> 5));
    pre |= (uint64_t)((w >> (g & 31)) & 1u) << t;
    g += dl;
    g = g >= p.m ? g - p.m : g;
  }
  p.st_g0[idx] = g0;
  p.st_d[idx] = dl;
  p.st_pre[idx] = pre;
  const uint64_t full = (p.k == 64) ? ~0ull : ((1ull << p.k) - 1);
  if (pre == full) p.dup[i] = 1;
}

// K4: insert pre-unset probes; detect contested positions.
__global__ void __launch_bounds__(BL_THREADS) k4_insert(const BloomParams p) {
  const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (*p.err || idx >= (uint64_t)p.nsb * p.bl) return;
  const uint64_t full = (p.k == 64) ? ~0ull : ((1ull << p.k) - 1);
  const uint64_t pre = p.st_pre[idx];
  if (pre == full) return;
  const uint32_t jl = (uint32_t)(idx % p.bl);
  const uint32_t i = p.i0 + (uint32_t)(idx / p.bl);
  uint32_t* F = p.F + (uint64_t)jl * p.W;
  uint32_t* T2 = p.T2 + (uint64_t)jl * p.W;
  const uint64_t dl = p.st_d[idx];
  const uint64_t tag = (p.gen << 32) | (uint64_t)(~i);
  uint64_t g = p.st_g0[idx], arr = 0;
  for (uint32_t t = 0; t < p.k; t++) {
    if (!((pre >> t) & 1)) {
      const uint32_t bit = 1u << (g & 31);
      const uint32_t old = atomicOr(F + (g >> 5), bit);
      if (old & bit) {
        atomicOr(T2 + (g >> 5), bit);
        e_upsert(p, ekey_of(p.gen, jl, g), tag);
      } else {
        arr |= 1ull << t;
      }
    }
    g += dl;
    g = g >= p.m ? g - p.m : g;
  }
  p.st_arr[idx] = arr;
}

// K5: first arrivals consult T2; contested ones join E; sole probers make the band miss.
__global__ void __launch_bounds__(BL_THREADS) k5_resolve(const BloomParams p) {
  const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (*p.err || idx >= (uint64_t)p.nsb * p.bl) return;
  const uint64_t full = (p.k == 64) ? ~0ull : ((1ull << p.k) - 1);
  const uint64_t pre = p.st_pre[idx];
  if (pre == full) return;
  const uint64_t arr = p.st_arr[idx];
  const uint32_t jl = (uint32_t)(idx % p.bl);
  const uint32_t i = p.i0 + (uint32_t)(idx / p.bl);
  uint32_t* T2 = p.T2 + (uint64_t)jl * p.W;
  bool maybe = true;
  if (arr) {
    const uint64_t dl = p.st_d[idx];
    const uint64_t tag = (p.gen << 32) | (uint64_t)(~i);
    uint64_t g = p.st_g0[idx];
    for (uint32_t t = 0; t < p.k; t++) {
      if ((arr >> t) & 1) {
        const uint32_t bit = 1u << (g & 31);
        if (__ldcg(T2 + (g >> 5)) & bit) {
          e_upsert(p, ekey_of(p.gen, jl, g), tag);
          atomicAnd(T2 + (g >> 5), ~bit);
        } else {
          maybe = false;   // only this document probes g: not set before it
        }
      }
      g += dl;
      g = g >= p.m ? g - p.m : g;
    }
  }
  if (maybe) {
    const uint32_t c = atomicAdd(p.cand_count, 1u);
    p.cand[c] = (uint32_t)idx;
  }
}

// K6: verdict for candidate (doc, band) pairs.
__global__ void __launch_bounds__(BL_THREADS) k6_verdict(const BloomParams p) {
  if (*p.err) return;
  const uint32_t nc = *p.cand_count;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    const uint32_t idx = p.cand[c];
    const uint32_t jl = idx % p.bl;
    const uint32_t i = p.i0 + idx / p.bl;
    const uint64_t pre = p.st_pre[idx];
    const uint64_t dl = p.st_d[idx];
    uint64_t g = p.st_g0[idx];
    bool hit = true;
    for (uint32_t t = 0; t < p.k && hit; t++) {
      if (!((pre >> t) & 1)) hit = e_lookup(p, ekey_of(p.gen, jl, g)) < i;
      g += dl;
      g = g >= p.m ? g - p.m : g;
    }
    if (hit) p.dup[i] = 1;
  }
}

int launch_bloom_subbatch(const BloomParams& p, int sm_count, cudaStream_t s) {
  const uint64_t n = (uint64_t)p.nsb * p.bl;
  const unsigned grid = (unsigned)((n + BL_THREADS - 1) / BL_THREADS);
  cudaMemsetAsync(p.cand_count, 0, sizeof(uint32_t), s);
  k3_probe<<<grid, BL_THREADS, 0, s>>>(p);
  k4_insert<<<grid, BL_THREADS, 0, s>>>(p);
  k5_resolve<<<grid, BL_THREADS, 0, s>>>(p);
  k6_verdict<<<(unsigned)sm_count, BL_THREADS, 0, s>>>(p);
  return 4;
}

}  // namespace lb
