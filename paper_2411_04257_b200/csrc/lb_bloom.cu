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
//                contested: the arrival is queued (clist) and its position flagged in a small
//                contested-position summary bitmap (cb).
//   K5 resolve : queued contested probes enter E (earliest setter, atomicMin); first arrivals
//                whose summary bit is set enter E too; a first arrival with a clear bit is its
//                position's sole prober, so its band misses (E[p] = i).  Bands whose every
//                pre-unset probe is contested become candidates.
//   K6 verdict : candidate hit <=> E[p] < i for every pre-unset probe p.  (The sub-batch's E
//                buffer and summary are cleared by memsets queued before K3.)
// E holds the contested positions (and the rare summary collisions).  Its primary form Q is a compact open-addressed table of
// packed u64 slots ((band, position) << 22 | doc - i0; atomicMin keeps the earliest doc), two
// buffers alternating by sub-batch, small enough to stay L2-resident.  A key whose probe
// sequence in Q is full (64 slots) lives in the overflow table instead -- consistently, since
// slots are never freed within a sub-batch -- a worst-case-sized table keyed by
// (generation, band, position) holding (generation << 32 | ~doc) under atomicMax, which never
// needs clearing.  Probe positions are recomputed from the band hash in every kernel.
#include <cstdint>

#include "lb_internal.h"
#include "lb_probes.cuh"

namespace lb {

#ifndef BL_THREADS
#define BL_THREADS 128
#endif

__device__ __forceinline__ uint64_t eslot(uint64_t key, uint32_t log2cap) {
  return (key * 0x9E3779B97F4A7C15ull) >> (64 - log2cap);
}
constexpr uint64_t kQEmpty = ~0ull;
constexpr int kQProbe = 64;
__device__ __forceinline__ uint64_t qkey(uint32_t jl, uint64_t g) { return ((uint64_t)jl << 36) | g; }
__device__ __forceinline__ uint64_t qslot(const BloomParams& p, uint64_t key) {
  return (key * 0xD6E8FEB86659FD93ull) >> (64 - p.q_log2);
}

// Contested-position summary: one bit per hash(band, position), set for every contested probe
// (K4b).  A clear bit proves a position has a single prober in the sub-batch, so K5 decides most
// first arrivals without a Q lookup; a hash collision only costs a lookup.
__device__ __forceinline__ uint32_t cbit(const BloomParams& p, uint32_t jl, uint64_t g) {
  const uint32_t x = ((uint32_t)g ^ (uint32_t)(g >> 32)) * 0x9E3779B1u + jl * 0x85EBCA77u;
  return (x * 0xC2B2AE35u) >> (32 - p.cb_log2);
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

// K4: enter doc i as a setter of contested key (earliest wins).
__device__ void e_add(const BloomParams& p, uint64_t key, uint32_t i) {
  LB_ASSERT(i >= p.i0 && i - p.i0 < (1u << 22) && key < (1ull << 42));
  const uint64_t packed = (key << 22) | (uint64_t)(i - p.i0);
  const uint64_t mask = (1ull << p.q_log2) - 1;
  uint64_t s = qslot(p, key);
  for (int n = 0; n < kQProbe; n++, s = (s + 1) & mask) {
    LB_ASSERT(s <= mask);
    uint64_t cur = __ldcg(p.Q + s);
    if (cur == kQEmpty) {
      cur = atomicCAS((unsigned long long*)(p.Q + s), (unsigned long long)kQEmpty, (unsigned long long)packed);
      if (cur == kQEmpty) return;                       // claimed the slot
    }
    if ((cur >> 22) == key) {
      atomicMin((unsigned long long*)(p.Q + s), (unsigned long long)packed);
      return;
    }
  }
  e_upsert(p, (p.gen << 42) | key, (p.gen << 32) | (uint64_t)(~i));   // overflow table
}

// K6: earliest setter of key (batch document index), ~0u if absent.
__device__ uint32_t e_find(const BloomParams& p, uint64_t key) {
  const uint64_t mask = (1ull << p.q_log2) - 1;
  uint64_t s = qslot(p, key);
  for (int n = 0; n < kQProbe; n++, s = (s + 1) & mask) {
    const uint64_t cur = __ldcg(p.Q + s);
    if (cur == kQEmpty) return 0xFFFFFFFFu;
    if ((cur >> 22) == key) return p.i0 + (uint32_t)(cur & 0x3FFFFFull);
  }
  return e_lookup(p, (p.gen << 42) | key);
}

__device__ __forceinline__ uint64_t full_mask(uint32_t k) { return k == 64 ? ~0ull : ((1ull << k) - 1); }

// K3: probe positions + pre-sub-batch test.
template <int KT, typename PT, typename GEN>
__global__ void __launch_bounds__(BL_THREADS) k3_probe(const BloomParams p) {
  // grid (doc blocks, bands): blocks run x-fastest, so a wave works in one band's filter
  const uint32_t il = blockIdx.x * blockDim.x + threadIdx.x, jl = blockIdx.y;
  if (*p.err || il >= p.nsb) return;
  const uint32_t idx = jl * p.nsb + il, i = p.i0 + il;
  LB_ASSERT(jl < p.bl);
  const uint64_t bh = p.bh[(uint64_t)jl * p.bh_sj + (uint64_t)i * p.bh_si];
  const uint32_t* F = p.F + (uint64_t)jl * p.W;
  asm volatile("" : "+l"(F));   // opaque: keep the band's base in a register (no per-probe remat)
  uint64_t pre = 0;
  if constexpr (KT > 0) {
    const Probes<KT, PT, GEN> pr(p, bh, jl);
    uint32_t w[KT];
#pragma unroll
    for (int t = 0; t < KT; t++) w[t] = __ldcg(F + (pr.g[t] >> 5));   // all loads in flight
#pragma unroll
    for (int t = 0; t < KT; t++) pre |= (uint64_t)((w[t] >> (pr.g[t] & 31)) & 1u) << t;
  } else {
    GEN gen(p, bh, jl);
    for (uint32_t t = 0; t < p.k; t++) {
      const uint64_t g = gen.next();
      pre |= (uint64_t)((__ldcg(F + (g >> 5)) >> (g & 31)) & 1u) << t;
    }
  }
  p.st_pre[idx] = pre;
  if (pre == full_mask(p.k)) raise_dup(p.dup, i);
}

// K4: insert pre-unset probes; detect contested positions.
template <int KT, typename PT, typename GEN>
__global__ void __launch_bounds__(BL_THREADS) k4_insert(const BloomParams p) {
  const uint32_t il = blockIdx.x * blockDim.x + threadIdx.x, jl = blockIdx.y;
  if (*p.err || il >= p.nsb) return;
  const uint32_t idx = jl * p.nsb + il, i = p.i0 + il;
  const uint64_t pre = p.st_pre[idx];
  if (pre == full_mask(p.k)) return;
  LB_ASSERT(jl < p.bl);
  const uint64_t bh = p.bh[(uint64_t)jl * p.bh_sj + (uint64_t)i * p.bh_si];
  uint32_t* F = p.F + (uint64_t)jl * p.W;
  asm volatile("" : "+l"(F));
  uint64_t arr = 0;
  auto settle = [&](uint32_t t, uint64_t g, uint32_t old) {
    const uint32_t bit = 1u << (g & 31);
    if (old & bit) {                     // someone else set it in this sub-batch: contested
      // queued for K5 (entering E here would make whole warps wait on one lane's table walk)
      const uint64_t key = qkey(jl, g);
      const uint32_t c = atomicAdd(p.cand_count + 1, 1u);
      LB_ASSERT(c < (uint64_t)p.nsb * p.bl * p.k);
      p.clist[c] = (key << 22) | (uint64_t)(i - p.i0);
      const uint32_t h = cbit(p, jl, g);
      atomicOr(p.cb + (h >> 5), 1u << (h & 31));
    } else {
      arr |= 1ull << t;                  // first arrival
    }
  };
  if constexpr (KT > 0) {
    const Probes<KT, PT, GEN> pr(p, bh, jl);
    uint32_t old[KT];
#pragma unroll
    for (int t = 0; t < KT; t++)         // all atomics in flight before any result is used
      old[t] = ((pre >> t) & 1) ? 0u : atomicOr(F + (pr.g[t] >> 5), 1u << (pr.g[t] & 31));
#pragma unroll
    for (int t = 0; t < KT; t++)
      if (!((pre >> t) & 1)) settle(t, pr.g[t], old[t]);
  } else {
    GEN gen(p, bh, jl);
    for (uint32_t t = 0; t < p.k; t++) {
      const uint64_t g = gen.next();
      if (!((pre >> t) & 1)) settle(t, g, atomicOr(F + (g >> 5), 1u << (g & 31)));
    }
  }
  p.st_arr[idx] = arr;
}

// K5: (a) the contested probes K4 queued enter E; (b) every first arrival whose position is
// flagged in the contested-position summary enters E too (insert-or-min, so the order of (a)
// and (b) across threads does not matter; a summary collision only adds an entry that no other
// document reads and that makes its own band miss, as a sole prober must).  A first arrival
// with a clear summary bit is a sole prober: its band misses.  Bands whose first arrivals are
// all flagged become candidates for K6.
template <int KT, typename PT, typename GEN>
__global__ void __launch_bounds__(BL_THREADS) k5_resolve(const BloomParams p) {
  const uint32_t il = blockIdx.x * blockDim.x + threadIdx.x, jl = blockIdx.y;
  if (*p.err) return;
  {
    const uint32_t nc = p.cand_count[1];
    const uint32_t stride = gridDim.x * gridDim.y * blockDim.x;
    for (uint32_t c = (blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; c < nc; c += stride) {
      const uint64_t e = p.clist[c];
      e_add(p, e >> 22, p.i0 + (uint32_t)(e & 0x3FFFFFull));
    }
  }
  if (il >= p.nsb) return;
  const uint32_t idx = jl * p.nsb + il, i = p.i0 + il;
  const uint64_t pre = p.st_pre[idx];
  if (pre == full_mask(p.k)) return;
  const uint64_t arr = p.st_arr[idx];
  bool maybe = true;
  if (arr) {
    const uint64_t bh = p.bh[(uint64_t)jl * p.bh_sj + (uint64_t)i * p.bh_si];
    // (not early-exiting: every contested first arrival must join E for the other docs)
    // Flagged first arrivals are collected (up to 2 per lane) and entered in E after the scan
    // with the warp's lanes together, rather than one divergent table walk per probe index.
    uint64_t pk0 = 0, pk1 = 0;
    uint32_t np = 0;
    GEN gen(p, bh, jl);
    for (uint32_t t = 0; t < p.k; t++) {
      const uint64_t g = gen.next();
      if ((arr >> t) & 1) {
        const uint32_t h = cbit(p, jl, g);
        if (!((__ldg(p.cb + (h >> 5)) >> (h & 31)) & 1u)) {
          maybe = false;                                   // sole prober
        } else {                                           // (possibly) contested: join E
          const uint64_t key = qkey(jl, g);
          if (np == 0) pk0 = key;
          else if (np == 1) pk1 = key;
          else e_add(p, key, i);
          np++;
        }
      }
    }
    if (np > 0) e_add(p, pk0, i);
    if (np > 1) e_add(p, pk1, i);
  }
  if (maybe) {
    const uint32_t c = atomicAdd(p.cand_count, 1u);
    p.cand[c] = idx;
  }
}

// K6: verdict for candidate (doc, band) pairs.
template <int KT, typename PT, typename GEN>
__global__ void __launch_bounds__(BL_THREADS) k6_verdict(const BloomParams p) {
  if (*p.err) return;
  const uint32_t nc = *p.cand_count;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += stride) {
    const uint32_t idx = p.cand[c];
    LB_ASSERT(idx < (uint64_t)p.nsb * p.bl);
    const uint32_t jl = idx / p.nsb;
    const uint32_t i = p.i0 + idx % p.nsb;
    const uint64_t pre = p.st_pre[idx];
    GEN gen(p, p.bh[(uint64_t)jl * p.bh_sj + (uint64_t)i * p.bh_si], jl);
    bool hit = true;
    for (uint32_t t = 0; t < p.k && hit; t++) {
      const uint64_t g = gen.next();
      if (!((pre >> t) & 1)) hit = e_find(p, qkey(jl, g)) < i;
    }
    if (hit) raise_dup(p.dup, i);
  }

}

template <int KT, typename PT, typename GEN = ProbeGen>
static void launch_k(const BloomParams& p, dim3 grid, int sm_count, cudaStream_t s) {
  k3_probe<KT, PT, GEN><<<grid, BL_THREADS, 0, s>>>(p);
  k4_insert<KT, PT, GEN><<<grid, BL_THREADS, 0, s>>>(p);
  k5_resolve<KT, PT, GEN><<<grid, BL_THREADS, 0, s>>>(p);
  k6_verdict<KT, PT, GEN><<<(unsigned)sm_count * 2, BL_THREADS, 0, s>>>(p);
}

int launch_bloom_subbatch(const BloomParams& p, int sm_count, cudaStream_t s) {
  const dim3 grid((p.nsb + BL_THREADS - 1) / BL_THREADS, p.bl);   // (doc blocks, bands)
  cudaMemsetAsync(p.cand_count, 0, 2 * sizeof(uint32_t), s);   // candidates, contested probes
  cudaMemsetAsync(p.Q, 0xFF, 8ull << p.q_log2, s);   // this sub-batch's E: all slots empty
  cudaMemsetAsync(p.cb, 0, 1ull << (p.cb_log2 - 3), s);
  if (p.nb) {                                           // blocked variant
    if (p.k == 17) {
      if (p.m <= (1ull << 32)) launch_k<17, uint32_t, BlockedGen>(p, grid, sm_count, s);
      else launch_k<17, uint64_t, BlockedGen>(p, grid, sm_count, s);
    } else {
      launch_k<0, uint64_t, BlockedGen>(p, grid, sm_count, s);
    }
    return 4;
  }
  if (p.k == 17) {                                      // every BASELINE config (p = 1e-5)
    if (p.m <= (1ull << 32)) launch_k<17, uint32_t, ProbeGen32>(p, grid, sm_count, s);
    else launch_k<17, uint64_t>(p, grid, sm_count, s);   // C5: m = 23,962,645,944
  } else {
    launch_k<0, uint64_t>(p, grid, sm_count, s);
  }
  return 4;
}

}  // namespace lb
