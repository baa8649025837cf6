// lb_sweep.cu -- K7-K9: the window-sweep form of the per-band Bloom query-then-insert.
//
// Same semantics as K3-K6 (lb_bloom.cu; P:213 insert, P:218 query, S:390 query-then-insert,
// S:427 serial order): for band j and batch document i,
//   hit_j(i) = every probe bit g of BH_j(i) is set before i  <=>  F_pre[g] or E[g] < i,
// E[g] = the smallest batch document probing g (every document inserts unconditionally, DESIGN
// R12, so this lemma needs no iteration).  K3-K6 evaluate it with random accesses into HBM: a
// probe's 128-B line is fetched for the read and again for the atomic (246 DRAM bytes per probe
// measured at C5 geometry).  Here a batch is applied window by window instead:
//   K7 bin    : every probe (doc, band, t) becomes a record (g mod 2^wb) << 32 | (doc - i0) in
//               bin (band, g >> wb); fixed-capacity bins, one atomicAdd per record.
//   K7x exact : only if a bin overflowed (device flag): scan the bin counts, re-scatter exactly.
//   K8 sweep  : one CTA per non-empty window at a time: TMA bulk copy of the window's 2^wb bits
//               HBM -> shared memory, the lemma applied to all of the window's records in shared
//               memory (pre-read; atomicOr whose return value separates each position's first
//               arrival from the contested rest; the earliest setter of contested positions in a
//               small shared table), the window written back with one bulk store.  A record that
//               finds its bit not set before its document marks (doc, band) as a miss.
//   K9 verdict: doc i is a duplicate iff some owned band has no miss.
// Every filter line a batch touches crosses HBM once each way per sweep, plus 16 B per probe for
// its record: for dense batches (C5: 4M documents on 60 GB, ~2.9 probes per 128-B line) that is
// well under one random line fetch per probe.
#include <cstdint>

#include "lb_internal.h"
#include "lb_probes.cuh"

namespace lb {

#ifndef SW_BIN_THREADS
#define SW_BIN_THREADS 128
#endif

constexpr uint32_t kEcapLog2 = 10;                 // shared earliest-setter table: 1024 slots
constexpr uint32_t kEcap = 1u << kEcapLog2;        //   >= distinct keys of a bin of <= 1024 records
constexpr uint32_t kSummLog2 = 12;                 // contested-position summary: 4096 bits
constexpr uint64_t kEEmpty = ~0ull;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n"
      "SW_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra SW_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// L2 policies: the filter windows and records stream through once per sweep (evict first), so
// they do not push the per-document miss words (red.or from every SM) out of L2 (evict last).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// TMA bulk copies (no tensor map: 1-D, 16-B multiples)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_or_keep(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("red.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t sweep_full(uint32_t bl) { return bl >= 64 ? ~0ull : ((1ull << bl) - 1); }

// ------------------------------------------------------------------------------------------ K7

// Thread per (document, band), grid (document blocks, bands): blocks run x-fastest, so the GPU
// bins one band at a time and the bins receiving records at any moment are one band's (their
// partly written tail lines stay in L2).  (A band-fastest mapping, which would coalesce the
// band-hash reads of row-major input, spreads the tails over every band: 2x slower at C5.)
template <int KT, typename PT, typename GEN, bool EXACT>
__global__ void __launch_bounds__(SW_BIN_THREADS) k7_bin(const SweepParams p, uint32_t lo, uint32_t cnt) {
  const uint32_t jl = blockIdx.y;
  if (*p.g.err) return;
  if (EXACT && !*p.ovf) return;                              // (the common case: a few hundred CTAs exit)
  for (uint32_t il = blockIdx.x * blockDim.x + threadIdx.x; il < cnt; il += gridDim.x * blockDim.x) {
    const uint32_t i = lo + il;
    LB_ASSERT(i >= p.i0 && i - p.i0 < p.n && jl < p.g.bl);
    const uint64_t bh = p.g.bh[(uint64_t)jl * p.g.bh_sj + (uint64_t)i * p.g.bh_si];
    const uint64_t doc = i - p.i0;
    const uint64_t bin0 = (uint64_t)jl * p.nw;
    const uint64_t wmask = (1ull << p.wb) - 1;
    uint32_t* cur = EXACT ? p.cursor2 : p.cursor;
    auto place = [&](uint64_t g, uint32_t slot) -> bool {
      const uint64_t bin = bin0 + (g >> p.wb);
      const uint64_t r = ((g & wmask) << 32) | doc;
      if (EXACT) {
        p.rec[p.start[bin] + slot] = r;
        return true;
      }
      if (slot >= p.cap) return false;
      p.rec[bin * p.cap + slot] = r;
      return true;
    };
    bool over = false;
    if constexpr (KT > 0) {
      const Probes<KT, PT, GEN> pr(p.g, bh, jl);
      uint32_t slot[KT];
#pragma unroll
      for (int t = 0; t < KT; t++) slot[t] = atomicAdd(cur + bin0 + ((uint64_t)pr.g[t] >> p.wb), 1u);
#pragma unroll
      for (int t = 0; t < KT; t++) over |= !place(pr.g[t], slot[t]);
    } else {
      GEN gen(p.g, bh, jl);
      for (uint32_t t = 0; t < p.g.k; t++) {
        const uint64_t g = gen.next();
        over |= !place(g, atomicAdd(cur + bin0 + (g >> p.wb), 1u));
      }
    }
    if (over) *p.ovf = 1;
  }
}

// K7x scan (one CTA, exact layout only): start[b] = sum_{b' < b} cursor[b'], cursor2 = 0.
__global__ void __launch_bounds__(1024) k7_scan(const SweepParams p) {
  if (*p.g.err || !*p.ovf) return;
  __shared__ uint64_t part[1024];
  const uint32_t T = blockDim.x, t = threadIdx.x;
  const uint64_t nb = p.nbins, seg = (nb + T - 1) / T;
  const uint64_t b0 = umin64(nb, t * seg), b1 = umin64(nb, b0 + seg);
  uint64_t s = 0;
  for (uint64_t b = b0; b < b1; b++) s += p.cursor[b];
  part[t] = s;
  __syncthreads();
  for (uint32_t off = 1; off < T; off <<= 1) {    // inclusive Hillis-Steele scan of the parts
    const uint64_t v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint64_t acc = part[t] - s;                      // exclusive prefix of this segment
  for (uint64_t b = b0; b < b1; b++) {
    p.start[b] = acc;
    acc += p.cursor[b];
    p.cursor2[b] = 0;
  }
  if (t == T - 1) p.start[nb] = part[t];
}

// ------------------------------------------------------------------------------------------ K7a / K7b
// Scattering 8-byte records one by one runs at the L2's rate for uncoalesced stores (~54 G/s on
// B200, tools/micro/scatter.cu), whatever the bin count.  The two-level form writes every record
// as part of a run instead: K7a sorts a 512-document tile's 8704 records by coarse bucket
// (2^cb windows, <= 512 buckets per band) in shared memory and writes each bucket's run (~17
// records) at a position reserved with one atomicAdd; K7b takes one coarse bucket per CTA and
// re-sorts its records by window, 4096 at a time, into the window bins K8 reads.  Runs are padded
// with sentinel records (~0) to whole 32-byte sectors, so no store is a partial-sector write.

// Exclusive prefix sum over the block (blockDim.x <= 1024); *total = the sum.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wsum, uint32_t& total) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= (uint32_t)o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  total = wsum[nw - 1];
  const uint32_t ex = x - v + (w ? wsum[w - 1] : 0);
  __syncthreads();
  return ex;
}

constexpr uint64_t kSentinel = ~0ull;

// Shared-memory layout of K7a / K7b (dynamic): srt[cap_slots] u64 | skey[cap_slots] u16 |
// hist, lst, gb [nkeys] u32 | wsum[32] u32.
struct RunSmem {
  uint64_t* srt;
  uint16_t* skey;
  uint32_t *hist, *lst, *gb, *wsum;
  __device__ RunSmem(uint8_t* base, uint32_t slots, uint32_t nkeys) {
    srt = (uint64_t*)base;
    skey = (uint16_t*)(srt + slots);
    hist = (uint32_t*)(((uintptr_t)(skey + slots) + 15) & ~(uintptr_t)15);
    lst = hist + nkeys;
    gb = lst + nkeys;
    wsum = gb + nkeys;
  }
};
__host__ __device__ constexpr size_t run_smem_bytes(uint32_t slots, uint32_t nkeys) {
  return (size_t)slots * 10 + 16 + (size_t)nkeys * 12 + 32 * 4;
}

// After hist[] holds per-key counts: pad every key's run to whole sectors (4 records), reserve
// space with one atomicAdd on its cursor, lay the runs out in srt (padding = sentinels).
// Returns the number of slots used.  key k's cursor: cur(k).
template <typename CurF>
__device__ __forceinline__ uint32_t runs_reserve(RunSmem& sm, uint32_t nkeys, CurF cur) {
  const uint32_t tid = threadIdx.x;
  const uint32_t c = tid < nkeys ? sm.hist[tid] : 0, pc = (c + 3u) & ~3u;
  uint32_t total;
  const uint32_t ex = block_excl_scan(pc, sm.wsum, total);
  if (tid < nkeys) {
    sm.lst[tid] = ex;
    if (pc) sm.gb[tid] = atomicAdd(cur(tid), pc);
    for (uint32_t q = c; q < pc; q++) {
      sm.srt[ex + q] = kSentinel;
      sm.skey[ex + q] = (uint16_t)tid;
    }
  }
  return total;
}

template <typename PT, typename GEN>
__global__ void __launch_bounds__(kSweepTileDocs, 1) k7a_coarse(const SweepParams p, uint32_t lo, uint32_t cnt) {
  constexpr int KT = 17;
  extern __shared__ __align__(16) uint8_t dsm[];
  const uint32_t ncb = (uint32_t)p.ncb;
  RunSmem sm(dsm, kSweepTileDocs * KT + 3 * kSweepMaxCoarse, kSweepMaxCoarse);
  if (*p.g.err) return;
  const uint32_t tid = threadIdx.x, jl = blockIdx.y;
  const uint32_t il = blockIdx.x * kSweepTileDocs + tid;
  const bool valid = il < cnt;
  const uint32_t i = lo + il;
  if (tid < ncb) sm.hist[tid] = 0;
  __syncthreads();
  const uint32_t shift = p.wb + p.cb;
  uint32_t key[KT], rank[KT];
  uint64_t bh = 0;
  if (valid) {
    bh = p.g.bh[(uint64_t)jl * p.g.bh_sj + (uint64_t)i * p.g.bh_si];
    const Probes<KT, PT, GEN> pr(p.g, bh, jl);
#pragma unroll
    for (int t = 0; t < KT; t++) {
      key[t] = (uint32_t)((uint64_t)pr.g[t] >> shift);
      LB_ASSERT(key[t] < ncb);
      rank[t] = atomicAdd(&sm.hist[key[t]], 1u);
    }
  }
  __syncthreads();
  uint32_t* ccur = p.ccursor + (uint64_t)jl * ncb;
  const uint32_t total = runs_reserve(sm, ncb, [&](uint32_t k) { return ccur + k; });
  __syncthreads();
  if (valid) {
    const Probes<KT, PT, GEN> pr(p.g, bh, jl);
    const uint64_t pmask = (1ull << shift) - 1, doc = i - p.i0;
#pragma unroll
    for (int t = 0; t < KT; t++) {
      const uint32_t x = sm.lst[key[t]] + rank[t];
      sm.srt[x] = (((uint64_t)pr.g[t] & pmask) << 32) | doc;
      sm.skey[x] = (uint16_t)key[t];
    }
  }
  __syncthreads();
  uint64_t* out = p.crec + (uint64_t)jl * ncb * p.ccap;
  for (uint32_t x = tid; x < total; x += blockDim.x) {
    const uint32_t k = sm.skey[x];
    const uint32_t off = sm.gb[k] + (x - sm.lst[k]);
    if (off < p.ccap) out[(uint64_t)k * p.ccap + off] = sm.srt[x];
    else *p.ovf = 1;
  }
}

// K7b: one coarse bucket per CTA (grid: bl * ncb).  The CTA owns the bucket's windows, so their
// write positions are shared-memory counters (no global atomics); records are staged per window
// in shared memory and written 16 at a time -- whole 128-byte lines -- as they accumulate.
constexpr size_t k7b_smem_bytes() { return (size_t)kSweepMaxW * (kSweepStage * 8 + 12) + 16; }

__global__ void __launch_bounds__(kSweepBThreads) k7b_fine(const SweepParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  uint64_t(*stage)[kSweepStage] = (uint64_t(*)[kSweepStage])dsm;
  uint32_t* scnt = (uint32_t*)(dsm + (size_t)kSweepMaxW * kSweepStage * 8);
  uint32_t* gcur = scnt + kSweepMaxW;
  uint32_t* fullq = gcur + kSweepMaxW;                   // windows that reached 16 staged records
  uint32_t* nfull = fullq + kSweepMaxW;
  constexpr uint32_t RPT = kSweepChunk / kSweepBThreads;
  if (*p.g.err || *p.ovf) return;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint64_t cidx = blockIdx.x;                      // jl * ncb + coarse bucket
  const uint32_t jl = (uint32_t)(cidx / p.ncb), cbk = (uint32_t)(cidx - (uint64_t)jl * p.ncb);
  const uint32_t W = 1u << p.cb;
  const uint32_t nwin = (uint32_t)umin64(W, p.nw - (uint64_t)cbk * W);
  const uint32_t R = min(p.ccursor[cidx], p.ccap);
  const uint64_t* in = p.crec + cidx * p.ccap;
  const uint64_t bin0 = (uint64_t)jl * p.nw + (uint64_t)cbk * W;
  const uint64_t wmask = (1ull << p.wb) - 1;
  for (uint32_t w = tid; w < W; w += blockDim.x) scnt[w] = gcur[w] = 0;
  if (tid == 0) *nfull = 0;
  __syncthreads();
  bool over = false;
  auto out = [&](uint32_t w) { return p.rec + (bin0 + w) * p.cap; };
  for (uint32_t c0 = 0; c0 < R; c0 += kSweepChunk) {
    uint64_t r[RPT];
#pragma unroll
    for (uint32_t q = 0; q < RPT; q++) {
      const uint32_t x = c0 + tid + q * blockDim.x;
      r[q] = x < R ? __ldcs(in + x) : kSentinel;
    }
#pragma unroll
    for (uint32_t q = 0; q < RPT; q++) {
      if (r[q] == kSentinel) continue;
      const uint32_t pos = (uint32_t)(r[q] >> 32), w = pos >> p.wb;
      const uint64_t rec = (((uint64_t)pos & wmask) << 32) | (uint32_t)r[q];
      const uint32_t slot = atomicAdd(&scnt[w], 1u);
      if (slot < kSweepStage) {
        stage[w][slot] = rec;
        if (slot == 15) fullq[atomicAdd(nfull, 1u)] = w;   // a whole line is ready
      } else {                                             // staging full (rare): write it now
        const uint32_t o = atomicAdd(&gcur[w], 1u);
        if (o < p.cap) out(w)[o] = rec;
        else over = true;
      }
    }
    __syncthreads();
    const uint32_t nf = *nfull;
    __syncthreads();                                     // everyone has read the count
    if (tid == 0) *nfull = 0;                            // (appends resume after the next barrier)
    for (uint32_t fi = warp; fi < nf; fi += nwarps) {    // flush whole lines of the full windows
      const uint32_t w = fullq[fi];
      const uint32_t c = min(scnt[w], kSweepStage), full = c & ~15u;
      if (full) {
        const uint32_t base = gcur[w];
        if (base + full <= p.cap) {
          for (uint32_t x = lane; x < full; x += 32) out(w)[base + x] = stage[w][x];
        } else {
          over = true;
        }
        uint64_t keep = lane < c - full ? stage[w][full + lane] : 0;
        __syncwarp();
        if (lane < c - full) stage[w][lane] = keep;
        if (lane == 0) {
          gcur[w] = base + full;
          scnt[w] = c - full;
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  for (uint32_t w = warp; w < nwin; w += nwarps) {       // the rest, padded to whole sectors
    const uint32_t c = min(scnt[w], kSweepStage), pc = (c + 3u) & ~3u, base = gcur[w];
    if (base + pc <= p.cap) {
      if (lane < pc) out(w)[base + lane] = lane < c ? stage[w][lane] : kSentinel;
    } else if (c) {
      over = true;
    }
    if (lane == 0) p.cursor[bin0 + w] = base + pc;
  }
  if (over) *p.ovf = 1;
}

// Exact-layout fallback (any bin over capacity): recount every window bin from the band hashes.
__global__ void kf_zero(const SweepParams p) {
  if (!*p.ovf) return;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < p.nbins; b += (uint64_t)gridDim.x * blockDim.x)
    p.cursor[b] = 0;
}

template <int KT, typename PT, typename GEN>
__global__ void __launch_bounds__(SW_BIN_THREADS) kf_count(const SweepParams p, uint32_t lo, uint32_t cnt) {
  const uint32_t jl = blockIdx.y;
  if (*p.g.err || !*p.ovf) return;
  for (uint32_t il = blockIdx.x * blockDim.x + threadIdx.x; il < cnt; il += gridDim.x * blockDim.x) {
    const uint32_t i = lo + il;
    const uint64_t bh = p.g.bh[(uint64_t)jl * p.g.bh_sj + (uint64_t)i * p.g.bh_si];
    const uint64_t bin0 = (uint64_t)jl * p.nw;
    GEN gen(p.g, bh, jl);
    for (uint32_t t = 0; t < p.g.k; t++) atomicAdd(p.cursor + bin0 + (gen.next() >> p.wb), 1u);
  }
}

// Band hashes [n][bl] (row-major, query_insert_bands) -> columns [col0, col0 + n) of a band-major
// [bl][ld] buffer, so that the binning kernels read them coalesced.
__global__ void k7_transpose(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, uint32_t n, uint32_t bl,
                             uint64_t ld, uint64_t col0) {
  __shared__ uint64_t t[32][33];
  const uint32_t d0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t d = d0 + y, j = j0 + threadIdx.x;
    if (d < n && j < bl) t[y][threadIdx.x] = in[(uint64_t)d * bl + j];
  }
  __syncthreads();
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t j = j0 + y, d = d0 + threadIdx.x;
    if (d < n && j < bl) out[(uint64_t)j * ld + col0 + d] = t[threadIdx.x][y];
  }
}

int launch_transpose_bh(const uint64_t* in, uint64_t* out, uint32_t n, uint32_t bl, cudaStream_t s,
                        uint64_t ld, uint64_t col0) {
  k7_transpose<<<dim3((n + 31) / 32, (bl + 31) / 32), dim3(32, 8), 0, s>>>(in, out, n, bl, ld ? ld : n, col0);
  return 1;
}

// ------------------------------------------------------------------------------------------ K8

__device__ __forceinline__ uint32_t ehash(uint32_t gl) { return (gl * 0x9E3779B1u) >> (32 - kEcapLog2); }
__device__ __forceinline__ uint32_t shash(uint32_t gl) { return (gl * 0x85EBCA77u) >> (32 - kSummLog2); }

// earliest setter table in shared memory: slot = gl << 32 | doc, min doc per gl.  Returns the
// slot, which the inserting record empties again after the window (the table is never cleared
// wholesale: a window has only a handful of contested positions).
__device__ __forceinline__ uint32_t e_insert_min(uint64_t* etab, uint32_t gl, uint32_t doc) {
  const uint64_t packed = ((uint64_t)gl << 32) | doc;
  uint32_t s = ehash(gl);
  for (;;) {
    uint64_t cur = *(volatile uint64_t*)(etab + s);
    if (cur == kEEmpty) {
      cur = atomicCAS((unsigned long long*)(etab + s), (unsigned long long)kEEmpty, (unsigned long long)packed);
      if (cur == kEEmpty) return s;
    }
    if ((uint32_t)(cur >> 32) == gl) {
      atomicMin((unsigned long long*)(etab + s), (unsigned long long)packed);
      return s;
    }
    s = (s + 1) & (kEcap - 1);
  }
}
__device__ __forceinline__ uint32_t e_find_min(const uint64_t* etab, uint32_t gl) {
  uint32_t s = ehash(gl);
  for (;;) {
    const uint64_t cur = *(volatile const uint64_t*)(etab + s);
    if ((uint32_t)(cur >> 32) == gl) return (uint32_t)cur;
    LB_ASSERT(cur != kEEmpty);   // every caller inserted its own key
    s = (s + 1) & (kEcap - 1);
  }
}

// Shared memory of K8: two stages, each a window (2^wb bits) and its records (<= kSweepCapReg,
// fixed layout: prefetched by TMA with the window), then the earliest-setter table, the
// contested-position summary and the two stages' mbarriers.
__host__ __device__ constexpr uint32_t k8_rec_bytes() { return kSweepCapReg * 8; }
__host__ __device__ inline uint32_t k8_stage_bytes(uint32_t wb) { return ((1u << wb) >> 3) + k8_rec_bytes(); }

// Persistent CTAs stride over the window bins.  A ring of p.stages stages keeps the windows and
// records of the next stages-1 non-empty bins in flight (TMA bulk copies) while one is processed.
struct K8Meta {                      // per stage, written by thread 0 when it issues the copies
  uint64_t bin;                      // ~0: no more bins
  uint32_t* gwin;
  uint32_t jl, R, bytes, pad;
};

__global__ void __launch_bounds__(kSweepThreads, 4) k8_sweep(const SweepParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr uint32_t kMaxStages = 8;
  __shared__ K8Meta meta[kMaxStages];
  const uint32_t S = p.stages;
  const uint32_t wbytes_max = (1u << p.wb) >> 3, stage = k8_stage_bytes(p.wb);
  uint64_t* etab = (uint64_t*)(smem + S * stage);
  uint32_t* summ = (uint32_t*)(etab + kEcap);
  uint64_t* bar = (uint64_t*)(summ + (1u << kSummLog2) / 32);
  if (*p.g.err) return;
  const uint32_t tid = threadIdx.x, T = blockDim.x;
  const bool exact = *p.ovf != 0;
  const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last(),
                 pol_normal = policy_evict_normal();
  const uint64_t wwords = (uint64_t)1 << (p.wb - 5);
  uint32_t* eg = p.eg + (uint64_t)blockIdx.x * (1ull << p.wb);
  // records go through shared memory with the window when they can (fixed layout, register path)
  auto staged = [&](uint32_t R) { return !exact && R <= kSweepCapReg; };
  // Thread 0 walks this CTA's bins (bin = blockIdx.x + k * gridDim.x, band-major: band jl, window
  // w), skipping untouched windows, and issues each one's copies into the next free stage.
  uint64_t nb = blockIdx.x, nw_w = 0;
  uint32_t nb_jl = 0;
  if (tid == 0) {
    nb_jl = (uint32_t)(nb / p.nw);
    nw_w = nb - (uint64_t)nb_jl * p.nw;
  }
  auto advance = [&]() {                                     // thread 0: to the next non-empty bin
    while (nb < p.nbins && p.cursor[nb] == 0) {
      nb += gridDim.x;
      nw_w += gridDim.x;
      while (nw_w >= p.nw) { nw_w -= p.nw; nb_jl++; }
    }
  };
  auto issue = [&](uint32_t st) {                            // thread 0: bin nb -> stage st
    K8Meta m;
    m.bin = ~0ull;
    if (nb < p.nbins) {
      m.bin = nb;
      m.jl = nb_jl;
      m.gwin = p.g.F + (uint64_t)nb_jl * p.g.W + nw_w * wwords;
      m.bytes = (uint32_t)(umin64(wwords, p.g.W - nw_w * wwords) * 4);
      m.R = p.cursor[nb];
      const uint32_t rb = staged(m.R) ? ((m.R * 8 + 15) & ~15u) : 0;
      uint8_t* sb = smem + st * stage;
      mbar_expect_tx(bar + st, m.bytes + rb);
      bulk_load(sb, m.gwin, m.bytes, bar + st, pol_stream);
      if (rb) bulk_load(sb + wbytes_max, p.rec + nb * p.cap, rb, bar + st, pol_stream);
      nb += gridDim.x;
      nw_w += gridDim.x;
      while (nw_w >= p.nw) { nw_w -= p.nw; nb_jl++; }
    }
    meta[st] = m;
  };
  if (tid == 0) {
    for (uint32_t i = 0; i < S; i++) mbar_init(bar + i);
    for (uint32_t i = 0; i + 1 < S; i++) {                   // prologue: S - 1 stages in flight
      advance();
      issue(i);
    }
  }
  for (uint32_t q = tid; q < kEcap; q += T) etab[q] = kEEmpty;          // kept empty between windows
  for (uint32_t q = tid; q < (1u << kSummLog2) / 32; q += T) summ[q] = 0;
  __syncthreads();
  uint32_t parity_bits = 0;                                  // bit i: phase of stage i's barrier
  uint32_t st = 0;
  for (;;) {
    const K8Meta m = meta[st];
    if (m.bin == ~0ull) break;
    const uint32_t fill = st == 0 ? S - 1 : st - 1;          // the stage processed last iteration
    if (tid == 0) {
      bulk_wait_read_all();                                  // its window store has left smem
      advance();
      issue(fill);                                           // (published to all by the barriers below)
    }
    const uint32_t parity = (parity_bits >> st) & 1u;
    parity_bits ^= 1u << st;
    const uint64_t bin = m.bin;
    const uint32_t jl = m.jl, bytes = m.bytes, R = m.R;
    uint32_t* gwin = m.gwin;
    uint32_t* win = (uint32_t*)(smem + st * stage);
    const uint64_t* srec = (const uint64_t*)(smem + st * stage + wbytes_max);
    const uint64_t* rec = p.rec + (exact ? p.start[bin] : bin * p.cap);
    LB_ASSERT(exact || R <= p.cap);
    const uint64_t bitj = 1ull << jl;
    if (R <= kSweepCapReg) {
      // ---- records in registers, earliest setters in a shared table
      uint64_t r[kSweepRPT];
      if (!staged(R)) {
#pragma unroll
        for (int q = 0; q < kSweepRPT; q++) {
          const uint32_t idx = tid + q * T;
          r[q] = idx < R ? ld_stream(rec + idx, pol_stream) : ~0ull;
        }
      }
      mbar_wait(bar + st, parity);
      if (staged(R)) {
#pragma unroll
        for (int q = 0; q < kSweepRPT; q++) {
          const uint32_t idx = tid + q * T;
          r[q] = idx < R ? srec[idx] : ~0ull;
        }
      }
      uint32_t pre = 0, first = 0;                           // per-record flags (bit q)
      bool touched = false;                                  // this thread wrote etab / summ
      uint32_t es[kSweepRPT];                                // etab slot each record entered
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        if (r[q] == ~0ull) { pre |= 1u << q; continue; }     // (padding: treated as pre-set)
        const uint32_t gl = (uint32_t)(r[q] >> 32);
        LB_ASSERT(gl < (1u << p.wb));
        pre |= ((win[gl >> 5] >> (gl & 31)) & 1u) << q;
      }
      __syncthreads();                                       // every pre-read before any insert
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        if ((pre >> q) & 1) continue;
        const uint32_t gl = (uint32_t)(r[q] >> 32), doc = (uint32_t)r[q];
        const uint32_t bit = 1u << (gl & 31);
        const uint32_t old = atomicOr(win + (gl >> 5), bit);
        if (old & bit) {                                     // contested: another record set it
          const uint32_t h = shash(gl);
          atomicOr(summ + (h >> 5), 1u << (h & 31));
          es[q] = e_insert_min(etab, gl, doc);
          touched = true;
        } else {
          first |= 1u << q;
        }
      }
      fence_proxy_async();                                   // this thread's window writes -> async proxy
      __syncthreads();                                       // window final, summary complete
      if (tid == 0) bulk_store(gwin, win, bytes, pol_stream);
      uint32_t joined = 0;
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        if (!((first >> q) & 1)) continue;
        const uint32_t gl = (uint32_t)(r[q] >> 32);
        const uint32_t h = shash(gl);
        if ((summ[h >> 5] >> (h & 31)) & 1u) {               // (possibly) contested position
          es[q] = e_insert_min(etab, gl, (uint32_t)r[q]);
          joined |= 1u << q;
          touched = true;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        if ((pre >> q) & 1) continue;
        const uint32_t gl = (uint32_t)(r[q] >> 32), doc = (uint32_t)r[q];
        bool set_before = false;                             // sole prober: not set before
        if (!((first >> q) & 1) || ((joined >> q) & 1)) set_before = e_find_min(etab, gl) < doc;
        if (!set_before) red_or_keep(p.miss + doc, bitj, pol_keep);
      }
      // Every table read done.  This is also the iteration's last barrier: meta[] of the next
      // stages was published by the barriers above, and the next window's first table write comes
      // after its own first barrier, which every thread reaches only after emptying its entries.
      __syncthreads();
      if (touched) {                                         // empty what this thread filled
#pragma unroll
        for (int q = 0; q < kSweepRPT; q++) {
          if ((pre >> q) & 1) continue;
          if (((first >> q) & 1) && !((joined >> q) & 1)) continue;
          const uint32_t h = shash((uint32_t)(r[q] >> 32));
          summ[h >> 5] = 0;
          etab[es[q]] = kEEmpty;
        }
      }
    } else {
      // ---- a bin beyond kSweepCapReg records: records streamed from global memory, earliest
      // setters in this CTA's direct-mapped global array (one entry per window position)
      const uint32_t np = 1u << p.wb;
      for (uint32_t q = tid; q < np; q += T) eg[q] = 0xFFFFFFFFu;
      mbar_wait(bar + st, parity);
      uint64_t* wrec = p.rec + (exact ? p.start[bin] : bin * p.cap);
      for (uint32_t idx = tid; idx < R; idx += T) {
        const uint64_t rr = wrec[idx];
        if (rr == kSentinel) continue;                       // run padding
        const uint32_t gl = (uint32_t)(rr >> 32);
        if ((win[gl >> 5] >> (gl & 31)) & 1u) wrec[idx] = rr | (1ull << 63);   // pre-set
      }
      __syncthreads();
      for (uint32_t idx = tid; idx < R; idx += T) {
        const uint64_t rr = wrec[idx];
        if (rr >> 63) continue;                              // pre-set or padding
        const uint32_t gl = (uint32_t)(rr >> 32);
        atomicOr(win + (gl >> 5), 1u << (gl & 31));
        atomicMin(eg + gl, (uint32_t)rr);
      }
      __syncthreads();
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) bulk_store(gwin, win, bytes, pol_stream);
      for (uint32_t idx = tid; idx < R; idx += T) {
        const uint64_t rr = wrec[idx];
        if (rr >> 63) continue;
        const uint32_t gl = (uint32_t)(rr >> 32), doc = (uint32_t)rr;
        if (!(__ldcg(eg + gl) < doc)) atomicOr((unsigned long long*)(p.miss + doc), (unsigned long long)bitj);
      }
      __syncthreads();                                       // eg[] reads done before the next reset
    }
    // (no barrier here: thread 0 writes meta[fill] at the top of the next iteration only after
    // every thread has read meta[st] -- they all passed this window's barriers since)
    st = st + 1 == S ? 0 : st + 1;
  }
  if (tid == 0) bulk_wait_all();
}

// ------------------------------------------------------------------------------------------ K9

__global__ void __launch_bounds__(256) k9_verdict(const SweepParams p) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= p.n) return;
  const uint64_t ms = p.miss[d];
  p.miss[d] = 0;                                             // ready for the next sweep
  if (*p.g.err) return;
  if (ms != sweep_full(p.g.bl)) raise_dup(p.g.dup, p.i0 + d);
}

// ------------------------------------------------------------------------------------------ launchers

template <int KT, typename PT, typename GEN>
static void bin_launch(const SweepParams& p, uint32_t lo, uint32_t hi, bool exact, cudaStream_t s) {
  const uint32_t blocks = (hi - lo + SW_BIN_THREADS - 1) / SW_BIN_THREADS;
  const dim3 grid(exact ? (blocks < 64u ? blocks : 64u) : blocks, p.g.bl);   // exact: gated, grid-stride
  if (exact) k7_bin<KT, PT, GEN, true><<<grid, SW_BIN_THREADS, 0, s>>>(p, lo, hi - lo);
  else k7_bin<KT, PT, GEN, false><<<grid, SW_BIN_THREADS, 0, s>>>(p, lo, hi - lo);
}

static void bin_dispatch(const SweepParams& p, uint32_t lo, uint32_t hi, bool exact, cudaStream_t s) {
  if (p.g.nb) {
    if (p.g.k == 17) {
      if (p.g.m <= (1ull << 32)) bin_launch<17, uint32_t, BlockedGen>(p, lo, hi, exact, s);
      else bin_launch<17, uint64_t, BlockedGen>(p, lo, hi, exact, s);
    } else {
      bin_launch<0, uint64_t, BlockedGen>(p, lo, hi, exact, s);
    }
    return;
  }
  if (p.g.k == 17) {
    if (p.g.m <= (1ull << 32)) bin_launch<17, uint32_t, ProbeGen32>(p, lo, hi, exact, s);
    else bin_launch<17, uint64_t, ProbeGen>(p, lo, hi, exact, s);
  } else {
    bin_launch<0, uint64_t, ProbeGen>(p, lo, hi, exact, s);
  }
}

template <typename PT, typename GEN>
static void k7a_launch(const SweepParams& p, uint32_t lo, uint32_t hi, cudaStream_t s) {
  const size_t sm = run_smem_bytes(kSweepTileDocs * 17 + 3 * kSweepMaxCoarse, kSweepMaxCoarse);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k7a_coarse<PT, GEN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  const dim3 grid((hi - lo + kSweepTileDocs - 1) / kSweepTileDocs, p.g.bl);
  k7a_coarse<PT, GEN><<<grid, kSweepTileDocs, sm, s>>>(p, lo, hi - lo);
}

int launch_sweep_bin(const SweepParams& p, uint32_t lo, uint32_t hi, cudaStream_t s) {
  if (hi <= lo) return 0;
  if (p.two_level) {                                   // k = 17 (host-checked)
    if (p.g.nb) {
      if (p.g.m <= (1ull << 32)) k7a_launch<uint32_t, BlockedGen>(p, lo, hi, s);
      else k7a_launch<uint64_t, BlockedGen>(p, lo, hi, s);
    } else {
      if (p.g.m <= (1ull << 32)) k7a_launch<uint32_t, ProbeGen32>(p, lo, hi, s);
      else k7a_launch<uint64_t, ProbeGen>(p, lo, hi, s);
    }
    return 1;
  }
  bin_dispatch(p, lo, hi, false, s);
  return 1;
}

static void count_dispatch(const SweepParams& p, cudaStream_t s) {
  const uint32_t blocks = (p.n + SW_BIN_THREADS - 1) / SW_BIN_THREADS;
  const dim3 grid(blocks < 64u ? blocks : 64u, p.g.bl);      // gated on the overflow flag, grid-stride
  if (p.g.nb) kf_count<0, uint64_t, BlockedGen><<<grid, SW_BIN_THREADS, 0, s>>>(p, p.i0, p.n);
  else kf_count<0, uint64_t, ProbeGen><<<grid, SW_BIN_THREADS, 0, s>>>(p, p.i0, p.n);
}

static size_t sweep_smem(uint32_t wb, uint32_t stages) {
  return (size_t)stages * k8_stage_bytes(wb) + kEcap * 8 + (1u << kSummLog2) / 8 + 8 * 8;
}

// K8: persistent CTAs, as many per SM as fit (LSHBLOOM_K8_CTAS caps it), each with a ring of
// `stages` pipeline stages (LSHBLOOM_K8_STAGES, default 2).  The grid never exceeds what is
// resident at once (a second wave of persistent CTAs would serialise).
SweepLaunch sweep_launch_cfg(int sm_count, uint32_t wb) {
  static const int env_ctas = [] { const char* e = getenv("LSHBLOOM_K8_CTAS"); return e ? atoi(e) : 0; }();
  static const int env_st = [] { const char* e = getenv("LSHBLOOM_K8_STAGES"); return e ? atoi(e) : 0; }();
  static bool attr = false;
  if (!attr) {
    // (227 KB per block minus K8's static meta array)
    cudaFuncSetAttribute(k8_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
    attr = true;
  }
  uint32_t st = env_st ? (uint32_t)env_st : 2u;
  st = st < 2 ? 2 : st > 8 ? 8 : st;
  while (st > 2 && sweep_smem(wb, st) > 224 * 1024) st--;
  SweepLaunch c;
  c.stages = st;
  c.smem = sweep_smem(wb, st);
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k8_sweep, kSweepThreads, c.smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  // K8 is bound by its per-window barrier phases, not by HBM latency: more resident CTAs help up
  // to the three per SM the 16 KB windows allow (C5: 2 per SM 36.1 ms for K7b + K8; a staging
  // layout that fitted four was slower, 40.4 vs 36.6 ms per Bloom stage), deeper pipelines do
  // not (2 / 3 / 4 stages within 0.1 ms)
  if (env_ctas > 0 && env_ctas < per_sm) per_sm = env_ctas;
  c.grid = sm_count * per_sm;
  return c;
}

int sweep_grid(int sm_count, uint32_t wb) { return sweep_launch_cfg(sm_count, wb).grid; }

int launch_sweep_finish(const SweepParams& p_in, int grid_unused, cudaStream_t s) {
  (void)grid_unused;
  SweepParams p = p_in;
  const SweepLaunch lc = sweep_launch_cfg(0, p.wb);
  p.stages = lc.stages;
  int l = 0;
  if (p.two_level) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k7b_fine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k7b_smem_bytes());
      attr = true;
    }
    k7b_fine<<<(unsigned)(p.ncb * p.g.bl), kSweepBThreads, k7b_smem_bytes(), s>>>(p);
    l++;
  }
  // exact layout, only if a bin overflowed (every kernel checks the device flag first)
  kf_zero<<<256, 256, 0, s>>>(p);
  count_dispatch(p, s);
  k7_scan<<<1, 1024, 0, s>>>(p);
  bin_dispatch(p, p.i0, p.i0 + p.n, true, s);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k8_sweep<<<sweep_launch_cfg(sms, p.wb).grid, kSweepThreads, lc.smem, s>>>(p);
  k9_verdict<<<(p.n + 255) / 256, 256, 0, s>>>(p);
  return l + 6;
}

}  // namespace lb
