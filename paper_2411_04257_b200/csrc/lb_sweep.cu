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

constexpr uint32_t kEcapLog2 = 11;                 // shared earliest-setter table: 2048 slots
constexpr uint32_t kEcap = 1u << kEcapLog2;        //   >= distinct keys of a bin of <= 2048 records
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
// TMA bulk copies (no tensor map: 1-D, 16-B multiples)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t sweep_full(uint32_t bl) { return bl >= 64 ? ~0ull : ((1ull << bl) - 1); }

// ------------------------------------------------------------------------------------------ K7

template <int KT, typename PT, typename GEN, bool EXACT>
__global__ void __launch_bounds__(SW_BIN_THREADS) k7_bin(const SweepParams p, uint32_t lo, uint32_t cnt) {
  const uint32_t il = blockIdx.x * blockDim.x + threadIdx.x, jl = blockIdx.y;
  if (*p.g.err || il >= cnt) return;
  if (EXACT && !*p.ovf) return;
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

// ------------------------------------------------------------------------------------------ K8

__device__ __forceinline__ uint32_t ehash(uint32_t gl) { return (gl * 0x9E3779B1u) >> (32 - kEcapLog2); }
__device__ __forceinline__ uint32_t shash(uint32_t gl) { return (gl * 0x85EBCA77u) >> (32 - kSummLog2); }

// earliest setter table in shared memory: slot = gl << 32 | doc, min doc per gl
__device__ __forceinline__ void e_insert_min(uint64_t* etab, uint32_t gl, uint32_t doc) {
  const uint64_t packed = ((uint64_t)gl << 32) | doc;
  uint32_t s = ehash(gl);
  for (;;) {
    uint64_t cur = *(volatile uint64_t*)(etab + s);
    if (cur == kEEmpty) {
      cur = atomicCAS((unsigned long long*)(etab + s), (unsigned long long)kEEmpty, (unsigned long long)packed);
      if (cur == kEEmpty) return;
    }
    if ((uint32_t)(cur >> 32) == gl) {
      atomicMin((unsigned long long*)(etab + s), (unsigned long long)packed);
      return;
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

__global__ void __launch_bounds__(kSweepThreads, 2) k8_sweep(const SweepParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t wbytes_max = (1u << p.wb) >> 3;
  uint32_t* win = (uint32_t*)smem;
  uint64_t* etab = (uint64_t*)(smem + wbytes_max);
  uint32_t* summ = (uint32_t*)(etab + kEcap);
  uint64_t* bar = (uint64_t*)(summ + (1u << kSummLog2) / 32);
  if (*p.g.err) return;
  const uint32_t tid = threadIdx.x, T = blockDim.x;
  const bool exact = *p.ovf != 0;
  if (tid == 0) mbar_init(bar);
  __syncthreads();
  uint32_t parity = 0;
  const uint64_t wwords = (uint64_t)1 << (p.wb - 5);
  uint32_t* eg = p.eg + (uint64_t)blockIdx.x * (1ull << p.wb);
  for (uint64_t bin = blockIdx.x; bin < p.nbins; bin += gridDim.x) {
    const uint32_t R = p.cursor[bin];
    if (R == 0) continue;                                    // window untouched by this batch
    const uint32_t jl = (uint32_t)(bin / p.nw);
    const uint64_t w = bin - (uint64_t)jl * p.nw;
    uint32_t* gwin = p.g.F + (uint64_t)jl * p.g.W + w * wwords;
    const uint32_t bytes = (uint32_t)(umin64(wwords, p.g.W - w * wwords) * 4);
    const uint64_t* rec = p.rec + (exact ? p.start[bin] : bin * p.cap);
    LB_ASSERT(exact || R <= p.cap);
    if (tid == 0) {
      bulk_wait_read_all();                                  // the last store has left smem
      mbar_expect_tx(bar, bytes);
      bulk_load(win, gwin, bytes, bar);
    }
    const uint64_t bitj = 1ull << jl;
    if (R <= kSweepCapReg) {
      // ---- records in registers, earliest setters in a shared table
      uint64_t r[kSweepRPT];
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        const uint32_t idx = tid + q * T;
        r[q] = idx < R ? __ldcs(rec + idx) : ~0ull;
      }
      for (uint32_t s = tid; s < kEcap; s += T) etab[s] = kEEmpty;
      for (uint32_t s = tid; s < (1u << kSummLog2) / 32; s += T) summ[s] = 0;
      mbar_wait(bar, parity);
      parity ^= 1;
      uint32_t pre = 0, first = 0;                           // per-record flags (bit q)
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
          e_insert_min(etab, gl, doc);
        } else {
          first |= 1u << q;
        }
      }
      __syncthreads();                                       // window final, summary complete
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) bulk_store(gwin, win, bytes);
      uint32_t joined = 0;
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        if (!((first >> q) & 1)) continue;
        const uint32_t gl = (uint32_t)(r[q] >> 32);
        const uint32_t h = shash(gl);
        if ((summ[h >> 5] >> (h & 31)) & 1u) {               // (possibly) contested position
          e_insert_min(etab, gl, (uint32_t)r[q]);
          joined |= 1u << q;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kSweepRPT; q++) {
        if ((pre >> q) & 1) continue;
        const uint32_t gl = (uint32_t)(r[q] >> 32), doc = (uint32_t)r[q];
        bool set_before = false;                             // sole prober: not set before
        if (!((first >> q) & 1) || ((joined >> q) & 1)) set_before = e_find_min(etab, gl) < doc;
        if (!set_before) atomicOr((unsigned long long*)(p.miss + doc), (unsigned long long)bitj);
      }
      __syncthreads();                                       // table reads done before the next clear
    } else {
      // ---- a bin beyond 2048 records (exact layout only): records streamed from global memory,
      // earliest setters in this CTA's direct-mapped global array (one entry per window position)
      const uint32_t np = 1u << p.wb;
      for (uint32_t s = tid; s < np; s += T) eg[s] = 0xFFFFFFFFu;
      mbar_wait(bar, parity);
      parity ^= 1;
      uint64_t* wrec = p.rec + (exact ? p.start[bin] : bin * p.cap);
      for (uint32_t idx = tid; idx < R; idx += T) {
        const uint64_t rr = wrec[idx];
        const uint32_t gl = (uint32_t)(rr >> 32);
        if ((win[gl >> 5] >> (gl & 31)) & 1u) wrec[idx] = rr | (1ull << 63);   // pre-set
      }
      __syncthreads();
      for (uint32_t idx = tid; idx < R; idx += T) {
        const uint64_t rr = wrec[idx];
        if (rr >> 63) continue;
        const uint32_t gl = (uint32_t)(rr >> 32);
        atomicOr(win + (gl >> 5), 1u << (gl & 31));
        atomicMin(eg + gl, (uint32_t)rr);
      }
      __syncthreads();
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) bulk_store(gwin, win, bytes);
      for (uint32_t idx = tid; idx < R; idx += T) {
        const uint64_t rr = wrec[idx];
        if (rr >> 63) continue;
        const uint32_t gl = (uint32_t)(rr >> 32), doc = (uint32_t)rr;
        if (!(__ldcg(eg + gl) < doc)) atomicOr((unsigned long long*)(p.miss + doc), (unsigned long long)bitj);
      }
      __syncthreads();
    }
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
  const dim3 grid((hi - lo + SW_BIN_THREADS - 1) / SW_BIN_THREADS, p.g.bl);
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

int launch_sweep_bin(const SweepParams& p, uint32_t lo, uint32_t hi, cudaStream_t s) {
  if (hi <= lo) return 0;
  bin_dispatch(p, lo, hi, false, s);
  return 1;
}

static size_t sweep_smem(uint32_t wb) {
  return ((size_t)1 << wb) / 8 + kEcap * 8 + (1u << kSummLog2) / 8 + 16;
}

int sweep_grid(int sm_count, uint32_t wb) {
  const size_t sm = sweep_smem(wb);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k8_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sweep_smem(19));
    attr = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k8_sweep, kSweepThreads, sm) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return sm_count * per_sm;
}

int launch_sweep_finish(const SweepParams& p, int grid, cudaStream_t s) {
  k7_scan<<<1, 1024, 0, s>>>(p);
  bin_dispatch(p, p.i0, p.i0 + p.n, true, s);
  k8_sweep<<<grid, kSweepThreads, sweep_smem(p.wb), s>>>(p);
  k9_verdict<<<(p.n + 255) / 256, 256, 0, s>>>(p);
  return 4;
}

}  // namespace lb
