// lb_minhash.cu -- K1: shingle fingerprints + MinHash + band-hash epilogue (sm_100a).
//
// One warp per document (persistent warps pull documents from an atomic counter).  Lanes own
// permutations p = lane + 32 q (q < NPL): their coefficients stay in registers for the whole
// launch, the running minima too, so no cross-lane reduction is ever needed.  The warp walks
// the document's shingles in chunks of 32: lane l fingerprints shingle s0 + l (DESIGN
// R1) and parks x = fp mod P, pre-split into 30/31-bit limbs, in shared memory; then every
// lane evaluates its NPL permutations on each of the 32 shingles (a warp-uniform shared-memory
// broadcast per shingle).
//
// The eval (DESIGN R3/R4):  y = ((a x + b) mod P) mod 2^32, exact.
//   a = a1 2^31 + a0, x = xh 2^30 + xl  =>  a x = a1 xh 2^61 + 2^30 (a0 xh + 2 a1 xl) + a0 xl
//   2^61 = 1 (mod P)  =>  a x + b + 1 = A + 2^30 G (mod P),
//       A = a0 xl + a1 xh + (b+1)            (< 3 2^61, two IMAD.WIDE with 64-bit addends)
//       G' = 2G = a0 (2 xh) + a1 (4 xl)      (< 2^64,   two IMAD.WIDE)
//   2^30 G = 2^29 G' = G'_hi 2^61 + G'_lo 2^29 = G'_hi + G'_lo 2^29 (mod P)
//   S' = A + G'_hi + G'_lo 2^29  (< 2^63 + 2^32),  S' = S + 1 with S = a x + b (mod P)
//   q = floor(S / P) = (S' + (S' >> 61)) >> 61,   y = low32(S - q P) = low32(S') - 1 + q.
// Four 32x32->64 multiplies (the minimum for a 61x61-bit product; IMAD.WIDE issues at 1/4 rate)
// plus ~8 ALU ops; tools/micro measured the per-opcode rates.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "lb_internal.h"

namespace lb {

#ifndef K1_THREADS
#define K1_THREADS 256
#endif
#ifndef LB_K1_MINB
#define LB_K1_MINB 1
#endif
#ifndef LB_UNR4
#define LB_UNR4 4
#endif
#define K1_WARPS (K1_THREADS / 32)

// Coefficients: a = a1 2^31 + a0 (a0 < 2^31, a1 < 2^30), b = b1 2^32 + b0 (b < P), stored per
// permutation as PermCoef{a0, a1, b1, b0}; shingle x = xh 2^30 + xl with xh2 = 2 xh, xl4 = 4 xl.
//   a x = a1 xh 2^61 + 2^30 (a0 xh + 2 a1 xl) + a0 xl,   2^61 = 1 (mod P)
//   A = a0 xl + a1 xh + b (< 3 2^61),  G = a0 xh2 + a1 xl4 (< 2^64),  2^30 (G/2) = G_hi + G_lo 2^29
//   S = A + G_hi + G_lo 2^29 = a x + b (mod P),  0 <= S < 2^63 + 2^61
// and y = low32(S mod P) = low32(S) + q with q = floor(S / P) <= 4 (low32(q P) = -q).

// Exact: q = (S' + (S' >> 61)) >> 61 with S' = S + 1 (proved in DESIGN.md), carries included.
__device__ __forceinline__ uint32_t eval_exact(const PermCoef& c, const XLimbs& x) {
  uint32_t y;
  asm("{\n\t"
      ".reg .u64 A, G, B;\n\t"
      ".reg .u32 s0, s1, g0, g1, t1, t2, q;\n\t"
      "mov.b64 B, {%3, %4};\n\t"
      "add.u64 B, B, 1;\n\t"              // b + 1
      "mad.wide.u32 A, %1, %5, B;\n\t"
      "mad.wide.u32 A, %2, %6, A;\n\t"
      "mul.wide.u32 G, %1, %7;\n\t"
      "mad.wide.u32 G, %2, %8, G;\n\t"
      "mov.b64 {s0, s1}, A;\n\t"
      "mov.b64 {g0, g1}, G;\n\t"
      "shl.b32 t1, g0, 29;\n\t"
      "shr.u32 t2, g0, 3;\n\t"
      "add.cc.u32 s0, s0, t1;\n\t"
      "addc.u32 s1, s1, t2;\n\t"
      "add.cc.u32 s0, s0, g1;\n\t"
      "addc.u32 s1, s1, 0;\n\t"           // S' = s1:s0 = S + 1
      "shr.u32 q, s1, 29;\n\t"
      "add.cc.u32 t1, s0, q;\n\t"
      "addc.u32 t2, s1, 0;\n\t"           // W = S' + (S' >> 61)
      "shr.u32 q, t2, 29;\n\t"            // q = W >> 61 = floor(S / P)
      "add.u32 s0, s0, q;\n\t"
      "sub.u32 %0, s0, 1;\n\t"            // low32(S' - 1) + q
      "}"
      : "=r"(y)
      : "r"(c.a0), "r"(c.a1), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
  return y;
}

// Carry-free: s0 = low32(S) is exact without carries; the high word is taken without the
// carries out of the low word (s1a = A_hi + (G_lo >> 3), at most 2 below the true high word), and
// q is taken as s1a >> 29.  This equals floor(S / P) unless bits 32..60 of S are within 5 of
// all-ones, i.e. unless (s1a | 0xE0000000) >= 0xFFFFFFFB (p ~ 1e-8 per evaluation); the running
// max of that word is returned in fmax and a flagged document is recomputed with eval_exact.
// No unflagged mismatch against big integers on 4e5 random and adversarial triples.
__device__ __forceinline__ uint32_t eval_fast(const PermCoef& c, const XLimbs& x, uint32_t& f) {
  uint32_t y;
  asm("{\n\t"
      ".reg .u64 A, G, B;\n\t"
      ".reg .u32 s0, s1, g0, g1, t1, t2;\n\t"
      "mov.b64 B, {%3, %4};\n\t"
      "mad.wide.u32 A, %2, %5, B;\n\t"    // a0*xl + b
      "mad.wide.u32 A, %6, %7, A;\n\t"    // + a1*xh
      "mul.wide.u32 G, %2, %8;\n\t"       // a0*(2xh)
      "mad.wide.u32 G, %6, %9, G;\n\t"    // + a1*(4xl)
      "mov.b64 {s0, s1}, A;\n\t"
      "mov.b64 {g0, g1}, G;\n\t"
      "shl.b32 t1, g0, 29;\n\t"
      "shr.u32 t2, g0, 3;\n\t"
      "add.u32 s0, s0, t1;\n\t"
      "add.u32 s0, s0, g1;\n\t"           // low32(S)
      "add.u32 s1, s1, t2;\n\t"           // high word, low-word carries dropped
      "or.b32 %1, s1, 0xE0000000;\n\t"
      "shr.u32 t1, s1, 29;\n\t"
      "add.u32 %0, s0, t1;\n\t"           // low32(S) + q
      "}"
      : "=r"(y), "=r"(f)
      : "r"(c.a0), "r"(c.b0), "r"(c.b1), "r"(x.xl), "r"(c.a1), "r"(x.xh), "r"(x.xh2), "r"(x.xl4));
  return y;
}


// Token loads: read-only path, L1-allocating (each token is read by up to n lanes), and marked
// evict-first in L2 -- the 0.8 GB of tokens a C2 batch streams through once must not push the
// concurrently running Bloom kernels' filters (48 MB, L2-resident) out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t ld_token(const uint32_t* ptr, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}

// Landing gate (MinhashParams::landed): called by one thread for document d (token end o1)
// before any lane reads the document.  Returns false if the tokens did not land within
// kLandTimeoutNs (the batch is then rejected; see MinhashParams).
constexpr uint64_t kLandTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// `known`: the largest counter value already acquired.  The acquire load compiles to a strong
// load plus an L1 invalidation (CCTL.IVALL), which also evicts other warps' L1-resident lines;
// once a value is acquired, the pieces it covers stay visible, so documents within it need no new
// load.  The polling loop and its error path are a separate (not inlined) function.
__device__ __noinline__ uint32_t await_tokens_slow(const uint32_t* landed, const int* gate, ErrState* es,
                                                   uint32_t need) {
  if (*(volatile const int*)&es->flags & 2) return 0;      // an earlier wait timed out: fail fast
  uint32_t v = ld_acquire_u32(landed);
  if (v >= need) return v;
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
    __nanosleep(256);
    v = ld_acquire_u32(landed);
    if (v >= need) return v;
    if (*(volatile const int*)gate) return 0;                 // the batch was rejected meanwhile
    if (globaltimer_ns() - t0 > kLandTimeoutNs) {
      atomicOr(&es->flags, 2);
      atomicExch(&es->pad, 1);
      return 0;
    }
  }
}
__device__ __forceinline__ bool await_tokens_impl(const uint32_t* landed, uint32_t land_log2, uint64_t tok_total,
                                              const int* gate, ErrState* es, uint64_t o1, uint32_t& known) {
  const uint64_t r32 = (o1 + 31) & ~(uint64_t)31, end = tok_total < r32 ? tok_total : r32;
  const uint32_t need = (uint32_t)((end + (1ull << land_log2) - 1) >> land_log2);
  if (known >= need) return true;
  const uint32_t v = await_tokens_slow(landed, gate, es, need);
  if (v < need) return false;
  known = v;
  return true;
}
__device__ __forceinline__ bool await_tokens(const MinhashParams& p, uint64_t o1, uint32_t& known) {
  return await_tokens_impl(p.landed, p.land_log2, p.tok_total, p.err, p.err_state, o1, known);
}
// Warp-uniform form: every lane computes the same `need` and holds the same `known`, and the
// waiting lane's counter value is broadcast, so the branch is uniform by construction (with the
// verdict of lane 0 alone, ptxas moved the FP32-screen loop's uniform address and loop arithmetic
// from the uniform datapath onto the fma pipe and dropped operand-reuse flags: C3 K1 +3.5 ms).
__device__ __forceinline__ bool warp_await_tokens_u(const MinhashParams& p, uint32_t d, uint32_t& known) {
  if (!p.landed) return true;
  const uint64_t o1 = p.offsets[d + 1];
  const uint64_t r32 = (o1 + 31) & ~(uint64_t)31, end = p.tok_total < r32 ? p.tok_total : r32;
  const uint32_t need = (uint32_t)((end + (1ull << p.land_log2) - 1) >> p.land_log2);
  if (known >= need) return true;
  const uint32_t v = __shfl_sync(0xffffffffu, await_tokens_slow(p.landed, p.err, p.err_state, need), 0);
  if (v < need) return false;
  known = v;
  return true;
}

__device__ __forceinline__ XLimbs make_limbs(uint64_t fp) {
  uint64_t x = mod_p(fp);
  XLimbs l;
  l.xl = (uint32_t)x & 0x3FFFFFFFu;
  l.xh = (uint32_t)(x >> 30);
  l.xh2 = l.xh << 1;
  l.xl4 = l.xl << 2;
  return l;
}

// PASSES > 1: the lane's 32 NPL PASSES permutations are evaluated NPL at a time, one pass over
// the document's shingles each (coefficients reloaded per pass, the signature row collected in
// shared memory for the band hashes): the register footprint of NPL permutations per lane for
// PASSES x NPL of them -- 256 permutations on short documents at 4 per lane run at the 128-
// permutation kernel's occupancy instead of the 8-per-lane kernel's.
template <int NPL, int UNR, int MINB = LB_K1_MINB, int PASSES = 1, bool GATED = false>
__global__ void __launch_bounds__(K1_THREADS, MINB) k1_minhash(const MinhashParams p) {
  __shared__ XLimbs xs[K1_WARPS][32];
  __shared__ uint32_t sg[K1_WARPS][32 * NPL * PASSES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (*p.err) return;
  const uint64_t tpol = l2_evict_first_policy();
  uint32_t land_known = 0;   // landing counter value already acquired (gated launches)
  PermCoef c[NPL];
#pragma unroll
  for (int q = 0; q < NPL; q++) c[q] = p.coef[lane + 32 * q];

  for (;;) {
    uint32_t di = 0;
    if (lane == 0) di = atomicAdd(p.counter, 1u);
    di = __shfl_sync(0xffffffffu, di, 0);
    if (di >= (p.list ? *p.list_n : p.n_docs)) break;
    const uint32_t d = p.list ? p.list[di] : p.doc0 + di;
    if (GATED && !warp_await_tokens_u(p, d, land_known)) continue;
    const uint64_t o0 = p.offsets[d];
    const uint64_t L = p.offsets[d + 1] - o0;
    LB_ASSERT(L >= 1 && o0 >= p.tok_base);
    const uint32_t* tk = p.tokens + (o0 - p.tok_base);
    const uint32_t n = p.shingle_n;
    const uint32_t S = L >= n ? (uint32_t)(L - n + 1) : 1u;     // the bag of n-grams
    const uint32_t t = L >= n ? n : (uint32_t)L;
    const uint64_t init = (t == n) ? p.fp_init_n : mix64(kFpSalt + t);

    for (int pass = 0; pass < PASSES; pass++) {
    if (PASSES > 1) {
#pragma unroll
      for (int q = 0; q < NPL; q++) c[q] = p.coef[pass * 32 * NPL + lane + 32 * q];
    }
    uint32_t mn[NPL];
#pragma unroll
    for (int q = 0; q < NPL; q++) mn[q] = 0xFFFFFFFFu;
    uint32_t fmax = 0;

    for (uint32_t s0 = 0; s0 < S; s0 += 32) {
      const uint32_t s = s0 + lane;
      if (s < S) {
        uint64_t h = init;
        for (uint32_t j = 0; j < t; j++) h = mix64(h ^ (uint64_t)ld_token(tk + s + j, tpol));
        xs[w][lane] = make_limbs(h);
      }
      __syncwarp();
      const uint32_t cnt = min(32u, S - s0);
      uint32_t j = 0;
      for (; j + UNR <= cnt; j += UNR) {
        XLimbs xv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) xv[u] = xs[w][j + u];
#pragma unroll
        for (int q = 0; q < NPL; q++) {
#pragma unroll
          for (int u = 0; u < UNR; u += 2) {
            uint32_t f0, f1;
            const uint32_t y0 = eval_fast(c[q], xv[u], f0);
            const uint32_t y1 = eval_fast(c[q], xv[u + 1], f1);
            mn[q] = min(mn[q], min(y0, y1));
            fmax = max(fmax, max(f0, f1));
          }
        }
      }
      for (; j < cnt; j++) {
        const XLimbs xv = xs[w][j];
#pragma unroll
        for (int q = 0; q < NPL; q++) {
          uint32_t f0;
          mn[q] = min(mn[q], eval_fast(c[q], xv, f0));
          fmax = max(fmax, f0);
        }
      }
      __syncwarp();
    }
    if (__any_sync(0xffffffffu, fmax >= 0xFFFFFFFBu)) {   // rare: redo the document exactly
#pragma unroll
      for (int q = 0; q < NPL; q++) mn[q] = 0xFFFFFFFFu;
      for (uint32_t s0 = 0; s0 < S; s0 += 32) {
        const uint32_t s = s0 + lane;
        if (s < S) {
          uint64_t h = init;
          for (uint32_t j = 0; j < t; j++) h = mix64(h ^ (uint64_t)ld_token(tk + s + j, tpol));
          xs[w][lane] = make_limbs(h);
        }
        __syncwarp();
        const uint32_t cnt = min(32u, S - s0);
        for (uint32_t j = 0; j < cnt; j++) {
          const XLimbs xv = xs[w][j];
#pragma unroll
          for (int q = 0; q < NPL; q++) mn[q] = min(mn[q], eval_exact(c[q], xv));
        }
        __syncwarp();
      }
    }

    if (p.sig_out) {
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const uint32_t pm = pass * 32 * NPL + lane + 32 * q;
        if (pm < p.num_perm) p.sig_out[(uint64_t)d * p.num_perm + pm] = mn[q];
      }
    }
    if (p.bh_out) {
#pragma unroll
      for (int q = 0; q < NPL; q++) sg[w][pass * 32 * NPL + lane + 32 * q] = mn[q];
    }
    }  // pass
    if (p.bh_out) {
      __syncwarp();
      for (uint32_t j = lane; j < p.b; j += 32) {
        if (p.map.ncol[j] == 0) continue;
        uint64_t acc = 0;                               // BH_j, P:207-208 (DESIGN R6/R7)
        for (uint32_t u = 0; u < p.r; u++) {
          acc += affine32_mod_p(__ldg(p.bcoef + u), sg[w][j * p.r + u], __ldg(p.bcoef + p.r + u));
          acc = acc >= kP ? acc - kP : acc;
        }
        p.map.ptr[j][(uint64_t)d * p.map.ncol[j]] = acc;
      }
      __syncwarp();
    }
  }
}


// ---------------------------------------------------------------------------------------------
// Screened K1.  Almost no evaluation can lower a running minimum once a document's first few
// shingles are in (P(y < m) ~ 1/s after s shingles), and whether one can is decided by the low
// 32 bits of S' alone: with S' = A + G'_hi + G'_lo 2^29 and y = low32(S') - 1 + q, q in [0, 4],
//   y >= m is guaranteed  <=>  u = low32(S') - 1 lies in [m, 2^32 - 5]
//                         <=>  w = low32(S') - (m + 1)  <=  K = 2^32 - 5 - m      (mod 2^32)
// and low32(S') needs only low32(A) (two 32-bit IMADs: half the fmaheavy cost of IMAD.WIDE) and
// G' (two IMAD.WIDE).  Every evaluation is screened this way; the rare candidates (w > K) are
// queued per lane and per permutation slot in shared memory and evaluated exactly (eval_exact)
// when the queues are flushed (every 32-shingle chunk, or earlier when a queue nears capacity).
// The first shingle of every document is evaluated exactly to seed m; if any m > 2^32 - 5
// (probability ~2^-30 per document) the warp keeps evaluating that document exactly.
// Screening against a stale (larger) m only admits more candidates, so results are exact.
#define K1S_QCAP 16
#ifndef LB_K1S_MINB
#define LB_K1S_MINB 1
#endif

__device__ __forceinline__ bool screen(const PermCoef& c, const XLimbs& x, uint32_t bias, uint32_t K,
                                       uint32_t sh29) {
  // w = low32(S') - (m + 1) = low32(S) - m = a0 xl + a1 xh + [b_lo - m] + G_hi + (G_lo << 29)
  uint32_t w;
  asm("{\n\t"
      ".reg .u64 G;\n\t"
      ".reg .u32 t, g0, g1;\n\t"
      "mad.lo.u32 t, %1, %3, %7;\n\t"
      "mad.lo.u32 t, %2, %4, t;\n\t"
      "mul.wide.u32 G, %1, %5;\n\t"
      "mad.wide.u32 G, %2, %6, G;\n\t"
      "mov.b64 {g0, g1}, G;\n\t"
      "shl.b32 g0, g0, %8;\n\t"          // run-time 29: keeps the shift-add off the fmaheavy pipe
      "add.u32 t, t, g1;\n\t"
      "add.u32 %0, t, g0;\n\t"
      "}"
      : "=r"(w)
      : "r"(c.a0), "r"(c.a1), "r"(x.xl), "r"(x.xh), "r"(x.xh2), "r"(x.xl4), "r"(bias), "r"(sh29));
  return w > K;
}

__device__ __forceinline__ void st_shared_u8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ uint32_t ld_shared_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// BLOCKDOC: one document per block instead of per warp -- warp w takes the 32-shingle chunks
// w, w + 8, w + 16, ... of the document, and the 8 warps' minima are merged in shared memory
// before the epilogue.  For long documents: a launch over a few thousand full texts (a fused
// chunk's long list) is then balanced over blocks instead of lasting as long as its slowest
// warp (C4's fused step: 4 full texts per warp at most vs ~2.7 per warp with one each).
template <int NPL, bool BLOCKDOC = false, bool GATED = false>
__global__ void __launch_bounds__(K1_THREADS, BLOCKDOC ? 2 : LB_K1S_MINB) k1_minhash_scr(const MinhashParams p) {
  __shared__ XLimbs xs[K1_WARPS][32];
  __shared__ uint8_t qb[K1_WARPS][NPL][K1S_QCAP][32];   // [slot][lane]: conflict-free byte stores
  __shared__ uint32_t sg[K1_WARPS][32 * NPL];
  __shared__ uint32_t s_doc;
  __shared__ uint32_t smin[BLOCKDOC ? 32 * NPL : 1];   // BLOCKDOC: the block's running minima
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (*p.err) return;
  if (p.block_gate && p.list && ((*p.list_n < p.block_gate) != BLOCKDOC)) return;   // the other mode runs
  const uint64_t tpol = l2_evict_first_policy();
  uint32_t land_known = 0;   // landing counter value already acquired (gated launches)
  PermCoef c[NPL];
#pragma unroll
  for (int q = 0; q < NPL; q++) c[q] = p.coef[lane + 32 * q];
  const uint32_t sh29 = p.sh29;
  const uint32_t s_first = BLOCKDOC ? 32u * w : 0u, s_step = BLOCKDOC ? 32u * K1_WARPS : 32u;

  for (;;) {
    uint32_t di = 0;
    if (BLOCKDOC) {
      __syncthreads();                                   // the previous document's merge is done
      if (threadIdx.x == 0) {   // (the whole block takes the gate's verdict: no barrier divergence)
        uint32_t v = atomicAdd(p.counter, 1u);
        const uint32_t nd = p.list ? *p.list_n : p.n_docs;
        if (GATED && v < nd && !await_tokens(p, p.offsets[(p.list ? p.list[v] : p.doc0 + v) + 1], land_known))
          v = 0xFFFFFFFFu;
        s_doc = v;
      }
      if (BLOCKDOC)
        for (uint32_t i = threadIdx.x; i < 32u * NPL; i += K1_THREADS) smin[i] = 0xFFFFFFFFu;
      __syncthreads();
      di = s_doc;
    } else {
      if (lane == 0) di = atomicAdd(p.counter, 1u);
      di = __shfl_sync(0xffffffffu, di, 0);
    }
    if (di >= (p.list ? *p.list_n : p.n_docs)) break;
    const uint32_t d = p.list ? p.list[di] : p.doc0 + di;
    if (GATED && !BLOCKDOC && !warp_await_tokens_u(p, d, land_known)) continue;
    const uint64_t o0 = p.offsets[d];
    const uint64_t L = p.offsets[d + 1] - o0;
    LB_ASSERT(L >= 1 && o0 >= p.tok_base);
    const uint32_t* tk = p.tokens + (o0 - p.tok_base);
    const uint32_t n = p.shingle_n;
    const uint32_t S = L >= n ? (uint32_t)(L - n + 1) : 1u;
    const uint32_t t = L >= n ? n : (uint32_t)L;
    const uint64_t init = (t == n) ? p.fp_init_n : mix64(kFpSalt + t);

    uint32_t mn[NPL], bias[NPL], K[NPL];
#pragma unroll
    for (int q = 0; q < NPL; q++) mn[q] = 0xFFFFFFFFu;   // (a warp with no chunk keeps these)
    bool exact_mode = false;
    for (uint32_t s0 = s_first; s0 < S; s0 += s_step) {
      const uint32_t s = s0 + lane;
      if (s < S) {
        uint64_t h = init;
        for (uint32_t j = 0; j < t; j++) h = mix64(h ^ (uint64_t)ld_token(tk + s + j, tpol));
        xs[w][lane] = make_limbs(h);
      }
      __syncwarp();
      const uint32_t cnt = min(32u, S - s0);
      uint32_t j = 0;
      if (s0 == s_first) {   // seed the minima with the warp's first shingle, exactly
        const XLimbs x0 = xs[w][0];
        bool big = false;
#pragma unroll
        for (int q = 0; q < NPL; q++) {
          mn[q] = eval_exact(c[q], x0);
          bias[q] = c[q].b0 - mn[q];
          K[q] = 0xFFFFFFFBu - mn[q];
          big |= mn[q] > 0xFFFFFFFBu;
        }
        exact_mode = __any_sync(0xffffffffu, big);
        j = 1;
      }
      if (exact_mode) {
        for (; j < cnt; j++) {
          const XLimbs xv = xs[w][j];
#pragma unroll
          for (int q = 0; q < NPL; q++) mn[q] = min(mn[q], eval_exact(c[q], xv));
        }
      } else {
        uint32_t rsh29;
        asm volatile("mov.u32 %0, %1;" : "=r"(rsh29) : "r"(sh29));   // opaque register copy
        // per-slot queue write pointers (shared-memory byte addresses, stride 32 = one slot)
        uint32_t qp[NPL];
        const uint32_t qbase = (uint32_t)__cvta_generic_to_shared(&qb[w][0][0][lane]);
#pragma unroll
        for (int q = 0; q < NPL; q++) qp[q] = qbase + q * (K1S_QCAP * 32);
        auto flush = [&]() {
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            const uint32_t n = (qp[q] - (qbase + q * (K1S_QCAP * 32))) >> 5;
            const uint32_t rounds = __reduce_max_sync(0xffffffffu, n);
            for (uint32_t i = 0; i < rounds; i++) {
              if (i < n) {
                const uint32_t js = ld_shared_u8(qbase + q * (K1S_QCAP * 32) + i * 32);
                const uint32_t y = eval_exact(c[q], xs[w][js]);
                if (y < mn[q]) {
                  mn[q] = y;
                  bias[q] = c[q].b0 - y;
                  K[q] = 0xFFFFFFFBu - y;
                }
              }
            }
            qp[q] = qbase + q * (K1S_QCAP * 32);
          }
        };
        for (; j + 4 <= cnt; j += 4) {       // full groups: straight-line screening
          XLimbs xv[4];
#pragma unroll
          for (int u = 0; u < 4; u++) xv[u] = xs[w][j + u];
#pragma unroll
          for (int q = 0; q < NPL; q++) {
#pragma unroll
            for (int u = 0; u < 4; u++) {
              if (screen(c[q], xv[u], bias[q], K[q], rsh29)) {
                LB_ASSERT(qp[q] < qbase + (q + 1) * (K1S_QCAP * 32));
                st_shared_u8(qp[q], j + u);
                qp[q] += 32;
              }
            }
          }
          bool full = false;
#pragma unroll
          for (int q = 0; q < NPL; q++) full |= qp[q] - (qbase + q * (K1S_QCAP * 32)) > (K1S_QCAP - 4) * 32;
          if (__any_sync(0xffffffffu, full)) flush();
        }
        for (; j < cnt; j++) {               // ragged tail of the chunk
          const XLimbs xv = xs[w][j];
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            if (screen(c[q], xv, bias[q], K[q], rsh29)) {
              LB_ASSERT(qp[q] < qbase + (q + 1) * (K1S_QCAP * 32));
              st_shared_u8(qp[q], j);
              qp[q] += 32;
            }
          }
        }
        __syncwarp();
        flush();
        if (BLOCKDOC) {
          // share minima across the block's warps: each warp then screens against the smallest
          // value any warp has found (still exact: an evaluation >= a value already achieved by
          // another shingle cannot change the minimum), as one warp walking the whole document
          // would, instead of against its own 1/8 of the shingles
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            const uint32_t g = atomicMin(&smin[lane + 32 * q], mn[q]);
            if (g < mn[q]) {
              mn[q] = g;
              bias[q] = c[q].b0 - g;
              K[q] = 0xFFFFFFFBu - g;
            }
          }
        }
      }
      __syncwarp();
    }

    if (BLOCKDOC) {
      // merge the warps' minima: warp w reduces permutations [32 w', ...) for w' = w, w + 8, ...
#pragma unroll
      for (int q = 0; q < NPL; q++) sg[w][lane + 32 * q] = mn[q];
      __syncthreads();
      uint32_t fin[(NPL + K1_WARPS - 1) / K1_WARPS];
#pragma unroll
      for (int k = 0; k < (NPL + K1_WARPS - 1) / K1_WARPS; k++) {
        const uint32_t pm = 32u * (w + K1_WARPS * k) + lane;
        uint32_t v = 0xFFFFFFFFu;
        if (pm < 32u * NPL) {
#pragma unroll
          for (int r = 0; r < K1_WARPS; r++) v = min(v, sg[r][pm]);
        }
        fin[k] = v;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < (NPL + K1_WARPS - 1) / K1_WARPS; k++) {
        const uint32_t pm = 32u * (w + K1_WARPS * k) + lane;
        if (pm < 32u * NPL) sg[0][pm] = fin[k];
      }
      __syncthreads();
      if (w != 0) continue;                              // warp 0 writes the outputs
#pragma unroll
      for (int q = 0; q < NPL; q++) mn[q] = sg[0][lane + 32 * q];
    }
    if (p.sig_out) {
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const uint32_t pm = lane + 32 * q;
        if (pm < p.num_perm) p.sig_out[(uint64_t)d * p.num_perm + pm] = mn[q];
      }
    }
    if (p.bh_out) {
#pragma unroll
      for (int q = 0; q < NPL; q++) sg[w][lane + 32 * q] = mn[q];
      __syncwarp();
      for (uint32_t jb = lane; jb < p.b; jb += 32) {
        if (p.map.ncol[jb] == 0) continue;
        uint64_t acc = 0;                               // BH_j, P:207-208 (DESIGN R6/R7)
        for (uint32_t u = 0; u < p.r; u++) {
          acc += affine32_mod_p(__ldg(p.bcoef + u), sg[w][jb * p.r + u], __ldg(p.bcoef + p.r + u));
          acc = acc >= kP ? acc - kP : acc;
        }
        p.map.ptr[jb][(uint64_t)d * p.map.ncol[jb]] = acc;
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Screened K1, lean form (warp per document).  Same screen and the same exactness argument as
// k1_minhash_scr, with less state per lane so that more warps are resident (the screened loop
// stalls on fixed-latency dependencies -- "wait" -- with the 4 warps per scheduler the 127-register
// kernel allows):
//  * per permutation only a0, a1 (the screen's multipliers), bias = b0 - m and K = 2^32 - 5 - m
//    live in registers; m = 2^32 - 5 - K is implicit, b0 / b1 are re-read (L1) on an update;
//  * each screen that admits a candidate sets a bit in a per-permutation mask over the chunk's
//    32 shingles (ISETP + a predicated LOP3) instead of queueing it in shared memory (STS + add);
//    the candidates are evaluated exactly at the end of the chunk, all lanes in step;
//  * PASSES > 1 walks the document PASSES times with NPL permutations each (the fingerprints are
//    recomputed, ~2 % of the work) -- 256 permutations as 2 x 4 per lane.
template <int NPL, int PASSES, int MINB = 3, bool GATED = false>
__global__ void __launch_bounds__(K1_THREADS, MINB) k1_minhash_scr2(const MinhashParams p) {
  __shared__ XLimbs xs[K1_WARPS][32];
  __shared__ uint32_t sg[K1_WARPS][32 * NPL * PASSES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (*p.err) return;
  if (p.block_gate && p.list && *p.list_n < p.block_gate) return;   // the block-per-document kernel runs
  const uint64_t tpol = l2_evict_first_policy();
  uint32_t land_known = 0;   // landing counter value already acquired (gated launches)
  const uint32_t sh29 = p.sh29;

  for (;;) {
    uint32_t di = 0;
    if (lane == 0) di = atomicAdd(p.counter, 1u);
    di = __shfl_sync(0xffffffffu, di, 0);
    if (di >= (p.list ? *p.list_n : p.n_docs)) break;
    const uint32_t d = p.list ? p.list[di] : p.doc0 + di;
    if (GATED && !warp_await_tokens_u(p, d, land_known)) continue;
    const uint64_t o0 = p.offsets[d];
    const uint64_t L = p.offsets[d + 1] - o0;
    LB_ASSERT(L >= 1 && o0 >= p.tok_base);
    const uint32_t* tk = p.tokens + (o0 - p.tok_base);
    const uint32_t n = p.shingle_n;
    const uint32_t S = L >= n ? (uint32_t)(L - n + 1) : 1u;
    const uint32_t t = L >= n ? n : (uint32_t)L;
    const uint64_t init = (t == n) ? p.fp_init_n : mix64(kFpSalt + t);

    for (int pass = 0; pass < PASSES; pass++) {
      const uint32_t pm0 = pass * 32 * NPL + lane;           // permutation of slot q: pm0 + 32 q
      uint32_t a0[NPL], a1[NPL], bias[NPL], K[NPL];
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const PermCoef c = p.coef[pm0 + 32 * q];
        a0[q] = c.a0;
        a1[q] = c.a1;
      }
      bool exact_mode = false;
      for (uint32_t s0 = 0; s0 < S; s0 += 32) {
        const uint32_t s = s0 + lane;
        if (s < S) {
          uint64_t h = init;
          for (uint32_t j = 0; j < t; j++) h = mix64(h ^ (uint64_t)ld_token(tk + s + j, tpol));
          xs[w][lane] = make_limbs(h);
        }
        __syncwarp();
        const uint32_t cnt = min(32u, S - s0);
        uint32_t j = 0;
        if (s0 == 0) {   // seed the minima with the first shingle, exactly
          const XLimbs x0 = xs[w][0];
          bool big = false;
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            K[q] = eval_exact(p.coef[pm0 + 32 * q], x0);     // (the raw minimum, for now)
            big |= K[q] > 0xFFFFFFFBu;
          }
          exact_mode = __any_sync(0xffffffffu, big);
          if (!exact_mode) {
#pragma unroll
            for (int q = 0; q < NPL; q++) {
              bias[q] = p.coef[pm0 + 32 * q].b0 - K[q];
              K[q] = 0xFFFFFFFBu - K[q];
            }
          }
          j = 1;
        }
        if (exact_mode) {     // (probability ~2^-30 per document) K holds the raw minima
          for (; j < cnt; j++) {
            const XLimbs xv = xs[w][j];
#pragma unroll
            for (int q = 0; q < NPL; q++) K[q] = min(K[q], eval_exact(p.coef[pm0 + 32 * q], xv));
          }
        } else {
          uint32_t rsh29;
          asm volatile("mov.u32 %0, %1;" : "=r"(rsh29) : "r"(sh29));   // opaque: shift stays on the ALU pipe
          uint32_t mask[NPL];
#pragma unroll
          for (int q = 0; q < NPL; q++) mask[q] = 0;
          for (; j + 4 <= cnt; j += 4) {
            XLimbs xv[4];
#pragma unroll
            for (int u = 0; u < 4; u++) xv[u] = xs[w][j + u];
#pragma unroll
            for (int q = 0; q < NPL; q++) {
              const PermCoef cq = {a0[q], a1[q], 0u, 0u};
#pragma unroll
              for (int u = 0; u < 4; u++)
                if (screen(cq, xv[u], bias[q], K[q], rsh29)) mask[q] |= 1u << (j + u);
            }
          }
          for (; j < cnt; j++) {
            const XLimbs xv = xs[w][j];
#pragma unroll
            for (int q = 0; q < NPL; q++) {
              const PermCoef cq = {a0[q], a1[q], 0u, 0u};
              if (screen(cq, xv, bias[q], K[q], rsh29)) mask[q] |= 1u << j;
            }
          }
          // exact evaluation of the candidates, all lanes in step (rounds = the warp's largest count)
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            const uint32_t rounds = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(mask[q]));
            if (!rounds) continue;
            const PermCoef c = p.coef[pm0 + 32 * q];
            for (uint32_t i = 0; i < rounds; i++) {
              if (mask[q]) {
                const uint32_t js = __ffs(mask[q]) - 1;
                mask[q] &= mask[q] - 1;
                const uint32_t y = eval_exact(c, xs[w][js]);
                if (y < 0xFFFFFFFBu - K[q]) {
                  bias[q] = c.b0 - y;
                  K[q] = 0xFFFFFFFBu - y;
                }
              }
            }
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const uint32_t m = exact_mode ? K[q] : 0xFFFFFFFBu - K[q];
        const uint32_t pm = pm0 + 32 * q;
        if (p.sig_out && pm < p.num_perm) p.sig_out[(uint64_t)d * p.num_perm + pm] = m;
        if (p.bh_out) sg[w][pm] = m;
      }
    }  // pass
    if (p.bh_out) {
      __syncwarp();
      for (uint32_t jb = lane; jb < p.b; jb += 32) {
        if (p.map.ncol[jb] == 0) continue;
        uint64_t acc = 0;                               // BH_j, P:207-208 (DESIGN R6/R7)
        for (uint32_t u = 0; u < p.r; u++) {
          acc += affine32_mod_p(__ldg(p.bcoef + u), sg[w][jb * p.r + u], __ldg(p.bcoef + p.r + u));
          acc = acc >= kP ? acc - kP : acc;
        }
        p.map.ptr[jb][(uint64_t)d * p.map.ncol[jb]] = acc;
      }
      __syncwarp();
    }
  }
}

template <int NPL, int PASSES, int MINB = 3>
static int launch_s2(const MinhashParams& p, int sm_count, cudaStream_t s, int max_bps) {
  static int bps_of[2] = {0, 0};   // [gated]
  const int gi = p.landed ? 1 : 0;
  if (!bps_of[gi]) {
    if (gi) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr2<NPL, PASSES, MINB, true>, K1_THREADS, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr2<NPL, PASSES, MINB, false>, K1_THREADS, 0);
    if (bps_of[gi] < 1) bps_of[gi] = 1;
  }
  const int blocks_per_sm = bps_of[gi];
  uint64_t want = ((uint64_t)p.n_docs + K1_WARPS - 1) / K1_WARPS;
  const int bps = (max_bps > 0 && max_bps < blocks_per_sm) ? max_bps : blocks_per_sm;
  uint64_t grid = (uint64_t)sm_count * bps;
  if (want < grid) grid = want ? want : 1;
  if (p.landed) k1_minhash_scr2<NPL, PASSES, MINB, true><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  else k1_minhash_scr2<NPL, PASSES, MINB, false><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  return 1;
}

// ---------------------------------------------------------------------------------------------
// Screened K1 with the FP64 pipe (k1_minhash_scr3).  The integer screen needs the high half of
// the 64-bit products (two IMAD.WIDE: 8 of its 12 fmaheavy cycles per warp-evaluation).  Split
// instead a = ah 2^32 + al, x = xh 2^32 + xl (ah, xh < 2^29) and M = ah xl + al xh (< 2^62):
//   a x = al xl + M 2^32 + ah xh 2^64,   M 2^32 = M_hi 2^61 + M_lo 2^32  (M_hi = floor(M / 2^29)),
//   2^61 = 1, 2^64 = 8 (mod P)  =>  a x + b = T (mod P),  T = al xl + M_lo 2^32 + M_hi + 8 ah xh + b,
//   0 <= T < 2^64 + 3 2^61 + 2^33 < 11 2^61 + 2^33, so q = floor(T / P) <= 11 and
//   y = low32((a x + b) mod P) = L + q (mod 2^32),  L = lo(al xl) + lo(8ah xh) + M_hi + lo(b).
// M_hi is only needed to within +-1 for a screen, and two DFMA give that:
//   r = fma(ah, xl 2^-29, fma(al, xh 2^-29, 1.5 2^52))  (every operand exact in binary64; both
//   results lie in [2^52, 2^53) where the ulp is 1, so each rounding moves by <= 1/2) = 1.5 2^52
//   + M / 2^29 + eps, |eps| <= 1, and the low word of r is N mod 2^32 with N - M_hi in {-1, 0, 1}.
// With L' = lo(al xl) + lo(8ah xh) + N + lo(b) = L + e, e in [-1, 1]: L in [m, 2^32 - 1 - 11]
// guarantees y >= m, and L' in [m + 1, 2^32 - 13] guarantees that, i.e. with u = L' + 12 and
// T = m + 13 (mod 2^32):  u >= T  =>  skip;  u < T: a candidate, evaluated exactly (eval_exact).
// (m > 2^32 - 14, only possible for a document's first shingle, keeps the document exact.)  The
// constant lo(b) + 12 rides in the magic addend: r1 = fma(al, xh 2^-29, 1.5 2^52 + lo(b) + 12)
// (exact: < 2^53), so u = al xl + 8ah xh + lo32(r2) -- two IMAD, no add.  DFMA issues at 1/4 rate on the unit IMAD.WIDE uses, IMAD at 1/2
// on fmaheavy, and the two overlap (tools/micro/pipe_micro.cu: fma.f64 + mad.lo 0.494 warp-inst/clk
// /SMSP together), so a screen costs 8 cycles of the FP64 unit instead of 12 of fmaheavy; the
// whole screen loop runs at 2.36 evaluations/clk/SMSP in isolation vs 1.91 for the integer one
// (tools/micro/dfma_screen.cu, which also checks 2^32 random and near-P triples: no screened-out
// y < m).  B200 (GB100) has full-rate-for-Blackwell FP64; on parts with vestigial FP64 this
// kernel must not be selected.
constexpr uint32_t kScr3Q = 13;   // T = m + kScr3Q: q <= 11 plus the +-1 of N, plus 1
struct __align__(16) XLimbsF {     // shingle x for the FP64 screen
  double XL, XH;                   // xl 2^-29, xh 2^-29 (exact)
  uint32_t xl, xh;                 // x mod 2^32, x >> 32
};
__device__ __forceinline__ uint32_t screen_u_f64(uint32_t al, uint32_t a8h, double AL, double AH, double CB,
                                                 const XLimbsF& x) {
  const double r1 = fma(AL, x.XH, CB);                   // CB = 1.5 2^52 + lo(b) + 12
  const double r2 = fma(AH, x.XL, r1);
  return al * x.xl + a8h * x.xh + (uint32_t)__double2loint(r2);
}

template <int NPL, int PASSES, int MINB = 3, bool GATED = false>
__global__ void __launch_bounds__(K1_THREADS, MINB) k1_minhash_scr3(const MinhashParams p) {
  __shared__ XLimbs xs[K1_WARPS][32];        // exact-evaluation limbs
  __shared__ XLimbsF xf[K1_WARPS][32];       // screen limbs
  __shared__ uint32_t sg[K1_WARPS][32 * NPL * PASSES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (*p.err) return;
  if (p.block_gate && p.list && *p.list_n < p.block_gate) return;   // the block-per-document kernel runs
  const uint64_t tpol = l2_evict_first_policy();
  uint32_t land_known = 0;   // landing counter value already acquired (gated launches)

  for (;;) {
    uint32_t di = 0;
    if (lane == 0) di = atomicAdd(p.counter, 1u);
    di = __shfl_sync(0xffffffffu, di, 0);
    if (di >= (p.list ? *p.list_n : p.n_docs)) break;
    const uint32_t d = p.list ? p.list[di] : p.doc0 + di;
    if (GATED && !warp_await_tokens_u(p, d, land_known)) continue;
    const uint64_t o0 = p.offsets[d];
    const uint64_t L = p.offsets[d + 1] - o0;
    LB_ASSERT(L >= 1 && o0 >= p.tok_base);
    const uint32_t* tk = p.tokens + (o0 - p.tok_base);
    const uint32_t n = p.shingle_n;
    const uint32_t S = L >= n ? (uint32_t)(L - n + 1) : 1u;
    const uint32_t t = L >= n ? n : (uint32_t)L;
    const uint64_t init = (t == n) ? p.fp_init_n : mix64(kFpSalt + t);

    for (int pass = 0; pass < PASSES; pass++) {
      const uint32_t pm0 = pass * 32 * NPL + lane;           // permutation of slot q: pm0 + 32 q
      uint32_t al[NPL], a8h[NPL], K[NPL];                   // K: the threshold T = m + 13 (raw m in exact mode)
      double AL[NPL], AH[NPL], CB[NPL];
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const PermCoef c = p.coef[pm0 + 32 * q];             // a = a1 2^31 + a0
        al[q] = c.a0 | (c.a1 << 31);
        a8h[q] = (c.a1 >> 1) << 3;
        AL[q] = (double)al[q];
        AH[q] = (double)(c.a1 >> 1);
        CB[q] = 6755399441055744.0 + (double)(c.b0 + 12u);   // 1.5 2^52 + lo(b) + 12 (mod 2^32)
      }
      // exact prefix: the first p.exact_prefix chunks are evaluated exactly (K = raw minima), where
      // candidates would be frequent (P(candidate) ~ 1/s after s shingles); then the screen
      bool exact_mode = true;
#pragma unroll
      for (int q = 0; q < NPL; q++) K[q] = 0xFFFFFFFFu;
      const uint32_t pre = 32u * p.exact_prefix;
      for (uint32_t s0 = 0; s0 < S; s0 += 32) {
        const uint32_t s = s0 + lane;
        if (s < S) {
          uint64_t h = init;
          for (uint32_t j = 0; j < t; j++) h = mix64(h ^ (uint64_t)ld_token(tk + s + j, tpol));
          const uint64_t x = mod_p(h);
          xs[w][lane] = make_limbs(h);
          XLimbsF f;
          f.xl = (uint32_t)x;
          f.xh = (uint32_t)(x >> 32);
          f.XL = (double)f.xl * 0x1p-29;
          f.XH = (double)f.xh * 0x1p-29;
          xf[w][lane] = f;
        }
        __syncwarp();
        const uint32_t cnt = min(32u, S - s0);
        uint32_t j = 0;
        if (exact_mode && s0 >= pre) {   // leave exact mode (seeding with shingle 0 if no prefix)
          bool big = false;
          const XLimbs x0 = xs[w][0];
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            if (s0 == 0) K[q] = eval_exact(p.coef[pm0 + 32 * q], x0);   // (the raw minimum, for now)
            big |= K[q] > 0xFFFFFFFFu - kScr3Q;               // T = m + 13 would wrap
          }
          if (s0 == 0) j = 1;
          exact_mode = __any_sync(0xffffffffu, big);
          if (!exact_mode) {
#pragma unroll
            for (int q = 0; q < NPL; q++) K[q] += kScr3Q;
          }
        }
        if (exact_mode) {     // the prefix, or (probability ~2^-28) a minimum near 2^32: raw minima
          for (; j < cnt; j++) {
            const XLimbs xv = xs[w][j];
#pragma unroll
            for (int q = 0; q < NPL; q++) K[q] = min(K[q], eval_exact(p.coef[pm0 + 32 * q], xv));
          }
        } else {
          uint32_t mask[NPL];
#pragma unroll
          for (int q = 0; q < NPL; q++) mask[q] = 0;
          for (; j + 4 <= cnt; j += 4) {
            XLimbsF xv[4];
#pragma unroll
            for (int u = 0; u < 4; u++) xv[u] = xf[w][j + u];
#pragma unroll
            for (int q = 0; q < NPL; q++) {
#pragma unroll
              for (int u = 0; u < 4; u++)
                if (screen_u_f64(al[q], a8h[q], AL[q], AH[q], CB[q], xv[u]) < K[q]) mask[q] |= 1u << (j + u);
            }
          }
          for (; j < cnt; j++) {
            const XLimbsF xv = xf[w][j];
#pragma unroll
            for (int q = 0; q < NPL; q++)
              if (screen_u_f64(al[q], a8h[q], AL[q], AH[q], CB[q], xv) < K[q]) mask[q] |= 1u << j;
          }
          // exact evaluation of the candidates, all lanes in step (rounds = the warp's largest count)
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            const uint32_t rounds = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(mask[q]));
            if (!rounds) continue;
            const PermCoef c = p.coef[pm0 + 32 * q];
            for (uint32_t i = 0; i < rounds; i++) {
              if (mask[q]) {
                const uint32_t js = __ffs(mask[q]) - 1;
                mask[q] &= mask[q] - 1;
                const uint32_t y = eval_exact(c, xs[w][js]);
                if (y < K[q] - kScr3Q) K[q] = y + kScr3Q;    // (y < m; y + 13 may wrap for a false candidate)
              }
            }
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const uint32_t m = exact_mode ? K[q] : K[q] - kScr3Q;
        const uint32_t pm = pm0 + 32 * q;
        if (p.sig_out && pm < p.num_perm) p.sig_out[(uint64_t)d * p.num_perm + pm] = m;
        if (p.bh_out) sg[w][pm] = m;
      }
    }  // pass
    if (p.bh_out) {
      __syncwarp();
      for (uint32_t jb = lane; jb < p.b; jb += 32) {
        if (p.map.ncol[jb] == 0) continue;
        uint64_t acc = 0;                               // BH_j, P:207-208 (DESIGN R6/R7)
        for (uint32_t u = 0; u < p.r; u++) {
          acc += affine32_mod_p(__ldg(p.bcoef + u), sg[w][jb * p.r + u], __ldg(p.bcoef + p.r + u));
          acc = acc >= kP ? acc - kP : acc;
        }
        p.map.ptr[jb][(uint64_t)d * p.map.ncol[jb]] = acc;
      }
      __syncwarp();
    }
  }
}

template <int NPL, int PASSES, int MINB = 3>
static int launch_s3(const MinhashParams& p, int sm_count, cudaStream_t s, int max_bps) {
  static int bps_of[2] = {0, 0};   // [gated]
  const int gi = p.landed ? 1 : 0;
  if (!bps_of[gi]) {
    if (gi) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr3<NPL, PASSES, MINB, true>, K1_THREADS, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr3<NPL, PASSES, MINB, false>, K1_THREADS, 0);
    if (bps_of[gi] < 1) bps_of[gi] = 1;
  }
  const int blocks_per_sm = bps_of[gi];
  uint64_t want = ((uint64_t)p.n_docs + K1_WARPS - 1) / K1_WARPS;
  const int bps = (max_bps > 0 && max_bps < blocks_per_sm) ? max_bps : blocks_per_sm;
  uint64_t grid = (uint64_t)sm_count * bps;
  if (want < grid) grid = want ? want : 1;
  if (p.landed) k1_minhash_scr3<NPL, PASSES, MINB, true><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  else k1_minhash_scr3<NPL, PASSES, MINB, false><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  return 1;
}

// ---------------------------------------------------------------------------------------------
// Screened K1 with the FP32 pipe (k1_minhash_scr4; round 2).  Same split and T as scr3:
//   y = low32((a x + b) mod P) = L + H + q (mod 2^32),  L = lo(al xl) + lo(8ah xh) + lo(b),
//   H = floor(M / 2^29), M = ah xl + al xh,  q in [0, 11].
// A screen needs H only to within a few thousand, and two binary32 FMA give that:
//   r = fmaf(AH, XL, fmaf(AL, XH, 1.5 2^34)),  AL = fl(al), AH = fl(ah), XL = fl(xl) 2^-29,
//   XH = fl(xh) 2^-29 (each rounded to nearest: relative error <= 2^-24).  Both sums lie in
//   [2^34, 2^35] where the ulp is 2^11, and bits(r) << 11 = r - 1.5 2^34 (mod 2^32) (at r = 2^35
//   both sides are 2^33 = 0).  Error of Hc = bits(r) << 11 against H: the two products' operand
//   rounding <= 2^32 (2^-23 + 2^-48) each (~2^9), the two roundings <= 2^10 each, the floor < 1:
//   |Hc - H| <= 3074.  With u = lo(al xl) + lo(8ah xh) + (lo(b) + 4096) + Hc:
//   u - y = 4096 + (Hc - H) - q in [1011, 7170] (mod 2^32), so for m <= 2^32 - 1 - 8192,
//   y < m  =>  u < m + 7171 < m + 8192 = K;  u >= K: skip;  u < K: a candidate, evaluated exactly.
// Per evaluation: 2 IMAD + 2 FFMA (one with an immediate) + a shift-add (LEA) + half a 3-input min
// (the min over each 4-shingle group is compared once) -- the FFMA share the fma pipe with IMAD
// but the second product's high half no longer costs a 1/4-rate DFMA or IMAD.WIDE.  Measured
// in isolation (tools/micro/fp32_screen.cu, profiles/r02s_fp32_screen_micro.txt): 3.75
// evaluations/clk/SMSP at 2 blocks per SM vs 2.39-2.53 for the FP64 screen; 2^32 random and
// adversarial triples: no screened-out y < m, largest |Hc - H| 2471.
constexpr uint32_t kScr4W = 8192, kScr4D = 4096;
constexpr float kScr4Magic = 25769803776.0f;   // 1.5 2^34
struct __align__(16) XLimbsS {                 // shingle x for the FP32 screen
  uint32_t xl, xh;                             // x mod 2^32, x >> 32
  float XL, XH;                                // fl(xl) 2^-29, fl(xh) 2^-29
};
// SPLIT: both products take the magic addend as an immediate (two 1-cycle FFMA instead of a 1- and a
// 2-cycle one) and their bit patterns are added on the ALU: bits(r1) + bits(r2) = 2 bits(1.5 2^34) +
// (the two rounded products) / 2^11, and 2 bits(1.5 2^34) << 11 = 0 (mod 2^32) (bits(1.5 2^34) = 0x50C00000),
// so (bits(r1) + bits(r2)) << 11 = the same Hc with the same two roundings (|Hc - H| <= 3074 still holds: each sum
// lies in [1.5 2^34, 1.75 2^34), ulp 2^11).  One fma-pipe cycle less, one ALU instruction more.
#ifndef LB_SCR4_SPLITQ
#define LB_SCR4_SPLITQ 0   // permutation slots per lane (of NPL) screened in the split form
#endif
__device__ __forceinline__ uint32_t screen_u_f32(uint32_t al, uint32_t a8h, uint32_t lb, float AL, float AH,
                                                 const XLimbsS& x, const bool SPLIT = false) {
  const float r1 = __fmaf_rn(AL, x.XH, kScr4Magic);
  float r2;
  uint32_t t, hb;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(al), "r"(x.xl), "r"(lb));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a8h), "r"(x.xh), "r"(t));
  if (SPLIT) {
    r2 = __fmaf_rn(AH, x.XL, kScr4Magic);
    // (two funnel-shift-adds: a plain add of the bit patterns became IMAD.IADD on the fma pipe)
    uint32_t hb1;
    asm("shf.l.wrap.b32 %0, %1, %2, 11;" : "=r"(hb1) : "r"(0u), "r"(__float_as_uint(r1)));
    asm("shf.l.wrap.b32 %0, %1, %2, 11;" : "=r"(hb) : "r"(0u), "r"(__float_as_uint(r2)));
    return (t + hb1) + hb;
  }
  r2 = __fmaf_rn(AH, x.XL, r1);
  // bits << 11 as a funnel shift ({bits, 0} << 11, high word): ptxas then fuses it with the add
  // into LEA.HI on the ALU pipe; a plain shl + add became IMAD (x 2048 + t) on the fma pipe -- the
  // loop's bottleneck -- for 7 of every 8 evaluations (4.9 instead of 4.0 fma-pipe ops each)
  asm("shf.l.wrap.b32 %0, %1, %2, 11;" : "=r"(hb) : "r"(0u), "r"(__float_as_uint(r2)));
  return t + hb;
}

template <int NPL, int PASSES, int MINB = 2, bool GATED = false, int G = 4, int R = 1, bool BAL = true>
__global__ void __launch_bounds__(K1_THREADS, MINB) k1_minhash_scr4(const MinhashParams p) {
  static_assert(R == 1 || (R == 2 && G == 8), "deferred resolution packs two chunks' 4 groups");
  __shared__ XLimbs xs[R][K1_WARPS][32];     // exact-evaluation limbs (R chunks)
  __shared__ XLimbsS xf[R][K1_WARPS][32];    // screen limbs
  __shared__ uint32_t sg[K1_WARPS][32 * NPL * PASSES];
  __shared__ uint32_t kq[K1_WARPS][NPL][32];  // thresholds while flagged groups are resolved
  constexpr uint32_t kRQ = 512;                 // balanced-resolution queue per warp (the rest per lane)
  __shared__ uint16_t rq[BAL ? K1_WARPS : 1][BAL ? kRQ : 1];   // flagged (lane, bit) items
  __shared__ PermCoef cs[32 * NPL * PASSES];   // the coefficient table (exact evaluations read it
                                              // by permutation; shared memory is immune to the
                                              // L1 invalidations of gated launches)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < 32 * NPL * PASSES; i += K1_THREADS) cs[i] = p.coef[i];
  __syncthreads();
  if (*p.err) return;
  if (p.block_gate && p.list && *p.list_n < p.block_gate) return;   // the block-per-document kernel runs
  const uint64_t tpol = l2_evict_first_policy();
  uint32_t land_known = 0;   // landing counter value already acquired (gated launches)

  for (;;) {
    uint32_t di = 0;
    if (lane == 0) di = atomicAdd(p.counter, 1u);
    di = __shfl_sync(0xffffffffu, di, 0);
    if (di >= (p.list ? *p.list_n : p.n_docs)) break;
    const uint32_t d = p.list ? p.list[di] : p.doc0 + di;
    if (GATED && !warp_await_tokens_u(p, d, land_known)) continue;   // (rejected batch: the rest fail fast)
    const uint64_t o0 = p.offsets[d];
    const uint64_t L = p.offsets[d + 1] - o0;
    LB_ASSERT(L >= 1 && o0 >= p.tok_base);
    const uint32_t* tk = p.tokens + (o0 - p.tok_base);
    const uint32_t n = p.shingle_n;
    const uint32_t S = L >= n ? (uint32_t)(L - n + 1) : 1u;
    const uint32_t t = L >= n ? n : (uint32_t)L;
    const uint64_t init = (t == n) ? p.fp_init_n : mix64(kFpSalt + t);

    for (int pass = 0; pass < PASSES; pass++) {
      const uint32_t pm0 = pass * 32 * NPL + lane;           // permutation of slot q: pm0 + 32 q
      uint32_t al[NPL], a8h[NPL], lb[NPL], K[NPL];          // K: the threshold m + W (raw m in exact mode)
      float AL[NPL], AH[NPL];
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const PermCoef c = cs[pm0 + 32 * q];             // a = a1 2^31 + a0
        al[q] = c.a0 | (c.a1 << 31);
        a8h[q] = (c.a1 >> 1) << 3;
        lb[q] = c.b0 + kScr4D;
        AL[q] = __uint2float_rn(al[q]);
        AH[q] = __uint2float_rn(c.a1 >> 1);
      }
      bool exact_mode = true;
#pragma unroll
      for (int q = 0; q < NPL; q++) K[q] = 0xFFFFFFFFu;
      const uint32_t pre = 32u * p.exact_prefix;
      // Tokens (shingles of <= 8 ids): one coalesced 32-token load per chunk, issued a chunk ahead
      // (tw0 = tokens [s0, s0 + 32), tw1 = [s0 + 32, s0 + 64), tw2 in flight), and the shingle's
      // ids gathered with shuffles -- the per-lane chain of t dependent loads held the warps at the
      // start of every chunk (ncu: 17 % of the stall samples for 5 % of the instructions).
      const bool shfl_fp = t <= 8;
      uint32_t tw0 = 0, tw1 = 0;
      if (shfl_fp) {
        if (lane < L) tw0 = ld_token(tk + lane, tpol);
        if (32 + lane < L) tw1 = ld_token(tk + 32 + lane, tpol);
      }
      uint64_t cm = 0;                  // flagged (permutation, group) bits of the unresolved chunks
      uint32_t j0s0 = 0, j0s1 = 0;      // first screened shingle of the chunks in buffers 0 / 1
      for (uint32_t s0 = 0, ci = 0; s0 < S; s0 += 32, ci++) {
        const uint32_t s = s0 + lane;
        const uint32_t bf = R == 2 ? (ci & 1) : 0;   // limb buffer of this chunk
        uint32_t tw2 = 0;
        if (shfl_fp && s0 + 64 + lane < L) tw2 = ld_token(tk + s0 + 64 + lane, tpol);
        uint64_t h = init;
#ifdef LB_DIAG_NOFP
        if (s0 >= 64) { tw0 = tw1; tw1 = tw2; h = (uint64_t)(s + 1) * 0x9E3779B97F4A7C15ull + o0; } else   // diagnostic: cheap distinct x
#endif
        if (shfl_fp) {
#pragma unroll
          for (uint32_t j = 0; j < 8; j++) {
            if (j < t) {
              const uint32_t src = (lane + j) & 31;
              const uint32_t a0 = __shfl_sync(0xffffffffu, tw0, src), a1 = __shfl_sync(0xffffffffu, tw1, src);
              h = mix64(h ^ (uint64_t)(lane + j < 32 ? a0 : a1));
            }
          }
          tw0 = tw1;
          tw1 = tw2;
        } else if (s < S) {
          for (uint32_t j = 0; j < t; j++) h = mix64(h ^ (uint64_t)ld_token(tk + s + j, tpol));
        }
        if (s < S) {
          const uint64_t x = mod_p(h);
          xs[bf][w][lane] = make_limbs(h);
          XLimbsS f;
          f.xl = (uint32_t)x;
          f.xh = (uint32_t)(x >> 32);
          f.XL = __uint2float_rn(f.xl) * 0x1p-29f;
          f.XH = __uint2float_rn(f.xh) * 0x1p-29f;
          xf[bf][w][lane] = f;
        }
        __syncwarp();
        const uint32_t cnt = min(32u, S - s0);
        uint32_t j = 0;
        if (exact_mode && s0 >= pre) {   // leave exact mode (seeding with shingle 0 if no prefix)
          bool big = false;
          const XLimbs x0 = xs[bf][w][0];
#pragma unroll
          for (int q = 0; q < NPL; q++) {
            if (s0 == 0) K[q] = eval_exact(cs[pm0 + 32 * q], x0);   // (the raw minimum, for now)
            big |= K[q] > 0xFFFFFFFFu - kScr4W;               // m + W would wrap
          }
          if (s0 == 0) j = 1;
          exact_mode = __any_sync(0xffffffffu, big);
          if (!exact_mode) {
#pragma unroll
            for (int q = 0; q < NPL; q++) K[q] += kScr4W;
          }
        }
        if (exact_mode) {     // the prefix, or (probability ~2^-19 per permutation) a minimum near 2^32
          for (; j < cnt; j++) {
            const XLimbs xv = xs[bf][w][j];
#pragma unroll
            for (int q = 0; q < NPL; q++) K[q] = min(K[q], eval_exact(cs[pm0 + 32 * q], xv));
          }
        } else {
          // groups of G shingles from j0: a flag per (slot q, group g) = some u of the group is below K[q]
          if (bf) j0s1 = j; else j0s0 = j;
          // the flag of (slot q, group g) goes straight into cm (bit 8 q + 4 bf + g) with a predicated
          // OR of a warp-uniform bit (setp + @p or -> ISETP + @P LOP3; `if (mn < K) mask[q] |= bit` on
          // per-slot mask registers compiled to ISETP + SEL + LOP3, a combine after the loop, and --
          // the registers gone -- eight I2FP per group rematerialising AL[]): the loop is issue-bound,
          // 404 -> 386 instructions per 64 evaluations, C3 K1 alone 60.4 -> 57.0 ms
          uint32_t cml = 0, cmh = 0;
          uint32_t gb0 = R == 2 ? (bf ? 16u : 1u) : 1u;   // 1 << (4 bf + g)
          for (; j + G <= cnt; j += G, gb0 <<= 1) {
            XLimbsS xv[G];
            const uint32_t gb[4] = {gb0, gb0 << 8, gb0 << 16, gb0 << 24};
#pragma unroll
            for (int u = 0; u < G; u++) xv[u] = xf[bf][w][j + u];
#pragma unroll
            for (int q = 0; q < NPL; q++) {
              uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
              for (int u = 0; u < G; u++) mn = min(mn, screen_u_f32(al[q], a8h[q], lb[q], AL[q], AH[q], xv[u], q < LB_SCR4_SPLITQ));
              if (q < 4) asm("{ .reg .pred p; setp.lt.u32 p, %1, %2; @p or.b32 %0, %0, %3; }" : "+r"(cml) : "r"(mn), "r"(K[q]), "r"(gb[q & 3]));
              else asm("{ .reg .pred p; setp.lt.u32 p, %1, %2; @p or.b32 %0, %0, %3; }" : "+r"(cmh) : "r"(mn), "r"(K[q]), "r"(gb[q & 3]));
            }
          }
          cm |= ((uint64_t)cmh << 32) | cml;
          // the chunk's last (cnt - j0) mod G shingles: exactly (warp-uniform)
          for (; j < cnt; j++) {
            const XLimbs xv = xs[bf][w][j];
#pragma unroll
            for (int q = 0; q < NPL; q++) {
              const uint32_t y = eval_exact(cs[pm0 + 32 * q], xv);
              if (y < K[q] - kScr4W) K[q] = y + kScr4W;
            }
          }
        }
        // exact evaluation of the flagged groups (every chunk, or with R = 2 every second chunk and
        // the last: a chunk's flags wait in cm while the next chunk is screened against the older
        // threshold, and one set of rounds serves both): each lane walks its own (permutation,
        // group) pairs, whichever permutation they belong to, so a round serves every lane that
        // still has one (rounds = the warp's largest per-lane count, not a sum over permutations);
        // the slot's coefficients come from the (L1-resident) table, its threshold from shared memory
#ifdef LB_DIAG_NORES
        K[0] ^= (uint32_t)__popcll(cm) & 1u;   // diagnostic build only: skip the resolution (wrong signatures)
        cm = 0;
#endif
        if ((R == 1 || bf == 1 || s0 + 32 >= S) && __any_sync(0xffffffffu, cm != 0)) {
#pragma unroll
          for (int q = 0; q < NPL; q++) kq[w][q][lane] = K[q];
          if (BAL) {
            // (128 permutations: abstract-length documents have many flagged groups per chunk,
            // unevenly spread over the lanes -- C5 K1 28.3 -> 26.9 ms per 2M documents, C2 14.2 ->
            // 13.5 ms; with 256 the long documents' sparse flags favour the per-lane walk below,
            // C3 63.4 vs 65.8 ms)
            // the warp's flagged (lane, permutation, group) items, load-balanced over the lanes:
            // each lane's items go to a shared queue at its prefix-sum offset and lane l takes items
            // l, l + 32, ... (rounds = ceil(items / 32) instead of the largest per-lane count);
            // thresholds live in kq meanwhile, lowered with shared-memory atomicMin
            const uint32_t cnt = (uint32_t)__popcll(cm);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += t;
            }
            const uint32_t total = min(kRQ, __shfl_sync(0xffffffffu, incl, 31));
            for (uint32_t off = incl - cnt; cm && off < kRQ; cm &= cm - 1) rq[w][off++] = (uint16_t)((lane << 8) | (__ffsll(cm) - 1));
            __syncwarp();
            for (uint32_t it = lane; it < total; it += 32) {
              const uint32_t item = rq[w][it], ol = item >> 8, bit = item & 0xFFu;
              const uint32_t hb = R == 2 ? ((bit >> 2) & 1) : 0;          // the chunk's buffer
              const uint32_t q = bit >> 3, gs = (hb ? j0s1 : j0s0) + G * (R == 2 ? (bit & 3) : (bit & 7));
              const PermCoef c = cs[pass * 32 * NPL + ol + 32 * q];
              const uint32_t cal = c.a0 | (c.a1 << 31), ca8h = (c.a1 >> 1) << 3, clb = c.b0 + kScr4D;
              const float cAL = __uint2float_rn(cal), cAH = __uint2float_rn(c.a1 >> 1);
              const uint32_t Kq = *(volatile uint32_t*)&kq[w][q][ol];   // (stale only admits more)
              uint32_t pass_bits = 0;
#pragma unroll
              for (uint32_t u = 0; u < G; u++)
                pass_bits |= (uint32_t)(screen_u_f32(cal, ca8h, clb, cAL, cAH, xf[hb][w][gs + u]) < Kq) << u;
              uint32_t ymin = 0xFFFFFFFFu;
              while (pass_bits) {
                const uint32_t u = __ffs(pass_bits) - 1;
                pass_bits &= pass_bits - 1;
                ymin = min(ymin, eval_exact(c, xs[hb][w][gs + u]));
              }
              if (ymin < Kq - kScr4W) atomicMin(&kq[w][q][ol], ymin + kScr4W);   // (y < m: no wrap)
            }
            __syncwarp();
          }
          {   // items beyond the queue (or all of them without BAL): each lane its own
          while (cm) {
            const uint32_t bit = __ffsll(cm) - 1;
            cm &= cm - 1;
            const uint32_t hb = R == 2 ? ((bit >> 2) & 1) : 0;          // the chunk's buffer
            const uint32_t q = bit >> 3, gs = (hb ? j0s1 : j0s0) + G * (R == 2 ? (bit & 3) : (bit & 7));
            const PermCoef c = cs[pm0 + 32 * q];
            const uint32_t cal = c.a0 | (c.a1 << 31), ca8h = (c.a1 >> 1) << 3, clb = c.b0 + kScr4D;
            const float cAL = __uint2float_rn(cal), cAH = __uint2float_rn(c.a1 >> 1);
            uint32_t Kq = kq[w][q][lane];
            // re-screen the group against the current threshold, then the passing shingles exactly
            uint32_t pass = 0;
#pragma unroll
            for (uint32_t u = 0; u < G; u++)
              pass |= (uint32_t)(screen_u_f32(cal, ca8h, clb, cAL, cAH, xf[hb][w][gs + u]) < Kq) << u;
            while (pass) {
              const uint32_t u = __ffs(pass) - 1;
              pass &= pass - 1;
              const uint32_t y = eval_exact(c, xs[hb][w][gs + u]);
              if (y < Kq - kScr4W) Kq = y + kScr4W;   // (y < m <= 2^32 - 1 - W: no wrap)
            }
            kq[w][q][lane] = Kq;
          }
          }
#pragma unroll
          for (int q = 0; q < NPL; q++) K[q] = kq[w][q][lane];
        }
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < NPL; q++) {
        const uint32_t m = exact_mode ? K[q] : K[q] - kScr4W;
        const uint32_t pm = pm0 + 32 * q;
        if (p.sig_out && pm < p.num_perm) p.sig_out[(uint64_t)d * p.num_perm + pm] = m;
        if (p.bh_out) sg[w][pm] = m;
      }
    }  // pass
    if (p.bh_out) {
      __syncwarp();
      for (uint32_t jb = lane; jb < p.b; jb += 32) {
        if (p.map.ncol[jb] == 0) continue;
        uint64_t acc = 0;                               // BH_j, P:207-208 (DESIGN R6/R7)
        for (uint32_t u = 0; u < p.r; u++) {
          acc += affine32_mod_p(__ldg(p.bcoef + u), sg[w][jb * p.r + u], __ldg(p.bcoef + p.r + u));
          acc = acc >= kP ? acc - kP : acc;
        }
        p.map.ptr[jb][(uint64_t)d * p.map.ncol[jb]] = acc;
      }
      __syncwarp();
    }
  }
}

template <int NPL, int PASSES, int MINB = 2, int G = 4, int R = 1, bool BAL = true>
static int launch_s4(const MinhashParams& p, int sm_count, cudaStream_t s, int max_bps) {
  static int bps_of[2] = {0, 0};   // [gated]
  const int gi = p.landed ? 1 : 0;
  if (!bps_of[gi]) {
    if (gi) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr4<NPL, PASSES, MINB, true, G, R, BAL>, K1_THREADS, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr4<NPL, PASSES, MINB, false, G, R, BAL>, K1_THREADS, 0);
    if (bps_of[gi] < 1) bps_of[gi] = 1;
  }
  const int blocks_per_sm = bps_of[gi];
  uint64_t want = ((uint64_t)p.n_docs + K1_WARPS - 1) / K1_WARPS;
  const int bps = (max_bps > 0 && max_bps < blocks_per_sm) ? max_bps : blocks_per_sm;
  uint64_t grid = (uint64_t)sm_count * bps;
  if (want < grid) grid = want ? want : 1;
  if (p.landed) k1_minhash_scr4<NPL, PASSES, MINB, true, G, R, BAL><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  else k1_minhash_scr4<NPL, PASSES, MINB, false, G, R, BAL><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  return 1;
}

template <int NPL, bool BLOCKDOC = false>
static int launch_s(const MinhashParams& p, int sm_count, cudaStream_t s, int max_bps) {
  static int bps_of[2] = {0, 0};   // [gated]
  const int gi = p.landed ? 1 : 0;
  if (!bps_of[gi]) {
    if (gi) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr<NPL, BLOCKDOC, true>, K1_THREADS, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash_scr<NPL, BLOCKDOC, false>, K1_THREADS, 0);
    if (bps_of[gi] < 1) bps_of[gi] = 1;
  }
  const int blocks_per_sm = bps_of[gi];
  uint64_t want = BLOCKDOC ? (uint64_t)p.n_docs : ((uint64_t)p.n_docs + K1_WARPS - 1) / K1_WARPS;
  const int bps = (max_bps > 0 && max_bps < blocks_per_sm) ? max_bps : blocks_per_sm;
  uint64_t grid = (uint64_t)sm_count * bps;
  if (want < grid) grid = want ? want : 1;
  if (p.landed) k1_minhash_scr<NPL, BLOCKDOC, true><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  else k1_minhash_scr<NPL, BLOCKDOC, false><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  return 1;
}


template <int NPL, int UNR, int MINB = LB_K1_MINB, int PASSES = 1>
static int launch_t(const MinhashParams& p, int sm_count, cudaStream_t s, int max_bps) {
  static int bps_of[2] = {0, 0};   // [gated]
  const int gi = p.landed ? 1 : 0;
  if (!bps_of[gi]) {
    if (gi) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash<NPL, UNR, MINB, PASSES, true>, K1_THREADS, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_of[gi], k1_minhash<NPL, UNR, MINB, PASSES, false>, K1_THREADS, 0);
    if (bps_of[gi] < 1) bps_of[gi] = 1;
  }
  const int blocks_per_sm = bps_of[gi];
  uint64_t want = ((uint64_t)p.n_docs + K1_WARPS - 1) / K1_WARPS;
  const int bps = (max_bps > 0 && max_bps < blocks_per_sm) ? max_bps : blocks_per_sm;
  uint64_t grid = (uint64_t)sm_count * bps;
  if (want < grid) grid = want ? want : 1;
  if (p.landed) k1_minhash<NPL, UNR, MINB, PASSES, true><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  else k1_minhash<NPL, UNR, MINB, PASSES, false><<<(unsigned)grid, K1_THREADS, 0, s>>>(p);
  return 1;
}

// K1p: split this launch's documents into short (S < split_s shingles) and long ones, stably
// (each list in document order: a landing-gated launch takes its documents in list order, and
// the tokens land in document order).  K1p1 counts long documents per 1024-document block;
// K1p2 scans the counts of the preceding blocks and places each document with warp ballots.
constexpr int kPartBlock = 1024;
__device__ __forceinline__ uint32_t doc_shingles(const MinhashParams& p, uint32_t d) {
  const uint64_t L = p.offsets[d + 1] - p.offsets[d];
  return (uint32_t)(L >= p.shingle_n ? L - p.shingle_n + 1 : 1);
}
// Three classes: short (S < split_s), long, and very long (S >= vlong_s; a subset of the long
// list placed at its front, so the longest documents start first and the launch does not end on
// a warp still walking one of them).  part_blk[b] = long | very long << 16 for block b.
__global__ void __launch_bounds__(kPartBlock) k1_partition_count(const MinhashParams p, uint32_t split_s,
                                                                 uint32_t vlong_s) {
  __shared__ uint32_t wsum[kPartBlock / 32];
  if (*p.err) return;
  const uint32_t di = blockIdx.x * kPartBlock + threadIdx.x;
  const uint32_t S = di < p.n_docs ? doc_shingles(p, p.doc0 + di) : 0;
  const uint32_t bl = __ballot_sync(0xffffffffu, di < p.n_docs && S >= split_s);
  const uint32_t bv = __ballot_sync(0xffffffffu, di < p.n_docs && S >= split_s && S >= vlong_s);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = __popc(bl) | (__popc(bv) << 16);
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = wsum[threadIdx.x];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) p.part_blk[blockIdx.x] = v;
  }
}
__global__ void __launch_bounds__(kPartBlock) k1_partition_place(const MinhashParams p, uint32_t split_s,
                                                                 uint32_t vlong_s) {
  __shared__ uint32_t wl[kPartBlock / 32];
  __shared__ uint32_t base_long, base_vlong, tot_vlong;
  if (*p.err) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == 0) {   // long / very long documents in the preceding blocks; very long ones in all blocks
    uint32_t acc = 0, accv = 0, totv = 0;
    for (uint32_t b = lane; b < gridDim.x; b += 32) {
      const uint32_t v = p.part_blk[b];
      if (b < blockIdx.x) { acc += v & 0xFFFFu; accv += v >> 16; }
      totv += v >> 16;
    }
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      accv += __shfl_xor_sync(0xffffffffu, accv, o);
      totv += __shfl_xor_sync(0xffffffffu, totv, o);
    }
    if (lane == 0) { base_long = acc; base_vlong = accv; tot_vlong = totv; }
  }
  const uint32_t di = blockIdx.x * kPartBlock + threadIdx.x;
  const bool in = di < p.n_docs;
  const uint32_t S = in ? doc_shingles(p, p.doc0 + di) : 0;
  const bool lg = in && S >= split_s, vl = lg && S >= vlong_s;
  const uint32_t bl = __ballot_sync(0xffffffffu, lg), bv = __ballot_sync(0xffffffffu, vl);
  if (lane == 0) wl[w] = __popc(bl) | (__popc(bv) << 16);
  __syncthreads();
  uint32_t before = 0;                          // long | very long << 16 of the earlier warps of the block
  for (int i = 0; i < w; i++) before += wl[i];
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t rank_long = base_long + (before & 0xFFFFu) + __popc(bl & lt);     // among all long
  const uint32_t rank_vl = base_vlong + (before >> 16) + __popc(bv & lt);          // among very long
  if (in) {
    if (vl) p.part_lists[(uint64_t)p.n_docs + rank_vl] = p.doc0 + di;
    else if (lg) p.part_lists[(uint64_t)p.n_docs + tot_vlong + (rank_long - rank_vl)] = p.doc0 + di;
    else p.part_lists[di - rank_long] = p.doc0 + di;        // short rank = documents before - long before
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kPartBlock - 1) {
    const uint32_t n_long = rank_long + (lg ? 1 : 0);
    p.part_counts[0] = p.n_docs - n_long;
    p.part_counts[1] = n_long;
  }
}

// The screened kernel for long documents (LSHBLOOM_K1_SCR): 5 = the FP32 screen (default), 4 = the
// FP64 screen, 3 = the FP64 screen at 2 x 4 permutations per lane, 2 / 1 = the integer screens.
static int k1_scr_choice() {
  static const int scr = [] { const char* e = getenv("LSHBLOOM_K1_SCR"); return e ? atoi(e) : 5; }();
  return scr;
}

int launch_minhash(const MinhashParams& p, int npl, int sm_count, cudaStream_t s, int max_bps) {
  // Kernel choice (measured on B200, tools/k1_variants.py): with 128 permutations (npl 4) the
  // exact kernel wins on abstract-length documents (C2: 1203 vs ~1100 Geval/s); with 256
  // (npl 8) the screened kernel wins by 1.7x on full-text lengths (C3: 1489 vs 860 Geval/s).
  // LSHBLOOM_K1=exact|screened overrides.
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("LSHBLOOM_K1");
    mode = !e ? 2 : (e[0] == 'e' ? 0 : (e[0] == 'h' ? 3 : 1));
  }
  // 65-128 permutations (C1, C2, C5): the screen kernel (FP32 since round 2; LSHBLOOM_K1_SCR=4 the
  // FP64 one) with the documents' first 32 shingles evaluated exactly (where candidates are dense).
  // Round 1 kept the exact kernel when the caller runs K1 beside the
  // random-access Bloom kernels (L2-resident filters), whose latency-bound kernels need the SM room
  // the 92-register exact kernel leaves (C2 step 18.9 vs 19.4 ms with the screen at 2 blocks per
  // SM).  K1 alone on C2 batches: 14.1 vs 17.1 ms; C5 fused sweep step 46.6 vs 53.3 ms per 2M
  // documents (prefix 0 / 1 / 2 / 3 / 4 chunks: 18.0 / 14.1 / 14.8 / 15.7 / 16.8 ms on C2).
  // LSHBLOOM_K1=exact keeps the exact kernel everywhere, =hyb forces the screen.
  //
  // Round 2: with the FP32 screen this holds beside the random-access kernels too once K1 is capped
  // at one block (8 warps) per SM, which leaves them the registers and warp slots the exact
  // kernel's two blocks took: C2 step 18.9 -> 17.9 ms (2 / 3 blocks: 19.2 / 20.7 ms; the exact
  // kernel at one block: 19.1 ms).  LSHBLOOM_K1_SCR_BPS overrides the cap.
  if (npl == 4 && (mode == 3 || mode == 2)) {
    static const uint32_t pre = [] { const char* e = getenv("LSHBLOOM_K1_PREFIX"); return e ? (uint32_t)atoi(e) : 1u; }();
    static const int scr_bps = [] { const char* e = getenv("LSHBLOOM_K1_SCR_BPS"); return e ? atoi(e) : 1; }();
    if (mode == 2 && p.beside_random_bloom && max_bps > 0) max_bps = std::min(max_bps, scr_bps);
    MinhashParams q = p;
    q.exact_prefix = pre;
    if (k1_scr_choice() == 4) return launch_s3<4, 1, 3>(q, sm_count, s, max_bps);
    if (k1_scr_choice() == 7) return launch_s4<4, 1, 2>(q, sm_count, s, max_bps);
    if (k1_scr_choice() == 9) return launch_s4<4, 1, 3, 8>(q, sm_count, s, max_bps);
    if (k1_scr_choice() == 11) return launch_s4<4, 1, 3, 4, 1, false>(q, sm_count, s, max_bps);   // (per-lane)
    return launch_s4<4, 1, 3>(q, sm_count, s, max_bps);
  }
  if (mode == 2 && npl == 8 && p.part_lists && p.n_docs > 0) {
    // 256 permutations: the screened kernel wins on full-text lengths (C3: 1760 vs 1236 Geval/s)
    // but loses on abstracts (C2 shapes: 680 vs 1269), so split each launch by length
    // (C4 is 31M abstracts + 8M full texts) and run each part on its kernel.
    static uint32_t split_s = 0;
    if (!split_s) {
      const char* e = getenv("LSHBLOOM_K1_SPLIT_S");
      split_s = e ? (uint32_t)atoi(e) : 128u;   // (FP32 screen: C4 49.4 -> 38.7 ms per 400K at 1024 -> 128)
    }
    // very long documents first, except on landing-gated launches (the tokens land in document
    // order, and a warp waits for its document's): LSHBLOOM_K1_VLONG_S shingles (0 = off)
    static const uint32_t vlong_env = [] {
      const char* e = getenv("LSHBLOOM_K1_VLONG_S");
      return e ? (uint32_t)atoi(e) : 8192u;
    }();
    const uint32_t vlong_s = (p.landed || vlong_env == 0) ? 0xFFFFFFFFu : vlong_env;
    const unsigned pblocks = (p.n_docs + kPartBlock - 1) / kPartBlock;
    k1_partition_count<<<pblocks, kPartBlock, 0, s>>>(p, split_s, vlong_s);
    k1_partition_place<<<pblocks, kPartBlock, 0, s>>>(p, split_s, vlong_s);
    MinhashParams a = p, b = p;
    a.list = p.part_lists;
    a.list_n = p.part_counts;
    b.list = p.part_lists + p.n_docs;
    b.list_n = p.part_counts + 1;
    auto short_docs = [&] {
      cudaMemsetAsync(p.counter, 0, 4, s);
      if (max_bps == 0) launch_t<4, LB_UNR4, 4, 2>(a, sm_count, s, 0);   // 256 = 2 passes x 4 x 32
      else launch_t<4, LB_UNR4, LB_K1_MINB, 2>(a, sm_count, s, max_bps);
    };
    // With a landing gate (host batch still being copied) the long documents go first: the short
    // ones (~2 % of C3's) are spread over the whole batch, and their kernel would wait for the
    // copy's end with every warp parked on one of them.
    static const bool long_first_env = [] { const char* e = getenv("LSHBLOOM_K1_LONG_FIRST"); return e && atoi(e); }();
    const bool long_first = p.landed || long_first_env;
    if (!long_first) short_docs();
    // long documents: a warp each when there are enough of them to balance the warps (>= 16 per
    // resident warp), else a block each (a few thousand full texts over ~2400 warps would last as
    // long as the slowest warp: C4's fused step 43.9 -> 37.2 ms); both kernels are launched and
    // the one the device-side count does not select returns at once
    b.block_gate = 16u * (uint32_t)sm_count * 2u * K1_WARPS;
    cudaMemsetAsync(p.counter, 0, 4, s);
    // warp-per-document long documents: the FP64-screen kernel, 8 permutations per lane in one
    // pass (128 registers, 2 blocks per SM; C3 200K full texts alone: 81.2 ms; 2 x 4 per lane at 3
    // blocks, LSHBLOOM_K1_SCR=3: 90.4 ms; the integer screens: 101.8 ms k1_minhash_scr2 = 2,
    // 111.4 ms k1_minhash_scr = 1; a min over each 4-shingle group with the mask bits built in a
    // branch: 86.1 ms; the same min with the flagged groups re-screened after the chunk: 109.8 ms)
    const int scr = k1_scr_choice();
    static const uint32_t lpre = [] { const char* e = getenv("LSHBLOOM_K1_LPREFIX"); return e ? (uint32_t)atoi(e) : 1u; }();
    if (scr >= 5) b.exact_prefix = lpre;
    if (scr == 1) launch_s<8, false>(b, sm_count, s, max_bps);
    else if (scr == 2) launch_s2<8, 1>(b, sm_count, s, max_bps);
    else if (scr == 3) launch_s3<4, 2>(b, sm_count, s, max_bps);
    else if (scr == 4) launch_s3<8, 1, 2>(b, sm_count, s, max_bps);
    else if (scr == 6) launch_s4<8, 1, 3>(b, sm_count, s, max_bps);   // (3 blocks per SM: diagnostic)
    else if (scr == 8) launch_s4<8, 1, 2, 4>(b, sm_count, s, max_bps);   // (4-shingle groups: diagnostic)
    else if (scr == 10) launch_s4<8, 1, 2, 8, 1>(b, sm_count, s, max_bps);   // (resolution every chunk: diagnostic)
    else if (scr == 11) launch_s4<8, 1, 2, 8, 2, true>(b, sm_count, s, max_bps);   // (balanced resolution: diagnostic)
    else launch_s4<8, 1, 2, 8, 2, false>(b, sm_count, s, max_bps);
    cudaMemsetAsync(p.counter, 0, 4, s);
    launch_s<8, true>(b, sm_count, s, max_bps);
    if (long_first) short_docs();
    return 5;
  }
  const bool screened = mode == 1 || (mode == 2 && npl >= 8);
  if (screened && npl <= 8) {
    switch (npl) {
      case 1: return launch_s<1>(p, sm_count, s, max_bps);
      case 2: return launch_s<2>(p, sm_count, s, max_bps);
      case 4: return launch_s<4>(p, sm_count, s, max_bps);
      case 8: return launch_s<8>(p, sm_count, s, max_bps);
    }
  }
  switch (npl) {
    case 1: return launch_t<1, 4>(p, sm_count, s, max_bps);
    case 2: return launch_t<2, 4>(p, sm_count, s, max_bps);
    // alone (max_bps == 0: signatures, band hashes, the sharded paths) K1 takes the whole GPU
    // and a 64-register build runs 4 blocks per SM (1467 vs 1421 Geval/s on C2); beside the
    // Bloom kernels (fused query_insert) the 92-register build at 2 blocks per SM leaves them
    // room (19.6 vs 20.5+ ms per C2 step, tools/k1_variants.py + bench.py)
    case 4: return max_bps == 0 ? launch_t<4, LB_UNR4, 4>(p, sm_count, s, 0)
                                : launch_t<4, LB_UNR4>(p, sm_count, s, max_bps);
    case 8: return launch_t<8, 2>(p, sm_count, s, max_bps);
    case 16: return launch_t<16, 2>(p, sm_count, s, max_bps);
    case 32: return launch_t<32, 2>(p, sm_count, s, max_bps);
    default: return -1;
  }
}

// K0: CSR validation (S:64 empty document; malformed offsets).
__global__ void k0_validate(const uint64_t* __restrict__ off, uint64_t n, ErrState* err) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && off[0] != 0) atomicOr(&err->flags, 1);
  if (i < n) {
    uint64_t a = off[i], b = off[i + 1];
    if (b < a) atomicOr(&err->flags, 1);
    else if (b == a) atomicMin(&err->first_empty, (unsigned long long)i);
  }
}

__global__ void k0_fold(ErrState* err, int* gate) {
  *gate = (err->flags != 0 || err->first_empty != ~0ull) ? 1 : 0;
}

int launch_validate(const uint64_t* offsets, uint64_t n_docs, ErrState* err, cudaStream_t s) {
  unsigned grid = (unsigned)((n_docs + 255) / 256);
  k0_validate<<<grid ? grid : 1, 256, 0, s>>>(offsets, n_docs, err);
  k0_fold<<<1, 1, 0, s>>>(err, &err->pad);
  return 2;
}

}  // namespace lb
