// lb_classic.cu -- the classic MinHashLSH index on the GPU.
//
// MinHashLSH declares a candidate pair when two documents' band hashes are exactly equal in
// some band ("if two bands of the MinHash signature matrix are exactly identical for two
// documents ... then those two documents have Jaccard similarity greater than or equal to T";
// S:186-189).  In stream order a document is a (classic) duplicate iff one of its
// band hashes was inserted by an earlier document; then all its band hashes are inserted.  It
// is the exact reference LSHBloom's Bloom filters approximate (LSHBloom's duplicates
// contain the classic ones), and the index whose size the paper contrasts with its own.
//
// Per owned band, an open-addressing table of `cap` slots: key = band hash (< P = 2^61-1, so
// ~0 marks an empty slot) and value = the earliest global document index holding that key.
// Because every document inserts (unconditionally) all its band hashes, the stream-order
// verdict is a single pass over any batch:
//     hit_j(i) = E_j[BH_j(i)] < i,   E_j[v] = min{ i' : BH_j(i') = v }
// (the same earliest-setter lemma as the Bloom stage, with the key itself in place
// of k bit positions).  Two launches per batch: KC1 inserts every (doc, band) key and takes
// the minimum document index with atomicMin; KC2 reads each key's minimum back.
#include <cstdint>

#include "lb_internal.h"

namespace lb {

#ifndef KC_THREADS
#define KC_THREADS 256
#endif

__device__ __forceinline__ uint64_t cslot(uint64_t key, uint32_t log2cap) {
  return (key * 0x9E3779B97F4A7C15ull) >> (64 - log2cap);
}

__global__ void __launch_bounds__(KC_THREADS) kc_insert(const ClassicParams p) {
  // grid (doc blocks, bands): blocks run x-fastest, so a wave works in one band's table
  const uint64_t il = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t jl = blockIdx.y;
  if (*p.err || il >= p.n) return;
  const uint32_t i = p.i0 + (uint32_t)il;
  const uint64_t key = p.bh[(uint64_t)jl * p.bh_sj + (uint64_t)i * p.bh_si];
  const unsigned long long gdoc = p.doc_base + i;
  unsigned long long* keys = (unsigned long long*)p.keys + ((uint64_t)jl << p.log2cap);
  unsigned long long* vals = (unsigned long long*)p.vals + ((uint64_t)jl << p.log2cap);
  const uint64_t mask = (1ull << p.log2cap) - 1;
  uint64_t s = cslot(key, p.log2cap);
  LB_ASSERT(key < 0x1FFFFFFFFFFFFFFFull);
  for (uint64_t n = 0; n <= mask; n++, s = (s + 1) & mask) {
    unsigned long long cur = __ldcg(keys + s);
    if (cur == ~0ull) {
      cur = atomicCAS(keys + s, ~0ull, (unsigned long long)key);
      if (cur == ~0ull) cur = key;                      // claimed the slot
    }
    if (cur == key) {
      atomicMin(vals + s, gdoc);
      return;
    }
  }
  atomicOr((int*)p.full, 1);   // unreachable while the host keeps the load factor <= 0.9
}

__global__ void __launch_bounds__(KC_THREADS) kc_verdict(const ClassicParams p) {
  const uint64_t il = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t jl = blockIdx.y;
  if (*p.err || il >= p.n) return;
  const uint32_t i = p.i0 + (uint32_t)il;
  const uint64_t key = p.bh[(uint64_t)jl * p.bh_sj + (uint64_t)i * p.bh_si];
  const unsigned long long* keys = (const unsigned long long*)p.keys + ((uint64_t)jl << p.log2cap);
  const unsigned long long* vals = (const unsigned long long*)p.vals + ((uint64_t)jl << p.log2cap);
  const uint64_t mask = (1ull << p.log2cap) - 1;
  uint64_t s = cslot(key, p.log2cap);
  for (uint64_t n = 0; n <= mask; n++, s = (s + 1) & mask) {
    const unsigned long long cur = __ldcg(keys + s);
    if (cur == key) {
      if (__ldcg(vals + s) < p.doc_base + i) raise_dup(p.dup, i);   // an earlier document holds it
      return;
    }
    LB_ASSERT(cur != ~0ull);                                 // KC1 inserted every key
    if (cur == ~0ull) return;
  }
}

int launch_classic(const ClassicParams& p, cudaStream_t s) {
  const dim3 grid((unsigned)(((uint64_t)p.n + KC_THREADS - 1) / KC_THREADS), p.bl);   // (doc blocks, bands)
  kc_insert<<<grid, KC_THREADS, 0, s>>>(p);
  kc_verdict<<<grid, KC_THREADS, 0, s>>>(p);
  return 2;
}

}  // namespace lb
