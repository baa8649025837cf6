// lb_internal.h -- kernel parameter blocks and launchers shared by the library's .cu files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lb_common.cuh"

namespace lb {

constexpr int kMaxBands = 64;

// Where the K1 epilogue writes band hash j of batch document d (d indexes the whole batch,
// not the launch's chunk):  ptr[j][d * ncol[j]]  (skip ncol[j] == 0).  The host builds ptr[j]
// either inside one local output, bh_out + blockstart[j] + col[j], or inside the owner rank's
// receive buffer in peer memory (lshbloom_band_hashes_to_peers), so the same epilogue stores
// band hashes locally or straight across NVLink.
struct BandMap {
  uint64_t blockstart[kMaxBands];
  uint32_t ncol[kMaxBands];
  uint32_t col[kMaxBands];
  uint64_t* ptr[kMaxBands];
};

constexpr int kMaxPeers = 64;

// Where a (document, band) hit raises its document's duplicate flag.  Local: dup[i] = 1.  Peer
// mode (lshbloom_query_insert_bands_peers, world = npeers > 0): document i of the global batch
// belongs to rank r with start[r] <= i < start[r + 1] and its flag lives in that rank's buffer
// peer[r] (peer memory over NVLink), so the OR over band owners is done by the stores themselves
// (every writer stores the same value 1) instead of an all-reduce.
struct DupSink {
  uint8_t* local;
  uint32_t npeers;
  uint8_t* peer[kMaxPeers];
  uint64_t start[kMaxPeers + 1];
};

__device__ __forceinline__ void raise_dup(const DupSink& d, uint32_t i) {
  if (d.npeers == 0) {
    d.local[i] = 1;
    return;
  }
  uint32_t lo = 0, hi = d.npeers;                 // largest r with start[r] <= i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (d.start[mid] <= i) lo = mid;
    else hi = mid;
  }
  d.peer[lo][i - d.start[lo]] = 1;
}

struct ErrState {
  int flags;                 // bit0: usage (offsets[0] != 0 or decreasing); bit1: landing-gate timeout
  int pad;
  unsigned long long first_empty;  // first empty document (~0 if none)
};

struct MinhashParams {
  const uint64_t* offsets;   // batch offsets (device), n+1
  const uint32_t* tokens;    // device tokens; document d starts at tokens[offsets[d] - tok_base]
  uint64_t tok_base;
  uint32_t doc0;             // first batch document of this launch
  uint32_t n_docs;           // documents in this launch
  uint32_t* counter;         // work counter (zeroed before launch)
  uint32_t shingle_n;
  uint32_t sh29, sh3;         // the constants 29 and 3 (kept opaque to ptxas)
  uint64_t fp_init_n;        // mix64(kFpSalt + shingle_n)
  const PermCoef* coef;      // [32 * npl] (padded)
  uint32_t num_perm;
  uint32_t* sig_out;         // [n][num_perm] (batch-indexed) or null
  uint64_t* bh_out;          // band hashes (see BandMap) or null
  uint32_t b, r;
  const uint64_t* bcoef;     // c[0..r), d[0..r)
  BandMap map;
  const int* err;            // nonzero: batch rejected, do nothing
  // Length-partitioned launches (npl >= 8): this launch handles batch documents list[0, *list_n)
  // instead of [doc0, doc0 + n_docs); part_* is scratch for the partition (2 lists of n_docs).
  const uint32_t* list;
  const uint32_t* list_n;
  uint32_t* part_lists;      // [2][n_docs]: short documents, long documents
  uint32_t* part_counts;     // [2]
  uint32_t* part_blk;        // [ceil(n_docs / 1024)]: long documents per partition block
  uint32_t block_gate;       // screened kernel: block-per-document mode iff *list_n < block_gate
  uint32_t exact_prefix;     // FP64-screen kernel: 32-shingle chunks evaluated exactly before screening
  uint32_t beside_random_bloom;  // K1 runs beside the random-access Bloom kernels (kernel choice only)
  // Landing gate (host batches streamed into one device token buffer while K1 runs): the copy
  // engine lands the tokens in pieces of 2^land_log2 tokens, in order, and after piece i a
  // stream memory operation (no SM involved) writes *landed = i + 1.  A warp starts document d
  // only when every 128-B line it can touch has landed -- tokens [0, roundup32(offsets[d+1]))
  // clipped to tok_total -- so no SM ever caches a line that is still being written.  Null:
  // the tokens are resident.  A wait beyond kLandTimeoutNs sets err_state->flags bit 1 and the
  // gate (the batch is rejected with LSHBLOOM_ECUDA instead of hanging the device).
  const uint32_t* landed;
  uint32_t land_log2;
  uint64_t tok_total;
  ErrState* err_state;
};

struct BloomParams {
  uint32_t* F;               // owned filters, bl * W uint32 words
  uint64_t* Q;               // compact earliest-setter table of this sub-batch (2^q_log2 slots)
  uint32_t q_log2;
  uint64_t W;                // uint32 words per band
  uint64_t m, m_inv;         // probe modulus and Barrett reciprocal
  uint64_t nb, nb_inv;       // blocked variant: 1024-bit blocks per band and Barrett reciprocal
  uint32_t k, bl;            // probes, owned bands
  const uint64_t* s1;        // [bl] filter seeds of the owned bands (global band index)
  const uint64_t* s2;
  uint64_t* ekey;            // overflow earliest-setter table (open addressing), 2^ecap_log2 slots
  uint64_t* eval;
  uint32_t ecap_log2;
  uint64_t gen;              // sub-batch generation tag (1 .. 2^22-1)
  const uint64_t* bh;        // band hashes of the batch: owned band jl of doc i at bh[jl*bh_sj + i*bh_si]
  uint64_t bh_sj, bh_si;     //   ([bl][n] band-major from K1: (n, 1); [n][bl] row-major: (1, bl))
  uint32_t i0, nsb;          // sub-batch = batch documents [i0, i0 + nsb); thread idx = jl * nsb + (i - i0)
  uint64_t* st_pre;          // [nsb * bl] per (doc, band): pre-set probe mask (K3)
  uint64_t* st_arr;          //   and first-arrival probe mask (K4)
  uint32_t* cand;            // candidate (doc, band) pairs
  uint32_t* cand_count;      //   and their count; cand_count[1] counts clist
  uint64_t* clist;           // contested probes of the sub-batch, packed (band, position) << 22 | doc - i0
  uint32_t* cb;              // contested-position summary: 2^cb_log2 bits, bit hash(band, position)
  uint32_t cb_log2;
  DupSink dup;               // [n] batch flags (OR over owned bands), local or in peer memory
  const int* err;
};

// Window-sweep Bloom stage (lb_sweep.cu).  Each band's filter is cut into windows of 2^wb bits;
// K7 bins every probe of a batch by (band, window) into fixed-capacity bins (records
// (position in window) << 32 | (document - i0)), K8 streams each non-empty window HBM -> shared
// memory with a TMA bulk copy, applies all of its records with the stream-order lemma in shared
// memory and writes the window back (one read + one write of every touched filter line per batch
// instead of two random line fetches per probe), K9 turns the per-(document, band) miss bits into
// duplicate flags.  A bin that exceeds its capacity switches the whole sweep to an exact layout
// (scan of the bin counts + re-scatter), decided on the device.
struct SweepParams {
  BloomParams g;             // geometry, seeds, filters, band hashes, dup sink, error gate
  uint32_t wb;               // log2 window bits (10..19)
  uint32_t cap;              // records per window bin in the fixed-capacity layout
  uint64_t nw;               // windows per band = ceil(m / 2^wb)
  uint64_t nbins;            // bl * nw, band-major
  uint32_t* cursor;          // [nbins] records (+ sentinel padding) per window bin
  uint32_t* cursor2;         // [nbins] exact-layout scatter cursors
  uint64_t* start;           // [nbins + 1] exact layout: exclusive scan of cursor
  uint64_t* rec;             // records: fixed layout bin * cap + slot, exact layout start[bin] + slot
  uint32_t* ovf;             // nonzero: some bin exceeded its capacity -> exact layout
  uint64_t* miss;            // [n] bit jl set: band jl of sweep document d missed
  uint32_t* eg;              // [grid][2^wb] earliest setter per position, for bins beyond kSweepCapReg
  uint32_t i0, n;            // this sweep = batch documents [i0, i0 + n)
  uint32_t stages;           // K8 pipeline depth (windows + records in flight per CTA)
  // two-level binning (k = 17): K7a sorts each 512-document tile's records by coarse bucket
  // (2^cb windows) in shared memory and writes them as runs; K7b re-sorts each coarse bucket by
  // window in 4096-record chunks -- every record is written in coalesced runs, never scattered
  uint32_t two_level;        // 1: K7a + K7b; 0: K7 writes records straight into window bins
  uint32_t cb;               // log2 windows per coarse bucket
  uint64_t ncb;              // coarse buckets per band = ceil(nw / 2^cb) (<= kSweepMaxCoarse)
  uint32_t ccap;             // records (+ padding) per coarse bucket
  uint32_t* ccursor;         // [bl * ncb]
  uint64_t* crec;            // [bl * ncb * ccap]
};

struct ClassicParams {        // classic MinHashLSH index (lb_classic.cu)
  uint64_t* keys;            // [bl][2^log2cap] band hashes (~0 = empty slot)
  uint64_t* vals;            // [bl][2^log2cap] earliest global document index per key
  uint32_t log2cap, bl;
  uint64_t doc_base;         // global index of batch document 0
  const uint64_t* bh;        // band hashes: owned band jl of doc i at bh[jl*bh_sj + i*bh_si]
  uint64_t bh_sj, bh_si;
  uint32_t i0, n;            // batch documents [i0, i0 + n)
  DupSink dup;               // [batch] flags (OR over owned bands), local or in peer memory
  int* full;                 // set if a probe sequence wrapped (cannot happen at load <= 0.9)
  const int* err;
};

// launchers (return number of kernel launches issued)
int launch_validate(const uint64_t* offsets, uint64_t n_docs, ErrState* err, cudaStream_t s);
int launch_minhash(const MinhashParams& p, int npl, int sm_count, cudaStream_t s, int max_bps);
int launch_bloom_subbatch(const BloomParams& p, int sm_count, cudaStream_t s);
int launch_classic(const ClassicParams& p, cudaStream_t s);
int launch_sweep_bin(const SweepParams& p, uint32_t lo, uint32_t hi, cudaStream_t s);
int launch_sweep_finish(const SweepParams& p, int grid, cudaStream_t s);
struct SweepLaunch { int grid; uint32_t stages; size_t smem; };
SweepLaunch sweep_launch_cfg(int sm_count, uint32_t wb);   // K8 persistent grid / pipeline depth
int sweep_grid(int sm_count, uint32_t wb);                 // = sweep_launch_cfg().grid
// [n][bl] -> columns [col0, col0 + n) of a [bl][ld] buffer (ld = 0: ld = n)
int launch_transpose_bh(const uint64_t* in, uint64_t* out, uint32_t n, uint32_t bl, cudaStream_t s,
                        uint64_t ld = 0, uint64_t col0 = 0);
constexpr int kSweepThreads = 256;               // K8 block size
constexpr int kSweepRPT = 4;                     // records per thread held in registers
constexpr uint32_t kSweepCapReg = kSweepThreads * kSweepRPT;   // 1024: larger bins take the global path
constexpr uint32_t kSweepMaxCoarse = 1024;       // coarse buckets per band (K7a: one per thread)
constexpr uint32_t kSweepTileDocs = 1024;        // K7a: documents per tile (= threads)
constexpr uint32_t kSweepMaxW = 256;             // K7b: windows per coarse bucket (line staging each)
constexpr uint32_t kSweepStage = 32;             // K7b: staged records per window (flushed in 16s)
constexpr uint32_t kSweepBThreads = 512;         // K7b block size
constexpr uint32_t kSweepChunk = 2048;           // K7b: records per chunk (4 per thread)

}  // namespace lb
