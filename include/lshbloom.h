/*
 * lshbloom.h -- C-ABI of the B200-native LSHBloom hot path (arXiv 2411.04257).
 *
 * The library computes, for every document of a CSR batch of uint32 word ids:
 *   word n-gram shingle fingerprints,
 *   a num_perm-wide MinHash signature sig[i] = min_x ((a_i x + b_i) mod (2^61-1)) mod 2^32
 *     (S:132-140),
 *   b band hashes over r rows each, BH_j = (sum_u (c_u sig[j r + u] + d_u) mod P) mod P
 *     (S:202-210),
 *   a k-probe query-then-insert of each band hash into that band's own Bloom filter of
 *     m = ceil(-n ln p / (ln 2)^2) bits, k = max(1, round((m/n) ln 2)) probes
 *     (S:263),
 *   and the duplicate flag = OR over bands ("If there is a collision for any band of
 *     signatures, we mark that document as a duplicate").
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.  Every convention the paper
 * leaves open (fingerprint, family PRNG, truncation order, probe derivation) is fixed in
 * DESIGN.md section 3; outputs are bit-identical to the CPU oracle in oracle/.
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  - Return codes mirror SPEC's exit codes:
 *      LSHBLOOM_OK 0, LSHBLOOM_EUSAGE 1 (bad argument / NULL pointer / malformed offsets),
 *      LSHBLOOM_EDATA 2 (an empty document, S:64 -- the whole batch is rejected before any
 *      filter is modified; lshbloom_last_error names the first bad index),
 *      LSHBLOOM_ERUNTIME 3 (CUDA failure: the handle is poisoned and every later call
 *      returns 3), LSHBLOOM_ENOMEM 4 (device allocation failed).
 *  - Ownership: the caller owns every batch and output buffer; outputs live in the same
 *    memory space as the batch (device memory of the handle's GPU when on_device = 1, host
 *    memory otherwise; pinned host memory enables overlapped copies).  The library owns
 *    filters, coefficients and scratch (cudaMalloc) and frees them in lshbloom_destroy.
 *  - A handle is not thread-safe.  query_insert calls are serialised by the caller and
 *    their order is the stream order.  Every call except
 *    lshbloom_query_insert_async (and lshbloom_reset while async batches are in flight) is
 *    complete when it returns.
 *  - Outputs are pure functions of (parameters, seed, ordered concatenation of batches):
 *    independent of batch boundaries, GPU count and launch configuration.
 */
#ifndef LSHBLOOM_H
#define LSHBLOOM_H

#include <stdint.h>

#if defined(__GNUC__)
#define LSHBLOOM_API __attribute__((visibility("default")))
#else
#define LSHBLOOM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define LSHBLOOM_OK 0
#define LSHBLOOM_EUSAGE 1
#define LSHBLOOM_EDATA 2
#define LSHBLOOM_ERUNTIME 3
#define LSHBLOOM_ENOMEM 4
#define LSHBLOOM_EFORMAT 5     /* checkpoint: bad magic / unsupported version / inconsistent header */
#define LSHBLOOM_ETRUNC 6      /* checkpoint: file shorter than its header says */
#define LSHBLOOM_ECHECKSUM 7   /* checkpoint: CRC32C mismatch */
#define LSHBLOOM_EIO 8         /* checkpoint: open / read / write failure */

#define LSHBLOOM_MAX_BANDS 64   /* bands per handle */
#define LSHBLOOM_MAX_PERM 1024  /* num_perm */
#define LSHBLOOM_MAX_K 64       /* probes per band hash (p >= ~5e-20) */
#define LSHBLOOM_NSTAGES 3      /* lshbloom_stage_times entries */

typedef struct lshbloom lshbloom; /* opaque */

/* A CSR batch.  Document d is tokens[offsets[d], offsets[d+1]).
 *   n_docs    >= 1 and < 2^32
 *   offsets   n_docs+1 entries, offsets[0] = 0, non-decreasing; an equal pair is an
 *             empty document (error 2)
 *   tokens    offsets[n_docs] word ids (any uint32 value, including 0)
 *   on_device 1: offsets/tokens (and outputs) are device pointers on the handle's GPU;
 *             0: host pointers (pinned preferred) -- host<->device copies are done inside
 *   stream    cudaStream_t to run on (NULL: the handle's own stream) */
typedef struct {
    uint64_t n_docs;
    const uint64_t *offsets;
    const uint32_t *tokens;
    int32_t on_device;
    void *stream;
} lshbloom_batch;

/* Extended configuration (lshbloom_create fills shingle_n = 5, device = current,
 * rank = 0, world = 1, sub_batch = 0 = default). */
typedef struct {
    uint32_t num_perm;   /* 1..LSHBLOOM_MAX_PERM */
    uint32_t b;          /* bands, 1..LSHBLOOM_MAX_BANDS */
    uint32_t r;          /* rows per band, b*r <= num_perm */
    uint32_t shingle_n;  /* word n-gram width, >= 1 (DESIGN R2: 5) */
    uint64_t n_expected; /* capacity n of every filter, >= 1 */
    double fp_rate;      /* per-filter false-positive rate p in (0,1) (DESIGN R8) */
    uint64_t seed;       /* hash-family seed (DESIGN R5) */
    int32_t device;      /* CUDA device ordinal, -1 = current */
    uint32_t rank;       /* band sharding: this rank owns bands [band_lo, band_hi) */
    uint32_t world;      /*   over world ranks (bands split as evenly as possible) */
    uint32_t sub_batch;  /* documents per Bloom sub-batch (0 = default 32768); results do
                            not depend on it */
    uint32_t index_kind; /* LSHBLOOM_INDEX_BLOOM (0, the paper's method),
                            LSHBLOOM_INDEX_CLASSIC (1) or LSHBLOOM_INDEX_BLOCKED (2); see below */
    uint32_t bloom_path; /* how a batch is applied to Bloom filters (results never depend on it):
                            LSHBLOOM_PATH_AUTO (0), _RANDOM (1) or _SWEEP (2); see below */
    uint32_t sweep_log2_window; /* sweep window 2^w bits, w in [10, 19] (0 = chosen per batch) */
    uint32_t sweep_cap;  /* sweep records per bin before the exact layout (0 = from the batch's
                            expected load; tests use tiny values to force the exact layout) */
    double lsh_threshold;/* Jaccard threshold T the (b, r) were chosen for, carried
                            into the LSHB checkpoint header; 0 = unknown: the header then holds
                            (1/b)^(1/r), the S-curve's approximate threshold.  No effect on results */
} lshbloom_config;

/* Bloom paths.  Both evaluate the same stream-order rule -- bit g of band j is set before
 * document i iff it was set before the batch or some earlier document of the batch probes g
 * (every document inserts all its band hashes) -- and give identical results:
 * LSHBLOOM_PATH_RANDOM: per sub-batch of documents, every probe reads and atomically sets its
 *   filter word in place (K3-K6): the fast form while the filters fit in L2 (<= ~64 MB) or a
 *   batch probes few lines of large filters.
 * LSHBLOOM_PATH_SWEEP: probes are binned by filter window (2^w bits), then every touched window
 *   is copied HBM -> shared memory once (TMA bulk copy), updated there for all of its probes,
 *   and written back once (K7-K9): one read + one write per touched filter line per batch
 *   instead of two random 128-byte line fetches per probe -- the fast form for dense batches on
 *   HBM-resident filters (C3-C5).  Batches of more than 4,194,304 documents are swept in
 *   pieces of that size.
 * LSHBLOOM_PATH_AUTO: the sweep when the owned filters exceed 96 MB and a batch puts at least
 *   256 probes per 64 KB window, else random access.  (Environment LSHBLOOM_BLOOM_PATH =
 *   random|sweep overrides AUTO for experiments.) */
#define LSHBLOOM_PATH_AUTO 0
#define LSHBLOOM_PATH_RANDOM 1
#define LSHBLOOM_PATH_SWEEP 2

/* Index kinds.
 * LSHBLOOM_INDEX_BLOOM: one Bloom filter per band -- the paper's method.
 * LSHBLOOM_INDEX_CLASSIC: the classic MinHashLSH index it replaces (P:134 exact band
 *   equality): per band the set of band hashes seen, a document being a
 *   duplicate iff one of its band hashes was inserted by an earlier document.  Same entry
 *   points and stream semantics; no false positives beyond LSH's own (the Bloom
 *   index's duplicates contain these).  Device memory: per owned band 16 B x cap slots,
 *   cap = the power of two >= n_expected / 0.7; a batch that would take doc_count past
 *   0.9 cap is rejected (error 1) before any mutation.  fp_rate is ignored; filter_copy and
 *   save/load return error 1. */
#define LSHBLOOM_INDEX_BLOOM 0
#define LSHBLOOM_INDEX_CLASSIC 1
/* LSHBLOOM_INDEX_BLOCKED: a blocked Bloom variant (not the paper's filter,
 *   whose layout SPEC S:328 leaves open): each filter is nb = ceil(m / 1024) blocks of 1024
 *   bits (one 128-byte line, the unit B200 moves from HBM per random access) and all k probes
 *   of a band hash fall in one block: block = h1 mod nb, offset_t = bits [10 (t mod 6),
 *   10 (t mod 6) + 10) of mix64(h2 + floor(t / 6)), position = 1024 block + offset_t (h1, h2 as
 *   for the standard filter, DESIGN R10).  m, k from (n_expected, fp_rate) as for the standard
 *   filter, m rounded up to whole blocks; same stream semantics, 1 random line per (document,
 *   band) instead of k.  Its false-positive rate at capacity is the Poisson mixture
 *   sum_i Pois(i; n/nb) (1 - (1 - 1/1024)^(k i))^k (3.4x p at p = 1e-5, k = 17): ask for a
 *   smaller fp_rate to compensate.  save/load return error 1. */
#define LSHBLOOM_INDEX_BLOCKED 2

typedef struct {
    uint64_t m;               /* bits per filter (analytic, the probe modulus) */
    uint32_t k;               /* probes per band hash */
    uint32_t num_perm, b, r, shingle_n;
    uint32_t band_lo, band_hi;/* owned bands (global indices) */
    uint64_t words_per_band;  /* uint32 words per filter = 4*ceil(m/128): the S:314 storage
                                 rounded up to 16 bytes (TMA bulk-copy granularity); padding bits
                                 are never set */
    uint64_t filter_bytes;    /* device bytes of the owned filters */
    double p_eff;             /* 1-(1-p)^b */
    uint64_t doc_count;       /* documents inserted so far */
    int32_t oversubscribed;   /* doc_count > n_expected */
    uint64_t seed;
    uint64_t n_expected;
    double fp_rate;
    uint32_t index_kind;      /* LSHBLOOM_INDEX_BLOOM / _CLASSIC / _BLOCKED */
    uint64_t classic_slots;   /* classic: table slots per band (0 for Bloom) */
    uint64_t sweeps;          /* batches (or 4M-document pieces) applied by the sweep path */
    double lsh_threshold;     /* the configured Jaccard threshold (0 = unknown) */
} lshbloom_info_t;

/* Create an index of b Bloom filters: sizes them from (n_expected, fp_rate),
 * expands the hash family from seed and zeroes the filters.  shingle n = 5.
 * On error *out is NULL and lshbloom_last_error(NULL) describes it. */
LSHBLOOM_API int lshbloom_create(uint32_t num_perm, uint32_t b, uint32_t r, uint64_t n_expected,
                    double fp_rate, uint64_t seed, lshbloom **out);
LSHBLOOM_API int lshbloom_create_ex(const lshbloom_config *cfg, lshbloom **out);

/* Release every resource; NULL-safe. */
LSHBLOOM_API void lshbloom_destroy(lshbloom *h);

/* MinHash signatures sig_out[n_docs][num_perm] (uint32, row-major).  Pure: no filter
 * state is read or written.  Rows >= b*r are computed too. */
LSHBLOOM_API int lshbloom_signatures(lshbloom *h, const lshbloom_batch *batch, uint32_t *sig_out);

/* Band hashes bh_out[n_docs][b] (uint64, values < 2^61-1) for ALL b bands.  Pure. */
LSHBLOOM_API int lshbloom_band_hashes(lshbloom *h, const lshbloom_batch *batch, uint64_t *bh_out);

/* Band hashes of ALL b bands laid out for the band-sharded exchange (world > 1): one
 * contiguous block per owner rank o = 0..world-1, block o = [n_docs][band_hi(o)-band_lo(o)]
 * (global band j of document d at block_start(o) + d*(hi-lo) + (j-lo)), so that the
 * all-to-all sends block o to rank o unchanged.  With world = 1 identical to
 * lshbloom_band_hashes.  Pure. */
LSHBLOOM_API int lshbloom_band_hashes_sharded(lshbloom *h, const lshbloom_batch *batch, uint64_t *bh_out);

/* Query-then-insert every document of the batch in stream order against the owned band
 * filters (all bands when world = 1): dup_out[d] = 1 iff some owned band's k probe bits
 * were all set before document d (by earlier batches or earlier documents of this batch),
 * else 0; then all band hashes are inserted (insert is unconditional).  Mutates the
 * filters.  With world > 1 the flags cover only the owned bands (combine with a max over
 * ranks; see lshbloom_query_insert_bands and paper_2411_04257_b200.sharded). */
LSHBLOOM_API int lshbloom_query_insert(lshbloom *h, const lshbloom_batch *batch, uint8_t *dup_out);

/* Asynchronous form of lshbloom_query_insert, for streams of batches (the index is a
 * stream; S:427 serial order).  Enqueues the batch and returns without waiting: the batch's
 * MinHash kernels run while the previous batch's Bloom stage is still working, and Bloom stages
 * run in call order, so the flags are exactly those of the synchronous calls in the same order.
 * At most two batches are in flight; a third call first waits for the oldest.  dup_out, and for
 * host batches the offsets / tokens (pinned memory, or the copies serialise), must stay valid
 * and unmodified until lshbloom_sync returns.  Host-checkable errors (NULL pointers, offsets[0],
 * chunk bounds) are returned at once; the device-side verdict on the CSR (malformed offsets,
 * empty document) is returned by lshbloom_sync -- a rejected batch inserts nothing, later
 * batches are processed normally.  Other entry points wait for the batches in flight first;
 * lshbloom_reset does not (it is ordered on the device between the batches around it). */
LSHBLOOM_API int lshbloom_query_insert_async(lshbloom *h, const lshbloom_batch *batch, uint8_t *dup_out);

/* Wait for every batch enqueued with lshbloom_query_insert_async; returns the first device-side
 * error among them (1 or 2, lshbloom_last_error names it) or 0, and clears it. */
LSHBLOOM_API int lshbloom_sync(lshbloom *h);

/* Bloom stage only, for band-sharded use: bh_owned[n_docs][band_hi-band_lo] holds the
 * band hashes of the owned bands for n_docs documents in global stream order;
 * hit_out[n_docs] = OR over the owned bands of the per-band verdicts.  Pointers are device
 * pointers when on_device = 1, host otherwise.  Mutates the owned filters. */
LSHBLOOM_API int lshbloom_query_insert_bands(lshbloom *h, const uint64_t *bh_owned, uint64_t n_docs,
                                int32_t on_device, void *stream, uint8_t *hit_out);

/* A batch of the owned bands assembled from band-hash chunks, for pipelined sharded steps: the
 * chunks of the global batch can be handed over in any order (disjoint document ranges, global
 * stream order is the document index), and with the window sweep each chunk's probes are binned
 * as soon as it arrives -- so the exchange and binning of chunk c overlap the MinHash of chunk
 * c+1 on every rank -- while the query-then-insert itself runs at finish in exact stream order.
 *  lshbloom_bands_begin(h, n_global): start a batch of n_global (< 2^32) documents (waits for
 *    earlier work of the handle).
 *  lshbloom_bands_add(h, bh_owned, doc0, n_docs, stream): bh_owned = device [n_docs][band_hi -
 *    band_lo] band hashes of global documents [doc0, doc0 + n_docs), produced on `stream`;
 *    copied into the batch (stream-ordered: reusable once `stream` passes this call).
 *  lshbloom_bands_finish(h, hit_out, stream): every document added exactly once, else error 1;
 *    hit_out (device, n_global) = OR over the owned bands of the stream-order verdicts, as
 *    lshbloom_query_insert_bands would give for the whole batch.  Mutates the filters;
 *    synchronises. */
LSHBLOOM_API int lshbloom_bands_begin(lshbloom *h, uint64_t n_global);
LSHBLOOM_API int lshbloom_bands_add(lshbloom *h, const uint64_t *bh_owned, uint64_t doc0, uint64_t n_docs,
                                    void *stream);
LSHBLOOM_API int lshbloom_bands_finish(lshbloom *h, uint8_t *hit_out, void *stream);

/* Band-sharded exchange over peer memory (world > 1 on GPUs with
 * peer access, e.g. NVLink / NVSwitch via torch symmetric memory).  Instead of an owner-major
 * local buffer + all-to-all + all-reduce:
 *  lshbloom_band_hashes_to_peers: K1 over this rank's documents, whose first document is
 *    global_doc0 of the global batch, stores each band hash straight into its owner's receive
 *    buffer: peer_recv[o] (a host array of `world` device pointers valid in this process, e.g.
 *    symmetric-memory peer pointers) holds [n_global][band_hi(o) - band_lo(o)] uint64 in global
 *    document order, and band j of global document g goes to
 *    peer_recv[o][g * (hi - lo) + (j - lo)] for the o owning j.  Synchronises its stream.
 *  lshbloom_query_insert_bands_peers: once every rank's band hashes have landed (a barrier
 *    between the two calls is the caller's), query-then-insert the owned bands for all n_global
 *    documents (bh_owned: this rank's receive buffer, device) and raise each hit document's flag
 *    directly in its home rank's buffer: document g with doc_start[r] <= g < doc_start[r+1]
 *    (host array of world+1 entries, doc_start[0] = 0, doc_start[world] = n_global) sets
 *    peer_flags[r][g - doc_start[r]] = 1 (every owner stores the same 1, so no reduction is
 *    needed).  Flag buffers must be zeroed before the first writer runs (the caller's barrier).
 *    Mutates the owned filters; synchronises its stream.
 * Results are bit-identical to lshbloom_query_insert on one GPU. */
LSHBLOOM_API int lshbloom_band_hashes_to_peers(lshbloom *h, const lshbloom_batch *batch, uint64_t global_doc0,
                                               void *const *peer_recv);
LSHBLOOM_API int lshbloom_query_insert_bands_peers(lshbloom *h, const uint64_t *bh_owned, uint64_t n_global,
                                                   const uint64_t *doc_start, void *const *peer_flags, void *stream);

/* Zero every owned filter and the document count (as right after create).  Ordered on the device
 * after the batches already enqueued and before later ones; waits for completion unless async
 * batches are in flight. */
LSHBLOOM_API int lshbloom_reset(lshbloom *h);

/* Copy owned band (band_hi > j >= band_lo, global index j) filter words to host memory
 * dst (words_per_band uint32 words; bit g of the filter = bit g&31 of word g>>5). */
LSHBLOOM_API int lshbloom_filter_copy(lshbloom *h, uint32_t j, uint32_t *dst);

/* Parameters and derived sizes. */
LSHBLOOM_API int lshbloom_info(const lshbloom *h, lshbloom_info_t *out);

/* Last error message of h (or of the last failed create when h is NULL). */
LSHBLOOM_API const char *lshbloom_last_error(const lshbloom *h);

/* Stage timing with CUDA events recorded around the MinHash (K1) launches, the Bloom stage
 * (K3-K6 sub-batch loop, or the sweep path's binning + sweep, on the Bloom stream) and the
 * sweep path's final kernels (exact-layout fix-up, window sweep, verdict).  enable != 0 turns
 * recording on for later calls.  ms_out[0..LSHBLOOM_NSTAGES) receive the K1 / Bloom / sweep
 * milliseconds accumulated since the previous read, n_out[] the number of timed stages; the
 * accumulators are then reset.  Either pointer may be NULL. */
LSHBLOOM_API int lshbloom_stage_times(lshbloom *h, int32_t enable, double *ms_out, uint64_t *n_out);

/* Checkpoint / resume.
 * lshbloom_save writes the index (world = 1 handles) as SPEC's little-endian "LSHB" container:
 *   "LSHB" | version u32 (1) | threshold f64 (config lsh_threshold; if 0, (1/b)^(1/r), the S-curve
 *            midpoint -- create takes b, r; load carries it back into the config)
 *   | num_perm u32 | b u32 | r u32 | signature_seed u64 | band_hash_seed u64 (both = seed)
 *   | n_docs u64 (n_expected) | p_effective f64 (1-(1-p)^b) | doc_count u64
 *   | b filter encodings | CRC32C u32 of every preceding byte,
 * each filter encoding being SPEC's "LBF1" record:
 *   "LBF1" | version u32 (1) | seed u64 (s1_j) | capacity_n u64 | target_p f64 (per-filter p)
 *   | m u64 | k u32 | inserted u64 | payload ceil(m/8) bytes (bit i at byte i>>3, mask
 *   1<<(i&7)) | CRC32C u32 of the preceding bytes of this record.
 * Shingle width n is not part of SPEC's format; files are written only for n = 5.
 * lshbloom_load reads such a file onto `device` (-1 = current) and returns a handle whose
 * later query_insert calls continue the stream exactly where the saved one stopped.
 * Errors: 1 usage (world > 1, n != 5, NULL), 5 format, 6 truncation, 7 checksum, 8 I/O. */
LSHBLOOM_API int lshbloom_save(lshbloom *h, const char *path);
LSHBLOOM_API int lshbloom_load(const char *path, int32_t device, lshbloom **out);

/* Band selection and capacity planning (host-only).
 * lshbloom_optimal_params: the (b, r) with b*r <= num_perm minimising
 *   fp_weight * int_0^T (1 - (1 - s^r)^b) ds + fn_weight * int_T^1 (1 - s^r)^b ds
 * ("given a desired Jaccard similarity threshold, T, one can determine an optimal band
 * size, b"), each integral by composite Simpson's rule with 1000 subintervals
 * (S:232); ties go to the smaller b, then the smaller r.  T in (0, 1], num_perm >= 2,
 * weights >= 0; error 1 otherwise.  (T = 0.8, 128 permutations -> b = 9.)
 * lshbloom_plan: sizes an index for n_docs documents at an effective false-positive rate
 * p_effective (P:227 p_eff = 1 - (1 - p)^b, inverted for the per-filter p) with b from
 * lshbloom_optimal_params(T, num_perm, 0.5, 0.5) and m, k per filter as lshbloom_create does;
 * total_bytes = b * ceil(m / 8) (Tables 1-2; P:229's 590 GB). */
typedef struct {
    uint32_t b, r;
    double p;                 /* per-filter false-positive rate */
    uint64_t m;               /* bits per filter */
    uint32_t k;               /* probes per band hash */
    uint64_t total_bytes;     /* b * ceil(m / 8) */
} lshbloom_plan_t;

LSHBLOOM_API int lshbloom_optimal_params(double threshold, uint32_t num_perm, double fp_weight,
                                         double fn_weight, uint32_t *b_out, uint32_t *r_out);
LSHBLOOM_API int lshbloom_plan(uint64_t n_docs, double p_effective, double threshold, uint32_t num_perm,
                               lshbloom_plan_t *out);

/* Number of kernel launches the library issued since create (launch-count evidence). */
LSHBLOOM_API uint64_t lshbloom_launch_count(const lshbloom *h);

#ifdef __cplusplus
}
#endif
#endif /* LSHBLOOM_H */
