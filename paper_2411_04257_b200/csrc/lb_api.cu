// lb_api.cu -- the C-ABI of include/lshbloom.h: handle, sizing, hash-family expansion, batch
// staging (pinned host -> HBM, double-buffered against K1), and the per-call kernel sequence.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>   // CUstream / CUdeviceptr types for the stream memory operation (no -lcuda)

#include "../../include/lshbloom.h"
#include "lb_internal.h"

using namespace lb;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

// Grow b to at least `bytes` (25 % slack); *fresh (optional) tells whether it was (re)allocated --
// cudaMalloc may hand back the address it just freed, so callers must not compare pointers.
cudaError_t ensure(DevBuf& b, size_t bytes, bool* fresh = nullptr) {
  if (fresh) *fresh = false;
  if (bytes <= b.cap && b.p) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t c = bytes + bytes / 4 + 256;
  cudaError_t e = cudaMalloc(&b.p, c);
  if (e == cudaSuccess) {
    b.cap = c;
    if (fresh) *fresh = true;
  }
  return e;
}

thread_local std::string g_create_error;

constexpr uint32_t kDefaultSubBatch = 32768;
constexpr uint64_t kChunkTokens = 16ull << 20;   // host-batch staging chunk (64 MB of tokens)
constexpr uint32_t K1_THREADS_HOST = 256;          // K1 block size (lb_minhash.cu), for chunk sizing
constexpr uint64_t kGenMax = (1ull << 22) - 1;

// Counter-mode expansion R(seed, dom, i) (DESIGN R5).
uint64_t R(uint64_t seed, uint64_t dom, uint64_t i) { return mix64(seed + kGamma * ((dom << 32) + i + 1)); }

struct SweepPlan {
  bool use = false;
  uint32_t wb = 0, cap = 0;
  uint64_t nw = 0, nbins = 0, piece = 0;
  bool two_level = false;         // K7a + K7b (k = 17)
  uint32_t cb = 0, ccap = 0;
  uint64_t ncb = 0;
};

}  // namespace

struct lshbloom {
  lshbloom_config cfg{};
  uint64_t m = 0, m_inv = 0, W = 0;
  uint64_t nb = 0, nb_inv = 0;    // blocked variant: 1024-bit blocks per band
  uint32_t k = 0, band_lo = 0, band_hi = 0, bl = 0, npl = 0, sub_batch = 0;
  int device = 0, sm_count = 148;
  size_t total_mem = 0;
  cudaStream_t own_stream = nullptr, copy_stream = nullptr, bloom_stream = nullptr;
  cudaStream_t k1_stream2 = nullptr, k1_stream3 = nullptr;  // fused step: K1 chunks round-robin, a chunk's tail overlaps the next
  cudaEvent_t ev_fuse = nullptr, ev_join = nullptr, ev_join3 = nullptr;
  int k1_nstreams = 2;
  bool k1_alt = true;
  int k1_bps = 0;                 // K1 blocks per SM cap (0 = occupancy limit)
  cudaEvent_t ev_h2d[3] = {nullptr, nullptr, nullptr}, ev_k1[3] = {nullptr, nullptr, nullptr};
  PermCoef* d_coef = nullptr;
  uint64_t* d_bcoef = nullptr;
  uint64_t* d_s1 = nullptr;
  uint64_t* d_s2 = nullptr;
  uint32_t* d_F = nullptr;
  uint64_t* d_Q = nullptr;        // 2 compact earliest-setter tables of 2^q_log2 slots
  uint32_t q_log2 = 19;
  uint64_t* d_ekey = nullptr;
  uint64_t* d_eval = nullptr;
  uint32_t ecap_log2 = 0;
  uint64_t gen = 1;
  uint64_t* d_st = nullptr;       // 2 * sub_batch * bl
  uint32_t* d_cand = nullptr;     // sub_batch * bl
  uint32_t* d_counters = nullptr; // [1..3] K1 work counters, [8] classic full, [12..13] Bloom candidates / contested
  uint64_t* d_clist = nullptr;    // contested probes of a sub-batch (sub_batch * bl * k)
  uint32_t* d_cb = nullptr;       // contested-position summary bits (2^cb_log2)
  uint32_t cb_log2 = 26;            // 8 MB: ~0.2 % of first arrivals collide with a contested position
  ErrState* d_err_base = nullptr; // [0]: synchronous calls; [1 + slot]: async query_insert batches
  ErrState* d_err = nullptr;      // the state of the call being enqueued
  DevBuf off, tok[3], bh, dup, sig, part;   // tok: host-batch staging buffers
  // query_insert batches in flight (lshbloom_query_insert_async / lshbloom_sync): at most two,
  // each with its own band-hash, offsets and flag buffers and error state, so that batch t+1's K1
  // runs while batch t's Bloom stage is still working (the Bloom stream keeps them in order)
  struct Slot {
    bool busy = false;
    uint64_t n = 0, seq = 0;
    cudaEvent_t done = nullptr;
    DevBuf bh, off, dup;
    // landing-gated host batches: the whole token array lands here while K1 runs; *landed counts
    // landed pieces (written by cuStreamWriteValue32 on the copy stream); tok_free is recorded
    // when the batch's last K1 launch is done (the next copy into this buffer waits for it)
    DevBuf tokall;
    uint32_t* landed = nullptr;
    cudaEvent_t tok_free = nullptr, land_zero = nullptr;   // land_zero: this batch's counter zeroed (copy stream)
  } slot[2];
  int next_slot = 0;
  uint64_t seq = 0;
  int async_rc = 0;               // first error of a completed async batch, until lshbloom_sync
  std::string async_msg;
  cudaStream_t k1_stream1 = nullptr;
  cudaEvent_t ev_in = nullptr, ev_pre = nullptr;
  // cuStreamWriteValue32 (driver entry point, resolved at create; null: host batches use the
  // staging path) and the landing piece, 2^land_log2 tokens
  CUresult (*write_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  uint32_t land_log2 = 21;
  bool land_enabled = true;
  // a batch assembled from band-hash chunks (lshbloom_bands_begin / _add / _finish)
  bool bands_open = false;
  uint64_t bands_n = 0, bands_added = 0;
  SweepPlan bands_plan;
  DevBuf bands_bh;                // [bl][n_global] band-major
  uint64_t doc_count = 0, launches = 0;
  // classic MinHashLSH index (index_kind = LSHBLOOM_INDEX_CLASSIC)
  uint64_t* d_ckeys = nullptr;    // [bl][2^c_log2cap]
  uint64_t* d_cvals = nullptr;
  uint32_t c_log2cap = 0;
  // window-sweep Bloom stage (lb_sweep.cu)
  uint32_t bloom_path = 0;        // LSHBLOOM_PATH_AUTO / _RANDOM / _SWEEP
  uint32_t sweep_wb_force = 0, sweep_cap_force = 0;
  DevBuf sw_cursor, sw_cursor2, sw_start, sw_rec, sw_miss, sw_eg, sw_ccursor, sw_crec, sw_bht;
  uint64_t sweeps = 0;            // sweeps run (lshbloom_info)
  // stage timing (lshbloom_stage_times): K1, Bloom stage, sweep kernels (K7x-K9)
  bool timing = false;
  int tset = 0;                   // event set of the call being enqueued: 0, 1 (async slots), 2 (sync)
  cudaEvent_t tev[3][2 * LSHBLOOM_NSTAGES] = {};
  bool pend[3][LSHBLOOM_NSTAGES] = {};
  double stage_ms[LSHBLOOM_NSTAGES] = {};
  uint64_t stage_n[LSHBLOOM_NSTAGES] = {};
  std::string err;
  bool poisoned = false;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int fail(lshbloom* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  else g_create_error = msg;
  return code;
}

int fail_cuda(lshbloom* h, cudaError_t e, const char* what) {
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(h, LSHBLOOM_ENOMEM, msg);
  }
  if (h) h->poisoned = true;
  return fail(h, LSHBLOOM_ERUNTIME, msg);
}

#define LB_CUDA(h, call)                                 \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return fail_cuda(h, e_, #call); \
  } while (0)

int check_handle(lshbloom* h) {
  if (!h) return fail(nullptr, LSHBLOOM_EUSAGE, "NULL handle");
  if (h->poisoned) return fail(h, LSHBLOOM_ERUNTIME, "handle poisoned by an earlier CUDA error: " + h->err);
  return LSHBLOOM_OK;
}

void free_all(lshbloom* h) {
  auto F = [](void* p) { if (p) cudaFree(p); };
  F(h->d_coef); F(h->d_bcoef); F(h->d_s1); F(h->d_s2); F(h->d_F); F(h->d_Q); F(h->d_clist); F(h->d_cb); F(h->d_ekey);
  F(h->d_eval); F(h->d_st); F(h->d_ckeys); F(h->d_cvals); F(h->d_cand); F(h->d_counters); F(h->d_err_base);
  for (auto& sl : h->slot) {
    F(sl.bh.p); F(sl.off.p); F(sl.dup.p); F(sl.tokall.p); F(sl.landed);
    if (sl.done) cudaEventDestroy(sl.done);
    if (sl.tok_free) cudaEventDestroy(sl.tok_free);
    if (sl.land_zero) cudaEventDestroy(sl.land_zero);
  }
  if (h->k1_stream1) cudaStreamDestroy(h->k1_stream1);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_pre) cudaEventDestroy(h->ev_pre);
  F(h->off.p); F(h->tok[0].p); F(h->tok[1].p); F(h->tok[2].p); F(h->bh.p); F(h->dup.p); F(h->sig.p); F(h->part.p);
  F(h->sw_cursor.p); F(h->sw_cursor2.p); F(h->sw_start.p); F(h->sw_rec.p); F(h->sw_miss.p); F(h->sw_eg.p);
  F(h->sw_ccursor.p); F(h->sw_crec.p); F(h->sw_bht.p); F(h->bands_bh.p);
  for (int i = 0; i < 3; i++) {
    if (h->ev_h2d[i]) cudaEventDestroy(h->ev_h2d[i]);
    if (h->ev_k1[i]) cudaEventDestroy(h->ev_k1[i]);
  }
  for (auto& set : h->tev)
    for (auto& e : set)
      if (e) cudaEventDestroy(e);
  if (h->ev_fuse) cudaEventDestroy(h->ev_fuse);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->k1_stream2) cudaStreamDestroy(h->k1_stream2);
  if (h->k1_stream3) cudaStreamDestroy(h->k1_stream3);
  if (h->ev_join3) cudaEventDestroy(h->ev_join3);
  if (h->bloom_stream) cudaStreamDestroy(h->bloom_stream);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
}

// Landing-gated host batches (MinhashParams::landed): resolve cuStreamWriteValue32 through the
// runtime's driver entry point (no link against libcuda) and check once that a stream write
// lands; otherwise host batches keep the staging path.  LSHBLOOM_LANDING=0 disables the gate,
// LSHBLOOM_LAND_LOG2 sets the landing piece (2^k tokens, 18..28; default 2^21 = 8 MB: C3 e2e 106.4 / 106.9 / 108.0 ms per 200K documents at 2^21 / 2^23 / 2^25).
void init_landing(lshbloom* h) {
  h->write_value32 = nullptr;
  if (const char* e = getenv("LSHBLOOM_LANDING")) h->land_enabled = atoi(e) != 0;
  if (const char* e = getenv("LSHBLOOM_LAND_LOG2")) h->land_log2 = (uint32_t)std::min(28, std::max(18, atoi(e)));
  if (!h->land_enabled) return;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return;
  }
  auto wv = (CUresult(*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int))fn;
  uint32_t got = 0;
  if (wv((CUstream)h->own_stream, (CUdeviceptr)h->slot[0].landed, 0x1A2B3C4Du, 0) != CUDA_SUCCESS ||
      cudaMemcpyAsync(&got, h->slot[0].landed, 4, cudaMemcpyDeviceToHost, h->own_stream) != cudaSuccess ||
      cudaStreamSynchronize(h->own_stream) != cudaSuccess || got != 0x1A2B3C4Du) {
    cudaGetLastError();
    return;
  }
  cudaMemset(h->slot[0].landed, 0, 4);
  h->write_value32 = wv;
}

// Host-side CSR validation; returns 0, 1 (usage) or 2 (empty doc).
int validate_host(lshbloom* h, const uint64_t* off, uint64_t n) {
  if (off[0] != 0) return fail(h, LSHBLOOM_EUSAGE, "offsets[0] must be 0");
  for (uint64_t i = 0; i < n; i++) {
    if (off[i + 1] < off[i]) return fail(h, LSHBLOOM_EUSAGE, "offsets decrease at index " + std::to_string(i));
    if (off[i + 1] == off[i])
      return fail(h, LSHBLOOM_EDATA, "empty document at index " + std::to_string(i));
  }
  return LSHBLOOM_OK;
}

int check_batch(lshbloom* h, const lshbloom_batch* b) {
  if (!b || !b->offsets || !b->tokens) return fail(h, LSHBLOOM_EUSAGE, "NULL batch / offsets / tokens");
  if (b->n_docs == 0 || b->n_docs > 0xFFFFFFFFull) return fail(h, LSHBLOOM_EUSAGE, "n_docs must be in [1, 2^32)");
  return LSHBLOOM_OK;
}

void stage_begin(lshbloom* h, int st, cudaStream_t s) {
  if (h->timing) cudaEventRecord(h->tev[h->tset][2 * st], s);
}
void stage_end(lshbloom* h, int st, cudaStream_t s) {
  if (h->timing) {
    cudaEventRecord(h->tev[h->tset][2 * st + 1], s);
    h->pend[h->tset][st] = true;
  }
}
// after the work of event set `set` is complete
void stage_collect(lshbloom* h, int set = 2) {
  for (int st = 0; st < LSHBLOOM_NSTAGES; st++) {
    if (!h->pend[set][st]) continue;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, h->tev[set][2 * st], h->tev[set][2 * st + 1]) == cudaSuccess) {
      h->stage_ms[st] += ms;
      h->stage_n[st] += 1;
    }
    h->pend[set][st] = false;
  }
}

// Host-side completion of an async batch: its error state (offsets / empty document, the
// device-side K0 verdict) becomes the pending async result; a rejected batch inserted nothing.
int collect(lshbloom* h, int si) {
  lshbloom::Slot& sl = h->slot[si];
  if (!sl.busy) return LSHBLOOM_OK;
  LB_CUDA(h, cudaEventSynchronize(sl.done));
  sl.busy = false;
  stage_collect(h, si);
  ErrState e;
  LB_CUDA(h, cudaMemcpy(&e, h->d_err_base + 1 + si, sizeof e, cudaMemcpyDeviceToHost));
  if (e.flags || e.first_empty != ~0ull) {
    h->doc_count -= std::min(h->doc_count, sl.n);
    if (!h->async_rc) {
      h->async_rc = (e.flags & 2) ? LSHBLOOM_ERUNTIME : e.flags ? LSHBLOOM_EUSAGE : LSHBLOOM_EDATA;
      h->async_msg = (e.flags & 2) ? "timed out waiting for the batch's tokens to land in device memory"
                     : e.flags ? "malformed offsets (offsets[0] != 0 or decreasing)"
                               : "empty document at index " + std::to_string(e.first_empty);
    }
  }
  return LSHBLOOM_OK;
}

// Wait for every batch in flight, oldest first.
int drain(lshbloom* h) {
  const int first = h->slot[0].busy && h->slot[1].busy ? (h->slot[0].seq < h->slot[1].seq ? 0 : 1)
                                                       : (h->slot[0].busy ? 0 : 1);
  int rc = collect(h, first);
  if (!rc) rc = collect(h, first ^ 1);
  return rc;
}

// ensure() for scratch shared by the batches in flight: growing it first drains them.
int grow(lshbloom* h, DevBuf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return LSHBLOOM_OK;
  int rc = drain(h);
  if (rc) return rc;
  LB_CUDA(h, ensure(b, bytes));
  return LSHBLOOM_OK;
}

// Owner-major layout for the band-sharded all-to-all (lshbloom_band_hashes_sharded).
BandMap sharded_map(const lshbloom* h, uint64_t n) {
  BandMap m;
  memset(&m, 0, sizeof m);
  const uint32_t b = h->cfg.b, world = h->cfg.world, base = b / world, rem = b % world;
  uint64_t start = 0;
  for (uint32_t o = 0; o < world; o++) {
    const uint32_t lo = o * base + std::min(o, rem), cnt = base + (o < rem ? 1 : 0);
    for (uint32_t j = lo; j < lo + cnt; j++) {
      m.blockstart[j] = start;
      m.ncol[j] = cnt;
      m.col[j] = j - lo;
    }
    start += n * cnt;
  }
  return m;
}


// Band-major [b_local][n] layout for the fused query_insert path (the Bloom kernels walk one
// band's filter at a time).
BandMap owned_band_major_map(const lshbloom* h, uint64_t n) {
  BandMap m;
  memset(&m, 0, sizeof m);
  for (uint32_t j = h->band_lo; j < h->band_hi; j++) {
    m.blockstart[j] = (uint64_t)(j - h->band_lo) * n;
    m.ncol[j] = 1;
    m.col[j] = 0;
  }
  return m;
}

BandMap full_map(const lshbloom* h) {
  BandMap m;
  memset(&m, 0, sizeof m);
  for (uint32_t j = 0; j < h->cfg.b; j++) {
    m.ncol[j] = h->cfg.b;
    m.col[j] = j;
  }
  return m;
}

// Absolute store pointers of a local layout (peer layouts come with ptr[] already set).
BandMap resolve_map(BandMap m, uint64_t* out, uint32_t b) {
  for (uint32_t j = 0; j < b; j++)
    if (m.ncol[j] && !m.ptr[j]) m.ptr[j] = out + m.blockstart[j] + m.col[j];
  return m;
}

// Reset the error gate: flags = 0, gate = 0, first_empty = ~0.
int reset_err(lshbloom* h, cudaStream_t s) {
  LB_CUDA(h, cudaMemsetAsync(h->d_err, 0, 8, s));
  LB_CUDA(h, cudaMemsetAsync(&h->d_err->first_empty, 0xFF, 8, s));
  return LSHBLOOM_OK;
}

// After the stream is synchronised: translate the device validation result.
int read_err(lshbloom* h) {
  ErrState e;
  LB_CUDA(h, cudaMemcpy(&e, h->d_err, sizeof e, cudaMemcpyDeviceToHost));
  if (e.flags) return fail(h, LSHBLOOM_EUSAGE, "malformed offsets (offsets[0] != 0 or decreasing)");
  if (e.first_empty != ~0ull)
    return fail(h, LSHBLOOM_EDATA, "empty document at index " + std::to_string(e.first_empty));
  return LSHBLOOM_OK;
}

MinhashParams base_params(lshbloom* h) {
  MinhashParams p;
  memset(&p, 0, sizeof p);
  p.shingle_n = h->cfg.shingle_n;
  p.sh29 = 29;
  p.sh3 = 3;
  p.fp_init_n = mix64(kFpSalt + h->cfg.shingle_n);
  p.coef = h->d_coef;
  p.num_perm = h->cfg.num_perm;
  p.b = h->cfg.b;
  p.r = h->cfg.r;
  p.bcoef = h->d_bcoef;
  p.err = &h->d_err->pad;
  return p;
}

// K0 + K1 over a batch.  sig_dev / bh_dev are device outputs (either may be null).
int run_minhash(lshbloom* h, const lshbloom_batch* b, cudaStream_t s, uint32_t* sig_dev,
                uint64_t* bh_dev, const BandMap& map) {
  const uint64_t n = b->n_docs;
  MinhashParams p = base_params(h);
  if (h->npl >= 8) {   // scratch of the length-partitioned K1 launches (lb_minhash.cu)
    LB_CUDA(h, ensure(h->part, (2 * (size_t)b->n_docs + 2 + b->n_docs / 1024 + 1) * sizeof(uint32_t)));
    p.part_lists = (uint32_t*)h->part.p;
    p.part_counts = (uint32_t*)h->part.p + 2 * b->n_docs;
    p.part_blk = p.part_counts + 2;
  }
  p.sig_out = sig_dev;
  p.bh_out = bh_dev;
  p.map = resolve_map(map, bh_dev, h->cfg.b);
  int rc = reset_err(h, s);
  if (rc) return rc;
  if (b->on_device) {
    h->launches += launch_validate(b->offsets, n, h->d_err, s);
    p.offsets = b->offsets;
    p.tokens = b->tokens;
    p.tok_base = 0;
    p.doc0 = 0;
    p.n_docs = (uint32_t)n;
    p.counter = h->d_counters + 1;
    LB_CUDA(h, cudaMemsetAsync(p.counter, 0, 4, s));
    stage_begin(h, 0, s);
    int l = launch_minhash(p, (int)h->npl, h->sm_count, s, 0);   // K1 alone: whole GPU
    if (l < 0) return fail(h, LSHBLOOM_EUSAGE, "unsupported num_perm");
    stage_end(h, 0, s);
    h->launches += l;
    LB_CUDA(h, cudaGetLastError());
    return LSHBLOOM_OK;
  }
  // host batch: validate here, then stream token chunks through two staging buffers
  rc = validate_host(h, b->offsets, n);
  if (rc) return rc;
  LB_CUDA(h, ensure(h->off, (n + 1) * sizeof(uint64_t)));
  LB_CUDA(h, cudaMemcpyAsync(h->off.p, b->offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  uint64_t maxdoc = 0;
  for (uint64_t i = 0; i < n; i++) maxdoc = std::max(maxdoc, b->offsets[i + 1] - b->offsets[i]);
  const uint64_t chunk = std::max(kChunkTokens, maxdoc);
  const uint64_t total = b->offsets[n];
  const uint64_t buf_tokens = std::min(chunk, total);
  for (int i = 0; i < 2; i++) LB_CUDA(h, ensure(h->tok[i], buf_tokens * sizeof(uint32_t)));
  p.offsets = (const uint64_t*)h->off.p;
  uint64_t d0 = 0;
  int c = 0;
  stage_begin(h, 0, s);
  while (d0 < n) {
    // largest d1 with tokens [off[d0], off[d1]) <= chunk, but at least ~16 documents per
    // resident K1 warp (long documents) and at least one document; buffers grow to fit
    const uint64_t t0 = b->offsets[d0];
    const uint64_t* lim = std::upper_bound(b->offsets + d0 + 1, b->offsets + n + 1, t0 + chunk);
    uint64_t d1 = (uint64_t)(lim - b->offsets) - 1;
    d1 = std::max<uint64_t>(d1, std::min<uint64_t>(n, d0 + 16ull * h->sm_count * 2 * (K1_THREADS_HOST / 32)));
    if (d1 <= d0) d1 = d0 + 1;
    const uint64_t t1 = b->offsets[d1];
    const int buf = c & 1;
    if ((t1 - t0) * sizeof(uint32_t) > h->tok[buf].cap) {   // a chunk larger than the buffer
      LB_CUDA(h, cudaStreamSynchronize(s));
      LB_CUDA(h, ensure(h->tok[buf], (t1 - t0) * sizeof(uint32_t)));
    }
    LB_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_k1[buf], 0));
    LB_CUDA(h, cudaMemcpyAsync(h->tok[buf].p, b->tokens + t0, (t1 - t0) * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, h->copy_stream));
    LB_CUDA(h, cudaEventRecord(h->ev_h2d[buf], h->copy_stream));
    LB_CUDA(h, cudaStreamWaitEvent(s, h->ev_h2d[buf], 0));
    p.tokens = (const uint32_t*)h->tok[buf].p;
    p.tok_base = t0;
    p.doc0 = (uint32_t)d0;
    p.n_docs = (uint32_t)(d1 - d0);
    p.counter = h->d_counters + 1 + buf;
    LB_CUDA(h, cudaMemsetAsync(p.counter, 0, 4, s));
    int l = launch_minhash(p, (int)h->npl, h->sm_count, s, 0);
    if (l < 0) return fail(h, LSHBLOOM_EUSAGE, "unsupported num_perm");
    h->launches += l;
    LB_CUDA(h, cudaGetLastError());
    LB_CUDA(h, cudaEventRecord(h->ev_k1[buf], s));
    d0 = d1;
    c++;
  }
  stage_end(h, 0, s);
  return LSHBLOOM_OK;
}

// Classic index (lb_classic.cu): KC1 + KC2 over batch documents [i_begin, i_end).
int run_classic(lshbloom* h, const uint64_t* bh_dev, uint64_t bh_sj, uint64_t bh_si, uint64_t i_begin,
                uint64_t i_end, uint8_t* dup_dev, cudaStream_t s, bool first, bool last, const DupSink* peers) {
  ClassicParams p;
  memset(&p, 0, sizeof p);
  p.keys = h->d_ckeys;
  p.vals = h->d_cvals;
  p.log2cap = h->c_log2cap;
  p.bl = h->bl;
  p.doc_base = h->doc_count;
  p.bh = bh_dev;
  p.bh_sj = bh_sj;
  p.bh_si = bh_si;
  p.i0 = (uint32_t)i_begin;
  p.n = (uint32_t)(i_end - i_begin);
  if (peers) p.dup = *peers;
  else p.dup.local = dup_dev;
  p.full = (int*)h->d_counters + 8;
  p.err = &h->d_err->pad;
  if (first) stage_begin(h, 1, s);
  if (p.n) h->launches += launch_classic(p, s);
  LB_CUDA(h, cudaGetLastError());
  if (last) stage_end(h, 1, s);
  return LSHBLOOM_OK;
}

// Classic index capacity: the batch may not take doc_count past 0.9 of the table (checked
// before any mutation, so the probe loops always find a free slot).
int classic_capacity(lshbloom* h, uint64_t n) {
  if (h->cfg.index_kind != LSHBLOOM_INDEX_CLASSIC) return LSHBLOOM_OK;
  const double cap = (double)(1ull << h->c_log2cap);
  if ((double)(h->doc_count + n) > 0.9 * cap)
    return fail(h, LSHBLOOM_EUSAGE, "classic index full: doc_count + batch > 0.9 x " + std::to_string((uint64_t)cap) +
                                        " slots (raise n_expected)");
  return LSHBLOOM_OK;
}

// Filter geometry, seeds, band-hash layout and flag sink of a Bloom launch.
BloomParams bloom_params(lshbloom* h, const uint64_t* bh_dev, uint64_t bh_sj, uint64_t bh_si, uint8_t* dup_dev,
                         const DupSink* peers) {
  BloomParams p;
  memset(&p, 0, sizeof p);
  p.F = h->d_F;
  p.q_log2 = h->q_log2;
  p.W = h->W;
  p.m = h->m;
  p.m_inv = h->m_inv;
  p.nb = h->nb;
  p.nb_inv = h->nb_inv;
  p.k = h->k;
  p.bl = h->bl;
  p.s1 = h->d_s1;
  p.s2 = h->d_s2;
  p.ekey = h->d_ekey;
  p.eval = h->d_eval;
  p.ecap_log2 = h->ecap_log2;
  p.bh = bh_dev;
  p.bh_sj = bh_sj;
  p.bh_si = bh_si;
  const uint64_t SB = h->sub_batch;
  p.st_pre = h->d_st;
  p.st_arr = h->d_st + SB * h->bl;
  p.cand = h->d_cand;
  p.cand_count = h->d_counters + 12;
  p.clist = h->d_clist;
  p.cb = h->d_cb;
  p.cb_log2 = h->cb_log2;
  if (peers) p.dup = *peers;
  else p.dup.local = dup_dev;
  p.err = &h->d_err->pad;
  return p;
}

// K3-K6 over bh_dev[n][bl] in sub-batches; dup_dev[n] must be zeroed by the caller.
int run_bloom(lshbloom* h, const uint64_t* bh_dev, uint64_t bh_sj, uint64_t bh_si, uint64_t i_begin, uint64_t i_end,
              uint8_t* dup_dev, cudaStream_t s, bool first = true, bool last = true, const DupSink* peers = nullptr) {
  if (h->cfg.index_kind == LSHBLOOM_INDEX_CLASSIC)
    return run_classic(h, bh_dev, bh_sj, bh_si, i_begin, i_end, dup_dev, s, first, last, peers);
  BloomParams p = bloom_params(h, bh_dev, bh_sj, bh_si, dup_dev, peers);
  const uint64_t SB = h->sub_batch;
  if (first) stage_begin(h, 1, s);
  for (uint64_t i0 = i_begin; i0 < i_end; i0 += SB) {
    if (h->gen >= kGenMax) {   // generation tags exhausted: clear E once every ~4M sub-batches
      const uint64_t cap = 1ull << h->ecap_log2;
      LB_CUDA(h, cudaMemsetAsync(h->d_ekey, 0, cap * 8, s));
      LB_CUDA(h, cudaMemsetAsync(h->d_eval, 0, cap * 8, s));
      h->gen = 1;
    }
    p.gen = h->gen++;
    const uint64_t qslots = 1ull << h->q_log2;
    p.Q = h->d_Q + (p.gen & 1) * qslots;
    p.i0 = (uint32_t)i0;
    p.nsb = (uint32_t)std::min<uint64_t>(SB, i_end - i0);
    h->launches += launch_bloom_subbatch(p, h->sm_count, s);
    LB_CUDA(h, cudaGetLastError());
  }
  if (last) stage_end(h, 1, s);
  return LSHBLOOM_OK;
}

// ------------------------------------------------------------------ window-sweep Bloom path

constexpr uint64_t kSweepMaxDocs = 1ull << 22;   // documents per sweep (records carry 32-bit
                                                 // document offsets; path (b) keeps 32-bit minima)

// Bin capacity for an expected load of mu records: 7 standard deviations of a Poisson load, slack
// for the band hashes near-duplicates share, and `pad` records of sector padding.
// Rounded up to whole 32-byte sectors so that every bin starts sector-aligned.
uint32_t sweep_cap_for(double mu, double pad = 0.0) {
  return ((uint32_t)std::ceil(mu + 7.0 * std::sqrt(mu) + 64.0 + pad) + 3u) & ~3u;
}

// Window size and bin capacities for a batch of n documents (pieces of <= kSweepMaxDocs): the
// largest window whose bin capacity (expected load mu = n k 2^wb / m, plus the sector padding
// K7b adds per chunk) fits the K8 CTA's kSweepCapReg register-held records, the coarse buckets
// of the two-level binning (<= kSweepMaxCoarse per band, <= 512 windows each), and whether the
// sweep beats random access (AUTO: owned filters beyond 96 MB, i.e. not L2-resident, and >= 256
// probes per 64 KB window).
SweepPlan plan_sweep(const lshbloom* h, uint64_t n, uint64_t max_piece = kSweepMaxDocs) {
  SweepPlan sp;
  if (h->cfg.index_kind == LSHBLOOM_INDEX_CLASSIC || h->bloom_path == LSHBLOOM_PATH_RANDOM || n == 0) return sp;
  sp.piece = std::min<uint64_t>(n, max_piece);
  const double rho = (double)sp.piece * h->k / (double)h->m;      // records per filter bit
  const double tiles = std::ceil((double)sp.piece / kSweepTileDocs);
  auto coarse = [&](uint32_t wb, uint32_t& cb, uint64_t& ncb, uint32_t& ccap) {
    const uint64_t nw = (h->m + (1ull << wb) - 1) >> wb;
    cb = 0;
    while ((1u << cb) < kSweepMaxW && ((nw + (1ull << cb) - 1) >> cb) > kSweepMaxCoarse) cb++;
    ncb = (nw + (1ull << cb) - 1) >> cb;
    const double mu_c = rho * (double)(1ull << (wb + cb));
    ccap = sweep_cap_for(mu_c, 3.0 * std::min(tiles, mu_c));
    return ncb <= kSweepMaxCoarse;
  };
  // window bins: Poisson load + K7b's rounding of each window's tail to a whole sector; rounded
  // to 16 records so that every bin starts on a 128-byte line (K7b writes whole lines)
  auto fine_cap = [&](uint32_t wb, bool two) {
    const double mu = rho * (double)(1ull << wb);
    if (!two) return sweep_cap_for(mu);
    return (sweep_cap_for(mu, 3.0) + 15u) & ~15u;
  };
  // windows up to 2^17 bits (16 KB: four K8 CTAs per SM fit; C5 4M-document sweeps measured
  // 36.4 ms at 2^17 vs 38.0 ms at 2^18 with two CTAs per SM)
  const bool two = h->k == 17;
  uint32_t wb = 10;
  while (wb < 17 && fine_cap(wb + 1, two) <= kSweepCapReg) wb++;
  if (h->sweep_wb_force) wb = h->sweep_wb_force;
  if (h->bloom_path == LSHBLOOM_PATH_AUTO) {
    const double fbytes = (double)h->bl * (double)h->W * 4.0;
    if (!(fbytes > 96e6 && rho * 524288.0 >= 256.0 && fine_cap(10, two) <= kSweepCapReg)) return sp;
  }
  sp.use = true;
  sp.wb = wb;
  sp.nw = (h->m + (1ull << wb) - 1) >> wb;
  sp.nbins = sp.nw * h->bl;
  sp.two_level = two && coarse(wb, sp.cb, sp.ncb, sp.ccap);
  if (getenv("LSHBLOOM_SWEEP_ONE_LEVEL")) sp.two_level = false;
  sp.cap = h->sweep_cap_force ? h->sweep_cap_force : fine_cap(wb, sp.two_level);
  if (sp.two_level && h->sweep_cap_force) {
    sp.ccap = (std::max<uint32_t>(4, h->sweep_cap_force) + 3u) & ~3u;
    sp.cap = (sp.cap + 15u) & ~15u;
  }
  return sp;
}

// ensure() for buffers that must start zeroed (the miss words are re-zeroed by K9 after use).
int ensure_zeroed(lshbloom* h, DevBuf& b, size_t bytes, cudaStream_t s) {
  bool fresh = false;
  LB_CUDA(h, ensure(b, bytes, &fresh));
  if (fresh) LB_CUDA(h, cudaMemsetAsync(b.p, 0, b.cap, s));
  return LSHBLOOM_OK;
}

int sweep_alloc(lshbloom* h, const SweepPlan& sp, cudaStream_t s) {
  const uint64_t recs = std::max<uint64_t>(sp.nbins * sp.cap, sp.piece * h->k * h->bl);
  int rc = 0;
  if (sp.two_level &&
      ((rc = grow(h, h->sw_ccursor, h->bl * sp.ncb * 4)) || (rc = grow(h, h->sw_crec, h->bl * sp.ncb * sp.ccap * 8))))
    return rc;
  if ((rc = grow(h, h->sw_cursor, sp.nbins * 4)) || (rc = grow(h, h->sw_cursor2, sp.nbins * 4)) ||
      (rc = grow(h, h->sw_start, (sp.nbins + 1) * 8)) || (rc = grow(h, h->sw_rec, recs * 8)) ||
      (rc = grow(h, h->sw_eg, (size_t)sweep_grid(h->sm_count, sp.wb) << sp.wb << 2)))
    return rc;
  if (sp.piece * 8 > h->sw_miss.cap && (rc = drain(h))) return rc;
  return ensure_zeroed(h, h->sw_miss, sp.piece * 8, s);
}

SweepParams sweep_params(lshbloom* h, const SweepPlan& sp, const BloomParams& g, uint64_t i0, uint64_t n) {
  SweepParams p;
  memset(&p, 0, sizeof p);
  p.g = g;
  p.wb = sp.wb;
  p.cap = sp.cap;
  p.nw = sp.nw;
  p.nbins = sp.nbins;
  p.cursor = (uint32_t*)h->sw_cursor.p;
  p.cursor2 = (uint32_t*)h->sw_cursor2.p;
  p.start = (uint64_t*)h->sw_start.p;
  p.rec = (uint64_t*)h->sw_rec.p;
  p.ovf = h->d_counters + 14;
  p.miss = (uint64_t*)h->sw_miss.p;
  p.eg = (uint32_t*)h->sw_eg.p;
  p.i0 = (uint32_t)i0;
  p.n = (uint32_t)n;
  p.two_level = sp.two_level ? 1 : 0;
  if (sp.two_level) {
    p.cb = sp.cb;
    p.ncb = sp.ncb;
    p.ccap = sp.ccap;
    p.ccursor = (uint32_t*)h->sw_ccursor.p;
    p.crec = (uint64_t*)h->sw_crec.p;
  }
  return p;
}

int sweep_begin(lshbloom* h, const SweepParams& p, cudaStream_t s) {
  LB_CUDA(h, cudaMemsetAsync(p.cursor, 0, p.nbins * 4, s));
  LB_CUDA(h, cudaMemsetAsync(p.ovf, 0, 4, s));
  if (p.two_level) LB_CUDA(h, cudaMemsetAsync(p.ccursor, 0, p.g.bl * p.ncb * 4, s));
  return LSHBLOOM_OK;
}

int sweep_bin(lshbloom* h, const SweepParams& p, uint64_t lo, uint64_t hi, cudaStream_t s) {
  h->launches += launch_sweep_bin(p, (uint32_t)lo, (uint32_t)hi, s);
  LB_CUDA(h, cudaGetLastError());
  return LSHBLOOM_OK;
}

int sweep_finish(lshbloom* h, const SweepParams& p, cudaStream_t s, bool first, bool last) {
  if (first) stage_begin(h, 2, s);
  h->launches += launch_sweep_finish(p, sweep_grid(h->sm_count, p.wb), s);
  LB_CUDA(h, cudaGetLastError());
  if (getenv("LSHBLOOM_SWEEP_DEBUG")) {   // diagnostic: record counts of the bins
    cudaStreamSynchronize(s);
    std::vector<uint32_t> cur(p.nbins), cc(p.two_level ? p.g.bl * p.ncb : 0);
    uint32_t ovf = 0;
    cudaMemcpy(cur.data(), p.cursor, p.nbins * 4, cudaMemcpyDeviceToHost);
    if (p.two_level) cudaMemcpy(cc.data(), p.ccursor, cc.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ovf, p.ovf, 4, cudaMemcpyDeviceToHost);
    uint64_t sf = 0, sc = 0, mf = 0, mc = 0;
    for (auto v : cur) { sf += v; mf = std::max<uint64_t>(mf, v); }
    for (auto v : cc) { sc += v; mc = std::max<uint64_t>(mc, v); }
    fprintf(stderr, "sweep n=%u wb=%u cap=%u two=%u cb=%u ncb=%lu ccap=%u ovf=%u records=%lu fine_sum=%lu fine_max=%lu coarse_sum=%lu coarse_max=%lu\n",
            p.n, p.wb, p.cap, p.two_level, p.cb, (unsigned long)p.ncb, p.ccap, ovf, (unsigned long)((uint64_t)p.n * h->k * h->bl),
            (unsigned long)sf, (unsigned long)mf, (unsigned long)sc, (unsigned long)mc);
  }
  if (last) stage_end(h, 2, s);
  h->sweeps++;
  return LSHBLOOM_OK;
}

// The sweep path over band hashes that already exist (query_insert_bands): pieces of
// <= kSweepMaxDocs documents, each binned then swept.
int run_bloom_sweep(lshbloom* h, const SweepPlan& sp, const uint64_t* bh_dev, uint64_t bh_sj, uint64_t bh_si,
                    uint64_t n, uint8_t* dup_dev, cudaStream_t s, const DupSink* peers) {
  int rc = sweep_alloc(h, sp, s);
  if (rc) return rc;
  if (bh_si != 1 && h->bl > 1) {          // row-major [n][bl]: transpose so the binning reads coalesced
    LB_CUDA(h, ensure(h->sw_bht, n * h->bl * 8));
    h->launches += launch_transpose_bh(bh_dev, (uint64_t*)h->sw_bht.p, (uint32_t)n, h->bl, s);
    bh_dev = (const uint64_t*)h->sw_bht.p;
    bh_sj = n;
    bh_si = 1;
  }
  const BloomParams g = bloom_params(h, bh_dev, bh_sj, bh_si, dup_dev, peers);
  stage_begin(h, 1, s);
  for (uint64_t i0 = 0; i0 < n; i0 += kSweepMaxDocs) {
    const uint64_t i1 = std::min(n, i0 + kSweepMaxDocs);
    const SweepParams p = sweep_params(h, sp, g, i0, i1 - i0);
    if ((rc = sweep_begin(h, p, s)) || (rc = sweep_bin(h, p, i0, i1, s)) ||
        (rc = sweep_finish(h, p, s, i0 == 0, i1 == n)))
      return rc;
  }
  stage_end(h, 1, s);
  return LSHBLOOM_OK;
}

// The Bloom stage over bh_dev for documents [0, n): sweep or random access (results identical).
int run_bloom_any(lshbloom* h, const uint64_t* bh_dev, uint64_t bh_sj, uint64_t bh_si, uint64_t n,
                  uint8_t* dup_dev, cudaStream_t s, const DupSink* peers = nullptr) {
  const SweepPlan sp = plan_sweep(h, n);
  if (sp.use) return run_bloom_sweep(h, sp, bh_dev, bh_sj, bh_si, n, dup_dev, s, peers);
  return run_bloom(h, bh_dev, bh_sj, bh_si, 0, n, dup_dev, s, true, true, peers);
}

// query_insert: K1 over document chunks (alternately on the caller's stream s and k1_stream2),
// each chunk's Bloom sub-batches on bloom_stream as soon as its band hashes exist, so the
// integer-bound K1 of chunk c+1 overlaps the memory-bound Bloom kernels of chunk c.  Bloom
// sub-batches stay in document order (one stream), which is all the exact semantics need.
// Staging buffers of a host batch in the fused step.  A third buffer lets the copy of chunk
// c+3 start when K1 of chunk c ends instead of c+1's: with long documents (large chunks) that
// keeps the copy ahead (C3 e2e 70.8 -> 67.5 ms per 100K, C4 35.8 -> 33.8 ms per 200K); with
// abstract lengths it costs a little (C2 19.64 -> 19.72 ms), so: 3 when the batch averages
// more than 512 tokens per document.  LSHBLOOM_HOST_BUFS=2|3 overrides.
int host_bufs(uint64_t n_docs, uint64_t n_tokens) {
  static const int v = [] {
    const char* e = getenv("LSHBLOOM_HOST_BUFS");
    return e ? (atoi(e) == 3 ? 3 : 2) : 0;
  }();
  if (v) return v;
  return n_tokens > 512 * n_docs ? 3 : 2;
}

uint64_t fuse_edge_docs() {   // small first / last chunks: Bloom starts early, short tail
  static uint64_t v = 0;
  if (!v) {
    const char* e = getenv("LSHBLOOM_FUSE_EDGE");
    v = e ? std::max<uint64_t>(1024, strtoull(e, nullptr, 10)) : 16384;
  }
  return v;
}

// Middle K1 chunk, swept per workload with the two K1 streams: 128 permutations (C2) 32K
// documents (16K: 19.16 vs 18.98 ms); 256 (the length-split K1 of C3 / C4) 16K (C4 32.3 vs
// 34.2 ms per 200K, C3 63.3 vs 64.5 ms per 100K; 8K and 12K slower).
uint64_t fuse_docs(uint32_t npl) {
  static const uint64_t v = [] {
    const char* e = getenv("LSHBLOOM_FUSE_DOCS");
    return e ? std::max<uint64_t>(1024, strtoull(e, nullptr, 10)) : 0;
  }();
  return v ? v : (npl >= 8 ? 16384 : 32768);
}

uint64_t fuse_chunk_end(uint64_t d0, uint64_t n, uint32_t npl) {
  const uint64_t kFuseDocs = fuse_docs(npl);
  const uint64_t kFuseEdgeDocs = fuse_edge_docs();
  if (d0 == 0) return std::min(n, kFuseEdgeDocs);
  const uint64_t left = n - d0;
  if (left <= kFuseEdgeDocs) return n;
  if (left <= kFuseDocs + kFuseEdgeDocs) return n - kFuseEdgeDocs;
  return d0 + kFuseDocs;
}

// Enqueue one query_insert batch into slot `si` (its buffers and error state) without waiting for
// it: K1 chunks on the handle's K1 streams, the Bloom stage on the Bloom stream (stream order =
// batch order, which is all the exact semantics need), the flags copied out (host batches) and
// the slot's `done` event recorded on the Bloom stream.  The caller's stream s only provides the
// inputs: the K1 streams wait for its current position; nothing on s waits for this batch.
// ddup: device flag buffer (the caller's when on_device, else the slot's); dup_host: host flags.
int run_query_insert(lshbloom* h, const lshbloom_batch* b, cudaStream_t s, int si, uint8_t* ddup, uint8_t* dup_host) {
  const uint64_t n = b->n_docs;
  lshbloom::Slot& sl = h->slot[si];
  h->d_err = h->d_err_base + 1 + si;
  h->tset = si;
  LB_CUDA(h, ensure(sl.bh, n * h->bl * sizeof(uint64_t)));
  uint64_t* bh = (uint64_t*)sl.bh.p;
  MinhashParams p = base_params(h);
  if (h->npl >= 8) {   // scratch of the length-partitioned K1 launches (lb_minhash.cu), per K1 stream
    int rc0 = grow(h, h->part, (6 * (size_t)b->n_docs + 6 + 3 * (b->n_docs / 1024 + 1)) * sizeof(uint32_t));
    if (rc0) return rc0;
  }
  p.bh_out = bh;
  p.map = resolve_map(owned_band_major_map(h, n), bh, h->cfg.b);
  const uint64_t chunk_tokens = b->on_device ? 0 : kChunkTokens;
  if (!b->on_device && b->offsets[0] != 0) return fail(h, LSHBLOOM_EUSAGE, "offsets[0] must be 0");
  // Landing-gated host batch: the whole token array is copied into the slot's device buffer in
  // 2^land_log2-token pieces on the copy stream while K1 runs over it in the device-resident
  // chunking, each warp waiting only for its own document's tokens (MinhashParams::landed):
  // no staging-sized K1 chunks, no tails per staging buffer.  Needs the stream write and a
  // buffer of the batch's size (at most 1/8 of device memory); otherwise the staging path.
  const uint64_t n_tok_host = b->on_device ? 0 : b->offsets[n];
  const bool landing = !b->on_device && h->write_value32 &&
                       n_tok_host * sizeof(uint32_t) <= h->total_mem / 8;
  const bool dev_chunks = b->on_device || landing;
  // Bloom path: with the sweep, each chunk's probes are binned right after its K1 (overlapping
  // the next chunk's K1) and every piece of <= kSweepMaxDocs documents is swept once complete;
  // chunk boundaries fall on piece boundaries.
  const SweepPlan sp = plan_sweep(h, n);
  // With the sweep the Bloom work per chunk is only the binning, so K1 runs in larger chunks (a
  // K1 launch ends with a tail on a few warps; fewer launches, fewer tails):
  // LSHBLOOM_FUSE_DOCS_SWEEP documents per chunk.
  static const uint64_t sweep_chunk = [] {
    const char* e = getenv("LSHBLOOM_FUSE_DOCS_SWEEP");
    return e ? std::max<uint64_t>(1024, strtoull(e, nullptr, 10)) : (uint64_t)262144;
  }();
  // (host batches keep their staging-sized chunks: those overlap the H2D copy with K1)
  auto clip = [&](uint64_t d0, uint64_t d1) {
    if (!sp.use) return d1;
    if (dev_chunks) d1 = std::max(d1, std::min(n, d0 + sweep_chunk));
    return std::min(d1, (d0 / kSweepMaxDocs + 1) * kSweepMaxDocs);
  };
  // Chunk bounds first, all of them checked before anything is enqueued: a host batch's copies
  // read tokens [offsets[d0], offsets[d1]) of the caller's buffer, so every bound must satisfy
  // 0 <= t0 <= t1 <= offsets[n] (the rest of the CSR is validated on the device by K0, which gates
  // every kernel before any filter mutation).
  std::vector<std::pair<uint64_t, uint64_t>> chunks;
  {
    uint64_t d0 = 0;
    while (d0 < n) {
      uint64_t d1;
      if (dev_chunks) {
        d1 = clip(d0, fuse_chunk_end(d0, n, h->npl));
        if (landing && (b->offsets[d1] < b->offsets[d0] || b->offsets[d1] > n_tok_host))
          return fail(h, LSHBLOOM_EUSAGE, "malformed offsets near index " + std::to_string(d0) +
                                              " (decreasing, or beyond offsets[n_docs])");
      } else {
        const uint64_t t0 = b->offsets[d0];
        const uint64_t* lim = std::upper_bound(b->offsets + d0 + 1, b->offsets + n + 1, t0 + chunk_tokens);
        d1 = (uint64_t)(lim - b->offsets) - 1;
        // at least ~3.5 documents per resident K1 warp (8192 on 148 SMs), however long the
        // documents: with full-text lengths 64 MB is ~1.7 documents per warp and a chunk would last
        // as long as its slowest warp (C3 e2e: 155 vs 66 ms per 100K documents).  With the two K1
        // streams the next chunk fills that tail, so the floor is lower than with one stream (16
        // per warp): C3 e2e 71.8 -> 70.0 ms per 100K, C4 36.5 -> 35.7 ms per 200K (2K-16K swept).
        static const uint64_t env_min_docs = [] {
          const char* e = getenv("LSHBLOOM_HOST_MIN_DOCS");
          return e ? std::max<uint64_t>(1, strtoull(e, nullptr, 10)) : 0;
        }();
        const uint64_t min_docs =
            env_min_docs ? env_min_docs : (7ull * h->sm_count * 2 * (K1_THREADS_HOST / 32) + 1) / 2;
        d1 = std::max(d1, std::min(n, d0 + min_docs));
        if (d1 <= d0) d1 = d0 + 1;
        d1 = clip(d0, std::min(d1, fuse_chunk_end(d0, n, h->npl)));
        const uint64_t t1 = b->offsets[d1];
        if (t1 < t0 || t1 > b->offsets[n])
          return fail(h, LSHBLOOM_EUSAGE, "malformed offsets near index " + std::to_string(d0) +
                                              " (decreasing, or beyond offsets[n_docs])");
      }
      chunks.emplace_back(d0, d1);
      d0 = d1;
    }
  }
  int rc;
  if (sp.use && (rc = sweep_alloc(h, sp, h->bloom_stream))) return rc;
  const BloomParams bp = bloom_params(h, bh, n, 1, ddup, nullptr);
  p.beside_random_bloom = sp.use ? 0u : 1u;
  // K1 chunks alternate between the K1 streams: each launch ends with a tail in which its last
  // documents finish on a few warps, and the next chunk's blocks fill the SM slots meanwhile.
  // Each stream has its own work counter, partition scratch and staging buffer (host batches).
  const bool alt = h->k1_alt;
  const int nks = alt ? h->k1_nstreams : 1;
  cudaStream_t kst[3] = {h->k1_stream1, h->k1_stream2, h->k1_stream3};
  cudaStream_t s0 = kst[0];
  LB_CUDA(h, cudaEventRecord(h->ev_in, s));                // the inputs, as of this call
  LB_CUDA(h, cudaStreamWaitEvent(s0, h->ev_in, 0));
  if ((rc = reset_err(h, s0))) return rc;
  int nbuf = 2;
  if (b->on_device) {
    h->launches += launch_validate(b->offsets, n, h->d_err, s0);
    p.offsets = b->offsets;
    p.tokens = b->tokens;
    p.tok_base = 0;
  } else {
    // No O(n) host pass: the offsets are validated on the device (K0), which gates every kernel;
    // the host only checked what its own copies depend on (offsets[0], chunk bounds, above).
    LB_CUDA(h, ensure(sl.off, (n + 1) * sizeof(uint64_t)));
    LB_CUDA(h, cudaMemcpyAsync(sl.off.p, b->offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s0));
    h->launches += launch_validate((const uint64_t*)sl.off.p, n, h->d_err, s0);
    p.offsets = (const uint64_t*)sl.off.p;
    if (landing) {
      LB_CUDA(h, ensure(sl.tokall, n_tok_host * sizeof(uint32_t)));   // (the slot is idle: collected)
      p.tokens = (const uint32_t*)sl.tokall.p;
      p.tok_base = 0;
      p.landed = sl.landed;
      p.land_log2 = h->land_log2;
      p.tok_total = n_tok_host;
      p.err_state = h->d_err;
    } else {
      nbuf = host_bufs(n, b->offsets[n]);
      const uint64_t buf_tokens = std::max<uint64_t>(1, std::min(chunk_tokens, b->offsets[n]));
      for (int i = 0; i < nbuf; i++)
        if (buf_tokens * sizeof(uint32_t) > h->tok[i].cap) {
          LB_CUDA(h, cudaEventSynchronize(h->ev_k1[i]));     // its last reader is done
          LB_CUDA(h, ensure(h->tok[i], buf_tokens * sizeof(uint32_t)));
        }
    }
  }
  LB_CUDA(h, cudaEventRecord(h->ev_pre, s0));               // error gate and offsets ready
  if (landing) {
    // every piece and its landing mark are enqueued before any K1 launch, so a waiting warp
    // only ever waits on copy-engine work (no SM involved).  The copies depend only on the
    // caller's inputs and on the slot's previous K1 reader -- not on the K1 streams' position --
    // so with two slots batch t+1's tokens land while batch t's K1 still runs (the copy engine
    // never idles between streamed host batches); the landing counter is zeroed on the copy
    // stream itself, and the K1 streams wait for that (a stale count would open the gate early)
    LB_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_in, 0));
    LB_CUDA(h, cudaStreamWaitEvent(h->copy_stream, sl.tok_free, 0));
    // (a stream write, not a memset: a memset kernel would queue behind the resident K1 blocks)
    if (h->write_value32((CUstream)h->copy_stream, (CUdeviceptr)sl.landed, 0u, 0) != CUDA_SUCCESS)
      return fail(h, LSHBLOOM_ERUNTIME, "cuStreamWriteValue32 failed");
    LB_CUDA(h, cudaEventRecord(sl.land_zero, h->copy_stream));
    const uint64_t piece = 1ull << h->land_log2;
    uint32_t i = 0;
    for (uint64_t t0 = 0; t0 < n_tok_host; t0 += piece) {
      const uint64_t t1 = std::min(n_tok_host, t0 + piece);
      LB_CUDA(h, cudaMemcpyAsync((uint32_t*)sl.tokall.p + t0, b->tokens + t0, (t1 - t0) * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, h->copy_stream));
      if (h->write_value32((CUstream)h->copy_stream, (CUdeviceptr)sl.landed, ++i, 0) != CUDA_SUCCESS)
        return fail(h, LSHBLOOM_ERUNTIME, "cuStreamWriteValue32 failed");
    }
    static const bool land_diag = [] { const char* e = getenv("LSHBLOOM_LAND_DIAG"); return e && atoi(e); }();
    if (land_diag) {   // diagnostic: K1 starts only after the whole copy (no overlap)
      LB_CUDA(h, cudaEventRecord(h->ev_h2d[0], h->copy_stream));
      for (int k = 0; k < nks; k++) LB_CUDA(h, cudaStreamWaitEvent(kst[k], h->ev_h2d[0], 0));
    }
  }
  for (int k = 1; k < nks; k++) LB_CUDA(h, cudaStreamWaitEvent(kst[k], h->ev_pre, 0));
  if (landing)
    for (int k = 0; k < nks; k++) LB_CUDA(h, cudaStreamWaitEvent(kst[k], sl.land_zero, 0));
  LB_CUDA(h, cudaStreamWaitEvent(h->bloom_stream, h->ev_pre, 0));
  LB_CUDA(h, cudaMemsetAsync(ddup, 0, n, h->bloom_stream));
  int c = 0;
  stage_begin(h, 0, s0);
  for (const auto& ch : chunks) {
    const uint64_t d0 = ch.first, d1 = ch.second;
    if (!dev_chunks) {
      const uint64_t t0 = b->offsets[d0], t1 = b->offsets[d1];
      const int buf = c % nbuf;
      if ((t1 - t0) * sizeof(uint32_t) > h->tok[buf].cap) {   // a chunk larger than the buffer
        LB_CUDA(h, cudaEventSynchronize(h->ev_k1[buf]));   // its last reader is done
        LB_CUDA(h, ensure(h->tok[buf], (t1 - t0) * sizeof(uint32_t)));
      }
      LB_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_k1[buf], 0));
      LB_CUDA(h, cudaMemcpyAsync(h->tok[buf].p, b->tokens + t0, (t1 - t0) * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, h->copy_stream));
      LB_CUDA(h, cudaEventRecord(h->ev_h2d[buf], h->copy_stream));
      LB_CUDA(h, cudaStreamWaitEvent(kst[c % nks], h->ev_h2d[buf], 0));
      p.tokens = (const uint32_t*)h->tok[buf].p;
      p.tok_base = t0;
    }
    const int par = c % nks;
    cudaStream_t ks = kst[par];
    p.doc0 = (uint32_t)d0;
    p.n_docs = (uint32_t)(d1 - d0);
    p.counter = h->d_counters + 1 + par;
    if (h->npl >= 8) {
      p.part_lists = (uint32_t*)h->part.p + (size_t)par * 2 * n;
      p.part_counts = (uint32_t*)h->part.p + 6 * n + 2 * par;
      p.part_blk = (uint32_t*)h->part.p + 6 * n + 6 + (size_t)par * (n / 1024 + 1);
    }
    LB_CUDA(h, cudaMemsetAsync(p.counter, 0, 4, ks));
    int l = launch_minhash(p, (int)h->npl, h->sm_count, ks, h->k1_bps);
    if (l < 0) return fail(h, LSHBLOOM_EUSAGE, "unsupported num_perm");
    h->launches += l;
    LB_CUDA(h, cudaGetLastError());
    if (!dev_chunks) LB_CUDA(h, cudaEventRecord(h->ev_k1[c % nbuf], ks));
    LB_CUDA(h, cudaEventRecord(h->ev_fuse, ks));
    if (d1 == n) {   // every K1 stream joined into the first before the stage's end mark
      cudaEvent_t ej[3] = {nullptr, h->ev_join, h->ev_join3};
      for (int k = 1; k < nks; k++) {
        LB_CUDA(h, cudaEventRecord(ej[k], kst[k]));
        LB_CUDA(h, cudaStreamWaitEvent(s0, ej[k], 0));
      }
      stage_end(h, 0, s0);
      if (landing) LB_CUDA(h, cudaEventRecord(sl.tok_free, s0));
    }
    LB_CUDA(h, cudaStreamWaitEvent(h->bloom_stream, h->ev_fuse, 0));
    if (!sp.use) {
      if ((rc = run_bloom(h, bh, n, 1, d0, d1, ddup, h->bloom_stream, d0 == 0, d1 == n))) return rc;
    } else {
      const uint64_t p0 = d0 / kSweepMaxDocs * kSweepMaxDocs, p1 = std::min(n, p0 + kSweepMaxDocs);
      const SweepParams sw = sweep_params(h, sp, bp, p0, p1 - p0);
      if (d0 == 0) stage_begin(h, 1, h->bloom_stream);
      if (d0 == p0 && (rc = sweep_begin(h, sw, h->bloom_stream))) return rc;
      if ((rc = sweep_bin(h, sw, d0, d1, h->bloom_stream))) return rc;
      if (d1 == p1 && (rc = sweep_finish(h, sw, h->bloom_stream, p0 == 0, p1 == n))) return rc;
      if (d1 == n) stage_end(h, 1, h->bloom_stream);
    }
    c++;
  }
  if (dup_host) LB_CUDA(h, cudaMemcpyAsync(dup_host, ddup, n, cudaMemcpyDeviceToHost, h->bloom_stream));
  LB_CUDA(h, cudaEventRecord(sl.done, h->bloom_stream));
  return LSHBLOOM_OK;
}

int finish(lshbloom* h, cudaStream_t s) {
  LB_CUDA(h, cudaStreamSynchronize(s));
  LB_CUDA(h, cudaGetLastError());
  stage_collect(h, 2);
  return read_err(h);
}

// Synchronous entry points other than query_insert: drain the async batches first, then run on
// error state 0 / event set 2.
int begin_sync(lshbloom* h) {
  int rc = drain(h);
  if (rc) return rc;
  h->d_err = h->d_err_base;
  h->tset = 2;
  return LSHBLOOM_OK;
}

}  // namespace

extern "C" {

int lshbloom_create(uint32_t num_perm, uint32_t b, uint32_t r, uint64_t n_expected, double fp_rate,
                    uint64_t seed, lshbloom** out) {
  lshbloom_config c;
  memset(&c, 0, sizeof c);
  c.num_perm = num_perm;
  c.b = b;
  c.r = r;
  c.shingle_n = 5;
  c.n_expected = n_expected;
  c.fp_rate = fp_rate;
  c.seed = seed;
  c.device = -1;
  c.rank = 0;
  c.world = 1;
  c.sub_batch = 0;
  c.index_kind = LSHBLOOM_INDEX_BLOOM;
  return lshbloom_create_ex(&c, out);
}

int lshbloom_create_ex(const lshbloom_config* cfg, lshbloom** out) {
  if (!out) return fail(nullptr, LSHBLOOM_EUSAGE, "NULL out");
  *out = nullptr;
  if (!cfg) return fail(nullptr, LSHBLOOM_EUSAGE, "NULL config");
  lshbloom_config c = *cfg;
  if (c.num_perm == 0 || c.num_perm > LSHBLOOM_MAX_PERM) return fail(nullptr, LSHBLOOM_EUSAGE, "num_perm must be in [1, 1024]");
  if (c.b == 0 || c.b > LSHBLOOM_MAX_BANDS) return fail(nullptr, LSHBLOOM_EUSAGE, "b must be in [1, 64]");
  if (c.r == 0 || (uint64_t)c.b * c.r > c.num_perm) return fail(nullptr, LSHBLOOM_EUSAGE, "need r >= 1 and b*r <= num_perm (S:183)");
  if (c.shingle_n == 0) return fail(nullptr, LSHBLOOM_EUSAGE, "shingle_n must be >= 1");
  if (c.n_expected == 0) return fail(nullptr, LSHBLOOM_EUSAGE, "n_expected must be >= 1");
  if (c.index_kind > LSHBLOOM_INDEX_BLOCKED)
    return fail(nullptr, LSHBLOOM_EUSAGE, "index_kind must be 0 (Bloom), 1 (classic) or 2 (blocked Bloom)");
  const bool classic = c.index_kind == LSHBLOOM_INDEX_CLASSIC;
  if (!classic && !(c.fp_rate > 0.0 && c.fp_rate < 1.0)) return fail(nullptr, LSHBLOOM_EUSAGE, "fp_rate must be in (0, 1) (S:273)");
  if (c.bloom_path > LSHBLOOM_PATH_SWEEP) return fail(nullptr, LSHBLOOM_EUSAGE, "bloom_path must be 0 (auto), 1 (random) or 2 (sweep)");
  if (c.sweep_log2_window && (c.sweep_log2_window < 10 || c.sweep_log2_window > 19))
    return fail(nullptr, LSHBLOOM_EUSAGE, "sweep_log2_window must be 0 or in [10, 19]");
  if (!(c.lsh_threshold >= 0.0 && c.lsh_threshold <= 1.0))
    return fail(nullptr, LSHBLOOM_EUSAGE, "lsh_threshold must be 0 (unknown) or in (0, 1]");
  if (c.world == 0) c.world = 1;
  if (c.rank >= c.world) return fail(nullptr, LSHBLOOM_EUSAGE, "rank must be < world");
  if (c.world > c.b) return fail(nullptr, LSHBLOOM_EUSAGE, "world must be <= b (every rank owns >= 1 band)");

  // Sizing, P:224-225 / S:263 (DESIGN R9): natural log, ceil for m, llround for k.
  // (The classic index has no filters; a nominal p keeps the arithmetic below finite.)
  const double psz = classic ? 0.5 : c.fp_rate;
  const double md = ceil(-(double)c.n_expected * log(psz) / (log(2.0) * log(2.0)));
  if (!(md >= 1.0) || md >= 68719476736.0) return fail(nullptr, LSHBLOOM_EUSAGE, "filter size m must be < 2^36 bits");
  long long kk = llround((md / (double)c.n_expected) * log(2.0));
  if (kk < 1) kk = 1;
  if (kk > LSHBLOOM_MAX_K) return fail(nullptr, LSHBLOOM_EUSAGE, "k > 64 probes (fp_rate too small)");

  lshbloom* h = new lshbloom();
  h->cfg = c;
  h->m = (uint64_t)md;
  h->k = (uint32_t)kk;
  if (c.index_kind == LSHBLOOM_INDEX_BLOCKED) {   // m rounded up to whole 1024-bit blocks
    h->nb = (h->m + 1023) / 1024;
    h->nb_inv = ~0ull / h->nb;
    h->m = h->nb * 1024;
  }
  h->m_inv = ~0ull / h->m;
  h->W = 4 * ((h->m + 127) / 128);   // S:314 storage rounded up to 16 B (TMA bulk-copy granularity)
  const uint32_t base = c.b / c.world, rem = c.b % c.world;
  h->band_lo = c.rank * base + std::min(c.rank, rem);
  h->bl = base + (c.rank < rem ? 1 : 0);
  h->band_hi = h->band_lo + h->bl;
  uint32_t npl = 1;
  while (npl * 32 < c.num_perm) npl *= 2;
  h->npl = npl;
  h->sub_batch = c.sub_batch ? std::min<uint32_t>(c.sub_batch, 1u << 22) : kDefaultSubBatch;   // doc offsets: 22 bits in Q
  h->bloom_path = c.bloom_path;
  if (h->bloom_path == LSHBLOOM_PATH_AUTO)
    if (const char* e = getenv("LSHBLOOM_BLOOM_PATH"))
      h->bloom_path = !strcmp(e, "sweep") ? LSHBLOOM_PATH_SWEEP : !strcmp(e, "random") ? LSHBLOOM_PATH_RANDOM : 0;
  h->sweep_wb_force = c.sweep_log2_window;
  h->sweep_cap_force = c.sweep_cap;

  int dev = c.device;
  if (dev < 0) cudaGetDevice(&dev);
  h->device = dev;
  h->cfg.device = dev;
  DeviceGuard guard(dev);
  cudaError_t e;
#define CR(call)                                     \
  do {                                               \
    e = (call);                                      \
    if (e != cudaSuccess) {                          \
      int rc_ = fail_cuda(nullptr, e, #call);        \
      free_all(h);                                   \
      delete h;                                      \
      return rc_;                                    \
    }                                                \
  } while (0)
  CR(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, dev));
  {
    size_t fr = 0;
    CR(cudaMemGetInfo(&fr, &h->total_mem));
  }
  CR(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
  CR(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  {
    // the latency-bound Bloom kernels get priority over K1 for SM slots as blocks retire
    int lo = 0, hi = 0;
    CR(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (const char* e = getenv("LSHBLOOM_BLOOM_PRIO")) hi = atoi(e) ? hi : lo;
    CR(cudaStreamCreateWithPriority(&h->bloom_stream, cudaStreamNonBlocking, hi));
  }
  CR(cudaEventCreateWithFlags(&h->ev_fuse, cudaEventDisableTiming));
  CR(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CR(cudaStreamCreateWithFlags(&h->k1_stream2, cudaStreamNonBlocking));
  CR(cudaStreamCreateWithFlags(&h->k1_stream3, cudaStreamNonBlocking));
  CR(cudaEventCreateWithFlags(&h->ev_join3, cudaEventDisableTiming));
  CR(cudaStreamCreateWithFlags(&h->k1_stream1, cudaStreamNonBlocking));
  CR(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  CR(cudaEventCreateWithFlags(&h->ev_pre, cudaEventDisableTiming));
  for (auto& sl : h->slot) {
    CR(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    CR(cudaEventCreateWithFlags(&sl.tok_free, cudaEventDisableTiming));
    CR(cudaEventCreateWithFlags(&sl.land_zero, cudaEventDisableTiming));
    CR(cudaMalloc(&sl.landed, 4));
    CR(cudaMemset(sl.landed, 0, 4));
  }
  init_landing(h);
  if (const char* e = getenv("LSHBLOOM_K1_STREAMS")) h->k1_nstreams = std::min(3, std::max(1, atoi(e)));
  if (const char* e = getenv("LSHBLOOM_K1_ALT")) h->k1_alt = atoi(e) != 0;
  h->k1_bps = 4;   // leave room on every SM for the concurrent Bloom kernels
  if (const char* e = getenv("LSHBLOOM_K1_BPS")) h->k1_bps = atoi(e);
  for (int i = 0; i < 3; i++) {
    CR(cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming));
    CR(cudaEventCreateWithFlags(&h->ev_k1[i], cudaEventDisableTiming));
    CR(cudaEventRecord(h->ev_k1[i], h->own_stream));
  }
  for (auto& set : h->tev)
    for (auto& ev : set) CR(cudaEventCreate(&ev));

  // Hash family (DESIGN R5), in the kernel's limb layout.
  std::vector<PermCoef> coef(32 * npl);
  for (uint32_t i = 0; i < 32 * npl; i++) {
    uint64_t a = 1, bb = 0;
    if (i < c.num_perm) {
      a = 1 + R(c.seed, 1, 2ull * i) % (kP - 1);
      bb = R(c.seed, 1, 2ull * i + 1) % kP;
    }
    coef[i].a0 = (uint32_t)(a & 0x7FFFFFFFull);
    coef[i].a1 = (uint32_t)(a >> 31);
    coef[i].b0 = (uint32_t)bb;
    coef[i].b1 = (uint32_t)(bb >> 32);
  }
  std::vector<uint64_t> bcoef(2 * c.r);
  for (uint32_t u = 0; u < c.r; u++) {
    bcoef[u] = 1 + R(c.seed, 2, 2ull * u) % (kP - 1);
    bcoef[c.r + u] = R(c.seed, 2, 2ull * u + 1) % kP;
  }
  std::vector<uint64_t> s1(h->bl), s2(h->bl);
  for (uint32_t jl = 0; jl < h->bl; jl++) {
    s1[jl] = R(c.seed, 3, h->band_lo + jl);
    s2[jl] = R(c.seed, 4, h->band_lo + jl);
  }
  CR(cudaMalloc(&h->d_coef, coef.size() * sizeof(PermCoef)));
  CR(cudaMemcpy(h->d_coef, coef.data(), coef.size() * sizeof(PermCoef), cudaMemcpyHostToDevice));
  CR(cudaMalloc(&h->d_bcoef, bcoef.size() * 8));
  CR(cudaMemcpy(h->d_bcoef, bcoef.data(), bcoef.size() * 8, cudaMemcpyHostToDevice));
  CR(cudaMalloc(&h->d_s1, h->bl * 8));
  CR(cudaMalloc(&h->d_s2, h->bl * 8));
  CR(cudaMemcpy(h->d_s1, s1.data(), h->bl * 8, cudaMemcpyHostToDevice));
  CR(cudaMemcpy(h->d_s2, s2.data(), h->bl * 8, cudaMemcpyHostToDevice));

  if (classic) {
    // per owned band 2^c_log2cap slots, load factor <= 0.7 at n_expected documents
    uint32_t lg = 10;
    while ((double)(1ull << lg) * 0.7 < (double)c.n_expected) lg++;
    if (lg > 40) { free_all(h); delete h; return fail(nullptr, LSHBLOOM_EUSAGE, "n_expected too large for the classic index"); }
    h->c_log2cap = lg;
    h->m = 0;
    h->k = 0;
    h->W = 0;
    const size_t tbytes = ((size_t)h->bl << lg) * 8;
    CR(cudaMalloc(&h->d_ckeys, tbytes));
    CR(cudaMalloc(&h->d_cvals, tbytes));
    CR(cudaMemset(h->d_ckeys, 0xFF, tbytes));   // all slots empty
    CR(cudaMemset(h->d_cvals, 0xFF, tbytes));   // no document yet
    CR(cudaMalloc(&h->d_counters, 16 * 4));
    CR(cudaMemset(h->d_counters, 0, 16 * 4));
    CR(cudaMalloc(&h->d_err_base, 3 * sizeof(ErrState)));
    CR(cudaMemset(h->d_err_base, 0, 3 * sizeof(ErrState)));
    h->d_err = h->d_err_base;
    CR(cudaDeviceSynchronize());
    *out = h;
    return LSHBLOOM_OK;
  }

  // Filters "with all bits initially set to 0".
  const size_t fbytes = (size_t)h->bl * h->W * 4;
  CR(cudaMalloc(&h->d_F, fbytes));
  CR(cudaMemset(h->d_F, 0, fbytes));
  CR(cudaMalloc(&h->d_Q, 2 * (8ull << h->q_log2)));
  CR(cudaMemset(h->d_Q, 0xFF, 2 * (8ull << h->q_log2)));   // all slots empty (~0)

  // Earliest-setter table: >= 2x the most contested positions a sub-batch can produce
  // (each contested position has >= 2 of the sub_batch * bl * k probes).
  const uint64_t probes = (uint64_t)h->sub_batch * h->bl * h->k;
  uint32_t lg = 10;
  while ((1ull << lg) < probes) lg++;
  h->ecap_log2 = lg;
  CR(cudaMalloc(&h->d_ekey, (8ull << lg)));
  CR(cudaMalloc(&h->d_eval, (8ull << lg)));
  CR(cudaMemset(h->d_ekey, 0, (8ull << lg)));
  CR(cudaMemset(h->d_eval, 0, (8ull << lg)));
  CR(cudaMalloc(&h->d_st, 2ull * h->sub_batch * h->bl * 8));
  CR(cudaMalloc(&h->d_cand, (size_t)h->sub_batch * h->bl * 4));
  CR(cudaMalloc(&h->d_clist, (size_t)h->sub_batch * h->bl * h->k * 8));
  if (const char* e = getenv("LSHBLOOM_CB_LOG2")) h->cb_log2 = std::max(10, std::min(30, atoi(e)));
  CR(cudaMalloc(&h->d_cb, 1ull << (h->cb_log2 - 3)));
  CR(cudaMalloc(&h->d_counters, 16 * 4));
  CR(cudaMemset(h->d_counters, 0, 16 * 4));
  CR(cudaMalloc(&h->d_err_base, 3 * sizeof(ErrState)));
  CR(cudaMemset(h->d_err_base, 0, 3 * sizeof(ErrState)));
  h->d_err = h->d_err_base;
  CR(cudaDeviceSynchronize());
#undef CR
  *out = h;
  return LSHBLOOM_OK;
}

void lshbloom_destroy(lshbloom* h) {
  if (!h) return;
  {
    DeviceGuard g(h->device);
    cudaDeviceSynchronize();                 // batches in flight, every internal stream
    free_all(h);
  }
  delete h;
}

int lshbloom_signatures(lshbloom* h, const lshbloom_batch* b, uint32_t* sig_out) {
  int rc = check_handle(h);
  if (rc) return rc;
  if ((rc = check_batch(h, b))) return rc;
  if (!sig_out) return fail(h, LSHBLOOM_EUSAGE, "NULL sig_out");
  if ((rc = begin_sync(h))) return rc;
  DeviceGuard g(h->device);
  cudaStream_t s = b->stream ? (cudaStream_t)b->stream : h->own_stream;
  const size_t bytes = b->n_docs * h->cfg.num_perm * sizeof(uint32_t);
  uint32_t* dsig = sig_out;
  if (!b->on_device) {
    LB_CUDA(h, ensure(h->sig, bytes));
    dsig = (uint32_t*)h->sig.p;
  }
  BandMap none;
  memset(&none, 0, sizeof none);
  if ((rc = run_minhash(h, b, s, dsig, nullptr, none))) return rc;
  if (!b->on_device) LB_CUDA(h, cudaMemcpyAsync(sig_out, dsig, bytes, cudaMemcpyDeviceToHost, s));
  return finish(h, s);
}

static int band_hashes_impl(lshbloom* h, const lshbloom_batch* b, uint64_t* bh_out, bool sharded) {
  int rc = check_handle(h);
  if (rc) return rc;
  if ((rc = check_batch(h, b))) return rc;
  if (!bh_out) return fail(h, LSHBLOOM_EUSAGE, "NULL bh_out");
  if ((rc = begin_sync(h))) return rc;
  DeviceGuard g(h->device);
  cudaStream_t s = b->stream ? (cudaStream_t)b->stream : h->own_stream;
  const size_t bytes = b->n_docs * h->cfg.b * sizeof(uint64_t);
  uint64_t* dbh = bh_out;
  if (!b->on_device) {
    LB_CUDA(h, ensure(h->bh, bytes));
    dbh = (uint64_t*)h->bh.p;
  }
  if ((rc = run_minhash(h, b, s, nullptr, dbh, sharded ? sharded_map(h, b->n_docs) : full_map(h)))) return rc;
  if (!b->on_device) LB_CUDA(h, cudaMemcpyAsync(bh_out, dbh, bytes, cudaMemcpyDeviceToHost, s));
  return finish(h, s);
}

int lshbloom_band_hashes(lshbloom* h, const lshbloom_batch* b, uint64_t* bh_out) {
  return band_hashes_impl(h, b, bh_out, false);
}

int lshbloom_band_hashes_sharded(lshbloom* h, const lshbloom_batch* b, uint64_t* bh_out) {
  return band_hashes_impl(h, b, bh_out, true);
}

int lshbloom_stage_times(lshbloom* h, int32_t enable, double* ms_out, uint64_t* n_out) {
  int rc = check_handle(h);
  if (rc) return rc;
  h->timing = enable != 0;
  for (int st = 0; st < LSHBLOOM_NSTAGES; st++) {
    if (ms_out) ms_out[st] = h->stage_ms[st];
    if (n_out) n_out[st] = h->stage_n[st];
    h->stage_ms[st] = 0;
    h->stage_n[st] = 0;
  }
  return LSHBLOOM_OK;
}

// Shared by the synchronous and asynchronous forms: validate, take the next slot (waiting for
// the batch that last used it), enqueue.
static int enqueue_query_insert(lshbloom* h, const lshbloom_batch* b, uint8_t* dup_out, int* slot_out) {
  int rc = check_handle(h);
  if (rc) return rc;
  if ((rc = check_batch(h, b))) return rc;
  if (!dup_out) return fail(h, LSHBLOOM_EUSAGE, "NULL dup_out");
  if (h->cfg.index_kind == LSHBLOOM_INDEX_CLASSIC) {
    // the classic index keeps the document count in its table layout: no batches in flight
    if ((rc = drain(h))) return rc;
    if ((rc = classic_capacity(h, b->n_docs))) return rc;
  }
  DeviceGuard g(h->device);
  cudaStream_t s = b->stream ? (cudaStream_t)b->stream : h->own_stream;
  const int si = h->next_slot;
  if ((rc = collect(h, si))) return rc;                    // the batch two calls back is done
  lshbloom::Slot& sl = h->slot[si];
  uint8_t* ddup = dup_out;
  if (!b->on_device) {
    LB_CUDA(h, ensure(sl.dup, b->n_docs));
    ddup = (uint8_t*)sl.dup.p;
  }
  if ((rc = run_query_insert(h, b, s, si, ddup, b->on_device ? nullptr : dup_out))) {
    // nothing of this batch can have mutated the filters (its K0 gate or a host check failed
    // before any launch), but kernels and copies may be queued: let them finish before returning
    for (cudaStream_t q : {h->k1_stream1, h->k1_stream2, h->k1_stream3, h->copy_stream, h->bloom_stream})
      cudaStreamSynchronize(q);
    return rc;
  }
  sl.busy = true;
  sl.n = b->n_docs;
  sl.seq = ++h->seq;
  h->next_slot ^= 1;
  h->doc_count += b->n_docs;
  if (slot_out) *slot_out = si;
  return LSHBLOOM_OK;
}

int lshbloom_query_insert(lshbloom* h, const lshbloom_batch* b, uint8_t* dup_out) {
  int rc = check_handle(h);
  if (rc) return rc;
  if ((rc = drain(h))) return rc;
  int si = 0;
  if ((rc = enqueue_query_insert(h, b, dup_out, &si))) return rc;
  DeviceGuard g(h->device);
  cudaStream_t s = b->stream ? (cudaStream_t)b->stream : h->own_stream;
  LB_CUDA(h, cudaStreamWaitEvent(s, h->slot[si].done, 0));  // stream order for the caller's later work
  LB_CUDA(h, cudaGetLastError());
  if ((rc = collect(h, si))) return rc;
  rc = h->async_rc;
  if (rc) {
    h->err = h->async_msg;
    h->async_rc = 0;
  }
  return rc;
}

int lshbloom_query_insert_async(lshbloom* h, const lshbloom_batch* b, uint8_t* dup_out) {
  return enqueue_query_insert(h, b, dup_out, nullptr);
}

int lshbloom_sync(lshbloom* h) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard g(h->device);
  if ((rc = drain(h))) return rc;
  LB_CUDA(h, cudaStreamSynchronize(h->bloom_stream));
  rc = h->async_rc;
  if (rc) {
    h->err = h->async_msg;
    h->async_rc = 0;
  }
  return rc;
}

int lshbloom_query_insert_bands(lshbloom* h, const uint64_t* bh_owned, uint64_t n_docs, int32_t on_device,
                                void* stream, uint8_t* hit_out) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!bh_owned || !hit_out) return fail(h, LSHBLOOM_EUSAGE, "NULL bh_owned / hit_out");
  if (n_docs == 0 || n_docs > 0xFFFFFFFFull) return fail(h, LSHBLOOM_EUSAGE, "n_docs must be in [1, 2^32)");
  if ((rc = begin_sync(h))) return rc;
  if ((rc = classic_capacity(h, n_docs))) return rc;
  DeviceGuard g(h->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : h->own_stream;
  const size_t bytes = n_docs * h->bl * sizeof(uint64_t);
  const uint64_t* dbh = bh_owned;
  uint8_t* dhit = hit_out;
  if (!on_device) {
    LB_CUDA(h, ensure(h->bh, bytes));
    LB_CUDA(h, ensure(h->dup, n_docs));
    LB_CUDA(h, cudaMemcpyAsync(h->bh.p, bh_owned, bytes, cudaMemcpyHostToDevice, s));
    dbh = (const uint64_t*)h->bh.p;
    dhit = (uint8_t*)h->dup.p;
  }
  if ((rc = reset_err(h, s))) return rc;
  LB_CUDA(h, cudaMemsetAsync(dhit, 0, n_docs, s));
  if ((rc = run_bloom_any(h, dbh, 1, h->bl, n_docs, dhit, s))) return rc;
  if (!on_device) LB_CUDA(h, cudaMemcpyAsync(hit_out, dhit, n_docs, cudaMemcpyDeviceToHost, s));
  if ((rc = finish(h, s))) return rc;
  h->doc_count += n_docs;
  return LSHBLOOM_OK;
}

// ---- a batch of the owned bands assembled from band-hash chunks (pipelined sharded steps)
int lshbloom_bands_begin(lshbloom* h, uint64_t n_global) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (n_global == 0 || n_global > 0xFFFFFFFFull) return fail(h, LSHBLOOM_EUSAGE, "n_global must be in [1, 2^32)");
  if ((rc = classic_capacity(h, n_global))) return rc;
  DeviceGuard g(h->device);
  if ((rc = begin_sync(h))) return rc;
  LB_CUDA(h, cudaStreamSynchronize(h->bloom_stream));
  h->bands_plan = plan_sweep(h, n_global, n_global);          // one sweep over the whole batch
  LB_CUDA(h, ensure(h->bands_bh, n_global * h->bl * sizeof(uint64_t)));
  if (h->bands_plan.use) {
    if ((rc = sweep_alloc(h, h->bands_plan, h->bloom_stream))) return rc;
    const BloomParams bp = bloom_params(h, (const uint64_t*)h->bands_bh.p, n_global, 1, nullptr, nullptr);
    if ((rc = sweep_begin(h, sweep_params(h, h->bands_plan, bp, 0, n_global), h->bloom_stream))) return rc;
  }
  if ((rc = reset_err(h, h->bloom_stream))) return rc;
  h->bands_open = true;
  h->bands_n = n_global;
  h->bands_added = 0;
  return LSHBLOOM_OK;
}

int lshbloom_bands_add(lshbloom* h, const uint64_t* bh_owned, uint64_t doc0, uint64_t n_docs, void* stream) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->bands_open) return fail(h, LSHBLOOM_EUSAGE, "lshbloom_bands_add without lshbloom_bands_begin");
  if (n_docs == 0) return LSHBLOOM_OK;
  if (!bh_owned) return fail(h, LSHBLOOM_EUSAGE, "NULL bh_owned");
  if (doc0 > h->bands_n || n_docs > h->bands_n - doc0) return fail(h, LSHBLOOM_EUSAGE, "chunk beyond n_global");
  DeviceGuard g(h->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : h->own_stream;
  const uint64_t n = h->bands_n;
  // the chunk is copied (transposed) into the batch's band-major buffer on the Bloom stream, after
  // the caller's stream has produced it; the caller may reuse it once its stream passes ev_fuse
  LB_CUDA(h, cudaEventRecord(h->ev_in, s));
  LB_CUDA(h, cudaStreamWaitEvent(h->bloom_stream, h->ev_in, 0));
  h->launches += launch_transpose_bh(bh_owned, (uint64_t*)h->bands_bh.p, (uint32_t)n_docs, h->bl, h->bloom_stream, n,
                                     doc0);
  if (h->bands_plan.use) {                                     // bin this chunk's probes now
    const BloomParams bp = bloom_params(h, (const uint64_t*)h->bands_bh.p, n, 1, nullptr, nullptr);
    if ((rc = sweep_bin(h, sweep_params(h, h->bands_plan, bp, 0, n), doc0, doc0 + n_docs, h->bloom_stream))) return rc;
  }
  LB_CUDA(h, cudaEventRecord(h->ev_fuse, h->bloom_stream));
  LB_CUDA(h, cudaStreamWaitEvent(s, h->ev_fuse, 0));
  LB_CUDA(h, cudaGetLastError());
  h->bands_added += n_docs;
  return LSHBLOOM_OK;
}

int lshbloom_bands_finish(lshbloom* h, uint8_t* hit_out, void* stream) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->bands_open) return fail(h, LSHBLOOM_EUSAGE, "lshbloom_bands_finish without lshbloom_bands_begin");
  if (!hit_out) return fail(h, LSHBLOOM_EUSAGE, "NULL hit_out");
  h->bands_open = false;
  if (h->bands_added != h->bands_n)
    return fail(h, LSHBLOOM_EUSAGE, "lshbloom_bands_add covered " + std::to_string(h->bands_added) + " of " +
                                        std::to_string(h->bands_n) + " documents");
  DeviceGuard g(h->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : h->own_stream;
  const uint64_t n = h->bands_n;
  LB_CUDA(h, cudaEventRecord(h->ev_in, s));
  LB_CUDA(h, cudaStreamWaitEvent(h->bloom_stream, h->ev_in, 0));
  LB_CUDA(h, cudaMemsetAsync(hit_out, 0, n, h->bloom_stream));
  const uint64_t* bh = (const uint64_t*)h->bands_bh.p;
  if (h->bands_plan.use) {
    const BloomParams bp = bloom_params(h, bh, n, 1, hit_out, nullptr);
    stage_begin(h, 1, h->bloom_stream);
    if ((rc = sweep_finish(h, sweep_params(h, h->bands_plan, bp, 0, n), h->bloom_stream, true, true))) return rc;
    stage_end(h, 1, h->bloom_stream);
  } else if ((rc = run_bloom(h, bh, n, 1, 0, n, hit_out, h->bloom_stream))) {
    return rc;
  }
  LB_CUDA(h, cudaEventRecord(h->ev_fuse, h->bloom_stream));
  LB_CUDA(h, cudaStreamWaitEvent(s, h->ev_fuse, 0));
  if ((rc = finish(h, h->bloom_stream))) return rc;
  h->doc_count += n;
  return LSHBLOOM_OK;
}

int lshbloom_band_hashes_to_peers(lshbloom* h, const lshbloom_batch* b, uint64_t global_doc0, void* const* peer_recv) {
  int rc = check_handle(h);
  if (rc) return rc;
  if ((rc = check_batch(h, b))) return rc;
  const uint32_t world = h->cfg.world, nb = h->cfg.b, base = nb / world, rem = nb % world;
  if (!peer_recv) return fail(h, LSHBLOOM_EUSAGE, "NULL peer_recv");
  if ((rc = begin_sync(h))) return rc;
  for (uint32_t o = 0; o < world; o++)
    if (!peer_recv[o]) return fail(h, LSHBLOOM_EUSAGE, "NULL receive buffer of rank " + std::to_string(o));
  BandMap m;
  memset(&m, 0, sizeof m);
  for (uint32_t o = 0; o < world; o++) {
    const uint32_t lo = o * base + std::min(o, rem), cnt = base + (o < rem ? 1 : 0);
    for (uint32_t j = lo; j < lo + cnt; j++) {
      m.ncol[j] = cnt;
      m.ptr[j] = (uint64_t*)peer_recv[o] + global_doc0 * cnt + (j - lo);   // owner's [n_global][cnt] buffer
    }
  }
  DeviceGuard g(h->device);
  cudaStream_t s = b->stream ? (cudaStream_t)b->stream : h->own_stream;
  if ((rc = run_minhash(h, b, s, nullptr, (uint64_t*)peer_recv[0], m))) return rc;
  return finish(h, s);
}

int lshbloom_query_insert_bands_peers(lshbloom* h, const uint64_t* bh_owned, uint64_t n_global, const uint64_t* doc_start,
                                      void* const* peer_flags, void* stream) {
  int rc = check_handle(h);
  if (rc) return rc;
  const uint32_t world = h->cfg.world;
  if (!bh_owned || !doc_start || !peer_flags) return fail(h, LSHBLOOM_EUSAGE, "NULL bh_owned / doc_start / peer_flags");
  if (n_global == 0 || n_global > 0xFFFFFFFFull) return fail(h, LSHBLOOM_EUSAGE, "n_global must be in [1, 2^32)");
  if (world > (uint32_t)kMaxPeers) return fail(h, LSHBLOOM_EUSAGE, "world > 64");
  if (doc_start[0] != 0 || doc_start[world] != n_global)
    return fail(h, LSHBLOOM_EUSAGE, "doc_start must run from 0 to n_global");
  if ((rc = begin_sync(h))) return rc;
  DupSink sink;
  memset(&sink, 0, sizeof sink);
  sink.npeers = world;
  for (uint32_t r = 0; r < world; r++) {
    if (doc_start[r + 1] < doc_start[r]) return fail(h, LSHBLOOM_EUSAGE, "doc_start must be non-decreasing");
    if (doc_start[r + 1] > doc_start[r] && !peer_flags[r])
      return fail(h, LSHBLOOM_EUSAGE, "NULL flag buffer of rank " + std::to_string(r));
    sink.peer[r] = (uint8_t*)peer_flags[r];
    sink.start[r] = doc_start[r];
  }
  sink.start[world] = doc_start[world];
  if ((rc = classic_capacity(h, n_global))) return rc;
  DeviceGuard g(h->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : h->own_stream;
  if ((rc = reset_err(h, s))) return rc;
  if ((rc = run_bloom_any(h, bh_owned, 1, h->bl, n_global, nullptr, s, &sink))) return rc;
  if ((rc = finish(h, s))) return rc;
  h->doc_count += n_global;
  return LSHBLOOM_OK;
}

// Stream-ordered: the filters are zeroed on the Bloom stream after every batch enqueued before and
// before every batch enqueued after, so a reset between async batches does not drain them; with
// nothing in flight the call also waits for the zeroing (the synchronous behaviour).
int lshbloom_reset(lshbloom* h) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard g(h->device);
  const bool inflight = h->slot[0].busy || h->slot[1].busy;
  if (h->cfg.index_kind == LSHBLOOM_INDEX_CLASSIC) {
    const size_t tbytes = ((size_t)h->bl << h->c_log2cap) * 8;
    LB_CUDA(h, cudaMemsetAsync(h->d_ckeys, 0xFF, tbytes, h->bloom_stream));
    LB_CUDA(h, cudaMemsetAsync(h->d_cvals, 0xFF, tbytes, h->bloom_stream));
  } else {
    LB_CUDA(h, cudaMemsetAsync(h->d_F, 0, (size_t)h->bl * h->W * 4, h->bloom_stream));
  }
  if (!inflight) LB_CUDA(h, cudaStreamSynchronize(h->bloom_stream));
  h->doc_count = 0;
  for (auto& sl : h->slot) sl.n = 0;      // counted before the reset
  return LSHBLOOM_OK;
}

int lshbloom_filter_copy(lshbloom* h, uint32_t j, uint32_t* dst) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!dst || j < h->band_lo || j >= h->band_hi) return fail(h, LSHBLOOM_EUSAGE, "band not owned by this handle / NULL dst");
  if (h->cfg.index_kind == LSHBLOOM_INDEX_CLASSIC) return fail(h, LSHBLOOM_EUSAGE, "not a Bloom index");
  DeviceGuard g(h->device);
  if ((rc = drain(h))) return rc;
  LB_CUDA(h, cudaStreamSynchronize(h->bloom_stream));
  LB_CUDA(h, cudaMemcpy(dst, h->d_F + (uint64_t)(j - h->band_lo) * h->W, h->W * 4, cudaMemcpyDeviceToHost));
  return LSHBLOOM_OK;
}

int lshbloom_info(const lshbloom* h, lshbloom_info_t* out) {
  if (!h || !out) {
    g_create_error = "lshbloom_info: NULL handle / output";
    return LSHBLOOM_EUSAGE;
  }
  memset(out, 0, sizeof *out);
  out->m = h->m;
  out->k = h->k;
  out->num_perm = h->cfg.num_perm;
  out->b = h->cfg.b;
  out->r = h->cfg.r;
  out->shingle_n = h->cfg.shingle_n;
  out->band_lo = h->band_lo;
  out->band_hi = h->band_hi;
  out->words_per_band = h->W;
  out->filter_bytes = (uint64_t)h->bl * h->W * 4;
  out->p_eff = -expm1((double)h->cfg.b * log1p(-h->cfg.fp_rate));   // 1-(1-p)^b
  out->doc_count = h->doc_count;
  out->oversubscribed = h->doc_count > h->cfg.n_expected ? 1 : 0;
  out->seed = h->cfg.seed;
  out->n_expected = h->cfg.n_expected;
  out->fp_rate = h->cfg.fp_rate;
  out->index_kind = h->cfg.index_kind;
  out->lsh_threshold = h->cfg.lsh_threshold;
  out->sweeps = h->sweeps;
  if (h->cfg.index_kind == LSHBLOOM_INDEX_CLASSIC) {
    out->classic_slots = 1ull << h->c_log2cap;
    out->filter_bytes = ((uint64_t)h->bl << h->c_log2cap) * 16;
    out->p_eff = 0.0;
    out->oversubscribed = (double)h->doc_count > 0.7 * (double)out->classic_slots ? 1 : 0;
  }
  return LSHBLOOM_OK;
}

const char* lshbloom_last_error(const lshbloom* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

uint64_t lshbloom_launch_count(const lshbloom* h) { return h ? h->launches : 0; }

// S-curve objective of a (b, r) pair: weighted areas of false positives
// below T and false negatives above T, composite Simpson with 1000 subintervals.
static double scurve_area(double lo, double hi, uint32_t b, uint32_t r, bool fn) {
  const int N = 1000;
  const double h = (hi - lo) / N;
  auto f = [&](double s) {
    const double miss = std::pow(1.0 - std::pow(s, (double)r), (double)b);   // P(no band collides)
    return fn ? miss : 1.0 - miss;
  };
  double acc = f(lo) + f(hi);
  for (int i = 1; i < N; i++) acc += (i % 2 ? 4.0 : 2.0) * f(lo + i * h);
  return acc * h / 3.0;
}

int lshbloom_optimal_params(double threshold, uint32_t num_perm, double fp_weight, double fn_weight,
                            uint32_t* b_out, uint32_t* r_out) {
  if (!b_out || !r_out) return fail(nullptr, LSHBLOOM_EUSAGE, "NULL output");
  if (!(threshold > 0.0 && threshold <= 1.0)) return fail(nullptr, LSHBLOOM_EUSAGE, "threshold must be in (0, 1]");
  if (num_perm < 2) return fail(nullptr, LSHBLOOM_EUSAGE, "num_perm must be >= 2");
  if (!(fp_weight >= 0.0 && fn_weight >= 0.0)) return fail(nullptr, LSHBLOOM_EUSAGE, "weights must be >= 0");
  double best = INFINITY;
  uint32_t bb = 0, br = 0;
  for (uint32_t b = 1; b <= num_perm; b++)
    for (uint32_t r = 1; (uint64_t)b * r <= num_perm; r++) {
      const double e = fp_weight * scurve_area(0.0, threshold, b, r, false) +
                       fn_weight * scurve_area(threshold, 1.0, b, r, true);
      if (e < best) {   // strict: ties keep the smaller b, then the smaller r
        best = e;
        bb = b;
        br = r;
      }
    }
  *b_out = bb;
  *r_out = br;
  return LSHBLOOM_OK;
}

int lshbloom_plan(uint64_t n_docs, double p_effective, double threshold, uint32_t num_perm, lshbloom_plan_t* out) {
  if (!out) return fail(nullptr, LSHBLOOM_EUSAGE, "NULL output");
  if (n_docs == 0) return fail(nullptr, LSHBLOOM_EUSAGE, "n_docs must be >= 1");
  if (!(p_effective > 0.0 && p_effective < 1.0)) return fail(nullptr, LSHBLOOM_EUSAGE, "p_effective must be in (0, 1)");
  memset(out, 0, sizeof *out);
  int rc = lshbloom_optimal_params(threshold, num_perm, 0.5, 0.5, &out->b, &out->r);
  if (rc) return rc;
  out->p = -std::expm1(std::log1p(-p_effective) / out->b);    // 1-(1-p)^b = p_eff
  const double md = std::ceil(-(double)n_docs * std::log(out->p) / (std::log(2.0) * std::log(2.0)));
  long long kk = std::llround((md / (double)n_docs) * std::log(2.0));
  out->m = (uint64_t)md;
  out->k = (uint32_t)(kk < 1 ? 1 : kk);
  out->total_bytes = (uint64_t)out->b * ((out->m + 7) / 8);
  return LSHBLOOM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Checkpoint / resume in SPEC's LSHB / LBF1 little-endian formats.
#include <cstdio>
#if defined(__x86_64__)
#include <nmmintrin.h>
#endif

namespace {

uint32_t crc32c_table[256];
bool crc32c_init_done = false;

void crc32c_init() {
  if (crc32c_init_done) return;
  for (uint32_t i = 0; i < 256; i++) {
    uint32_t c = i;
    for (int k = 0; k < 8; k++) c = (c >> 1) ^ (0x82F63B78u & (0u - (c & 1)));
    crc32c_table[i] = c;
  }
  crc32c_init_done = true;
}

#if defined(__x86_64__)
__attribute__((target("sse4.2"))) uint32_t crc32c_hw(uint32_t crc, const uint8_t* p, size_t n) {
  uint64_t c = crc;
  while (n >= 8) {
    uint64_t v;
    memcpy(&v, p, 8);
    c = _mm_crc32_u64(c, v);
    p += 8;
    n -= 8;
  }
  uint32_t c32 = (uint32_t)c;
  while (n--) c32 = _mm_crc32_u8(c32, *p++);
  return c32;
}
#endif

// CRC32C (Castagnoli), running form: start with crc = 0, feed chunks, result is the CRC.
struct Crc32c {
  uint32_t state = 0xFFFFFFFFu;
  void update(const void* data, size_t n) {
    const uint8_t* p = (const uint8_t*)data;
#if defined(__x86_64__)
    if (__builtin_cpu_supports("sse4.2")) {
      state = crc32c_hw(state, p, n);
      return;
    }
#endif
    crc32c_init();
    uint32_t c = state;
    for (size_t i = 0; i < n; i++) c = crc32c_table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    state = c;
  }
  uint32_t value() const { return state ^ 0xFFFFFFFFu; }
};

struct Writer {
  FILE* f;
  Crc32c outer, inner;
  bool ok = true;
  void put(const void* d, size_t n, bool in_filter) {
    if (ok && fwrite(d, 1, n, f) != n) ok = false;
    outer.update(d, n);
    if (in_filter) inner.update(d, n);
  }
  template <class T> void put_v(T v, bool in_filter) { put(&v, sizeof v, in_filter); }
};

struct Reader {
  FILE* f;
  Crc32c outer, inner;
  int err = 0;   // 0 ok, 6 truncated, 8 io
  bool get(void* d, size_t n, bool in_filter) {
    if (err) return false;
    size_t got = fread(d, 1, n, f);
    if (got != n) {
      err = ferror(f) ? LSHBLOOM_EIO : LSHBLOOM_ETRUNC;
      return false;
    }
    outer.update(d, n);
    if (in_filter) inner.update(d, n);
    return true;
  }
  template <class T> bool get_v(T& v, bool in_filter) { return get(&v, sizeof v, in_filter); }
};

constexpr size_t kIoChunk = 64ull << 20;

}  // namespace

extern "C" {

int lshbloom_save(lshbloom* h, const char* path) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!path) return fail(h, LSHBLOOM_EUSAGE, "NULL path");
  if (h->cfg.world != 1) return fail(h, LSHBLOOM_EUSAGE, "save needs an unsharded handle (world = 1)");
  if (h->cfg.index_kind != LSHBLOOM_INDEX_BLOOM) return fail(h, LSHBLOOM_EUSAGE, "save: SPEC's LBF1 format holds standard Bloom filters only");
  if (h->cfg.shingle_n != 5) return fail(h, LSHBLOOM_EUSAGE, "the LSHB format carries no shingle width; save needs n = 5");
  DeviceGuard g(h->device);
  if ((rc = drain(h))) return rc;
  LB_CUDA(h, cudaDeviceSynchronize());
  FILE* f = fopen(path, "wb");
  if (!f) return fail(h, LSHBLOOM_EIO, std::string("cannot open ") + path + " for writing");
  Writer w{f};
  const lshbloom_config& c = h->cfg;
  // the threshold the (b, r) were chosen for; unknown: the S-curve's approximate (1/b)^(1/r)
  const double threshold = c.lsh_threshold > 0.0 ? c.lsh_threshold : pow(1.0 / c.b, 1.0 / c.r);
  const double p_eff = -expm1((double)c.b * log1p(-c.fp_rate));
  w.put("LSHB", 4, false);
  w.put_v<uint32_t>(1, false);
  w.put_v<double>(threshold, false);
  w.put_v<uint32_t>(c.num_perm, false);
  w.put_v<uint32_t>(c.b, false);
  w.put_v<uint32_t>(c.r, false);
  w.put_v<uint64_t>(c.seed, false);
  w.put_v<uint64_t>(c.seed, false);
  w.put_v<uint64_t>(c.n_expected, false);
  w.put_v<double>(p_eff, false);
  w.put_v<uint64_t>(h->doc_count, false);
  const uint64_t payload = (h->m + 7) / 8;
  std::vector<uint8_t> buf(std::min<uint64_t>(payload, kIoChunk));
  for (uint32_t j = 0; j < c.b; j++) {
    w.inner = Crc32c();
    w.put("LBF1", 4, true);
    w.put_v<uint32_t>(1, true);
    w.put_v<uint64_t>(R(c.seed, 3, j), true);
    w.put_v<uint64_t>(c.n_expected, true);
    w.put_v<double>(c.fp_rate, true);
    w.put_v<uint64_t>(h->m, true);
    w.put_v<uint32_t>(h->k, true);
    w.put_v<uint64_t>(h->doc_count, true);
    const uint8_t* src = (const uint8_t*)(h->d_F + (uint64_t)j * h->W);
    for (uint64_t off = 0; off < payload; off += buf.size()) {
      const size_t n = (size_t)std::min<uint64_t>(buf.size(), payload - off);
      cudaError_t e = cudaMemcpy(buf.data(), src + off, n, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        fclose(f);
        return fail_cuda(h, e, "cudaMemcpy(filter -> host)");
      }
      w.put(buf.data(), n, true);
    }
    w.put_v<uint32_t>(w.inner.value(), false);
  }
  const uint32_t crc = w.outer.value();
  w.put_v<uint32_t>(crc, false);
  const bool ok = w.ok && fclose(f) == 0;
  if (!ok) return fail(h, LSHBLOOM_EIO, std::string("write failed: ") + path);
  return LSHBLOOM_OK;
}

int lshbloom_load(const char* path, int32_t device, lshbloom** out) {
  if (!out || !path) return fail(nullptr, LSHBLOOM_EUSAGE, "NULL path / out");
  *out = nullptr;
  FILE* f = fopen(path, "rb");
  if (!f) return fail(nullptr, LSHBLOOM_EIO, std::string("cannot open ") + path);
  Reader r{f};
  auto bail = [&](int code, const std::string& msg, lshbloom* h) {
    fclose(f);
    if (h) lshbloom_destroy(h);
    return fail(nullptr, code, msg);
  };
  char magic[4];
  uint32_t version, num_perm, b, rr;
  double threshold, p_eff;
  uint64_t sseed, bseed, n_docs, doc_count;
  r.get(magic, 4, false);
  r.get_v(version, false);
  r.get_v(threshold, false);
  r.get_v(num_perm, false);
  r.get_v(b, false);
  r.get_v(rr, false);
  r.get_v(sseed, false);
  r.get_v(bseed, false);
  r.get_v(n_docs, false);
  r.get_v(p_eff, false);
  r.get_v(doc_count, false);
  if (r.err) return bail(r.err, "truncated LSHB header", nullptr);
  if (memcmp(magic, "LSHB", 4) != 0) return bail(LSHBLOOM_EFORMAT, "bad magic (not an LSHB file)", nullptr);
  if (version != 1) return bail(LSHBLOOM_EFORMAT, "unsupported LSHB version " + std::to_string(version), nullptr);
  if (sseed != bseed) return bail(LSHBLOOM_EFORMAT, "signature and band-hash seeds differ (unsupported)", nullptr);
  lshbloom* h = nullptr;
  bool created = false;
  for (uint32_t j = 0; j < b; j++) {
    r.inner = Crc32c();
    char fm[4];
    uint32_t fv, k;
    uint64_t fseed, cap, m, inserted;
    double tp;
    r.get(fm, 4, true);
    r.get_v(fv, true);
    r.get_v(fseed, true);
    r.get_v(cap, true);
    r.get_v(tp, true);
    r.get_v(m, true);
    r.get_v(k, true);
    r.get_v(inserted, true);
    if (r.err) return bail(r.err, "truncated LBF1 header of band " + std::to_string(j), h);
    if (memcmp(fm, "LBF1", 4) != 0 || fv != 1) return bail(LSHBLOOM_EFORMAT, "bad LBF1 record for band " + std::to_string(j), h);
    if (!created) {
      lshbloom_config c;
      memset(&c, 0, sizeof c);
      c.num_perm = num_perm;
      c.b = b;
      c.r = rr;
      c.shingle_n = 5;
      c.n_expected = cap;
      c.fp_rate = tp;
      c.seed = sseed;
      c.device = device;
      c.world = 1;
      c.lsh_threshold = threshold > 0.0 && threshold <= 1.0 ? threshold : 0.0;
      int rc = lshbloom_create_ex(&c, &h);
      if (rc) return bail(rc == LSHBLOOM_EUSAGE ? LSHBLOOM_EFORMAT : rc, "header parameters rejected: " + g_create_error, nullptr);
      created = true;
      if (n_docs != cap) return bail(LSHBLOOM_EFORMAT, "n_docs != capacity_n", h);
    }
    if (m != h->m || k != h->k || cap != h->cfg.n_expected || tp != h->cfg.fp_rate || fseed != R(sseed, 3, j))
      return bail(LSHBLOOM_EFORMAT, "LBF1 geometry of band " + std::to_string(j) + " disagrees with its parameters", h);
    const uint64_t payload = (m + 7) / 8;
    std::vector<uint8_t> buf(std::min<uint64_t>(payload, kIoChunk));
    uint8_t* dst = (uint8_t*)(h->d_F + (uint64_t)j * h->W);
    for (uint64_t off = 0; off < payload; off += buf.size()) {
      const size_t n = (size_t)std::min<uint64_t>(buf.size(), payload - off);
      if (!r.get(buf.data(), n, true)) return bail(r.err, "truncated payload of band " + std::to_string(j), h);
      cudaError_t e = cudaMemcpy(dst + off, buf.data(), n, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return bail(LSHBLOOM_ERUNTIME, std::string("cudaMemcpy: ") + cudaGetErrorString(e), h);
    }
    const uint32_t want = r.inner.value();
    uint32_t stored;
    if (!r.get_v(stored, false)) return bail(r.err, "truncated LBF1 checksum", h);
    if (stored != want) return bail(LSHBLOOM_ECHECKSUM, "LBF1 checksum mismatch in band " + std::to_string(j), h);
    h->doc_count = inserted;
  }
  if (!created) return bail(LSHBLOOM_EFORMAT, "LSHB file with b = 0", nullptr);
  const uint32_t want = r.outer.value();
  uint32_t stored;
  if (!r.get_v(stored, false)) return bail(r.err, "truncated LSHB checksum", h);
  if (stored != want) return bail(LSHBLOOM_ECHECKSUM, "LSHB checksum mismatch", h);
  h->doc_count = doc_count;
  fclose(f);
  *out = h;
  return LSHBLOOM_OK;
}

}  // extern "C"
