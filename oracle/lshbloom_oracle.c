/*
 * lshbloom_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * LSHBloom hot path (arXiv 2411.04257).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this file.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2411_04257_b200/csrc/ (which re-implements every step independently).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 * Conventions that the paper leaves open are fixed in DESIGN.md §3 ("readings")
 * and are written out here literally, in the paper's order:
 *
 *   shingles        word n-grams of the uint32 id sequence;
 *                                      a document shorter than n is one shingle
 *   fingerprint (DESIGN R1)      h = mix64(0x6C7368626C6F6F6D + t);
 *                                      for w in shingle: h = mix64(h ^ w)
 *   MinHash   sig[i] = min_x ((a_i*x + b_i) mod P) mod 2^32,
 *                                      x = fingerprint mod P, P = 2^61-1,
 *                                      exact 128-bit products
 *   band hash   BH_j = (sum_{u<r} ((c_u*sig[j*r+u] + d_u) mod P)) mod P
 *   Bloom   m = ceil(-n ln p / (ln 2)^2), k = max(1, round((m/n) ln 2))
 *                                      (P:224-225); probes g_t = (h1 + t*h2) mod m
 *                                      with h1 = mix64(BH^s1_j), h2 = mix64(BH^s2_j)|1
 *   LSHBloom   one filter per band; a document is a duplicate
 *                                      iff some band's k bits were all set before it
 *                                      (query), then all b band hashes are inserted
 *                                      (insert is unconditional), in stream order.
 *
 * Parity pins (tests/test_oracle_*.py): sizing against S:275-276 and the
 * paper's Tables 1-2 and P:229; mix64 against the published
 * SplitMix64 output sequence; MinHash against the singleton closed form
 * (S:139), x in {0, 1, P-1} closed forms, brute-force set minima and the
 * Jaccard estimator bound; band hash against r=1 and
 * all-equal-row closed forms; probes against the non-incremental closed form;
 * the streaming verdict against a brute-force set formulation and the classic
 * exact-band-equality index; Bloom FP / fill against their
 * analytic values.
 *
 * Conventions the paper leaves open (orc_fingerprint, DESIGN R1; orc_family,
 * R5; orc_probes_blocked's in-block offsets) are pinned
 * element by element against an independent pure-Python big-integer
 * re-implementation written from DESIGN.md's prose (tests/support/
 * micro_oracle.py, tests/test_oracle_micro.py) and by known-answer vectors
 * (tests/golden/conventions_kat.json).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define ORC_P ((uint64_t)0x1FFFFFFFFFFFFFFFull) /* 2^61 - 1 */

/* SplitMix64 finaliser (DESIGN R5). All arithmetic wraps mod 2^64. */
uint64_t orc_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

/* Counter-mode expansion R(seed, dom, i) ("specified counter-mode"; DESIGN R5). */
uint64_t orc_R(uint64_t seed, uint64_t dom, uint64_t i) {
    return orc_mix64(seed + 0x9E3779B97F4A7C15ull * ((dom << 32) + i + 1));
}

/* Bloom sizing, "m = -n * log(p)/(log(2))^2" (natural log),
 * k = max(1, round((m/n) ln 2)).  Returns 1 on usage error. */
int orc_bloom_size(uint64_t n, double p, uint64_t *m_out, uint32_t *k_out) {
    if (n == 0 || !(p > 0.0 && p < 1.0)) return 1;
    double m = ceil(-(double)n * log(p) / (log(2.0) * log(2.0)));
    long long k = llround((m / (double)n) * log(2.0));
    if (k < 1) k = 1;
    *m_out = (uint64_t)m;
    *k_out = (uint32_t)k;
    return 0;
}

/* Universal hash family and the per-band filter seeds.
 * Any output pointer may be NULL. */
void orc_family(uint64_t seed, uint32_t num_perm, uint32_t r, uint32_t b,
                uint64_t *a, uint64_t *bb, uint64_t *c, uint64_t *d,
                uint64_t *s1, uint64_t *s2) {
    for (uint32_t i = 0; i < num_perm; i++) {
        if (a) a[i] = 1 + orc_R(seed, 1, 2ull * i) % (ORC_P - 1);
        if (bb) bb[i] = orc_R(seed, 1, 2ull * i + 1) % ORC_P;
    }
    for (uint32_t u = 0; u < r; u++) {
        if (c) c[u] = 1 + orc_R(seed, 2, 2ull * u) % (ORC_P - 1);
        if (d) d[u] = orc_R(seed, 2, 2ull * u + 1) % ORC_P;
    }
    for (uint32_t j = 0; j < b; j++) {
        if (s1) s1[j] = orc_R(seed, 3, j);
        if (s2) s2[j] = orc_R(seed, 4, j);
    }
}

/* Shingle fingerprint of the id sequence w[0..t) ("documented 64-bit hash
 * with token boundaries encoded"; DESIGN R1: fixed-width ids, length salt). */
uint64_t orc_fingerprint(const uint32_t *w, uint32_t t) {
    uint64_t h = orc_mix64(0x6C7368626C6F6F6Dull + t);
    for (uint32_t q = 0; q < t; q++) h = orc_mix64(h ^ (uint64_t)w[q]);
    return h;
}

/* (a*x + b) mod P with an exact 128-bit intermediate. */
static uint64_t orc_affine_mod_p(uint64_t a, uint64_t x, uint64_t b) {
    return (uint64_t)(((u128)a * (u128)x + (u128)b) % (u128)ORC_P);
}

/* MinHash signature of one document ("repeatedly apply random
 * permutations ... MinHash signatures").  ids[0..L), L >= 1. */
void orc_signature_doc(const uint32_t *ids, uint64_t L, uint32_t n,
                       const uint64_t *a, const uint64_t *bb, uint32_t num_perm,
                       uint32_t *sig) {
    /* the bag of n-grams: every contiguous n-gram, or the whole doc if L < n */
    uint64_t S = (L >= n) ? (L - n + 1) : 1;
    uint32_t t = (L >= n) ? n : (uint32_t)L;
    uint64_t *X = (uint64_t *)malloc(sizeof(uint64_t) * S);
    for (uint64_t q = 0; q < S; q++) X[q] = orc_fingerprint(ids + q, t) % ORC_P;
    /* sig[i] = min over the set of ((a_i x + b_i) mod P) truncated to 32 bits (DESIGN R3) */
    for (uint32_t i = 0; i < num_perm; i++) {
        uint32_t best = 0xFFFFFFFFu;
        for (uint64_t q = 0; q < S; q++) {
            uint32_t v = (uint32_t)(orc_affine_mod_p(a[i], X[q], bb[i]) & 0xFFFFFFFFull);
            if (v < best) best = v;
        }
        sig[i] = best;
    }
    free(X);
}

/* Band hash: h(x) = (sum_{i=1..r} h_i(x_i)) mod N, N = P, h_u(x) = (c_u x + d_u) mod P,
 * band j = rows [j r, j r + r). */
uint64_t orc_band_hash(const uint32_t *sig, uint32_t j, uint32_t r,
                       const uint64_t *c, const uint64_t *d) {
    uint64_t acc = 0;
    for (uint32_t u = 0; u < r; u++) {
        uint64_t hu = orc_affine_mod_p(c[u], (uint64_t)sig[(uint64_t)j * r + u], d[u]);
        acc = (uint64_t)(((u128)acc + hu) % ORC_P);
    }
    return acc;
}

/* k probe positions of one band hash in a filter of m bits:
 * g_t = (h1 + t*h2) mod m over the integers. */
void orc_probes(uint64_t bh, uint64_t s1, uint64_t s2, uint64_t m, uint32_t k, uint64_t *g) {
    uint64_t h1 = orc_mix64(bh ^ s1);
    uint64_t h2 = orc_mix64(bh ^ s2) | 1ull;
    for (uint32_t t = 0; t < k; t++) g[t] = (uint64_t)(((u128)h1 + (u128)t * (u128)h2) % (u128)m);
}

/* Blocked variant (SPEC S:328 leaves the filter layout open): the
 * filter is nb blocks of 1024 bits (one 128-byte line) and all k probes of a band hash fall
 * in one block:  block = h1 mod nb;  offsets are the 10-bit fields of w_j = mix64(h2 + j):
 * o_t = (w_{t / 6} >> (10 (t mod 6))) & 1023;  g_t = 1024 * block + o_t,  t < k.
 * h1, h2 as for the standard filter.  Offsets are independent and uniform (they may repeat,
 * as positions of the standard filter may). */
#define ORC_BLOCK_BITS 1024u
void orc_probes_blocked(uint64_t bh, uint64_t s1, uint64_t s2, uint64_t nb, uint32_t k, uint64_t *g) {
    uint64_t h1 = orc_mix64(bh ^ s1);
    uint64_t h2 = orc_mix64(bh ^ s2) | 1ull;
    uint64_t block = h1 % nb;
    for (uint32_t t = 0; t < k; t++) {
        uint64_t w = orc_mix64(h2 + t / 6);
        g[t] = block * ORC_BLOCK_BITS + ((w >> (10 * (t % 6))) & (ORC_BLOCK_BITS - 1));
    }
}

/* ------------------------------------------------------------------------ */
/* Signatures + band hashes over a CSR batch, threads over documents.        */

typedef struct {
    uint64_t lo, hi;
    const uint64_t *offsets;
    const uint32_t *tokens;
    uint32_t num_perm, n, b, r;
    const uint64_t *a, *bb, *c, *d;
    uint32_t *sig_out;   /* [n_docs][num_perm] or NULL */
    uint64_t *bh_out;    /* [n_docs][b] or NULL */
} orc_sig_job;

static void *orc_sig_worker(void *arg) {
    orc_sig_job *J = (orc_sig_job *)arg;
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * J->num_perm);
    for (uint64_t i = J->lo; i < J->hi; i++) {
        uint64_t L = J->offsets[i + 1] - J->offsets[i];
        uint32_t *sig = J->sig_out ? J->sig_out + i * J->num_perm : tmp;
        orc_signature_doc(J->tokens + J->offsets[i], L, J->n, J->a, J->bb, J->num_perm, sig);
        if (J->bh_out)
            for (uint32_t j = 0; j < J->b; j++)
                J->bh_out[i * J->b + j] = orc_band_hash(sig, j, J->r, J->c, J->d);
    }
    free(tmp);
    return NULL;
}

/* Returns 0 ok, 1 usage, 2 "empty document" -- *bad_doc = first empty doc. */
int orc_signatures(uint64_t n_docs, const uint64_t *offsets, const uint32_t *tokens,
                   uint32_t num_perm, uint32_t shingle_n, uint32_t b, uint32_t r,
                   uint64_t seed, int nthreads, uint32_t *sig_out, uint64_t *bh_out,
                   uint64_t *bad_doc) {
    if (num_perm == 0 || shingle_n == 0 || (bh_out && (b == 0 || r == 0 || (uint64_t)b * r > num_perm)))
        return 1;
    if (offsets[0] != 0) return 1;
    for (uint64_t i = 0; i < n_docs; i++) {
        if (offsets[i + 1] < offsets[i]) return 1;
        if (offsets[i + 1] == offsets[i]) { if (bad_doc) *bad_doc = i; return 2; }
    }
    uint64_t *a = malloc(8 * (size_t)num_perm), *bb = malloc(8 * (size_t)num_perm);
    uint64_t *c = malloc(8 * (size_t)(r ? r : 1)), *d = malloc(8 * (size_t)(r ? r : 1));
    orc_family(seed, num_perm, r, 0, a, bb, c, d, NULL, NULL);
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > n_docs) nthreads = n_docs ? (int)n_docs : 1;
    pthread_t *th = malloc(sizeof(pthread_t) * nthreads);
    orc_sig_job *jobs = malloc(sizeof(orc_sig_job) * nthreads);
    for (int t = 0; t < nthreads; t++) {
        orc_sig_job J = {n_docs * t / nthreads, n_docs * (t + 1) / nthreads, offsets, tokens,
                         num_perm, shingle_n, b, r, a, bb, c, d, sig_out, bh_out};
        jobs[t] = J;
        pthread_create(&th[t], NULL, orc_sig_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th); free(jobs); free(a); free(bb); free(c); free(d);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* The LSHBloom index: b Bloom filters of m bits.  Bit g of a    */
/* filter lives in byte g>>3 at mask 1<<(g&7) (S:322 payload layout).        */

typedef struct {
    uint32_t b, k;
    int blocked;           /* 0: standard filter; 1: blocked variant (orc_probes_blocked) */
    uint64_t nb;           /* blocked: number of 1024-bit blocks */
    uint64_t m, n_expected, doc_count;
    uint64_t seed;
    uint64_t *s1, *s2;
    uint8_t **bits; /* b arrays of ceil(m/8) bytes */
} orc_index;

/* blocked = 1: the standard m rounded up to whole 1024-bit blocks, same k. */
void *orc_index_new2(uint32_t b, uint64_t n_expected, double fp_rate, uint64_t seed, int blocked) {
    uint64_t m; uint32_t k;
    if (b == 0 || orc_bloom_size(n_expected, fp_rate, &m, &k)) return NULL;
    orc_index *X = calloc(1, sizeof(orc_index));
    if (blocked) {
        X->blocked = 1;
        X->nb = (m + ORC_BLOCK_BITS - 1) / ORC_BLOCK_BITS;
        m = X->nb * ORC_BLOCK_BITS;
    }
    X->b = b; X->k = k; X->m = m; X->n_expected = n_expected; X->seed = seed;
    X->s1 = malloc(8 * (size_t)b); X->s2 = malloc(8 * (size_t)b);
    orc_family(seed, 0, 0, b, NULL, NULL, NULL, NULL, X->s1, X->s2);
    X->bits = malloc(sizeof(uint8_t *) * b);
    for (uint32_t j = 0; j < b; j++) {
        X->bits[j] = calloc((size_t)((m + 7) / 8), 1);   /* "all bits initially set to 0" */
        if (!X->bits[j]) return NULL;
    }
    return X;
}

void *orc_index_new(uint32_t b, uint64_t n_expected, double fp_rate, uint64_t seed) {
    return orc_index_new2(b, n_expected, fp_rate, seed, 0);
}

void orc_index_free(void *p) {
    orc_index *X = (orc_index *)p;
    if (!X) return;
    for (uint32_t j = 0; j < X->b; j++) free(X->bits[j]);
    free(X->bits); free(X->s1); free(X->s2); free(X);
}

uint64_t orc_index_m(void *p) { return ((orc_index *)p)->m; }
uint32_t orc_index_k(void *p) { return ((orc_index *)p)->k; }
uint64_t orc_index_doc_count(void *p) { return ((orc_index *)p)->doc_count; }
const uint8_t *orc_index_bits(void *p, uint32_t j) { return ((orc_index *)p)->bits[j]; }

static int orc_get_bit(const uint8_t *F, uint64_t g) { return (F[g >> 3] >> (g & 7)) & 1; }
static void orc_set_bit(uint8_t *F, uint64_t g) { F[g >> 3] |= (uint8_t)(1u << (g & 7)); }

typedef struct {
    orc_index *X;
    uint32_t j;            /* global band index */
    uint32_t col, ncol;    /* column of band j in bh[n][ncol] */
    uint64_t n_docs;
    const uint64_t *bh;
    uint8_t *hit;          /* [n_docs] for this band */
} orc_band_job;

/* One band, stream order (S:390 query then insert; S:427 serialised). */
static void *orc_band_worker(void *arg) {
    orc_band_job *J = (orc_band_job *)arg;
    orc_index *X = J->X;
    uint8_t *F = X->bits[J->j];
    uint64_t *g = malloc(8 * (size_t)X->k);
    for (uint64_t i = 0; i < J->n_docs; i++) {
        if (X->blocked) orc_probes_blocked(J->bh[i * J->ncol + J->col], X->s1[J->j], X->s2[J->j], X->nb, X->k, g);
        else orc_probes(J->bh[i * J->ncol + J->col], X->s1[J->j], X->s2[J->j], X->m, X->k, g);
        int all = 1;                                          /* query: all k bits set */
        for (uint32_t t = 0; t < X->k; t++) all &= orc_get_bit(F, g[t]);
        for (uint32_t t = 0; t < X->k; t++) orc_set_bit(F, g[t]);   /* insert */
        J->hit[i] = (uint8_t)all;
    }
    free(g);
    return NULL;
}

/* Query-then-insert a batch of band hashes bh[n_docs][ncol] for bands
 * [band_lo, band_lo + ncol) in stream order.  dup_out[i] = OR over those bands
 * ("collision for any band ... mark that document as a duplicate").
 * hits_out (optional) = per-band verdicts [n_docs][ncol].  Bands are processed
 * on separate threads: each band's filter evolves independently because every
 * document inserts all its band hashes (DESIGN R12). */
int orc_index_query_insert(void *p, uint64_t n_docs, const uint64_t *bh, uint32_t band_lo,
                           uint32_t ncol, int nthreads, uint8_t *dup_out, uint8_t *hits_out) {
    orc_index *X = (orc_index *)p;
    if (!X || band_lo + ncol > X->b) return 1;
    uint8_t *hit = malloc((size_t)n_docs * ncol + 1);
    orc_band_job *jobs = malloc(sizeof(orc_band_job) * ncol);
    pthread_t *th = malloc(sizeof(pthread_t) * ncol);
    if (nthreads < 1) nthreads = 1;
    for (uint32_t c0 = 0; c0 < ncol; c0 += (uint32_t)nthreads) {
        uint32_t c1 = c0 + (uint32_t)nthreads < ncol ? c0 + (uint32_t)nthreads : ncol;
        for (uint32_t c = c0; c < c1; c++) {
            orc_band_job J = {X, band_lo + c, c, ncol, n_docs, bh, hit + (size_t)c * n_docs};
            jobs[c] = J;
            pthread_create(&th[c], NULL, orc_band_worker, &jobs[c]);
        }
        for (uint32_t c = c0; c < c1; c++) pthread_join(th[c], NULL);
    }
    for (uint64_t i = 0; i < n_docs; i++) {
        uint8_t any = 0;
        for (uint32_t c = 0; c < ncol; c++) {
            uint8_t h = hit[(size_t)c * n_docs + i];
            any |= h;
            if (hits_out) hits_out[i * ncol + c] = h;
        }
        if (dup_out) dup_out[i] = any;
    }
    X->doc_count += n_docs;
    free(hit); free(jobs); free(th);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* The classic MinHashLSH index ("if two bands ... are exactly      */
/* identical ... candidate pairs"; S:186-189 ClassicLshIndex      */
/* classic_insert / classic_query): b maps from band hash to the documents    */
/* holding it.  A document is a classic duplicate iff some band hash of it    */
/* was already inserted by an earlier document of the stream; then all its   */
/* band hashes are inserted.  Only membership matters for that verdict, so    */
/* each band keeps the set of band-hash values seen (a plain linear-probing   */
/* hash set; band hashes are < P = 2^61 - 1, so UINT64_MAX marks empty).      */

typedef struct {
    uint64_t cap, used;
    uint64_t *keys;
} orc_set;

static int orc_set_contains(const orc_set *S, uint64_t v) {
    if (!S->cap) return 0;
    uint64_t s = orc_mix64(v) & (S->cap - 1);
    while (S->keys[s] != UINT64_MAX) {
        if (S->keys[s] == v) return 1;
        s = (s + 1) & (S->cap - 1);
    }
    return 0;
}

static void orc_set_add(orc_set *S, uint64_t v);

static void orc_set_grow(orc_set *S) {
    orc_set T = {S->cap ? 2 * S->cap : 1024, 0, NULL};
    T.keys = malloc(8 * (size_t)T.cap);
    memset(T.keys, 0xFF, 8 * (size_t)T.cap);
    for (uint64_t i = 0; i < S->cap; i++)
        if (S->keys[i] != UINT64_MAX) orc_set_add(&T, S->keys[i]);
    free(S->keys);
    *S = T;
}

static void orc_set_add(orc_set *S, uint64_t v) {
    if (2 * (S->used + 1) > S->cap) orc_set_grow(S);
    uint64_t s = orc_mix64(v) & (S->cap - 1);
    while (S->keys[s] != UINT64_MAX) {
        if (S->keys[s] == v) return;
        s = (s + 1) & (S->cap - 1);
    }
    S->keys[s] = v;
    S->used++;
}

typedef struct {
    uint32_t b;
    uint64_t doc_count;
    orc_set *sets;
} orc_classic;

void *orc_classic_new(uint32_t b) {
    if (b == 0) return NULL;
    orc_classic *X = calloc(1, sizeof(orc_classic));
    X->b = b;
    X->sets = calloc(b, sizeof(orc_set));
    return X;
}

void orc_classic_free(void *p) {
    orc_classic *X = (orc_classic *)p;
    if (!X) return;
    for (uint32_t j = 0; j < X->b; j++) free(X->sets[j].keys);
    free(X->sets); free(X);
}

uint64_t orc_classic_keys(void *p, uint32_t j) { return ((orc_classic *)p)->sets[j].used; }

/* Stream order, one document at a time: query every band ("union over bands of ids in
 * the bucket matching that band's hash"; non-empty = duplicate), then insert. */
int orc_classic_query_insert(void *p, uint64_t n_docs, const uint64_t *bh, uint32_t band_lo,
                             uint32_t ncol, uint8_t *dup_out, uint8_t *hits_out) {
    orc_classic *X = (orc_classic *)p;
    if (!X || band_lo + ncol > X->b) return 1;
    for (uint64_t i = 0; i < n_docs; i++) {
        uint8_t any = 0;
        for (uint32_t c = 0; c < ncol; c++) {
            uint8_t h = (uint8_t)orc_set_contains(&X->sets[band_lo + c], bh[i * ncol + c]);
            any |= h;
            if (hits_out) hits_out[i * ncol + c] = h;
        }
        for (uint32_t c = 0; c < ncol; c++) orc_set_add(&X->sets[band_lo + c], bh[i * ncol + c]);
        if (dup_out) dup_out[i] = any;
    }
    X->doc_count += n_docs;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Band selection ("determine an optimal band size b", S:193-199   */
/* optimal_params): over all b*r <= num_perm minimise                         */
/*   fp_w * int_0^T (1-(1-s^r)^b) ds + fn_w * int_T^1 (1-s^r)^b ds           */
/* with composite Simpson's rule, 1000 subintervals per integral;     */
/* ties toward smaller b, then smaller r.                                     */

static double orc_fp_integrand(double s, uint32_t b, uint32_t r) { return 1.0 - pow(1.0 - pow(s, r), b); }
static double orc_fn_integrand(double s, uint32_t b, uint32_t r) { return pow(1.0 - pow(s, r), b); }

static double orc_simpson(double (*f)(double, uint32_t, uint32_t), double lo, double hi, uint32_t b, uint32_t r) {
    const int N = 1000;
    double h = (hi - lo) / N, acc = f(lo, b, r) + f(hi, b, r);
    for (int i = 1; i < N; i++) acc += f(lo + i * h, b, r) * ((i & 1) ? 4.0 : 2.0);
    return acc * h / 3.0;
}

int orc_optimal_params(double T, uint32_t num_perm, double fp_w, double fn_w, uint32_t *b_out, uint32_t *r_out) {
    if (!(T > 0.0 && T <= 1.0) || num_perm < 2) return 1;
    double best = INFINITY;
    uint32_t bb = 0, br = 0;
    for (uint32_t b = 1; b <= num_perm; b++) {
        for (uint32_t r = 1; b * r <= num_perm; r++) {
            double e = fp_w * orc_simpson(orc_fp_integrand, 0.0, T, b, r) +
                       fn_w * orc_simpson(orc_fn_integrand, T, 1.0, b, r);
            if (e < best) { best = e; bb = b; br = r; }
        }
    }
    *b_out = bb; *r_out = br;
    return 0;
}
