"""Pins for the CPU oracle: each oracle function is checked against something
other than itself -- values printed by the paper / SPEC, published reference
outputs, closed forms, brute force on tiny inputs, invariants and statistical
fixed points (SPEC "[PAPER]" / "[DERIVED]" examples).  No GPU needed."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import P61

MASK32 = 0xFFFFFFFF


# --------------------------------------------------------------------------- sizing

def _sizing():
    here = os.path.join(os.path.dirname(__file__), "golden", "sizing.json")
    with open(here) as f:
        return json.load(f)


@pytest.mark.parametrize("row", _sizing()["bloom_size"], ids=lambda r: r["src"])
def test_bloom_size_spec_examples(row):
    assert oracle.bloom_size(row["n"], row["p"]) == (row["m"], row["k"])


def _index_size(n, p_eff, b):
    # per-filter p from p_effective = 1-(1-p)^b, inverted stably
    p = -math.expm1(math.log1p(-p_eff) / b)
    m, _ = oracle.bloom_size(int(n), p)
    return b * ((m + 7) // 8)          # S:398 total_bytes = b * ceil(bits/8)


@pytest.mark.parametrize("row", _sizing()["index_size"], ids=lambda r: r["src"])
def test_index_size_paper_tables(row):
    got = _index_size(row["n"], row["p_eff"], row["b"]) / row["unit_bytes"]
    if row["exact"]:
        assert round(got, row["digits"]) == pytest.approx(row["size"], abs=1e-9)
    else:
        assert got == pytest.approx(row["size"], rel=row["rel_tol"])


def test_index_size_pes2o_per_filter_p():
    row = _sizing()["per_filter_p"][0]
    m, _ = oracle.bloom_size(row["n"], row["p"])
    assert round(row["b"] * ((m + 7) // 8) / 1e9, row["digits"]) == row["size_gb"]


def test_bloom_size_rejects_bad_p():
    for p in (0.0, 1.0, -0.1, 1.5, float("nan")):
        with pytest.raises(ValueError):
            oracle.bloom_size(10, p)
    with pytest.raises(ValueError):
        oracle.bloom_size(0, 0.1)


def test_bloom_size_k_is_rounded_ln2_ratio():
    # k = round((m/n) ln 2); for p = 2^-j the optimum k is j (ln p = -j ln 2)
    for j in range(1, 20):
        m, k = oracle.bloom_size(1000, 2.0 ** -j)
        assert k == j


# --------------------------------------------------------------------------- mix64 / counter

def _splitmix_vectors():
    path = os.path.join(os.path.dirname(__file__), "golden", "splitmix64_seed0.txt")
    return [int(l, 16) for l in open(path) if l.strip() and not l.startswith("#")]


def test_mix64_matches_published_splitmix64():
    gamma = 0x9E3779B97F4A7C15
    for i, want in enumerate(_splitmix_vectors()):
        assert oracle.mix64((gamma * (i + 1)) % 2**64) == want
        assert oracle.counter(0, 0, i) == want   # R(0, 0, i) is SplitMix64's i-th output


def test_mix64_is_a_bijection_sample():
    # inverse via the modular inverses of the two odd multipliers (independent of the forward code)
    inv1 = pow(0xBF58476D1CE4E5B9, -1, 2**64)
    inv2 = pow(0x94D049BB133111EB, -1, 2**64)

    def unxorshift(z, s):
        x = z
        for _ in range(64 // s + 1):
            x = z ^ (x >> s)
        return x

    rng = np.random.default_rng(5)
    for z in rng.integers(0, 2**63, 200, dtype=np.uint64).tolist() + [0, 2**64 - 1]:
        h = oracle.mix64(z)
        x = unxorshift(h, 31)
        x = (x * inv2) % 2**64
        x = unxorshift(x, 27)
        x = (x * inv1) % 2**64
        x = unxorshift(x, 30)
        assert x == z


# --------------------------------------------------------------------------- family

def test_family_ranges_prefix_and_determinism():
    a, b, c, d, s1, s2 = oracle.family(42, 256, 8, 32)
    assert (a >= 1).all() and (a < P61).all() and (b < P61).all()
    assert (c >= 1).all() and (c < P61).all() and (d < P61).all()
    a2, b2, *_ = oracle.family(42, 128, 8, 32)
    assert (a2 == a[:128]).all() and (b2 == b[:128]).all()               # prefix property
    a3, b3, *_ = oracle.family(42, 256, 8, 32)
    assert (a3 == a).all() and (b3 == b).all()                           # determinism
    a4, *_ = oracle.family(43, 256, 8, 32)
    assert (a4 != a).any()
    assert len(set(s1.tolist())) == 32 and len(set(s2.tolist()) | set(s1.tolist())) == 64


# --------------------------------------------------------------------------- fingerprint

def test_fingerprint_encodes_boundaries_and_length():
    assert oracle.fingerprint([0]) != oracle.fingerprint([0, 0])          # length salt (DESIGN R1)
    assert oracle.fingerprint([1, 2]) != oracle.fingerprint([2, 1])
    assert oracle.fingerprint([7, 8, 9]) == oracle.fingerprint(np.array([7, 8, 9], np.uint32))
    fps = {oracle.fingerprint(list(w)) for w in itertools.product(range(4), repeat=5)}
    assert len(fps) == 4 ** 5                                            # no collisions on 1024 5-grams


# --------------------------------------------------------------------------- MinHash

def _affine_low32(a, x, b):
    return ((a * x + b) % P61) & MASK32


def test_singleton_signature_closed_form():
    # singleton set {x} -> values[i] = (a_i x + b_i) mod P (then truncated, DESIGN R3)
    a, b, *_ = oracle.family(7, 128, 0, 0)
    for ids in ([5], [1, 2, 3], [9, 9, 9, 9], [0, 1, 2, 3, 4], [2**32 - 1] * 5):
        x = oracle.fingerprint(ids) % P61
        want = np.array([_affine_low32(int(a[i]), x, int(b[i])) for i in range(128)], np.uint32)
        assert (oracle.signature_doc(ids, 128, 7) == want).all()


def test_signature_is_min_over_the_shingle_set():
    # brute force: sig(doc) = elementwise min over its 5-gram shingles, each a 5-token doc
    rng = np.random.default_rng(1)
    for L in (5, 6, 13, 40):
        ids = rng.integers(0, 50, L).astype(np.uint32)
        parts = np.stack([oracle.signature_doc(ids[q:q + 5], 64, 3) for q in range(L - 4)])
        assert (oracle.signature_doc(ids, 64, 3) == parts.min(axis=0)).all()


def test_signature_set_semantics_and_identity():
    ids = np.array([1, 2, 3, 4, 5, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5], np.uint32)
    once = np.array([1, 2, 3, 4, 5, 1, 2, 3, 4, 5], np.uint32)   # same shingle set
    assert (oracle.signature_doc(ids, 128, 0) == oracle.signature_doc(once, 128, 0)).all()
    with pytest.raises(ValueError):
        oracle.signature_doc([], 128, 0)


def _shingle_set(ids, n=5):
    ids = list(ids)
    if len(ids) < n:
        return {tuple(ids)}
    return {tuple(ids[q:q + n]) for q in range(len(ids) - n + 1)}


@pytest.mark.parametrize("target", [0.3, 0.5, 0.9])
def test_minhash_estimator_within_3sigma(target):
    # S:140 / S:595: estimate within J +- 3 sqrt(J(1-J)/256) for >= 99% of 200 seeds
    rng = np.random.default_rng(int(target * 100))
    n_sh = 200
    common = int(round(2 * target * n_sh / (1 + target)))
    base = rng.permutation(10**6)[: 2 * n_sh + 10].astype(np.uint32)
    A = np.concatenate([base[:common + 4], base[common + 4: n_sh + 4 + 0]])
    B = np.concatenate([base[:common + 4], base[n_sh + 4: 2 * n_sh + 4 - common + 0]])
    sa, sb = _shingle_set(A), _shingle_set(B)
    J = len(sa & sb) / len(sa | sb)                                      # exact Jaccard (brute force)
    sd = math.sqrt(J * (1 - J) / 256)
    ok = 0
    for seed in range(200):
        est = (oracle.signature_doc(A, 256, seed) == oracle.signature_doc(B, 256, seed)).mean()
        ok += abs(est - J) <= 3 * sd + 1e-12
    assert ok >= 198, (J, ok)


def test_identical_documents_identical_signatures():
    ids = np.arange(100, 400, dtype=np.uint32)
    assert (oracle.signature_doc(ids, 128, 0) == oracle.signature_doc(ids.copy(), 128, 0)).all()


# --------------------------------------------------------------------------- band hash

def test_band_hash_closed_forms():
    seed = 11
    _, _, c, d, _, _ = oracle.family(seed, 0, 8, 0)
    c = [int(v) for v in c]
    d = [int(v) for v in d]
    # r = 1: h = h_1(x_1) mod P
    for x in (0, 1, 12345, MASK32):
        assert oracle.band_hash(np.array([x], np.uint32), 0, 1, seed) == (c[0] * x + d[0]) % P61
    # all rows 0: sum d_u mod P; all rows 1: sum (c_u + d_u) mod P
    assert oracle.band_hash(np.zeros(8, np.uint32), 0, 8, seed) == sum(d) % P61
    assert oracle.band_hash(np.ones(8, np.uint32), 0, 8, seed) == sum(ci + di for ci, di in zip(c, d)) % P61
    # band j reads rows [j r, j r + r): band 2 of a signature = band 0 of its shifted copy
    sig = np.arange(1, 33, dtype=np.uint32) * 1000003
    assert oracle.band_hash(sig, 2, 8, seed) == oracle.band_hash(sig[16:], 0, 8, seed)


def test_band_hash_distinct_on_single_row_change():
    rng = np.random.default_rng(2)
    for _ in range(2000):
        s = rng.integers(0, 2**32, 8, dtype=np.uint64).astype(np.uint32)
        t = s.copy()
        t[rng.integers(0, 8)] ^= np.uint32(1 + rng.integers(0, 2**31))
        assert oracle.band_hash(s, 0, 8, 3) != oracle.band_hash(t, 0, 8, 3)


# --------------------------------------------------------------------------- probes

def test_probes_are_arithmetic_progression_mod_m():
    rng = np.random.default_rng(3)
    for m in (1, 2, 97, 23962646, 23962645944, 2**40 + 7):
        bh = int(rng.integers(0, P61))
        s1, s2 = 0x1234, 0x5678
        g = [int(v) for v in oracle.probes(bh, s1, s2, m, 17)]
        h1 = oracle.mix64(bh ^ s1)
        h2 = oracle.mix64(bh ^ s2) | 1
        assert all(0 <= v < m for v in g)
        assert g[0] == h1 % m
        assert all((g[t + 1] - g[t]) % m == h2 % m for t in range(16))


# --------------------------------------------------------------------------- stream semantics

def _positions(bh, j, s1, s2, m, k):
    return {int(v) for v in oracle.probes(int(bh), int(s1[j]), int(s2[j]), m, k)}


def _brute_force_flags(bh, s1, s2, m, k):
    """dup_i <=> exists band j: Pos_j(i) subset of union_{i'<i} Pos_j(i') (set form, no bit array)."""
    n, b = bh.shape
    seen = [set() for _ in range(b)]
    out = np.zeros(n, np.uint8)
    hits = np.zeros((n, b), np.uint8)
    for i in range(n):
        for j in range(b):
            pos = _positions(bh[i, j], j, s1, s2, m, k)
            hits[i, j] = pos <= seen[j]
            seen[j] |= pos
        out[i] = hits[i].any()
    return out, hits


@pytest.mark.parametrize("n_expected,fp", [(8, 0.3), (40, 0.05), (200, 0.01)])
def test_stream_flags_match_brute_force_sets(n_expected, fp):
    rng = np.random.default_rng(n_expected)
    b = 4
    n = 3 * n_expected
    bh = rng.integers(0, 64, (n, b), dtype=np.uint64)       # tiny range -> many repeats
    bh[5] = bh[2]                                             # planted exact repeat
    idx = oracle.Index(b, n_expected, fp, seed=9)
    _, _, _, _, s1, s2 = oracle.family(9, 0, 0, b)
    dup, hits = idx.query_insert(bh, want_hits=True, nthreads=2)
    want, want_hits = _brute_force_flags(bh, s1, s2, idx.m, idx.k)
    assert (dup == want).all() and (hits == want_hits).all()
    assert dup[5] == 1 and hits[5].all()


def test_stream_in_two_calls_equals_one_call():
    rng = np.random.default_rng(4)
    bh = rng.integers(0, 1000, (300, 3), dtype=np.uint64)
    one = oracle.Index(3, 100, 0.05, 1).query_insert(bh)
    ix = oracle.Index(3, 100, 0.05, 1)
    two = np.concatenate([ix.query_insert(bh[:137]), ix.query_insert(bh[137:])])
    assert (one == two).all() and ix.doc_count == 300


def _csr(docs):
    off = np.zeros(len(docs) + 1, np.uint64)
    off[1:] = np.cumsum([len(d) for d in docs])
    return off, np.concatenate([np.asarray(d, np.uint32) for d in docs])


def test_same_document_twice_is_unique_then_duplicate():
    # same document streamed twice -> [unique, duplicate]; all b bands collide
    d = np.arange(1000, 1200, dtype=np.uint32)
    off, tok = _csr([d, np.arange(5000, 5300, dtype=np.uint32), d])
    sig, bh, dup, idx = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=1000,
                                   fp_rate=1e-5, seed=0)
    assert dup.tolist() == [0, 0, 1]
    assert (bh[0] == bh[2]).all() and (sig[0] == sig[2]).all()


def test_empty_document_is_rejected():
    off = np.array([0, 3, 3, 5], np.uint64)
    with pytest.raises(oracle.OracleError) as e:
        oracle.signatures(off, np.arange(5, dtype=np.uint32), 128, 0, b=16, r=8)
    assert e.value.code == 2 and "index 1" in str(e.value)


def test_short_documents_use_one_whole_shingle():
    # fewer than n tokens -> a single shingle over all tokens
    for L in range(1, 5):
        ids = np.arange(L, dtype=np.uint32) + 17
        x = oracle.fingerprint(ids) % P61
        a, b, *_ = oracle.family(0, 32, 0, 0)
        want = [_affine_low32(int(a[i]), x, int(b[i])) for i in range(32)]
        assert oracle.signature_doc(ids, 32, 0).tolist() == want


def test_lshbloom_flags_superset_of_classic_lsh():
    # LSHBloom duplicates contain the classic exact-band-equality duplicates; the
    # excess is bounded by the Bloom FP tail.
    from synthetic.corpus import CONFIGS, gen_range
    cfg = CONFIGS["C1"].with_docs(3000)
    off, tok = gen_range(cfg, 0, 3000)
    sig, bh, dup, idx = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=3000,
                                   fp_rate=1e-3, seed=0)
    seen = [set() for _ in range(16)]
    classic = np.zeros(len(dup), np.uint8)
    for i in range(len(dup)):
        classic[i] = any(int(bh[i, j]) in seen[j] for j in range(16))
        for j in range(16):
            seen[j].add(int(bh[i, j]))
    assert (dup >= classic).all()
    p_eff = 1 - (1 - 1e-3) ** 16
    excess = int((dup > classic).sum())
    assert excess <= len(dup) * p_eff + 6 * math.sqrt(len(dup) * p_eff) + 3


# --------------------------------------------------------------------------- Bloom geometry

def test_bloom_fill_and_false_positive_rate():
    # S:286 fill ~ m(1-(1-1/m)^{kn}) within 1%; S:309 FP at capacity within [p/2, 2p]
    n, p = 20000, 1e-3
    rng = np.random.default_rng(6)
    ix = oracle.Index(1, n, p, seed=5)
    ix.query_insert(rng.integers(0, 2**61, (n, 1), dtype=np.uint64))
    m, k = ix.m, ix.k
    bits = np.unpackbits(ix.filter_bytes(0), bitorder="little")[:m]
    fill = bits.sum() / m
    assert fill == pytest.approx(1 - (1 - 1 / m) ** (k * n), rel=0.01)
    _, _, _, _, s1, s2 = oracle.family(5, 0, 0, 1)
    fresh = rng.integers(2**61, 2**62, 100000, dtype=np.uint64)
    fp = sum(all(bits[int(g)] for g in oracle.probes(int(x), int(s1[0]), int(s2[0]), m, k))
             for x in fresh) / len(fresh)
    assert p / 2 <= fp <= 2 * p, fp


def test_lsh_s_curve():
    # S:233 / S:597: candidate probability 1-(1-s^r)^b within 3 SE over 500 trials
    rng = np.random.default_rng(8)
    b, r, trials = 4, 3, 500
    for s in (0.3, 0.6, 0.9):
        hits = 0
        for _ in range(trials):
            x = rng.integers(0, 2**32, b * r, dtype=np.uint64).astype(np.uint32)
            y = np.where(rng.random(b * r) < s, x,
                         rng.integers(0, 2**32, b * r, dtype=np.uint64).astype(np.uint32))
            hits += any(oracle.band_hash(x, j, r, 1) == oracle.band_hash(y, j, r, 1) for j in range(b))
        pr = 1 - (1 - s ** r) ** b
        assert abs(hits / trials - pr) <= 3 * math.sqrt(pr * (1 - pr) / trials) + 1e-9
