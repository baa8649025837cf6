"""The C oracle against an independent second implementation of its conventions.

tests/support/micro_oracle.py re-implements DESIGN.md section 3 (R1 fingerprint, R3-R6 family /
MinHash / band hash, R9 sizing, R10 probes, R12-R13 stream order) and the blocked variant's
offsets from their prose definitions, in pure Python big integers.  Element-by-element equality
here pins the exact values of orc_fingerprint, orc_family, orc_probes_blocked and everything built
on them, which the closed-form / statistical pins in test_oracle_pins.py only constrain by
properties.  The known-answer file tests/golden/conventions_kat.json (written by
tools/gen_conventions_kat.py, which calls only oracle/) freezes a few of those values so a later
change to either implementation is caught even if both drift together.  No GPU needed."""
import json
import os

import numpy as np
import pytest

import oracle
from support import micro_oracle as mo

SEEDS = [0, 1, 42, 0xDEADBEEF, 2**64 - 1]


@pytest.mark.parametrize("seed", SEEDS)
def test_family_matches_micro_oracle(seed):
    a, b, c, d, s1, s2 = oracle.family(seed, 256, 8, 32)
    ma, mb = mo.permutation_coefficients(seed, 256)
    mc, md = mo.band_coefficients(seed, 8)
    ms1, ms2 = mo.filter_seeds(seed, range(32))
    assert a.tolist() == ma and b.tolist() == mb
    assert c.tolist() == mc and d.tolist() == md
    assert s1.tolist() == ms1 and s2.tolist() == ms2


def test_fingerprint_matches_micro_oracle():
    rng = np.random.default_rng(11)
    cases = [[0], [0, 0], [1], [2**32 - 1], [0, 1, 2, 3, 4], [2**32 - 1] * 5, [7, 7, 7, 7, 7, 7, 7]]
    for t in range(1, 9):
        for _ in range(40):
            cases.append(rng.integers(0, 2**32, t, dtype=np.uint64).tolist())
            cases.append(rng.integers(0, 5, t, dtype=np.uint64).tolist())
    for ids in cases:
        assert oracle.fingerprint(ids) == mo.shingle_fingerprint(ids), ids


@pytest.mark.parametrize("seed", [0, 42])
def test_signatures_and_band_hashes_match_micro_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    docs = []
    for i in range(48):
        L = int(rng.integers(1, 40))
        docs.append(rng.integers(0, 2**32 if i % 3 == 0 else 50, L, dtype=np.uint64).astype(np.uint32))
    docs.append(docs[5].copy())                     # an exact duplicate
    docs.append(np.concatenate([docs[7], docs[7]]))  # a repeated shingle set
    off = np.zeros(len(docs) + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in docs])
    tok = np.concatenate(docs).astype(np.uint32)
    sig, bh = oracle.signatures(off, tok, 64, seed, b=8, r=8)
    for i, ids in enumerate(docs):
        ms = mo.signature(ids.tolist(), 64, seed)
        assert sig[i].tolist() == ms, i
        assert bh[i].tolist() == [mo.band_hash(ms, j, 8, seed) for j in range(8)], i


def test_band_hash_rows_beyond_b_r_ignored_and_r_general():
    # b*r < num_perm (C5: 20 x 6 of 128 rows) and a larger r (sums reduce mod P after each add)
    rng = np.random.default_rng(3)
    for r in (1, 6, 13):
        sig = rng.integers(0, 2**32, 128, dtype=np.uint64).astype(np.uint32)
        for j in range(128 // r):
            assert oracle.band_hash(sig, j, r, 9) == mo.band_hash(sig.tolist(), j, r, 9)


@pytest.mark.parametrize("m", [1, 2, 97, 239_627, 23_962_646, 2**32 + 15, 23_962_645_944, 2**40 + 3])
def test_probe_positions_match_micro_oracle(m):
    rng = np.random.default_rng(m % 1000)
    for _ in range(60):
        bh = int(rng.integers(0, mo.P))
        s1, s2 = int(rng.integers(0, 2**63)) * 2 + 1, int(rng.integers(0, 2**63))
        assert oracle.probes(bh, s1, s2, m, 17).tolist() == mo.probe_positions(bh, s1, s2, m, 17)


@pytest.mark.parametrize("nb", [1, 3, 23_402, 23_401_022])
def test_blocked_positions_match_micro_oracle(nb):
    rng = np.random.default_rng(nb % 997)
    for k in (1, 6, 7, 17, 40):
        for _ in range(20):
            bh = int(rng.integers(0, mo.P))
            s1, s2 = int(rng.integers(0, 2**64, dtype=np.uint64)), int(rng.integers(0, 2**64, dtype=np.uint64))
            assert oracle.probes_blocked(bh, s1, s2, nb, k).tolist() == mo.blocked_positions(bh, s1, s2, nb, k)


def test_sizing_matches_micro_oracle():
    for n in (1, 2, 7, 1000, 10_000, 1_000_000, 8_000_000, 39_000_000, 1_000_000_000, 5 * 10**9):
        for p in (0.5, 0.1, 1e-3, 1e-5, 1e-10, 2.0**-17):
            assert oracle.bloom_size(n, p) == mo.bloom_geometry(n, p), (n, p)


@pytest.mark.parametrize("blocked", [False, True])
def test_stream_flags_match_micro_oracle(blocked):
    """Dense filters (n_expected far below the stream length) so bits collide often; planted
    duplicates and near-duplicates; per-band hits and final filter bytes too."""
    rng = np.random.default_rng(7 + blocked)
    docs = []
    for i in range(150):
        if i > 3 and rng.random() < 0.25:
            src = docs[int(rng.integers(0, len(docs)))].copy()
            if rng.random() < 0.5 and len(src) > 6:
                src[int(rng.integers(0, len(src)))] = int(rng.integers(0, 30))
            docs.append(src)
        else:
            docs.append(rng.integers(0, 30, int(rng.integers(1, 25))).astype(np.uint32))
    b, r, num_perm, n_exp, p, seed = 6, 3, 20, 40, 1e-2, 5
    msig, mbh, mdup, midx = mo.run([d.tolist() for d in docs], num_perm=num_perm, b=b, r=r,
                                   n_expected=n_exp, p=p, seed=seed, blocked=blocked)
    off = np.zeros(len(docs) + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in docs])
    tok = np.concatenate(docs).astype(np.uint32)
    sig, bh = oracle.signatures(off, tok, num_perm, seed, b=b, r=r)
    idx = oracle.Index(b, n_exp, p, seed, blocked=blocked)
    dup, hits = idx.query_insert(bh, want_hits=True)
    assert sig.tolist() == msig and bh.tolist() == mbh
    assert dup.tolist() == mdup
    assert 0 < sum(mdup) < len(docs)
    assert idx.m == midx.m and idx.k == midx.k
    for j in range(b):
        assert idx.filter_bytes(j).tobytes() == midx.filter_bytes(j)


def _kat():
    with open(os.path.join(os.path.dirname(__file__), "golden", "conventions_kat.json")) as f:
        return json.load(f)


def test_known_answers_both_implementations():
    kat = _kat()
    for row in kat["fingerprint"]:
        want = int(row["fp"], 16)
        assert oracle.fingerprint(row["ids"]) == want
        assert mo.shingle_fingerprint(row["ids"]) == want
    for row in kat["family"]:
        a, b, c, d, s1, s2 = oracle.family(row["seed"], len(row["a"]), len(row["c"]), len(row["s1"]))
        got = {"a": a, "b": b, "c": c, "d": d, "s1": s1, "s2": s2}
        for key, arr in got.items():
            assert [int(x, 16) for x in row[key]] == arr.tolist(), key
        ma, mb = mo.permutation_coefficients(row["seed"], len(row["a"]))
        assert [int(x, 16) for x in row["a"]] == ma and [int(x, 16) for x in row["b"]] == mb
    for row in kat["signature"]:
        sig = oracle.signature_doc(row["ids"], row["num_perm"], row["seed"])
        assert sig.tolist() == row["sig"]
        assert mo.signature(row["ids"], row["num_perm"], row["seed"]) == row["sig"]
        assert [mo.band_hash(row["sig"], j, row["r"], row["seed"]) for j in range(row["b"])] == \
            [int(x, 16) for x in row["band_hashes"]]
    for row in kat["probes"]:
        want = [int(x) for x in row["g"]]
        bh, s1, s2 = (int(row[k], 16) for k in ("bh", "s1", "s2"))
        if row["blocked"]:
            assert oracle.probes_blocked(bh, s1, s2, row["nb"], row["k"]).tolist() == want
            assert mo.blocked_positions(bh, s1, s2, row["nb"], row["k"]) == want
        else:
            assert oracle.probes(bh, s1, s2, row["m"], row["k"]).tolist() == want
            assert mo.probe_positions(bh, s1, s2, row["m"], row["k"]) == want
