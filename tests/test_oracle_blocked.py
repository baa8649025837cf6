"""Pins for the oracle's blocked Bloom variant: every band hash's k probes
fall in one 1024-bit block.  Checked against the structure it promises, uniformity, a
brute-force set formulation of the stream semantics, the analytic fill and the Poisson-mixture
false-positive rate of a blocked filter, zero false negatives and the classic index.
No GPU needed."""
import math

import numpy as np
import pytest
from scipy.stats import chisquare, poisson

import oracle


def _params(seed=5):
    _, _, _, _, s1, s2 = oracle.family(seed, 0, 0, 1)
    return int(s1[0]), int(s2[0])


def test_blocked_probe_structure_and_uniformity():
    rng = np.random.default_rng(1)
    s1, s2 = _params()
    nb, k = 64, 17
    blocks, offs = [], []
    for bh in rng.integers(0, 2**61 - 1, 6000, dtype=np.uint64):
        g = oracle.probes_blocked(int(bh), s1, s2, nb, k).astype(np.int64)
        blk = g // 1024
        assert (blk == blk[0]).all() and 0 <= blk[0] < nb      # one block, in range
        blocks.append(int(blk[0]))
        offs.extend((g % 1024).tolist())
    # block index and in-block offsets uniform (chi-square, 6000 and 102000 draws)
    assert chisquare(np.bincount(blocks, minlength=nb)).pvalue > 1e-4
    assert chisquare(np.bincount(np.asarray(offs) // 16, minlength=64)).pvalue > 1e-4
    # the k offsets of one key behave like independent draws: repeats at the birthday rate
    rep = np.mean([len(set(oracle.probes_blocked(int(x), s1, s2, nb, k).tolist())) < k
                   for x in rng.integers(0, 2**61 - 1, 4000, dtype=np.uint64)])
    expect = 1 - math.prod(1 - t / 1024 for t in range(k))
    assert abs(rep - expect) < 5 * math.sqrt(expect * (1 - expect) / 4000)


def test_blocked_stream_semantics_bruteforce():
    # dup_i <=> exists band j: Pos_j(i) is a subset of the union of earlier documents' Pos_j
    # (set formulation, no bit array), with dense collisions from a tiny filter
    rng = np.random.default_rng(2)
    n, b = 1500, 3
    bh = rng.integers(0, 2**61 - 1, (n, b), dtype=np.uint64)
    bh[rng.integers(1, n, 200)] = bh[rng.integers(0, 1, 200)]
    ix = oracle.Index(b, 60, 0.2, seed=7, blocked=True)
    assert ix.m % 1024 == 0
    got = ix.query_insert(bh)
    _, _, _, _, s1, s2 = oracle.family(7, 0, 0, b)
    nb = ix.m // 1024
    seen = [set() for _ in range(b)]
    want = np.zeros(n, np.uint8)
    for i in range(n):
        hit = False
        for j in range(b):
            pos = set(oracle.probes_blocked(int(bh[i, j]), int(s1[j]), int(s2[j]), nb, ix.k).tolist())
            hit |= pos <= seen[j]
            seen[j] |= pos
        want[i] = hit
    assert (got == want).all() and 0 < want.sum() < n


@pytest.mark.parametrize("n,p", [(20000, 1e-2), (20000, 1e-3)])
def test_blocked_fill_fp_and_no_false_negatives(n, p):
    rng = np.random.default_rng(6)
    ix = oracle.Index(1, n, p, seed=5, blocked=True)
    keys = rng.integers(0, 2**61, (n, 1), dtype=np.uint64)
    ix.query_insert(keys)
    m, k = ix.m, ix.k
    nb = m // 1024
    bits = np.unpackbits(ix.filter_bytes(0), bitorder="little")[:m]
    # every probe is uniform over the m bits -> the standard fill formula
    assert bits.mean() == pytest.approx(1 - (1 - 1 / m) ** (k * n), rel=0.01)
    s1, s2 = _params()
    for x in keys[:300, 0]:                                       # no false negatives
        assert all(bits[int(g)] for g in oracle.probes_blocked(int(x), s1, s2, nb, k))
    # false positives: Poisson mixture over block loads, P = sum_i Pois(i; n/nb) (1-(1-1/1024)^(k i))^k
    fresh = rng.integers(2**61, 2**62, 120000, dtype=np.uint64)
    fp = np.mean([all(bits[int(g)] for g in oracle.probes_blocked(int(x), s1, s2, nb, k)) for x in fresh])
    lam = n / nb
    i = np.arange(0, int(lam * 4 + 80))
    an = float((poisson.pmf(i, lam) * (1 - (1 - 1 / 1024) ** (k * i)) ** k).sum())
    assert abs(fp - an) < 5 * math.sqrt(an / len(fresh)) + 1e-4, (fp, an)
    # and it costs more false positives than the standard filter of the same m (P:227 analysis)
    assert an > (1 - math.exp(-k * n / m)) ** k


def test_blocked_flags_superset_of_classic():
    from synthetic.corpus import CONFIGS, gen_range
    cfg = CONFIGS["C1"].with_docs(3000)
    off, tok = gen_range(cfg, 0, 3000)
    _, bh = oracle.signatures(off, tok, 128, 0, b=16, r=8, want_sig=False)
    dup = oracle.Index(16, 3000, 1e-3, 0, blocked=True).query_insert(bh)
    classic = oracle.Classic(16).query_insert(bh)
    assert (dup >= classic).all() and classic.sum() > 0
