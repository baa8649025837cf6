"""Pins for the oracle's classic MinHashLSH index and capacity planner:
brute-force set formulations, the paper's printed band count and index sizes, and an
independent quadrature of the S-curve objective.  No GPU needed."""
import math

import numpy as np
import pytest

import oracle


def _classic_bruteforce(bh):
    """dup_i = exists j: bh[i][j] in {bh[i'][j] : i' < i}  (P:134 exact band equality)."""
    n, b = bh.shape
    seen = [set() for _ in range(b)]
    out = np.zeros(n, np.uint8)
    for i in range(n):
        out[i] = any(int(bh[i, j]) in seen[j] for j in range(b))
        for j in range(b):
            seen[j].add(int(bh[i, j]))
    return out


def test_classic_matches_bruteforce_with_planted_repeats():
    rng = np.random.default_rng(11)
    n, b = 5000, 7
    bh = rng.integers(0, 2**61 - 1, (n, b), dtype=np.uint64)
    for _ in range(1500):               # copy single bands and whole rows from earlier documents
        i = int(rng.integers(1, n))
        src = int(rng.integers(0, i))
        if rng.random() < 0.3:
            bh[i] = bh[src]
        else:
            j = int(rng.integers(0, b))
            bh[i, j] = bh[src, j]
    # repeats inside one document's own bands must not count (bands are separate maps)
    bh[10, 1] = bh[10, 0]
    ix = oracle.Classic(b)
    dup, hits = ix.query_insert(bh, want_hits=True)
    assert (dup == _classic_bruteforce(bh)).all()
    assert (dup == hits.max(axis=1)).all()
    for j in range(b):
        assert ix.keys(j) == len(set(bh[:, j].tolist()))


def test_classic_identical_documents_and_batch_split():
    # S:393 analogue: [d, d] -> [unique, dup]; results independent of batch boundaries
    rng = np.random.default_rng(12)
    bh = rng.integers(0, 2**61 - 1, (3000, 4), dtype=np.uint64)
    bh[1] = bh[0]
    bh[2999] = bh[5]
    whole = oracle.Classic(4).query_insert(bh)
    assert whole[0] == 0 and whole[1] == 1 and whole[2999] == 1
    ix = oracle.Classic(4)
    parts = [ix.query_insert(bh[a:c]) for a, c in [(0, 1), (1, 777), (777, 778), (778, 3000)]]
    assert (np.concatenate(parts) == whole).all()


def test_classic_band_range_and_lshbloom_superset():
    # LSHBloom duplicates contain the classic duplicates; a sharded band range of the
    # classic index ORs to the whole.
    from synthetic.corpus import CONFIGS, gen_range
    cfg = CONFIGS["C1"].with_docs(3000)
    off, tok = gen_range(cfg, 0, 3000)
    _, bh, dup, _ = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=3000, fp_rate=1e-3, seed=0)
    classic = oracle.Classic(16).query_insert(bh)
    assert (classic == _classic_bruteforce(bh)).all()
    assert (dup >= classic).all()
    lo = oracle.Classic(16)
    a = lo.query_insert(bh[:, :5], band_lo=0)
    c = lo.query_insert(bh[:, 5:], band_lo=5)
    assert ((a | c) == classic).all()


def _objective(T, b, r, w=0.5):
    from scipy.integrate import quad
    fp = quad(lambda s: 1 - (1 - s**r) ** b, 0, T, limit=200)[0]
    fn = quad(lambda s: (1 - s**r) ** b, T, 1, limit=200)[0]
    return w * fp + (1 - w) * fn


def test_optimal_params_paper_nine_bands():
    # "T of 0.8, and 128 random permutations ... MinHashLSH creates nine bands"
    b, r = oracle.optimal_params(0.8, 128)
    assert b == 9 and b * r <= 128


@pytest.mark.parametrize("T,num_perm", [(0.5, 48), (0.8, 128), (0.3, 64), (0.9, 32), (0.7, 256)])
def test_optimal_params_vs_independent_quadrature(T, num_perm):
    # exhaustive search with adaptive Gauss-Kronrod quadrature (an independent integrator)
    b, r = oracle.optimal_params(T, num_perm)
    assert b * r <= num_perm
    best = min(_objective(T, bb, rr) for bb in range(1, num_perm + 1) for rr in range(1, num_perm // bb + 1))
    assert _objective(T, b, r) <= best + 1e-7


def test_optimal_params_rejects_bad_threshold():
    for T in (0.0, -0.5, 1.5, float("nan")):
        with pytest.raises(ValueError):
            oracle.optimal_params(T, 128)


@pytest.mark.parametrize("n,p_eff,size,unit,tol", [
    (5e9, 1e-5, 160.51, 1e9, 0.0005),     # Table 1, 5B docs, p_eff 1e-5
    (1e10, 1e-10, 590.0, 1e9, 0.005),     # P:229 "would only require 590 GB"
    (1e11, 1e-5, 3.21, 1e12, 0.005),      # Table 2, 100B docs
])
def test_plan_reproduces_paper_sizes(n, p_eff, size, unit, tol):
    pl = oracle.plan(n, p_eff, 0.8, 128)
    assert pl["b"] == 9
    assert pl["total_bytes"] / unit == pytest.approx(size, rel=tol)
    assert 1 - (1 - pl["p"]) ** pl["b"] == pytest.approx(p_eff, rel=1e-9)
