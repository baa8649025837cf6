"""Full-size parity at BASELINE.json's bench workload (config C2: 1M documents, 128 perms,
b16 r8, fp 1e-5) in the launch configuration bench.py times (device-resident batch, default
sub-batch, one query_insert per step) and through the host (e2e) path.  The oracle computes
every document (plain C, all host cores), so every signature, band hash and flag is compared
element by element."""
import os

import numpy as np
import pytest

import oracle
from synthetic.corpus import CONFIGS, checksum, gen_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def c2():
    cfg = CONFIGS["C2"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    sig, bh, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=cfg.n_docs,
                                 fp_rate=cfg.fp_rate, seed=cfg.seed)
    return cfg, off, tok, sig, bh, dup


def test_c2_full_parity_bench_configuration(c2):
    cfg, off, tok, sig, bh, dup = c2
    print("C2 checksum", checksum(off, tok), "flagged", int(dup.sum()))
    d_off = torch.from_numpy(off.view(np.int64)).to(DEV)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(DEV)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    got_dup = idx.query_insert(d_off, d_tok).cpu().numpy()
    assert (got_dup == dup).all(), np.flatnonzero(got_dup != dup)[:20]
    got_bh = idx.band_hashes(d_off, d_tok).cpu().numpy().view(np.uint64)
    assert (got_bh == bh).all()
    got_sig = idx.signatures(d_off, d_tok).cpu().numpy().view(np.uint32)
    assert (got_sig == sig).all()
    # a second step after reset (what bench.py repeats) gives the same flags
    idx.reset()
    assert (idx.query_insert(d_off, d_tok).cpu().numpy() == dup).all()


def test_c2_full_parity_host_path(c2):
    cfg, off, tok, sig, bh, dup = c2
    p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
    p_tok = torch.from_numpy(tok.view(np.int32)).pin_memory()
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    assert (idx.query_insert(p_off, p_tok) == dup).all()


def test_c2_planted_near_duplicates_are_detected(c2):
    # statistical fixed point: planted near-dups at J in [0.7, 0.99] are flagged at least at the
    # S-curve rate 1-(1-s^r)^b (s ~ J); almost all non-planted docs are not flagged.
    from synthetic.corpus import planted_pairs
    cfg, off, tok, sig, bh, dup = c2
    d, src, e = planted_pairs(cfg, 0, cfg.n_docs)
    rate = dup[d].mean()
    J = (2 * (1 - e) ** 5) / (2 - (1 - e) ** 5)
    expect = np.mean(1 - (1 - J ** cfg.r) ** cfg.b)
    assert rate >= expect - 0.03, (rate, expect)
    others = np.ones(cfg.n_docs, bool)
    others[d] = False
    assert dup[others].mean() < 0.01
