"""Parity on prefixes of BASELINE.json's larger configs, each with its own LSH shape and filter
geometry: C3 (full-text lengths up to tens of thousands of words, 256 perms, b32 r8), C4 (the
8:31 full-text / abstract mixture with cross-length copies), C5 (b20 r6, filters sized for 1e9
documents so m = 23,962,645,944 > 2^32 and probe positions need 64 bits)."""
import numpy as np
import pytest

import oracle
from synthetic.corpus import CONFIGS, gen_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(off, tok):
    return (torch.from_numpy(off.view(np.int64)).to(DEV), torch.from_numpy(tok.view(np.int32)).to(DEV))


@pytest.mark.parametrize("name,n_docs,n_expected,sub_batch", [
    ("C3", 3000, None, 0),
    ("C4", 20000, None, 4096),
    ("C5", 60000, None, 0),
])
def test_config_prefix_parity(name, n_docs, n_expected, sub_batch):
    cfg = CONFIGS[name]
    n_exp = n_expected or cfg.n_docs            # filter geometry of the full config
    off, tok = gen_range(cfg, 0, n_docs)
    sig, bh, dup, ref = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=n_exp,
                                   fp_rate=cfg.fp_rate, seed=cfg.seed)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n_exp, cfg.fp_rate, cfg.seed, device=0, sub_batch=sub_batch)
    assert (idx.m, idx.k) == (ref.m, ref.k)
    d = to_dev(off, tok)
    assert (idx.signatures(*d).cpu().numpy().view(np.uint32) == sig).all()
    assert (idx.band_hashes(*d).cpu().numpy().view(np.uint64) == bh).all()
    got = idx.query_insert(*d).cpu().numpy()
    assert (got == dup).all(), np.flatnonzero(got != dup)[:10]
    assert dup.sum() > 0
    if name == "C5":
        assert idx.m > 2**32


def test_c3_longest_documents():
    # the longest documents of a large C3 sample (tails of the lognormal)
    cfg = CONFIGS["C3"]
    from synthetic.corpus import base_lengths
    L = base_lengths(cfg, np.arange(200_000))
    longest = np.sort(np.argsort(L)[-40:])
    from synthetic.corpus import gen_docs
    off, tok = gen_docs(cfg, longest)
    assert np.diff(off.astype(np.int64)).max() > 25_000
    sig, bh, dup, _ = oracle.run(off, tok, num_perm=256, b=32, r=8, n_expected=cfg.n_docs, fp_rate=cfg.fp_rate,
                                 seed=cfg.seed)
    idx = LSHBloom(256, 32, 8, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    d = to_dev(off, tok)
    assert (idx.signatures(*d).cpu().numpy().view(np.uint32) == sig).all()
    assert (idx.query_insert(*d).cpu().numpy() == dup).all()
