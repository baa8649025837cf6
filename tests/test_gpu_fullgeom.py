"""Parity at the full geometry of BASELINE.json's larger configs, in the launch configuration
bench.py times: the filters sized for the config's whole corpus (n_expected = its document
count, so they are HBM-resident: C3 767 MB, C4 3.74 GB, C5 59.9 GB with m > 2^32) and whole
per-step batches (C3 200K full texts, C4 400K mixed documents, C5 two consecutive 4M-document
stream batches on one handle).  Every duplicate flag is compared with the CPU oracle's
sequential stream; band hashes too, and filter bytes for sampled
bands.  These run the sweep path the library picks for them (checked via info()["sweeps"])."""
import numpy as np
import pytest

import oracle
from synthetic.corpus import CONFIGS, gen_range_parallel

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom  # noqa: E402

DEV = torch.device("cuda:0")
STEP_DOCS = {"C3": 200_000, "C4": 400_000}


def to_dev(off, tok):
    return (torch.from_numpy(off.view(np.int64)).to(DEV), torch.from_numpy(tok.view(np.int32)).to(DEV))


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_step_at_config_geometry(name):
    cfg = CONFIGS[name]
    n = STEP_DOCS[name]
    off, tok = gen_range_parallel(cfg, 0, n)
    _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
    ref = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed)
    dup = ref.query_insert(bh)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    assert idx.info()["filter_bytes"] > 700e6
    d = to_dev(off, tok)
    got = idx.query_insert(*d).cpu().numpy()
    assert (got == dup).all(), np.flatnonzero(got != dup)[:20]
    assert idx.info()["sweeps"] >= 1
    assert (idx.band_hashes(*d).cpu().numpy().view(np.uint64) == bh).all()
    for j in (0, 13, cfg.b - 1):
        words = idx.filter_words(j).view(np.uint8)
        assert (words[:(ref.m + 7) // 8] == ref.filter_bytes(j)).all(), j
    # the bench's e2e form: pinned host batch, host flags
    idx2 = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
    p_tok = torch.from_numpy(tok.view(np.int32)).pin_memory()
    assert (np.asarray(idx2.query_insert(p_off, p_tok)) == dup).all()


def test_c5_two_full_stream_batches():
    """C5: 20 filters of m = 23,962,645,944 bits (59.9 GB) and two consecutive 4M-document batches
    of the 1B-document stream on one handle -- the second batch queries what the first inserted."""
    cfg = CONFIGS["C5"]
    B = cfg.batch_docs
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    assert idx.m > 2**32 and idx.info()["filter_bytes"] > 59e9
    ref = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed)
    for t in range(2):
        off, tok = gen_range_parallel(cfg, t * B, (t + 1) * B)
        _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
        dup = ref.query_insert(bh)
        got = idx.query_insert(*to_dev(off, tok)).cpu().numpy()
        assert (got == dup).all(), (t, np.flatnonzero(got != dup)[:20])
        assert dup.sum() > 0.05 * B
        torch.cuda.empty_cache()
    assert idx.info()["sweeps"] == 2 and idx.info()["doc_count"] == 2 * B
    for j in (0, cfg.b - 1):
        words = idx.filter_words(j).view(np.uint8)
        assert (words[:(ref.m + 7) // 8] == ref.filter_bytes(j)).all(), j
