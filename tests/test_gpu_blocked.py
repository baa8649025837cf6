"""Parity of the GPU blocked Bloom variant (index="blocked") with the
oracle's blocked index (oracle.Index(blocked=True), pinned in tests/test_oracle_blocked.py):
duplicate flags and filter bytes bit-identical in stream order, under sub-batch sizes, batch
splits, dense collisions and C5's m > 2^32 geometry."""
import numpy as np
import pytest

import oracle
from synthetic.corpus import CONFIGS, gen_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom, LSHBloomError  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(off, tok):
    return (torch.from_numpy(np.ascontiguousarray(off, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(tok, np.uint32).view(np.int32)).to(DEV))


def dbh(bh):
    return torch.from_numpy(np.ascontiguousarray(bh).view(np.int64)).to(DEV)


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
    ref = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed, blocked=True)
    dup = ref.query_insert(bh)
    return cfg, off, tok, bh, dup, ref


def test_c1_blocked_flags_and_filters(c1):
    cfg, off, tok, bh, dup, ref = c1
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, index="blocked")
    assert idx.index == "blocked" and (idx.m, idx.k) == (ref.m, ref.k) and idx.m % 1024 == 0
    got = idx.query_insert(*to_dev(off, tok)).cpu().numpy()
    assert (got == dup).all(), np.flatnonzero(got != dup)[:10]
    assert dup.sum() > 0
    for j in (0, 7, cfg.b - 1):
        words = idx.filter_words(j)
        assert (words.view(np.uint8)[:(ref.m + 7) // 8] == ref.filter_bytes(j)).all()
    with pytest.raises(LSHBloomError):
        idx.save("/tmp/never_written.lshb")


@pytest.mark.parametrize("sub_batch", [1, 7, 1000, 0])
def test_c1_blocked_sub_batch_and_splits(c1, sub_batch):
    cfg, off, tok, bh, dup, _ = c1
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, index="blocked",
                   sub_batch=sub_batch)
    cuts = [0, 1, 2500, 2501, 9000, cfg.n_docs]
    got = np.concatenate([idx.query_insert_bands(dbh(bh[a:c])).cpu().numpy() for a, c in zip(cuts[:-1], cuts[1:])])
    assert (got == dup).all()


def test_blocked_dense_collisions():
    # a tiny filter (few blocks): most positions are contested inside a sub-batch
    rng = np.random.default_rng(4)
    n, b = 40000, 3
    bh = rng.integers(0, 2**61 - 1, (n, b), dtype=np.uint64)
    bh[rng.integers(1, n, 3000)] = bh[rng.integers(0, 50, 3000)]
    ref = oracle.Index(b, 300, 0.05, 11, blocked=True)
    want = ref.query_insert(bh)
    for sb in (0, 333):
        h = LSHBloom(32, b, 4, 300, 0.05, 11, device=0, index="blocked", sub_batch=sb)
        assert h.m == ref.m
        got = h.query_insert_bands(dbh(bh)).cpu().numpy()
        assert (got == want).all(), (sb, np.flatnonzero(got != want)[:10])
    assert 0 < want.sum() < n


def test_c5_geometry_blocked_prefix():
    # C5's filters (n_expected = 1e9, m > 2^32 bits, 64-bit positions) on 2 bands of a prefix
    cfg = CONFIGS["C5"]
    off, tok = gen_range(cfg, 0, 30000)
    _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
    bh2 = np.ascontiguousarray(bh[:, :2])
    ref = oracle.Index(2, cfg.n_docs, cfg.fp_rate, cfg.seed, blocked=True)
    want = ref.query_insert(bh2)
    h = LSHBloom(cfg.num_perm, 2, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, index="blocked")
    assert h.m == ref.m and h.m > 2**32
    got = h.query_insert_bands(dbh(bh2)).cpu().numpy()
    assert (got == want).all()
    assert want.sum() > 0
