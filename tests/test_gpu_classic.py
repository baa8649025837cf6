"""Parity of the GPU classic MinHashLSH index (index="classic", lb_classic.cu) with the oracle's
classic index (oracle.Classic, pinned in tests/test_oracle_classic.py): duplicate flags
bit-identical in stream order, on C1 and the full C2 batch, under batch splits, band sharding,
dense collisions and the capacity limit."""
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


def classic(cfg, n_expected=None, **kw):
    return LSHBloom(cfg.num_perm, cfg.b, cfg.r, n_expected or cfg.n_docs, cfg.fp_rate, cfg.seed,
                    device=0, index="classic", **kw)


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
    dup_c = oracle.Classic(cfg.b).query_insert(bh)
    dup_b = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed).query_insert(bh)
    return cfg, off, tok, bh, dup_c, dup_b


def test_c1_classic_flags_device_and_host(c1):
    cfg, off, tok, bh, dup_c, dup_b = c1
    assert dup_c.sum() > 0
    idx = classic(cfg)
    assert idx.index == "classic" and idx.info()["classic_slots"] >= cfg.n_docs / 0.7
    d_off, d_tok = to_dev(off, tok)
    got = idx.query_insert(d_off, d_tok).cpu().numpy()
    assert (got == dup_c).all(), np.flatnonzero(got != dup_c)[:10]
    idx.reset()
    assert (idx.query_insert(off, tok) == dup_c).all()
    # the Bloom index's duplicates contain the classic ones
    assert (dup_b >= got).all()


def test_c1_classic_batch_splits_and_bands_path(c1):
    cfg, off, tok, bh, dup_c, _ = c1
    rng = np.random.default_rng(3)
    cuts = np.unique(np.concatenate([[0, 1, 2, cfg.n_docs], rng.integers(3, cfg.n_docs, 12)]))
    idx = classic(cfg)
    parts = []
    for a, c in zip(cuts[:-1], cuts[1:]):
        o = off[a:c + 1] - off[a]
        parts.append(idx.query_insert(*to_dev(o, tok[off[a]:off[c]])).cpu().numpy())
    assert (np.concatenate(parts) == dup_c).all()
    idx2 = classic(cfg)
    got = idx2.query_insert_bands(torch.from_numpy(bh.view(np.int64)).to(DEV)).cpu().numpy()
    assert (got == dup_c).all()


def test_c1_classic_band_sharded_handles(c1):
    cfg, off, tok, bh, dup_c, _ = c1
    world = 3
    acc = np.zeros(cfg.n_docs, np.uint8)
    for rank in range(world):
        h = classic(cfg, rank=rank, world=world)
        lo, hi = h.band_lo, h.band_hi
        part = h.query_insert_bands(torch.from_numpy(np.ascontiguousarray(bh[:, lo:hi]).view(np.int64)).to(DEV))
        acc |= part.cpu().numpy()
    assert (acc == dup_c).all()


def test_classic_dense_collisions():
    # every document identical in some bands, distinct in others; long runs of equal keys
    rng = np.random.default_rng(5)
    n, b = 70000, 6
    bh = rng.integers(0, 2**61 - 1, (n, b), dtype=np.uint64)
    bh[:, 0] = 12345                       # band 0: one key for everybody
    bh[::7, 1] = bh[0, 1]                  # band 1: every 7th document repeats document 0
    bh[1::3, 2] = rng.integers(0, 50, len(bh[1::3, 2]), dtype=np.uint64)
    want = oracle.Classic(b).query_insert(bh)
    assert want[0] == 0 and want[1:].all()
    h = LSHBloom(64, b, 4, n, 1e-5, 0, device=0, index="classic")
    got = h.query_insert_bands(torch.from_numpy(bh.view(np.int64)).to(DEV)).cpu().numpy()
    assert (got == want).all()
    # without band 0 the verdicts are mixed
    want2 = oracle.Classic(b - 1).query_insert(np.ascontiguousarray(bh[:, 1:]))
    h2 = LSHBloom(64, b - 1, 4, n, 1e-5, 0, device=0, index="classic")
    got2 = h2.query_insert_bands(torch.from_numpy(np.ascontiguousarray(bh[:, 1:]).view(np.int64)).to(DEV))
    assert (got2.cpu().numpy() == want2).all() and 0 < want2.sum() < n


def test_classic_capacity_rejects_before_mutation():
    rng = np.random.default_rng(9)
    h = LSHBloom(32, 2, 4, 100, 1e-5, 0, device=0, index="classic")
    slots = h.info()["classic_slots"]
    bh = rng.integers(0, 2**61 - 1, (int(0.9 * slots) + 5, 2), dtype=np.uint64)
    with pytest.raises(LSHBloomError) as e:
        h.query_insert_bands(torch.from_numpy(bh.view(np.int64)).to(DEV))
    assert e.value.code == 1 and h.info()["doc_count"] == 0
    small = bh[:100]
    got = h.query_insert_bands(torch.from_numpy(small.view(np.int64)).to(DEV)).cpu().numpy()
    assert (got == oracle.Classic(2).query_insert(small)).all()
    with pytest.raises(LSHBloomError):
        h.filter_words(0)


@pytest.mark.slow
def test_c2_full_classic_flags():
    cfg = CONFIGS["C2"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
    want = oracle.Classic(cfg.b).query_insert(bh)
    idx = classic(cfg)
    got = idx.query_insert(*to_dev(off, tok)).cpu().numpy()
    assert (got == want).all(), np.flatnonzero(got != want)[:10]
    bloom = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    gb = bloom.query_insert(*to_dev(off, tok)).cpu().numpy()
    assert (gb >= got).all()
    p_eff = bloom.info()["p_eff"]
    assert (gb > got).sum() <= cfg.n_docs * p_eff + 6 * np.sqrt(cfg.n_docs * p_eff) + 3
