"""lshbloom_bands_begin / _add / _finish (the pipelined sharded step's owner side): band-hash
chunks of a global batch handed over in any order -- as the chunks of several ranks arrive in a
pipelined exchange -- give the flags of lshbloom_query_insert_bands on the whole batch, i.e. the
oracle's stream order, for both Bloom paths, the classic and
blocked indexes, and simulated band-sharded ranks on one GPU."""
import numpy as np
import pytest

import oracle
from synthetic.corpus import CONFIGS, gen_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom, LSHBloomError  # noqa: E402
from paper_2411_04257_b200.sharded import band_range  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    _, bh, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=cfg.n_docs,
                               fp_rate=cfg.fp_rate, seed=cfg.seed)
    return cfg, bh, dup


def chunks_interleaved(n_ranks_docs, chunk):
    """(doc0, n) pieces in pipelined arrival order: chunk c of every rank, then chunk c + 1."""
    starts = np.concatenate([[0], np.cumsum(n_ranks_docs)])
    out, c = [], 0
    while True:
        got = False
        for r, nr in enumerate(n_ranks_docs):
            a, b = min(c * chunk, nr), min((c + 1) * chunk, nr)
            if b > a:
                out.append((int(starts[r] + a), int(b - a)))
                got = True
        if not got:
            return out
        c += 1


@pytest.mark.parametrize("path,world,chunk", [("sweep", 1, 700), ("sweep", 3, 257), ("random", 2, 1000),
                                              ("sweep", 4, 5000)])
def test_bands_assembled_out_of_order_match_oracle(c1, path, world, chunk):
    cfg, bh, dup = c1
    n = cfg.n_docs
    ranks_docs = [n // 3, 1, n - n // 3 - 1]                      # three producer ranks, one tiny
    pieces = chunks_interleaved(ranks_docs, chunk)
    hits = []
    for g in range(world):                                       # simulated band owners
        h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, rank=g, world=world,
                     bloom_path=path)
        own = torch.from_numpy(np.ascontiguousarray(bh[:, h.band_lo:h.band_hi]).view(np.int64)).to(DEV)
        h.bands_begin(n)
        for doc0, k in pieces:
            h.bands_add(own[doc0:doc0 + k], doc0)
        hits.append(h.bands_finish().cpu().numpy())
        assert h.info()["doc_count"] == n
    assert (np.maximum.reduce(hits) == dup).all()


@pytest.mark.parametrize("kind", ["classic", "blocked"])
def test_bands_other_index_kinds(c1, kind):
    cfg, bh, _ = c1
    ref = oracle.Classic(cfg.b) if kind == "classic" else oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed,
                                                                          blocked=True)
    want = ref.query_insert(bh)
    h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, index=kind,
                 bloom_path="sweep")
    d = torch.from_numpy(bh.view(np.int64)).to(DEV)
    h.bands_begin(cfg.n_docs)
    for doc0, k in chunks_interleaved([cfg.n_docs // 2, cfg.n_docs - cfg.n_docs // 2], 999):
        h.bands_add(d[doc0:doc0 + k], doc0)
    assert (h.bands_finish().cpu().numpy() == want).all()


def test_bands_incomplete_batch_rejected(c1):
    cfg, bh, dup = c1
    h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    d = torch.from_numpy(bh.view(np.int64)).to(DEV)
    h.bands_begin(100)
    h.bands_add(d[:60], 0)
    with pytest.raises(LSHBloomError) as e:
        h.bands_finish()
    assert e.value.code == 1
    with pytest.raises(LSHBloomError):
        h.bands_begin(10)
        h.bands_add(d[:20], 0)                                   # beyond n_global
    # the handle still works, and nothing was inserted
    assert (h.query_insert_bands(d) == torch.from_numpy(dup).to(DEV)).all()
