"""The window-sweep Bloom path (K7-K9, lb_sweep.cu) against the CPU oracle, element by element.

The sweep applies a whole batch window by window (TMA bulk copy of 2^w filter bits into shared
memory, all of the window's probes applied there with the stream-order lemma, one bulk store
back).  Its flags and final filter bits must equal the oracle's sequential query-then-insert
 for every window size, bin capacity (tiny capacities force the
device-side exact layout; one-window bands force bins beyond 2048 records onto the global-memory
branch), batch and call split, index kind, and the peer / band-sharded entry points."""
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
    return (torch.from_numpy(np.ascontiguousarray(off, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(tok, np.uint32).view(np.int32)).to(DEV))


def u8(t):
    return t.cpu().numpy() if torch.is_tensor(t) else t


def csr(docs):
    off = np.zeros(len(docs) + 1, np.uint64)
    off[1:] = np.cumsum([len(d) for d in docs])
    tok = np.concatenate([np.asarray(d, np.uint32) for d in docs]) if docs else np.zeros(0, np.uint32)
    return off, tok


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    sig, bh, dup, ref = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r,
                                   n_expected=cfg.n_docs, fp_rate=cfg.fp_rate, seed=cfg.seed)
    return cfg, off, tok, bh, dup, ref


def sweep(cfg, n_expected=None, **kw):
    kw.setdefault("bloom_path", "sweep")
    return LSHBloom(cfg.num_perm, cfg.b, cfg.r, n_expected or cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, **kw)


def assert_filters_equal(idx, ref, bands):
    for j in bands:
        words = idx.filter_words(j).view(np.uint8)
        nb = (ref.m + 7) // 8
        assert (words[:nb] == ref.filter_bytes(j)).all(), j
        assert not words[nb:].any()


@pytest.mark.parametrize("wlog2", [0, 10, 12, 16, 19])
def test_c1_sweep_flags_and_filters(c1, wlog2):
    cfg, off, tok, bh, dup, ref = c1
    idx = sweep(cfg, sweep_window_log2=wlog2)
    got = u8(idx.query_insert(*to_dev(off, tok)))
    assert (got == dup).all(), np.flatnonzero(got != dup)[:10]
    assert idx.info()["sweeps"] == 1
    assert_filters_equal(idx, ref, range(cfg.b))


@pytest.mark.parametrize("cap", [1, 3, 64])
def test_exact_layout_after_overflow(c1, cap):
    # a capacity far below the load: every sweep switches to the exact (scanned) layout
    cfg, off, tok, bh, dup, ref = c1
    idx = sweep(cfg, sweep_window_log2=12, sweep_cap=cap)
    assert (u8(idx.query_insert(*to_dev(off, tok))) == dup).all()
    assert_filters_equal(idx, ref, (0, 5, cfg.b - 1))


@pytest.mark.parametrize("cap", [0, 2])
def test_bins_beyond_register_capacity(c1, cap):
    # m = 239,627 < 2^19: one window per band, ~170K records per bin -> the global-memory branch
    cfg, off, tok, bh, dup, ref = c1
    idx = sweep(cfg, sweep_window_log2=19, sweep_cap=cap)
    assert (u8(idx.query_insert(*to_dev(off, tok))) == dup).all()
    assert_filters_equal(idx, ref, range(cfg.b))


def test_sweep_call_boundaries_and_host_path(c1):
    cfg, off, tok, bh, dup, ref = c1
    rng = np.random.default_rng(4)
    cuts = np.unique(np.concatenate([[0, cfg.n_docs], rng.integers(1, cfg.n_docs, 9), [1, 2]]))
    for host in (False, True):
        idx = sweep(cfg)
        got = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            o = off[a:b + 1] - off[a]
            t = tok[int(off[a]):int(off[b])]
            got.append(u8(idx.query_insert(o, t) if host else idx.query_insert(*to_dev(o, t))))
        assert (np.concatenate(got) == dup).all()


def test_sweep_dense_collisions_tiny_filters():
    cfg = CONFIGS["C1"]
    n = 6000
    off, tok = gen_range(cfg, 0, n)
    docs = [tok[int(off[i]):int(off[i + 1])] for i in range(n)]
    rng = np.random.default_rng(3)
    for i in rng.integers(1, n, 800):
        docs[i] = docs[rng.integers(0, i)]
    off, tok = csr(docs)
    for n_exp, fp, wl, cap in [(50, 0.2, 10, 0), (300, 0.05, 11, 5), (20, 0.5, 10, 2048), (2000, 1e-3, 14, 0)]:
        idx = LSHBloom(64, 8, 4, n_exp, fp, 11, device=0, bloom_path="sweep", sweep_window_log2=wl, sweep_cap=cap)
        _, _, o_dup, _ = oracle.run(off, tok, num_perm=64, b=8, r=4, n_expected=n_exp, fp_rate=fp, seed=11)
        got = u8(idx.query_insert(*to_dev(off, tok)))
        assert (got == o_dup).all(), (n_exp, fp, wl, cap, np.flatnonzero(got != o_dup)[:10])


def test_sweep_all_identical_documents():
    # adversarial: every document the same -> each band's 17 positions get all records
    docs = [[1, 2, 3, 4, 5, 6, 7]] * 5000 + [[9, 9, 9, 9, 9]] * 3000
    off, tok = csr(docs)
    idx = LSHBloom(128, 16, 8, 10_000, 1e-5, 0, device=0, bloom_path="sweep")
    _, _, o_dup, _ = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=10_000, fp_rate=1e-5, seed=0)
    got = u8(idx.query_insert(*to_dev(off, tok)))
    assert (got == o_dup).all() and got.sum() == 7998


def test_sweep_blocked_variant(c1):
    cfg, off, tok, bh, dup, _ = c1
    ref = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed, blocked=True)
    o_dup = ref.query_insert(bh)
    for wl in (0, 10, 19):
        idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, index="blocked",
                       bloom_path="sweep", sweep_window_log2=wl)
        assert (u8(idx.query_insert(*to_dev(off, tok))) == o_dup).all()
        assert_filters_equal(idx, ref, (0, cfg.b - 1))


def test_sweep_band_sharded_query_insert_bands(c1):
    cfg, off, tok, bh, dup, _ = c1
    for world in (1, 3):
        hits = []
        for rank in range(world):
            h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, rank=rank,
                         world=world, bloom_path="sweep")
            owned = torch.from_numpy(np.ascontiguousarray(bh[:, h.band_lo:h.band_hi]).view(np.int64)).to(DEV)
            hits.append(u8(h.query_insert_bands(owned)))
        assert (np.maximum.reduce(hits) == dup).all()


def test_sweep_and_random_paths_agree_on_c3_shapes():
    # C3 geometry (256 perms, b=32, n_expected = 8M): both paths on the same 3000 full-text docs
    cfg = CONFIGS["C3"]
    off, tok = gen_range(cfg, 0, 3000)
    d = to_dev(off, tok)
    a = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, bloom_path="sweep")
    b = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, bloom_path="random")
    fa, fb = u8(a.query_insert(*d)), u8(b.query_insert(*d))
    assert (fa == fb).all()
    for j in (0, 31):
        assert (a.filter_words(j) == b.filter_words(j)).all()


@pytest.mark.slow
def test_sweep_pieces_beyond_4m_documents():
    # > 2^22 documents in one call: two sweeps, the second continuing the first's filters
    rng = np.random.default_rng(9)
    n = (1 << 22) + 123_457
    lens = rng.integers(1, 4, n)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    tok = rng.integers(0, 2000, int(off[-1])).astype(np.uint32)
    idx = LSHBloom(32, 4, 8, n, 1e-3, 3, device=0, bloom_path="sweep")
    _, _, o_dup, _ = oracle.run(off, tok, num_perm=32, b=4, r=8, n_expected=n, fp_rate=1e-3, seed=3)
    got = u8(idx.query_insert(*to_dev(off, tok)))
    assert (got == o_dup).all(), np.flatnonzero(got != o_dup)[:10]
    assert idx.info()["sweeps"] == 2
