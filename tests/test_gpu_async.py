"""lshbloom_query_insert_async / lshbloom_sync: batches of a stream enqueued back to back (the
next batch's MinHash overlapping the previous batch's Bloom stage) give exactly the flags of the
sequential stream -- checked against the CPU oracle for both Bloom
paths, index kinds, host and device batches, a reset between batches, and a rejected batch in the
middle of a stream."""
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


def u8(t):
    return t.cpu().numpy() if torch.is_tensor(t) else np.asarray(t)


def pieces(off, tok, cuts):
    for a, b in zip(cuts[:-1], cuts[1:]):
        yield off[a:b + 1] - off[a], tok[int(off[a]):int(off[b])]


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    _, bh, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=cfg.n_docs,
                               fp_rate=cfg.fp_rate, seed=cfg.seed)
    return cfg, off, tok, bh, dup


@pytest.mark.parametrize("path,host", [("random", False), ("sweep", False), ("random", True), ("sweep", True)])
def test_async_stream_equals_oracle(c1, path, host):
    cfg, off, tok, bh, dup = c1
    cuts = [0, 1, 700, 2000, 2001, 5000, 8000, cfg.n_docs]
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, bloom_path=path)
    outs = []
    for o, t in pieces(off, tok, cuts):
        if host:
            o = torch.from_numpy(o.view(np.int64)).pin_memory()
            t = torch.from_numpy(t.view(np.int32)).pin_memory()
            out = torch.empty(len(o) - 1, dtype=torch.uint8).pin_memory()
            outs.append(idx.query_insert_async(o, t, out=out))
        else:
            outs.append(idx.query_insert_async(*to_dev(o, t)))
    idx.sync()
    got = np.concatenate([u8(x) for x in outs])
    assert (got == dup).all(), np.flatnonzero(got != dup)[:10]
    assert idx.info()["doc_count"] == cfg.n_docs


def test_async_reset_between_batches(c1):
    cfg, off, tok, bh, dup = c1
    d = to_dev(off, tok)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    outs = []
    for _ in range(3):                       # what bench.py's steps do: zero, then the batch
        idx.reset()
        outs.append(idx.query_insert_async(*d))
    idx.sync()
    for x in outs:
        assert (u8(x) == dup).all()


def test_async_rejected_batch_mid_stream(c1):
    cfg, off, tok, bh, dup = c1
    n1, n2 = 3000, 6000
    a = (off[:n1 + 1], tok[:int(off[n1])])
    bad_off = (off[n1:n2 + 1] - off[n1]).copy()
    bad_off[10] = bad_off[9]                 # an empty document: the whole batch is rejected
    bad = (bad_off, tok[int(off[n1]):int(off[n2])])
    c = (off[n1:] - off[n1], tok[int(off[n1]):])
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    fa = idx.query_insert_async(*to_dev(*a))
    idx.query_insert_async(*to_dev(*bad))
    fc = idx.query_insert_async(*to_dev(*c))
    with pytest.raises(LSHBloomError) as e:
        idx.sync()
    assert e.value.code == 2 and "index 9" in str(e.value)
    idx.sync()                               # the error was cleared
    got = np.concatenate([u8(fa), u8(fc)])
    assert (got == dup).all()                # as if the rejected batch had never been sent
    assert idx.info()["doc_count"] == cfg.n_docs


def test_async_classic_and_blocked(c1):
    cfg, off, tok, bh, dup = c1
    cuts = [0, 4000, 4001, cfg.n_docs]
    for kind, ref in (("classic", oracle.Classic(cfg.b)),
                      ("blocked", oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed, blocked=True))):
        want = ref.query_insert(bh)
        idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, index=kind)
        outs = [idx.query_insert_async(*to_dev(o, t)) for o, t in pieces(off, tok, cuts)]
        idx.sync()
        assert (np.concatenate([u8(x) for x in outs]) == want).all(), kind


def test_async_c3_sweep_stream():
    # full-text documents at C3 geometry (sweep path), four batches in a row
    cfg = CONFIGS["C3"]
    off, tok = gen_range(cfg, 0, 4000)
    _, _, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=cfg.n_docs,
                              fp_rate=cfg.fp_rate, seed=cfg.seed)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, bloom_path="sweep")
    outs = [idx.query_insert_async(*to_dev(o, t)) for o, t in pieces(off, tok, [0, 1000, 2000, 3000, 4000])]
    idx.sync()
    assert (np.concatenate([u8(x) for x in outs]) == dup).all()
    assert idx.info()["sweeps"] == 4


def test_async_c3_host_stream_varying_sizes():
    # landing-gated host batches of very different sizes in a row (3-4 landing pieces, then one,
    # ...): each slot's landing counter restarts from zero on the copy stream before the batch's
    # K1 may read it, and batch t+1's copy runs while batch t's K1 does (Overlap)
    cfg = CONFIGS["C3"]
    off, tok = gen_range(cfg, 0, 4000)
    _, _, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=cfg.n_docs,
                              fp_rate=cfg.fp_rate, seed=cfg.seed)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    outs, keep = [], []
    for o, t in pieces(off, tok, [0, 1500, 1600, 3200, 3300, 3301, 4000]):
        o = torch.from_numpy(o.view(np.int64)).pin_memory()
        t = torch.from_numpy(t.view(np.int32)).pin_memory()
        out = torch.empty(len(o) - 1, dtype=torch.uint8).pin_memory()
        keep.append((o, t))
        outs.append(idx.query_insert_async(o, t, out=out))
    idx.sync()
    got = np.concatenate([u8(x) for x in outs])
    assert (got == dup).all(), np.flatnonzero(got != dup)[:10]
    assert dup.sum() > 0 and idx.info()["doc_count"] == 4000
