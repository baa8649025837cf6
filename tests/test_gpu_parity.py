"""Parity of the CUDA path (called through the C-ABI) with the CPU oracle, element by element:
signatures, band hashes and duplicate flags must be bit-identical (north_star: all work is
integer, tolerance 0).  Sizes span many warps / CTAs / sub-batches with ragged tails."""
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


def u32(t):
    return t.cpu().numpy().view(np.uint32) if torch.is_tensor(t) else t


def u64(t):
    return t.cpu().numpy().view(np.uint64) if torch.is_tensor(t) else t


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
    sig, bh, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r,
                                 n_expected=cfg.n_docs, fp_rate=cfg.fp_rate, seed=cfg.seed)
    return cfg, off, tok, sig, bh, dup


def make(cfg, n_expected=None, **kw):
    return LSHBloom(cfg.num_perm, cfg.b, cfg.r, n_expected or cfg.n_docs, cfg.fp_rate, cfg.seed,
                    device=0, **kw)


def test_c1_signatures_band_hashes_flags_device(c1):
    cfg, off, tok, sig, bh, dup = c1
    d_off, d_tok = to_dev(off, tok)
    idx = make(cfg)
    assert (u32(idx.signatures(d_off, d_tok)) == sig).all()
    assert (u64(idx.band_hashes(d_off, d_tok)) == bh).all()
    got = u8(idx.query_insert(d_off, d_tok))
    assert (got == dup).all(), np.flatnonzero(got != dup)[:10]
    assert dup.sum() > 0 and idx.info()["doc_count"] == cfg.n_docs


def test_c1_host_path_matches(c1):
    cfg, off, tok, sig, bh, dup = c1
    idx = make(cfg)
    assert (idx.signatures(off, tok) == sig).all()
    assert (idx.band_hashes(off, tok) == bh).all()
    assert (idx.query_insert(off, tok) == dup).all()


def test_c1_pinned_host_path_matches(c1):
    cfg, off, tok, sig, bh, dup = c1
    p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
    p_tok = torch.from_numpy(tok.view(np.int32)).pin_memory()
    idx = make(cfg)
    assert (u8(idx.query_insert(p_off, p_tok)) == dup).all()


@pytest.mark.parametrize("sub_batch", [1, 7, 333, 4096, 1 << 20])
def test_flags_independent_of_sub_batch(c1, sub_batch):
    cfg, off, tok, sig, bh, dup = c1
    d_off, d_tok = to_dev(off, tok)
    idx = make(cfg, sub_batch=sub_batch)
    assert (u8(idx.query_insert(d_off, d_tok)) == dup).all()


def test_flags_independent_of_call_boundaries(c1):
    cfg, off, tok, sig, bh, dup = c1
    rng = np.random.default_rng(0)
    cuts = np.unique(np.concatenate([[0, cfg.n_docs], rng.integers(1, cfg.n_docs, 12), [1, 2, 3]]))
    idx = make(cfg)
    got = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        o = off[a:b + 1] - off[a]
        t = tok[int(off[a]):int(off[b])]
        got.append(u8(idx.query_insert(*to_dev(o, t))))
    assert (np.concatenate(got) == dup).all()


def test_dense_collisions_tiny_filters():
    # tiny filters + many exact and near duplicates: dense contested positions in every sub-batch
    cfg = CONFIGS["C1"]
    n = 6000
    off, tok = gen_range(cfg, 0, n)
    docs = [tok[int(off[i]):int(off[i + 1])] for i in range(n)]
    rng = np.random.default_rng(3)
    for i in rng.integers(1, n, 800):
        docs[i] = docs[rng.integers(0, i)]
    off, tok = csr(docs)
    for n_exp, fp, sb in [(50, 0.2, 64), (300, 0.05, 1000), (20, 0.5, 6000)]:
        idx = LSHBloom(64, 8, 4, n_exp, fp, 11, device=0, sub_batch=sb)
        _, _, o_dup, _ = oracle.run(off, tok, num_perm=64, b=8, r=4, n_expected=n_exp, fp_rate=fp, seed=11)
        got = u8(idx.query_insert(*to_dev(off, tok)))
        assert (got == o_dup).all(), (n_exp, fp, sb, np.flatnonzero(got != o_dup)[:10])


@pytest.mark.parametrize("num_perm,b,r,n", [(128, 16, 8, 5), (256, 32, 8, 5), (100, 10, 9, 5),
                                            (50, 5, 10, 3), (33, 33, 1, 1), (32, 1, 32, 5),
                                            (512, 64, 8, 5), (1024, 4, 200, 7)])
def test_lsh_shapes(num_perm, b, r, n):
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, 700)
    idx = LSHBloom(num_perm, b, r, 700, 1e-3, 5, device=0, shingle_n=n)
    d = to_dev(off, tok)
    o_sig, o_bh, o_dup, _ = oracle.run(off, tok, num_perm=num_perm, b=b, r=r, n_expected=700,
                                       fp_rate=1e-3, seed=5, shingle_n=n)
    assert (u32(idx.signatures(*d)) == o_sig).all()
    assert (u64(idx.band_hashes(*d)) == o_bh).all()
    assert (u8(idx.query_insert(*d)) == o_dup).all()


def test_edge_documents():
    docs = [[7], [7], [1, 2], [1, 2, 3, 4], [1, 2, 3, 4, 5], [1, 2, 3, 4, 5], [0, 0, 0, 0, 0, 0],
            [2**32 - 1] * 9, list(range(40)), list(range(40)), [5, 4, 3, 2, 1]]
    rng = np.random.default_rng(1)
    docs.append(rng.integers(0, 2**32, 150_000, dtype=np.uint64).astype(np.uint32))  # > 1 chunk of warps
    docs.append(docs[-1].copy())
    off, tok = csr(docs)
    idx = LSHBloom(128, 16, 8, 100, 1e-5, 0, device=0)
    o_sig, o_bh, o_dup, _ = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=100, fp_rate=1e-5, seed=0)
    d = to_dev(off, tok)
    assert (u32(idx.signatures(*d)) == o_sig).all()
    assert (u64(idx.band_hashes(*d)) == o_bh).all()
    got = u8(idx.query_insert(*d))
    assert (got == o_dup).all()
    assert got[1] == 1 and got[5] == 1 and got[9] == 1 and got[-1] == 1 and got[0] == 0


def test_single_document_batches():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, 60)
    idx = make(cfg, n_expected=60)
    got = [u8(idx.query_insert(off[i:i + 2] - off[i], tok[int(off[i]):int(off[i + 1])]))[0] for i in range(60)]
    _, _, o_dup, _ = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=60, fp_rate=cfg.fp_rate, seed=0)
    assert (np.array(got) == o_dup).all()


@pytest.mark.parametrize("on_device", [True, False])
def test_empty_document_rejected_without_mutation(on_device):
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, 300)
    idx = make(cfg, n_expected=300)
    bad_off = off.copy()
    bad_off[121] = bad_off[120]                    # doc 120 becomes empty
    bad_off = np.concatenate([bad_off[:121], bad_off[121:]])
    args = to_dev(bad_off, tok) if on_device else (bad_off, tok)
    with pytest.raises(LSHBloomError) as e:
        idx.query_insert(*args)
    assert e.value.code == 2 and "index 120" in str(e.value)
    assert all((idx.filter_words(j) == 0).all() for j in range(16))   # no filter was touched
    _, _, o_dup, _ = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=300, fp_rate=cfg.fp_rate, seed=0)
    assert (u8(idx.query_insert(*to_dev(off, tok))) == o_dup).all()  # handle still usable


def test_malformed_offsets_rejected():
    idx = LSHBloom(128, 16, 8, 100, 1e-5, 0, device=0)
    off = np.array([0, 5, 3, 9], np.uint64)
    tok = np.arange(9, dtype=np.uint32)
    for args in ((off, tok), to_dev(off, tok)):
        with pytest.raises(LSHBloomError) as e:
            idx.query_insert(*args)
        assert e.value.code == 1
    off2 = np.array([1, 5, 9], np.uint64)
    with pytest.raises(LSHBloomError) as e:
        idx.query_insert(*to_dev(off2, tok))
    assert e.value.code == 1


def test_filters_match_oracle_bits_and_reset(c1):
    cfg, off, tok, sig, bh, dup = c1
    idx = make(cfg)
    idx.query_insert(*to_dev(off, tok))
    ref = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed)
    ref.query_insert(bh)
    for j in range(cfg.b):
        gpu_bytes = idx.filter_words(j).view(np.uint8)
        m = ref.m
        assert (np.unpackbits(gpu_bytes, bitorder="little")[:m] ==
                np.unpackbits(ref.filter_bytes(j), bitorder="little")[:m]).all()
        assert not np.unpackbits(gpu_bytes, bitorder="little")[m:].any()   # padding never set
    idx.reset()
    assert idx.info()["doc_count"] == 0
    assert (u8(idx.query_insert(*to_dev(off, tok))) == dup).all()


def test_info_sizing_matches_oracle():
    for n, p in [(10_000, 1e-5), (10**6, 1e-5), (10**9, 1e-5), (1, 0.5), (1000, 1e-3)]:
        idx = LSHBloom(128, 16, 8, n, p, 0, device=0, sub_batch=1024)
        inf = idx.info()
        assert (inf["m"], inf["k"]) == oracle.bloom_size(n, p)
        assert inf["words_per_band"] == 4 * ((inf["m"] + 127) // 128)   # S:314 storage, 16-B rounded
        assert inf["p_eff"] == pytest.approx(1 - (1 - p) ** 16, rel=1e-12)
        idx.close()


def test_band_sharded_handles_partition_the_flags(c1):
    # world ranks each own a band subset; OR of their per-band hits == the single-GPU flags
    cfg, off, tok, sig, bh, dup = c1
    for world in (2, 3, 16):
        hits = []
        for rank in range(world):
            idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0,
                           rank=rank, world=world)
            lo, hi = idx.band_lo, idx.band_hi
            owned = torch.from_numpy(np.ascontiguousarray(bh[:, lo:hi]).view(np.int64)).to(DEV)
            hits.append(u8(idx.query_insert_bands(owned)))
        assert (np.maximum.reduce(hits) == dup).all()


def test_query_insert_on_sharded_handle_covers_owned_bands(c1):
    cfg, off, tok, sig, bh, dup = c1
    hits = []
    for rank in range(4):
        idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0,
                       rank=rank, world=4)
        hits.append(u8(idx.query_insert(*to_dev(off, tok))))
    assert (np.maximum.reduce(hits) == dup).all()


def test_band_hashes_sharded_layout(c1):
    from paper_2411_04257_b200.sharded import band_range
    cfg, off, tok, sig, bh, dup = c1
    for world in (1, 3, 8):
        idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, rank=0, world=world)
        got = u64(idx.band_hashes_sharded(*to_dev(off, tok)))
        want = np.concatenate([np.ascontiguousarray(bh[:, lo:hi]).ravel()
                               for lo, hi in (band_range(o, world, cfg.b) for o in range(world))])
        assert (got == want).all()


def test_sharded_layer_world1_nccl(c1):
    import os
    import torch.distributed as dist
    from paper_2411_04257_b200.sharded import ShardedLSHBloom
    cfg, off, tok, sig, bh, dup = c1
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        sx = ShardedLSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
        half = 4321
        a = sx.query_insert(*to_dev(off[:half + 1], tok[:int(off[half])]))
        b = sx.query_insert(*to_dev(off[half:] - off[half], tok[int(off[half]):]))
        assert (np.concatenate([u8(a), u8(b)]) == dup).all()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("on_device", [True, False])
def test_many_chunks_short_docs(on_device):
    # many fused K1/Bloom chunks (alternating K1 streams) and, on the host path, > 1 staging chunk
    from synthetic.corpus import CorpusConfig, LengthDist
    cfg = CorpusConfig("short", 300_000, LengthDist(60, 30), 5000, 1.1, 0.1, "edit", 0.0, 0.1,
                       num_perm=64, b=8, r=8, fp_rate=1e-4)
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    _, bh, dup, _ = oracle.run(off, tok, num_perm=64, b=8, r=8, n_expected=cfg.n_docs, fp_rate=1e-4, seed=3)
    idx = LSHBloom(64, 8, 8, cfg.n_docs, 1e-4, 3, device=0, sub_batch=50_000)
    args = to_dev(off, tok) if on_device else (off, tok)
    assert (u8(idx.query_insert(*args)) == dup).all()
    assert (u64(idx.band_hashes(*args)) == bh).all()


@pytest.mark.parametrize("mode", ["exact", "screened", "hyb:0", "hyb:1", "hyb:3", "scr:2", "scr:3", "scr:4", "scr:8", "scr:10", "scr:11", "scr:4+hyb:1"])
def test_both_minhash_kernels(mode):
    # exact / screened: LSHBLOOM_K1 for every launch; hyb:k the FP64-screen kernel with a k-chunk
    # exact prefix for 128 permutations; scr:k the long-document kernel of the 256-permutation
    # split (2: integer screen, 3: FP64 screen in two passes, 4: FP64 screen in one pass; default:
    # the FP32 screen in 8-shingle groups resolved every second chunk, 10: resolved every chunk,
    # 8: in 4-shingle groups as the 128-permutation hyb batches run it unless scr:4+hyb; 11: the
    # other resolution (balanced over the lanes for 256 permutations, per lane for 128))
    # run in a subprocess: the kernel choice is read once per process from LSHBLOOM_K1
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle
from synthetic.corpus import CONFIGS, gen_range
from paper_2411_04257_b200 import LSHBloom
for name, n in (("C1", 3000), ("C3", 300)):
    cfg = CONFIGS[name]
    off, tok = gen_range(cfg, 0, n)
    sig, bh, dup, _ = oracle.run(off, tok, num_perm=cfg.num_perm, b=cfg.b, r=cfg.r, n_expected=n,
                                 fp_rate=cfg.fp_rate, seed=cfg.seed)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n, cfg.fp_rate, cfg.seed, device=0)
    d = (torch.from_numpy(off.view(np.int64)).cuda(), torch.from_numpy(tok.view(np.int32)).cuda())
    assert (idx.signatures(*d).cpu().numpy().view(np.uint32) == sig).all(), name
    assert (idx.query_insert(*d).cpu().numpy() == dup).all(), name
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root)
    if "+" in mode:   # the FP64 screen for both the long documents and 128-permutation batches
        env.update(LSHBLOOM_K1_SCR="4", LSHBLOOM_K1="hyb", LSHBLOOM_K1_PREFIX="1")
        mode = "none"
    kind, _, arg = mode.partition(":")
    if kind == "none":
        pass
    elif kind == "hyb":
        env.update(LSHBLOOM_K1="hyb", LSHBLOOM_K1_PREFIX=arg)
    elif kind == "scr":
        env.update(LSHBLOOM_K1_SCR=arg)
        env.pop("LSHBLOOM_K1", None)
    else:
        env.update(LSHBLOOM_K1=mode)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("split", ["1", "300", "100000", "300:2000", "1:1", "300:0"])
def test_length_partitioned_k1(split):
    # 256 permutations: each K1 launch is split by shingle count into an exact-kernel part and a
    # screened-kernel part (lb_minhash.cu); every threshold must give the oracle's outputs,
    # including all-long (1) and all-short (100000) partitions; subprocess because the
    # threshold is read once per process
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle
from synthetic.corpus import CONFIGS, gen_range
from paper_2411_04257_b200 import LSHBloom
for name, n in (("C4", 2000), ("C1", 1500)):
    cfg = CONFIGS[name]
    off, tok = gen_range(cfg, 0, n)
    sig, bh, dup, _ = oracle.run(off, tok, num_perm=256, b=32, r=8, n_expected=n, fp_rate=1e-4, seed=3)
    idx = LSHBloom(256, 32, 8, n, 1e-4, 3, device=0)
    d = (torch.from_numpy(off.view(np.int64)).cuda(), torch.from_numpy(tok.view(np.int32)).cuda())
    assert (idx.signatures(*d).cpu().numpy().view(np.uint32) == sig).all(), name
    assert (idx.band_hashes(off, tok) == bh).all(), name
    assert (idx.query_insert(*d).cpu().numpy() == dup).all(), name
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # "split:vlong": also the very-long class placed first (LSHBLOOM_K1_VLONG_S; 0 = off)
    split, _, vlong = split.partition(":")
    env = dict(os.environ, LSHBLOOM_K1_SPLIT_S=split, PYTHONPATH=root)
    if vlong:
        env["LSHBLOOM_K1_VLONG_S"] = vlong
    env.pop("LSHBLOOM_K1", None)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("env", [{"LSHBLOOM_K1_ALT": "0"},
                                 {"LSHBLOOM_FUSE_DOCS": "1024", "LSHBLOOM_FUSE_EDGE": "1024"},
                                 {"LSHBLOOM_FUSE_DOCS": "1500", "LSHBLOOM_FUSE_EDGE": "1100", "LSHBLOOM_K1_ALT": "1"},
                                 {"LSHBLOOM_FUSE_DOCS": "1024", "LSHBLOOM_HOST_BUFS": "3", "LSHBLOOM_HOST_MIN_DOCS": "300",
                                  "LSHBLOOM_LANDING": "0"},
                                 {"LSHBLOOM_FUSE_DOCS": "1024", "LSHBLOOM_HOST_BUFS": "2", "LSHBLOOM_HOST_MIN_DOCS": "300",
                                  "LSHBLOOM_LANDING": "0"},
                                 {"LSHBLOOM_FUSE_DOCS": "1024", "LSHBLOOM_LAND_LOG2": "18"},
                                 {"LSHBLOOM_LAND_LOG2": "18", "LSHBLOOM_BLOOM_PATH": "sweep", "LSHBLOOM_FUSE_DOCS_SWEEP": "2048"}])
def test_fused_chunking_knobs(env):
    # the fused step's K1 chunking (one or two K1 streams, chunk sizes, 2 or 3 host staging
    # buffers, the host chunk floor, landing-gated host batches with 2^18-token pieces, with
    # either Bloom path) changes only the schedule:
    # flags equal the oracle's with 128 and 256 permutations (the latter with the length-split
    # K1 and its per-stream partition scratch), device and host inputs, many chunks per call
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle
from synthetic.corpus import CONFIGS, gen_range
from paper_2411_04257_b200 import LSHBloom
for name, n, P, b, r in (("C1", 9000, 128, 16, 8), ("C4", 7000, 256, 32, 8)):
    cfg = CONFIGS[name]
    off, tok = gen_range(cfg, 0, n)
    _, bh, dup, _ = oracle.run(off, tok, num_perm=P, b=b, r=r, n_expected=n, fp_rate=1e-4, seed=5)
    assert 0 < dup.sum() < n
    d = (torch.from_numpy(off.view(np.int64)).cuda(), torch.from_numpy(tok.view(np.int32)).cuda())
    for args in (d, (off, tok)):
        idx = LSHBloom(P, b, r, n, 1e-4, 5, device=0)
        got = idx.query_insert(*args)
        got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
        assert (got == dup).all(), (name, np.flatnonzero(got != dup)[:10])
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    full = dict(os.environ, PYTHONPATH=root, **env)
    for k in ("LSHBLOOM_K1", "LSHBLOOM_K1_SPLIT_S"):
        full.pop(k, None)
    out = subprocess.run([sys.executable, "-c", code], env=full, cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_gpu_known_answers():
    """The CUDA path against the known-answer vectors of the documented conventions
    (tests/golden/conventions_kat.json, pinned to the independent micro-oracle)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "conventions_kat.json")) as f:
        kat = json.load(f)
    for row in kat["signature"]:
        off, tok = csr([row["ids"]])
        d_off, d_tok = to_dev(off, tok)
        idx = LSHBloom(row["num_perm"], row["b"], row["r"], 1000, 1e-5, row["seed"], device=0)
        assert u32(idx.signatures(d_off, d_tok))[0].tolist() == row["sig"]
        assert u64(idx.band_hashes(d_off, d_tok))[0].tolist() == [int(x, 16) for x in row["band_hashes"]]
        idx.close()
