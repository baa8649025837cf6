"""Checkpoint / resume: lshbloom_save writes SPEC's LSHB / LBF1 container
 and lshbloom_load resumes the stream exactly."""
import os

import numpy as np
import pytest

import oracle
from support.lshb_format import read_lshb
from synthetic.corpus import CONFIGS, gen_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom, LSHBloomError  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(off, tok):
    return (torch.from_numpy(off.view(np.int64)).to(DEV), torch.from_numpy(tok.view(np.int32)).to(DEV))


@pytest.fixture(scope="module")
def stream():
    cfg = CONFIGS["C1"]
    off, tok = gen_range(cfg, 0, cfg.n_docs)
    sig, bh, dup, ref = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=cfg.n_docs, fp_rate=1e-4, seed=7)
    return cfg, off, tok, bh, dup, ref


def _split(off, tok, a, b):
    return off[a:b + 1] - off[a], tok[int(off[a]):int(off[b])]


def test_save_load_resume_equals_uninterrupted(stream, tmp_path):
    cfg, off, tok, bh, dup, ref = stream
    idx = LSHBloom(128, 16, 8, cfg.n_docs, 1e-4, 7, device=0)
    cut = 6123
    first = idx.query_insert(*to_dev(*_split(off, tok, 0, cut))).cpu().numpy()
    path = str(tmp_path / "index.lshb")
    idx.save(path)
    idx.close()
    res = LSHBloom.load(path, device=0)
    assert res.info()["doc_count"] == cut
    second = res.query_insert(*to_dev(*_split(off, tok, cut, cfg.n_docs))).cpu().numpy()
    assert (np.concatenate([first, second]) == dup).all()
    assert res.info()["doc_count"] == cfg.n_docs


def test_file_layout_matches_spec_and_oracle_filters(stream, tmp_path):
    cfg, off, tok, bh, dup, ref = stream
    idx = LSHBloom(128, 16, 8, cfg.n_docs, 1e-4, 7, device=0)
    idx.query_insert(*to_dev(off, tok))
    path = str(tmp_path / "index.lshb")
    idx.save(path)
    blob = open(path, "rb").read()
    hdr, filters = read_lshb(blob)
    assert hdr["magic"] == b"LSHB" and hdr["version"] == 1 and hdr["crc_ok"] and hdr["size"] == len(blob)
    assert (hdr["num_perm"], hdr["b"], hdr["r"]) == (128, 16, 8)
    assert hdr["signature_seed"] == hdr["band_hash_seed"] == 7
    assert hdr["n_docs"] == cfg.n_docs and hdr["doc_count"] == cfg.n_docs
    assert hdr["p_effective"] == pytest.approx(1 - (1 - 1e-4) ** 16, rel=1e-12)
    assert hdr["threshold"] == pytest.approx((1 / 16) ** (1 / 8))
    _, _, _, _, s1, _ = oracle.family(7, 0, 0, 16)
    for j, f in enumerate(filters):
        assert f["magic"] == b"LBF1" and f["version"] == 1 and f["crc_ok"]
        assert (f["m"], f["k"]) == (ref.m, ref.k)
        assert f["capacity_n"] == cfg.n_docs and f["target_p"] == 1e-4 and f["inserted"] == cfg.n_docs
        assert f["seed"] == int(s1[j])
        assert f["payload"] == ref.filter_bytes(j).tobytes()      # bit-exact filter state vs oracle


def test_configured_threshold_round_trips(stream, tmp_path):
    """The header's threshold field holds the T the (b, r) were chosen for when the config names
    it (SPEC LshParams), and load carries it back."""
    cfg, off, tok, bh, dup, ref = stream
    idx = LSHBloom(128, 16, 8, 2000, 1e-3, 7, device=0, lsh_threshold=0.8)
    assert idx.info()["lsh_threshold"] == 0.8
    path = str(tmp_path / "t.lshb")
    idx.save(path)
    hdr, _ = read_lshb(open(path, "rb").read())
    assert hdr["threshold"] == 0.8
    assert LSHBloom.load(path, device=0).info()["lsh_threshold"] == 0.8
    with pytest.raises(LSHBloomError):
        LSHBloom(128, 16, 8, 2000, 1e-3, 7, device=0, lsh_threshold=1.5)


def test_corrupt_truncated_and_foreign_files(stream, tmp_path):
    cfg, off, tok, bh, dup, ref = stream
    idx = LSHBloom(128, 16, 8, 2000, 1e-3, 7, device=0)
    idx.query_insert(*to_dev(*_split(off, tok, 0, 500)))
    path = str(tmp_path / "a.lshb")
    idx.save(path)
    blob = bytearray(open(path, "rb").read())
    cases = {}
    bad = bytearray(blob)
    bad[len(bad) // 2] ^= 0x10
    cases["corrupt"] = (bytes(bad), 7)
    cases["truncated"] = (bytes(blob[:len(blob) - 100]), 6)
    cases["header_only"] = (bytes(blob[:20]), 6)
    cases["magic"] = (b"XXXX" + bytes(blob[4:]), 5)
    bad = bytearray(blob)
    bad[4] = 2
    cases["version"] = (bytes(bad), 5)
    for name, (data, code) in cases.items():
        p = str(tmp_path / (name + ".lshb"))
        open(p, "wb").write(data)
        with pytest.raises(LSHBloomError) as e:
            LSHBloom.load(p, device=0)
        assert e.value.code == code, (name, e.value)
    with pytest.raises(LSHBloomError) as e:
        LSHBloom.load(str(tmp_path / "missing.lshb"), device=0)
    assert e.value.code == 8


def test_save_rejects_sharded_handles(tmp_path):
    idx = LSHBloom(128, 16, 8, 1000, 1e-3, 0, device=0, rank=0, world=2)
    with pytest.raises(LSHBloomError) as e:
        idx.save(str(tmp_path / "x.lshb"))
    assert e.value.code == 1
