"""Seeded synthetic corpora shaped like BASELINE.json's configs C1-C5.

This module is the ONE piece shared by the CUDA path's tests/bench and the CPU
oracle: it produces inputs only and holds none of the method's arithmetic (no
shingling, MinHash, band hashing or Bloom logic).  Its random numbers come from
Murmur3's fmix64 finaliser in counter mode -- a different mixer from the
SplitMix64 finaliser the method itself uses -- so any document is a pure
function of (corpus seed, document index) and a 1B-document stream can be
generated batch by batch.

Recipe (after SURVEY.md §8(d)):
  * length  L = max(1, round(exp(mu + sigma Z))), sigma^2 = ln(1 + sd^2/mean^2),
    mu = ln(mean) - sigma^2/2, Z standard normal (Box-Muller);
  * tokens  Zipf(s) over ranks 1..V, id = rank - 1 (Walker/Vose alias table);
  * near-duplicates: doc d >= 1 is a near-dup with probability q; its source is
    uniform over [0, d) (resolved recursively if the source is itself a near-dup);
    the copy keeps the source's length and each position is independently
    replaced by a fresh Zipf token with probability e.  e ~ U(e_lo, e_hi)
    ("edit" mode) or, for a target Jaccard J ~ U(J_lo, J_hi) over word 5-grams,
    e = 1 - (2J/(1+J))^(1/5) ("jaccard" mode);
  * C4's mixture: 8 of every 39 documents (evenly interleaved) are full-text-like.
"""
from __future__ import annotations

import dataclasses
import functools
import hashlib
import math

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_C1 = np.uint64(0xFF51AFD7ED558CCD)
_C2 = np.uint64(0xC4CEB9FE1A85EC53)
_K_STREAM = np.uint64(0x9E6C63D0676A9A99)
_K_DOC = np.uint64(0xD6E8FEB86659FD93)
_K_POS = np.uint64(0xC2B2AE3D27D4EB4F)
_K_ADD = np.uint64(0x165667B19E3779F9)
_S33 = np.uint64(33)

STREAM_LEN, STREAM_DUP, STREAM_TOK, STREAM_EDIT, STREAM_EDTOK = 1, 2, 3, 4, 5


def fmix64(z: np.ndarray) -> np.ndarray:
    """Murmur3 64-bit finaliser, elementwise on uint64 (wrapping)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> _S33)
        z = z * _C1
        z = z ^ (z >> _S33)
        z = z * _C2
        z = z ^ (z >> _S33)
    return z


def _doc_keys(seed: int, stream: int, docs: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = fmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (_K_STREAM * np.uint64(stream + 1)))
        return fmix64(base ^ (np.asarray(docs, np.uint64) * _K_DOC + np.uint64(1)))


def _rand(keys: np.ndarray, pos) -> np.ndarray:
    with np.errstate(over="ignore"):
        return fmix64(keys + np.asarray(pos, np.uint64) * _K_POS + _K_ADD)


def _unif53(u: np.ndarray) -> np.ndarray:
    """Uniform in (0, 1) from the top 53 bits."""
    return ((u >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


@functools.lru_cache(maxsize=8)
def zipf_alias(vocab: int, s: float):
    """Vose alias table for P(rank) ~ rank^-s, rank = 1..vocab."""
    w = np.arange(1, vocab + 1, dtype=np.float64) ** (-s)
    p = w * (vocab / w.sum())
    prob = np.zeros(vocab, np.float64)
    alias = np.zeros(vocab, np.int64)
    small = [i for i in range(vocab) if p[i] < 1.0]
    large = [i for i in range(vocab) if p[i] >= 1.0]
    p = p.tolist()
    while small and large:
        l, g = small.pop(), large.pop()
        prob[l] = p[l]
        alias[l] = g
        p[g] = (p[g] + p[l]) - 1.0
        (small if p[g] < 1.0 else large).append(g)
    for i in large + small:
        prob[i] = 1.0
        alias[i] = i
    # acceptance threshold as a 32-bit integer so the draw is integer-exact
    thr = np.minimum(np.floor(prob * 4294967296.0), 4294967296.0).astype(np.uint64)
    return thr, alias.astype(np.uint32)


def _zipf_tokens(u: np.ndarray, vocab: int, s: float) -> np.ndarray:
    thr, alias = zipf_alias(vocab, s)
    idx = ((u >> np.uint64(32)) * np.uint64(vocab)) >> np.uint64(32)
    keep = (u & np.uint64(0xFFFFFFFF)) < thr[idx]
    return np.where(keep, idx.astype(np.uint32), alias[idx])


@dataclasses.dataclass(frozen=True)
class LengthDist:
    mean: float
    sd: float

    @property
    def sigma(self) -> float:
        return math.sqrt(math.log(1.0 + (self.sd / self.mean) ** 2))

    @property
    def mu(self) -> float:
        return math.log(self.mean) - self.sigma ** 2 / 2.0


@dataclasses.dataclass(frozen=True)
class CorpusConfig:
    name: str
    n_docs: int
    length: LengthDist
    vocab: int
    zipf_s: float
    dup_frac: float
    dup_mode: str            # "edit" or "jaccard"
    dup_lo: float
    dup_hi: float
    # LSH / filter parameters of the config (consumed by tests/bench, not here)
    num_perm: int = 128
    b: int = 16
    r: int = 8
    fp_rate: float = 1e-5
    seed: int = 0            # hash-family seed
    corpus_seed: int = 0
    shingle_n: int = 5
    long_length: LengthDist | None = None   # C4 mixture: full-text class
    long_per: tuple[int, int] | None = None  # (8, 39): 8 of every 39 docs are full-text
    batch_docs: int = 0      # C5: stream batch size

    def with_docs(self, n: int) -> "CorpusConfig":
        return dataclasses.replace(self, n_docs=n)


CONFIGS = {
    "C1": CorpusConfig("C1", 10_000, LengthDist(150, 60), 50_000, 1.1, 0.05, "edit", 0.05, 0.15,
                       num_perm=128, b=16, r=8),
    "C2": CorpusConfig("C2", 1_000_000, LengthDist(200, 80), 200_000, 1.1, 0.10, "jaccard", 0.7,
                       0.99, num_perm=128, b=16, r=8),
    "C3": CorpusConfig("C3", 8_000_000, LengthDist(4000, 2500), 1_000_000, 1.05, 0.08, "edit", 0.01,
                       0.20, num_perm=256, b=32, r=8),
    "C4": CorpusConfig("C4", 39_000_000, LengthDist(200, 80), 1_000_000, 1.05, 0.10, "edit", 0.01,
                       0.20, num_perm=256, b=32, r=8, long_length=LengthDist(4000, 2500),
                       long_per=(8, 39)),
    "C5": CorpusConfig("C5", 1_000_000_000, LengthDist(200, 80), 1_000_000, 1.1, 0.10, "jaccard", 0.7,
                       0.99, num_perm=128, b=20, r=6, batch_docs=4_000_000),
}


def _is_long(cfg: CorpusConfig, docs: np.ndarray) -> np.ndarray:
    if cfg.long_per is None:
        return np.zeros(len(docs), bool)
    a, c = cfg.long_per
    d = docs.astype(np.int64)
    return ((d + 1) * a) // c > (d * a) // c


def base_lengths(cfg: CorpusConfig, docs: np.ndarray) -> np.ndarray:
    keys = _doc_keys(cfg.corpus_seed, STREAM_LEN, docs)
    u1 = _unif53(_rand(keys, 0))
    u2 = _unif53(_rand(keys, 1))
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    mu = np.full(len(docs), cfg.length.mu)
    sg = np.full(len(docs), cfg.length.sigma)
    if cfg.long_length is not None:
        lg = _is_long(cfg, docs)
        mu[lg] = cfg.long_length.mu
        sg[lg] = cfg.long_length.sigma
    return np.maximum(1, np.rint(np.exp(mu + sg * z))).astype(np.int64)


def dup_params(cfg: CorpusConfig, docs: np.ndarray):
    """(is_dup, source, edit_rate) per doc."""
    docs = np.asarray(docs, np.int64)
    keys = _doc_keys(cfg.corpus_seed, STREAM_DUP, docs)
    is_dup = (_unif53(_rand(keys, 0)) < cfg.dup_frac) & (docs >= 1)
    src = np.floor(_unif53(_rand(keys, 1)) * docs).astype(np.int64)
    src = np.minimum(src, np.maximum(docs - 1, 0))
    v = cfg.dup_lo + (cfg.dup_hi - cfg.dup_lo) * _unif53(_rand(keys, 2))
    if cfg.dup_mode == "jaccard":
        e = 1.0 - (2.0 * v / (1.0 + v)) ** (1.0 / cfg.shingle_n)
    else:
        e = v
    return is_dup, np.where(is_dup, src, -1), e


def _expand(docs: np.ndarray, lengths: np.ndarray):
    """Flattened (doc index into `docs`, position) for CSR token generation."""
    owner = np.repeat(np.arange(len(docs)), lengths)
    starts = np.zeros(len(docs) + 1, np.int64)
    np.cumsum(lengths, out=starts[1:])
    pos = np.arange(starts[-1], dtype=np.int64) - starts[owner]
    return owner, pos, starts


def gen_docs(cfg: CorpusConfig, docs: np.ndarray):
    """Generate the documents with the given (sorted, unique) indices.

    Returns (offsets u64[n+1], tokens u32[...]) in the order of `docs`."""
    docs = np.asarray(docs, np.int64)
    if len(docs) == 0:
        return np.zeros(1, np.uint64), np.zeros(0, np.uint32)
    is_dup, src, e = dup_params(cfg, docs)
    lengths = base_lengths(cfg, docs)
    if is_dup.any():
        need = np.unique(src[is_dup])
        s_off, s_tok = gen_docs(cfg, need)
        s_len = np.diff(s_off.astype(np.int64))
        where = np.searchsorted(need, src[is_dup])
        lengths[is_dup] = s_len[where]
    owner, pos, starts = _expand(docs, lengths)
    tokens = np.empty(starts[-1], np.uint32)
    # fresh documents: i.i.d. Zipf tokens
    fresh_tok = ~is_dup[owner]
    if fresh_tok.any():
        keys = _doc_keys(cfg.corpus_seed, STREAM_TOK, docs)
        u = _rand(keys[owner[fresh_tok]], pos[fresh_tok])
        tokens[fresh_tok] = _zipf_tokens(u, cfg.vocab, cfg.zipf_s)
    # near-duplicates: copy the source, replace each position w.p. e
    dup_tok = ~fresh_tok
    if dup_tok.any():
        o = owner[dup_tok]
        p = pos[dup_tok]
        srow = np.searchsorted(need, src[o])
        copied = s_tok[s_off[srow].astype(np.int64) + p]
        ekeys = _doc_keys(cfg.corpus_seed, STREAM_EDIT, docs)
        ue = _unif53(_rand(ekeys[o], p))
        edit = ue < e[o]
        tkeys = _doc_keys(cfg.corpus_seed, STREAM_EDTOK, docs)
        fresh = _zipf_tokens(_rand(tkeys[o[edit]], p[edit]), cfg.vocab, cfg.zipf_s)
        copied[edit] = fresh
        tokens[dup_tok] = copied
    return starts.astype(np.uint64), tokens


def gen_range(cfg: CorpusConfig, start: int, stop: int, chunk: int = 65536):
    """CSR for documents [start, stop), generated in chunks to bound memory."""
    offs = [np.zeros(1, np.uint64)]
    toks = []
    base = 0
    for c0 in range(start, stop, chunk):
        o, t = gen_docs(cfg, np.arange(c0, min(stop, c0 + chunk)))
        offs.append(o[1:] + np.uint64(base))
        toks.append(t)
        base += len(t)
    return np.concatenate(offs), (np.concatenate(toks) if toks else np.zeros(0, np.uint32))


def _gen_chunk(args):
    cfg, c0, c1 = args
    return gen_docs(cfg, np.arange(c0, c1))


def gen_range_parallel(cfg: CorpusConfig, start: int, stop: int, workers: int | None = None,
                       chunk: int = 0):
    """gen_range over a process pool (chunks are independent: every document is a pure function
    of (corpus seed, index)).  Byte-identical to gen_range; used for the multi-GB C3-C5 batches."""
    import multiprocessing as mp
    import os
    workers = workers or min(32, os.cpu_count() or 1)
    chunk = chunk or max(2048, min(65536, (stop - start) // (4 * workers) + 1))
    jobs = [(cfg, c0, min(stop, c0 + chunk)) for c0 in range(start, stop, chunk)]
    if workers <= 1 or len(jobs) <= 1:
        return gen_range(cfg, start, stop, chunk)
    with mp.get_context("fork").Pool(min(workers, len(jobs))) as pool:
        parts = pool.map(_gen_chunk, jobs, chunksize=1)
    lens = [len(t) for _, t in parts]
    total = int(sum(lens))
    offsets = np.empty(stop - start + 1, np.uint64)
    offsets[0] = 0
    tokens = np.empty(total, np.uint32)
    base, d = 0, 0
    for o, t in parts:
        n = len(o) - 1
        offsets[d + 1:d + 1 + n] = o[1:] + np.uint64(base)
        tokens[base:base + len(t)] = t
        base += len(t)
        d += n
    return offsets, tokens


def checksum(offsets: np.ndarray, tokens: np.ndarray) -> str:
    """64-bit digest of a CSR batch, logged so GPU and oracle provably read the same bytes."""
    h = hashlib.blake2b(digest_size=8)
    h.update(np.ascontiguousarray(offsets, np.uint64).tobytes())
    h.update(np.ascontiguousarray(tokens, np.uint32).tobytes())
    return h.hexdigest()


def planted_pairs(cfg: CorpusConfig, start: int, stop: int):
    """(doc, source, edit_rate) for every planted near-duplicate in [start, stop)."""
    docs = np.arange(start, stop)
    is_dup, src, e = dup_params(cfg, docs)
    return docs[is_dup], src[is_dup], e[is_dup]
