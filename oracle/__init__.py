"""CPU oracle for the LSHBloom hot path (arXiv 2411.04257).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2411_04257_b200``) never imports it and
shares no code with it; see ``oracle/lshbloom_oracle.c`` for the algorithm,
written out in the paper's order with citations (PAPER.md = "P:line",
SPEC.md = "S:line").

This module is argument marshalling (numpy <-> C) plus building the plain C
file with gcc.  Every oracle function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_pins.py`` against values the paper/SPEC print, closed forms,
brute force on tiny inputs or statistical fixed points.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lshbloom_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None

P61 = (1 << 61) - 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2; no vectorisation pragmas)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build())
        u64, u32, i32, dbl, vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_void_p)
        lib.orc_mix64.restype = u64
        lib.orc_mix64.argtypes = [u64]
        lib.orc_R.restype = u64
        lib.orc_R.argtypes = [u64, u64, u64]
        lib.orc_bloom_size.restype = i32
        lib.orc_bloom_size.argtypes = [u64, dbl, ctypes.POINTER(u64), ctypes.POINTER(u32)]
        lib.orc_family.restype = None
        lib.orc_family.argtypes = [u64, u32, u32, u32, vp, vp, vp, vp, vp, vp]
        lib.orc_fingerprint.restype = u64
        lib.orc_fingerprint.argtypes = [vp, u32]
        lib.orc_signature_doc.restype = None
        lib.orc_signature_doc.argtypes = [vp, u64, u32, vp, vp, u32, vp]
        lib.orc_band_hash.restype = u64
        lib.orc_band_hash.argtypes = [vp, u32, u32, vp, vp]
        lib.orc_probes.restype = None
        lib.orc_probes.argtypes = [u64, u64, u64, u64, u32, vp]
        lib.orc_signatures.restype = i32
        lib.orc_signatures.argtypes = [u64, vp, vp, u32, u32, u32, u32, u64, i32, vp, vp,
                                       ctypes.POINTER(u64)]
        lib.orc_index_new.restype = vp
        lib.orc_index_new.argtypes = [u32, u64, dbl, u64]
        lib.orc_index_new2.restype = vp
        lib.orc_index_new2.argtypes = [u32, u64, dbl, u64, i32]
        lib.orc_probes_blocked.restype = None
        lib.orc_probes_blocked.argtypes = [u64, u64, u64, u64, u32, vp]
        lib.orc_index_free.restype = None
        lib.orc_index_free.argtypes = [vp]
        lib.orc_index_m.restype = u64
        lib.orc_index_m.argtypes = [vp]
        lib.orc_index_k.restype = u32
        lib.orc_index_k.argtypes = [vp]
        lib.orc_index_doc_count.restype = u64
        lib.orc_index_doc_count.argtypes = [vp]
        lib.orc_index_bits.restype = vp
        lib.orc_index_bits.argtypes = [vp, u32]
        lib.orc_index_query_insert.restype = i32
        lib.orc_index_query_insert.argtypes = [vp, u64, vp, u32, u32, i32, vp, vp]
        lib.orc_classic_new.restype = vp
        lib.orc_classic_new.argtypes = [u32]
        lib.orc_classic_free.restype = None
        lib.orc_classic_free.argtypes = [vp]
        lib.orc_classic_keys.restype = u64
        lib.orc_classic_keys.argtypes = [vp, u32]
        lib.orc_classic_query_insert.restype = i32
        lib.orc_classic_query_insert.argtypes = [vp, u64, vp, u32, u32, vp, vp]
        lib.orc_optimal_params.restype = i32
        lib.orc_optimal_params.argtypes = [dbl, u32, dbl, dbl, ctypes.POINTER(u32), ctypes.POINTER(u32)]
        _lib = lib
        return lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# --------------------------------------------------------------------------- scalars

def mix64(z: int) -> int:
    return int(_load().orc_mix64(z & (2**64 - 1)))


def counter(seed: int, dom: int, i: int) -> int:
    return int(_load().orc_R(seed & (2**64 - 1), dom, i))


def bloom_size(n: int, p: float) -> tuple[int, int]:
    """(m bits, k probes), P:224-225 / S:263.  Raises ValueError on bad input."""
    m = ctypes.c_uint64()
    k = ctypes.c_uint32()
    if _load().orc_bloom_size(n, p, ctypes.byref(m), ctypes.byref(k)):
        raise ValueError("bloom_size: need n >= 1 and 0 < p < 1")
    return int(m.value), int(k.value)


def family(seed: int, num_perm: int, r: int, b: int):
    """(a, b, c, d, s1, s2) as uint64 arrays (DESIGN R5)."""
    a = np.zeros(max(num_perm, 1), np.uint64)
    bb = np.zeros(max(num_perm, 1), np.uint64)
    c = np.zeros(max(r, 1), np.uint64)
    d = np.zeros(max(r, 1), np.uint64)
    s1 = np.zeros(max(b, 1), np.uint64)
    s2 = np.zeros(max(b, 1), np.uint64)
    _load().orc_family(seed & (2**64 - 1), num_perm, r, b, _ptr(a), _ptr(bb), _ptr(c), _ptr(d),
                       _ptr(s1), _ptr(s2))
    return a[:num_perm], bb[:num_perm], c[:r], d[:r], s1[:b], s2[:b]


def fingerprint(ids) -> int:
    w = np.ascontiguousarray(ids, dtype=np.uint32)
    return int(_load().orc_fingerprint(_ptr(w), len(w)))


def signature_doc(ids, num_perm: int, seed: int, shingle_n: int = 5) -> np.ndarray:
    w = np.ascontiguousarray(ids, dtype=np.uint32)
    if len(w) == 0:
        raise ValueError("empty document")
    a, bb, *_ = family(seed, num_perm, 0, 0)
    sig = np.zeros(num_perm, np.uint32)
    _load().orc_signature_doc(_ptr(w), len(w), shingle_n, _ptr(a), _ptr(bb), num_perm, _ptr(sig))
    return sig


def band_hash(sig, j: int, r: int, seed: int) -> int:
    s = np.ascontiguousarray(sig, dtype=np.uint32)
    _, _, c, d, _, _ = family(seed, 0, r, 0)
    return int(_load().orc_band_hash(_ptr(s), j, r, _ptr(c), _ptr(d)))


def probes(bh: int, s1: int, s2: int, m: int, k: int) -> np.ndarray:
    g = np.zeros(k, np.uint64)
    _load().orc_probes(bh, s1, s2, m, k, _ptr(g))
    return g


def probes_blocked(bh: int, s1: int, s2: int, nb: int, k: int) -> np.ndarray:
    """Blocked variant: k positions inside one 1024-bit block."""
    g = np.zeros(k, np.uint64)
    _load().orc_probes_blocked(bh, s1, s2, nb, k, _ptr(g))
    return g


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def signatures(offsets, tokens, num_perm: int, seed: int, *, b: int = 0, r: int = 0,
               shingle_n: int = 5, nthreads: int | None = None, want_sig: bool = True,
               want_bh: bool = True):
    """Signatures [n][num_perm] u32 and band hashes [n][b] u64 for a CSR batch."""
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    tok = np.ascontiguousarray(tokens, dtype=np.uint32)
    n = len(off) - 1
    sig = np.zeros((n, num_perm), np.uint32) if want_sig else None
    bh = np.zeros((n, b), np.uint64) if (want_bh and b) else None
    bad = ctypes.c_uint64(0)
    rc = _load().orc_signatures(n, _ptr(off), _ptr(tok) if len(tok) else 0, num_perm, shingle_n,
                                b, r, seed & (2**64 - 1), nthreads or default_threads(),
                                _ptr(sig) if sig is not None else 0,
                                _ptr(bh) if bh is not None else 0, ctypes.byref(bad))
    if rc == 2:
        raise OracleError(2, "empty document at index %d" % bad.value)
    if rc:
        raise OracleError(rc, "usage error")
    return sig, bh


class Index:
    """The LSHBloom index of b Bloom filters, stream-order semantics."""

    def __init__(self, b: int, n_expected: int, fp_rate: float, seed: int, blocked: bool = False):
        self._lib = _load()
        self._h = self._lib.orc_index_new2(b, n_expected, fp_rate, seed & (2**64 - 1), 1 if blocked else 0)
        self.blocked = blocked
        if not self._h:
            raise ValueError("orc_index_new: bad parameters")
        self.b = b

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.orc_index_free(h)

    @property
    def m(self) -> int:
        return int(self._lib.orc_index_m(self._h))

    @property
    def k(self) -> int:
        return int(self._lib.orc_index_k(self._h))

    @property
    def doc_count(self) -> int:
        return int(self._lib.orc_index_doc_count(self._h))

    def filter_bytes(self, j: int) -> np.ndarray:
        n = (self.m + 7) // 8
        buf = (ctypes.c_uint8 * n).from_address(self._lib.orc_index_bits(self._h, j))
        return np.frombuffer(buf, dtype=np.uint8).copy()

    def query_insert(self, bh, *, band_lo: int = 0, nthreads: int | None = None,
                     want_hits: bool = False):
        arr = np.ascontiguousarray(bh, dtype=np.uint64)
        n, ncol = arr.shape
        dup = np.zeros(n, np.uint8)
        hits = np.zeros((n, ncol), np.uint8) if want_hits else None
        rc = self._lib.orc_index_query_insert(self._h, n, _ptr(arr), band_lo, ncol,
                                              nthreads or default_threads(), _ptr(dup),
                                              _ptr(hits) if hits is not None else 0)
        if rc:
            raise OracleError(rc, "usage error")
        return (dup, hits) if want_hits else dup


def run(offsets, tokens, *, num_perm: int, b: int, r: int, n_expected: int, fp_rate: float,
        seed: int, shingle_n: int = 5, index: Index | None = None, nthreads: int | None = None):
    """Whole hot path: signatures, band hashes, stream-order flags."""
    sig, bh = signatures(offsets, tokens, num_perm, seed, b=b, r=r, shingle_n=shingle_n,
                         nthreads=nthreads)
    idx = index if index is not None else Index(b, n_expected, fp_rate, seed)
    dup = idx.query_insert(bh, nthreads=nthreads)
    return sig, bh, dup, idx


class Classic:
    """The classic MinHashLSH index (P:134 exact band equality): per band the set of
    band hashes seen; a document is a duplicate iff some band hash of it was seen before."""

    def __init__(self, b: int):
        self._lib = _load()
        self._h = self._lib.orc_classic_new(b)
        if not self._h:
            raise ValueError("orc_classic_new: b must be >= 1")
        self.b = b

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.orc_classic_free(h)

    def keys(self, j: int) -> int:
        """Distinct band-hash values stored for band j."""
        return int(self._lib.orc_classic_keys(self._h, j))

    def query_insert(self, bh, *, band_lo: int = 0, want_hits: bool = False):
        arr = np.ascontiguousarray(bh, dtype=np.uint64)
        n, ncol = arr.shape
        dup = np.zeros(n, np.uint8)
        hits = np.zeros((n, ncol), np.uint8) if want_hits else None
        rc = self._lib.orc_classic_query_insert(self._h, n, _ptr(arr), band_lo, ncol, _ptr(dup),
                                                _ptr(hits) if hits is not None else 0)
        if rc:
            raise OracleError(rc, "usage error")
        return (dup, hits) if want_hits else dup


def optimal_params(threshold: float, num_perm: int, fp_weight: float = 0.5,
                   fn_weight: float = 0.5) -> tuple[int, int]:
    """(b, r) minimising the weighted FP/FN areas of the LSH S-curve."""
    b = ctypes.c_uint32()
    r = ctypes.c_uint32()
    if _load().orc_optimal_params(threshold, num_perm, fp_weight, fn_weight, ctypes.byref(b), ctypes.byref(r)):
        raise ValueError("optimal_params: need 0 < threshold <= 1 and num_perm >= 2")
    return int(b.value), int(r.value)


def plan(n_docs: int, p_effective: float, threshold: float, num_perm: int) -> dict:
    """Capacity plan (Tables 1-2): b from optimal_params, per-filter p from
    p_effective = 1 - (1 - p)^b, m and k per filter, total = b * ceil(m / 8) bytes."""
    b, r = optimal_params(threshold, num_perm)
    p = -np.expm1(np.log1p(-p_effective) / b)
    m, k = bloom_size(int(n_docs), float(p))
    return {"b": b, "r": r, "p": float(p), "m": m, "k": k, "total_bytes": b * ((m + 7) // 8)}
