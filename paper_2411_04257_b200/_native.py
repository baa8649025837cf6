"""ctypes binding of include/lshbloom.h -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``liblshbloom.so``; this module only
converts torch tensors / numpy arrays into pointers and sizes, allocates outputs with torch
(device memory, streams) and translates return codes into exceptions.  There is no CPU
fallback: if the library is missing, importing this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB_PATH = os.environ.get("LSHBLOOM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                           "liblshbloom.so")

OK, EUSAGE, EDATA, ERUNTIME, ENOMEM, EFORMAT, ETRUNC, ECHECKSUM, EIO = range(9)
NSTAGES = 3                      # LSHBLOOM_NSTAGES: K1, Bloom stage, sweep kernels
BLOOM_PATHS = {"auto": 0, "random": 1, "sweep": 2}


class LSHBloomError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("lshbloom error %d: %s" % (code, msg))
        self.code = code


class _Batch(ctypes.Structure):
    _fields_ = [("n_docs", ctypes.c_uint64), ("offsets", ctypes.c_void_p),
                ("tokens", ctypes.c_void_p), ("on_device", ctypes.c_int32),
                ("stream", ctypes.c_void_p)]


class _Config(ctypes.Structure):
    _fields_ = [("num_perm", ctypes.c_uint32), ("b", ctypes.c_uint32), ("r", ctypes.c_uint32),
                ("shingle_n", ctypes.c_uint32), ("n_expected", ctypes.c_uint64),
                ("fp_rate", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("device", ctypes.c_int32), ("rank", ctypes.c_uint32), ("world", ctypes.c_uint32),
                ("sub_batch", ctypes.c_uint32), ("index_kind", ctypes.c_uint32),
                ("bloom_path", ctypes.c_uint32), ("sweep_log2_window", ctypes.c_uint32),
                ("sweep_cap", ctypes.c_uint32), ("lsh_threshold", ctypes.c_double)]


class _Info(ctypes.Structure):
    _fields_ = [("m", ctypes.c_uint64), ("k", ctypes.c_uint32), ("num_perm", ctypes.c_uint32),
                ("b", ctypes.c_uint32), ("r", ctypes.c_uint32), ("shingle_n", ctypes.c_uint32),
                ("band_lo", ctypes.c_uint32), ("band_hi", ctypes.c_uint32),
                ("words_per_band", ctypes.c_uint64), ("filter_bytes", ctypes.c_uint64),
                ("p_eff", ctypes.c_double), ("doc_count", ctypes.c_uint64),
                ("oversubscribed", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("n_expected", ctypes.c_uint64), ("fp_rate", ctypes.c_double),
                ("index_kind", ctypes.c_uint32), ("classic_slots", ctypes.c_uint64),
                ("sweeps", ctypes.c_uint64), ("lsh_threshold", ctypes.c_double)]


class _Plan(ctypes.Structure):
    _fields_ = [("b", ctypes.c_uint32), ("r", ctypes.c_uint32), ("p", ctypes.c_double),
                ("m", ctypes.c_uint64), ("k", ctypes.c_uint32), ("total_bytes", ctypes.c_uint64)]


EXPORTS = ("lshbloom_create", "lshbloom_create_ex", "lshbloom_destroy", "lshbloom_signatures",
           "lshbloom_band_hashes", "lshbloom_band_hashes_sharded", "lshbloom_query_insert",
           "lshbloom_query_insert_bands", "lshbloom_reset", "lshbloom_filter_copy", "lshbloom_info",
           "lshbloom_stage_times", "lshbloom_save", "lshbloom_load", "lshbloom_last_error",
           "lshbloom_launch_count", "lshbloom_optimal_params", "lshbloom_plan",
           "lshbloom_band_hashes_to_peers", "lshbloom_query_insert_bands_peers", "lshbloom_query_insert_async",
           "lshbloom_sync", "lshbloom_bands_begin", "lshbloom_bands_add", "lshbloom_bands_finish")


def load_library(path: str = _LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError("liblshbloom.so not built (%s); run `python -c 'import __graft_entry__ as g; "
                          "g.build()'`" % path)
    lib = ctypes.CDLL(path)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    lib.lshbloom_create.argtypes = [u32, u32, u32, u64, ctypes.c_double, u64, ctypes.POINTER(vp)]
    lib.lshbloom_create_ex.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(vp)]
    lib.lshbloom_destroy.argtypes = [vp]
    lib.lshbloom_destroy.restype = None
    for f in ("lshbloom_signatures", "lshbloom_band_hashes", "lshbloom_band_hashes_sharded",
              "lshbloom_query_insert", "lshbloom_query_insert_async"):
        getattr(lib, f).argtypes = [vp, ctypes.POINTER(_Batch), vp]
    lib.lshbloom_sync.argtypes = [vp]
    lib.lshbloom_bands_begin.argtypes = [vp, u64]
    lib.lshbloom_bands_add.argtypes = [vp, vp, u64, u64, vp]
    lib.lshbloom_bands_finish.argtypes = [vp, vp, vp]
    lib.lshbloom_query_insert_bands.argtypes = [vp, vp, u64, i32, vp, vp]
    lib.lshbloom_reset.argtypes = [vp]
    lib.lshbloom_filter_copy.argtypes = [vp, u32, vp]
    lib.lshbloom_info.argtypes = [vp, ctypes.POINTER(_Info)]
    lib.lshbloom_stage_times.argtypes = [vp, i32, vp, vp]
    lib.lshbloom_save.argtypes = [vp, ctypes.c_char_p]
    lib.lshbloom_load.argtypes = [ctypes.c_char_p, i32, ctypes.POINTER(vp)]
    lib.lshbloom_last_error.argtypes = [vp]
    lib.lshbloom_last_error.restype = ctypes.c_char_p
    lib.lshbloom_launch_count.argtypes = [vp]
    lib.lshbloom_optimal_params.argtypes = [ctypes.c_double, u32, ctypes.c_double, ctypes.c_double,
                                            ctypes.POINTER(u32), ctypes.POINTER(u32)]
    lib.lshbloom_plan.argtypes = [u64, ctypes.c_double, ctypes.c_double, u32, ctypes.POINTER(_Plan)]
    lib.lshbloom_band_hashes_to_peers.argtypes = [vp, ctypes.POINTER(_Batch), u64, ctypes.POINTER(vp)]
    lib.lshbloom_query_insert_bands_peers.argtypes = [vp, vp, u64, ctypes.POINTER(u64), ctypes.POINTER(vp), vp]
    lib.lshbloom_launch_count.restype = u64
    for f in EXPORTS:
        if f not in ("lshbloom_destroy", "lshbloom_last_error", "lshbloom_launch_count", "lshbloom_optimal_params", "lshbloom_plan",
           "lshbloom_band_hashes_to_peers", "lshbloom_query_insert_bands_peers", "lshbloom_query_insert_async",
           "lshbloom_sync", "lshbloom_bands_begin", "lshbloom_bands_add", "lshbloom_bands_finish"):
            getattr(lib, f).restype = ctypes.c_int
    return lib


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


_INT_KINDS = "iu"


def _raw(x, kind: str, itemsize: int | None = None):
    """(pointer, on_device, keepalive) for a contiguous tensor / array of integers; `itemsize`
    (bytes per element) is enforced when given -- the library reads offsets as u64 and tokens as
    u32, so e.g. numpy's default int64 token array would otherwise be misread silently."""
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("%s must be contiguous" % kind)
        if x.dtype.is_floating_point or x.dtype.is_complex or x.dtype == __import__("torch").bool:
            raise TypeError("%s must be an integer tensor, got %s" % (kind, x.dtype))
        if itemsize is not None and x.element_size() != itemsize:
            raise TypeError("%s must have %d-byte elements, got %s" % (kind, itemsize, x.dtype))
        return x.data_ptr(), (1 if x.is_cuda else 0), x
    a = np.ascontiguousarray(x)
    if a.dtype.kind not in _INT_KINDS:
        raise TypeError("%s must be an integer array, got %s" % (kind, a.dtype))
    if itemsize is not None and a.dtype.itemsize != itemsize:
        raise TypeError("%s must have %d-byte elements, got %s" % (kind, itemsize, a.dtype))
    return a.ctypes.data, 0, a


def _check_out(out, n: int, itemsize: int, on_device: bool, kind: str = "out"):
    """A caller-supplied output: contiguous, `n` elements of `itemsize` bytes, in the batch's
    memory space."""
    if _is_torch(out):
        ok = out.is_contiguous() and out.numel() == n and out.element_size() == itemsize
        dev = out.is_cuda
    else:
        ok = isinstance(out, np.ndarray) and out.flags.c_contiguous and out.size == n and \
            out.dtype.itemsize == itemsize and out.dtype.kind in _INT_KINDS
        dev = False
    if not ok:
        raise ValueError("%s must be a contiguous buffer of %d %d-byte integers" % (kind, n, itemsize))
    if dev != on_device:
        raise ValueError("%s must live in the same memory space as the inputs" % kind)


class LSHBloom:
    """One LSHBloom index (b Bloom filters, one per band) on one GPU.

    Inputs are CSR batches: ``offsets`` (n+1, int64/uint64) and ``tokens`` (uint32/int32 word
    ids).  CUDA tensors run device-resident on torch's current stream; host arrays / CPU
    tensors are copied in and out inside the call (pinned memory enables overlap)."""

    def __init__(self, num_perm: int, b: int, r: int, n_expected: int, fp_rate: float, seed: int = 0,
                 *, shingle_n: int = 5, device: int | None = None, rank: int = 0, world: int = 1,
                 sub_batch: int = 0, index: str = "bloom", bloom_path: str = "auto", sweep_window_log2: int = 0,
                 sweep_cap: int = 0, lsh_threshold: float = 0.0, _handle=None):
        """index: "bloom" (the paper's per-band Bloom filters), "classic" (the exact
        band-equality MinHashLSH index it replaces; fp_rate is ignored) or "blocked" (a blocked
        Bloom variant: all k probes of a band hash in one 1024-bit block).
        bloom_path: "auto", "random" (K3-K6, random access per probe) or "sweep" (K7-K9, windows
        streamed through shared memory); results are identical.  sweep_window_log2 / sweep_cap
        override the sweep's window size (2^w bits, w in [10, 19]) and bin capacity.
        lsh_threshold: the Jaccard threshold the (b, r) were chosen for, recorded in checkpoints
        (0: unknown, (1/b)^(1/r) is recorded)."""
        self._lib = lib()
        kinds = {"bloom": 0, "classic": 1, "blocked": 2}
        if index not in kinds:
            raise ValueError("index must be 'bloom', 'classic' or 'blocked'")
        if device is None:
            try:
                import torch
                device = torch.cuda.current_device() if torch.cuda.is_available() else -1
            except Exception:
                device = -1
        if _handle is None:
            if bloom_path not in BLOOM_PATHS:
                raise ValueError("bloom_path must be 'auto', 'random' or 'sweep'")
            cfg = _Config(num_perm, b, r, shingle_n, n_expected, fp_rate, seed & (2**64 - 1), device,
                          rank, world, sub_batch, kinds[index], BLOOM_PATHS[bloom_path], sweep_window_log2,
                          sweep_cap, float(lsh_threshold))
            h = ctypes.c_void_p()
            rc = self._lib.lshbloom_create_ex(ctypes.byref(cfg), ctypes.byref(h))
            if rc:
                raise LSHBloomError(rc, self._lib.lshbloom_last_error(None).decode())
            _handle = h
        self._h = _handle
        inf = self.info()
        self.num_perm, self.b, self.r = inf["num_perm"], inf["b"], inf["r"]
        self.device = device
        self.m, self.k = inf["m"], inf["k"]
        self.band_lo, self.band_hi = inf["band_lo"], inf["band_hi"]
        self.index = {0: "bloom", 1: "classic", 2: "blocked"}[inf["index_kind"]]

    # ------------------------------------------------------------------ plumbing
    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.lshbloom_destroy(h)

    __del__ = close

    def _check(self, rc: int):
        if rc:
            raise LSHBloomError(rc, self._lib.lshbloom_last_error(self._h).decode())

    def _batch(self, offsets, tokens, stream):
        po, do, ko = _raw(offsets, "offsets", 8)
        pt, dt, kt = _raw(tokens, "tokens", 4)
        if do != dt:
            raise ValueError("offsets and tokens must live in the same memory space")
        n = (offsets.numel() if _is_torch(offsets) else len(ko)) - 1
        if stream is None and do:
            import torch
            stream = torch.cuda.current_stream(offsets.device).cuda_stream
        return _Batch(n, po, pt, do, stream or None), (ko, kt), n, bool(do)

    def _out(self, shape, np_dtype, torch_dtype, on_device, like):
        if on_device:
            import torch
            return torch.empty(shape, dtype=torch_dtype, device=like.device)
        return np.empty(shape, dtype=np_dtype)

    @staticmethod
    def _ptr(x):
        return x.data_ptr() if _is_torch(x) else x.ctypes.data

    # ------------------------------------------------------------------ the C-ABI calls
    def signatures(self, offsets, tokens, *, stream=None):
        """MinHash signatures [n][num_perm] uint32 (int32 when on the GPU)."""
        import_torch_dtype = _torch_dtype("int32")
        bt, keep, n, dev = self._batch(offsets, tokens, stream)
        out = self._out((n, self.num_perm), np.uint32, import_torch_dtype, dev, offsets)
        self._check(self._lib.lshbloom_signatures(self._h, ctypes.byref(bt), self._ptr(out)))
        return out

    def band_hashes(self, offsets, tokens, *, stream=None):
        """Band hashes [n][b] uint64 (int64 when on the GPU) for all bands."""
        bt, keep, n, dev = self._batch(offsets, tokens, stream)
        out = self._out((n, self.b), np.uint64, _torch_dtype("int64"), dev, offsets)
        self._check(self._lib.lshbloom_band_hashes(self._h, ctypes.byref(bt), self._ptr(out)))
        return out

    def band_hashes_sharded(self, offsets, tokens, *, stream=None):
        """Band hashes of all bands in owner-major blocks (flat, n*b entries) for the all-to-all."""
        bt, keep, n, dev = self._batch(offsets, tokens, stream)
        out = self._out((n * self.b,), np.uint64, _torch_dtype("int64"), dev, offsets)
        self._check(self._lib.lshbloom_band_hashes_sharded(self._h, ctypes.byref(bt), self._ptr(out)))
        return out

    def stage_times(self, enable: bool = True, all_stages: bool = False):
        """(K1 ms, Bloom ms), (K1 launches, Bloom stages) since the last read; resets them.
        all_stages: also the sweep kernels' ms / count (third entries)."""
        ms = (ctypes.c_double * NSTAGES)()
        nn = (ctypes.c_uint64 * NSTAGES)()
        self._check(self._lib.lshbloom_stage_times(self._h, 1 if enable else 0, ms, nn))
        if all_stages:
            return tuple(ms), tuple(nn)
        return (ms[0], ms[1]), (nn[0], nn[1])

    def query_insert(self, offsets, tokens, *, out=None, stream=None):
        """Duplicate flags [n] uint8, stream order; mutates the filters."""
        bt, keep, n, dev = self._batch(offsets, tokens, stream)
        if out is None:
            out = self._out((n,), np.uint8, _torch_dtype("uint8"), dev, offsets)
        else:
            _check_out(out, n, 1, dev)
        self._check(self._lib.lshbloom_query_insert(self._h, ctypes.byref(bt), self._ptr(out)))
        return out

    def query_insert_async(self, offsets, tokens, *, out=None, stream=None):
        """Enqueue a batch (lshbloom_query_insert_async): returns its flag buffer at once; the
        flags are valid after sync().  The inputs and the returned buffer are kept alive until
        then."""
        bt, keep, n, dev = self._batch(offsets, tokens, stream)
        if out is None:
            out = self._out((n,), np.uint8, _torch_dtype("uint8"), dev, offsets)
        else:
            _check_out(out, n, 1, dev)
        self._check(self._lib.lshbloom_query_insert_async(self._h, ctypes.byref(bt), self._ptr(out)))
        self._inflight = (getattr(self, "_inflight", []) + [(keep, out)])[-2:]
        return out

    def sync(self):
        """Wait for the async batches; raises the first device-side error among them."""
        try:
            self._check(self._lib.lshbloom_sync(self._h))
        finally:
            self._inflight = []

    def query_insert_bands(self, bh_owned, *, out=None, stream=None):
        """Bloom stage only: bh_owned [n][band_hi-band_lo] -> hit flags [n] (OR over owned bands)."""
        p, dev, keep = _raw(bh_owned, "bh_owned", 8)
        if tuple(bh_owned.shape) != (bh_owned.shape[0], self.band_hi - self.band_lo):
            raise ValueError("bh_owned must be [n][%d] (the owned bands)" % (self.band_hi - self.band_lo))
        n = bh_owned.shape[0]
        if out is None:
            out = self._out((n,), np.uint8, _torch_dtype("uint8"), dev, bh_owned)
        else:
            _check_out(out, n, 1, bool(dev))
        if stream is None and dev:
            import torch
            stream = torch.cuda.current_stream(bh_owned.device).cuda_stream
        self._check(self._lib.lshbloom_query_insert_bands(self._h, p, n, dev, stream or None,
                                                          self._ptr(out)))
        return out

    def bands_begin(self, n_global: int):
        """Start a batch of n_global documents assembled from band-hash chunks."""
        self._check(self._lib.lshbloom_bands_begin(self._h, int(n_global)))
        self._bands_n = int(n_global)

    def bands_add(self, bh_owned, doc0: int, *, stream=None):
        """Add bh_owned [n][band_hi - band_lo] (device) for global documents [doc0, doc0 + n)."""
        p, dev, keep = _raw(bh_owned, "bh_owned", 8)
        if not dev:
            raise ValueError("bh_owned must be a device tensor")
        n = bh_owned.shape[0]
        if n and tuple(bh_owned.shape) != (n, self.band_hi - self.band_lo):
            raise ValueError("bh_owned must be [n][%d]" % (self.band_hi - self.band_lo))
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(bh_owned.device).cuda_stream
        self._check(self._lib.lshbloom_bands_add(self._h, p, int(doc0), n, stream or None))

    def bands_finish(self, *, out=None, device=None, stream=None):
        """Hit flags [n_global] (uint8, device) of the assembled batch; mutates the filters."""
        import torch
        n = self._bands_n
        if out is None:
            out = torch.empty(n, dtype=torch.uint8, device=device if device is not None else "cuda:%d" % self.device)
        else:
            _check_out(out, n, 1, True)
        if stream is None:
            stream = torch.cuda.current_stream(out.device).cuda_stream
        self._check(self._lib.lshbloom_bands_finish(self._h, out.data_ptr(), stream or None))
        return out

    def band_hashes_to_peers(self, offsets, tokens, global_doc0: int, peer_recv, *, stream=None):
        """K1 over this rank's documents with every band hash stored straight into its owner
        rank's receive buffer (peer_recv: `world` device pointers, e.g. symmetric memory)."""
        bt, keep, n, dev = self._batch(offsets, tokens, stream)
        ptrs = (ctypes.c_void_p * len(peer_recv))(*[int(x) for x in peer_recv])
        self._check(self._lib.lshbloom_band_hashes_to_peers(self._h, ctypes.byref(bt), int(global_doc0), ptrs))

    def query_insert_bands_peers(self, bh_owned, doc_start, peer_flags, *, stream=None):
        """Bloom stage of the owned bands for all documents of the global batch, raising each hit
        document's flag in its home rank's buffer (peer_flags: `world` device pointers)."""
        p, dev, keep = _raw(bh_owned, "bh_owned", 8)
        if not dev:
            raise ValueError("bh_owned must be a device tensor")
        n = int(doc_start[-1])
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(bh_owned.device).cuda_stream
        starts = (ctypes.c_uint64 * len(doc_start))(*[int(x) for x in doc_start])
        ptrs = (ctypes.c_void_p * len(peer_flags))(*[int(x) for x in peer_flags])
        self._check(self._lib.lshbloom_query_insert_bands_peers(self._h, p, n, starts, ptrs, stream or None))

    def save(self, path: str):
        """Checkpoint the filters and document count (SPEC's LSHB / LBF1 container)."""
        self._check(self._lib.lshbloom_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, device: int | None = None) -> "LSHBloom":
        """Resume an index saved with save(); the stream continues where it stopped."""
        if device is None:
            try:
                import torch
                device = torch.cuda.current_device() if torch.cuda.is_available() else -1
            except Exception:
                device = -1
        l = lib()
        h = ctypes.c_void_p()
        rc = l.lshbloom_load(os.fsencode(path), device, ctypes.byref(h))
        if rc:
            raise LSHBloomError(rc, l.lshbloom_last_error(None).decode())
        return cls(0, 0, 0, 0, 0.0, device=device, _handle=h)

    def reset(self):
        self._check(self._lib.lshbloom_reset(self._h))

    def filter_words(self, j: int) -> np.ndarray:
        out = np.empty(self.info()["words_per_band"], np.uint32)
        self._check(self._lib.lshbloom_filter_copy(self._h, j, out.ctypes.data))
        return out

    def info(self) -> dict:
        inf = _Info()
        self._check(self._lib.lshbloom_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in _Info._fields_}

    @property
    def launch_count(self) -> int:
        return int(self._lib.lshbloom_launch_count(self._h))


def _torch_dtype(name: str):
    import torch
    return getattr(torch, name)


def optimal_params(threshold: float, num_perm: int, fp_weight: float = 0.5, fn_weight: float = 0.5):
    """(b, r) minimising the weighted S-curve error areas (lshbloom_optimal_params; host-only)."""
    b, r = ctypes.c_uint32(), ctypes.c_uint32()
    L = lib()
    rc = L.lshbloom_optimal_params(threshold, num_perm, fp_weight, fn_weight, ctypes.byref(b), ctypes.byref(r))
    if rc:
        raise LSHBloomError(rc, L.lshbloom_last_error(None).decode())
    return int(b.value), int(r.value)


def plan(n_docs: int, p_effective: float, threshold: float = 0.8, num_perm: int = 128) -> dict:
    """Capacity plan of an index (lshbloom_plan; host-only): b, r, per-filter p, m, k, total bytes."""
    out = _Plan()
    L = lib()
    rc = L.lshbloom_plan(int(n_docs), p_effective, threshold, num_perm, ctypes.byref(out))
    if rc:
        raise LSHBloomError(rc, L.lshbloom_last_error(None).decode())
    return {f: getattr(out, f) for f, _ in _Plan._fields_}
