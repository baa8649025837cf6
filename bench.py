#!/usr/bin/env python3
"""bench.py -- LSHBloom hot path throughput on B200 (documents/s), BASELINE.json's metric.

Headline workload (N=1): config C3 of BASELINE.json, the largest configuration that runs on one
GPU without band sharding -- 8M full-text-like documents (lognormal(4000, 2500) words, Zipf(1.05)
over 1M ids, 8% near-duplicates), word 5-grams, num_perm=256, b=32, r=8, per-filter fp 1e-5,
filters sized for the whole corpus (n_expected = 8M: 32 x 24 MB = 767 MB, HBM-resident).  A
step = one pass of the whole hot path over one 200K-document batch of the stream: zero the
filters (a0), then lshbloom_query_insert (shingle fingerprints, MinHash, band hashes, k-probe
query-then-insert in exact stream order, duplicate flags).  N > 1 (torchrun): weak scaling,
200K documents per rank, bands sharded over ranks (paper_2411_04257_b200.sharded).

`value` is device-resident (inputs already in HBM); `e2e` is the same step through the C-ABI
with pinned HOST buffers (H2D of the CSR batch and D2H of the flags inside the timed region).
Secondary lines in the same JSON object: `secondary.C2` (1M abstracts per step, 48 MB of
L2-resident filters) and `roofline_bloom_hbm` (C5 geometry: 20 x 3.0 GB filters, 4M-document
stream batches -- the Bloom stage at its HBM-bound worst, alone and inside the fused step).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic.corpus import CONFIGS, checksum, gen_range, gen_range_parallel  # noqa: E402

METRIC = "documents/sec end-to-end at 1/2/4/8 B200; % of INT-pipe and HBM roofline"
UNIT = "docs/s"
# documents per rank per step (one batch of the config's stream)
DOCS_PER_STEP = {"C1": 10_000, "C2": 1_000_000, "C3": 200_000, "C4": 400_000, "C5": 4_000_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--docs", type=int, default=0, help="documents per rank per step (default: per config)")
    ap.add_argument("--n-expected", type=int, default=0,
                    help="index capacity n (default: the config's corpus size, BASELINE.json)")
    ap.add_argument("--sub-batch", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hbm", action="store_true", help="skip the HBM-resident Bloom leg (C5 geometry)")
    ap.add_argument("--index", default="bloom", choices=["bloom", "classic", "blocked"],
                    help="index kind: the paper's Bloom filters (default), the classic MinHashLSH "
                         "index, or the blocked Bloom variant")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: band-hash / flag exchange over peer memory (default) or NCCL")
    ap.add_argument("--hbm-docs", type=int, default=4_000_000, help="C5 leg: documents per stream batch")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary C2 line")
    ap.add_argument("--sync-steps", action="store_true",
                    help="one synchronous lshbloom_query_insert per step (default: the async stream form)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle wall time")
    a = ap.parse_args()
    if not a.docs:
        a.docs = DOCS_PER_STEP[a.config]
    if not a.n_expected:
        a.n_expected = CONFIGS[a.config].n_docs
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            if os.environ.get("LSHBLOOM_BENCH_NO_CLOCKS"):   # diagnostic: measure the sampler's own cost
                raise RuntimeError("disabled")
            ms = os.environ.get("LSHBLOOM_BENCH_CLOCK_MS", "200")
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", ms, "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- workload

def workload(cfg, rank: int, n_docs: int):
    t = time.time()
    off, tok = gen_range_parallel(cfg, rank * n_docs, (rank + 1) * n_docs)
    return off, tok, time.time() - t


def minhash_evals(off: np.ndarray, num_perm: int, n: int = 5, split_s: int = 128, prefix: int = 32):
    """(total, exact-form, screened-form) evaluations: S_d x num_perm per document, S_d =
    max(1, L_d - n + 1).  The library runs the FP32-screen kernel for 65-128 permutations and, with
    256, for documents of >= split_s shingles (lb_minhash.cu, LSHBLOOM_K1_SPLIT_S); that kernel
    evaluates each document's first `prefix` shingles exactly (LSHBLOOM_K1_PREFIX / _LPREFIX = one
    32-shingle chunk) and screens the rest.  Everything else runs the exact kernel."""
    L = np.diff(off.astype(np.int64))
    S = np.where(L >= n, L - n + 1, 1)
    total = int(S.sum()) * num_perm
    if num_perm > 128:
        scr_docs = S >= split_s
    elif num_perm > 64:
        scr_docs = np.ones(len(S), dtype=bool)
    else:
        return total, total, 0
    screened = int(np.maximum(S[scr_docs] - prefix, 0).sum()) * num_perm
    return total, total - screened, screened


# K1 bounds per evaluation (tools/micro/pipe_micro.cu, profiles/r02h_microbench.txt +
# r02j_pipe_micro_fp64.txt + r02s_fp32_screen_micro.txt): the exact form needs four 32x32->64
# products (IMAD.WIDE.U32 at 0.25 warp-instr/clk/SMSP: 16 cycles per warp-evaluation -> 2
# evaluations/clk/SMSP); the screened form (long documents, 256 permutations, lb_minhash.cu
# k1_minhash_scr4) decides almost every evaluation from two 32-bit IMAD and two FFMA, all on the
# fma pipe: IMAD 2 cycles each, the FFMA with an immediate 1, the other 2 -> 7 cycles per
# warp-evaluation = 32/7 = 4.57 evaluations/clk/SMSP (measured for that instruction pair alone:
# 4.555).  (The round-2 FP64 screen, k1_minhash_scr3, was bounded at 4 by its two DFMA.)
K1_EVALS_PER_CLK_SMSP = {"exact": 2.0, "screened": 32.0 / 7.0}


def k1_peak(evals, f_hz: float, sms: int = 148, screened: float | None = None):
    """Evaluation-weighted bound (Geval/s) of K1 for a batch split over the two kernels."""
    total, ex, sc = evals
    t = (ex / K1_EVALS_PER_CLK_SMSP["exact"] + sc / (screened or K1_EVALS_PER_CLK_SMSP["screened"])) / (sms * 4 * f_hz)
    return total / t


def load_traffic(config: str):
    path = os.path.join(ROOT, "profiles", "k1_traffic_%s.json" % config)
    try:
        with open(path) as f:
            return json.load(f).get("bytes_per_launch")
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------------------- CPU oracle timing

def oracle_sample(cfg, off, tok, n_docs_total: int, sample: int, nthreads: int):
    """Oracle (signatures + band hashes + stream-order Bloom) on the first `sample` documents."""
    import oracle
    o = off[:sample + 1]
    t = tok[:int(o[-1])]
    t0 = time.perf_counter()
    _, bh = oracle.signatures(o, t, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False,
                              nthreads=nthreads)
    idx = oracle.Index(cfg.b, n_docs_total, cfg.fp_rate, cfg.seed)
    idx.query_insert(bh, nthreads=nthreads)
    return time.perf_counter() - t0


def calibrate_sample(cfg, off, tok, n_total, nthreads, target_s):
    n0 = min(4000, len(off) - 1)
    dt = oracle_sample(cfg, off, tok, n_total, n0, nthreads)
    s = int(n0 * target_s / max(dt, 1e-3))
    return max(n0, min(s, len(off) - 1))


def run_reference(args, cfg):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    nthreads = os.cpu_count() or 1
    off, tok, _ = workload(cfg, 0, args.docs)
    # each step: a bounded sample so (warmup + steps) finishes within a few minutes
    per_step = max(2.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    sample = calibrate_sample(cfg, off, tok, args.n_expected, nthreads, per_step)
    for _ in range(args.warmup):
        oracle_sample(cfg, off, tok, args.n_expected, sample, nthreads)
    t = 0.0
    for _ in range(args.steps):
        t += oracle_sample(cfg, off, tok, args.n_expected, sample, nthreads)
    value = sample * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": "%s sample: first %d of %d docs per step" % (cfg.name, sample, args.docs),
                   "num_perm": cfg.num_perm, "b": cfg.b, "r": cfg.r, "fp_rate": cfg.fp_rate},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                         "sample": "first %d docs of %s per step (signatures, band hashes, stream-order Bloom)"
                                   % (sample, cfg.name)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- Bloom stage timing

def load_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def bloom_alone(torch, dev, make_engine, bhs, probes, peaks, peak_src, steps):
    """The Bloom stage by itself (lshbloom_query_insert_bands: binning + window sweep + verdict,
    or the random-access kernels, whichever the library picks) on freshly zeroed filters, one
    batch of band hashes per step (bhs[0] warms up).  CUDA events on the launching stream around
    each call.  Algorithmic traffic per probe = one 32-B sector read + one 32-B write-back
    (SURVEY §8d), against the measured HBM copy peak."""
    eng = make_engine()
    stream = torch.cuda.current_stream(dev)
    ms = []
    for i in range(steps + 1):
        eng.reset()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.stage_times(enable=True)
        e0.record(stream)
        eng.query_insert_bands(bhs[i % len(bhs)])
        e1.record(stream)
        torch.cuda.synchronize(dev)
        st, _ = eng.stage_times(enable=False, all_stages=True)
        if i:
            ms.append((e0.elapsed_time(e1), st[2]))
    info = eng.info()
    eng.close()
    t = statistics.median(m for m, _ in ms)
    sweep_ms = statistics.median(x for _, x in ms)
    peak = float(peaks.get("hbm_gbs", 6546.0))
    alg = probes * 64.0
    return {"bound": "hbm", "achieved": alg / t / 1e6, "peak": peak, "unit": "GB/s", "frac": alg / t / 1e6 / peak,
            "ms_per_batch": t, "sweep_kernels_ms": sweep_ms, "probes": probes, "Gprobe_per_s": probes / t / 1e6,
            "bytes_per_probe_algorithmic": 64, "path": "sweep" if info["sweeps"] else "random",
            "filter_bytes": info["filter_bytes"], "peak_source": "%s hbm_gbs (copy)" % peak_src}


def c5_leg(args, torch, dev, peaks, peak_src):
    """C5 geometry (128 perms, b=20 r=6, n_expected=1e9 -> 20 x 3.0 GB filters, m > 2^32), 4M-
    document stream batches: (a) the fused lshbloom_query_insert per batch (device-resident CSR,
    filters zeroed between steps outside the timed call), (b) the Bloom stage alone on fresh
    band hashes of the same documents under other hash seeds."""
    from paper_2411_04257_b200 import LSHBloom
    cfg = CONFIGS["C5"]
    n = args.hbm_docs
    off, tok = gen_range_parallel(cfg, 0, n)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
    steps = max(3, min(args.steps, 6))
    stream = torch.cuda.current_stream(dev)
    eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=dev.index)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    times, stages = [], []
    for i in range(2 + steps):
        eng.reset()
        torch.cuda.synchronize(dev)
        eng.stage_times(enable=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.query_insert(d_off, d_tok, out=out)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        st, _ = eng.stage_times(enable=False, all_stages=True)
        if i >= 2:
            times.append(e0.elapsed_time(e1))
            stages.append(st)
    fused_ms = statistics.median(times)
    dup_frac = float(out.float().mean().item())
    # the same batch as a stream: reset + lshbloom_query_insert_async per step, each step's MinHash
    # overlapping the previous step's Bloom stage; one event pair around all steps
    for _ in range(2):
        eng.reset()
        eng.query_insert_async(d_off, d_tok, out=out)
    eng.sync()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        eng.reset()
        eng.query_insert_async(d_off, d_tok, out=out)
    eng.sync()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    stream_ms = e0.elapsed_time(e1) / steps
    info = eng.info()
    eng.close()
    del eng
    bhs = []
    for s in range(3):
        h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n, cfg.fp_rate, cfg.seed + 1000 + s, device=dev.index)
        bhs.append(h.band_hashes(d_off, d_tok))
        h.close()
    del d_off, d_tok
    torch.cuda.empty_cache()
    probes = n * cfg.b * info["k"]
    alone = bloom_alone(torch, dev, lambda: LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed,
                                                     device=dev.index), bhs, probes, peaks, peak_src, steps)
    tr = load_json("bloom_sweep_traffic_C5.json")
    alone["traffic"] = tr["dram_bytes_per_probe"] * probes if tr else None
    alone["traffic_source"] = "profiles/bloom_sweep_traffic_C5.json (ncu, same batch shape)" if tr else None
    del bhs
    torch.cuda.empty_cache()
    return {"workload": "C5 geometry: 128 perms, b=20 r=6, n_expected=1e9 (%.1f GB of filters, m=%d > 2^32), "
                        "%d-document stream batches" % (info["filter_bytes"] / 1e9, info["m"], n),
            "stream": {"docs_per_s": n / (stream_ms / 1e3), "ms_per_batch": stream_ms, "steps": steps,
                       "timing": "CUDA events around %d async steps (reset + query_insert_async each)" % steps},
            "fused_step": {"docs_per_s": n / (fused_ms / 1e3), "ms_per_batch": fused_ms,
                           "stages_ms": {"minhash_k1": statistics.median(x[0] for x in stages),
                                         "bloom_stage_span": statistics.median(x[1] for x in stages),
                                         "sweep_kernels": statistics.median(x[2] for x in stages)},
                           "dup_frac": dup_frac, "timing": "CUDA events around each query_insert call; "
                                                           "filters zeroed between calls, untimed"},
            "bloom_alone": alone}


def secondary_c2(args, torch, dev, peaks, name="C2"):
    """C2 (1M abstract-like documents per step, 128 perms, b16 r8, n_expected = 1M: 48 MB of
    L2-resident filters) or C4 (the 8:31 full-text : abstract mixture, 400K documents per step, 256
    perms, b32 r8, n_expected = 39M: 3.74 GB of filters): the fused step, device-resident, filters
    zeroed inside each step."""
    from paper_2411_04257_b200 import LSHBloom
    cfg = CONFIGS[name]
    n = DOCS_PER_STEP[name]
    off, tok = gen_range_parallel(cfg, 0, n)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
    eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=dev.index)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    steps = max(5, min(args.steps, 20))
    for _ in range(3):
        eng.reset()
        eng.query_insert(d_off, d_tok, out=out)
    torch.cuda.synchronize(dev)
    eng.stage_times(enable=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        eng.reset()
        eng.query_insert(d_off, d_tok, out=out)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    (k1_ms, _), (k1_n, _) = eng.stage_times(enable=False)
    ms = e0.elapsed_time(e1) / steps
    evals = minhash_evals(off, cfg.num_perm, cfg.shingle_n)
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    ach = evals[0] / (k1_ms / max(1, k1_n) / 1e3)
    # K1 alone (band hashes only, the whole GPU): inside the C2 step K1 is capped at one block per
    # SM beside the random-access Bloom kernels, so its in-step rate is not the kernel's own
    eng.band_hashes(d_off, d_tok)
    eng.stage_times(enable=True)
    for _ in range(3):
        eng.band_hashes(d_off, d_tok)
    (a_ms, _), (a_n, _) = eng.stage_times(enable=False)
    alone = evals[0] / (a_ms / max(1, a_n) / 1e3) if a_n else None
    res = {"workload": ("C2: 1M abstract-like docs per step, 128 perms, b16 r8, n_expected 1M (%.0f MB of filters)"
                        if name == "C2" else
                        "C4: 400K docs per step (8 of every 39 full-text), 256 perms, b32 r8, n_expected 39M "
                        "(%.0f MB of filters)") % (eng.info()["filter_bytes"] / 1e6),
           "docs_per_s": n / (ms / 1e3), "ms_per_step": ms, "dup_frac": float(out.float().mean().item()),
           "k1_roofline": {"achieved": ach / 1e9, "peak": k1_peak(evals, f_max) / 1e9, "unit": "Geval/s",
                           "frac": ach / k1_peak(evals, f_max), "ms_per_launch": k1_ms / max(1, k1_n),
                           "note": ("in-step K1 stage (capped at one block per SM beside the random-access Bloom "
                                    "kernels)" if name == "C2" else "in-step K1 stage (beside the sweep's binning)"),
                           "alone_achieved": alone / 1e9 if alone else None,
                           "alone_frac": alone / k1_peak(evals, f_max) if alone else None,
                           "alone_ms_per_launch": a_ms / max(1, a_n) if a_n else None}}
    eng.close()
    del d_off, d_tok
    torch.cuda.empty_cache()
    return res


# --------------------------------------------------------------------------- GPU arm

def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2411_04257_b200 import LSHBloom
    from paper_2411_04257_b200.sharded import ShardedLSHBloom

    world, rank, local = dist_env()
    if world != args.gpus:
        print("warning: --gpus %d but WORLD_SIZE %d" % (args.gpus, world), file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n_total = args.docs * world
    off, tok, gen_s = workload(cfg, rank, args.docs)
    csum = checksum(off, tok)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
    evals = minhash_evals(off, cfg.num_perm, cfg.shingle_n)   # (total, exact-kernel, screened-kernel)

    if world > 1:
        sx = ShardedLSHBloom(cfg.num_perm, cfg.b, cfg.r, args.n_expected, cfg.fp_rate, cfg.seed,
                             device=local, sub_batch=args.sub_batch, exchange=args.exchange, index=args.index)
        if args.exchange == "p2p":
            try:                              # symmetric-memory rendezvous; NCCL if unavailable
                sx._p2p_buffers(args.docs * world, args.docs, dev)
            except Exception as e:            # noqa: BLE001
                print("p2p exchange unavailable (%s); using NCCL" % e, file=sys.stderr)
                sx.exchange = args.exchange = "nccl"
        eng = sx.engine
        counts = [args.docs] * world                 # fixed per-rank batches: no count all-gather
        step = lambda o, t: sx.query_insert(o, t, counts=counts)  # noqa: E731
    else:
        eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, args.n_expected, cfg.fp_rate, cfg.seed, device=local,
                       sub_batch=args.sub_batch, index=args.index)
        sx = None
        d_flags = torch.empty(args.docs, dtype=torch.uint8, device=dev)   # caller-owned output (no allocation per step)
        # a stream of batches: each step's MinHash overlaps the previous step's Bloom stage
        # (lshbloom_query_insert_async); --sync-steps times one synchronous call per step instead
        if args.sync_steps:
            step = lambda o, t: eng.query_insert(o, t, out=d_flags)  # noqa: E731
        else:
            step = lambda o, t: eng.query_insert_async(o, t, out=d_flags)  # noqa: E731

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream(dev)

    step_wall = []   # host wall time per step (diagnostic only: every call synchronises its stream)
    step_stage = []  # with LSHBLOOM_BENCH_DIAG: per-step (reset wall ms, K1 ms, Bloom ms)
    diag = bool(os.environ.get("LSHBLOOM_BENCH_DIAG"))

    def timed(fn, steps):
        step_wall.clear()
        step_stage.clear()
        gc.collect()
        gc.disable()   # a Python collection pause is not part of the GPU path
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = None
        for _ in range(steps):
            t0 = time.perf_counter()
            eng.reset()
            t1 = time.perf_counter()
            out = fn()
            step_wall.append(1e3 * (time.perf_counter() - t0))
            if diag:
                (a, b), _ = eng.stage_times(enable=True)
                step_stage.append((round(1e3 * (t1 - t0), 2), a, b))
        if world == 1:
            eng.sync()                # the batches still in flight (async steps)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        gc.enable()
        barrier()
        return e0.elapsed_time(e1), out

    def wall_summary():
        w = sorted(step_wall)
        if not w:
            return None
        out = {"min": round(w[0], 3), "median": round(w[len(w) // 2], 3), "max": round(w[-1], 3)}
        if diag:
            med = w[len(w) // 2]
            out["outliers"] = [(i, round(x, 2), [round(v, 2) for v in step_stage[i]] if i < len(step_stage) else None)
                               for i, x in enumerate(step_wall) if x > 1.3 * med]
        return out

    # ---- device-resident arm
    clk = ClockSampler(local)
    clk.start()                                       # started before warm-up: its start-up is untimed
    for _ in range(args.warmup):
        eng.reset()
        flags = step(d_off, d_tok)
    if world == 1:
        eng.sync()
    torch.cuda.synchronize(dev)
    eng.stage_times(enable=True)                      # reset accumulators, start recording
    launches0 = eng.launch_count
    clk.lines.clear()
    ms, flags = timed(lambda: step(d_off, d_tok), args.steps)
    clocks = clk.stop()
    device_step_wall = wall_summary()
    launches = eng.launch_count - launches0
    (k1_ms, bl_ms), (k1_n, bl_n) = eng.stage_times(enable=False)
    ms = max_over_ranks(ms)
    dup_frac = float(flags.float().mean().item())

    # ---- end-to-end arm: pinned host CSR in, host flags out, through the same C-ABI call
    e2e = None
    if not args.no_e2e:
        p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
        p_tok = torch.from_numpy(tok.view(np.int32)).pin_memory()
        if world > 1:
            e2e_step = lambda: sx.query_insert(p_off.to(dev, non_blocking=True),  # noqa: E731
                                               p_tok.to(dev, non_blocking=True), counts=counts).cpu()
        else:
            h_flags = torch.empty(args.docs, dtype=torch.uint8).pin_memory()
            if args.sync_steps:
                e2e_step = lambda: eng.query_insert(p_off, p_tok, out=h_flags)  # noqa: E731
            else:
                e2e_step = lambda: eng.query_insert_async(p_off, p_tok, out=h_flags)  # noqa: E731
        for _ in range(max(1, args.warmup // 2)):
            eng.reset()
            e2e_step()
        if world == 1:
            eng.sync()
        e2e_ms, _ = timed(e2e_step, args.steps)
        e2e_ms = max_over_ranks(e2e_ms)
        e2e = {"value": n_total * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(off.nbytes + tok.nbytes), "d2h_bytes_per_step": int(args.docs),
               "ms_per_step": e2e_ms / args.steps, "step_wall_ms": wall_summary()}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (K1: shingles + MinHash + band hashes)
    peaks, peak_src = load_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_evals = k1_peak(evals, f_max)
    k1_per_launch_ms = k1_ms / max(1, k1_n)
    achieved = evals[0] / (k1_per_launch_ms / 1e3) if k1_n else None
    roofline = {"bound": "alu", "achieved": achieved / 1e9 if achieved else None,
                "peak": peak_evals / 1e9, "unit": "Geval/s",
                "frac": (achieved / peak_evals) if achieved else None,
                "traffic": load_traffic(args.config),
                "kernel": "k1_minhash (fingerprints + MinHash + band hashes)",
                "peak_source": "%s sm_max_mhz %.0f x 148 SMs x 4 SMSP x evaluations/clk/SMSP of the kernel each "
                               "document runs on (exact: 2 = four IMAD.WIDE at 1/4 rate; screened, >= 1024 "
                               "shingles with 256 permutations: 32/7 = two IMAD + two FFMA on the fma pipe, 7 cycles per "
                               "warp-evaluation), "
                               "weighted by evaluations" % (peak_src, f_max / 1e6),
                "frac_of_exact_form_bound": (achieved / (2.0 * 148 * 4 * f_max)) if achieved else None,
                # a stricter reading of the screened bound: with operand reuse the 3-register FFMA also
                # issues at ~1/clk (profiles/r02v_reuse_micro_and_land.log), i.e. 6 fma-pipe cycles per
                # warp-evaluation instead of the 7 `peak` assumes
                "frac_of_6_cycle_screen_bound": (achieved / k1_peak(evals, f_max, screened=32.0 / 6.0)) if achieved else None,
                "evals_per_launch": evals[0], "evals_exact_kernel": evals[1], "evals_screened_kernel": evals[2],
                "ms_per_launch": k1_per_launch_ms,
                "share_of_step": (k1_ms / max(1, args.steps)) / (ms / args.steps)}

    # K1 alone (lshbloom_band_hashes: one launch over the batch, the whole GPU, no Bloom
    # kernels beside it) -- the kernel's own rate, next to its rate inside the overlapped step
    roofline_bloom = None
    if world == 1:
        bh_step = eng.band_hashes(d_off, d_tok)
        eng.stage_times(enable=True)
        for _ in range(3):
            eng.band_hashes(d_off, d_tok)
        (a_ms, _), (a_n, _) = eng.stage_times(enable=False)
        if a_n:
            roofline["alone_ms_per_launch"] = a_ms / a_n
            roofline["alone_achieved"] = evals[0] / (a_ms / a_n / 1e3) / 1e9
            roofline["alone_frac"] = roofline["alone_achieved"] / roofline["peak"]
        # the headline config's Bloom stage by itself (same band hashes, filters zeroed per step)
        if args.index != "classic":
            probes = args.docs * cfg.b * eng.k
            roofline_bloom = bloom_alone(
                torch, dev, lambda: LSHBloom(cfg.num_perm, cfg.b, cfg.r, args.n_expected, cfg.fp_rate, cfg.seed,
                                             device=local, index=args.index), [bh_step], probes, peaks, peak_src,
                max(3, min(args.steps, 10)))
        del bh_step

    secondary = {}
    if world == 1 and not args.no_secondary and args.config != "C2":
        secondary["C2"] = secondary_c2(args, torch, dev, peaks)
    if world == 1 and not args.no_secondary and args.config != "C4":
        secondary["C4"] = secondary_c2(args, torch, dev, peaks, "C4")

    bloom_hbm = None
    if not args.no_hbm and world == 1:
        del flags
        torch.cuda.empty_cache()
        bloom_hbm = c5_leg(args, torch, dev, peaks, peak_src)

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        nthreads = os.cpu_count() or 1
        sample = calibrate_sample(cfg, off, tok, args.n_expected, nthreads, args.cpu_seconds)
        dt = oracle_sample(cfg, off, tok, args.n_expected, sample, nthreads)
        cpu = {"value": sample / dt, "unit": UNIT, "cores": nthreads, "kind": "oracle",
               "sample": "first %d of %d docs of %s (signatures, band hashes, stream-order Bloom), %.1f s"
                         % (sample, args.docs, cfg.name, dt)}

    value = n_total * args.steps / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "%s: %d docs/rank/step, lognormal(%g,%g) words, Zipf(%g) vocab %d, "
                               "%d%% near-dups; word %d-grams" % (cfg.name, args.docs, cfg.length.mean,
                                                                    cfg.length.sd, cfg.zipf_s, cfg.vocab,
                                                                    int(cfg.dup_frac * 100), cfg.shingle_n),
                   "num_perm": cfg.num_perm, "b": cfg.b, "r": cfg.r, "fp_rate": cfg.fp_rate,
                   "n_expected": args.n_expected, "docs_per_step": n_total, "tokens_per_rank": int(len(tok)),
                   "index": args.index, "index_bytes": int(eng.info()["filter_bytes"]),
                   "parallelism": ("band-sharded x%d, %s exchange" % (world, args.exchange)) if world > 1
                                  else "single GPU",
                   "l2": "inputs %.0f MB > 126 MB L2; filters zeroed each step" % (tok.nbytes / 1e6),
                   "sub_batch": args.sub_batch or 32768, "csr_checksum_rank0": csum,
                   "dup_frac": dup_frac, "gen_s": round(gen_s, 1)},
        "roofline": roofline,
        "roofline_bloom": roofline_bloom,
        "roofline_bloom_hbm": bloom_hbm,
        "secondary": secondary,
        "step_wall_ms": device_step_wall,
        "stages_ms_per_step": {"minhash_k1": k1_ms / max(1, args.steps),
                               "bloom_stage_span": bl_ms / max(1, args.steps),
                               "note": "the Bloom stage runs on its own stream beside K1 (span, not busy time)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
