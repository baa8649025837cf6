#!/usr/bin/env python3
"""bench.py -- LSHBloom hot path throughput on B200 (documents/s), BASELINE.json's metric.

Workload (N=1): config C2 of BASELINE.json -- 1M abstract-like documents (lognormal(200, 80)
words, Zipf(1.1) over 200k ids, 10% near-duplicates at Jaccard 0.7-0.99), word 5-grams,
num_perm=128, b=16, r=8, per-filter fp 1e-5, seed 0.  A step = one pass of the whole hot path
over the 1M-document batch: zero the filters (a0), then lshbloom_query_insert (shingle
fingerprints, MinHash, band hashes, k-probe query-then-insert in exact stream order,
duplicate flags).  N > 1 (torchrun): weak scaling, 1M documents per rank, bands sharded over
ranks with one NCCL all-to-all + one all-reduce(max) per step (paper_2411_04257_b200.sharded).

`value` is device-resident (inputs already in HBM); `e2e` is the same step through the C-ABI
with pinned HOST buffers (H2D of the CSR batch and D2H of the flags inside the timed region).
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
    ap.add_argument("--hbm-docs", type=int, default=1_000_000)
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


def minhash_evals(off: np.ndarray, num_perm: int, n: int = 5) -> int:
    L = np.diff(off.astype(np.int64))
    S = np.where(L >= n, L - n + 1, 1)
    return int(S.sum()) * num_perm


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


# --------------------------------------------------------------------------- HBM-resident Bloom leg

def hbm_leg(args, torch, dev, peaks, peak_src):
    """The Bloom stage where it is HBM-bound: C5's index geometry (128 perms, b=20 r=6,
    n_expected=1e9 -> 20 x 3.0 GB filters, m > 2^32) over C5's first documents, one fused
    lshbloom_query_insert per step on freshly zeroed filters (every probe sets a new bit: the
    stage's worst case).  Timed with CUDA events around the call; the library's stage events
    give the Bloom (K3-K6) time.  Algorithmic traffic per probe = one 32-B sector read + one
    32-B sector write-back; B200 moves a whole 128-B line per random access, which
    the measured random-access peak (tools/micro/rand_sector.cu) reflects."""
    cfg = CONFIGS["C5"]
    n = args.hbm_docs
    off, tok = gen_range(cfg, 0, n)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
    res = hbm_run(args, torch, dev, peaks, peak_src, cfg, d_off, d_tok, "bloom")
    # the blocked variant: one 128-B line per (document, band)
    res["blocked_variant"] = hbm_run(args, torch, dev, peaks, peak_src, cfg, d_off, d_tok, "blocked")
    del d_off, d_tok
    torch.cuda.empty_cache()
    return res


def hbm_traffic(index, probes):
    """DRAM bytes per step (read + write) of the standard filter's Bloom stage from the committed
    ncu capture (profiles/bloom_hbm_traffic_C5.json, per probe x probes per step): a random probe
    moves a whole 128-B line for K3's read and again for K4's atomic."""
    if index != "bloom":
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "bloom_hbm_traffic_C5.json")) as f:
            return json.load(f)["dram_bytes_per_probe"] * probes
    except Exception:
        return None


def hbm_run(args, torch, dev, peaks, peak_src, cfg, d_off, d_tok, index):
    from paper_2411_04257_b200 import LSHBloom
    n = d_off.numel() - 1
    eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=dev.index, index=index)
    stream = torch.cuda.current_stream(dev)
    steps, warm = max(3, min(args.steps, 10)), 2
    tot = 0.0
    for i in range(warm + steps):
        eng.reset()
        if i == warm:
            eng.stage_times(enable=True)
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        flags = eng.query_insert(d_off, d_tok)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= warm:
            tot += e0.elapsed_time(e1)
    (k1_ms, bl_ms), (k1_n, bl_n) = eng.stage_times(enable=False)
    info = eng.info()
    probes = n * cfg.b * eng.k
    bl_step = bl_ms / max(1, bl_n)
    # standard: a 32-B sector read + write-back per probe; blocked: one 128-B line read +
    # write-back per (document, band), i.e. 256 / k bytes per probe
    bpp = 64.0 if index == "bloom" else 256.0 / eng.k
    alg_bytes = probes * bpp
    peak = float(peaks.get("hbm_gbs", 6546.0))
    res = {"bound": "hbm", "index": index,
           "workload": "C5 geometry (128 perms, b=20 r=6, n_expected=1e9, %.1f GB filters), "
                       "first %d C5 documents per step, fresh filters" % (info["filter_bytes"] / 1e9, n),
           "docs_per_s": n * steps / (tot / 1e3), "ms_per_step": tot / steps,
           "bloom_ms_per_step": bl_step, "probes_per_step": probes,
           "Gprobe_per_s": probes / bl_step / 1e6,
           "achieved": alg_bytes / bl_step / 1e6, "peak": peak, "unit": "GB/s", "frac": alg_bytes / bl_step / 1e6 / peak,
           "peak_source": "%s hbm_gbs" % peak_src,
           "bytes_per_probe_algorithmic": round(bpp, 3),
           "traffic": hbm_traffic(index, probes),
           "dup_frac": float(flags.float().mean().item())}
    eng.close()
    del eng
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
    evals = minhash_evals(off, cfg.num_perm, cfg.shingle_n)

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
        step = lambda o, t: sx.query_insert(o, t)  # noqa: E731
    else:
        eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, args.n_expected, cfg.fp_rate, cfg.seed, device=local,
                       sub_batch=args.sub_batch, index=args.index)
        sx = None
        d_flags = torch.empty(args.docs, dtype=torch.uint8, device=dev)   # caller-owned output (no allocation per step)
        step = lambda o, t: eng.query_insert(o, t, out=d_flags)  # noqa: E731

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
                                               p_tok.to(dev, non_blocking=True)).cpu()
        else:
            h_flags = torch.empty(args.docs, dtype=torch.uint8).pin_memory()
            e2e_step = lambda: eng.query_insert(p_off, p_tok, out=h_flags)  # noqa: E731
        for _ in range(max(1, args.warmup // 2)):
            eng.reset()
            e2e_step()
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
    # 4 IMAD.WIDE.U32 per (a x + b) mod P evaluation (two 61-bit operands -> four 32x32->64
    # partial products); IMAD.WIDE issues at 0.25 warp-inst/clk/SMSP on sm_100a (fmaheavy,
    # tools/micro/pipe_micro.cu) -> 2 evaluations / clk / SMSP.
    peak_evals = 2.0 * 148 * 4 * f_max
    k1_per_launch_ms = k1_ms / max(1, k1_n)
    achieved = evals / (k1_per_launch_ms / 1e3) if k1_n else None
    roofline = {"bound": "alu", "achieved": achieved / 1e9 if achieved else None,
                "peak": peak_evals / 1e9, "unit": "Geval/s",
                "frac": (achieved / peak_evals) if achieved else None,
                "traffic": load_traffic(args.config),
                "kernel": "k1_minhash (fingerprints + MinHash + band hashes)",
                "peak_source": "%s sm_max_mhz %.0f x 148 SMs x 4 SMSP x 2 evals/clk (fmaheavy IMAD.WIDE bound)"
                               % (peak_src, f_max / 1e6),
                "evals_per_launch": evals, "ms_per_launch": k1_per_launch_ms,
                "share_of_step": (k1_ms / max(1, args.steps)) / (ms / args.steps)}

    # K1 alone (lshbloom_band_hashes: one launch over the batch, the whole GPU, no Bloom
    # kernels beside it) -- the kernel's own rate, next to its rate inside the overlapped step
    if world == 1:
        eng.band_hashes(d_off, d_tok)
        eng.stage_times(enable=True)
        for _ in range(3):
            eng.band_hashes(d_off, d_tok)
        (a_ms, _), (a_n, _) = eng.stage_times(enable=False)
        if a_n:
            roofline["alone_ms_per_launch"] = a_ms / a_n
            roofline["alone_achieved"] = evals / (a_ms / a_n / 1e3) / 1e9
            roofline["alone_frac"] = roofline["alone_achieved"] / roofline["peak"]

    bloom_hbm = None
    if not args.no_hbm and world == 1:
        del flags
        bloom_hbm = hbm_leg(args, torch, dev, peaks, peak_src)

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
        "roofline_bloom_hbm": bloom_hbm,
        "step_wall_ms": device_step_wall,
        "stages_ms_per_step": {"minhash_k1": k1_ms / max(1, args.steps), "bloom_k3_k6": bl_ms / max(1, args.steps)},
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
