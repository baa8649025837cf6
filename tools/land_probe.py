"""Landing-gated host batches: the H2D copy alone (whole, and in landing pieces) against the
device-resident step and the host-batch step (synchronous calls), per landing piece size.
Usage: python tools/land_probe.py [CONFIG=C3] [DOCS=200000]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range_parallel  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
n_docs = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
off, tok = gen_range_parallel(cfg, 0, n_docs)
dev = torch.device("cuda:0")
p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
p_tok = torch.from_numpy(tok.view(np.int32)).pin_memory()
d_off = p_off.to(dev)
d_tok = p_tok.to(dev)
d_dst = torch.empty_like(d_tok)
s = torch.cuda.Stream(dev)


def ev_time(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            fn()
            e1.record(s)
        torch.cuda.synchronize(dev)
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


nb = p_tok.numel() * 4
ms = ev_time(lambda: d_dst.copy_(p_tok, non_blocking=True))
print(json.dumps({"h2d_whole_ms": round(ms, 2), "GBps": round(nb / ms / 1e6, 1), "bytes": nb}), flush=True)
for lg in (21, 23, 25):
    piece = 1 << lg

    def pieces():
        for t0 in range(0, p_tok.numel(), piece):
            d_dst[t0:t0 + piece].copy_(p_tok[t0:t0 + piece], non_blocking=True)
    ms = ev_time(pieces)
    print(json.dumps({"h2d_pieces_log2": lg, "ms": round(ms, 2), "GBps": round(nb / ms / 1e6, 1)}), flush=True)

h_out = torch.empty(n_docs, dtype=torch.uint8).pin_memory()
d_out = torch.empty(n_docs, dtype=torch.uint8, device=dev)
arms = [("device", {}, lambda e: e.query_insert(d_off, d_tok, out=d_out))]
for env in ({"LSHBLOOM_LANDING": "0"}, {"LSHBLOOM_LAND_LOG2": "21"}, {"LSHBLOOM_LAND_LOG2": "23"},
            {"LSHBLOOM_LAND_LOG2": "25"}):
    arms.append(("host " + " ".join("%s=%s" % kv for kv in env.items()), env,
                 lambda e: e.query_insert(p_off, p_tok, out=h_out)))
for name, env, fn in arms:
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    for _ in range(2):
        eng.reset()
        fn(eng)
    rows = []
    for _ in range(4):
        eng.reset()
        torch.cuda.synchronize(dev)
        eng.stage_times(True)
        t0 = time.perf_counter()
        fn(eng)
        torch.cuda.synchronize(dev)
        wall = 1e3 * (time.perf_counter() - t0)
        (k1, bl), _ = eng.stage_times(False)
        rows.append((wall, k1, bl))
    w = np.array(rows)
    print(json.dumps({"arm": name, "wall_ms": round(float(np.median(w[:, 0])), 2),
                      "k1_stage_ms": round(float(np.median(w[:, 1])), 2),
                      "bloom_stage_ms": round(float(np.median(w[:, 2])), 2)}), flush=True)
    del eng
    torch.cuda.empty_cache()
