"""C5 geometry stream timing: N async steps (reset + query_insert_async) of one 4M-document batch on
the 60 GB index, plus the synchronous per-call time and stage split.  Usage: python tools/c5_stream.py [docs] [steps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range_parallel  # noqa: E402

cfg = CONFIGS["C5"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
off, tok = gen_range_parallel(cfg, 0, n)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
out = torch.empty(n, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
res = {}
for mode in ("sync", "async"):
    for _ in range(2):
        eng.reset()
        (eng.query_insert if mode == "sync" else eng.query_insert_async)(d_off, d_tok, out=out)
    eng.sync()
    torch.cuda.synchronize()
    eng.stage_times(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        eng.reset()
        (eng.query_insert if mode == "sync" else eng.query_insert_async)(d_off, d_tok, out=out)
    eng.sync()
    e1.record(st)
    torch.cuda.synchronize()
    ms, cnt = eng.stage_times(False, all_stages=True)
    res[mode] = {"ms_per_batch": round(e0.elapsed_time(e1) / steps, 2),
                 "docs_per_s": round(n * steps / (e0.elapsed_time(e1) / 1e3)),
                 "k1_ms": round(ms[0] / max(1, cnt[0]), 2), "bloom_span_ms": round(ms[1] / max(1, cnt[1]), 2),
                 "sweep_ms": round(ms[2] / max(1, cnt[2]), 2)}
print(json.dumps({"docs": n, "steps": steps, "env": {k: v for k, v in os.environ.items() if k.startswith("LSHBLOOM")},
                  **res}))
