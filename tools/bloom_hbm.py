"""Bloom stage on HBM-resident filters (C5 sizing: b=20 r=6, n_expected=1e9 -> 20 x 3.0 GB).

Band hashes come from K1 over C5's first documents; steps after the first reuse the same
documents under a different hash seed (fresh band hashes with the same duplicate structure), so
the filter keeps filling like a stream.  Reports ms per 1M-document step, probes/s and the
algorithmic bytes/s (32 B sector read per probe + 32 B write-back per newly set bit).
Usage: python tools/bloom_hbm.py [docs=1000000] [steps=4] [sub_batch,...=0] [n_expected=1e9] [bloom|blocked]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range  # noqa: E402

cfg = CONFIGS["C5"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sbs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
n_expected = int(float(sys.argv[4])) if len(sys.argv) > 4 else CONFIGS["C5"].n_docs
kind = sys.argv[5] if len(sys.argv) > 5 else "bloom"
off, tok = gen_range(cfg, 0, n)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
bhs = []
for s in range(steps + 1):
    h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n, cfg.fp_rate, cfg.seed + 1000 + s, device=0)
    bhs.append(h.band_hashes(d_off, d_tok))
    del h
torch.cuda.synchronize()
for sb in sbs:
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n_expected, cfg.fp_rate, cfg.seed, device=0, sub_batch=sb,
                   index=kind)
    info = idx.info()
    idx.query_insert_bands(bhs[0])           # warm-up (also fills a little)
    res = []
    for s in range(1, steps + 1):
        idx.stage_times(True)
        hits = idx.query_insert_bands(bhs[s])
        (_, ms), (_, cnt) = idx.stage_times(False)
        probes = n * cfg.b * idx.k
        res.append({"step": s, "ms": round(ms, 3), "Gprobe_per_s": round(probes / ms / 1e6, 3),
                    "flagged": int(hits.sum().item())})
    print(json.dumps({"index": kind, "sub_batch": sb, "filters_GB": info["filter_bytes"] / 1e9, "m": info["m"], "k": info["k"],
                      "docs": n, "probes_per_step": n * cfg.b * idx.k, "steps": res}), flush=True)
    idx.close()
    del idx
    torch.cuda.empty_cache()
