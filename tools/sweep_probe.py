"""Bloom stage at C5 geometry on the sweep path, per-kernel CUDA-event timing.
Usage: python tools/sweep_probe.py [docs=4000000] [steps=3] [path=sweep] [wlog2=0]"""
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
path = sys.argv[3] if len(sys.argv) > 3 else "sweep"
wl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
off, tok = gen_range_parallel(cfg, 0, n)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
bhs = []
for s in range(steps + 1):
    h = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n, cfg.fp_rate, cfg.seed + 1000 + s, device=0)
    bhs.append(h.band_hashes(d_off, d_tok))
    h.close()
del d_tok
torch.cuda.synchronize()
idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, bloom_path=path,
               sweep_window_log2=wl)
idx.query_insert_bands(bhs[0])
res = []
for s in range(1, steps + 1):
    idx.stage_times(True)
    hits = idx.query_insert_bands(bhs[s])
    ms, cnt = idx.stage_times(False, all_stages=True)
    probes = n * cfg.b * idx.k
    res.append({"step": s, "bloom_ms": round(ms[1], 3), "sweep_finish_ms": round(ms[2], 3),
                "Gprobe_per_s": round(probes / ms[1] / 1e6, 3), "frac_64B": round(probes * 64 / ms[1] / 1e6 / 6546.2, 4),
                "flagged": int(hits.sum().item())})
print(json.dumps({"path": path, "wlog2": wl, "docs": n, "steps": res, "info_sweeps": idx.info()["sweeps"]}))
