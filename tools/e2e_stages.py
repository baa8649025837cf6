"""Where the end-to-end (host-buffer) step spends its time versus the device-resident one:
per-step wall time and the library's K1 / Bloom stage times for both arms.
Usage: python tools/e2e_stages.py [CONFIG=C2] [DOCS]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n_docs = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_docs
off, tok = gen_range(cfg, 0, n_docs)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
p_tok = torch.from_numpy(tok.view(np.int32)).pin_memory()
eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, n_docs, cfg.fp_rate, cfg.seed, device=0)
d_out = torch.empty(n_docs, dtype=torch.uint8, device=dev)
h_out = torch.empty(n_docs, dtype=torch.uint8).pin_memory()
for name, fn in (("device", lambda: eng.query_insert(d_off, d_tok, out=d_out)),
                 ("host", lambda: eng.query_insert(p_off, p_tok, out=h_out))):
    for _ in range(3):
        eng.reset()
        fn()
    rows = []
    for _ in range(4):
        eng.reset()
        eng.stage_times(True)
        t0 = time.perf_counter()
        fn()
        wall = 1e3 * (time.perf_counter() - t0)
        (k1, bl), _ = eng.stage_times(False)
        rows.append((wall, k1, bl))
    w = np.array(rows)
    print(json.dumps({"arm": name, "wall_ms": round(float(np.median(w[:, 0])), 3),
                      "k1_stage_ms": round(float(np.median(w[:, 1])), 3),
                      "bloom_stage_ms": round(float(np.median(w[:, 2])), 3)}), flush=True)
