"""K1 alone (lshbloom_band_hashes) on a config's documents: ms per launch and Geval/s.
Usage: python tools/k1_probe.py [config=C3] [docs=200000] [reps=3]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range_parallel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = CONFIGS[name]
off, tok = gen_range_parallel(cfg, 0, n)
L = np.diff(off.astype(np.int64))
evals = int(np.where(L >= 5, L - 4, 1).sum()) * cfg.num_perm
d_off = torch.from_numpy(off.view(np.int64)).cuda()
d_tok = torch.from_numpy(tok.view(np.int32)).cuda()
eng = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
eng.band_hashes(d_off, d_tok)
eng.stage_times(True)
for _ in range(reps):
    bh = eng.band_hashes(d_off, d_tok)
(ms, _), (cnt, _) = eng.stage_times(False)
t = ms / max(1, cnt)
print(json.dumps({"config": name, "docs": n, "evals": evals, "ms": round(t, 3), "Geval_per_s": round(evals / t / 1e6, 1),
                  "checksum": int(bh.cpu().numpy().view(np.uint64)[:, 0].astype(np.uint64).sum() % (1 << 61)),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("LSHBLOOM")}}))
