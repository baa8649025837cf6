"""K1 rate on one corpus for several (num_perm, kernel) choices: band_hashes timed with the
library's stage events.  Usage: python tools/k1_perm_split.py CONFIG DOCS"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
n = int(sys.argv[2])
off, tok = gen_range(cfg, 0, n)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
L = np.diff(off.astype(np.int64))
S = int(np.where(L >= 5, L - 4, 1).sum())
for num_perm in (128, 256):
    idx = LSHBloom(num_perm, 16, 8, n, 1e-5, 0, device=0)
    idx.band_hashes(d_off, d_tok)
    idx.stage_times(True)
    for _ in range(3):
        idx.band_hashes(d_off, d_tok)
    (ms, _), (cnt, _) = idx.stage_times(False)
    print(json.dumps({"config": cfg.name, "num_perm": num_perm, "kernel": os.environ.get("LSHBLOOM_K1", "auto"),
                      "ms": ms / cnt, "Geval_s": S * num_perm / (ms / cnt) / 1e6}), flush=True)
