"""Bloom stage in isolation: lshbloom_query_insert_bands over C2's band hashes (1M docs x 16
bands), timed with the library's stage events; reports ms and probes/s."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range  # noqa: E402

cfg = CONFIGS["C2"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_docs
sbs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [65536]
nexp = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [cfg.n_docs]
off, tok = gen_range(cfg, 0, n)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
base = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0)
bh = base.band_hashes(d_off, d_tok)
ref = {}
for ne, sb in [(a, b) for a in nexp for b in sbs]:
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, ne, cfg.fp_rate, cfg.seed, device=0, sub_batch=sb)
    idx.query_insert_bands(bh)
    idx.stage_times(True)
    reps = 5
    for _ in range(reps):
        idx.reset()
        hits = idx.query_insert_bands(bh)
    (_, ms), (_, cnt) = idx.stage_times(False)
    h = hits.cpu().numpy()
    ref.setdefault(ne, h)
    probes = n * cfg.b * idx.k
    print("n_expected %10d (filters %7.1f MB) sub_batch %7d: bloom %.3f ms/step  %.2f Gprobe/s  flagged %d  same=%s" % (
        ne, idx.info()["filter_bytes"] / 1e6, sb, ms / cnt, probes / (ms / cnt) / 1e6, int(h.sum()),
        bool((h == ref[ne]).all())))
