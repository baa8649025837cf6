"""K1 kernel choice on one workload: K1 alone (band_hashes) and the fused query_insert step, for
the kernel selected by LSHBLOOM_K1 in this process (exact / screened / scr2 / default), with a
digest of the band hashes so variants can be checked against each other.
Usage: LSHBLOOM_K1=... python tools/k1_mode_probe.py CONFIG DOCS [reps]"""
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range_parallel  # noqa: E402

name = sys.argv[1]
docs = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = CONFIGS[name]
cache = "/tmp/k1probe_%s_%d.npz" % (name, docs)
if os.path.exists(cache):
    z = np.load(cache)
    off, tok = z["off"], z["tok"]
else:
    off, tok = gen_range_parallel(cfg, 0, docs)
    np.savez(cache, off=off, tok=tok)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
L = np.diff(off.astype(np.int64))
evals = int(np.where(L >= 5, L - 4, 1).sum()) * cfg.num_perm
idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs if name != "C5" else docs * 250, cfg.fp_rate, cfg.seed, device=0)
bh = idx.band_hashes(d_off, d_tok)
idx.stage_times(True)
for _ in range(reps):
    idx.band_hashes(d_off, d_tok)
(k1, _), (n, _) = idx.stage_times(False)
out = torch.empty(docs, dtype=torch.uint8, device=dev)
for _ in range(2):
    idx.reset()
    idx.query_insert(d_off, d_tok, out=out)
torch.cuda.synchronize()
step = []
for _ in range(reps):
    idx.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx.query_insert(d_off, d_tok, out=out)
    e1.record()
    torch.cuda.synchronize()
    step.append(e0.elapsed_time(e1))
h = bh.cpu().numpy().view(np.uint64)
print(json.dumps({"config": name, "docs": docs, "mode": os.environ.get("LSHBLOOM_K1", "default"),
                  "k1_alone_ms": round(k1 / n, 3), "Geval_s_alone": round(evals / (k1 / n) / 1e6, 1),
                  "step_ms": round(float(np.median(step)), 3), "docs_per_s": round(docs / np.median(step) * 1e3),
                  "flags": int(out.sum().item()),
                  "bh_digest": hashlib.blake2b(h.tobytes(), digest_size=8).hexdigest()}), flush=True)
