"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): C1 prefix with
tiny filters (dense collisions) and several sub-batches, device and host paths, both K1 kernels."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range  # noqa: E402

cfg = CONFIGS["C1"]
off, tok = gen_range(cfg, 0, 1500)
d_off = torch.from_numpy(off.view(np.int64)).cuda()
d_tok = torch.from_numpy(tok.view(np.int32)).cuda()
for (np_, b, r) in ((128, 16, 8), (256, 32, 8)):
    _, bh, dup, _ = oracle.run(off, tok, num_perm=np_, b=b, r=r, n_expected=300, fp_rate=0.01, seed=1)
    idx = LSHBloom(np_, b, r, 300, 0.01, 1, device=0, sub_batch=500)
    assert (idx.query_insert(d_off, d_tok).cpu().numpy() == dup).all()
    idx.reset()
    assert (idx.query_insert(off, tok) == dup).all()
    assert (idx.band_hashes(d_off, d_tok).cpu().numpy().view(np.uint64) == bh).all()
    idx.signatures(d_off, d_tok)
torch.cuda.synchronize()
print("sanitize run ok")
