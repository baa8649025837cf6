import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle
from synthetic.corpus import CONFIGS, gen_range
from paper_2411_04257_b200 import LSHBloom
cfg = CONFIGS["C2"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
off, tok = gen_range(cfg, 0, n)
_, bh, dup, _ = oracle.run(off, tok, num_perm=128, b=16, r=8, n_expected=cfg.n_docs, fp_rate=cfg.fp_rate, seed=0)
dev = torch.device("cuda:0")
d_off = torch.from_numpy(off.view(np.int64)).to(dev); d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
for sb in [0, 1 << 20, 32768, 4096]:
    idx = LSHBloom(128, 16, 8, cfg.n_docs, cfg.fp_rate, 0, device=0, sub_batch=sb)
    g = idx.query_insert(d_off, d_tok).cpu().numpy()
    bad = np.flatnonzero(g != dup)
    print("sub_batch", sb, "mismatches", len(bad), "gpu1/oracle0", int(((g == 1) & (dup == 0)).sum()), "gpu0/oracle1", int(((g == 0) & (dup == 1)).sum()), bad[:5])
    # bands-only path on oracle band hashes
    idx2 = LSHBloom(128, 16, 8, cfg.n_docs, cfg.fp_rate, 0, device=0, sub_batch=sb)
    h = idx2.query_insert_bands(torch.from_numpy(bh.view(np.int64)).to(dev)).cpu().numpy()
    print("   bands-only mismatches", int((h != dup).sum()))
