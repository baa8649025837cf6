"""K1 design exploration: build liblshbloom variants (-D flags) and time K1 on the C2 corpus.

  python tools/k1_variants.py build NAME=FLAGS ...     (here; nvcc cross-compiles)
  python tools/k1_variants.py run [docs]               (on the GPU box; one subprocess per variant)
"""
import glob
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "tools", "variants")


def build(specs):
    from paper_2411_04257_b200 import build as b
    os.makedirs(VDIR, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = os.path.join(VDIR, "lib_%s.so" % name)
        cmd = [b.NVCC, *b.FLAGS, *flags.split(), "-o", out, *b.sources()]
        subprocess.check_call(cmd)
        print("built", out, flags)


def one(path, docs, reps, config="C2"):
    import numpy as np
    import torch
    os.environ["LSHBLOOM_LIB"] = path
    from paper_2411_04257_b200 import LSHBloom
    from synthetic.corpus import CONFIGS, gen_range
    cfg = CONFIGS[config]
    cache = "/tmp/%s_%d.npz" % (config, docs)
    if os.path.exists(cache):
        z = np.load(cache)
        off, tok = z["off"], z["tok"]
    else:
        off, tok = gen_range(cfg, 0, docs)
        np.savez(cache, off=off, tok=tok)
    dev = torch.device("cuda:0")
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
    idx = LSHBloom(cfg.num_perm, cfg.b, cfg.r, docs, cfg.fp_rate, cfg.seed, device=0)
    bh = idx.band_hashes(d_off, d_tok)
    idx.stage_times(True)
    for _ in range(reps):
        idx.band_hashes(d_off, d_tok)
    (k1, _), (n, _) = idx.stage_times(False)
    L = np.diff(off.astype(np.int64))
    evals = int(np.where(L >= 5, L - 4, 1).sum()) * cfg.num_perm
    h = bh.cpu().numpy().view(np.uint64)
    import hashlib
    return {"k1_ms": k1 / n, "Geval_s": evals / (k1 / n) / 1e6, "bh_digest": hashlib.blake2b(h.tobytes(), digest_size=8).hexdigest()}


def run(docs, reps=10):
    res = {}
    for path in sorted(glob.glob(os.path.join(VDIR, "lib_*.so"))):
        name = os.path.basename(path)[4:-3]
        out = subprocess.run([sys.executable, __file__, "one", path, str(docs), str(reps)], capture_output=True, text=True)
        try:
            res[name] = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            res[name] = {"error": (out.stdout + out.stderr)[-500:]}
        print(name, res[name], flush=True)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    elif sys.argv[1] == "one":
        print(json.dumps(one(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]),
                             sys.argv[5] if len(sys.argv) > 5 else "C2")))
    else:
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000)
