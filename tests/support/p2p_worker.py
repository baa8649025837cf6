"""torchrun worker for tests/test_gpu_p2p.py: the band-sharded path with exchange="p2p" (torch
symmetric memory) or "nccl" on real process groups; rank 0 compares every rank's flags (gathered)
with a single-handle run of the same stream and prints PASS / FAIL."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from paper_2411_04257_b200.sharded import ShardedLSHBloom  # noqa: E402
from synthetic.corpus import CONFIGS, gen_range  # noqa: E402


def main():
    exchange = sys.argv[1] if len(sys.argv) > 1 else "p2p"
    pipeline = 262144
    if ":" in exchange:                      # "nccl:<pipeline_docs>"
        exchange, pipeline = exchange.split(":")[0], int(exchange.split(":")[1])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS["C1"]
    per = 2500
    batches = [(0, per * world), (per * world, per * world + 777 * world)]
    sx = ShardedLSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=local,
                         exchange=exchange, pipeline_docs=pipeline)
    ok = True
    ref = LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=local) if rank == 0 else None
    for a, c in batches:
        n = (c - a) // world
        off, tok = gen_range(cfg, a + rank * n, a + (rank + 1) * n)
        d_off = torch.from_numpy(off.view(np.int64)).to(dev)
        d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
        got = sx.query_insert(d_off, d_tok)
        allg = [torch.empty_like(got) for _ in range(world)]
        dist.all_gather(allg, got)
        if rank == 0:
            off_all, tok_all = gen_range(cfg, a, c)
            want = ref.query_insert(torch.from_numpy(off_all.view(np.int64)).to(dev),
                                    torch.from_numpy(tok_all.view(np.int32)).to(dev))
            ok &= bool((torch.cat(allg) == want).all().item())
    if rank == 0:
        print("PASS" if ok else "FAIL", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
