"""The peer-memory band-sharded exchange (lshbloom_band_hashes_to_peers +
lshbloom_query_insert_bands_peers).  Only one GPU is available to this build, so:
  * the store pattern (each band hash into its owner's [n_global][bl] buffer, each hit flag into
    its home rank's buffer) is checked bit-exactly with W simulated ranks on one GPU -- W handles,
    plain device buffers standing in for the peer buffers, phases run one after the other (no
    rank waits on another);
  * the torch symmetric-memory plumbing of ShardedLSHBloom(exchange="p2p") runs under torchrun
    with world size 1 against a plain handle (the multi-rank barriers are correct by
    construction and untested on hardware here)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
from synthetic.corpus import CONFIGS, gen_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_04257_b200 import LSHBloom  # noqa: E402
from paper_2411_04257_b200.sharded import band_range  # noqa: E402

DEV = torch.device("cuda:0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def to_dev(off, tok):
    return (torch.from_numpy(np.ascontiguousarray(off, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(tok, np.uint32).view(np.int32)).to(DEV))


@pytest.mark.parametrize("world,index", [(2, "bloom"), (3, "bloom"), (5, "bloom"), (16, "bloom"),
                                         (3, "classic"), (4, "blocked")])
def test_simulated_ranks_match_oracle(world, index):
    cfg = CONFIGS["C1"]
    n_total = 6000
    off, tok = gen_range(cfg, 0, n_total)
    _, bh = oracle.signatures(off, tok, cfg.num_perm, cfg.seed, b=cfg.b, r=cfg.r, want_sig=False)
    if index == "classic":
        want = oracle.Classic(cfg.b).query_insert(bh)
    else:
        want = oracle.Index(cfg.b, cfg.n_docs, cfg.fp_rate, cfg.seed, blocked=index == "blocked").query_insert(bh)
    engines = [LSHBloom(cfg.num_perm, cfg.b, cfg.r, cfg.n_docs, cfg.fp_rate, cfg.seed, device=0, rank=r,
                        world=world, index=index) for r in range(world)]
    widths = [band_range(r, world, cfg.b)[1] - band_range(r, world, cfg.b)[0] for r in range(world)]
    # two batches with uneven per-rank document counts (including a rank with none in batch 2)
    got = []
    for a, c in [(0, 4000), (4000, n_total)]:
        n = c - a
        cuts = np.linspace(a, c, world + 1).astype(int)
        if a == 4000 and world > 2:
            cuts[1] = cuts[0]                                   # rank 0 has no documents
        starts = [int(x - a) for x in cuts]
        recv = [torch.full((n * widths[o],), -1, dtype=torch.int64, device=DEV) for o in range(world)]
        flags = [torch.zeros(max(1, starts[r + 1] - starts[r]), dtype=torch.uint8, device=DEV) for r in range(world)]
        for r in range(world):                                   # phase 1: K1 -> owners' buffers
            if starts[r + 1] > starts[r]:
                o_r = off[cuts[r]:cuts[r + 1] + 1] - off[cuts[r]]
                engines[r].band_hashes_to_peers(*to_dev(o_r, tok[off[cuts[r]]:off[cuts[r + 1]]]), starts[r],
                                                [t.data_ptr() for t in recv])
        for o in range(world):                                   # the owners' buffers hold the oracle's columns
            lo, hi = band_range(o, world, cfg.b)
            assert (recv[o].view(n, hi - lo).cpu().numpy().view(np.uint64) == bh[a:c, lo:hi]).all()
        for r in range(world):                                   # phase 2: Bloom -> home ranks' flags
            engines[r].query_insert_bands_peers(recv[r].view(n, widths[r]), starts, [t.data_ptr() for t in flags])
        got.append(np.concatenate([flags[r][:starts[r + 1] - starts[r]].cpu().numpy() for r in range(world)]))
    got = np.concatenate(got)
    assert (got == want).all(), np.flatnonzero(got != want)[:10]
    assert want.sum() > 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("exchange", ["p2p", "nccl", "nccl:0", "nccl:300"])
def test_torchrun_world1_symmetric_memory(exchange):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "support", "p2p_worker.py"), exchange]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert "PASS" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]
