"""The band-sharded multi-GPU layer (paper_2411_04257_b200.sharded) run as world_size 2 and 3
with the gloo backend on CPU.  The per-rank compute is a stand-in engine built on the CPU
oracle (test infrastructure); what is tested is the host logic: band ownership, the
owner-major exchange layout, the all-to-all split sizes and document order, the
all-reduce(MAX) combine and the local slice -- against a single-process oracle run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2411_04257_b200.sharded import ShardedLSHBloom, band_range
from synthetic.corpus import CONFIGS, gen_range

B, R, NP, SEED, FP = 16, 8, 128, 0, 1e-4


class OracleEngine:
    """Stand-in for the CUDA engine with the same methods, computed by the oracle."""

    def __init__(self, rank, world, n_expected):
        self.band_lo, self.band_hi = band_range(rank, world, B)
        self.world = world
        self.index = oracle.Index(B, n_expected, FP, SEED)

    def band_hashes_sharded(self, offsets, tokens):
        _, bh = oracle.signatures(offsets.numpy().view(np.uint64), tokens.numpy().view(np.uint32),
                                  NP, SEED, b=B, r=R, want_sig=False, nthreads=2)
        blocks = []
        for o in range(self.world):
            lo, hi = band_range(o, self.world, B)
            blocks.append(np.ascontiguousarray(bh[:, lo:hi]).ravel())
        return torch.from_numpy(np.concatenate(blocks).view(np.int64))

    def query_insert_bands(self, bh_owned):
        dup = self.index.query_insert(bh_owned.numpy().view(np.uint64), band_lo=self.band_lo, nthreads=2)
        return torch.from_numpy(dup)

    # pipelined form (lshbloom_bands_begin / _add / _finish)
    def bands_begin(self, n_global):
        self._rows = np.full((n_global, self.band_hi - self.band_lo), -1, np.int64)
        self._seen = np.zeros(n_global, bool)

    def bands_add(self, bh_owned, doc0):
        n = bh_owned.shape[0]
        assert not self._seen[doc0:doc0 + n].any()          # every document exactly once
        self._rows[doc0:doc0 + n] = bh_owned.numpy()
        self._seen[doc0:doc0 + n] = True

    def bands_finish(self, device=None):
        assert self._seen.all()
        return self.query_insert_bands(torch.from_numpy(self._rows))

    def reset(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cuts, n_total, out_path, pipeline_docs=0, pass_counts=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["C1"]
    sx = ShardedLSHBloom(NP, B, R, n_total, FP, SEED, engine=OracleEngine(rank, world, n_total),
                         pipeline_docs=pipeline_docs)
    flags = []
    for batch in cuts:                       # several batches: filter state persists across calls
        a, b = batch[rank], batch[rank + 1]
        off, tok = gen_range(cfg, a, b)
        counts = [batch[r + 1] - batch[r] for r in range(world)] if pass_counts else None
        got = sx.query_insert(torch.from_numpy(off.view(np.int64)), torch.from_numpy(tok.view(np.int32)),
                              counts=counts)
        flags.append(got.numpy().copy())
    np.save(out_path % rank, np.concatenate(flags))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,pipeline_docs,pass_counts", [(2, 0, False), (3, 0, False), (2, 97, False),
                                                             (3, 500, False), (3, 1 << 18, False), (3, 500, True)])
def test_sharded_flags_equal_single_process_oracle(world, pipeline_docs, pass_counts, tmp_path):
    # two stream batches; each split into `world` unequal contiguous rank shards
    rng = np.random.default_rng(world)
    bounds = [0, 1400, 1401, 3000]                       # includes a one-document batch
    cuts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        if b - a < world:                                 # fewer documents than ranks: empty shards
            cuts.append([a] * world + [b])
            continue
        inner = sorted(rng.choice(np.arange(a + 1, b), world - 1, replace=False).tolist())
        cuts.append([a] + inner + [b])
    out = str(tmp_path / "flags_%d.npy")
    mp.spawn(_worker, args=(world, _free_port(), cuts, bounds[-1], out, pipeline_docs, pass_counts), nprocs=world,
             join=True)
    got = []
    per_rank = [np.load(out % r) for r in range(world)]
    # reassemble global order: batch by batch, rank by rank
    pos = [0] * world
    for batch in cuts:
        for r in range(world):
            n = batch[r + 1] - batch[r]
            got.append(per_rank[r][pos[r]:pos[r] + n])
            pos[r] += n
    got = np.concatenate(got)
    off, tok = gen_range(CONFIGS["C1"], 0, bounds[-1])
    _, _, want, _ = oracle.run(off, tok, num_perm=NP, b=B, r=R, n_expected=bounds[-1], fp_rate=FP, seed=SEED)
    assert want.sum() > 0
    assert (got == want).all()


def test_band_range_partitions_bands():
    for b in (1, 9, 16, 20, 32, 64):
        for world in range(1, min(b, 8) + 1):
            rs = [band_range(g, world, b) for g in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == b
            assert all(rs[g][1] == rs[g + 1][0] for g in range(world - 1))
            widths = [h - l for l, h in rs]
            assert max(widths) - min(widths) <= 1 and min(widths) >= 1
    assert [h - l for l, h in (band_range(g, 8, 20) for g in range(8))] == [3, 3, 3, 3, 2, 2, 2, 2]
