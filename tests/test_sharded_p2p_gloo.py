"""The peer-memory exchange of the band-sharded layer (ShardedLSHBloom(exchange="p2p")) run as
world_size 2 and 3 with gloo on CPU.  torch's symmetric memory is replaced by a stand-in whose
"peer pointers" name files in /dev/shm that every rank maps (so one rank's stores land in another
rank's buffer, as over NVLink), and the CUDA engine by an oracle-backed stand-in with the same
two methods.  What is tested is the host logic of the p2p path: document ranges and global
offsets, receive-buffer shapes per owner, the three barriers, the flag slices -- against a
single-process oracle run over several batches."""
import os
import socket
import sys
import types
import uuid

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2411_04257_b200.sharded import ShardedLSHBloom, band_range
from synthetic.corpus import CONFIGS, gen_range

B, R, NP, SEED, FP = 16, 8, 128, 0, 1e-4


class _FakeSymm:
    """Symmetric memory stand-in: every allocation is a shared file per rank; buffer_ptrs are
    ids (allocation number, rank) that the engine stand-in maps back to those files."""

    def __init__(self, prefix, rank, world):
        self.prefix, self.rank, self.world, self.k = prefix, rank, world, 0
        self.sizes = {}

    def path(self, k, r):
        return "/dev/shm/%s_%d_%d" % (self.prefix, k, r)

    def empty(self, n, dtype, device=None):
        k = self.k
        self.k += 1
        t = torch.from_file(self.path(k, self.rank), shared=True, size=n, dtype=dtype)
        t.zero_()
        t._fake_k = k
        self.sizes[k] = (n, dtype)
        return t

    def rendezvous(self, t, group):
        k = t._fake_k
        h = types.SimpleNamespace()
        h.buffer_ptrs = [(k << 8) | r for r in range(self.world)]
        h.barrier = lambda channel=0: dist.barrier()
        dist.barrier()                                    # every rank has created its file
        return h

    def open(self, ptr):
        k, r = ptr >> 8, ptr & 0xFF
        n, dtype = self.sizes[k]
        return torch.from_file(self.path(k, r), shared=True, size=n, dtype=dtype)


class OracleP2PEngine:
    def __init__(self, rank, world, n_expected, symm):
        self.band_lo, self.band_hi = band_range(rank, world, B)
        self.world, self.symm = world, symm
        self.index = oracle.Index(B, n_expected, FP, SEED)

    def band_hashes_to_peers(self, offsets, tokens, global_doc0, peer_recv):
        _, bh = oracle.signatures(offsets.numpy().view(np.uint64), tokens.numpy().view(np.uint32),
                                  NP, SEED, b=B, r=R, want_sig=False, nthreads=2)
        n = bh.shape[0]
        for o in range(self.world):                       # store into each owner's buffer
            lo, hi = band_range(o, self.world, B)
            dst = self.symm.open(peer_recv[o]).numpy().view(np.uint64)
            w = hi - lo
            dst[global_doc0 * w:(global_doc0 + n) * w] = np.ascontiguousarray(bh[:, lo:hi]).ravel()

    def query_insert_bands_peers(self, recv, doc_start, peer_flags):
        hits = self.index.query_insert(recv.numpy().view(np.uint64), band_lo=self.band_lo, nthreads=2)
        for r in range(self.world):                       # raise flags at their home ranks
            a, c = doc_start[r], doc_start[r + 1]
            if c > a:
                f = self.symm.open(peer_flags[r]).numpy()
                f[:c - a] |= hits[a:c]

    def reset(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cuts, n_total, out_path, prefix):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    symm = _FakeSymm(prefix, rank, world)
    fake = types.ModuleType("torch.distributed._symmetric_memory")
    fake.empty, fake.rendezvous = symm.empty, symm.rendezvous
    sys.modules["torch.distributed._symmetric_memory"] = fake
    torch.distributed._symmetric_memory = fake
    cfg = CONFIGS["C1"]
    sx = ShardedLSHBloom(NP, B, R, n_total, FP, SEED, exchange="p2p",
                         engine=OracleP2PEngine(rank, world, n_total, symm))
    flags = []
    for batch in cuts:
        a, b = batch[rank], batch[rank + 1]
        off, tok = gen_range(cfg, a, b)
        got = sx.query_insert(torch.from_numpy(off.view(np.int64)), torch.from_numpy(tok.view(np.int32)))
        flags.append(got.numpy().copy())
    np.save(out_path % rank, np.concatenate(flags))
    dist.barrier()
    dist.destroy_process_group()
    for k in range(symm.k):
        try:
            os.unlink(symm.path(k, rank))
        except OSError:
            pass


@pytest.mark.skipif(not os.path.isdir("/dev/shm"), reason="needs /dev/shm")
@pytest.mark.parametrize("world", [2, 3])
def test_p2p_exchange_flags_equal_single_process_oracle(world, tmp_path):
    rng = np.random.default_rng(10 + world)
    bounds = [0, 1200, 1201, 2600]                        # includes a one-document batch
    cuts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        if b - a < world:                                  # fewer documents than ranks: empty shards
            cuts.append([a] * world + [b])
            continue
        inner = sorted(rng.choice(np.arange(a + 1, b), world - 1, replace=False).tolist())
        cuts.append([a] + inner + [b])
    out = str(tmp_path / "flags_%d.npy")
    prefix = "lshb_test_%s" % uuid.uuid4().hex[:12]
    mp.spawn(_worker, args=(world, _free_port(), cuts, bounds[-1], out, prefix), nprocs=world, join=True)
    per_rank = [np.load(out % r) for r in range(world)]
    got, pos = [], [0] * world
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
