"""Band-sharded multi-GPU LSHBloom over torch.distributed (north_star).

One process per GPU.  Documents are sharded for MinHash (rank g holds a contiguous range, so
global stream order = rank order).  Bands are sharded for the Bloom stage: because every
document inserts all its band hashes (DESIGN R12) each band's filter evolves independently, so
rank g owns bands [band_lo(g), band_hi(g)) and processes ALL documents of the batch for them.
Per batch:
  1. K1 on the local documents writes band hashes owner-major (lshbloom_band_hashes_sharded),
  2. one all-to-all (NCCL over NVLink) delivers every rank its bands for all documents in
     global order,
  3. K3-K6 query-then-insert the owned bands (lshbloom_query_insert_bands),
  4. one all-reduce(MAX) of the uint8 hit flags combines the bands (any band hits),
  5. each rank keeps its own documents' flags.
Results are bit-identical for every world size.  The collectives are plumbing (torch /
NCCL); every arithmetic step runs in the library's kernels.

With the NCCL exchange the step is pipelined over chunks of `pipeline_docs` local documents
(default 262144): chunk c's band hashes are exchanged (one all_to_all per chunk) and handed to
the owners' engines (lshbloom_bands_add: copied into the batch and, with the window sweep,
binned at once) while every rank computes chunk c+1's MinHash; the query-then-insert runs once
per batch (lshbloom_bands_finish) over the whole global batch in stream order = rank order, so
the flags do not depend on the world size or the chunk size.  pipeline_docs=0 exchanges the
batch in one piece (steps 1-4 above).

exchange="p2p" replaces steps 1-4 by stores into peer memory: K1's
epilogue writes every band hash straight into its owner's receive buffer (torch symmetric
memory over NVLink / NVSwitch; lshbloom_band_hashes_to_peers), and the Bloom kernels raise each
hit document's flag directly in its home rank's flag buffer (lshbloom_query_insert_bands_peers),
with three device-side barriers per batch and no all-to-all, all-reduce or pack pass.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def band_range(rank: int, world: int, b: int) -> tuple[int, int]:
    """Bands owned by `rank`: as even a split as possible, lower ranks take the remainder."""
    base, rem = divmod(b, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class ShardedLSHBloom:
    def __init__(self, num_perm: int, b: int, r: int, n_expected: int, fp_rate: float, seed: int = 0,
                 *, group=None, device: int | None = None, sub_batch: int = 0, index: str = "bloom",
                 exchange: str = "nccl", engine=None, pipeline_docs: int = 262144):
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange = exchange
        self.pipeline_docs = int(pipeline_docs)
        self._p2p = None
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.b = b
        if engine is None:
            from ._native import LSHBloom
            engine = LSHBloom(num_perm, b, r, n_expected, fp_rate, seed, device=device,
                              rank=self.rank, world=self.world, sub_batch=sub_batch, index=index)
        self.engine = engine
        self.band_lo, self.band_hi = band_range(self.rank, self.world, b)
        assert (engine.band_lo, engine.band_hi) == (self.band_lo, self.band_hi)
        self.bl = self.band_hi - self.band_lo
        self.widths = [band_range(o, self.world, b)[1] - band_range(o, self.world, b)[0]
                       for o in range(self.world)]

    def _counts(self, n_local: int, device) -> list[int]:
        t = torch.tensor([n_local], dtype=torch.int64, device=device)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]

    def query_insert(self, offsets, tokens, counts: list[int] | None = None):
        """Local documents' duplicate flags (uint8), global stream order = rank order.
        counts: every rank's document count of this batch, when the caller knows them (the
        same list on every rank); otherwise they are all-gathered (one host sync per batch)."""
        device = offsets.device
        n_local = offsets.numel() - 1
        if counts is None:
            counts = self._counts(n_local, device)
        elif len(counts) != self.world or counts[self.rank] != n_local:
            raise ValueError("counts must list every rank's document count (this rank: %d)" % n_local)
        counts = [int(c) for c in counts]
        if self.exchange == "p2p":
            return self._query_insert_p2p(offsets, tokens, counts, device)
        if self.pipeline_docs > 0:
            return self._query_insert_pipelined(offsets, tokens, counts, device)
        if n_local:
            send = self.engine.band_hashes_sharded(offsets, tokens)      # owner-major, flat
        else:                                                            # this rank has no documents
            send = torch.empty(0, dtype=torch.int64, device=device)
        in_splits = [n_local * w for w in self.widths]
        out_splits = [c * self.bl for c in counts]
        recv = torch.empty(sum(out_splits), dtype=send.dtype, device=device)
        dist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)
        n_global = sum(counts)
        hits = self.engine.query_insert_bands(recv.view(n_global, self.bl))
        dist.all_reduce(hits, op=dist.ReduceOp.MAX, group=self.group)
        start = sum(counts[:self.rank])
        return hits[start:start + n_local]

    def _query_insert_pipelined(self, offsets, tokens, counts, device):
        n_local = counts[self.rank]
        n_global = sum(counts)
        starts = [0]
        for c in counts:
            starts.append(starts[-1] + c)
        C = self.pipeline_docs
        nchunks = max(1, -(-max(counts) // C))
        off_h = offsets.cpu().numpy().view(np.uint64) if n_local else None   # chunk bounds (one copy)
        self.engine.bands_begin(n_global)
        for c in range(nchunks):
            a, b = min(c * C, n_local), min((c + 1) * C, n_local)
            if b > a:
                o = torch.from_numpy((off_h[a:b + 1] - off_h[a]).view(np.int64)).to(device, non_blocking=True)
                t = tokens[int(off_h[a]):int(off_h[b])]
                send = self.engine.band_hashes_sharded(o, t)             # owner-major, flat
            else:
                send = torch.empty(0, dtype=torch.int64, device=device)
            part = [max(0, min(C, counts[r] - c * C)) for r in range(self.world)]
            in_splits = [(b - a) * w for w in self.widths]
            out_splits = [k * self.bl for k in part]
            recv = torch.empty(sum(out_splits), dtype=torch.int64, device=device)
            dist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)
            pos = 0
            for r in range(self.world):                                 # rank r's chunk c, in place
                if part[r]:
                    self.engine.bands_add(recv[pos:pos + part[r] * self.bl].view(part[r], self.bl),
                                          starts[r] + c * C)
                pos += part[r] * self.bl
        hits = self.engine.bands_finish(device=device)
        dist.all_reduce(hits, op=dist.ReduceOp.MAX, group=self.group)
        return hits[starts[self.rank]:starts[self.rank] + n_local]

    def reset(self):
        self.engine.reset()

    # ------------------------------------------------------------------ peer-memory exchange
    def _p2p_buffers(self, n_global: int, n_local_max: int, device):
        """Symmetric receive / flag buffers (same size on every rank; every rank takes the same
        decision because it sees the same all-gathered counts)."""
        import torch.distributed._symmetric_memory as symm_mem
        bl_max = max(self.widths)
        cur = self._p2p
        if cur is not None and cur["cap_g"] >= n_global and cur["cap_l"] >= n_local_max:
            return cur
        cap_g = max(n_global, (cur or {}).get("cap_g", 0))
        cap_l = max(n_local_max, (cur or {}).get("cap_l", 0))
        recv = symm_mem.empty(cap_g * bl_max, dtype=torch.int64, device=device)
        flags = symm_mem.empty(cap_l, dtype=torch.uint8, device=device)
        hr = symm_mem.rendezvous(recv, self.group if self.group is not None else dist.group.WORLD)
        hf = symm_mem.rendezvous(flags, self.group if self.group is not None else dist.group.WORLD)
        self._p2p = {"cap_g": cap_g, "cap_l": cap_l, "recv": recv, "flags": flags, "hr": hr, "hf": hf,
                     "peer_recv": [int(x) for x in hr.buffer_ptrs], "peer_flags": [int(x) for x in hf.buffer_ptrs]}
        return self._p2p

    def _query_insert_p2p(self, offsets, tokens, counts, device):
        n_local = counts[self.rank]
        n_global = sum(counts)
        starts = [0]
        for c in counts:
            starts.append(starts[-1] + c)
        buf = self._p2p_buffers(n_global, max(counts), device)
        buf["flags"][:n_local].zero_()
        buf["hr"].barrier(channel=0)            # flags zeroed everywhere; last batch's readers done
        if n_local:
            self.engine.band_hashes_to_peers(offsets, tokens, starts[self.rank], buf["peer_recv"])
        buf["hr"].barrier(channel=1)            # every band hash has landed in its owner's buffer
        recv = buf["recv"][:n_global * self.bl].view(n_global, self.bl)
        self.engine.query_insert_bands_peers(recv, starts, buf["peer_flags"])
        buf["hr"].barrier(channel=2)            # every hit flag has landed at its home rank
        return buf["flags"][:n_local].clone()
