"""Device batch queue: groups of Q prepared mini-batches (mq_prep_batches).

MQ-GNN overlaps sampling/transfer with compute through per-device queues of
prepared batches (runtime.py:380-612, BoundedQueue pipeline.py:109-167).  On
the B200 a queue group is Q device slots filled by ONE pass of batched
kernels (csrc/mq_prep.cu): device batch plan -> per hop sample + relabel ->
feature gather + target labels, every launch covering all Q batches.  The
trainer consumes the slots one window at a time while the next group is
prepared on another stream.

Buffers are [Q, ...] tensors so slot q of every array sits at a fixed stride;
``SlotView`` exposes one slot with the per-batch attribute names the train
workspaces expect (targets, hops[h].row_ptr, x0, labels, ...).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from ._lib import I32, I64, P, lib, ptr
from .engine import hop_bounds

MQ_MAX_HOPS = 4
# node-indexed relabel tables up to 16 GB (all slots): the hashed layout is
# a memory saver, not a speed-up (papers shape 2.30M -> 2.17M seeds/s, products
# 2.53M -> 2.31M with it forced: probes and the key CAS cost more than the
# smaller span saves)
RANK_TABLE_BYTES = 16 << 30
PREP_SETUP, PREP_SAMPLE, PREP_RELABEL, PREP_GATHER, PREP_LABELS = 1, 2, 4, 8, 16


class PrepHop(C.Structure):
    _fields_ = [("fanout", I32), ("n_dst_max", I32), ("n_src_max", I32), ("pad_", I32),
                ("nbr", P), ("nbr_s", I64), ("cnt", P), ("cnt_s", I64),
                ("row_ptr", P), ("row_ptr_s", I64),
                ("rows", P), ("cols", P), ("vals", P), ("edge_s", I64),
                ("src_ids", P), ("src_s", I64), ("counts", P), ("counts_s", I64)]


class PrepDesc(C.Structure):
    _fields_ = [("nslots", I32), ("num_hops", I32), ("batch_size", I32), ("world", I32),
                ("rank", I32), ("d", I32),
                ("perm", P), ("n_perm", I64), ("cursor", P),
                ("targets", P), ("targets_s", I64), ("n_targets", P), ("n_targets_s", I64),
                ("key", P), ("key_s", I64),
                ("hop", PrepHop * MQ_MAX_HOPS),
                ("node_rank", P), ("reserved_", P), ("table_s", I64),
                ("scratch", P), ("scratch_s", I64),
                ("row_off", P), ("col", P), ("hot_arc", P), ("hot_off", P),
                ("cache_tbl", P), ("cache_pitch", I32), ("store_pitch", I32),
                ("slot_of", P), ("store", P),
                ("x0", P), ("x0_s", I64), ("x0_pitch", I32), ("stage_mask", C.c_uint32),
                ("hit_miss", P),
                ("all_labels", P), ("labels", P), ("labels_s", I64),
                ("store_shard", P * 8), ("n_shards", I32), ("hash_lg", I32)]


class PrepShared:
    """Per-runner state every group's prep pass reuses (prep passes are
    serialised on one stream): node relabel tables and scan scratch."""

    def __init__(self, g, fanouts, batch_size: int, Q: int):
        dev = g.device
        self.Q = int(Q)
        bounds = hop_bounds(batch_size, fanouts, g.num_nodes)
        # the relabel's node-rank words, one int32 per node and slot (INT32_MAX
        # at rest): 4 B x nodes x Q, L2-resident up to products-sized graphs
        # (papers-sized: 8 x 111M x 4 B = 3.5 GB).  Past RANK_TABLE_BYTES a hash
        # of the touched nodes per slot instead: 2^k (key, word) pairs, load
        # <= 0.8 at the bound on a pass's distinct nodes (~0.3 in practice),
        # then the position -> entry list (MQ_PREP_HASH=1 / 0 forces it)
        n_src = bounds[-1].n_src_max
        force = os.environ.get("MQ_PREP_HASH")
        direct = Q * g.num_nodes * 4
        self.hash_lg = 0
        if force == "1" or (force != "0" and direct > RANK_TABLE_BYTES):
            lg = max(4, (int(1.25 * n_src) - 1).bit_length())
            if force == "1" or (2 << lg) + n_src < g.num_nodes:
                self.hash_lg = lg
        if self.hash_lg:
            cap = 1 << self.hash_lg
            self.tbl = torch.zeros((Q, 2 * cap + n_src), dtype=torch.int32, device=dev)
            self.tbl[:, 1:2 * cap:2] = 2 ** 31 - 1
        else:
            self.tbl = torch.full((Q, g.num_nodes), 2 ** 31 - 1, dtype=torch.int32, device=dev)
        per = max(int(lib().mq_prep_scratch_bytes(b.n_dst_max, b.fanout)) for b in bounds)
        self.scratch_s = per
        self.scratch = torch.zeros(Q * per, dtype=torch.uint8, device=dev)


class HopView:
    __slots__ = ("nbr", "cnt", "row_ptr", "rows", "cols", "vals", "src_ids", "counts")


class SlotView:
    """One slot of a PrepGroup with SampleWorkspace's attribute names."""

    def __init__(self, grp: "PrepGroup", q: int):
        self.graph = grp.graph
        self.fanouts = grp.fanouts
        self.batch_size = grp.batch_size
        self.bounds = grp.bounds
        self.q = q
        self.targets = grp.targets[q]
        self.n_targets = grp.n_targets[q]
        self.key = grp.key[q]
        self.x0 = grp.x0[q]
        self.labels = grp.labels[q]
        self.hops = []
        for hb in grp.hops:
            v = HopView()
            for name in HopView.__slots__:
                setattr(v, name, getattr(hb, name)[q])
            self.hops.append(v)

    def n_dst_dev(self, h: int) -> torch.Tensor:
        return self.n_targets if h == 0 else self.hops[h - 1].counts[0:1]

    def dst(self, h: int) -> torch.Tensor:
        return self.targets if h == 0 else self.hops[h - 1].src_ids

    @property
    def input_ids(self) -> torch.Tensor:
        return self.hops[-1].src_ids

    @property
    def n_input_dev(self) -> torch.Tensor:
        return self.hops[-1].counts[0:1]


class _HopBufs:
    pass


class PrepGroup:
    """Q device slots of prepared batches plus the descriptor of their pass."""

    def __init__(self, g, fanouts, batch_size: int, Q: int, shared: PrepShared):
        if not fanouts or len(fanouts) > MQ_MAX_HOPS:
            raise ValueError(f"need 1..{MQ_MAX_HOPS} hops")
        if any(f < 1 or f > 32 for f in fanouts):
            raise ValueError("fanouts must lie in [1, 32]")
        dev = g.device
        i32 = dict(dtype=torch.int32, device=dev)
        self.graph = g
        self.fanouts = tuple(int(f) for f in fanouts)
        self.batch_size = int(batch_size)
        self.Q = int(Q)
        self.shared = shared
        self.bounds = hop_bounds(self.batch_size, self.fanouts, g.num_nodes)
        B = max(self.batch_size, 1)
        self.targets = torch.zeros((Q, B), **i32)
        self.n_targets = torch.zeros((Q, 1), **i32)
        self.key = torch.zeros((Q, 3), **i32)  # uint32 {seed, epoch, batch}
        self.hops = []
        for b in self.bounds:
            hb = _HopBufs()
            nnz = max(b.nnz_max, 1)
            hb.nbr = torch.zeros((Q, nnz), **i32)
            hb.cnt = torch.zeros((Q, max(b.n_dst_max, 1)), **i32)
            hb.row_ptr = torch.zeros((Q, b.n_dst_max + 1), **i32)
            hb.rows = torch.zeros((Q, nnz), **i32)
            hb.cols = torch.zeros((Q, nnz), **i32)
            hb.vals = torch.zeros((Q, nnz), dtype=torch.float32, device=dev)
            hb.src_ids = torch.zeros((Q, max(b.n_src_max, 1)), **i32)
            hb.counts = torch.zeros((Q, 2), **i32)
            self.hops.append(hb)
        self.x0 = torch.zeros((Q, max(self.bounds[-1].n_src_max, 1), g.pitch),
                              dtype=torch.float32, device=dev)
        self.labels = torch.zeros((Q, B), **i32)
        self.slots = [SlotView(self, q) for q in range(Q)]

    def set_key(self, seed: int, epoch: int):
        # fills with the words' int32 bit patterns: kernel arguments, no
        # pageable host copy (which would block the host until the stream
        # drains, e.g. at every epoch boundary)
        def i32(x):
            x &= 0xFFFFFFFF
            return x - (1 << 32) if x >= 1 << 31 else x
        self.key[:, 0].fill_(i32(seed))
        self.key[:, 1].fill_(i32(epoch))

    def desc(self, cache, perm, cursor, world: int, rank: int) -> PrepDesc:
        """Descriptor of one pass; cursor=None means host-staged targets."""
        g = self.graph
        sh = self.shared
        d = PrepDesc()
        d.nslots = self.Q
        d.num_hops = len(self.fanouts)
        d.batch_size = self.batch_size
        d.world = int(world)
        d.rank = int(rank)
        d.d = g.feature_dim
        d.perm = ptr(perm)
        d.n_perm = int(perm.numel()) if perm is not None else 0
        d.cursor = ptr(cursor)
        d.targets, d.targets_s = ptr(self.targets), self.targets.stride(0)
        d.n_targets, d.n_targets_s = ptr(self.n_targets), self.n_targets.stride(0)
        d.key, d.key_s = ptr(self.key), self.key.stride(0)
        for h, (hb, b) in enumerate(zip(self.hops, self.bounds)):
            hp = d.hop[h]
            hp.fanout, hp.n_dst_max, hp.n_src_max = b.fanout, b.n_dst_max, b.n_src_max
            hp.nbr, hp.nbr_s = ptr(hb.nbr), hb.nbr.stride(0)
            hp.cnt, hp.cnt_s = ptr(hb.cnt), hb.cnt.stride(0)
            hp.row_ptr, hp.row_ptr_s = ptr(hb.row_ptr), hb.row_ptr.stride(0)
            hp.rows, hp.cols, hp.vals = ptr(hb.rows), ptr(hb.cols), ptr(hb.vals)
            hp.edge_s = hb.rows.stride(0)
            hp.src_ids, hp.src_s = ptr(hb.src_ids), hb.src_ids.stride(0)
            hp.counts, hp.counts_s = ptr(hb.counts), hb.counts.stride(0)
        d.node_rank, d.table_s, d.hash_lg = ptr(sh.tbl), sh.tbl.stride(0), sh.hash_lg
        d.scratch, d.scratch_s = ptr(sh.scratch), sh.scratch_s
        d.row_off, d.col = ptr(g.row_off), ptr(g.col)
        d.store_pitch = g.pitch
        if g.shards is not None:  # seed-partitioned store (graph.DeviceGraph.shard_features)
            d.n_shards = len(g.shards)
            for q, p in enumerate(g.shards):
                d.store_shard[q] = p
        else:
            d.store = ptr(g.features)
        if cache is not None:
            d.hot_arc, d.hot_off = ptr(cache.hot_arc), ptr(cache.hot_off)
            d.cache_tbl, d.cache_pitch = ptr(cache.table), g.pitch
            d.slot_of, d.hit_miss = ptr(cache.slot_of), ptr(cache.hit_miss)
        d.x0, d.x0_s, d.x0_pitch = ptr(self.x0), self.x0.stride(0), g.pitch
        d.all_labels = ptr(g.labels)
        d.labels, d.labels_s = ptr(self.labels), self.labels.stride(0)
        return d

    def launch(self, desc: PrepDesc, stream: int):
        lib().mq_prep_batches(C.byref(desc), stream)

    # ------------------------------------------------ host staging / read-back
    def stage(self, batches, seed: int, epoch: int):
        """Host-staged slot contents (the descriptor with cursor=None):
        ``batches`` = [(batch_id, int targets)] for slots 0..len-1, the rest
        empty (n = 0).  Synchronous; for tests and the drop-in API."""
        import numpy as np
        if len(batches) > self.Q:
            raise ValueError("more batches than slots")
        tg = np.zeros(tuple(self.targets.shape), dtype=np.int32)
        meta = np.zeros((self.Q, 4), dtype=np.uint32)
        for q in range(self.Q):
            meta[q, 1:3] = (seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF)
            if q < len(batches):
                bid, t = batches[q]
                t = np.asarray(t, dtype=np.int64).ravel()
                if t.size > self.batch_size:
                    raise ValueError("batch larger than the slot")
                tg[q, :t.size] = t
                meta[q, 0] = t.size
                meta[q, 3] = bid & 0xFFFFFFFF
        dev = self.targets.device
        self.targets.copy_(torch.from_numpy(tg).to(dev))
        m = torch.from_numpy(meta.view(np.int32)).to(dev)
        self.n_targets.copy_(m[:, 0:1])
        self.key.copy_(m[:, 1:4])

    def minibatch(self, q: int, epoch: int = 0, with_features: bool = True):
        """Slot ``q`` as a reference-shaped ``MiniBatch`` (samplers.py:49-72):
        bottom-up blocks, targets, labels and the gathered input features,
        copied out of the slot buffers — the parity read-back of the
        production prep pass."""
        from .samplers import Block, MiniBatch
        torch.cuda.synchronize(self.targets.device)
        dev = self.targets.device
        n = int(self.n_targets[q, 0])
        counts = torch.stack([hb.counts[q] for hb in self.hops]).cpu().numpy()
        tg = self.targets[q, :n].clone()
        blocks, nd, dst = [], n, tg
        for h, hb in enumerate(self.hops):
            n_src, nnz = int(counts[h, 0]), int(counts[h, 1])
            blk = Block(rows=hb.rows[q, :nnz].clone(), cols=hb.cols[q, :nnz].clone(),
                        values=hb.vals[q, :nnz].clone(), src_ids=hb.src_ids[q, :n_src].clone(),
                        dst_ids=dst, row_ptr=hb.row_ptr[q, :nd + 1].clone(),
                        dst_in_src=torch.arange(nd, device=dev, dtype=torch.int32))
            blocks.append(blk)
            dst, nd = blk.src_ids, n_src
        blocks.reverse()
        n_in = int(counts[-1, 0])
        feats = (self.x0[q, :n_in, :self.graph.feature_dim].clone() if with_features else None)
        bid = int(self.key[q, 2].item()) & 0xFFFFFFFF
        return MiniBatch(batch_id=bid, epoch=epoch, target_ids=tg,
                         target_labels=self.labels[q, :n].clone(), layers=tuple(blocks),
                         input_ids=blocks[0].src_ids, features=feats)
