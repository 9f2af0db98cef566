"""Device-resident graph store (replaces GraphCSR's arrays on the GPU).

Reference: ``mqpipe/graph.py:28-91`` (GraphCSR: int64 row_offsets, sorted
deduped rows, f32 features, int32 labels, split masks).

HBM layout:
  * ``row_off``  int64 [n+1] and ``col`` int32 [E'] — the reference CSR with
    stored self loops removed.  The sampler drops the loop from every
    neighbour list anyway (``samplers.py:162``), so stripping once at upload
    makes every row's pool contiguous.
  * ``features`` f32 [n, pitch], pitch = round_up(d, 4) floats so every row is
    16-byte aligned for vector loads (Reddit's 602-d rows are 2,408 B).
    Placement "hbm" keeps the table in device memory; "host" keeps it in
    pinned host memory and the gather reads misses over the host link;
    "sharded" (``shard_features``) partitions it by node across the ranks:
    node v's row lives on rank v % G at row v // G, and the other ranks'
    shards are mapped over NVLink (CUDA IPC), so the gather reads remote
    rows peer-to-peer (BASELINE configs[4]).
  * ``labels`` int32 [n].
"""

from __future__ import annotations

import numpy as np
import torch

import ctypes as C

from ._lib import lib, ptr

INT32_MAX = 2 ** 31 - 1


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def _as_tensor(a, dtype, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype)
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=device)


class DeviceGraph:
    """GraphCSR resident on one GPU.  Build with :meth:`from_csr`."""

    def __init__(self):
        raise TypeError("use DeviceGraph.from_csr(g)")

    @classmethod
    def from_csr(cls, g, device=None, feature_placement: str = "hbm") -> "DeviceGraph":
        """Upload any GraphCSR-like object (reference ``GraphCSR`` or
        ``synth.SynthGraph``).  ``feature_placement``: "hbm", "host" or
        "sharded" (collective over torch.distributed: ``g.features`` holds
        either every node's row or only this rank's rows v = rank, rank+G, ...)."""
        if feature_placement not in ("hbm", "host", "sharded"):
            raise ValueError(f"unknown feature placement {feature_placement!r}")
        self = object.__new__(cls)
        dev = torch.device(device or "cuda")
        if dev.type != "cuda":
            raise ValueError("DeviceGraph lives on a CUDA device")
        self.device = dev
        self.num_nodes = int(g.num_nodes)
        self.num_classes = int(g.num_classes)
        feats = g.features
        self.feature_dim = int(feats.shape[1])
        self.pitch = round_up(self.feature_dim, 4)
        self.train_mask = np.asarray(_host(g.train_mask), dtype=bool)
        self.val_mask = np.asarray(_host(g.val_mask), dtype=bool)
        self.test_mask = np.asarray(_host(g.test_mask), dtype=bool)
        self.source = g
        self.shards = None   # seed-partitioned store: device pointers of the G shards
        self._shard_keep = None
        n = self.num_nodes
        if n >= INT32_MAX:
            raise ValueError("node ids must fit in int32")
        stream = torch.cuda.current_stream(dev).cuda_stream
        with torch.cuda.device(dev):
            row_off = _as_tensor(g.row_offsets, torch.int64, dev)
            col = _as_tensor(g.col_indices, torch.int32, dev)
            e = int(col.numel())
            self.num_arcs_stored = e
            out_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
            scratch = torch.empty(int(lib().mq_scan_scratch_bytes(max(n, 1))), dtype=torch.uint8,
                                  device=dev)
            out_col = torch.empty(max(e, 1), dtype=torch.int32, device=dev)
            lib().mq_strip_self_loops(ptr(row_off), ptr(col), n, e, ptr(out_off), ptr(out_col),
                                      ptr(scratch), stream)
            kept = int(out_off[-1].item())
            self.row_off = out_off
            self.col = out_col[:max(kept, 1)].clone() if kept != e else out_col
            self.num_arcs = kept
            self.self_loops = e - kept
            # stripped loops per row: they still count toward in-degrees and
            # the cache walk's flow (cache.py:41-76 use the stored CSR)
            self.loops = (((row_off[1:] - row_off[:-1]) - (out_off[1:] - out_off[:-1]))
                          .to(torch.int32) if self.self_loops else None)
            del row_off, col, scratch
            self.labels = _as_tensor(g.labels, torch.int32, dev)
            self.feature_placement = feature_placement
            if feature_placement == "sharded":
                self.features = None
                self._install_shard(feats)
                return self
            if feature_placement == "hbm":
                if (isinstance(feats, torch.Tensor) and feats.device == dev
                        and feats.dtype == torch.float32 and feats.is_contiguous()
                        and self.feature_dim == self.pitch):
                    table = feats  # already a pitched device table: share it (57 GB at papers)
                else:
                    table = torch.zeros((n, self.pitch), dtype=torch.float32, device=dev)
                    table[:, :self.feature_dim] = _as_tensor(feats, torch.float32, dev)
            else:
                table = torch.zeros((n, self.pitch), dtype=torch.float32, pin_memory=True)
                table[:, :self.feature_dim] = _as_tensor(feats, torch.float32, "cpu")
            self.features = table
        return self

    # ---- seed-partitioned feature store
    def shard_features(self, group=None):
        """Collective: keep only this rank's rows of the (full) table and map
        the other ranks' shards; the full table is released."""
        if self.features is None:
            raise ValueError("features are already sharded")
        full = self.features
        self.features = None
        self._install_shard(full, group)
        self.feature_placement = "sharded"
        del full
        torch.cuda.empty_cache()

    def _install_shard(self, feats, group=None):
        import torch.distributed as dist
        from .peer import PeerArena, exchange_handles, open_handle
        on = dist.is_available() and dist.is_initialized()
        G, r = (dist.get_world_size(group), dist.get_rank(group)) if on else (1, 0)
        if G > MQ_MAX_SHARDS:
            raise ValueError(f"at most {MQ_MAX_SHARDS} feature shards")
        n, d, P = self.num_nodes, self.feature_dim, self.pitch
        rows = shard_rows(n, G, r)
        if int(feats.shape[0]) == n:
            own = feats[r::G]
        elif int(feats.shape[0]) == rows:
            own = feats
        else:
            raise ValueError(f"features must hold all {n} rows or this rank's {rows}")
        arena = PeerArena(max(rows, 1) * P * 4, self.device)
        stage = torch.zeros((max(rows, 1), P), dtype=torch.float32, device=self.device)
        stage[:rows, :d] = _as_tensor(own, torch.float32, self.device)
        lib().mq_memcpy_async(arena.ptr, ptr(stage), stage.numel() * 4,
                              torch.cuda.current_stream(self.device).cuda_stream)
        torch.cuda.synchronize(self.device)
        del stage
        infos = exchange_handles(arena.export(), group) if on else [(None, None)]
        import os
        ptrs, opened = [], []
        for q, (pid, h) in enumerate(infos):
            if q == r:
                ptrs.append(arena.ptr)
            elif pid == os.getpid():
                raise RuntimeError("two ranks in one process: use use_local_shards")
            else:
                p = open_handle(h, self.device)
                opened.append(p)
                ptrs.append(p)
        if on:
            dist.barrier(group)
        self.shards = ptrs
        self._shard_keep = (arena, opened)
        self.shard_rank, self.num_shards = r, G

    def use_local_shards(self, world: int):
        """Split this process's table into ``world`` node-partitioned shards
        (one process standing in for G ranks; tests of the sharded gather)."""
        if self.features is None or world < 1 or world > MQ_MAX_SHARDS:
            raise ValueError("need a full table and 1..8 shards")
        keep = [self.features[q::world].contiguous() for q in range(world)]
        self.shards = [t.data_ptr() for t in keep]
        self._shard_keep = keep
        self.num_shards = world

    def gather_rows(self, ids, n_dev, n_max: int, out, out_pitch: int, stream, cache=None,
                    hit_miss=None):
        """gather_features into ``out``: cache hits from the HBM table, misses
        from the store (one table, pinned host, or the node-partitioned shards)."""
        tbl = ptr(cache.table) if cache is not None else None
        slot = ptr(cache.slot_of) if cache is not None else None
        hm = ptr(hit_miss) if cache is not None else None
        if self.shards is not None:
            arr = (C.c_void_p * len(self.shards))(*self.shards)
            lib().mq_gather_sharded(tbl, self.pitch, slot, arr, len(self.shards), self.pitch,
                                    ptr(ids), ptr(n_dev), n_max, self.feature_dim, ptr(out),
                                    out_pitch, hm, stream)
        else:
            lib().mq_gather(tbl, self.pitch, slot, ptr(self.features), self.pitch, ptr(ids),
                            ptr(n_dev), n_max, self.feature_dim, ptr(out), out_pitch, hm, stream)

    def require_full_table(self, what: str):
        if self.features is None:
            raise NotImplementedError(f"{what} reads the whole feature table; this graph's "
                                      "features are sharded across ranks")

    # ---- reference-compatible views
    @property
    def num_edges(self) -> int:
        return self.num_arcs_stored

    def features_view(self) -> torch.Tensor:
        self.require_full_table("features_view")
        return self.features[:, :self.feature_dim]

    def degree(self) -> torch.Tensor:
        """Out-degree without self loops (the sampler's pool size)."""
        return self.row_off[1:] - self.row_off[:-1]

    def in_degrees(self) -> torch.Tensor:
        """In-degree counts of the stored CSR (graph.py:47-49), self loops
        included, as the reference's cache_probs_degree uses them (int64,
        computed on the device by mq_in_degrees)."""
        deg = torch.empty(max(self.num_nodes, 1), dtype=torch.int64, device=self.device)
        lib().mq_in_degrees(ptr(self.col), self.num_nodes, self.num_arcs, ptr(self.loops),
                            ptr(deg), torch.cuda.current_stream(self.device).cuda_stream)
        return deg[:self.num_nodes]


MQ_MAX_SHARDS = 8


def shard_rows(num_nodes: int, world: int, rank: int) -> int:
    """Rows of rank's shard: nodes rank, rank + world, ... < num_nodes."""
    return max(0, (num_nodes - rank + world - 1) // world)


def _host(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return a


# ------------------------------------------------------------------ ingest
MAGIC = b"MQG1"


def _stream(device):
    return torch.cuda.current_stream(device).cuda_stream


def build_csr(edges, num_nodes: int, features=None, labels=None, num_classes: int | None = None,
              device=None):
    """The reference's build_csr (graph.py:94-139) on the device: duplicate
    arcs collapse, rows come out sorted; default features are the one-hot
    degree buckets (graph.py:142-149).  Returns a GraphCSR-like ``SynthGraph``
    whose arrays live on ``device`` (int64 row_offsets, int32 col_indices);
    ``DeviceGraph.from_csr`` takes it as is."""
    from .synth import SynthGraph
    dev = torch.device(device or "cuda")
    n = int(num_nodes)
    if n < 1 or n >= INT32_MAX:
        raise ValueError("num_nodes must lie in [1, 2^31 - 1)")
    e = edges if isinstance(edges, torch.Tensor) else torch.as_tensor(
        np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges, dtype=np.int64))
    e = e.to(device=dev, dtype=torch.int64).reshape(-1, 2).contiguous()
    m = int(e.shape[0])
    lb = lib()
    s = _stream(dev)
    scr = torch.empty(int(lb.mq_build_csr_scratch_bytes(m)), dtype=torch.uint8, device=dev)
    uniq = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    lb.mq_build_csr_keys(ptr(e), m, n, ptr(scr), ptr(uniq), ptr(cnt), ptr(bad), s)
    if int(bad.item()):
        raise ValueError("edge endpoint out of range")
    nu = int(cnt.item())
    del scr
    row_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(nu, 1), dtype=torch.int32, device=dev)
    lb.mq_build_csr_finish(ptr(uniq), nu, n, ptr(row_off), ptr(col), s)
    col = col[:nu]
    if features is None:
        bucket = torch.empty(n, dtype=torch.int32, device=dev)
        lb.mq_degree_buckets(ptr(row_off), n, ptr(bucket), s)
        dim = int(bucket.max().item()) + 1
        features = torch.zeros((n, dim), dtype=torch.float32, device=dev)
        features[torch.arange(n, device=dev), bucket.long()] = 1.0
    else:
        features = _as_tensor(features, torch.float32, dev)
        if features.shape[0] != n:
            raise ValueError("features must have one row per node")
    labels = (torch.zeros(n, dtype=torch.int32, device=dev) if labels is None
              else _as_tensor(labels, torch.int32, dev))
    if num_classes is None:
        num_classes = int(labels.max().item()) + 1
    empty = np.zeros(n, dtype=bool)
    return SynthGraph(n, row_off, col, features.contiguous(), labels, int(num_classes),
                      empty.copy(), empty.copy(), empty.copy())


def load(path: str, device=None):
    """Read the reference's MQG1 container (graph.py:325-395: magic, u64
    header, u64 CSR arrays, f32 features, i32 labels, bit-packed masks)
    straight to the device: u64 columns are narrowed to int32 by a kernel."""
    from .synth import SynthGraph
    dev = torch.device(device or "cuda")
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    if raw.size < 36:
        raise ValueError("buffer too short for header")
    if bytes(raw[:4]) != MAGIC:
        raise ValueError(f"bad magic {bytes(raw[:4])!r}")
    n, e, d, c = (int(x) for x in np.frombuffer(raw[4:36].tobytes(), dtype="<u8"))
    mask_bytes = (n + 7) // 8
    off = 36
    need = off + 8 * (n + 1) + 8 * e + 4 * n * d + 4 * n + 3 * mask_bytes
    if raw.size < need:
        raise ValueError(f"buffer truncated: need {need} bytes, have {raw.size}")

    def take(count, dtype):
        nonlocal off
        nb = count * np.dtype(dtype).itemsize
        a = np.frombuffer(raw, dtype=dtype, count=count, offset=off)
        off += nb
        return np.array(a)  # an owned, writable copy (the map is read-only)

    row_off = torch.as_tensor(take(n + 1, "<u8").astype(np.int64)).to(dev)
    cols64 = torch.as_tensor(take(e, "<u8").view(np.int64)).to(dev)
    col = torch.empty(max(e, 1), dtype=torch.int32, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    lib().mq_narrow_cols(ptr(cols64), e, n, ptr(col), ptr(bad), _stream(dev))
    if int(bad.item()):
        raise ValueError("column index out of range")
    del cols64
    feats = torch.as_tensor(take(n * d, "<f4").reshape(n, d)).to(dev)
    labels = torch.as_tensor(take(n, "<i4")).to(dev)
    masks = []
    for _ in range(3):
        bits = np.unpackbits(np.asarray(raw[off:off + mask_bytes]), bitorder="little")
        masks.append(bits[:n].astype(bool))
        off += mask_bytes
    return SynthGraph(n, row_off, col[:e], feats, labels, c, *masks)
