"""Drop-in node-wise (GraphSAGE) sampling API backed by the CUDA kernels.

Mirrors the reference's public surface in ``mqpipe/samplers.py``:

* ``SamplerParams``     — ``samplers.py:75-85`` (+ per-hop ``fanout`` tuples)
* ``Block``/``MiniBatch`` — ``samplers.py:27-72`` (device tensors; ``digest()``
  hashes the same bytes as the reference's SHA-256, ``samplers.py:63-72``)
* ``node_wise_block``   — ``samplers.py:142-210`` (SAGE arm)
* ``sample_node_wise``  — ``samplers.py:213-226``
* ``build_minibatch``   — ``samplers.py:502-540`` (node-wise methods)

``rng`` is a :class:`PhiloxStream` — the injected counter-based stream
 that replaces NumPy's PCG64 so that every row's draws are
addressable in parallel.  Under the same stream the reference's own code
produces bit-identical blocks (tests/golden).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np
import torch

from .cache import DeviceCache, gather_features
from .engine import SampleWorkspace, current_stream
from .graph import DeviceGraph


from .layerwise import LayerBlock, SamplingError, gcn_block_from_sage, sample_fastgcn, sample_ladies


@dataclass(frozen=True)
class PhiloxStream:
    """Key of the injected draw stream: (seed, epoch, batch_id); the hop and
    row complete the Philox counter inside the kernels."""

    seed: int = 0
    epoch: int = 0
    batch_id: int = 0
    hop: int = 0

    def at_hop(self, hop: int) -> "PhiloxStream":
        return PhiloxStream(self.seed, self.epoch, self.batch_id, hop)


@dataclass(frozen=True)
class SamplerParams:
    method: str = "sage"
    fanout: object = 5            # int (every hop) or tuple (hop 0 = seeds)
    nodes_per_layer: int = 512    # layer-wise methods (ladies, fastgcn)
    num_layers: int = 2
    flat: bool = False
    debias: bool = False
    replace: bool = False

    @property
    def hop_fanouts(self) -> tuple:
        if isinstance(self.fanout, (tuple, list)):
            f = tuple(int(x) for x in self.fanout)
            if len(f) != self.num_layers:
                raise ValueError("one fanout per layer required")
            return f
        return (int(self.fanout),) * self.num_layers


@dataclass(frozen=True)
class Block:
    """One sampled layer (dst rows x src cols) on the device.

    ``values`` are the float32 weights the forward applies
    (``effective_values`` in the reference); ``values64()`` restores the
    reference's float64 ``1/s``.  ``row_ptr`` is the CSR view of the
    row-sorted triplets."""

    rows: torch.Tensor
    cols: torch.Tensor
    values: torch.Tensor
    src_ids: torch.Tensor
    dst_ids: torch.Tensor
    row_ptr: torch.Tensor
    dst_in_src: torch.Tensor = None

    @property
    def effective_values(self):
        return self.values

    @property
    def num_dst(self) -> int:
        return int(self.dst_ids.numel())

    @property
    def num_src(self) -> int:
        return int(self.src_ids.numel())

    @property
    def nnz(self) -> int:
        return int(self.rows.numel())

    def values64(self) -> np.ndarray:
        rp = self.row_ptr.cpu().numpy().astype(np.int64)
        s = np.diff(rp)
        rows = self.rows.cpu().numpy().astype(np.int64)
        return 1.0 / s[rows].astype(np.float64) if rows.size else np.empty(0, np.float64)

    def to_reference(self) -> dict:
        """int64/f64 NumPy arrays laid out as the reference's Block."""
        return dict(rows=self.rows.cpu().numpy().astype(np.int64),
                    cols=self.cols.cpu().numpy().astype(np.int64),
                    values=self.values64(),
                    src_ids=self.src_ids.cpu().numpy().astype(np.int64),
                    dst_ids=self.dst_ids.cpu().numpy().astype(np.int64),
                    dst_in_src=np.arange(self.num_dst, dtype=np.int64))


@dataclass
class MiniBatch:
    batch_id: int
    epoch: int
    target_ids: torch.Tensor
    target_labels: torch.Tensor
    layers: tuple
    input_ids: torch.Tensor
    features: torch.Tensor | None = None
    cache_hits: int = 0
    cache_misses: int = 0
    dropped_targets: int = 0
    method: str = "sage"
    miss_bytes: int = 0  # feature bytes served from the (host) store by transfer_stage

    def digest(self) -> str:
        """Same SHA-256 as the reference (samplers.py:63-72) over int64 ids,
        int64 rows/cols, f64 values and the f32 features."""
        h = hashlib.sha256()
        h.update(self.target_ids.cpu().numpy().astype(np.int64).tobytes())
        for blk in self.layers:
            r = blk.to_reference()
            for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
                h.update(np.ascontiguousarray(r[k]).tobytes())
        if self.features is not None:
            h.update(np.ascontiguousarray(self.features.cpu().numpy(), dtype=np.float32).tobytes())
        return h.hexdigest()


# ---------------------------------------------------------------- internals
def _workspace(g: DeviceGraph, fanouts, batch_size: int) -> SampleWorkspace:
    cache = g.__dict__.setdefault("_sample_ws", {})
    key = (tuple(fanouts), batch_size)
    ws = cache.get(key)
    if ws is None:
        if len(cache) > 8:
            cache.clear()
        ws = SampleWorkspace(g, fanouts, batch_size)
        cache[key] = ws
    return ws


def _as_cache(g: DeviceGraph, cached_mask):
    if cached_mask is None or isinstance(cached_mask, DeviceCache):
        return cached_mask
    return DeviceCache(g, cached_mask)


def _run_hops(g, targets, fanouts, rng: PhiloxStream, cache, hop0: int = 0):
    tg = torch.as_tensor(np.asarray(targets, dtype=np.int64)) if not isinstance(
        targets, torch.Tensor) else targets
    tg = tg.to(device=g.device, dtype=torch.int32).flatten()
    n = int(tg.numel())
    if n == 0:
        raise SamplingError("empty target set")
    if int(tg.min()) < 0 or int(tg.max()) >= g.num_nodes:
        raise ValueError("target id out of range")
    ws = _workspace(g, fanouts, n)
    ws.targets[:n].copy_(tg)
    ws.n_targets.fill_(n)
    stream = current_stream(g.device)
    if hop0 == 0:
        ws.launch(cache, stream, seed=rng.seed, epoch=rng.epoch, batch=rng.batch_id)
    else:  # a lone hop at depth hop0 (node_wise_block called directly)
        from ._lib import lib, ptr
        hb, b = ws.hops[0], ws.bounds[0]
        hot_arc = ptr(cache.hot_arc) if cache is not None else None
        hot_off = ptr(cache.hot_off) if cache is not None else None
        lib().mq_sample_hop(ptr(g.row_off), ptr(g.col), hot_arc, hot_off, ptr(ws.targets),
                            ptr(ws.n_targets), b.n_dst_max, b.fanout, rng.seed & 0xFFFFFFFF,
                            rng.epoch & 0xFFFFFFFF, rng.batch_id & 0xFFFFFFFF, hop0, None,
                            ptr(hb.nbr), ptr(hb.cnt), stream)
        lib().mq_relabel(ptr(ws.targets), ptr(ws.n_targets), b.n_dst_max, ptr(hb.nbr), ptr(hb.cnt),
                         b.fanout, ptr(ws.dpos), ptr(ws.first), ptr(hb.row_ptr), ptr(hb.rows),
                         ptr(hb.cols), ptr(hb.vals), ptr(hb.src_ids), ptr(hb.counts),
                         ptr(ws.scratch), stream)
    counts = torch.stack([hb.counts for hb in ws.hops]).cpu().numpy()
    blocks = []
    nd = n
    dst = tg.clone()
    for h, hb in enumerate(ws.hops):
        n_src, nnz = int(counts[h, 0]), int(counts[h, 1])
        blk = Block(rows=hb.rows[:nnz].clone(), cols=hb.cols[:nnz].clone(),
                    values=hb.vals[:nnz].clone(), src_ids=hb.src_ids[:n_src].clone(),
                    dst_ids=dst, row_ptr=hb.row_ptr[:nd + 1].clone(),
                    dst_in_src=torch.arange(nd, device=g.device, dtype=torch.int32))
        blocks.append(blk)
        dst = blk.src_ids
        nd = n_src
    return blocks


# ---------------------------------------------------------------- public API
def _gcn_arm(g: DeviceGraph, blk: Block) -> LayerBlock:
    """The GCN rows of a SAGE block of the same draws (samplers.py:178-191)."""
    row_ptr, rows, cols, vals = gcn_block_from_sage(g, blk, blk.dst_ids)
    return LayerBlock(rows=rows, cols=cols, values=vals.to(torch.float32), src_ids=blk.src_ids,
                      dst_ids=blk.dst_ids, row_ptr=row_ptr, exact=vals, exact_effective=vals,
                      dst_in_src=blk.dst_in_src)


def _check_arch(arch):
    if arch not in ("sage", "gcn"):
        raise ValueError(f"unknown arch {arch!r}")


def node_wise_block(g: DeviceGraph, dst_ids, fanout: int, rng: PhiloxStream,
                    arch: str = "gcn", cached_mask=None):
    """One node-wise block (samplers.py:142-210) at hop ``rng.hop``: the SAGE
    arm (mean weights 1/s) or the GCN arm (normalised adjacency entries)."""
    _check_arch(arch)
    blk = _run_hops(g, dst_ids, (fanout,), rng, _as_cache(g, cached_mask), hop0=rng.hop)[0]
    return _gcn_arm(g, blk) if arch == "gcn" else blk


def sample_node_wise(g: DeviceGraph, targets, fanout, layers: int, rng: PhiloxStream,
                     arch: str = "gcn", cached_mask=None) -> list:
    """Top-down hops, blocks returned bottom-up (samplers.py:213-226)."""
    _check_arch(arch)
    fanouts = tuple(fanout) if isinstance(fanout, (tuple, list)) else (int(fanout),) * layers
    if len(fanouts) != layers:
        raise ValueError("one fanout per layer required")
    blocks = _run_hops(g, targets, fanouts, rng, _as_cache(g, cached_mask))
    if arch == "gcn":
        blocks = [_gcn_arm(g, b) for b in blocks]
    blocks.reverse()
    return blocks


def build_minibatch(g: DeviceGraph, targets, params: SamplerParams, rng: PhiloxStream,
                    batch_id: int = 0, epoch: int = 0, cached_mask=None) -> MiniBatch:
    """Batch assembly (samplers.py:502-540): the method's blocks, labels,
    input features (gathered on device) and the cache hit/miss count."""
    cache = _as_cache(g, cached_mask)
    dropped = 0
    if params.method in ("gcn", "sage"):
        blocks = sample_node_wise(g, targets, params.hop_fanouts, params.num_layers, rng,
                                  arch=params.method, cached_mask=cache)
    elif params.method == "ladies":
        blocks, dropped = sample_ladies(g, targets, params.nodes_per_layer, params.num_layers,
                                        rng, flat=params.flat, debias=params.debias,
                                        replace=params.replace)
    elif params.method == "fastgcn":
        blocks = sample_fastgcn(g, targets, params.nodes_per_layer, params.num_layers, rng,
                                flat=params.flat, debias=params.debias)
    else:
        raise ValueError(f"unknown method {params.method!r}")
    kept = blocks[-1].dst_ids
    input_ids = blocks[0].src_ids
    hits = misses = 0
    if cache is not None and input_ids.numel():
        hits = int(cache.cached_mask[input_ids.long()].sum().item())
        misses = int(input_ids.numel()) - hits
    feats = gather_features(None, g, input_ids).clone()
    return MiniBatch(batch_id=batch_id, epoch=epoch, target_ids=kept,
                     target_labels=g.labels[kept.long()], layers=tuple(blocks),
                     input_ids=input_ids, features=feats, cache_hits=hits, cache_misses=misses,
                     dropped_targets=dropped, method=params.method)
