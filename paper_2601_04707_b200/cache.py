"""GNS feature cache on the device: residency bitmap, O(fanout) residency
index for the sampler, slot map and the HBM cache table.

Reference: ``mqpipe/cache.py`` —
  * ``CacheState`` (``cache.py:20-38``): sorted ``cached_ids``, bool
    ``cached_mask``, ``cached_features`` copy, locked hit/miss counters;
  * ``lookup`` / ``gather_features`` (``cache.py:111-134``);
  * ``cache_probs_degree`` / ``cache_probs_walk`` / ``refresh_cache``
    (``cache.py:41-108``) — per-epoch residency, on the device
    (mq_refresh.cu) under the refresh injected-draw contract.

Per-epoch device structures built from the mask:
  * ``bits``      uint32 [ceil(n/32)] residency bitmap;
  * ``hot_arc``   int64 [H] arcs whose head is resident, ``hot_off`` int64
    [n+1] — the sampler's hot/cold split in O(fanout) per row;
  * ``slot_of``   int32 [n] rank among resident ids (−1 = miss);
  * ``table``     f32 [|C|, pitch] HBM copy of the resident rows.
"""

from __future__ import annotations

import math
import threading

import numpy as np
import torch

from ._lib import lib, ptr
from .graph import DeviceGraph


class DeviceCache:
    """Device form of ``CacheState``; counters are device u64 accumulators."""

    def __init__(self, g: DeviceGraph, cached_mask, fraction: float | None = None):
        dev = g.device
        n = g.num_nodes
        mask = cached_mask
        if isinstance(mask, np.ndarray) or not isinstance(mask, torch.Tensor):
            mask = torch.as_tensor(np.asarray(mask, dtype=bool))
        mask = mask.to(device=dev, dtype=torch.bool)
        if mask.shape != (n,):
            raise ValueError("cached_mask must have one entry per node")
        self.graph = g
        self.fraction = fraction
        self.cached_mask = mask
        self.cached_ids = torch.nonzero(mask).flatten()           # ascending ids
        self.size = int(self.cached_ids.numel())
        self.bits = _pack_bits(mask)
        stream = torch.cuda.current_stream(dev).cuda_stream
        with torch.cuda.device(dev):
            scr = torch.empty(int(lib().mq_scan_scratch_bytes(max(g.num_arcs, n, 1))),
                              dtype=torch.uint8, device=dev)
            hot_arc = torch.empty(max(g.num_arcs, 1), dtype=torch.int64, device=dev)
            self.hot_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
            n_hot = torch.zeros(1, dtype=torch.int64, device=dev)
            lib().mq_residency_index(ptr(g.row_off), ptr(g.col), n, g.num_arcs, ptr(self.bits),
                                     ptr(hot_arc), ptr(self.hot_off), ptr(n_hot), ptr(scr), stream)
            self.num_hot_arcs = int(n_hot.item())
            self.hot_arc = hot_arc[:max(self.num_hot_arcs, 1)].clone()
            del hot_arc
            self.slot_of = torch.empty(n, dtype=torch.int32, device=dev)
            n_res = torch.zeros(1, dtype=torch.int32, device=dev)
            lib().mq_residency_slots(ptr(self.bits), n, ptr(self.slot_of), ptr(n_res), ptr(scr),
                                     stream)
            table = torch.zeros((max(self.size, 1), g.pitch), dtype=torch.float32, device=dev)
            if self.size:
                ids32 = self.cached_ids.to(torch.int32)
                nd = torch.tensor([self.size], dtype=torch.int32, device=dev)
                g.gather_rows(ids32, nd, self.size, table, g.pitch, stream)
            self.table = table
            self.hit_miss = torch.zeros(2, dtype=torch.int64, device=dev)
        self._lock = threading.Lock()
        self._host_hits = 0
        self._host_misses = 0

    # CacheState-compatible counters (cache.py:28-38)
    @property
    def hits(self) -> int:
        return int(self.hit_miss[0].item()) + self._host_hits

    @property
    def misses(self) -> int:
        return int(self.hit_miss[1].item()) + self._host_misses

    def hit_rate(self) -> float:
        total = self.hits + self.misses
        return self.hits / total if total else 0.0

    @property
    def cached_features(self) -> torch.Tensor:
        return self.table[:self.size, :self.graph.feature_dim]


def _pack_bits(mask: torch.Tensor) -> torch.Tensor:
    n = mask.numel()
    words = (n + 31) // 32
    padded = torch.zeros(words * 32, dtype=torch.int64, device=mask.device)
    padded[:n] = mask.to(torch.int64)
    weights = (torch.ones(32, dtype=torch.int64, device=mask.device)
               << torch.arange(32, device=mask.device, dtype=torch.int64))
    packed = (padded.view(words, 32) * weights).sum(dim=1)
    # two's-complement wrap into int32 storage, read as uint32 by the kernels
    packed = torch.where(packed >= 2 ** 31, packed - 2 ** 32, packed)
    return packed.to(torch.int32).contiguous()


# ---------------------------------------------------------------- per-epoch
class RefreshStream:
    """Key of the per-epoch refresh's injected draws (oracle/philox.py
    RefreshRng): ``random(n)`` and the shortfall ``choice`` come from reserved
    Philox row streams of (seed, epoch), so the device refresh reproduces the
    reference's refresh_cache driven by the same draws."""

    def __init__(self, seed: int, epoch: int = 0):
        self.seed, self.epoch = int(seed), int(epoch)

    def uniforms(self, n) -> np.ndarray:
        """random(n) of the contract (the library's host restatement; tests)."""
        out = np.empty(int(n), dtype=np.float64)
        lib().mq_refresh_uniforms_host(self.seed, self.epoch, int(n),
                                       out.ctypes.data if n else None)
        return out


def _stream(g):
    return torch.cuda.current_stream(g.device).cuda_stream


def cache_probs_degree(g: DeviceGraph) -> torch.Tensor:
    """In-degree importance (cache.py:41-48) as a device f64 tensor."""
    deg = g.in_degrees()
    probs = torch.empty(max(g.num_nodes, 1), dtype=torch.float64, device=g.device)
    lib().mq_degree_probs(ptr(deg), g.num_nodes, g.num_edges, ptr(probs), _stream(g))
    return probs[:g.num_nodes]


def cache_probs_walk(g: DeviceGraph, fanout: int, steps: int) -> torch.Tensor:
    """Sampling-reachability walk p <- D A p + p from the training set
    (cache.py:51-76), bit-exact, as a device f64 tensor."""
    train = np.asarray(g.train_mask, dtype=bool)
    n_train = int(train.sum())
    if n_train == 0:
        raise ValueError("walk probabilities need a nonempty training set")
    dev = g.device
    deg = g.in_degrees()
    tm = torch.as_tensor(train.astype(np.uint8)).to(dev)
    probs = torch.empty(g.num_nodes, dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    scr = torch.empty(int(lib().mq_walk_scratch_bytes(g.num_nodes)), dtype=torch.uint8, device=dev)
    lib().mq_walk_probs(ptr(g.row_off), ptr(g.col), g.num_nodes, ptr(g.loops), ptr(deg), ptr(tm),
                        n_train, int(fanout), int(steps), ptr(probs), ptr(bad), ptr(scr),
                        _stream(g))
    if int(bad.item()):
        raise ValueError("walk produced no probability mass")
    return probs


def refresh_mask(g: DeviceGraph, probs: torch.Tensor, fraction: float,
                 key: RefreshStream) -> torch.Tensor:
    """Device resident set of refresh_cache (cache.py:79-108) as a bool mask."""
    if not (0.0 < fraction <= 1.0):
        raise ValueError("fraction must lie in (0, 1]")
    n = g.num_nodes
    dev = g.device
    probs = torch.as_tensor(probs, dtype=torch.float64).to(dev).contiguous()
    if probs.shape != (n,):
        raise ValueError("probs must have one entry per node")
    budget = int(math.ceil(fraction * n))
    chosen = torch.empty(n, dtype=torch.uint8, device=dev)
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    scr = torch.empty(int(lib().mq_refresh_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    lib().mq_refresh_select(ptr(probs), n, budget, key.seed, key.epoch, ptr(chosen), ptr(counts),
                            ptr(scr), _stream(g))
    return chosen.view(torch.bool)


def weighted_sample_without_replacement(weights, k: int, rng) -> np.ndarray:
    """Exponential-key WOR draw (samplers.py:113-135), host form for a
    caller-supplied generator (the device refresh does not use it)."""
    w = np.asarray(weights, dtype=np.float64)
    if np.any(w < 0) or not np.all(np.isfinite(w)):
        raise ValueError("weights must be finite and nonnegative")
    positive = np.flatnonzero(w > 0)
    if k < 0 or k > positive.size:
        raise ValueError(f"k={k} out of range for {positive.size} positive weights")
    if k == 0:
        return np.empty(0, dtype=np.int64)
    u = rng.random(positive.size)
    keys = u ** (1.0 / w[positive])
    order = np.lexsort((positive, -keys))
    return positive[order[:k]].astype(np.int64)


def refresh_cache(g: DeviceGraph, probs, fraction: float, rng) -> DeviceCache:
    """ceil(fraction * |V|) residents drawn WOR by probs (cache.py:79-108).

    With a :class:`RefreshStream` key (the injected-draw contract) the whole
    selection runs on the device (mq_refresh_select).  Any other ``rng``
    (e.g. a NumPy Generator, whose draw stream a GPU cannot replay) is
    honoured on the host, as the reference does."""
    if isinstance(rng, RefreshStream):
        return DeviceCache(g, refresh_mask(g, probs, fraction, rng), fraction)
    if not (0.0 < fraction <= 1.0):
        raise ValueError("fraction must lie in (0, 1]")
    if isinstance(probs, torch.Tensor):
        probs = probs.detach().cpu().numpy()
    probs = np.asarray(probs, dtype=np.float64)
    if probs.shape != (g.num_nodes,):
        raise ValueError("probs must have one entry per node")
    budget = int(math.ceil(fraction * g.num_nodes))
    positive = int(np.count_nonzero(probs > 0))
    take = min(budget, positive)
    chosen = weighted_sample_without_replacement(probs, take, rng)
    if take < budget:
        rest = np.setdiff1d(np.arange(g.num_nodes), chosen)
        extra = rng.choice(rest, size=budget - take, replace=False)
        chosen = np.concatenate([chosen, extra])
    mask = np.zeros(g.num_nodes, dtype=bool)
    mask[chosen] = True
    return DeviceCache(g, mask, fraction)


# ---------------------------------------------------------------- per batch
def lookup(cache: DeviceCache, ids):
    """Order-preserving (hits, misses) partition; bumps counters (cache.py:111-120)."""
    ids = _ids_tensor(ids, cache.graph.device)
    hit = cache.cached_mask[ids.long()]
    hits, misses = ids[hit], ids[~hit]
    with cache._lock:
        cache._host_hits += int(hits.numel())
        cache._host_misses += int(misses.numel())
    return hits, misses


def gather_features(cache: DeviceCache | None, g: DeviceGraph, ids, *, out=None,
                    out_pitch=None, count_hits: bool = False) -> torch.Tensor:
    """Feature rows for ids: hits from the HBM cache table, misses from the
    store (HBM or pinned host) — cache.py:123-134.  Returns f32 [n, d]."""
    ids = _ids_tensor(ids, g.device)
    n = int(ids.numel())
    n_dev = torch.tensor([n], dtype=torch.int32, device=g.device)
    pitch = out_pitch or g.pitch
    if out is None:
        out = torch.empty((max(n, 1), pitch), dtype=torch.float32, device=g.device)
    stream = torch.cuda.current_stream(g.device).cuda_stream
    hm = None
    if cache is not None:
        hm = cache.hit_miss if count_hits else torch.zeros(2, dtype=torch.int64, device=g.device)
    g.gather_rows(ids, n_dev, n, out, pitch, stream, cache=cache, hit_miss=hm)
    return out[:n, :g.feature_dim]


def _ids_tensor(ids, device):
    if isinstance(ids, torch.Tensor):
        return ids.to(device=device, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.asarray(ids, dtype=np.int64).astype(np.int32), device=device)
