"""CPU restatement of the GNS cache's per-batch lookup and gather — test oracle.

* ``lookup``          — ``mqpipe/cache.py:111-120``
* ``gather_features`` — ``mqpipe/cache.py:123-134``
* ``degree_probs``    — ``mqpipe/cache.py:41-48``
* ``walk_probs``      — ``mqpipe/cache.py:51-76``
* ``weighted_sample_without_replacement`` — ``mqpipe/samplers.py:113-135``
* ``refresh_cache_ids`` — ``mqpipe/cache.py:79-108`` (resident ids)
"""

from __future__ import annotations

import numpy as np


def lookup(cached_mask, ids):
    """Order-preserving hit/miss partition (cache.py:111-120)."""
    ids = np.asarray(ids, dtype=np.int64)
    hit = cached_mask[ids]
    return ids[hit], ids[~hit]


def gather_features(cached_ids, cached_mask, cached_features, features, ids):
    """Hits from the cache copy, misses from the store (cache.py:123-134)."""
    ids = np.asarray(ids, dtype=np.int64)
    if cached_ids is None:
        return features[ids].copy()
    out = np.empty((ids.size, features.shape[1]), dtype=features.dtype)
    hit = cached_mask[ids]
    pos = np.searchsorted(cached_ids, ids[hit])
    out[hit] = cached_features[pos]
    out[~hit] = features[ids[~hit]]
    return out


def degree_probs(col_indices, num_nodes):
    """In-degree importance (cache.py:41-48)."""
    deg = np.bincount(col_indices, minlength=num_nodes).astype(np.float64)
    total = deg.sum()
    if total == 0:
        return np.full(num_nodes, 1.0 / num_nodes)
    return deg / total


def walk_probs(row_offsets, col_indices, train_mask, fanout, steps):
    """Sampling-reachability walk p <- D A p + p (cache.py:51-76)."""
    n = train_mask.size
    train_ids = np.flatnonzero(train_mask)
    if train_ids.size == 0:
        raise ValueError("walk probabilities need a nonempty training set")
    p = np.zeros(n, dtype=np.float64)
    p[train_ids] = 1.0 / train_ids.size
    indeg = np.bincount(col_indices, minlength=n).astype(np.float64)
    d = np.zeros(n, dtype=np.float64)
    nz = indeg > 0
    d[nz] = np.minimum(fanout, indeg[nz]) / indeg[nz]
    src = np.repeat(np.arange(n), np.diff(row_offsets))
    for _ in range(steps):
        flow = np.bincount(src, weights=p[col_indices], minlength=n)
        p = d * flow + p
    total = p.sum()
    if total <= 0:
        raise ValueError("walk produced no probability mass")
    return p / total


def weighted_sample_without_replacement(weights, k, rng):
    """Exponential keys u^(1/w), descending, ties to the lower index
    (samplers.py:113-135)."""
    w = np.asarray(weights, dtype=np.float64)
    positive = np.flatnonzero(w > 0)
    if k > positive.size:
        raise ValueError(f"k={k} exceeds {positive.size} positive weights")
    if k == 0:
        return np.empty(0, dtype=np.int64)
    u = rng.random(positive.size)
    keys = u ** (1.0 / w[positive])
    order = np.lexsort((positive, -keys))
    return positive[order[:k]].astype(np.int64)


def refresh_cache_ids(num_nodes, probs, fraction, rng):
    """Resident ids of refresh_cache (cache.py:79-108): ceil(f*|V|) drawn WOR
    by probs, shortfall filled uniformly from the zero-probability rest."""
    if not (0.0 < fraction <= 1.0):
        raise ValueError("fraction must lie in (0, 1]")
    probs = np.asarray(probs, dtype=np.float64)
    budget = int(np.ceil(fraction * num_nodes))
    positive = int(np.count_nonzero(probs > 0))
    take = min(budget, positive)
    chosen = weighted_sample_without_replacement(probs, take, rng)
    if take < budget:
        rest = np.setdiff1d(np.arange(num_nodes), chosen, assume_unique=False)
        extra = rng.choice(rest, size=budget - take, replace=False)
        chosen = np.concatenate([chosen, extra])
    return np.sort(chosen.astype(np.int64))
