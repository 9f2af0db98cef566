"""CPU restatement of the GNS cache's per-batch lookup and gather — test oracle.

* ``lookup``          — ``mqpipe/cache.py:111-120``
* ``gather_features`` — ``mqpipe/cache.py:123-134``
* ``degree_probs``    — ``mqpipe/cache.py:41-48``
* ``walk_probs``      — ``mqpipe/cache.py:51-76``
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
