"""CPU restatement of GNS-biased node-wise sampling (SAGE arm) — test oracle.

Follows ``mqpipe/samplers.py`` of the reference:

* ``node_wise_block``   — ``samplers.py:142-210`` (SAGE arm ``:192-200``)
* ``sample_node_wise``  — ``samplers.py:213-226`` (extended with per-hop fanouts)
* ``build_minibatch``   — ``samplers.py:502-540`` (node-wise dispatch only)
* ``digest``            — ``samplers.py:63-72``

The reference's ``rng.choice`` is replaced by the injected Philox row stream
(``oracle.philox``), the contract under which the reference itself produced
the golden vectors in ``tests/golden``.

* ``build_csr`` / ``degree_bucket_features`` — ``mqpipe/graph.py:94-149`` (ingest)
"""

from __future__ import annotations

import hashlib

import numpy as np

from .philox import draws, fisher_yates_positions, philox4x32_10


class OracleBlock:
    __slots__ = ("rows", "cols", "values", "src_ids", "dst_ids", "dst_in_src")

    def __init__(self, rows, cols, values, src_ids, dst_ids):
        self.rows = rows
        self.cols = cols
        self.values = values
        self.src_ids = src_ids
        self.dst_ids = dst_ids
        self.dst_in_src = np.arange(dst_ids.size, dtype=np.int64)

    @property
    def effective_values(self):
        return self.values

    @property
    def num_dst(self):
        return int(self.dst_ids.size)

    @property
    def num_src(self):
        return int(self.src_ids.size)


def _choice(pool: np.ndarray, k: int, key, x=None) -> np.ndarray:
    """Injected ``rng.choice(pool, size=k, replace=False)`` (samplers.py:172-177)."""
    if x is None:
        x = draws(*key, count=k)
    return pool[fisher_yates_positions(x, pool.size, k)]


def _row_draws(n_rows, count, seed, epoch, batch_id, hop):
    """x_0..x_{count-1} of every row stream of a hop, vectorised: [n_rows, count]."""
    blocks = (count + 3) // 4
    ctr = np.zeros((n_rows, blocks, 4), dtype=np.uint64)
    ctr[:, :, 0] = np.arange(blocks, dtype=np.uint64)[None, :]
    ctr[:, :, 1] = np.arange(n_rows, dtype=np.uint64)[:, None] & np.uint64(0xFFFFFFFF)
    ctr[:, :, 2] = hop & 0xFFFFFFFF
    ctr[:, :, 3] = batch_id & 0xFFFFFFFF
    key = np.array([seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF], dtype=np.uint64)
    return philox4x32_10(ctr, key).reshape(n_rows, blocks * 4)[:, :count]


def node_wise_block(row_offsets, col_indices, dst_ids, fanout: int, *, seed: int,
                    epoch: int, batch_id: int, hop: int, cached_mask=None):
    """One SAGE block (samplers.py:142-210, arch == 'sage')."""
    dst_ids = np.asarray(dst_ids, dtype=np.int64)
    src_list = list(dst_ids.tolist())
    # last occurrence wins, as with the dict comprehension at samplers.py:156
    src_pos = {int(v): i for i, v in enumerate(dst_ids)}
    rows, cols, vals = [], [], []
    xs = _row_draws(dst_ids.size, fanout, seed, epoch, batch_id, hop) if dst_ids.size else None
    for r, v in enumerate(dst_ids.tolist()):
        nbrs = col_indices[row_offsets[v]:row_offsets[v + 1]]
        nbrs = nbrs[nbrs != v]                      # samplers.py:162
        n = nbrs.size
        key = (seed, epoch, batch_id, hop, r)
        if n <= fanout:                             # :164-167
            sampled = nbrs
        elif cached_mask is not None:               # :168-175
            hot_sel = cached_mask[nbrs]
            hot, cold = nbrs[hot_sel], nbrs[~hot_sel]
            if hot.size >= fanout:
                sampled = _choice(hot, fanout, key, xs[r])
            else:
                sampled = np.concatenate(
                    [hot, _choice(cold, fanout - hot.size, key, xs[r])])
        else:                                       # :176-177
            sampled = _choice(nbrs, fanout, key, xs[r])
        s = sampled.size
        for u in sampled.tolist():                  # :192-200
            if u not in src_pos:
                src_pos[u] = len(src_list)
                src_list.append(u)
            rows.append(r)
            cols.append(src_pos[u])
            vals.append(1.0 / s)
    return OracleBlock(np.asarray(rows, dtype=np.int64),
                       np.asarray(cols, dtype=np.int64),
                       np.asarray(vals, dtype=np.float64),
                       np.asarray(src_list, dtype=np.int64), dst_ids)


def sample_node_wise(row_offsets, col_indices, targets, fanouts, *, seed, epoch,
                     batch_id, cached_mask=None):
    """Hop chaining top-down, blocks returned bottom-up (samplers.py:213-226).

    ``fanouts[h]`` is applied at hop h counted from the seeds.
    """
    dst = np.asarray(targets, dtype=np.int64)
    if dst.size == 0:
        raise ValueError("empty target set")        # SamplingError in the reference
    blocks = []
    for hop, f in enumerate(fanouts):
        blk = node_wise_block(row_offsets, col_indices, dst, int(f), seed=seed,
                              epoch=epoch, batch_id=batch_id, hop=hop,
                              cached_mask=cached_mask)
        blocks.append(blk)
        dst = blk.src_ids
    blocks.reverse()
    return blocks


class OracleMiniBatch:
    def __init__(self, batch_id, epoch, target_ids, target_labels, layers,
                 input_ids, features, hits, misses):
        self.batch_id = batch_id
        self.epoch = epoch
        self.target_ids = target_ids
        self.target_labels = target_labels
        self.layers = tuple(layers)
        self.input_ids = input_ids
        self.features = features
        self.cache_hits = hits
        self.cache_misses = misses

    def digest(self) -> str:
        """SHA-256 over ids, triplets and features (samplers.py:63-72)."""
        return digest_of(self.target_ids, self.layers, self.features)


def digest_of(target_ids, layers, features) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(target_ids, dtype=np.int64).tobytes())
    for blk in layers:
        h.update(np.ascontiguousarray(blk.rows, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(blk.cols, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(blk.values, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(blk.src_ids, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(blk.dst_ids, dtype=np.int64).tobytes())
    if features is not None:
        h.update(np.ascontiguousarray(features, dtype=np.float32).tobytes())
    return h.hexdigest()


def build_minibatch(row_offsets, col_indices, features, labels, targets, fanouts,
                    *, seed, epoch, batch_id, cached_mask=None):
    """Node-wise arm of build_minibatch (samplers.py:502-540)."""
    targets = np.asarray(targets, dtype=np.int64)
    blocks = sample_node_wise(row_offsets, col_indices, targets, fanouts,
                              seed=seed, epoch=epoch, batch_id=batch_id,
                              cached_mask=cached_mask)
    kept = blocks[-1].dst_ids
    input_ids = blocks[0].src_ids
    hits = misses = 0
    if cached_mask is not None and input_ids.size:
        hits = int(np.count_nonzero(cached_mask[input_ids]))
        misses = int(input_ids.size - hits)
    return OracleMiniBatch(batch_id, epoch, kept, labels[kept], blocks,
                           input_ids, features[input_ids].copy(), hits, misses)


def build_csr(edges, num_nodes):
    """graph.py:94-139: (row_offsets, col_indices) of the deduplicated,
    sorted arc set (np.unique of src * n + dst)."""
    arr = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if arr.size and (arr.min() < 0 or arr.max() >= num_nodes):
        raise ValueError("edge endpoint out of range")
    keys = np.unique(arr[:, 0] * num_nodes + arr[:, 1]) if arr.size else np.empty(0, np.int64)
    src, dst = keys // num_nodes, keys % num_nodes
    row_offsets = np.zeros(num_nodes + 1, dtype=np.int64)
    np.add.at(row_offsets, src + 1, 1)
    return np.cumsum(row_offsets), dst.copy()


def degree_bucket_features(row_offsets):
    """graph.py:142-149: one-hot of floor(log2(out_degree + 1))."""
    deg = np.diff(row_offsets)
    buckets = np.floor(np.log2(deg + 1)).astype(np.int64)
    dim = int(buckets.max()) + 1 if buckets.size else 1
    feats = np.zeros((deg.size, dim), dtype=np.float32)
    feats[np.arange(deg.size), buckets] = 1.0
    return feats
