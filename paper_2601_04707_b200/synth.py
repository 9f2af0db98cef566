"""Synthetic power-law graphs of the benchmark shapes (measurement infra).

The reference's own generator (``graph.py:252-289``, configuration model on
zipf degrees) cannot target an edge count and took minutes at Reddit scale
(SURVEY.md §2 C0b, §8d).  This Chung-Lu variant draws one endpoint of every
edge proportional to a power-law weight (exponent 2.1, the reference default)
and the other uniformly, stores both arcs, drops self loops and dedups —
i.e. exactly ``build_csr`` semantics (``graph.py:94-139``: sorted rows,
unique arcs) — topping up until the arc target is reached.

``generate_numpy`` is deterministic NumPy (small graphs, golden fixtures);
``generate_torch`` runs the same construction with torch ops on a GPU for the
114M-arc benchmark shape.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SHAPES = {
    # configs[0]: the reference's CPU-runnable case
    "cfg1": dict(num_nodes=10_000, num_arcs=100_000, feature_dim=64, num_classes=4,
                 fanouts=(10, 5), train=0.66),
    # configs[1]: Reddit-shaped, 1 B200 (the headline workload)
    "reddit": dict(num_nodes=232_965, num_arcs=114_000_000, feature_dim=602, num_classes=41,
                   fanouts=(10, 5), train=0.66),
    # configs[2..3]: ogbn-products-shaped
    "products": dict(num_nodes=2_449_029, num_arcs=62_000_000, feature_dim=100, num_classes=47,
                     fanouts=(15, 10, 5), train=0.08),
    # configs[4]: ogbn-papers100M-shaped (1.1% training nodes, as the OGB split);
    # CSR (7.3 GB) + features (57 GB) fit one B200's 180 GB HBM
    "papers": dict(num_nodes=111_059_956, num_arcs=1_600_000_000, feature_dim=128,
                   num_classes=172, fanouts=(15, 10, 5), train=0.011),
}


@dataclass
class SynthGraph:
    """Duck-typed stand-in for the reference ``GraphCSR`` (graph.py:28-91)."""

    num_nodes: int
    row_offsets: object      # int64 [n+1]
    col_indices: object      # int32/int64 [E]
    features: object         # f32 [n, d]
    labels: object           # int32 [n]
    num_classes: int
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray

    @property
    def num_edges(self) -> int:
        return int(self.col_indices.shape[0])

    @property
    def feature_dim(self) -> int:
        return int(self.features.shape[1])


def _weights(num_nodes, exponent, rng_perm):
    w = (np.arange(num_nodes, dtype=np.float64) + 1.0) ** (-1.0 / (exponent - 1.0))
    return w[rng_perm]


def split_masks(num_nodes, ratios, seed):
    """Disjoint floor-sized splits, as ``split_masks`` (graph.py:220-249)."""
    rng = np.random.default_rng(seed)
    order = rng.permutation(num_nodes)
    n_train = int(ratios[0] * num_nodes)
    n_val = int(ratios[1] * num_nodes)
    n_test = int(ratios[2] * num_nodes)
    masks = []
    lo = 0
    for k in (n_train, n_val, n_test):
        m = np.zeros(num_nodes, dtype=bool)
        m[order[lo:lo + k]] = True
        masks.append(m)
        lo += k
    return masks


def ratios_for(train):
    rest = 1.0 - train
    return (train, rest * 0.3, rest * 0.7)


def chung_lu_keys_numpy(num_nodes, num_arcs, exponent=2.1, seed=0):
    """Sorted unique arc keys src*n+dst (symmetric, no self loops)."""
    rng = np.random.default_rng(seed)
    w = _weights(num_nodes, exponent, rng.permutation(num_nodes))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    n = np.int64(num_nodes)
    keys = np.empty(0, dtype=np.int64)
    while keys.size < num_arcs:
        need = num_arcs - keys.size
        m = int(need * 0.55) + 16
        src = np.minimum(np.searchsorted(cdf, rng.random(m), side="right"), num_nodes - 1)
        dst = rng.integers(0, num_nodes, m)
        keep = src != dst
        s, d = src[keep].astype(np.int64), dst[keep].astype(np.int64)
        keys = np.unique(np.concatenate([keys, s * n + d, d * n + s]))
    return keys


def keys_to_csr(keys, num_nodes):
    src = keys // num_nodes
    col = (keys % num_nodes).astype(np.int64)
    counts = np.bincount(src, minlength=num_nodes)
    row_offsets = np.zeros(num_nodes + 1, dtype=np.int64)
    np.cumsum(counts, out=row_offsets[1:])
    return row_offsets, col


def teacher_labels_numpy(features, num_classes, seed):
    rng = np.random.default_rng(seed)
    proj = rng.standard_normal((features.shape[1], num_classes)).astype(np.float32)
    return np.argmax(features @ proj, axis=1).astype(np.int32)


def generate_numpy(num_nodes, num_arcs, feature_dim, num_classes, *, train=0.66,
                   exponent=2.1, seed=0) -> SynthGraph:
    """Deterministic small-graph generator (seeds: graph s, features s+1,
    labels s+2, splits s+4)."""
    keys = chung_lu_keys_numpy(num_nodes, num_arcs, exponent, seed)
    row_offsets, col = keys_to_csr(keys, num_nodes)
    feats = np.random.default_rng(seed + 1).standard_normal(
        (num_nodes, feature_dim), dtype=np.float32)
    labels = teacher_labels_numpy(feats, num_classes, seed + 2)
    tr, va, te = split_masks(num_nodes, ratios_for(train), seed + 4)
    return SynthGraph(num_nodes, row_offsets, col, feats, labels, num_classes, tr, va, te)


def generate_torch(num_nodes, num_arcs, feature_dim, num_classes, *, train=0.66,
                   exponent=2.1, seed=0, device="cuda", feature_shard=None) -> SynthGraph:
    """Same construction with torch ops (GPU); arrays stay on ``device``.

    Masks are NumPy (host) like the reference's; row_offsets int64, col int32.
    Features are drawn in fixed row chunks, so ``feature_shard=(G, r)`` —
    keep only rows v = r, r + G, ... (the seed-partitioned store) — yields
    exactly those rows of the unsharded table; labels always see every row.
    """
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    n = num_nodes
    perm = torch.randperm(n, generator=gen, device=device)
    w = (torch.arange(n, device=device, dtype=torch.float64) + 1.0) ** (-1.0 / (exponent - 1.0))
    w = w[perm]
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < num_arcs:
        need = num_arcs - keys.numel()
        m = int(need * 0.55) + 16
        u = torch.rand(m, generator=gen, device=device, dtype=torch.float64)
        src = torch.clamp(torch.searchsorted(cdf, u, right=True), max=n - 1)
        dst = torch.randint(0, n, (m,), generator=gen, device=device)
        keep = src != dst
        s, d = src[keep], dst[keep]
        cat = torch.cat([keys, s * n + d, d * n + s])
        del s, d, src, dst, u, keep
        keys = torch.unique(cat, sorted=True)
        del cat
    src = keys // n
    col = (keys - src * n).to(torch.int32)
    counts = torch.bincount(src, minlength=n)
    del keys, src
    row_offsets = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=row_offsets[1:])
    del counts
    proj = torch.randn((feature_dim, num_classes), generator=gen, device=device)
    labels = torch.empty(n, dtype=torch.int32, device=device)
    G, r = feature_shard if feature_shard is not None else (1, 0)
    feats = torch.empty(((n - r + G - 1) // G, feature_dim), dtype=torch.float32, device=device)
    chunk = 1 << 20  # a multiple of every shard count <= 8
    for lo in range(0, n, chunk):  # [n x C] logits would be 76 GB at papers
        hi = min(n, lo + chunk)
        x = torch.randn((hi - lo, feature_dim), generator=gen, device=device, dtype=torch.float32)
        labels[lo:hi] = torch.argmax(x @ proj, dim=1).to(torch.int32)
        first = (r - lo) % G  # first row of this chunk owned by shard r
        feats[(lo + first - r) // G:(lo + first - r) // G + len(range(first, hi - lo, G))] = \
            x[first::G]
        del x
    tr, va, te = split_masks(n, ratios_for(train), seed + 4)
    return SynthGraph(n, row_offsets, col, feats, labels, num_classes, tr, va, te)


def generate_shape(name: str, seed: int = 0, device: str | None = None, feature_shard=None,
                   **overrides):
    spec = dict(SHAPES[name])
    spec.update(overrides)
    fanouts = spec.pop("fanouts")
    train = spec.pop("train")
    if device is None or device == "cpu":
        g = generate_numpy(spec["num_nodes"], spec["num_arcs"], spec["feature_dim"],
                           spec["num_classes"], train=train, seed=seed)
    else:
        g = generate_torch(spec["num_nodes"], spec["num_arcs"], spec["feature_dim"],
                           spec["num_classes"], train=train, seed=seed, device=device,
                           feature_shard=feature_shard)
    return g, tuple(fanouts)


def degree_cache_mask(col_indices, num_nodes, fraction):
    """Deterministic top-in-degree residency (ties -> lower id), the expected
    content of the reference's degree-mode cache (cache.py:41-48, 79-108)
    without its random draw; used for the benchmark shapes."""
    budget = int(math.ceil(fraction * num_nodes))
    try:
        import torch
        if isinstance(col_indices, torch.Tensor):
            indeg = torch.bincount(col_indices.long(), minlength=num_nodes)
            order = torch.argsort(-indeg, stable=True)[:budget]
            mask = torch.zeros(num_nodes, dtype=torch.bool, device=col_indices.device)
            mask[order] = True
            return mask
    except ImportError:  # pragma: no cover
        pass
    indeg = np.bincount(np.asarray(col_indices), minlength=num_nodes)
    order = np.argsort(-indeg, kind="stable")[:budget]
    mask = np.zeros(num_nodes, dtype=bool)
    mask[order] = True
    return mask
