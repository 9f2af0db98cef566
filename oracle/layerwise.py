"""CPU restatement of the layer-wise samplers and the GCN block arm — TEST ORACLE.

Test infrastructure only (see ``oracle/__init__.py``).  Follows
``mqpipe/samplers.py`` of the reference:

* ``_slice_csr`` / ``_restricted_rows``   — ``samplers.py:233-262``
* ``ladies_candidates``                   — ``samplers.py:265-271``
* ``_candidate_norms``                    — ``samplers.py:274-283``
* ``ladies_probs`` / ``flat_probs``       — ``samplers.py:286-311``
* ``fastgcn_probs``                       — ``samplers.py:314-318``
* ``debias_coefficients``                 — ``samplers.py:353-373``
* ``_layer_wise_block``                   — ``samplers.py:376-440``
* ``sample_ladies`` / ``sample_fastgcn``  — ``samplers.py:443-495``
* ``build_minibatch`` (layer-wise arms)   — ``samplers.py:502-540``
* ``node_wise_block`` GCN arm values      — ``samplers.py:178-191``

Injected draws (the layer-wise contract, pinned by ``tests/golden/
make_golden_layerwise.py`` which drives the reference's own functions through
``LayerRng``): a batch's rng makes exactly one public call per layer
(``random`` for the WOR arms, ``choice(.., replace=True, p=..)`` for the
with-replacement arm), and call l (0 = the targets' layer) draws from the
Philox stream (seed, epoch; ctr (i, 0xFFFFFFFF, l, batch_id)):

    random(n)[i]  = ((x_{4i} >> 5) * 2^26 + (x_{4i+1} >> 6)) * 2^-53
    choice(m, s, replace=True, p) = NumPy's Generator.choice algorithm:
        cdf = cumsum(p); cdf /= cdf[-1]; searchsorted(cdf, random(s), 'right')
"""

from __future__ import annotations

import numpy as np

from .cache import weighted_sample_without_replacement
from .philox import draws

LW_ROW = 0xFFFFFFFF


class SamplingError(RuntimeError):
    pass


def layer_uniforms(seed: int, epoch: int, batch_id: int, layer: int, n: int) -> np.ndarray:
    """random(n) of layer ``layer``'s stream (module docstring)."""
    if n <= 0:
        return np.empty(0, dtype=np.float64)
    x = draws(seed, epoch, batch_id, layer, LW_ROW, 4 * n).reshape(n, 4)
    hi = (x[:, 0] >> np.uint32(5)).astype(np.float64)
    lo = (x[:, 1] >> np.uint32(6)).astype(np.float64)
    return (hi * 67108864.0 + lo) / 9007199254740992.0


class LayerRng:
    """Duck-typed ``rng`` of one batch: the k-th public call is layer k."""

    def __init__(self, seed: int, epoch: int, batch_id: int):
        self.seed, self.epoch, self.batch_id = int(seed), int(epoch), int(batch_id)
        self.calls = 0

    def _uniforms(self, n):
        return layer_uniforms(self.seed, self.epoch, self.batch_id, self.calls, int(n))

    def random(self, n):
        u = self._uniforms(n)
        self.calls += 1
        return u

    def choice(self, a, size, replace=True, p=None):
        if not replace or p is None:
            raise ValueError("the layer-wise contract draws weighted, with replacement")
        m = int(a) if np.ndim(a) == 0 else len(a)
        p = np.asarray(p, dtype=np.float64)
        if p.shape != (m,):
            raise ValueError("p must match the population")
        cdf = np.cumsum(p)
        cdf /= cdf[-1]
        idx = np.searchsorted(cdf, self._uniforms(size), side="right")
        self.calls += 1
        return idx if np.ndim(a) == 0 else np.asarray(a)[idx]


# --------------------------------------------------------------------- graph
def a_hat_degrees(row_offsets, col_indices):
    """Row sums of A + I (graph.py:53-60): out-degree, +1 unless a loop is stored."""
    n = row_offsets.size - 1
    out = np.diff(row_offsets)
    owner = np.repeat(np.arange(n), out)
    loop = np.zeros(n, dtype=bool)
    loop[owner[col_indices == owner]] = True
    return (out + (~loop)).astype(np.int64)


def csr_slice(row_offsets, col_indices, nodes):
    """(local row, neighbour id) of every stored entry of ``nodes``, row-major."""
    nodes = np.asarray(nodes, dtype=np.int64)
    lo = row_offsets[nodes].astype(np.int64)
    cnt = row_offsets[nodes + 1].astype(np.int64) - lo
    local = np.repeat(np.arange(nodes.size, dtype=np.int64), cnt)
    first = np.cumsum(cnt) - cnt
    pos = np.arange(int(cnt.sum()), dtype=np.int64) - np.repeat(first, cnt) + np.repeat(lo, cnt)
    return local, col_indices[pos].astype(np.int64)


def restricted_rows(row_offsets, col_indices, deg_hat, prev):
    """Rows of D^-1/2 (A+I) D^-1/2 for ``prev``, the loop entry present in
    every row at its sorted place (samplers.py:247-262)."""
    prev = np.asarray(prev, dtype=np.int64)
    r, c = csr_slice(row_offsets, col_indices, prev)
    has = np.zeros(prev.size, dtype=bool)
    has[r[c == prev[r]]] = True
    if not has.all():
        miss = np.flatnonzero(~has)
        r = np.concatenate([r, miss])
        c = np.concatenate([c, prev[miss]])
        o = np.lexsort((c, r))
        r, c = r[o], c[o]
    dh = deg_hat.astype(np.float64)
    v = 1.0 / np.sqrt(dh[prev[r]] * dh[c])
    return r, c, v


def candidates_of(row_offsets, col_indices, prev):
    """Sorted unique neighbour ids of ``prev`` (stored entries only)."""
    prev = np.asarray(prev, dtype=np.int64)
    if prev.size == 0:
        return np.empty(0, dtype=np.int64)
    return np.unique(csr_slice(row_offsets, col_indices, prev)[1]).astype(np.int64)


def column_norms(row_offsets, col_indices, deg_hat, cand, prev, squared):
    """Column norms of the restricted Laplacian over ``cand``: the squares
    summed per column in entry order (np.add.at), sqrt unless ``squared``."""
    r, c, v = restricted_rows(row_offsets, col_indices, deg_hat, prev)
    if cand.size == 0:
        return np.zeros(0, dtype=np.float64)
    at = np.minimum(np.searchsorted(cand, c), cand.size - 1)
    hit = cand[at] == c
    acc = np.zeros(cand.size, dtype=np.float64)
    np.add.at(acc, at[hit], v[hit] ** 2)
    return acc if squared else np.sqrt(acc)


def layer_probs(row_offsets, col_indices, deg_hat, cand, prev, flat):
    """ladies_probs (squared) / flat_probs (unsquared), normalised."""
    if cand.size == 0:
        raise SamplingError("empty candidate set")
    x = column_norms(row_offsets, col_indices, deg_hat, cand, prev, squared=not flat)
    t = x.sum()
    if t <= 0:
        raise SamplingError("all candidate columns have zero norm")
    return x / t


def fastgcn_probs(row_offsets, col_indices, deg_hat, flat=False):
    n = row_offsets.size - 1
    every = np.arange(n, dtype=np.int64)
    x = column_norms(row_offsets, col_indices, deg_hat, every, every, squared=not flat)
    return x / x.sum()


def debias_coefficients(p_draw, n):
    """Weights c with estimate = c @ x_rows for the recursive WOR estimator."""
    p_draw = np.asarray(p_draw, dtype=np.float64)
    s = p_draw.size
    alpha = np.array([1.0] + [n / ((n - i) * (i + 1)) for i in range(1, s)], dtype=np.float64)
    beta = np.empty(s)
    tail = 1.0
    for i in range(s - 1, -1, -1):
        beta[i] = alpha[i] * tail
        tail *= 1.0 - alpha[i]
    left = 1.0 - np.concatenate([[0.0], np.cumsum(p_draw[:-1])])
    later = np.concatenate([np.cumsum(beta[::-1])[::-1][1:], [0.0]])
    return beta / (p_draw / left) + later


class LayerBlock:
    __slots__ = ("rows", "cols", "values", "effective_values", "src_ids", "dst_ids",
                 "dst_in_src", "sample_probs")

    def __init__(self, **kw):
        for k in self.__slots__:
            setattr(self, k, kw.get(k))

    @property
    def num_dst(self):
        return int(self.dst_ids.size)

    @property
    def num_src(self):
        return int(self.src_ids.size)


def layer_block(row_offsets, col_indices, deg_hat, prev, cand, probs, budget, rng,
                debias, replace):
    """One layer-wise block from candidate probabilities (samplers.py:376-440)."""
    prev = np.asarray(prev, dtype=np.int64)
    rr, rc, rv = restricted_rows(row_offsets, col_indices, deg_hat, prev)

    def restrict(chosen, scale):
        at = np.minimum(np.searchsorted(chosen, rc), chosen.size - 1)
        keep = (chosen[at] == rc)
        return rr[keep], at[keep], rv[keep] * scale[at[keep]]

    positive = int(np.count_nonzero(probs > 0))
    if debias:
        s = min(budget, positive)
        order = weighted_sample_without_replacement(probs, s, rng)
        coef = debias_coefficients(probs[order], cand.size)
        asc = np.argsort(order, kind="stable")
        picked = order[asc]
        rows, cols, vals = restrict(cand[picked], coef[asc])
        eff = vals
    elif replace:
        s = budget
        d = rng.choice(cand.size, size=s, replace=True, p=probs)
        picked, counts = np.unique(d, return_counts=True)
        rows, cols, vals = restrict(cand[picked], counts / (s * probs[picked]))
        eff = vals
    else:
        s = min(budget, positive)
        picked = np.sort(weighted_sample_without_replacement(probs, s, rng))
        rows, cols, vals = restrict(cand[picked], 1.0 / (s * probs[picked]))
        sums = np.zeros(prev.size, dtype=np.float64)
        np.add.at(sums, rows, vals)
        eff = vals / np.where(sums > 0, sums, 1.0)[rows]
    return LayerBlock(rows=rows, cols=cols, values=vals, effective_values=eff,
                      src_ids=cand[picked].astype(np.int64), dst_ids=prev,
                      dst_in_src=None, sample_probs=probs[picked])


def sample_ladies(row_offsets, col_indices, targets, nodes_per_layer, layers, rng,
                  flat=False, debias=False, replace=False, deg_hat=None):
    """LADIES (samplers.py:443-472): blocks bottom-up and the dropped count."""
    if deg_hat is None:
        deg_hat = a_hat_degrees(row_offsets, col_indices)
    targets = np.asarray(targets, dtype=np.int64)
    out = np.diff(row_offsets)[targets]
    dropped = int(np.count_nonzero(out == 0))
    prev = targets[out > 0]
    if prev.size == 0:
        raise SamplingError("no targets with outgoing edges")
    blocks = []
    for _ in range(layers):
        cand = candidates_of(row_offsets, col_indices, prev)
        if cand.size == 0:
            raise SamplingError("empty candidate set mid-chain")
        p = layer_probs(row_offsets, col_indices, deg_hat, cand, prev, flat)
        blk = layer_block(row_offsets, col_indices, deg_hat, prev, cand, p, nodes_per_layer,
                          rng, debias=debias, replace=replace)
        blocks.append(blk)
        prev = blk.src_ids
    return blocks[::-1], dropped


def sample_fastgcn(row_offsets, col_indices, targets, nodes_per_layer, layers, rng,
                   flat=False, debias=False, probs=None, deg_hat=None):
    """FastGCN (samplers.py:475-495): i.i.d. draws from the global norms."""
    if deg_hat is None:
        deg_hat = a_hat_degrees(row_offsets, col_indices)
    targets = np.asarray(targets, dtype=np.int64)
    if targets.size == 0:
        raise SamplingError("empty target set")
    if probs is None:
        probs = fastgcn_probs(row_offsets, col_indices, deg_hat, flat=flat)
    every = np.arange(row_offsets.size - 1, dtype=np.int64)
    prev, blocks = targets, []
    for _ in range(layers):
        blk = layer_block(row_offsets, col_indices, deg_hat, prev, every, probs,
                          nodes_per_layer, rng, debias=debias, replace=not debias)
        blocks.append(blk)
        prev = blk.src_ids
    return blocks[::-1]


def gcn_block_values(row_offsets, col_indices, deg_hat, sage_block):
    """GCN arm of node_wise_block (samplers.py:178-191) from the SAGE block of
    the same draws: per row the self entry (r, r, 1/deg_hat[v]) first, then
    the sampled entries in order with (n/s)/sqrt(deg_hat[v] deg_hat[u])."""
    dst, src = sage_block.dst_ids, sage_block.src_ids
    dh = deg_hat.astype(np.float64)
    counts = np.bincount(sage_block.rows, minlength=dst.size)
    rows, cols, vals = [], [], []
    e = 0
    for r, v in enumerate(dst.tolist()):
        nb = col_indices[row_offsets[v]:row_offsets[v + 1]]
        n = int(np.count_nonzero(nb != v))
        s = int(counts[r])
        rows.append(r)
        cols.append(r)
        vals.append(1.0 / deg_hat[v])
        scale = n / s if s else 0.0
        for k in range(s):
            u = int(src[sage_block.cols[e + k]])
            rows.append(r)
            cols.append(int(sage_block.cols[e + k]))
            vals.append(scale / np.sqrt(dh[v] * dh[u]))
        e += s
    return (np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64),
            np.asarray(vals, dtype=np.float64))
