"""Layer-wise samplers (LADIES, FastGCN; flat / debias / with replacement)
and the GCN node-wise arm, backed by the CUDA kernels of ``mq_layerwise.cu``.

Mirrors ``mqpipe/samplers.py``:

* ``ladies_candidates`` / ``ladies_probs`` / ``flat_probs`` — ``:265-311``
  (computed inside ``mq_layer_block``; exposed through the block's
  ``sample_probs`` and ``LayerBlock.num_candidates``)
* ``fastgcn_probs``     — ``:314-318`` (``mq_layer_fastgcn_probs``)
* ``sample_ladies``     — ``:443-472``
* ``sample_fastgcn``    — ``:475-495``
* ``node_wise_block`` GCN arm — ``:178-191`` (``mq_gcn_block``)

``rng`` is the batch's :class:`samplers.PhiloxStream`; layer l of the batch
draws from the Philox stream (seed, epoch; ctr (i, 0xFFFFFFFF, l, batch)) —
the contract under which the reference's own sampler produced the fixtures
in ``tests/golden/layerwise.npz``.  The calls synchronise their stream (the
reference returns host arrays; each layer's sizes come from the device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._lib import MQSamplingError, lib, ptr
from .engine import current_stream

_MODE_WOR, _MODE_REPLACE, _MODE_DEBIAS = 0, 1, 2


class SamplingError(RuntimeError):
    """samplers.py:23-24 (re-exported by ``samplers``)."""


@dataclass(frozen=True)
class LayerBlock:
    """One layer-wise block on the device.  ``values`` are the float32 weights
    the forward applies (``effective_values`` cast, as ``block_apply`` does,
    nn.py:79-89); ``exact`` / ``exact_effective`` the reference's float64
    estimator values; ``row_ptr`` the CSR view of the row-sorted triplets."""

    rows: torch.Tensor
    cols: torch.Tensor
    values: torch.Tensor
    src_ids: torch.Tensor
    dst_ids: torch.Tensor
    row_ptr: torch.Tensor
    exact: torch.Tensor
    exact_effective: torch.Tensor
    sample_probs: torch.Tensor = None
    num_candidates: int = 0
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
        return self.exact.cpu().numpy()

    def to_reference(self) -> dict:
        return dict(rows=self.rows.cpu().numpy().astype(np.int64),
                    cols=self.cols.cpu().numpy().astype(np.int64),
                    values=self.exact.cpu().numpy(),
                    effective_values=self.exact_effective.cpu().numpy(),
                    src_ids=self.src_ids.cpu().numpy().astype(np.int64),
                    dst_ids=self.dst_ids.cpu().numpy().astype(np.int64),
                    dst_in_src=(None if self.dst_in_src is None
                                else self.dst_in_src.cpu().numpy().astype(np.int64)),
                    sample_probs=(None if self.sample_probs is None
                                  else self.sample_probs.cpu().numpy()))


class _Tables:
    """Per-graph node tables of the LADIES candidate pass (flags stay zero)."""

    def __init__(self, g):
        n = max(g.num_nodes, 1)
        self.flags = torch.zeros(n, dtype=torch.uint8, device=g.device)
        self.pos = torch.empty(n, dtype=torch.int32, device=g.device)
        self.fastgcn = {}  # flat -> (probs, cdf)


def _tables(g) -> _Tables:
    t = g.__dict__.get("_lw_tables")
    if t is None:
        t = _Tables(g)
        g._lw_tables = t
    return t


def _i32(x, g) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.int64))
    t = t.to(device=g.device, dtype=torch.int32).flatten().contiguous()
    if t.numel() and (int(t.min()) < 0 or int(t.max()) >= g.num_nodes):
        raise ValueError("node id out of range")
    return t


def fastgcn_probs(g, flat: bool = False) -> torch.Tensor:
    """Global importance: column norms of the full Laplacian (samplers.py:314-318),
    float64 on the device; cached per graph."""
    return _fastgcn(g, flat)[0]


def _fastgcn(g, flat):
    t = _tables(g)
    hit = t.fastgcn.get(bool(flat))
    if hit is None:
        n = g.num_nodes
        probs = torch.empty(n, dtype=torch.float64, device=g.device)
        cdf = torch.empty(n, dtype=torch.float64, device=g.device)
        lib().mq_layer_fastgcn_probs(ptr(g.row_off), ptr(g.col), ptr(g.loops), n, int(flat),
                                     ptr(probs), ptr(cdf), current_stream(g.device))
        hit = (probs, cdf)
        t.fastgcn[bool(flat)] = hit
    return hit


def _layer(g, prev: torch.Tensor, budget: int, rng, layer: int, mode: int, flat: bool,
           probs=None, cdf=None) -> LayerBlock:
    dev, stream = g.device, current_stream(g.device)
    n_prev = int(prev.numel())
    roff = torch.empty(n_prev + 1, dtype=torch.int64, device=dev)
    scr = torch.empty(int(lib().mq_layer_scratch_bytes(max(n_prev, 1))), dtype=torch.uint8,
                      device=dev)
    lib().mq_layer_entries(ptr(g.row_off), ptr(g.loops), ptr(prev), n_prev, ptr(roff), ptr(scr),
                           stream)
    ne = int(roff[-1].item())
    budget = int(budget)
    i32 = dict(dtype=torch.int32, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    rows, cols = torch.empty(max(ne, 1), **i32), torch.empty(max(ne, 1), **i32)
    vals, eff = torch.empty(max(ne, 1), **f64), torch.empty(max(ne, 1), **f64)
    row_ptr = torch.empty(n_prev + 1, **i32)
    src, sp = torch.empty(max(budget, 1), **i32), torch.empty(max(budget, 1), **f64)
    counts = torch.zeros(4, dtype=torch.int64, device=dev)
    tb = _tables(g)
    try:
        lib().mq_layer_block(ptr(g.row_off), ptr(g.col), ptr(g.loops), g.num_nodes, ptr(prev),
                             n_prev, ptr(roff), ne, ptr(probs), ptr(cdf), int(flat), mode, budget,
                             rng.seed & 0xFFFFFFFFFFFFFFFF, rng.epoch & 0xFFFFFFFFFFFFFFFF,
                             rng.batch_id & 0xFFFFFFFF, layer, ptr(tb.flags), ptr(tb.pos),
                             ptr(rows), ptr(cols), ptr(vals), ptr(eff), ptr(row_ptr), ptr(src),
                             ptr(sp), ptr(counts), stream)
    except MQSamplingError as e:
        raise SamplingError(str(e)) from None
    nnz, n_src, n_cand, _ = (int(x) for x in counts.cpu().tolist())
    return LayerBlock(rows=rows[:nnz], cols=cols[:nnz], values=eff[:nnz].to(torch.float32),
                      src_ids=src[:n_src], dst_ids=prev, row_ptr=row_ptr,
                      exact=vals[:nnz], exact_effective=eff[:nnz], sample_probs=sp[:n_src],
                      num_candidates=n_cand)


def _mode(debias: bool, replace: bool) -> int:
    return _MODE_DEBIAS if debias else (_MODE_REPLACE if replace else _MODE_WOR)


def sample_ladies(g, targets, nodes_per_layer: int, layers: int, rng, flat: bool = False,
                  debias: bool = False, replace: bool = False) -> tuple[list, int]:
    """LADIES (samplers.py:443-472): (blocks bottom-up, dropped targets)."""
    tg = _i32(targets, g)
    n = int(tg.numel())
    kept = torch.empty(max(n, 1), dtype=torch.int32, device=g.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=g.device)
    scr = torch.empty(int(lib().mq_layer_scratch_bytes(max(n, 1))), dtype=torch.uint8,
                      device=g.device)
    lib().mq_layer_live_targets(ptr(g.row_off), ptr(g.loops), ptr(tg), n, ptr(kept), ptr(cnt),
                                ptr(scr), current_stream(g.device))
    k = int(cnt.item())
    dropped = n - k
    if k == 0:
        raise SamplingError("no targets with outgoing edges")
    prev, blocks = kept[:k], []
    for layer in range(layers):
        blk = _layer(g, prev, nodes_per_layer, rng, layer, _mode(debias, replace), flat)
        blocks.append(blk)
        prev = blk.src_ids
    blocks.reverse()
    return blocks, dropped


def sample_fastgcn(g, targets, nodes_per_layer: int, layers: int, rng, flat: bool = False,
                   debias: bool = False, probs=None) -> list:
    """FastGCN (samplers.py:475-495): i.i.d. draws from the global norms (with
    replacement), or WOR with the recursive correction when ``debias``."""
    tg = _i32(targets, g)
    if tg.numel() == 0:
        raise SamplingError("empty target set")
    if probs is None:
        probs, cdf = _fastgcn(g, flat)
    else:
        probs = torch.as_tensor(probs, dtype=torch.float64).to(g.device).contiguous()
        if probs.numel() != g.num_nodes:
            raise ValueError("probs must hold one entry per node")
        cdf = None if debias else _cdf_of(probs)
    prev, blocks = tg, []
    mode = _MODE_DEBIAS if debias else _MODE_REPLACE
    for layer in range(layers):
        blk = _layer(g, prev, nodes_per_layer, rng, layer, mode, flat, probs=probs, cdf=cdf)
        blocks.append(blk)
        prev = blk.src_ids
    blocks.reverse()
    return blocks


def _cdf_of(probs: torch.Tensor) -> torch.Tensor:
    """NumPy's choice(p) cdf of user-given probabilities: cumsum (sequential)
    divided by its last element (mq_layer_cdf)."""
    out = torch.empty_like(probs)
    lib().mq_layer_cdf(ptr(probs), int(probs.numel()), ptr(out), current_stream(probs.device))
    return out


def gcn_block_from_sage(g, sage_blk, dst: torch.Tensor):
    """GCN arm of node_wise_block (samplers.py:178-191) from the SAGE block of
    the same draws: returns (row_ptr, rows, cols, values f64)."""
    dev = g.device
    n_dst = int(dst.numel())
    nnz = sage_blk.nnz + n_dst
    i32 = dict(dtype=torch.int32, device=dev)
    row_ptr = torch.empty(n_dst + 1, **i32)
    rows, cols = torch.empty(max(nnz, 1), **i32), torch.empty(max(nnz, 1), **i32)
    vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    lib().mq_gcn_block(ptr(g.row_off), ptr(g.loops), ptr(dst), ptr(sage_blk.src_ids),
                       ptr(sage_blk.row_ptr), ptr(sage_blk.cols), n_dst, ptr(row_ptr), ptr(rows),
                       ptr(cols), ptr(vals), current_stream(dev))
    return row_ptr, rows[:nnz], cols[:nnz], vals[:nnz]
