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
    pinned host memory and the gather reads misses over the host link.
  * ``labels`` int32 [n].
"""

from __future__ import annotations

import numpy as np
import torch

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
        ``synth.SynthGraph``).  ``feature_placement``: "hbm" or "host"."""
        if feature_placement not in ("hbm", "host"):
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

    # ---- reference-compatible views
    @property
    def num_edges(self) -> int:
        return self.num_arcs_stored

    def features_view(self) -> torch.Tensor:
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


def _host(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return a
