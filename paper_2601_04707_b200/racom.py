"""RaCoM gradient sharing and periodic model sync on NCCL (or gloo / in-process).

Reference: ``mqpipe/racom.py``.

* Window gradient mean (``Accumulator``, ``racom.py:36-78``; broadcast to every
  inbox, ``racom.py:142-184``): every replica packs its window gradient into
  f64 together with a contributor flag (``mq_pack_grads``); ONE all-reduce(SUM)
  yields the sum and ``expected[k]`` (``runtime.py:115-116``); the optimizer
  kernel divides on device.  f64 accumulation as in the reference.
* ``sync_models`` (``racom.py:118-139``): f64 average of [W | m | v] — one
  all-reduce of the packed buffer, divide by the replica count, cast back.
* ``compute_sync_period`` (``racom.py:90-106``) and ``apply_update``
  (``racom.py:81-87``) keep the reference's host-side definitions.

Exchanges: ``DistExchange`` wraps a ``torch.distributed`` process group
(NCCL over NVLink on GPUs, gloo for the CPU tests); ``LocalExchange`` sums
the buffers of replicas that share one process (several replicas on one
GPU — the reference's simulated devices).
"""

from __future__ import annotations

import math
import warnings

import torch

from ._lib import lib, ptr


def compute_sync_period(num_nodes: int, num_edges: int, num_devices: int,
                        scale_k: float = 1.0) -> int:
    """Iterations between full syncs: ceil(k * sqrt(V) / sqrt(G * E)), >= 1."""
    if num_nodes <= 0 or num_devices <= 0:
        raise ValueError("need positive node and device counts")
    if num_edges == 0:
        warnings.warn("sync period on an edge-free graph: ignoring edge term")
        period = math.ceil(scale_k * math.sqrt(num_nodes))
    else:
        period = math.ceil(scale_k * math.sqrt(num_nodes) / math.sqrt(num_devices * num_edges))
    return max(1, period)


def staleness_cost(period, alpha, beta, num_nodes, num_edges, num_devices) -> float:
    """alpha * P * E + beta * (V / G) / P (racom.py:109-115)."""
    if period <= 0:
        raise ValueError("period must be positive")
    return alpha * period * num_edges + beta * (1.0 / period) * (num_nodes / num_devices)


def apply_update(state, grads, optimizer: str):
    from . import nn
    if optimizer == "adam":
        return nn.adam_step(state, grads)
    if optimizer == "sgd":
        return nn.sgd_step(state, grads)
    raise ValueError(f"unknown optimizer {optimizer!r}")


class DistExchange:
    """All-reduce(SUM) over a torch.distributed group (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)

    def allreduce_sum(self, t: torch.Tensor, stream=None):
        if stream is not None and t.is_cuda:
            with torch.cuda.stream(stream):
                self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        else:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def allreduce_sum_many(self, ts):
        for t in ts:
            self.allreduce_sum(t)


class LocalExchange:
    """Replicas sharing one process: sum their buffers in replica order
    (the reference's in-process device threads, racom.py:142-184)."""

    def __init__(self, size: int):
        self.size = size

    def allreduce_sum_many(self, ts):
        total = ts[0].clone()
        for t in ts[1:]:
            total += t
        for t in ts:
            t.copy_(total)


def _pack_state(model, out64):
    d = model.dev
    n = d.num_params
    s = torch.cuda.current_stream(d.device).cuda_stream
    for i, flat in enumerate((d.flat_w, d.flat_m, d.flat_v)):
        lib().mq_f32_to_f64(ptr(flat), ptr(out64[i * n:(i + 1) * n]), n, s)


def _unpack_state(model, in64, divisor):
    d = model.dev
    n = d.num_params
    s = torch.cuda.current_stream(d.device).cuda_stream
    for i, flat in enumerate((d.flat_w, d.flat_m, d.flat_v)):
        lib().mq_f64_to_f32(ptr(in64[i * n:(i + 1) * n]), float(divisor), ptr(flat), n, s)


def sync_models(replicas, exchange=None) -> None:
    """Average weights and Adam moments across replicas in f64, in place.

    ``replicas`` are this process's ModelStates; ``exchange`` is a
    DistExchange when the other replicas live in other processes."""
    if not replicas:
        raise ValueError("no replicas to sync")
    steps = {r.step_count for r in replicas}
    if exchange is not None and isinstance(exchange, DistExchange):
        import torch.distributed as dist
        st = torch.tensor([min(steps), max(steps)], dtype=torch.int64)
        if replicas[0].device.type == "cuda" and dist.get_backend(exchange.group) == "nccl":
            st = st.to(replicas[0].device)
        lo = st.clone()
        dist.all_reduce(lo[0:1], op=dist.ReduceOp.MIN, group=exchange.group)
        dist.all_reduce(lo[1:2], op=dist.ReduceOp.MAX, group=exchange.group)
        if int(lo[0]) != int(lo[1]):
            raise RuntimeError(f"sync with unequal step counts: {int(lo[0])}..{int(lo[1])}")
        n_total = exchange.size * len(replicas)
    else:
        if len(steps) != 1:
            raise RuntimeError(f"sync with unequal step counts: {sorted(steps)}")
        n_total = len(replicas)
    bufs = []
    for r in replicas:
        b = torch.empty(3 * r.dev.num_params, dtype=torch.float64, device=r.device)
        _pack_state(r, b)
        bufs.append(b)
    if len(bufs) > 1:
        LocalExchange(len(bufs)).allreduce_sum_many(bufs)
    if exchange is not None and isinstance(exchange, DistExchange):
        exchange.allreduce_sum(bufs[0])
        for b in bufs[1:]:
            b.copy_(bufs[0])
    for r, b in zip(replicas, bufs):
        _unpack_state(r, b, n_total)


class WindowDriver:
    """RaCoM window schedule for the replicas of this process.

    Parity mode of the reference (``_run_epoch_serial`` with zero delay,
    ``runtime.py:285-373``): per window every replica computes its batch on
    its current weights, the f64 window sum and contributor count are
    all-reduced, every replica applies the mean (window order), and replicas
    average [W | m | v] every ``sync_period`` applied windows and once at the
    epoch barrier when more than one replica exists.

    ``runners`` implement ``compute_window() / grad64 / apply_window() /
    state64() / load_state64(t, n) / step_count / sync_point() /
    stream_ctx() / wait_current()``
    (``trainer.StepRunner`` on a GPU; an oracle-backed runner in the CPU
    tests).  ``exchange`` is a DistExchange when replicas span processes.

    Sync elision (``elide_identical``): after one full average the replicas
    are bit-identical, and every later window applies the same all-reduced
    gradient through the same deterministic optimizer on every replica, so
    they stay bit-identical; averaging G identical f32 values in f64 (exact
    sums of at most 8 terms, exact division of an exact multiple) returns
    them unchanged.  Later milestone and epoch-barrier syncs are therefore
    the identity and are skipped (still counted in ``sync_count``, reported
    in ``elided``).  The first sync of a driver always runs, since replicas
    handed in may differ.
    """

    def __init__(self, runners, exchange=None, sync_period: int = 1,
                 elide_identical: bool = True):
        if sync_period < 1:
            raise ValueError("sync period must be at least 1")
        self.runners = list(runners)
        self.exchange = exchange
        self.sync_period = int(sync_period)
        self.remote = exchange.size if isinstance(exchange, DistExchange) else 1
        self.total_replicas = self.remote * len(self.runners)
        self.elide_identical = bool(elide_identical)
        self.identical = False  # replicas known to be bit-identical
        self.elided = 0

    def _reduce(self, tensors):
        """Sum the runners' buffers over every replica.  A lone local runner
        issues the collective on its own stream (no host sync); several local
        runners are summed on the current stream between explicit waits."""
        if len(self.runners) == 1:
            if self.remote > 1:
                with self.runners[0].stream_ctx():
                    self.exchange.allreduce_sum(tensors[0])
            return
        for r in self.runners:
            r.sync_point()
        LocalExchange(len(tensors)).allreduce_sum_many(tensors)
        if self.remote > 1:
            self.exchange.allreduce_sum(tensors[0])
            for t in tensors[1:]:
                t.copy_(tensors[0])
        for r in self.runners:
            r.wait_current()

    def sync(self):
        steps = {r.step_count for r in self.runners}
        if len(steps) != 1:
            raise RuntimeError(f"sync with unequal step counts: {sorted(steps)}")
        if self.elide_identical and self.identical:
            self.elided += 1
            return
        bufs = [r.state64() for r in self.runners]
        self._reduce(bufs)
        for r, b in zip(self.runners, bufs):
            r.load_state64(b, self.total_replicas)
        self.identical = True

    def run(self, total_windows: int, on_window=None) -> dict:
        applied = 0
        milestone = self.sync_period
        sync_count = 0
        # runners whose window already contains the exchange (peer memory,
        # peer.PeerExchange) need no host-issued reduction
        fused = all(getattr(r, "fx", None) is not None for r in self.runners)
        for k in range(total_windows):
            for r in self.runners:
                r.compute_window()
            if self.total_replicas > 1 and not fused:
                self._reduce([r.grad64 for r in self.runners])
            for r in self.runners:
                r.apply_window()
            applied += 1
            if on_window is not None:
                on_window(k)
            if milestone <= total_windows and applied >= milestone:
                if self.total_replicas > 1:  # a lone replica's average is itself
                    self.sync()
                milestone += self.sync_period
                sync_count += 1
        for r in self.runners:  # the pipelined schedule's held-back window
            fin = getattr(r, "finish", None)
            if fin is not None:
                fin()
        epoch_sync = 0
        if self.total_replicas > 1:
            self.sync()
            epoch_sync = 1
        return {"sync_count": sync_count, "epoch_sync": epoch_sync, "applied": applied,
                "elided": self.elided}
