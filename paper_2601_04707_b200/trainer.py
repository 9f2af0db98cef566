"""One replica's per-iteration hot path as captured CUDA graphs.

A step = batch setup (device-side plan), L hops of sample + relabel, feature
gather, SAGE forward, summed softmax-CE, backward and the optimizer — the
``_run_epoch_serial`` per-batch body of the reference (``runtime.py:294-323``)
with the RaCoM window apply (``runtime.py:167-195``) folded in.  Everything is
enqueued through the C-ABI on one stream; after an eager warm-up the sequence
is captured once and replayed per batch, so a step costs one graph launch.

Multi-replica (RaCoM) steps split the graph in two around the gradient
exchange: compute graph -> f64 all-reduce of [grads | contributor count]
(NCCL in production, gloo/in-process in tests) -> update graph.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import lib, ptr
from .engine import SampleWorkspace, TrainWorkspace


class StepRunner:
    """Per-iteration path for one replica on one GPU."""

    def __init__(self, g, model, *, fanouts, batch_size: int, num_train: int, cache=None,
                 optimizer: str = "adam", seed: int = 0, world: int = 1, rank: int = 0,
                 multi: bool = False, use_graph: bool = True, ring_len: int = 1 << 16):
        if optimizer not in ("adam", "sgd"):
            raise ValueError(f"unknown optimizer {optimizer!r}")
        self.g = g
        self.model = model
        self.dm = model.dev
        self.cache = cache
        self.optimizer = optimizer
        self.seed = int(seed)
        self.world, self.rank = int(world), int(rank)
        self.multi = bool(multi)
        self.use_graph = use_graph
        dev = g.device
        self.device = dev
        self.sw = SampleWorkspace(g, fanouts, batch_size)
        dims = [g.feature_dim] + [int(w.shape[1]) for w in model.weights]
        if dims[-1] != g.num_classes:
            raise ValueError("model output width must equal num_classes")
        self.tw = TrainWorkspace(self.sw, dims, g.num_classes)
        self.num_train = int(num_train)
        self.perm = torch.zeros(max(self.num_train, 1), dtype=torch.int32, device=dev)
        self.cursor = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ring_len = int(ring_len)
        self.loss_ring = torch.zeros(self.ring_len, dtype=torch.float64, device=dev)
        self.grad64 = (torch.zeros(self.dm.num_params + 1, dtype=torch.float64, device=dev)
                       if self.multi else None)
        self.stream = torch.cuda.Stream(device=dev)
        self.graphs = {}
        self.windows_done = 0
        self.epoch = 0

    # ---------------------------------------------------------------- epochs
    def begin_epoch(self, epoch: int, perm: np.ndarray):
        """Upload this epoch's shuffled train ids (plan_epoch, runtime.py:95-117)."""
        perm = np.asarray(perm)
        if perm.size != self.num_train:
            raise ValueError("permutation length changed; build a new StepRunner")
        # stream-ordered and host-asynchronous: pinned staging + non_blocking
        # copies, so an epoch boundary does not drain the step pipeline
        staged = torch.from_numpy(perm.astype(np.int32)).pin_memory()
        key = torch.from_numpy(np.array([self.seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF, 0],
                                        dtype=np.uint32).view(np.int32)).pin_memory()
        with torch.cuda.stream(self.stream):
            self.perm.copy_(staged, non_blocking=True)
            self.cursor.zero_()
            self.sw.key.copy_(key, non_blocking=True)
        self.epoch = epoch
        self.windows_done = 0
        n_windows = -(-self.num_train // (self.sw.batch_size * self.world))
        self.dm.ensure_bias(self.dm.host_steps + n_windows + 8)

    # --------------------------------------------------------------- enqueue
    def _enqueue_setup(self, s):
        lib().mq_batch_setup(ptr(self.perm), self.num_train, self.sw.batch_size, self.world,
                             self.rank, ptr(self.cursor), ptr(self.sw.targets),
                             ptr(self.sw.n_targets), ptr(self.sw.key), s)

    def _enqueue_compute(self, s, commit=True):
        self.sw.launch(self.cache, s, key_on_device=True)
        self.tw.launch_gather(self.cache, s)
        self.tw.launch_forward(self.dm, s)
        self.tw.launch_loss(self.dm, s)
        if commit:
            lib().mq_step_commit(ptr(self.tw.loss), ptr(self.cursor), ptr(self.loss_ring),
                                 self.ring_len, s)
        self.tw.launch_backward(self.dm, s)
        if self.grad64 is not None:
            lib().mq_pack_grads(ptr(self.dm.flat_g), self.dm.num_params, ptr(self.sw.n_targets),
                                ptr(self.grad64), s)

    def _enqueue_update(self, s):
        if self.grad64 is None:
            self.tw.launch_optimizer(self.dm, self.optimizer, s)
        else:  # scale 0: divide by the all-reduced contributor count (expected[k])
            self.tw.launch_optimizer(self.dm, self.optimizer, s, grad64=self.grad64, scale=0.0)

    def _phases(self):
        if self.grad64 is None:
            return {"full": lambda s: (self._enqueue_setup(s), self._enqueue_compute(s),
                                       self._enqueue_update(s))}
        return {"compute": lambda s: (self._enqueue_setup(s), self._enqueue_compute(s)),
                "update": self._enqueue_update}

    # ----------------------------------------------------------------- graphs
    def _snapshot(self):
        d = self.dm
        return [t.clone() for t in (d.flat_w, d.flat_m, d.flat_v, d.step_dev, self.cursor,
                                    self.loss_ring)] + (
            [self.cache.hit_miss.clone()] if self.cache is not None else [])

    def _restore(self, snap):
        d = self.dm
        targets = [d.flat_w, d.flat_m, d.flat_v, d.step_dev, self.cursor, self.loss_ring] + (
            [self.cache.hit_miss] if self.cache is not None else [])
        for t, v in zip(targets, snap):
            t.copy_(v)

    def capture(self):
        """Eager warm-up (state restored afterwards), then capture each phase."""
        if self.graphs:
            return
        phases = self._phases()
        with torch.cuda.stream(self.stream):
            snap = self._snapshot()
            s = self.stream.cuda_stream
            for fn in phases.values():
                fn(s)  # warm-up only: no collective in between
            self.stream.synchronize()
            self._restore(snap)
            self.tw.loss.zero_()
            self.dm.nonfinite.zero_()
            self.stream.synchronize()
        for name, fn in phases.items():
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=self.stream):
                fn(torch.cuda.current_stream().cuda_stream)
            self.graphs[name] = graph
        torch.cuda.synchronize(self.device)

    def kernels_per_step(self) -> int:
        """Number of libmqgnn kernel launches one step enqueues."""
        lib().mq_prof_reset()
        before = lib().mq_launch_count()
        with torch.cuda.stream(self.stream):
            snap = self._snapshot()
            for fn in self._phases().values():
                fn(self.stream.cuda_stream)
            self.stream.synchronize()
            self._restore(snap)
            self.tw.loss.zero_()
        return int(lib().mq_launch_count() - before)

    # ------------------------------------------------------------------ step
    def _replay(self, name):
        with torch.cuda.stream(self.stream):
            if self.use_graph:
                self.graphs[name].replay()
            elif name == "update":
                self._enqueue_update(self.stream.cuda_stream)
            else:
                self._phases()[name](self.stream.cuda_stream)

    # RaCoM protocol (racom.WindowDriver): compute -> exchange grad64 -> apply.
    # A lone replica's compute already contains its update ("full" graph).
    def compute_window(self):
        self._replay("compute" if self.multi else "full")

    def apply_window(self):
        if self.multi:
            self._replay("update")
        self.dm.host_steps += 1
        self.windows_done += 1

    def step(self):
        """One window (async; nothing is read back)."""
        if self.multi:
            raise RuntimeError("multi-replica runners need the exchange: use racom.WindowDriver")
        self.compute_window()
        self.apply_window()

    def state64(self) -> torch.Tensor:
        from .racom import _pack_state
        with torch.cuda.stream(self.stream):
            out = torch.empty(3 * self.dm.num_params, dtype=torch.float64, device=self.device)
            _pack_state(self.model, out)
        return out

    def load_state64(self, t: torch.Tensor, divisor: int):
        from .racom import _unpack_state
        with torch.cuda.stream(self.stream):
            _unpack_state(self.model, t, divisor)

    @property
    def step_count(self) -> int:
        return self.dm.host_steps

    def sync_point(self):
        self.stream.synchronize()

    def stream_ctx(self):
        return torch.cuda.stream(self.stream)

    def wait_current(self):
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def read_counts(self) -> dict:
        """Device counts of the last step: targets and (n_dst, n_src, nnz) per hop."""
        self.stream.synchronize()
        c = torch.cat([self.sw.n_targets] + [hb.counts for hb in self.sw.hops]).cpu().tolist()
        hops, nd = [], c[0]
        for h in range(len(self.sw.hops)):
            ns, nnz = c[1 + 2 * h], c[2 + 2 * h]
            hops.append((nd, ns, nnz))
            nd = ns
        return {"n_targets": c[0], "hops": hops}

    def losses(self, n_windows: int) -> np.ndarray:
        self.stream.synchronize()
        return self.loss_ring[:n_windows].cpu().numpy()

    def check_finite(self):
        self.stream.synchronize()
        flag = int(self.dm.nonfinite.item())
        if flag:
            self.dm.nonfinite.zero_()
            if flag & 2:
                raise RuntimeError("Adam bias-correction table exhausted")
            raise FloatingPointError("training step produced NaN or Inf")

    # ------------------------------------------------- host-input (e2e) path
    def capture_host_input(self):
        """Graph variant that reads targets staged by the host (no device plan)."""
        if "host" in self.graphs:
            return
        if self.multi:
            raise NotImplementedError("host-input steps are single-replica")

        def fn(s):
            self._enqueue_compute(s, commit=False)
            self._enqueue_update(s)
        with torch.cuda.stream(self.stream):
            snap = self._snapshot()
            fn(self.stream.cuda_stream)
            self.stream.synchronize()
            self._restore(snap)
            self.tw.loss.zero_()
            self.stream.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=self.stream):
            fn(torch.cuda.current_stream().cuda_stream)
        self.graphs["host"] = graph
        self._stage = torch.zeros(4, dtype=torch.int32, pin_memory=True)
        self._loss_host = torch.zeros(1, dtype=torch.float64, pin_memory=True)

    def step_from_host(self, targets_pinned: torch.Tensor, batch_id: int) -> float:
        """H2D the batch's targets, run the step, D2H its loss (synchronous)."""
        n = int(targets_pinned.numel())
        with torch.cuda.stream(self.stream):
            self.sw.targets[:n].copy_(targets_pinned, non_blocking=True)
            self._stage.numpy().view(np.uint32)[:] = (n, self.seed & 0xFFFFFFFF,
                                                      self.epoch & 0xFFFFFFFF,
                                                      batch_id & 0xFFFFFFFF)
            self.sw.n_targets.copy_(self._stage[0:1], non_blocking=True)
            self.sw.key.copy_(self._stage[1:4], non_blocking=True)
            self.graphs["host"].replay()
            self._loss_host.copy_(self.tw.loss, non_blocking=True)
            self.tw.loss.zero_()
        self.stream.synchronize()
        self.dm.host_steps += 1
        return float(self._loss_host[0])
