"""One replica's per-iteration hot path as captured, pipelined CUDA graphs.

A step = batch setup (device-side plan), L hops of sample + relabel, feature
gather ("prep": the reference's sample + transfer stages, samplers.py:502-540
and runtime.py:127-143) followed by SAGE forward, summed softmax-CE,
backward and the optimizer ("train": nn.py:116-206 and the RaCoM window
apply, runtime.py:167-195).

The multi-queue pipeline of MQ-GNN (sample -> transfer -> compute -> update,
runtime.py:380-612) is expressed with two CUDA streams inside ONE graph per
step: the prep of batch k+1 runs on the prep stream into the other of two
double-buffered slots while batch k trains on the train stream; the graph
joins both branches, so the host launches one graph per window and never
synchronises.  Queue depth is the slot count (2).

Multi-replica (RaCoM) steps split the graph around the gradient exchange:
[prep k+1 || train k + pack] -> f64 all-reduce of [grads | contributor
count] (NCCL in production, gloo / in-process in tests) -> update graph.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import lib, ptr
from .engine import FusedTrainWorkspace, SampleWorkspace, TrainWorkspace


class StepRunner:
    """Per-iteration path for one replica on one GPU."""

    def __init__(self, g, model, *, fanouts, batch_size: int, num_train: int, cache=None,
                 optimizer: str = "adam", seed: int = 0, world: int = 1, rank: int = 0,
                 multi: bool = False, use_graph: bool = True, pipeline: bool = True,
                 ring_len: int = 1 << 16, fused: bool = True):
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
        self.pipeline = bool(pipeline)
        dev = g.device
        self.device = dev
        self.slots = [SampleWorkspace(g, fanouts, batch_size)
                      for _ in range(2 if self.pipeline else 1)]
        self.sw = self.slots[0]
        dims = [g.feature_dim] + [int(w.shape[1]) for w in model.weights]
        if dims[-1] != g.num_classes:
            raise ValueError("model output width must equal num_classes")
        # fused: transform-first hidden layers + one-launch head (mq_fused.cu);
        # otherwise the reference-shaped per-op kernels (aggregate-first)
        self.fused = bool(fused)
        self.tw = (FusedTrainWorkspace if self.fused else TrainWorkspace)(self.sw, dims,
                                                                          g.num_classes)
        self.num_train = int(num_train)
        self.batch_size = int(batch_size)
        self.perm = torch.zeros(max(self.num_train, 1), dtype=torch.int32, device=dev)
        self.cursor = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ring_len = int(ring_len)
        self.loss_ring = torch.zeros(self.ring_len, dtype=torch.float64, device=dev)
        self.grad64 = (torch.zeros(self.dm.num_params + 1, dtype=torch.float64, device=dev)
                       if self.multi else None)
        self.stream = torch.cuda.Stream(device=dev)       # train stream
        self.prep_stream = torch.cuda.Stream(device=dev)  # sample + transfer stream
        self.graphs = {}
        self.launches_per_phase = {}
        self.windows_done = 0
        self.epoch = 0
        self._primed = False

    # ---------------------------------------------------------------- epochs
    def begin_epoch(self, epoch: int, perm: np.ndarray):
        """Upload this epoch's shuffled train ids (plan_epoch, runtime.py:95-117)
        and, when pipelined, prepare batch 0 (the pipeline prologue)."""
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
            for sw in self.slots:
                sw.key.copy_(key, non_blocking=True)
        self.epoch = epoch
        self.windows_done = 0
        n_windows = -(-self.num_train // (self.batch_size * self.world))
        self.dm.ensure_bias(self.dm.host_steps + n_windows + 8)
        self._primed = False
        if self.pipeline and self.graphs:
            self._prologue()

    def _prologue(self):
        with torch.cuda.stream(self.stream):
            if self.use_graph:
                self.graphs["prologue"].replay()
            else:
                self._enqueue_prep(self.slots[0], self.stream.cuda_stream)
        self._primed = True

    # --------------------------------------------------------------- enqueue
    def _enqueue_setup(self, sw, s):
        lib().mq_batch_setup(ptr(self.perm), self.num_train, self.batch_size, self.world,
                             self.rank, ptr(self.cursor), ptr(sw.targets), ptr(sw.n_targets),
                             ptr(sw.key), s)

    def _enqueue_prep(self, sw, s, setup=True):
        if setup:
            self._enqueue_setup(sw, s)
        sw.launch(self.cache, s, key_on_device=True)
        self.tw.launch_gather(sw, self.cache, s)

    def _enqueue_train(self, sw, s, commit=True):
        if self.fused:
            self.tw.launch_train(self.dm, s, sw, ring=self.loss_ring if commit else None,
                                 ring_len=self.ring_len, world=self.world)
        else:
            self.tw.launch_forward(self.dm, s, sw)
            self.tw.launch_loss(self.dm, s, sw)
            if commit:
                lib().mq_step_commit(ptr(self.tw.loss), ptr(sw.key), self.world,
                                     ptr(self.loss_ring), self.ring_len, s)
            self.tw.launch_backward(self.dm, s, sw)
        if self.grad64 is not None:
            src = self.tw.grad_src(self.dm) if self.fused else None
            lib().mq_pack_grads(ptr(self.dm.flat_g), self.dm.num_params, ptr(sw.n_targets),
                                ptr(self.grad64), C.byref(src) if src is not None else None, s)

    def _enqueue_update(self, s):
        if self.grad64 is None:
            self.tw.launch_optimizer(self.dm, self.optimizer, s)
        else:  # scale 0: divide by the all-reduced contributor count (expected[k])
            self.tw.launch_optimizer(self.dm, self.optimizer, s, grad64=self.grad64, scale=0.0)

    def _fork_join(self, s_train, prep_fn, train_fn):
        """prep_fn on the prep stream in parallel with train_fn on s_train."""
        cur = torch.cuda.current_stream(self.device)
        self.prep_stream.wait_stream(cur)
        with torch.cuda.stream(self.prep_stream):
            prep_fn(self.prep_stream.cuda_stream)
        train_fn(s_train)
        cur.wait_stream(self.prep_stream)

    def _phases(self):
        """name -> fn(stream) for every graph this runner captures."""
        ph = {}
        if not self.pipeline:
            sw = self.slots[0]

            def full(s):
                self._enqueue_prep(sw, s)
                self._enqueue_train(sw, s)
                if not self.multi:
                    self._enqueue_update(s)
            ph["step0" if not self.multi else "compute0"] = full
        else:
            ph["prologue"] = lambda s: self._enqueue_prep(self.slots[0], s)
            for i in (0, 1):
                cur, nxt = self.slots[i], self.slots[1 - i]

                def step(s, cur=cur, nxt=nxt):
                    def train(st):
                        self._enqueue_train(cur, st)
                        if not self.multi:
                            self._enqueue_update(st)
                    self._fork_join(s, lambda sp: self._enqueue_prep(nxt, sp), train)
                ph[("step" if not self.multi else "compute") + str(i)] = step
        if self.multi:
            ph["update"] = self._enqueue_update
        return ph

    # ----------------------------------------------------------------- graphs
    def _state_tensors(self):
        d = self.dm
        ts = [d.flat_w, d.flat_m, d.flat_v, d.step_dev, self.cursor, self.loss_ring]
        if self.cache is not None:
            ts.append(self.cache.hit_miss)
        return ts

    def _warm(self):
        """Run every phase once eagerly (module loading, first-touch) and
        restore all mutable state afterwards."""
        snap = [t.clone() for t in self._state_tensors()]
        with torch.cuda.stream(self.stream):
            for fn in self._phases().values():
                fn(self.stream.cuda_stream)
        torch.cuda.synchronize(self.device)
        for t, v in zip(self._state_tensors(), snap):
            t.copy_(v)
        self.tw.loss.zero_()
        self.dm.nonfinite.zero_()
        torch.cuda.synchronize(self.device)

    def capture(self):
        """Eager warm-up (state restored), then capture each phase as a graph."""
        if self.graphs:
            return
        self._warm()
        self.launches_per_phase = {}
        for name, fn in self._phases().items():
            graph = torch.cuda.CUDAGraph()
            before = lib().mq_launch_count()
            with torch.cuda.graph(graph, stream=self.stream):
                fn(torch.cuda.current_stream().cuda_stream)
            self.launches_per_phase[name] = int(lib().mq_launch_count() - before)
            self.graphs[name] = graph
        torch.cuda.synchronize(self.device)
        if self.pipeline and not self._primed:
            self._prologue()

    def kernels_per_step(self) -> int:
        """libmqgnn kernel launches in one steady-state step (counted while the
        step's graphs were captured)."""
        ph = self.launches_per_phase
        if self.multi:
            return ph.get("compute0", 0) + ph.get("update", 0)
        return ph.get("step0", 0)

    def eager_window(self):
        """One window enqueued eagerly (not from the graphs) — used by the bench
        to time each kernel with CUDA events; same kernels, same buffers."""
        g = self.use_graph
        self.use_graph = False
        try:
            self.compute_window()
            if not self.multi:
                self.apply_window()
        finally:
            self.use_graph = g

    def _replay(self, name):
        with torch.cuda.stream(self.stream):
            if self.use_graph:
                self.graphs[name].replay()
            else:
                self._phases()[name](self.stream.cuda_stream)

    # RaCoM protocol (racom.WindowDriver): compute -> exchange grad64 -> apply.
    # A lone replica's compute already contains its update ("step" graph).
    def compute_window(self):
        if self.pipeline and not self._primed:
            self._prologue()
        i = self.windows_done % 2 if self.pipeline else 0
        self._replay(("compute" if self.multi else "step") + str(i))

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

    def read_counts(self, slot: int | None = None) -> dict:
        """Device counts of a slot's batch: targets and (n_dst, n_src, nnz) per hop."""
        torch.cuda.synchronize(self.device)
        sw = self.slots[slot if slot is not None else
                        ((self.windows_done - 1) % 2 if self.pipeline else 0)]
        c = torch.cat([sw.n_targets] + [hb.counts for hb in sw.hops]).cpu().tolist()
        hops, nd = [], c[0]
        for h in range(len(sw.hops)):
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
        """Graphs whose prep reads targets staged by the host (no device plan):
        slot i trains while the other slot's host-staged batch is prepared."""
        if "host0" in self.graphs:
            return
        if self.multi:
            raise NotImplementedError("host-input steps are single-replica")
        self._stage = [torch.zeros(4, dtype=torch.int32, pin_memory=True) for _ in self.slots]
        self._loss_host = torch.zeros(1, dtype=torch.float64, pin_memory=True)
        phases = {}
        if not self.pipeline:
            sw = self.slots[0]

            def host0(s):
                self._enqueue_prep(sw, s, setup=False)
                self._enqueue_train(sw, s, commit=False)
                self._enqueue_update(s)
            phases["host0"] = host0
        else:
            phases["hostpro"] = lambda s: self._enqueue_prep(self.slots[0], s, setup=False)
            for i in (0, 1):
                cur, nxt = self.slots[i], self.slots[1 - i]

                def hstep(s, cur=cur, nxt=nxt):
                    def train(st):
                        self._enqueue_train(cur, st, commit=False)
                        self._enqueue_update(st)
                    self._fork_join(s, lambda sp: self._enqueue_prep(nxt, sp, setup=False), train)
                phases[f"host{i}"] = hstep
        snap = [t.clone() for t in self._state_tensors()]
        with torch.cuda.stream(self.stream):
            for fn in phases.values():
                fn(self.stream.cuda_stream)
        torch.cuda.synchronize(self.device)
        for t, v in zip(self._state_tensors(), snap):
            t.copy_(v)
        self.tw.loss.zero_()
        torch.cuda.synchronize(self.device)
        for name, fn in phases.items():
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=self.stream):
                fn(torch.cuda.current_stream().cuda_stream)
            self.graphs[name] = graph
        torch.cuda.synchronize(self.device)

    def _stage_batch(self, slot: int, targets_pinned: torch.Tensor, batch_id: int):
        sw = self.slots[slot]
        n = int(targets_pinned.numel())
        st = self._stage[slot]
        st.numpy().view(np.uint32)[:] = (n, self.seed & 0xFFFFFFFF, self.epoch & 0xFFFFFFFF,
                                        batch_id & 0xFFFFFFFF)
        sw.targets[:n].copy_(targets_pinned, non_blocking=True)
        sw.n_targets.copy_(st[0:1], non_blocking=True)
        sw.key.copy_(st[1:4], non_blocking=True)

    def run_host_batches(self, batches):
        """Public host-buffer entry point (one replica): for each pinned int32
        target batch (batch_id, targets) the step H2D-copies its inputs, trains,
        and D2H-reads its summed loss.  With pipelining, batch k+1 is staged and
        prepared while batch k trains; every batch still gets its own H2D copy
        and its own loss read-back.  Yields (batch_id, loss)."""
        batches = list(batches)
        if not batches:
            return
        with torch.cuda.stream(self.stream):
            if not self.pipeline:
                for bid, t in batches:
                    self._stage_batch(0, t, bid)
                    self.graphs["host0"].replay()
                    self._loss_host.copy_(self.tw.loss, non_blocking=True)
                    self.tw.loss.zero_()
                    self.stream.synchronize()
                    self.dm.host_steps += 1
                    yield bid, float(self._loss_host[0])
                return
            # the host runs one step ahead: step k's loss is read back (its own
            # D2H + event wait) right after step k+1 has been launched
            if not hasattr(self, "_loss_ring_host"):
                self._loss_ring_host = torch.zeros(2, dtype=torch.float64, pin_memory=True)
                self._loss_ev = [torch.cuda.Event(), torch.cuda.Event()]
            self._stage_batch(0, batches[0][1], batches[0][0])
            self.graphs["hostpro"].replay()
            pending = None
            for k, (bid, t) in enumerate(batches):
                cur, nxt = k % 2, 1 - (k % 2)
                if k + 1 < len(batches):
                    self._stage_batch(nxt, batches[k + 1][1], batches[k + 1][0])
                else:  # nothing left to prepare: an empty batch keeps the graph fixed
                    self.slots[nxt].n_targets.zero_()
                self.graphs[f"host{cur}"].replay()
                self._loss_ring_host[cur:cur + 1].copy_(self.tw.loss, non_blocking=True)
                self.tw.loss.zero_()
                self._loss_ev[cur].record(self.stream)
                self.dm.host_steps += 1
                if pending is not None:
                    pbid, pslot = pending
                    self._loss_ev[pslot].synchronize()
                    yield pbid, float(self._loss_ring_host[pslot])
                pending = (bid, cur)
            pbid, pslot = pending
            self._loss_ev[pslot].synchronize()
            yield pbid, float(self._loss_ring_host[pslot])

    def step_from_host(self, targets_pinned: torch.Tensor, batch_id: int) -> float:
        """Single synchronous step from one host batch (no cross-step overlap)."""
        return next(iter(self.run_host_batches([(batch_id, targets_pinned)])))[1]
