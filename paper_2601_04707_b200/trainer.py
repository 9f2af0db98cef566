"""One replica's per-iteration hot path as captured, pipelined CUDA graphs.

A window = one batch of SAGE forward, summed softmax-CE, backward and the
optimizer ("train": nn.py:116-206 and the RaCoM window apply,
runtime.py:167-195) on a slot that was prepared earlier by the device batch
queue (prep.PrepGroup: batch plan, L hops of sample + relabel, feature gather
— the reference's sample + transfer stages, samplers.py:502-540,
runtime.py:127-143).

The multi-queue pipeline of MQ-GNN (sample -> transfer -> compute -> update,
runtime.py:380-612) is two CUDA streams and two slot groups of depth Q: while
the train stream works through group i one window at a time, the prep stream
fills group 1-i with the next Q batches in ONE batched pass
(mq_prep_batches).  Cross-stream order is carried by CUDA events recorded
between graph launches, so the host never synchronises.

Multi-replica (RaCoM) windows either run the fused peer-memory exchange
inside the train graph ([train -> mq_racom_publish -> mq_racom_apply],
peer.PeerExchange: no host synchronisation, group graphs as for one replica)
or split the train graph around a host-issued collective: [train + pack] ->
f64 all-reduce of [grads | contributor count] (torch.distributed, or
in-process replicas) -> update graph.
"""

from __future__ import annotations

import gc
import os

import ctypes as C

import numpy as np
import torch

from ._lib import lib, ptr
from .engine import FusedTrainWorkspace, TrainWorkspace, capture_graph
from .pipeline import PipelineTimeout
from .prep import PrepGroup, PrepShared


DEFAULT_QUEUE_DEPTH = 16  # measured on B200: 2 < 4 < 8 < 16 (Reddit 20.70M -> 20.92M seeds/s, e2e +2 %)


# device stage stamp tags (mq_trace_stamp; decoded by runtime.device_trace)
TAG_PREP_START, TAG_SAMPLE_END, TAG_GATHER_END = 1, 2, 3
TAG_COMPUTE_START, TAG_FWD_END, TAG_BWD_END, TAG_SHARE_END, TAG_APPLY_END = 10, 11, 12, 13, 14
TAG_SYNC_START, TAG_SYNC_END = 20, 21


class PeerTimeout(PipelineTimeout):
    """A rank waited past the timeout for a peer's window gradient (the
    reference's PipelineTimeout at the rendezvous, pipeline.py:101-106)."""


def raise_device_flag(dm):
    """Raise for the device status word the step kernels set (and clear it):
    bit 0 a non-finite loss / weight (nn.py:74-76), bit 1 an optimizer step
    counter overflow, bit 2 a block row longer than MQ_MAX_FANOUT (structural,
    the head truncated it), bit 3 a peer-exchange wait that timed out."""
    flag = int(dm.nonfinite.item())
    if not flag:
        return
    dm.nonfinite.zero_()
    if flag & 8:
        raise PeerTimeout("a peer rank never published its window gradient (RaCoM apply "
                          "timed out); the replica skipped that update")
    if flag & 4:
        raise ValueError("a sampled block row has more edges than the fused head supports "
                         "(MQ_MAX_FANOUT): the fanout is too large for the fused step")
    if flag & 2:
        raise RuntimeError("optimizer step counter overflow")
    raise FloatingPointError("training step produced NaN or Inf")


class StepRunner:
    """Per-iteration path for one replica on one GPU."""

    def __init__(self, g, model, *, fanouts, batch_size: int, num_train: int, cache=None,
                 optimizer: str = "adam", seed: int = 0, world: int = 1, rank: int = 0,
                 multi: bool = False, use_graph: bool = True, pipeline: bool = True,
                 ring_len: int = 1 << 16, fused: bool = True, queue_depth: int | None = None,
                 layer0: str = "auto", exchange=None, trace_cap: int = 0):
        if optimizer not in ("adam", "sgd"):
            raise ValueError(f"unknown optimizer {optimizer!r}")
        Q = DEFAULT_QUEUE_DEPTH if queue_depth is None else int(queue_depth)
        if Q < 1:
            raise ValueError("queue depth must be at least 1")
        self.g = g
        self.model = model
        self.dm = model.dev
        self.cache = cache
        self.optimizer = optimizer
        self.seed = int(seed)
        self.world, self.rank = int(world), int(rank)
        self.multi = bool(multi)
        # fused peer-memory exchange (peer.PeerExchange): publish + apply run
        # inside the train graph, so multi-rank windows need no host step
        self.fx = exchange if getattr(exchange, "fused", False) else None
        if self.fx is not None and (self.fx.world != self.world or self.fx.rank != self.rank):
            raise ValueError("peer exchange world/rank differ from the runner's")
        self.use_graph = use_graph
        self.pipeline = bool(pipeline)
        self.Q = Q
        dev = g.device
        self.device = dev
        self.shared = PrepShared(g, fanouts, batch_size, Q)
        self.groups = [PrepGroup(g, fanouts, batch_size, Q, self.shared)
                       for _ in range(2 if self.pipeline else 1)]
        self.slots = [s for grp in self.groups for s in grp.slots]
        self.sw = self.slots[0]
        dims = [g.feature_dim] + [int(w.shape[1]) for w in model.weights]
        if dims[-1] != g.num_classes:
            raise ValueError("model output width must equal num_classes")
        # fused: transform-first hidden layers + one-launch head (mq_fused.cu);
        # otherwise the reference-shaped per-op kernels (aggregate-first)
        self.fused = bool(fused)
        if self.fused:
            self.tw = FusedTrainWorkspace(self.sw, dims, g.num_classes, layer0=layer0)
        else:
            self.tw = TrainWorkspace(self.sw, dims, g.num_classes)
        self.num_train = int(num_train)
        self.batch_size = int(batch_size)
        self.perm = torch.zeros(max(self.num_train, 1), dtype=torch.int32, device=dev)
        self.cursor = torch.zeros(2, dtype=torch.int32, device=dev)  # [window, arrivals]
        self.ring_len = int(ring_len)
        self.loss_ring = torch.zeros(self.ring_len, dtype=torch.float64, device=dev)
        self.grad64 = (torch.zeros(self.dm.num_params + 1, dtype=torch.float64, device=dev)
                       if self.multi and self.fx is None else None)
        self.stream = torch.cuda.Stream(device=dev)       # train stream
        self.prep_stream = torch.cuda.Stream(device=dev)  # sample + transfer stream
        # device stage stamps (mq_trace_stamp): [cap][t_ns, tag << 32 | batch]
        self.trace_cap = int(trace_cap)
        self.trace_buf = (torch.zeros(2 * self.trace_cap, dtype=torch.int64, device=dev)
                          if self.trace_cap else None)
        self.trace_cur = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ev_prep = [torch.cuda.Event() for _ in self.groups]
        self.ev_train = [torch.cuda.Event() for _ in self.groups]
        self._desc = {}
        self._hphases = None
        self.graphs = {}
        self.launches_per_phase = {}
        self.windows_done = 0
        self.epoch = 0
        self._primed = False
        self._last = (0, 0)
        # epoch-boundary overlap (single replica, group graphs): g0 is the slot
        # group an epoch starts on; when the previous epoch ended with its
        # train-only last-group graph (_tail_clean), the next epoch's first
        # prep runs on the prep stream while that group still trains, in the
        # OTHER group's slots (g0 alternates), instead of after it
        self.g0 = 0
        self._tail_clean = False
        self._pending_prep = None  # group whose prep a train-only tail deferred
        self._perm_stage = None
        self._perm_i = 0
        self._epoch_windows = -(-self.num_train // (self.batch_size * self.world))
        self._join_current()

    def _join_current(self):
        """Order the runner's streams after the work already queued on the
        caller's current stream: buffers, weights and the cache were created
        (zero-filled, copied) there, and the step graphs run on the side
        streams — without this a fill could land after the first prep pass
        (found by compute-sanitizer racecheck: stale targets in the second
        runner of a process)."""
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)
        self.prep_stream.wait_stream(cur)

    # ---------------------------------------------------------------- epochs
    def begin_epoch(self, epoch: int, perm: np.ndarray):
        """Upload this epoch's shuffled train ids (plan_epoch, runtime.py:95-117)
        and, when pipelined, prepare the first slot group (the prologue)."""
        perm = np.asarray(perm)
        if perm.size != self.num_train:
            raise ValueError("permutation length changed; build a new StepRunner")
        # two persistent pinned staging rows, reused every other epoch once the
        # copy that read them has executed (with a fresh pinned tensor per
        # epoch, a host running epochs ahead of the device hit one 10-60 ms
        # device stall in ~half the 10-epoch bench runs, measured per epoch)
        if self._perm_stage is None:
            self._perm_stage = [torch.empty(perm.size, dtype=torch.int32, pin_memory=True)
                                for _ in range(2)]
            self._perm_ev = [torch.cuda.Event() for _ in range(2)]
        si = self._perm_i
        self._perm_i ^= 1
        self._perm_ev[si].synchronize()
        staged = self._perm_stage[si]
        staged.numpy()[:] = perm
        # the caller's queued work (model / cache updates) first
        self._join_current()
        overlap = (self._tail_clean and self.pipeline and self.use_graph
                   and self.trace_buf is None and self.windows_done == self._epoch_windows
                   and os.environ.get("MQ_EPOCH_OVERLAP", "1") != "0")
        if overlap:
            # the last group (self._last[0]) may still be training: the prep
            # stream alone switches perm / cursor / keys (only prep passes read
            # perm and cursor; the trains read key[2], set_key writes key[0:2])
            # and prepares the other group once its previous trains are done
            self.g0 = 1 - self._last[0]
            self.prep_stream.wait_event(self.ev_train[self.g0])
            cs = self.prep_stream
        else:
            # an in-flight prep pass may still read perm / cursor
            self.stream.wait_stream(self.prep_stream)
            self.g0 = 0
            cs = self.stream
        with torch.cuda.stream(cs):
            self.perm.copy_(staged, non_blocking=True)
            self._perm_ev[si].record(cs)
            self.cursor.zero_()
            if not overlap:
                self.trace_cur.zero_()
            for grp in self.groups:
                grp.set_key(self.seed, epoch)
        self.epoch = epoch
        self.windows_done = 0
        self._tail_clean = False
        self._pending_prep = None  # the new epoch's prologue prepares its first group
        self.dm.ensure_bias(self.dm.host_steps + self._epoch_windows + 8)
        self._primed = False
        if self.pipeline and (self.graphs or not self.use_graph):
            self._prologue(overlap)

    def _prologue(self, overlap: bool = False):
        if not overlap:
            self.prep_stream.wait_stream(self.stream)
        self._run(f"prep{self.g0}", self.prep_stream)
        self.ev_prep[self.g0].record(self.prep_stream)
        self._primed = True

    # --------------------------------------------------------------- enqueue
    def _prep_desc(self, gi: int, host: bool):
        key = (gi, host)
        if key not in self._desc:
            self._desc[key] = self.groups[gi].desc(self.cache, self.perm,
                                                   None if host else self.cursor,
                                                   self.world, self.rank)
        return self._desc[key]

    def _stamp(self, tag: int, s, key=None):
        if self.trace_buf is not None:
            lib().mq_trace_stamp(ptr(self.trace_buf), self.trace_cap, ptr(self.trace_cur), tag,
                                 ptr(key), s)

    def _launch_prep(self, gi: int, host: bool, s):
        """One batched prep pass over group gi; traced runs split it at the
        sample | transfer boundary with stage stamps."""
        grp, desc = self.groups[gi], self._prep_desc(gi, host)
        if self.trace_buf is None:
            grp.launch(desc, s)
            return
        from .prep import PREP_GATHER, PREP_LABELS, PREP_RELABEL, PREP_SAMPLE, PREP_SETUP
        self._stamp(TAG_PREP_START, s)
        try:
            desc.stage_mask = PREP_SETUP | PREP_SAMPLE | PREP_RELABEL
            grp.launch(desc, s)
            self._stamp(TAG_SAMPLE_END, s)
            desc.stage_mask = PREP_GATHER | PREP_LABELS
            grp.launch(desc, s)
        finally:
            desc.stage_mask = 0
        self._stamp(TAG_GATHER_END, s)

    def _enqueue_prep(self, sw, s, setup=True):
        """One batched prep pass filling the whole group that holds slot ``sw``."""
        gi = next(i for i, grp in enumerate(self.groups) if sw in grp.slots)
        self._launch_prep(gi, not setup, s)

    def _enqueue_train(self, sw, s, commit=True, ring=None):
        ring = self.loss_ring if ring is None else ring
        self._stamp(TAG_COMPUTE_START, s, sw.key)
        if self.fused:
            for name, op in self.tw.train_ops(self.dm, sw, ring if commit else None,
                                              self.ring_len, self.world):
                op(s)
                if name == "sage_head":  # loss + dlogits: the forward ends here
                    self._stamp(TAG_FWD_END, s, sw.key)
        else:
            self.tw.launch_forward(self.dm, s, sw)
            self.tw.launch_loss(self.dm, s, sw)
            if commit:
                lib().mq_step_commit(ptr(self.tw.loss), ptr(sw.key), self.world,
                                     ptr(ring), self.ring_len, s)
            self._stamp(TAG_FWD_END, s, sw.key)
            self.tw.launch_backward(self.dm, s, sw)
        self._stamp(TAG_BWD_END, s, sw.key)
        if self.fx is not None:
            self.fx.publish(self.dm.flat_g, self.tw.grad_src(self.dm) if self.fused else None,
                            sw.n_targets, s)
        elif self.grad64 is not None:
            src = self.tw.grad_src(self.dm) if self.fused else None
            lib().mq_pack_grads(ptr(self.dm.flat_g), self.dm.num_params, ptr(sw.n_targets),
                                ptr(self.grad64), C.byref(src) if src is not None else None, s)
        self._stamp(TAG_SHARE_END, s, sw.key)

    def _enqueue_update(self, s):
        self._update(s)
        self._stamp(TAG_APPLY_END, s)

    def _update(self, s):
        if self.fx is not None:
            self.fx.apply(self.dm, self.optimizer, s)
        elif self.grad64 is None:
            self.tw.launch_optimizer(self.dm, self.optimizer, s)
        else:  # scale 0: divide by the all-reduced contributor count (expected[k])
            self.tw.launch_optimizer(self.dm, self.optimizer, s, grad64=self.grad64, scale=0.0)

    def _phases(self):
        """name -> fn(stream) for every graph this runner captures."""
        ph = {}
        for gi, grp in enumerate(self.groups):
            ph[f"prep{gi}"] = (lambda s, gi=gi: self._launch_prep(gi, False, s))
            for q, sw in enumerate(grp.slots):
                def train(s, sw=sw):
                    self._enqueue_train(sw, s)
                    if self._host_exchange is False:
                        self._enqueue_update(s)
                ph[f"train{gi}_{q}"] = train
        if self._host_exchange:
            ph["update"] = self._enqueue_update
        return ph

    @property
    def _host_exchange(self) -> bool:
        """True when the window's gradient exchange is issued by the host
        between a train graph and an update graph."""
        return self.multi and self.fx is None

    # ----------------------------------------------------------------- graphs
    def _state_tensors(self):
        d = self.dm
        ts = [d.flat_w, d.flat_m, d.flat_v, d.step_dev, self.cursor, self.loss_ring]
        if self.cache is not None:
            ts.append(self.cache.hit_miss)
        return ts

    def _warm(self, phases):
        """Run phases once eagerly (module loading, first-touch) and restore
        all mutable state afterwards."""
        snap = [t.clone() for t in self._state_tensors()]
        with torch.cuda.stream(self.stream):
            for fn in phases.values():
                fn(self.stream.cuda_stream)
        # a lagged peer exchange holds the last warm-up window back: apply it
        # now (every rank warms the same windows) so the first real window
        # starts with nothing pending
        self.finish()
        torch.cuda.synchronize(self.device)
        self.trace_cur.zero_()
        for t, v in zip(self._state_tensors(), snap):
            t.copy_(v)
        self.tw.loss.zero_()
        self.dm.nonfinite.zero_()
        torch.cuda.synchronize(self.device)

    def _capture(self, phases):
        for name, fn in phases.items():
            graph = torch.cuda.CUDAGraph()
            before = lib().mq_launch_count()
            with capture_graph(graph, self.stream):
                fn(torch.cuda.current_stream().cuda_stream)
            self.launches_per_phase[name] = int(lib().mq_launch_count() - before)
            self.graphs[name] = graph
        torch.cuda.synchronize(self.device)

    def capture(self):
        """Eager warm-up (state restored), then capture each phase as a graph,
        plus (single replica, pipelined) one graph per slot group that runs
        all Q windows of the group while the other group is prepared."""
        if self.graphs:
            return
        phases = self._phases()
        self._warm(phases)
        self._capture(phases)
        if self.pipeline and not self._host_exchange:
            # whole groups, plus the leading k < Q windows of a group (an
            # epoch's last group, the tail of a steps() call): every window a
            # group-aligned caller issues runs inside a group graph
            for gi in range(2):
                for k in range(1, self.Q + 1):
                    def group(s, gi=gi, k=k):
                        cur = torch.cuda.current_stream(self.device)
                        self.prep_stream.wait_stream(cur)
                        with torch.cuda.stream(self.prep_stream):
                            self._launch_prep(1 - gi, False, self.prep_stream.cuda_stream)
                        for q in range(k):
                            ph = phases[f"train{gi}_{q}"]
                            ph(cur.cuda_stream)
                        cur.wait_stream(self.prep_stream)
                    self._capture({f"group{gi}" if k == self.Q else f"group{gi}_{k}": group})
            if self.trace_buf is None:
                # train-only groups, without the forked prep of the group after
                # them: an epoch's last group (the next epoch's first prep
                # replaces that fork) and a steps() call's partial tail (the
                # fork waits until more windows are asked for)
                sizes = set(range(1, self.Q)) | {(self._epoch_windows - 1) % self.Q + 1}
                for gi in range(2):
                    for c in sorted(sizes):
                        def tgroup(s, gi=gi, c=c):
                            for q in range(c):
                                phases[f"train{gi}_{q}"](s)
                        self._capture({f"tgroup{gi}_{c}": tgroup})
        if self.pipeline and not self._primed:
            self._prologue()

    def kernels_per_step(self) -> float:
        """libmqgnn kernel launches per steady-state window (counted while the
        graphs were captured): the train graph plus 1/Q of a prep pass."""
        ph = self.launches_per_phase
        n = ph.get("train0_0", 0) + ph.get("prep0", 0) / self.Q
        if self._host_exchange:
            n += ph.get("update", 0)
        return n

    def _run(self, name, stream):
        with torch.cuda.stream(stream):
            if self.use_graph:
                self.graphs[name].replay()
            else:
                self._phases()[name](stream.cuda_stream)

    def eager_window(self):
        """One window enqueued eagerly (not from the graphs) — used by the bench
        to time each kernel with CUDA events; same kernels, same buffers."""
        g = self.use_graph
        self.use_graph = False
        try:
            self.compute_window()
            if not self._host_exchange:
                self.apply_window()
        finally:
            self.use_graph = g

    # RaCoM protocol (racom.WindowDriver): compute -> exchange grad64 -> apply.
    # A lone replica's train graph already contains its update.
    def _flush_prep(self):
        """Issue the next group's prep that a train-only tail held back."""
        p = self._pending_prep
        if p is None:
            return
        self._pending_prep = None
        self.prep_stream.wait_event(self.ev_train[p])  # its previous trains
        self._run(f"prep{p}", self.prep_stream)
        self.ev_prep[p].record(self.prep_stream)

    def compute_window(self):
        k, Q = self.windows_done, self.Q
        q = k % Q
        self._flush_prep()
        self._tail_clean = False
        if self.pipeline:
            if not self._primed:
                self._prologue()
            gi = (k // Q + self.g0) % 2
            if q == 0:  # the next group fills the other half while this one trains
                nxt = 1 - gi
                self.prep_stream.wait_event(self.ev_train[nxt])
                self._run(f"prep{nxt}", self.prep_stream)
                self.ev_prep[nxt].record(self.prep_stream)
                self.stream.wait_event(self.ev_prep[gi])
        else:
            gi = 0
            if q == 0:
                self._run("prep0", self.stream)
        self._run(f"train{gi}_{q}", self.stream)
        if self.pipeline and q == Q - 1:
            self.ev_train[gi].record(self.stream)
        self._last = (gi, q)

    def apply_window(self):
        if self._host_exchange:
            self._run("update", self.stream)
        self.dm.host_steps += 1
        self.windows_done += 1

    def finish(self):
        """End of epoch: apply what the pipelined schedule still holds back
        (lag 1: the last window), so every window is applied at the barrier."""
        if self.fx is not None and self.fx.lag > 0:
            with torch.cuda.stream(self.stream):
                self.fx.apply(self.dm, self.optimizer, self.stream.cuda_stream, lag=0)

    def step(self):
        """One window (async; nothing is read back)."""
        if self._host_exchange:
            raise RuntimeError("multi-replica runners need the exchange: use racom.WindowDriver")
        self.compute_window()
        self.apply_window()

    def steps(self, n: int, epoch_windows: int | None = None) -> int:
        """Up to n windows of this epoch (async).  Whole slot groups run as ONE
        graph launch each (prep of the next group forked inside it), the
        rest window by window.  Returns the number of windows issued."""
        if self._host_exchange:
            raise RuntimeError("multi-replica runners need the exchange: use racom.WindowDriver")
        if epoch_windows is None:
            epoch_windows = -(-self.num_train // (self.batch_size * self.world))
        n = min(n, epoch_windows - self.windows_done)
        done = 0
        Q = self.Q
        self._flush_prep()
        while done < n:
            k = self.windows_done
            if self.use_graph and self.pipeline and "group0" in self.graphs and k % Q == 0:
                if not self._primed:
                    self._prologue()
                gi = (k // Q + self.g0) % 2
                c = min(Q, n - done)
                # the epoch's last group: train-only graph (begin_epoch forks
                # the next epoch's first prep beside it)
                tail = f"tgroup{gi}_{c}"
                last = k + c == epoch_windows and tail in self.graphs
                # this call's partial tail mid-epoch: train only as well; the
                # next group's prep is issued by the next call (_flush_prep)
                defer = not last and c < Q and tail in self.graphs
                with torch.cuda.stream(self.stream):
                    # the group graph joins its own prep branch; prep(1-gi)
                    # overwrites the other half, whose last trains preceded it
                    self.stream.wait_event(self.ev_prep[gi])
                    self.graphs[tail if last or defer else
                                f"group{gi}" if c == Q else f"group{gi}_{c}"].replay()
                # every group graph marks its trains done (the overlapped
                # prologue waits on the group it overwrites)
                self.ev_train[gi].record(self.stream)
                if defer:
                    self._pending_prep = 1 - gi
                elif not last:
                    self.ev_prep[1 - gi].record(self.stream)
                self._tail_clean = last
                self._last = (gi, c - 1)
                self.dm.host_steps += c
                self.windows_done += c
                done += c
            else:
                self.compute_window()
                self.apply_window()
                done += 1
        return done

    def state64(self) -> torch.Tensor:
        from .racom import _pack_state
        with torch.cuda.stream(self.stream):
            self._stamp(TAG_SYNC_START, self.stream.cuda_stream)
            out = torch.empty(3 * self.dm.num_params, dtype=torch.float64, device=self.device)
            _pack_state(self.model, out)
        return out

    def load_state64(self, t: torch.Tensor, divisor: int):
        from .racom import _unpack_state
        with torch.cuda.stream(self.stream):
            _unpack_state(self.model, t, divisor)
            self._stamp(TAG_SYNC_END, self.stream.cuda_stream)

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
        """Device counts of a slot's batch: targets and (n_dst, n_src, nnz) per hop
        (default: the slot trained last)."""
        torch.cuda.synchronize(self.device)
        if slot is None:
            gi, q = self._last
            sw = self.groups[gi].slots[q]
        else:
            sw = self.slots[slot]
        c = torch.cat([sw.n_targets] + [hb.counts for hb in sw.hops]).cpu().tolist()
        hops, nd = [], c[0]
        for h in range(len(sw.hops)):
            ns, nnz = c[1 + 2 * h], c[2 + 2 * h]
            hops.append((nd, ns, nnz))
            nd = ns
        return {"n_targets": c[0], "hops": hops}

    def read_trace(self) -> np.ndarray:
        """The epoch's stage stamps as int64 [k, 3] = (t_ns, tag, batch id), in
        append order (stream order per stream)."""
        if self.trace_buf is None:
            return np.zeros((0, 3), dtype=np.int64)
        torch.cuda.synchronize(self.device)
        n = min(int(self.trace_cur.item()), self.trace_cap)
        raw = self.trace_buf[:2 * n].view(n, 2).cpu().numpy()
        out = np.empty((n, 3), dtype=np.int64)
        out[:, 0] = raw[:, 0]
        out[:, 1] = (raw[:, 1].view(np.uint64) >> np.uint64(32)).astype(np.int64)
        out[:, 2] = (raw[:, 1].view(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
        return out

    def losses(self, n_windows: int) -> np.ndarray:
        self.stream.synchronize()
        return self.loss_ring[:n_windows].cpu().numpy()

    def check_finite(self):
        self.stream.synchronize()
        raise_device_flag(self.dm)

    # ------------------------------------------------- host-input (e2e) path
    def capture_host_input(self):
        """Graphs whose prep reads targets staged by the host (no device plan)
        and whose train step leaves the batch loss for a per-step read-back."""
        if self._hphases is not None:
            return
        if self._host_exchange:
            raise NotImplementedError("host-input steps need the fused (peer) exchange "
                                      "when replicas span processes")
        Q = self.Q
        # a ring of pinned staging rows: a row set is reused only after the copies
        # that read it (4 groups earlier) have executed, so the host never waits
        # on the group that is about to train
        self._stage = [torch.zeros((Q, 4), dtype=torch.int32, pin_memory=True) for _ in range(4)]
        # the group's targets, staged host-side by memcpy and sent as ONE H2D
        # copy (per-slot tensor copies cost ~10 us of host time each)
        self._tstage = [torch.zeros(tuple(self.groups[0].targets.shape), dtype=torch.int32,
                                    pin_memory=True) for _ in range(4)]
        self._stage_ev = [torch.cuda.Event() for _ in range(4)]
        self._stage_i = 0
        # the step's loss commit (the head's last CTA) writes straight into this
        # pinned, device-mapped ring (index batch_id % ring_len): the per-step
        # D2H read-back needs no copy node between the step's kernels
        self._loss_hring = torch.zeros(self.ring_len, dtype=torch.float64, pin_memory=True)
        self._win_ev = [torch.cuda.Event() for _ in range(2)]
        self._join_current()
        self._grp_ev = [torch.cuda.Event() for _ in self.groups]
        phases = {}
        for gi, grp in enumerate(self.groups):
            phases[f"hprep{gi}"] = (lambda s, gi=gi: self._launch_prep(gi, True, s))
            for q, sw in enumerate(grp.slots):
                def htrain(s, sw=sw):
                    self._enqueue_train(sw, s, commit=True, ring=self._loss_hring)
                    self._enqueue_update(s)
                phases[f"htrain{gi}_{q}"] = htrain
        if self.use_graph:
            self._warm(phases)
            self._capture(phases)
            groups = {}
            for gi, grp in enumerate(self.groups):
                for k in range(1, Q + 1):  # whole groups and a last partial one
                    def hgroup(s, gi=gi, k=k):
                        for q in range(k):
                            phases[f"htrain{gi}_{q}"](s)
                    groups[f"hgroup{gi}" if k == Q else f"hgroup{gi}_{k}"] = hgroup
            self._capture(groups)
        self._hphases = phases

    def _hrun(self, name, stream):
        with torch.cuda.stream(stream):
            if self.use_graph:
                self.graphs[name].replay()
            else:
                self._hphases[name](stream.cuda_stream)

    def _stage_group(self, gi: int, group, stream):
        """H2D: every slot's targets and {n, seed, epoch, batch} (empty slots: n = 0)."""
        grp = self.groups[gi]
        si = self._stage_i
        self._stage_i = (si + 1) % len(self._stage)
        st = self._stage[si]
        self._stage_ev[si].synchronize()
        sv = st.numpy().view(np.uint32)
        tv = self._tstage[si].numpy()
        for q in range(self.Q):
            if q < len(group):
                bid, t = group[q]
                tn = t.numpy()
                tv[q, :tn.size] = tn
                sv[q] = (tn.size, self.seed & 0xFFFFFFFF, self.epoch & 0xFFFFFFFF,
                         bid & 0xFFFFFFFF)
            else:
                sv[q] = (0, self.seed & 0xFFFFFFFF, self.epoch & 0xFFFFFFFF, 0)
        with torch.cuda.stream(stream):
            grp.targets.copy_(self._tstage[si], non_blocking=True)
            grp.n_targets.copy_(st[:, 0:1], non_blocking=True)
            grp.key.copy_(st[:, 1:4], non_blocking=True)
        self._stage_ev[si].record(stream)

    def run_host_batches(self, batches):
        """Public host-buffer entry point (one replica): for each pinned int32
        target batch (batch_id, targets) the step H2D-copies its inputs, trains,
        and D2H-reads its summed loss.  Batches are prepared Q at a time (the
        device queue); group j+1 is staged and prepared while group j trains.
        A full group of Q windows runs as one graph; every window's loss is
        written by the device into a pinned host ring (the D2H read-back of
        the step's result) and the host reads group j's losses after group
        j+1 is enqueued, so the GPU never idles on the host.  Yields
        (batch_id, loss) in order."""
        batches = list(batches)
        if not batches:
            return
        self.capture_host_input()
        # the loop is host-bound at ~60 us per batch: a cyclic-GC pass over
        # the process heap (milliseconds) would stall the device queue
        gc_was = gc.isenabled()
        gc.disable()
        try:
            yield from self._run_host_batches(batches)
        finally:
            if gc_was:
                gc.enable()

    def _run_host_batches(self, batches):
        Q = self.Q
        self._flush_prep()
        self._tail_clean = False
        chunks = [batches[i:i + Q] for i in range(0, len(batches), Q)]
        prep_s = self.prep_stream if self.pipeline else self.stream
        ngroups = len(self.groups)

        def stage_and_prep(j):
            gi = j % ngroups
            prep_s.wait_event(self.ev_train[gi])
            self._stage_group(gi, chunks[j], prep_s)
            self._hrun(f"hprep{gi}", prep_s)
            self.ev_prep[gi].record(prep_s)

        stage_and_prep(0)
        pending = []   # (event, [batch ids]) of enqueued work whose losses are unread
        ring = self._loss_hring.numpy()  # pinned, device-written: a NumPy view reads it directly
        slot_of = lambda bid: ((bid & 0xFFFFFFFF) // self.world) % self.ring_len  # noqa: E731

        def drain(keep):
            while len(pending) > keep:
                ev, ids = pending.pop(0)
                ev.synchronize()
                for bid in ids:
                    yield bid, float(ring[slot_of(bid)])

        def clash(ids):  # a pending loss would be overwritten before it is read
            busy = {slot_of(b) for _, pids in pending for b in pids}
            return any(slot_of(b) in busy for b in ids)

        nwin = 0
        for j, chunk in enumerate(chunks):
            gi = j % ngroups
            if j + 1 < len(chunks) and self.pipeline:
                stage_and_prep(j + 1)
            elif j > 0 and not self.pipeline:
                stage_and_prep(j)
            self.stream.wait_event(self.ev_prep[gi])
            ids = [bid for bid, _ in chunk]
            gname = f"hgroup{gi}" if len(chunk) == Q else f"hgroup{gi}_{len(chunk)}"
            if self.use_graph and gname in self.graphs:
                yield from drain(0 if clash(ids) else 1)
                with torch.cuda.stream(self.stream):
                    self.graphs[gname].replay()
                ev = self._grp_ev[gi]
                ev.record(self.stream)
                self.dm.host_steps += len(chunk)
                pending.append((ev, ids))
            else:
                for q, bid in enumerate(ids):
                    yield from drain(0 if clash([bid]) else 1)
                    self._hrun(f"htrain{gi}_{q}", self.stream)
                    ev = self._win_ev[nwin % 2]
                    nwin += 1
                    ev.record(self.stream)
                    self.dm.host_steps += 1
                    pending.append((ev, [bid]))
            self.ev_train[gi].record(self.stream)
            yield from drain(1)
        yield from drain(0)
        raise_device_flag(self.dm)

    def step_from_host(self, targets_pinned: torch.Tensor, batch_id: int) -> float:
        """Single synchronous step from one host batch."""
        return next(iter(self.run_host_batches([(batch_id, targets_pinned)])))[1]
