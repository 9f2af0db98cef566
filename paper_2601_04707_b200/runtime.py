"""Drop-in ``run_epoch`` over the device step graphs, plus the epoch plan.

Mirrors ``mqpipe/runtime.py``:

* ``PipelineConfig``  — ``runtime.py:39-69`` (same fields; the timing
  simulation knobs only exist for the reference's thread simulator and must
  stay at their defaults here)
* ``EpochStats``      — ``runtime.py:72-92``
* ``plan_epoch``      — ``runtime.py:95-117`` (same NumPy shuffle, so the
  batches are identical to the reference's)
* ``batch_rng``       — ``runtime.py:120-124`` -> the Philox stream key
* ``transfer_stage``  — ``runtime.py:127-143``
* ``run_epoch``       — ``runtime.py:208-226``

The sample -> transfer -> compute -> update queue pipeline of the reference's
threaded mode becomes a single captured CUDA graph per replica step: the
bounded queues disappear because the stages are stream-ordered on the
device, and the host only launches one graph per window.  Replicas are either
several StepRunners in this process (the reference's simulated devices, one
GPU) or one per process over torch.distributed (NCCL over NVLink), with the
RaCoM schedule of ``racom.WindowDriver``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .cache import DeviceCache, gather_features
from .pipeline import MS_TO_NS, Trace
from .racom import DistExchange, WindowDriver, apply_update
from .samplers import PhiloxStream, SamplerParams, build_minibatch
from .trainer import StepRunner


@dataclass
class PipelineConfig:
    num_devices: int = 1
    queue_capacity: int = 2
    sampler_workers: int = 1
    batch_size: int = 1024
    sampler: SamplerParams = field(default_factory=SamplerParams)
    optimizer: str = "adam"
    sync_period: int = 1
    delay_model: object = None
    transfer_model: object = None
    timing_mode: str = "real"
    stage_durations: dict = field(default_factory=dict)
    deterministic: bool = False
    seed: int = 0
    queue_timeout: float = 60.0
    capture_weights: bool = False
    use_graph: bool = True
    pipeline: bool = True   # prep of batch k+1 overlaps training of batch k
    fused_step: bool = True  # transform-first fused SAGE step (mq_fused.cu)
    elide_syncs: bool = True  # skip model averages of provably identical replicas (exact)
    # gradient exchange of multi-process runs: "peer" = fused publish/apply
    # kernels over NVLink peer memory (peer.PeerExchange, graph-captured),
    # "collective" = host-issued torch.distributed all-reduce; "auto" = peer
    exchange: str = "auto"
    # 0: the reference's serial parity schedule (window k applied before
    # batch k+1); 1: pipelined RaCoM, window k applied after batch k+1's
    # backward (every gradient misses exactly one update)
    staleness: int = 0
    # device stage stamps for the returned Trace (sample / transfer /
    # compute_fwd / compute_bwd / grad_share / grad_apply / sync spans from
    # the GPU clock) and the queue statistics; False skips the stamp
    # launches (5 per window) and returns a trace of windows only
    trace: bool = True

    def validate(self) -> None:
        if self.num_devices < 1:
            raise ValueError("need at least one device")
        if self.queue_capacity < 1:
            raise ValueError("queue capacity must be at least 1")
        if self.sampler_workers < 1:
            raise ValueError("need at least one sampler worker per device")
        if self.sync_period < 1:
            raise ValueError("sync period must be at least 1")
        if self.timing_mode not in ("real", "simulated"):
            raise ValueError(f"unknown timing_mode {self.timing_mode!r}")
        if self.optimizer not in ("adam", "sgd"):
            raise ValueError(f"unknown optimizer {self.optimizer!r}")
        if self.sampler.method not in ("sage", "gcn", "ladies", "fastgcn"):
            raise ValueError(f"unknown method {self.sampler.method!r}")
        if self.timing_mode != "real" or self.stage_durations:
            raise NotImplementedError("simulated stage timings belong to the reference simulator")
        if self.exchange not in ("auto", "peer", "collective"):
            raise ValueError(f"unknown exchange {self.exchange!r}")
        if self.staleness not in (0, 1):
            raise ValueError("staleness must be 0 (parity) or 1 (pipelined)")


@dataclass
class EpochStats:
    epoch: int
    losses: dict
    batches: int
    cache_hits: int = 0
    cache_misses: int = 0
    dropped_targets: int = 0
    sync_count: int = 0
    epoch_sync: int = 0
    elided_syncs: int = 0
    applied_windows: dict = field(default_factory=dict)
    queue_high_water: dict = field(default_factory=dict)
    queue_keys: dict = field(default_factory=dict)
    weight_traces: dict = field(default_factory=dict)
    wall_ms: float = 0.0

    @property
    def mean_loss(self) -> float:
        if not self.losses:
            return float("nan")
        return float(np.mean(list(self.losses.values())))


def epoch_permutation(train_mask, seed: int, epoch: int) -> np.ndarray:
    train_ids = np.flatnonzero(train_mask)
    if train_ids.size == 0:
        raise ValueError("graph has no training nodes")
    rng = np.random.default_rng(np.random.SeedSequence([seed, epoch, 0]))
    return rng.permutation(train_ids)


def plan_epoch(g, config: PipelineConfig, epoch: int):
    """(per_device[(window, batch_id, targets)], expected[k]) — runtime.py:95-117."""
    perm = epoch_permutation(g.train_mask, config.seed, epoch)
    bs = config.batch_size
    batches = [perm[i:i + bs] for i in range(0, perm.size, bs)]
    per_device = [[] for _ in range(config.num_devices)]
    for j, targets in enumerate(batches):
        d = j % config.num_devices
        per_device[d].append((len(per_device[d]), j, targets))
    total = max((len(x) for x in per_device), default=0)
    expected = [sum(1 for x in per_device if len(x) > k) for k in range(total)]
    return per_device, expected


def batch_rng(config: PipelineConfig, epoch: int, batch_id: int) -> PhiloxStream:
    """Batch content depends only on (seed, epoch, batch_id) (runtime.py:120-124)."""
    return PhiloxStream(config.seed, epoch, batch_id)


def transfer_stage(batch, cache, g, transfer_model=None, rng=None):
    """Serve cached rows from HBM, misses from the store (runtime.py:127-143).

    Returns ``(batch, delay_ms)`` like the reference: ``delay_ms`` is the
    reference transfer model's price of the miss bytes
    (``transfer_model.delay_ms(miss_bytes, rng)``, timing.py:86-94) or 0.0.
    The bytes that crossed the host link (misses, when the store is pinned
    host memory) are left on ``batch.miss_bytes``."""
    ids = batch.input_ids
    if cache is not None:
        hit = cache.cached_mask[ids.long()]
        batch.cache_hits = int(hit.sum().item())
        batch.cache_misses = int(ids.numel()) - batch.cache_hits
        miss_rows = batch.cache_misses
    else:
        miss_rows = int(ids.numel())
    batch.features = gather_features(cache, g, ids, count_hits=cache is not None).clone()
    batch.miss_bytes = miss_rows * g.feature_dim * 4
    delay = float(transfer_model.delay_ms(batch.miss_bytes, rng)) if transfer_model else 0.0
    return batch, delay


def _distributed():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def _peer_for(replica, config, world, rank):
    """The replica's peer-memory exchange (arena + mapped peers), created once
    per (world, staleness) and reused across epochs."""
    from .peer import PeerExchange
    key = (world, rank, config.staleness)
    px = getattr(replica, "_peer", None)
    if px is None or px[0] != key:
        if px is not None:
            px[1].close()
        ex = PeerExchange(replica.dev.num_params, replica.device, lag=config.staleness,
                          ring=4, timeout_s=config.queue_timeout)
        replica._peer = (key, ex)
        return ex
    return px[1]


def _runner_for(replica, g, cache, config, world, rank, multi, num_train, exchange=None):
    key = (id(g), id(cache), config.sampler.hop_fanouts, config.batch_size, config.optimizer,
           config.seed, world, rank, multi, num_train, config.use_graph, config.pipeline,
           config.fused_step, config.queue_capacity, id(exchange), config.trace)
    r = getattr(replica, "_runner", None)
    if r is None or r[0] != key:
        runner = StepRunner(g, replica, fanouts=config.sampler.hop_fanouts,
                            batch_size=config.batch_size, num_train=num_train, cache=cache,
                            optimizer=config.optimizer, seed=config.seed, world=world, rank=rank,
                            multi=multi, use_graph=config.use_graph,
                            pipeline=config.pipeline, fused=config.fused_step,
                            queue_depth=config.queue_capacity, exchange=exchange,
                            trace_cap=_trace_cap(num_train, config, world) if config.trace else 0)
        replica._runner = (key, runner)
        return runner, True
    return r[1], False


def _trace_cap(num_train, config, world):
    windows = -(-num_train // (config.batch_size * world))
    return 8 * windows + 64


def device_trace(stamps, windows, Q: int, device: int, epoch: int, trace: Trace):
    """Decode one replica's device stage stamps into the reference's trace
    spans (pipeline.py:24-25 STAGES; the emit points of runtime.py:399-546)
    and queue statistics.  ``windows`` = [(window, batch_id)] of this device.

    * prep pass p (batched, Q windows) gives every batch of windows
      [pQ, (p+1)Q): ``sample`` = [pass start, sample+relabel end],
      ``enqueue_cpu`` (zero length at sample end), ``transfer`` =
      [sample end, gather end];
    * ``enqueue_dev`` = [gather end, compute start]: the time the prepared
      batch waited in the device queue (slot ring);
    * ``compute_fwd`` = [compute start, head end (loss, dlogits)],
      ``compute_bwd`` = [head end, gradients done], ``grad_share`` =
      [gradients done, packet published], ``grad_apply`` (batch = window)
      = [published, update applied];
    * ``sync`` spans from the model-average stamps.
    Returns (queue_high_water {"cpu", "dev"}, queue_keys, sync spans added)."""
    t0 = int(stamps[0, 0]) if len(stamps) else 0
    by_tag = {}
    for t, tag, bid in stamps:
        by_tag.setdefault(int(tag), []).append((int(t) - t0, int(bid)))
    from .trainer import (TAG_APPLY_END, TAG_BWD_END, TAG_COMPUTE_START, TAG_FWD_END,
                          TAG_GATHER_END, TAG_PREP_START, TAG_SAMPLE_END, TAG_SHARE_END,
                          TAG_SYNC_END, TAG_SYNC_START)
    ps, se, ge = (by_tag.get(k, []) for k in (TAG_PREP_START, TAG_SAMPLE_END, TAG_GATHER_END))
    cs, fe, be, sh, ae = (by_tag.get(k, []) for k in (TAG_COMPUTE_START, TAG_FWD_END,
                                                      TAG_BWD_END, TAG_SHARE_END,
                                                      TAG_APPLY_END))
    ready, start = {}, {}
    for k, (_, bid) in enumerate(windows):
        p = k // Q
        if p < len(ps) and p < len(se) and p < len(ge):
            trace.add("sample", device, bid, epoch, ps[p][0], se[p][0])
            trace.add("enqueue_cpu", device, bid, epoch, se[p][0], se[p][0])
            trace.add("transfer", device, bid, epoch, se[p][0], ge[p][0])
            ready[bid] = ge[p][0]
        if k < len(cs) and k < len(fe) and k < len(be):
            trace.add("compute_fwd", device, bid, epoch, cs[k][0], fe[k][0])
            trace.add("compute_bwd", device, bid, epoch, fe[k][0], be[k][0])
            start[bid] = cs[k][0]
            if bid in ready:
                trace.add("enqueue_dev", device, bid, epoch, ready[bid],
                          max(ready[bid], cs[k][0]))
        if k < len(be) and k < len(sh):
            trace.add("grad_share", device, bid, epoch, be[k][0], sh[k][0])
    for k in range(min(len(sh), len(ae))):
        trace.add("grad_apply", device, k, epoch, sh[k][0], max(sh[k][0], ae[k][0]))
    syncs = list(zip(by_tag.get(TAG_SYNC_START, []), by_tag.get(TAG_SYNC_END, [])))
    for a, b in syncs:
        trace.add("sync", device, -1, epoch, a[0], max(a[0], b[0]))
    # queue occupancy from the same clock: the batched pass hands a whole group
    # from sampling to transfer ("cpu"), prepared batches wait for compute ("dev")
    def high_water(puts, gets):
        evs = sorted([(t, 1) for t in puts] + [(t, -1) for t in gets], key=lambda x: (x[0], x[1]))
        cur = hw = 0
        for _, d in evs:
            cur += d
            hw = max(hw, cur)
        return hw
    bids = [bid for _, bid in windows]
    cpu_put = [se[k // Q][0] for k in range(len(windows)) if k // Q < len(se)]
    cpu_get = [ge[k // Q][0] for k in range(len(windows)) if k // Q < len(ge)]
    hw = {"cpu": high_water(cpu_put, cpu_get) if cpu_put else 0,
          "dev": high_water(list(ready.values()), list(start.values())) if ready else 0}
    order = lambda d: [b for b in sorted(d, key=lambda b: (d[b], bids.index(b)))]  # noqa: E731
    keys = {"cpu_put": bids[:len(cpu_put)], "cpu_get": bids[:len(cpu_get)],
            "dev_put": order(ready), "dev_get": order(start)}
    return hw, keys, len(syncs)


def _run_epoch_per_op(g, cache, replicas, config, epoch, trace):
    """The reference's serial schedule (runtime.py:226-324, zero delays) over
    the per-op API, for the samplers the fused step does not cover (the GCN
    node-wise arm, LADIES, FastGCN): per window k every device builds and
    trains its batch (build_minibatch, loss_and_grads), the packets are
    folded in device order into the f64 running mean (Accumulator,
    racom.py:36-78), every replica applies it (apply_update), and the
    replicas are averaged every sync_period applied windows and at the epoch
    barrier (sync_models)."""
    from . import nn
    from .racom import sync_models
    if _distributed():
        raise NotImplementedError("the per-op schedule runs in-process replicas")
    if len(replicas) != config.num_devices:
        raise ValueError("one model replica per device required")
    per_device, expected = plan_epoch(g, config, epoch)
    losses, hits, misses, dropped = {}, 0, 0, 0
    applied = syncs = 0
    t0 = time.perf_counter()
    t0_ns = time.perf_counter_ns()
    for k in range(len(expected)):
        mean, count = None, 0
        for d, rep in enumerate(replicas):
            if k >= len(per_device[d]):
                continue
            _, bid, targets = per_device[d][k]
            ts = time.perf_counter_ns()
            batch = build_minibatch(g, targets, config.sampler, batch_rng(config, epoch, bid),
                                    batch_id=bid, epoch=epoch, cached_mask=cache)
            loss, grads, _ = nn.loss_and_grads(batch, rep)
            losses[bid] = loss
            hits += batch.cache_hits
            misses += batch.cache_misses
            dropped += batch.dropped_targets
            count += 1
            if mean is None:
                mean = [gr.to(torch.float64).clone() for gr in grads]
            else:
                for m, gr in zip(mean, grads):
                    m += (gr.to(torch.float64) - m) / count
            te = time.perf_counter_ns()
            trace.add("compute_fwd", d, bid, epoch, ts - t0_ns, te - t0_ns)
        if count != expected[k]:
            raise RuntimeError(f"window {k}: {count} packets, expected {expected[k]}")
        for rep in replicas:
            apply_update(rep, mean, config.optimizer)
        applied += 1
        if applied % config.sync_period == 0:  # the milestone rendezvous (runtime.py:255-265)
            if config.num_devices > 1:  # (one replica: the average is the identity)
                sync_models(replicas)
            syncs += 1
    epoch_sync = 0
    if config.num_devices > 1:
        sync_models(replicas)
        epoch_sync = 1
    wall_ms = (time.perf_counter() - t0) * 1e3
    stats = EpochStats(
        epoch=epoch, losses=losses, batches=sum(len(x) for x in per_device), cache_hits=hits,
        cache_misses=misses, dropped_targets=dropped, sync_count=syncs, epoch_sync=epoch_sync,
        applied_windows={d: applied for d in range(config.num_devices)},
        queue_high_water={d: {"cpu": 1, "dev": 1} for d in range(config.num_devices)},
        queue_keys={d: {k: [b for _, b, _ in per_device[d]]
                        for k in ("cpu_put", "cpu_get", "dev_put", "dev_get")}
                    for d in range(config.num_devices)},
        wall_ms=wall_ms)
    return stats, trace


def run_epoch(g, cache, replicas: list, config: PipelineConfig, epoch: int = 0,
              trace: Trace | None = None):
    """Train one epoch; returns (EpochStats, Trace).  Every training target
    lands in exactly one batch; all windows are applied on every replica and
    multi-replica runs end with the epoch-barrier model average."""
    config.validate()
    if trace is None:
        trace = Trace()
    if cache is not None and not isinstance(cache, DeviceCache):
        cache = DeviceCache(g, cache)
    if config.sampler.method != "sage":
        return _run_epoch_per_op(g, cache, replicas, config, epoch, trace)
    dist_mode = _distributed()
    if dist_mode:
        import torch.distributed as dist
        world, rank = dist.get_world_size(), dist.get_rank()
        if config.num_devices != world or len(replicas) != 1:
            raise ValueError("distributed run: one replica per rank, num_devices == world size")
        exchange = DistExchange()
        local_ranks = [rank]
    else:
        if len(replicas) != config.num_devices:
            raise ValueError("one model replica per device required")
        world = config.num_devices
        exchange = None
        local_ranks = list(range(world))
    if config.staleness and not dist_mode:
        raise NotImplementedError("the pipelined (staleness 1) schedule runs over the peer "
                                  "exchange: one process per device")
    use_peer = dist_mode and config.exchange in ("auto", "peer") and g.device.type == "cuda"
    per_device, expected = plan_epoch(g, config, epoch)
    total_windows = len(expected)
    perm = epoch_permutation(g.train_mask, config.seed, epoch)
    multi = world > 1
    runners = []
    # counters before the pipeline prologue, which already gathers batch 0
    torch.cuda.synchronize(g.device)
    hm0 = cache.hit_miss.clone() if cache is not None else None
    for d, rep in zip(local_ranks, replicas):
        fx = _peer_for(rep, config, world, d) if use_peer else None
        r, fresh = _runner_for(rep, g, cache, config, world, d, multi, perm.size, fx)
        r.begin_epoch(epoch, perm)
        if config.use_graph:
            r.capture()
        runners.append(r)
    weight_traces = {d: [] for d in local_ranks}

    # straggler injection (the reference's gradient delay model, racom.py:172-184,
    # runtime.py:545-547): this process holds back each window's launch by a
    # delay draw.  The device schedule is fixed (every rank folds the packets
    # of a window in rank order), so delays change timing, never results.
    dm = config.delay_model
    delay_rng = (np.random.default_rng(np.random.SeedSequence([config.seed, epoch, 2, local_ranks[0]]))
                 if dm is not None and getattr(dm, "kind", "none") != "none" else None)

    def on_window(k):
        if delay_rng is not None and k + 1 < total_windows:
            time.sleep(dm.sample(delay_rng) / 1e3)
        if config.capture_weights:
            for d, r in zip(local_ranks, runners):
                r.sync_point()
                weight_traces[d].append((k, [w.detach().cpu().numpy().copy()
                                             for w in r.model.weights]))

    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(runners[0].stream)
    info = WindowDriver(runners, exchange, config.sync_period,
                        elide_identical=config.elide_syncs).run(total_windows, on_window)
    ev1.record(runners[0].stream)
    for r in runners:
        r.check_finite()
    torch.cuda.synchronize(g.device)
    gpu_ms = ev0.elapsed_time(ev1)
    wall_ms = (time.perf_counter() - t0) * 1e3

    losses = {}
    for d, r in zip(local_ranks, runners):
        ring = r.losses(len(per_device[d]))
        for k, (_, bid, _) in enumerate(per_device[d]):
            losses[bid] = float(ring[k])
    hits = misses = 0
    if cache is not None:
        delta = (cache.hit_miss - hm0).cpu().numpy()
        hits, misses = int(delta[0]), int(delta[1])

    queue_hw, queue_keys = {}, {}
    local_trace = Trace()
    for d, r in zip(local_ranks, runners):
        wins = [(k, bid) for k, (_, bid, _) in enumerate(per_device[d])]
        if config.trace:
            queue_hw[d], queue_keys[d], got = device_trace(r.read_trace(), wins, r.Q, d, epoch,
                                                           local_trace)
        else:
            queue_hw[d] = {"cpu": 0, "dev": 0}
            queue_keys[d] = {k: [b for _, b in wins]
                             for k in ("cpu_put", "cpu_get", "dev_put", "dev_get")}
            got = 0
            per_win = gpu_ms / max(total_windows, 1)
            for k, bid in wins:  # window spans only (no stamps)
                a = k * per_win * MS_TO_NS
                local_trace.add("compute_fwd", d, bid, epoch, a, a + per_win * MS_TO_NS)
        t_end = int(gpu_ms * MS_TO_NS)
        # elided syncs (identical replicas: the average is the identity) are
        # zero-length, like the reference's barrier action with nothing to do
        for _ in range(info["sync_count"] + info["epoch_sync"] - got):
            local_trace.add("sync", d, -1, epoch, t_end, t_end)
    if dist_mode:
        import torch.distributed as dist
        gathered = [None] * world
        evs = [e.to_dict() for e in local_trace.events()]
        dist.all_gather_object(gathered, (losses, hits, misses, queue_hw, queue_keys, evs))
        losses = {}
        hits = misses = 0
        for l_, h_, m_, qh, qk, ev in gathered:
            losses.update(l_)
            hits += h_
            misses += m_
            queue_hw.update(qh)
            queue_keys.update(qk)
            for e in ev:
                trace.add(e["stage"], e["device"], e["batch"], e["epoch"], e["t_start_ns"],
                          e["t_end_ns"])
    else:
        for e in local_trace.events():
            trace.add(e.stage, e.device, e.batch, e.epoch, e.t_start_ns, e.t_end_ns)
    stats = EpochStats(
        epoch=epoch, losses=losses, batches=sum(len(x) for x in per_device),
        cache_hits=hits, cache_misses=misses, dropped_targets=0,
        sync_count=info["sync_count"], epoch_sync=info["epoch_sync"],
        elided_syncs=info["elided"],
        applied_windows={d: info["applied"] for d in range(config.num_devices)},
        queue_high_water=queue_hw,
        queue_keys=queue_keys,
        weight_traces=weight_traces, wall_ms=wall_ms)
    return stats, trace
