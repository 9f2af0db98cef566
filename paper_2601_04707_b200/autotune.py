"""Queue sizing for the device batch queue (MQ-GNN's adaptive queue, the
reference's ``mqpipe/autotune.py``).

The reference picks the queue depth that hides preparation behind compute
(Eq. 24, ``compute_queue_size``: ceil(max_prep / mean_compute) clamped to
[2, cap]) under a device-memory cap (``compute_cap``: staged batches that fit
beside the model's padded peak).  Those two formulas are kept verbatim here.

On the B200 the queue is a group of Q slots prepared by ONE batched pass
(``mq_prep_batches``), so Q also sets how well the prep kernels amortise
their launch and latency: the per-batch prep time is itself a function of Q,
and the reference's ratio (measured at one Q) under-sizes the queue.
``auto_queue_depth`` therefore measures the pipelined step at each candidate
depth that fits the memory cap and keeps the fastest — the same objective
(prep hidden behind compute, memory-bounded), decided by measurement.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

DEFAULT_DEVICE_MEMORY = None  # None: the device's free memory
MEMORY_MARGIN = 0.075         # autotune.py:20
WARMUP_BATCHES = 20           # autotune.py:21
MIN_FOR_EXCLUSION = 60        # autotune.py:22


class AutotuneError(ValueError):
    pass


def steady_slice(n: int, exclude: int = WARMUP_BATCHES,
                 min_for_exclusion: int = MIN_FOR_EXCLUSION) -> slice:
    """Trim warmup and cooldown batches when enough remain (autotune.py:29-34)."""
    if n >= min_for_exclusion and n > 2 * exclude:
        return slice(exclude, n - exclude)
    return slice(0, n)


def compute_cap(total_memory_bytes: int, peak_memory_bytes: int,
                minibatch_memory_bytes: int, margin: float = MEMORY_MARGIN) -> int:
    """Staged minibatches that fit beside the padded peak (autotune.py:112-129)."""
    if minibatch_memory_bytes <= 0:
        raise AutotuneError("minibatch memory must be positive")
    budget = total_memory_bytes - peak_memory_bytes * (1.0 + margin)
    cap = int(math.floor(budget / minibatch_memory_bytes))
    if cap < 1:
        raise AutotuneError(
            f"no headroom for staged batches: budget {budget:.0f} bytes, "
            f"minibatch {minibatch_memory_bytes} bytes")
    return cap


def compute_queue_size(max_prep_ms: float, mean_compute_ms: float, cap: int) -> int:
    """Depth hiding preparation behind compute, clamped to [2, cap] (Eq. 24,
    autotune.py:132-141)."""
    if mean_compute_ms <= 0:
        raise AutotuneError("mean compute time must be positive")
    if cap < 1:
        raise AutotuneError("memory cap must allow at least one batch")
    depth = math.ceil(max_prep_ms / mean_compute_ms)
    return min(cap, max(2, depth))


@dataclass
class QueueChoice:
    depth: int
    cap: int
    ms_per_window: dict      # depth -> measured pipelined ms per window
    formula_depth: int       # Eq. 24 from the probe's per-batch prep / compute


def _slot_bytes(runner) -> int:
    """Device bytes one queue slot holds (its share of a group's prep buffers:
    targets, per-hop blocks, gathered input rows, labels)."""
    grp = runner.groups[0]
    ts = [grp.targets, grp.n_targets, grp.key, grp.x0, grp.labels]
    for hb in grp.hops:
        ts += [t for t in hb.__dict__.values() if isinstance(t, torch.Tensor)]
    total = sum(t.numel() * t.element_size() for t in ts)
    return max(1, total // max(runner.Q, 1))


def auto_queue_depth(g, model, *, fanouts, batch_size: int, num_train: int, cache=None,
                     optimizer: str = "adam", seed: int = 0, candidates=(2, 4, 8, 16),
                     windows: int = 60, total_memory_bytes=DEFAULT_DEVICE_MEMORY,
                     margin: float = MEMORY_MARGIN) -> QueueChoice:
    """Measure the pipelined step at each candidate queue depth that fits the
    memory cap; return the fastest (ties to the shallower queue).  The model
    is copied, so tuning never perturbs it."""
    from .runtime import epoch_permutation
    from .trainer import StepRunner
    if total_memory_bytes is None:
        total_memory_bytes, _ = torch.cuda.mem_get_info(g.device)
        total_memory_bytes += torch.cuda.memory_allocated(g.device)
    perm = epoch_permutation(g.train_mask, seed, 0)
    timings, cap, formula = {}, None, None
    for q in sorted(set(int(c) for c in candidates)):
        probe = model.copy()
        runner = StepRunner(g, probe, fanouts=fanouts, batch_size=batch_size, num_train=num_train,
                            cache=cache, optimizer=optimizer, seed=seed, queue_depth=q)
        if cap is None:
            peak = torch.cuda.max_memory_allocated(g.device)
            cap = compute_cap(total_memory_bytes, peak, _slot_bytes(runner), margin)
        if q > cap:
            del runner, probe
            continue
        runner.capture()
        runner.begin_epoch(0, perm)
        n_win = -(-num_train // batch_size)
        w = min(windows, max(n_win - 2 * q, q))
        runner.steps(2 * q)  # warm
        torch.cuda.synchronize(g.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(runner.stream)
        done = runner.steps(w)
        e1.record(runner.stream)
        torch.cuda.synchronize(g.device)
        timings[q] = e0.elapsed_time(e1) / max(done, 1)
        if formula is None:  # the reference's Eq. 24 from this probe's per-op times
            from .profiling import op_table
            tab = op_table(runner, reps=5)["ops"]
            prep = sum(v["us"] for k, v in tab.items() if k.startswith("prep_")) / runner.Q
            comp = sum(v["us"] for k, v in tab.items() if not k.startswith("prep_"))
            formula = compute_queue_size(prep, comp, cap)
        del runner, probe
        torch.cuda.empty_cache()
    if not timings:
        raise AutotuneError(f"no candidate depth fits the memory cap {cap}")
    best = min(timings, key=lambda q: (round(timings[q], 4), q))
    return QueueChoice(best, cap, timings, formula if formula is not None else 2)
