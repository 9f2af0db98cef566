"""CPU restatement of RaCoM windowing and the epoch plan — test oracle.

* ``plan_epoch``          — ``mqpipe/runtime.py:95-117``
* ``RunningMean``         — ``mqpipe/racom.py:36-78`` (f64 running mean)
* ``sync_models``         — ``mqpipe/racom.py:118-139``
* ``compute_sync_period`` — ``mqpipe/racom.py:90-106``
* ``run_epoch_serial``    — ``mqpipe/runtime.py:233-373`` restricted to the
  zero-delay schedule (no duration/delay models), which is the reference's
  bit-reproducible parity mode: per window every device computes its batch on
  its current replica, the f64 mean over ``expected[k]`` contributors is
  applied in window order, and replicas are averaged every ``sync_period``
  applied windows plus once at the epoch barrier.
"""

from __future__ import annotations

import math

import numpy as np

from . import nn as onn
from .sampler import build_minibatch


def plan_epoch(train_mask, num_devices, batch_size, seed, epoch):
    train_ids = np.flatnonzero(train_mask)
    if train_ids.size == 0:
        raise ValueError("graph has no training nodes")
    rng = np.random.default_rng(np.random.SeedSequence([seed, epoch, 0]))
    perm = rng.permutation(train_ids)
    batches = [perm[i:i + batch_size] for i in range(0, perm.size, batch_size)]
    per_device = [[] for _ in range(num_devices)]
    for j, targets in enumerate(batches):
        d = j % num_devices
        per_device[d].append((len(per_device[d]), j, targets))
    total = max((len(x) for x in per_device), default=0)
    expected = [sum(1 for x in per_device if len(x) > k) for k in range(total)]
    return per_device, expected


class RunningMean:
    """mean += (g - mean) / count in f64 (racom.py:47-57)."""

    def __init__(self):
        self.mean = None
        self.count = 0

    def add(self, grads):
        self.count += 1
        if self.mean is None:
            self.mean = [np.asarray(g, dtype=np.float64).copy() for g in grads]
        else:
            for acc, g in zip(self.mean, grads):
                acc += (np.asarray(g, dtype=np.float64) - acc) / self.count


def sync_models(models):
    steps = {m.step_count for m in models}
    if len(steps) != 1:
        raise RuntimeError(f"sync with unequal step counts: {sorted(steps)}")
    n = len(models)
    for l in range(len(models[0].weights)):
        for attr in ("weights", "m", "v"):
            mean = sum(getattr(r, attr)[l].astype(np.float64) for r in models) / n
            for r in models:
                arr = getattr(r, attr)[l]
                arr[...] = mean.astype(arr.dtype)


def compute_sync_period(num_nodes, num_edges, num_devices, scale_k=1.0):
    if num_nodes <= 0 or num_devices <= 0:
        raise ValueError("need positive node and device counts")
    if num_edges == 0:
        period = math.ceil(scale_k * math.sqrt(num_nodes))
    else:
        period = math.ceil(scale_k * math.sqrt(num_nodes)
                           / math.sqrt(num_devices * num_edges))
    return max(1, period)


def run_epoch_serial(graph, models, *, fanouts, batch_size, seed, epoch,
                     optimizer="adam", sync_period=1, cached_mask=None,
                     capture_weights=False, staleness=0):
    """Zero-delay serial schedule; returns (losses{bid: loss}, weight_traces).

    staleness=1 is the pipelined RaCoM schedule (the threaded
    reference's one-window run-ahead, runtime.py:489-511, made deterministic):
    window k's gradients are computed before window k-1's mean is applied,
    so every gradient misses exactly one update; the last window is applied
    at the epoch barrier.  Milestone syncs count processed windows."""
    G = len(models)
    per_device, expected = plan_epoch(graph["train_mask"], G, batch_size, seed,
                                      epoch)
    step = onn.adam_step if optimizer == "adam" else onn.sgd_step
    losses = {}
    traces = {d: [] for d in range(G)}
    applied = 0
    milestone = sync_period
    pending = None
    for k in range(len(expected)):
        acc = RunningMean()
        for d in range(G):
            if k >= len(per_device[d]):
                continue
            _, bid, targets = per_device[d][k]
            mb = build_minibatch(graph["row_offsets"], graph["col_indices"],
                                 graph["features"], graph["labels"], targets,
                                 fanouts, seed=seed, epoch=epoch, batch_id=bid,
                                 cached_mask=cached_mask)
            loss, grads, _ = onn.loss_and_grads(mb.layers, mb.features,
                                                mb.target_labels,
                                                models[d].weights)
            losses[bid] = loss
            acc.add(grads)
        assert acc.count == expected[k]
        if staleness:
            ready, pending = pending, acc.mean
        else:
            ready = acc.mean
        if ready is not None:
            for d in range(G):
                step(models[d], ready)
                if capture_weights:
                    traces[d].append((k, [w.copy() for w in models[d].weights]))
        applied += 1
        if applied >= milestone:
            sync_models(models)
            milestone += sync_period
    if staleness and pending is not None:
        for d in range(G):
            step(models[d], pending)
    if G > 1:
        sync_models(models)
    return losses, traces
