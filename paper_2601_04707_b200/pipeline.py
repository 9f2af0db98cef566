"""Trace schema kept from the reference (``mqpipe/pipeline.py:24-98``).

The stage vocabulary and the JSONL event layout are unchanged so the
reference's offline tools (``utilization``, ``mqpipe report``, autotune's
``profile_from_trace``) can read traces produced by the device runtime.
Timestamps come from CUDA events on the runtime's streams.
"""

from __future__ import annotations

import json
import threading
from dataclasses import dataclass

STAGES = ("sample", "enqueue_cpu", "transfer", "enqueue_dev",
          "compute_fwd", "compute_bwd", "grad_share", "grad_apply", "sync")

MS_TO_NS = 1_000_000


class PipelineTimeout(RuntimeError):
    """A stage starved past its deadline (pipeline.py:101-102)."""


class PipelineStopped(RuntimeError):
    """Another worker failed (pipeline.py:105-106)."""


@dataclass(frozen=True)
class TraceEvent:
    stage: str
    device: int
    batch: int
    epoch: int
    t_start_ns: int
    t_end_ns: int

    def __post_init__(self):
        if self.stage not in STAGES:
            raise ValueError(f"unknown stage {self.stage!r}")
        if self.t_end_ns < self.t_start_ns:
            raise ValueError("event ends before it starts")

    def to_dict(self) -> dict:
        return {"stage": self.stage, "device": self.device, "batch": self.batch,
                "epoch": self.epoch, "t_start_ns": self.t_start_ns, "t_end_ns": self.t_end_ns}


class Trace:
    """Append-only, thread-safe event collector (pipeline.py:51-98)."""

    def __init__(self):
        self._events = []
        self._lock = threading.Lock()

    def add(self, stage, device, batch, epoch, t_start_ns, t_end_ns):
        ev = TraceEvent(stage, int(device), int(batch), int(epoch), int(t_start_ns),
                        int(t_end_ns))
        with self._lock:
            self._events.append(ev)

    def events(self, stage=None, device=None):
        with self._lock:
            evs = list(self._events)
        if stage is not None:
            evs = [e for e in evs if e.stage == stage]
        if device is not None:
            evs = [e for e in evs if e.device == device]
        return evs

    def __len__(self):
        with self._lock:
            return len(self._events)

    def extend(self, other: "Trace"):
        with self._lock, other._lock:
            self._events.extend(other._events)

    def dump_jsonl(self, path: str):
        with open(path, "w") as fh:
            for ev in self.events():
                fh.write(json.dumps(ev.to_dict()) + "\n")

    @staticmethod
    def load_jsonl(path: str) -> "Trace":
        tr = Trace()
        with open(path) as fh:
            for line in fh:
                line = line.strip()
                if line:
                    d = json.loads(line)
                    tr.add(d["stage"], d["device"], d["batch"], d["epoch"], d["t_start_ns"],
                           d["t_end_ns"])
        return tr


def utilization(trace: Trace, device: int = 0, exclude: int = 20,
                min_for_exclusion: int = 60) -> float:
    """Compute-busy fraction of the traced span (pipeline.py:170-196)."""
    events = [e for e in trace.events(device=device) if e.stage in ("compute_fwd", "compute_bwd")]
    if not events:
        return 0.0
    by_epoch: dict = {}
    for e in events:
        by_epoch.setdefault(e.epoch, {}).setdefault(e.batch, []).append(e)
    busy = span = 0
    for per_batch in by_epoch.values():
        batches = sorted(per_batch.values(), key=lambda evs: min(e.t_start_ns for e in evs))
        if len(batches) >= min_for_exclusion and len(batches) > 2 * exclude:
            batches = batches[exclude:-exclude]
        busy += sum(e.t_end_ns - e.t_start_ns for evs in batches for e in evs)
        span += (max(e.t_end_ns for evs in batches for e in evs)
                 - min(e.t_start_ns for evs in batches for e in evs))
    return busy / span if span > 0 else (1.0 if busy > 0 else 0.0)
