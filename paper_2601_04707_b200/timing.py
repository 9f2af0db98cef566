"""Delay models (``mqpipe/timing.py:10-54``), kept as the host-side straggler
injector of ``run_epoch`` (``PipelineConfig.delay_model``).

The reference uses them to price simulated transfers and to delay gradient
packets between its thread "devices"; on real devices the schedule is fixed
by stream order and the rank-ordered fold, so a delay only holds back a
rank's launches (a straggler) and never changes results.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class DurationModel:
    """A nonnegative duration in milliseconds: none, fixed, or uniform[a, b]."""

    kind: str = "fixed"  # fixed | uniform | none
    a: float = 0.0
    b: float = 0.0

    @staticmethod
    def parse(spec: str) -> "DurationModel":
        """'none' | 'fixed:10' | 'uniform:2,5' | bare number (timing.py:17-33)."""
        spec = spec.strip().lower()
        if spec in ("none", ""):
            return DurationModel("none")
        if ":" not in spec:
            return DurationModel("fixed", float(spec))
        kind, _, args = spec.partition(":")
        if kind == "fixed":
            return DurationModel("fixed", float(args))
        if kind == "uniform":
            lo, hi = (float(x) for x in args.split(","))
            if hi < lo:
                raise ValueError(f"uniform range reversed in {spec!r}")
            return DurationModel("uniform", lo, hi)
        raise ValueError(f"unknown duration spec {spec!r}")

    def sample(self, rng) -> float:
        if self.kind == "none":
            return 0.0
        if self.kind == "fixed":
            return self.a
        return float(rng.uniform(self.a, self.b))

    @property
    def max_value(self) -> float:
        return {"none": 0.0, "fixed": self.a, "uniform": self.b}[self.kind]


NO_DELAY = DurationModel("none")
