"""Result records: what one measurement produced and how it is ranked and stored.

Behaviour contract (reference ``pkg/src/jouletune/tuner.py:65-224``):

* a :class:`BenchmarkResult` resolves a metric name against the core fields
  (``time`` in s, ``energy`` in J), then observer readings, then user metrics;
* an :class:`Objective` turns a result into a scalar to *minimise*; failed
  results rank last (+inf), ``maximize`` negates;
* :class:`UserMetric` expressions see ``time``/``energy``, every observer key
  and the run constants, and must produce a finite number;
* :class:`ResultCache` is an append-only JSON-lines file keyed by
  ``KernelConfig.key()``; re-opening it replays every line, so an interrupted
  tuning run resumes with zero repeated device work.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any, Mapping

from .errors import ConfigurationError, MeasurementError
from .expressions import Expression
from .spaces import KernelConfig

__all__ = ["BenchmarkResult", "Objective", "UserMetric", "default_metrics", "ResultCache", "CORE_FIELDS"]

CORE_FIELDS = frozenset({"time", "energy"})
@dataclass(frozen=True)
class BenchmarkResult:
    config: KernelConfig
    time: float
    energy: float
    observer_results: dict[str, float] = field(default_factory=dict)
    metrics: dict[str, float] = field(default_factory=dict)
    failed: bool = False
    failure_reason: str | None = None

    def lookup(self, name: str) -> float:
        """Core field, then observer reading, then user metric."""
        if name in CORE_FIELDS:
            return self.time if name == "time" else self.energy
        for table in (self.observer_results, self.metrics):
            if name in table:
                return table[name]
        known = ["time", "energy"] + sorted(self.observer_results) + sorted(self.metrics)
        raise ConfigurationError(f"result has no metric {name!r}; available: {known}")

    def to_dict(self) -> dict[str, Any]:
        return {
            "config": self.config.as_dict(),
            "time": self.time,
            "energy": self.energy,
            "observer_results": dict(self.observer_results),
            "metrics": dict(self.metrics),
            "failed": self.failed,
            "failure_reason": self.failure_reason,
        }

    @classmethod
    def from_dict(cls, data: Mapping[str, Any]) -> "BenchmarkResult":
        return cls(
            config=KernelConfig.from_dict(data["config"]),
            time=data["time"],
            energy=data["energy"],
            observer_results=dict(data.get("observer_results", {})),
            metrics=dict(data.get("metrics", {})),
            failed=data.get("failed", False),
            failure_reason=data.get("failure_reason"),
        )


@dataclass(frozen=True)
class Objective:
    metric: str = "time"
    direction: str = "minimize"

    def __post_init__(self):
        if self.direction not in ("minimize", "maximize"):
            raise ConfigurationError(f"direction must be minimize or maximize, got {self.direction!r}")

    @classmethod
    def parse(cls, text: str) -> "Objective":
        """``'energy'``, ``'time:min'``, ``'gflops_per_w:max'``."""
        name, _, suffix = text.partition(":")
        direction = {"": "minimize", "min": "minimize", "max": "maximize"}.get(suffix)
        if not name or direction is None:
            raise ConfigurationError(f"bad objective {text!r}; expected NAME[:min|:max]")
        return cls(name, direction)

    def fitness(self, result: BenchmarkResult) -> float:
        if result.failed:
            return math.inf
        value = result.lookup(self.metric)
        return -value if self.direction == "maximize" else value

    def better(self, a: BenchmarkResult, b: BenchmarkResult) -> bool:
        return self.fitness(a) < self.fitness(b)


@dataclass(frozen=True)
class UserMetric:
    name: str
    expression: str

    def __post_init__(self):
        if not self.name.isidentifier():
            raise ConfigurationError(f"metric name {self.name!r} is not an identifier")

    def evaluate(self, env: Mapping[str, float]) -> float:
        value = Expression(self.expression)(env)
        if not isinstance(value, (int, float)) or not math.isfinite(value):
            raise MeasurementError(f"metric {self.name!r} = {self.expression!r} is not finite: {value!r}")
        return float(value)


def default_metrics(total_flops: float) -> tuple[UserMetric, ...]:
    """``gflops`` and ``gflops_per_w`` from a known operation count (time in s)."""
    if total_flops <= 0:
        raise ConfigurationError("total_flops must be positive")
    return (
        UserMetric("gflops", "total_flops / time / 1e9"),
        UserMetric("gflops_per_w", "total_flops / energy / 1e9"),
    )


class ResultCache:
    """Append-only result store keyed by canonical config hash (JSON lines)."""

    def __init__(self, path: str | Path | None = None):
        self.path = None if path is None else Path(path)
        self._entries: dict[str, BenchmarkResult] = {}
        if self.path is not None and self.path.exists():
            for lineno, raw in enumerate(self.path.read_text().splitlines(), 1):
                raw = raw.strip()
                if not raw:
                    continue
                try:
                    result = BenchmarkResult.from_dict(json.loads(raw))
                except (json.JSONDecodeError, KeyError) as exc:
                    raise ConfigurationError(f"corrupt cache line in {self.path}: {exc}") from exc
                self._entries[result.config.key()] = result

    def __len__(self) -> int:
        return len(self._entries)

    def __contains__(self, config: KernelConfig) -> bool:
        return config.key() in self._entries

    def get(self, config: KernelConfig) -> BenchmarkResult | None:
        return self._entries.get(config.key())

    def put(self, result: BenchmarkResult) -> None:
        k = result.config.key()
        if k in self._entries:
            return
        self._entries[k] = result
        if self.path is not None:
            with open(self.path, "a") as fh:
                fh.write(json.dumps(result.to_dict(), sort_keys=True) + "\n")

    def results(self) -> list[BenchmarkResult]:
        return list(self._entries.values())


