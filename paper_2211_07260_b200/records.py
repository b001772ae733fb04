"""Result records: what one measurement produced, how it ranks, where it is kept.

Behaviour contract (reference ``pkg/src/jouletune/tuner.py:65-224``):

* a :class:`BenchmarkResult` resolves a metric name against the core fields
  (``time`` in s, ``energy`` in J), then observer readings, then user metrics;
* an :class:`Objective` maps a result to a scalar to *minimise*: failed
  results rank last (+inf) and ``maximize`` negates the metric;
* :class:`UserMetric` expressions see ``time``/``energy``, every observer key
  and the run constants, and must evaluate to a finite number;
* :class:`ResultCache` is an append-only JSON-lines file keyed by
  ``KernelConfig.key()``; re-opening it replays every line, so an interrupted
  run resumes with no repeated device work, and the line format is the
  reference's (``sort_keys`` JSON of ``BenchmarkResult.to_dict()``).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any, Iterator, Mapping

from .errors import ConfigurationError, MeasurementError
from .expressions import Expression
from .spaces import KernelConfig

__all__ = ["BenchmarkResult", "Objective", "UserMetric", "default_metrics", "ResultCache", "CORE_FIELDS"]

CORE_FIELDS = frozenset({"time", "energy"})
_DIRECTIONS = {"": "minimize", "min": "minimize", "max": "maximize"}


@dataclass(frozen=True)
class BenchmarkResult:
    """One evaluated config (failed evaluations carry inf time/energy and a reason)."""

    config: KernelConfig
    time: float
    energy: float
    observer_results: dict[str, float] = field(default_factory=dict)
    metrics: dict[str, float] = field(default_factory=dict)
    failed: bool = False
    failure_reason: str | None = None

    def _namespaces(self) -> Iterator[Mapping[str, float]]:
        yield {"time": self.time, "energy": self.energy}
        yield self.observer_results
        yield self.metrics

    def lookup(self, name: str) -> float:
        for table in self._namespaces():
            if name in table:
                return table[name]
        available = ["time", "energy", *sorted(self.observer_results), *sorted(self.metrics)]
        raise ConfigurationError(f"result has no metric {name!r}; available: {available}")

    def to_dict(self) -> dict[str, Any]:
        doc: dict[str, Any] = {"config": self.config.as_dict(), "time": self.time, "energy": self.energy}
        doc["observer_results"] = dict(self.observer_results)
        doc["metrics"] = dict(self.metrics)
        doc["failed"] = self.failed
        doc["failure_reason"] = self.failure_reason
        return doc

    @classmethod
    def from_dict(cls, doc: Mapping[str, Any]) -> "BenchmarkResult":
        optional = {
            "observer_results": dict(doc.get("observer_results", {})),
            "metrics": dict(doc.get("metrics", {})),
            "failed": doc.get("failed", False),
            "failure_reason": doc.get("failure_reason"),
        }
        return cls(KernelConfig.from_dict(doc["config"]), doc["time"], doc["energy"], **optional)


@dataclass(frozen=True)
class Objective:
    """Metric name + direction; ``fitness`` is what every strategy minimises."""

    metric: str = "time"
    direction: str = "minimize"

    def __post_init__(self):
        if self.direction not in _DIRECTIONS.values():
            raise ConfigurationError(f"direction must be minimize or maximize, got {self.direction!r}")

    @classmethod
    def parse(cls, text: str) -> "Objective":
        """``'energy'``, ``'time:min'``, ``'gflops_per_w:max'``."""
        name, _, suffix = text.partition(":")
        if not name or suffix not in _DIRECTIONS:
            raise ConfigurationError(f"bad objective {text!r}; expected NAME[:min|:max]")
        return cls(name, _DIRECTIONS[suffix])

    def fitness(self, result: BenchmarkResult) -> float:
        if result.failed:
            return math.inf
        sign = -1.0 if self.direction == "maximize" else 1.0
        value = result.lookup(self.metric)
        return value if sign > 0 else -value

    def better(self, a: BenchmarkResult, b: BenchmarkResult) -> bool:
        return self.fitness(a) < self.fitness(b)


@dataclass(frozen=True)
class UserMetric:
    """A named expression derived from every result (e.g. GFLOPS/W)."""

    name: str
    expression: str

    def __post_init__(self):
        if not self.name.isidentifier():
            raise ConfigurationError(f"metric name {self.name!r} is not an identifier")

    def evaluate(self, env: Mapping[str, float]) -> float:
        value = Expression(self.expression)(env)
        finite = isinstance(value, (int, float)) and math.isfinite(value)
        if not finite:
            raise MeasurementError(f"metric {self.name!r} = {self.expression!r} is not finite: {value!r}")
        return float(value)


def default_metrics(total_flops: float) -> tuple[UserMetric, ...]:
    """``gflops`` and ``gflops_per_w`` for a known operation count (time in s, energy in J)."""
    if total_flops <= 0:
        raise ConfigurationError("total_flops must be positive")
    return UserMetric("gflops", "total_flops / time / 1e9"), UserMetric("gflops_per_w", "total_flops / energy / 1e9")


class ResultCache:
    """Results keyed by config hash, optionally mirrored to a JSON-lines file."""

    def __init__(self, path: str | Path | None = None):
        self.path = Path(path) if path is not None else None
        self._by_key: dict[str, BenchmarkResult] = {}
        if self.path is not None and self.path.exists():
            self._replay(self.path)

    def _replay(self, path: Path) -> None:
        for raw in path.read_text().splitlines():
            if not raw.strip():
                continue
            try:
                result = BenchmarkResult.from_dict(json.loads(raw))
            except (json.JSONDecodeError, KeyError) as exc:
                raise ConfigurationError(f"corrupt cache line in {path}: {exc}") from exc
            self._by_key[result.config.key()] = result

    def __len__(self) -> int:
        return len(self._by_key)

    def __contains__(self, config: KernelConfig) -> bool:
        return config.key() in self._by_key

    def get(self, config: KernelConfig) -> BenchmarkResult | None:
        return self._by_key.get(config.key())

    def put(self, result: BenchmarkResult) -> None:
        """Store once (first write wins) and append it to the file."""
        key = result.config.key()
        if key in self._by_key:
            return
        self._by_key[key] = result
        if self.path is not None:
            with self.path.open("a") as fh:
                fh.write(json.dumps(result.to_dict(), sort_keys=True) + "\n")

    def results(self) -> list[BenchmarkResult]:
        return list(self._by_key.values())
