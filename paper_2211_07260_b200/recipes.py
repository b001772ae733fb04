"""The paper's five tuning pipelines over a clock-augmented space.

Reference: ``pkg/src/jouletune/tuner.py:509-645`` (paper ``PAPER.md:385-399``):
race-to-idle (time at the top clock), energy-to-solution at the top clock,
each of those followed by a clock sweep for energy with the kernel parameters
pinned, and the global (config x clock) energy search. The base clock is the
listed value nearest ``device.spec.base_clock`` (ties go higher).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Iterable, Mapping, Sequence

from .hardware import CLOCK_PARAM
from .errors import ConfigurationError
from .observer_hooks import BenchmarkObserver
from .records import BenchmarkResult, Objective, ResultCache, UserMetric
from .search import TuningRun, run_strategy
from .sensors import AveragedSensorConfig
from .spaces import KernelConfig, SearchSpace

__all__ = ["PIPELINES", "StageReport", "PipelineReport", "run_pipeline"]

PIPELINES = (
    "race_to_idle",
    "energy_to_solution_maxclock",
    "race_to_idle_plus_clocks",
    "energy_to_solution_plus_clocks",
    "global",
)


@dataclass(frozen=True)
class StageReport:
    label: str
    space_size: int
    best: BenchmarkResult


@dataclass(frozen=True)
class PipelineReport:
    name: str
    stages: tuple[StageReport, ...]
    best: BenchmarkResult

    def to_dict(self) -> dict[str, Any]:
        return {
            "name": self.name,
            "stages": [{"label": s.label, "space_size": s.space_size, "best": s.best.to_dict()} for s in self.stages],
            "best": self.best.to_dict(),
        }


def _nearest_value(values: Iterable[float], target: float) -> float:
    return min(values, key=lambda v: (abs(v - target), -v))


def _pin_kernel_params(space: SearchSpace, config: KernelConfig, clock_param: str) -> SearchSpace:
    out = space
    for p in space.parameters:
        if p.name != clock_param:
            out = out.with_values(p.name, [config[p.name]])
    return out


def run_pipeline(
    name: str,
    space: SearchSpace,
    device,
    observers: Sequence[BenchmarkObserver] = (),
    *,
    clock_param: str = CLOCK_PARAM,
    strategy: str = "exhaustive",
    budget: int | None = None,
    seed: int = 0,
    user_metrics: Sequence[UserMetric] = (),
    constants: Mapping[str, float] | None = None,
    cache: ResultCache | None = None,
    averaged_cfg: AveragedSensorConfig | None = None,
) -> PipelineReport:
    """One of the paper's five recipes over a clock-augmented space."""
    if name not in PIPELINES:
        raise ConfigurationError(f"unknown pipeline {name!r}; choose from {PIPELINES}")
    if clock_param not in space.names:
        raise ConfigurationError(f"pipeline {name!r} needs a {clock_param!r} parameter in the space")
    cache = ResultCache() if cache is None else cache
    clocks = space.parameter(clock_param).values
    top = max(clocks)
    base = _nearest_value(clocks, device.spec.base_clock)
    shared = dict(user_metrics=user_metrics, constants=constants, cache=cache, averaged_cfg=averaged_cfg)
    by_time, by_energy = Objective("time", "minimize"), Objective("energy", "minimize")

    def stage(label: str, sub: SearchSpace, objective: Objective, stage_seed: int) -> StageReport:
        tuning = TuningRun(space=sub, strategy=strategy, objective=objective, budget=budget, seed=stage_seed)
        return StageReport(label, sub.size(), run_strategy(tuning, device, observers, **shared).best)

    at_top = space.with_values(clock_param, [top])
    if name == "race_to_idle":
        stages = (stage("time at max clock", at_top, by_time, seed),)
    elif name == "energy_to_solution_maxclock":
        stages = (stage("energy at max clock", at_top, by_energy, seed),)
    elif name in ("race_to_idle_plus_clocks", "energy_to_solution_plus_clocks"):
        if name == "race_to_idle_plus_clocks":
            first = stage("time at max clock", at_top, by_time, seed)
        else:
            first = stage("energy at base clock", space.with_values(clock_param, [base]), by_energy, seed)
        sweep = _pin_kernel_params(space, first.best.config, clock_param)
        stages = (first, stage("clock sweep for energy", sweep, by_energy, seed + 1))
    else:
        stages = (stage("energy over full space", space, by_energy, seed),)
    return PipelineReport(name=name, stages=stages, best=stages[-1].best)
