"""Search strategies over a space: exhaustive, random, randomised local search.

Reference: ``pkg/src/jouletune/tuner.py:341-506``. The budget counts device
executions (cache hits are free); the history records every evaluation in
order, hits included; the best result is the first minimum of the objective
in history order. RNG use (``default_rng(seed)``: ``permutation`` for random
order, ``integers`` for local-search starts, ``permutation`` for neighbour
order) is kept call for call, so histories match the reference seed for seed.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .errors import ConfigurationError, TuningError
from .measure import MeasurementSetup, benchmark
from .observer_hooks import BenchmarkObserver
from .records import BenchmarkResult, Objective, ResultCache, UserMetric
from .sensors import AveragedSensorConfig
from .spaces import KernelConfig, SearchSpace

__all__ = ["STRATEGIES", "TuningRun", "StrategyOutcome", "run_strategy"]

STRATEGIES = ("exhaustive", "random", "local_search")


@dataclass(frozen=True)
class TuningRun:
    space: SearchSpace
    strategy: str = "exhaustive"
    objective: Objective = field(default_factory=Objective)
    budget: int | None = None
    seed: int = 0

    def __post_init__(self):
        if self.strategy not in STRATEGIES:
            raise ConfigurationError(f"unknown strategy {self.strategy!r}; choose from {STRATEGIES}")
        if self.budget is not None and self.budget < 1:
            raise ConfigurationError("budget must be >= 1")


@dataclass
class StrategyOutcome:
    best: BenchmarkResult
    history: list[BenchmarkResult]
    minima_reached: list[KernelConfig]
    device_executions: int
    evaluations: int


class _Evaluator:
    """Cache-aware benchmark wrapper counting real device executions."""

    def __init__(self, device, setup: MeasurementSetup, user_metrics, constants, cache):
        self.device = device
        self.setup = setup
        self.user_metrics = tuple(user_metrics)
        self.constants = dict(constants or {})
        self.cache = cache if cache is not None else ResultCache()
        self.device_executions = 0
        self.evaluations = 0

    def evaluate(self, config: KernelConfig) -> tuple[BenchmarkResult, bool]:
        self.evaluations += 1
        hit = self.cache.get(config)
        if hit is not None:
            return hit, False
        result = benchmark(
            self.device,
            config,
            self.setup.observers,
            user_metrics=self.user_metrics,
            constants=self.constants,
            averaged_cfg=self.setup.averaged,
        )
        self.cache.put(result)
        self.device_executions += 1
        return result, True


class _Budget:
    def __init__(self, limit: int):
        self.left = limit

    def spent(self) -> bool:
        return self.left <= 0

    def charge(self, executed: bool) -> None:
        if executed:
            self.left -= 1


def run_strategy(
    run: TuningRun,
    device,
    observers: Sequence[BenchmarkObserver] = (),
    *,
    user_metrics: Sequence[UserMetric] = (),
    constants: Mapping[str, float] | None = None,
    cache: ResultCache | None = None,
    averaged_cfg: AveragedSensorConfig | None = None,
) -> StrategyOutcome:
    """One search; history includes cache hits, the budget counts executions."""
    setup = MeasurementSetup(tuple(observers), averaged_cfg or AveragedSensorConfig())
    evaluator = _Evaluator(device, setup, user_metrics, constants, cache)
    configs = run.space.enumerate()
    if not configs:
        raise TuningError("the search space has no valid configurations")
    rng = np.random.default_rng(run.seed)
    history: list[BenchmarkResult] = []
    minima: list[KernelConfig] = []

    if run.strategy == "exhaustive":
        history.extend(evaluator.evaluate(c)[0] for c in configs)
    elif run.strategy == "random":
        budget = _Budget(len(configs) if run.budget is None else run.budget)
        for idx in rng.permutation(len(configs)):
            if budget.spent():
                break
            result, executed = evaluator.evaluate(configs[idx])
            history.append(result)
            budget.charge(executed)
    else:
        _local_search(run, configs, evaluator, rng, history, minima)

    ok = [r for r in history if not r.failed]
    if not ok:
        raise TuningError(f"no successful evaluations in {len(history)} attempts")
    return StrategyOutcome(
        best=min(ok, key=run.objective.fitness),
        history=history,
        minima_reached=minima,
        device_executions=evaluator.device_executions,
        evaluations=evaluator.evaluations,
    )


def _local_search(run, configs, evaluator: _Evaluator, rng, history, minima) -> None:
    """First-improvement walks from random starts until the budget is spent.

    Once every config is cached the search stops after the current walk, as
    further restarts could only replay cached results.
    """
    fitness = run.objective.fitness
    budget = _Budget(len(configs) if run.budget is None else run.budget)

    def visit(config):
        if budget.spent():
            return None
        result, executed = evaluator.evaluate(config)
        budget.charge(executed)
        history.append(result)
        return result

    while not budget.spent():
        here = visit(configs[int(rng.integers(len(configs)))])
        if here is None:
            return
        improved = True
        while improved:
            improved = False
            around = run.space.neighbors(here.config)
            for idx in rng.permutation(len(around)):
                candidate = visit(around[int(idx)])
                if candidate is None:
                    return
                if fitness(candidate) < fitness(here):
                    here, improved = candidate, True
                    break
            if not improved:
                minima.append(here.config)
        if len(evaluator.cache) >= len(configs):
            return


