"""Search-space partitioner: (config x clock) points sharded over GPUs.

SURVEY §8(e). Every (kernel config, clock) point is independent, so N GPUs
tune N disjoint shards with no data-path collective:

1. ``plan`` enumerates the kernel configs once (the clock product stays
   lazy) and deals whole configs to workers by LPT on an estimated cost
   (uniform cost = round robin), so each config is compiled on one worker
   only and every worker sweeps the full clock list of its configs.
2. ``run_shard`` runs on one worker (one process per GPU, its own device):
   *clock-major* — set a clock once, measure all of the shard's configs at
   it, then move on — so clock switches per worker equal the number of
   clocks, not points. Results go to a per-worker JSON-lines shard in the
   reference ``ResultCache`` format.
3. ``merge`` is the host-side gather: it unions the shards (numeric values
   normalised, so ``810`` and ``810.0`` key alike), restores enumeration
   order and picks the best exactly like a single-process exhaustive
   ``run_strategy`` (first minimum in enumeration order).

``run_distributed`` wires this to ``torch.distributed`` only for a barrier
(gloo): the gather itself is the filesystem.
"""

from __future__ import annotations

import heapq
import json
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Mapping, Sequence

from .hardware import CLOCK_PARAM
from .errors import ConfigurationError, TuningError
from .observer_hooks import BenchmarkObserver
from .sensors import AveragedSensorConfig
from .spaces import KernelConfig, SearchSpace, normalize_value
from .measure import MeasurementSetup
from .records import BenchmarkResult, Objective, ResultCache, UserMetric
from .search import _Evaluator

__all__ = ["Shard", "plan", "run_shard", "merge", "MergedRun", "run_distributed"]


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    configs: tuple[KernelConfig, ...]  # kernel configs (no clock)
    clocks: tuple  # clock values (empty if the space has no clock parameter)
    clock_param: str = CLOCK_PARAM

    def points(self) -> int:
        return len(self.configs) * max(1, len(self.clocks))

    def iter_points(self):
        """Clock-major: every config at clock c before moving to the next clock."""
        if not self.clocks:
            yield from self.configs
            return
        for clock in self.clocks:
            for cfg in self.configs:
                yield KernelConfig(cfg.items + ((self.clock_param, clock),))


def _split_clock(space: SearchSpace, clock_param: str) -> tuple[SearchSpace, tuple]:
    if clock_param not in space.names:
        return space, ()
    clocks = space.parameter(clock_param).values
    for rule in space.restrictions:
        if clock_param in rule.names:
            raise ConfigurationError(f"restriction {rule.expression!r} couples {clock_param}; cannot shard lazily")
    rest = SearchSpace(tuple(p for p in space.parameters if p.name != clock_param), space.restrictions)
    return rest, tuple(clocks)


def plan(
    space: SearchSpace,
    world: int,
    *,
    clock_param: str = CLOCK_PARAM,
    cost: Callable[[KernelConfig], float] | None = None,
) -> list[Shard]:
    """Deal kernel configs to ``world`` workers (LPT on ``cost``, stable)."""
    if world < 1:
        raise ConfigurationError("world must be >= 1")
    kernel_space, clocks = _split_clock(space, clock_param)
    configs = kernel_space.enumerate()
    if not configs:
        raise TuningError("the search space has no valid configurations")
    weights = [float(cost(c)) if cost else 1.0 for c in configs]
    order = sorted(range(len(configs)), key=lambda i: (-weights[i], i))
    heap = [(0.0, r) for r in range(world)]
    owned: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        owned[r].append(i)
        heapq.heappush(heap, (load + weights[i], r))
    return [
        Shard(r, world, tuple(configs[i] for i in sorted(owned[r])), clocks, clock_param) for r in range(world)
    ]


def run_shard(
    shard: Shard,
    device,
    observers: Sequence[BenchmarkObserver] = (),
    *,
    out: str | Path,
    user_metrics: Sequence[UserMetric] = (),
    constants: Mapping[str, float] | None = None,
    averaged_cfg: AveragedSensorConfig | None = None,
) -> dict:
    """Measure every point of one shard (clock-major) into a JSONL shard file."""
    setup = MeasurementSetup(tuple(observers), averaged_cfg or AveragedSensorConfig())
    cache = ResultCache(out)
    evaluator = _Evaluator(device, setup, user_metrics, constants, cache)
    t0 = time.perf_counter()
    for point in shard.iter_points():
        evaluator.evaluate(point)
    elapsed = time.perf_counter() - t0
    stats = {"rank": shard.rank, "points": shard.points(), "executed": evaluator.device_executions,
             "seconds": elapsed}
    Path(str(out) + ".stats.json").write_text(json.dumps(stats) + "\n")
    return stats


@dataclass
class MergedRun:
    best: BenchmarkResult
    history: list[BenchmarkResult]
    cache: ResultCache
    shard_stats: list[dict] = field(default_factory=list)

    @property
    def points_per_second(self) -> float | None:
        if not self.shard_stats:
            return None
        wall = max(s["seconds"] for s in self.shard_stats)
        return sum(s["executed"] for s in self.shard_stats) / wall if wall > 0 else None


def _normalized(result: BenchmarkResult) -> BenchmarkResult:
    cfg = result.config.normalized()
    if cfg == result.config and cfg.key() == result.config.key():
        return result
    return BenchmarkResult(cfg, result.time, result.energy, result.observer_results, result.metrics, result.failed,
                           result.failure_reason)


def merge(
    space: SearchSpace,
    shard_files: Sequence[str | Path],
    *,
    objective: Objective | None = None,
    out: str | Path | None = None,
) -> MergedRun:
    """Host-side gather of shard files into enumeration order + best."""
    objective = objective or Objective("energy")
    merged = ResultCache(out)
    by_key: dict[str, BenchmarkResult] = {}
    stats = []
    for path in shard_files:
        for result in ResultCache(path).results():
            r = _normalized(result)
            by_key.setdefault(r.config.key(), r)
        side = Path(str(path) + ".stats.json")
        if side.exists():
            stats.append(json.loads(side.read_text()))
    history = []
    for cfg in space.enumerate():
        r = by_key.get(cfg.normalized().key())
        if r is None:
            raise TuningError(f"point {cfg} missing from every shard")
        history.append(r)
        merged.put(r)
    ok = [r for r in history if not r.failed]
    if not ok:
        raise TuningError(f"no successful evaluations in {len(history)} attempts")
    return MergedRun(best=min(ok, key=objective.fitness), history=history, cache=merged, shard_stats=stats)


def run_distributed(
    space: SearchSpace,
    make_device: Callable[[int], object],
    observers_factory: Callable[[], Sequence[BenchmarkObserver]],
    *,
    workdir: str | Path,
    rank: int,
    world: int,
    local_rank: int | None = None,
    barrier: Callable[[], None] | None = None,
    objective: Objective | None = None,
    user_metrics: Sequence[UserMetric] = (),
    constants: Mapping[str, float] | None = None,
    cost: Callable[[KernelConfig], float] | None = None,
) -> MergedRun | dict:
    """One rank's part of a sharded exhaustive search; rank 0 returns the merge.

    ``barrier`` is the only synchronisation (e.g. ``torch.distributed.barrier``
    on a gloo group); results travel through ``workdir``.
    """
    workdir = Path(workdir)
    workdir.mkdir(parents=True, exist_ok=True)
    shards = plan(space, world, cost=cost)
    device = make_device(rank if local_rank is None else local_rank)
    stats = run_shard(shards[rank], device, observers_factory(), out=workdir / f"shard{rank}.jsonl",
                      user_metrics=user_metrics, constants=constants)
    if barrier:
        barrier()
    if rank != 0:
        return stats
    return merge(space, [workdir / f"shard{r}.jsonl" for r in range(world)], objective=objective,
                 out=workdir / "merged.jsonl")


def normalize_doc(doc: Mapping) -> dict:
    """JSON-safe copy of a config dict with integral floats as ints."""
    return {k: normalize_value(v) for k, v in doc.items()}
