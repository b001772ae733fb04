"""Tuning-landscape analysis over a result cache: Pareto fronts and search difficulty.

Behaviour contract (reference ``pkg/src/jouletune/analysis.py``; SURVEY §8(f)
row 3), applied to B200 caches:

* a :class:`ParetoPoint` has two *maximised* axes (e.g. ``gflops`` and
  ``gflops_per_w``); :func:`pareto_front` keeps the non-dominated points,
  ordered by performance descending, with duplicate coordinate pairs kept
  only at their first occurrence (``analysis.py:51-73``);
* a fitness flow graph has an edge from every valid config to each
  Hamming-1 neighbour with *strictly* lower (minimised) fitness; its sinks
  are the local optima (``analysis.py:76-115``);
* :func:`minima_arrival_distribution` weighs each optimum by where random
  strictly-improving walks end: the exact absorbing-chain solution (walks
  start uniformly on every node, a walk that starts on a sink counts for it)
  or PageRank (damping 0.85, uniform teleport and dangling mass, L1
  tolerance 1e-10) restricted to the optima (``analysis.py:118-202``);
* :func:`proportion_of_centrality` is the share of that weight on optima
  within ``p`` times the global best fitness (``analysis.py:205-243``);
* CSV outputs use the reference columns and ``%.9g`` (``analysis.py:248-268``).

The graph algorithms are vectorised (edge arrays, ``bincount`` scatter) so
a CLBlast-sized space analyses in seconds; results agree with the reference
to rounding (``tests/test_api_parity.py``).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path
from typing import Mapping, Sequence

import numpy as np

from .errors import AnalysisError, ConfigurationError
from .spaces import KernelConfig, SearchSpace

__all__ = ["ParetoPoint", "dominates", "pareto_front", "FitnessFlowGraph", "build_ffg",
           "minima_arrival_distribution", "CentralityCurve", "proportion_of_centrality", "write_pareto_csv",
           "write_centrality_csv"]

DAMPING = 0.85
PAGERANK_TOL = 1e-10
PAGERANK_MAX_ITERS = 10_000
WEIGHT_MODES = ("absorbing", "pagerank")


@dataclass(frozen=True)
class ParetoPoint:
    """One measured config on two maximised axes (performance, efficiency)."""

    config: KernelConfig
    performance: float
    efficiency: float


def dominates(a: ParetoPoint, b: ParetoPoint) -> bool:
    """``a`` is no worse on both axes and strictly better on at least one."""
    no_worse = a.performance >= b.performance and a.efficiency >= b.efficiency
    return no_worse and (a.performance, a.efficiency) != (b.performance, b.efficiency)


def pareto_front(points: Sequence[ParetoPoint]) -> list[ParetoPoint]:
    """Non-dominated points, best performance first (O(n log n) sweep)."""
    if not points:
        return []
    perf = np.array([p.performance for p in points], dtype=float)
    eff = np.array([p.efficiency for p in points], dtype=float)
    # performance descending, then efficiency descending, then input order
    order = np.lexsort((np.arange(len(points)), -eff, -perf))
    front, best = [], -np.inf
    for i in order:
        if eff[i] > best:  # strictly better than every faster point seen so far
            front.append(points[i])
            best = eff[i]
    return front


@dataclass(frozen=True)
class FitnessFlowGraph:
    """Strict-improvement edges between Hamming-1 neighbours (fitness minimised)."""

    nodes: tuple[KernelConfig, ...]
    fitness: Mapping[KernelConfig, float]
    successors: Mapping[KernelConfig, tuple[KernelConfig, ...]]

    @property
    def minima(self) -> tuple[KernelConfig, ...]:
        return tuple(n for n in self.nodes if not self.successors[n])

    def edge_count(self) -> int:
        return sum(map(len, self.successors.values()))

    def edge_arrays(self) -> tuple[np.ndarray, np.ndarray, dict[KernelConfig, int]]:
        """(source, target) node indices of every edge, and the node index."""
        index = {n: i for i, n in enumerate(self.nodes)}
        src = [index[n] for n in self.nodes for _ in self.successors[n]]
        dst = [index[s] for n in self.nodes for s in self.successors[n]]
        return np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64), index


def build_ffg(space: SearchSpace, fitness: Mapping[KernelConfig, float]) -> FitnessFlowGraph:
    """The flow graph of ``space``; every valid config needs a fitness value."""
    nodes = tuple(space.enumerate())
    missing = [n for n in nodes if n not in fitness]
    if missing:
        sample = ", ".join(repr(m.as_dict()) for m in missing[:3])
        raise AnalysisError(f"fitness missing for {len(missing)} of {len(nodes)} configs (e.g. {sample})")
    successors = {n: tuple(m for m in space.neighbors(n) if fitness[m] < fitness[n]) for n in nodes}
    return FitnessFlowGraph(nodes=nodes, fitness=fitness, successors=successors)


def minima_arrival_distribution(graph: FitnessFlowGraph, mode: str = "absorbing") -> dict[KernelConfig, float]:
    """Weight of each local optimum (sums to one) under random improving walks."""
    if mode not in WEIGHT_MODES:
        raise ConfigurationError(f"unknown mode {mode!r}; use absorbing or pagerank")
    if not graph.nodes:
        raise AnalysisError("graph has no nodes")
    return _absorbing(graph) if mode == "absorbing" else _pagerank(graph)


def _absorbing(graph: FitnessFlowGraph) -> dict[KernelConfig, float]:
    """Absorption probabilities B = (I - Q)^-1 R of the uniform improving walk."""
    nodes, sinks = graph.nodes, graph.minima
    n = len(nodes)
    is_sink = {s: j for j, s in enumerate(sinks)}
    transient = [x for x in nodes if x not in is_sink]
    if not transient:
        return {s: 1.0 / len(sinks) for s in sinks}
    row = {x: i for i, x in enumerate(transient)}
    q = np.zeros((len(transient), len(transient)))
    r = np.zeros((len(transient), len(sinks)))
    for x in transient:
        nxt = graph.successors[x]
        step = 1.0 / len(nxt)
        for y in nxt:
            if y in is_sink:
                r[row[x], is_sink[y]] += step
            else:
                q[row[x], row[y]] += step
    absorbed = np.linalg.solve(np.eye(len(transient)) - q, r).sum(axis=0)
    raw = {s: (absorbed[j] + 1.0) / n for s, j in is_sink.items()}  # +1: the walk starting on s
    total = sum(raw.values())
    return {s: w / total for s, w in raw.items()}


def _pagerank(graph: FitnessFlowGraph) -> dict[KernelConfig, float]:
    """Power iteration with uniform teleport and dangling mass, restricted to the optima."""
    n = len(graph.nodes)
    src, dst, index = graph.edge_arrays()
    out_degree = np.bincount(src, minlength=n).astype(float)
    dangling = out_degree == 0
    share = np.zeros(n)
    rank = np.full(n, 1.0 / n)
    for _ in range(PAGERANK_MAX_ITERS):
        np.divide(rank, out_degree, out=share, where=~dangling)
        incoming = np.bincount(dst, weights=share[src], minlength=n)
        updated = (1.0 - DAMPING) / n + DAMPING * (incoming + rank[dangling].sum() / n)
        converged = np.abs(updated - rank).sum() < PAGERANK_TOL
        rank = updated
        if converged:
            break
    sinks = graph.minima
    weights = np.array([rank[index[s]] for s in sinks])
    weights /= weights.sum()
    return {s: float(w) for s, w in zip(sinks, weights)}


@dataclass(frozen=True)
class CentralityCurve:
    p_values: tuple[float, ...]
    proportions: tuple[float, ...]
    f_optimal: float


def proportion_of_centrality(graph: FitnessFlowGraph, weights: Mapping[KernelConfig, float],
                             p_values: Sequence[float]) -> CentralityCurve:
    """Share of arrival weight on optima with fitness <= p * (best fitness), per p >= 1."""
    if any(p < 1.0 for p in p_values):
        raise ConfigurationError("p values must be >= 1")
    if not graph.nodes:
        raise AnalysisError("graph has no nodes")
    f_opt = min(graph.fitness[x] for x in graph.nodes)
    if f_opt <= 0:
        raise AnalysisError(f"proportion of centrality needs positive fitness, best is {f_opt}")
    total = sum(weights.values())
    if total <= 0:
        raise AnalysisError("arrival weights sum to zero")
    shares = tuple(sum(w for x, w in weights.items() if graph.fitness[x] <= p * f_opt) / total for p in p_values)
    return CentralityCurve(tuple(p_values), shares, f_opt)


def write_pareto_csv(points: Sequence[ParetoPoint], front: Sequence[ParetoPoint], path: str | Path) -> None:
    """Every point with an ``is_front`` flag (coordinates shared with a front point count)."""
    front_ids = {id(p) for p in front}
    front_xy = {(p.performance, p.efficiency) for p in front}
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["performance", "efficiency", "is_front"])
        for p in points:
            flag = id(p) in front_ids or (p.performance, p.efficiency) in front_xy
            out.writerow([f"{p.performance:.9g}", f"{p.efficiency:.9g}", int(flag)])


def write_centrality_csv(curve: CentralityCurve, path: str | Path) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["p", "proportion"])
        out.writerows([f"{p:.9g}", f"{share:.9g}"] for p, share in zip(curve.p_values, curve.proportions))
