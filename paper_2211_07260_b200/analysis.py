"""``jouletune.analysis`` module path; the implementation lives in :mod:`.landscape`."""

from .landscape import (  # noqa: F401
    CentralityCurve, FitnessFlowGraph, ParetoPoint, build_ffg, dominates, minima_arrival_distribution, pareto_front,
    proportion_of_centrality, write_centrality_csv, write_pareto_csv,
)
