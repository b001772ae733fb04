"""Tuned configurations found on B200 (loaded from ``tuned_b200.json``).

The JSON is written by ``scripts/tune_suite.py`` from tuning runs on the GPU
box: per kernel, the time-optimal and energy-optimal (config, clock) plus
the measured GFLOP/s and GFLOPS/W. ``bench.py`` measures the time-optimal
config; ``build()`` precompiles every config listed here.
"""

from __future__ import annotations

import json
from pathlib import Path

TUNED_PATH = Path(__file__).resolve().parent / "tuned_b200.json"


def load() -> dict:
    if TUNED_PATH.exists():
        return json.loads(TUNED_PATH.read_text())
    return {}


def configs_for(kernel: str) -> list[dict]:
    entry = load().get(kernel, {})
    out = []
    for key in ("time_optimal", "energy_optimal"):
        cfg = entry.get(key, {}).get("config")
        if cfg:
            out.append({k: v for k, v in cfg.items() if not k.startswith("nvml_")})
    return out


def best_config(kernel: str, objective: str = "time_optimal") -> dict | None:
    cfg = load().get(kernel, {}).get(objective, {}).get("config")
    if not cfg:
        return None
    return {k: v for k, v in cfg.items() if not k.startswith("nvml_")}
