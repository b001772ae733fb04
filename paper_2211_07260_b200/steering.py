"""From a fitted P*(f) to the clocks worth sweeping (and the sweep files).

* ``optimal_frequency`` — argmin over the grid of P*(f)/f, ties to the higher
  clock (reference ``powermodel.py:387-402``);
* ``frequency_band`` — supported clocks within +-pct of it, never empty
  (``powermodel.py:405-431``);
* CSV / JSON I/O in the reference formats (``powermodel.py:434-497``).

B200 addition: :func:`prepare_sweep` cleans a measured sweep *before* the
unchanged fit — it keys samples by the observed SM clock and drops samples
taken while the board sat on its power cap. On a 1 kW part a long, noisy cap
plateau otherwise defeats the 2 % trailing-run test and the fit snaps the
optimum to the top clock (measured with the reference code).
"""

from __future__ import annotations

import csv
import json
import math
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import ConfigurationError
from .pmodel import FrequencySample, PowerModel

__all__ = ["optimal_frequency", "FrequencyBand", "frequency_band", "prepare_sweep", "read_samples_csv",
           "write_samples_csv", "model_to_json", "model_from_json"]


def optimal_frequency(model: PowerModel, grid: Sequence[float]) -> float:
    """Grid clock minimising P*(f)/f; ties go to the higher clock."""
    if not grid:
        raise ConfigurationError("empty frequency grid")
    best, best_e = None, math.inf
    for f in grid:
        if f <= 0:
            raise ConfigurationError(f"non-positive frequency {f} in grid")
        e = model.predict_power(f) / f
        if e < best_e or (e == best_e and (best is None or f > best)):
            best, best_e = f, e
    return best


@dataclass(frozen=True)
class FrequencyBand:
    clocks: tuple[float, ...]
    reduction: float


def frequency_band(f_opt: float, supported: Sequence[float], pct: float = 0.10) -> FrequencyBand:
    """Supported clocks in [f_opt(1-pct), f_opt(1+pct)]; nearest clock if none."""
    if not supported:
        raise ConfigurationError("empty supported clock list")
    if not 0 <= pct < 1:
        raise ConfigurationError(f"pct must be in [0, 1), got {pct}")
    grid = sorted(supported)
    lo, hi = f_opt * (1.0 - pct), f_opt * (1.0 + pct)
    inside = tuple(c for c in grid if lo <= c <= hi)
    if not inside:
        inside = (min(grid, key=lambda c: (abs(c - f_opt), -c)),)
    return FrequencyBand(inside, 1.0 - len(inside) / len(grid))


def prepare_sweep(
    records: Sequence[dict],
    *,
    power_limit: float | None = None,
    cap_fraction: float = 0.97,
    clock_tolerance: float = 0.03,
) -> tuple[list[FrequencySample], list[dict]]:
    """B200 sweep hygiene before :func:`fit` (reference algorithm untouched).

    ``records`` are dicts with ``requested_mhz``, ``observed_mhz``, ``power_w``
    and optionally ``power_capped`` (NVML SW-power-cap reason seen) and
    ``voltage_v``. A record is dropped when the board was power capped, when
    the observed clock undershoots the requested one by more than
    ``clock_tolerance`` (throttled), or when power sits within
    ``cap_fraction`` of ``power_limit``. Surviving samples are keyed by the
    *observed* clock; duplicates of the same observed clock are averaged.
    Returns (samples sorted by clock, dropped records with a reason).
    """
    kept: dict[float, list[dict]] = {}
    dropped: list[dict] = []
    for rec in records:
        why = None
        if rec.get("power_capped"):
            why = "power cap active"
        elif rec["observed_mhz"] < (1.0 - clock_tolerance) * rec["requested_mhz"]:
            why = "observed clock below requested"
        elif power_limit is not None and rec["power_w"] >= cap_fraction * power_limit:
            why = "power at the limit"
        if why:
            dropped.append({**rec, "dropped": why})
            continue
        kept.setdefault(float(round(rec["observed_mhz"])), []).append(rec)
    samples = []
    for clock in sorted(kept):
        group = kept[clock]
        volts = [g.get("voltage_v") for g in group]
        samples.append(
            FrequencySample(
                frequency=clock,
                power=float(np.mean([g["power_w"] for g in group])),
                voltage=float(np.mean(volts)) if all(x is not None for x in volts) else None,
            )
        )
    return samples, dropped


# -- files --------------------------------------------------------------------------


def read_samples_csv(path: str | Path) -> list[FrequencySample]:
    """Sweep CSV with columns frequency_mhz, power_w[, voltage_v]."""
    try:
        with open(path, newline="") as fh:
            rows = csv.DictReader(fh)
            if rows.fieldnames is None or not {"frequency_mhz", "power_w"} <= set(rows.fieldnames):
                raise ConfigurationError(f"{path} must have columns frequency_mhz, power_w[, voltage_v]")
            out = []
            for row in rows:
                volt = row.get("voltage_v")
                out.append(
                    FrequencySample(
                        float(row["frequency_mhz"]),
                        float(row["power_w"]),
                        float(volt) if volt not in (None, "") else None,
                    )
                )
            return out
    except OSError as exc:
        raise ConfigurationError(f"cannot read {path}: {exc}") from exc
    except ValueError as exc:
        raise ConfigurationError(f"bad numeric value in {path}: {exc}") from exc


def write_samples_csv(samples: Sequence[FrequencySample], path: str | Path) -> None:
    volts = any(s.voltage is not None for s in samples)
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["frequency_mhz", "power_w"] + (["voltage_v"] if volts else []))
        for s in samples:
            row = [f"{s.frequency:.6g}", f"{s.power:.6f}"]
            if volts:
                row.append("" if s.voltage is None else f"{s.voltage:.6f}")
            out.writerow(row)


def model_to_json(model: PowerModel, path: str | Path) -> None:
    with open(path, "w") as fh:
        json.dump(model.to_dict(), fh, indent=2)
        fh.write("\n")


def model_from_json(path: str | Path) -> PowerModel:
    """Bare parameter object, or a fit report nesting it under ``model``."""
    try:
        data = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise ConfigurationError(f"cannot load model from {path}: {exc}") from exc
    if isinstance(data, dict) and isinstance(data.get("model"), dict):
        data = data["model"]
    return PowerModel.from_dict(data)
