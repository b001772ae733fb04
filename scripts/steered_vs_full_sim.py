"""Model-steered vs full clock sweep, simulated with B200-calibrated ground truths.

On this pool NVML refuses clock locks and power limits, so the
north star's steered-vs-full comparison cannot run on the hardware. This
study runs the same pipeline on simulated devices whose parameters come from
the round's B200 measurements:

* the board: 1 kW cap, 195..1965 MHz in 15 MHz steps (the B200's supported
  SM clocks), a P(f) ground truth P = min(p_max, p_idle + u * alpha * f * v(f)^2)
  (reference device.py:107-115) with the B200-like knee of SURVEY §7;
* per kernel: alpha * u set so P(1965 MHz) equals the counter-slope power
  measured for the tuned config (tuned_b200.json), and the reference runtime
  law t(f) = t_ref * (kappa * f_ref / f + 1 - kappa) (device.py:169-172) with
  t_ref the measured time, kappa = 1 for the FP32-pipe-bound kernels and 0.5
  for the memory/latency-bound PnPoly slab / grid / cells kernels;
* steered: a noisy (1%) full-load burner sweep -> prepare_sweep (drops the
  power-capped samples) -> fit -> optimal_frequency -> frequency_band(+-10%);
  each kernel is then swept only over the band (powermodel.py:387-431).

Pass criterion (north star): steered best GFLOPS/W >= 0.95 x full-sweep best.

    python scripts/steered_vs_full_sim.py  ->  results/steered_vs_full_sim.json
"""

from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import fit, frequency_band, optimal_frequency, prepare_sweep  # noqa: E402
from paper_2211_07260_b200.device import GroundTruth  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402
from paper_2211_07260_b200.tuned import TUNED_PATH  # noqa: E402

GRID = [float(f) for f in np.arange(195.0, 1966.0, 15.0)]
F_REF = 1965.0
P_IDLE, P_MAX, TAU, BETA = 180.0, 1000.0, 1200.0, 0.0012
KAPPA = {"conv2d": 1.0, "sgemm": 1.0, "pnpoly": 1.0, "pnpoly_slab": 0.5, "pnpoly_grid": 0.5, "pnpoly_cells": 0.5}


def board(alpha_u: float) -> GroundTruth:
    return GroundTruth(p_idle=P_IDLE, p_max=P_MAX, alpha=alpha_u, tau_ft=TAU, beta=BETA, noise_stddev=0.0)


def alpha_for(power_at_ref: float) -> float:
    v = 1.0 + BETA * (F_REF - TAU)
    return (power_at_ref - P_IDLE) / (F_REF * v * v)


def steered_band(seed: int, burner_power: float) -> tuple[float, list[float]]:
    truth = board(alpha_for(burner_power))
    rng = np.random.default_rng(seed)
    recs = []
    for f in GRID:
        p = truth.power(f)
        recs.append({"requested_mhz": f, "observed_mhz": f, "power_w": p * (1 + rng.normal(0, 0.01)),
                     "power_capped": p >= P_MAX})
    samples, _ = prepare_sweep(recs, power_limit=P_MAX)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model = fit(samples, tdp=P_MAX)
    f_opt = optimal_frequency(model, GRID)
    band = frequency_band(f_opt, GRID, 0.10)
    return f_opt, list(band.clocks)


def main():
    tuned = json.loads(TUNED_PATH.read_text())
    # the burner (full FP32 load) draws more than any tuned FP32 kernel; take the highest
    # measured kernel power + 10% as its P(1965 MHz), capped just below the limit
    burner_power = min(0.99 * P_MAX, 1.1 * max(tuned[k]["time_optimal"]["power_w"] for k in ("conv2d", "sgemm")))
    out = {"board": {"p_idle": P_IDLE, "p_max": P_MAX, "tau_mhz": TAU, "beta": BETA, "grid_mhz": [GRID[0], GRID[-1], 15],
                     "burner_power_at_1965": burner_power},
           "kernels": {}}
    seeds = range(20)
    bands = [steered_band(s, burner_power) for s in seeds]
    out["steered_f_opt_mhz"] = [b[0] for b in bands]
    for name, kappa in KAPPA.items():
        entry = tuned.get(name, {}).get("time_optimal")
        if not entry:
            continue
        flops = make_problem(name, **({"n_points": 4096} if "pnpoly" in name else {})).total_flops
        if "pnpoly" in name:
            flops = make_problem("pnpoly").total_flops  # GFLOP/s convention of the brute-force workload
        truth = board(alpha_for(entry["power_w"]))
        t_ref = entry["time_s"]

        def gflops_per_w(f):
            t = t_ref * (kappa * F_REF / f + 1.0 - kappa)
            return flops / (truth.power(f) * t) / 1e9

        full = {f: gflops_per_w(f) for f in GRID}
        f_full = max(full, key=full.get)
        ratios, reductions = [], []
        for f_opt, band in bands:
            best = max(full[f] for f in band)
            ratios.append(best / full[f_full])
            reductions.append(1.0 - len(band) / len(GRID))
        out["kernels"][name] = {
            "kappa": kappa, "measured_power_w_at_1965": entry["power_w"], "measured_time_s": t_ref,
            "full_sweep_optimum_mhz": f_full, "full_sweep_gflops_per_w": round(full[f_full], 3),
            "gflops_per_w_at_1965": round(full[max(GRID)], 3),
            "steered_over_full_min": round(min(ratios), 4), "steered_over_full_median": round(float(np.median(ratios)), 4),
            "pass_fraction": sum(r >= 0.95 for r in ratios) / len(ratios),
            "grid_reduction_median": round(float(np.median(reductions)), 3),
        }
    path = ROOT / "results" / "steered_vs_full_sim.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out["kernels"], indent=1))
    print("steered f_opt (MHz):", sorted(set(out["steered_f_opt_mhz"])))


if __name__ == "__main__":
    main()
