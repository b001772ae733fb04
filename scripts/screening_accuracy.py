"""How well do 0.3 s sweep windows rank configs by energy? (CPU, over committed B200 results)

Every exhaustive sweep (scripts/tune_paper_space.py) measures each config once in a
0.3 s loop: energy = the NVML energy-counter slope over its two updates inside the
steady window x per-launch runtime, with the instant-power median of the same window
recorded beside it. ``confirm`` then re-measures the leaders of four screening rankings
in 3 interleaved 1 s loops. Taking the confirmed energies as the truth for those
configs, this script reports the relative error of each screening estimator:

* counter: the sweep's energy (counter slope x runtime);
* instant: instant-power median x runtime;
* max: the larger of the two (what ``confirm`` also ranks by).

    python scripts/screening_accuracy.py [space ...]   # default: sgemm_clblast pnpoly_space
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import ResultCache  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

SPACES = {"sgemm_clblast": ("sgemm_clblast_report.json", "cache_sgemm_clblast.jsonl",
                            lambda: make_problem("sgemm", value_set="clblast")),
          "pnpoly": ("pnpoly_report.json", "cache_pnpoly.jsonl", lambda: make_problem("pnpoly"))}


def main() -> None:
    names = sys.argv[1:] or list(SPACES)
    out = {}
    for name in names:
        rep_name, cache_name, factory = SPACES[name]
        rep_path = ROOT / "results" / rep_name
        if not rep_path.exists():
            continue
        report = json.loads(rep_path.read_text())
        space = factory().space()
        cache = ResultCache(ROOT / "results" / cache_name)
        rows = []
        for cand in report["confirmed"]["candidates"]:
            r = cache.get(space.config(cand["config"]))
            if r is None or r.failed:
                continue
            inst = r.observer_results.get("nvml_power_instant")
            truth = cand["energy_j"]
            est = {"counter": r.energy, "instant": r.time * inst if inst else float("nan")}
            est["max"] = max(est["counter"], est["instant"])
            rows.append({k: v / truth - 1.0 for k, v in est.items()})
        if not rows:
            continue
        stats = {}
        for k in ("counter", "instant", "max"):
            e = np.array([row[k] for row in rows])
            e = e[np.isfinite(e)]
            stats[k] = {"median_rel_error": float(np.median(e)), "median_abs_rel_error": float(np.median(np.abs(e))),
                        "p90_abs_rel_error": float(np.quantile(np.abs(e), 0.9)), "n": int(e.size)}
        out[name] = {"candidates": len(rows), "vs_confirmed_1s_energy": stats,
                     "confirmed_energy_optimum_rank": report.get("screening", {}).get("confirmed_energy_optimum_rank")}
    print(json.dumps(out, indent=1))
    (ROOT / "results" / "screening_accuracy.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
