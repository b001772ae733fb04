"""How well do 0.3 s sweep windows rank configs by energy? (CPU, over committed B200 results)

Every exhaustive sweep (scripts/tune_paper_space.py) measures each config once in a
0.3 s loop: energy = the NVML energy-counter slope over its two updates inside the
steady window x per-launch runtime, with the instant-power median of the same window
recorded beside it. ``confirm`` then re-measures the leaders of four screening rankings
in 3 interleaved 1 s loops. Taking the confirmed energies as the truth for those
configs, this script reports the relative error of each screening estimator:

* counter: the sweep's energy (counter power x runtime: a two-change slope before the round-2
  fixes, whole counter periods after them);
* instant: instant-power median x runtime;
* max: the larger of the two (what ``confirm`` also ranks by).

    python scripts/screening_accuracy.py [space ...]   # default: every space below
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
          "pnpoly": ("pnpoly_report.json", "cache_pnpoly.jsonl", lambda: make_problem("pnpoly")),
          # tune_suite sweeps: their confirmed candidates live in tuned_b200.json
          "conv2d": ("tuned:conv2d", "cache_conv2d.jsonl", lambda: make_problem("conv2d")),
          "sgemm_tf32": ("tuned:sgemm_tf32", "cache_sgemm_tf32.jsonl", lambda: make_problem("sgemm_tf32"))}
TUNED = ROOT / "paper_2211_07260_b200" / "tuned_b200.json"


def main() -> None:
    names = sys.argv[1:] or list(SPACES)
    out = {}
    for name in names:
        rep_name, cache_name, factory = SPACES[name]
        if rep_name.startswith("tuned:"):
            entry = json.loads(TUNED.read_text()).get(rep_name[6:])
            if not entry or not (ROOT / "results" / cache_name).exists():
                continue
            report = {"confirmed": {"candidates": entry["confirm"]["candidates"]},
                      "energy_optimal_config": entry["energy_optimal"]["config"]}
        else:
            rep_path = ROOT / "results" / rep_name
            if not rep_path.exists():
                continue
            report = json.loads(rep_path.read_text())
        space = factory().space()
        cache = ResultCache(ROOT / "results" / cache_name)
        rows = []
        for cand in report["confirmed"]["candidates"]:
            try:
                r = cache.get(space.config({k: v for k, v in cand["config"].items() if not k.startswith("nvml_")}))
            except Exception:  # noqa: BLE001 (a candidate outside this cache's space)
                continue
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
        rank = report.get("screening", {}).get("confirmed_energy_optimum_rank")
        if rank is None and report.get("energy_optimal_config"):
            sys.path.insert(0, str(ROOT / "scripts"))
            from tune_suite import RANKINGS  # noqa: E402

            ok = [r for r in cache.results() if not r.failed]
            best = space.config({k: v for k, v in report["energy_optimal_config"].items()
                                 if not k.startswith("nvml_")}).key()
            rank = {n: 1 + [r.config.key() for r in sorted(ok, key=key)].index(best) for n, key in RANKINGS.items()}
        out[name] = {"candidates": len(rows), "vs_confirmed_1s_energy": stats, "confirmed_energy_optimum_rank": rank}
    print(json.dumps(out, indent=1))
    (ROOT / "results" / "screening_accuracy.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
