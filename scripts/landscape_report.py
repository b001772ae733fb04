"""Fig. 3-style speed-vs-efficiency report over the B200 tuning caches.

For every reference-format cache in results/ this runs the package's own
``analyze`` CLI (reference ``cli.py:367-443``, ``analysis.py:50-240``):

* ``--mode pareto``: the performance / efficiency front (GFLOP/s vs GFLOPS/W
  for flop-counted kernels; points/s vs points/J for the work-skipping PnPoly
  kernels, which are not credited with brute-force flops);
* ``--mode difficulty``: the fitness-flow graph of the energy objective and its
  proportion-of-centrality curve, when the cache covers its whole space;

then writes one SVG scatter per kernel (every config, the front, the time- and
energy-optimal configs; the paper's Fig. 3 view) and results/landscape/REPORT.md.
CPU only: it reads caches measured on the B200 (scripts/tune_suite.py,
scripts/tune_paper_space.py).

    python scripts/landscape_report.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import ResultCache, SearchSpace, commands  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

RESULTS = ROOT / "results"
OUT = RESULTS / "landscape"

#: cache -> (problem name, problem kwargs, performance metric, efficiency metric, units)
CACHES = {
    "conv2d": ("conv2d", {}, "gflops", "gflops_per_w", ("GFLOP/s", "GFLOPS/W")),
    "sgemm": ("sgemm", {}, "gflops", "gflops_per_w", ("GFLOP/s", "GFLOPS/W")),
    "sgemm_wide": ("sgemm", {"value_set": "b200"}, "gflops", "gflops_per_w", ("GFLOP/s", "GFLOPS/W")),
    "sgemm_clblast": ("sgemm", {"value_set": "clblast"}, "gflops", "gflops_per_w", ("GFLOP/s", "GFLOPS/W")),
    "sgemm_tf32": ("sgemm_tf32", {}, "gflops", "gflops_per_w", ("GFLOP/s", "GFLOPS/W")),
    "pnpoly": ("pnpoly", {}, "gflops", "gflops_per_w", ("GFLOP/s (3 ops/edge)", "GFLOPS/W")),
    "pnpoly_slab": ("pnpoly_slab", {}, "points_per_s", "points_per_j", ("points/s", "points/J")),
    "pnpoly_grid": ("pnpoly_grid", {}, "points_per_s", "points_per_j", ("points/s", "points/J")),
    "pnpoly_cells": ("pnpoly_cells", {}, "points_per_s", "points_per_j", ("points/s", "points/J")),
}


def cache_space(results) -> dict:
    """The space document the cache enumerates: every parameter it sets, the values it saw."""
    values: dict[str, set] = {}
    for r in results:
        for k, v in r.config.as_dict().items():
            values.setdefault(k, set()).add(v)
    return {"parameters": {k: sorted(v) for k, v in values.items()}, "restrictions": []}


def difficulty_space(problem, results) -> dict | None:
    """A space whose every valid config the cache holds: the problem's own, else the cache's
    value lists under the problem's restrictions (None if neither is covered)."""
    have = {r.config for r in results}
    for doc in (problem.space_document(), {**cache_space(results), "restrictions": problem.restrictions()}):
        names = set(doc["parameters"])
        if any(set(r.config.as_dict()) != names for r in results[:1]):
            continue
        try:
            configs = SearchSpace.from_dict(doc).enumerate()
        except Exception:  # noqa: BLE001 (a restriction naming a parameter this cache does not set)
            continue
        if configs and all(c in have for c in configs):
            return doc
    return None


def screening_quality(results) -> dict:
    """Which energy estimator a cache was measured with, read off its observer keys, and how far
    its counter power strays from the instant-power median of the same window (1st-99th pct)."""
    keys = set().union(*(r.observer_results.keys() for r in results))
    if "nvml_power_disagree" in keys:
        estimator = "counter periods, re-runs"
    elif "nvml_stale_retries" in keys or "nvml_counter_updates" in keys:
        estimator = "counter (2-3 changes)"
    else:
        estimator = "counter slope (r1)"
    ratio = sorted(r.observer_results["nvml_power"] / r.observer_results["nvml_power_instant"] for r in results
                   if r.observer_results.get("nvml_power") and r.observer_results.get("nvml_power_instant"))
    q = (lambda f: ratio[int(f * (len(ratio) - 1))]) if ratio else None
    return {"estimator": estimator, "ratio": f"{q(0.01):.2f}-{q(0.99):.2f}" if q else "-"}


def svg_scatter(points, front, t_opt, e_opt, units, title, path: Path) -> None:
    """Performance (x) vs efficiency (y): all configs grey, the Pareto front blue, optima marked."""
    w, h, m = 640, 440, 60
    xs = [p[0] for p in points]
    ys = [p[1] for p in points]
    x0, x1 = min(xs), max(xs)
    y0, y1 = min(ys), max(ys)
    sx = lambda x: m + (x - x0) / ((x1 - x0) or 1) * (w - 2 * m)  # noqa: E731
    sy = lambda y: h - m - (y - y0) / ((y1 - y0) or 1) * (h - 2 * m)  # noqa: E731
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{w}" height="{h}" font-family="sans-serif" font-size="12">',
           f'<rect width="{w}" height="{h}" fill="white"/>',
           f'<text x="{w / 2}" y="20" text-anchor="middle" font-size="14">{title}</text>',
           f'<line x1="{m}" y1="{h - m}" x2="{w - m}" y2="{h - m}" stroke="black"/>',
           f'<line x1="{m}" y1="{m}" x2="{m}" y2="{h - m}" stroke="black"/>',
           f'<text x="{w / 2}" y="{h - 15}" text-anchor="middle">{units[0]}</text>',
           f'<text x="15" y="{h / 2}" transform="rotate(-90 15 {h / 2})" text-anchor="middle">{units[1]}</text>']
    for frac in (0.0, 0.5, 1.0):
        xv, yv = x0 + frac * (x1 - x0), y0 + frac * (y1 - y0)
        out.append(f'<text x="{sx(xv)}" y="{h - m + 15}" text-anchor="middle">{xv:.4g}</text>')
        out.append(f'<text x="{m - 5}" y="{sy(yv) + 4}" text-anchor="end">{yv:.4g}</text>')
    for x, y in points:
        out.append(f'<circle cx="{sx(x):.1f}" cy="{sy(y):.1f}" r="2" fill="#999" fill-opacity="0.5"/>')
    fr = sorted(front)
    out.append('<polyline fill="none" stroke="#1f5fbf" stroke-width="1.5" points="'
               + " ".join(f"{sx(x):.1f},{sy(y):.1f}" for x, y in fr) + '"/>')
    for x, y in fr:
        out.append(f'<circle cx="{sx(x):.1f}" cy="{sy(y):.1f}" r="3" fill="#1f5fbf"/>')
    for (x, y), label, color in ((t_opt, "time-optimal", "#d62728"), (e_opt, "energy-optimal", "#2ca02c")):
        out.append(f'<circle cx="{sx(x):.1f}" cy="{sy(y):.1f}" r="6" fill="none" stroke="{color}" stroke-width="2"/>')
        out.append(f'<text x="{sx(x) - 8:.1f}" y="{sy(y) - 9:.1f}" text-anchor="end" fill="{color}">{label}</text>')
    out.append("</svg>")
    path.write_text("\n".join(out) + "\n")


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    rows = []
    for name, (pname, kwargs, perf, eff, units) in CACHES.items():
        cache_path = RESULTS / f"cache_{name}.jsonl"
        if not cache_path.exists():
            continue
        results = [r for r in ResultCache(cache_path).results() if not r.failed]
        if not results:
            continue
        d = OUT / name
        d.mkdir(exist_ok=True)
        commands.main(["analyze", "--mode", "pareto", "--cache", str(cache_path), "--performance", perf,
                       "--efficiency", eff, "--out", str(d)])
        front_doc = json.loads((d / "analyze.json").read_text())
        (d / "analyze.json").rename(d / "pareto.json")
        problem = make_problem(pname, **kwargs)
        space_doc = difficulty_space(problem, results)
        diff = None
        if space_doc is not None:
            (d / "space.json").write_text(json.dumps(space_doc, indent=1) + "\n")
            commands.main(["analyze", "--mode", "difficulty", "--cache", str(cache_path), "--space",
                           str(d / "space.json"), "--objective", "energy", "--out", str(d)])
            diff = json.loads((d / "analyze.json").read_text())
            (d / "analyze.json").rename(d / "difficulty.json")
        t_best = min(results, key=lambda r: r.time)
        e_best = min(results, key=lambda r: r.energy)
        pts = [(r.lookup(perf), r.lookup(eff)) for r in results]
        front = [(p["performance"], p["efficiency"]) for p in front_doc["front"]]
        svg_scatter(pts, front, (t_best.lookup(perf), t_best.lookup(eff)), (e_best.lookup(perf), e_best.lookup(eff)),
                    units, f"{name}: {len(results)} configs on B200 (speed vs efficiency)", d / "speed_vs_efficiency.svg")
        rows.append({
            "kernel": name, "configs": len(results), "front": len(front), "units": units,
            "time_opt": (t_best.lookup(perf), t_best.lookup(eff)), "energy_opt": (e_best.lookup(perf), e_best.lookup(eff)),
            "energy_saving": 1.0 - e_best.energy / t_best.energy, "slowdown": e_best.time / t_best.time - 1.0,
            "eff_spread": max(p[1] for p in pts) / min(p[1] for p in pts),
            "minima": None if diff is None else diff["minima"],
            "f_optimal": None if diff is None else diff["f_optimal"],
            **screening_quality(results),
        })
    lines = ["# Speed vs efficiency over the B200 tuning caches (Fig. 3 view)", "",
             "Generated by `scripts/landscape_report.py` from `results/cache_*.jsonl` (sweep-window values: "
             "0.2-0.4 s loops; confirmed optima are in `tuned_b200.json`). The `estimator` column says how "
             "each cache's energies were taken, and `counter/instant` how far its counter power strays from "
             "the instant-power median of the same window (1st-99th percentile): caches taken before the "
             "round-2 measurement fixes (DESIGN.md §5, `results/screening_accuracy.json`) hold a few "
             "energies off by tens of percent, so their screening energy optima and efficiency spreads "
             "are noise-inflated; the confirmed table at the end is the measurement of record. "
             "Each kernel's directory holds `pareto.csv` / `pareto.json` (the package's `analyze --mode pareto`), "
             "`difficulty.csv` / `difficulty.json` (`analyze --mode difficulty`, energy objective, when the cache "
             "covers its whole space) and `speed_vs_efficiency.svg`.", "",
             "| kernel | configs | estimator | counter/instant | front | time-optimal (perf, eff) | energy-optimal "
             "(perf, eff) | energy saved by the energy optimum | its slowdown | eff. spread max/min | local optima "
             "(FFG) | f_optimal |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        u = r["units"]
        fo = "-" if r["f_optimal"] is None else f"{r['f_optimal']:.3f}"
        minima = "-" if r["minima"] is None else r["minima"]
        lines.append(
            f"| {r['kernel']} | {r['configs']} | {r['estimator']} | {r['ratio']} | {r['front']} | "
            f"{r['time_opt'][0]:.4g} {u[0]}, {r['time_opt'][1]:.4g} "
            f"{u[1]} | {r['energy_opt'][0]:.4g}, {r['energy_opt'][1]:.4g} | {100 * r['energy_saving']:.1f}% | "
            f"{100 * r['slowdown']:.1f}% | {r['eff_spread']:.1f}x | {minima} | {fo} |")
    # the optima confirmed in 3 x 1 s interleaved loops are the ones to quote
    tuned = json.loads((ROOT / "paper_2211_07260_b200" / "tuned_b200.json").read_text())
    lines += ["", "Confirmed optima (`tuned_b200.json`: the sweep's energy and time leaders re-measured in 3 "
              "interleaved 1 s loops, energy from 0.25 s in; what bench.py's per_kernel reports):", "",
              "| kernel | time-optimal: ms, perf, eff | energy-optimal: ms, perf, eff | energy saved | slowdown |",
              "|---|---|---|---|---|"]
    for name, entry in tuned.items():
        t, e = entry.get("time_optimal"), entry.get("energy_optimal")
        if not t or not e or name.endswith("_sweep"):
            continue
        key = ("points_per_s", "j_per_bitmap") if "points_per_s" in t else ("gflops", "gflops_per_w")
        fmt = lambda r: f"{r['time_s'] * 1e3:.4g}, {r[key[0]]:.4g}, {r[key[1]]:.4g}"  # noqa: E731
        lines.append(f"| {name} ({key[0]}, {key[1]}) | {fmt(t)} | {fmt(e)} | "
                     f"{100 * (1 - e['energy_j'] / t['energy_j']):.1f}% | {100 * (e['time_s'] / t['time_s'] - 1):.1f}% |")
    (OUT / "REPORT.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
