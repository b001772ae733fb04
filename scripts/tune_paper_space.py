"""Exhaustive tuning of whole kernel spaces on B200.

The paper benchmarks every config of Kernel Tuner's CLBlast xgemm space
(17,472 configs, ``SgemmProblem(value_set="clblast")``) at
4096^3. This script does the same through the reference API (``benchmark`` +
``NVMLObserver``, energy from the NVML counter), resumable across GPU calls
through a reference-format JSONL cache per space, for:

* ``--space sgemm_clblast``: the paper's 17,472-config GEMM space (default);
* ``--space pnpoly``: the whole brute-force PnPoly space (10,624 configs,
  20 M points x 600 vertices), bit-exact verification against the oracle
  formulation each config computes;
* ``--space sgemm_tf32``: the tcgen05 TF32 space (153 configs).

    python scripts/tune_paper_space.py [--space S] verify       # every config at a small shape vs the oracle
    python scripts/tune_paper_space.py [--space S] sweep --seconds 1800   # measure uncached configs (resumable)
    python scripts/tune_paper_space.py [--space S] confirm      # leaders in 3 x 1 s loops -> tuned_b200.json

Clock control is refused on this pool (profiles/r2_knob_probe.json), so the
(config x clock) product of the paper is config-only here; the space runs at
the driver-managed clock and every result records the observed clock.
Outputs (also mirrored under gpurun_out/ so they come back from the box):
results/cache_<space>.jsonl, results/<space>_verify.json,
results/<space>_report.json.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import NVMLObserver, ResultCache, benchmark  # noqa: E402
from paper_2211_07260_b200.b200 import B200Device  # noqa: E402
from paper_2211_07260_b200.gpu import GPU, fp32_peak_tflops  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

RESULTS = ROOT / "results"
MIRROR = ROOT / "gpurun_out" / "results"

#: space -> (problem factory at full size, factory at the verification size, description)
SPACES = {
    "sgemm_clblast": (lambda: make_problem("sgemm", value_set="clblast"),
                      lambda: make_problem("sgemm", value_set="clblast", m=256, n=256, k=128),
                      "Kernel Tuner CLBlast xgemm, 17,472 configs (PAPER.md:318), 4096^3 FP32, alpha 1 beta 0.5"),
    "pnpoly": (lambda: make_problem("pnpoly"), lambda: make_problem("pnpoly", n_points=100_003),
               "brute-force PnPoly, whole space (10,624 configs), 20 M points x 600 vertices"),
    "sgemm_tf32": (lambda: make_problem("sgemm_tf32"), lambda: make_problem("sgemm_tf32", m=512, n=512, k=256),
                   "tcgen05 TF32 SGEMM, whole space, 4096^3, alpha 1 beta 0.5"),
}


def cache_path(space: str) -> Path:
    return RESULTS / f"cache_{space}.jsonl"


def check_output(problem, cfg, ref) -> tuple[bool, str, float]:
    """(ok, message, error) of the problem's current output against the oracle ``ref``."""
    got = problem.fetch_output()
    if problem.name.startswith("pnpoly"):
        bad = int((got != ref[problem.formula(cfg)]).sum())
        return bad == 0, f"{bad} points differ", float(bad)
    err = O.sgemm_error(got, ref)
    tol = O.SGEMM_TF32_TOL if problem.name == "sgemm_tf32" else O.SGEMM_TOL
    return err <= tol, f"normalised error {err:.3g}", err


def oracle_refs(problem):
    inp = problem.inputs
    if problem.name.startswith("pnpoly"):
        return {f: O.pnpoly(inp["points"], inp["vx"], inp["vy"], f) for f in (0, 1, 2, 3)}
    return O.sgemm(inp["a"], inp["b"], inp["c0"], problem.alpha, problem.beta)


def mirror(*paths: Path) -> None:
    MIRROR.mkdir(parents=True, exist_ok=True)
    for p in paths:
        if p.exists():
            shutil.copy(p, MIRROR / p.name)


def compile_all(problem, configs) -> dict:
    """NVRTC-compile every config on all host cores; returns {key: error} for the ones that fail."""
    errors = {}

    def one(c):
        try:
            problem.cubin({**problem.default_config(), **c.as_dict()})
        except Exception as exc:  # noqa: BLE001 (recorded; the benchmark records the failure too)
            errors[c.key()] = str(exc)[:200]

    with ThreadPoolExecutor(os.cpu_count() or 8) as pool:
        list(pool.map(one, configs))
    return errors


def cmd_verify(args) -> None:
    """Every config of the space, once, at a small shape, against the oracle."""
    problem = SPACES[args.space][1]()
    configs = problem.space().enumerate()
    t0 = time.time()
    errors = compile_all(problem, configs)
    compile_s = time.time() - t0
    worst, failed = 0.0, []
    with GPU(0) as gpu:
        problem.prepare(gpu)
        ref = oracle_refs(problem)
        for c in configs:
            cfg = {**problem.default_config(), **c.as_dict()}
            try:
                k = problem.kernel(cfg)
                problem.bind(k, cfg)  # __constant__ polygon (PnPoly poly_smem 0, ASM 8)
                problem.reset_output()
                gpu.launch(k, problem.launch(cfg), problem.args(cfg))
                gpu.synchronize()
                ok, msg, err = check_output(problem, cfg, ref)
            except Exception as exc:  # noqa: BLE001
                failed.append({"config": c.as_dict(), "error": str(exc)[:200]})
                continue
            worst = max(worst, err)
            if not ok:
                failed.append({"config": c.as_dict(), "error": msg})
    pn = problem.name.startswith("pnpoly")
    doc = {"space": SPACES[args.space][2], "configs": len(configs),
           "shape": [problem.n_points, problem.n_vertices] if pn else [problem.m, problem.n, problem.k],
           "compile_errors": len(errors), "failed": failed,
           ("worst_points_differing" if pn else "worst_normalised_error"): worst,
           "bar": "bit-exact vs the oracle formulation each config computes" if pn else
           (O.SGEMM_TF32_TOL if problem.name == "sgemm_tf32" else O.SGEMM_TOL),
           "compile_s": round(compile_s, 1), "run_s": round(time.time() - t0 - compile_s, 1)}
    out = RESULTS / f"{args.space}_verify.json"
    out.write_text(json.dumps(doc, indent=1) + "\n")
    mirror(out)
    print(json.dumps({k: v for k, v in doc.items() if k != "failed"}), "failed:", len(failed), flush=True)


def cmd_sweep(args) -> None:
    problem = SPACES[args.space][0]()
    configs = problem.space().enumerate()
    CACHE = cache_path(args.space)
    cache = ResultCache(CACHE)
    todo = [c for c in configs if c not in cache]
    print(f"{len(configs)} configs, {len(configs) - len(todo)} cached, {len(todo)} to measure", flush=True)
    deadline = time.time() + args.seconds
    # compile only what this call can plausibly measure (~0.3 s per point)
    batch = todo[: max(1, int(args.seconds / 0.25))]
    t0 = time.time()
    errors = compile_all(problem, batch)
    print(f"compiled {len(batch)} in {time.time() - t0:.0f} s ({len(errors)} errors)", flush=True)
    metrics, consts = problem.user_metrics()
    done = 0
    with GPU(0) as gpu:
        dev = B200Device(problem, gpu=gpu, min_window=args.window, settle=args.settle)
        obs = [NVMLObserver(args.window)]
        t1 = time.time()
        for c in batch:
            if time.time() > deadline:
                break
            cache.put(benchmark(dev, c, obs, user_metrics=metrics, constants=consts))
            done += 1
            if done % 500 == 0:
                print(f"{done} measured, {(time.time() - t1) / done * 1e3:.0f} ms per point", flush=True)
                mirror(CACHE)
        dev.close()
    mirror(CACHE)
    print(f"measured {done} points in {time.time() - t1:.0f} s; cache now {len(cache)} of {len(configs)}", flush=True)


def cmd_confirm(args) -> None:
    sys.path.insert(0, str(ROOT / "scripts"))
    from tune_suite import RANKINGS, TUNED_PATH, confirm, oracle_check, screening_leaders  # noqa: E402

    problem = SPACES[args.space][0]()
    space = problem.space()
    configs = space.enumerate()
    cache = ResultCache(cache_path(args.space))
    results = [cache.get(c) for c in configs]
    have = [r for r in results if r is not None]
    ok = [r for r in have if not r.failed]
    rankings = RANKINGS
    leaders = screening_leaders(ok, args.top)
    with GPU(0) as gpu:
        dev = B200Device(problem, gpu=gpu, min_window=args.window)
        confirmed = confirm(dev, problem, leaders)
        by_time = min(confirmed, key=lambda r: r["time_s"])
        by_energy = min(confirmed, key=lambda r: r["energy_j"])
        for rec in (by_time, by_energy):
            cfg = {**problem.default_config(), **rec["config"]}
            k = problem.kernel(cfg)
            problem.bind(k, cfg)
            problem.reset_output()
            gpu.launch(k, problem.launch(cfg), problem.args(cfg))
            gpu.synchronize()
            rec["oracle_ok"], rec["oracle_metric"] = oracle_check(problem, cfg)
        sm = gpu.sm_count
        dev.close()
    # distribution over the whole space (the paper's Fig. 3 view): GFLOP/s vs GFLOPS/W
    gf = np.array([r.metrics["gflops"] for r in ok])
    gw = np.array([r.metrics["gflops_per_w"] for r in ok])
    tmin = min(r.time for r in ok)
    emin = min(r.energy for r in ok)
    best_t = min(ok, key=lambda r: r.time)
    best_e = min(ok, key=lambda r: r.energy)
    report = {
        "space": SPACES[args.space][2],
        "measured": len(have), "failed": len(have) - len(ok), "space_size": len(configs),
        "window_s": args.window, "observer": "NVMLObserver (energy-counter slope x per-launch runtime)",
        "clock": "driver-managed (clock control refused: profiles/r2_knob_probe.json); observed clock per result",
        "gflops": {"max": float(gf.max()), "median": float(np.median(gf)), "min": float(gf.min())},
        "gflops_per_w": {"max": float(gw.max()), "median": float(np.median(gw)), "min": float(gw.min())},
        "sweep_time_optimal": {"config": best_t.config.as_dict(), "gflops": best_t.metrics["gflops"],
                               "gflops_per_w": best_t.metrics["gflops_per_w"]},
        "sweep_energy_optimal": {"config": best_e.config.as_dict(), "gflops": best_e.metrics["gflops"],
                                 "gflops_per_w": best_e.metrics["gflops_per_w"]},
        "energy_optimal_vs_time_optimal_in_sweep": {
            "energy_saving": 1.0 - emin / best_t.energy, "slowdown": best_e.time / tmin - 1.0},
        "within_5pct_of_best_time": int(sum(r.time <= 1.05 * tmin for r in ok)),
        "within_5pct_of_best_energy": int(sum(r.energy <= 1.05 * emin for r in ok)),
        "fp32_peak_tflops_at_1965": fp32_peak_tflops(sm, 1965.0),
        "confirmed": {"time_optimal": by_time, "energy_optimal": by_energy, "candidates": confirmed},
    }
    # screening noise: counter / instant power in the same window, and where the confirmed
    # optimum ranked under each screening estimator
    ratio = np.array([r.observer_results["nvml_power"] / r.observer_results["nvml_power_instant"] for r in ok
                      if r.observer_results.get("nvml_power_instant") and r.observer_results.get("nvml_power")])
    report["screening"] = {
        "counter_over_instant_power_quantiles": {str(q): float(np.quantile(ratio, q)) for q in
                                                 (0.01, 0.05, 0.25, 0.5, 0.75, 0.95, 0.99)} if ratio.size else None,
        "confirmed_energy_optimum_rank": {
            name: 1 + [r.config.key() for r in sorted(ok, key=key)].index(space.config(by_energy["config"]).key())
            for name, key in rankings.items()},
        "candidates_per_ranking": args.top,
    }
    out = RESULTS / f"{args.space}_report.json"
    out.write_text(json.dumps(report, indent=1) + "\n")
    data = json.loads(TUNED_PATH.read_text()) if TUNED_PATH.exists() else {}
    data[args.space if args.space != "pnpoly" else "pnpoly_space"] = {"space_size": len(configs), "strategy": "exhaustive", "evaluations": len(have),
                             "failed": len(have) - len(ok), "time_optimal": by_time, "energy_optimal": by_energy,
                             "confirm": {"rounds": 3, "window_s": 1.0, "candidates": confirmed}}
    TUNED_PATH.write_text(json.dumps(data, indent=1) + "\n")
    shutil.copy(TUNED_PATH, ROOT / "gpurun_out" / "tuned_b200.json")
    mirror(out)
    print(json.dumps({k: report[k] for k in ("measured", "failed", "gflops", "gflops_per_w")}), flush=True)
    print("time-opt  ", by_time, "\nenergy-opt", by_energy, flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--space", choices=sorted(SPACES), default="sgemm_clblast")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("verify")
    s = sub.add_parser("sweep")
    s.add_argument("--seconds", type=float, default=1800.0)
    # 0.3 s loops hold two whole 100 ms energy-counter periods after the settle (b200.counter_power)
    s.add_argument("--window", type=float, default=0.3)
    s.add_argument("--settle", type=float, default=0.02)
    c = sub.add_parser("confirm")
    c.add_argument("--top", type=int, default=8)
    c.add_argument("--window", type=float, default=0.2)
    args = ap.parse_args()
    {"verify": cmd_verify, "sweep": cmd_sweep, "confirm": cmd_confirm}[args.cmd](args)


if __name__ == "__main__":
    main()
