"""Generate tests/golden/reference_golden.json from the reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``jouletune`` read-only from /root/reference/pkg/src
and records, on its own simulated devices and fixtures, the outputs the drop-in
API must reproduce: enumeration keys, tuning histories for the three
strategies and five pipelines, sensor readings, power-model fits, optimal
clocks and bands, and the CLI workflow of pkg/README.md. The device spec and
space fixtures used are embedded so the tests never read /root/reference.
"""

from __future__ import annotations

import json
import sys
import tempfile
import warnings
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "reference_golden.json"


def main():
    sys.path.insert(0, str(REF))
    import jouletune as J
    from jouletune import powermodel as PM
    from jouletune import presets
    from jouletune.cli import main as cli_main

    gold: dict = {"reference": "jouletune " + J.__version__}
    specs = {n: json.loads(presets.spec_path(n).read_text()) for n in presets.DEVICE_NAMES}
    gold["specs"] = specs
    gold["spaces"] = {
        "gemm_space": json.loads(presets.fixture_path("gemm_space.json").read_text()),
        "a100_mimic_space": json.loads(presets.fixture_path("a100_mimic_space.json").read_text()),
    }

    # -- search spaces ---------------------------------------------------------
    sp = {}
    for name, doc in gold["spaces"].items():
        space = J.SearchSpace.from_dict(doc)
        cfgs = space.enumerate()
        sp[name] = {
            "size": len(cfgs),
            "keys": [c.key() for c in cfgs],
            "first_neighbors": [c.key() for c in space.neighbors(cfgs[0])],
            "mid_neighbors": [c.key() for c in space.neighbors(cfgs[len(cfgs) // 2])],
        }
    gold["searchspace"] = sp

    # -- strategies on the mimic fixture -----------------------------------------
    runs = {}
    for strategy, budget, seed in (("exhaustive", None, 0), ("random", 150, 7), ("local_search", 200, 7),
                                   ("local_search", 60, 3)):
        space, dev = presets.a100_mimic()
        out = J.run_strategy(J.TuningRun(space, strategy, J.Objective("energy"), budget=budget, seed=seed), dev,
                             [J.InstantPowerObserver()],
                             user_metrics=J.default_metrics(presets.GEMM_TOTAL_FLOPS),
                             constants={"total_flops": presets.GEMM_TOTAL_FLOPS})
        runs[f"{strategy}:{budget}:{seed}"] = {
            "history": [[r.config.key(), r.time, r.energy, r.metrics.get("gflops_per_w")] for r in out.history],
            "best": [out.best.config.key(), out.best.energy],
            "minima": [c.key() for c in out.minima_reached],
            "device_executions": out.device_executions,
        }
    # averaged observer on a noisy device (RNG stream parity)
    dev = presets.device("a100_like", seed=3)
    space = J.SearchSpace.from_dict({"parameters": {"x": [1, 2, 3],
                                                    "nvml_gr_clock": list(dev.spec.supported_core_clocks[::16])}})
    out = J.run_strategy(J.TuningRun(space, "exhaustive", J.Objective("time")), dev, [J.AveragedPowerObserver()])
    runs["averaged:a100_like:3"] = {
        "history": [[r.config.key(), r.time, r.energy, r.observer_results.get("nvml_power")] for r in out.history],
        "best": [out.best.config.key(), out.best.energy],
    }
    gold["strategies"] = runs

    pipes = {}
    space, _ = presets.a100_mimic()
    for name in J.PIPELINES:
        rep = J.run_pipeline(name, space, presets.device("a100_mimic"), [J.InstantPowerObserver()])
        pipes[name] = rep.to_dict()
    gold["pipelines"] = pipes

    # -- sensors ----------------------------------------------------------------
    ramp = [J.PowerSample(float(t), 20.0 + 50.0 * float(t)) for t in np.linspace(0.0, 1.0, 101)]
    cfg = J.AveragedSensorConfig(refresh_rate=10.0, continuous_duration=1.0)
    gold["sensors"] = {
        "ramp_readings": {str(t): J.averaged_reading(ramp, t, cfg) for t in (0.1, 0.201, 0.25, 0.31, 0.99, 1.0)},
        "instant_energy": J.instant_energy([J.PowerSample(0.5, 100.0), J.PowerSample(1.0, 110.0),
                                            J.PowerSample(1.5, 120.0)], 0.0, 2.0),
    }

    # -- power model ------------------------------------------------------------
    fits = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for name in ("a100_like", "a4000_like", "a6000_like", "v100_like", "titan_rtx_like", "a100_mimic"):
            dev = presets.device(name, seed=11)
            for voltage in (True, False):
                samples = []
                for f in dev.spec.supported_core_clocks[::3]:
                    p = dev.ground_truth.power(f) * (1.0 + 0.01 * np.sin(f))
                    v = dev.ground_truth.voltage(f) if voltage else None
                    samples.append(PM.FrequencySample(float(f), float(p), v))
                key = f"{name}:{'v' if voltage else 'nov'}"
                try:
                    m = PM.fit(samples, tdp=dev.spec.tdp)
                    f_opt = PM.optimal_frequency(m, dev.spec.supported_core_clocks)
                    band = PM.frequency_band(f_opt, dev.spec.supported_core_clocks)
                    fits[key] = {"samples": [[s.frequency, s.power, s.voltage] for s in samples],
                                 "tdp": dev.spec.tdp, "model": m.to_dict(), "f_opt": f_opt,
                                 "band": list(band.clocks), "reduction": band.reduction}
                except Exception as exc:  # noqa: BLE001
                    fits[key] = {"samples": [[s.frequency, s.power, s.voltage] for s in samples],
                                 "tdp": dev.spec.tdp, "error": type(exc).__name__}
    # noisy 4-parameter fits (numeric path exercised hardest)
    truth = J.GroundTruth(p_idle=55.0, p_max=250.0, alpha=0.135, tau_ft=1015.0, beta=0.00108, v0=0.7)
    for seed in range(5):
        rng = np.random.default_rng(seed)
        samples = [PM.FrequencySample(float(f), float(truth.power(f) * (1 + rng.normal(0, 0.01))), None)
                   for f in np.linspace(210.0, 1410.0, 25)]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            m = PM.fit(samples, tdp=250.0)
        fits[f"noisy:{seed}"] = {"samples": [[s.frequency, s.power, None] for s in samples], "tdp": 250.0,
                                 "model": m.to_dict()}
    gold["fits"] = fits

    # -- CLI workflow (pkg/README.md) ----------------------------------------------
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        spec = str(presets.spec_path("a100_mimic"))
        space_path = str(presets.fixture_path("a100_mimic_space.json"))
        rc = [cli_main(["simulate-sweep", "--device", spec, "--out", str(tmp / "sweep.csv"), "--points", "25"])]
        rc.append(cli_main(["fit", "--samples", str(tmp / "sweep.csv"), "--device", spec, "--out",
                            str(tmp / "model.json")]))
        rc.append(cli_main(["steer", "--space", space_path, "--device", spec, "--model", str(tmp / "model.json"),
                            "--out", str(tmp / "steer"), "--observer", "instant", "--total-flops", "1.374e11"]))
        gold["cli"] = {
            "rc": rc,
            "sweep_csv": (tmp / "sweep.csv").read_text(),
            "model": json.loads((tmp / "model.json").read_text()),
            "steer_report": json.loads((tmp / "steer" / "report.json").read_text()),
        }
        # analyze over the steer run's cache: Pareto front and both difficulty weightings
        band = gold["cli"]["steer_report"]["steering"]["band"]
        steered = J.SearchSpace.from_dict(gold["spaces"]["a100_mimic_space"]).with_values("nvml_gr_clock", band)
        (tmp / "steered.json").write_text(json.dumps(steered.to_dict()))
        cache = str(tmp / "steer" / "cache.jsonl")
        analyze = {}
        for label, extra in (("pareto", ["--mode", "pareto"]),
                             ("absorbing", ["--mode", "difficulty", "--space", str(tmp / "steered.json")]),
                             ("pagerank", ["--mode", "difficulty", "--space", str(tmp / "steered.json"),
                                           "--weights", "pagerank", "--p-max", "2.0", "--p-steps", "11"]),
                             ("time", ["--mode", "difficulty", "--space", str(tmp / "steered.json"),
                                       "--objective", "time"])):
            out = tmp / f"analyze_{label}"
            rc = cli_main(["analyze", "--cache", cache, "--out", str(out), *extra])
            doc = json.loads((out / "analyze.json").read_text())
            csv_name = "pareto.csv" if label == "pareto" else "difficulty.csv"
            analyze[label] = {"rc": rc, "report": {k: v for k, v in doc.items() if not k.startswith("manifest")},
                              "manifest_keys": sorted(doc["manifest"]), "csv": (out / csv_name).read_text()}
        gold["analyze"] = analyze
    OUT.write_text(json.dumps(gold, indent=None, separators=(",", ":")) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
