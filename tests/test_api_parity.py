"""The drop-in API reproduces the reference on its own golden vectors.

Golden data: tests/golden/reference_golden.json, generated from the live
reference (``jouletune``) by tests/golden/make_golden.py. Tolerances: exact
for keys, orders and simulated energies (same RNG stream); 1e-9 relative for
power-model fits (LM arithmetic is restated, not copied).
"""

import json
import math
import warnings

import numpy as np
import pytest

import paper_2211_07260_b200 as B
from paper_2211_07260_b200 import powermodel as PM
from paper_2211_07260_b200.cli import main as cli_main


def _close(a, b, rel=1e-9):
    if a is None or b is None:
        return a is b
    return math.isclose(a, b, rel_tol=rel, abs_tol=1e-12)


def test_enumeration_keys_and_neighbors(golden):
    for name, doc in golden["spaces"].items():
        space = B.SearchSpace.from_dict(doc)
        want = golden["searchspace"][name]
        cfgs = space.enumerate()
        assert space.size() == want["size"]
        assert [c.key() for c in cfgs] == want["keys"]
        assert [c.key() for c in space.neighbors(cfgs[0])] == want["first_neighbors"]
        assert [c.key() for c in space.neighbors(cfgs[len(cfgs) // 2])] == want["mid_neighbors"]
    assert golden["searchspace"]["gemm_space"]["size"] == 1328  # tests/test_searchspace.py:128-134


@pytest.mark.parametrize("run_key", ["exhaustive:None:0", "random:150:7", "local_search:200:7", "local_search:60:3"])
def test_strategies_reproduce_reference_histories(golden, spec_file, run_key):
    strategy, budget, seed = run_key.split(":")
    budget = None if budget == "None" else int(budget)
    space = B.SearchSpace.from_dict(golden["spaces"]["a100_mimic_space"])
    dev = B.load_device(spec_file("a100_mimic"))
    flops = 2.0 * 4096.0**3
    out = B.run_strategy(B.TuningRun(space, strategy, B.Objective("energy"), budget=budget, seed=int(seed)), dev,
                         [B.InstantPowerObserver()], user_metrics=B.default_metrics(flops),
                         constants={"total_flops": flops})
    want = golden["strategies"][run_key]
    got = [[r.config.key(), r.time, r.energy, r.metrics.get("gflops_per_w")] for r in out.history]
    assert got == want["history"]
    assert [out.best.config.key(), out.best.energy] == want["best"]
    assert [c.key() for c in out.minima_reached] == want["minima"]
    assert out.device_executions == want["device_executions"]


def test_averaged_observer_rng_stream_parity(golden, spec_file):
    dev = B.load_device(spec_file("a100_like"), seed=3)
    space = B.SearchSpace.from_dict(
        {"parameters": {"x": [1, 2, 3], "nvml_gr_clock": list(dev.spec.supported_core_clocks[::16])}})
    out = B.run_strategy(B.TuningRun(space, "exhaustive", B.Objective("time")), dev, [B.AveragedPowerObserver()])
    want = golden["strategies"]["averaged:a100_like:3"]
    got = [[r.config.key(), r.time, r.energy, r.observer_results.get("nvml_power")] for r in out.history]
    assert got == want["history"]


@pytest.mark.parametrize("name", B.PIPELINES)
def test_pipelines_match_reference(golden, spec_file, name):
    space = B.SearchSpace.from_dict(golden["spaces"]["a100_mimic_space"])
    rep = B.run_pipeline(name, space, B.load_device(spec_file("a100_mimic")), [B.InstantPowerObserver()])
    assert json.loads(json.dumps(rep.to_dict())) == golden["pipelines"][name]


def test_global_pipeline_beats_staged(golden):
    # tests/test_acceptance.py:170-180 on the golden pipeline results
    e = {k: v["best"]["energy"] for k, v in golden["pipelines"].items()}
    assert all(e["global"] <= e[k] for k in e)
    assert e["global"] == pytest.approx(0.0566676, rel=1e-6)  # pkg/README.md:81-83


def test_sensor_readings(golden):
    ramp = [B.PowerSample(float(t), 20.0 + 50.0 * float(t)) for t in np.linspace(0.0, 1.0, 101)]
    cfg = B.AveragedSensorConfig(refresh_rate=10.0, continuous_duration=1.0)
    for t, want in golden["sensors"]["ramp_readings"].items():
        assert B.averaged_reading(ramp, float(t), cfg) == want
    pts = [B.PowerSample(0.5, 100.0), B.PowerSample(1.0, 110.0), B.PowerSample(1.5, 120.0)]
    assert B.instant_energy(pts, 0.0, 2.0) == golden["sensors"]["instant_energy"] == 220.0


def test_power_model_fits_match_reference(golden):
    for key, case in golden["fits"].items():
        samples = [PM.FrequencySample(f, p, v) for f, p, v in case["samples"]]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            if "error" in case:
                with pytest.raises(B.JouleTuneError):
                    PM.fit(samples, tdp=case["tdp"])
                continue
            model = PM.fit(samples, tdp=case["tdp"])
        for field, want in case["model"].items():
            assert _close(getattr(model, field), want), (key, field, getattr(model, field), want)


def test_power_model_optimum_and_band(golden, spec_file):
    for key, case in golden["fits"].items():
        if "f_opt" not in case:
            continue
        name = key.split(":")[0]
        grid = B.load_device(spec_file(name)).spec.supported_core_clocks
        model = PM.PowerModel(**case["model"])
        f_opt = PM.optimal_frequency(model, grid)
        assert f_opt == case["f_opt"]
        band = PM.frequency_band(f_opt, grid)
        assert list(band.clocks) == case["band"] and band.reduction == case["reduction"]


def test_band_worked_example():
    # tests/test_powermodel.py:291-296
    grid = list(np.arange(300.0, 2101.0, 75.0))
    band = PM.frequency_band(1300.0, grid, pct=0.10)
    assert list(band.clocks) == [1200.0, 1275.0, 1350.0, 1425.0]
    assert band.reduction == pytest.approx(0.84)


def test_cli_readme_workflow_matches_reference(golden, spec_file, tmp_path):
    spec = str(spec_file("a100_mimic"))
    space_path = tmp_path / "space.json"
    space_path.write_text(json.dumps(golden["spaces"]["a100_mimic_space"]))
    assert cli_main(["simulate-sweep", "--device", spec, "--out", str(tmp_path / "sweep.csv"), "--points", "25"]) == 0
    assert (tmp_path / "sweep.csv").read_text() == golden["cli"]["sweep_csv"]
    assert cli_main(["fit", "--samples", str(tmp_path / "sweep.csv"), "--device", spec, "--out",
                     str(tmp_path / "model.json")]) == 0
    model = json.loads((tmp_path / "model.json").read_text())
    want = golden["cli"]["model"]
    for k in ("optimal_frequency", "band", "band_reduction", "supported_clocks", "ridge"):
        assert model[k] == want[k]
    for k, v in want["model"].items():
        assert _close(model["model"][k], v)
    assert cli_main(["steer", "--space", str(space_path), "--device", spec, "--model", str(tmp_path / "model.json"),
                     "--out", str(tmp_path / "steer"), "--observer", "instant", "--total-flops", "1.374e11"]) == 0
    rep = json.loads((tmp_path / "steer" / "report.json").read_text())
    ref = golden["cli"]["steer_report"]
    assert rep["steering"] == ref["steering"]
    assert rep["result"]["best"] == ref["result"]["best"]
    assert rep["history"] == ref["history"]
    assert rep["space_size"] == ref["space_size"] == 1144


def test_cli_exit_codes(tmp_path):
    assert cli_main(["fit", "--samples", str(tmp_path / "missing.csv"), "--device", "x.json", "--out", "m.json"]) == 2
    bad = tmp_path / "sweep.csv"
    bad.write_text("frequency_mhz,power_w\n100,1\n200,2\n")
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"name": "t", "supported_core_clocks": [100, 200], "base_clock": 100,
                                "peak_clock": 200, "power_limit_range": [10, 20], "tdp": 20,
                                "ground_truth": {"p_idle": 1, "p_max": 20, "alpha": 0.1, "tau_ft": 150,
                                                 "beta": 0.001}}))
    assert cli_main(["fit", "--samples", str(bad), "--device", str(spec), "--out", str(tmp_path / "m.json")]) == 1


def test_live_reference_agrees_on_random_expressions(reference):
    from jouletune.expressions import Expression as RefExpr

    rng = np.random.default_rng(5)
    exprs = ["a % b == 0", "a / b + c", "a // b * c - 1", "min(a, b) <= c < max(a, c)", "not a or b and c",
             "abs(a - b) ** 2", "a * b % (c / a)", "a < b < c", "a or 0", "b and c"]
    for _ in range(200):
        env = {k: int(v) for k, v in zip("abc", rng.integers(1, 9, 3))}
        for e in exprs:
            assert B.Expression(e)(env) == RefExpr(e)(env), (e, env)


def test_live_reference_fit_parity(reference):
    from jouletune import powermodel as RPM

    rng = np.random.default_rng(17)
    for trial in range(25):
        p_idle, alpha = rng.uniform(40, 180), rng.uniform(0.05, 0.3)
        tau, beta = rng.uniform(700, 1300), rng.uniform(5e-4, 2e-3)
        grid = np.linspace(300, 1965, int(rng.integers(8, 40)))
        pw = [min(1000.0, p_idle + alpha * f * (1 if f < tau else 1 + beta * (f - tau)) ** 2)
              * (1 + rng.normal(0, 0.01)) for f in grid]
        ours = [PM.FrequencySample(float(f), float(p)) for f, p in zip(grid, pw)]
        theirs = [RPM.FrequencySample(float(f), float(p)) for f, p in zip(grid, pw)]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                ref = RPM.fit(theirs, tdp=1000.0)
            except Exception as exc:  # noqa: BLE001
                with pytest.raises(B.JouleTuneError) as info:
                    PM.fit(ours, tdp=1000.0)
                assert type(info.value).__name__ == type(exc).__name__
                continue
            got = PM.fit(ours, tdp=1000.0)
        for k, v in ref.to_dict().items():
            assert _close(getattr(got, k), v, rel=1e-9), (trial, k)


def test_cli_analyze_matches_reference(golden, spec_file, tmp_path):
    """``analyze`` (Pareto front, difficulty curve under both weightings) on the
    steer run's cache: same reports and CSVs as the reference (analysis.py, cli.py:367-443)."""
    spec = str(spec_file("a100_mimic"))
    space_path = tmp_path / "space.json"
    space_path.write_text(json.dumps(golden["spaces"]["a100_mimic_space"]))
    assert cli_main(["simulate-sweep", "--device", spec, "--out", str(tmp_path / "sweep.csv"), "--points", "25"]) == 0
    assert cli_main(["fit", "--samples", str(tmp_path / "sweep.csv"), "--device", spec, "--out",
                     str(tmp_path / "model.json")]) == 0
    assert cli_main(["steer", "--space", str(space_path), "--device", spec, "--model", str(tmp_path / "model.json"),
                     "--out", str(tmp_path / "steer"), "--observer", "instant", "--total-flops", "1.374e11"]) == 0
    band = golden["cli"]["steer_report"]["steering"]["band"]
    steered = B.SearchSpace.from_dict(golden["spaces"]["a100_mimic_space"]).with_values("nvml_gr_clock", band)
    (tmp_path / "steered.json").write_text(json.dumps(steered.to_dict()))
    cache = str(tmp_path / "steer" / "cache.jsonl")
    runs = {"pareto": ["--mode", "pareto"],
            "absorbing": ["--mode", "difficulty", "--space", str(tmp_path / "steered.json")],
            "pagerank": ["--mode", "difficulty", "--space", str(tmp_path / "steered.json"), "--weights", "pagerank",
                         "--p-max", "2.0", "--p-steps", "11"],
            "time": ["--mode", "difficulty", "--space", str(tmp_path / "steered.json"), "--objective", "time"]}
    for label, extra in runs.items():
        want = golden["analyze"][label]
        out = tmp_path / f"analyze_{label}"
        assert cli_main(["analyze", "--cache", cache, "--out", str(out), *extra]) == want["rc"] == 0
        doc = json.loads((out / "analyze.json").read_text())
        assert sorted(doc["manifest"]) == want["manifest_keys"], label
        body = {k: v for k, v in doc.items() if not k.startswith("manifest")}
        assert body.keys() == want["report"].keys(), label
        for k, v in want["report"].items():
            if isinstance(v, float):
                assert _close(body[k], v), (label, k)
            else:
                assert body[k] == v, (label, k)
        csv_name = "pareto.csv" if label == "pareto" else "difficulty.csv"
        assert (out / csv_name).read_text() == want["csv"], label


def test_landscape_units():
    """Pareto and flow-graph rules on hand-checkable cases."""
    from paper_2211_07260_b200 import landscape as L

    K = lambda **kw: B.KernelConfig.from_dict(kw)  # noqa: E731
    pts = [L.ParetoPoint(K(i=i), p, e) for i, (p, e) in enumerate([(3, 1), (2, 2), (2, 2), (1, 3), (1, 1), (3, 0.5)])]
    front = L.pareto_front(pts)
    assert [(p.performance, p.efficiency) for p in front] == [(3, 1), (2, 2), (1, 3)]
    assert front[1] is pts[1]  # duplicate coordinates: first occurrence only
    assert L.dominates(pts[0], pts[5]) and not L.dominates(pts[1], pts[2]) and not L.dominates(pts[0], pts[1])
    space = B.SearchSpace.from_dict({"parameters": {"a": [0, 1], "b": [0, 1]}})
    fit = {K(a=0, b=0): 1.0, K(a=1, b=1): 1.5, K(a=0, b=1): 3.0, K(a=1, b=0): 2.0}
    g = L.build_ffg(space, fit)
    assert set(g.minima) == {K(a=0, b=0), K(a=1, b=1)} and g.edge_count() == 4
    w = L.minima_arrival_distribution(g)  # each transient node splits 1/2 : 1/2, each sink keeps its own walk
    assert w[K(a=0, b=0)] == pytest.approx(0.5) and w[K(a=1, b=1)] == pytest.approx(0.5)
    pr = L.minima_arrival_distribution(g, mode="pagerank")
    assert sum(pr.values()) == pytest.approx(1.0) and pr[K(a=0, b=0)] == pytest.approx(pr[K(a=1, b=1)])
    curve = L.proportion_of_centrality(g, w, [1.0, 1.4, 1.5])
    assert curve.f_optimal == 1.0 and curve.proportions == pytest.approx((0.5, 0.5, 1.0))
    with pytest.raises(B.AnalysisError):
        L.build_ffg(space, {K(a=0, b=0): 1.0})
    with pytest.raises(B.ConfigurationError):
        L.minima_arrival_distribution(g, mode="random")
