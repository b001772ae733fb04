"""Unit tests of the API layer in the style of the reference suite
(brute-force / closed-form oracles)."""

import itertools
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2211_07260_b200 as B
from paper_2211_07260_b200.device import ConstantSurface, DeviceSpec, GroundTruth, SimulatedDevice
from paper_2211_07260_b200.errors import ConfigurationError, ExpressionError, UnknownNameError

# -- expressions (reference expressions.py semantics) -------------------------------


@pytest.mark.parametrize(
    "src, env, want",
    [
        ("Kwg % Kwi == 0", {"Kwg": 32, "Kwi": 8}, True),
        ("total_flops / time / 1e9", {"total_flops": 2e9, "time": 0.5}, 4.0),
        ("a / b", {"a": 3, "b": 2}, 1.5),
        ("a // b", {"a": 7, "b": 2}, 3),
        ("1 < a <= 3 < b", {"a": 3, "b": 4}, True),
        ("1 < a <= 3 < b", {"a": 3, "b": 3}, False),
        ("a or b", {"a": 0, "b": 5}, 5),
        ("a and b", {"a": 2, "b": 0}, 0),
        ("not a", {"a": 0}, True),
        ("max(a, b) - min(a, b) + abs(-a)", {"a": 2, "b": 7}, 7),
        ("-a ** 2", {"a": 3}, -9),
        ("True + 1", {}, 2),
    ],
)
def test_expression_values(src, env, want):
    assert B.Expression(src)(env) == want


@pytest.mark.parametrize("src", ["a & b", "a in b", "len(a)", "a.b", "'s'", "lambda: 1", "min(a, key=b)", "x[0]",
                                 "", "a is b", "f(1)", "(1,)"])
def test_expression_rejects_syntax(src):
    with pytest.raises(ExpressionError):
        B.Expression(src)


def test_expression_unknown_name_and_names():
    e = B.Expression("a + b * c")
    assert e.names == frozenset("abc")
    with pytest.raises(UnknownNameError) as info:
        e({"a": 1, "b": 2})
    assert info.value.name == "c"


# -- search spaces (brute-force oracle, reference tests/test_searchspace.py:28-35) ----


def brute(space):
    out = []
    for combo in itertools.product(*[p.values for p in space.parameters]):
        env = dict(zip(space.names, combo))
        if all(eval(r.expression, {"min": min, "max": max, "abs": abs}, dict(env)) for r in space.restrictions):
            out.append(B.KernelConfig(tuple(env.items())))
    return out


@settings(max_examples=60, deadline=None)
@given(
    st.lists(st.lists(st.integers(1, 12), min_size=1, max_size=4, unique=True), min_size=1, max_size=4),
    st.sampled_from(["p0 % p1 == 0", "p0 * p1 <= 24", "p0 + p1 > p2", "p0 < 5 or p2 == p1", "p1 / p0 >= 1"]),
)
def test_enumeration_matches_brute_force(value_lists, rule):
    params = tuple(B.TunableParameter(f"p{i}", tuple(v)) for i, v in enumerate(value_lists))
    names = {p.name for p in params}
    rules = (B.Restriction(rule),) if B.Expression(rule).names <= names else ()
    space = B.SearchSpace(params, rules)
    assert space.enumerate() == brute(space)


def test_augment_with_values_and_neighbors():
    space = B.SearchSpace.from_dict({"parameters": {"a": [1, 2, 4], "b": [1, 2, 3, 4]}, "restrictions": ["b % a == 0"]})
    aug = space.augment(B.TunableParameter("nvml_gr_clock", (100, 200, 300)))
    assert aug.size() == 3 * space.size()
    assert aug.enumerate()[0]["nvml_gr_clock"] == 100 and aug.enumerate()[1]["nvml_gr_clock"] == 200
    pinned = aug.with_values("nvml_gr_clock", [200])
    assert pinned.size() == space.size()
    for cfg in space.enumerate():
        want = [c for c in space.enumerate() if sum(c[n] != cfg[n] for n in space.names) == 1]
        assert sorted(space.neighbors(cfg), key=lambda c: c.items) == sorted(want, key=lambda c: c.items)
    with pytest.raises(ConfigurationError):
        space.augment(B.TunableParameter("a", (1,)))
    with pytest.raises(UnknownNameError):
        B.SearchSpace.from_dict({"parameters": {"a": [1]}, "restrictions": ["zz > 1"]})


def test_config_key_and_normalisation():
    a = B.KernelConfig.from_dict({"x": 1, "nvml_gr_clock": 810})
    b = B.KernelConfig.from_dict({"nvml_gr_clock": 810.0, "x": 1})
    assert a == b and hash(a) == hash(b)
    assert a.key() != b.key()  # reference hazard, kept for cache compatibility
    assert b.normalized().key() == a.key()
    assert B.normalize_value(True) is True and B.normalize_value(2.5) == 2.5


# -- sensors (reference tests/test_observers.py closed forms) ------------------------


def test_averaged_window_closed_form():
    ramp = [B.PowerSample(float(t), 20.0 + 50.0 * float(t)) for t in np.linspace(0.0, 1.0, 101)]
    cfg = B.AveragedSensorConfig(refresh_rate=10.0)
    assert B.averaged_reading(ramp, 0.201, cfg) == pytest.approx(27.5, abs=1e-9)
    with pytest.raises(B.SensorNotReadyError):
        B.averaged_reading(ramp, 0.05, cfg)
    step = [B.PowerSample(0.0, 100.0), B.PowerSample(0.5, 100.0), B.PowerSample(0.5, 200.0), B.PowerSample(1.0, 200.0)]
    assert B.averaged_reading(step, 1.0, B.AveragedSensorConfig(refresh_rate=1.0)) == pytest.approx(150.0)
    with pytest.raises(B.MeasurementError):
        B.averaged_reading([B.PowerSample(0.5, 1.0), B.PowerSample(0.9, 1.0)], 1.0, B.AveragedSensorConfig(1.0))


def _steady_device(noise=0.0):
    spec = DeviceSpec("steady", (500, 1000), 1000, 1000, (50.0, 300.0), 300.0)
    truth = GroundTruth(p_idle=50.0, p_max=300.0, alpha=0.1, tau_ft=1000.0, beta=1e-9, noise_stddev=noise)
    return SimulatedDevice(spec, truth, ConstantSurface(reference_clock=1000.0, base_time=3e-3))


def test_continuous_benchmark_steady_state():
    dev = _steady_device()
    out = B.continuous_benchmark(dev, B.KernelConfig(()), B.AveragedSensorConfig(10.0, 1.0))
    assert out.energy == pytest.approx(dev.modeled_power(1000) * out.duration, rel=0.005)
    assert out.duration >= 1.0 and not out.long_kernel


def test_instant_observer_ignores_tail_samples():
    obs = B.InstantPowerObserver()
    trace = tuple(B.PowerSample(t, 100.0 if t <= 0.002 else 500.0) for t in np.linspace(0, 0.01, 11))
    run = B.Execution(0.002, trace, 1000.0, 5, 0.01)
    pb = B.observers.TracePlayback(run)
    obs.before_start()
    obs.after_start(pb)
    while pb.advance(0.001):
        obs.during(pb)
    obs.after_finish(pb)
    assert obs.get_results()["ps_power"] == 100.0


# -- tuner behaviour ---------------------------------------------------------------


class FailingDevice:
    """Wraps a simulated device; configs with x == 2 raise DomainError."""

    def __init__(self):
        self.inner = _steady_device()
        self.spec = self.inner.spec
        self.sample_rate_hz = self.inner.sample_rate_hz
        self.execution_count = 0

    def set_core_clock(self, c):
        return self.inner.set_core_clock(c)

    def set_power_limit(self, w):
        return self.inner.set_power_limit(w)

    def execute(self, config, duration_hint=0.0):
        if config.get("x") == 2:
            raise B.DomainError("launch rejected")
        self.execution_count += 1
        return self.inner.execute(config, duration_hint)


def test_failures_become_results_and_all_failed_raises():
    space = B.SearchSpace.from_dict({"parameters": {"x": [1, 2, 3]}})
    out = B.run_strategy(B.TuningRun(space), FailingDevice(), [B.InstantPowerObserver()])
    failed = [r for r in out.history if r.failed]
    assert len(failed) == 1 and math.isinf(failed[0].time) and "DomainError" in failed[0].failure_reason
    with pytest.raises(B.TuningError):
        B.run_strategy(B.TuningRun(B.SearchSpace.from_dict({"parameters": {"x": [2]}})), FailingDevice())


def test_observer_key_collision_is_a_configuration_error():
    class Dup(B.BenchmarkObserver):
        def get_results(self):
            return {"ps_power": 1.0}

    with pytest.raises(ConfigurationError):
        B.benchmark(_steady_device(), B.KernelConfig(()), [B.InstantPowerObserver(), Dup()])


class CounterDevice:
    """A device reporting a real-hardware style Execution (window + counter)."""

    spec = DeviceSpec("fake-b200", (1000, 1965), 1965, 1965, (200.0, 1000.0), 1000.0)
    sample_rate_hz = 1000.0

    def __init__(self):
        self.execution_count = 0

    def set_core_clock(self, c):
        return None

    def execute(self, config, duration_hint=0.0):
        self.execution_count += 1
        trace = tuple(B.PowerSample(t, 200.0 if t < 0.02 else 600.0) for t in np.arange(0, 0.3, 0.001))
        return B.Execution(runtime=1e-3, samples=trace, effective_clock=1965.0, repetitions=300, total_duration=0.3,
                           window=(0.02, 0.3), counter_power=610.0, counter_energy=183.0,
                           telemetry={"sm_clock": 1965.0, "temperature": 50.0, "clock_locked": 0.0})


def test_counter_mode_and_windowed_instant_rule():
    dev = CounterDevice()
    res = B.benchmark(dev, B.KernelConfig(()), [B.NVMLObserver(0.3)])
    assert res.energy == pytest.approx(610.0 * 1e-3)
    assert res.observer_results["nvml_power"] == 610.0
    assert res.observer_results["nvml_power_instant"] == 600.0
    assert res.observer_results["nvml_clock_locked"] == 0.0
    # instant rule on a real trace uses the steady window, not [0, runtime]
    res = B.benchmark(dev, B.KernelConfig(()), [B.InstantPowerObserver()])
    assert res.energy == pytest.approx(600.0 * 1e-3)
    assert res.observer_results["ps_power"] == 600.0


def test_result_cache_round_trip_and_warm_cache(tmp_path):
    path = tmp_path / "c.jsonl"
    space = B.SearchSpace.from_dict({"parameters": {"nvml_gr_clock": [500, 1000]}})
    dev = _steady_device()
    first = B.run_strategy(B.TuningRun(space), dev, [B.InstantPowerObserver()], cache=B.ResultCache(path))
    warm = B.run_strategy(B.TuningRun(space), dev, [B.InstantPowerObserver()], cache=B.ResultCache(path))
    assert first.device_executions == 2 and warm.device_executions == 0
    assert [r.to_dict() for r in first.history] == [r.to_dict() for r in warm.history]


def test_prepare_sweep_drops_capped_and_keys_by_observed_clock():
    recs = [
        {"requested_mhz": 1000, "observed_mhz": 1000, "power_w": 500.0},
        {"requested_mhz": 1500, "observed_mhz": 1500, "power_w": 700.0},
        {"requested_mhz": 1800, "observed_mhz": 1650, "power_w": 990.0, "power_capped": True},
        {"requested_mhz": 1965, "observed_mhz": 1650, "power_w": 995.0},
        {"requested_mhz": 1600, "observed_mhz": 1600, "power_w": 980.0},
    ]
    samples, dropped = B.prepare_sweep(recs, power_limit=1000.0)
    assert [s.frequency for s in samples] == [1000.0, 1500.0]
    assert {d["dropped"] for d in dropped} == {"power cap active", "observed clock below requested",
                                               "power at the limit"}


def test_steered_power_capped_fit_recovers_optimum():
    """a noisy 1 kW cap plateau defeats the reference fit unless the
    capped samples are dropped first (prepare_sweep)."""
    truth = GroundTruth(p_idle=180, p_max=1000, alpha=0.30, tau_ft=1200, beta=0.0012, noise_stddev=0.0)
    grid = np.arange(195.0, 1966.0, 15.0)
    hits = 0
    for seed in range(10):
        rng = np.random.default_rng(seed)
        recs = []
        for f in grid:
            p = truth.power(f) * (1 + rng.normal(0, 0.01))
            recs.append({"requested_mhz": f, "observed_mhz": f, "power_w": p,
                         "power_capped": truth.power(f) >= 1000.0})
        samples, _ = B.prepare_sweep(recs, power_limit=1000.0)
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model = B.fit(samples, tdp=1000.0)
        f_opt = B.optimal_frequency(model, list(grid))
        hits += abs(f_opt - 1200.0) <= 0.1 * 1200.0
    assert hits >= 9


def test_callable_metric_uses_milliseconds():
    from paper_2211_07260_b200.facade import CallableMetric

    m = CallableMetric("gflops", "0", fn=lambda p: 2e9 / 1e9 / (p["time"] / 1e3))
    assert m.evaluate({"time": 0.5, "energy": 1.0}) == pytest.approx(4.0)
    with pytest.raises(ConfigurationError):
        CallableMetric("not an id", "0", fn=lambda p: 0)
