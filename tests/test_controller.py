"""Clock / power controller of B200Device against a scripted NVML (CPU only).

The GPU pool refuses every knob (``profiles/r2_knob_probe.json``: NVML
``Not Supported``, code 3, as root), so the refusal path is the one that
runs in production there; these tests pin its semantics:

* a refused request is a failed result with NVML's reason, never a result
  stored under a clock (or limit) the board did not run at;
* the default clock with no lock active is the driver-managed state and is
  measured (``clock_locked`` False);
* an active lock is always undone on release / close, even after a later
  refusal flipped ``clock_mode``;
* a power limit is read back after an accepted set.
"""

from __future__ import annotations

import json
import types

import pytest

import paper_2211_07260_b200 as B
from paper_2211_07260_b200.b200 import B200Device
from paper_2211_07260_b200.kernels import make_problem


class FakeGPU:
    """Just enough of gpu.GPU for the controller; ``accept`` scripts NVML."""

    def __init__(self, accept_lock=False, accept_app=False, accept_limit=False, enforce=None):
        self.info = types.SimpleNamespace(default_sm_clock_mhz=1965, power_limit_min_mw=200_000,
                                          power_limit_max_mw=1_000_000, power_limit_default_mw=1_000_000,
                                          power_limit_mw=1_000_000, mem_clock_mhz=3996,
                                          pci_bus_id=b"00000000:E5:00.0")
        self.name, self.ordinal, self.sm_count = "NVIDIA B200", 0, 148
        self.accept_lock, self.accept_app, self.accept_limit, self.enforce = accept_lock, accept_app, accept_limit, enforce
        self.calls = []
        self.last_refusal = None

    def supported_clocks(self):
        return list(range(120, 1966, 15))

    def _answer(self, ok, what):
        if not ok:
            self.last_refusal = f"{what}: Not Supported"
        return ok

    def lock_clocks(self, lo, hi):
        self.calls.append(("lock", lo))
        return self._answer(self.accept_lock, "nvmlDeviceSetGpuLockedClocks")

    def reset_clocks(self):
        self.calls.append(("reset_lock",))
        return True

    def set_app_clocks(self, mem, sm):
        self.calls.append(("app", sm))
        return self._answer(self.accept_app, "nvmlDeviceSetApplicationsClocks")

    def reset_app_clocks(self):
        self.calls.append(("reset_app",))
        return True

    def set_power_limit(self, w):
        self.calls.append(("limit", w))
        ok = self._answer(self.accept_limit, "nvmlDeviceSetPowerManagementLimit")
        if ok:
            self.info.power_limit_mw = int((self.enforce or w) * 1000)
        return ok

    def reset_power_limit(self):
        self.calls.append(("reset_limit",))
        self.info.power_limit_mw = self.info.power_limit_default_mw
        return True

    def enforced_power_limit_w(self):
        return self.info.power_limit_mw / 1000.0

    def close(self):
        pass


def device(gpu):
    problem = make_problem("burner")
    problem.gpu = gpu
    return B200Device(problem, gpu=gpu, clock_settle=0.0)


def test_refused_clock_is_a_failure_not_a_mislabelled_result():
    gpu = FakeGPU()
    dev = device(gpu)
    with pytest.raises(B.ControlRefusedError) as exc:
        dev.set_core_clock(1005.0)
    assert exc.value.knob == "core_clock" and "Not Supported" in exc.value.reason
    assert isinstance(exc.value, B.CapabilityError)  # -> failed result in benchmark (tuner.py:257-271)
    assert dev.clock_mode == "refused" and dev.refusals[-1]["requested"] == 1005.0
    assert dev.state.core_clock == 1965.0  # state not moved to the refused label
    # the default clock with no lock active is the driver-managed state: measured, flagged unlocked
    dev.set_core_clock(1965.0)
    assert dev.clock_locked is False and dev.state.core_clock == 1965.0


def test_benchmark_records_refusal_as_failed_result():
    gpu = FakeGPU()
    dev = device(gpu)
    dev.execute = lambda cfg, duration_hint=0.0: pytest.fail("must not execute under a refused clock")
    res = B.benchmark(dev, B.KernelConfig.from_dict({"nvml_gr_clock": 1500}), [B.NVMLObserver(0.1)])
    assert res.failed and "ControlRefusedError" in res.failure_reason and "Not Supported" in res.failure_reason


def test_lock_then_refusal_still_releases_the_active_lock():
    gpu = FakeGPU(accept_lock=True)
    dev = device(gpu)
    dev.set_core_clock(1500.0)
    assert dev.clock_locked and dev.clock_mode == "locked"
    gpu.accept_lock = False
    with pytest.raises(B.ControlRefusedError):
        dev.set_core_clock(1005.0)
    assert dev.refusals[-1]["active_lock_mhz"] == 1500.0
    dev.release_clock()
    assert ("reset_lock",) in gpu.calls
    gpu.calls.clear()
    dev.close()
    assert ("reset_lock",) not in gpu.calls  # nothing left to undo


def test_application_clock_fallback_and_close_resets_it():
    gpu = FakeGPU(accept_app=True)
    dev = device(gpu)
    dev.set_core_clock(1200.0)
    assert dev.clock_mode == "application" and dev.clock_locked
    dev.set_core_clock(1200.0)  # idempotent: no second NVML call
    assert [c for c in gpu.calls if c[0] == "app"] == [("app", 1200)]
    dev.close()
    assert ("reset_app",) in gpu.calls


def test_power_limit_refused_accepted_and_read_back():
    gpu = FakeGPU()
    dev = device(gpu)
    with pytest.raises(B.ControlRefusedError) as exc:
        dev.set_power_limit(600.0)
    assert exc.value.knob == "power_limit"
    dev.set_power_limit(1000.0)  # the limit already in force: nothing to change
    assert dev.state.power_limit == 1000.0
    gpu2 = FakeGPU(accept_limit=True)
    dev2 = device(gpu2)
    dev2.set_power_limit(600.0)
    assert dev2.state.power_limit == 600.0
    gpu3 = FakeGPU(accept_limit=True, enforce=700.0)
    dev3 = device(gpu3)
    with pytest.raises(B.ControlRefusedError, match="enforces 700"):
        dev3.set_power_limit(600.0)
    with pytest.raises(B.DomainError):
        dev.set_power_limit(50.0)


def test_simulate_sweep_on_refusing_device_writes_no_sweep(tmp_path, monkeypatch):
    from paper_2211_07260_b200 import commands

    gpu = FakeGPU()
    dev = device(gpu)
    trace = tuple(B.PowerSample(t / 100, 900.0) for t in range(11))
    dev.execute = lambda cfg, duration_hint=0.0: B.Execution(
        runtime=1e-3, samples=trace, effective_clock=1965.0, repetitions=100, total_duration=0.1,
        window=(0.02, 0.1), counter_power=900.0, counter_energy=90.0, telemetry={"clock_locked": 0.0})
    monkeypatch.setattr(commands, "open_device", lambda *a, **k: dev)
    out = tmp_path / "sweep.csv"
    rc = commands.main(["simulate-sweep", "--device", "b200", "--out", str(out), "--points", "7",
                        "--observer", "nvml", "--duration", "0.1"])
    assert rc == 1 and not out.exists()
    meta = json.loads((tmp_path / "sweep.csv.meta.json").read_text())
    assert len(meta["refused"]) == 6 and meta["clock_mode"] == "refused"
    assert all("Not Supported" in r["reason"] for r in meta["refused"])


def _sensor_execution(avg_watts):
    trace = tuple(B.PowerSample(t / 1000, 500.0 + (t % 7)) for t in range(0, 2501, 1))
    sensor = tuple(B.PowerSample(t / 10, w) for t, w in avg_watts)
    return B.Execution(runtime=1e-3, samples=trace, effective_clock=1965.0, repetitions=2500, total_duration=2.5,
                       window=(0.02, 2.5), counter_power=505.0, sensor_samples=sensor, sensor_window=1.0)


def test_sensor_reading_uses_the_boards_own_average():
    from paper_2211_07260_b200.sensors import sensor_reading

    run = _sensor_execution([(2, 200.0), (9, 400.0), (12, 480.0), (24, 510.0), (26, 999.0)])
    cfg = B.AveragedSensorConfig(refresh_rate=1.0, continuous_duration=2.5)
    assert sensor_reading(run, 2.5, cfg) == 510.0  # last reading at or before t, not the later one
    assert sensor_reading(run, 1.25, cfg) == 480.0  # the 0.2 s reading's window started before the trace
    with pytest.raises(B.SensorNotReadyError):
        sensor_reading(run, 0.5, cfg)
    with pytest.raises(B.ConfigurationError, match="refresh_rate must be 1"):
        sensor_reading(run, 2.5, B.AveragedSensorConfig(refresh_rate=10.0))
    # without a board sensor the reference window rule over the instant trace applies
    plain = B.Execution(runtime=1e-3, samples=run.samples, effective_clock=1965.0, repetitions=1, total_duration=2.5)
    assert sensor_reading(plain, 2.5, cfg) == pytest.approx(B.averaged_reading(run.samples, 2.5, cfg))


def test_averaged_mode_benchmark_reads_board_sensor():
    class SensorDevice:
        spec = B.DeviceSpec("fake-b200", (1000, 1965), 1965, 1965, (200.0, 1000.0), 1000.0)
        sample_rate_hz = 1000.0
        execution_count = 0

        def execute(self, config, duration_hint=0.0):
            assert duration_hint == 2.5
            return _sensor_execution([(12, 480.0), (24, 510.0)])

    cfg = B.AveragedSensorConfig(refresh_rate=1.0, continuous_duration=2.5)
    res = B.benchmark(SensorDevice(), B.KernelConfig(()), [B.AveragedPowerObserver(cfg)], averaged_cfg=cfg)
    assert res.energy == pytest.approx(510.0 * 1e-3)
    assert res.observer_results["nvml_power"] == 510.0
    with pytest.raises(B.ConfigurationError):
        B.benchmark(SensorDevice(), B.KernelConfig(()), [B.AveragedPowerObserver()],
                    averaged_cfg=B.AveragedSensorConfig(continuous_duration=2.5))


def test_counter_updates_and_slope_window():
    from paper_2211_07260_b200.b200 import counter_slope, counter_updates

    nan = float("nan")
    # (t, p_inst, p_avg, energy J, energy stamp, sm, mem, temp, reasons): counter steps every 0.1 s at 500 W
    samples = [(0.01 * i, 500.0, 500.0, 100.0 + 50.0 * (i // 10), 0.1 * (i // 10), 1965, 3996, 50, 0)
               for i in range(60)]
    assert counter_updates(samples, 0.05, 0.33) == 3  # stamps 0.1, 0.2, 0.3
    assert counter_slope(samples, 0.05, 0.33) == pytest.approx(500.0)
    assert counter_updates(samples, 0.12, 0.19) == 0 and counter_slope(samples, 0.12, 0.19) is None
    samples.append((0.7, 500.0, 500.0, nan, nan, 1965, 3996, 50, 0))  # a missing reading is ignored
    assert counter_updates(samples, 0.0, 1.0) == 6


def test_counter_power_whole_periods_ignore_timestamp_jitter():
    """The counter adds one 100 ms period per change; change times jitter by +-35 ms. A dE/dt slope
    over two changes scatters with the jitter, whole periods do not (profiles/r2_energy_probe.json)."""
    import numpy as np

    from paper_2211_07260_b200.b200 import counter_power, counter_slope

    rng = np.random.default_rng(5)
    nan = float("nan")
    # 400 W before t = 1.0 (previous config), 750 W in the loop [1.0, 1.31], 250 W after
    def power(t):
        return 400.0 if t < 1.0 else (750.0 if t < 1.31 else 250.0)

    changes, e = [], 1000.0
    for j in range(1, 25):  # period ends every 0.1 s (offset 0.03), seen with jitter
        end = 0.03 + 0.1 * j
        e += sum(power(end - 0.1 + 0.001 * i) for i in range(100)) * 0.001
        changes.append((end + rng.uniform(-0.035, 0.035) + 0.004, e))
    samples, k = [], 0
    for i in range(2600):
        t = 0.001 * i
        while k < len(changes) and changes[k][0] <= t:
            k += 1
        energy = changes[k - 1][1] if k else 1000.0
        samples.append((t, 500.0, 500.0, energy, nan, 1965, 3996, 50, 0))
    watts, periods = counter_power(samples, 1.0, 1.31)
    assert periods >= 2
    assert watts == pytest.approx(750.0, rel=0.02)
    # the long trace estimates the period itself
    assert counter_power(samples, 0.0, 2.5)[1] >= 20
    # a window shorter than one whole period has none
    assert counter_power(samples, 1.0, 1.09) == (None, 0)
    assert counter_slope(samples, 1.0, 1.31) is not None  # the old estimator still exists for comparison


def test_stale_nvml_loop_is_rerun():
    """A loop whose trace holds no whole energy-counter period (a stalled NVML call returned its
    reading after the loop) is measured again; the result records the re-run."""
    from paper_2211_07260_b200.gpu import BenchRun

    nan = float("nan")

    def trace(t0, stale):
        # counter periods end at t0 + 0.1 k; a stale trace sees the first change stamped after the loop
        out, e = [], 5000.0
        for i in range(300):
            t = t0 + 0.001 * i
            k = int((t - t0) / 0.1)
            stamp = t0 + 0.1 * k
            if stale:
                k, stamp = 0, t0
            out.append((t, 700.0, 700.0, e + 70.0 * k, stamp, 1965, 3996, 50, 0))
        if stale:
            out.append((t0 + 0.31, 700.0, 700.0, e + 210.0, t0 + 0.6, 1965, 3996, 50, 0))
        return out

    gpu = FakeGPU()
    runs = iter([True, True, False])
    calls = []

    def bench(kernel, launch, args, *, min_seconds, sample_period_us=1000, **kw):
        stale = next(runs)
        calls.append(stale)
        t0 = 10.0 * len(calls)
        return BenchRun(1e-3, 1e-3, 0.3, 300, t0, t0 + 0.3, trace(t0, stale))

    gpu.bench = bench
    dev = device(gpu)
    dev._compiled = lambda config: ({}, None, types.SimpleNamespace(threads=128))
    dev.problem.bind = lambda kernel, cfg: None
    dev.problem.args = lambda cfg: []
    ex = dev.execute(B.KernelConfig(()), duration_hint=0.3)
    assert calls == [True, True, False]
    assert ex.telemetry["stale_retries"] == 2.0
    assert ex.counter_power == pytest.approx(700.0, rel=0.01)
    # at most two re-runs: a board that stays stale is measured three times and falls back
    runs = iter([True, True, True])
    calls.clear()
    ex = dev.execute(B.KernelConfig(()), duration_hint=0.3)
    assert calls == [True, True, True] and ex.telemetry["stale_retries"] == 2.0


def test_counter_instant_disagreement_is_rerun():
    """A loop whose counter power is half its instant-power median (one bad increment) is measured
    again; the agreeing re-run is the one kept."""
    from paper_2211_07260_b200.gpu import BenchRun

    def trace(t0, per_period_j):
        out = []
        for i in range(300):
            t = t0 + 0.001 * i
            k = int((t - t0) / 0.1)
            out.append((t, 700.0, 700.0, 5000.0 + per_period_j * k, t0 + 0.1 * k, 1965, 3996, 50, 0))
        return out

    gpu = FakeGPU()
    energies = iter([35.0, 70.0])
    calls = []

    def bench(kernel, launch, args, *, min_seconds, sample_period_us=1000, **kw):
        calls.append(1)
        t0 = 10.0 * len(calls)
        return BenchRun(1e-3, 1e-3, 0.3, 300, t0, t0 + 0.3, trace(t0, next(energies)))

    gpu.bench = bench
    dev = device(gpu)
    dev._compiled = lambda config: ({}, None, types.SimpleNamespace(threads=128))
    dev.problem.bind = lambda kernel, cfg: None
    dev.problem.args = lambda cfg: []
    ex = dev.execute(B.KernelConfig(()), duration_hint=0.3)
    assert len(calls) == 2 and ex.telemetry["stale_retries"] == 1.0 and ex.telemetry["power_disagree"] == 0.0
    assert ex.counter_power == pytest.approx(700.0, rel=0.01)
