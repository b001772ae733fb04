"""Observers: the lifecycle hooks that turn a measured trace into readings.

Lifecycle ``before_start -> after_start -> during* -> after_finish ->
get_results`` (reference ``pkg/src/jouletune/observers.py:207-287``); keys
carry the observer's prefix so several observers can be attached together.

Added for the B200 backend: :class:`NVMLObserver` reports what the NVML
sampler inside ``libjt`` recorded around the device-timed loop (energy
counter slope, instant-power median, SM clock, temperature, clock-lock
status) under the ``nvml_`` prefix. It replaces — and must not be attached
together with — :class:`AveragedPowerObserver`, which owns the same prefix.
"""

from __future__ import annotations

import statistics

from .errors import ConfigurationError, SensorNotReadyError
from .sensors import AveragedSensorConfig, InstantSensorConfig, TracePlayback

__all__ = ["BenchmarkObserver", "InstantPowerObserver", "AveragedPowerObserver", "NVMLObserver"]


class BenchmarkObserver:
    """Observer base class; ``get_results`` keys carry the observer's prefix."""

    def before_start(self) -> None:
        pass

    def after_start(self, playback: TracePlayback) -> None:
        pass

    def during(self, playback: TracePlayback) -> None:
        pass

    def after_finish(self, playback: TracePlayback) -> None:
        pass

    def get_results(self) -> dict[str, float]:
        return {}


class InstantPowerObserver(BenchmarkObserver):
    """External fast power meter (``ps_`` prefix): median over [0, runtime]."""

    prefix = "ps_"

    def __init__(self, cfg: InstantSensorConfig | None = None):
        self.cfg = cfg or InstantSensorConfig()
        self._readings: list[tuple[float, float]] = []
        self._runtime = 0.0
        self._window: tuple[float, float] | None = None

    def before_start(self) -> None:
        self._readings = []
        self._window = None

    def after_start(self, playback: TracePlayback) -> None:
        self._readings.append((playback.now, playback.instant_power()))

    def during(self, playback: TracePlayback) -> None:
        self._readings.append((playback.now, playback.instant_power()))

    def after_finish(self, playback: TracePlayback) -> None:
        self._runtime = playback.runtime
        self._window = playback.execution.window

    def get_results(self) -> dict[str, float]:
        if self._window is not None:
            # real trace: median over the steady loop window (B200 rule, see tuner)
            t0, t1 = self._window
            powers = [p for t, p in self._readings if t0 - 1e-12 <= t <= t1 + 1e-12]
        else:
            powers = [p for t, p in self._readings if t <= self._runtime + 1e-12]
        if not powers:
            return {}
        med = statistics.median(powers)
        return {"ps_power": med, "ps_energy": med * self._runtime}


class AveragedPowerObserver(BenchmarkObserver):
    """On-board averaged sensor (``nvml_`` prefix), reference semantics."""

    prefix = "nvml_"

    def __init__(self, cfg: AveragedSensorConfig | None = None):
        self.cfg = cfg or AveragedSensorConfig()
        self._final_reading: float | None = None
        self._duration = 0.0

    def before_start(self) -> None:
        self._final_reading = None

    def after_finish(self, playback: TracePlayback) -> None:
        self._duration = playback.total_duration
        try:
            self._final_reading = playback.final_averaged_power(self.cfg)
        except SensorNotReadyError:
            self._final_reading = None

    def get_results(self) -> dict[str, float]:
        if self._final_reading is None:
            return {}
        return {"nvml_power": self._final_reading, "nvml_energy": self._final_reading * self._duration}


class NVMLObserver(BenchmarkObserver):
    """B200 NVML readings around a device-timed loop (``nvml_`` prefix).

    Results per benchmark (energies are per single kernel execution):

    * ``nvml_energy`` — energy-counter power over the steady window x runtime
      (the primary energy source, ``nvmlDeviceGetTotalEnergyConsumption``): the
      counter's whole fixed periods inside the window, summed and divided by
      their duration (``b200.counter_power``);
    * ``nvml_power`` — that counter power in W;
    * ``nvml_power_instant`` — median instant power over the window;
    * ``nvml_sm_clock`` / ``nvml_temperature`` / ``nvml_mem_clock`` — medians;
    * ``nvml_clock_locked`` — 1.0 if the controller held the requested clock,
      0.0 if NVML refused (the observed clock is then the truth);
    * ``nvml_energy_source`` — 1.0 counter periods inside the steady window,
      0.5 counter periods anywhere in the loop (none after the settle), 0.0
      instant-power median (a loop shorter than one counter period);
    * ``nvml_counter_updates`` — counter periods the energy used;
    * ``nvml_stale_retries`` — loops re-run because NVML showed no whole
      counter period during them (stalled readings) or its counter and
      instant-power estimates disagreed by more than 15%;
    * ``nvml_power_disagree`` — 1.0 if they still disagreed after the re-runs.

    Attaching it switches the benchmark energy rule to ``counter`` mode
    (see ``tuner.MeasurementSetup``).
    """

    prefix = "nvml_"

    def __init__(self, duration: float = 0.25):
        if duration <= 0:
            raise ConfigurationError("NVMLObserver duration must be positive")
        #: length of the back-to-back launch loop per benchmark (s)
        self.duration = float(duration)
        self._result: dict[str, float] = {}

    def before_start(self) -> None:
        self._result = {}

    def after_finish(self, playback: TracePlayback) -> None:
        run = playback.execution
        tele = dict(run.telemetry or {})
        out: dict[str, float] = {}
        if run.counter_power is not None:
            out["nvml_power"] = run.counter_power
            out["nvml_energy"] = run.counter_power * run.runtime
        window = run.window or (0.0, run.total_duration)
        inside = [s.power for s in run.samples if window[0] <= s.timestamp <= window[1]]
        if inside:
            out["nvml_power_instant"] = statistics.median(inside)
        for key in ("sm_clock", "mem_clock", "temperature", "clock_locked", "throttle_reasons", "energy_source",
                    "counter_updates", "stale_retries", "power_disagree"):
            if key in tele:
                out[f"nvml_{key}"] = float(tele[key])
        self._result = out

    def get_results(self) -> dict[str, float]:
        return dict(self._result)
