"""Measuring one configuration: apply execution parameters, run, derive energy.

Reference: ``pkg/src/jouletune/tuner.py:227-338``. Device-side failures
(any ``JouleTuneError`` that is not a ``ConfigurationError``) come back as
failed results, so a search can rank and keep them; configuration errors are
caller mistakes and propagate.

Energy rules (``MeasurementSetup.mode``):

* ``instant`` — median power over the measurement window x runtime. The
  window is ``[0, runtime]`` for a simulated trace (reference) and the
  steady-state part of the device-timed loop for a real trace
  (``Execution.window``): a 0.1-3 ms kernel gets at most one NVML sample in
  ``[0, runtime]``, so the reference window would fail every config.
* ``averaged`` — last completed averaged-sensor window x runtime.
* ``counter`` (new, when an :class:`NVMLObserver` is attached and neither of
  the above) — NVML energy-counter slope over the steady window x runtime.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Mapping, Sequence

from .hardware import CLOCK_PARAM, POWER_LIMIT_PARAM
from .errors import ConfigurationError, JouleTuneError, MeasurementError
from .observer_hooks import AveragedPowerObserver, BenchmarkObserver, InstantPowerObserver, NVMLObserver
from .records import CORE_FIELDS, BenchmarkResult, UserMetric
from .sensors import AveragedSensorConfig, TracePlayback, instant_energy, sensor_reading
from .spaces import KernelConfig

__all__ = ["MeasurementSetup", "benchmark"]


@dataclass(frozen=True)
class MeasurementSetup:
    observers: tuple[BenchmarkObserver, ...] = ()
    averaged: AveragedSensorConfig = field(default_factory=AveragedSensorConfig)

    def _has(self, kind) -> bool:
        return any(isinstance(o, kind) for o in self.observers)

    def mode(self) -> str:
        if self._has(InstantPowerObserver):
            return "instant"
        if self._has(AveragedPowerObserver):
            return "averaged"
        if self._has(NVMLObserver):
            return "counter"
        return "instant"

    def duration_hint(self) -> float:
        mode = self.mode()
        if mode == "averaged":
            return self.averaged.continuous_duration
        if mode == "counter":
            return max(o.duration for o in self.observers if isinstance(o, NVMLObserver))
        return 0.0


def benchmark(
    device,
    config: KernelConfig,
    observers: Sequence[BenchmarkObserver] = (),
    *,
    user_metrics: Sequence[UserMetric] = (),
    constants: Mapping[str, float] | None = None,
    averaged_cfg: AveragedSensorConfig | None = None,
) -> BenchmarkResult:
    """Measure one config; device-side failures become ``failed`` results."""
    setup = MeasurementSetup(tuple(observers), averaged_cfg or AveragedSensorConfig())
    try:
        return _measure(device, config, setup, user_metrics, constants or {})
    except ConfigurationError:
        raise  # caller mistake: failing every config silently would hide it
    except JouleTuneError as exc:
        return BenchmarkResult(
            config=config,
            time=math.inf,
            energy=math.inf,
            failed=True,
            failure_reason=f"{type(exc).__name__}: {exc}",
        )


def _overrides_during(observer: BenchmarkObserver) -> bool:
    return type(observer).during is not BenchmarkObserver.during


def _measure(device, config, setup: MeasurementSetup, user_metrics, constants) -> BenchmarkResult:
    if CLOCK_PARAM in config:
        device.set_core_clock(config[CLOCK_PARAM])
    if POWER_LIMIT_PARAM in config:
        device.set_power_limit(config[POWER_LIMIT_PARAM])
    # nvml_mem_clock is accepted and ignored (B200 exposes a single memory clock).

    mode = setup.mode()
    observers = setup.observers
    for o in observers:
        o.before_start()
    run = device.execute(config, duration_hint=setup.duration_hint())
    playback = TracePlayback(run)
    for o in observers:
        o.after_start(playback)
    stepping = [o for o in observers if _overrides_during(o)]
    if stepping:
        meters = [o for o in observers if isinstance(o, InstantPowerObserver)]
        dt = 1.0 / (meters[0].cfg.sample_rate if meters else device.sample_rate_hz)
        while playback.advance(dt):
            for o in observers:
                o.during(playback)
    else:
        playback.now = run.total_duration
    for o in observers:
        o.after_finish(playback)

    readings: dict[str, float] = {}
    for o in observers:
        for key, value in o.get_results().items():
            if key in CORE_FIELDS or key in readings:
                raise ConfigurationError(f"observer result key collision: {key!r}")
            readings[key] = value

    runtime = run.runtime
    if mode == "averaged":
        watts = sensor_reading(run, run.total_duration, setup.averaged)
    elif mode == "counter":
        if run.counter_power is None:
            raise MeasurementError("device reported no energy-counter reading")
        watts = run.counter_power
    else:
        t0, t1 = run.window if run.window is not None else (0.0, runtime)
        watts = instant_energy(run.samples, t0, t1) / (t1 - t0)
    energy = watts * runtime

    env: dict[str, float] = {"time": runtime, "energy": energy, **readings, **constants}
    derived: dict[str, float] = {}
    for metric in user_metrics:
        derived[metric.name] = env[metric.name] = metric.evaluate(env)
    return BenchmarkResult(config=config, time=runtime, energy=energy, observer_results=readings, metrics=derived)


