"""Sensor semantics over execution traces (the measurement rules).

Reference rules kept exactly (``pkg/src/jouletune/observers.py:35-204``):

* averaged sensor — trapezoid mean of the last refresh window completed at
  or before ``t``; windows are aligned at t = 0;
* instant sensor — median of the samples in ``[t0, t1]`` times ``t1 - t0``;
* continuous benchmark — repeat for ``continuous_duration``; energy is the
  final window reading times the loop duration;
* :class:`TracePlayback` steps a virtual clock through a recorded trace.
"""

from __future__ import annotations

import bisect
import math
import statistics
import warnings
from dataclasses import dataclass
from typing import Sequence

from .errors import ConfigurationError, MeasurementError, SensorNotReadyError
from .hardware import Execution, PowerSample
from .spaces import KernelConfig

__all__ = ["AveragedSensorConfig", "InstantSensorConfig", "averaged_reading", "sensor_reading", "instant_energy",
           "ContinuousResult", "continuous_benchmark", "TracePlayback"]


@dataclass(frozen=True)
class AveragedSensorConfig:
    refresh_rate: float = 10.0  # Hz
    continuous_duration: float = 1.0  # s

    def __post_init__(self):
        if self.refresh_rate <= 0 or self.continuous_duration <= 0:
            raise ConfigurationError("sensor rates and durations must be positive")


@dataclass(frozen=True)
class InstantSensorConfig:
    sample_rate: float = 2870.0  # Hz

    def __post_init__(self):
        if self.sample_rate <= 0:
            raise ConfigurationError("sensor rates and durations must be positive")


def _stamps(samples: Sequence[PowerSample]) -> list[float]:
    return [s.timestamp for s in samples]


def _value_at(samples: Sequence[PowerSample], stamps: Sequence[float], t: float) -> float:
    """Piecewise-linear trace value at t, clamped to the first/last sample."""
    if t <= stamps[0]:
        return samples[0].power
    if t >= stamps[-1]:
        return samples[-1].power
    hi = bisect.bisect_right(stamps, t)
    lo = hi - 1
    a, b = samples[lo], samples[hi]
    if a.timestamp == b.timestamp:
        return b.power
    return a.power + (t - a.timestamp) / (b.timestamp - a.timestamp) * (b.power - a.power)


def averaged_reading(
    samples: Sequence[PowerSample], t: float, cfg: AveragedSensorConfig | None = None
) -> float:
    """What the averaged sensor reports at time ``t`` (see module docstring)."""
    cfg = cfg or AveragedSensorConfig()
    if not samples:
        raise MeasurementError("empty trace")
    width = 1.0 / cfg.refresh_rate
    done = math.floor(t * cfg.refresh_rate + 1e-9)
    if done < 1:
        raise SensorNotReadyError(f"no completed {width:.3g}s window at t={t:.6g}s")
    end = done * width
    start = end - width
    first, last = samples[0].timestamp, samples[-1].timestamp
    if first > start + 1e-12 or last < end - 1e-12:
        raise MeasurementError(
            f"trace [{first:.6g}, {last:.6g}] does not cover window [{start:.6g}, {end:.6g}]"
        )
    stamps = _stamps(samples)
    # knots: window edges (interpolated) plus every sample strictly inside
    lo = bisect.bisect_right(stamps, start)
    hi = bisect.bisect_left(stamps, end)
    xs = [start] + stamps[lo:hi] + [end]
    ys = [_value_at(samples, stamps, start)] + [s.power for s in samples[lo:hi]] + [_value_at(samples, stamps, end)]
    area = 0.0
    for i in range(1, len(xs)):
        area += 0.5 * (ys[i] + ys[i - 1]) * (xs[i] - xs[i - 1])
    return area / width


def sensor_reading(execution: Execution, t: float, cfg: AveragedSensorConfig | None = None) -> float:
    """What the averaged sensor reports at ``t`` for one execution.

    Simulated traces: :func:`averaged_reading` over the instant trace (the
    reference rule, ``observers.py:81-107``). A real board with its own
    averaging sensor (``execution.sensor_samples``, NVML's 1 s average on
    B200): the value that sensor reported at or before ``t``. Its window is
    fixed by the hardware, so ``cfg.refresh_rate`` must be its inverse (1 Hz
    on B200) — anything else is a configuration error, not a silently
    different measurement — and nothing is ready before one full window.
    """
    cfg = cfg or AveragedSensorConfig()
    if execution.sensor_samples is None:
        return averaged_reading(execution.samples, t, cfg)
    width = float(execution.sensor_window or 1.0)
    if abs(1.0 / cfg.refresh_rate - width) > 1e-6 * width:
        raise ConfigurationError(
            f"this device's averaged sensor reports {width:g} s averages: refresh_rate must be {1.0 / width:g} Hz "
            f"(got {cfg.refresh_rate:g} Hz)")
    if t < width - 1e-9:
        raise SensorNotReadyError(f"no completed {width:.3g}s window at t={t:.6g}s")
    # the board's average covers (t_s - width, t_s]: only readings whose window lies inside the trace
    ready = [s for s in execution.sensor_samples if width - 1e-9 <= s.timestamp <= t + 1e-12 and math.isfinite(s.power)]
    if not ready:
        raise MeasurementError(f"the averaged sensor reported nothing in [{width:.3g}, {t:.6g}] s")
    return ready[-1].power


def instant_energy(samples: Sequence[PowerSample], t0: float, t1: float) -> float:
    """Median sample power inside [t0, t1] times the elapsed time."""
    if t0 >= t1:
        raise MeasurementError(f"inverted window: t0={t0} >= t1={t1}")
    inside = [s.power for s in samples if t0 <= s.timestamp <= t1]
    if not inside:
        raise MeasurementError(f"no samples in [{t0}, {t1}]")
    return statistics.median(inside) * (t1 - t0)


@dataclass(frozen=True)
class ContinuousResult:
    energy: float
    mean_power: float
    repetitions: int
    duration: float
    long_kernel: bool = False


def _single_runtime(device, config: KernelConfig) -> float:
    probe = getattr(device, "probe_runtime", None)
    if probe is not None:
        return probe(config)
    kernel = device.kernel_view(config)
    surface = device.surface
    return surface.runtime(kernel, device.effective_clock(utilization=surface.utilization(kernel)))


def continuous_benchmark(device, config: KernelConfig, cfg: AveragedSensorConfig | None = None) -> ContinuousResult:
    """Averaged-sensor benchmark of one config (see module docstring).

    The reference probes the runtime through the simulator-only ``surface``
    (``observers.py:150-153``); here any device exposing ``probe_runtime``
    works (the B200 backend times one launch with CUDA events).
    """
    cfg = cfg or AveragedSensorConfig()
    probe = _single_runtime(device, config)
    too_long = probe > 10.0 * cfg.continuous_duration
    if too_long:
        warnings.warn(
            f"kernel runtime {probe:.3g}s dwarfs the {cfg.continuous_duration:.3g}s "
            "benchmark duration; measuring a single execution",
            stacklevel=2,
        )
    run = device.execute(config, duration_hint=0.0 if too_long else cfg.continuous_duration)
    watts = sensor_reading(run, run.total_duration, cfg)
    return ContinuousResult(
        energy=watts * run.total_duration,
        mean_power=watts,
        repetitions=run.repetitions,
        duration=run.total_duration,
        long_kernel=too_long,
    )


class TracePlayback:
    """Steps a virtual clock through a recorded execution trace."""

    def __init__(self, execution: Execution):
        self.execution = execution
        self.now = 0.0
        self._stamps = _stamps(execution.samples)

    @property
    def runtime(self) -> float:
        return self.execution.runtime

    @property
    def total_duration(self) -> float:
        return self.execution.total_duration

    def advance(self, dt: float) -> bool:
        if self.now >= self.total_duration:
            return False
        self.now = min(self.now + dt, self.total_duration)
        return True

    def instant_power(self) -> float:
        return _value_at(self.execution.samples, self._stamps, self.now)

    def averaged_power(self, cfg: AveragedSensorConfig) -> float:
        return sensor_reading(self.execution, self.now, cfg)

    def final_averaged_power(self, cfg: AveragedSensorConfig) -> float:
        return sensor_reading(self.execution, self.total_duration, cfg)


