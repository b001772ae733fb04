"""Device-facing value types shared by the simulated and the real device.

Execution parameters (``nvml_gr_clock``, ``nvml_mem_clock``,
``nvml_pwr_limit``) are ordinary tunables that the benchmark applies to the
device instead of passing to the kernel (reference
``pkg/src/jouletune/device.py:38-41``).

The duck-typed device interface the engine, observers and CLI call
(SURVEY §8(b)): ``spec``, ``state``, ``sample_rate_hz``, ``execution_count``,
``set_core_clock``, ``set_power_limit``, ``effective_clock``,
``read_voltage``, ``kernel_view``, ``execute`` and (new) ``probe_runtime``.
Implementations: :class:`.simulator.SimulatedDevice` (deterministic test
backend) and :class:`.b200.B200Device` (the GPU).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping

from .errors import ConfigurationError

CLOCK_PARAM = "nvml_gr_clock"
MEM_CLOCK_PARAM = "nvml_mem_clock"
POWER_LIMIT_PARAM = "nvml_pwr_limit"
EXECUTION_PARAMS = (CLOCK_PARAM, MEM_CLOCK_PARAM, POWER_LIMIT_PARAM)

__all__ = ["CLOCK_PARAM", "MEM_CLOCK_PARAM", "POWER_LIMIT_PARAM", "EXECUTION_PARAMS", "DeviceSpec", "DeviceState",
           "PowerSample", "Execution"]


@dataclass(frozen=True)
class DeviceSpec:
    """Capabilities: clock grid (MHz, ascending, floats), anchors, power-limit range (W)."""

    name: str
    supported_core_clocks: tuple[float, ...]
    base_clock: float
    peak_clock: float
    power_limit_range: tuple[float, float]
    tdp: float
    voltage_readable: bool = False

    def __post_init__(self):
        grid = tuple(float(c) for c in self.supported_core_clocks)
        object.__setattr__(self, "supported_core_clocks", grid)
        object.__setattr__(self, "power_limit_range", tuple(self.power_limit_range))
        lo, hi = self.power_limit_range
        checks = (
            (len(grid) >= 2 and list(grid) == sorted(set(grid)), "supported clocks must be a sorted set of >= 2 values"),
            (self.base_clock in grid and self.peak_clock in grid, "base and peak clock must be supported clocks"),
            (self.base_clock <= self.peak_clock, "base clock above peak clock"),
            (0 < lo < hi, f"bad power limit range {lo}..{hi}"),
            (hi <= self.tdp, f"power limit range exceeds TDP {self.tdp}"),
        )
        for ok, problem in checks:
            if not ok:
                raise ConfigurationError(f"{self.name}: {problem}")


@dataclass(frozen=True)
class DeviceState:
    core_clock: float
    power_limit: float


@dataclass(frozen=True)
class PowerSample:
    timestamp: float  # s since the start of the execution
    power: float  # W


@dataclass(frozen=True)
class Execution:
    """One measured execution (possibly a back-to-back repetition loop).

    The first five fields are the reference's (``device.py:130-138``):
    per-execution runtime (s), the power trace, the granted clock, the
    repetition count and the traced duration. The real device fills the
    optional tail:

    * ``window`` — ``(t0, t1)`` steady-state part of the loop inside the
      trace; energy rules the reference evaluates over ``[0, runtime]`` use
      this window when present;
    * ``counter_energy`` / ``counter_power`` — NVML energy-counter delta over
      the loop (J) and its slope over the steady window (W);
    * ``telemetry`` — medians of SM / memory clock, temperature and the
      controller / throttle status over the window;
    * ``sensor_samples`` / ``sensor_window`` — the board's own averaged
      power sensor as it reported during the loop (NVML's 1 s average on
      B200) and its averaging window (s). When present, the averaged-sensor
      rules read this sensor instead of re-averaging the instant trace
      (``sensors.sensor_reading``).
    """

    runtime: float
    samples: tuple[PowerSample, ...]
    effective_clock: float
    repetitions: int
    total_duration: float
    window: tuple[float, float] | None = None
    counter_energy: float | None = None
    counter_power: float | None = None
    telemetry: Mapping[str, float] | None = None
    sensor_samples: tuple[PowerSample, ...] | None = None
    sensor_window: float | None = None
