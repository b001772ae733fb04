"""Device-facing value types shared by the simulated and the real device.

Reference: ``pkg/src/jouletune/device.py:38-138``. The execution parameters
(``nvml_gr_clock``, ``nvml_mem_clock``, ``nvml_pwr_limit``) are ordinary
tunables that the benchmark applies to the device instead of passing to the
kernel. The duck-typed device interface the tuner, observers and CLI call is
listed in SURVEY §8(b): ``spec``, ``state``, ``sample_rate_hz``,
``execution_count``, ``set_core_clock``, ``set_power_limit``,
``effective_clock``, ``read_voltage``, ``kernel_view``, ``execute`` and (new
here) ``probe_runtime``. Implementations: :class:`.simulator.SimulatedDevice`
(deterministic test backend) and :class:`.b200.B200Device` (the GPU).
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
    """What a device can do: clock grid, clock anchors, power-limit range."""

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
        if len(grid) < 2 or list(grid) != sorted(set(grid)):
            raise ConfigurationError(f"{self.name}: supported clocks must be a sorted set of >= 2 values")
        if self.base_clock not in grid or self.peak_clock not in grid:
            raise ConfigurationError(f"{self.name}: base and peak clock must be supported clocks")
        if self.base_clock > self.peak_clock:
            raise ConfigurationError(f"{self.name}: base clock above peak clock")
        lo, hi = self.power_limit_range
        if not 0 < lo < hi:
            raise ConfigurationError(f"{self.name}: bad power limit range {lo}..{hi}")
        if hi > self.tdp:
            raise ConfigurationError(f"{self.name}: power limit range exceeds TDP {self.tdp}")


@dataclass(frozen=True)
class DeviceState:
    core_clock: float
    power_limit: float


@dataclass(frozen=True)
class PowerSample:
    timestamp: float
    power: float


@dataclass(frozen=True)
class Execution:
    """One measured execution (possibly a back-to-back repetition loop).

    The first five fields are the reference's (``device.py:130-138``).
    The B200 backend fills the optional tail:

    * ``window`` — ``(t0, t1)`` of the steady-state part of the loop inside
      the trace; energy rules that the reference evaluates over
      ``[0, runtime]`` use this window instead when present;
    * ``counter_energy`` — energy-counter delta over the whole loop (J);
    * ``counter_power`` — counter slope over the steady window (W);
    * ``telemetry`` — medians of SM clock, temperature etc. over the window.
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


