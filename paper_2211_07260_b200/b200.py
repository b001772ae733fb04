"""The real device: a B200 behind libjt, drop-in for ``SimulatedDevice``.

``B200Device`` implements the duck-typed device interface the tuner,
observers and CLI call (reference ``device.py:246-382``) for
one bound :class:`~.kernels.KernelProblem` — the way Kernel Tuner's
``tune_kernel`` binds one kernel source to a device:

* ``set_core_clock(MHz)`` — ``DomainError`` if not an NVML-supported clock;
  otherwise locks the SM clock with ``nvmlDeviceSetGpuLockedClocks`` (else
  applications clocks; no-op if unchanged, settle wait only on a real
  change). If NVML refuses, :class:`ControlRefusedError` is raised — the
  tuner records a failed result with NVML's reason — except for the default
  clock with no lock active, which is the driver-managed state itself
  (results carry ``nvml_clock_locked=0`` and the observed clock).
* ``set_power_limit(W)`` — range-checked ``nvmlDeviceSetPowerManagementLimit``,
  read back; refused → :class:`ControlRefusedError`.
* ``execute(config, duration_hint)`` — compile (NVRTC, cached) and load the
  config's module, run one probe launch and then a CUDA-event-timed
  back-to-back loop of >= max(duration_hint, min_window) seconds while the
  NVML sampler thread in libjt records instant power, the energy counter, SM
  clock, temperature and clock-event reasons. The returned
  :class:`~.device.Execution` has ``runtime`` = loop time / reps, a power
  trace re-based to the loop start, ``window`` = the steady part of the loop,
  ``counter_power`` = energy-counter slope over that window and
  ``effective_clock`` = median observed SM clock.
* ``read_voltage`` — ``CapabilityError`` (B200 exposes no core voltage).

All controller changes are undone by :meth:`close` (and by libjt at exit).
"""

from __future__ import annotations

import math
import statistics
import time
from dataclasses import replace
from typing import Any, Callable, Mapping

import numpy as np

from .hardware import EXECUTION_PARAMS, DeviceSpec, DeviceState, Execution, PowerSample
from .errors import CapabilityError, ControlRefusedError, DomainError
from .gpu import ENERGY, E_STAMP, GPU, MEM_MHZ, P_AVG, P_INST, REASONS, SM_MHZ, SW_POWER_CAP, TEMP, T
from .kernels import KernelProblem, make_problem
from .spaces import KernelConfig, normalize_value

__all__ = ["B200Device", "counter_power", "counter_slope", "steady_window", "NVML_AVERAGE_WINDOW_S"]

#: The B200 energy counter (nvmlDeviceGetTotalEnergyConsumption) accumulates in fixed periods:
#: every change adds the energy of one period, while the host-observed change times and the
#: driver's field timestamps jitter by +-20-40 ms around it (profiles/r2_energy_probe.json:
#: increments of 74-78 J at ~750 W, 25 J idle, 50 J at ~505 W; 72 changes over 7.20 s).
COUNTER_PERIOD_S = 0.1
#: allowance between the end of a counter period and the change's stamp
COUNTER_LAG_S = 0.015

#: nvmlDeviceGetPowerUsage on Ampere and newer (incl. B200) reports power averaged over 1 s
NVML_AVERAGE_WINDOW_S = 1.0


def steady_window(total: float, settle: float) -> tuple[float, float]:
    """Skip the first ``settle`` s (power ramp), but keep >= half the loop."""
    skip = min(settle, 0.5 * total)
    return (skip, total)


def counter_updates(samples, t0: float, t1: float) -> int:
    """Distinct energy-counter readings (change points) stamped inside [t0, t1]."""
    n, last_e = 0, None
    for s in samples:
        e = s[ENERGY]
        if not math.isfinite(e) or e == last_e:
            continue
        last_e = e
        t = s[E_STAMP] if math.isfinite(s[E_STAMP]) else s[T]
        n += t0 <= t <= t1
    return n


def _change_points(samples) -> list[tuple[float, float]]:
    """(time, energy) of every energy-counter change, in order. The time is the driver's field
    timestamp when present: an NVML call can stall for hundreds of ms (profiles/
    r2_energy_probe2.json: a reading requested at +0.069 s came back stamped +0.617 s), so the
    host time at which a sample was requested can lie far before the value it returned."""
    pts, last_e = [], None
    for s in samples:
        e = s[ENERGY]
        if math.isfinite(e) and e != last_e:
            pts.append((s[E_STAMP] if math.isfinite(s[E_STAMP]) else s[T], e))
            last_e = e
    return pts


def counter_power(samples, t0: float, t1: float) -> tuple[float | None, int]:
    """Energy-counter power (W) over [t0, t1] and the number of counter periods it used.

    The counter adds one fixed period's energy per change (``COUNTER_PERIOD_S``), but the
    times at which changes are seen jitter by a large fraction of the period, so a slope
    dE / dt over two or three changes scatters by tens of percent (a 0.3 s loop: +37% on
    one config in the r2 probe). Instead: sum the increments whose whole period lies inside
    the window (the change stamped t covers about [t - period, t]) and divide by their
    number of periods. Every change carries one period, however far from its neighbours it
    is stamped (the probe saw gaps of 45-141 ms, each with one period's energy), unless the
    gap exceeds 1.75 periods (changes the sampler did not see: a stalled NVML call returns
    several periods at once). The period is the median change interval of the trace when it
    holds enough changes."""
    pts = _change_points(samples)
    if len(pts) < 2:
        return None, 0
    gaps = [b[0] - a[0] for a, b in zip(pts, pts[1:])]
    period = statistics.median(gaps) if len(gaps) >= 8 else COUNTER_PERIOD_S
    if not 0.5 * COUNTER_PERIOD_S <= period <= 2.0 * COUNTER_PERIOD_S:
        period = COUNTER_PERIOD_S
    energy, periods = 0.0, 0
    for (ta, ea), (tb, eb) in zip(pts, pts[1:]):
        gap = (tb - ta) / period
        k = round(gap) if gap > 1.75 else 1
        if tb - k * period >= t0 + COUNTER_LAG_S and tb <= t1:
            energy += eb - ea
            periods += k
    if periods == 0:
        return None, 0
    return energy / (periods * period), periods


def counter_slope(samples, t0: float, t1: float) -> float | None:
    """Energy-counter power (W) over [t0, t1] from (time, energy) samples.

    The counter updates in steps (cadence is device specific), so the slope
    is taken between the first and last *change points* inside the window,
    stamped with the driver's own field timestamp when available. Returns
    None when fewer than two distinct readings fall in the window.
    """
    pts = []
    last_e = None
    for s in samples:
        e = s[ENERGY]
        if not math.isfinite(e):
            continue
        t = s[E_STAMP] if math.isfinite(s[E_STAMP]) else s[T]
        if e != last_e:
            pts.append((t, e))
            last_e = e
    inside = [(t, e) for t, e in pts if t0 <= t <= t1]
    if len(inside) < 2:
        return None
    (ta, ea), (tb, eb) = inside[0], inside[-1]
    if tb - ta <= 0:
        return None
    return (eb - ea) / (tb - ta)


class B200Device:
    """One CUDA ordinal + one bound kernel problem (see module docstring)."""

    def __init__(
        self,
        problem: KernelProblem | str = "conv2d",
        ordinal: int = 0,
        *,
        gpu: GPU | None = None,
        min_window: float = 0.25,
        settle: float = 0.02,
        clock_settle: float = 0.05,
        sample_period_us: int = 1000,
        answer: np.ndarray | None = None,
        verify: Callable[[np.ndarray, np.ndarray, Mapping[str, Any]], bool] | None = None,
        problem_kwargs: Mapping[str, Any] | None = None,
    ):
        self.problem = make_problem(problem, **(problem_kwargs or {})) if isinstance(problem, str) else problem
        self.gpu = gpu if gpu is not None else GPU(ordinal)
        self._owns_gpu = gpu is None
        self.min_window = float(min_window)
        self.settle = float(settle)
        #: re-runs of a loop whose NVML trace held no whole counter period, or whose counter and
        #: instant-power estimates disagree by more than ``disagree`` (see ``execute``)
        self.max_stale_retries = 2
        self.disagree = 0.15
        self.clock_settle = float(clock_settle)
        self.sample_period_us = int(sample_period_us)
        self.sample_rate_hz = 1e6 / self.sample_period_us
        self.answer = answer
        self.verify = verify
        self.execution_count = 0
        self.clock_locked: bool | None = None  # None = never requested
        #: "locked" (nvmlDeviceSetGpuLockedClocks), "application" (applications
        #: clocks), "refused" (observed clocks recorded instead) or None (untried)
        self.clock_mode: str | None = None
        self.last_observed_clock: float | None = None
        self.spec = self._probe_spec()
        self.state = DeviceState(self.spec.base_clock, self.spec.power_limit_range[1])
        self._requested_clock: float | None = None
        self._requested_limit: float | None = None
        #: which knob holds a clock lock right now ("locked" / "application" / None)
        self._lock_kind: str | None = None
        #: every refused controller request: {"knob", "requested", "reason", ...}
        self.refusals: list[dict] = []
        if self.problem.gpu is not self.gpu:
            self.problem.prepare(self.gpu)

    # -- construction helpers ---------------------------------------------
    def _probe_spec(self) -> DeviceSpec:
        info = self.gpu.info
        clocks = self.gpu.supported_clocks()
        if len(clocks) < 2:
            raise CapabilityError(f"NVML reports no supported SM clocks for {self.gpu.name}")
        peak = max(clocks)
        base_req = info.default_sm_clock_mhz or peak
        base = min(clocks, key=lambda c: (abs(c - base_req), -c))
        lo = info.power_limit_min_mw / 1000.0 or 100.0
        hi = info.power_limit_max_mw / 1000.0 or 1000.0
        tdp = max(info.power_limit_default_mw / 1000.0, hi)
        if not 0 < lo < hi:
            lo, hi = 0.5 * hi, hi
        return DeviceSpec(
            name=f"{self.gpu.name} (cuda:{self.gpu.ordinal}, {info.pci_bus_id.decode()})",
            supported_core_clocks=tuple(float(c) for c in clocks),
            base_clock=float(base),
            peak_clock=float(peak),
            power_limit_range=(lo, hi),
            tdp=tdp,
            voltage_readable=False,
        )

    @classmethod
    def from_document(cls, data: Mapping[str, Any]) -> "B200Device":
        """``{"kind": "b200", "kernel": "conv2d", "ordinal": 0, ...}`` device files."""
        extra = {k: data[k] for k in ("min_window", "settle", "clock_settle", "sample_period_us") if k in data}
        return cls(data.get("kernel", "conv2d"), int(data.get("ordinal", 0)),
                   problem_kwargs=data.get("problem", {}), **extra)

    def close(self) -> None:
        try:
            self._reset_clock()
            if self._requested_limit is not None:
                self.gpu.reset_power_limit()
        finally:
            self._requested_clock = None
            self._requested_limit = None
            if self._owns_gpu:
                self.gpu.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- controller -----------------------------------------------------------
    def set_core_clock(self, clock: float) -> DeviceState:
        """Lock the SM clock (reference ``device.py:277-284``).

        A refused lock raises :class:`ControlRefusedError` (a failed result in
        ``benchmark``), except for a request for the default clock while no
        lock is active: that is the driver-managed state the board is already
        in, measured with ``nvml_clock_locked = 0`` and the observed clock.
        Every refusal is kept in ``refusals`` with NVML's own text.
        """
        if clock not in self.spec.supported_core_clocks:
            raise DomainError(
                f"{clock} MHz is not supported on {self.spec.name}; supported: {list(self.spec.supported_core_clocks)}"
            )
        clock = float(clock)
        if self._requested_clock != clock:
            if self._apply_clock(int(clock)):
                self.clock_locked = True
                self._requested_clock = clock
                time.sleep(self.clock_settle)
            elif clock == self.spec.base_clock and self._lock_kind is None:
                self.clock_locked = False
                self._requested_clock = clock
            else:
                reason = self.gpu.last_refusal or "refused"
                self.refusals.append({"knob": "core_clock", "requested": clock, "reason": reason,
                                      "active_lock_mhz": self._requested_clock if self._lock_kind else None})
                raise ControlRefusedError("core_clock", clock, reason)
        self.state = replace(self.state, core_clock=clock)
        return self.state

    def _apply_clock(self, mhz: int) -> bool:
        """Locked clocks, else applications clocks; False if NVML refuses both.

        ``_lock_kind`` remembers which knob holds the board now, independently
        of later refusals, so :meth:`release_clock` / :meth:`close` always
        undo a lock that is still active."""
        if self.clock_mode in (None, "locked", "refused") and self._lock_kind in (None, "locked"):
            if self.gpu.lock_clocks(mhz, mhz):
                self.clock_mode = self._lock_kind = "locked"
                return True
        if self.clock_mode in (None, "application", "refused") and self._lock_kind in (None, "application"):
            if self.gpu.set_app_clocks(int(self.gpu.info.mem_clock_mhz), mhz):
                self.clock_mode = self._lock_kind = "application"
                return True
        if self._lock_kind is None:
            self.clock_mode = "refused"
        return False

    def release_clock(self) -> None:
        """Back to driver-managed clocks (e.g. before an untuned measurement)."""
        if self._requested_clock is not None:
            locked = self._lock_kind is not None
            self._reset_clock()
            self._requested_clock = None
            self.clock_locked = None
            if locked:
                time.sleep(self.clock_settle)

    def _reset_clock(self) -> None:
        if self._lock_kind == "locked":
            self.gpu.reset_clocks()
        elif self._lock_kind == "application":
            self.gpu.reset_app_clocks()
        self._lock_kind = None

    def set_power_limit(self, watts: float) -> DeviceState:
        """Board power limit (reference ``device.py:286-293``).

        NVML refusing the change raises :class:`ControlRefusedError` unless the
        limit already in force equals the request; an accepted change is read
        back and must be the enforced limit."""
        lo, hi = self.spec.power_limit_range
        if not lo <= watts <= hi:
            raise DomainError(f"power limit {watts} W outside [{lo}, {hi}] W on {self.spec.name}")
        watts = float(watts)
        if self._requested_limit != watts:
            if self.gpu.set_power_limit(watts):
                self._requested_limit = watts
                time.sleep(self.clock_settle)
                enforced = self.gpu.enforced_power_limit_w()
                if abs(enforced - watts) > 1.0:
                    reason = f"NVML accepted the limit but enforces {enforced:g} W"
                    self.refusals.append({"knob": "power_limit", "requested": watts, "reason": reason})
                    raise ControlRefusedError("power_limit", watts, reason)
            elif abs(self.gpu.enforced_power_limit_w() - watts) <= 1.0:
                pass  # already the limit in force: nothing to change
            else:
                reason = self.gpu.last_refusal or "refused"
                self.refusals.append({"knob": "power_limit", "requested": watts, "reason": reason})
                raise ControlRefusedError("power_limit", watts, reason)
        self.state = replace(self.state, power_limit=watts)
        return self.state

    def effective_clock(self, requested: float | None = None, *, utilization: float = 1.0) -> float:
        if self.last_observed_clock is not None:
            return self.last_observed_clock
        return self.state.core_clock if requested is None else requested

    def read_voltage(self, clock: float) -> float:
        raise CapabilityError(f"{self.spec.name} does not expose core voltage through NVML")

    # -- execution ----------------------------------------------------------------
    def kernel_view(self, config: KernelConfig) -> KernelConfig:
        return config.drop(*EXECUTION_PARAMS)

    def _compiled(self, config: KernelConfig):
        kernel_cfg = self.kernel_view(config).normalized().as_dict()
        defaults = self.problem.default_config()
        merged = {**defaults, **kernel_cfg} if kernel_cfg.keys() <= defaults.keys() else kernel_cfg
        kernel = self.problem.kernel(merged)
        launch = self.problem.launch(merged)
        if launch.threads > 1024:
            raise DomainError(f"{launch.threads} threads per block exceed the 1024 limit")
        return merged, kernel, launch

    def probe_runtime(self, config: KernelConfig) -> float:
        merged, kernel, launch = self._compiled(config)
        self.problem.bind(kernel, merged)
        args = self.problem.args(merged)
        self.gpu.time(kernel, launch, args, reps=1)  # warm-up
        return self.gpu.time(kernel, launch, args, reps=1)

    def execute(self, config: KernelConfig, duration_hint: float = 0.0) -> Execution:
        merged, kernel, launch = self._compiled(config)
        self.problem.bind(kernel, merged)
        args = self.problem.args(merged)
        if self.answer is not None:
            self.problem.reset_output()
        retries = 0
        while True:
            run = self.gpu.bench(
                kernel,
                launch,
                args,
                min_seconds=max(float(duration_hint), self.min_window),
                sample_period_us=self.sample_period_us,
            )
            self.execution_count += 1
            # A loop spanning >= 2.5 counter periods without one whole counter period inside its
            # steady window carries no energy information (NVML stalled: a reading requested
            # early in the loop returned after it, and the instant field then lags too): run it
            # again, at most twice.
            # The same goes for a loop whose counter power and instant-power median disagree by
            # more than DISAGREE (one bad counter increment among two, or an instant field still
            # showing the previous config): the re-run follows a loop of the same config, so a
            # lagging instant field has caught up and a bad increment is not repeated.
            w0, w1 = steady_window(run.total_s, self.settle)
            t0, t1 = run.loop_t0 + w0, run.loop_t0 + w1
            watts = counter_power(run.samples, t0, t1)[0]
            inst = [smp[P_INST] for smp in run.samples if t0 <= smp[T] <= t1 and math.isfinite(smp[P_INST])]
            disagree = bool(watts and inst) and abs(watts / statistics.median(inst) - 1.0) > self.disagree
            stale = run.total_s >= 2.5 * COUNTER_PERIOD_S and (watts is None or disagree)
            if not stale or retries == self.max_stale_retries:
                break
            retries += 1
        if self.answer is not None:
            self._check_answer(merged)
        ex = self._execution(run)
        ex.telemetry["stale_retries"] = float(retries)
        ex.telemetry["power_disagree"] = 1.0 if disagree else 0.0
        return ex

    def _check_answer(self, config) -> None:
        got = self.problem.fetch_output()
        if self.verify is not None:
            ok = self.verify(got, self.answer, config)
        else:
            ok = np.array_equal(got, self.answer)
        if not ok:
            raise DomainError(f"output of {self.problem.name} config {config} does not match the answer")

    def _execution(self, run) -> Execution:
        total = run.total_s
        t0 = run.loop_t0
        trace: list[PowerSample] = []
        before = [s for s in run.samples if s[T] < t0]
        during = [s for s in run.samples if t0 <= s[T] <= t0 + total]
        after = [s for s in run.samples if s[T] > t0 + total]
        if before and math.isfinite(before[-1][P_INST]):
            trace.append(PowerSample(0.0, before[-1][P_INST]))
        for s in during:
            if math.isfinite(s[P_INST]):
                trace.append(PowerSample(s[T] - t0, s[P_INST]))
        if after and math.isfinite(after[0][P_INST]):
            trace.append(PowerSample(total, after[0][P_INST]))
        window = steady_window(total, self.settle)
        steady = [s for s in during if window[0] <= s[T] - t0 <= window[1]] or during or run.samples
        slope, updates = counter_power(run.samples, t0 + window[0], t0 + window[1])
        source = 1.0  # whole energy-counter periods inside the steady window
        if slope is None:
            # no whole counter period after the settle: whole periods anywhere in the loop
            slope, updates = counter_power(run.samples, t0, t0 + total)
            source = 0.5
        if slope is None:
            # a loop shorter than one counter period: median instant power over the steady window
            inst = [s[P_INST] for s in steady if math.isfinite(s[P_INST])]
            slope = float(statistics.median(inst)) if inst else None
            source = 0.0
        clocks = [s[SM_MHZ] for s in steady if s[SM_MHZ]]
        observed = float(statistics.median(clocks)) if clocks else float(self.state.core_clock)
        self.last_observed_clock = observed
        reasons = 0
        for s in steady:
            reasons |= int(s[REASONS])
        telemetry = {
            "sm_clock": observed,
            "mem_clock": float(statistics.median([s[MEM_MHZ] for s in steady])) if steady else math.nan,
            "temperature": float(statistics.median([s[TEMP] for s in steady])) if steady else math.nan,
            "clock_locked": 1.0 if self.clock_locked else 0.0,
            "throttle_reasons": float(reasons),
            "power_capped": 1.0 if reasons & SW_POWER_CAP else 0.0,
            "reps": float(run.reps),
            "energy_source": source,
            "counter_updates": float(updates),
        }
        # NVML's own 1 s average as the board reported it during the loop (averaged-sensor mode)
        sensor = tuple(PowerSample(s[T] - t0, s[P_AVG]) for s in during if math.isfinite(s[P_AVG]))
        return Execution(
            runtime=run.per_launch_s,
            samples=tuple(trace),
            effective_clock=observed,
            repetitions=run.reps,
            total_duration=total,
            window=window,
            counter_energy=None if slope is None else slope * total,
            counter_power=slope,
            telemetry=telemetry,
            sensor_samples=sensor or None,
            sensor_window=NVML_AVERAGE_WINDOW_S,
        )

    # -- helpers for workflows ---------------------------------------------------
    def clock_grid(self, step_mhz: float | None = None, lo: float | None = None) -> list[int]:
        """Supported clocks, optionally thinned to >= step_mhz apart and >= lo."""
        grid = [int(normalize_value(c)) for c in self.spec.supported_core_clocks]
        if lo is not None:
            grid = [c for c in grid if c >= lo]
        if step_mhz:
            thinned = [grid[-1]]
            for c in reversed(grid[:-1]):
                if thinned[-1] - c >= step_mhz:
                    thinned.append(c)
            grid = sorted(thinned)
        return grid
