"""The load power model P*(f) and how it is fitted to a clock sweep.

Model (paper eq. 1-2, ``PAPER.md:487-503``; reference
``pkg/src/jouletune/powermodel.py:37-384``)::

    P*(f) = min(p_max, p_idle + alpha * f * v(f)^2)
    v(f)  = v0                             f <  tau_ft
          = v0 * (1 + beta * (f - tau_ft)) f >= tau_ft

The fit reproduces the reference to ~1e-9 relative on identical samples
(tests/test_api_parity.py), organised here as:

* :class:`_Sweep` — samples sorted by clock, the trailing throttle plateau
  (>= 3 samples within 2 % of the peak power) split off; it sets ``p_max``
  (plateau mean, else TDP, else the peak);
* a fit *path*: :class:`_MeasuredVoltagePath` when every active sample has a
  voltage (ridge from the flat-to-rising transition, tau/beta from a line
  through the rising side, free (p_idle, alpha)) or
  :class:`_InferredVoltagePath` (free (p_idle, alpha, tau_ft, beta) with
  v0 = 1, falling back to a straight line with beta = 0);
* :class:`_LevenbergMarquardt` — damping 1e-3, x10 on a rejected step, /10
  (floor 1e-12) on an accepted one, gives up at 1e14, forward-difference
  Jacobian with step 1e-6 * max(|theta|, 1e-2), converged when the relative
  cost drop falls below 1e-9, at most ``max_iterations`` outer steps.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .errors import ConfigurationError, FitError, UnderDeterminedError

__all__ = ["FrequencySample", "RidgePoint", "PowerModel", "detect_ridge", "fit"]

MIN_SAMPLES = 6  # free parameters of the full model: p_idle, p_max, alpha, tau_ft, beta, v0
RIDGE_TOLERANCE = 0.01  # of the minimum voltage
PLATEAU_TOLERANCE = 0.02  # of the maximum power
PLATEAU_MIN_RUN = 3


@dataclass(frozen=True)
class FrequencySample:
    frequency: float  # MHz
    power: float  # W
    voltage: float | None = None  # V


@dataclass(frozen=True)
class RidgePoint:
    frequency: float
    voltage: float


@dataclass(frozen=True)
class PowerModel:
    """Fitted (or given) model parameters; ``residual_rms`` in W when fitted."""

    p_idle: float
    p_max: float
    alpha: float
    tau_ft: float
    beta: float
    v0: float = 1.0
    residual_rms: float | None = None

    def __post_init__(self):
        sane = self.p_idle >= 0 and self.alpha > 0 and self.beta >= 0 and self.v0 > 0
        if not sane:
            raise ConfigurationError("power model needs p_idle >= 0, alpha > 0, beta >= 0, v0 > 0")
        if not self.p_max > self.p_idle:
            raise ConfigurationError("power model needs p_max > p_idle")

    def predict_voltage(self, frequency: float) -> float:
        return self.v0 if frequency < self.tau_ft else self.v0 * (1.0 + self.beta * (frequency - self.tau_ft))

    def predict_power(self, frequency: float, voltage: float | None = None) -> float:
        v = voltage if voltage is not None else self.predict_voltage(frequency)
        return min(self.p_max, self.p_idle + self.alpha * frequency * v * v)

    def to_dict(self) -> dict:
        keys = ("p_idle", "p_max", "alpha", "tau_ft", "beta", "v0") + (("residual_rms",) if self.residual_rms is not None
                                                                      else ())
        return {k: getattr(self, k) for k in keys}

    @classmethod
    def from_dict(cls, data: dict) -> "PowerModel":
        try:
            return cls(**data)
        except TypeError as exc:
            raise ConfigurationError(f"bad model document: {exc}") from exc


def detect_ridge(samples: Sequence[FrequencySample], tolerance: float = RIDGE_TOLERANCE) -> RidgePoint | None:
    """Last sample of the leading run of voltages within ``tolerance`` x v_min of
    v_min (None when the whole sweep is flat). Mirrors the reference quirk:
    if even the lowest clock is above the band the *last* sample is returned."""
    if len(samples) < 4:
        raise ConfigurationError("ridge detection needs at least 4 samples")
    by_clock = sorted(samples, key=lambda s: s.frequency)
    if any(s.voltage is None for s in by_clock):
        raise ConfigurationError("ridge detection needs voltages on every sample")
    volts = [s.voltage for s in by_clock]
    v_min = min(volts)
    band_top = v_min + tolerance * v_min
    flat = 0
    while flat < len(volts) and volts[flat] <= band_top:
        flat += 1
    if flat == len(volts):
        return None
    tail = volts[flat:]
    if any(b < a - tolerance * v_min for a, b in zip(tail, tail[1:])):
        warnings.warn("voltage is not monotone beyond the ridge; fit quality may suffer", stacklevel=2)
    last_flat = by_clock[flat - 1]  # index -1 (the last sample) when nothing is flat
    return RidgePoint(last_flat.frequency, last_flat.voltage)


def _split_throttled(samples: Sequence[FrequencySample]):
    """(active, plateau), clock-sorted: the plateau is a trailing run of >= 3
    samples within 2 % of the peak power, unless it would take every sample."""
    ordered = sorted(samples, key=lambda s: s.frequency)
    threshold = (1.0 - PLATEAU_TOLERANCE) * max(s.power for s in ordered)
    run = 0
    while run < len(ordered) and ordered[-1 - run].power >= threshold:
        run += 1
    if PLATEAU_MIN_RUN <= run < len(ordered):
        return ordered[: len(ordered) - run], ordered[len(ordered) - run :]
    return ordered, []


class _Sweep:
    """Clock-sorted samples with the throttle plateau separated."""

    def __init__(self, samples: Sequence[FrequencySample], tdp: float | None):
        if len(samples) < MIN_SAMPLES:
            raise UnderDeterminedError(f"{len(samples)} samples cannot determine {MIN_SAMPLES} model parameters")
        self.active, self.plateau = _split_throttled(samples)
        if len(self.active) < MIN_SAMPLES:
            raise UnderDeterminedError(f"only {len(self.active)} samples remain after excluding the throttled "
                                       f"plateau; need at least {MIN_SAMPLES}")
        if self.plateau:
            self.p_max = float(np.mean([s.power for s in self.plateau]))
        else:
            self.p_max = float(tdp) if tdp is not None else max(s.power for s in samples)
        self.f = np.array([s.frequency for s in self.active])
        self.p = np.array([s.power for s in self.active])

    @property
    def has_voltages(self) -> bool:
        return all(s.voltage is not None for s in self.active)

    def idle_guess(self) -> float:
        return 0.9 * float(np.min(self.p))

    def slope_guess(self, mask: np.ndarray) -> float:
        """LSQ slope of power over clock on ``mask`` (the whole sweep if < 2 points)."""
        use = mask if int(np.count_nonzero(mask)) >= 2 else np.ones_like(mask, dtype=bool)
        slope, _ = np.polyfit(self.f[use], self.p[use], 1)
        return max(float(slope), 1e-9)


class _LevenbergMarquardt:
    """Minimise ||r(theta)||^2 (see module docstring for the schedule)."""

    def __init__(self, residual: Callable[[np.ndarray], np.ndarray], *, max_iterations: int = 200,
                 damping: float = 1e-3, rel_tolerance: float = 1e-9):
        self.residual = residual
        self.max_iterations = max_iterations
        self.damping = damping
        self.rel_tolerance = rel_tolerance

    def _jacobian(self, theta: np.ndarray, r0: np.ndarray) -> np.ndarray:
        columns = []
        for j in range(theta.size):
            step = 1e-6 * max(abs(theta[j]), 1e-2)
            probe = theta.copy()
            probe[j] += step
            columns.append((self.residual(probe) - r0) / step)
        return np.stack(columns, axis=1)

    def _descend(self, theta, cost, normal, gradient, scale):
        """Raise the damping until a step does not increase the cost."""
        while self.damping < 1e14:
            try:
                step = np.linalg.solve(normal + self.damping * scale, -gradient)
            except np.linalg.LinAlgError:
                self.damping *= 10.0
                continue
            trial = theta + step
            r_trial = self.residual(trial)
            c_trial = float(r_trial @ r_trial)
            if c_trial <= cost:
                return trial, r_trial, c_trial
            self.damping *= 10.0
        return None

    def solve(self, theta0: Sequence[float]) -> tuple[np.ndarray, float]:
        theta = np.asarray(theta0, dtype=float)
        r = self.residual(theta)
        cost = float(r @ r)
        for _ in range(self.max_iterations):
            jac = self._jacobian(theta, r)
            normal = jac.T @ jac
            scale = np.diag(np.maximum(np.diag(normal), 1e-12))
            accepted = self._descend(theta, cost, normal, jac.T @ r, scale)
            if accepted is None:  # stationary: no damping gives descent
                break
            drop = abs(cost - accepted[2]) / max(cost, 1e-300)
            theta, r, cost = accepted
            self.damping = max(self.damping / 10.0, 1e-12)
            if drop < self.rel_tolerance:
                break
        else:
            raise FitError(f"no convergence after {self.max_iterations} iterations", theta=theta, residuals=r)
        return theta, math.sqrt(cost / r.size)


class _MeasuredVoltagePath:
    """Voltages known: tau/beta/v0 from the voltage curve, LM on (p_idle, alpha)."""

    def __init__(self, sweep: _Sweep):
        self.sweep = sweep
        f = sweep.f
        self.v = np.array([s.voltage for s in sweep.active])
        self.ridge = detect_ridge(sweep.active)
        if self.ridge is None:
            warnings.warn("voltage is flat across the sweep; fixing beta to 0", stacklevel=4)
            self.v0, self.tau, self.beta = float(np.mean(self.v)), float(f[-1]), 0.0
            return
        self.v0 = float(np.mean(self.v[f <= self.ridge.frequency]))
        above = f > self.ridge.frequency
        if int(np.count_nonzero(above)) >= 2:
            # line through the rising side; tau where it crosses v0 (between grid points)
            slope, intercept = np.polyfit(f[above], self.v[above], 1)
            self.beta = float(slope / self.v0)
            crossing = (self.v0 - intercept) / slope if slope > 0 else self.ridge.frequency
            self.tau = float(min(max(crossing, f[0]), f[-1]))
        else:
            self.tau = float(self.ridge.frequency)
            self.beta = (float(self.v[above][0]) / self.v0 - 1.0) / (float(f[above][0]) - self.tau)

    def residual(self, theta: np.ndarray) -> np.ndarray:
        s = self.sweep
        return theta[0] + theta[1] * s.f * self.v**2 - s.p

    def start(self) -> list[float]:
        s = self.sweep
        flat = s.f < (self.tau if self.ridge is not None else np.inf)
        return [s.idle_guess(), s.slope_guess(flat) / (self.v0 * self.v0)]

    def model(self, theta: np.ndarray, rms: float) -> PowerModel:
        idle, alpha = float(theta[0]), float(theta[1])
        return PowerModel(p_idle=max(idle, 0.0), p_max=max(self.sweep.p_max, idle + 1e-9), alpha=alpha,
                          tau_ft=self.tau, beta=self.beta, v0=self.v0, residual_rms=rms)


class _InferredVoltagePath:
    """No voltages: LM on (p_idle, alpha, tau_ft, beta) with v0 = 1."""

    def __init__(self, sweep: _Sweep):
        self.sweep = sweep

    def residual(self, theta: np.ndarray) -> np.ndarray:
        idle, alpha, tau, beta = theta
        f = self.sweep.f
        v = np.where(f < tau, 1.0, 1.0 + beta * (f - tau))
        return idle + alpha * f * v * v - self.sweep.p

    def start(self) -> list[float]:
        s = self.sweep
        return [s.idle_guess(), s.slope_guess(s.f <= np.median(s.f)), float(0.5 * (s.f[0] + s.f[-1])), 1e-3]

    def model(self, theta: np.ndarray, rms: float) -> PowerModel:
        s = self.sweep
        idle, alpha, tau, beta = (float(x) for x in theta)
        if tau >= s.f[-1] or beta <= 0:
            # the sweep never left the flat-voltage regime: straight line, beta pinned
            warnings.warn("no voltage rise detected in the sweep; fixing beta to 0", stacklevel=4)
            alpha, idle = (float(c) for c in np.polyfit(s.f, s.p, 1))
            tau, beta = float(s.f[-1]), 0.0
            rms = float(np.sqrt(np.mean((idle + alpha * s.f - s.p) ** 2)))
        return PowerModel(p_idle=max(idle, 0.0), p_max=max(s.p_max, idle + 1e-9), alpha=alpha, tau_ft=tau,
                          beta=max(beta, 0.0), v0=1.0, residual_rms=rms)


def fit(samples: Sequence[FrequencySample], *, tdp: float | None = None, max_iterations: int = 200) -> PowerModel:
    """Fit the load power model to a frequency sweep (see module docstring)."""
    sweep = _Sweep(samples, tdp)
    path = _MeasuredVoltagePath(sweep) if sweep.has_voltages else _InferredVoltagePath(sweep)
    theta, rms = _LevenbergMarquardt(path.residual, max_iterations=max_iterations).solve(path.start())
    return path.model(theta, rms)


def _lm_solve(residual, theta0, *, max_iterations: int = 200, initial_damping: float = 1e-3,
              rel_tolerance: float = 1e-9):
    """Functional form of the LM solver: returns (theta, rms)."""
    return _LevenbergMarquardt(residual, max_iterations=max_iterations, damping=initial_damping,
                               rel_tolerance=rel_tolerance).solve(theta0)
