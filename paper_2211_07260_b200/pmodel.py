"""The load power model P*(f) and its Levenberg-Marquardt fit.

Model (paper eq. 1-2, ``PAPER.md:487-503``; reference
``pkg/src/jouletune/powermodel.py:37-384``)::

    P*(f) = min(p_max, p_idle + alpha * f * v(f)^2)
    v(f)  = v0                             f <  tau_ft
          = v0 * (1 + beta * (f - tau_ft)) f >= tau_ft

Fit procedure kept from the reference so that fitted parameters agree to
~1e-9 relative on identical samples:

* a trailing plateau of >= 3 samples within 2 % of the maximum power is the
  throttled region and defines ``p_max`` (else TDP, else max power);
* with voltages on every active sample: ridge = flat-to-rising transition
  (1 % of v_min), tau/beta from a line through the rising side, LM on
  (p_idle, alpha);
* without voltages: LM on (p_idle, alpha, tau_ft, beta) with v0 = 1, falling
  back to a linear fit with beta = 0 when no rise materialises;
* LM: damping 1e-3 (x10 on reject, /10 on accept, floor 1e-12, give-up at
  1e14), forward-difference Jacobian with step 1e-6 * max(|theta|, 1e-2),
  stop on relative cost change < 1e-9, at most 200 iterations.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .errors import ConfigurationError, FitError, UnderDeterminedError

__all__ = ["FrequencySample", "RidgePoint", "PowerModel", "detect_ridge", "fit"]

_N_PARAMS = 6  # p_idle, p_max, alpha, tau_ft, beta, v0
_RIDGE_REL = 0.01
_PLATEAU_REL = 0.02
_PLATEAU_MIN = 3


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
    p_idle: float
    p_max: float
    alpha: float
    tau_ft: float
    beta: float
    v0: float = 1.0
    residual_rms: float | None = None

    def __post_init__(self):
        if self.p_idle < 0 or self.alpha <= 0 or self.beta < 0 or self.v0 <= 0:
            raise ConfigurationError("power model needs p_idle >= 0, alpha > 0, beta >= 0, v0 > 0")
        if self.p_max <= self.p_idle:
            raise ConfigurationError("power model needs p_max > p_idle")

    def predict_voltage(self, frequency: float) -> float:
        if frequency < self.tau_ft:
            return self.v0
        return self.v0 * (1.0 + self.beta * (frequency - self.tau_ft))

    def predict_power(self, frequency: float, voltage: float | None = None) -> float:
        v = self.predict_voltage(frequency) if voltage is None else voltage
        return min(self.p_max, self.p_idle + self.alpha * frequency * v * v)

    def to_dict(self) -> dict:
        doc = {k: getattr(self, k) for k in ("p_idle", "p_max", "alpha", "tau_ft", "beta", "v0")}
        if self.residual_rms is not None:
            doc["residual_rms"] = self.residual_rms
        return doc

    @classmethod
    def from_dict(cls, data: dict) -> "PowerModel":
        try:
            return cls(**data)
        except TypeError as exc:
            raise ConfigurationError(f"bad model document: {exc}") from exc


def detect_ridge(samples: Sequence[FrequencySample], tolerance: float = _RIDGE_REL) -> RidgePoint | None:
    """Highest clock whose voltage (and every lower one's) stays within
    ``tolerance`` x v_min of v_min while the next one rises; None if flat."""
    if len(samples) < 4:
        raise ConfigurationError("ridge detection needs at least 4 samples")
    ordered = sorted(samples, key=lambda s: s.frequency)
    if any(s.voltage is None for s in ordered):
        raise ConfigurationError("ridge detection needs voltages on every sample")
    volts = [s.voltage for s in ordered]
    floor = min(volts)
    ceiling = floor + tolerance * floor
    flat_end = -1
    while flat_end + 1 < len(volts) and volts[flat_end + 1] <= ceiling:
        flat_end += 1
    if flat_end == len(ordered) - 1:
        return None
    rise = volts[flat_end + 1 :]
    if any(nxt < cur - tolerance * floor for cur, nxt in zip(rise, rise[1:])):
        warnings.warn("voltage is not monotone beyond the ridge; fit quality may suffer", stacklevel=2)
    anchor = ordered[flat_end]
    return RidgePoint(anchor.frequency, anchor.voltage)


def _split_throttled(samples: Sequence[FrequencySample]):
    """(active, plateau): plateau = trailing >= 3 samples within 2 % of max power."""
    ordered = sorted(samples, key=lambda s: s.frequency)
    cutoff = (1.0 - _PLATEAU_REL) * max(s.power for s in ordered)
    tail = 0
    for s in reversed(ordered):
        if s.power < cutoff:
            break
        tail += 1
    if _PLATEAU_MIN <= tail < len(ordered):
        split = len(ordered) - tail
        return ordered[:split], ordered[split:]
    return ordered, []


def _jacobian(residual: Callable[[np.ndarray], np.ndarray], theta: np.ndarray, r0: np.ndarray) -> np.ndarray:
    cols = []
    for j in range(theta.size):
        h = 1e-6 * max(abs(theta[j]), 1e-2)
        shifted = theta.copy()
        shifted[j] += h
        cols.append((residual(shifted) - r0) / h)
    return np.stack(cols, axis=1)


def _lm_solve(
    residual: Callable[[np.ndarray], np.ndarray],
    theta0: Sequence[float],
    *,
    max_iterations: int = 200,
    initial_damping: float = 1e-3,
    rel_tolerance: float = 1e-9,
) -> tuple[np.ndarray, float]:
    """Levenberg-Marquardt with Marquardt diagonal scaling; returns (theta, rms)."""
    theta = np.asarray(theta0, dtype=float)
    r = residual(theta)
    cost = float(r @ r)
    lam = initial_damping
    for _ in range(max_iterations):
        jac = _jacobian(residual, theta, r)
        jtj = jac.T @ jac
        grad = jac.T @ r
        diag = np.diag(np.maximum(np.diag(jtj), 1e-12))
        trial = None
        while lam < 1e14:
            try:
                delta = np.linalg.solve(jtj + lam * diag, -grad)
            except np.linalg.LinAlgError:
                lam *= 10.0
                continue
            candidate = theta + delta
            r_c = residual(candidate)
            cost_c = float(r_c @ r_c)
            if cost_c <= cost:
                trial = (candidate, r_c, cost_c)
                break
            lam *= 10.0
        if trial is None:  # no damping yields descent: stationary point
            return theta, math.sqrt(cost / r.size)
        rel_drop = abs(cost - trial[2]) / max(cost, 1e-300)
        theta, r, cost = trial
        lam = max(lam / 10.0, 1e-12)
        if rel_drop < rel_tolerance:
            return theta, math.sqrt(cost / r.size)
    raise FitError(f"no convergence after {max_iterations} iterations", theta=theta, residuals=r)


def fit(samples: Sequence[FrequencySample], *, tdp: float | None = None, max_iterations: int = 200) -> PowerModel:
    """Fit the load power model to a frequency sweep (see module docstring)."""
    if len(samples) < _N_PARAMS:
        raise UnderDeterminedError(f"{len(samples)} samples cannot determine {_N_PARAMS} model parameters")
    active, plateau = _split_throttled(samples)
    if len(active) < _N_PARAMS:
        raise UnderDeterminedError(
            f"only {len(active)} samples remain after excluding the throttled plateau; need at least {_N_PARAMS}"
        )
    if plateau:
        p_max = float(np.mean([s.power for s in plateau]))
    elif tdp is not None:
        p_max = float(tdp)
    else:
        p_max = max(s.power for s in samples)
    f = np.array([s.frequency for s in active])
    p = np.array([s.power for s in active])
    if all(s.voltage is not None for s in active):
        return _fit_measured_voltage(active, f, p, p_max, max_iterations)
    return _fit_inferred_voltage(f, p, p_max, max_iterations)


def _idle_guess(p: np.ndarray) -> float:
    return 0.9 * float(np.min(p))


def _slope_guess(f: np.ndarray, p: np.ndarray, mask: np.ndarray) -> float:
    """LSQ slope of power vs clock on ``mask`` (whole sweep if < 2 points)."""
    if int(np.count_nonzero(mask)) < 2:
        mask = np.ones_like(mask, dtype=bool)
    slope, _ = np.polyfit(f[mask], p[mask], 1)
    return max(float(slope), 1e-9)


def _fit_measured_voltage(active, f, p, p_max, max_iterations) -> PowerModel:
    v = np.array([s.voltage for s in active])
    ridge = detect_ridge(active)
    if ridge is None:
        warnings.warn("voltage is flat across the sweep; fixing beta to 0", stacklevel=3)
        v0, tau, beta = float(np.mean(v)), float(f[-1]), 0.0
    else:
        v0 = float(np.mean(v[f <= ridge.frequency]))
        rising = f > ridge.frequency
        if int(np.count_nonzero(rising)) >= 2:
            slope, intercept = np.polyfit(f[rising], v[rising], 1)
            beta = float(slope / v0)
            cross = (v0 - intercept) / slope if slope > 0 else ridge.frequency
            tau = float(min(max(cross, f[0]), f[-1]))
        else:
            tau = float(ridge.frequency)
            beta = (float(v[rising][0]) / v0 - 1.0) / (float(f[rising][0]) - tau)

    def residual(theta):
        return theta[0] + theta[1] * f * v**2 - p

    flat = f < (tau if ridge is not None else np.inf)
    theta, rms = _lm_solve(
        residual, [_idle_guess(p), _slope_guess(f, p, flat) / (v0 * v0)], max_iterations=max_iterations
    )
    idle, alpha = float(theta[0]), float(theta[1])
    return PowerModel(
        p_idle=max(idle, 0.0), p_max=max(p_max, idle + 1e-9), alpha=alpha, tau_ft=tau, beta=beta, v0=v0,
        residual_rms=rms,
    )


def _fit_inferred_voltage(f, p, p_max, max_iterations) -> PowerModel:
    def residual(theta):
        idle, alpha, tau, beta = theta
        v = np.where(f < tau, 1.0, 1.0 + beta * (f - tau))
        return idle + alpha * f * v * v - p

    start = [_idle_guess(p), _slope_guess(f, p, f <= np.median(f)), float(0.5 * (f[0] + f[-1])), 1e-3]
    theta, rms = _lm_solve(residual, start, max_iterations=max_iterations)
    idle, alpha, tau, beta = (float(x) for x in theta)
    if tau >= f[-1] or beta <= 0:
        warnings.warn("no voltage rise detected in the sweep; fixing beta to 0", stacklevel=3)
        alpha, idle = (float(c) for c in np.polyfit(f, p, 1))
        tau, beta = float(f[-1]), 0.0
        rms = float(np.sqrt(np.mean((idle + alpha * f - p) ** 2)))
    return PowerModel(
        p_idle=max(idle, 0.0), p_max=max(p_max, idle + 1e-9), alpha=alpha, tau_ft=tau, beta=max(beta, 0.0),
        v0=1.0, residual_rms=rms,
    )


