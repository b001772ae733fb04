"""Pin the CPU oracles against implementations that share no code or op order with them.

The reference has no kernel code, so kernel parity cannot be
pinned to reference outputs; test_oracle.py pins the oracles against their own
restatements and committed fixtures. These tests add checks that are
independent of both:

* conv2d: scipy.signal.correlate2d (a third-party 'valid' correlation) — the
  Kernel Tuner convolution (output[y][x] = sum_j sum_i in[y+j][x+i] * f[j][i]);
* sgemm: scipy's BLAS dgemm wrapper, called directly;
* PnPoly: the crossing-number test evaluated in float64, where every step but
  the one division and one addition is exact for float32 inputs, so its answer
  is the exact geometric one except for points within ~1e-15 of a crossing.
  The float32 oracle (every formulation, and the PnPoly kernels bit for bit)
  may differ from it only at points whose distance to a crossing is within
  float32 rounding of the crossing's x coordinate — checked point by point.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import kernels_oracle as O
from paper_2211_07260_b200.kernels import PnPolyProblem

scipy_signal = pytest.importorskip("scipy.signal")
scipy_blas = pytest.importorskip("scipy.linalg.blas")


def test_conv_oracle_equals_scipy_correlate2d():
    rng = np.random.default_rng(11)
    img = rng.uniform(0, 1, (83, 71)).astype(np.float32)
    f = rng.uniform(0, 1, (17, 17)).astype(np.float32)
    ref = O.conv2d(img, f)
    sp = scipy_signal.correlate2d(img.astype(np.float64), f.astype(np.float64), mode="valid")
    assert ref.shape == sp.shape == (83 - 16, 71 - 16)
    np.testing.assert_allclose(ref, sp, rtol=1e-12, atol=0)


def test_sgemm_oracle_equals_scipy_dgemm():
    rng = np.random.default_rng(12)
    a, b, c = rng.uniform(-1, 1, (64, 48)), rng.uniform(-1, 1, (48, 40)), rng.uniform(-1, 1, (64, 40))
    ref = O.sgemm(a, b, c, 1.0, 0.5)
    d = scipy_blas.dgemm(1.0, a, b, beta=0.5, c=c.copy())
    np.testing.assert_allclose(ref, d, rtol=1e-13, atol=1e-13)


def crossing_float64(points: np.ndarray, vx: np.ndarray, vy: np.ndarray, chunk: int = 8192):
    """Crossing-number point-in-polygon in float64 (W. R. Franklin's test, the paper's PnPoly),
    plus each point's smallest |px - x_crossing| over the edges whose y-test passes."""
    px = points[:, 0].astype(np.float64)
    py = points[:, 1].astype(np.float64)
    xi, yi = vx.astype(np.float64), vy.astype(np.float64)
    xj, yj = np.roll(xi, 1), np.roll(yi, 1)  # edge k joins vertex k-1 -> k, as in the kernels
    inside = np.zeros(len(px), bool)
    margin = np.full(len(px), np.inf)
    for s in range(0, len(px), chunk):
        X, Y = px[s:s + chunk, None], py[s:s + chunk, None]
        ycond = (yi > Y) != (yj > Y)
        with np.errstate(divide="ignore", invalid="ignore"):
            # (xj - xi), (Y - yi) exact in float64 for float32 data; their product exact (48 bits)
            xc = (xj - xi) * (Y - yi) / (yj - yi) + xi
        cross = ycond & (X < xc)
        inside[s:s + chunk] = (np.count_nonzero(cross, axis=1) & 1).astype(bool)
        dist = np.where(ycond, np.abs(X - xc), np.inf)
        margin[s:s + chunk] = dist.min(axis=1)
    return inside.astype(np.int32), margin


@pytest.mark.parametrize("method", [0, 1, 2, 3])
def test_pnpoly_oracle_is_the_geometric_crossing_test(method):
    inp = PnPolyProblem(n_points=120_000, seed=21).host_inputs()
    pts, vx, vy = inp["points"], inp["vx"], inp["vy"]
    exact, margin = crossing_float64(pts, vx, vy)
    got = O.pnpoly(pts, vx, vy, method)
    assert 0.2 < exact.mean() < 0.45
    bad = np.flatnonzero(got != exact)
    # every disagreement sits within float32 rounding of a crossing (|x| <= ~1 here: a few ulps)
    scale = float(np.abs(vx).max())
    assert np.all(margin[bad] <= 8 * np.finfo(np.float32).eps * scale), (method, bad[:10], margin[bad][:10])
    assert len(bad) <= 3, (method, len(bad))


def test_pnpoly_geometric_test_on_points_near_edges():
    """Points placed ON the polygon's edges (worst case): disagreements with the float64 test
    are confined to points whose crossing margin is within float32 rounding."""
    inp = PnPolyProblem(n_points=1000, seed=22).host_inputs()
    vx, vy = inp["vx"], inp["vy"]
    rng = np.random.default_rng(5)
    k = rng.integers(0, len(vx), 20_000)
    t = rng.uniform(0, 1, 20_000)
    x = vx[k - 1] + t * (vx[k] - vx[k - 1])
    y = vy[k - 1] + t * (vy[k] - vy[k - 1])
    pts = np.stack([x, y], 1).astype(np.float32)
    exact, margin = crossing_float64(pts, vx, vy)
    scale = float(np.abs(vx).max())
    for method in range(4):
        got = O.pnpoly(pts, vx, vy, method)
        bad = np.flatnonzero(got != exact)
        assert np.all(margin[bad] <= 8 * np.finfo(np.float32).eps * scale), method
