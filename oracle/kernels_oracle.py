"""TEST INFRASTRUCTURE ONLY — CPU oracles for the kernel suite.

May be imported only by tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs, as the checker or the timed CPU
baseline. The product (``paper_2211_07260_b200``) never imports it.

Parity status of kernel outputs: UNPINNED by the reference. The reference
package (``/root/reference/pkg/src/jouletune``) simulates kernels with a
``PerformanceSurface`` (``device.py:148-243``) and contains no SGEMM,
convolution or PnPoly code; the paper cites CLBlast's
GEMM (``PAPER.md:244, 309-316``) and Kernel Tuner's benchmarks. These
restatements are therefore the definition of correct output:

* ``sgemm`` — ``alpha * (A @ B) + beta * C0`` in float64 (numpy);
  the FP32 kernel must satisfy ``max|C - C64| / max|C64| <= 1e-5``.
* ``conv2d`` — direct float64 correlation (289 shifted multiply-adds);
  FP32 tolerance ``max|out - ref| / (sum|f| * max|x|) <= 1e-5``.
* ``pnpoly`` — float32 crossing number with a pinned op sequence per
  crossing formula (oracle/pnpoly_oracle.c, compiled with
  ``-ffp-contract=off``); the bitmap must match bit for bit. A pure-numpy
  restatement of formula 0 (``pnpoly_numpy``) cross-checks the C oracle.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
LIB = ORACLE_DIR / "_build" / "liboracle.so"

SGEMM_TOL = 1e-5
SGEMM_TF32_TOL = 5e-3
CONV_TOL = 1e-5


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    return LIB


_lib = None


def _liboracle():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        lib.pnpoly_oracle.restype = ctypes.c_int
        lib.pnpoly_oracle.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def pnpoly(points: np.ndarray, vx: np.ndarray, vy: np.ndarray, method: int = 0, threads: int | None = None):
    """int32 bitmap (1 = inside) for float32 points (n, 2) and vertices."""
    points = np.ascontiguousarray(points, dtype=np.float32)
    vx = np.ascontiguousarray(vx, dtype=np.float32)
    vy = np.ascontiguousarray(vy, dtype=np.float32)
    out = np.empty(points.shape[0], dtype=np.int32)
    rc = _liboracle().pnpoly_oracle(points.ctypes.data, points.shape[0], vx.ctypes.data, vy.ctypes.data, vx.size,
                                    int(method), out.ctypes.data, int(threads or host_threads()))
    if rc:
        raise RuntimeError(f"pnpoly_oracle failed ({rc})")
    return out


def pnpoly_numpy(points: np.ndarray, vx: np.ndarray, vy: np.ndarray) -> np.ndarray:
    """Formula 0 in numpy float32 (every op rounds to float32; numpy never contracts)."""
    px = points[:, 0].astype(np.float32)
    py = points[:, 1].astype(np.float32)
    inside = np.zeros(px.shape, dtype=bool)
    n = vx.size
    with np.errstate(divide="ignore", invalid="ignore"):
        for k in range(n):
            j = (k - 1) % n
            dx = np.float32(vx[j] - vx[k])
            dy = np.float32(vy[j] - vy[k])
            spans = (vy[k] > py) != (vy[j] > py)
            x = ((dx * (py - vy[k])) / dy + vx[k]).astype(np.float32)
            inside ^= spans & (px < x)
    return inside.astype(np.int32)


def conv2d(image: np.ndarray, filt: np.ndarray) -> np.ndarray:
    """Valid-mode correlation in float64: out[y, x] = sum_ij image[y+i, x+j] * f[i, j]."""
    fh, fw = filt.shape
    h, w = image.shape[0] - fh + 1, image.shape[1] - fw + 1
    img = image.astype(np.float64)
    f64 = filt.astype(np.float64)
    out = np.zeros((h, w), dtype=np.float64)
    for i in range(fh):
        for j in range(fw):
            out += f64[i, j] * img[i : i + h, j : j + w]
    return out


def conv2d_rows(image: np.ndarray, filt: np.ndarray, rows: slice) -> np.ndarray:
    """Same as conv2d for a band of output rows (bounded CPU samples)."""
    fh, _ = filt.shape
    r0, r1 = rows.start, rows.stop
    return conv2d(image[r0 : r1 + fh - 1], filt)


def conv2d_error(out: np.ndarray, ref: np.ndarray, image: np.ndarray, filt: np.ndarray) -> float:
    scale = float(np.abs(filt).sum(dtype=np.float64) * np.abs(image).max())
    return float(np.abs(out.astype(np.float64) - ref).max() / scale)


def sgemm(a: np.ndarray, b: np.ndarray, c0: np.ndarray, alpha: float, beta: float) -> np.ndarray:
    return alpha * (a.astype(np.float64) @ b.astype(np.float64)) + beta * c0.astype(np.float64)


def sgemm_error(c: np.ndarray, ref: np.ndarray) -> float:
    return float(np.abs(c.astype(np.float64) - ref).max() / np.abs(ref).max())
