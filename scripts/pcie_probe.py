"""PCIe copy probe: H2D alone, D2H alone, both on separate streams (pinned host memory)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_07260_b200.gpu import GPU, rows  # noqa: E402

MB = 1 << 20
gpu = GPU(0)
n = 64 * MB // 4
src = gpu.pinned((n,), np.float32)
dst = gpu.pinned((n,), np.float32)
src[...] = 1.0
da = gpu.empty((n,), np.float32)
db = gpu.empty((n,), np.float32)
gpu.reserve_streams(3)


def timed(fn, reps=10):
    fn()
    gpu.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    gpu.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    gpu.use_stream(1)
    gpu.h2d_async(da, src)
    gpu.use_stream(0)


def d2h():
    gpu.use_stream(2)
    gpu.d2h_async(dst, db)
    gpu.use_stream(0)


def both():
    h2d()
    d2h()


def chunked(k):
    def run():
        step = n // k
        for i in range(k):
            gpu.use_stream(1)
            gpu.h2d_async(rows(da, i * step, (i + 1) * step), src[i * step:(i + 1) * step])
            gpu.use_stream(2)
            gpu.d2h_async(dst[i * step:(i + 1) * step], rows(db, i * step, (i + 1) * step))
        gpu.use_stream(0)
    return run


for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both), ("chunked16", chunked(16)), ("chunked64", chunked(64))]:
    t = timed(fn)
    print(f"{name:10s} {t * 1e3:7.3f} ms  {64 * MB / t / 1e9:6.1f} GB/s per direction", flush=True)
