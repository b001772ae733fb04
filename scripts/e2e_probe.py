"""Wall time of the pipelined host-buffer conv2d / pnpoly calls vs strip count (pinned host arrays)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_07260_b200 import suite, tuned  # noqa: E402
from paper_2211_07260_b200.kernels import Conv2DProblem, PnPolyProblem  # noqa: E402


def sweep(label, call, flops, counts, reps=20):
    for strips in counts:
        for _ in range(3):
            call(strips)
        t0 = time.perf_counter()
        for _ in range(reps):
            call(strips)
        dt = (time.perf_counter() - t0) / reps
        print(f"{label} strips={strips:3d} {dt * 1e3:7.3f} ms  {flops / dt / 1e9:8.1f} G/s", flush=True)


p = Conv2DProblem()
inp = p.host_inputs()
img = suite.pinned(inp["image"].shape)
img[...] = inp["image"]
out = suite.pinned((p.height, p.width))
cfg = tuned.best_config("conv2d")
sweep("conv2d", lambda s: suite.conv2d(img, inp["filter"], out=out, config=cfg, strips=s), p.total_flops,
      (1, 2, 3, 4, 5, 6, 8, 10, 12, 16))
q = PnPolyProblem()
pin = q.host_inputs()
pts = suite.pinned(pin["points"].shape)
pts[...] = pin["points"]
res = suite.pinned((q.n_points,), np.int32)
qcfg = tuned.best_config("pnpoly")
sweep("pnpoly", lambda s: suite.pnpoly(pts, pin["vx"], pin["vy"], out=res, config=qcfg, strips=s), q.total_flops,
      (1, 2, 3, 4, 6, 8, 12), reps=8)
