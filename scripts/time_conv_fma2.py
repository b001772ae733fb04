"""conv2d: packed FFMA2 (fma2=1) vs scalar on the tuned and nearby configs (device-timed,
4 rotating inputs > L2); checks the fma2 output is bit-identical to fma2=0."""
import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import Conv2DProblem  # noqa: E402

gpu = GPU(0)
p = Conv2DProblem()
p.prepare(gpu)
ref = O.conv2d(p.inputs["image"], p.inputs["filter"])
best = tuned.best_config("conv2d")
for bx, by, tx, ty, sm in itertools.product((32, 64), (4, 8), (4, 8), (1, 2, 4), (0, 1)):
    base = dict(best, block_size_x=bx, block_size_y=by, tile_size_x=tx, tile_size_y=ty, use_shmem=sm, use_padding=0)
    outs = {}
    for f2 in (0, 1):
        cfg = dict(base, fma2=f2)
        if not p.is_valid(cfg):
            continue
        k = p.kernel(cfg)
        p.bind(k, cfg)
        p.reset_output()
        gpu.launch(k, p.launch(cfg), p.args(cfg))
        gpu.synchronize()
        outs[f2] = p.fetch_output()
        err = O.conv2d_error(outs[f2], ref, p.inputs["image"], p.inputs["filter"])
        t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=50) / 50
        same = bool(np.array_equal(outs[f2].view(np.uint32), outs[0].view(np.uint32))) if 0 in outs else None
        print(f"{cfg} err={err:.1e} same_as_fma={same} regs={k.regs} {t * 1e6:.1f} us "
              f"{p.total_flops / t / 1e12:.2f} TF/s = {p.total_flops / t / 74.45e12:.3f}", flush=True)
