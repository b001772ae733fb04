"""Brute-force PnPoly ASM 7: occupancy sweep via MIN_BLOCKS (register cap), full size, bit-exact check."""
import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import native  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import PnPolyProblem  # noqa: E402

gpu = GPU(0)
p = PnPolyProblem()
p.prepare(gpu)
want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 3)
peak_slots = gpu.sm_count * 128 * 1965e6
for b, t, mb in itertools.product((128, 192, 256, 384), (4, 6, 8), (1, 4, 5, 6, 8)):
    cfg = dict(block_size_x=b, tile=t, vec=2, method=2, between=0, poly_smem=1, asm=7, persist=0)
    if mb * b > 2048:
        continue
    defs = {**p.defines(cfg), "MIN_BLOCKS": mb}
    try:
        cub = native.compile_cubin(native.kernel_source(p.source), p.name, native._nvrtc_options(defs))
    except Exception as e:  # noqa: BLE001
        print(cfg, mb, "compile failed", str(e)[:80])
        continue
    k = gpu.load(cub, p.symbol)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    ok = np.array_equal(p.fetch_output(), want)
    dt = gpu.time(k, p.launch(cfg), p.args(cfg), reps=10) / 10
    print(f"block {b} tile {t} minb {mb} regs {k.regs} local {k.local_bytes} ok={ok} {dt * 1e3:.3f} ms "
          f"frac={p.total_flops / dt / peak_slots:.3f}", flush=True)
