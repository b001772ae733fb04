"""Full-size PnPoly timing of selected configs (device-timed loops) + bit-exact check."""
import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import PnPolyProblem  # noqa: E402

gpu = GPU(0)
p = PnPolyProblem()
p.prepare(gpu)
want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 3)
# usage: time_pnpoly.py [ASMS [TILES [BLOCKS]]]   e.g.  time_pnpoly.py 3,7 4,8 128,256,512
lists = [[int(v) for v in a.split(",")] for a in sys.argv[1:4]]
asms, tiles, blocks = lists + [[3, 7], [4, 8], [128, 256, 512]][len(lists):]
configs = [dict(block_size_x=b, tile=t, vec=2, method=2, between=0, poly_smem=int(a != 8), asm=a, persist=ps)
           for a, b, t, ps in itertools.product(asms, blocks, tiles, (0, 1))]
peak_slots = gpu.sm_count * 128 * 1965e6
for cfg in configs:
    k = p.kernel(cfg)
    p.bind(k, cfg)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    ok = np.array_equal(p.fetch_output(), want)
    t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=20) / 20
    print(f"{cfg} ok={ok} {t * 1e3:.3f} ms  frac(3-op, 1965 MHz)={p.total_flops / t / peak_slots:.3f}", flush=True)
