"""Full-size PnPoly slab-kernel timing over its whole tuning space (device-timed, L2-cold
inputs: 20 M points = 160 MB > L2) + bit-exact check against the brute-force oracle."""
import json
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

gpu = GPU(0)
# usage: time_slab.py [--grid | --cells] [key=value ...]  (--grid: pnpoly_grid.cu, --cells: pnpoly_cells.cu)
grid_mode = "--grid" in sys.argv
cells_mode = "--cells" in sys.argv
sys.argv = [a for a in sys.argv if a not in ("--grid", "--cells")]
p = make_problem("pnpoly_cells" if cells_mode else "pnpoly_grid" if grid_mode else "pnpoly_slab")
p.prepare(gpu)
want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)
configs = [c.as_dict() for c in p.space().enumerate()]
if len(sys.argv) > 1:
    configs = [c for c in configs if all(str(c.get(k)) == v for k, v in (a.split("=") for a in sys.argv[1:]))]
with ThreadPoolExecutor(16) as pool:
    list(pool.map(p.cubin, configs))
hbm = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
rows = []
for cfg in configs:
    k = p.kernel(cfg)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    ok = bool(np.array_equal(p.fetch_output(), want))
    t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=20) / 20
    rows.append((t, cfg, ok))
    print(f"{cfg} ok={ok} {t * 1e6:.1f} us  hbm_frac={p.algorithmic_bytes / t / 1e9 / hbm:.3f} "
          f"regs={k.regs}", flush=True)
rows.sort(key=lambda r: r[0])
print("BEST", [(round(t * 1e6, 1), c, ok) for t, c, ok in rows[:8]])
print("useful edge tests per point", p.useful_edge_tests() / p.n_points)
if grid_mode or cells_mode:
    print("clean fraction", {g: round(p.clean_fraction(g), 4) for g in (256, 512)})
