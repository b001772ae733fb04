"""Memory floor of the pnpoly_cells loop: the same kernel compiled with -DPROBE_FLOOR=1 (the
cell lookup replaced by px < py, nothing queued), -DPROBE_FLOOR=2 (the lookups, nothing
queued) and -DPROBE_FLOOR=3 (lookups and queue pushes, drained points dropped) next to the
real one, device-timed on the
20 M-point input (160 MB read, 80 MB written per launch).

    python scripts/cells_floor.py [key=value ...]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_07260_b200 import native  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

gpu = GPU(0)
p = make_problem("pnpoly_cells")
p.prepare(gpu)
hbm = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
base = p.default_config()
variants = [dict(base, **dict(a.split("=") for a in sys.argv[1:]))] if len(sys.argv) > 1 else [
    dict(base, block_size_x=b, tile=t, regpf=0, prefetch=f) for b in (256, 512, 1024) for t in (1, 2, 4)
    for f in (0, 1, 2) if p.is_valid(dict(base, block_size_x=b, tile=t, regpf=0, prefetch=f))]
for cfg in variants:
    cfg = {k: int(v) for k, v in cfg.items()}
    for probe in (0, 1, 2, 3):
        opts = native._nvrtc_options({**p.defines(cfg), "PROBE_FLOOR": probe})
        k = gpu.load(native.compile_cubin(native.kernel_source(p.source), p.name, opts), p.symbol)
        t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=50) / 50
        print(json.dumps({"config": cfg, "probe_floor": probe, "us": round(t * 1e6, 2),
                          "hbm_frac": round(p.algorithmic_bytes / t / 1e9 / hbm, 3)}), flush=True)
