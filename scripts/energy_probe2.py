"""Raw NVML trace over a sweep of 0.3 s loops (B200): what do the energy-counter changes look like in the
loops whose whole-period power reads about half the instant power? (round 2)

80 conv2d configs are measured back to back in 0.3 s loops exactly as tune_suite measures them
(jt_bench's own sampler around each loop); every loop's raw trace goes to gpurun_out/energy_probe2.json.

    python scripts/energy_probe2.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def main() -> None:
    with GPU(0) as gpu:
        conv = make_problem("conv2d")
        conv.prepare(gpu)
        configs = [c.as_dict() for c in conv.space().enumerate()][::25][:80]
        kernels = []
        for c in configs:
            cfg = {**conv.default_config(), **c}
            try:
                k = conv.kernel(cfg)
            except Exception:  # noqa: BLE001
                continue
            kernels.append((cfg, k))
        loops = []
        for cfg, k in kernels:  # the tuning path: jt_bench's own sampler around each loop
            conv.bind(k, cfg)
            run = gpu.bench(k, conv.launch(cfg), conv.args(cfg), min_seconds=0.3, sample=True)
            loops.append({"t0": run.loop_t0, "t1": run.loop_t0 + run.total_s, "per_launch_ms": run.per_launch_s * 1e3,
                          "samples": run.samples})
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/energy_probe2.json").write_text(json.dumps({"loops": loops}))
    print(len(loops), "loops")


if __name__ == "__main__":
    main()
