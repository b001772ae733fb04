"""Raw NVML trace around a sweep-like sequence of loops (B200): how do the energy counter and the
instant-power field follow short loads?

One continuous libjt sampler (1 ms) runs while the script idles, then runs device-timed
loops back to back the way a tuning sweep does (0.3 s loops of different configs, a
short idle gap, a slow config, and a 1.5 s loop), so the counter's update cadence, its
driver timestamps and its lag behind the load, and the instant field's lag, can be read
off against the known loop intervals.

    python scripts/energy_probe.py      # -> gpurun_out/energy_probe.json
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def main() -> None:
    with GPU(0) as gpu:
        conv = make_problem("conv2d")
        conv.prepare(gpu)
        sg = make_problem("sgemm")
        sg.prepare(gpu)
        runs = {}
        for name, prob, cfg in (
            ("conv_tuned", conv, tuned.best_config("conv2d")),
            ("conv_small", conv, {**conv.default_config(), "block_size_x": 16, "block_size_y": 2, "tile_size_x": 1,
                                  "tile_size_y": 1}),
            ("sgemm_tuned", sg, tuned.best_config("sgemm")),
        ):
            k = prob.kernel(cfg)
            prob.bind(k, cfg)
            runs[name] = (k, prob.launch(cfg), prob.args(cfg))
        plan = [("idle", 0.6), ("conv_tuned", 0.3), ("sgemm_tuned", 0.3), ("conv_small", 0.3), ("conv_tuned", 0.3),
                ("idle", 0.25), ("sgemm_tuned", 0.3), ("conv_small", 0.3), ("idle", 0.05), ("conv_tuned", 0.3),
                ("sgemm_tuned", 1.5), ("idle", 0.5), ("conv_small", 1.5), ("idle", 0.6)]
        marks = []
        gpu.sampler_start(period_us=1000)
        for name, dur in plan:
            if name == "idle":
                t0 = gpu.sample()[0]
                time.sleep(dur)
                marks.append({"what": "idle", "t0": t0, "t1": gpu.sample()[0]})
                continue
            k, lau, args = runs[name]
            run = gpu.bench(k, lau, args, min_seconds=dur, sample=False)
            marks.append({"what": name, "t0": run.loop_t0, "t1": run.loop_t0 + run.total_s,
                          "per_launch_ms": run.per_launch_s * 1e3, "reps": run.reps})
        samples = gpu.sampler_stop()
    out = {"fields": ["t", "p_inst", "p_avg", "energy_j", "energy_stamp", "sm_mhz", "mem_mhz", "temp_c", "reasons"],
           "marks": marks, "samples": samples}
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/energy_probe.json").write_text(json.dumps(out))
    print(json.dumps(marks, indent=0)[:3000])
    print(len(samples), "samples")


if __name__ == "__main__":
    main()
