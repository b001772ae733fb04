"""Where a 20-launch timed region loses time against a 1 s loop (bench.py headline, conv2d tuned config).

After the same warm-up + synchronize as bench.py, times K launches three ways on the same
stream with CUDA events: (a) the bench's Python loop of pre-packed native launches over 4 rotating
sets; (b) libjt's C loop (jt_time) on one set; (c) (a) with K = 200 and 2000. Prints per-launch ms.

    python scripts/short_loop_probe.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import Conv2DProblem  # noqa: E402


def main():
    with GPU(0) as gpu:
        prob = Conv2DProblem()
        cfg = tuned.best_config("conv2d", "time_optimal")
        prob.prepare(gpu)
        k = prob.kernel(cfg)
        prob.bind(k, cfg)
        launch = prob.launch(cfg)
        sets = [prob.args(cfg)]
        for _ in range(3):
            img = gpu.array(prob.inputs["image"], slack=64)
            out = gpu.empty((prob.height, prob.width), np.float32)
            sets.append([out, img])
        prepared = [gpu.prepare_launch(k, launch, s) for s in sets]
        gpu.reserve_events(3)
        res = {}
        for trial in range(3):
            for steps in (20, 200, 2000):
                for i in range(5):
                    gpu.launch_prepared(prepared[i % 4])
                gpu.synchronize()
                gpu.record(0)
                for i in range(steps):
                    gpu.launch_prepared(prepared[i % 4])
                gpu.record(1)
                res.setdefault(f"python_loop_{steps}", []).append(gpu.elapsed(0, 1) / steps * 1e3)
                gpu.synchronize()
            for i in range(5):
                gpu.launch_prepared(prepared[i % 4])
            gpu.synchronize()
            res.setdefault("c_loop_20_one_set", []).append(gpu.time(k, launch, sets[0], reps=20) / 20 * 1e3)
            # back to back: the second 20-launch region follows the first with no idle gap
            gpu.record(0)
            for i in range(20):
                gpu.launch_prepared(prepared[i % 4])
            gpu.record(1)
            for i in range(20):
                gpu.launch_prepared(prepared[i % 4])
            gpu.record(2)
            res.setdefault("python_loop_20_after_idle", []).append(gpu.elapsed(0, 1) / 20 * 1e3)
            res.setdefault("python_loop_20_after_busy", []).append(gpu.elapsed(1, 2) / 20 * 1e3)
            gpu.synchronize()
        # with the bench's NVML sampler running: ungated vs gated 20-launch regions
        gpu.sampler_start(1000, 1 << 20)
        for trial in range(5):
            for gated in (False, True):
                for i in range(5):
                    gpu.launch_prepared(prepared[i % 4])
                gpu.synchronize()
                if gated:
                    gpu.gate()
                gpu.record(0)
                for i in range(20):
                    gpu.launch_prepared(prepared[i % 4])
                gpu.record(1)
                if gated:
                    gpu.release()
                key = "sampler_on_20_gated" if gated else "sampler_on_20"
                res.setdefault(key, []).append(gpu.elapsed(0, 1) / 20 * 1e3)
                gpu.synchronize()
        gpu.sampler_stop(1 << 20)
        print(json.dumps({k: [round(v, 5) for v in vs] for k, vs in res.items()}), flush=True)


if __name__ == "__main__":
    main()
