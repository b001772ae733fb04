"""Our tuned TF32 SGEMM at beta = 0.5 (the benchmark problem) and beta = 0 (C = A.B, what the cuBLAS
calibration times) in the same 1 s device-timed loops bench.py uses, with the NVML clock / power
record, so scripts/cublas_calibration.py's sustained TF32 number has a like-for-like counterpart.

    python scripts/tf32_vs_cublas.py        # then: python scripts/cublas_calibration.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import summarize_samples  # noqa: E402
from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def main():
    with GPU(0) as gpu:
        for beta in (0.5, 0.0):
            prob = make_problem("sgemm_tf32", beta=beta)
            prob.prepare(gpu)
            cfg = {**prob.default_config(), **tuned.best_config("sgemm_tf32", "time_optimal")}
            k = prob.kernel(cfg)
            prob.bind(k, cfg)
            rot = prob.rotation_sets(cfg, 2)
            gpu.bench(k, prob.launch(cfg), prob.args(cfg), min_seconds=0.3, rotate=rot)  # warm
            r = gpu.bench(k, prob.launch(cfg), prob.args(cfg), min_seconds=1.0, rotate=rot)
            s = summarize_samples(r.samples, r.loop_t0 + 0.25, r.loop_t1)
            ms = r.per_launch_s * 1e3
            print(json.dumps({"impl": "ours", "beta": beta, "config": cfg, "ms": round(ms, 4),
                              "tflops": round(prob.total_flops / r.per_launch_s / 1e12, 1),
                              "sm_mhz": s["sm_mhz"], "power_w": s["counter_w"], "reasons": s["reasons"]}),
                  flush=True)
            for b in prob.buffers.values():
                b.free()


if __name__ == "__main__":
    main()
