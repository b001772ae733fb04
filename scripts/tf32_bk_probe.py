"""TF32 persistent CTA-pair kernel: k-rows per pipeline stage (BK 32 / 64) around the tuned config.

Fewer, larger TMA boxes and half the mbarrier round trips per flop at BK 64 (the operand bytes
per flop are unchanged: DESIGN.md §4, "What feeds the TF32 tensor cores"). Each variant is first
checked against the fp64 oracle at 512 x 512 x 512, then timed at 4096^3 in a 20-launch burst and
a 1 s loop (2 rotating input sets, NVML clock and counter power). One JSON line per variant.

    python scripts/tf32_bk_probe.py check BK STAGES     # small-shape oracle check (run under `timeout`)
    python scripts/tf32_bk_probe.py time BK STAGES      # full-size timing
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402  (checker only)
from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def config(prob, bk, stages):
    return {**prob.default_config(), **tuned.best_config("sgemm_tf32", "time_optimal"), "BK": bk, "STAGES": stages}


def main():
    mode, bk, stages = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    with GPU(0) as gpu:
        if mode == "check":
            prob = make_problem("sgemm_tf32", m=512, n=512, k=512)
            prob.prepare(gpu)
            cfg = config(prob, bk, stages)
            k = prob.kernel(cfg)
            prob.bind(k, cfg)
            prob.reset_output()
            gpu.launch(k, prob.launch(cfg), prob.args(cfg))
            gpu.synchronize()
            ref = O.sgemm(prob.inputs["a"], prob.inputs["b"], prob.inputs["c0"], prob.alpha, prob.beta)
            err = O.sgemm_error(prob.fetch_output(), ref)
            print(json.dumps({"mode": "check", "BK": bk, "STAGES": stages, "err": float(err), "ok": bool(err <= 5e-3)}),
                  flush=True)
            return
        prob = make_problem("sgemm_tf32")
        prob.prepare(gpu)
        cfg = config(prob, bk, stages)
        k = prob.kernel(cfg)
        prob.bind(k, cfg)
        prob.reset_output()
        gpu.launch(k, prob.launch(cfg), prob.args(cfg))
        gpu.synchronize()
        ref = O.sgemm(prob.inputs["a"], prob.inputs["b"], prob.inputs["c0"], prob.alpha, prob.beta)
        err = O.sgemm_error(prob.fetch_output(), ref)
        gpu.time(k, prob.launch(cfg), prob.args(cfg), reps=5)
        burst = gpu.time(k, prob.launch(cfg), prob.args(cfg), reps=20) / 20
        from bench import summarize_samples

        rot = prob.rotation_sets(cfg, 2)
        r = gpu.bench(k, prob.launch(cfg), prob.args(cfg), min_seconds=1.0, rotate=rot)
        s = summarize_samples(r.samples, r.loop_t0 + 0.25, r.loop_t1)
        f = prob.total_flops
        print(json.dumps({"mode": "time", "BK": bk, "STAGES": stages, "err": float(err), "regs": k.regs,
                          "burst_ms": round(burst * 1e3, 4), "burst_tflops": round(f / burst / 1e12, 1),
                          "loop_ms": round(r.per_launch_s * 1e3, 4), "loop_tflops": round(f / r.per_launch_s / 1e12, 1),
                          "sm_mhz": s["sm_mhz"], "power_w": s["counter_w"],
                          "gflops_per_w": round(f / r.per_launch_s / 1e9 / s["counter_w"], 1) if s["counter_w"] else None}),
              flush=True)


if __name__ == "__main__":
    main()
