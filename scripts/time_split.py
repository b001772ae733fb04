"""SPLIT_TAIL (K-split of the last partial wave) x GROUP_M for the FP32 SGEMM at 4096^3, plus
nearby CTA shapes, against cuBLAS FP32 (torch.matmul with TF32 off) on the same box.

    python scripts/time_split.py     # 1 s rotating loops -> gpurun_out/time_split.jsonl
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402  (checker only)
from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU, fp32_peak_tflops  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def median_clock(run):
    return sorted(s[5] for s in run.samples)[len(run.samples) // 2] if run.samples else None


def main():
    out = []
    with GPU(0) as gpu:
        p = make_problem("sgemm", value_set="b200")
        p.prepare(gpu)
        ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
        base = {**p.default_config(), **(tuned.best_config("sgemm") or {})}
        variants = []
        for g in (1, 8, 16):
            for s in (0, 2, 4):
                variants.append({**base, "GROUP_M": g, "SPLIT_TAIL": s})
        # the same tile with other thread shapes / stage counts, split tail on
        for extra in ({"ASYNC": 3}, {"KWG": 32, "ASYNC": 3}, {"MDIMC": 8, "NDIMC": 16, "VWM": 4, "VWN": 2},
                      {"KWI": 2}):
            variants.append({**base, "GROUP_M": 8, "SPLIT_TAIL": 2, **extra})
        for cfg in variants:
            if not p.is_valid(cfg):
                print("invalid", cfg, flush=True)
                continue
            k = p.kernel(cfg)
            p.reset_output()
            gpu.launch(k, p.launch(cfg), p.args(cfg))
            gpu.synchronize()
            err = O.sgemm_error(p.fetch_output(), ref)
            run = gpu.bench(k, p.launch(cfg), p.args(cfg), min_seconds=1.0, rotate=p.rotation_sets(cfg, 2))
            mhz = median_clock(run)
            tf = p.total_flops / run.per_launch_s / 1e12
            rec = {"config": cfg, "plan": list(p.tail_plan(cfg)), "regs": k.regs,
                   "per_sm": k.occupancy(cfg["MDIMC"] * cfg["NDIMC"], p.smem_bytes(cfg)),
                   "ms": round(run.per_launch_s * 1e3, 4), "tflops": round(tf, 2), "sm_mhz": mhz,
                   "frac_fp32": round(tf / fp32_peak_tflops(gpu.sm_count, mhz or 1965.0), 4), "err": err,
                   "ok": err <= O.SGEMM_TOL}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    try:  # library calibration, not the product
        import torch

        torch.backends.cuda.matmul.allow_tf32 = False
        a = torch.rand(4096, 4096, device="cuda") * 2 - 1
        b = torch.rand(4096, 4096, device="cuda") * 2 - 1
        for _ in range(5):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(300):
            torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 300
        rec = {"cublas_fp32": True, "ms": round(ms, 4), "tflops": round(2 * 4096 ** 3 / ms / 1e9, 2),
               "frac_fp32_at_1965": round(2 * 4096 ** 3 / ms / 1e9 / fp32_peak_tflops(148, 1965.0), 4)}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    except Exception as exc:  # noqa: BLE001
        print("cublas calibration failed:", exc, flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/time_split.jsonl").write_text("\n".join(json.dumps(r) for r in out) + "\n")


if __name__ == "__main__":
    main()
