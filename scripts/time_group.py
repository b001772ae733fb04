"""GROUP_M (CTA / tile-walk rasterisation) sweep for the tuned SGEMM FP32 and TF32 configs.

    python scripts/time_group.py            # 1 s rotating loops: ms, TF/s per GROUP_M
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        python scripts/time_group.py --once  # one launch per config for DRAM bytes
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--groups", default="1,2,4,8,16")
    args = ap.parse_args()
    groups = [int(g) for g in args.groups.split(",")]
    out = []
    with GPU(0) as gpu:
        for name in ("sgemm", "sgemm_tf32"):
            p = make_problem(name)
            p.prepare(gpu)
            base = {**p.default_config(), **(tuned.best_config(name) or {})}
            for g in groups:
                if name == "sgemm_tf32" and g > 8:
                    continue
                cfg = {**base, "GROUP_M": g}
                k = p.kernel(cfg)
                if args.once:
                    for _ in range(2):
                        gpu.launch(k, p.launch(cfg), p.args(cfg))
                    gpu.synchronize()
                    print(name, g, flush=True)
                    continue
                run = gpu.bench(k, p.launch(cfg), p.args(cfg), min_seconds=1.0, rotate=p.rotation_sets(cfg, 2))
                rec = {"kernel": name, "GROUP_M": g, "ms": run.per_launch_s * 1e3,
                       "tflops": p.total_flops / run.per_launch_s / 1e12,
                       "sm_mhz": sorted(s[5] for s in run.samples)[len(run.samples) // 2] if run.samples else None}
                print(json.dumps(rec), flush=True)
                out.append(rec)
            for b in p.buffers.values():
                b.free()
    if out:
        Path("gpurun_out").mkdir(exist_ok=True)
        Path("gpurun_out/time_group.jsonl").write_text("\n".join(json.dumps(r) for r in out) + "\n")


if __name__ == "__main__":
    main()
