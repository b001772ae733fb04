"""Measure a list of kernel configs on one GPU: device time, GFLOP/s, correctness.

  python scripts/sweep.py --kernel pnpoly --configs '[{...}, ...]'
  python scripts/sweep.py --kernel sgemm --sample 200 --seed 1
  python scripts/sweep.py --kernel conv2d --all

Compiles every config with NVRTC on a host thread pool first, then runs each
as a device-timed back-to-back loop (no NVML sampling), verifies its output
against the CPU oracle (test infrastructure, used here only as the checker)
and writes gpurun_out/sweep_<kernel>.json sorted by time.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402  (checker only)
from paper_2211_07260_b200.errors import JouleTuneError  # noqa: E402
from paper_2211_07260_b200.gpu import GPU, fp32_peak_tflops  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def reference(problem):
    inp = problem.inputs
    if problem.name == "pnpoly":
        return {m: O.pnpoly(inp["points"], inp["vx"], inp["vy"], m) for m in (0, 1, 2, 3)}
    if problem.name == "conv2d":
        return O.conv2d(inp["image"], inp["filter"])
    if problem.name in ("sgemm", "sgemm_tf32"):
        return O.sgemm(inp["a"], inp["b"], inp["c0"], problem.alpha, problem.beta)
    return None


def check(problem, ref, cfg):
    out = problem.fetch_output()
    if problem.name == "pnpoly":
        bad = int((out != ref[problem.formula(cfg)]).sum())
        return bad == 0, float(bad)
    if problem.name == "conv2d":
        err = O.conv2d_error(out, ref, problem.inputs["image"], problem.inputs["filter"])
        return err <= O.CONV_TOL, err
    if problem.name in ("sgemm", "sgemm_tf32"):
        err = O.sgemm_error(out, ref)
        return err <= (O.SGEMM_TF32_TOL if problem.name == "sgemm_tf32" else O.SGEMM_TOL), err
    return True, 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--configs", default=None, help="JSON list of configs")
    ap.add_argument("--sample", type=int, default=None)
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--min-seconds", type=float, default=0.2)
    ap.add_argument("--problem", default="{}", help="JSON problem kwargs")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--value-set", default=None)
    args = ap.parse_args()

    kwargs = json.loads(args.problem)
    if args.value_set:
        kwargs["value_set"] = args.value_set
    problem = make_problem(args.kernel, **kwargs)
    if args.configs:
        configs = json.loads(args.configs)
    else:
        space = problem.space()
        every = [c.as_dict() for c in space.enumerate()]
        if args.all:
            configs = every
        else:
            rng = np.random.default_rng(args.seed)
            idx = rng.choice(len(every), size=min(args.sample or 50, len(every)), replace=False)
            configs = [every[i] for i in sorted(idx)]
    configs = [{**problem.default_config(), **c} for c in configs]
    print(f"{args.kernel}: {len(configs)} configs", flush=True)

    t0 = time.time()
    workers = max(1, min(32, (os.cpu_count() or 8)))

    def build(cfg):
        try:
            problem.cubin(cfg)
            return None
        except JouleTuneError as exc:
            return str(exc)[:300]

    with ThreadPoolExecutor(workers) as pool:
        errors = list(pool.map(build, configs))
    print(f"compiled in {time.time() - t0:.1f}s with {workers} threads", flush=True)

    gpu = GPU(0)
    problem.prepare(gpu)
    ref = None if args.no_verify else reference(problem)
    rows = []
    for cfg, err in zip(configs, errors):
        row = {"config": cfg}
        if err:
            row["error"] = err
            rows.append(row)
            continue
        try:
            k = problem.kernel(cfg)
            problem.bind(k, cfg)
            problem.reset_output()
            launch = problem.launch(cfg)
            run = gpu.bench(k, launch, problem.args(cfg), min_seconds=args.min_seconds, sample=False)
            row.update(ms=run.per_launch_s * 1e3, reps=run.reps, regs=k.regs, smem=k.static_smem,
                       tflops=problem.total_flops / run.per_launch_s / 1e12)
            if ref is not None:
                # fresh single launch from a clean output for the check
                problem.reset_output()
                gpu.launch(k, launch, problem.args(cfg))
                gpu.synchronize()
                ok, metric = check(problem, ref, cfg)
                row.update(ok=ok, check=metric)
        except JouleTuneError as exc:
            row["error"] = str(exc)[:300]
        rows.append(row)
        print(json.dumps(row), flush=True)
    good = sorted([r for r in rows if "ms" in r], key=lambda r: r["ms"])
    peak = fp32_peak_tflops(gpu.sm_count, 1965)
    print("best:")
    for r in good[:10]:
        print(f"  {r['ms']:.4f} ms  {r['tflops']:.2f} TF ({r['tflops'] / peak:.1%} of 1965-MHz FP32)  "
              f"ok={r.get('ok')} regs={r['regs']} {r['config']}")
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/sweep_{args.kernel}.json").write_text(json.dumps(rows, indent=1))
    gpu.close()


if __name__ == "__main__":
    main()
