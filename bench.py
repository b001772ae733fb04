"""Benchmark of the B200 kernel suite (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): 2D correlation of a 4096x4096 fp32
image with a 17x17 filter at the B200-tuned time-optimal config. One *step*
is one kernel launch over one 4096^2 image. Inputs are resident in HBM and
rotate over 4 image/output sets (4 x 135 MB = 540 MB > 126 MB L2), so no
step reads an L2-warm image. ``value`` = GFLOP/s of the whole job (all
ranks; weak scaling: every rank convolves its own image stream), timed with
CUDA events on the launching stream, max over ranks. The NVML sampler in
libjt records power / energy counter / SM clock during the timed region, so
the same run reports GFLOPS/W. ``e2e`` times the public host-buffer API
(``paper_2211_07260_b200.suite.conv2d``) with pinned inputs: H2D image +
kernel + D2H output per step. ``per_kernel`` reports the tuned PnPoly and
SGEMM configs the same way. ``cpu_baseline`` times the numpy oracle port on
this host's cores (rank 0, N=1).

``--impl reference`` times the reference CPU path (the numpy restatement in
oracle/, the reference package has no kernel code) on the same metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import types
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GFLOPS/W and GFLOP/s at energy- vs time-optimal config+clock, per kernel"
PROFILE_SUMMARY = ROOT / "profiles" / "ncu_summary.json"
REASON_NAMES = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


# -- distributed plumbing (host-side only: barrier + max over ranks) ----------------


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        # test hook: BENCH_SAME_GPU=1 puts every rank on cuda:0, so the N > 1 control flow
        # (barriers, shard plan, gather, max over ranks) can be exercised on a 1-GPU box
        # (its numbers are then meaningless)
        if os.environ.get("BENCH_SAME_GPU") == "1":
            self.local_rank = 0
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


E2E_STRIPS = 4  # row bands of the pipelined host-buffer call (suite.CONV2D_STRIPS)
GATE_MAX_STEPS = 256  # timed regions up to this many launches are enqueued behind a stream gate
ENERGY_LOOP_S = 1.5  # the headline's dedicated energy loop (>= 10 energy-counter updates)
ISSUE_MIX_CYCLES = 5.15  # scheduler cycles per 32 brute-force edge tests (ASM 7 mix, measured)
ENERGY_SETTLE_S = 0.25  # skipped at its start: power ramp after the timed region


def torch_sync():
    """The contract's torch.cuda.synchronize(); our work runs on libjt's stream,
    which is synchronised explicitly as well."""
    try:
        import torch

        if torch.cuda.is_available():
            torch.cuda.synchronize()
    except Exception:  # noqa: BLE001
        pass


# -- CPU reference path (oracle port; test infrastructure used as the baseline) -------


def cpu_conv_rate(budget_s: float, threads: int, rows_per_task: int = 32):
    """GFLOP/s of the numpy conv oracle port over row bands of the §8(d) image."""
    from oracle import kernels_oracle as O
    from paper_2211_07260_b200.kernels import Conv2DProblem

    prob = Conv2DProblem()
    inp = prob.host_inputs()
    image, filt = inp["image"], inp["filter"]
    bands = [slice(r, r + rows_per_task) for r in range(0, prob.height, rows_per_task)]
    done_rows = 0
    t0 = time.perf_counter()

    def work(sl):
        O.conv2d_rows(image, filt, sl)
        return sl.stop - sl.start

    with ThreadPoolExecutor(threads) as pool:
        futures = []
        for sl in bands:
            futures.append(pool.submit(work, sl))
            if len(futures) >= threads * 2:
                done_rows += futures.pop(0).result()
                if time.perf_counter() - t0 > budget_s:
                    break
        for f in futures:
            done_rows += f.result()
    dt = time.perf_counter() - t0
    flops = 2.0 * prob.fw * prob.fh * prob.width * done_rows
    return flops / dt / 1e9, done_rows, dt


def cpu_kernel_rates() -> dict:
    """The CPU oracle ports of the other kernels on bounded samples of their BASELINE workloads
    (host cores, the same run), for the per-kernel GPU / CPU ratio. Test infrastructure as the
    reported baseline only."""
    from oracle import kernels_oracle as O
    from paper_2211_07260_b200.kernels import PnPolyProblem, SgemmProblem

    out = {}
    threads = O.host_threads()
    p = PnPolyProblem()
    inp = p.host_inputs()
    n = p.n_points
    t0 = time.perf_counter()
    O.pnpoly(inp["points"][:n], inp["vx"], inp["vy"], 2, threads=threads)
    dt = time.perf_counter() - t0
    out["pnpoly"] = {"value": round(3.0 * n * p.n_vertices / dt / 1e9, 3), "unit": "GFLOP/s (3 ops per edge test)",
                     "cores": threads, "kind": "port",
                     "sample": f"all {n} points x 600 edges ({dt:.1f} s), C float32 crossing test, formulation 2"}
    s = SgemmProblem()
    inp = s.host_inputs()
    t0 = time.perf_counter()
    O.sgemm(inp["a"], inp["b"], inp["c0"], s.alpha, s.beta)
    dt = time.perf_counter() - t0
    out["sgemm"] = {"value": round(s.total_flops / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
                    "sample": f"4096^3 ({dt:.1f} s), numpy float64 matmul oracle (OpenBLAS threads)"}
    return out


def run_reference(args, dist: Dist) -> int:
    if dist.rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    rates = []
    for i in range(args.warmup + args.steps):
        rate, rows, dt = cpu_conv_rate(budget_s=2.0, threads=threads)
        if i >= args.warmup:
            rates.append((rate, rows, dt))
    value = statistics.median(r[0] for r in rates)
    rows = rates[0][1]
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GFLOP/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(r[2] for r in rates), 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seed 3, U[0,1) image and filter)",
        "config": {"workload": "conv2d 4096x4096 fp32, 17x17 filter (numpy oracle port, CPU)",
                   "image": [4096, 4096], "filter": [17, 17]},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "sample": f"{rows} output rows x 4096 per step (2 s budget), float64 shift-add, "
                                   f"{threads} threads over 32-row bands"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# -- GPU path ------------------------------------------------------------------------


def summarize_samples(samples, t0, t1):
    from paper_2211_07260_b200.b200 import counter_power

    inside = [s for s in samples if t0 <= s[0] <= t1]
    watts, _ = counter_power(samples, t0, t1)
    clocks = [s[5] for s in inside if s[5]]
    reasons = 0
    for s in inside:
        reasons |= int(s[8])
    inst = [s[1] for s in inside if math.isfinite(s[1])]
    return {
        "n": len(inside),
        "counter_w": watts,
        "instant_w": statistics.median(inst) if inst else None,
        "sm_mhz": statistics.median(clocks) if clocks else None,
        "temp_c": statistics.median([s[7] for s in inside]) if inside else None,
        "reasons": [name for bit, name in REASON_NAMES.items() if reasons & bit and bit != 0x1],
    }


def kernel_profile(name: str, config: dict):
    """DRAM traffic per launch from the committed ncu summary, if captured."""
    if not PROFILE_SUMMARY.exists():
        return None
    data = json.loads(PROFILE_SUMMARY.read_text())
    entry = data.get(name)
    if not entry:
        return None
    if entry.get("config") and {k: v for k, v in entry["config"].items()} != config:
        return None
    return entry.get("dram_bytes_per_launch")


def tf32_peak_gflops(sustained: bool = False) -> float:
    """Dense TF32 peak = half the MEASURED dense bf16 rate (same tcgen05 cycles, K=8 vs K=16 per MMA).
    ``sustained``: the back-to-back figure (power-capped clocks), for kernels timed in long loops."""
    peaks = ROOT / "MEASURED_PEAKS.json"
    doc = json.loads(peaks.read_text()) if peaks.exists() else {}
    bf16 = doc.get("bf16_tflops_sustained" if sustained else "bf16_tflops") or doc.get("bf16_tflops", 1590.0)
    return bf16 / 2.0 * 1e3


def measure_tuned(gpu, name: str, objective: str, seconds: float = 1.0, settle: float = 0.25, sets: int = 2,
                  config: dict | None = None, loops: int = 1):
    """One tuned config (or ``config``) in ``loops`` >= 1 s device-timed loops over ``sets`` rotating
    input/output sets (each larger than L2 or alone in it, so no launch reads an L2-warm input), energy
    from whole NVML energy-counter periods taken ``settle`` s into each loop; with several loops the
    median time and the median power are reported."""
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.gpu import fp32_peak_tflops
    from paper_2211_07260_b200.kernels import make_problem

    prob = make_problem(name)
    prob.prepare(gpu)
    cfg = config or tuned.best_config(name, objective) or prob.default_config()
    k = prob.kernel(cfg)
    prob.bind(k, cfg)
    rotation = prob.rotation_sets(cfg, sets)
    measured = []
    for _ in range(max(1, loops)):
        r = gpu.bench(k, prob.launch(cfg), prob.args(cfg), min_seconds=seconds, rotate=rotation)
        measured.append((r, summarize_samples(r.samples, r.loop_t0 + settle, r.loop_t1)))
    powers = [m[1]["counter_w"] for m in measured if m[1]["counter_w"]]
    watts = statistics.median(powers) if powers else None
    run, summ = sorted(measured, key=lambda m: m[0].per_launch_s)[len(measured) // 2]
    run_s = statistics.median([m[0].per_launch_s for m in measured])
    run = types.SimpleNamespace(per_launch_s=run_s)
    out = {"config": cfg, "ms": round(run.per_launch_s * 1e3, 4), "rotating_sets": sets, "loops": len(measured),
           "power_w": round(watts, 1) if watts else None, "sm_mhz": summ["sm_mhz"], "reasons": summ["reasons"]}
    if prob.roofline_kind == "hbm":
        # work-skipping PnPoly kernels: no flop credit for the edge tests they do not run
        peaks = ROOT / "MEASURED_PEAKS.json"
        hbm = (json.loads(peaks.read_text()) if peaks.exists() else {}).get("hbm_gbs") or 7700.0
        gbs = prob.algorithmic_bytes / run.per_launch_s / 1e9
        out.update({
            "points_per_s": round(prob.n_points / run.per_launch_s, 1),
            "gb_per_s": round(gbs, 1),
            "j_per_bitmap": round(watts * run.per_launch_s, 6) if watts else None,
            "roofline_frac": round(gbs / hbm, 4),
            "roofline_basis": (f"HBM: {prob.algorithmic_bytes / 1e6:.1f} MB algorithmic (points + bitmap) per "
                               f"launch = {gbs:.0f} GB/s vs {hbm} GB/s (MEASURED_PEAKS hbm_gbs)"),
        })
        if name == "pnpoly_grid":
            out["clean_cell_fraction"] = round(prob.clean_fraction(cfg["grid"]), 4)
        if name == "pnpoly_cells":
            out["decided_cell_fraction"] = round(prob.clean_fraction(cfg["grid"], cfg["lmax"]), 4)
    else:
        rate = prob.total_flops / run.per_launch_s / 1e9
        out["gflops"] = round(rate, 1)
        out["gflops_per_w"] = round(prob.total_flops / (watts * run.per_launch_s) / 1e9, 2) if watts else None
        if prob.roofline_kind == "tensor":
            # a >= 1 s back-to-back loop runs at the power cap: the sustained measured peak is the
            # denominator (the burst one is reported beside it)
            peak = tf32_peak_gflops(sustained=True)
            out["roofline_frac"] = round(rate / peak, 4)
            out["roofline_peak_gflops"] = peak
            out["roofline_frac_vs_burst"] = round(rate / tf32_peak_gflops(), 4)
            out["roofline_basis"] = ("MEASURED_PEAKS bf16_tflops_sustained / 2 (tcgen05 kind::tf32 issues K=8 per "
                                     "MMA vs K=16; loop runs power-capped like the sustained bf16 measurement)")
        elif summ["sm_mhz"]:
            peak = fp32_peak_tflops(gpu.sm_count, summ["sm_mhz"]) * 1e3
            if prob.roofline_kind == "issue":
                peak /= 2.0  # 1 lane-instruction slot per lane per clock, not 2 flop/FFMA
                out["edge_tests_per_s"] = round(prob.edge_tests / run.per_launch_s, 1)
                out["j_per_bitmap"] = round(watts * run.per_launch_s, 6) if watts else None
                # the measured issue bound of the crossing-test instruction mix (DESIGN.md §4,
                # profiles/r1_issue_probe.jsonl): 5.15 scheduler cycles per 32 edge tests
                bound_s = prob.edge_tests / 32 * ISSUE_MIX_CYCLES / (4 * gpu.sm_count * summ["sm_mhz"] * 1e6)
                out["issue_mix_bound_ms"] = round(bound_s * 1e3, 4)
                out["roofline_frac_issue_mix"] = round(bound_s / run.per_launch_s, 4)
            out["roofline_frac"] = round(rate / peak, 4)
    for b in prob.buffers.values():
        b.free()
    return out


#: the sharded tuning leg: a fixed slice of the conv2d space (strong scaling over ranks), 516 points so that
#: each of 8 ranks measures >= 64 of them
TUNE_SPACE = {"block_size_x": [32, 64], "block_size_y": [2, 4, 8, 16], "tile_size_x": [2, 4, 8],
              "tile_size_y": [1, 2, 4], "use_shmem": [0, 1], "use_padding": [0], "fma2": [0, 1], "min_blocks": [0, 2]}
TUNE_WINDOW_S = 0.25  # launch loop per point: >= 2 energy-counter updates (~100 ms cadence)


def tuning_leg(gpu, dist: Dist) -> dict:
    """Tuning throughput: this rank's shard of a fixed (config) space through the reference API.

    ``partition.plan`` deals the configs over the ranks (LPT); each
    rank measures its shard on its own GPU with the NVML observer
    (``run_strategy``'s evaluator, energy objective), writes a JSONL shard, and
    rank 0 merges them on the filesystem after a barrier. Per-rank fixed costs
    (input upload + device setup, compilation) are timed apart from the shard
    loop; points/s = all points / slowest shard loop.
    """
    import tempfile

    from paper_2211_07260_b200 import NVMLObserver, Objective, SearchSpace, partition
    from paper_2211_07260_b200.b200 import B200Device
    from paper_2211_07260_b200.kernels import make_problem

    problem = make_problem("conv2d")
    space = SearchSpace.from_dict({"parameters": TUNE_SPACE, "restrictions": problem.restrictions()})
    shards = partition.plan(space, dist.world)
    mine = shards[dist.rank]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(8) as pool:
        list(pool.map(lambda c: problem.cubin({**problem.default_config(), **c.as_dict()}), mine.configs))
    compile_s = time.perf_counter() - t0
    base = os.environ.get("BENCH_TUNE_DIR") or os.path.join(tempfile.gettempdir(),
                                                            f"bench_tune_{os.environ.get('MASTER_PORT', 'solo')}")
    workdir = Path(base)
    if dist.rank == 0:
        workdir.mkdir(parents=True, exist_ok=True)
        for f in workdir.iterdir():
            f.unlink()
    dist.barrier()
    t0 = time.perf_counter()
    device = B200Device(problem, gpu=gpu, min_window=TUNE_WINDOW_S)  # uploads this rank's inputs
    setup_s = time.perf_counter() - t0
    metrics, consts = problem.user_metrics()
    stats = partition.run_shard(mine, device, [NVMLObserver(TUNE_WINDOW_S)], out=workdir / f"shard{dist.rank}.jsonl",
                                user_metrics=metrics, constants=consts)
    dist.barrier()
    slowest = dist.max(stats["seconds"])
    points = len(space.enumerate())
    per_point_ms = 1e3 * stats["seconds"] / max(1, mine.points())
    out = {"space": "conv2d slice " + json.dumps(TUNE_SPACE, separators=(",", ":")), "points": points,
           "window_s": TUNE_WINDOW_S, "points_per_s": round(points / slowest, 3), "slowest_shard_s": round(slowest, 2),
           "shard_points": [s.points() for s in shards],
           "per_point_ms_max": round(dist.max(per_point_ms), 1),
           "fixed_cost_s": {"setup_max": round(dist.max(setup_s), 3), "compile_max": round(dist.max(compile_s), 2),
                            "note": "per rank, outside the shard loop: input upload + device probe; NVRTC compile "
                                    "of the shard's configs (8 host threads, cubin cache cold or warm)"},
           "points_per_s_incl_fixed": round(points / dist.max(stats["seconds"] + setup_s + compile_s), 3),
           "timing": "wall clock of each rank's shard loop, max over ranks",
           "note": "0.25 s windows hold two whole energy-counter periods (loops that stalled or whose counter "
                   "and instant power disagree are re-run): the optima below are screening values, each "
                   "re-measured in a 1 s loop under confirmed_1s (tune_suite.py confirms leaders in 3 x 1 s "
                   "loops; per_kernel holds those)"}
    if dist.rank == 0:
        merged = partition.merge(space, [workdir / f"shard{r}.jsonl" for r in range(dist.world)],
                                 objective=Objective("energy"))
        ok = [r for r in merged.history if not r.failed]
        best_t = min(ok, key=lambda r: r.time)
        out["failed"] = len(merged.history) - len(ok)
        out["energy_optimal"] = {"config": merged.best.config.as_dict(),
                                 "gflops_per_w": round(merged.best.metrics.get("gflops_per_w", 0.0), 2),
                                 "gflops": round(merged.best.metrics.get("gflops", 0.0), 1)}
        out["time_optimal"] = {"config": best_t.config.as_dict(),
                               "gflops_per_w": round(best_t.metrics.get("gflops_per_w", 0.0), 2),
                               "gflops": round(best_t.metrics.get("gflops", 0.0), 1)}
    for b in problem.buffers.values():
        b.free()
    if dist.rank == 0:
        # the screening optima re-measured the way per_kernel measures (1 s loops, energy from 0.25 s in),
        # after the timed shard loop: a 0.25 s window can read a low-power stretch and flatter a config
        for key in ("energy_optimal", "time_optimal"):
            cfg = {**problem.default_config(), **out[key]["config"]}
            conf = measure_tuned(gpu, "conv2d", key, config=cfg)
            out[key]["confirmed_1s"] = {k: conf.get(k) for k in ("ms", "power_w", "gflops", "gflops_per_w", "sm_mhz")}
    return out


def run_ours(args, dist: Dist) -> int:
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.gpu import GPU, fp32_peak_tflops
    from paper_2211_07260_b200.kernels import Conv2DProblem
    from paper_2211_07260_b200 import suite

    gpu = GPU(dist.local_rank)
    prob = Conv2DProblem()
    cfg = tuned.best_config("conv2d", "time_optimal") or prob.default_config()
    prob.prepare(gpu)
    kernel = prob.kernel(cfg)
    prob.bind(kernel, cfg)
    launch = prob.launch(cfg)
    sets = [prob.args(cfg)]
    for _ in range(3):  # rotate inputs: 4 x 135 MB > L2
        img = gpu.array(prob.inputs["image"], slack=64)
        out = gpu.empty((prob.height, prob.width), np.float32)
        sets.append([out, img])
    # each set's launch packed once: the timed loop below issues back-to-back native launches with no
    # per-launch Python argument packing (the kernel is ~150 us; the first launch follows the start event)
    prepared = [gpu.prepare_launch(kernel, launch, s) for s in sets]
    from paper_2211_07260_b200 import native

    gpu.reserve_events(2)
    # the NVML sampler (its first calls can stall) starts before the warm-up, so the only idle time
    # between the warm-up and the timed region is the barrier + synchronize the contract requires
    gpu.sampler_start(1000, 1 << 20)
    for i in range(args.warmup):
        gpu.launch_prepared(prepared[i % 4])
    gpu.synchronize()
    dist.barrier()
    torch_sync()
    gpu.synchronize()
    t_host0 = native.now()
    # the stream is gated while the start event, the K launches and the stop event are enqueued, then
    # released: the events time K back-to-back kernels, with no host submission (or driver lock held by
    # the NVML sampler thread) between them
    # not under a profiler / sanitizer (CUDA_INJECTION64_PATH): those complete each launch inside the
    # launch call, which would wait forever on a gated stream
    # Only short regions are gated: launches pile up in the driver's queue behind the gate, and a queue
    # that fills blocks the enqueueing thread (long regions have no start-up gap to hide anyway).
    gated = False
    tool = any(k.startswith(("CUDA_INJECTION", "NV_NSIGHT", "NSIGHT", "NV_COMPUTE_PROFILER", "NV_TPS"))
               for k in os.environ) or any(t in os.environ.get("LD_PRELOAD", "").lower()
                                           for t in ("nsight", "sanitizer", "injection"))
    if args.steps <= GATE_MAX_STEPS and not tool and not os.environ.get("BENCH_NO_GATE"):
        try:
            gpu.gate()
            gated = True
        except Exception:  # noqa: BLE001  (no stream memory operations on this driver: plain enqueue)
            gated = False
    # a tool that blocks inside the launch call anyway is freed by a watchdog release (its timing would
    # then include the wait; numbers taken under a profiler are never bench values)
    watchdog = None
    if gated:
        import threading

        watchdog = threading.Timer(5.0, gpu.release)
        watchdog.daemon = True
        watchdog.start()
    try:
        gpu.record(0)
        for i in range(args.steps):
            gpu.launch_prepared(prepared[i % 4])
        gpu.record(1)
    finally:
        if gated:
            gpu.release()
            watchdog.cancel()
    elapsed = gpu.elapsed(0, 1)
    gpu.synchronize()
    torch_sync()
    t_host1 = native.now()
    samples = gpu.sampler_stop(1 << 20)
    dist.barrier()
    elapsed_max = dist.max(elapsed)
    ranks_flops = dist.sum(prob.total_flops * args.steps)
    # the loop occupied the last `elapsed` seconds before t_host1; skip 0.1 s of ramp
    loop_t0 = max(t_host0, t_host1 - elapsed)
    summ = summarize_samples(samples, loop_t0 + min(0.1, 0.5 * elapsed), t_host1)

    # energy: a dedicated loop of the same kernel and config over the same 4 rotating sets, independent
    # of --steps (a 20-step timed region lasts ~3 ms, far below the ~100 ms energy-counter cadence)
    erun = gpu.bench(kernel, launch, sets[0], rotate=sets[1:], min_seconds=ENERGY_LOOP_S)
    esumm = summarize_samples(erun.samples, erun.loop_t0 + ENERGY_SETTLE_S, erun.loop_t1)

    per_step = elapsed / args.steps
    value = ranks_flops / elapsed_max / 1e9
    if summ["sm_mhz"]:
        sm, sm_basis, clock_src = summ["sm_mhz"], "observed median in the timed region", summ
    elif esumm["sm_mhz"]:
        sm, sm_basis, clock_src = esumm["sm_mhz"], "observed median in the energy loop (timed region unsampled)", esumm
    else:
        sm, sm_basis, clock_src = 1965.0, "assumed 1965 MHz max clock (no NVML clock sample)", esumm
    achieved_tf = prob.total_flops / per_step / 1e12
    peak_tf = fp32_peak_tflops(gpu.sm_count, sm)
    traffic = kernel_profile("conv2d", cfg)

    # e2e through the public host-buffer API, pinned host memory
    e2e_steps = max(1, min(args.steps, 100))
    img_host = suite.pinned(prob.inputs["image"].shape, np.float32, dist.local_rank)
    img_host[...] = prob.inputs["image"]
    out_host = suite.pinned((prob.height, prob.width), np.float32, dist.local_rank)
    for _ in range(3):
        suite.conv2d(img_host, prob.inputs["filter"], config=cfg, out=out_host, ordinal=dist.local_rank)

    def e2e_rate(strips):
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            suite.conv2d(img_host, prob.inputs["filter"], config=cfg, out=out_host, ordinal=dist.local_rank,
                         strips=strips)
        return dist.sum(prob.total_flops * e2e_steps) / dist.max(time.perf_counter() - t0) / 1e9

    e2e_single = e2e_rate(1)
    e2e_per_call = e2e_rate(E2E_STRIPS)
    # the stream API: every step still uploads its image and downloads its result, but the
    # copies of step j+1 / j-1 overlap the launches of step j (two device buffer sets)
    out_host_b = suite.pinned((prob.height, prob.width), np.float32, dist.local_rank)
    suite.conv2d_many([img_host] * 4, prob.inputs["filter"], config=cfg, outs=[out_host, out_host_b] * 2,
                      ordinal=dist.local_rank, strips=E2E_STRIPS)
    dist.barrier()
    t0 = time.perf_counter()
    suite.conv2d_many([img_host] * e2e_steps, prob.inputs["filter"], config=cfg,
                      outs=[out_host, out_host_b] * (e2e_steps // 2) + [out_host] * (e2e_steps % 2),
                      ordinal=dist.local_rank, strips=E2E_STRIPS)
    e2e_value = dist.sum(prob.total_flops * e2e_steps) / dist.max(time.perf_counter() - t0) / 1e9

    tuning = None if args.no_tune else tuning_leg(gpu, dist)

    # per-kernel tuned summaries (time- and energy-optimal) on this rank's GPU
    per_kernel = {}
    if dist.rank == 0 and not args.quick:
        for name in ("conv2d", "pnpoly", "pnpoly_slab", "pnpoly_grid", "pnpoly_cells", "sgemm", "sgemm_tf32"):
            # 2 loops per config, medians; a config that is both optima is measured once and reported twice
            from paper_2211_07260_b200 import tuned as _tuned
            t_cfg = _tuned.best_config(name, "time_optimal")
            entry = {"time_optimal": measure_tuned(gpu, name, "time_optimal", loops=2)}
            if t_cfg is not None and t_cfg == _tuned.best_config(name, "energy_optimal"):
                entry["energy_optimal"] = {**entry["time_optimal"], "same_config_as": "time_optimal"}
            else:
                entry["energy_optimal"] = measure_tuned(gpu, name, "energy_optimal", loops=2)
            per_kernel[name] = entry

    cpu = None
    cpu_kernels = None
    if dist.rank == 0 and dist.world == 1 and not args.quick:
        cpu_kernels = cpu_kernel_rates()
        threads = len(os.sched_getaffinity(0))
        rate, rows, dt = cpu_conv_rate(budget_s=10.0, threads=threads)
        cpu = {"value": round(rate, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
               "sample": f"{rows} of 4096 output rows ({dt:.1f} s), numpy float64 shift-add oracle, "
                         f"{threads} threads over 32-row bands"}

    if dist.rank == 0:
        ew = esumm["counter_w"]
        gflops_per_w = prob.total_flops / (ew * erun.per_launch_s) / 1e9 if ew else None
        line = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": "GFLOP/s",
            "n_gpus": dist.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(1e3 * elapsed_max / args.steps, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seed 3: U[0,1) 4112x4112 image, U[0,1) 17x17 filter)",
            "config": {
                "workload": "conv2d 4096x4096 fp32 17x17 (BASELINE configs[1]) at the B200-tuned time-optimal config",
                "kernel_config": cfg,
                "image": [4096, 4096],
                "filter": [17, 17],
                "l2": "4 rotating resident image/output sets, 540 MB > 126 MB L2",
                "parallelism": f"replicas x{dist.world} (independent images per GPU, no collective)",
                "clock_control": "none in the timed region (driver-managed clocks)",
                "timed_region": ("stream gated while start event + K launches + stop event are enqueued, then "
                                 "released (jt_stream_gate)" if gated else "launches enqueued behind the start event"),
            },
            "energy": {
                "gflops_per_w": round(gflops_per_w, 2) if gflops_per_w else None,
                "power_w_counter": round(ew, 1) if ew else None,
                "power_w_instant_median": esumm["instant_w"],
                "gflops": round(prob.total_flops / erun.per_launch_s / 1e9, 1),
                "ms_per_launch": round(erun.per_launch_s * 1e3, 5),
                "sm_mhz": esumm["sm_mhz"],
                "reasons": esumm["reasons"],
                "source": (f"NVML total-energy counter, whole 100 ms counter periods (libjt sampler) over a dedicated {erun.total_s:.2f} s "
                           f"loop of {erun.reps} launches of the same kernel/config over the same 4 rotating sets, "
                           f"from {ENERGY_SETTLE_S} s in (past the power ramp); GFLOPS/W = flop / (W x s per launch)"),
            },
            "roofline": {
                "bound": "fp32",
                "achieved": round(achieved_tf, 2),
                "peak": round(peak_tf, 2),
                "unit": "TFLOP/s",
                "frac": round(achieved_tf / peak_tf, 4),
                "traffic": traffic,
                "peak_basis": f"FP32 FFMA peak 2 x {gpu.sm_count} SMs x 128 lanes x {sm:.0f} MHz ({sm_basis}); "
                              "MEASURED_PEAKS.json has no FP32 figure",
                "frac_at_1965mhz": round(achieved_tf / fp32_peak_tflops(gpu.sm_count, 1965.0), 4),
                "algorithmic_flops_per_launch": prob.total_flops,
            },
            "clocks": {"sm_mhz": clock_src["sm_mhz"], "sm_max_mhz": gpu.info.max_sm_clock_mhz,
                       "reasons": sorted(set(summ["reasons"]) | set(esumm["reasons"])), "temp_c": clock_src["temp_c"],
                       "source": sm_basis, "timed_region_samples": summ["n"]},
            "e2e": {"value": round(e2e_value, 1), "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(prob.inputs["image"].nbytes),
                    "d2h_bytes_per_step": int(prob.width * prob.height * 4),
                    "timing": f"wall clock around paper_2211_07260_b200.suite.conv2d_many over {e2e_steps} steps "
                              "(pinned host arrays): every step uploads its 4112^2 image and downloads its "
                              f"4096^2 result; {E2E_STRIPS} row bands per step over H2D / compute / D2H "
                              "streams, pipelined across steps",
                    "per_call_value": round(e2e_per_call, 1),
                    "single_launch_value": round(e2e_single, 1)},
            "gpu_launches": args.steps,
            "per_kernel": per_kernel,
        }
        if tuning:
            line["tuning"] = tuning
        if cpu:
            line["cpu_baseline"] = cpu
        if cpu_kernels:
            line["cpu_per_kernel"] = cpu_kernels
        print(json.dumps(line))
    gpu.close()
    return 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=6000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--quick", action="store_true", help="skip per-kernel and CPU-baseline legs")
    ap.add_argument("--no-tune", action="store_true", help="skip the sharded tuning-throughput leg")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    dist = Dist()
    try:
        return run_reference(args, dist) if args.impl == "reference" else run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    sys.exit(main())
