"""Sharded exhaustive tuning over N GPUs of one box (one process per GPU).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        scripts/tune_sharded.py --kernel conv2d --workdir gpurun_out/shard_conv2d

Each rank tunes its shard of the (config x clock) space (``partition.plan``:
LPT over whole configs, clock-major per worker) on its own B200 through the
reference API, writes a JSONL shard, and rank 0 merges the shards on the
filesystem after a gloo barrier. No NCCL, no data-path collective. Prints
one JSON line with the merged best and the tuning throughput
(points / max worker seconds).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import (  # noqa: E402
    CLOCK_PARAM, NVMLObserver, Objective, SearchSpace, TunableParameter, default_metrics, partition,
)
from paper_2211_07260_b200.b200 import B200Device  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="conv2d")
    ap.add_argument("--workdir", default="gpurun_out/shards")
    ap.add_argument("--duration", type=float, default=0.25)
    ap.add_argument("--clocks", default="", help="comma list of MHz to add as nvml_gr_clock")
    ap.add_argument("--limit", type=int, default=None, help="first N kernel configs only")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    barrier = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        barrier = dist.barrier
    problem = make_problem(args.kernel)
    doc = problem.space_document()
    if args.limit:
        cfgs = SearchSpace.from_dict(doc).enumerate()[: args.limit]
        doc = {"parameters": {k: sorted({c[k] for c in cfgs}) for k in doc["parameters"]},
               "restrictions": doc["restrictions"]}
    space = SearchSpace.from_dict(doc)
    if args.clocks:
        space = space.augment(TunableParameter(CLOCK_PARAM, tuple(int(c) for c in args.clocks.split(","))))
    shards = partition.plan(space, world)
    mine = shards[rank]
    with ThreadPoolExecutor(min(16, os.cpu_count() or 4)) as pool:  # compile this shard's configs
        list(pool.map(lambda c: problem.cubin({**problem.default_config(), **c.as_dict()}), mine.configs))
    out = partition.run_distributed(
        space,
        lambda ordinal: B200Device(problem, ordinal, min_window=args.duration),
        lambda: [NVMLObserver(args.duration)],
        workdir=args.workdir, rank=rank, world=world, local_rank=local, barrier=barrier,
        objective=Objective("energy"), user_metrics=problem.user_metrics()[0],
        constants=problem.user_metrics()[1],
    )
    if rank == 0:
        best_t = min((r for r in out.history if not r.failed), key=lambda r: r.time)
        print(json.dumps({
            "kernel": args.kernel, "world": world, "points": len(out.history),
            "points_per_second": out.points_per_second,
            "shard_seconds": [s["seconds"] for s in sorted(out.shard_stats, key=lambda s: s["rank"])],
            "energy_optimal": {"config": out.best.config.as_dict(), **out.best.metrics},
            "time_optimal": {"config": best_t.config.as_dict(), **best_t.metrics},
        }))
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
