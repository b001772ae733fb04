"""Sharded (config x clock) tuning == single-process exhaustive tuning.

Multi-process coverage on CPU: torch.distributed with the gloo backend,
world size 2, one simulated device per rank (the B200 path is identical
with one B200Device per rank). The only collective is a barrier; the gather
is the filesystem, as in production."""

import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2211_07260_b200 as B
from paper_2211_07260_b200 import partition


def _space(golden):
    return B.SearchSpace.from_dict(golden["spaces"]["a100_mimic_space"])


def test_plan_covers_every_point_once_and_is_clock_major(golden):
    space = _space(golden)
    shards = partition.plan(space, 3)
    points = [p for s in shards for p in s.iter_points()]
    assert sorted(p.key() for p in points) == sorted(c.key() for c in space.enumerate())
    assert sum(s.points() for s in shards) == space.size()
    first = list(shards[0].iter_points())
    n = len(shards[0].configs)
    assert {p["nvml_gr_clock"] for p in first[:n]} == {shards[0].clocks[0]}
    assert max(len(s.configs) for s in shards) - min(len(s.configs) for s in shards) <= 1


def test_lpt_balances_weighted_configs(golden):
    space = _space(golden)
    cost = lambda c: c["Mwg"] * c["Nwg"]  # noqa: E731
    shards = partition.plan(space, 4, cost=cost)
    loads = [sum(cost(c) for c in s.configs) for s in shards]
    assert max(loads) / min(loads) < 1.05


def test_merge_normalises_float_clocks(golden, spec_file, tmp_path):
    space = B.SearchSpace.from_dict({"parameters": {"Mwg": [16, 32], "nvml_gr_clock": [810, 1410]}})
    floats = space.with_values("nvml_gr_clock", [810.0, 1410.0])
    dev = B.load_device(spec_file("a100_mimic"))
    shard = partition.plan(floats, 1)[0]
    partition.run_shard(shard, dev, [B.InstantPowerObserver()], out=tmp_path / "s0.jsonl")
    merged = partition.merge(space, [tmp_path / "s0.jsonl"])
    assert [r.config.key() for r in merged.history] == [c.key() for c in space.enumerate()]


def test_single_process_shards_equal_exhaustive(golden, spec_file, tmp_path):
    space = _space(golden)
    files = []
    for shard in partition.plan(space, 3):
        dev = B.load_device(spec_file("a100_mimic"))
        path = tmp_path / f"s{shard.rank}.jsonl"
        partition.run_shard(shard, dev, [B.InstantPowerObserver()], out=path)
        files.append(path)
    merged = partition.merge(space, files)
    ref = B.run_strategy(B.TuningRun(space, "exhaustive", B.Objective("energy")),
                         B.load_device(spec_file("a100_mimic")), [B.InstantPowerObserver()])
    assert [r.to_dict() for r in merged.history] == [r.to_dict() for r in ref.history]
    assert merged.best.to_dict() == ref.best.to_dict()
    assert merged.points_per_second and merged.points_per_second > 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, spec_path, space_doc, workdir, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        space = B.SearchSpace.from_dict(space_doc)
        out = partition.run_distributed(
            space, lambda _: B.load_device(spec_path), lambda: [B.InstantPowerObserver()], workdir=workdir,
            rank=rank, world=world, barrier=dist.barrier)
        if rank == 0:
            with open(result_path, "w") as fh:
                json.dump({"history": [r.to_dict() for r in out.history], "best": out.best.to_dict(),
                           "stats": out.shard_stats}, fh)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_sharded_tuning_matches_single_process(golden, spec_file, tmp_path):
    space_doc = golden["spaces"]["a100_mimic_space"]
    result = tmp_path / "merged.json"
    mp.spawn(_worker, args=(2, _free_port(), str(spec_file("a100_mimic")), space_doc, str(tmp_path / "w"),
                            str(result)), nprocs=2, join=True)
    got = json.loads(result.read_text())
    space = B.SearchSpace.from_dict(space_doc)
    ref = B.run_strategy(B.TuningRun(space, "exhaustive", B.Objective("energy")),
                         B.load_device(spec_file("a100_mimic")), [B.InstantPowerObserver()])
    assert got["history"] == json.loads(json.dumps([r.to_dict() for r in ref.history]))
    assert got["best"]["energy"] == ref.best.energy
    assert sorted(s["rank"] for s in got["stats"]) == [0, 1]
    assert sum(s["points"] for s in got["stats"]) == space.size()
