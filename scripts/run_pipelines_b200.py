"""The paper's five tuning pipelines on B200 measurements.

Reference: ``tuner.py:541-645`` (recipes), ``scripts/run_pipelines.py:36-77``
(the reference's driver on simulated boards), ``PAPER.md:385-399`` (race-to-
idle vs global energy gap).

1. ``replay`` (CPU): every kernel's B200 tuning cache (results/cache_*.jsonl,
   reference JSONL format) becomes the cache of a (config x clock) space whose
   clock axis holds the one clock this pool runs at: NVML refuses every clock
   and power knob (profiles/r2_knob_probe.json: "Not Supported", code 3), so
   the driver-managed default clock (1965 MHz) is the only clock a
   ``B200Device`` accepts (``set_core_clock``), and the cached measurements
   were taken in exactly that state. ``run_pipeline`` then runs all five
   recipes against a device that refuses to execute, so every evaluation is a
   cache hit of a real measurement. With one clock the "+clocks" stages have
   nothing to sweep; the recipes still differ in their objective (time vs
   energy) at that clock, which is the paper's race-to-idle vs global gap.
2. ``confirm`` (GPU): the distinct configs the recipes picked are re-measured
   in 3 interleaved 1 s loops (the sweep windows read energy 5-25 % low after
   lighter configs), so each gap is quoted on confirmed energies too.

    python scripts/run_pipelines_b200.py replay      # -> results/pipelines_b200.json
    python scripts/run_pipelines_b200.py confirm     # GPU; adds the confirmed numbers
"""

from __future__ import annotations

import argparse
import json
import shutil
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import (  # noqa: E402
    CLOCK_PARAM, PIPELINES, DeviceSpec, DomainError, KernelConfig, ResultCache, SearchSpace, TunableParameter,
    run_pipeline,
)
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

sys.path.insert(0, str(ROOT / "scripts"))
from landscape_report import difficulty_space  # noqa: E402

RESULTS = ROOT / "results"
OUT = RESULTS / "pipelines_b200.json"
CLOCK = 1965.0  # the driver-managed clock every cached measurement ran at (observed median per result)

#: cache name -> (problem, kwargs)
KERNELS = {
    "conv2d": ("conv2d", {}), "sgemm_clblast": ("sgemm", {"value_set": "clblast"}), "sgemm": ("sgemm", {}),
    "sgemm_tf32": ("sgemm_tf32", {}), "pnpoly": ("pnpoly", {}), "pnpoly_slab": ("pnpoly_slab", {}),
    "pnpoly_grid": ("pnpoly_grid", {}), "pnpoly_cells": ("pnpoly_cells", {}),
}


class ReplayDevice:
    """A B200 spec whose only job is to make a cache miss loud: execute() refuses."""

    def __init__(self):
        self.spec = DeviceSpec("B200 (replay of measured cache)", (CLOCK - 15.0, CLOCK), CLOCK, CLOCK,
                               (200.0, 1000.0), 1000.0)
        self.sample_rate_hz = 1000.0
        self.execution_count = 0

    def set_core_clock(self, clock):
        return None

    def execute(self, config, duration_hint=0.0):
        self.execution_count += 1
        raise DomainError(f"not measured on the B200: {config.as_dict()}")


def replay() -> dict:
    out = {}
    for name, (pname, kwargs) in KERNELS.items():
        path = RESULTS / f"cache_{name}.jsonl"
        if not path.exists():
            continue
        measured = [r for r in ResultCache(path).results()]
        if not measured:
            continue
        # the measured configs, clock-augmented; the space is restricted to exactly those configs
        cache = ResultCache()
        keys = set()
        for r in measured:
            cfg = KernelConfig(r.config.items + ((CLOCK_PARAM, CLOCK),))
            cache.put(type(r)(config=cfg, time=r.time, energy=r.energy, observer_results=r.observer_results,
                              metrics=r.metrics, failed=r.failed, failure_reason=r.failure_reason))
            keys.add(r.config.key())
        doc = difficulty_space(make_problem(pname, **kwargs), [r for r in measured])
        if doc is None:  # a sampled (not exhaustive) cache: no space the recipes could enumerate
            print(name, "skipped: the cache does not cover a whole space", flush=True)
            continue
        space = SearchSpace.from_dict(doc).augment(TunableParameter(CLOCK_PARAM, (CLOCK,)))
        enumerated = space.enumerate()
        missing = [c for c in enumerated if KernelConfig(tuple(i for i in c.items if i[0] != CLOCK_PARAM)).key()
                   not in keys]
        dev = ReplayDevice()
        reports = {}
        for pipe in PIPELINES:
            rep = run_pipeline(pipe, space, dev, [], cache=cache)
            reports[pipe] = {"config": {k: v for k, v in rep.best.config.as_dict().items()},
                             "time_s": rep.best.time, "energy_j": rep.best.energy,
                             "stages": [s.label for s in rep.stages]}
        glob = reports["global"]["energy_j"]
        for pipe, rec in reports.items():
            rec["gap_vs_global"] = rec["energy_j"] / glob - 1.0
        out[name] = {"measured_configs": len(measured), "space_product": len(enumerated),
                     "unmeasured_in_product": len(missing), "clock_mhz": CLOCK, "device_executions": dev.execution_count,
                     "pipelines": reports}
        print(name, {p: f"{100 * r['gap_vs_global']:+.1f}%" for p, r in reports.items()}, flush=True)
    return out


def cmd_replay(args) -> None:
    doc = {"what": "the five pipelines (tuner.py:541-645) replayed on B200 tuning caches at the pool's one "
                   "available clock (clock control refused: profiles/r2_knob_probe.json)",
           "kernels": replay()}
    OUT.write_text(json.dumps(doc, indent=1) + "\n")


def cmd_confirm(args) -> None:
    sys.path.insert(0, str(ROOT / "scripts"))
    from paper_2211_07260_b200.b200 import B200Device
    from paper_2211_07260_b200.gpu import GPU
    from tune_suite import confirm  # noqa: E402

    doc = json.loads(OUT.read_text())

    class Picked:
        def __init__(self, cfg):
            self.config = KernelConfig.from_dict(cfg)
            self.energy = None  # confirm() records the sweep energy beside the confirmed one

    with GPU(0) as gpu:
        for name, entry in doc["kernels"].items():
            pname, kwargs = KERNELS[name]
            problem = make_problem(pname, **kwargs)
            dev = B200Device(problem, gpu=gpu)
            picks = [Picked({k: v for k, v in r["config"].items() if k != CLOCK_PARAM})
                     for r in entry["pipelines"].values()]
            confirmed = {json.dumps(c["config"], sort_keys=True): c for c in confirm(dev, problem, picks)}
            glob = None
            for pipe in ("global", *PIPELINES):
                rec = entry["pipelines"][pipe]
                key = json.dumps({k: v for k, v in rec["config"].items() if k != CLOCK_PARAM}, sort_keys=True)
                c = confirmed.get(key)
                if c is None:
                    continue
                rec["confirmed_time_s"], rec["confirmed_energy_j"] = c["time_s"], c["energy_j"]
                if pipe == "global":
                    glob = c["energy_j"]
                rec["confirmed_gap_vs_global"] = c["energy_j"] / glob - 1.0 if glob else None
            dev.close()
            for b in problem.buffers.values():
                b.free()
            print(name, {p: r.get("confirmed_gap_vs_global") for p, r in entry["pipelines"].items()}, flush=True)
    OUT.write_text(json.dumps(doc, indent=1) + "\n")
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    shutil.copy(OUT, ROOT / "gpurun_out" / OUT.name)


def main() -> None:
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("replay")
    sub.add_parser("confirm")
    args = ap.parse_args()
    {"replay": cmd_replay, "confirm": cmd_confirm}[args.cmd](args)


if __name__ == "__main__":
    main()
