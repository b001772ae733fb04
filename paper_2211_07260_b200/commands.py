"""Command line: ``simulate-sweep``, ``fit``, ``tune``, ``steer``, ``analyze``.

Behaviour contract (reference ``pkg/src/jouletune/cli.py``): the same
subcommands, flags, report documents (``report.json`` / model JSON / sweep
CSV) and exit codes — 0 ok, 1 runtime failure, 2 configuration error — so
that reports are byte-identical on simulated devices. A report header holds
the package version, the seed, the run manifest (every input that decides
the outputs, ``None`` entries dropped) and a 16-hex sha256 of that manifest;
there are no timestamps.

Additions for the real GPU:

* ``--device`` also accepts ``b200`` / ``b200:<kernel>[:<ordinal>]`` or a JSON
  file ``{"kind": "b200", "kernel": ..., "ordinal": ...}``;
* on a B200 the clock sweep runs the full-load burner kernel (the
  reference's ``ConstantSurface(kappa=1, load=1)``), keys each sample by the
  *observed* SM clock and drops power-capped samples (``prepare_sweep``)
  before writing the CSV; a ``.meta.json`` sidecar keeps the raw records;
* ``--observer nvml`` selects the NVML energy-counter observer.

``analyze`` reads any result cache, simulated or B200:
``--mode pareto`` writes the performance / efficiency front and
``--mode difficulty`` the proportion-of-centrality curve of the space's
fitness flow graph (reference ``cli.py:367-443``).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import warnings
from pathlib import Path
from typing import Any

import numpy as np

from . import __version__, landscape, pmodel, recipes, records, search, steering
from .errors import CapabilityError, ConfigurationError, ControlRefusedError, JouleTuneError
from .hardware import CLOCK_PARAM
from .observer_hooks import AveragedPowerObserver, InstantPowerObserver, NVMLObserver
from .sensors import AveragedSensorConfig, averaged_reading, instant_energy
from .simulator import ConstantSurface, load_device
from .spaces import KernelConfig, SearchSpace

OBSERVERS = ("averaged", "instant", "nvml")

# manifest entries that always appear (with these defaults) in a report header
_MANIFEST_DEFAULTS: dict[str, Any] = {"seed": 0, "pct": 0.10, "observer": "averaged", "duration": 1.0}
_MANIFEST_FILES = ("space", "device", "samples", "model", "cache")


class RunManifest:
    """Inputs of one command run; ``to_dict`` / ``hash`` feed the report header."""

    def __init__(self, command: str, **inputs: Any):
        entries = dict(_MANIFEST_DEFAULTS)
        entries.update(inputs)
        entries["command"] = command
        self._entries = {k: v for k, v in entries.items() if v is not None}

    def __getattr__(self, name: str):
        if name.startswith("_"):
            raise AttributeError(name)
        return self._entries.get(name)

    def validate(self) -> None:
        for key in _MANIFEST_FILES:
            path = self._entries.get(key)
            if path is None or Path(path).exists():
                continue
            creates_it = key == "cache" and self.command in ("tune", "steer")
            if creates_it or (key == "device" and _is_b200_token(path)):
                continue
            raise ConfigurationError(f"--{key}: no such file: {path}")
        if not 0 <= self.pct < 1:
            raise ConfigurationError(f"--pct must be in [0, 1), got {self.pct}")
        if self.duration <= 0:
            raise ConfigurationError(f"--duration must be positive, got {self.duration}")
        if self.observer not in OBSERVERS:
            raise ConfigurationError(f"--observer must be averaged or instant, got {self.observer!r}")

    def to_dict(self) -> dict:
        return dict(self._entries)

    def hash(self) -> str:
        canonical = json.dumps(self._entries, sort_keys=True, separators=(",", ":"))
        return hashlib.sha256(canonical.encode()).hexdigest()[:16]

    def header(self) -> dict:
        return {"version": __version__, "seed": self.seed, "manifest": self.to_dict(), "manifest_hash": self.hash()}


def _is_b200_token(text: str) -> bool:
    return text == "b200" or text.startswith("b200:")


def open_device(token: str, *, seed: int = 0, kernel: str | None = None):
    """Simulated device file, B200 device file, or ``b200[:kernel[:ordinal]]``."""
    if not _is_b200_token(token):
        return load_device(token, seed=seed)
    from .b200 import B200Device

    _, *rest = token.split(":")
    name = rest[0] if rest and rest[0] else (kernel or "burner")
    return B200Device(name, int(rest[1]) if len(rest) > 1 else 0)


def _write_report(doc: dict, path: Path) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def _measurement(m: RunManifest):
    """(observers, averaged-sensor config, user metrics, constants) of a run."""
    averaged = AveragedSensorConfig(continuous_duration=m.duration)
    observer = {
        "instant": lambda: InstantPowerObserver(),
        "nvml": lambda: NVMLObserver(m.duration),
    }.get(m.observer, lambda: AveragedPowerObserver(averaged))()
    if m.total_flops is None:
        return [observer], averaged, (), {}
    return [observer], averaged, records.default_metrics(m.total_flops), {"total_flops": m.total_flops}


# -- simulate-sweep / fit --------------------------------------------------------------


def _sweep_clocks(device, points: int | None) -> list:
    grid = list(device.spec.supported_core_clocks)
    if points is None:
        return grid
    if not 2 <= points <= len(grid):
        raise ConfigurationError(f"--points must be in [2, {len(grid)}], got {points}")
    picks = sorted(set(np.linspace(0, len(grid) - 1, points).round().astype(int).tolist()))
    return [grid[i] for i in picks]


def _sweep_power(run, observer: str, cfg: AveragedSensorConfig) -> float:
    if observer == "averaged":
        return averaged_reading(run.samples, run.total_duration, cfg)
    if observer == "nvml" and run.counter_power is not None:
        return run.counter_power
    t0, t1 = run.window or (0.0, run.total_duration)
    return instant_energy(run.samples, t0, t1) / (t1 - t0)


def cmd_simulate_sweep(args) -> int:
    m = RunManifest("simulate-sweep", device=args.device, out=args.out, seed=args.seed, observer=args.observer,
                    duration=args.duration)
    m.validate()
    device = open_device(args.device, seed=args.seed, kernel="burner")
    if hasattr(device, "surface"):  # simulator: a full-load kernel scaling with the clock
        device.surface = ConstantSurface(reference_clock=device.spec.peak_clock, base_time=1e-3, kappa=1.0, load=1.0)
    cfg = AveragedSensorConfig(continuous_duration=args.duration)
    samples, raw, refused = [], [], []
    for clock in _sweep_clocks(device, args.points):
        try:
            device.set_core_clock(clock)
        except ControlRefusedError as exc:  # real device only: no sample under a label the board never ran at
            refused.append({"requested_mhz": clock, "reason": exc.reason})
            continue
        run = device.execute(KernelConfig(()), duration_hint=args.duration)
        watts = _sweep_power(run, args.observer, cfg)
        volts = device.read_voltage(clock) if device.spec.voltage_readable else None
        samples.append(pmodel.FrequencySample(frequency=clock, power=watts, voltage=volts))
        tele = run.telemetry or {}
        raw.append({"requested_mhz": clock, "observed_mhz": float(run.effective_clock), "power_w": watts,
                    "voltage_v": volts, "power_capped": bool(tele.get("power_capped", 0.0)),
                    "clock_locked": tele.get("clock_locked")})
    if hasattr(device, "release_clock"):  # real device: observed clocks, capped samples out
        device.release_clock()
        samples, dropped = steering.prepare_sweep(raw, power_limit=device.spec.tdp)
        sidecar = {"records": raw, "dropped": dropped, "refused": refused, "clock_mode": device.clock_mode}
        Path(str(args.out) + ".meta.json").write_text(json.dumps(sidecar, indent=1) + "\n")
        distinct = {round(s.frequency) for s in samples}
        if refused and len(distinct) < 4:
            # too few clocks the board actually ran at for a P(f) fit: no CSV, the refusal is the result
            raise CapabilityError(
                f"clock control refused for {len(refused)} of {len(refused) + len(raw)} sweep clocks "
                f"({refused[0]['reason']}); {len(distinct)} usable sample(s), no sweep written "
                f"(records in {args.out}.meta.json)")
    steering.write_samples_csv(samples, args.out)
    print(f"wrote {len(samples)} sweep samples to {args.out}")
    return 0


def cmd_fit(args) -> int:
    m = RunManifest("fit", samples=args.samples, device=args.device, out=args.out, pct=args.pct, seed=args.seed)
    m.validate()
    device = open_device(args.device, seed=args.seed)
    samples = steering.read_samples_csv(args.samples)
    model = pmodel.fit(samples, tdp=device.spec.tdp)
    grid = device.spec.supported_core_clocks
    f_opt = steering.optimal_frequency(model, grid)
    band = steering.frequency_band(f_opt, grid, pct=args.pct)
    ridge = None
    if len(samples) >= 4 and all(s.voltage is not None for s in samples):
        point = pmodel.detect_ridge(samples)
        ridge = None if point is None else {"frequency": point.frequency, "voltage": point.voltage}
    _write_report({**m.header(), "model": model.to_dict(), "ridge": ridge, "optimal_frequency": f_opt,
                   "band": list(band.clocks), "band_reduction": band.reduction, "supported_clocks": len(grid)},
                  Path(args.out))
    print(f"fit: p_idle={model.p_idle:.3f} W alpha={model.alpha:.6g} tau_ft={model.tau_ft:.1f} MHz "
          f"beta={model.beta:.6g} rms={model.residual_rms:.4g} W")
    print(f"optimal frequency {f_opt:.0f} MHz, band of {len(band.clocks)} clocks "
          f"({band.reduction:.1%} reduction) -> {args.out}")
    return 0


# -- tune / steer ---------------------------------------------------------------------------


def _tuning_manifest(args, command: str, **more) -> RunManifest:
    m = RunManifest(
        command, space=args.space, device=args.device, pipeline=args.pipeline, strategy=args.strategy,
        objective=args.objective, seed=args.seed, budget=args.budget, out=args.out,
        cache=args.cache or str(Path(args.out or ".") / "cache.jsonl"), observer=args.observer,
        duration=args.duration, total_flops=args.total_flops, **more,
    )
    m.validate()
    return m


def _run_tuning(m: RunManifest, space: SearchSpace, extra: dict, device=None) -> int:
    device = device if device is not None else open_device(m.device, seed=m.seed)
    observers, averaged, metrics, constants = _measurement(m)
    out_dir = Path(m.out or ".")
    out_dir.mkdir(parents=True, exist_ok=True)
    Path(m.cache).parent.mkdir(parents=True, exist_ok=True)
    cache = records.ResultCache(m.cache)
    before = device.execution_count
    common = dict(user_metrics=metrics, constants=constants, cache=cache, averaged_cfg=averaged)
    history = None
    if m.pipeline is not None:
        body = recipes.run_pipeline(m.pipeline, space, device, observers, strategy=m.strategy or "exhaustive",
                                    budget=m.budget, seed=m.seed, **common).to_dict()
    else:
        objective = records.Objective.parse(m.objective or "energy")
        run = search.TuningRun(space=space, strategy=m.strategy or "exhaustive", objective=objective, budget=m.budget,
                               seed=m.seed)
        outcome = search.run_strategy(run, device, observers, **common)
        body = {"strategy": run.strategy, "objective": f"{objective.metric}:{objective.direction}",
                "best": outcome.best.to_dict(), "evaluations": outcome.evaluations}
        history = [r.to_dict() for r in outcome.history]
    report = {**m.header(), "space_size": space.size(), "device_executions": device.execution_count - before,
              "cache_entries": len(cache), **extra, "result": body}
    if history is not None:
        report["history"] = history
    _write_report(report, out_dir / "report.json")
    best = body["best"]
    print(f"best config {best['config']} time={best['time']:.6g}s energy={best['energy']:.6g}J "
          f"({report['device_executions']} device executions) -> {out_dir / 'report.json'}")
    return 0


def cmd_tune(args) -> int:
    if args.pipeline is not None and args.strategy == "local_search" and args.budget is None:
        raise ConfigurationError("local_search pipelines need an explicit --budget")
    m = _tuning_manifest(args, "tune")
    return _run_tuning(m, SearchSpace.from_json(m.space), {})


def cmd_steer(args) -> int:
    m = _tuning_manifest(args, "steer", model=args.model, pct=args.pct)
    space = SearchSpace.from_json(m.space)
    if CLOCK_PARAM not in space.names:
        raise ConfigurationError(f"steering needs a {CLOCK_PARAM!r} parameter in the space")
    device = open_device(m.device, seed=m.seed)
    grid = device.spec.supported_core_clocks
    f_opt = steering.optimal_frequency(steering.model_from_json(m.model), grid)
    band = steering.frequency_band(f_opt, grid, pct=m.pct)
    steered = space.with_values(CLOCK_PARAM, band.clocks)
    info = {"optimal_frequency": f_opt, "band": list(band.clocks), "band_reduction": band.reduction,
            "pre_space_size": space.size(), "post_space_size": steered.size()}
    print(f"steering clocks to {len(band.clocks)} of {len(grid)} supported ({band.reduction:.1%} reduction); "
          f"space {info['pre_space_size']} -> {info['post_space_size']}")
    return _run_tuning(m, steered, {"steering": info}, device=device)


# -- analyze ------------------------------------------------------------------------------------


def cmd_analyze(args) -> int:
    pareto = args.mode == "pareto"
    m = RunManifest(
        "analyze", cache=args.cache, space=args.space, objective=args.objective, out=args.out, seed=args.seed,
        mode=args.mode, performance=args.performance if pareto else None,
        efficiency=args.efficiency if pareto else None, weights=None if pareto else args.weights,
        p_max=None if pareto else args.p_max, p_steps=None if pareto else args.p_steps,
    )
    m.validate()
    results = [r for r in records.ResultCache(args.cache).results() if not r.failed]
    if not results:
        raise JouleTuneError(f"cache {args.cache} holds no successful results")
    out_dir = Path(args.out or ".")
    out_dir.mkdir(parents=True, exist_ok=True)
    if pareto:
        points = [landscape.ParetoPoint(r.config, r.lookup(args.performance), r.lookup(args.efficiency))
                  for r in results]
        front = landscape.pareto_front(points)
        landscape.write_pareto_csv(points, front, out_dir / "pareto.csv")
        body = {"points": len(points), "front_size": len(front),
                "front": [{"config": p.config.as_dict(), "performance": p.performance, "efficiency": p.efficiency}
                          for p in front]}
        _write_report({**m.header(), **body}, out_dir / "analyze.json")
        print(f"pareto front: {len(front)} of {len(points)} points -> {out_dir}")
        return 0
    if args.space is None:
        raise ConfigurationError("--space is required for difficulty analysis")
    space = SearchSpace.from_json(args.space)
    objective = records.Objective.parse(args.objective or "energy")
    graph = landscape.build_ffg(space, {r.config: objective.fitness(r) for r in results})
    weights = landscape.minima_arrival_distribution(graph, mode=args.weights)
    curve = landscape.proportion_of_centrality(graph, weights, np.linspace(1.0, args.p_max, args.p_steps).tolist())
    landscape.write_centrality_csv(curve, out_dir / "difficulty.csv")
    body = {"objective": f"{objective.metric}:{objective.direction}", "nodes": len(graph.nodes),
            "edges": graph.edge_count(), "minima": len(graph.minima), "f_optimal": curve.f_optimal,
            "weights_mode": args.weights}
    _write_report({**m.header(), **body}, out_dir / "analyze.json")
    print(f"difficulty: {len(graph.minima)} local optima over {len(graph.nodes)} configs -> {out_dir}")
    return 0


# -- parser (flag tables) ----------------------------------------------------------------------

_TUNING_FLAGS = [
    ("--space", dict(required=True, help="search space JSON")),
    ("--device", dict(required=True, help="device spec JSON, or b200[:kernel[:ordinal]]")),
    ("--pipeline", dict(choices=recipes.PIPELINES, default=None)),
    ("--strategy", dict(choices=search.STRATEGIES, default=None)),
    ("--objective", dict(default=None, help="NAME[:min|:max], default energy")),
    ("--seed", dict(type=int, default=0)),
    ("--budget", dict(type=int, default=None, help="max device executions")),
    ("--out", dict(default=None, help="output directory")),
    ("--cache", dict(default=None, help="JSON-lines result cache")),
    ("--observer", dict(choices=list(OBSERVERS), default="averaged")),
    ("--duration", dict(type=float, default=1.0, help="continuous benchmark duration (s)")),
    ("--total-flops", dict(type=float, default=None, help="operation count; enables gflops and gflops_per_w")),
]

_COMMANDS = {
    "simulate-sweep": ("measure a full-load clock sweep", cmd_simulate_sweep, [
        ("--device", dict(required=True)),
        ("--out", dict(required=True, help="sweep CSV path")),
        ("--points", dict(type=int, default=None, help="subsample the clock grid")),
        ("--seed", dict(type=int, default=0)),
        ("--observer", dict(choices=list(OBSERVERS), default="averaged")),
        ("--duration", dict(type=float, default=1.0)),
    ]),
    "fit": ("fit the power model to a sweep CSV", cmd_fit, [
        ("--samples", dict(required=True, help="sweep CSV")),
        ("--device", dict(required=True)),
        ("--out", dict(required=True, help="model JSON path")),
        ("--pct", dict(type=float, default=0.10)),
        ("--seed", dict(type=int, default=0)),
    ]),
    "tune": ("tune a space on a device", cmd_tune, _TUNING_FLAGS),
    "steer": ("tune with the clock parameter reduced to the model band", cmd_steer, _TUNING_FLAGS + [
        ("--model", dict(required=True, help="fitted model JSON")),
        ("--pct", dict(type=float, default=0.10)),
    ]),
    "analyze": ("analyze a result cache", cmd_analyze, [
        ("--cache", dict(required=True)),
        ("--mode", dict(choices=["pareto", "difficulty"], required=True)),
        ("--space", dict(default=None, help="needed for difficulty")),
        ("--objective", dict(default=None)),
        ("--performance", dict(default="gflops")),
        ("--efficiency", dict(default="gflops_per_w")),
        ("--weights", dict(choices=list(landscape.WEIGHT_MODES), default="absorbing")),
        ("--p-max", dict(type=float, default=1.5)),
        ("--p-steps", dict(type=int, default=26)),
        ("--out", dict(default=None)),
        ("--seed", dict(type=int, default=0)),
    ]),
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="jouletune", description="Energy-aware kernel tuning on B200 GPUs")
    parser.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (help_text, handler, flags) in _COMMANDS.items():
        p = sub.add_parser(name, help=help_text)
        for flag, options in flags:
            p.add_argument(flag, **options)
        p.set_defaults(func=handler)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("default")
            return args.func(args)
    except ConfigurationError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except JouleTuneError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
