"""``tune_kernel``: the paper's Kernel-Tuner-style entry point over ``run_strategy``.

The reference package has no ``tune_kernel``; its entry
points are ``run_strategy`` / ``run_pipeline``. The paper's usage
(``PAPER.md:96, 191, 205-208``) is Kernel Tuner's::

    tune_kernel(kernel_name, kernel_source, problem_size, arguments, tune_params,
                observers=[...], metrics={...}, ...)

This façade builds ``SearchSpace.from_dict({"parameters": tune_params,
"restrictions": restrictions})`` (reference ``searchspace.py:253-264``),
binds the kernel to a :class:`~.b200.B200Device` and calls
:func:`~.tuner.run_strategy`. ``nvml_gr_clock`` / ``nvml_pwr_limit`` are
ordinary tunables (the controller applies them; ``PAPER.md:191``).

Kernels: either one of the built-in suite problems (``kernel_source=None``
and ``kernel_name`` in ``pnpoly``/``conv2d``/``sgemm``/``burner``) or any
``extern "C" __global__`` CUDA source, compiled per config for sm_100a by
NVRTC with every tunable as a ``-D`` define. Grid sizing follows Kernel
Tuner: ``grid = ceil(problem_size / (block_size * grid_div))`` per
dimension, block sizes from the ``block_size_x/y/z`` tunables.

Metrics: ``UserMetric`` expression strings (reference semantics, time in s)
or Kernel-Tuner lambdas ``{name: f(p)}`` where ``p["time"]`` is in **ms**
(Kernel Tuner's unit) and ``p["energy"]`` in J.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any, Callable, Mapping, Sequence

import numpy as np

from . import native
from .b200 import B200Device
from .gpu import DeviceArray, Launch, f32, f64, i32, i64
from .kernels import KernelProblem, make_problem
from .observer_hooks import BenchmarkObserver, NVMLObserver
from .spaces import SearchSpace
from .records import Objective, ResultCache, UserMetric, default_metrics
from .search import StrategyOutcome, TuningRun, run_strategy

__all__ = ["tune_kernel", "SourceProblem", "CallableMetric"]


@dataclass(frozen=True)
class CallableMetric(UserMetric):
    """A Kernel-Tuner-style metric ``fn(p)`` with ``p['time']`` in milliseconds."""

    fn: Callable[[Mapping[str, float]], float] = field(default=None, compare=False, repr=False)

    def evaluate(self, env: Mapping[str, float]) -> float:
        p = dict(env)
        p["time"] = env["time"] * 1e3
        return float(self.fn(p))


def _scalar(value):
    """numpy scalar types pick the C type (Kernel Tuner convention); Python
    floats are float32 and Python ints int32."""
    if type(value) is np.float64:
        return f64(value)
    if isinstance(value, (np.floating, float)):
        return f32(value)
    if type(value) is np.int64:
        return i64(value)
    if isinstance(value, (bool, int, np.integer)):
        return i32(int(value))
    raise TypeError(f"unsupported kernel argument type {type(value)}")


@dataclass
class SourceProblem(KernelProblem):
    """An arbitrary CUDA kernel, Kernel Tuner style (arguments as numpy arrays/scalars)."""

    name: str = "kernel"
    kernel_source: str = ""
    symbol: str = ""
    problem_size: tuple = (1,)
    arguments: list = field(default_factory=list)
    tune_params_doc: dict = field(default_factory=dict)
    restriction_list: list = field(default_factory=list)
    grid_div: tuple = (None, None, None)
    total_flops_value: float = 1.0
    compiler_options: tuple = ()

    @property
    def total_flops(self) -> float:
        return self.total_flops_value

    @property
    def algorithmic_bytes(self) -> float:
        return float(sum(a.nbytes for a in self.arguments if isinstance(a, np.ndarray)))

    def tune_params(self):
        return dict(self.tune_params_doc)

    def restrictions(self):
        return list(self.restriction_list)

    def default_config(self):
        return {k: v[0] for k, v in self.tune_params_doc.items() if not k.startswith("nvml_")}

    def defines(self, config):
        return {k: (int(v) if isinstance(v, bool) else v) for k, v in dict(config).items()}

    def options(self, config):
        return native._nvrtc_options(self.defines(config), tuple(self.compiler_options))

    def cubin(self, config):
        return native.compile_cubin(self.kernel_source, self.name, self.options(config))

    def launch(self, config):
        c = dict(config)
        block = tuple(int(c.get(f"block_size_{d}", default)) for d, default in zip("xyz", (256, 1, 1)))
        size = tuple(self.problem_size) + (1,) * (3 - len(self.problem_size))
        grid = []
        for dim, (n, b, div) in enumerate(zip(size, block, self.grid_div)):
            divisor = b if div is None else math.prod(int(c[name]) for name in div) if isinstance(div, (list, tuple)) \
                else int(c[div]) if isinstance(div, str) else int(div)
            grid.append(max(1, math.ceil(n / divisor)))
        return Launch(tuple(grid), block)

    def host_inputs(self):
        return {}

    def prepare(self, gpu, inputs=None):
        self.gpu = gpu
        self.inputs = {}
        self._args = []
        self.buffers = {}
        for i, a in enumerate(self.arguments):
            if isinstance(a, np.ndarray):
                buf = gpu.array(a)
                self.buffers[f"arg{i}"] = buf
                self._args.append(buf)
            else:
                self._args.append(_scalar(a))
        self._initial = [a.copy() if isinstance(a, np.ndarray) else None for a in self.arguments]

    def args(self, config):
        return self._args

    def reset_output(self):
        for i, a in enumerate(self._initial):
            if a is not None:
                self.buffers[f"arg{i}"].upload(a)

    def fetch_output(self):
        return [b.download() if isinstance(b, DeviceArray) else None for b in self._args]


def _verify_list(got, answer, config, atol: float) -> bool:
    for g, a in zip(got, answer):
        if a is None:
            continue
        if g is None or g.shape != np.asarray(a).shape:
            return False
        a = np.asarray(a)
        if np.issubdtype(a.dtype, np.floating):
            if not np.allclose(g, a, atol=atol, rtol=0):
                return False
        elif not np.array_equal(g, a):
            return False
    return True


def tune_kernel(
    kernel_name: str,
    kernel_source: str | None = None,
    problem_size=None,
    arguments: Sequence | None = None,
    tune_params: Mapping[str, Sequence] | None = None,
    *,
    restrictions: Sequence[str] = (),
    grid_div_x=None,
    grid_div_y=None,
    grid_div_z=None,
    answer: Sequence | np.ndarray | None = None,
    atol: float = 1e-6,
    verify: Callable | None = None,
    observers: Sequence[BenchmarkObserver] | None = None,
    metrics: Mapping[str, Callable] | Sequence[UserMetric] | None = None,
    constants: Mapping[str, float] | None = None,
    objective: str = "energy",
    strategy: str = "exhaustive",
    budget: int | None = None,
    seed: int = 0,
    cache: str | ResultCache | None = None,
    device: B200Device | None = None,
    ordinal: int = 0,
    total_flops: float | None = None,
    compiler_options: Sequence[str] = (),
    problem_kwargs: Mapping[str, Any] | None = None,
    duration: float = 0.25,
) -> tuple[list[dict], StrategyOutcome]:
    """Tune ``kernel_name`` on a B200; returns (results as dicts, outcome).

    Without ``tune_params`` the built-in problem's own space is used.
    """
    if kernel_source is None:
        problem = make_problem(kernel_name, **(problem_kwargs or {}))
        doc = problem.space_document() if tune_params is None else {"parameters": dict(tune_params),
                                                                    "restrictions": list(restrictions)}
    else:
        if tune_params is None or arguments is None or problem_size is None:
            raise TypeError("custom kernels need problem_size, arguments and tune_params")
        size = tuple(problem_size) if isinstance(problem_size, (list, tuple)) else (int(problem_size),)
        problem = SourceProblem(
            name=kernel_name, kernel_source=kernel_source, symbol=kernel_name, problem_size=size,
            arguments=list(arguments), tune_params_doc=dict(tune_params), restriction_list=list(restrictions),
            grid_div=(grid_div_x, grid_div_y, grid_div_z), total_flops_value=float(total_flops or 1.0),
            compiler_options=tuple(compiler_options),
        )
        doc = {"parameters": dict(tune_params), "restrictions": list(restrictions)}
    space = SearchSpace.from_dict(doc)
    if device is None:
        checker = verify
        if checker is None and answer is not None and kernel_source is not None:
            checker = lambda got, ans, cfg: _verify_list(got, ans, cfg, atol)  # noqa: E731
        device = B200Device(problem, ordinal, answer=answer, verify=checker, min_window=duration)
    observers = list(observers) if observers is not None else [NVMLObserver(duration)]
    if total_flops is not None:
        defaults, consts = default_metrics(total_flops), {"total_flops": float(total_flops)}
    else:
        defaults, consts = problem.user_metrics()
    if metrics is None:
        user_metrics: list[UserMetric] = list(defaults)
    elif isinstance(metrics, Mapping):
        user_metrics = [CallableMetric(name.replace("/", "_per_").replace(" ", "_"), "0", fn=fn)
                        if callable(fn) else UserMetric(name, fn) for name, fn in metrics.items()]
    else:
        user_metrics = list(metrics)
    consts = {**consts, **(constants or {})}
    if isinstance(cache, str):
        cache = ResultCache(cache)
    outcome = run_strategy(TuningRun(space, strategy, Objective.parse(objective), budget, seed), device, observers,
                           user_metrics=user_metrics, constants=consts, cache=cache)
    rows = [{**r.config.as_dict(), "time_ms": r.time * 1e3, "energy_j": r.energy, **r.observer_results,
             **r.metrics, "failed": r.failed} for r in outcome.history]
    return rows, outcome
