"""Host-buffer entry points of the kernel suite (what a user calls).

``conv2d(image, filt)``, ``pnpoly(points, vx, vy)`` and ``sgemm(a, b, c)``
take numpy arrays, copy the inputs to the B200 (asynchronously, fast when
the arrays are page-locked — see :func:`pinned`), launch the tuned sm_100a
kernel through libjt and copy the result back. Runners are cached per
(kernel, shape, config, device) so repeated calls reuse compiled modules and
device buffers. Configs default to the B200-tuned time-optimal ones
(:mod:`.tuned`), else the kernel's default.
"""

from __future__ import annotations

import threading
from typing import Any, Mapping

import numpy as np

from . import tuned
from .errors import ConfigurationError
from .gpu import GPU
from .kernels import KernelProblem, make_problem

__all__ = ["Runner", "conv2d", "conv2d_many", "pnpoly", "sgemm", "sgemm_tf32", "pinned", "device"]

_lock = threading.Lock()
_gpus: dict[int, GPU] = {}
_runners: dict[tuple, "Runner"] = {}


def device(ordinal: int = 0) -> GPU:
    with _lock:
        gpu = _gpus.get(ordinal)
        if gpu is None:
            gpu = _gpus[ordinal] = GPU(ordinal)
        return gpu


def pinned(shape, dtype=np.float32, ordinal: int = 0) -> np.ndarray:
    """Page-locked host array (H2D/D2H at full PCIe speed, fully async)."""
    return device(ordinal).pinned(shape, dtype)


class Runner:
    """One prepared (problem, config) on one GPU: inputs in, output out."""

    def __init__(self, problem: KernelProblem, config: Mapping[str, Any], gpu: GPU, inputs: dict[str, np.ndarray]):
        self.problem = problem
        self.config = dict(config)
        self.gpu = gpu
        problem.prepare(gpu, inputs)
        self.kernel = problem.kernel(self.config)
        self.launch_shape = problem.launch(self.config)
        self.args = problem.args(self.config)

    # event indices below EVENT_BASE are left to callers (bench.py)
    EVENT_BASE = 64
    H2D, COMPUTE, D2H = 1, 0, 2

    def run(self, uploads: Mapping[str, np.ndarray], out: np.ndarray | None = None, *,
            strips: int | None = None) -> np.ndarray:
        """H2D the inputs, launch, D2H the output.

        With ``strips`` > 1 and a problem that splits (conv2d bands, pnpoly
        chunks) the call is pipelined over three streams: the H2D of strip
        i+1 and the D2H of strip i-1 overlap the launch of strip i, so a
        PCIe-bound call costs about max(H2D, D2H) instead of their sum.
        """
        dst = self.problem.buffers["out"]
        if out is None:
            out = np.empty(dst.shape, dtype=dst.dtype)
        if strips and strips > 1:
            uploads = {k: np.ascontiguousarray(v) for k, v in uploads.items()}
            plan = self.problem.strips(self.config, uploads, out, strips)
            if plan:
                return self._pipelined(plan, out)
        return self._single(uploads, out)

    def _pipelined(self, plan, out: np.ndarray) -> np.ndarray:
        gpu, base = self.gpu, self.EVENT_BASE
        gpu.reserve_streams(3)
        gpu.reserve_events(base + 2 * len(plan))
        self.problem.bind(self.kernel, self.config)
        try:
            for i, strip in enumerate(plan):
                gpu.use_stream(self.H2D)
                for dev, host in strip.h2d:
                    gpu.h2d_async(dev, host)
                gpu.record(base + 2 * i)
                gpu.use_stream(self.COMPUTE)
                gpu.wait_event(base + 2 * i)
                gpu.launch(self.kernel, strip.launch, strip.args)
                gpu.record(base + 2 * i + 1)
                gpu.use_stream(self.D2H)
                gpu.wait_event(base + 2 * i + 1)
                for host, dev in strip.d2h:
                    gpu.d2h_async(host, dev)
        finally:
            gpu.use_stream(self.COMPUTE)
            gpu.synchronize()
        return out

    def run_many(self, partner: "Runner", uploads: list, outs: list, *, strips: int) -> list:
        """A sequence of calls pipelined across calls as well as within them.

        Call j runs on ``self`` (even j) or ``partner`` (odd j), two prepared
        copies of the same problem with their own device buffers, so the H2D of
        call j+1 and the D2H of call j-1 overlap the launches of call j. Call j
        reuses the buffers of call j-2 only after that call's kernels (input
        buffer) and D2H copies (output buffer) are done (stream events).
        """
        runners = (self, partner)
        plans = []
        for j, up in enumerate(uploads):
            r = runners[j % 2]
            up = {k: np.ascontiguousarray(v) for k, v in up.items()}
            plan = r.problem.strips(r.config, up, outs[j], max(1, strips))
            if not plan:
                raise ValueError(f"{r.problem.name} does not split into strips")
            plans.append(plan)
        gpu, base = self.gpu, self.EVENT_BASE
        n_strips = sum(len(p) for p in plans)
        gpu.reserve_streams(3)
        gpu.reserve_events(base + 2 * n_strips + 2 * len(plans))
        for r in runners:
            r.problem.bind(r.kernel, r.config)
        done_k, done_d2h = {}, {}  # call -> event index
        ev = base
        try:
            for j, plan in enumerate(plans):
                r = runners[j % 2]
                for i, strip in enumerate(plan):
                    gpu.use_stream(self.H2D)
                    if i == 0 and j >= 2:
                        gpu.wait_event(done_k[j - 2])  # call j-2 no longer reads these inputs
                    for dev, host in strip.h2d:
                        gpu.h2d_async(dev, host)
                    gpu.record(ev)
                    gpu.use_stream(self.COMPUTE)
                    gpu.wait_event(ev)
                    if i == 0 and j >= 2:
                        gpu.wait_event(done_d2h[j - 2])  # call j-2's output has left the device
                    gpu.launch(r.kernel, strip.launch, strip.args)
                    gpu.record(ev + 1)
                    gpu.use_stream(self.D2H)
                    gpu.wait_event(ev + 1)
                    for host, dev in strip.d2h:
                        gpu.d2h_async(host, dev)
                    ev += 2
                done_k[j] = ev - 1
                gpu.use_stream(self.D2H)
                gpu.record(ev)
                done_d2h[j] = ev
                ev += 1
        finally:
            gpu.use_stream(self.COMPUTE)
            gpu.synchronize()
        return outs

    def _single(self, uploads: Mapping[str, np.ndarray], out: np.ndarray) -> np.ndarray:
        gpu = self.gpu
        for name, host in uploads.items():
            gpu.h2d_async(self.problem.buffers[name], np.ascontiguousarray(host))
        self.problem.bind(self.kernel, self.config)
        gpu.launch(self.kernel, self.launch_shape, self.args)
        gpu.d2h_async(out, self.problem.buffers["out"])
        gpu.synchronize()
        return out


class PaddedRunner(Runner):
    """A problem prepared at its tile-padded size; calls copy the valid region in and out.

    Shapes the tuned kernels cannot tile exactly (conv2d 4095^2, SGEMM 1000^3) run
    on buffers padded up to the config's tile multiples, CLBlast's "indirect"
    approach: operands go in with pitched copies (the padding stays zero, so the
    extra K terms of a GEMM are 0 * 0 and conv2d outputs only read their own
    window), a row-major A is transposed and padded on the device
    (``csrc/kernels/layout.cu``) instead of on the host, and only the valid block
    of the result comes back.
    """

    def __init__(self, problem: KernelProblem, config, gpu: GPU, inputs, shape: dict[str, int]):
        super().__init__(problem, config, gpu, inputs)
        self.shape = shape  # the caller's (unpadded) sizes
        out = problem.buffers.get("out")
        if out is not None:  # inputs were prepared from zeros; padding regions start (and stay) zero
            out.fill(0)
        self._transpose = None
        self._staging = None

    def transpose_kernel(self):
        if self._transpose is None:
            from . import native

            cubin = native.compile_cubin(native.kernel_source("layout.cu"), "layout", native._nvrtc_options({}))
            self._transpose = self.gpu.load(cubin, "transpose_pad")
        return self._transpose

    def run_gemm(self, a: np.ndarray, b: np.ndarray, c: np.ndarray) -> np.ndarray:
        from .gpu import Launch, i32

        gpu, p = self.gpu, self.problem
        m, n, k = self.shape["m"], self.shape["n"], self.shape["k"]
        bufs = p.buffers
        if a.flags.f_contiguous and not a.flags.c_contiguous:  # column-major A: already the kernel's layout
            gpu.h2d_2d_async(bufs["at"], p.m * 4, a.T)
        else:
            if self._staging is None:
                self._staging = gpu.empty((m, k), np.float32)
            gpu.h2d_async(self._staging, np.ascontiguousarray(a))
            gpu.launch(self.transpose_kernel(), Launch((-(-p.k // 32), -(-p.m // 32), 1), (32, 8, 1)),
                       [bufs["at"], self._staging, i32(m), i32(k), i32(p.k), i32(p.m)])
        gpu.h2d_2d_async(bufs["b"], p.n * 4, b)
        gpu.h2d_2d_async(bufs["out"], p.n * 4, c)
        p.bind(self.kernel, self.config)
        gpu.launch(self.kernel, self.launch_shape, self.args)
        out = np.empty((m, n), np.float32)
        gpu.d2h_2d_async(out, bufs["out"], p.n * 4)
        gpu.synchronize()
        return out

    def run_conv(self, image: np.ndarray, out: np.ndarray | None) -> np.ndarray:
        gpu, p = self.gpu, self.problem
        h, w = self.shape["height"], self.shape["width"]
        gpu.h2d_2d_async(p.buffers["image"], (p.width + p.fw - 1) * 4, np.ascontiguousarray(image))
        p.bind(self.kernel, self.config)
        gpu.launch(self.kernel, self.launch_shape, self.args)
        if out is None:
            out = np.empty((h, w), np.float32)
        gpu.d2h_2d_async(out, p.buffers["out"], p.width * 4)
        gpu.synchronize()
        return out


def _choose_config(name: str, config, problem_kwargs: dict, pad: bool) -> dict:
    probe = make_problem(name, **problem_kwargs)
    if config:
        return {**probe.default_config(), **dict(config)}
    # tuned configs were tuned at the BASELINE size: padded calls take the tuned one as is, the
    # others the first that divides this shape
    candidates = [tuned.best_config(name), tuned.best_config(name, "energy_optimal"), probe.default_config()]
    if pad:
        return {**probe.default_config(), **next(c for c in candidates if c)}
    return probe.fitting_config(candidates)


def _runner(name: str, key: tuple, config, problem_kwargs: dict, inputs, ordinal: int, pad: bool = False,
            staged: bool = False) -> Runner:
    """A cached runner. ``pad``: sizes in ``problem_kwargs`` that the config cannot tile are padded up
    (``inputs`` is then a callable building zero inputs for the padded kwargs); ``staged``: always a
    :class:`PaddedRunner` (the GEMM entry points stage A through the device transpose)."""
    cfg = _choose_config(name, config, problem_kwargs, pad)
    kwargs = dict(problem_kwargs)
    if pad:
        for field_name, multiple in make_problem(name, **kwargs).tile_multiples(cfg).items():
            kwargs[field_name] = -(-kwargs[field_name] // multiple) * multiple
    padded = kwargs != problem_kwargs
    cache_key = (name, key, tuple(sorted(cfg.items())), ordinal)
    with _lock:
        hit = _runners.get(cache_key)
    if hit is None:
        problem = make_problem(name, **kwargs)
        broken = problem.broken_restrictions(cfg)
        if broken or not problem.is_valid(cfg):
            raise ConfigurationError(f"{name} config {cfg} is not valid for {kwargs}: breaks {broken or 'value lists'}")
        if padded or staged:
            hit = PaddedRunner(problem, cfg, device(ordinal), inputs(kwargs), problem_kwargs)
        else:
            hit = Runner(problem, cfg, device(ordinal), inputs(kwargs) if callable(inputs) else inputs)
        with _lock:
            _runners[cache_key] = hit
    return hit


# Measured on the B200 pool's PCIe Gen5 x16 (scripts/e2e_probe.py): concurrent H2D + D2H reach
# ~90 GB/s combined but every extra strip costs ~25 us of copy-engine turnaround, so a few
# large strips win: conv2d 4096^2 2.58 -> 1.97 ms at 4 bands, pnpoly 20M 6.30 -> 4.08 ms at 6 chunks.
CONV2D_STRIPS = 4
PNPOLY_STRIPS = 6


def conv2d(image: np.ndarray, filt: np.ndarray, *, config=None, out=None, ordinal: int = 0,
           strips: int = CONV2D_STRIPS) -> np.ndarray:
    """Valid-mode 2D correlation of a pre-padded float32 image with a 17x17-style filter
    (``strips`` row bands pipelined over copy/compute streams; 1 = one launch). Output
    sizes the config's tile does not divide run on a padded problem (:class:`PaddedRunner`)."""
    image = np.asarray(image, dtype=np.float32)
    filt = np.asarray(filt, dtype=np.float32)
    if image.ndim != 2 or filt.ndim != 2:
        raise ConfigurationError("conv2d takes a 2D image and a 2D filter")
    fh, fw = filt.shape
    h, w = image.shape[0] - fh + 1, image.shape[1] - fw + 1
    if h < 1 or w < 1:
        raise ConfigurationError(f"image {image.shape} is smaller than the filter {filt.shape}")

    def zero_inputs(kw):
        return {"image": np.zeros((kw["height"] + fh - 1, kw["width"] + fw - 1), np.float32), "filter": filt}

    r = _runner("conv2d", (h, w, fh, fw), config, {"width": w, "height": h, "fw": fw, "fh": fh}, zero_inputs,
                ordinal, pad=True)
    r.problem.inputs["filter"] = filt
    if isinstance(r, PaddedRunner):
        return r.run_conv(image, out)
    return r.run({"image": image}, out, strips=strips)


def conv2d_many(images: list, filt: np.ndarray, *, config=None, outs: list | None = None, ordinal: int = 0,
                strips: int = CONV2D_STRIPS) -> list:
    """``conv2d`` over a sequence of same-shape images, pipelined across images too: the
    upload of image j+1 and the download of result j-1 overlap the convolution of image
    j (two device buffer sets). Every image is still copied in and its result copied out."""
    filt = np.asarray(filt, dtype=np.float32)
    if not images:
        return []
    image = np.asarray(images[0], dtype=np.float32)
    fh, fw = filt.shape
    h, w = image.shape[0] - fh + 1, image.shape[1] - fw + 1
    key = (h, w, fh, fw)
    kwargs = {"width": w, "height": h, "fw": fw, "fh": fh}
    try:
        _choose_config("conv2d", config, kwargs, pad=False)
    except ConfigurationError:  # the tiles do not divide this shape: padded calls, one after the other
        outs = outs or [None] * len(images)
        return [conv2d(im, filt, config=config, out=o, ordinal=ordinal) for im, o in zip(images, outs)]
    a = _runner("conv2d", key, config, kwargs, {"image": image, "filter": filt}, ordinal)
    b = _runner("conv2d", key + ("partner",), a.config, kwargs, {"image": image, "filter": filt}, ordinal)
    for r in (a, b):
        r.problem.inputs["filter"] = filt
    if outs is None:
        outs = [np.empty((h, w), np.float32) for _ in images]
    return a.run_many(b, [{"image": np.asarray(im, dtype=np.float32)} for im in images], outs, strips=strips)


def pnpoly(points: np.ndarray, vx: np.ndarray, vy: np.ndarray, *, config=None, out=None, ordinal: int = 0,
           strips: int = PNPOLY_STRIPS, algorithm: str = "brute"):
    """int32 inside/outside bitmap for float32 points (n, 2) against a polygon
    (``strips`` point chunks pipelined over copy/compute streams; 1 = one launch).

    ``algorithm``: "brute" tests every edge (pnpoly.cu, the paper's kernel);
    "slab" locates each point's y-slab and x-position first (pnpoly_slab.cu);
    "grid" answers points in provably clean cells with one lookup and runs the
    slab search for the rest (pnpoly_grid.cu); "cells" answers the rest from
    per-cell lists of the few undecided edges (pnpoly_cells.cu). All four give
    the brute-force METHOD 2 bitmap bit for bit."""
    names = {"brute": "pnpoly", "slab": "pnpoly_slab", "grid": "pnpoly_grid", "cells": "pnpoly_cells"}
    if algorithm not in names:
        raise ConfigurationError(f"algorithm must be one of {sorted(names)}, not {algorithm!r}")
    points = np.asarray(points, dtype=np.float32)
    vx = np.asarray(vx, dtype=np.float32)
    vy = np.asarray(vy, dtype=np.float32)
    key = (points.shape[0], vx.size, vx.tobytes(), vy.tobytes())
    name = names[algorithm]
    r = _runner(name, key, config, {"n_points": points.shape[0], "n_vertices": vx.size},
                {"points": points, "vx": vx, "vy": vy}, ordinal)
    return r.run({"points": points}, out, strips=strips)


def sgemm(a: np.ndarray, b: np.ndarray, c: np.ndarray, alpha: float = 1.0, beta: float = 0.0, *, config=None,
          ordinal: int = 0) -> np.ndarray:
    """alpha * a @ b + beta * c in FP32 (a is staged column-major, as BLAS 'N')."""
    return _gemm("sgemm", a, b, c, alpha, beta, config, ordinal)


def sgemm_tf32(a: np.ndarray, b: np.ndarray, c: np.ndarray, alpha: float = 1.0, beta: float = 0.0, *, config=None,
               ordinal: int = 0) -> np.ndarray:
    """The same product on the tcgen05 tensor cores: TF32 inputs, FP32 accumulation
    (oracle SGEMM_TF32_TOL). Shapes must be multiples of the config's tile (M % 128 or
    % 256 for the CTA-pair kernel, N % BN, K % 32)."""
    return _gemm("sgemm_tf32", a, b, c, alpha, beta, config, ordinal)


def _gemm(name, a, b, c, alpha, beta, config, ordinal) -> np.ndarray:
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    c = np.asarray(c, dtype=np.float32)
    if a.ndim != 2 or b.ndim != 2 or c.ndim != 2 or a.shape[1] != b.shape[0] or c.shape != (a.shape[0], b.shape[1]):
        raise ConfigurationError(f"{name}: shapes {a.shape} x {b.shape} + {c.shape} do not form a GEMM")
    m, k = a.shape
    n = b.shape[1]

    def zero_inputs(kw):
        return {"a": np.zeros((kw["m"], kw["k"]), np.float32), "b": np.zeros((kw["k"], kw["n"]), np.float32),
                "c0": np.zeros((kw["m"], kw["n"]), np.float32)}

    r = _runner(name, (m, n, k, float(alpha), float(beta)), config,
                {"m": m, "n": n, "k": k, "alpha": float(alpha), "beta": float(beta)}, zero_inputs, ordinal, pad=True,
                staged=True)
    return r.run_gemm(a, b, c)
