"""Thin object layer over a ``jt_ctx``: device buffers, loaded kernels, timed loops.

One :class:`GPU` per (process, CUDA ordinal). Buffers and modules are owned
by the context (freed with it). Nothing here falls back to the CPU: if libjt
or the GPU is missing, construction raises ``CapabilityError``.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import native
from .native import ARG_BLOB, ARG_F32, ARG_F64, ARG_I32, ARG_I64, ARG_PTR, JTArg, JTBenchResult, JTLaunchShape, JTSample, check

__all__ = ["GPU", "DeviceArray", "DeviceSlice", "rows", "Kernel", "Launch", "BenchRun", "i32", "f32", "f64", "i64"]


class _Scalar:
    __slots__ = ("kind", "value")

    def __init__(self, kind, value):
        self.kind, self.value = kind, value


def i32(v) -> _Scalar:
    return _Scalar(ARG_I32, int(v))


def i64(v) -> _Scalar:
    return _Scalar(ARG_I64, int(v))


def f32(v) -> _Scalar:
    return _Scalar(ARG_F32, float(v))


def f64(v) -> _Scalar:
    return _Scalar(ARG_F64, float(v))


class Blob:
    """A by-value kernel parameter (e.g. a 128-byte CUtensorMap), 64-byte aligned."""

    def __init__(self, data: bytes):
        self._raw = ctypes.create_string_buffer(len(data) + 64)
        base = ctypes.addressof(self._raw)
        self.address = (base + 63) & ~63
        ctypes.memmove(self.address, data, len(data))
        self.nbytes = len(data)


class DeviceArray:
    """A device allocation with a numpy-ish shape/dtype for host copies."""

    def __init__(self, gpu: "GPU", nbytes: int, shape=None, dtype=np.uint8):
        self.gpu = gpu
        self.nbytes = int(nbytes)
        self.dtype = np.dtype(dtype)
        self.shape = tuple(shape) if shape is not None else (self.nbytes // self.dtype.itemsize,)
        ptr = ctypes.c_ulonglong()
        check(native.lib().jt_alloc(gpu.handle, self.nbytes, ctypes.byref(ptr)), "jt_alloc")
        self.ptr = ptr.value

    def upload(self, host: np.ndarray) -> "DeviceArray":
        host = np.ascontiguousarray(host)
        if host.nbytes > self.nbytes:
            raise ValueError(f"host array ({host.nbytes} B) larger than device buffer ({self.nbytes} B)")
        check(native.lib().jt_h2d(self.gpu.handle, self.ptr, host.ctypes.data, host.nbytes), "jt_h2d")
        return self

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.shape, dtype=self.dtype)
        check(native.lib().jt_d2h(self.gpu.handle, out.ctypes.data, self.ptr, out.nbytes), "jt_d2h")
        return out

    def clone(self) -> "DeviceArray":
        """A new allocation holding the same bytes (slack included), staged through the host."""
        raw = np.empty(self.nbytes, np.uint8)
        check(native.lib().jt_d2h(self.gpu.handle, raw.ctypes.data, self.ptr, self.nbytes), "jt_d2h")
        copy = DeviceArray(self.gpu, self.nbytes, self.shape, self.dtype)
        check(native.lib().jt_h2d(self.gpu.handle, copy.ptr, raw.ctypes.data, self.nbytes), "jt_h2d")
        return copy

    def fill(self, byte: int = 0) -> None:
        check(native.lib().jt_memset_d8(self.gpu.handle, self.ptr, byte, self.nbytes), "jt_memset_d8")
        self.gpu.synchronize()

    def free(self) -> None:
        if self.ptr:
            check(native.lib().jt_free(self.gpu.handle, self.ptr), "jt_free")
            self.ptr = 0


class DeviceSlice:
    """A byte range of a :class:`DeviceArray` (kernel argument / async-copy endpoint; not owning)."""

    __slots__ = ("gpu", "ptr", "nbytes", "shape", "dtype")

    def __init__(self, base: DeviceArray, offset: int, nbytes: int, shape=None):
        if offset < 0 or nbytes < 0 or offset + nbytes > base.nbytes:
            raise ValueError(f"slice [{offset}, {offset + nbytes}) outside a {base.nbytes}-byte buffer")
        self.gpu = base.gpu
        self.ptr = base.ptr + offset
        self.nbytes = nbytes
        self.dtype = base.dtype
        self.shape = tuple(shape) if shape is not None else (nbytes // base.dtype.itemsize,)


def rows(base: DeviceArray, r0: int, r1: int) -> DeviceSlice:
    """Rows [r0, r1) of a row-major device array (its shape[1:] is the row)."""
    row = int(np.prod(base.shape[1:])) * base.dtype.itemsize if len(base.shape) > 1 else base.dtype.itemsize
    return DeviceSlice(base, r0 * row, (r1 - r0) * row, (r1 - r0, *base.shape[1:]))


@dataclass(frozen=True)
class Launch:
    grid: tuple[int, int, int]
    block: tuple[int, int, int]
    smem: int = 0
    cluster_x: int = 1

    def shape(self) -> JTLaunchShape:
        s = JTLaunchShape()
        for i in range(3):
            s.grid[i] = int(self.grid[i])
            s.block[i] = int(self.block[i])
        s.smem_bytes = int(self.smem)
        s.cluster_x = int(self.cluster_x)
        return s

    @property
    def threads(self) -> int:
        return self.block[0] * self.block[1] * self.block[2]

    @property
    def blocks(self) -> int:
        return self.grid[0] * self.grid[1] * self.grid[2]


def _pack(args: Sequence) -> ctypes.Array:
    arr = (JTArg * max(len(args), 1))()
    for i, a in enumerate(args):
        if isinstance(a, (DeviceArray, DeviceSlice)):
            arr[i].kind = ARG_PTR
            arr[i].v.ptr = a.ptr
        elif isinstance(a, Blob):
            arr[i].kind = ARG_BLOB
            arr[i].v.ptr = a.address
        elif isinstance(a, _Scalar):
            arr[i].kind = a.kind
            if a.kind == ARG_I32:
                arr[i].v.i32 = a.value
            elif a.kind == ARG_F32:
                arr[i].v.f32 = a.value
            elif a.kind == ARG_F64:
                arr[i].v.f64 = a.value
            else:
                arr[i].v.i64 = a.value
        else:
            raise TypeError(f"kernel argument {i}: expected DeviceArray or i32/f32/f64/i64 scalar, got {type(a)}")
    return arr


@dataclass
class Kernel:
    gpu: "GPU"
    module: int
    handle: int
    name: str
    regs: int = 0
    static_smem: int = 0
    local_bytes: int = 0
    max_threads: int = 0

    def set_global(self, symbol: str, host: np.ndarray) -> None:
        host = np.ascontiguousarray(host)
        check(
            native.lib().jt_module_set_global(self.gpu.handle, self.module, symbol.encode(), host.ctypes.data,
                                              host.nbytes),
            f"set {symbol}",
        )

    def occupancy(self, block_threads: int, dynamic_smem: int = 0) -> int:
        """Resident CTAs per SM at this block size and dynamic shared memory (``jt_kernel_occupancy``)."""
        n = ctypes.c_int()
        check(native.lib().jt_kernel_occupancy(self.gpu.handle, self.handle, int(block_threads), int(dynamic_smem),
                                               ctypes.byref(n)), f"occupancy {self.name}")
        return n.value


@dataclass
class BenchRun:
    """One device-timed loop plus its NVML trace (times on the jt_now clock)."""

    first_launch_s: float
    per_launch_s: float
    total_s: float
    reps: int
    loop_t0: float
    loop_t1: float
    samples: list = field(default_factory=list)  # list[JTSample-like tuples]


class GPU:
    """A libjt context on one CUDA ordinal."""

    def __init__(self, ordinal: int = 0):
        L = native.lib()
        h = ctypes.c_void_p()
        check(L.jt_open(int(ordinal), ctypes.byref(h)), f"jt_open({ordinal})")
        self.handle = h
        self.ordinal = int(ordinal)
        info = native.JTDeviceInfo()
        check(L.jt_device_info_get(self.handle, ctypes.byref(info)), "jt_device_info_get")
        self.info = info
        self._modules: dict[str, Kernel] = {}
        self._pinned: list = []

    # -- lifecycle --------------------------------------------------------
    def close(self) -> None:
        if self.handle:
            for ptr in self._pinned:
                native.lib().jt_host_free(self.handle, ptr)
            self._pinned = []
            native.lib().jt_close(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- facts --------------------------------------------------------------
    @property
    def name(self) -> str:
        return self.info.name.decode()

    @property
    def sm_count(self) -> int:
        return self.info.sm_count

    def refresh_info(self):
        check(native.lib().jt_device_info_get(self.handle, ctypes.byref(self.info)), "jt_device_info_get")
        return self.info

    def supported_clocks(self) -> list[int]:
        return [int(self.info.clocks_mhz[i]) for i in range(self.info.n_clocks)]

    # -- memory -------------------------------------------------------------
    def array(self, host: np.ndarray, *, slack: int = 0) -> DeviceArray:
        host = np.ascontiguousarray(host)
        buf = DeviceArray(self, host.nbytes + slack, host.shape, host.dtype)
        if slack:
            buf.fill(0)
        return buf.upload(host)

    def empty(self, shape, dtype=np.float32, *, slack: int = 0) -> DeviceArray:
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        return DeviceArray(self, nbytes + slack, shape, dtype)

    def synchronize(self) -> None:
        check(native.lib().jt_synchronize(self.handle), "jt_synchronize")

    # -- events / async copies (bench.py) --------------------------------------
    def reserve_events(self, n: int) -> None:
        check(native.lib().jt_events_reserve(self.handle, int(n)), "jt_events_reserve")

    def record(self, index: int) -> None:
        check(native.lib().jt_event_record(self.handle, int(index)), "jt_event_record")

    def gate(self) -> None:
        """Hold the active stream until :meth:`release` (work enqueued in between starts together)."""
        check(native.lib().jt_stream_gate(self.handle), "jt_stream_gate")

    def release(self) -> None:
        check(native.lib().jt_stream_release(self.handle), "jt_stream_release")

    def elapsed(self, start: int, stop: int) -> float:
        out = ctypes.c_double()
        check(native.lib().jt_event_elapsed(self.handle, int(start), int(stop), ctypes.byref(out)), "jt_event_elapsed")
        return out.value

    # -- streams: 0 = the context's own; copies / launches / events follow the selected one
    def reserve_streams(self, n: int) -> None:
        check(native.lib().jt_streams_reserve(self.handle, int(n)), "jt_streams_reserve")

    def use_stream(self, index: int) -> None:
        check(native.lib().jt_stream_select(self.handle, int(index)), "jt_stream_select")

    def wait_event(self, index: int) -> None:
        """The selected stream waits for event ``index`` (recorded on any stream)."""
        check(native.lib().jt_stream_wait_event(self.handle, int(index)), "jt_stream_wait_event")

    def h2d_async(self, dst: "DeviceArray", host: np.ndarray) -> None:
        check(native.lib().jt_h2d_async(self.handle, dst.ptr, host.ctypes.data, host.nbytes), "jt_h2d_async")

    def d2h_async(self, host: np.ndarray, src: "DeviceArray") -> None:
        check(native.lib().jt_d2h_async(self.handle, host.ctypes.data, src.ptr, host.nbytes), "jt_d2h_async")

    def h2d_2d_async(self, dst: "DeviceArray", dst_pitch: int, host: np.ndarray) -> None:
        """A row-major 2D host array into the top-left of a pitched device buffer (``dst_pitch`` bytes/row)."""
        host = np.ascontiguousarray(host)
        rows, row_bytes = host.shape[0], host.strides[0]
        check(native.lib().jt_h2d_2d_async(self.handle, dst.ptr, int(dst_pitch), host.ctypes.data, row_bytes,
                                            row_bytes, rows), "jt_h2d_2d_async")

    def d2h_2d_async(self, host: np.ndarray, src: "DeviceArray", src_pitch: int) -> None:
        """The top-left ``host.shape`` block of a pitched device buffer into a C-contiguous host array."""
        if not host.flags.c_contiguous:
            raise ValueError("destination must be C-contiguous")
        rows, row_bytes = host.shape[0], host.strides[0]
        check(native.lib().jt_d2h_2d_async(self.handle, host.ctypes.data, row_bytes, src.ptr, int(src_pitch),
                                            row_bytes, rows), "jt_d2h_2d_async")

    SWIZZLE_128B = 3
    SWIZZLE_128B_ATOM_32B = 4

    def tensor_map_2d(self, array: "DeviceArray", rows: int, cols: int, box_rows: int, box_cols: int,
                      swizzle: int = SWIZZLE_128B) -> Blob:
        """TMA descriptor for a row-major fp32 [rows][cols] device matrix."""
        out = ctypes.create_string_buffer(128)
        check(native.lib().jt_tensor_map_2d(self.handle, array.ptr, int(rows), int(cols), int(box_rows),
                                             int(box_cols), int(swizzle), out), "jt_tensor_map_2d")
        return Blob(out.raw)

    def pinned(self, shape, dtype=np.float32) -> np.ndarray:
        """A numpy array backed by page-locked host memory owned by this context."""
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        ptr = ctypes.c_void_p()
        check(native.lib().jt_host_alloc(self.handle, nbytes, ctypes.byref(ptr)), "jt_host_alloc")
        buf = (ctypes.c_byte * nbytes).from_address(ptr.value)
        arr = np.frombuffer(buf, dtype=dtype).reshape(shape)
        self._pinned.append(ptr)
        return arr

    def l2_flush(self) -> None:
        check(native.lib().jt_l2_flush(self.handle), "jt_l2_flush")

    # -- kernels --------------------------------------------------------------
    def load(self, cubin: bytes, name: str) -> Kernel:
        key = hashlib.sha1(cubin).hexdigest() + name
        hit = self._modules.get(key)
        if hit is not None:
            return hit
        L = native.lib()
        mod = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(cubin, len(cubin))
        check(L.jt_module_load(self.handle, buf, len(cubin), ctypes.byref(mod)), f"load {name}")
        fn = ctypes.c_void_p()
        check(L.jt_kernel_get(self.handle, mod, name.encode(), ctypes.byref(fn)), f"kernel {name}")
        regs, smem, local, mt = (ctypes.c_int() for _ in range(4))
        check(
            L.jt_kernel_attributes(self.handle, fn, ctypes.byref(regs), ctypes.byref(smem), ctypes.byref(local),
                                   ctypes.byref(mt)),
            "attributes",
        )
        k = Kernel(self, mod, fn, name, regs.value, smem.value, local.value, mt.value)
        self._modules[key] = k
        return k

    def launch(self, kernel: Kernel, launch: Launch, args: Sequence) -> None:
        packed = _pack(args)
        shape = launch.shape()
        check(native.lib().jt_launch(self.handle, kernel.handle, ctypes.byref(shape), packed, len(args)),
              f"launch {kernel.name}")

    def prepare_launch(self, kernel: Kernel, launch: Launch, args: Sequence) -> tuple:
        """Pack one launch's shape and arguments once, for :meth:`launch_prepared` in a timed loop
        (no per-launch Python argument packing between the kernels)."""
        shape = launch.shape()
        packed = _pack(args)
        return (kernel.handle, ctypes.byref(shape), packed, len(args), shape, kernel.name)

    def launch_prepared(self, prepared: tuple) -> None:
        handle, shape_ref, packed, n, _shape, name = prepared
        rc = native.lib().jt_launch(self.handle, handle, shape_ref, packed, n)
        if rc:
            check(rc, f"launch {name}")

    def time(self, kernel: Kernel, launch: Launch, args: Sequence, reps: int = 1) -> float:
        packed = _pack(args)
        shape = launch.shape()
        out = ctypes.c_double()
        check(
            native.lib().jt_time(self.handle, kernel.handle, ctypes.byref(shape), packed, len(args), int(reps),
                                 ctypes.byref(out)),
            f"time {kernel.name}",
        )
        return out.value

    def bench(
        self,
        kernel: Kernel,
        launch: Launch,
        args: Sequence,
        *,
        min_seconds: float,
        min_reps: int = 1,
        max_reps: int = 1 << 20,
        sample_period_us: int = 1000,
        sample: bool = True,
        rotate: Sequence[Sequence] = (),
    ) -> BenchRun:
        """``jt_bench``: device-timed loop + NVML trace. ``rotate``: further argument
        sets; launch i then uses set i % (1 + len(rotate)) (``jt_bench_sets``)."""
        sets = [list(args), *[list(r) for r in rotate]]
        if any(len(s) != len(args) for s in sets):
            raise ValueError("every rotated argument set needs the same arity")
        packed = _pack([a for s in sets for a in s])
        shape = launch.shape()
        res = JTBenchResult()
        cap = int(max(64, min(1 << 20, (min_seconds + 2.0) * 1e6 / max(sample_period_us, 100) + 64))) if sample else 0
        buf = (JTSample * max(cap, 1))()
        check(
            native.lib().jt_bench_sets(
                self.handle, kernel.handle, ctypes.byref(shape), packed, len(args), len(sets), float(min_seconds),
                int(min_reps), int(max_reps), int(sample_period_us), ctypes.byref(res),
                buf if sample else None, cap,
            ),
            f"bench {kernel.name}",
        )
        samples = [
            (s.t_s, s.power_w, s.power_avg_w, s.energy_j, s.energy_stamp_s, s.sm_mhz, s.mem_mhz, s.temp_c, s.reasons)
            for s in buf[: res.n_samples]
        ]
        return BenchRun(res.first_launch_s, res.per_launch_s, res.total_s, res.reps, res.loop_t0, res.host_t_done,
                        samples)

    # -- sensors / controller --------------------------------------------------
    def sample(self):
        s = JTSample()
        check(native.lib().jt_sample_now(self.handle, ctypes.byref(s)), "jt_sample_now")
        return (s.t_s, s.power_w, s.power_avg_w, s.energy_j, s.energy_stamp_s, s.sm_mhz, s.mem_mhz, s.temp_c,
                s.reasons)

    def sampler_start(self, period_us: int = 1000, cap: int = 1 << 20) -> None:
        check(native.lib().jt_sampler_start(self.handle, int(period_us), int(cap)), "jt_sampler_start")

    def sampler_stop(self, cap: int = 1 << 20) -> list:
        buf = (JTSample * cap)()
        n = ctypes.c_int()
        check(native.lib().jt_sampler_stop(self.handle, buf, cap, ctypes.byref(n)), "jt_sampler_stop")
        return [
            (s.t_s, s.power_w, s.power_avg_w, s.energy_j, s.energy_stamp_s, s.sm_mhz, s.mem_mhz, s.temp_c, s.reasons)
            for s in buf[: n.value]
        ]

    _REFUSED = (native.JT_ENOPERM, native.JT_ENOTSUP)
    #: NVML's text for the last refused controller call (e.g. "nvmlDeviceSetGpuLockedClocks: Not Supported")
    last_refusal: str | None = None

    def _control(self, status: int, what: str, tolerate: tuple[int, ...] = _REFUSED) -> bool:
        st = check(status, what, tolerate=tolerate)
        if st != native.JT_OK:
            self.last_refusal = native.last_error()
        return st == native.JT_OK

    def lock_clocks(self, mhz_min: int, mhz_max: int) -> bool:
        """True if NVML accepted the lock; False if it refused (NO_PERMISSION or
        NOT_SUPPORTED, text in ``last_refusal``): the caller decides, never raised here."""
        return self._control(native.lib().jt_clock_lock(self.handle, int(mhz_min), int(mhz_max)), "jt_clock_lock")

    def reset_clocks(self) -> bool:
        return self._control(native.lib().jt_clock_reset(self.handle), "jt_clock_reset")

    def set_app_clocks(self, mem_mhz: int, sm_mhz: int) -> bool:
        return self._control(native.lib().jt_app_clocks_set(self.handle, int(mem_mhz), int(sm_mhz)),
                             "jt_app_clocks_set", self._REFUSED + (native.JT_EINVAL,))

    def reset_app_clocks(self) -> bool:
        return self._control(native.lib().jt_app_clocks_reset(self.handle), "jt_app_clocks_reset")

    def set_power_limit(self, watts: float) -> bool:
        return self._control(native.lib().jt_power_limit_set(self.handle, int(round(watts * 1000))),
                             "jt_power_limit_set")

    def reset_power_limit(self) -> bool:
        return self._control(native.lib().jt_power_limit_reset(self.handle), "jt_power_limit_reset")

    def enforced_power_limit_w(self) -> float:
        """The limit NVML reports now (read back after a set)."""
        return self.refresh_info().power_limit_mw / 1000.0


# sample tuple field indices
T, P_INST, P_AVG, ENERGY, E_STAMP, SM_MHZ, MEM_MHZ, TEMP, REASONS = range(9)
SW_POWER_CAP = 0x4
HW_SLOWDOWN = 0x8
SW_THERMAL = 0x20
HW_THERMAL = 0x40
HW_POWER_BRAKE = 0x80


def fp32_peak_tflops(sm_count: int, mhz: float) -> float:
    """FP32 FMA peak: SMs x 128 lanes x 2 flop x clock."""
    return 2.0 * sm_count * 128 * mhz * 1e6 / 1e12


def isfinite(x) -> bool:
    return x is not None and math.isfinite(x)
