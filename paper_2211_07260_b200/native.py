"""ctypes binding of ``libjt`` (include/jt.h) plus its in-tree build.

This is the only module that talks to the C-ABI. It maps ``jt_status``
codes onto the reference's exception convention (``errors.py``):

=============  ===========================  ==================================
status         exception                    tuner behaviour (tuner.py:242-271)
=============  ===========================  ==================================
JT_EINVAL      ConfigurationError           re-raised (caller mistake)
JT_ENOGPU      CapabilityError              config fails
JT_ECUDA       DomainError                  config fails
JT_ECOMPILE    DomainError                  config fails (e.g. smem overflow)
JT_ELAUNCH     DomainError                  config fails (launch shape)
JT_ENVML       CapabilityError              config fails
JT_ENOPERM     (returned, not raised)       observed clock recorded instead
JT_ENOTSUP     CapabilityError              config fails
=============  ===========================  ==================================

There is no CPU fallback anywhere: without the library or a GPU every entry
point raises.
"""

from __future__ import annotations

import ctypes
import functools
import hashlib
import os
import subprocess
import threading
from pathlib import Path

from .errors import CapabilityError, ConfigurationError, DomainError, JouleTuneError

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
KERNEL_DIR = CSRC / "kernels"
LIB_PATH = PKG_DIR / "libjt.so"
INCLUDE_DIR = REPO_DIR / "include"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
ARCH = "sm_100a"

JT_OK, JT_EINVAL, JT_ENOGPU, JT_ECUDA, JT_ECOMPILE, JT_ELAUNCH, JT_ENVML, JT_ENOPERM, JT_ENOTSUP = range(9)
ARG_PTR, ARG_I32, ARG_F32, ARG_F64, ARG_I64, ARG_BLOB = range(6)

# every function include/jt.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "jt_abi_version", "jt_now", "jt_last_error", "jt_device_count", "jt_open", "jt_close",
    "jt_device_info_get", "jt_alloc", "jt_free", "jt_host_alloc", "jt_host_free", "jt_h2d", "jt_d2h",
    "jt_memset_d8", "jt_synchronize", "jt_compile", "jt_free_image", "jt_module_load", "jt_module_unload",
    "jt_kernel_get", "jt_kernel_attributes", "jt_launch", "jt_time", "jt_bench", "jt_bench_sets", "jt_l2_flush",
    "jt_sample_now", "jt_sampler_start", "jt_sampler_stop", "jt_clock_lock", "jt_clock_reset",
    "jt_app_clocks_set", "jt_app_clocks_reset", "jt_power_limit_set", "jt_power_limit_reset",
    "jt_pnpoly_edges", "jt_module_set_global", "jt_events_reserve", "jt_event_record", "jt_event_elapsed",
    "jt_h2d_async", "jt_d2h_async", "jt_tensor_map_2d", "jt_streams_reserve", "jt_stream_select",
    "jt_stream_wait_event", "jt_pnpoly_slabs", "jt_pnpoly_grid", "jt_pnpoly_cells", "jt_h2d_2d_async",
    "jt_d2h_2d_async", "jt_nvrtc_version", "jt_kernel_occupancy", "jt_stream_gate", "jt_stream_release",
)


class JTSlabInfo(ctypes.Structure):
    _fields_ = [
        ("nu", ctypes.c_int), ("ng", ctypes.c_int), ("ne", ctypes.c_int), ("max_band", ctypes.c_int),
        ("u_off", ctypes.c_int), ("guess_off", ctypes.c_int), ("band_off", ctypes.c_int), ("pair_off", ctypes.c_int),
        ("words", ctypes.c_int), ("ybase", ctypes.c_float), ("yscale", ctypes.c_float),
        ("xlo_off", ctypes.c_int), ("pmax_off", ctypes.c_int), ("xpar_off", ctypes.c_int), ("xst_off", ctypes.c_int),
        ("xb", ctypes.c_int), ("half_off", ctypes.c_int),
    ]


class JTDeviceInfo(ctypes.Structure):
    _fields_ = [
        ("ordinal", ctypes.c_int),
        ("cc_major", ctypes.c_int),
        ("cc_minor", ctypes.c_int),
        ("sm_count", ctypes.c_int),
        ("max_smem_optin", ctypes.c_int),
        ("l2_bytes", ctypes.c_int),
        ("total_mem", ctypes.c_ulonglong),
        ("name", ctypes.c_char * 128),
        ("pci_bus_id", ctypes.c_char * 32),
        ("nvml_ok", ctypes.c_int),
        ("energy_counter_ok", ctypes.c_int),
        ("instant_power_ok", ctypes.c_int),
        ("n_clocks", ctypes.c_uint),
        ("clocks_mhz", ctypes.c_uint * 512),
        ("mem_clock_mhz", ctypes.c_uint),
        ("max_sm_clock_mhz", ctypes.c_uint),
        ("default_sm_clock_mhz", ctypes.c_uint),
        ("power_limit_min_mw", ctypes.c_uint),
        ("power_limit_max_mw", ctypes.c_uint),
        ("power_limit_default_mw", ctypes.c_uint),
        ("power_limit_mw", ctypes.c_uint),
        ("tdp_mw", ctypes.c_uint),
    ]


class JTSample(ctypes.Structure):
    _fields_ = [
        ("t_s", ctypes.c_double),
        ("power_w", ctypes.c_double),
        ("power_avg_w", ctypes.c_double),
        ("energy_j", ctypes.c_double),
        ("energy_stamp_s", ctypes.c_double),
        ("sm_mhz", ctypes.c_uint),
        ("mem_mhz", ctypes.c_uint),
        ("temp_c", ctypes.c_uint),
        ("pad", ctypes.c_uint),
        ("reasons", ctypes.c_ulonglong),
    ]


class _ArgValue(ctypes.Union):
    _fields_ = [
        ("ptr", ctypes.c_ulonglong),
        ("i64", ctypes.c_longlong),
        ("f64", ctypes.c_double),
        ("f32", ctypes.c_float),
        ("i32", ctypes.c_int),
    ]


class JTArg(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("pad", ctypes.c_int), ("v", _ArgValue)]


class JTLaunchShape(ctypes.Structure):
    _fields_ = [
        ("grid", ctypes.c_uint * 3),
        ("block", ctypes.c_uint * 3),
        ("smem_bytes", ctypes.c_uint),
        ("cluster_x", ctypes.c_uint),
    ]


class JTBenchResult(ctypes.Structure):
    _fields_ = [
        ("first_launch_s", ctypes.c_double),
        ("per_launch_s", ctypes.c_double),
        ("total_s", ctypes.c_double),
        ("reps", ctypes.c_int),
        ("n_samples", ctypes.c_int),
        ("host_t_enqueue", ctypes.c_double),
        ("host_t_done", ctypes.c_double),
        ("loop_t0", ctypes.c_double),
    ]


# -- build -------------------------------------------------------------------------


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/jt.cpp into the in-tree libjt.so (host code; the kernels
    are compiled per config for sm_100a by NVRTC through jt_compile)."""
    src = CSRC / "jt.cpp"
    header = INCLUDE_DIR / "jt.h"
    if LIB_PATH.exists() and not force:
        newest = max(src.stat().st_mtime, header.stat().st_mtime)
        if LIB_PATH.stat().st_mtime >= newest:
            return LIB_PATH
    cmd = [
        "g++", "-std=c++17", "-O2", "-g", "-ffp-contract=off", "-fPIC", "-shared", "-Wall", "-Wextra",
        "-Wno-unused-parameter", f"-I{INCLUDE_DIR}", f"-I{CUDA_HOME / 'include'}", str(src),
        "-o", str(LIB_PATH) + ".tmp", f"-L{CUDA_HOME / 'lib64'}", f"-Wl,-rpath,{CUDA_HOME / 'lib64'}",
        f'-DJT_CUDA_LIB_DIR="{CUDA_HOME / "lib64"}"',
        "-ldl", "-lpthread",  # NVRTC is dlopen'ed by full path (jt.cpp nvrtc_load)
    ]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(str(LIB_PATH) + ".tmp", LIB_PATH)
    return LIB_PATH


# -- loading -------------------------------------------------------------------------

_lib = None
_lib_lock = threading.Lock()


def _declare(lib) -> None:
    c = ctypes
    P = c.c_void_p
    sig = {
        "jt_abi_version": (c.c_int, []),
        "jt_now": (c.c_double, []),
        "jt_last_error": (c.c_char_p, []),
        "jt_device_count": (c.c_int, [c.POINTER(c.c_int)]),
        "jt_open": (c.c_int, [c.c_int, c.POINTER(P)]),
        "jt_close": (c.c_int, [P]),
        "jt_device_info_get": (c.c_int, [P, c.POINTER(JTDeviceInfo)]),
        "jt_alloc": (c.c_int, [P, c.c_size_t, c.POINTER(c.c_ulonglong)]),
        "jt_free": (c.c_int, [P, c.c_ulonglong]),
        "jt_host_alloc": (c.c_int, [P, c.c_size_t, c.POINTER(P)]),
        "jt_host_free": (c.c_int, [P, P]),
        "jt_h2d": (c.c_int, [P, c.c_ulonglong, P, c.c_size_t]),
        "jt_d2h": (c.c_int, [P, P, c.c_ulonglong, c.c_size_t]),
        "jt_memset_d8": (c.c_int, [P, c.c_ulonglong, c.c_ubyte, c.c_size_t]),
        "jt_synchronize": (c.c_int, [P]),
        "jt_compile": (
            c.c_int,
            [c.c_char_p, c.c_char_p, c.POINTER(c.c_char_p), c.c_int, c.POINTER(P), c.POINTER(c.c_size_t),
             c.c_char_p, c.c_size_t],
        ),
        "jt_free_image": (None, [P]),
        "jt_nvrtc_version": (c.c_int, [c.POINTER(c.c_int), c.POINTER(c.c_int), c.c_char_p, c.c_size_t]),
        "jt_module_load": (c.c_int, [P, P, c.c_size_t, c.POINTER(P)]),
        "jt_module_unload": (c.c_int, [P, P]),
        "jt_kernel_get": (c.c_int, [P, P, c.c_char_p, c.POINTER(P)]),
        "jt_kernel_attributes": (
            c.c_int, [P, P, c.POINTER(c.c_int), c.POINTER(c.c_int), c.POINTER(c.c_int), c.POINTER(c.c_int)]
        ),
        "jt_kernel_occupancy": (c.c_int, [P, P, c.c_int, c.c_size_t, c.POINTER(c.c_int)]),
        "jt_launch": (c.c_int, [P, P, c.POINTER(JTLaunchShape), c.POINTER(JTArg), c.c_int]),
        "jt_time": (
            c.c_int, [P, P, c.POINTER(JTLaunchShape), c.POINTER(JTArg), c.c_int, c.c_int, c.POINTER(c.c_double)]
        ),
        "jt_bench": (
            c.c_int,
            [P, P, c.POINTER(JTLaunchShape), c.POINTER(JTArg), c.c_int, c.c_double, c.c_int, c.c_int, c.c_int,
             c.POINTER(JTBenchResult), c.POINTER(JTSample), c.c_int],
        ),
        "jt_bench_sets": (
            c.c_int,
            [P, P, c.POINTER(JTLaunchShape), c.POINTER(JTArg), c.c_int, c.c_int, c.c_double, c.c_int, c.c_int,
             c.c_int, c.POINTER(JTBenchResult), c.POINTER(JTSample), c.c_int],
        ),
        "jt_l2_flush": (c.c_int, [P]),
        "jt_events_reserve": (c.c_int, [P, c.c_int]),
        "jt_event_record": (c.c_int, [P, c.c_int]),
        "jt_event_elapsed": (c.c_int, [P, c.c_int, c.c_int, c.POINTER(c.c_double)]),
        "jt_h2d_async": (c.c_int, [P, c.c_ulonglong, P, c.c_size_t]),
        "jt_streams_reserve": (c.c_int, [P, c.c_int]),
        "jt_stream_select": (c.c_int, [P, c.c_int]),
        "jt_stream_wait_event": (c.c_int, [P, c.c_int]),
        "jt_stream_gate": (c.c_int, [P]),
        "jt_stream_release": (c.c_int, [P]),
        "jt_tensor_map_2d": (c.c_int, [P, c.c_ulonglong, c.c_ulonglong, c.c_ulonglong, c.c_uint, c.c_uint, c.c_int, P]),
        "jt_d2h_async": (c.c_int, [P, P, c.c_ulonglong, c.c_size_t]),
        "jt_h2d_2d_async": (c.c_int, [P, c.c_ulonglong, c.c_size_t, P, c.c_size_t, c.c_size_t, c.c_size_t]),
        "jt_d2h_2d_async": (c.c_int, [P, P, c.c_size_t, c.c_ulonglong, c.c_size_t, c.c_size_t, c.c_size_t]),
        "jt_sample_now": (c.c_int, [P, c.POINTER(JTSample)]),
        "jt_sampler_start": (c.c_int, [P, c.c_int, c.c_int]),
        "jt_sampler_stop": (c.c_int, [P, c.POINTER(JTSample), c.c_int, c.POINTER(c.c_int)]),
        "jt_clock_lock": (c.c_int, [P, c.c_uint, c.c_uint]),
        "jt_clock_reset": (c.c_int, [P]),
        "jt_app_clocks_set": (c.c_int, [P, c.c_uint, c.c_uint]),
        "jt_app_clocks_reset": (c.c_int, [P]),
        "jt_power_limit_set": (c.c_int, [P, c.c_uint]),
        "jt_power_limit_reset": (c.c_int, [P]),
        "jt_pnpoly_edges": (c.c_int, [P, P, c.c_int, c.c_int, P, P]),
        "jt_pnpoly_slabs": (c.c_int, [P, P, c.c_int, c.c_int, c.c_int, c.c_int, P, c.c_longlong,
                                      c.POINTER(JTSlabInfo)]),
        "jt_pnpoly_grid": (c.c_int, [P, P, c.c_int, c.c_int, c.c_int, P, P, c.c_longlong, c.POINTER(c.c_int)]),
        "jt_pnpoly_cells": (c.c_int, [P, P, c.c_int, c.c_int, c.c_int, c.c_int, c.c_int, P, P, c.c_longlong, P,
                                      c.c_longlong, P, c.c_longlong, P]),
        "jt_module_set_global": (c.c_int, [P, P, c.c_char_p, P, c.c_size_t]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded libjt (raises if it was never built: there is no fallback)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise CapabilityError(
                        f"{LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(no CPU fallback exists)"
                    )
                handle = ctypes.CDLL(str(LIB_PATH))
                _declare(handle)
                _lib = handle
    return _lib


def last_error() -> str:
    raw = lib().jt_last_error()
    return raw.decode(errors="replace") if raw else ""


_EXC = {
    JT_EINVAL: ConfigurationError,
    JT_ENOGPU: CapabilityError,
    JT_ECUDA: DomainError,
    JT_ECOMPILE: DomainError,
    JT_ELAUNCH: DomainError,
    JT_ENVML: CapabilityError,
    JT_ENOTSUP: CapabilityError,
}


class NativeError(JouleTuneError):
    pass


def check(status: int, what: str = "", *, tolerate: tuple[int, ...] = (JT_ENOPERM,)) -> int:
    """Raise the mapped exception for a non-OK status; ``tolerate`` codes are returned."""
    if status == JT_OK or status in tolerate:
        return status
    msg = last_error()
    exc = _EXC.get(status, NativeError)
    raise exc(f"{what}: {msg}" if what else msg)


def now() -> float:
    return lib().jt_now()


# -- per-config kernel compilation with an on-disk cubin cache -----------------------

CUBIN_CACHE = Path(os.environ.get("JT_CUBIN_CACHE", PKG_DIR / "_cubins"))


def _nvrtc_options(defines: dict, extra: tuple[str, ...] = ()) -> list[str]:
    opts = [f"--gpu-architecture={ARCH}", "-std=c++17", "-lineinfo", "--extra-device-vectorization"]
    opts += [f"-D{k}={int(v) if isinstance(v, bool) else v}" for k, v in sorted(defines.items())]
    opts += list(extra)
    return opts


def kernel_source(filename: str) -> str:
    return (KERNEL_DIR / filename).read_text()


@functools.lru_cache(maxsize=1)
def nvrtc_version() -> tuple[int, int, str]:
    """(major, minor, library path) of the NVRTC behind jt_compile."""
    major, minor = ctypes.c_int(), ctypes.c_int()
    path = ctypes.create_string_buffer(4096)
    check(lib().jt_nvrtc_version(ctypes.byref(major), ctypes.byref(minor), path, len(path)), "jt_nvrtc_version")
    return major.value, minor.value, path.value.decode()


def cubin_key(source: str, options: list[str]) -> str:
    h = hashlib.sha256()
    h.update("nvrtc {}.{}\0".format(*nvrtc_version()[:2]).encode())  # a cubin belongs to its compiler
    h.update(source.encode())
    for o in options:
        h.update(b"\0" + o.encode())
    return h.hexdigest()[:40]


def compile_cubin(source: str, name: str, options: list[str], *, use_cache: bool = True) -> bytes:
    """NVRTC-compile ``source`` for sm_100a (thread safe, no GPU needed)."""
    key = cubin_key(source, options)
    path = CUBIN_CACHE / f"{name}-{key}.cubin"
    if use_cache and path.exists():
        return path.read_bytes()
    L = lib()
    arr = (ctypes.c_char_p * len(options))(*[o.encode() for o in options])
    image = ctypes.c_void_p()
    size = ctypes.c_size_t()
    log = ctypes.create_string_buffer(1 << 16)
    status = L.jt_compile(source.encode(), f"{name}.cu".encode(), arr, len(options), ctypes.byref(image),
                          ctypes.byref(size), log, len(log))
    if status != JT_OK:
        raise DomainError(f"{last_error()}\n{log.value.decode(errors='replace')[-4000:]}")
    try:
        blob = ctypes.string_at(image, size.value)
    finally:
        L.jt_free_image(image)
    if use_cache:
        CUBIN_CACHE.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".tmp{os.getpid()}.{threading.get_ident()}")
        tmp.write_bytes(blob)
        os.replace(tmp, path)
    return blob


def pnpoly_edges(vx, vy, method: int):
    """Edge table for csrc/kernels/pnpoly.cu, computed by libjt in float32."""
    import numpy as np

    vx = np.ascontiguousarray(vx, dtype=np.float32)
    vy = np.ascontiguousarray(vy, dtype=np.float32)
    n = vx.size
    edges = np.zeros((n, 4), dtype=np.float32)
    ybounds = np.zeros((n, 2), dtype=np.float32)
    check(
        lib().jt_pnpoly_edges(vx.ctypes.data, vy.ctypes.data, n, int(method), edges.ctypes.data, ybounds.ctypes.data),
        "jt_pnpoly_edges",
    )
    return edges, ybounds


def pnpoly_slabs(vx, vy, buckets: int, pad: int, xbuckets: int = 0):
    """Slab table for csrc/kernels/pnpoly_slab.cu (libjt ``jt_pnpoly_slabs``):
    returns (table as float32 words, JTSlabInfo)."""
    import numpy as np

    vx = np.ascontiguousarray(vx, dtype=np.float32)
    vy = np.ascontiguousarray(vy, dtype=np.float32)
    info = JTSlabInfo()
    L = lib()
    check(L.jt_pnpoly_slabs(vx.ctypes.data, vy.ctypes.data, vx.size, int(buckets), int(pad), int(xbuckets), None, 0,
                            ctypes.byref(info)), "jt_pnpoly_slabs")
    table = np.zeros(info.words, dtype=np.float32)
    check(L.jt_pnpoly_slabs(vx.ctypes.data, vy.ctypes.data, vx.size, int(buckets), int(pad), int(xbuckets), table.ctypes.data,
                            table.size, ctypes.byref(info)), "jt_pnpoly_slabs")
    return table, info


def pnpoly_grid(vx, vy, gw: int, gh: int):
    """Uniform-cell fast-path bits for csrc/kernels/pnpoly_grid.cu (libjt ``jt_pnpoly_grid``):
    returns (uint32 words, 2 bits per cell), params {x0, sx, y0, sy} and the clean-cell count."""
    import numpy as np

    vx = np.ascontiguousarray(vx, dtype=np.float32)
    vy = np.ascontiguousarray(vy, dtype=np.float32)
    params = np.zeros(4, dtype=np.float32)
    words = np.zeros((gw * gh + 15) // 16, dtype=np.uint32)
    clean = ctypes.c_int()
    check(lib().jt_pnpoly_grid(vx.ctypes.data, vy.ctypes.data, vx.size, int(gw), int(gh), params.ctypes.data,
                               words.ctypes.data, words.size, ctypes.byref(clean)), "jt_pnpoly_grid")
    return words, params, clean.value


def pnpoly_cells(vx, vy, gw: int, gh: int, lmax: int, head_words: int = 4):
    """Per-cell edge lists for csrc/kernels/pnpoly_cells.cu (libjt ``jt_pnpoly_cells``): returns
    (uint32 words, 2-bit codes, 16 cells per word), params {sx, ox, sy, oy}, uint32 heads
    (head_words per cell), float32 edge entries (k, 4) and stats {entries, decided, listed,
    fallback}."""
    import numpy as np

    vx = np.ascontiguousarray(vx, dtype=np.float32)
    vy = np.ascontiguousarray(vy, dtype=np.float32)
    params = np.zeros(4, dtype=np.float32)
    stats = np.zeros(4, dtype=np.int64)
    args = (vx.ctypes.data, vy.ctypes.data, vx.size, int(gw), int(gh), int(lmax), int(head_words), params.ctypes.data)
    check(lib().jt_pnpoly_cells(*args, None, 0, None, 0, None, 0, stats.ctypes.data), "jt_pnpoly_cells")
    words = np.zeros((gw * gh + 15) // 16, dtype=np.uint32)
    heads = np.zeros(int(head_words) * gw * gh, dtype=np.uint32)
    edges = np.zeros((max(1, int(stats[0])), 4), dtype=np.float32)
    check(lib().jt_pnpoly_cells(*args, words.ctypes.data, words.size, heads.ctypes.data, heads.size,
                                edges.ctypes.data, edges.shape[0], stats.ctypes.data), "jt_pnpoly_cells")
    return words, params, heads, edges, stats
