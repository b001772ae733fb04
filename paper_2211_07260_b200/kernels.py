"""The tuned kernel suite: problem definitions, tunable spaces, launch geometry.

Each :class:`KernelProblem` binds one sm_100a kernel source
(``csrc/kernels/*.cu``) to a synthetic, seeded input of the size
``BASELINE.json`` names, the Kernel-Tuner-style tunable-parameter dict
(``{"parameters": {name: [values]}, "restrictions": [expr]}``, the format of
the reference's ``SearchSpace.from_dict``, ``searchspace.py:253-264``), the
per-config ``-D`` defines, the launch shape and the algorithmic work used for
``gflops`` / ``gflops_per_w`` (``tuner.default_metrics``) and rooflines.

Inputs, all float32 from ``np.random.default_rng(seed)``:

* PnPoly: 20,000,000 points uniform in [-1,1]^2 (seed 4); a 600-vertex
  star-shaped polygon (sorted angles, radius 0.5 + 0.3 U); int32 bitmap.
* Conv2D: (4096+16)^2 input U[0,1) and a 17x17 filter U[0,1) (seed 3);
  4096^2 valid-mode output.
* SGEMM: A, B, C0 U[-1,1) 4096^2 (seeds 0/1/2), alpha 1, beta 0.5;
  A column-major, B and C row-major.

The kernels never see the oracle; verification against a user-provided
``answer`` happens in :mod:`.b200` and in the tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any, Mapping

import numpy as np

from . import native
from .gpu import GPU, Kernel, Launch, f32, i32, rows
from .records import UserMetric, default_metrics
from .spaces import KernelConfig, SearchSpace

__all__ = [
    "KernelProblem",
    "PnPolyProblem",
    "PnPolySlabProblem",
    "PnPolyGridProblem",
    "Conv2DProblem",
    "SgemmProblem",
    "SgemmTF32Problem",
    "BurnerProblem",
    "PROBLEMS",
    "make_problem",
]


@dataclass
class Strip:
    """One stage of a host-buffer pipeline: H2D copies, one launch, D2H copies.

    Consecutive strips run on three streams (H2D / compute / D2H) so the
    copies of strip i+1 and i-1 overlap the launch of strip i.
    """

    h2d: list  # [(DeviceSlice, host ndarray)]
    launch: Launch
    args: list
    d2h: list  # [(host ndarray, DeviceSlice)]


@dataclass
class KernelProblem:
    """Base class: subclasses fill the hooks below."""

    name: str = ""
    source: str = ""
    symbol: str = ""
    seed: int = 0
    # filled by prepare()
    gpu: GPU | None = field(default=None, repr=False)
    buffers: dict = field(default_factory=dict, repr=False)

    # -- description ------------------------------------------------------
    @property
    def total_flops(self) -> float:
        raise NotImplementedError

    @property
    def algorithmic_bytes(self) -> float:
        raise NotImplementedError

    #: "fp32" (FFMA-pipe roofline) or "issue" (lane-instruction roofline)
    roofline_kind = "fp32"

    def user_metrics(self) -> tuple[tuple, dict[str, float]]:
        """(tuner user metrics, their constants): ``gflops`` / ``gflops_per_w`` over
        the algorithmic flop count (``tuner.default_metrics``)."""
        return default_metrics(self.total_flops), {"total_flops": self.total_flops}

    def tune_params(self) -> dict[str, list]:
        raise NotImplementedError

    def restrictions(self) -> list[str]:
        return []

    def space_document(self) -> dict[str, Any]:
        return {"parameters": self.tune_params(), "restrictions": self.restrictions()}

    def space(self) -> SearchSpace:
        return SearchSpace.from_dict(self.space_document())

    def default_config(self) -> dict[str, Any]:
        raise NotImplementedError

    def is_valid(self, config: Mapping[str, Any]) -> bool:
        """Config satisfies this problem's value lists and restrictions."""
        merged = {**self.default_config(), **_as_dict(config)}
        space = self.space()
        return space.is_valid(KernelConfig.from_dict({k: merged[k] for k in space.names}))

    def fitting_config(self, preferred: list) -> dict[str, Any]:
        """First valid config among ``preferred`` (None entries skipped).

        Raises ``ConfigurationError`` naming the restrictions the first candidate
        breaks when none fits this problem's shape (no search over the space)."""
        from .errors import ConfigurationError

        candidates = [c for c in preferred if c]
        for cfg in candidates:
            if self.is_valid(cfg):
                return {**self.default_config(), **cfg}
        first = {**self.default_config(), **(candidates[0] if candidates else {})}
        broken = self.broken_restrictions(first)
        raise ConfigurationError(f"{self.name}: no tuned or default config fits this shape; {first} breaks "
                                 f"{broken or 'the value lists'}")

    def broken_restrictions(self, config: Mapping[str, Any]) -> list[str]:
        """The restriction expressions ``config`` violates on this problem's shape."""
        from .expressions import Expression

        env = {**self.default_config(), **_as_dict(config)}
        return [r for r in self.restrictions() if not Expression(r)(env)]

    def defines(self, config: Mapping[str, Any]) -> dict[str, Any]:
        return {k.upper(): v for k, v in config.items()}

    def tile_multiples(self, config: Mapping[str, Any]) -> dict[str, int]:
        """Problem-size fields and the multiple ``config`` needs each of them to be
        (the host API pads other shapes up to these, ``suite``); {} = any size."""
        return {}

    def launch(self, config: Mapping[str, Any]) -> Launch:
        raise NotImplementedError

    # -- device side ----------------------------------------------------------
    def host_inputs(self) -> dict[str, np.ndarray]:
        raise NotImplementedError

    def prepare(self, gpu: GPU) -> None:
        raise NotImplementedError

    def args(self, config: Mapping[str, Any]) -> list:
        raise NotImplementedError

    def bind(self, kernel: Kernel, config: Mapping[str, Any]) -> None:
        """Per-run constant-memory uploads (no-op by default)."""

    def reset_output(self) -> None:
        """Zero the output so a stale result can never pass verification."""
        out = self.buffers.get("out")
        if out is not None:
            out.fill(0)

    def fetch_output(self) -> np.ndarray:
        return self.buffers["out"].download()

    def strips(self, config, uploads: Mapping[str, np.ndarray], out: np.ndarray, n: int) -> list[Strip] | None:
        """Split one host-buffer call into ~n independent strips (None: not splittable)."""
        return None

    #: buffers a rotated argument set replaces: the streamed inputs and the output
    rotating = ("out",)

    def rotation_sets(self, config: Mapping[str, Any], n: int) -> list[list]:
        """``n - 1`` argument sets besides :meth:`args`, each over its own copies of the
        ``rotating`` buffers (kept in ``buffers`` as ``key@j``), for loops that must not
        re-read an L2-warm input (``GPU.bench(..., rotate=...)``). Tables stay shared."""
        base = self.args(config)
        sets = []
        for j in range(1, n):
            swap = {}
            for key in self.rotating:
                name = f"{key}@{j}"
                if name not in self.buffers:
                    self.buffers[name] = self.buffers[key].clone()
                swap[id(self.buffers[key])] = self.buffers[name]
            sets.append([swap.get(id(a), a) for a in base])
        return sets

    # -- compilation ------------------------------------------------------------
    def options(self, config: Mapping[str, Any]) -> list[str]:
        return native._nvrtc_options(self.defines(config))

    def cubin(self, config: Mapping[str, Any]) -> bytes:
        return native.compile_cubin(native.kernel_source(self.source), self.name, self.options(config))

    def kernel(self, config: Mapping[str, Any]) -> Kernel:
        if self.gpu is None:
            raise RuntimeError(f"{self.name}: prepare(gpu) first")
        return self.gpu.load(self.cubin(config), self.symbol)


def _as_dict(config) -> dict[str, Any]:
    return config.as_dict() if isinstance(config, KernelConfig) else dict(config)


# -- PnPoly -----------------------------------------------------------------------------


@dataclass
class PnPolyProblem(KernelProblem):
    name: str = "pnpoly"
    source: str = "pnpoly.cu"
    symbol: str = "pnpoly"
    seed: int = 4
    n_points: int = 20_000_000
    n_vertices: int = 600

    roofline_kind = "issue"
    #: lane-instruction slots credited per edge test (SURVEY §8(d) convention)
    ops_per_edge = 3
    rotating = ("points", "out")

    @property
    def edge_tests(self) -> float:
        return float(self.n_points) * self.n_vertices

    @property
    def total_flops(self) -> float:
        return self.ops_per_edge * self.edge_tests

    @property
    def algorithmic_bytes(self) -> float:
        return 8.0 * self.n_points + 4.0 * self.n_points + 8.0 * self.n_vertices

    def tune_params(self):
        return {
            "block_size_x": [32 * i for i in range(1, 33)],
            "tile": [1, 2, 4, 6, 8],
            "vec": [1, 2],
            "method": [0, 1, 2],
            "between": [0, 1],
            "poly_smem": [0, 1],
            "asm": [0, 1, 2, 3, 4, 5, 6, 7, 8, 9],
            "persist": [0, 1],
        }

    def restrictions(self):
        return [
            "vec == 1 or tile % 2 == 0",
            "asm == 0 or method == 2",
            "asm == 0 or (asm == 8 and poly_smem == 0) or (asm != 8 and poly_smem == 1)",
            "asm == 0 or asm >= 3 or (between == 1 and tile != 8)",
            "asm < 3 or (between == 0 and tile != 1)",
            "(asm != 4 and asm != 6) or (vec == 2 and (tile == 4 or tile == 8))",
        ]

    def default_config(self):
        return {"block_size_x": 256, "tile": 8, "vec": 2, "method": 2, "between": 0, "poly_smem": 1, "asm": 7,
                "persist": 0}

    @staticmethod
    def formula(config) -> int:
        """Which exactly-specified crossing formulation a config computes:
        0/1/2 = METHOD (IEEE compares), 3 = sign-bit form of METHOD 2 (ASM=3)."""
        c = _as_dict(config)
        return 3 if c.get("asm", 0) >= 3 else c["method"]

    def defines(self, config):
        c = _as_dict(config)
        return {
            "BLOCK_SIZE_X": c["block_size_x"],
            "TILE": c["tile"],
            "VEC": c["vec"],
            "METHOD": c["method"],
            "BETWEEN": c["between"],
            "POLY_SMEM": c["poly_smem"],
            "ASM": c.get("asm", 0),
            "VERTICES": self.n_vertices,
        }

    def launch(self, config, n_points: int | None = None):
        c = _as_dict(config)
        per_block = c["block_size_x"] * c["tile"]
        tiles = max(1, math.ceil((self.n_points if n_points is None else n_points) / per_block))
        if c.get("persist", 0):
            sms = self.gpu.sm_count if self.gpu is not None else 148
            resident = max(1, 2048 // c["block_size_x"])  # thread-limited residency per SM
            tiles = min(tiles, sms * resident)
        return Launch((tiles, 1, 1), (c["block_size_x"], 1, 1))

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        theta = np.sort(rng.uniform(0.0, 2.0 * np.pi, self.n_vertices))
        radius = 0.5 + 0.3 * rng.uniform(0.0, 1.0, self.n_vertices)
        vx = (radius * np.cos(theta)).astype(np.float32)
        vy = (radius * np.sin(theta)).astype(np.float32)
        points = rng.uniform(-1.0, 1.0, (self.n_points, 2)).astype(np.float32)
        return {"points": points, "vx": vx, "vy": vy}

    def prepare(self, gpu, inputs=None):
        self.gpu = gpu
        inputs = inputs or self.host_inputs()
        self.inputs = inputs
        self._tables = {m: native.pnpoly_edges(inputs["vx"], inputs["vy"], m) for m in (0, 1, 2)}
        self.buffers = {
            "out": gpu.empty((self.n_points,), np.int32),
            "points": gpu.array(inputs["points"], slack=16),
        }
        for m, (edges, yb) in self._tables.items():
            self.buffers[f"edges{m}"] = gpu.array(edges)
            self.buffers[f"ybounds{m}"] = gpu.array(yb)
        self.buffers["packed"] = gpu.array(self.packed_table())
        self.buffers["packed3"] = gpu.array(self.chain_table())
        self.buffers["packed7"] = gpu.array(self.pair_table())
        self.buffers["packed9"] = gpu.array(self.pair_table(bank_split=True))

    def chain_table(self) -> np.ndarray:
        """{vy_k, slope, icpt, 0} per edge for the sign-bit chain (ASM=3),
        padded to a multiple of 4 with copies of the last vertex's vy (a
        zero-length continuation of the chain, which never toggles)."""
        edges, _ = self._tables[2]
        n = edges.shape[0]
        npack = (n + 3) // 4 * 4
        table = np.zeros((npack, 4), dtype=np.float32)
        table[:, 0] = edges[n - 1, 0]
        table[:n, 0] = edges[:, 0]
        table[:n, 1] = edges[:, 2]
        table[:n, 2] = edges[:, 1]
        return table

    def pair_table(self, bank_split: bool = False) -> np.ndarray:
        """ASM=7 structure-of-arrays chain table: per group of 4 edges the 12
        floats {vy0..3, slope0..3, icpt0..3}, edges padded to a multiple of 8
        with the chain's zero-length continuation (vy of the last vertex,
        slope = icpt = 0). Pure repacking of chain_table().

        ``bank_split`` (ASM=9): {vy0..3, sl0, sl1, ic2, ic3, sl2, sl3, ic0, ic1},
        so each 128-bit load puts a slope pair and an intercept pair in opposite
        halves of its register quad (different register banks for FFMA2)."""
        edges, _ = self._tables[2]
        n = edges.shape[0]
        n8 = (n + 7) // 8 * 8
        chain = np.zeros((n8, 3), dtype=np.float32)
        chain[:, 0] = edges[n - 1, 0]
        chain[:n, 0] = edges[:, 0]
        chain[:n, 1] = edges[:, 2]
        chain[:n, 2] = edges[:, 1]
        groups = np.ascontiguousarray(chain.reshape(n8 // 4, 4, 3).transpose(0, 2, 1))  # [g][vy|sl|ic][4]
        if bank_split:
            vy, sl, ic = groups[:, 0], groups[:, 1], groups[:, 2]
            groups = np.concatenate([vy, sl[:, :2], ic[:, 2:], sl[:, 2:], ic[:, :2]], axis=1)
        return np.ascontiguousarray(groups).reshape(-1)

    def packed_table(self) -> np.ndarray:
        """{ymin, ymax, slope, icpt} per edge (METHOD 2), padded to a multiple
        of 4 with never-spanning dummies {+inf, -inf, 0, 0} (pure repacking of
        the libjt edge table; no arithmetic)."""
        edges, yb = self._tables[2]
        n = edges.shape[0]
        npack = (n + 3) // 4 * 4
        packed = np.zeros((npack, 4), dtype=np.float32)
        packed[:, 0] = np.inf
        packed[:, 1] = -np.inf
        packed[:n, 0] = yb[:, 0]
        packed[:n, 1] = yb[:, 1]
        packed[:n, 2] = edges[:, 2]
        packed[:n, 3] = edges[:, 1]
        return packed

    def args(self, config):
        m = _as_dict(config)["method"]
        b = self.buffers
        asm = _as_dict(config).get("asm", 0)
        packed = (b["packed9"] if asm == 9 else b["packed7"] if asm == 7 else b["packed3"] if asm >= 3
                  else b["packed"])
        return [b["out"], b["points"], i32(self.n_points), b[f"edges{m}"], b[f"ybounds{m}"], packed]

    def strips(self, config, uploads, out, n):
        """Point chunks (multiples of one block's tile): each is an independent launch."""
        c = _as_dict(config)
        points, per_block = uploads["points"], c["block_size_x"] * c["tile"]
        size = max(per_block, math.ceil(self.n_points / n / per_block) * per_block)
        tail = self.args(config)[3:]
        plan = []
        for p0 in range(0, self.n_points, size):
            p1 = min(self.n_points, p0 + size)
            dst = rows(self.buffers["points"], p0, p1)
            res = rows(self.buffers["out"], p0, p1)
            plan.append(Strip([(dst, points[p0:p1])], self.launch(c, p1 - p0), [res, dst, i32(p1 - p0), *tail],
                              [(out[p0:p1], res)]))
        return plan

    def bind(self, kernel, config):
        c = _as_dict(config)
        if c.get("asm", 0) == 8:
            kernel.set_global("c_pairs", self.pair_table())
            return
        if not c["poly_smem"]:
            edges, yb = self._tables[c["method"]]
            kernel.set_global("c_edges", edges)
            kernel.set_global("c_ybounds", yb)


@dataclass
class PnPolySlabProblem(PnPolyProblem):
    """PnPoly by y-slab point location (csrc/kernels/pnpoly_slab.cu).

    Same inputs and the same bitmap as :class:`PnPolyProblem` at METHOD 2
    (bit for bit: the skipped edges are exactly those whose y-test fails), but
    a different amount of work, so it is reported as its own kernel: its
    roofline is HBM (the 240 MB of points and bitmap). It is not credited with
    the brute-force edge tests it skips: ``total_flops`` raises, and its
    metrics are points/s, GB/s and joules per bitmap (:meth:`user_metrics`).
    ``edge_tests`` stays the brute-force-equivalent count, for reference only.
    """

    name: str = "pnpoly_slab"
    source: str = "pnpoly_slab.cu"
    symbol: str = "pnpoly_slab"

    roofline_kind = "hbm"
    #: slab lists are padded to a multiple of this (4 edges per trip of the edge loop)
    pad = 4

    @property
    def total_flops(self) -> float:
        from .errors import ConfigurationError

        raise ConfigurationError(f"{self.name} skips most edge tests and is not flop-counted; "
                                 "use user_metrics() (points/s, GB/s, J per bitmap)")

    def user_metrics(self):
        return ((UserMetric("points_per_s", "n_points / time"), UserMetric("gb_per_s", "hbm_bytes / time / 1e9"),
                 UserMetric("j_per_bitmap", "energy"), UserMetric("points_per_j", "n_points / energy")),
                {"n_points": float(self.n_points), "hbm_bytes": float(self.algorithmic_bytes)})

    def tune_params(self):
        return {
            "block_size_x": [128, 256, 512, 1024],
            "tile": [1, 2, 4, 8],
            "sort": [0, 1],
            "pairs_smem": [0, 1],
            "xbuckets": [0, 4, 8, 16],
            "exact_flags": [0, 1],
            "half": [0, 1],
            "buckets": [1024, 4096],
        }

    def restrictions(self):
        info = self.slab_info(4096)
        xinfo = self.slab_info(4096, 4)
        nu1 = info.nu + 1
        head = (info.nu + 3) // 4 * 4 + (info.nu + 2 + 3) // 4 * 4
        # x-search words past the slab starts: slab records, uint16 bucket starts, lo + pmax
        # (two float32 arrays, or one word per edge with HALF)
        xfix = 4 * nu1 + 4
        ne4 = (xinfo.ne + 3) // 4 * 4
        limit = 227 * 1024
        return [
            "block_size_x * tile <= 8192",
            "xbuckets == 0 or (sort == 0 and pairs_smem == 0)",
            "xbuckets > 0 or exact_flags == 1",
            "xbuckets > 0 or half == 0",
            f"({head} + buckets + pairs_smem * {2 * info.ne} + sort * ({(info.nu + 4) // 4 * 4} + "
            f"5 * block_size_x * tile) + (xbuckets > 0) * ({xfix} + (2 - half) * {ne4} + {nu1} * (xbuckets + 1) / 2)) * 4"
            f" <= {limit}",
        ]

    def default_config(self):
        return {"block_size_x": 1024, "tile": 8, "sort": 1, "pairs_smem": 0, "xbuckets": 0, "exact_flags": 1,
                "half": 0, "buckets": 4096}

    @staticmethod
    def formula(config) -> int:
        return 2

    def defines(self, config):
        c = _as_dict(config)
        return {"BLOCK_SIZE_X": c["block_size_x"], "TILE": c["tile"], "SORT": c["sort"],
                "PAIRS_SMEM": c["pairs_smem"], "XSEARCH": int(c.get("xbuckets", 0) > 0),
                "EXACT_FLAGS": c.get("exact_flags", 1), "HALF": c.get("half", 0)}

    def _polygon(self):
        inputs = getattr(self, "inputs", None)
        if inputs is None:
            inputs = self.host_inputs() if self.n_points <= (1 << 20) else self._vertices_only()
        return inputs["vx"], inputs["vy"]

    def _vertices_only(self):
        rng = np.random.default_rng(self.seed)
        theta = np.sort(rng.uniform(0.0, 2.0 * np.pi, self.n_vertices))
        radius = 0.5 + 0.3 * rng.uniform(0.0, 1.0, self.n_vertices)
        return {"vx": (radius * np.cos(theta)).astype(np.float32), "vy": (radius * np.sin(theta)).astype(np.float32)}

    def slab_table(self, buckets: int, xbuckets: int = 0):
        cache = self.__dict__.setdefault("_slab_tables", {})
        if (buckets, xbuckets) not in cache:
            vx, vy = self._polygon()
            cache[buckets, xbuckets] = native.pnpoly_slabs(vx, vy, buckets, self.pad, xbuckets)
        return cache[buckets, xbuckets]

    def slab_info(self, buckets: int, xbuckets: int = 0):
        return self.slab_table(buckets, xbuckets)[1]

    def smem_bytes(self, config) -> int:
        c = _as_dict(config)
        info = self.slab_info(c["buckets"], c.get("xbuckets", 0))
        words = sum(self._stage(c, info))
        if c["sort"]:
            words += (info.nu + 4) // 4 * 4 + 5 * c["block_size_x"] * c["tile"]
        return 4 * words

    def launch(self, config, n_points: int | None = None):
        c = _as_dict(config)
        chunk = c["block_size_x"] * c["tile"]
        chunks = max(1, math.ceil((self.n_points if n_points is None else n_points) / chunk))
        smem = self.smem_bytes(c)
        sms = self.gpu.sm_count if self.gpu is not None else 148
        resident = max(1, min(2048 // c["block_size_x"], (228 * 1024) // (smem + 1024)))
        return Launch((min(chunks, sms * resident), 1, 1), (c["block_size_x"], 1, 1), smem)

    def prepare(self, gpu, inputs=None):
        self.gpu = gpu
        inputs = inputs or self.host_inputs()
        self.inputs = inputs
        self.__dict__.pop("_slab_tables", None)
        self.buffers = {
            "out": gpu.empty((self.n_points,), np.int32),
            "points": gpu.array(inputs["points"], slack=16),
        }

    def _table_buffer(self, buckets: int, xbuckets: int):
        key = f"slabs{buckets}x{xbuckets}"
        if key not in self.buffers:
            self.buffers[key] = self.gpu.array(self.slab_table(buckets, xbuckets)[0])
        return self.buffers[key]

    @staticmethod
    def _stage(c, info):
        """(words staged from the table's start, words of the second staged range)."""
        if c.get("xbuckets", 0):
            if c.get("half", 0):
                return info.xlo_off, 0  # header + the binary16 lo|pmax words
            return info.half_off, info.pair_off - info.xlo_off  # header, then float32 lo and pmax
        return (info.words if c["pairs_smem"] else info.pair_off), 0

    def _tail(self, c):
        xb = c.get("xbuckets", 0)
        info = self.slab_info(c["buckets"], xb)
        staged, arr_words = self._stage(c, info)
        # x-search arrays as shared-memory word offsets (see pnpoly_slab.cu)
        xlo_s = info.half_off
        pmax_s = info.half_off + (info.pmax_off - info.xlo_off)
        return [self._table_buffer(c["buckets"], xb), i32(info.nu), i32(info.ng), i32(info.band_off),
                i32(info.pair_off), i32(staged), f32(info.ybase), f32(info.yscale), i32(xlo_s),
                i32(pmax_s), i32(info.xpar_off), i32(info.xst_off), i32(info.xb), i32(info.xlo_off),
                i32(arr_words)]

    def args(self, config):
        c = _as_dict(config)
        return [self.buffers["out"], self.buffers["points"], i32(self.n_points), *self._tail(c)]

    def strips(self, config, uploads, out, n):
        c = _as_dict(config)
        points, per_block = uploads["points"], c["block_size_x"] * c["tile"]
        size = max(per_block, math.ceil(self.n_points / n / per_block) * per_block)
        tail = self._tail(c)
        plan = []
        for p0 in range(0, self.n_points, size):
            p1 = min(self.n_points, p0 + size)
            dst = rows(self.buffers["points"], p0, p1)
            res = rows(self.buffers["out"], p0, p1)
            plan.append(Strip([(dst, points[p0:p1])], self.launch(c, p1 - p0), [res, dst, i32(p1 - p0), *tail],
                              [(out[p0:p1], res)]))
        return plan

    def bind(self, kernel, config):
        pass

    def useful_edge_tests(self) -> float:
        """Edges listed for the points' slabs on this input (incl. padding): what the
        edge-loop variants (xbuckets=0) evaluate per point."""
        info = self.slab_info(4096)
        table = self.slab_table(4096)[0]
        u = table[info.u_off:info.u_off + info.nu]
        band = table[info.band_off:info.band_off + info.nu + 2].view(np.int32)
        r = np.searchsorted(u, self.inputs["points"][:, 1], side="right")
        return float((band[r + 1] - band[r]).astype(np.int64).sum())


@dataclass
class PnPolyGridProblem(PnPolySlabProblem):
    """PnPoly with a uniform-cell fast path (csrc/kernels/pnpoly_grid.cu).

    The same bitmap as :class:`PnPolyProblem` at METHOD 2, bit for bit: a
    GRID x GRID raster of cells (libjt ``jt_pnpoly_grid``) answers every point
    whose cell is provably clean with one lookup; the others are queued per
    warp and run the exact x-search of the slab kernel (its table read
    through L1 / L2). Reported as its own kernel against the HBM roofline.
    """

    name: str = "pnpoly_grid"
    source: str = "pnpoly_grid.cu"
    symbol: str = "pnpoly_grid"

    def tune_params(self):
        return {
            "block_size_x": [256, 512, 1024],
            "tile": [1, 2, 4],
            "grid": [256, 512, 1024, 2048],
            "grid_smem": [0, 1],
            "xbuckets": [8, 16],
            "buckets": [1024, 4096],
        }

    def restrictions(self):
        return [f"(grid_smem * grid * grid / 4 + block_size_x / 32 * {16 * 64}) <= {227 * 1024}"]

    def default_config(self):
        return {"block_size_x": 1024, "tile": 2, "grid": 512, "grid_smem": 1, "xbuckets": 16, "buckets": 4096}

    def defines(self, config):
        c = _as_dict(config)
        return {"BLOCK_SIZE_X": c["block_size_x"], "TILE": c["tile"], "GRID": c["grid"],
                "GRID_SMEM": c.get("grid_smem", 1)}

    def grid_table(self, g: int):
        cache = self.__dict__.setdefault("_grid_tables", {})
        if g not in cache:
            vx, vy = self._polygon()
            cache[g] = native.pnpoly_grid(vx, vy, g, g)
        return cache[g]

    def smem_bytes(self, config) -> int:
        c = _as_dict(config)
        words = (c["grid"] * c["grid"] + 15) // 16 if c.get("grid_smem", 1) else 0
        return ((words + 3) // 4 * 4) * 4 + c["block_size_x"] // 32 * 64 * 16

    def launch(self, config, n_points: int | None = None):
        c = _as_dict(config)
        chunk = c["block_size_x"] * c["tile"]
        chunks = max(1, math.ceil((self.n_points if n_points is None else n_points) / chunk))
        smem = self.smem_bytes(c)
        sms = self.gpu.sm_count if self.gpu is not None else 148
        resident = max(1, min(2048 // c["block_size_x"], (228 * 1024) // (smem + 1024)))
        return Launch((min(chunks, sms * resident), 1, 1), (c["block_size_x"], 1, 1), smem)

    def prepare(self, gpu, inputs=None):
        super().prepare(gpu, inputs)
        self.__dict__.pop("_grid_tables", None)

    def _tail(self, c):
        g = c["grid"]
        key = f"grid{g}"
        words, params, _ = self.grid_table(g)
        if key not in self.buffers:
            self.buffers[key] = self.gpu.array(words)
        info = self.slab_info(c["buckets"], c["xbuckets"])
        return [self.buffers[key], f32(params[0]), f32(params[1]), f32(params[2]), f32(params[3]),
                self._table_buffer(c["buckets"], c["xbuckets"]), i32(info.nu), i32(info.ng), i32(info.xb),
                f32(info.ybase), f32(info.yscale), i32(info.guess_off), i32(info.xpar_off), i32(info.xst_off),
                i32(info.xlo_off), i32(info.pmax_off), i32(info.pair_off)]

    def clean_fraction(self, g: int) -> float:
        """Fraction of this input's points that land in a clean cell (the fast path)."""
        words, prm, _ = self.grid_table(g)
        pts = self.inputs["points"]

        def cell(v, scale, offset):  # fma emulated exactly: float32 x float32 is exact in float64
            with np.errstate(invalid="ignore", over="ignore"):
                f = (v.astype(np.float64) * np.float64(scale) + np.float64(offset)).astype(np.float32)
            k = np.trunc(np.nan_to_num(f, nan=0.0, posinf=2.0**32, neginf=0.0))
            return np.clip(k, 0, g - 1).astype(np.int64)

        idx = cell(pts[:, 1], prm[2], prm[3]) * g + cell(pts[:, 0], prm[0], prm[1])
        return float(((words[idx >> 4] >> ((idx & 15) * 2).astype(np.uint32)) & 1).mean())


@dataclass
class PnPolyCellsProblem(PnPolyGridProblem):
    """PnPoly with per-cell edge lists (csrc/kernels/pnpoly_cells.cu).

    The same bitmap as :class:`PnPolyProblem` at METHOD 2, bit for bit: libjt
    ``jt_pnpoly_cells`` decides every edge's test per cell of a GRID x GRID
    raster; decided cells answer with one shared-memory lookup, undecided ones
    list their few undecided edges (base parity ^ their tests), cells with more
    than ``lmax`` fall back to the slab search. Two points per 16-byte load.
    Reported as its own kernel against the HBM roofline.
    """

    name: str = "pnpoly_cells"
    source: str = "pnpoly_cells.cu"
    symbol: str = "pnpoly_cells"

    def tune_params(self):
        return {
            "block_size_x": [256, 512, 1024],
            "tile": [1, 2, 4],
            "grid": [256, 448, 512, 576, 640, 704, 768, 1024],
            "grid_smem": [0, 1],
            "lmax": [4, 16],
            "stream": [0, 1, 2],
            "prefetch": [0, 1, 2],
            "adrain": [0, 1],
            "head32": [0, 1],
            "quad": [0, 1],
            "min_blocks": [0, 1, 2],
            "regpf": [0, 1, 2],
        }
    # round 2: min_blocks 1 (one block per SM, registers uncapped) makes REGPF (register double
    # buffering) pay, so both joined the space (profiles/r2_cells_ring_minblocks_probe.jsonl);
    # DEFER (per-thread pending points, no ring) stays a kernel option: slower everywhere
    # (profiles/r2_cells_defer_probe.jsonl)

    def restrictions(self):
        # ring: 128 x 12-byte slots per warp, or 64 + a 16-byte head slot per thread with
        # the split drain (QCAP in pnpoly_cells.cu)
        return [f"(grid_smem * grid * grid / 4 + block_size_x / 32 * (1536 - 768 * adrain) + "
                f"16 * (1 + head32) * block_size_x * adrain) <= {227 * 1024}"]

    def default_config(self):
        return {"block_size_x": 1024, "tile": 2, "grid": 512, "grid_smem": 1, "lmax": 16, "stream": 0, "prefetch": 1, "regpf": 0,
                "adrain": 1, "head32": 0, "quad": 0, "min_blocks": 0}

    def defines(self, config):
        c = _as_dict(config)
        return {"BLOCK_SIZE_X": c["block_size_x"], "TILE": c["tile"], "GRID": c["grid"],
                "GRID_SMEM": c.get("grid_smem", 1), "STREAM": c.get("stream", 0), "PREFETCH": c.get("prefetch", 0),
                "REGPF": c.get("regpf", 0), "ADRAIN": c.get("adrain", 0), "HEAD32": c.get("head32", 0),
                **({"QUAD": 1} if c.get("quad", 0) else {}), **({"DEFER": 1} if c.get("defer", 0) else {}),
                **({"MIN_BLOCKS": c["min_blocks"]} if c.get("min_blocks", 0) else {}),
                **({"HPF": 1} if c.get("hpf", 0) else {}), **({"PUSHV": 1} if c.get("pushv", 0) else {}),
                **({"RING16": 1} if c.get("ring16", 0) else {})}

    def cell_table(self, g: int, lmax: int, head_words: int = 4):
        cache = self.__dict__.setdefault("_cell_tables", {})
        if (g, lmax, head_words) not in cache:
            vx, vy = self._polygon()
            cache[(g, lmax, head_words)] = native.pnpoly_cells(vx, vy, g, g, lmax, head_words)
        return cache[(g, lmax, head_words)]

    def smem_bytes(self, config) -> int:
        c = _as_dict(config)
        words = (c["grid"] * c["grid"] + 15) // 16 if c.get("grid_smem", 1) else 0
        ad, hw = c.get("adrain", 0), 1 + c.get("head32", 0)
        if c.get("defer", 0):  # no ring: the raster only
            return (words + 3) // 4 * 16
        qcap = 64 if ad else (256 if c.get("pushv", 0) and c.get("quad", 0) else 128)  # QCAP in the kernel
        slot = 16 if c.get("ring16", 0) else 12  # RSLOT
        return (words + 3) // 4 * 16 + c["block_size_x"] // 32 * qcap * slot + 16 * hw * c["block_size_x"] * ad

    def launch(self, config, n_points: int | None = None):
        c = _as_dict(config)
        chunk = (2 + 2 * c.get("quad", 0)) * c["block_size_x"] * c["tile"]
        chunks = max(1, math.ceil((self.n_points if n_points is None else n_points) / chunk))
        smem = self.smem_bytes(c)
        sms = self.gpu.sm_count if self.gpu is not None else 148
        blocks = c.get("min_blocks", 0) or 2048 // c["block_size_x"]  # the launch bounds' residency
        resident = max(1, min(blocks, 2048 // c["block_size_x"], (228 * 1024) // (smem + 1024)))
        return Launch((min(chunks, sms * resident), 1, 1), (c["block_size_x"], 1, 1), smem)

    def prepare(self, gpu, inputs=None):
        super().prepare(gpu, inputs)
        self.__dict__.pop("_cell_tables", None)

    def _tail(self, c):
        g, lmax, hw = c["grid"], c["lmax"], 4 + 4 * c.get("head32", 0)
        key = f"cells{g}x{lmax}h{hw}"
        words, params, heads, edges, _ = self.cell_table(g, lmax, hw)
        if key + "w" not in self.buffers:  # one entry per device buffer (buffers are freed one by one)
            self.buffers[key + "w"] = self.gpu.array(words)
            self.buffers[key + "h"] = self.gpu.array(heads)
            self.buffers[key + "e"] = self.gpu.array(edges)
        bw, bh, be = (self.buffers[key + x] for x in "whe")
        info = self.slab_info(1024, 16)
        return [bw, bh, be, f32(params[0]), f32(params[1]), f32(params[2]), f32(params[3]),
                self._table_buffer(1024, 16), i32(info.nu), i32(info.ng), i32(info.xb),
                f32(info.ybase), f32(info.yscale), i32(info.guess_off), i32(info.xpar_off), i32(info.xst_off),
                i32(info.xlo_off), i32(info.pmax_off), i32(info.pair_off)]

    def clean_fraction(self, g: int, lmax: int = 16) -> float:
        """Fraction of this input's points answered by the cell lookup alone (codes 0 / 1)."""
        words, prm, _, _, _ = self.cell_table(g, lmax)
        pts = self.inputs["points"]

        def cell(v, scale, offset):
            with np.errstate(invalid="ignore", over="ignore"):
                f = (v.astype(np.float64) * np.float64(scale) + np.float64(offset)).astype(np.float32)
            k = np.trunc(np.nan_to_num(f, nan=0.0, posinf=2.0**32, neginf=0.0))
            return np.clip(k, 0, g - 1).astype(np.int64)

        idx = cell(pts[:, 1], prm[2], prm[3]) * g + cell(pts[:, 0], prm[0], prm[1])
        return float((((words[idx >> 4] >> ((idx & 15) * 2).astype(np.uint32)) & 3) < 2).mean())


# -- Conv2D -------------------------------------------------------------------------------


@dataclass
class Conv2DProblem(KernelProblem):
    name: str = "conv2d"
    source: str = "conv2d.cu"
    symbol: str = "conv2d"
    seed: int = 3
    rotating = ("image", "out")
    width: int = 4096
    height: int = 4096
    fw: int = 17
    fh: int = 17

    @property
    def total_flops(self) -> float:
        return 2.0 * self.fw * self.fh * self.width * self.height

    @property
    def algorithmic_bytes(self) -> float:
        return 4.0 * ((self.width + self.fw - 1) * (self.height + self.fh - 1) + self.width * self.height
                      + self.fw * self.fh)

    def tune_params(self):
        return {
            "block_size_x": [16, 32, 64],
            "block_size_y": [1, 2, 4, 8, 16],
            "tile_size_x": [1, 2, 4, 8],
            "tile_size_y": [1, 2, 4, 8],
            "use_shmem": [0, 1],
            "use_padding": [0, 1],
            "fma2": [0, 1],
            "min_blocks": [0, 2],
        }

    def restrictions(self):
        return [
            "32 <= block_size_x * block_size_y <= 1024",
            "tile_size_x * tile_size_y <= 32",
            f"{self.width} % (block_size_x * tile_size_x) == 0",
            f"{self.height} % (block_size_y * tile_size_y) == 0",
            "use_shmem == 1 or use_padding == 0",
            "fma2 == 0 or tile_size_x % 2 == 0",
            "min_blocks * block_size_x * block_size_y <= 2048",
            f"use_shmem == 0 or (block_size_y * tile_size_y + {self.fh - 1}) * "
            f"(block_size_x * tile_size_x + {self.fw - 1} + 4 * use_padding) * 4 <= 48000",
        ]

    def default_config(self):
        return {"block_size_x": 32, "block_size_y": 4, "tile_size_x": 4, "tile_size_y": 4, "use_shmem": 1,
                "use_padding": 0, "fma2": 0, "min_blocks": 0}

    def defines(self, config):
        c = _as_dict(config)
        return {
            "BLOCK_X": c["block_size_x"],
            "BLOCK_Y": c["block_size_y"],
            "TILE_X": c["tile_size_x"],
            "TILE_Y": c["tile_size_y"],
            "USE_SMEM": c["use_shmem"],
            "PAD": 4 * c["use_padding"],
            "FMA2": c.get("fma2", 0),
            **({"MIN_BLOCKS": c["min_blocks"]} if c.get("min_blocks", 0) else {}),
            "IMAGE_W": self.width,
            "IMAGE_H": self.height,
            "FW": self.fw,
            "FH": self.fh,
        }

    def tile_multiples(self, config):
        c = _as_dict(config)
        return {"width": c["block_size_x"] * c["tile_size_x"], "height": c["block_size_y"] * c["tile_size_y"]}

    def launch(self, config):
        c = _as_dict(config)
        gx = self.width // (c["block_size_x"] * c["tile_size_x"])
        gy = self.height // (c["block_size_y"] * c["tile_size_y"])
        return Launch((gx, gy, 1), (c["block_size_x"], c["block_size_y"], 1))

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        image = rng.uniform(0.0, 1.0, (self.height + self.fh - 1, self.width + self.fw - 1)).astype(np.float32)
        filt = rng.uniform(0.0, 1.0, (self.fh, self.fw)).astype(np.float32)
        return {"image": image, "filter": filt}

    def prepare(self, gpu, inputs=None):
        self.gpu = gpu
        inputs = inputs or self.host_inputs()
        self.inputs = inputs
        self.buffers = {
            "out": gpu.empty((self.height, self.width), np.float32),
            "image": gpu.array(inputs["image"], slack=64),
        }

    def args(self, config):
        return [self.buffers["out"], self.buffers["image"]]

    def strips(self, config, uploads, out, n):
        """Bands of output rows (multiples of the block's tile height). Band i uploads only
        the input rows band i-1 has not (its halo of FH-1 rows is already resident)."""
        c = _as_dict(config)
        image, th = uploads["image"], c["block_size_y"] * c["tile_size_y"]
        band = max(th, math.ceil(self.height / n / th) * th)
        shape = self.launch(c)
        plan, uploaded = [], 0
        for r0 in range(0, self.height, band):
            r1 = min(self.height, r0 + band)
            need = r1 + self.fh - 1
            h2d = [(rows(self.buffers["image"], uploaded, need), image[uploaded:need])]
            uploaded = need
            res = rows(self.buffers["out"], r0, r1)
            launch = Launch((shape.grid[0], (r1 - r0) // th, 1), shape.block)
            plan.append(Strip(h2d, launch, [res, rows(self.buffers["image"], r0, need)], [(out[r0:r1], res)]))
        return plan

    def bind(self, kernel, config):
        kernel.set_global("d_filter", self.inputs["filter"])


# -- SGEMM --------------------------------------------------------------------------------


@dataclass
class SgemmProblem(KernelProblem):
    name: str = "sgemm"
    source: str = "sgemm.cu"
    symbol: str = "sgemm"
    seed: int = 0
    m: int = 4096
    n: int = 4096
    k: int = 4096
    alpha: float = 1.0
    beta: float = 0.5
    #: "paper": Kernel Tuner's CLBlast value lists; "b200": widened for 227 KB smem / 255 regs
    value_set: str = "paper"
    rotating = ("at", "b", "out")

    @property
    def total_flops(self) -> float:
        return 2.0 * self.m * self.n * self.k

    @property
    def algorithmic_bytes(self) -> float:
        return 4.0 * (self.m * self.k + self.k * self.n + 2 * self.m * self.n)

    #: the paper's space: Kernel Tuner's CLBlast xgemm lists and restrictions,
    #: 17,472 valid configs
    CLBLAST_PARAMS = {
        "MWG": [16, 32, 64, 128], "NWG": [16, 32, 64, 128], "KWG": [32], "MDIMC": [8, 16, 32], "NDIMC": [8, 16, 32],
        "MDIMA": [8, 16, 32], "NDIMB": [8, 16, 32], "KWI": [2], "VWM": [1, 2, 4, 8], "VWN": [1, 2, 4, 8],
        "STRM": [0], "STRN": [0], "SA": [0, 1], "SB": [0, 1],
    }
    CLBLAST_RESTRICTIONS = [
        "KWG % KWI == 0",
        "MWG % (MDIMC * VWM) == 0",
        "NWG % (NDIMC * VWN) == 0",
        "MWG % (MDIMA * VWM) == 0",
        "NWG % (NDIMB * VWN) == 0",
        "KWG % ((MDIMC * NDIMC) / MDIMA) == 0",
        "KWG % ((MDIMC * NDIMC) / NDIMB) == 0",
        "not (MWG == 128 and NWG == 128 and MDIMC == 8 and NDIMC == 8)",
    ]

    def tune_params(self):
        if self.value_set == "clblast":
            return dict(self.CLBLAST_PARAMS)
        if self.value_set == "b200":
            return {
                "MWG": [64, 128, 256], "NWG": [64, 128, 256], "KWG": [8, 16, 32],
                "MDIMC": [8, 16, 32], "NDIMC": [8, 16, 32], "MDIMA": [8, 16, 32, 64], "NDIMB": [8, 16, 32, 64],
                "KWI": [1, 2, 4, 8], "VWM": [1, 2, 4], "VWN": [1, 2, 4], "STRM": [0, 1], "STRN": [0, 1],
                "SA": [0, 1], "SB": [0, 1], "ASYNC": [0, 2, 3, 4], "FMA2": [0, 1], "GROUP_M": [1, 4, 8, 16],
                "SPLIT_TAIL": [0, 2, 4],
            }
        return {
            "MWG": [16, 32, 64, 128], "NWG": [16, 32, 64, 128], "KWG": [16, 32],
            "MDIMC": [8, 16, 32], "NDIMC": [8, 16, 32], "MDIMA": [8, 16, 32], "NDIMB": [8, 16, 32],
            "KWI": [2, 8], "VWM": [1, 2, 4, 8], "VWN": [1, 2, 4, 8], "STRM": [0, 1], "STRN": [0, 1],
            "SA": [0, 1], "SB": [0, 1], "ASYNC": [0, 2, 3, 4], "FMA2": [0, 1],
        }

    def restrictions(self):
        shape = f"{self.m} % MWG == 0 and {self.n} % NWG == 0 and {self.k} % KWG == 0"
        if self.value_set == "clblast":
            # every one of the 17,472 fits the B200 kernel (dynamic shared memory, float8 vectors)
            return [*self.CLBLAST_RESTRICTIONS, shape]
        # CLBlast's xgemm constraints (KWG % KWI, tile divisibility, load shapes) plus the B200
        # shared-memory budget (two buffers, or ASYNC cp.async stages) and the register cap.
        return [
            "KWG % KWI == 0",
            "MWG % (MDIMC * VWM) == 0",
            "NWG % (NDIMC * VWN) == 0",
            "MWG % (MDIMA * VWM) == 0",
            "NWG % (NDIMB * VWN) == 0",
            "KWG % ((MDIMC * NDIMC) / MDIMA) == 0",
            "KWG % ((MDIMC * NDIMC) / NDIMB) == 0",
            "(MDIMC * NDIMC) % MDIMA == 0",
            "(MDIMC * NDIMC) % NDIMB == 0",
            "ASYNC == 0 or (SA == 1 and SB == 1)",
            "(ASYNC == 0 and (SA * KWG * MWG + SB * KWG * NWG) * 2 * 4 <= 227 * 1024)"
            " or (ASYNC > 0 and KWG * (MWG + NWG) * 4 * ASYNC <= 227 * 1024)",
            "(MWG / MDIMC) * (NWG / NDIMC) <= 128",
            shape,
            "FMA2 == 0 or VWN % 2 == 0",
        ]

    def default_config(self):
        return {"MWG": 128, "NWG": 128, "KWG": 16, "MDIMC": 16, "NDIMC": 16, "MDIMA": 32, "NDIMB": 32,
                "KWI": 2, "VWM": 4, "VWN": 4, "STRM": 1, "STRN": 1, "SA": 1, "SB": 1, "ASYNC": 0, "FMA2": 0,
                "GROUP_M": 1, "SPLIT_TAIL": 0}

    def defines(self, config):
        return dict(_as_dict(config))

    def tile_multiples(self, config):
        c = _as_dict(config)
        return {"m": c["MWG"], "n": c["NWG"], "k": c["KWG"]}

    @staticmethod
    def smem_bytes(config) -> int:
        c = _as_dict(config)
        stages = c.get("ASYNC", 0)
        if stages:  # cp.async stages
            return c["KWG"] * (c["MWG"] + c["NWG"]) * 4 * stages
        return 2 * 4 * c["KWG"] * (c["SA"] * c["MWG"] + c["SB"] * c["NWG"])  # CLBlast's two buffers

    def tail_plan(self, config) -> tuple[int, int, int]:
        """SPLIT_TAIL = s > 0: (full_tiles, split, grid) for the 1D split-tail grid. Whole waves of
        SMs x resident CTAs (cuOccupancy for this config's registers and shared memory) run one
        tile per CTA; the remaining tiles are split along K over up to s CTAs each, as many as
        still fit one wave. Without a GPU (or no tail) every tile is whole."""
        c = _as_dict(config)
        tiles = (self.m // c["MWG"]) * (self.n // c["NWG"])
        s = int(c.get("SPLIT_TAIL", 0))
        if s < 2 or self.gpu is None:
            return tiles, 1, tiles
        key = ("tail", tuple(sorted(c.items())))
        hit = self._plans.get(key) if hasattr(self, "_plans") else None
        if hit:
            return hit
        per_sm = self.kernel(c).occupancy(c["MDIMC"] * c["NDIMC"], self.smem_bytes(c))
        slots = max(1, per_sm) * self.gpu.sm_count
        full = tiles // slots * slots
        tail = tiles - full
        split = min(s, slots // tail, self.k // c["KWG"]) if tail else 1
        if split < 2:
            full, split = tiles, 1
        plan = (full, split, full + (tiles - full) * split)
        if not hasattr(self, "_plans"):
            self._plans = {}
        self._plans[key] = plan
        # workspace: one MWG x NWG partial per split CTA; one arrival counter per split tile (zeroed
        # once; the last CTA of a tile resets its counter)
        need_ws = (tiles - full) * split * c["MWG"] * c["NWG"]
        if need_ws and ("tail_ws" not in self.buffers or self.buffers["tail_ws"].nbytes < 4 * need_ws):
            if "tail_ws" in self.buffers:
                self.buffers["tail_ws"].free()
            self.buffers["tail_ws"] = self.gpu.empty((need_ws,), np.float32)
        if "tail_counters" not in self.buffers or self.buffers["tail_counters"].nbytes < 4 * tiles:
            if "tail_counters" in self.buffers:
                self.buffers["tail_counters"].free()
            self.buffers["tail_counters"] = self.gpu.empty((tiles,), np.uint32)
            self.buffers["tail_counters"].fill(0)
        return plan

    def launch(self, config):
        c = _as_dict(config)
        block = (c["MDIMC"] * c["NDIMC"], 1, 1)
        if c.get("SPLIT_TAIL", 0):
            return Launch((self.tail_plan(c)[2], 1, 1), block, smem=self.smem_bytes(c))
        return Launch((self.m // c["MWG"], self.n // c["NWG"], 1), block, smem=self.smem_bytes(c))

    def host_inputs(self):
        a = np.random.default_rng(self.seed).uniform(-1.0, 1.0, (self.m, self.k)).astype(np.float32)
        b = np.random.default_rng(self.seed + 1).uniform(-1.0, 1.0, (self.k, self.n)).astype(np.float32)
        c0 = np.random.default_rng(self.seed + 2).uniform(-1.0, 1.0, (self.m, self.n)).astype(np.float32)
        return {"a": a, "b": b, "c0": c0}

    def prepare(self, gpu, inputs=None):
        self.gpu = gpu
        inputs = inputs or self.host_inputs()
        self.inputs = inputs
        self._plans = {}  # split-tail plans refer to this buffer set
        self.buffers = {
            "at": gpu.array(np.ascontiguousarray(inputs["a"].T)),  # column-major A == row-major A^T
            "b": gpu.array(inputs["b"]),
            "out": gpu.array(inputs["c0"]),
        }

    def reset_output(self):
        # C is read (beta != 0) and written: every run restarts from C0.
        self.buffers["out"].upload(self.inputs["c0"])

    def args(self, config):
        b = self.buffers
        base = [i32(self.m), i32(self.n), i32(self.k), f32(self.alpha), f32(self.beta), b["at"], b["b"], b["out"]]
        if _as_dict(config).get("SPLIT_TAIL", 0):
            full, split, _ = self.tail_plan(config)
            ws = b.get("tail_ws") or b["out"]  # no split tile: never touched
            counters = b.get("tail_counters") or b["out"]
            return [*base, ws, counters, i32(full), i32(split)]
        return base


@dataclass
class SgemmTF32Problem(SgemmProblem):
    """SGEMM on the 5th-gen tensor cores (tcgen05 kind::tf32, TMA, TMEM).

    Same inputs, storage and oracle as :class:`SgemmProblem`; TF32 inputs
    (10-bit mantissa) with FP32 accumulation, so it is held to its own
    tolerance (oracle SGEMM_TF32_TOL) and reported separately (K1').
    """

    name: str = "sgemm_tf32"
    source: str = "sgemm_tf32.cu"
    symbol: str = "sgemm_tf32"
    roofline_kind = "tensor"

    def tune_params(self):
        return {"BN": [64, 128, 256], "STAGES": [2, 3, 4, 5, 6, 7], "PERSIST": [0, 1], "SPLIT_TAIL": [0, 1],
                "PAIR": [0, 1], "GROUP_M": [1, 4, 8]}

    def restrictions(self):
        return [
            "STAGES * (16384 + BN * 128 / (1 + PAIR)) + 2048 <= 232448",
            "PERSIST == 0 or BN >= 128",
            "PERSIST == 1 or SPLIT_TAIL == 0",
            "PAIR == 0 or BN >= 128",
            "PAIR == 0 or PERSIST == 1 or SPLIT_TAIL == 0",
            "PERSIST == 1 or GROUP_M == 1",  # the tile walk of the persistent variants
            f"{self.m} % (128 * (1 + PAIR)) == 0 and {self.n} % BN == 0 and {self.k} % 32 == 0",
        ]

    def default_config(self):
        return {"BN": 256, "STAGES": 4, "PERSIST": 1, "SPLIT_TAIL": 1, "PAIR": 0, "GROUP_M": 1}

    def defines(self, config):
        c = _as_dict(config)
        d = {"BN": c["BN"], "STAGES": c["STAGES"]}
        if c.get("PERSIST", 0):
            d["SPLIT_TAIL"] = c.get("SPLIT_TAIL", 0)
            if c.get("GROUP_M", 1) > 1:
                d["GROUP_M"] = c["GROUP_M"]
        if self._bk(c) != 32:
            if not (c.get("PAIR", 0) and c.get("PERSIST", 0)):
                from .errors import ConfigurationError

                raise ConfigurationError("BK != 32 exists only for the persistent CTA-pair kernel (PAIR = PERSIST = 1)")
            d["BK"] = self._bk(c)
        return d

    @staticmethod
    def _bk(config) -> int:
        """k-rows per pipeline stage (optional key, default 32; 64 / 128 only for PAIR + PERSIST)."""
        return int(_as_dict(config).get("BK", 32))

    def tile_multiples(self, config):
        c = _as_dict(config)
        return {"m": 128 * (1 + c.get("PAIR", 0)), "n": c["BN"], "k": self._bk(c)}

    def _variant(self, config) -> tuple[str, str]:
        """(source file, kernel symbol): CTA-pair (cta_group::2), persistent warp-specialised, or one
        tile per CTA."""
        c = _as_dict(config)
        if c.get("PAIR", 0) and c.get("PERSIST", 0):
            return "sgemm_tf32c2p.cu", "sgemm_tf32c2p"
        if c.get("PAIR", 0):
            return "sgemm_tf32c2.cu", "sgemm_tf32c2"
        if c.get("PERSIST", 0):
            return "sgemm_tf32p.cu", "sgemm_tf32p"
        return "sgemm_tf32.cu", "sgemm_tf32"

    def cubin(self, config):
        source, _ = self._variant(config)
        return native.compile_cubin(native.kernel_source(source), self.name, self.options(config))

    def kernel(self, config):
        if self.gpu is None:
            raise RuntimeError(f"{self.name}: prepare(gpu) first")
        return self.gpu.load(self.cubin(config), self._variant(config)[1])

    def smem_bytes(self, config) -> int:
        c = _as_dict(config)
        bk = SgemmTF32Problem._bk(c)
        b_stage = c["BN"] * bk * 4 // (2 if c.get("PAIR", 0) else 1)
        return c["STAGES"] * (128 * bk * 4 + b_stage) + 1024 + 256

    def tiles(self, config) -> int:
        return (self.m // 128) * (self.n // _as_dict(config)["BN"])

    def launch(self, config):
        c = _as_dict(config)
        if c.get("PAIR", 0) and c.get("PERSIST", 0):  # persistent CTA pairs, one per TPC
            sms = self.gpu.sm_count if self.gpu is not None else 148
            pairs = min(sms // 2, (self.m // 256) * (self.n // c["BN"]))
            return Launch((2 * pairs, 1, 1), (192, 1, 1), smem=self.smem_bytes(c), cluster_x=2)
        if c.get("PAIR", 0):  # one 256 x BN tile per CTA pair (cluster of 2 on one TPC)
            return Launch((2 * (self.n // c["BN"]), self.m // 256, 1), (128, 1, 1), smem=self.smem_bytes(c),
                          cluster_x=2)
        if c.get("PERSIST", 0):
            sms = self.gpu.sm_count if self.gpu is not None else 148
            return Launch((min(sms, self.tiles(c)), 1, 1), (192, 1, 1), smem=self.smem_bytes(c))
        return Launch((self.n // c["BN"], self.m // 128, 1), (128, 1, 1), smem=self.smem_bytes(c))

    def prepare(self, gpu, inputs=None):
        super().prepare(gpu, inputs)
        # TMA descriptors: A^T is K x M row-major, B is K x N row-major; 32 x 32 fp32 boxes in the
        # 128B-span / 32B-atom swizzle, the only smem layout UMMA accepts for MN-major TF32
        self._maps = {}  # BK -> {"a", "b"}: boxes of BK k-rows x 32 fp32, built on first use
        # split-K tail workspace (two 128 x 256 partials per split tile, < one per SM) and counters
        self.buffers["workspace"] = gpu.empty((2 * gpu.sm_count * 128 * 256,), np.float32)
        counters = gpu.empty((gpu.sm_count,), np.uint32)
        counters.fill(0)
        self.buffers["counters"] = counters

    def rotation_sets(self, config, n):
        """As the base class, plus TMA descriptors of each set's own A and B copies."""
        sets = super().rotation_sets(config, n)
        sw, bk = self.gpu.SWIZZLE_128B_ATOM_32B, self._bk(config)
        for j, args in enumerate(sets, start=1):
            args[0] = self.gpu.tensor_map_2d(self.buffers[f"at@{j}"], self.k, self.m, bk, 32, sw)
            args[1] = self.gpu.tensor_map_2d(self.buffers[f"b@{j}"], self.k, self.n, bk, 32, sw)
        return sets

    def _maps_for(self, bk: int) -> dict:
        if bk not in self._maps:
            sw = self.gpu.SWIZZLE_128B_ATOM_32B
            self._maps[bk] = {"a": self.gpu.tensor_map_2d(self.buffers["at"], self.k, self.m, bk, 32, sw),
                              "b": self.gpu.tensor_map_2d(self.buffers["b"], self.k, self.n, bk, 32, sw)}
        return self._maps[bk]

    def args(self, config):
        c = _as_dict(config)
        b = self.buffers
        maps = self._maps_for(self._bk(c))
        scalars = [i32(self.m), i32(self.n), i32(self.k), f32(self.alpha), f32(self.beta)]
        if c.get("PERSIST", 0):
            return [maps["a"], maps["b"], b["out"], b["workspace"], b["counters"], *scalars]
        return [maps["a"], maps["b"], b["out"], *scalars]


# -- burner (P(f) sweep load) ---------------------------------------------------------------


@dataclass
class BurnerProblem(KernelProblem):
    name: str = "burner"
    source: str = "burner.cu"
    symbol: str = "burner"
    rotating = ()
    iters: int = 4096
    blocks_per_sm: int = 8

    @property
    def total_flops(self) -> float:
        sms = self.gpu.sm_count if self.gpu else 148
        return 2.0 * 16 * 8 * self.iters * 256 * self.blocks_per_sm * sms

    @property
    def algorithmic_bytes(self) -> float:
        return 0.0

    def tune_params(self):
        return {"chains": [8], "block": [256]}

    def default_config(self):
        return {"chains": 8, "block": 256}

    def launch(self, config):
        sms = self.gpu.sm_count if self.gpu else 148
        return Launch((sms * self.blocks_per_sm, 1, 1), (256, 1, 1))

    def host_inputs(self):
        return {}

    def prepare(self, gpu, inputs=None):
        self.gpu = gpu
        self.buffers = {"sink": gpu.empty((gpu.sm_count * self.blocks_per_sm * 256,), np.float32)}

    def reset_output(self):
        pass

    def args(self, config):
        return [self.buffers["sink"], i32(self.iters), f32(1.0)]


PROBLEMS = {"pnpoly": PnPolyProblem, "pnpoly_slab": PnPolySlabProblem, "pnpoly_grid": PnPolyGridProblem,
            "pnpoly_cells": PnPolyCellsProblem,
            "conv2d": Conv2DProblem, "sgemm": SgemmProblem, "sgemm_tf32": SgemmTF32Problem,
            "burner": BurnerProblem}


def make_problem(name: str, **kwargs) -> KernelProblem:
    try:
        return PROBLEMS[name](**kwargs)
    except KeyError:
        from .errors import ConfigurationError

        raise ConfigurationError(f"unknown kernel {name!r}; choose from {sorted(PROBLEMS)}") from None
