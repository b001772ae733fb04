"""Kernel parity on the B200 through libjt (the C-ABI) against the CPU oracles.

Bars: PnPoly bit-exact against the oracle formulation the
config computes; Conv2D max|out - ref| / (sum|f| max|x|) <= 1e-5; SGEMM
max|C - C64| / max|C64| <= 1e-5 (FP32, fp64 oracle).
"""

import itertools

import numpy as np
import pytest
from conftest import assert_full_size_pin

from oracle import kernels_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    from paper_2211_07260_b200.gpu import GPU

    g = GPU(0)
    yield g
    g.close()


def run_once(gpu, problem, cfg):
    k = problem.kernel(cfg)
    problem.bind(k, cfg)
    problem.reset_output()
    gpu.launch(k, problem.launch(cfg), problem.args(cfg))
    gpu.synchronize()
    return problem.fetch_output()


# -- PnPoly ---------------------------------------------------------------------------

PNPOLY_CONFIGS = (
    [dict(block_size_x=b, tile=t, vec=2, method=2, between=0, poly_smem=1, asm=a, persist=ps)
     for a, b, t, ps in itertools.product((3, 5, 7, 9), (96, 256, 1024), (2, 4, 6, 8), (0, 1))]
    + [dict(block_size_x=b, tile=t, vec=2, method=2, between=0, poly_smem=1, asm=a, persist=ps)
       for a, b, t, ps in itertools.product((4, 6), (128, 512), (4, 8), (0, 1))]
    + [dict(block_size_x=b, tile=t, vec=v, method=2, between=0, poly_smem=0, asm=8, persist=ps)
       for b, t, v, ps in itertools.product((128, 512), (2, 4, 6, 8), (1, 2), (0, 1))]
    + [dict(block_size_x=b, tile=t, vec=v, method=2, between=1, poly_smem=1, asm=a)
       for a, b, t, v in itertools.product((1, 2), (128,), (1, 2, 4, 6), (1, 2)) if not (v == 2 and t % 2)]
    + [dict(block_size_x=b, tile=t, vec=v, method=m, between=bt, poly_smem=s, asm=0)
       for m, bt, s, (b, t, v) in itertools.product((0, 1, 2), (0, 1), (0, 1), ((64, 1, 1), (256, 4, 2)))]
)


@pytest.fixture(scope="module")
def pnpoly_small(gpu):
    from paper_2211_07260_b200.kernels import PnPolyProblem

    p = PnPolyProblem(n_points=1_000_003)  # ragged: not a multiple of any block*tile
    p.prepare(gpu)
    inp = p.inputs
    refs = {m: O.pnpoly(inp["points"], inp["vx"], inp["vy"], m) for m in range(4)}
    return p, refs


@pytest.mark.parametrize("cfg", PNPOLY_CONFIGS, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_pnpoly_bit_exact_across_configs(gpu, pnpoly_small, cfg):
    p, refs = pnpoly_small
    got = run_once(gpu, p, cfg)
    want = refs[p.formula(cfg)]
    assert got.dtype == np.int32 and got.shape == want.shape
    assert np.array_equal(got, want), f"{int((got != want).sum())} points differ"


@pytest.mark.parametrize("n", [1, 7, 4097])
def test_pnpoly_tiny_and_ragged_inputs(gpu, n):
    from paper_2211_07260_b200.kernels import PnPolyProblem

    p = PnPolyProblem(n_points=n)
    p.prepare(gpu)
    for cfg in (p.default_config(), dict(p.default_config(), asm=0, between=1, vec=1, tile=1)):
        got = run_once(gpu, p, cfg)
        np.testing.assert_array_equal(got, O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"],
                                                    p.formula(cfg)))


def test_pnpoly_degenerate_points_and_polygon(gpu):
    """Points on vertices, on horizontal/vertical edges and at y = vertex y;
    a polygon with horizontal edges and a repeated vertex."""
    from paper_2211_07260_b200.kernels import PnPolyProblem

    vx = np.array([0.0, 0.5, 0.5, 1.0, 1.0, 0.0, 0.0], np.float32)
    vy = np.array([0.0, 0.0, 0.25, 0.25, 1.0, 1.0, 1.0], np.float32)  # last vertex repeated
    xs = np.unique(np.concatenate([vx, vx + 1e-7, vx - 1e-7, [0.25, 0.75, -0.5, 1.5]])).astype(np.float32)
    ys = np.unique(np.concatenate([vy, vy + 1e-7, vy - 1e-7, [0.1, 0.6, -0.5, 1.5]])).astype(np.float32)
    pts = np.array([[x, y] for x in xs for y in ys], np.float32)
    p = PnPolyProblem(n_points=len(pts), n_vertices=vx.size)
    p.prepare(gpu, {"points": pts, "vx": vx, "vy": vy})
    pairs = [dict(block_size_x=128, tile=t, vec=2, method=2, between=0, poly_smem=int(a != 8), asm=a, persist=1)
             for t in (2, 8) for a in (7, 8, 9)]
    for cfg in PNPOLY_CONFIGS[::5] + pairs:  # 7 vertices: ASM 7/8 pad their 8-edge groups
        got = run_once(gpu, p, cfg)
        np.testing.assert_array_equal(got, O.pnpoly(pts, vx, vy, p.formula(cfg)), err_msg=str(cfg))
    # the four formulations must agree with the textbook answer on clear cases
    inside = run_once(gpu, p, p.default_config())
    lookup = {(float(x), float(y)): v for (x, y), v in zip(pts, inside)}
    f = lambda x, y: lookup[(float(np.float32(x)), float(np.float32(y)))]  # noqa: E731
    assert f(0.25, 0.1) == 1 and f(0.75, 0.6) == 1 and f(0.75, 0.1) == 0
    assert f(-0.5, 0.6) == 0 and f(1.5, 0.6) == 0


def test_pnpoly_full_size_tuned_bit_exact(gpu):
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import PnPolyProblem

    p = PnPolyProblem()  # 20,000,000 points x 600 vertices (BASELINE configs[0])
    p.prepare(gpu)
    for cfg in [tuned.best_config("pnpoly") or p.default_config(), tuned.best_config("pnpoly", "energy_optimal")]:
        if cfg is None:
            continue
        got = run_once(gpu, p, cfg)
        want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], p.formula(cfg))
        assert np.array_equal(got, want), f"{int((got != want).sum())} of 20M points differ"
        assert_full_size_pin(got)  # == formula 2; differs from the paper op order exactly where pinned
        # formula 3 (sign-bit) and the IEEE-compare formula 2 agree on this input
        assert np.array_equal(want, O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2))


def test_pnpoly_full_size_paper_op_order(gpu):
    """The brute-force kernel in the paper's Kernel-Tuner op order (METHOD 0: (dx*(py-vy))/dy + vx with IEEE
    rounding per op) over the whole BASELINE input reproduces the formula-0 oracle bitmap bit for bit
    (pinned by SHA-256 in tests/golden/pnpoly_full_pin.json)."""
    import hashlib
    import json

    from conftest import FULL_PIN
    from paper_2211_07260_b200.kernels import PnPolyProblem

    pin = json.loads(FULL_PIN.read_text())
    p = PnPolyProblem()
    p.prepare(gpu)
    for cfg in (dict(p.default_config(), method=0, asm=0), dict(p.default_config(), method=0, asm=0, poly_smem=0)):
        got = np.ascontiguousarray(run_once(gpu, p, cfg), dtype=np.int32)
        assert hashlib.sha256(got.tobytes()).hexdigest() == pin["sha256"]["formula0"], cfg
        for d in pin["formula0_vs_formula2_differ"]:
            assert got[d["index"]] == d["formula0"]


# -- Conv2D ------------------------------------------------------------------------------

CONV_CONFIGS = [
    dict(block_size_x=32, block_size_y=4, tile_size_x=4, tile_size_y=4, use_shmem=1, use_padding=0),
    dict(block_size_x=32, block_size_y=4, tile_size_x=4, tile_size_y=4, use_shmem=1, use_padding=1),
    dict(block_size_x=64, block_size_y=8, tile_size_x=8, tile_size_y=2, use_shmem=0, use_padding=0),
    dict(block_size_x=16, block_size_y=16, tile_size_x=1, tile_size_y=1, use_shmem=1, use_padding=0),
    dict(block_size_x=16, block_size_y=2, tile_size_x=2, tile_size_y=8, use_shmem=0, use_padding=0),
    dict(block_size_x=64, block_size_y=1, tile_size_x=2, tile_size_y=4, use_shmem=1, use_padding=1),
    dict(block_size_x=32, block_size_y=16, tile_size_x=1, tile_size_y=8, use_shmem=1, use_padding=0),
    dict(block_size_x=64, block_size_y=8, tile_size_x=8, tile_size_y=2, use_shmem=0, use_padding=0, fma2=1,
         min_blocks=2),
    dict(block_size_x=32, block_size_y=4, tile_size_x=4, tile_size_y=4, use_shmem=1, use_padding=0, min_blocks=2),
]


@pytest.mark.parametrize("cfg", CONV_CONFIGS, ids=lambda c: "-".join(str(v) for v in c.values()))
@pytest.mark.parametrize("shape", [(512, 512), (512, 256)])
def test_conv2d_within_fp32_tolerance(gpu, cfg, shape):
    from paper_2211_07260_b200.kernels import Conv2DProblem

    w, h = shape
    p = Conv2DProblem(width=w, height=h)
    p.prepare(gpu)
    got = run_once(gpu, p, cfg)
    err = O.conv2d_error(got, O.conv2d(p.inputs["image"], p.inputs["filter"]), p.inputs["image"],
                         p.inputs["filter"])
    assert err <= O.CONV_TOL


@pytest.mark.parametrize("cfg", [c for c in CONV_CONFIGS if c["tile_size_x"] % 2 == 0],
                         ids=lambda c: "-".join(str(v) for v in c.values()))
def test_conv2d_fma2_bit_identical_to_scalar(gpu, cfg):
    """fma2=1 (packed FFMA2 on even filter columns) computes the same fma.rn sequence per
    output as fma2=0, so the images agree bit for bit (and with the oracle's tolerance)."""
    from paper_2211_07260_b200.kernels import Conv2DProblem

    p = Conv2DProblem(width=512, height=256)
    p.prepare(gpu)
    scalar = run_once(gpu, p, dict(cfg, fma2=0)).copy()
    packed = run_once(gpu, p, dict(cfg, fma2=1))
    assert np.array_equal(scalar.view(np.uint32), packed.view(np.uint32))
    ref = O.conv2d(p.inputs["image"], p.inputs["filter"])
    assert O.conv2d_error(packed, ref, p.inputs["image"], p.inputs["filter"]) <= O.CONV_TOL


def test_conv2d_full_size_tuned(gpu):
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import Conv2DProblem

    p = Conv2DProblem()
    p.prepare(gpu)
    ref = O.conv2d(p.inputs["image"], p.inputs["filter"])
    for obj in ("time_optimal", "energy_optimal"):
        cfg = tuned.best_config("conv2d", obj) or p.default_config()
        got = run_once(gpu, p, cfg)
        assert O.conv2d_error(got, ref, p.inputs["image"], p.inputs["filter"]) <= O.CONV_TOL


# -- SGEMM ---------------------------------------------------------------------------------

SGEMM_CONFIGS = [
    {},
    dict(MWG=64, NWG=128, KWG=32, MDIMC=8, NDIMC=16, MDIMA=16, NDIMB=32, KWI=8, VWM=2, VWN=4, STRM=1, STRN=0),
    dict(MWG=64, NWG=64, KWG=16, MDIMC=16, NDIMC=16, MDIMA=16, NDIMB=16, KWI=2, VWM=1, VWN=1, STRM=0, STRN=0),
    dict(MWG=128, NWG=64, KWG=16, MDIMC=16, NDIMC=8, MDIMA=32, NDIMB=8, KWI=2, VWM=2, VWN=2, SA=0, SB=1),
    dict(MWG=32, NWG=32, KWG=16, MDIMC=8, NDIMC=8, MDIMA=8, NDIMB=8, KWI=8, VWM=4, VWN=4, SA=0, SB=0),
    dict(MWG=128, NWG=128, KWG=16, MDIMC=32, NDIMC=8, MDIMA=32, NDIMB=32, KWI=2, VWM=4, VWN=4, STRM=0, STRN=1),
    # cp.async stages (ASYNC): 2 and 3 stages, vector widths 1 / 2 / 4 (4-, 8- and 16-byte copies)
    dict(MWG=128, NWG=128, KWG=32, MDIMC=16, NDIMC=16, MDIMA=32, NDIMB=32, KWI=8, VWM=4, VWN=4, ASYNC=2),
    dict(MWG=128, NWG=64, KWG=32, MDIMC=16, NDIMC=8, MDIMA=16, NDIMB=16, KWI=8, VWM=4, VWN=4, STRN=0, ASYNC=3),
    dict(MWG=64, NWG=64, KWG=16, MDIMC=16, NDIMC=16, MDIMA=16, NDIMB=16, KWI=2, VWM=1, VWN=2, STRM=0, ASYNC=2),
    dict(MWG=32, NWG=64, KWG=16, MDIMC=8, NDIMC=8, MDIMA=8, NDIMB=16, KWI=8, VWM=2, VWN=1, ASYNC=3),
]


@pytest.mark.parametrize("overrides", SGEMM_CONFIGS, ids=range(len(SGEMM_CONFIGS)))
@pytest.mark.parametrize("mnk,beta", [((512, 512, 512), 0.5), ((256, 384, 128), 0.0)])
def test_sgemm_within_fp32_tolerance(gpu, overrides, mnk, beta):
    from paper_2211_07260_b200.kernels import SgemmProblem

    m, n, k = mnk
    p = SgemmProblem(m=m, n=n, k=k, beta=beta)
    p.prepare(gpu)
    cfg = {**p.default_config(), **overrides}
    got = run_once(gpu, p, cfg)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    assert O.sgemm_error(got, ref) <= O.SGEMM_TOL


@pytest.mark.parametrize("overrides", [c for c in SGEMM_CONFIGS if c.get("VWN", 4) % 2 == 0],
                         ids=lambda c: str(sorted(c.items())))
def test_sgemm_fma2_bit_identical_to_scalar(gpu, overrides):
    """FMA2=1 (packed FFMA2 outer product) gives C bit for bit equal to FMA2=0."""
    from paper_2211_07260_b200.kernels import SgemmProblem

    p = SgemmProblem(m=512, n=512, k=512, beta=0.5)
    p.prepare(gpu)
    cfg = {**p.default_config(), **overrides}
    scalar = run_once(gpu, p, dict(cfg, FMA2=0)).copy()
    packed = run_once(gpu, p, dict(cfg, FMA2=1))
    assert np.array_equal(scalar.view(np.uint32), packed.view(np.uint32))
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    assert O.sgemm_error(packed, ref) <= O.SGEMM_TOL


def _clblast_sample(n=16, seed=7):
    import random

    from paper_2211_07260_b200.kernels import SgemmProblem

    cfgs = [c.as_dict() for c in SgemmProblem(value_set="clblast").space().enumerate()]
    rng = random.Random(seed)
    extremes = [c for c in cfgs if c["VWM"] == 8 and c["VWN"] == 8][:2] + \
        [c for c in cfgs if c["MWG"] == c["NWG"] == 128 and c["SA"] == c["SB"] == 1][:2] + \
        [c for c in cfgs if c["SA"] == c["SB"] == 0][:1]
    return extremes + rng.sample(cfgs, n)


@pytest.mark.parametrize("overrides", _clblast_sample(), ids=lambda c: "-".join(str(v) for v in c.values()))
def test_sgemm_paper_clblast_space(gpu, overrides):
    """Configs of the paper's 17,472-config CLBlast space (float8 vectors, > 48 KB of double-buffered
    shared memory, global-memory fragments) within the FP32 bar."""
    from paper_2211_07260_b200.kernels import SgemmProblem

    p = SgemmProblem(m=256, n=256, k=128, value_set="clblast")
    p.prepare(gpu)
    cfg = {**p.default_config(), **overrides}
    assert p.is_valid(cfg)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    assert O.sgemm_error(run_once(gpu, p, cfg), ref) <= O.SGEMM_TOL


def test_sgemm_group_m_rasterisation_bit_identical(gpu):
    """GROUP_M only reorders CTAs: the same bits as launch order."""
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import SgemmProblem

    p = SgemmProblem(m=1024, n=768, k=256)
    p.prepare(gpu)
    base = {**p.default_config(), **(tuned.best_config("sgemm") or {})}
    one = run_once(gpu, p, {**base, "GROUP_M": 1}).copy()
    for g in (4, 8, 16):
        np.testing.assert_array_equal(run_once(gpu, p, {**base, "GROUP_M": g}), one)


SPLIT_BASE = {"MWG": 128, "NWG": 128, "KWG": 16, "MDIMC": 16, "NDIMC": 8, "MDIMA": 16, "NDIMB": 16, "KWI": 8,
              "VWM": 4, "VWN": 4, "STRM": 1, "STRN": 1, "SA": 1, "SB": 1, "ASYNC": 4, "FMA2": 1, "GROUP_M": 1}


@pytest.mark.parametrize("overrides", [{}, {"GROUP_M": 8}, {"ASYNC": 0}, {"ASYNC": 0, "SA": 0, "SB": 0, "FMA2": 0},
                                       {"SPLIT_TAIL": 4}], ids=str)
@pytest.mark.parametrize("mnk", [(2816, 2304, 512), (2560, 2304, 272), (1024, 1024, 400)], ids=str)
def test_sgemm_split_tail(gpu, overrides, mnk):
    """SPLIT_TAIL: the last partial wave's tiles split along K over 2-4 CTAs, partials summed through
    the workspace by the last arriver. Within the FP32 bar, the per-tile counters left at zero, and
    bit-reproducible over relaunches (the partials are summed in part order, not arrival order)."""
    from paper_2211_07260_b200.kernels import SgemmProblem

    m, n, k = mnk
    p = SgemmProblem(m=m, n=n, k=k, beta=0.5, value_set="b200")
    p.prepare(gpu)
    cfg = {**SPLIT_BASE, "SPLIT_TAIL": 2, **overrides}
    full, split, grid = p.tail_plan(cfg)
    tiles = (m // 128) * (n // 128)
    assert full % gpu.sm_count == 0 and grid == full + (tiles - full) * split
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    first = run_once(gpu, p, cfg).copy()
    assert O.sgemm_error(first, ref) <= O.SGEMM_TOL
    for _ in range(2):
        np.testing.assert_array_equal(run_once(gpu, p, cfg).view(np.uint32), first.view(np.uint32))
    if (m, n) == (1024, 1024):  # 64 tiles < half of any wave: all of them split along K
        assert full == 0 and split >= 2, (full, split, grid)
    if split > 1:
        assert not p.buffers["tail_counters"].download().any()
    whole = run_once(gpu, p, {**cfg, "SPLIT_TAIL": 0})
    # whole tiles are bit-identical to the plain grid; split tiles differ by one rounding at most
    assert O.sgemm_error(whole, ref) <= O.SGEMM_TOL


def test_sgemm_split_tail_plan_at_4096(gpu):
    """At 4096^3 the tuned 128 x 128 config leaves a partial 4th wave (1024 tiles over 2 x 148
    resident CTAs): the plan runs 888 whole tiles and splits the other 136 in two."""
    from paper_2211_07260_b200.kernels import SgemmProblem

    p = SgemmProblem(value_set="b200")
    p.prepare(gpu)
    cfg = {**SPLIT_BASE, "SPLIT_TAIL": 2}
    per_sm = p.kernel(cfg).occupancy(128, p.smem_bytes(cfg))
    full, split, grid = p.tail_plan(cfg)
    slots = per_sm * gpu.sm_count
    assert full == 1024 // slots * slots and split == min(2, slots // (1024 - full))
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    assert O.sgemm_error(run_once(gpu, p, cfg), ref) <= O.SGEMM_TOL


def test_sgemm_tf32_group_m_walk(gpu):
    """GROUP_M reorders the persistent tile walk only: without split tails the same bits, with them
    (which tiles get K-split changes) still inside the TF32 bar."""
    from paper_2211_07260_b200.kernels import SgemmTF32Problem

    p = SgemmTF32Problem(m=1024, n=1024, k=256)
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    for pair in (0, 1):
        base = dict(BN=256, STAGES=4, PERSIST=1, SPLIT_TAIL=0, PAIR=pair, GROUP_M=1)
        one = run_once(gpu, p, base).copy()
        for g in (4, 8):
            np.testing.assert_array_equal(run_once(gpu, p, {**base, "GROUP_M": g}), one)
            err = O.sgemm_error(run_once(gpu, p, {**base, "GROUP_M": g, "SPLIT_TAIL": 1}), ref)
            assert 1e-6 < err <= O.SGEMM_TF32_TOL


def test_sgemm_full_size_tuned(gpu):
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import SgemmProblem

    p = SgemmProblem()
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    for obj in ("time_optimal", "energy_optimal"):
        cfg = tuned.best_config("sgemm", obj) or p.default_config()
        assert O.sgemm_error(run_once(gpu, p, cfg), ref) <= O.SGEMM_TOL


# -- host-buffer API (suite) ---------------------------------------------------------------


def test_suite_host_api_matches_oracles():
    from paper_2211_07260_b200 import suite
    from paper_2211_07260_b200.kernels import Conv2DProblem, PnPolyProblem, SgemmProblem

    ci = Conv2DProblem(width=256, height=256).host_inputs()
    out = suite.conv2d(ci["image"], ci["filter"])
    assert O.conv2d_error(out, O.conv2d(ci["image"], ci["filter"]), ci["image"], ci["filter"]) <= O.CONV_TOL
    # second call with a different image reuses the runner and re-uploads
    img2 = ci["image"][::-1].copy()
    out2 = suite.conv2d(img2, ci["filter"])
    assert O.conv2d_error(out2, O.conv2d(img2, ci["filter"]), img2, ci["filter"]) <= O.CONV_TOL
    pi = PnPolyProblem(n_points=100_000).host_inputs()
    got = suite.pnpoly(pi["points"], pi["vx"], pi["vy"])
    np.testing.assert_array_equal(got, O.pnpoly(pi["points"], pi["vx"], pi["vy"], 3))
    si = SgemmProblem(m=256, n=128, k=64).host_inputs()
    c = suite.sgemm(si["a"], si["b"], si["c0"], 1.0, 0.5, config=SgemmProblem().default_config() | {
        "MWG": 64, "NWG": 64, "MDIMC": 16, "NDIMC": 16, "MDIMA": 16, "NDIMB": 16})
    assert O.sgemm_error(c, O.sgemm(si["a"], si["b"], si["c0"], 1.0, 0.5)) <= O.SGEMM_TOL
    ti = SgemmProblem(m=512, n=256, k=96).host_inputs()
    t = suite.sgemm_tf32(ti["a"], ti["b"], ti["c0"], 1.0, 0.5)  # tuned CTA-pair config fits 512 x 256
    err = O.sgemm_error(t, O.sgemm(ti["a"], ti["b"], ti["c0"], 1.0, 0.5))
    assert 1e-6 < err <= O.SGEMM_TF32_TOL


@pytest.mark.parametrize("m,n,k", [(1000, 1000, 1000), (1023, 777, 513), (4096, 4096, 4096)])
def test_suite_sgemm_any_shape(m, n, k):
    """Shapes the tuned tiles do not divide run padded (CLBlast's indirect GEMM): A is uploaded row-major and
    transposed + zero-padded on the device (no host transpose), B / C go in with pitched copies."""
    from paper_2211_07260_b200 import suite

    rng = np.random.default_rng(m + n + k)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    c = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    ref = O.sgemm(a, b, c, 1.0, 0.5)
    assert O.sgemm_error(suite.sgemm(a, b, c, 1.0, 0.5), ref) <= O.SGEMM_TOL
    # column-major A (a Fortran-ordered view) is already the kernel's layout: pitched copy, same result
    np.testing.assert_array_equal(suite.sgemm(np.asfortranarray(a), b, c, 1.0, 0.5), suite.sgemm(a, b, c, 1.0, 0.5))
    err = O.sgemm_error(suite.sgemm_tf32(a, b, c, 1.0, 0.5), ref)
    assert 1e-6 < err <= O.SGEMM_TF32_TOL


def test_suite_conv2d_untileable_width_and_bad_shapes():
    from paper_2211_07260_b200 import suite
    from paper_2211_07260_b200.kernels import Conv2DProblem

    ci = Conv2DProblem(width=4095, height=4095).host_inputs()  # 4111^2 image -> 4095^2 output
    out = suite.conv2d(ci["image"], ci["filter"])
    assert out.shape == (4095, 4095)
    for rows in (slice(0, 24), slice(2000, 2008), slice(4071, 4095)):  # bounded oracle bands incl. the edges
        ref = O.conv2d_rows(ci["image"], ci["filter"], rows)
        assert O.conv2d_error(out[rows], ref, ci["image"], ci["filter"]) <= O.CONV_TOL
    small = Conv2DProblem(width=37, height=29).host_inputs()
    got = suite.conv2d(small["image"], small["filter"])
    assert O.conv2d_error(got, O.conv2d(small["image"], small["filter"]), small["image"], small["filter"]) <= O.CONV_TOL
    import paper_2211_07260_b200 as B

    with pytest.raises(B.ConfigurationError):
        suite.conv2d(np.zeros((8, 8), np.float32), ci["filter"])  # image smaller than the filter
    with pytest.raises(B.ConfigurationError):
        suite.sgemm(np.zeros((4, 5), np.float32), np.zeros((6, 4), np.float32), np.zeros((4, 4), np.float32))


def test_suite_pipelined_strips_match_single_launch():
    """Pipelined host calls (bands / chunks over 3 streams) give the single-launch bits."""
    from paper_2211_07260_b200 import suite
    from paper_2211_07260_b200.kernels import Conv2DProblem, PnPolyProblem

    ci = Conv2DProblem(width=512, height=496).host_inputs()  # 31 tile rows: ragged last band
    one = suite.conv2d(ci["image"], ci["filter"], strips=1)
    for n in (2, 5, 16):
        np.testing.assert_array_equal(suite.conv2d(ci["image"], ci["filter"], strips=n), one)
    assert O.conv2d_error(one, O.conv2d(ci["image"], ci["filter"]), ci["image"], ci["filter"]) <= O.CONV_TOL
    img_pinned = suite.pinned(ci["image"].shape)
    img_pinned[...] = ci["image"]
    out_pinned = suite.pinned(one.shape)
    suite.conv2d(img_pinned, ci["filter"], out=out_pinned, strips=8)
    np.testing.assert_array_equal(out_pinned, one)
    pi = PnPolyProblem(n_points=1_000_003).host_inputs()  # not a multiple of any chunk
    want = O.pnpoly(pi["points"], pi["vx"], pi["vy"], 3)
    for n in (1, 3, 16):
        np.testing.assert_array_equal(suite.pnpoly(pi["points"], pi["vx"], pi["vy"], strips=n), want)


def test_suite_conv2d_many_matches_single_calls():
    """conv2d_many (pipelined across images over two device buffer sets) gives, image for
    image, the bits of separate single-launch calls; odd counts and repeated output
    buffers included."""
    from paper_2211_07260_b200 import suite
    from paper_2211_07260_b200.kernels import Conv2DProblem

    rng = np.random.default_rng(5)
    filt = rng.uniform(0, 1, (17, 17)).astype(np.float32)
    images = [rng.uniform(0, 1, (496 + 16, 512 + 16)).astype(np.float32) for _ in range(5)]
    want = [suite.conv2d(im, filt, strips=1).copy() for im in images]
    for strips in (1, 4):
        got = suite.conv2d_many(images, filt, strips=strips)
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w)
    pinned = [suite.pinned(want[0].shape) for _ in range(2)]
    suite.conv2d_many(images[:4], filt, outs=[pinned[0], pinned[1], pinned[0], pinned[1]], strips=3)
    np.testing.assert_array_equal(pinned[0], want[2])
    np.testing.assert_array_equal(pinned[1], want[3])
    p = Conv2DProblem(width=512, height=496)
    assert O.conv2d_error(want[0], O.conv2d(images[0], filt), images[0], filt) <= O.CONV_TOL
    assert p.width == 512


# -- SGEMM on tcgen05 (TF32, its own tolerance) -------------------------------------------------


_TF32 = {"PERSIST": 0, "SPLIT_TAIL": 0, "PAIR": 0}
TF32_CONFIGS = [_TF32 | c for c in (
    {"BN": 64, "STAGES": 3}, {"BN": 128, "STAGES": 6}, {"BN": 256, "STAGES": 2}, {"BN": 256, "STAGES": 4},
    {"BN": 128, "STAGES": 4, "PERSIST": 1}, {"BN": 256, "STAGES": 4, "PERSIST": 1, "SPLIT_TAIL": 1},
    {"BN": 128, "STAGES": 6, "PAIR": 1}, {"BN": 256, "STAGES": 4, "PAIR": 1},
    # persistent CTA pairs (sgemm_tf32c2p.cu), with and without the split-K tail
    {"BN": 256, "STAGES": 4, "PAIR": 1, "PERSIST": 1}, {"BN": 128, "STAGES": 5, "PAIR": 1, "PERSIST": 1},
    {"BN": 256, "STAGES": 5, "PAIR": 1, "PERSIST": 1, "SPLIT_TAIL": 1})]


@pytest.mark.parametrize("cfg", TF32_CONFIGS, ids=str)
@pytest.mark.parametrize("mnk,beta", [((256, 256, 256), 0.5), ((384, 512, 96), 0.0), ((512, 768, 160), 1.0),
                                      ((2560, 2048, 1024), 0.5)])
def test_sgemm_tf32_tcgen05_within_tf32_tolerance(gpu, cfg, mnk, beta):
    from paper_2211_07260_b200.kernels import SgemmTF32Problem

    m, n, k = mnk
    p = SgemmTF32Problem(m=m, n=n, k=k, beta=beta)
    if not p.is_valid(cfg):
        pytest.skip("shape not a multiple of this config's tile")
    p.prepare(gpu)
    got = run_once(gpu, p, cfg)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    err = O.sgemm_error(got, ref)
    assert err <= O.SGEMM_TF32_TOL
    assert err > 1e-6  # really TF32 inputs, not an FP32 path
    if cfg.get("SPLIT_TAIL"):  # the split-K reduction has a fixed order: a relaunch gives the same bits
        again = run_once(gpu, p, cfg)
        assert np.array_equal(got.view(np.uint32), again.view(np.uint32))


def test_sgemm_tf32_full_size(gpu):
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import SgemmTF32Problem

    p = SgemmTF32Problem()
    p.prepare(gpu)
    cfg = tuned.best_config("sgemm_tf32") or p.default_config()
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    assert O.sgemm_error(run_once(gpu, p, cfg), ref) <= O.SGEMM_TF32_TOL


@pytest.mark.parametrize("cfg", [{"BN": 128, "STAGES": 4, "PERSIST": 1, "SPLIT_TAIL": 1, "PAIR": 0},
                                 {"BN": 256, "STAGES": 3, "PERSIST": 1, "SPLIT_TAIL": 1, "PAIR": 0}], ids=str)
def test_sgemm_tf32_persistent_split_tail(gpu, cfg):
    """More tiles than SMs with a short last wave: the tail tiles are split along K over two
    CTAs and reduced through the workspace. Relaunching must keep the result (the per-tile
    arrival counters only grow; their parity marks the second finisher)."""
    from paper_2211_07260_b200.kernels import SgemmTF32Problem

    p = SgemmTF32Problem(m=2304, n=2304, k=256, beta=0.5)
    p.prepare(gpu)
    tiles = p.tiles(cfg)
    assert tiles > gpu.sm_count and 0 < 2 * (tiles % gpu.sm_count) <= gpu.sm_count  # the split path runs
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    first = run_once(gpu, p, cfg)
    assert O.sgemm_error(first, ref) <= O.SGEMM_TF32_TOL
    for _ in range(2):
        np.testing.assert_array_equal(run_once(gpu, p, cfg), first)  # deterministic split-K reduction

