"""PnPoly slab kernel (csrc/kernels/pnpoly_slab.cu) on the B200 through libjt:
bit-exact against the brute-force oracle formulation 2 (oracle/pnpoly_oracle.c)."""

import itertools

import numpy as np
import pytest
from conftest import assert_full_size_pin

from oracle import kernels_oracle as O

pytestmark = pytest.mark.gpu

SLAB_CONFIGS = (
    [dict(block_size_x=b, tile=t, sort=s, pairs_smem=ps, xbuckets=0, buckets=4096)
     for b, t, s, ps in itertools.product((128, 512, 1024), (1, 4, 8), (0, 1), (0, 1))
     if not (ps and s and b * t > 2048)]
    + [dict(block_size_x=256, tile=8, sort=1, pairs_smem=0, xbuckets=0, buckets=1024),
       dict(block_size_x=1024, tile=8, sort=1, pairs_smem=0, xbuckets=0, buckets=1024)]
    + [dict(block_size_x=b, tile=t, sort=0, pairs_smem=0, xbuckets=x, exact_flags=f, half=h, buckets=g)
       for b, t, x, f, h, g in itertools.product((128, 512, 1024), (1, 4, 8), (4, 16), (0, 1), (0, 1), (1024, 4096))]
)


@pytest.fixture(scope="module")
def gpu():
    from paper_2211_07260_b200.gpu import GPU

    g = GPU(0)
    yield g
    g.close()


def run_once(gpu, problem, cfg):
    k = problem.kernel(cfg)
    problem.reset_output()
    gpu.launch(k, problem.launch(cfg), problem.args(cfg))
    gpu.synchronize()
    return problem.fetch_output()


@pytest.fixture(scope="module")
def slab_small(gpu):
    from paper_2211_07260_b200.kernels import PnPolySlabProblem

    p = PnPolySlabProblem(n_points=1_000_003)
    p.prepare(gpu)
    return p, O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)


@pytest.mark.parametrize("cfg", SLAB_CONFIGS, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_slab_bit_exact_across_configs(gpu, slab_small, cfg):
    p, want = slab_small
    assert p.is_valid(cfg)
    got = run_once(gpu, p, cfg)
    assert np.array_equal(got, want), f"{int((got != want).sum())} points differ"


@pytest.mark.parametrize("n", [1, 7, 4097])
def test_slab_tiny_and_ragged_inputs(gpu, n):
    from paper_2211_07260_b200.kernels import PnPolySlabProblem

    p = PnPolySlabProblem(n_points=n)
    p.prepare(gpu)
    for cfg in (p.default_config(), dict(p.default_config(), sort=0, tile=1)):
        np.testing.assert_array_equal(run_once(gpu, p, cfg),
                                      O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2))


def test_slab_degenerate_points_and_polygon(gpu):
    """Points on vertices / edges / at vertex ordinates, +-0.0, +-inf and NaN
    coordinates; a polygon with horizontal edges and a repeated vertex."""
    from paper_2211_07260_b200.kernels import PnPolySlabProblem

    vx = np.array([0.0, 0.5, 0.5, 1.0, 1.0, 0.0, 0.0], np.float32)
    vy = np.array([0.0, 0.0, 0.25, 0.25, 1.0, 1.0, 1.0], np.float32)
    special = [0.0, -0.0, np.inf, -np.inf, np.nan, 0.25, 0.75, -0.5, 1.5]
    xs = np.concatenate([vx, vx + 1e-7, vx - 1e-7, special]).astype(np.float32)
    ys = np.concatenate([vy, vy + 1e-7, vy - 1e-7, special]).astype(np.float32)
    pts = np.array([[x, y] for x in xs for y in ys], np.float32)
    p = PnPolySlabProblem(n_points=len(pts), n_vertices=vx.size)
    p.prepare(gpu, {"points": pts, "vx": vx, "vy": vy})
    want = O.pnpoly(pts, vx, vy, 2)
    for cfg in SLAB_CONFIGS[::3]:
        np.testing.assert_array_equal(run_once(gpu, p, cfg), want, err_msg=str(cfg))


def test_slab_matches_brute_force_kernel_full_size(gpu):
    """20 M points x 600 vertices: the slab bitmap equals the oracle's formulation 2
    (the precomputed slope / intercept form the brute-force METHOD 2 kernel computes)."""
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import PnPolySlabProblem

    p = PnPolySlabProblem()
    p.prepare(gpu)
    want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)
    for cfg in {str(c): c for c in [p.default_config(), tuned.best_config("pnpoly_slab"),
                                    tuned.best_config("pnpoly_slab", "energy_optimal")] if c}.values():
        got = run_once(gpu, p, cfg)
        assert np.array_equal(got, want), f"{int((got != want).sum())} of 20M points differ ({cfg})"
        assert_full_size_pin(got)  # == formula 2; differs from the paper op order exactly where pinned


@pytest.mark.parametrize("strips", [1, 5])
def test_slab_host_api_matches_brute_force(gpu, strips):
    """suite.pnpoly(algorithm="slab" / "grid" / "cells") through pinned host buffers equals the
    brute-force call."""
    from paper_2211_07260_b200 import suite
    from paper_2211_07260_b200.kernels import PnPolyProblem

    inp = PnPolyProblem(n_points=1_500_007).host_inputs()
    pts = suite.pinned(inp["points"].shape, np.float32)
    pts[...] = inp["points"]
    slab = suite.pnpoly(pts, inp["vx"], inp["vy"], strips=strips, algorithm="slab").copy()
    grid = suite.pnpoly(pts, inp["vx"], inp["vy"], strips=strips, algorithm="grid").copy()
    np.testing.assert_array_equal(grid, slab)
    cells = suite.pnpoly(pts, inp["vx"], inp["vy"], strips=strips, algorithm="cells").copy()
    np.testing.assert_array_equal(cells, slab)
    brute = suite.pnpoly(pts, inp["vx"], inp["vy"], strips=strips,
                         config=dict(PnPolyProblem().default_config(), asm=0, method=2)).copy()
    np.testing.assert_array_equal(slab, brute)
    np.testing.assert_array_equal(slab, O.pnpoly(inp["points"], inp["vx"], inp["vy"], 2))


EXTREME = {
    "flat": (np.array([0.0, 1.0, 2.0, 0.5], np.float32), np.array([0.25, 0.25, 0.25, 0.25], np.float32), 1.0),
    "tiny": (np.array([0.0, 3e-30, 1e-30], np.float32), np.array([0.0, 1e-30, 4e-30], np.float32), 5e-30),
    "huge": (np.array([-1e30, 2e30, 0.0, 5e29], np.float32), np.array([-1e30, 0.0, 3e30, 1e29], np.float32), 4e30),
}


@pytest.mark.parametrize("shape", sorted(EXTREME))
def test_slab_and_grid_extreme_polygons(gpu, shape):
    """Zero-height, 1e-30-sized and 1e30-sized polygons through the slab and grid kernels."""
    from paper_2211_07260_b200.kernels import PnPolyCellsProblem, PnPolyGridProblem, PnPolySlabProblem

    vx, vy, span = EXTREME[shape]
    rng = np.random.default_rng(21)
    pts = np.concatenate([rng.uniform(-span, span, (100_003, 2)), np.stack([vx, vy], 1)]).astype(np.float32)
    want = O.pnpoly(pts, vx, vy, 2)
    for cls, cfgs in ((PnPolySlabProblem, SLAB_CONFIGS[::6]), (PnPolyGridProblem, GRID_CONFIGS[::4]),
                      (PnPolyCellsProblem, CELLS_CONFIGS[::5])):
        p = cls(n_points=len(pts), n_vertices=vx.size)
        p.prepare(gpu, {"points": pts, "vx": vx, "vy": vy})
        for cfg in [c for c in cfgs if p.is_valid(c)] + [p.default_config()]:
            np.testing.assert_array_equal(run_once(gpu, p, cfg), want, err_msg=f"{shape} {cls.__name__} {cfg}")


@pytest.mark.parametrize("shape", ["star3000", "convex50", "comb"])
def test_slab_other_polygons(gpu, shape):
    """Slab kernel on polygons unlike the benchmark one: a 3000-vertex star (long slab
    lists), a 50-vertex convex polygon (2 edges per slab) and a comb with shared
    vertex ordinates and horizontal edges."""
    from paper_2211_07260_b200.kernels import PnPolySlabProblem

    rng = np.random.default_rng(11)
    if shape == "star3000":
        th = np.sort(rng.uniform(0, 2 * np.pi, 3000))
        rad = 0.4 + 0.5 * rng.uniform(0, 1, 3000)
    elif shape == "convex50":
        th = np.sort(rng.uniform(0, 2 * np.pi, 50))
        rad = np.full(50, 0.9)
    if shape == "comb":
        vx = np.array([0, 4, 4, 3, 3, 2, 2, 1, 1, 0], np.float32) / 4 - 0.5
        vy = np.array([0, 0, 3, 3, 1, 1, 3, 3, 1, 1], np.float32) / 3 - 0.5
    else:
        vx, vy = (rad * np.cos(th)).astype(np.float32), (rad * np.sin(th)).astype(np.float32)
    pts = rng.uniform(-1, 1, (300_001, 2)).astype(np.float32)
    pts[:vx.size] = np.stack([vx, vy], 1)  # exactly on the vertices
    p = PnPolySlabProblem(n_points=len(pts), n_vertices=vx.size)
    p.prepare(gpu, {"points": pts, "vx": vx, "vy": vy})
    want = O.pnpoly(pts, vx, vy, 2)
    cfgs = [c for c in SLAB_CONFIGS[::4] if p.is_valid(c)] + [p.default_config()]
    assert cfgs
    for cfg in cfgs:
        np.testing.assert_array_equal(run_once(gpu, p, cfg), want, err_msg=f"{shape} {cfg}")


def test_slab_through_tune_kernel():
    """The paper-style facade tunes the slab kernel as a built-in problem."""
    from paper_2211_07260_b200 import tune_kernel

    rows, outcome = tune_kernel("pnpoly_slab", tune_params={"block_size_x": [512, 1024], "tile": [2], "sort": [0],
                                                            "pairs_smem": [0], "xbuckets": [16], "exact_flags": [0],
                                                            "half": [0, 1], "buckets": [4096]},
                                problem_kwargs={"n_points": 1 << 20}, duration=0.05)
    assert len(rows) == 4 and not any(r["failed"] for r in rows)
    # a work-skipping kernel: points/s, GB/s and joules per bitmap, no brute-force flop credit
    best = outcome.best.metrics
    assert "gflops" not in best and best["points_per_s"] > 1e9 and best["j_per_bitmap"] == outcome.best.energy
    assert best["gb_per_s"] == pytest.approx(best["points_per_s"] * 12 / 1e9, rel=1e-3)


# -- uniform-cell fast path in front of the slab search (csrc/kernels/pnpoly_grid.cu) ---------

GRID_CONFIGS = ([dict(block_size_x=b, tile=t, grid=g, grid_smem=1, xbuckets=x, buckets=4096)
                 for b, t, g, x in itertools.product((256, 1024), (1, 4), (256, 512), (8, 16))]
                + [dict(block_size_x=b, tile=t, grid=g, grid_smem=0, xbuckets=16, buckets=1024)
                   for b, t, g in itertools.product((256, 1024), (2,), (512, 1024, 2048))])


@pytest.fixture(scope="module")
def grid_small(gpu):
    from paper_2211_07260_b200.kernels import PnPolyGridProblem

    p = PnPolyGridProblem(n_points=1_000_003)
    p.prepare(gpu)
    return p, O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)


@pytest.mark.parametrize("cfg", GRID_CONFIGS, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_grid_bit_exact_across_configs(gpu, grid_small, cfg):
    p, want = grid_small
    assert p.is_valid(cfg)
    got = run_once(gpu, p, cfg)
    assert np.array_equal(got, want), f"{int((got != want).sum())} points differ"


@pytest.mark.parametrize("n", [1, 7, 33, 4097])
def test_grid_tiny_and_ragged_inputs(gpu, n):
    from paper_2211_07260_b200.kernels import PnPolyGridProblem

    p = PnPolyGridProblem(n_points=n)
    p.prepare(gpu)
    for cfg in (p.default_config(), dict(p.default_config(), block_size_x=256, tile=1, grid=256),
                dict(p.default_config(), grid=2048, grid_smem=0)):
        np.testing.assert_array_equal(run_once(gpu, p, cfg),
                                      O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2))


@pytest.mark.parametrize("kind", ["grid", "cells"])
@pytest.mark.parametrize("shape", ["degenerate", "star3000", "convex50", "comb"])
def test_grid_other_polygons_and_special_points(gpu, shape, kind):
    """Degenerate polygon with +-0, +-inf and NaN coordinates; the slab tests' other polygons;
    points exactly on vertices and on cell borders (grid and cell-list kernels)."""
    from paper_2211_07260_b200 import native
    from paper_2211_07260_b200.kernels import PnPolyCellsProblem, PnPolyGridProblem

    rng = np.random.default_rng(12)
    if shape == "degenerate":
        vx = np.array([0.0, 0.5, 0.5, 1.0, 1.0, 0.0, 0.0], np.float32)
        vy = np.array([0.0, 0.0, 0.25, 0.25, 1.0, 1.0, 1.0], np.float32)
    elif shape == "comb":
        vx = np.array([0, 4, 4, 3, 3, 2, 2, 1, 1, 0], np.float32) / 4 - 0.5
        vy = np.array([0, 0, 3, 3, 1, 1, 3, 3, 1, 1], np.float32) / 3 - 0.5
    else:
        m = 3000 if shape == "star3000" else 50
        th = np.sort(rng.uniform(0, 2 * np.pi, m))
        rad = 0.4 + 0.5 * rng.uniform(0, 1, m) if m == 3000 else np.full(m, 0.9)
        vx, vy = (rad * np.cos(th)).astype(np.float32), (rad * np.sin(th)).astype(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 0.25, -0.5, 1.5], np.float32)
    pts = [rng.uniform(-1.2, 1.2, (200_001, 2)).astype(np.float32), np.stack([vx, vy], 1),
           np.array([[a, b] for a in special for b in special], np.float32)]
    for g in (256, 512, 2048):
        _, prm, _ = native.pnpoly_grid(vx, vy, g, g)
        xs = ((np.arange(g + 1, dtype=np.float64) - prm[1]) / prm[0]).astype(np.float32)
        pts.append(np.stack([xs, rng.uniform(-1, 1, xs.size).astype(np.float32)], 1))
    pts = np.ascontiguousarray(np.concatenate(pts).astype(np.float32))
    cls, configs = (PnPolyGridProblem, GRID_CONFIGS[::3]) if kind == "grid" else (PnPolyCellsProblem, CELLS_CONFIGS[::3])
    p = cls(n_points=len(pts), n_vertices=vx.size)
    p.prepare(gpu, {"points": pts, "vx": vx, "vy": vy})
    want = O.pnpoly(pts, vx, vy, 2)
    cfgs = [c for c in configs if p.is_valid(c)] + [p.default_config()]
    if kind == "cells":
        cfgs.append(dict(p.default_config(), lmax=0))  # every undecided cell -> slab search
        cfgs += [dict(p.default_config(), adrain=0, pushv=1, hpf=1, quad=1),
                 dict(p.default_config(), defer=1, min_blocks=1), dict(p.default_config(), defer=1, lmax=0, head32=1),
                 dict(p.default_config(), defer=1, quad=1, tile=2, block_size_x=512, min_blocks=2)]
    for cfg in cfgs:
        np.testing.assert_array_equal(run_once(gpu, p, cfg), want, err_msg=f"{shape} {cfg}")


def test_grid_full_size_matches_brute_force(gpu):
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import PnPolyGridProblem

    p = PnPolyGridProblem()
    p.prepare(gpu)
    want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)
    for cfg in {str(c): c for c in [p.default_config(), tuned.best_config("pnpoly_grid"),
                                    tuned.best_config("pnpoly_grid", "energy_optimal")] if c}.values():
        got = run_once(gpu, p, cfg)
        assert np.array_equal(got, want), f"{int((got != want).sum())} of 20M points differ ({cfg})"
        assert_full_size_pin(got)  # == formula 2; differs from the paper op order exactly where pinned
    assert p.clean_fraction(512) > 0.9


# -- per-cell edge lists (csrc/kernels/pnpoly_cells.cu) --------------------------------------

CELLS_CONFIGS = ([dict(block_size_x=b, tile=t, grid=g, grid_smem=1, lmax=l, stream=st, prefetch=(b + t + st) % 3,
                       regpf=(t + l) % 2, adrain=(g // 256 + st) % 2, head32=(b // 256 + l) % 2)
                  for b, t, g, l, st in itertools.product((256, 1024), (1, 2, 4), (256, 512), (4, 16), (0, 1))]
                 + [dict(block_size_x=b, tile=2, grid=g, grid_smem=0, lmax=16, stream=0, prefetch=pf, regpf=pf // 2, adrain=1, head32=pf // 2)
                    for b, g, pf in itertools.product((256, 1024), (512, 1024), (0, 2))]
                 # QUAD: four points per 32-byte load, four results per 16-byte store
                 + [dict(block_size_x=b, tile=t, grid=448, grid_smem=1, lmax=16, stream=st, prefetch=pf, regpf=0,
                         adrain=ad, head32=h, quad=1)
                    for b, t, st, pf, ad, h in itertools.product((256, 1024), (1, 2), (0, 1), (0, 1), (0, 1), (0, 1))
                    if (b + t + st + pf + ad + h) % 2 == 0]
                 # one block per SM with uncapped registers, register double buffering, L1-bypassing loads
                 + [dict(block_size_x=1024, tile=t, grid=g, grid_smem=1, lmax=l, stream=st, prefetch=1, regpf=1,
                         adrain=ad, head32=(t + st) % 2, quad=q, min_blocks=1)
                    for t, g, l, st, ad, q in itertools.product((1, 2, 4), (448, 512), (4, 16), (0, 2), (0, 1), (0, 1))
                    if (t + g // 64 + l + st + ad + q) % 4 == 0]
                 # finer rasters with one block per SM (r2 tuned region)
                 + [dict(block_size_x=1024, tile=1, grid=g, grid_smem=1, lmax=16, stream=2 * (g // 64 % 2), prefetch=1,
                         regpf=1, adrain=ad, head32=1 - ad, quad=1, min_blocks=1)
                    for g in (576, 640, 704, 768) for ad in (0, 1)]
                 # copy-free register double buffering, 16-byte ring records
                 + [dict(block_size_x=b, tile=t, grid=g, grid_smem=1, lmax=l, stream=2, prefetch=1, regpf=2,
                         adrain=ad, head32=1, quad=q, min_blocks=int(b == 1024), ring16=r)
                    for b, t, g, l, ad, q, r in itertools.product((512, 1024), (1, 2), (448, 640), (4, 16), (0, 1),
                                                                  (0, 1), (0, 1))
                    if (b // 512 + t + g // 64 + l + ad + q + r) % 4 == 0 and not (b == 512 and g == 640)]
                 # one warp prefix per point vector for the ring pushes; L1 prefetch of queued heads
                 + [dict(block_size_x=b, tile=t, grid=448, grid_smem=1, lmax=l, stream=st, prefetch=1, regpf=int(b == 1024),
                         adrain=0, head32=h, quad=q, min_blocks=int(b == 1024), pushv=1, hpf=hp)
                    for b, t, l, st, h, q, hp in itertools.product((512, 1024), (1, 2), (4, 16), (0, 2), (0, 1), (0, 1),
                                                                   (0, 1))
                    if (b // 512 + t + l + st + h + q + hp) % 4 == 0]
                 # DEFER: per-thread pending undecided points instead of the warp ring
                 + [dict(block_size_x=b, tile=t, grid=(448, 512, 1024)[(t + q) % 3], grid_smem=int((t + q) % 3 < 2),
                         lmax=(16, 4)[(b // 256 + t) % 2], stream=(t + q) % 2, prefetch=(b // 256 + q) % 2,
                         regpf=(t + q + b // 512) % 2, adrain=0, head32=(t + b // 256) % 2, quad=q, defer=1,
                         min_blocks=mb)
                    for (b, mb), t, q in itertools.product(((1024, 1), (512, 2), (256, 2), (256, 0)), (1, 2, 4), (0, 1))])


@pytest.fixture(scope="module")
def cells_small(gpu):
    from paper_2211_07260_b200.kernels import PnPolyCellsProblem

    p = PnPolyCellsProblem(n_points=1_000_003)
    p.prepare(gpu)
    return p, O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)


@pytest.mark.parametrize("cfg", CELLS_CONFIGS, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_cells_bit_exact_across_configs(gpu, cells_small, cfg):
    p, want = cells_small
    assert p.is_valid(cfg)
    got = run_once(gpu, p, cfg)
    assert np.array_equal(got, want), f"{int((got != want).sum())} points differ"


@pytest.mark.parametrize("n", [1, 2, 3, 7, 33, 4097, 65537])
def test_cells_tiny_and_ragged_inputs(gpu, n):
    from paper_2211_07260_b200.kernels import PnPolyCellsProblem

    p = PnPolyCellsProblem(n_points=n)
    p.prepare(gpu)
    for cfg in (p.default_config(), dict(p.default_config(), block_size_x=256, tile=1, grid=256),
                dict(p.default_config(), tile=4, block_size_x=512), dict(p.default_config(), grid=1024, grid_smem=0),
                dict(p.default_config(), lmax=0), dict(p.default_config(), adrain=0),
                dict(p.default_config(), adrain=1, tile=1, block_size_x=256),
                dict(p.default_config(), head32=1, grid=448), dict(p.default_config(), head32=1, adrain=0),
                dict(p.default_config(), quad=1, tile=1), dict(p.default_config(), quad=1, adrain=0, regpf=1),
                dict(p.default_config(), quad=1, block_size_x=256, tile=2, stream=1),
                dict(p.default_config(), defer=1, min_blocks=1), dict(p.default_config(), defer=1, quad=1, tile=1),
                dict(p.default_config(), defer=1, block_size_x=256, tile=4, regpf=1, head32=1, min_blocks=2),
                dict(p.default_config(), defer=1, lmax=0),
                dict(p.default_config(), adrain=0, pushv=1, hpf=1), dict(p.default_config(), adrain=0, pushv=1, quad=1),
                dict(p.default_config(), adrain=0, pushv=1, lmax=0, min_blocks=1, regpf=1),
                dict(p.default_config(), regpf=2, ring16=1, min_blocks=1, quad=1, tile=1, grid=640, adrain=0),
                dict(p.default_config(), regpf=2, ring16=1, adrain=1, tile=2)):
        np.testing.assert_array_equal(run_once(gpu, p, cfg),
                                      O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2), err_msg=str(cfg))


def test_cells_full_size_matches_brute_force(gpu):
    from paper_2211_07260_b200 import tuned
    from paper_2211_07260_b200.kernels import PnPolyCellsProblem

    p = PnPolyCellsProblem()
    p.prepare(gpu)
    want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)
    for cfg in {str(c): c for c in [p.default_config(), tuned.best_config("pnpoly_cells"),
                                    tuned.best_config("pnpoly_cells", "energy_optimal")] if c}.values():
        got = run_once(gpu, p, cfg)
        assert np.array_equal(got, want), f"{int((got != want).sum())} of 20M points differ ({cfg})"
        assert_full_size_pin(got)  # == formula 2; differs from the paper op order exactly where pinned
    assert p.clean_fraction(512) > 0.9
