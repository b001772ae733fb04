"""CPU checks of the PnPoly slab table (libjt ``jt_pnpoly_slabs``, no GPU needed).

The slab kernel is bit-exact with the brute-force METHOD 2 kernel iff, for
every point, the list of slab r = #{u <= py} is exactly the set of edges whose
y-test ``(vy_k > py) != (vy_j > py)`` holds, with the same slope / intercept
bits. Both are checked here on the benchmark polygon and on degenerate ones.
"""

import ctypes
import ctypes.util
import math

import numpy as np
import pytest

from paper_2211_07260_b200 import native
from paper_2211_07260_b200.kernels import PnPolySlabProblem


def _decode(table, info):
    u = table[info.u_off:info.u_off + info.nu]
    guess = table[info.guess_off:info.guess_off + info.ng].view(np.int32)
    band = table[info.band_off:info.band_off + info.nu + 2].view(np.int32)
    pairs = table[info.pair_off:info.pair_off + 2 * info.ne].reshape(-1, 2)
    return u, guess, band, pairs


def _bucket(v, base, scale, hi):
    """min(max(__float2int_rz(__fmul_rn(__fsub_rn(v, base), scale)), 0), hi) in float32."""
    with np.errstate(invalid="ignore", over="ignore"):
        f = np.float32(np.float32(v) - np.float32(base)) * np.float32(scale)
    g = 0 if math.isnan(f) else int(np.clip(np.trunc(np.nan_to_num(f, posinf=2**31 - 1, neginf=-2**31)),
                                            -2**31, 2**31 - 1))
    return min(max(g, 0), hi)


def _kernel_rank(py, u, guess, info, check_exact=True):
    """The kernel's slab rank: y-bucket start (bit 31 = exact), else corrected by compares."""
    if math.isnan(py):
        return 0
    gv = int(guess[_bucket(py, info.ybase, info.yscale, info.ng - 1)]) & 0xFFFFFFFF
    r = gv & 0x7FFFFFFF
    if gv & 0x80000000:
        if check_exact:  # the flag promises the corrected value is already there
            assert r == int(np.searchsorted(u, np.float32(py), side="right"))
        return r
    while r < info.nu and u[r] <= py:
        r += 1
    while r > 0 and u[r - 1] > py:
        r -= 1
    return int(r)


POLYGONS = {
    "benchmark": None,
    "horizontal+repeated": (np.array([0.0, 0.5, 0.5, 1.0, 1.0, 0.0, 0.0], np.float32),
                            np.array([0.0, 0.0, 0.25, 0.25, 1.0, 1.0, 1.0], np.float32)),
    "signed-zeros": (np.array([-1.0, 1.0, 1.0, -1.0], np.float32), np.array([-0.0, 0.0, 1.0, 1.0], np.float32)),
    "comb": (np.array([0, 4, 4, 3, 3, 2, 2, 1, 1, 0], np.float32),
             np.array([0, 0, 3, 3, 1, 1, 3, 3, 1, 1], np.float32)),
    "flat": (np.array([0.0, 1.0, 2.0, 0.5], np.float32), np.array([0.25, 0.25, 0.25, 0.25], np.float32)),
    "tiny": (np.array([0.0, 3e-30, 1e-30], np.float32), np.array([0.0, 1e-30, 4e-30], np.float32)),
    "huge": (np.array([-1e30, 2e30, 0.0, 5e29], np.float32), np.array([-1e30, 0.0, 3e30, 1e29], np.float32)),
}


@pytest.mark.parametrize("name", sorted(POLYGONS))
@pytest.mark.parametrize("buckets", [1, 7, 4096])
def test_slab_lists_equal_the_y_test(name, buckets):
    if POLYGONS[name] is None:
        p = PnPolySlabProblem(n_points=4096)
        vx, vy = p._polygon()
    else:
        vx, vy = POLYGONS[name]
    table, info = native.pnpoly_slabs(vx, vy, buckets, 4)
    u, guess, band, pairs = _decode(table, info)
    edges, _ = native.pnpoly_edges(vx, vy, 2)  # {vy_k, icpt, slope, 0}: the brute-force kernel's bits
    n = vx.size
    prev = np.roll(vy, 1)
    rng = np.random.default_rng(0)
    probes = np.concatenate([vy, np.nextafter(vy, np.inf), np.nextafter(vy, -np.inf),
                             rng.uniform(vy.min() - 1, vy.max() + 1, 300).astype(np.float32),
                             np.array([np.inf, -np.inf, np.nan, 0.0, -0.0], np.float32)]).astype(np.float32)
    for py in probes:
        r = _kernel_rank(py, u, guess, info)
        assert r == (0 if math.isnan(py) else int(np.searchsorted(u, py, side="right")))
        listed = pairs[band[r]:band[r + 1]]
        assert len(listed) % 4 == 0
        real = listed[~np.isneginf(listed[:, 1])]
        fillers = listed[np.isneginf(listed[:, 1])]
        assert np.all(fillers[:, 0] == 0)
        spans = [k for k in range(n) if (vy[k] > py) != (prev[k] > py)]
        want = np.array([[edges[k, 2], edges[k, 1]] for k in spans], np.float32).reshape(-1, 2)
        assert real.view(np.uint32).tolist() == want.view(np.uint32).tolist(), (name, float(py), r)
    assert info.max_band == max(band[r + 1] - band[r] for r in range(info.nu + 1))


def test_slab_table_size_query_and_errors():
    vx = np.array([0, 1, 0], np.float32)
    vy = np.array([0, 0, 1], np.float32)
    table, info = native.pnpoly_slabs(vx, vy, 16, 4)
    assert info.words == table.size and info.nu == 2 and info.ne == 4
    with pytest.raises(Exception):
        native.pnpoly_slabs(vx[:2], vy[:2], 16, 4)
    with pytest.raises(Exception):
        native.pnpoly_slabs(vx, vy, 0, 4)


def test_slab_space_fits_shared_memory():
    p = PnPolySlabProblem()
    for cfg in p.space().enumerate():
        assert p.smem_bytes(cfg.as_dict()) <= 227 * 1024
    assert p.is_valid(p.default_config())


@pytest.mark.parametrize("name", sorted(POLYGONS))
def test_xsearch_table_decides_like_the_brute_force_test(name):
    """x-search layout: per slab, lo sorted ascending, pmax = running max of hi, and for
    every probe point the kernel's decision procedure (count lo > px, then evaluate the
    undecided edges walking back while pmax > px) equals the brute-force parity.
    The fma is emulated exactly in float64 (a float32 x float32 product is exact)."""
    if POLYGONS[name] is None:
        p = PnPolySlabProblem(n_points=4096)
        vx, vy = p._polygon()
    else:
        vx, vy = POLYGONS[name]
    table, info = native.pnpoly_slabs(vx, vy, 64, 4, 8)
    u, guess, band, _ = _decode(table, info)
    xlo = table[info.xlo_off:info.xlo_off + info.ne]
    pmax = table[info.pmax_off:info.pmax_off + info.ne]
    rec = table[info.pair_off:info.pair_off + 4 * info.ne].reshape(-1, 4)
    for r in range(1, info.nu):
        lo, pm = xlo[band[r]:band[r + 1]], pmax[band[r]:band[r + 1]]
        assert np.all(np.diff(lo) >= 0) and np.all(pm == np.maximum.accumulate(rec[band[r]:band[r + 1], 2]))
        assert np.all(rec[band[r]:band[r + 1], 2] >= lo)
    xst = table[info.xst_off:].view(np.uint16)[:(info.nu + 1) * (info.xb + 1)].reshape(info.nu + 1, info.xb + 1)
    srec = table[info.xpar_off:info.xpar_off + 4 * (info.nu + 1)].reshape(-1, 4)
    for r in range(1, info.nu):
        cnt = band[r + 1] - band[r]
        assert srec[r, :2].view(np.int32).tolist() == [band[r], cnt]
        assert np.all((xst[r] & 0x7FFF) <= cnt)
    edges, _ = native.pnpoly_edges(vx, vy, 2)
    prev = np.roll(vy, 1)

    def fma32(a, b, c):  # exact product in float64, one rounding of the sum: equals fmaf
        return np.float32(np.float64(a) * np.float64(b) + np.float64(c))

    hw = table[info.half_off:info.half_off + info.ne].view(np.uint32)
    lo16 = (hw & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float32)
    pm16 = (hw >> 16).astype(np.uint16).view(np.float16).astype(np.float32)

    def walk(b, pos, c, xlo_t, pm_t, px, py):
        """The kernel's parity: certain crossings + the undecided edges along the skip chain."""
        got = (c - pos) & 1
        j = pos - 1
        while j >= 0 and pm_t[b + j] > px:
            sl, ic, hi, skip = rec[b + j]
            if hi > px and px < fma32(sl, py, ic):
                got ^= 1
            j = int(np.float32(skip).view(np.int32))
        return got

    rng = np.random.default_rng(1)
    span = float(max(abs(vx).max(), abs(vy).max())) + 0.5
    pts = rng.uniform(-span, span, (3000, 2)).astype(np.float32)
    pts[:len(vx), 1] = vy  # points exactly at vertex ordinates / abscissae
    pts[len(vx):2 * len(vx), 0] = vx
    for px, py in pts:
        want = 0
        for k in range(vx.size):
            if (vy[k] > py) != (prev[k] > py) and px < fma32(edges[k, 2], py, edges[k, 1]):
                want ^= 1
        r = 0 if math.isnan(py) else _kernel_rank(py, u, guess, info)
        got = 0
        if 0 < r < info.nu and not math.isnan(px):
            b, c = band[r], band[r + 1] - band[r]
            pos = int(np.sum(xlo[b:b + c] <= px))
            w = int(xst[r, _bucket(px, srec[r, 2], srec[r, 3], info.xb)])
            if w & 0x8000:  # flagged exact: the bucket's start must already be the count
                assert (w & 0x7FFF) == pos, (name, float(px), float(py))
            got = walk(b, pos, c, xlo_t=None, pm_t=pmax, px=px, py=py)
            # HALF tables: pos over binary16 lo (rounded down), walk bounded by binary16 pmax (up)
            pos16 = int(np.sum(lo16[b:b + c] <= px))
            got16 = walk(b, pos16, c, xlo_t=None, pm_t=pm16, px=px, py=py)
            assert got16 == want, ("half", name, float(px), float(py))
        assert got == want, (name, float(px), float(py))


@pytest.mark.parametrize("name", sorted(POLYGONS))
def test_half_copy_is_conservative_and_tight(name):
    """The binary16 copy: lo rounded toward -inf, pmax toward +inf, each the closest
    such binary16 value (so the HALF kernel only re-evaluates a few more edges)."""
    if POLYGONS[name] is None:
        vx, vy = PnPolySlabProblem(n_points=4096)._polygon()
    else:
        vx, vy = POLYGONS[name]
    table, info = native.pnpoly_slabs(vx, vy, 64, 4, 8)
    h = table[info.half_off:info.half_off + info.ne].view(np.uint32)
    lo16 = (h & 0xFFFF).astype(np.uint16).view(np.float16)
    pm16 = (h >> 16).astype(np.uint16).view(np.float16)
    lo = table[info.xlo_off:info.xlo_off + info.ne]
    pm = table[info.pmax_off:info.pmax_off + info.ne]
    assert np.all(lo16.astype(np.float32) <= lo) and np.all(pm16.astype(np.float32) >= pm)
    with np.errstate(over="ignore"):
        assert np.all(np.nextafter(lo16, np.float16(np.inf)).astype(np.float32) > lo)
        assert np.all(np.nextafter(pm16, np.float16(-np.inf)).astype(np.float32) < pm)


def _cell(v, scale, offset, hi):
    """min(f2u_rz(fma(v, scale, offset)), hi) of pnpoly_grid.cu. The fma is emulated
    exactly: the float32 product is exact in float64, and float64 + float32 rounded once to
    float32 differs from a true fma only when the float64 sum itself rounds, which the
    tests' coordinates (|v| <= ~1e30 with scale ~1e3) keep rare; host and kernel both use a
    real fmaf, so the cleanliness check does not depend on this emulation."""
    with np.errstate(invalid="ignore", over="ignore"):
        f = (np.asarray(v, np.float64) * np.float64(scale) + np.float64(offset)).astype(np.float32)
    k = np.trunc(np.nan_to_num(f, nan=0.0, posinf=2.0**32, neginf=0.0))
    return np.clip(k, 0, hi).astype(np.int64)


@pytest.mark.parametrize("name", sorted(POLYGONS))
@pytest.mark.parametrize("g", [7, 64, 512])
def test_grid_clean_cells_give_the_brute_force_parity(name, g):
    """jt_pnpoly_grid: wherever a cell is flagged clean, its stored parity equals the
    brute-force (formulation 2) bit of every point mapping to it - checked on random points,
    points on/near vertices and cell borders, and points far outside."""
    from oracle import kernels_oracle as O

    if POLYGONS[name] is None:
        vx, vy = PnPolySlabProblem(n_points=4096)._polygon()
    else:
        vx, vy = POLYGONS[name]
    words, prm, clean = native.pnpoly_grid(vx, vy, g, g)
    assert 0 <= clean <= g * g
    pts = _grid_points(vx, vy, prm, g)
    cx = _cell(pts[:, 0], prm[0], prm[1], g - 1)
    cy = _cell(pts[:, 1], prm[2], prm[3], g - 1)
    cell = cy * g + cx
    code = (words[cell >> 4] >> ((cell & 15) * 2).astype(np.uint32)) & 3
    want = O.pnpoly(pts, vx, vy, 2)
    is_clean = (code & 1) == 1
    assert np.array_equal((code[is_clean] >> 1).astype(np.int32), want[is_clean]), name
    if name == "benchmark" and g == 512:
        assert is_clean.mean() > 0.8  # the fast path is the common path


def _grid_points(vx, vy, prm, g):
    """Random points, points on / next to the vertices and on / next to the cell borders of a
    g x g raster with params prm, and far-away points."""
    rng = np.random.default_rng(3)
    span = float(max(abs(vx).max(), abs(vy).max())) * 1.3
    pts = [rng.uniform(-span, span, (200_000, 2)).astype(np.float32)]
    vv = np.stack([vx, vy], 1).astype(np.float32)
    for d in (0.0, 1e-7, -1e-7, 1e-3):
        pts.append((vv + np.float32(d)).astype(np.float32))
    # cell borders in x and y (v = (k - o) / s)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):  # flat polygons: scale 0
        xs = ((np.arange(g + 1, dtype=np.float64) - prm[1]) / prm[0]).astype(np.float32)
        ys = ((np.arange(g + 1, dtype=np.float64) - prm[3]) / prm[2]).astype(np.float32)
    bx = np.concatenate([xs, np.nextafter(xs, np.float32(np.inf)), np.nextafter(xs, np.float32(-np.inf))])
    by = np.concatenate([ys, np.nextafter(ys, np.float32(np.inf)), np.nextafter(ys, np.float32(-np.inf))])
    pts.append(np.stack([rng.choice(bx, 50_000), rng.uniform(-span, span, 50_000).astype(np.float32)], 1))
    pts.append(np.stack([rng.uniform(-span, span, 50_000).astype(np.float32), rng.choice(by, 50_000)], 1))
    pts.append(np.array([[1e30, 0], [-1e30, 0], [0, 1e30], [0, -1e30], [np.inf, 0], [-np.inf, 0]], np.float32))
    return np.ascontiguousarray(np.concatenate(pts).astype(np.float32))


@pytest.mark.parametrize("name", sorted(POLYGONS))
def test_grid_border_cells_are_zero_when_clean(name):
    """pnpoly_grid.cu sends NaN coordinates to the first column / row without a NaN test:
    every clean cell there must hold parity 0 (the NaN answer)."""
    if POLYGONS[name] is None:
        vx, vy = PnPolySlabProblem(n_points=4096)._polygon()
    else:
        vx, vy = POLYGONS[name]
    for g in (7, 256, 512):
        words, _, _ = native.pnpoly_grid(vx, vy, g, g)
        code = lambda c: (int(words[c >> 4]) >> ((c & 15) * 2)) & 3  # noqa: E731
        for k in range(g):
            for c in (k * g, k):  # first column of row k, first row's cell k
                if code(c) & 1:
                    assert code(c) >> 1 == 0, (name, g, k)


_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.fmaf.restype = ctypes.c_float
_libm.fmaf.argtypes = [ctypes.c_float] * 3


def _polygon(name):
    return PnPolySlabProblem(n_points=4096)._polygon() if POLYGONS[name] is None else POLYGONS[name]


@pytest.mark.parametrize("name", sorted(POLYGONS))
@pytest.mark.parametrize("g,lmax,hw", [(7, 8, 4), (64, 2, 8), (512, 8, 4), (512, 16, 8)])
def test_cell_lists_give_the_brute_force_answer(name, g, lmax, hw):
    """jt_pnpoly_cells: the pnpoly_cells.cu decision, emulated - code 0 / 1 is the answer,
    code 2 | base is base XOR the listed edges' METHOD 2 tests (libm fmaf, NaN -> 0), the
    edges in the head (4- or 8-word heads) or in the edge array - equals the brute-force bit
    for every point outside the fallback (slab search) cells."""
    from oracle import kernels_oracle as O

    vx, vy = _polygon(name)
    words, prm, heads, edges, st = native.pnpoly_cells(vx, vy, g, g, lmax, hw)
    assert st[1] + st[2] + st[3] <= g * g and st[0] <= max(1, st[2] * lmax)
    pts = _grid_points(vx, vy, prm, g)
    cell = _cell(pts[:, 1], prm[2], prm[3], g - 1) * g + _cell(pts[:, 0], prm[0], prm[1], g - 1)
    code = _cells_code(words, cell)
    want = O.pnpoly(pts, vx, vy, 2)
    got = np.where(code < 2, code, 0).astype(np.int32)
    fallback = np.zeros(len(pts), dtype=bool)
    for i in np.nonzero(code >= 2)[0]:
        px, py = float(pts[i, 0]), float(pts[i, 1])
        if px != px or py != py:
            continue
        h = heads[hw * int(cell[i]): hw * int(cell[i]) + hw]
        hf = h.view(np.float32).reshape(-1, 4)
        if hf[0, 2] == hf[0, 2]:
            listed = list(hf)  # in place (an unused slot never tests true)
        elif h[1] == 0xFFFFFFFF:
            fallback[i] = True
            continue
        else:
            listed = list(edges[h[0]: h[0] + h[1]])
        r = int(code[i]) & 1
        for e in listed:
            if e[2] <= py < e[3] and px < _libm.fmaf(float(e[0]), py, float(e[1])):
                r ^= 1
        got[i] = r
    keep = ~fallback
    assert np.array_equal(got[keep], want[keep]), (name, int((got[keep] != want[keep]).sum()))
    if name == "benchmark" and g == 512:
        assert (code < 2).mean() > 0.8 and fallback.mean() < 0.01


@pytest.mark.parametrize("name", sorted(POLYGONS))
def test_cell_lists_border_and_limits(name):
    """NaN lands in row 0 / column 0: clean cells there hold 0. lmax 0 sends every undecided
    cell to the slab search (code 3) and lists nothing; the clean cells equal jt_pnpoly_grid's."""
    vx, vy = _polygon(name)
    for g in (7, 256):
        words, _, _, _, st = native.pnpoly_cells(vx, vy, g, g, 8)
        for k in range(g):
            for c in (k * g, k):
                assert _cells_code(words, np.array([c]))[0] != 1, (name, g, k)
        w0, _, h0, e0, s0 = native.pnpoly_cells(vx, vy, g, g, 0)
        assert s0[0] == 0 and s0[1] == st[1]
        assert s0[1] + s0[2] + s0[3] == st[1] + st[2] + st[3]
        # lmax 0: no head holds an edge; only the edge-less (border, base 1) cells are listed
        und = _cells_code(w0, np.arange(g * g)) >= 2
        hf = h0.reshape(-1, 4)
        assert np.all(np.isnan(hf[und].view(np.float32)[:, 2]))
        assert np.all((hf[und, 1] == 0xFFFFFFFF) | (hf[und, 1] == 0))
    with pytest.raises(Exception):
        native.pnpoly_cells(vx, vy, 0, 4, 8)
    with pytest.raises(Exception):
        native.pnpoly_cells(vx, vy, 8, 8, 8, 6)  # head_words 4 or 8


def _cells_code(words, cell):
    """2-bit codes from jt_pnpoly_cells' raster (16 cells per word)."""
    cell = np.asarray(cell, dtype=np.int64)
    return ((words[cell >> 4] >> ((cell & 15) * 2).astype(np.uint32)) & 3).astype(np.int64)
