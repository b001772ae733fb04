"""One small launch per kernel family / variant, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python scripts/sanitize.py
    compute-sanitizer --tool racecheck python scripts/sanitize.py [--only tf32]
    compute-sanitizer --tool synccheck python scripts/sanitize.py

Each launch runs through the product path (libjt, NVRTC cubins) at the
smallest size its config accepts and is checked against the CPU oracle, so a
sanitizer run also proves the launch did real work. Logs: profiles/r2_sanitize_*.log.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import suite  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402


def once(gpu, p, cfg):
    k = p.kernel(cfg)
    p.bind(k, cfg)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    return p.fetch_output()


def pnpoly_family(gpu):
    p = make_problem("pnpoly", n_points=4099)  # ragged: a partial last tile
    p.prepare(gpu)
    base = dict(block_size_x=128, tile=2, vec=2, method=2, between=0, poly_smem=1, asm=0, persist=0)
    for cfg in [base, {**base, "poly_smem": 0}, {**base, "method": 0}, {**base, "asm": 3},
                {**base, "asm": 7}, {**base, "asm": 8, "poly_smem": 0}, {**base, "asm": 7, "persist": 1}]:
        got = once(gpu, p, cfg)
        want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], p.formula(cfg))
        assert np.array_equal(got, want), cfg
        yield "pnpoly", cfg
    want = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 2)
    for name, cfgs in (
        ("pnpoly_slab", [dict(block_size_x=128, tile=2, sort=0, pairs_smem=0, xbuckets=16, exact_flags=0, half=1,
                              buckets=1024),
                         dict(block_size_x=128, tile=2, sort=1, pairs_smem=1, xbuckets=0, exact_flags=1, half=0,
                              buckets=1024)]),
        ("pnpoly_grid", [None]),
        ("pnpoly_cells", [None, {"adrain": 0}, {"head32": 1}, {"prefetch": 1}, {"lmax": 0}]),
    ):
        q = make_problem(name, n_points=4099)
        q.prepare(gpu)
        for extra in cfgs:
            cfg = q.default_config() if extra is None else {**q.default_config(), **extra}
            if not q.is_valid(cfg):
                print("skip invalid", name, cfg, flush=True)
                continue
            got = once(gpu, q, cfg)
            assert np.array_equal(got, want), (name, cfg)
            yield name, cfg


def conv_family(gpu):
    p = make_problem("conv2d", width=128, height=64)
    p.prepare(gpu)
    ref = O.conv2d(p.inputs["image"], p.inputs["filter"])
    for cfg in [p.default_config(), {**p.default_config(), "use_shmem": 0},
                {**p.default_config(), "use_padding": 1},
                dict(block_size_x=64, block_size_y=8, tile_size_x=2, tile_size_y=2, use_shmem=0, use_padding=0,
                     fma2=1, min_blocks=2)]:
        if not p.is_valid(cfg):
            print("skip invalid conv2d", cfg, flush=True)
            continue
        err = O.conv2d_error(once(gpu, p, cfg), ref, p.inputs["image"], p.inputs["filter"])
        assert err <= O.CONV_TOL, (cfg, err)
        yield "conv2d", cfg


def sgemm_family(gpu):
    p = make_problem("sgemm", m=256, n=256, k=64)
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    base = p.default_config()
    for cfg in [base, {**base, "ASYNC": 3}, {**base, "ASYNC": 4, "FMA2": 1, "KWI": 8}, {**base, "SA": 0, "SB": 0}]:
        if not p.is_valid(cfg):
            print("skip invalid sgemm", cfg, flush=True)
            continue
        assert O.sgemm_error(once(gpu, p, cfg), ref) <= O.SGEMM_TOL, cfg
        yield "sgemm", cfg


def tf32_family(gpu):
    p = make_problem("sgemm_tf32", m=512, n=512, k=128)
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    for cfg in [dict(BN=128, STAGES=3, PERSIST=0, SPLIT_TAIL=0, PAIR=0),
                dict(BN=256, STAGES=4, PERSIST=1, SPLIT_TAIL=1, PAIR=0),
                dict(BN=256, STAGES=4, PERSIST=0, SPLIT_TAIL=0, PAIR=1),
                dict(BN=256, STAGES=7, PERSIST=1, SPLIT_TAIL=1, PAIR=1)]:
        err = O.sgemm_error(once(gpu, p, cfg), ref)
        assert 1e-6 < err <= O.SGEMM_TF32_TOL, (cfg, err)
        yield "sgemm_tf32", cfg


def misc_family(gpu):
    b = make_problem("burner", iters=16)
    b.prepare(gpu)
    cfg = b.default_config()
    gpu.launch(b.kernel(cfg), b.launch(cfg), b.args(cfg))
    gpu.synchronize()
    yield "burner", cfg
    rng = np.random.default_rng(0)
    a, bb, c = (rng.uniform(-1, 1, s).astype(np.float32) for s in ((100, 70), (70, 90), (100, 90)))
    got = suite.sgemm(a, bb, c, 1.0, 0.5, config={**make_problem("sgemm").default_config(), "MWG": 64, "NWG": 64,
                                                   "MDIMA": 16, "NDIMB": 16})
    assert O.sgemm_error(got, O.sgemm(a, bb, c, 1.0, 0.5)) <= O.SGEMM_TOL
    yield "transpose_pad+sgemm (suite, padded 100x90x70)", {}


FAMILIES = {"pnpoly": pnpoly_family, "conv": conv_family, "sgemm": sgemm_family, "tf32": tf32_family,
            "misc": misc_family}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(FAMILIES))
    args = ap.parse_args()
    with GPU(0) as gpu:
        for fam in args.only.split(","):
            for name, cfg in FAMILIES[fam](gpu):
                print(f"ok {name} {cfg}", flush=True)
    print("sanitize launches done", flush=True)


if __name__ == "__main__":
    main()
