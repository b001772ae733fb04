"""Regression fixtures for the kernel oracles (tests/golden/kernels_small.npz).

The reference package has no kernel code, so these vectors come from the
oracles themselves after they were pinned against independent restatements
(tests/test_oracle.py): PnPoly C oracle == numpy restatement, conv oracle ==
direct sums, SGEMM oracle == float64 BLAS. Freezing them catches any later
drift in the oracles or in the seeded input generators.
"""

from pathlib import Path
import sys

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.kernels import Conv2DProblem, PnPolyProblem, SgemmProblem  # noqa: E402


def main():
    pn = PnPolyProblem(n_points=20_000, seed=4)
    pi = pn.host_inputs()
    assert np.array_equal(O.pnpoly(pi["points"], pi["vx"], pi["vy"], 0), O.pnpoly_numpy(pi["points"], pi["vx"], pi["vy"]))
    out = {"pn_n": np.int64(pn.n_points), "pn_points": pi["points"]}
    for m in range(4):
        out[f"pn_bitmap{m}"] = O.pnpoly(pi["points"], pi["vx"], pi["vy"], m)
    cp = Conv2DProblem(width=64, height=48)
    ci = cp.host_inputs()
    out["conv_out"] = O.conv2d(ci["image"], ci["filter"])
    sp = SgemmProblem(m=64, n=32, k=48)
    si = sp.host_inputs()
    out["sgemm_out"] = O.sgemm(si["a"], si["b"], si["c0"], sp.alpha, sp.beta)
    path = Path(__file__).resolve().parent / "kernels_small.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
