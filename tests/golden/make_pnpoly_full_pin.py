"""Full-size PnPoly pin (tests/golden/pnpoly_full_pin.json).

The BASELINE PnPoly workload (20,000,000 points x 600 vertices, seed 4)
evaluated by the C oracle (oracle/pnpoly_oracle.c, test infrastructure) in
the paper's Kernel-Tuner op order (formula 0: (dx * (py - vy_k)) / dy + vx_k,
one IEEE float32 rounding per op) and in the precomputed slope / intercept
form every tuned kernel computes (formula 2: fmaf(slope, py, icpt); formula
3 = formula 2 with sign-bit compares). Records each bitmap's SHA-256 and
inside count, and every point where the tuned formulation and the paper's
op order disagree, with its coordinates, so the GPU tests can assert the
exact differing set at full size.

    python tests/golden/make_pnpoly_full_pin.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.kernels import PnPolyProblem  # noqa: E402

OUT = Path(__file__).resolve().parent / "pnpoly_full_pin.json"


def sha(bitmap: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(bitmap, dtype=np.int32).tobytes()).hexdigest()


def compute() -> dict:
    p = PnPolyProblem()
    inp = p.host_inputs()
    maps = {m: O.pnpoly(inp["points"], inp["vx"], inp["vy"], m) for m in (0, 2, 3)}
    diff = np.flatnonzero(maps[0] != maps[2])
    return {
        "workload": "pnpoly 20,000,000 points x 600 vertices, seed 4 (BASELINE configs[0] / SURVEY §8(d))",
        "n_points": p.n_points,
        "sha256": {f"formula{m}": sha(b) for m, b in maps.items()},
        "inside": {f"formula{m}": int(b.sum()) for m, b in maps.items()},
        "formula2_equals_formula3": bool(np.array_equal(maps[2], maps[3])),
        "formula0_vs_formula2_differ": [
            {"index": int(i), "px": float(inp["points"][i, 0]), "py": float(inp["points"][i, 1]),
             "formula0": int(maps[0][i]), "formula2": int(maps[2][i])} for i in diff],
    }


if __name__ == "__main__":
    doc = compute()
    OUT.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))
