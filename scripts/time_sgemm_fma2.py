"""SGEMM FP32: packed FFMA2 outer product (FMA2=1) vs scalar FFMA on the tuned and nearby configs.
Checks the FMA2 output is bit-identical to FMA2=0 and within the oracle tolerance."""
import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import SgemmProblem  # noqa: E402

gpu = GPU(0)
p = SgemmProblem()
p.prepare(gpu)
ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
best = tuned.best_config("sgemm")
bases = [best,
         dict(best, MDIMC=16, NDIMC=16, MDIMA=32, NDIMB=32, VWN=4, STRN=1),
         dict(best, KWG=32, KWI=8),
         dict(best, MWG=128, NWG=256, NDIMC=32, NDIMB=32),
         dict(best, VWN=4, NDIMC=8, NDIMB=16)]
for base, asy, f2 in itertools.product(bases, (2, 3), (0, 1)):
    cfg = dict(base, ASYNC=asy, FMA2=f2)
    if not p.is_valid(cfg):
        print(cfg, "invalid", flush=True)
        continue
    k = p.kernel(cfg)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    out = p.fetch_output()
    err = O.sgemm_error(out, ref)
    if f2 == 0:
        scalar_out = out
    same = bool(np.array_equal(out.view(np.uint32), scalar_out.view(np.uint32)))
    t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=10) / 10
    print(f"{cfg} err={err:.2e} ok={err <= O.SGEMM_TOL} bit_identical_to_fma={same} regs={k.regs} "
          f"{t * 1e3:.3f} ms {p.total_flops / t / 1e12:.1f} TF/s = {p.total_flops / t / 74.45e12:.3f}", flush=True)
