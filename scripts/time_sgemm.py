"""Full-size FP32 SGEMM timing of selected CLBlast configs x ASYNC staging, checked against the oracle."""
import itertools
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import SgemmProblem  # noqa: E402

gpu = GPU(0)
p = SgemmProblem()
p.prepare(gpu)
ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
bases = [
    {'KWG': 32, 'KWI': 8, 'MDIMA': 16, 'MDIMC': 16, 'MWG': 128, 'NDIMB': 16, 'NDIMC': 8, 'NWG': 64, 'SA': 1, 'SB': 1,
     'STRM': 1, 'STRN': 0, 'VWM': 4, 'VWN': 4},
    {'KWG': 16, 'KWI': 2, 'MDIMA': 32, 'MDIMC': 16, 'MWG': 128, 'NDIMB': 32, 'NDIMC': 16, 'NWG': 128, 'SA': 1,
     'SB': 1, 'STRM': 1, 'STRN': 1, 'VWM': 4, 'VWN': 4},
    {'KWG': 32, 'KWI': 8, 'MDIMA': 32, 'MDIMC': 16, 'MWG': 128, 'NDIMB': 32, 'NDIMC': 16, 'NWG': 128, 'SA': 1,
     'SB': 1, 'STRM': 1, 'STRN': 1, 'VWM': 4, 'VWN': 4},
    {'KWG': 16, 'KWI': 8, 'MDIMA': 16, 'MDIMC': 16, 'MWG': 128, 'NDIMB': 16, 'NDIMC': 8, 'NWG': 64, 'SA': 1, 'SB': 1,
     'STRM': 1, 'STRN': 0, 'VWM': 4, 'VWN': 4},
]
for base, asy in itertools.product(bases, (0, 2, 3, 4)):
    cfg = dict(base, ASYNC=asy)
    if not p.is_valid(cfg):
        print(cfg, "invalid")
        continue
    k = p.kernel(cfg)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    err = O.sgemm_error(p.fetch_output(), ref)
    t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=10) / 10
    print(f"{cfg} err={err:.2e} ok={err <= O.SGEMM_TOL} regs={k.regs} {t * 1e3:.3f} ms "
          f"{p.total_flops / t / 1e12:.1f} TF/s = {p.total_flops / t / 74.45e12:.3f}", flush=True)
