"""SGEMM FP32: MIN_BLOCKS (register cap -> resident CTAs) sweep around the tuned config, device-timed."""
import itertools
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import native, tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import SgemmProblem  # noqa: E402

gpu = GPU(0)
p = SgemmProblem()
p.prepare(gpu)
ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
best = tuned.best_config("sgemm")
for asy, mb in itertools.product((2, 3, 4), (0, 2, 3)):
    cfg = dict(best, ASYNC=asy)
    if not p.is_valid(cfg):
        continue
    defs = p.defines(cfg)
    if mb:
        defs["MIN_BLOCKS"] = mb
    k = gpu.load(native.compile_cubin(native.kernel_source(p.source), p.name, native._nvrtc_options(defs)), p.symbol)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    err = O.sgemm_error(p.fetch_output(), ref)
    t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=10) / 10
    print(f"ASYNC={asy} minb={mb} regs={k.regs} local={k.local_bytes} err={err:.1e} {t * 1e3:.3f} ms "
          f"{p.total_flops / t / 1e12:.1f} TF/s = {p.total_flops / t / 74.45e12:.3f}", flush=True)
