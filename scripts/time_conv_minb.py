"""conv2d: occupancy sweep of the tuned config family via MIN_BLOCKS (register cap), device-timed."""
import itertools
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import native, tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import Conv2DProblem  # noqa: E402

gpu = GPU(0)
p = Conv2DProblem()
p.prepare(gpu)
ref = O.conv2d(p.inputs["image"], p.inputs["filter"])
best = tuned.best_config("conv2d")
for by, ty, f2, mb in itertools.product((4, 8), (2, 4), (0, 1), (0, 2, 3, 4)):
    cfg = dict(best, block_size_y=by, tile_size_y=ty, fma2=f2)
    if not p.is_valid(cfg) or mb * 64 * by > 2048:
        continue
    defs = p.defines(cfg)
    if mb:
        defs["MIN_BLOCKS"] = mb
    try:
        k = gpu.load(native.compile_cubin(native.kernel_source(p.source), p.name, native._nvrtc_options(defs)),
                     p.symbol)
    except Exception as e:  # noqa: BLE001
        print(cfg, mb, "failed", str(e)[:60])
        continue
    p.bind(k, cfg)
    p.reset_output()
    gpu.launch(k, p.launch(cfg), p.args(cfg))
    gpu.synchronize()
    err = O.conv2d_error(p.fetch_output(), ref, p.inputs["image"], p.inputs["filter"])
    t = gpu.time(k, p.launch(cfg), p.args(cfg), reps=50) / 50
    print(f"by={by} ty={ty} fma2={f2} minb={mb} regs={k.regs} local={k.local_bytes} err={err:.1e} "
          f"{t * 1e6:.1f} us {p.total_flops / t / 74.45e12:.3f}", flush=True)
