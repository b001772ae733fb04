"""Event timeline of a pipelined conv2d host call: completion time of each strip's H2D / kernel / D2H."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_07260_b200 import suite, tuned  # noqa: E402
from paper_2211_07260_b200.kernels import Conv2DProblem  # noqa: E402

p = Conv2DProblem()
inp = p.host_inputs()
img = suite.pinned(inp["image"].shape)
img[...] = inp["image"]
out = suite.pinned((p.height, p.width))
cfg = tuned.best_config("conv2d")
suite.conv2d(img, inp["filter"], out=out, config=cfg, strips=16)
r = [v for k, v in suite._runners.items() if k[0] == "conv2d"][0]
gpu = r.gpu
for strips, with_kernel in ((16, True), (16, False), (4, True)):
    for rep in range(2):
        plan = r.problem.strips(r.config, {"image": img}, out, strips)
        n = len(plan)
        base = 64
        gpu.reserve_events(base + 3 * n + 1)
        START = base + 3 * n
        gpu.use_stream(1)
        gpu.record(START)
        for i, strip in enumerate(plan):
            gpu.use_stream(1)
            for dev, host in strip.h2d:
                gpu.h2d_async(dev, host)
            gpu.record(base + 3 * i)
            gpu.use_stream(0)
            gpu.wait_event(base + 3 * i)
            if with_kernel:
                gpu.launch(r.kernel, strip.launch, strip.args)
            gpu.record(base + 3 * i + 1)
            gpu.use_stream(2)
            gpu.wait_event(base + 3 * i + 1)
            for host, dev in strip.d2h:
                gpu.d2h_async(host, dev)
            gpu.record(base + 3 * i + 2)
        gpu.use_stream(0)
        gpu.synchronize()
        if rep:
            print(f"strips={strips} kernel={with_kernel}")
            for i in range(n):
                h, k, d = (gpu.elapsed(START, base + 3 * i + j) * 1e3 for j in range(3))
                print(f"  {i:2d} h2d {h:6.3f} kern {k:6.3f} d2h {d:6.3f}")
