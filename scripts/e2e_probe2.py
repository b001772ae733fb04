"""Where does a pipelined conv2d host call spend its time (enqueue vs wait)?"""
import sys
import time
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
for strips in (1, 4, 16):
    for it in range(4):
        t0 = time.perf_counter()
        plan = r.problem.strips(r.config, {"image": img}, out, strips)
        t1 = time.perf_counter()
        base = 64
        gpu.reserve_streams(3)
        gpu.reserve_events(base + 2 * len(plan))
        r.problem.bind(r.kernel, r.config)
        t2 = time.perf_counter()
        for i, strip in enumerate(plan):
            gpu.use_stream(1)
            for dev, host in strip.h2d:
                gpu.h2d_async(dev, host)
            gpu.record(base + 2 * i)
            gpu.use_stream(0)
            gpu.wait_event(base + 2 * i)
            gpu.launch(r.kernel, strip.launch, strip.args)
            gpu.record(base + 2 * i + 1)
            gpu.use_stream(2)
            gpu.wait_event(base + 2 * i + 1)
            for host, dev in strip.d2h:
                gpu.d2h_async(host, dev)
        t3 = time.perf_counter()
        gpu.use_stream(0)
        gpu.synchronize()
        t4 = time.perf_counter()
        print(f"strips={strips:2d} plan {1e3*(t1-t0):.3f} bind {1e3*(t2-t1):.3f} enqueue {1e3*(t3-t2):.3f} "
              f"wait {1e3*(t4-t3):.3f} total {1e3*(t4-t0):.3f} ms", flush=True)
# enqueue-only micro costs
import timeit  # noqa: E402
s = plan[0]
print("use_stream us", 1e6 * timeit.timeit(lambda: gpu.use_stream(0), number=2000) / 2000)
print("record us", 1e6 * timeit.timeit(lambda: gpu.record(64), number=2000) / 2000)
print("launch us", 1e6 * timeit.timeit(lambda: gpu.launch(r.kernel, s.launch, s.args), number=500) / 500)
gpu.synchronize()
print("h2d_async 4KB us", 1e6 * timeit.timeit(lambda: gpu.h2d_async(s.h2d[0][0], img[0:1]), number=500) / 500)
gpu.synchronize()
