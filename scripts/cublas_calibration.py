"""cuBLAS reference rates on the box (library calibration, not the product): FP32 SGEMM with TF32
disabled and enabled, 4096^3, C = A @ B (beta = 0), CUDA-event timed after warm-up.

Two regimes per precision: a short burst (10 / 200 launches, before the board's 1 kW power cap
settles) and a sustained 1 s loop whose last 0.5 s is timed (the regime bench.py's per_kernel
loops measure ours in), with the SM clock sampled through NVML during the sustained loop."""
import json
import threading
import time

import torch

try:
    import pynvml
except ImportError:  # nvidia_ml_py provides the pynvml module
    pynvml = None

n = 4096
a = torch.rand(n, n, device="cuda") * 2 - 1
b = torch.rand(n, n, device="cuda") * 2 - 1
flop = 2 * n ** 3


def timed(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def sustained(seconds=1.0):
    clocks, stop = [], threading.Event()
    if pynvml is not None:
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

        def sample():
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.02)
        th = threading.Thread(target=sample, daemon=True)
        th.start()
    ms = timed(20)
    warm = max(1, int(0.5 * seconds / (ms * 1e-3)))
    timed(warm)  # past the power ramp
    ms = timed(warm)
    stop.set()
    out = {"ms": round(ms, 4), "tflops": round(flop / ms / 1e9, 1), "loop_s": round(2 * warm * ms * 1e-3, 2)}
    if clocks:
        clocks.sort()
        out["sm_mhz_median"] = clocks[len(clocks) // 2]
    return out


out = {}
for label, tf32 in (("fp32", False), ("tf32", True)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    for _ in range(5):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    for reps in (10, 200):
        ms = timed(reps)
        out[f"{label}_reps{reps}"] = {"ms": round(ms, 4), "tflops": round(flop / ms / 1e9, 1)}
    out[f"{label}_sustained_1s"] = sustained(1.0)
    time.sleep(1.0)
print(json.dumps(out))
