"""cuBLAS reference rates on the box (library calibration, not the product): FP32 SGEMM with TF32
disabled and enabled, 4096^3, C = A @ B (beta = 0), CUDA-event timed after warm-up."""
import json

import torch

n = 4096
a = torch.rand(n, n, device="cuda") * 2 - 1
b = torch.rand(n, n, device="cuda") * 2 - 1
out = {}
for label, tf32 in (("fp32", False), ("tf32", True)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    for _ in range(5):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    for reps in (10, 200):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            torch.matmul(a, b)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / reps
        out[f"{label}_reps{reps}"] = {"ms": round(ms, 4), "tflops": round(2 * n ** 3 / ms / 1e9, 1)}
print(json.dumps(out))
