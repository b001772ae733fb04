"""Quick TF32 tcgen05 SGEMM check (small then larger) against the fp64 oracle."""
import sys
from pathlib import Path


ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import SgemmTF32Problem  # noqa: E402

sizes = [tuple(int(x) for x in s.split("x")) for s in (sys.argv[1:] or ["256x256x256"])]
gpu = GPU(0)
for m, n, k in sizes:
    p = SgemmTF32Problem(m=m, n=n, k=k)
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    for cfg in [c.as_dict() for c in p.space().enumerate()]:
        kern = p.kernel(cfg)
        p.reset_output()
        gpu.launch(kern, p.launch(cfg), p.args(cfg))
        gpu.synchronize()
        err = O.sgemm_error(p.fetch_output(), ref)
        t = gpu.time(kern, p.launch(cfg), p.args(cfg), reps=5) / 5 if m >= 2048 else float("nan")
        print(f"{m}x{n}x{k} {cfg} err={err:.3e} ok={err <= O.SGEMM_TF32_TOL} ms={t*1e3:.4f} "
              f"TF={p.total_flops / t / 1e12:.1f}", flush=True)
    for b in p.buffers.values():
        b.free()
try:
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    p = SgemmTF32Problem(m=sizes[-1][0], n=sizes[-1][1], k=sizes[-1][2])
    inp = p.host_inputs()
    a = torch.from_numpy(inp["a"]).cuda(); b = torch.from_numpy(inp["b"]).cuda(); c0 = torch.from_numpy(inp["c0"]).cuda()
    out = (p.alpha * (a @ b) + p.beta * c0).cpu().numpy()
    print("torch/cuBLAS TF32 calibration error", O.sgemm_error(out, O.sgemm(inp["a"], inp["b"], inp["c0"], p.alpha, p.beta)))
except Exception as exc:  # noqa: BLE001
    print("torch calibration skipped:", exc)
