"""Persistent CTA-pair TF32 SGEMM (sgemm_tf32c2p.cu): correctness at several shapes, then full-size
timing against the non-persistent pair kernel. Run under `timeout` (cluster barriers can hang)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200.gpu import GPU  # noqa: E402
from paper_2211_07260_b200.kernels import SgemmTF32Problem  # noqa: E402

gpu = GPU(0)
for (m, n, k) in [(512, 512, 512), (256, 256, 64), (1024, 768, 320), (2560, 2048, 1024), (4096, 4096, 4096)]:
    p = SgemmTF32Problem(m=m, n=n, k=k)
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    for cfg in [dict(BN=256, STAGES=4, PERSIST=1, SPLIT_TAIL=0, PAIR=1),
                dict(BN=256, STAGES=4, PERSIST=1, SPLIT_TAIL=1, PAIR=1),
                dict(BN=256, STAGES=5, PERSIST=1, SPLIT_TAIL=1, PAIR=1),
                dict(BN=128, STAGES=6, PERSIST=1, SPLIT_TAIL=0, PAIR=1),
                dict(BN=256, STAGES=3, PERSIST=0, SPLIT_TAIL=0, PAIR=1)]:
        if not p.is_valid(cfg):
            print((m, n, k), cfg, "invalid", flush=True)
            continue
        kern = p.kernel(cfg)
        p.reset_output()
        gpu.launch(kern, p.launch(cfg), p.args(cfg))
        gpu.synchronize()
        err = O.sgemm_error(p.fetch_output(), ref)
        first = p.fetch_output().copy()
        t = gpu.time(kern, p.launch(cfg), p.args(cfg), reps=20) / 20
        p.reset_output()
        gpu.launch(kern, p.launch(cfg), p.args(cfg))
        gpu.synchronize()
        again = bool((p.fetch_output() == first).all())  # relaunch gives the same bits (split reduction order)
        print((m, n, k), cfg, f"err={err:.2e} ok={1e-6 < err <= O.SGEMM_TF32_TOL} {t * 1e3:.4f} ms "
              f"{p.total_flops / t / 1e12:.1f} TF/s relaunch_identical={again}", flush=True)
    for b in p.buffers.values():
        b.free()
