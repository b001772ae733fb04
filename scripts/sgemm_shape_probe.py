"""SGEMM FP32 4096^3: CTA-shape / occupancy probe around the tuned config, device-timed, oracle-checked.

Variants the tuning samples did not cover together: 256-thread CTAs (8 x 8 and 8 x 16 per thread),
256-wide tiles with one CTA per SM, KWG 32 (half the barriers), each with and without a
MIN_BLOCKS register cap. Prints one JSON line per variant.

    python scripts/sgemm_shape_probe.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import kernels_oracle as O  # noqa: E402
from paper_2211_07260_b200 import native, tuned  # noqa: E402
from paper_2211_07260_b200.gpu import GPU, fp32_peak_tflops  # noqa: E402
from paper_2211_07260_b200.kernels import SgemmProblem  # noqa: E402

base = {**SgemmProblem(value_set="b200").default_config(), **tuned.best_config("sgemm")}
VARIANTS = [
    ({}, 0),
    ({"GROUP_M": 16}, 0),
    ({"KWG": 32, "ASYNC": 3}, 0),
    ({"KWG": 32, "ASYNC": 3, "GROUP_M": 16}, 0),
    # 256 threads, 8 x 8 per thread, two CTAs per SM (16 warps)
    ({"MDIMC": 16, "NDIMC": 16, "MDIMA": 16, "NDIMB": 16, "VWN": 4}, 0),
    ({"MDIMC": 16, "NDIMC": 16, "MDIMA": 16, "NDIMB": 16, "VWN": 4}, 2),
    ({"MDIMC": 16, "NDIMC": 16, "MDIMA": 16, "NDIMB": 16, "VWN": 4, "KWI": 4}, 2),
    ({"MDIMC": 16, "NDIMC": 16, "MDIMA": 16, "NDIMB": 16, "VWN": 4, "KWG": 32, "ASYNC": 3}, 2),
    # 256 threads, 8 x 16 per thread, 128 x 256 / 256 x 128 tiles, one CTA per SM
    ({"NWG": 256, "MDIMC": 16, "NDIMC": 16, "MDIMA": 16, "NDIMB": 32, "ASYNC": 3}, 0),
    ({"MWG": 256, "MDIMC": 32, "NDIMC": 8, "MDIMA": 32, "NDIMB": 16, "ASYNC": 3}, 0),
    # three 128-thread CTAs per SM with a lighter fragment prefetch
    ({"KWI": 2}, 3),
    ({"KWI": 4}, 3),
]


def main():
    gpu = GPU(0)
    p = SgemmProblem(value_set="b200")
    p.prepare(gpu)
    ref = O.sgemm(p.inputs["a"], p.inputs["b"], p.inputs["c0"], p.alpha, p.beta)
    for delta, mb in VARIANTS:
        cfg = {**base, **delta}
        rec = {"delta": delta, "min_blocks": mb}
        if not p.is_valid(cfg):
            rec["skipped"] = "invalid"
            print(json.dumps(rec), flush=True)
            continue
        defs = p.defines(cfg)
        if mb:
            defs["MIN_BLOCKS"] = mb
        try:
            k = gpu.load(native.compile_cubin(native.kernel_source(p.source), p.name, native._nvrtc_options(defs)),
                         p.symbol)
            p.reset_output()
            gpu.launch(k, p.launch(cfg), p.args(cfg))
            gpu.synchronize()
            err = O.sgemm_error(p.fetch_output(), ref)
            gpu.time(k, p.launch(cfg), p.args(cfg), reps=20)
            t = min(gpu.time(k, p.launch(cfg), p.args(cfg), reps=50) / 50 for _ in range(3))
        except Exception as e:  # noqa: BLE001
            rec["error"] = str(e)[:200]
            print(json.dumps(rec), flush=True)
            continue
        tf = p.total_flops / t / 1e12
        rec.update(regs=k.regs, local=k.local_bytes, err=float(err), ms=round(t * 1e3, 4), tflops=round(tf, 2),
                   frac_at_1965=round(tf / fp32_peak_tflops(gpu.sm_count, 1965.0), 4))
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
