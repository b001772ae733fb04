"""Why does a persistent PnPoly-shaped stream stop at ~93% of HBM? (cells kernel, round 2)

``scripts/stream_probe.py`` found that a one-pass grid reaches 99.4% of the
measured HBM copy peak on the 240 MB PnPoly stream (8 bytes read, 4 written per
point), while every persistent grid-stride variant stops at 92-94% whatever
its bytes in flight (up to 168 KB per SM with bulk-copy rings). The cells
kernel must be persistent (it stages a 49 KB raster in shared memory once per
block), so this probe tests the hypothesis that the persistent loss is the
static schedule's tail: 10 M vectors in chunks of BS x U over SMs x blocks
gives 16.5 rounds, so half the blocks run one chunk more than the average,
and SMs do not all stream at the same speed.

* SCHED 0: one pass (a block per chunk), the reference shape;
* SCHED 1: persistent, static round-robin chunks (the cells kernel today);
* SCHED 2: persistent, chunks claimed with one atomicAdd per block and chunk
  (double-buffered index in shared memory, one __syncthreads per chunk; the
  counter resets itself when the last block leaves);
* SCHED 3: persistent, static rounds except the last two, which are claimed
  dynamically (the atomic traffic of SCHED 2 cut to the tail).

    python scripts/persist_probe.py      # -> gpurun_out/persist_probe.jsonl
"""

from __future__ import annotations

import itertools
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_07260_b200 import native  # noqa: E402
from paper_2211_07260_b200.gpu import GPU, Launch, i32  # noqa: E402

SRC = r"""
#define BODY(c)                                                                                         \
    do {                                                                                                \
        float x[U][4];                                                                                  \
        _Pragma("unroll") for (int u = 0; u < U; ++u) {                                                 \
            const int v = (c) * BS * U + u * BS + threadIdx.x;                                          \
            if (v < nvec)                                                                               \
                asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"                 \
                             : "=f"(x[u][0]), "=f"(x[u][1]), "=f"(x[u][2]), "=f"(x[u][3])               \
                             : "l"(pts + (long long)v * 4));                                            \
        }                                                                                               \
        _Pragma("unroll") for (int u = 0; u < U; ++u) {                                                 \
            const int v = (c) * BS * U + u * BS + threadIdx.x;                                          \
            if (v < nvec)                                                                               \
                asm volatile("st.global.cs.v2.s32 [%0], {%1,%2};" ::"l"(out + (long long)v * 2),         \
                             "r"(x[u][0] < x[u][1] ? 1 : 0), "r"(x[u][2] < x[u][3] ? 1 : 0) : "memory"); \
        }                                                                                               \
    } while (0)

extern "C" __global__ void __launch_bounds__(BS, MINB)
stream(int *__restrict__ out, const float *__restrict__ pts, int nvec, unsigned *__restrict__ ctr) {
    __shared__ int s_c[2];
    const int nchunks = (nvec + BS * U - 1) / (BS * U);
    int c = blockIdx.x;
#if SCHED == 0
    if (c < nchunks) BODY(c);
    return;
#elif SCHED == 1
    for (; c < nchunks; c += gridDim.x) BODY(c);
    return;
#else
#if SCHED == 3
    // static rounds, no block-wide sync, except the last two rounds' worth of chunks
    const int rounds = (int)(nchunks / gridDim.x) - 2;
    const int n_static = (rounds > 1 ? rounds : 1) * (int)gridDim.x;
    for (; c + (int)gridDim.x < n_static; c += gridDim.x) BODY(c);
#else
    const int n_static = gridDim.x;  // the first chunk of every block is its own
#endif
    // c is this block's last static chunk; the rest are claimed, one ahead
    int it = 0;
    while (c < nchunks) {
        if (threadIdx.x == 0) s_c[(it + 1) & 1] = n_static + (int)atomicAdd(ctr, 1u);
        BODY(c);
        __syncthreads();
        c = s_c[(++it) & 1];
    }
    if (threadIdx.x == 0) {  // the last block out resets the counters for the next launch
        __threadfence();
        if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
            ctr[0] = 0;
            ctr[1] = 0;
            __threadfence();
        }
    }
#endif
}
"""

N_POINTS = 20_000_000


def main() -> None:
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6549.4)
    rng = np.random.default_rng(4)
    pts = rng.uniform(-1, 1, (N_POINTS, 2)).astype(np.float32)
    want = (pts[:, 0] < pts[:, 1]).astype(np.int32)
    rows = []
    with GPU(0) as gpu:
        sets = [(gpu.empty((N_POINTS,), np.int32), gpu.array(pts)) for _ in range(2)]
        ctr = gpu.array(np.zeros(2, np.uint32))
        sms = gpu.sm_count
        nvec = N_POINTS // 2
        for sched, u, bs, occ in itertools.product((0, 1, 2, 3), (1, 2, 4, 8), (256, 512, 1024), (1024, 2048)):
            if sched == 0 and occ == 1024:
                continue
            minb = occ // bs
            opts = native._nvrtc_options({"SCHED": sched, "U": u, "BS": bs, "MINB": minb})
            try:
                k = gpu.load(native.compile_cubin(SRC, "persist_probe", opts), "stream")
            except Exception as exc:  # noqa: BLE001
                print("compile failed", sched, u, bs, minb, exc, flush=True)
                continue
            blocks = -(-nvec // (bs * u))
            if sched:
                blocks = min(blocks, sms * minb)
            launch = Launch((blocks, 1, 1), (bs, 1, 1))
            args = [[o, p, i32(nvec), ctr] for o, p in sets]
            for rep in range(2):  # twice: the counter must have reset itself
                sets[0][0].fill(0)
                gpu.launch(k, launch, args[0])
                gpu.synchronize()
            ok = bool(np.array_equal(sets[0][0].download(), want))
            run = gpu.bench(k, launch, args[0], rotate=args[1:], min_seconds=0.3, sample=False)
            gbs = 12.0 * N_POINTS / run.per_launch_s / 1e9
            rec = {"SCHED": sched, "U": u, "BS": bs, "OCC": occ, "blocks": blocks, "regs": k.regs, "ok": ok,
                   "us": round(run.per_launch_s * 1e6, 2), "gb_s": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4)}
            print(json.dumps(rec), flush=True)
            rows.append(rec)
    for s in range(4):
        sub = [r for r in rows if r["SCHED"] == s]
        if sub:
            print("best SCHED", s, max(sub, key=lambda r: r["gb_s"]), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/persist_probe.jsonl").write_text("\n".join(json.dumps(r) for r in rows) + "\n")


if __name__ == "__main__":
    main()
