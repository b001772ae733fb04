"""Issue-rate microbenchmarks behind the PnPoly brute-force ceiling.

Each probe is a loop of independent chains of one instruction form (inline
PTX, so ptxas emits exactly that SASS op), run by as many 256-thread
blocks per SM as are resident at once (up to 4, register-limited). Every warp times its loop with clock64; the
issue rate per SMSP is warps_per_smsp x instructions_per_iteration x iters /
cycles. Forms:

  ffma_rrr   FFMA with three distinct register sources
  ffma_rri   FFMA with an immediate multiplicand (2 register sources)
  fadd_rr    FADD, two register sources
  fadd2_bc   FADD2 {s, s} - pair (the ASM 7 form: broadcast scalar + pair)
  ffma2_bc   FFMA2 pair * {s, s} + pair
  lop3_rrr   LOP3 with three register sources
  lop3_rri   LOP3 with two register sources and an immediate
  mix_f2_lop one FADD2 (broadcast form) + one 3-register LOP3 per chain step
  mix_f_lop  one FADD + one 3-register LOP3 per chain step
  asm7_edge2 the ASM 7 step for one point and two edges: FADD2, FFMA2, FADD2
             (broadcast scalar operands) and three 3-register LOP3s
  asm7_dep   the same, with the LOP3s reading the halves of the FADD2 results
             (the kernel's data flow)

The SASS op counts of each probe's loop (cuobjdump) are printed with it, so a
rate can be read per SASS instruction actually issued.

    python scripts/issue_probe.py            (prints one JSON line per form)
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_07260_b200 import native  # noqa: E402
from paper_2211_07260_b200.gpu import GPU, Launch, f32, i32  # noqa: E402

CHAINS = 8
UNROLL = 4  # body repeats per loop trip (the 3-instruction loop overhead is amortised)
FORMS = {
    # name: (per-chain PTX body using %c (chain reg) and per-chain invariants, instrs per chain per iter, regs)
    "ffma_rrr": ("fma.rn.f32 c{k}, c{k}, x{k}, y{k};", 1),
    "ffma_rri": ("fma.rn.f32 c{k}, c{k}, 0f3F800001, y{k};", 1),
    "fadd_rr": ("add.rn.f32 c{k}, c{k}, x{k};", 1),
    "fadd2_bc": ("mov.b64 t{k}, {{s, s}};\nsub.rn.f32x2 p{k}, t{k}, p{k};", 1),
    "ffma2_bc": ("mov.b64 t{k}, {{s, s}};\nfma.rn.f32x2 p{k}, p{k}, t{k}, q{k};", 1),
    "lop3_rrr": ("lop3.b32 u{k}, u{k}, v{k}, w{k}, 0x96;", 1),
    "lop3_rri": ("lop3.b32 u{k}, u{k}, v{k}, 0x5A5A5A5A, 0x96;", 1),
    "mix_f2_lop": ("mov.b64 t{k}, {{s, s}};\nsub.rn.f32x2 p{k}, t{k}, p{k};\nlop3.b32 u{k}, u{k}, v{k}, w{k}, 0x96;", 2),
    "mix_f_lop": ("add.rn.f32 c{k}, c{k}, x{k};\nlop3.b32 u{k}, u{k}, v{k}, w{k}, 0x96;", 2),
    # the same mix, but the LOP3s consume the halves of the f32x2 results (as in the kernel)
    "asm7_dep": ("{{\n.reg .b32 dl, dh, el, eh;\nmov.b64 t{k}, {{s, s}};\nsub.rn.f32x2 p{k}, t{k}, p{k};\n"
                 "fma.rn.f32x2 q{k}, q{k}, t{k}, p{k};\nsub.rn.f32x2 q{k}, t{k}, q{k};\n"
                 "mov.b64 {{dl, dh}}, p{k};\nmov.b64 {{el, eh}}, q{k};\n"
                 "lop3.b32 u{k}, dl, w{k}, el, 0x28;\nlop3.b32 v{k}, dh, dl, eh, 0x28;\n"
                 "lop3.b32 w{k}, w{k}, u{k}, v{k}, 0x96;\n}}", 6),
    # predicate forms (PnPoly ASM 1/2 style): FSETP chains and a predicated-toggle crossing step
    # (third field: chains, so the predicates fit the 7 hardware predicate registers)
    "fsetp_and": ("setp.lt.and.f32 P{k}, c{k}, x{k}, P{k};", 1, 6),
    "asm1_step": ("setp.ge.f32 S{k}, c{k}, x{k};\nsetp.lt.and.f32 S{k}, c{k}, y{k}, S{k};\n"
                  "fma.rn.f32 y{k}, y{k}, s, x{k};\n@S{k} setp.lt.xor.f32 P{k}, s, y{k}, P{k};", 4, 3),
    "asm7_edge2": ("mov.b64 t{k}, {{s, s}};\nsub.rn.f32x2 p{k}, t{k}, p{k};\nfma.rn.f32x2 q{k}, p{k}, t{k}, q{k};\n"
                   "sub.rn.f32x2 p{k}, t{k}, q{k};\nlop3.b32 u{k}, u{k}, v{k}, w{k}, 0x28;\n"
                   "lop3.b32 v{k}, u{k}, v{k}, w{k}, 0x28;\nlop3.b32 w{k}, u{k}, v{k}, w{k}, 0x96;", 6),
}

TEMPLATE = r"""
extern "C" __global__ void __launch_bounds__(256) probe(unsigned long long *cycles, float *sink, int iters, float s_in) {
    unsigned long long t0, t1;
    float out;
    asm volatile("{\n"
        ".reg .f32 s, %s;\n.reg .b32 %s;\n.reg .b64 %s;\n.reg .pred lp, %s;\n.reg .s32 it;\n"
        "mov.f32 s, %%3;\n"
        %s
        "mov.u64 %%0, %%clock64;\n"
        "mov.s32 it, %%4;\n"
        "LOOP:\n"
        %s
        "sub.s32 it, it, 1;\n"
        "setp.gt.s32 lp, it, 0;\n"
        "@lp bra LOOP;\n"
        "mov.u64 %%1, %%clock64;\n"
        %s
        "}\n" : "=l"(t0), "=l"(t1), "=f"(out) : "f"(s_in + 0.001f * threadIdx.x), "r"(iters));
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned smid;
    asm volatile("mov.u32 %%0, %%%%smid;" : "=r"(smid));
    if ((threadIdx.x & 31) == 0) {  // per warp: SM id, start and end of the timed loop (SM clock)
        cycles[3 * gw] = smid;
        cycles[3 * gw + 1] = t0;
        cycles[3 * gw + 2] = t1;
    }
    if (out == 12345.f) sink[threadIdx.x] = out;
}
"""


def kernel_source(body: str, chains: int = CHAINS) -> str:
    f32 = ", ".join(f"c{k}, x{k}, y{k}" for k in range(CHAINS))
    b32 = ", ".join(f"u{k}, v{k}, w{k}" for k in range(CHAINS))
    b64 = ", ".join(f"p{k}, q{k}, t{k}" for k in range(CHAINS))
    preds = ", ".join(f"P{k}, S{k}" for k in range(CHAINS))
    init = ""
    for k in range(CHAINS):
        init += (f"add.f32 c{k}, s, 0f3F8{k}0000;\nadd.f32 x{k}, s, 0f3F9{k}0000;\nadd.f32 y{k}, s, 0f3FA{k}0000;\n"
                 f"mov.b32 u{k}, c{k};\nmov.b32 v{k}, x{k};\nmov.b32 w{k}, y{k};\n"
                 f"mov.b64 p{k}, {{x{k}, y{k}}};\nmov.b64 q{k}, {{y{k}, c{k}}};\nmov.b64 t{k}, {{s, s}};\n"
                 f"setp.lt.f32 P{k}, c{k}, x{k};\nsetp.lt.f32 S{k}, x{k}, c{k};\n")
    loop = "".join(body.format(k=k) + "\n" for _ in range(UNROLL) for k in range(chains))
    fold = "mov.f32 %2, c0;\n"
    for k in range(CHAINS):
        fold += (f"add.f32 %2, %2, c{k};\nadd.f32 %2, %2, x{k};\nadd.f32 %2, %2, y{k};\n"
                 f"{{ .reg .f32 a, b; mov.b64 {{a, b}}, p{k}; add.f32 %2, %2, a; add.f32 %2, %2, b; "
                 f"mov.b64 {{a, b}}, q{k}; add.f32 %2, %2, a; }}\n"
                 f"{{ .reg .b32 z; xor.b32 z, u{k}, v{k}; xor.b32 z, z, w{k}; cvt.rn.f32.u32 x{k}, z; "
                 f"add.f32 %2, %2, x{k}; }}\n"
                 f"{{ .reg .f32 z; selp.f32 z, 1.0, 0.0, P{k}; add.f32 %2, %2, z; }}\n")
    return TEMPLATE % (f32, b32, b64, preds, cstr(init), cstr(loop), cstr(fold))


def cstr(ptx: str) -> str:
    """Multi-line PTX as concatenated C string literals."""
    return "".join(f'"{line}\\n"\n' for line in ptx.splitlines() if line.strip())


def loop_ops(cubin: bytes) -> dict:
    """SASS op histogram of the timed loop (branch target .. backward branch)."""
    import re
    import subprocess
    import tempfile
    from collections import Counter

    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(cubin)
        f.flush()
        sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
    rows = []
    for line in sass.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            rows.append((int(m.group(1), 16), m.group(2).strip()))
    for i, (addr, ins) in enumerate(rows):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", ins)
        if m and m.group(1) and int(m.group(1), 16) < addr:
            start = int(m.group(1), 16)
            body = [x for a, x in rows if start <= a <= addr]
            return dict(Counter((x.split()[1] if x.startswith("@") else x.split()[0]) for x in body))
    return {}


def main():
    gpu = GPU(0)
    sms = gpu.sm_count
    threads, iters = 256, 4096
    cycles = gpu.empty((3 * sms * 8 * threads // 32,), np.uint64)
    sink = gpu.empty((threads,), np.float32)
    for name, (body, per_chain, *rest) in FORMS.items():
        chains = rest[0] if rest else CHAINS
        src = kernel_source(body, chains)
        cubin = native.compile_cubin(src, f"probe_{name}", native._nvrtc_options({}))
        k = gpu.load(cubin, "probe")
        # launch only as many blocks as are resident at once (register-limited), so every
        # warp's clock64 window overlaps the others' and per-SM rates are not inflated
        resident = max(1, min(4, 65536 // (max(k.regs, 1) * threads)))
        blocks = sms * resident
        launch = Launch((blocks, 1, 1), (threads, 1, 1))
        args = [cycles, sink, i32(iters), f32(1.5)]
        gpu.launch(k, launch, args)
        gpu.synchronize()
        gpu.launch(k, launch, args)
        gpu.synchronize()
        raw = cycles.download()[: 3 * blocks * threads // 32].reshape(-1, 3)
        sm, t0, t1 = raw[:, 0].astype(np.int64), raw[:, 1].astype(np.float64), raw[:, 2].astype(np.float64)
        # per SM: all of its warps' instructions over the SM's busy window (first start to last
        # end on that SM's clock), per SMSP; blocks that ran in a second wave are then counted
        # against the time they really took
        instrs = per_chain * chains * UNROLL * iters
        ops = loop_ops(cubin)
        rates, issued_rates, spans = [], [], []
        for s_id in np.unique(sm):
            w = sm == s_id
            window = t1[w].max() - t0[w].min()
            rates.append(w.sum() / 4.0 * instrs / window)
            issued_rates.append(w.sum() / 4.0 * sum(ops.values()) * iters / window)
            spans.append(window / np.median(t1[w] - t0[w]))
        per_smsp = float(np.median(rates))
        issued = float(np.median(issued_rates))
        warps_per_smsp = float(np.median(np.bincount(sm)[np.unique(sm)])) / 4.0
        span = float(np.median(spans))  # 1 = the SM's warps all ran concurrently, 2 = two waves
        cyc = t1 - t0
        print(json.dumps({"form": name, "regs": k.regs, "blocks_per_sm": resident, "span": round(float(span), 3),
                          "instrs_per_trip_per_warp": per_chain * chains * UNROLL,
                          "sass_loop_ops": ops, "sass_issue_per_smsp_per_cycle": round(issued, 3),
                          "warp_instr_per_smsp_per_cycle": round(per_smsp, 3),
                          "median_cycles": float(np.median(cyc)), "warps_per_smsp": warps_per_smsp}), flush=True)
    gpu.close()


if __name__ == "__main__":
    main()
