// PnPoly point-in-polygon (crossing number), sm_100a, compiled per config by NVRTC.
//
// No reference code exists for this kernel: it is the paper's
// Kernel-Tuner PnPoly benchmark rebuilt for B200. Output bitmap[i] = 1 when
// point i is inside the polygon (odd number of edge crossings of the ray
// y = py, x > px).
//
// Tunables (-D):
//   BLOCK_SIZE_X  threads per block
//   TILE          points per thread (edge data is loaded once per TILE points)
//   VEC           1: float2 point loads; 2: float4 loads (two points per load)
//   METHOD        edge crossing formula, each bit-exact against its own
//                 float32 oracle (oracle/pnpoly_oracle.c):
//                   0  x = (dx * (py - vy)) / dy + vx      (IEEE div, no FMA)
//                   1  x = fma(slope, py - vy, vx)         (slope = dx / dy)
//                   2  x = fma(slope, py, icpt)            (icpt = fma(-slope, vy, vx))
//   BETWEEN       0: (vy_k > py) != (vy_prev > py)   1: ymin <= py < ymax
//                 (identical booleans; different instruction shapes)
//   POLY_SMEM     0: edge table in __constant__ memory; 1: staged in shared memory
//   VERTICES      polygon size (compile-time so the edge loop is counted)
//   MIN_BLOCKS    (optional) __launch_bounds__ minimum resident blocks per SM,
//                 capping registers so more warps fit. Swept by
//                 scripts/time_pnpoly_minb.py: no gain (occupancy is not what
//                 limits ASM 7), so it is not in the tuning space.
//   (launch)      persist=1 in the tuning space sizes the grid to the SMs'
//                 residency and the kernel strides over point tiles
//   ASM           1: hand-written PTX edge loop (needs BETWEEN=1, POLY_SMEM=1,
//                 METHOD 2, TILE in {1,2,4,6}): per edge one LDS.128 of the
//                 packed record {ymin, ymax, slope, icpt}, then per point
//                   setp.ge  s, py, ymin; setp.lt.and s, py, ymax, s;
//                   fma.rn x, slope, py, icpt;
//                   @s setp.lt.xor in, px, x, in      (toggle fused in the compare)
//                 with the inside flags living in predicate registers for the
//                 whole loop (TILE inside flags + 1 scratch <= 7 predicates).
//                 2: same, but two edges' crossings (s & left) are folded into
//                 the flag with one 3-input predicate XOR (PLOP3) per point.
//                 3: sign-bit formulation on the FMA pipe (needs POLY_SMEM=1,
//                 METHOD=2, TILE in {2,4,6,8}): per edge-point
//                   FADD d = py - vy_k; FFMA x; FADD e = px - x;
//                   LOP3 t = (d ^ d_prev) & e; (1/2) LOP3 acc ^= t1 ^ t2
//                 inside = sign bit of acc. Bit-exact against the oracle's
//                 formulation 3 (same as formula 2 unless a coordinate is -0.0).
//                 4: ASM 3 with point pairs in packed f32x2 registers
//                 (FADD2/FFMA2): 1.5 FMA-pipe + 1.5 ALU instructions per
//                 edge-point (VEC=2, TILE in {4,8}); same formulation 3.
//                 5: ASM 3 with sign(d_k ^ d_{k-1}) taken from an FMUL (IEEE
//                 product sign): 4 FMA-pipe + 1 LOP3 per edge-point.
//                 6: ASM 5 on point pairs (FADD2/FMUL2/FFMA2). Same formulation 3.
//                 7: ASM 3 with EDGE pairs in the packed f32x2 lanes and the
//                 point's coordinates as the broadcast scalar operand: per
//                 point and 2 edges FADD2 d, FFMA2 x, FADD2 e, then 1.5 LOP3
//                 per edge. The pairs come straight out of LDS.64 of the
//                 structure-of-arrays table {vy0..3, sl0..3, ic0..3} per 4
//                 edges, so no register shuffling: 3 issue slots per
//                 edge-point (1.5 FMA-pipe + 1.5 ALU). Same formulation 3.
//                 9: ASM 7 over a table whose 128-bit loads put each slope pair
//                 and intercept pair in opposite halves of a register quad (no
//                 register-bank overlap between the two FFMA2 pair operands).
//                 Measured identical to ASM 7 (1.775 ms): bank conflicts on the
//                 FFMA2 are not what holds ASM 7 back.
//                 8: ASM 7's arithmetic written in C++ over the same table
//                 held in __constant__ memory (POLY_SMEM=0): the edge pairs
//                 are warp-uniform loads, so ptxas can feed them to FADD2 /
//                 FFMA2 as uniform-register operands and the f32x2 ops read
//                 fewer vector registers (register-read bandwidth, not the
//                 FMA pipe, is what holds ASM 7's dispatch back).
//
// Edge table (built on the host in float32, see kernels.py): per edge k from
// vertex k-1 (cyclic) to vertex k, a float4 {vy_k, a, b, c} and a float2
// {ymin, ymax}:
//   METHOD 0: a = vx_k, b = dx = vx_{k-1} - vx_k, c = dy = vy_{k-1} - vy_k
//   METHOD 1: a = vx_k, b = slope = dx / dy, c = unused
//   METHOD 2: a = icpt, b = slope,           c = unused
#ifndef BLOCK_SIZE_X
#define BLOCK_SIZE_X 256
#endif
#ifndef TILE
#define TILE 4
#endif
#ifndef VEC
#define VEC 1
#endif
#ifndef METHOD
#define METHOD 2
#endif
#ifndef BETWEEN
#define BETWEEN 0
#endif
#ifndef POLY_SMEM
#define POLY_SMEM 0
#endif
#ifndef VERTICES
#define VERTICES 600
#endif
#ifndef ASM
#define ASM 0
#endif
#if VEC == 2 && (TILE % 2) != 0
#error "VEC=2 needs an even TILE"
#endif
#if (ASM == 1 || ASM == 2) && !(BETWEEN == 1 && POLY_SMEM == 1 && METHOD == 2 && \
             (TILE == 1 || TILE == 2 || TILE == 4 || TILE == 6))
#error "ASM=1|2 needs BETWEEN=1, POLY_SMEM=1, METHOD=2 and TILE in {1,2,4,6}"
#endif
#if ASM == 3 && !(POLY_SMEM == 1 && METHOD == 2 && (TILE == 2 || TILE == 4 || TILE == 6 || TILE == 8))
#error "ASM=3 needs POLY_SMEM=1, METHOD=2 and TILE in {2,4,6,8}"
#endif
#if (ASM == 4 || ASM == 6) && !(POLY_SMEM == 1 && METHOD == 2 && VEC == 2 && (TILE == 4 || TILE == 8))
#error "ASM=4|6 needs POLY_SMEM=1, METHOD=2, VEC=2 and TILE in {4,8}"
#endif
#if ASM == 5 && !(POLY_SMEM == 1 && METHOD == 2 && (TILE == 2 || TILE == 4 || TILE == 6 || TILE == 8))
#error "ASM=5 needs POLY_SMEM=1, METHOD=2 and TILE in {2,4,6,8}"
#endif
#if (ASM == 7 || ASM == 9) && !(POLY_SMEM == 1 && METHOD == 2 && (TILE == 2 || TILE == 4 || TILE == 6 || TILE == 8))
#error "ASM=7 needs POLY_SMEM=1, METHOD=2 and TILE in {2,4,6,8}"
#endif
#if ASM == 8 && !(POLY_SMEM == 0 && METHOD == 2)
#error "ASM=8 needs POLY_SMEM=0 and METHOD=2"
#endif
// packed records {ymin, ymax, slope, icpt} (METHOD 2) padded
// to a multiple of 4 with never-spanning dummies {+inf, -inf, 0, 0}
#define NPACK (((VERTICES) + 3) / 4 * 4)
// ASM 7 table: edges padded to a multiple of 8 (two 4-edge groups per loop
// trip), 12 floats per 4-edge group
#define NPAIR8 (((VERTICES) + 7) / 8 * 8)
#if ASM == 7 || ASM == 8 || ASM == 9
#define TAB_VEC4 (NPAIR8 * 3 / 4)
#else
#define TAB_VEC4 NPACK
#endif

#if ASM == 1 || ASM == 2
#define PT_X(PY) "fma.rn.f32 x, sl, %" PY ", ic;\n"
#define PT(PIN, PX, PY)                         \
    "setp.ge.f32 s, %" PY ", ylo;\n"            \
    "setp.lt.and.f32 s, %" PY ", yhi, s;\n"     \
    PT_X(PY)                                    \
    "@s setp.lt.xor.f32 " PIN ", %" PX ", x, " PIN ";\n"
#define LD_EDGE(OFF) "ld.shared.v4.f32 {ylo, yhi, sl, ic}, [ptr+" OFF "];\n"
#if TILE == 1
#define PTS PT("p0", "1", "2")
#define BASE_OP "3"
#define END_OP "5"
#define OUT_SELP "selp.u32 %0, 1, 0, p0;\n"
#define PREDS ".reg .pred p0, s;\n"
#define INIT "setp.ne.u32 p0, %4, 0;\n"
#elif TILE == 2
#define PTS PT("p0", "2", "4") PT("p1", "3", "5")
#define BASE_OP "6"
#define END_OP "8"
#define OUT_SELP "selp.u32 %0, 1, 0, p0;\n" "selp.u32 %1, 1, 0, p1;\n"
#define PREDS ".reg .pred p0, p1, s;\n"
#define INIT "setp.ne.u32 p0, %7, 0;\n" "mov.pred p1, p0;\n"
#elif TILE == 4
#define PTS PT("p0", "4", "8") PT("p1", "5", "9") PT("p2", "6", "10") PT("p3", "7", "11")
#define BASE_OP "12"
#define END_OP "14"
#define OUT_SELP "selp.u32 %0, 1, 0, p0;\n" "selp.u32 %1, 1, 0, p1;\n" \
                 "selp.u32 %2, 1, 0, p2;\n" "selp.u32 %3, 1, 0, p3;\n"
#define PREDS ".reg .pred p0, p1, p2, p3, s;\n"
#define INIT "setp.ne.u32 p0, %13, 0;\n" "mov.pred p1, p0;\n" "mov.pred p2, p0;\n" "mov.pred p3, p0;\n"
#else
#define PTS PT("p0", "6", "12") PT("p1", "7", "13") PT("p2", "8", "14") \
            PT("p3", "9", "15") PT("p4", "10", "16") PT("p5", "11", "17")
#define BASE_OP "18"
#define END_OP "20"
#define OUT_SELP "selp.u32 %0, 1, 0, p0;\n" "selp.u32 %1, 1, 0, p1;\n" "selp.u32 %2, 1, 0, p2;\n" \
                 "selp.u32 %3, 1, 0, p3;\n" "selp.u32 %4, 1, 0, p4;\n" "selp.u32 %5, 1, 0, p5;\n"
#define PREDS ".reg .pred p0, p1, p2, p3, p4, p5, s;\n"
#define INIT "setp.ne.u32 p0, %19, 0;\n" "mov.pred p1, p0;\n" "mov.pred p2, p0;\n" \
             "mov.pred p3, p0;\n" "mov.pred p4, p0;\n" "mov.pred p5, p0;\n"
#endif
#if ASM == 2
// pair mode: two edges per point feed one 3-input predicate XOR (PLOP3)
#define PT2(PIN, PX, PY)                                 \
    "setp.ge.f32 s, %" PY ", ylo;\n"                     \
    "setp.lt.and.f32 s, %" PY ", yhi, s;\n"              \
    "fma.rn.f32 x, sl, %" PY ", ic;\n"                   \
    "setp.lt.and.f32 q, %" PX ", x, s;\n"                \
    "setp.ge.f32 s, %" PY ", ylo2;\n"                    \
    "setp.lt.and.f32 s, %" PY ", yhi2, s;\n"             \
    "fma.rn.f32 x, sl2, %" PY ", ic2;\n"                 \
    "setp.lt.and.f32 s, %" PX ", x, s;\n"                \
    "xor.pred " PIN ", " PIN ", q;\n"                    \
    "xor.pred " PIN ", " PIN ", s;\n"
#define LD_EDGE2(OFF, OFF2) "ld.shared.v4.f32 {ylo, yhi, sl, ic}, [ptr+" OFF "];\n" \
                            "ld.shared.v4.f32 {ylo2, yhi2, sl2, ic2}, [ptr+" OFF2 "];\n"
#if TILE == 1
#define PTS2 PT2("p0", "1", "2")
#elif TILE == 2
#define PTS2 PT2("p0", "2", "4") PT2("p1", "3", "5")
#elif TILE == 4
#define PTS2 PT2("p0", "4", "8") PT2("p1", "5", "9") PT2("p2", "6", "10") PT2("p3", "7", "11")
#else
#define PTS2 PT2("p0", "6", "12") PT2("p1", "7", "13") PT2("p2", "8", "14") \
             PT2("p3", "9", "15") PT2("p4", "10", "16") PT2("p5", "11", "17")
#endif
#define EDGE(OFF) ""
#define BODY LD_EDGE2("0", "16") PTS2 LD_EDGE2("32", "48") PTS2
#define EXTRA_REGS ".reg .pred q;\n.reg .f32 ylo2, yhi2, sl2, ic2;\n"
#else
#define EDGE(OFF) LD_EDGE(OFF) PTS
#define BODY EDGE("0") EDGE("16") EDGE("32") EDGE("48")
#define EXTRA_REGS ""
#endif
#endif
#if ASM == 3
// sign-bit variant: every comparison becomes the sign of an exactly rounded
// float32 difference (FADD on the FMA pipe); the crossing bit of edge k for a
// point is  sign((py - vy_k) ^ (py - vy_{k-1})) & sign(px - x_k)  (one LOP3),
// and two edges' bits fold into the parity word with one 3-input XOR LOP3.
#if TILE == 2
#define S3_POINTS \
    "sub.rn.f32 da, %4, vy0;\n" "fma.rn.f32 x, sl0, %4, ic0;\n" "sub.rn.f32 e, %2, x;\n" "lop3.b32 t1, da, dp0, e, 0x28;\n" \
    "sub.rn.f32 db, %4, vy1;\n" "fma.rn.f32 x, sl1, %4, ic1;\n" "sub.rn.f32 e, %2, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %4, vy2;\n" "fma.rn.f32 x, sl2, %4, ic2;\n" "sub.rn.f32 e, %2, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp0, %4, vy3;\n" "fma.rn.f32 x, sl3, %4, ic3;\n" "sub.rn.f32 e, %2, x;\n" "lop3.b32 t2, dp0, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %5, vy0;\n" "fma.rn.f32 x, sl0, %5, ic0;\n" "sub.rn.f32 e, %3, x;\n" "lop3.b32 t1, da, dp1, e, 0x28;\n" \
    "sub.rn.f32 db, %5, vy1;\n" "fma.rn.f32 x, sl1, %5, ic1;\n" "sub.rn.f32 e, %3, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %5, vy2;\n" "fma.rn.f32 x, sl2, %5, ic2;\n" "sub.rn.f32 e, %3, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp1, %5, vy3;\n" "fma.rn.f32 x, sl3, %5, ic3;\n" "sub.rn.f32 e, %3, x;\n" "lop3.b32 t2, dp1, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n"
#define S3_INIT "sub.rn.f32 dp0, %4, %8;\n" "sub.rn.f32 dp1, %5, %8;\n"
#define S3_REGS ".reg .b32 dp0, dp1, da, db, e, t1, t2;\n"
#define S3_BASE "6"
#define S3_SPAN "7"
#elif TILE == 4
#define S3_POINTS \
    "sub.rn.f32 da, %8, vy0;\n" "fma.rn.f32 x, sl0, %8, ic0;\n" "sub.rn.f32 e, %4, x;\n" "lop3.b32 t1, da, dp0, e, 0x28;\n" \
    "sub.rn.f32 db, %8, vy1;\n" "fma.rn.f32 x, sl1, %8, ic1;\n" "sub.rn.f32 e, %4, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %8, vy2;\n" "fma.rn.f32 x, sl2, %8, ic2;\n" "sub.rn.f32 e, %4, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp0, %8, vy3;\n" "fma.rn.f32 x, sl3, %8, ic3;\n" "sub.rn.f32 e, %4, x;\n" "lop3.b32 t2, dp0, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %9, vy0;\n" "fma.rn.f32 x, sl0, %9, ic0;\n" "sub.rn.f32 e, %5, x;\n" "lop3.b32 t1, da, dp1, e, 0x28;\n" \
    "sub.rn.f32 db, %9, vy1;\n" "fma.rn.f32 x, sl1, %9, ic1;\n" "sub.rn.f32 e, %5, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %9, vy2;\n" "fma.rn.f32 x, sl2, %9, ic2;\n" "sub.rn.f32 e, %5, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp1, %9, vy3;\n" "fma.rn.f32 x, sl3, %9, ic3;\n" "sub.rn.f32 e, %5, x;\n" "lop3.b32 t2, dp1, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %10, vy0;\n" "fma.rn.f32 x, sl0, %10, ic0;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t1, da, dp2, e, 0x28;\n" \
    "sub.rn.f32 db, %10, vy1;\n" "fma.rn.f32 x, sl1, %10, ic1;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %2, %2, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %10, vy2;\n" "fma.rn.f32 x, sl2, %10, ic2;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp2, %10, vy3;\n" "fma.rn.f32 x, sl3, %10, ic3;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t2, dp2, da, e, 0x28;\n" \
    "lop3.b32 %2, %2, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %11, vy0;\n" "fma.rn.f32 x, sl0, %11, ic0;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t1, da, dp3, e, 0x28;\n" \
    "sub.rn.f32 db, %11, vy1;\n" "fma.rn.f32 x, sl1, %11, ic1;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %3, %3, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %11, vy2;\n" "fma.rn.f32 x, sl2, %11, ic2;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp3, %11, vy3;\n" "fma.rn.f32 x, sl3, %11, ic3;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t2, dp3, da, e, 0x28;\n" \
    "lop3.b32 %3, %3, t1, t2, 0x96;\n"
#define S3_INIT "sub.rn.f32 dp0, %8, %14;\n" "sub.rn.f32 dp1, %9, %14;\n" "sub.rn.f32 dp2, %10, %14;\n" "sub.rn.f32 dp3, %11, %14;\n"
#define S3_REGS ".reg .b32 dp0, dp1, dp2, dp3, da, db, e, t1, t2;\n"
#define S3_BASE "12"
#define S3_SPAN "13"
#elif TILE == 6
#define S3_POINTS \
    "sub.rn.f32 da, %12, vy0;\n" "fma.rn.f32 x, sl0, %12, ic0;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t1, da, dp0, e, 0x28;\n" \
    "sub.rn.f32 db, %12, vy1;\n" "fma.rn.f32 x, sl1, %12, ic1;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %12, vy2;\n" "fma.rn.f32 x, sl2, %12, ic2;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp0, %12, vy3;\n" "fma.rn.f32 x, sl3, %12, ic3;\n" "sub.rn.f32 e, %6, x;\n" "lop3.b32 t2, dp0, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %13, vy0;\n" "fma.rn.f32 x, sl0, %13, ic0;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t1, da, dp1, e, 0x28;\n" \
    "sub.rn.f32 db, %13, vy1;\n" "fma.rn.f32 x, sl1, %13, ic1;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %13, vy2;\n" "fma.rn.f32 x, sl2, %13, ic2;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp1, %13, vy3;\n" "fma.rn.f32 x, sl3, %13, ic3;\n" "sub.rn.f32 e, %7, x;\n" "lop3.b32 t2, dp1, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %14, vy0;\n" "fma.rn.f32 x, sl0, %14, ic0;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t1, da, dp2, e, 0x28;\n" \
    "sub.rn.f32 db, %14, vy1;\n" "fma.rn.f32 x, sl1, %14, ic1;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %2, %2, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %14, vy2;\n" "fma.rn.f32 x, sl2, %14, ic2;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp2, %14, vy3;\n" "fma.rn.f32 x, sl3, %14, ic3;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t2, dp2, da, e, 0x28;\n" \
    "lop3.b32 %2, %2, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %15, vy0;\n" "fma.rn.f32 x, sl0, %15, ic0;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t1, da, dp3, e, 0x28;\n" \
    "sub.rn.f32 db, %15, vy1;\n" "fma.rn.f32 x, sl1, %15, ic1;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %3, %3, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %15, vy2;\n" "fma.rn.f32 x, sl2, %15, ic2;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp3, %15, vy3;\n" "fma.rn.f32 x, sl3, %15, ic3;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t2, dp3, da, e, 0x28;\n" \
    "lop3.b32 %3, %3, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %16, vy0;\n" "fma.rn.f32 x, sl0, %16, ic0;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t1, da, dp4, e, 0x28;\n" \
    "sub.rn.f32 db, %16, vy1;\n" "fma.rn.f32 x, sl1, %16, ic1;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %4, %4, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %16, vy2;\n" "fma.rn.f32 x, sl2, %16, ic2;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp4, %16, vy3;\n" "fma.rn.f32 x, sl3, %16, ic3;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t2, dp4, da, e, 0x28;\n" \
    "lop3.b32 %4, %4, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %17, vy0;\n" "fma.rn.f32 x, sl0, %17, ic0;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t1, da, dp5, e, 0x28;\n" \
    "sub.rn.f32 db, %17, vy1;\n" "fma.rn.f32 x, sl1, %17, ic1;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %5, %5, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %17, vy2;\n" "fma.rn.f32 x, sl2, %17, ic2;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp5, %17, vy3;\n" "fma.rn.f32 x, sl3, %17, ic3;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t2, dp5, da, e, 0x28;\n" \
    "lop3.b32 %5, %5, t1, t2, 0x96;\n"
#define S3_INIT "sub.rn.f32 dp0, %12, %20;\n" "sub.rn.f32 dp1, %13, %20;\n" "sub.rn.f32 dp2, %14, %20;\n" "sub.rn.f32 dp3, %15, %20;\n" "sub.rn.f32 dp4, %16, %20;\n" "sub.rn.f32 dp5, %17, %20;\n"
#define S3_REGS ".reg .b32 dp0, dp1, dp2, dp3, dp4, dp5, da, db, e, t1, t2;\n"
#define S3_BASE "18"
#define S3_SPAN "19"
#elif TILE == 8
#define S3_POINTS \
    "sub.rn.f32 da, %16, vy0;\n" "fma.rn.f32 x, sl0, %16, ic0;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t1, da, dp0, e, 0x28;\n" \
    "sub.rn.f32 db, %16, vy1;\n" "fma.rn.f32 x, sl1, %16, ic1;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %16, vy2;\n" "fma.rn.f32 x, sl2, %16, ic2;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp0, %16, vy3;\n" "fma.rn.f32 x, sl3, %16, ic3;\n" "sub.rn.f32 e, %8, x;\n" "lop3.b32 t2, dp0, da, e, 0x28;\n" \
    "lop3.b32 %0, %0, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %17, vy0;\n" "fma.rn.f32 x, sl0, %17, ic0;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t1, da, dp1, e, 0x28;\n" \
    "sub.rn.f32 db, %17, vy1;\n" "fma.rn.f32 x, sl1, %17, ic1;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %17, vy2;\n" "fma.rn.f32 x, sl2, %17, ic2;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp1, %17, vy3;\n" "fma.rn.f32 x, sl3, %17, ic3;\n" "sub.rn.f32 e, %9, x;\n" "lop3.b32 t2, dp1, da, e, 0x28;\n" \
    "lop3.b32 %1, %1, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %18, vy0;\n" "fma.rn.f32 x, sl0, %18, ic0;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t1, da, dp2, e, 0x28;\n" \
    "sub.rn.f32 db, %18, vy1;\n" "fma.rn.f32 x, sl1, %18, ic1;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %2, %2, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %18, vy2;\n" "fma.rn.f32 x, sl2, %18, ic2;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp2, %18, vy3;\n" "fma.rn.f32 x, sl3, %18, ic3;\n" "sub.rn.f32 e, %10, x;\n" "lop3.b32 t2, dp2, da, e, 0x28;\n" \
    "lop3.b32 %2, %2, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %19, vy0;\n" "fma.rn.f32 x, sl0, %19, ic0;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t1, da, dp3, e, 0x28;\n" \
    "sub.rn.f32 db, %19, vy1;\n" "fma.rn.f32 x, sl1, %19, ic1;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %3, %3, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %19, vy2;\n" "fma.rn.f32 x, sl2, %19, ic2;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp3, %19, vy3;\n" "fma.rn.f32 x, sl3, %19, ic3;\n" "sub.rn.f32 e, %11, x;\n" "lop3.b32 t2, dp3, da, e, 0x28;\n" \
    "lop3.b32 %3, %3, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %20, vy0;\n" "fma.rn.f32 x, sl0, %20, ic0;\n" "sub.rn.f32 e, %12, x;\n" "lop3.b32 t1, da, dp4, e, 0x28;\n" \
    "sub.rn.f32 db, %20, vy1;\n" "fma.rn.f32 x, sl1, %20, ic1;\n" "sub.rn.f32 e, %12, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %4, %4, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %20, vy2;\n" "fma.rn.f32 x, sl2, %20, ic2;\n" "sub.rn.f32 e, %12, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp4, %20, vy3;\n" "fma.rn.f32 x, sl3, %20, ic3;\n" "sub.rn.f32 e, %12, x;\n" "lop3.b32 t2, dp4, da, e, 0x28;\n" \
    "lop3.b32 %4, %4, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %21, vy0;\n" "fma.rn.f32 x, sl0, %21, ic0;\n" "sub.rn.f32 e, %13, x;\n" "lop3.b32 t1, da, dp5, e, 0x28;\n" \
    "sub.rn.f32 db, %21, vy1;\n" "fma.rn.f32 x, sl1, %21, ic1;\n" "sub.rn.f32 e, %13, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %5, %5, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %21, vy2;\n" "fma.rn.f32 x, sl2, %21, ic2;\n" "sub.rn.f32 e, %13, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp5, %21, vy3;\n" "fma.rn.f32 x, sl3, %21, ic3;\n" "sub.rn.f32 e, %13, x;\n" "lop3.b32 t2, dp5, da, e, 0x28;\n" \
    "lop3.b32 %5, %5, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %22, vy0;\n" "fma.rn.f32 x, sl0, %22, ic0;\n" "sub.rn.f32 e, %14, x;\n" "lop3.b32 t1, da, dp6, e, 0x28;\n" \
    "sub.rn.f32 db, %22, vy1;\n" "fma.rn.f32 x, sl1, %22, ic1;\n" "sub.rn.f32 e, %14, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %6, %6, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %22, vy2;\n" "fma.rn.f32 x, sl2, %22, ic2;\n" "sub.rn.f32 e, %14, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp6, %22, vy3;\n" "fma.rn.f32 x, sl3, %22, ic3;\n" "sub.rn.f32 e, %14, x;\n" "lop3.b32 t2, dp6, da, e, 0x28;\n" \
    "lop3.b32 %6, %6, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %23, vy0;\n" "fma.rn.f32 x, sl0, %23, ic0;\n" "sub.rn.f32 e, %15, x;\n" "lop3.b32 t1, da, dp7, e, 0x28;\n" \
    "sub.rn.f32 db, %23, vy1;\n" "fma.rn.f32 x, sl1, %23, ic1;\n" "sub.rn.f32 e, %15, x;\n" "lop3.b32 t2, db, da, e, 0x28;\n" \
    "lop3.b32 %7, %7, t1, t2, 0x96;\n" \
    "sub.rn.f32 da, %23, vy2;\n" "fma.rn.f32 x, sl2, %23, ic2;\n" "sub.rn.f32 e, %15, x;\n" "lop3.b32 t1, da, db, e, 0x28;\n" \
    "sub.rn.f32 dp7, %23, vy3;\n" "fma.rn.f32 x, sl3, %23, ic3;\n" "sub.rn.f32 e, %15, x;\n" "lop3.b32 t2, dp7, da, e, 0x28;\n" \
    "lop3.b32 %7, %7, t1, t2, 0x96;\n"
#define S3_INIT "sub.rn.f32 dp0, %16, %26;\n" "sub.rn.f32 dp1, %17, %26;\n" "sub.rn.f32 dp2, %18, %26;\n" "sub.rn.f32 dp3, %19, %26;\n" "sub.rn.f32 dp4, %20, %26;\n" "sub.rn.f32 dp5, %21, %26;\n" "sub.rn.f32 dp6, %22, %26;\n" "sub.rn.f32 dp7, %23, %26;\n"
#define S3_REGS ".reg .b32 dp0, dp1, dp2, dp3, dp4, dp5, dp6, dp7, da, db, e, t1, t2;\n"
#define S3_BASE "24"
#define S3_SPAN "25"
#endif
#define S3_LD "ld.shared.v4.f32 {vy0, sl0, ic0, z}, [ptr+0];\n" "ld.shared.v4.f32 {vy1, sl1, ic1, z}, [ptr+16];\n" \
              "ld.shared.v4.f32 {vy2, sl2, ic2, z}, [ptr+32];\n" "ld.shared.v4.f32 {vy3, sl3, ic3, z}, [ptr+48];\n"
#define S3_ASM                                                                                     \
    "{\n" S3_REGS ".reg .f32 vy0, vy1, vy2, vy3, sl0, sl1, sl2, sl3, ic0, ic1, ic2, ic3, x, z;\n"  \
    ".reg .u32 ptr, end;\n.reg .pred s;\n" S3_INIT "mov.u32 ptr, %" S3_BASE ";\n"                  \
    "add.u32 end, ptr, %" S3_SPAN ";\n" "PNPOLY_S3_LOOP:\n" S3_LD S3_POINTS                        \
    "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_S3_LOOP;\n}\n"
#endif
#if ASM == 4
// paired variant of ASM 3: two points share every FP32 instruction through
// Blackwell's packed f32x2 ops (FADD2 / FFMA2, each lane IEEE .rn, no ftz),
// halving FMA-pipe issue; the sign-bit LOP3s stay per point on the ALU pipe.
#if TILE == 4
#define S4_REGS ".reg .b64 pxq0, pyq0, pxq1, pyq1, zz;\n.reg .u32 zr;\n.reg .b64 vy2, sl2, ic2, x2, e2, dp0, dA0, dB0, dp1, dA1, dB1;\n" \
    ".reg .b32 lo0, hi0, lo1, hi1, lo2, hi2, t0a, t0b, t1a, t1b, t2a, t2b, t3a, t3b;\n" \
    ".reg .f32 vy, sl, ic, z, vyl;\n"
#define S4_INIT "mov.u32 zr, %%tid.y;\n" "cvt.u64.u32 zz, zr;\n" \
    "xor.b64 pxq0, %4, zz;\n" \
    "xor.b64 pyq0, %6, zz;\n" \
    "xor.b64 pxq1, %5, zz;\n" \
    "xor.b64 pyq1, %7, zz;\n" \
    "mov.b32 vyl, %10;\n" \
    "mov.b64 vy2, {vyl, vyl};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n"
#define S4_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dA0;\n" \
    "mov.b64 {lo1, hi1}, dp0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dA1;\n" \
    "mov.b64 {lo1, hi1}, dp1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3a, hi0, hi1, hi2, 0x28;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dB0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dB0;\n" \
    "mov.b64 {lo1, hi1}, dA0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %0, %0, t0a, t0b, 0x96;\n" \
    "lop3.b32 %1, %1, t1a, t1b, 0x96;\n" \
    "sub.rn.f32x2 dB1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dB1;\n" \
    "mov.b64 {lo1, hi1}, dA1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %2, %2, t2a, t2b, 0x96;\n" \
    "lop3.b32 %3, %3, t3a, t3b, 0x96;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dA0;\n" \
    "mov.b64 {lo1, hi1}, dB0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dA1;\n" \
    "mov.b64 {lo1, hi1}, dB1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3a, hi0, hi1, hi2, 0x28;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dp0;\n" \
    "mov.b64 {lo1, hi1}, dA0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %0, %0, t0a, t0b, 0x96;\n" \
    "lop3.b32 %1, %1, t1a, t1b, 0x96;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dp1;\n" \
    "mov.b64 {lo1, hi1}, dA1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %2, %2, t2a, t2b, 0x96;\n" \
    "lop3.b32 %3, %3, t3a, t3b, 0x96;\n"
#define S4_BASE "8"
#define S4_SPAN "9"
#elif TILE == 8
#define S4_REGS ".reg .b64 pxq0, pyq0, pxq1, pyq1, pxq2, pyq2, pxq3, pyq3, zz;\n.reg .u32 zr;\n.reg .b64 vy2, sl2, ic2, x2, e2, dp0, dA0, dB0, dp1, dA1, dB1, dp2, dA2, dB2, dp3, dA3, dB3;\n" \
    ".reg .b32 lo0, hi0, lo1, hi1, lo2, hi2, t0a, t0b, t1a, t1b, t2a, t2b, t3a, t3b, t4a, t4b, t5a, t5b, t6a, t6b, t7a, t7b;\n" \
    ".reg .f32 vy, sl, ic, z, vyl;\n"
#define S4_INIT "mov.u32 zr, %%tid.y;\n" "cvt.u64.u32 zz, zr;\n" \
    "xor.b64 pxq0, %8, zz;\n" \
    "xor.b64 pyq0, %12, zz;\n" \
    "xor.b64 pxq1, %9, zz;\n" \
    "xor.b64 pyq1, %13, zz;\n" \
    "xor.b64 pxq2, %10, zz;\n" \
    "xor.b64 pyq2, %14, zz;\n" \
    "xor.b64 pxq3, %11, zz;\n" \
    "xor.b64 pyq3, %15, zz;\n" \
    "mov.b32 vyl, %18;\n" \
    "mov.b64 vy2, {vyl, vyl};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n" \
    "sub.rn.f32x2 dp2, pyq2, vy2;\n" \
    "sub.rn.f32x2 dp3, pyq3, vy2;\n"
#define S4_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dA0;\n" \
    "mov.b64 {lo1, hi1}, dp0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dA1;\n" \
    "mov.b64 {lo1, hi1}, dp1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA2, pyq2, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq2, ic2;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {lo0, hi0}, dA2;\n" \
    "mov.b64 {lo1, hi1}, dp2;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t4a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t5a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA3, pyq3, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq3, ic2;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {lo0, hi0}, dA3;\n" \
    "mov.b64 {lo1, hi1}, dp3;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t6a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t7a, hi0, hi1, hi2, 0x28;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dB0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dB0;\n" \
    "mov.b64 {lo1, hi1}, dA0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %0, %0, t0a, t0b, 0x96;\n" \
    "lop3.b32 %1, %1, t1a, t1b, 0x96;\n" \
    "sub.rn.f32x2 dB1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dB1;\n" \
    "mov.b64 {lo1, hi1}, dA1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %2, %2, t2a, t2b, 0x96;\n" \
    "lop3.b32 %3, %3, t3a, t3b, 0x96;\n" \
    "sub.rn.f32x2 dB2, pyq2, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq2, ic2;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {lo0, hi0}, dB2;\n" \
    "mov.b64 {lo1, hi1}, dA2;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t4b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t5b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %4, %4, t4a, t4b, 0x96;\n" \
    "lop3.b32 %5, %5, t5a, t5b, 0x96;\n" \
    "sub.rn.f32x2 dB3, pyq3, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq3, ic2;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {lo0, hi0}, dB3;\n" \
    "mov.b64 {lo1, hi1}, dA3;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t6b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t7b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %6, %6, t6a, t6b, 0x96;\n" \
    "lop3.b32 %7, %7, t7a, t7b, 0x96;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dA0;\n" \
    "mov.b64 {lo1, hi1}, dB0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dA1;\n" \
    "mov.b64 {lo1, hi1}, dB1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA2, pyq2, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq2, ic2;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {lo0, hi0}, dA2;\n" \
    "mov.b64 {lo1, hi1}, dB2;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t4a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t5a, hi0, hi1, hi2, 0x28;\n" \
    "sub.rn.f32x2 dA3, pyq3, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq3, ic2;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {lo0, hi0}, dA3;\n" \
    "mov.b64 {lo1, hi1}, dB3;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t6a, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t7a, hi0, hi1, hi2, 0x28;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2, {sl, sl};\n" \
    "mov.b64 ic2, {ic, ic};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq0, ic2;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {lo0, hi0}, dp0;\n" \
    "mov.b64 {lo1, hi1}, dA0;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t0b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t1b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %0, %0, t0a, t0b, 0x96;\n" \
    "lop3.b32 %1, %1, t1a, t1b, 0x96;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq1, ic2;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {lo0, hi0}, dp1;\n" \
    "mov.b64 {lo1, hi1}, dA1;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t2b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t3b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %2, %2, t2a, t2b, 0x96;\n" \
    "lop3.b32 %3, %3, t3a, t3b, 0x96;\n" \
    "sub.rn.f32x2 dp2, pyq2, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq2, ic2;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {lo0, hi0}, dp2;\n" \
    "mov.b64 {lo1, hi1}, dA2;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t4b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t5b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %4, %4, t4a, t4b, 0x96;\n" \
    "lop3.b32 %5, %5, t5a, t5b, 0x96;\n" \
    "sub.rn.f32x2 dp3, pyq3, vy2;\n" \
    "fma.rn.f32x2 x2, sl2, pyq3, ic2;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {lo0, hi0}, dp3;\n" \
    "mov.b64 {lo1, hi1}, dA3;\n" \
    "mov.b64 {lo2, hi2}, e2;\n" \
    "lop3.b32 t6b, lo0, lo1, lo2, 0x28;\n" \
    "lop3.b32 t7b, hi0, hi1, hi2, 0x28;\n" \
    "lop3.b32 %6, %6, t6a, t6b, 0x96;\n" \
    "lop3.b32 %7, %7, t7a, t7b, 0x96;\n"
#define S4_BASE "16"
#define S4_SPAN "17"
#endif
#define S4_ASM                                                                         \
    "{\n" S4_REGS ".reg .u32 ptr, end;\n.reg .pred s;\n" S4_INIT                       \
    "mov.u32 ptr, %" S4_BASE ";\nadd.u32 end, ptr, %" S4_SPAN ";\n" "PNPOLY_S4_LOOP:\n" \
    S4_BODY "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_S4_LOOP;\n}\n"
#endif
#if ASM == 7 || ASM == 9
// One 4-edge group for one point. vyA = {vy0, vy1}, vyB = {vy2, vy3} (same
// for sl / ic) come from LDS.64, so every f32x2 operand is an aligned pair;
// the point's px / py enter as broadcast scalars. PREV holds py - vy of the
// vertex before this group; LAST receives py - vy3 (chain to the next group).
// The six FMA-pipe ops of point t+1 are interleaved one-to-one with the six
// ALU LOP3s of point t (register set S = t % 2), so every warp's stream
// alternates pipes instead of bursting one pipe at a time. (Putting the
// vertex difference shared by consecutive edges in the same LOP3 operand slot
// lets ptxas set operand-reuse flags on 16 LOP3s; measured: no speed-up.)
#define S7_F1(S, PX, PY) "mov.b64 py2" S ", {%" PY ", %" PY "};\n" "mov.b64 px2" S ", {%" PX ", %" PX "};\n" \
                         "sub.rn.f32x2 dA" S ", py2" S ", vyA;\n"
#define S7_F2(S) "fma.rn.f32x2 xA" S ", slA, py2" S ", icA;\n"
#define S7_F3(S) "sub.rn.f32x2 eA" S ", px2" S ", xA" S ";\n"
#define S7_F4(S) "sub.rn.f32x2 dB" S ", py2" S ", vyB;\n"
#define S7_F5(S) "fma.rn.f32x2 xB" S ", slB, py2" S ", icB;\n"
#define S7_F6(S, LAST) "sub.rn.f32x2 eB" S ", px2" S ", xB" S ";\n"                                    \
    "mov.b64 {d0" S ", d1" S "}, dA" S ";\n" "mov.b64 {d2" S ", " LAST "}, dB" S ";\n"                   \
    "mov.b64 {e0" S ", e1" S "}, eA" S ";\n" "mov.b64 {e2" S ", e3" S "}, eB" S ";\n"
#define S7_L1(S, PREV) "lop3.b32 t0" S ", d0" S ", " PREV ", e0" S ", 0x28;\n"
#define S7_L2(S) "lop3.b32 t1" S ", d1" S ", d0" S ", e1" S ", 0x28;\n"
#define S7_L3(S, ACC) "lop3.b32 %" ACC ", %" ACC ", t0" S ", t1" S ", 0x96;\n"
#define S7_L4(S) "lop3.b32 t0" S ", d2" S ", d1" S ", e2" S ", 0x28;\n"
#define S7_L5(S, LAST) "lop3.b32 t1" S ", " LAST ", d2" S ", e3" S ", 0x28;\n"
#define S7_HEAD(S, PX, PY, LAST) S7_F1(S, PX, PY) S7_F2(S) S7_F3(S) S7_F4(S) S7_F5(S) S7_F6(S, LAST)
#define S7_TAIL(S, ACC, PREV, LAST) S7_L1(S, PREV) S7_L2(S) S7_L3(S, ACC) S7_L4(S) S7_L5(S, LAST) S7_L3(S, ACC)
#define S7_STEP(NS, NPX, NPY, NLAST, CS, CACC, CPREV, CLAST)                                         \
    S7_F1(NS, NPX, NPY) S7_L1(CS, CPREV) S7_F2(NS) S7_L2(CS) S7_F3(NS) S7_L3(CS, CACC)               \
    S7_F4(NS) S7_L4(CS) S7_F5(NS) S7_L5(CS, CLAST) S7_F6(NS, NLAST) S7_L3(CS, CACC)
#if ASM == 9
// register-bank-friendly table: {vy0..3}{sl0,sl1,ic2,ic3}{sl2,sl3,ic0,ic1}. A 128-bit load
// fills an aligned register quad, so slope and intercept pairs land in opposite halves of
// two quads and each FFMA2 (slope pair x py + intercept pair) reads its two pair operands
// from different register banks (ASM 7: both from the same half of their quads)
#define S7_LOAD(OFF)                                            \
    "ld.shared.v2.b64 {vyA, vyB}, [ptr+" OFF "];\n"             \
    "ld.shared.v2.b64 {slA, icB}, [ptr+" OFF "+16];\n"          \
    "ld.shared.v2.b64 {slB, icA}, [ptr+" OFF "+32];\n"
#else
#define S7_LOAD(OFF)                                            \
    "ld.shared.v2.b64 {vyA, vyB}, [ptr+" OFF "];\n"             \
    "ld.shared.v2.b64 {slA, slB}, [ptr+" OFF "+16];\n"          \
    "ld.shared.v2.b64 {icA, icB}, [ptr+" OFF "+32];\n"
#endif
#define S7_INIT1(I, PY, VL) "sub.rn.f32 dp" #I ", %" PY ", %" VL ";\n"
#if TILE == 2
#define S7_GROUP_P \
    S7_HEAD("0", "2", "4", "dq0") \
    S7_STEP("1", "3", "5", "dq1", "0", "0", "dp0", "dq0") \
    S7_TAIL("1", "1", "dp1", "dq1")
#define S7_GROUP_Q \
    S7_HEAD("0", "2", "4", "dp0") \
    S7_STEP("1", "3", "5", "dp1", "0", "0", "dq0", "dp0") \
    S7_TAIL("1", "1", "dq1", "dp1")
#define S7_INIT S7_INIT1(0, "4", "8") S7_INIT1(1, "5", "8")
#define S7_BASE "6"
#define S7_SPAN "7"
#elif TILE == 4
#define S7_GROUP_P \
    S7_HEAD("0", "4", "8", "dq0") \
    S7_STEP("1", "5", "9", "dq1", "0", "0", "dp0", "dq0") \
    S7_STEP("0", "6", "10", "dq2", "1", "1", "dp1", "dq1") \
    S7_STEP("1", "7", "11", "dq3", "0", "2", "dp2", "dq2") \
    S7_TAIL("1", "3", "dp3", "dq3")
#define S7_GROUP_Q \
    S7_HEAD("0", "4", "8", "dp0") \
    S7_STEP("1", "5", "9", "dp1", "0", "0", "dq0", "dp0") \
    S7_STEP("0", "6", "10", "dp2", "1", "1", "dq1", "dp1") \
    S7_STEP("1", "7", "11", "dp3", "0", "2", "dq2", "dp2") \
    S7_TAIL("1", "3", "dq3", "dp3")
#define S7_INIT S7_INIT1(0, "8", "14") S7_INIT1(1, "9", "14") S7_INIT1(2, "10", "14") S7_INIT1(3, "11", "14")
#define S7_BASE "12"
#define S7_SPAN "13"
#elif TILE == 6
#define S7_GROUP_P \
    S7_HEAD("0", "6", "12", "dq0") \
    S7_STEP("1", "7", "13", "dq1", "0", "0", "dp0", "dq0") \
    S7_STEP("0", "8", "14", "dq2", "1", "1", "dp1", "dq1") \
    S7_STEP("1", "9", "15", "dq3", "0", "2", "dp2", "dq2") \
    S7_STEP("0", "10", "16", "dq4", "1", "3", "dp3", "dq3") \
    S7_STEP("1", "11", "17", "dq5", "0", "4", "dp4", "dq4") \
    S7_TAIL("1", "5", "dp5", "dq5")
#define S7_GROUP_Q \
    S7_HEAD("0", "6", "12", "dp0") \
    S7_STEP("1", "7", "13", "dp1", "0", "0", "dq0", "dp0") \
    S7_STEP("0", "8", "14", "dp2", "1", "1", "dq1", "dp1") \
    S7_STEP("1", "9", "15", "dp3", "0", "2", "dq2", "dp2") \
    S7_STEP("0", "10", "16", "dp4", "1", "3", "dq3", "dp3") \
    S7_STEP("1", "11", "17", "dp5", "0", "4", "dq4", "dp4") \
    S7_TAIL("1", "5", "dq5", "dp5")
#define S7_INIT S7_INIT1(0, "12", "20") S7_INIT1(1, "13", "20") S7_INIT1(2, "14", "20") S7_INIT1(3, "15", "20") S7_INIT1(4, "16", "20") S7_INIT1(5, "17", "20")
#define S7_BASE "18"
#define S7_SPAN "19"
#elif TILE == 8
#define S7_GROUP_P \
    S7_HEAD("0", "8", "16", "dq0") \
    S7_STEP("1", "9", "17", "dq1", "0", "0", "dp0", "dq0") \
    S7_STEP("0", "10", "18", "dq2", "1", "1", "dp1", "dq1") \
    S7_STEP("1", "11", "19", "dq3", "0", "2", "dp2", "dq2") \
    S7_STEP("0", "12", "20", "dq4", "1", "3", "dp3", "dq3") \
    S7_STEP("1", "13", "21", "dq5", "0", "4", "dp4", "dq4") \
    S7_STEP("0", "14", "22", "dq6", "1", "5", "dp5", "dq5") \
    S7_STEP("1", "15", "23", "dq7", "0", "6", "dp6", "dq6") \
    S7_TAIL("1", "7", "dp7", "dq7")
#define S7_GROUP_Q \
    S7_HEAD("0", "8", "16", "dp0") \
    S7_STEP("1", "9", "17", "dp1", "0", "0", "dq0", "dp0") \
    S7_STEP("0", "10", "18", "dp2", "1", "1", "dq1", "dp1") \
    S7_STEP("1", "11", "19", "dp3", "0", "2", "dq2", "dp2") \
    S7_STEP("0", "12", "20", "dp4", "1", "3", "dq3", "dp3") \
    S7_STEP("1", "13", "21", "dp5", "0", "4", "dq4", "dp4") \
    S7_STEP("0", "14", "22", "dp6", "1", "5", "dq5", "dp5") \
    S7_STEP("1", "15", "23", "dp7", "0", "6", "dq6", "dp6") \
    S7_TAIL("1", "7", "dq7", "dp7")
#define S7_INIT S7_INIT1(0, "16", "26") S7_INIT1(1, "17", "26") S7_INIT1(2, "18", "26") S7_INIT1(3, "19", "26") S7_INIT1(4, "20", "26") S7_INIT1(5, "21", "26") S7_INIT1(6, "22", "26") S7_INIT1(7, "23", "26")
#define S7_BASE "24"
#define S7_SPAN "25"
#endif
#define S7_SETS ".reg .b64 py20, px20, dA0, dB0, xA0, xB0, eA0, eB0;\n" ".reg .b32 d00, d10, d20, e00, e10, e20, e30, t00, t10;\n" ".reg .b64 py21, px21, dA1, dB1, xA1, xB1, eA1, eB1;\n" ".reg .b32 d01, d11, d21, e01, e11, e21, e31, t01, t11;\n" ".reg .b64 py22, px22, dA2, dB2, xA2, xB2, eA2, eB2;\n" ".reg .b32 d02, d12, d22, e02, e12, e22, e32, t02, t12;\n" ".reg .b64 py23, px23, dA3, dB3, xA3, xB3, eA3, eB3;\n" ".reg .b32 d03, d13, d23, e03, e13, e23, e33, t03, t13;\n" ".reg .b64 py24, px24, dA4, dB4, xA4, xB4, eA4, eB4;\n" ".reg .b32 d04, d14, d24, e04, e14, e24, e34, t04, t14;\n" ".reg .b64 py25, px25, dA5, dB5, xA5, xB5, eA5, eB5;\n" ".reg .b32 d05, d15, d25, e05, e15, e25, e35, t05, t15;\n" ".reg .b64 py26, px26, dA6, dB6, xA6, xB6, eA6, eB6;\n" ".reg .b32 d06, d16, d26, e06, e16, e26, e36, t06, t16;\n" ".reg .b64 py27, px27, dA7, dB7, xA7, xB7, eA7, eB7;\n" ".reg .b32 d07, d17, d27, e07, e17, e27, e37, t07, t17;\n" 
#define S7_ASM                                                                                   \
    "{\n"                                                                                        \
    ".reg .b64 vyA, vyB, slA, slB, icA, icB;\n"                                                 \
    S7_SETS                                                                                      \
    ".reg .b32 dp0, dp1, dp2, dp3, dp4, dp5, dp6, dp7, dq0, dq1, dq2, dq3, dq4, dq5, dq6, dq7;\n" \
    ".reg .u32 ptr, end;\n.reg .pred s;\n" S7_INIT                                               \
    "mov.u32 ptr, %" S7_BASE ";\nadd.u32 end, ptr, %" S7_SPAN ";\n"                              \
    "PNPOLY_S7_LOOP:\n" S7_LOAD("0") S7_GROUP_P S7_LOAD("48") S7_GROUP_Q                         \
    "add.u32 ptr, ptr, 96;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_S7_LOOP;\n}\n"
#endif
#if ASM == 5
// ASM 3 with the sign XOR of consecutive (py - vy) moved to the FMA pipe:
// sign(d_k * d_{k-1}) == sign(d_k) ^ sign(d_{k-1}) exactly (IEEE product
// sign), leaving one 3-input LOP3 per edge-point: acc ^= m & e.
#if TILE == 2
#define S5_REGS ".reg .b32 m, e, dp0, dA0, dB0, dp1, dA1, dB1;\n" \
    ".reg .f32 vy, sl, ic, z, x;\n"
#define S5_INIT "sub.rn.f32 dp0, %4, %8;\n" \
    "sub.rn.f32 dp1, %5, %8;\n"
#define S5_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "sub.rn.f32 dA0, %4, vy;\n" \
    "mul.rn.f32 m, dA0, dp0;\n" \
    "fma.rn.f32 x, sl, %4, ic;\n" \
    "sub.rn.f32 e, %2, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %5, vy;\n" \
    "mul.rn.f32 m, dA1, dp1;\n" \
    "fma.rn.f32 x, sl, %5, ic;\n" \
    "sub.rn.f32 e, %3, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "sub.rn.f32 dB0, %4, vy;\n" \
    "mul.rn.f32 m, dB0, dA0;\n" \
    "fma.rn.f32 x, sl, %4, ic;\n" \
    "sub.rn.f32 e, %2, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dB1, %5, vy;\n" \
    "mul.rn.f32 m, dB1, dA1;\n" \
    "fma.rn.f32 x, sl, %5, ic;\n" \
    "sub.rn.f32 e, %3, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "sub.rn.f32 dA0, %4, vy;\n" \
    "mul.rn.f32 m, dA0, dB0;\n" \
    "fma.rn.f32 x, sl, %4, ic;\n" \
    "sub.rn.f32 e, %2, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %5, vy;\n" \
    "mul.rn.f32 m, dA1, dB1;\n" \
    "fma.rn.f32 x, sl, %5, ic;\n" \
    "sub.rn.f32 e, %3, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "sub.rn.f32 dp0, %4, vy;\n" \
    "mul.rn.f32 m, dp0, dA0;\n" \
    "fma.rn.f32 x, sl, %4, ic;\n" \
    "sub.rn.f32 e, %2, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dp1, %5, vy;\n" \
    "mul.rn.f32 m, dp1, dA1;\n" \
    "fma.rn.f32 x, sl, %5, ic;\n" \
    "sub.rn.f32 e, %3, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n"
#define S5_BASE "6"
#define S5_SPAN "7"
#elif TILE == 4
#define S5_REGS ".reg .b32 m, e, dp0, dA0, dB0, dp1, dA1, dB1, dp2, dA2, dB2, dp3, dA3, dB3;\n" \
    ".reg .f32 vy, sl, ic, z, x;\n"
#define S5_INIT "sub.rn.f32 dp0, %8, %14;\n" \
    "sub.rn.f32 dp1, %9, %14;\n" \
    "sub.rn.f32 dp2, %10, %14;\n" \
    "sub.rn.f32 dp3, %11, %14;\n"
#define S5_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "sub.rn.f32 dA0, %8, vy;\n" \
    "mul.rn.f32 m, dA0, dp0;\n" \
    "fma.rn.f32 x, sl, %8, ic;\n" \
    "sub.rn.f32 e, %4, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %9, vy;\n" \
    "mul.rn.f32 m, dA1, dp1;\n" \
    "fma.rn.f32 x, sl, %9, ic;\n" \
    "sub.rn.f32 e, %5, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dA2, %10, vy;\n" \
    "mul.rn.f32 m, dA2, dp2;\n" \
    "fma.rn.f32 x, sl, %10, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dA3, %11, vy;\n" \
    "mul.rn.f32 m, dA3, dp3;\n" \
    "fma.rn.f32 x, sl, %11, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "sub.rn.f32 dB0, %8, vy;\n" \
    "mul.rn.f32 m, dB0, dA0;\n" \
    "fma.rn.f32 x, sl, %8, ic;\n" \
    "sub.rn.f32 e, %4, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dB1, %9, vy;\n" \
    "mul.rn.f32 m, dB1, dA1;\n" \
    "fma.rn.f32 x, sl, %9, ic;\n" \
    "sub.rn.f32 e, %5, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dB2, %10, vy;\n" \
    "mul.rn.f32 m, dB2, dA2;\n" \
    "fma.rn.f32 x, sl, %10, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dB3, %11, vy;\n" \
    "mul.rn.f32 m, dB3, dA3;\n" \
    "fma.rn.f32 x, sl, %11, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "sub.rn.f32 dA0, %8, vy;\n" \
    "mul.rn.f32 m, dA0, dB0;\n" \
    "fma.rn.f32 x, sl, %8, ic;\n" \
    "sub.rn.f32 e, %4, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %9, vy;\n" \
    "mul.rn.f32 m, dA1, dB1;\n" \
    "fma.rn.f32 x, sl, %9, ic;\n" \
    "sub.rn.f32 e, %5, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dA2, %10, vy;\n" \
    "mul.rn.f32 m, dA2, dB2;\n" \
    "fma.rn.f32 x, sl, %10, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dA3, %11, vy;\n" \
    "mul.rn.f32 m, dA3, dB3;\n" \
    "fma.rn.f32 x, sl, %11, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "sub.rn.f32 dp0, %8, vy;\n" \
    "mul.rn.f32 m, dp0, dA0;\n" \
    "fma.rn.f32 x, sl, %8, ic;\n" \
    "sub.rn.f32 e, %4, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dp1, %9, vy;\n" \
    "mul.rn.f32 m, dp1, dA1;\n" \
    "fma.rn.f32 x, sl, %9, ic;\n" \
    "sub.rn.f32 e, %5, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dp2, %10, vy;\n" \
    "mul.rn.f32 m, dp2, dA2;\n" \
    "fma.rn.f32 x, sl, %10, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dp3, %11, vy;\n" \
    "mul.rn.f32 m, dp3, dA3;\n" \
    "fma.rn.f32 x, sl, %11, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n"
#define S5_BASE "12"
#define S5_SPAN "13"
#elif TILE == 6
#define S5_REGS ".reg .b32 m, e, dp0, dA0, dB0, dp1, dA1, dB1, dp2, dA2, dB2, dp3, dA3, dB3, dp4, dA4, dB4, dp5, dA5, dB5;\n" \
    ".reg .f32 vy, sl, ic, z, x;\n"
#define S5_INIT "sub.rn.f32 dp0, %12, %20;\n" \
    "sub.rn.f32 dp1, %13, %20;\n" \
    "sub.rn.f32 dp2, %14, %20;\n" \
    "sub.rn.f32 dp3, %15, %20;\n" \
    "sub.rn.f32 dp4, %16, %20;\n" \
    "sub.rn.f32 dp5, %17, %20;\n"
#define S5_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "sub.rn.f32 dA0, %12, vy;\n" \
    "mul.rn.f32 m, dA0, dp0;\n" \
    "fma.rn.f32 x, sl, %12, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %13, vy;\n" \
    "mul.rn.f32 m, dA1, dp1;\n" \
    "fma.rn.f32 x, sl, %13, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dA2, %14, vy;\n" \
    "mul.rn.f32 m, dA2, dp2;\n" \
    "fma.rn.f32 x, sl, %14, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dA3, %15, vy;\n" \
    "mul.rn.f32 m, dA3, dp3;\n" \
    "fma.rn.f32 x, sl, %15, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dA4, %16, vy;\n" \
    "mul.rn.f32 m, dA4, dp4;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dA5, %17, vy;\n" \
    "mul.rn.f32 m, dA5, dp5;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "sub.rn.f32 dB0, %12, vy;\n" \
    "mul.rn.f32 m, dB0, dA0;\n" \
    "fma.rn.f32 x, sl, %12, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dB1, %13, vy;\n" \
    "mul.rn.f32 m, dB1, dA1;\n" \
    "fma.rn.f32 x, sl, %13, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dB2, %14, vy;\n" \
    "mul.rn.f32 m, dB2, dA2;\n" \
    "fma.rn.f32 x, sl, %14, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dB3, %15, vy;\n" \
    "mul.rn.f32 m, dB3, dA3;\n" \
    "fma.rn.f32 x, sl, %15, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dB4, %16, vy;\n" \
    "mul.rn.f32 m, dB4, dA4;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dB5, %17, vy;\n" \
    "mul.rn.f32 m, dB5, dA5;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "sub.rn.f32 dA0, %12, vy;\n" \
    "mul.rn.f32 m, dA0, dB0;\n" \
    "fma.rn.f32 x, sl, %12, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %13, vy;\n" \
    "mul.rn.f32 m, dA1, dB1;\n" \
    "fma.rn.f32 x, sl, %13, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dA2, %14, vy;\n" \
    "mul.rn.f32 m, dA2, dB2;\n" \
    "fma.rn.f32 x, sl, %14, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dA3, %15, vy;\n" \
    "mul.rn.f32 m, dA3, dB3;\n" \
    "fma.rn.f32 x, sl, %15, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dA4, %16, vy;\n" \
    "mul.rn.f32 m, dA4, dB4;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dA5, %17, vy;\n" \
    "mul.rn.f32 m, dA5, dB5;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "sub.rn.f32 dp0, %12, vy;\n" \
    "mul.rn.f32 m, dp0, dA0;\n" \
    "fma.rn.f32 x, sl, %12, ic;\n" \
    "sub.rn.f32 e, %6, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dp1, %13, vy;\n" \
    "mul.rn.f32 m, dp1, dA1;\n" \
    "fma.rn.f32 x, sl, %13, ic;\n" \
    "sub.rn.f32 e, %7, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dp2, %14, vy;\n" \
    "mul.rn.f32 m, dp2, dA2;\n" \
    "fma.rn.f32 x, sl, %14, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dp3, %15, vy;\n" \
    "mul.rn.f32 m, dp3, dA3;\n" \
    "fma.rn.f32 x, sl, %15, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dp4, %16, vy;\n" \
    "mul.rn.f32 m, dp4, dA4;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dp5, %17, vy;\n" \
    "mul.rn.f32 m, dp5, dA5;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n"
#define S5_BASE "18"
#define S5_SPAN "19"
#elif TILE == 8
#define S5_REGS ".reg .b32 m, e, dp0, dA0, dB0, dp1, dA1, dB1, dp2, dA2, dB2, dp3, dA3, dB3, dp4, dA4, dB4, dp5, dA5, dB5, dp6, dA6, dB6, dp7, dA7, dB7;\n" \
    ".reg .f32 vy, sl, ic, z, x;\n"
#define S5_INIT "sub.rn.f32 dp0, %16, %26;\n" \
    "sub.rn.f32 dp1, %17, %26;\n" \
    "sub.rn.f32 dp2, %18, %26;\n" \
    "sub.rn.f32 dp3, %19, %26;\n" \
    "sub.rn.f32 dp4, %20, %26;\n" \
    "sub.rn.f32 dp5, %21, %26;\n" \
    "sub.rn.f32 dp6, %22, %26;\n" \
    "sub.rn.f32 dp7, %23, %26;\n"
#define S5_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "sub.rn.f32 dA0, %16, vy;\n" \
    "mul.rn.f32 m, dA0, dp0;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %17, vy;\n" \
    "mul.rn.f32 m, dA1, dp1;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dA2, %18, vy;\n" \
    "mul.rn.f32 m, dA2, dp2;\n" \
    "fma.rn.f32 x, sl, %18, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dA3, %19, vy;\n" \
    "mul.rn.f32 m, dA3, dp3;\n" \
    "fma.rn.f32 x, sl, %19, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dA4, %20, vy;\n" \
    "mul.rn.f32 m, dA4, dp4;\n" \
    "fma.rn.f32 x, sl, %20, ic;\n" \
    "sub.rn.f32 e, %12, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dA5, %21, vy;\n" \
    "mul.rn.f32 m, dA5, dp5;\n" \
    "fma.rn.f32 x, sl, %21, ic;\n" \
    "sub.rn.f32 e, %13, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "sub.rn.f32 dA6, %22, vy;\n" \
    "mul.rn.f32 m, dA6, dp6;\n" \
    "fma.rn.f32 x, sl, %22, ic;\n" \
    "sub.rn.f32 e, %14, x;\n" \
    "lop3.b32 %6, %6, m, e, 0x78;\n" \
    "sub.rn.f32 dA7, %23, vy;\n" \
    "mul.rn.f32 m, dA7, dp7;\n" \
    "fma.rn.f32 x, sl, %23, ic;\n" \
    "sub.rn.f32 e, %15, x;\n" \
    "lop3.b32 %7, %7, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "sub.rn.f32 dB0, %16, vy;\n" \
    "mul.rn.f32 m, dB0, dA0;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dB1, %17, vy;\n" \
    "mul.rn.f32 m, dB1, dA1;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dB2, %18, vy;\n" \
    "mul.rn.f32 m, dB2, dA2;\n" \
    "fma.rn.f32 x, sl, %18, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dB3, %19, vy;\n" \
    "mul.rn.f32 m, dB3, dA3;\n" \
    "fma.rn.f32 x, sl, %19, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dB4, %20, vy;\n" \
    "mul.rn.f32 m, dB4, dA4;\n" \
    "fma.rn.f32 x, sl, %20, ic;\n" \
    "sub.rn.f32 e, %12, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dB5, %21, vy;\n" \
    "mul.rn.f32 m, dB5, dA5;\n" \
    "fma.rn.f32 x, sl, %21, ic;\n" \
    "sub.rn.f32 e, %13, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "sub.rn.f32 dB6, %22, vy;\n" \
    "mul.rn.f32 m, dB6, dA6;\n" \
    "fma.rn.f32 x, sl, %22, ic;\n" \
    "sub.rn.f32 e, %14, x;\n" \
    "lop3.b32 %6, %6, m, e, 0x78;\n" \
    "sub.rn.f32 dB7, %23, vy;\n" \
    "mul.rn.f32 m, dB7, dA7;\n" \
    "fma.rn.f32 x, sl, %23, ic;\n" \
    "sub.rn.f32 e, %15, x;\n" \
    "lop3.b32 %7, %7, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "sub.rn.f32 dA0, %16, vy;\n" \
    "mul.rn.f32 m, dA0, dB0;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dA1, %17, vy;\n" \
    "mul.rn.f32 m, dA1, dB1;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dA2, %18, vy;\n" \
    "mul.rn.f32 m, dA2, dB2;\n" \
    "fma.rn.f32 x, sl, %18, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dA3, %19, vy;\n" \
    "mul.rn.f32 m, dA3, dB3;\n" \
    "fma.rn.f32 x, sl, %19, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dA4, %20, vy;\n" \
    "mul.rn.f32 m, dA4, dB4;\n" \
    "fma.rn.f32 x, sl, %20, ic;\n" \
    "sub.rn.f32 e, %12, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dA5, %21, vy;\n" \
    "mul.rn.f32 m, dA5, dB5;\n" \
    "fma.rn.f32 x, sl, %21, ic;\n" \
    "sub.rn.f32 e, %13, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "sub.rn.f32 dA6, %22, vy;\n" \
    "mul.rn.f32 m, dA6, dB6;\n" \
    "fma.rn.f32 x, sl, %22, ic;\n" \
    "sub.rn.f32 e, %14, x;\n" \
    "lop3.b32 %6, %6, m, e, 0x78;\n" \
    "sub.rn.f32 dA7, %23, vy;\n" \
    "mul.rn.f32 m, dA7, dB7;\n" \
    "fma.rn.f32 x, sl, %23, ic;\n" \
    "sub.rn.f32 e, %15, x;\n" \
    "lop3.b32 %7, %7, m, e, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "sub.rn.f32 dp0, %16, vy;\n" \
    "mul.rn.f32 m, dp0, dA0;\n" \
    "fma.rn.f32 x, sl, %16, ic;\n" \
    "sub.rn.f32 e, %8, x;\n" \
    "lop3.b32 %0, %0, m, e, 0x78;\n" \
    "sub.rn.f32 dp1, %17, vy;\n" \
    "mul.rn.f32 m, dp1, dA1;\n" \
    "fma.rn.f32 x, sl, %17, ic;\n" \
    "sub.rn.f32 e, %9, x;\n" \
    "lop3.b32 %1, %1, m, e, 0x78;\n" \
    "sub.rn.f32 dp2, %18, vy;\n" \
    "mul.rn.f32 m, dp2, dA2;\n" \
    "fma.rn.f32 x, sl, %18, ic;\n" \
    "sub.rn.f32 e, %10, x;\n" \
    "lop3.b32 %2, %2, m, e, 0x78;\n" \
    "sub.rn.f32 dp3, %19, vy;\n" \
    "mul.rn.f32 m, dp3, dA3;\n" \
    "fma.rn.f32 x, sl, %19, ic;\n" \
    "sub.rn.f32 e, %11, x;\n" \
    "lop3.b32 %3, %3, m, e, 0x78;\n" \
    "sub.rn.f32 dp4, %20, vy;\n" \
    "mul.rn.f32 m, dp4, dA4;\n" \
    "fma.rn.f32 x, sl, %20, ic;\n" \
    "sub.rn.f32 e, %12, x;\n" \
    "lop3.b32 %4, %4, m, e, 0x78;\n" \
    "sub.rn.f32 dp5, %21, vy;\n" \
    "mul.rn.f32 m, dp5, dA5;\n" \
    "fma.rn.f32 x, sl, %21, ic;\n" \
    "sub.rn.f32 e, %13, x;\n" \
    "lop3.b32 %5, %5, m, e, 0x78;\n" \
    "sub.rn.f32 dp6, %22, vy;\n" \
    "mul.rn.f32 m, dp6, dA6;\n" \
    "fma.rn.f32 x, sl, %22, ic;\n" \
    "sub.rn.f32 e, %14, x;\n" \
    "lop3.b32 %6, %6, m, e, 0x78;\n" \
    "sub.rn.f32 dp7, %23, vy;\n" \
    "mul.rn.f32 m, dp7, dA7;\n" \
    "fma.rn.f32 x, sl, %23, ic;\n" \
    "sub.rn.f32 e, %15, x;\n" \
    "lop3.b32 %7, %7, m, e, 0x78;\n"
#define S5_BASE "24"
#define S5_SPAN "25"
#endif
#define S5_ASM                                                                              \
    "{\n" S5_REGS ".reg .u32 ptr, end;\n.reg .pred s;\n" S5_INIT "mov.u32 ptr, %" S5_BASE ";\n" \
    "add.u32 end, ptr, %" S5_SPAN ";\n" "PNPOLY_S5_LOOP:\n" S5_BODY                              \
    "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_S5_LOOP;\n}\n"
#endif
#if ASM == 6
// ASM 5 on point pairs with packed f32x2 (FADD2 / FMUL2 / FFMA2).
#if TILE == 4
#define S6_REGS ".reg .b64 pxq0, pyq0, pxq1, pyq1, zz;\n.reg .u32 zr;\n.reg .b64 sl2b, ic2b, vy2, m2, x2, e2, dp0, dA0, dB0, dp1, dA1, dB1;\n" \
    ".reg .b32 mlo, mhi, elo, ehi;\n" \
    ".reg .f32 vy, sl, ic, z, vyl;\n"
#define S6_INIT "mov.u32 zr, %%tid.y;\n" "cvt.u64.u32 zz, zr;\n" \
    "xor.b64 pxq0, %4, zz;\n" \
    "xor.b64 pyq0, %6, zz;\n" \
    "xor.b64 pxq1, %5, zz;\n" \
    "xor.b64 pyq1, %7, zz;\n" \
    "mov.b32 vyl, %10;\n" \
    "mov.b64 vy2, {vyl, vyl};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n"
#define S6_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dA0, dp0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dA1, dp1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dB0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dB0, dA0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dB1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dB1, dA1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dA0, dB0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dA1, dB1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dp0, dA0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dp1, dA1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n"
#define S6_BASE "8"
#define S6_SPAN "9"
#elif TILE == 8
#define S6_REGS ".reg .b64 pxq0, pyq0, pxq1, pyq1, pxq2, pyq2, pxq3, pyq3, zz;\n.reg .u32 zr;\n.reg .b64 sl2b, ic2b, vy2, m2, x2, e2, dp0, dA0, dB0, dp1, dA1, dB1, dp2, dA2, dB2, dp3, dA3, dB3;\n" \
    ".reg .b32 mlo, mhi, elo, ehi;\n" \
    ".reg .f32 vy, sl, ic, z, vyl;\n"
#define S6_INIT "mov.u32 zr, %%tid.y;\n" "cvt.u64.u32 zz, zr;\n" \
    "xor.b64 pxq0, %8, zz;\n" \
    "xor.b64 pyq0, %12, zz;\n" \
    "xor.b64 pxq1, %9, zz;\n" \
    "xor.b64 pyq1, %13, zz;\n" \
    "xor.b64 pxq2, %10, zz;\n" \
    "xor.b64 pyq2, %14, zz;\n" \
    "xor.b64 pxq3, %11, zz;\n" \
    "xor.b64 pyq3, %15, zz;\n" \
    "mov.b32 vyl, %18;\n" \
    "mov.b64 vy2, {vyl, vyl};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n" \
    "sub.rn.f32x2 dp2, pyq2, vy2;\n" \
    "sub.rn.f32x2 dp3, pyq3, vy2;\n"
#define S6_BODY \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+0];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dA0, dp0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dA1, dp1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA2, pyq2, vy2;\n" \
    "mul.rn.f32x2 m2, dA2, dp2;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq2, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %4, %4, mlo, elo, 0x78;\n" \
    "lop3.b32 %5, %5, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA3, pyq3, vy2;\n" \
    "mul.rn.f32x2 m2, dA3, dp3;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq3, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %6, %6, mlo, elo, 0x78;\n" \
    "lop3.b32 %7, %7, mhi, ehi, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+16];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dB0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dB0, dA0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dB1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dB1, dA1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dB2, pyq2, vy2;\n" \
    "mul.rn.f32x2 m2, dB2, dA2;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq2, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %4, %4, mlo, elo, 0x78;\n" \
    "lop3.b32 %5, %5, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dB3, pyq3, vy2;\n" \
    "mul.rn.f32x2 m2, dB3, dA3;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq3, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %6, %6, mlo, elo, 0x78;\n" \
    "lop3.b32 %7, %7, mhi, ehi, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+32];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dA0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dA0, dB0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dA1, dB1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA2, pyq2, vy2;\n" \
    "mul.rn.f32x2 m2, dA2, dB2;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq2, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %4, %4, mlo, elo, 0x78;\n" \
    "lop3.b32 %5, %5, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dA3, pyq3, vy2;\n" \
    "mul.rn.f32x2 m2, dA3, dB3;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq3, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %6, %6, mlo, elo, 0x78;\n" \
    "lop3.b32 %7, %7, mhi, ehi, 0x78;\n" \
    "ld.shared.v4.f32 {vy, sl, ic, z}, [ptr+48];\n" \
    "mov.b64 vy2, {vy, vy};\n" \
    "mov.b64 sl2b, {sl, sl};\n" \
    "mov.b64 ic2b, {ic, ic};\n" \
    "sub.rn.f32x2 dp0, pyq0, vy2;\n" \
    "mul.rn.f32x2 m2, dp0, dA0;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq0, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq0, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %0, %0, mlo, elo, 0x78;\n" \
    "lop3.b32 %1, %1, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dp1, pyq1, vy2;\n" \
    "mul.rn.f32x2 m2, dp1, dA1;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq1, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq1, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %2, %2, mlo, elo, 0x78;\n" \
    "lop3.b32 %3, %3, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dp2, pyq2, vy2;\n" \
    "mul.rn.f32x2 m2, dp2, dA2;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq2, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq2, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %4, %4, mlo, elo, 0x78;\n" \
    "lop3.b32 %5, %5, mhi, ehi, 0x78;\n" \
    "sub.rn.f32x2 dp3, pyq3, vy2;\n" \
    "mul.rn.f32x2 m2, dp3, dA3;\n" \
    "fma.rn.f32x2 x2, sl2b, pyq3, ic2b;\n" \
    "sub.rn.f32x2 e2, pxq3, x2;\n" \
    "mov.b64 {mlo, mhi}, m2;\n" \
    "mov.b64 {elo, ehi}, e2;\n" \
    "lop3.b32 %6, %6, mlo, elo, 0x78;\n" \
    "lop3.b32 %7, %7, mhi, ehi, 0x78;\n"
#define S6_BASE "16"
#define S6_SPAN "17"
#endif
#define S6_ASM                                                                              \
    "{\n" S6_REGS ".reg .u32 ptr, end;\n.reg .pred s;\n" S6_INIT "mov.u32 ptr, %" S6_BASE ";\n" \
    "add.u32 end, ptr, %" S6_SPAN ";\n" "PNPOLY_S6_LOOP:\n" S6_BODY                              \
    "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_S6_LOOP;\n}\n"
#endif


__constant__ float4 c_edges[VERTICES];
__constant__ float2 c_ybounds[VERTICES];
#if ASM == 8
// the ASM 7 pair table: per 4-edge group {vy0..3}, {sl0..3}, {ic0..3}
__constant__ ulonglong2 c_pairs[TAB_VEC4];

// {a, a} - b and s * {a, a} + c on packed f32x2 lanes (IEEE .rn per lane, no ftz)
__device__ __forceinline__ unsigned long long f2_sub_bcast(float a, unsigned long long b) {
    unsigned long long r;
    asm("{\n.reg .b64 aa;\nmov.b64 aa, {%1, %1};\nsub.rn.f32x2 %0, aa, %2;\n}" : "=l"(r) : "f"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2_fma_bcast(unsigned long long sl, float a, unsigned long long c) {
    unsigned long long r;
    asm("{\n.reg .b64 aa;\nmov.b64 aa, {%2, %2};\nfma.rn.f32x2 %0, %1, aa, %3;\n}" : "=l"(r) : "l"(sl), "f"(a), "l"(c));
    return r;
}
#endif

__device__ __forceinline__ float crossing_x(float4 e, float py) {
#if METHOD == 0
    return __fadd_rn(__fdiv_rn(__fmul_rn(e.z, __fsub_rn(py, e.x)), e.w), e.y);
#elif METHOD == 1
    return __fmaf_rn(e.z, __fsub_rn(py, e.x), e.y);
#else
    return __fmaf_rn(e.z, py, e.y);
#endif
}

#ifdef MIN_BLOCKS
extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X, MIN_BLOCKS)
#else
extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X)
#endif
pnpoly(int *__restrict__ bitmap, const float2 *__restrict__ points, int n,
       const float4 *__restrict__ g_edges, const float2 *__restrict__ g_ybounds,
       const float4 *__restrict__ g_packed) {
#if ASM && ASM != 8
    // packed records, NPACK entries (ASM 1/2: {ymin, ymax, slope, icpt};
    // ASM 3: {vy_k, slope, icpt, 0})
    __shared__ __align__(16) float4 s_packed[TAB_VEC4];
    for (int k = threadIdx.x; k < TAB_VEC4; k += BLOCK_SIZE_X) s_packed[k] = g_packed[k];
    __syncthreads();
#elif POLY_SMEM
    __shared__ float4 s_edges[VERTICES];
#if BETWEEN == 1
    __shared__ float2 s_ybounds[VERTICES];
#endif
    for (int k = threadIdx.x; k < VERTICES; k += BLOCK_SIZE_X) {
        s_edges[k] = g_edges[k];
#if BETWEEN == 1
        s_ybounds[k] = g_ybounds[k];
#endif
    }
    __syncthreads();
    const float4 *edges = s_edges;
#if BETWEEN == 1
    const float2 *ybounds = s_ybounds;
#endif
#else
    const float4 *edges = c_edges;
#if BETWEEN == 1
    const float2 *ybounds = c_ybounds;
#endif
#endif

    // Coalesced: in step t, consecutive threads own consecutive points
    // (VEC=1: float2) or point pairs (VEC=2: float4).
    // PERSIST=1: a grid of ~SMs x resident blocks strides over point tiles, so
    // each block stages the polygon once (no per-tile barrier / table reload)
    const long long n_tiles = ((long long)n + BLOCK_SIZE_X * TILE - 1) / (BLOCK_SIZE_X * TILE);
    for (long long tile_id = blockIdx.x; tile_id < n_tiles; tile_id += gridDim.x) {
    const long long block_base = tile_id * (BLOCK_SIZE_X * TILE);
    float px[TILE], py[TILE];
    int idx[TILE];
#pragma unroll
    for (int t = 0; t < TILE / VEC; ++t) {
        const long long first = block_base + (long long)VEC * ((long long)t * BLOCK_SIZE_X + threadIdx.x);
#if VEC == 2
        idx[2 * t] = (int)first;
        idx[2 * t + 1] = (int)first + 1;
        if (first + 1 < n) {
            const float4 q = reinterpret_cast<const float4 *>(points)[first >> 1];
            px[2 * t] = q.x;
            py[2 * t] = q.y;
            px[2 * t + 1] = q.z;
            py[2 * t + 1] = q.w;
        } else {
            const float2 q = first < n ? points[first] : make_float2(0.f, 0.f);
            px[2 * t] = q.x;
            py[2 * t] = q.y;
            px[2 * t + 1] = 0.f;
            py[2 * t + 1] = 0.f;
        }
#else
        idx[t] = (int)first;
        const float2 q = first < n ? points[first] : make_float2(0.f, 0.f);
        px[t] = q.x;
        py[t] = q.y;
#endif
    }

#if ASM == 4 || ASM == 6
#if ASM == 4
#define SP_ASM S4_ASM
#else
#define SP_ASM S6_ASM
#endif
    unsigned inside[TILE];
    {
        unsigned acc[TILE];
        unsigned long long pxp[TILE / 2], pyp[TILE / 2];
#pragma unroll
        for (int t = 0; t < TILE; ++t) acc[t] = 0u;
#pragma unroll
        for (int q = 0; q < TILE / 2; ++q) {
            // pair (2q, 2q+1) came from one float4 {x0, y0, x1, y1}
            pxp[q] = ((unsigned long long)__float_as_uint(px[2 * q + 1]) << 32) | __float_as_uint(px[2 * q]);
            pyp[q] = ((unsigned long long)__float_as_uint(py[2 * q + 1]) << 32) | __float_as_uint(py[2 * q]);
        }
        const unsigned sbase = (unsigned)__cvta_generic_to_shared(s_packed);
        const unsigned span = NPACK * 16u;
        const float vy_last = s_packed[VERTICES - 1].x;
#if TILE == 4
        asm volatile(SP_ASM : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3])
                     : "l"(pxp[0]), "l"(pxp[1]), "l"(pyp[0]), "l"(pyp[1]), "r"(sbase), "r"(span), "f"(vy_last));
#else
        asm volatile(SP_ASM : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),
                     "+r"(acc[6]), "+r"(acc[7])
                     : "l"(pxp[0]), "l"(pxp[1]), "l"(pxp[2]), "l"(pxp[3]), "l"(pyp[0]), "l"(pyp[1]), "l"(pyp[2]),
                       "l"(pyp[3]), "r"(sbase), "r"(span), "f"(vy_last));
#endif
#pragma unroll
        for (int t = 0; t < TILE; ++t) inside[t] = acc[t] >> 31;
    }
#elif ASM == 8
    unsigned inside[TILE];
    {
        unsigned acc[TILE], dp[TILE];
        const float vy_last = reinterpret_cast<const float *>(c_pairs)[(VERTICES - 1) / 4 * 12 + (VERTICES - 1) % 4];
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            acc[t] = 0u;
            dp[t] = __float_as_uint(__fsub_rn(py[t], vy_last));
        }
#pragma unroll 2
        for (int g = 0; g < NPAIR8 / 4; ++g) {
            const ulonglong2 vy = c_pairs[3 * g], sl = c_pairs[3 * g + 1], ic = c_pairs[3 * g + 2];
#pragma unroll
            for (int t = 0; t < TILE; ++t) {
                const unsigned long long dA = f2_sub_bcast(py[t], vy.x), dB = f2_sub_bcast(py[t], vy.y);
                const unsigned long long eA = f2_sub_bcast(px[t], f2_fma_bcast(sl.x, py[t], ic.x));
                const unsigned long long eB = f2_sub_bcast(px[t], f2_fma_bcast(sl.y, py[t], ic.y));
                const unsigned d0 = (unsigned)dA, d1 = (unsigned)(dA >> 32);
                const unsigned d2 = (unsigned)dB, d3 = (unsigned)(dB >> 32);
                // crossing bit of each edge = sign((py - vy_k) ^ (py - vy_{k-1})) & sign(px - x_k)
                acc[t] ^= ((d0 ^ dp[t]) & (unsigned)eA) ^ ((d1 ^ d0) & (unsigned)(eA >> 32));
                acc[t] ^= ((d2 ^ d1) & (unsigned)eB) ^ ((d3 ^ d2) & (unsigned)(eB >> 32));
                dp[t] = d3;
            }
        }
#pragma unroll
        for (int t = 0; t < TILE; ++t) inside[t] = acc[t] >> 31;
    }
#elif ASM == 3 || ASM == 5 || ASM == 7 || ASM == 9
#if ASM == 3
#define SS_ASM S3_ASM
#elif ASM == 5
#define SS_ASM S5_ASM
#else
#define SS_ASM S7_ASM
#endif
    unsigned inside[TILE];
    {
        unsigned acc[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) acc[t] = 0u;
        const unsigned sbase = (unsigned)__cvta_generic_to_shared(s_packed);
#if ASM == 7 || ASM == 9
        const unsigned span = NPAIR8 * 12u;  // 4-edge groups of 12 floats
        const float vy_last = reinterpret_cast<const float *>(s_packed)[(VERTICES - 1) / 4 * 12 + (VERTICES - 1) % 4];
#else
        const unsigned span = NPACK * 16u;
        const float vy_last = s_packed[VERTICES - 1].x;
#endif
#if TILE == 2
        asm volatile(SS_ASM : "+r"(acc[0]), "+r"(acc[1]) : "f"(px[0]), "f"(px[1]), "f"(py[0]), "f"(py[1]),
                     "r"(sbase), "r"(span), "f"(vy_last));
#elif TILE == 4
        asm volatile(SS_ASM : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3])
                     : "f"(px[0]), "f"(px[1]), "f"(px[2]), "f"(px[3]), "f"(py[0]), "f"(py[1]), "f"(py[2]), "f"(py[3]),
                       "r"(sbase), "r"(span), "f"(vy_last));
#elif TILE == 6
        asm volatile(SS_ASM : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5])
                     : "f"(px[0]), "f"(px[1]), "f"(px[2]), "f"(px[3]), "f"(px[4]), "f"(px[5]), "f"(py[0]), "f"(py[1]),
                       "f"(py[2]), "f"(py[3]), "f"(py[4]), "f"(py[5]), "r"(sbase), "r"(span), "f"(vy_last));
#else
        asm volatile(SS_ASM : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),
                     "+r"(acc[6]), "+r"(acc[7])
                     : "f"(px[0]), "f"(px[1]), "f"(px[2]), "f"(px[3]), "f"(px[4]), "f"(px[5]), "f"(px[6]), "f"(px[7]),
                       "f"(py[0]), "f"(py[1]), "f"(py[2]), "f"(py[3]), "f"(py[4]), "f"(py[5]), "f"(py[6]), "f"(py[7]),
                       "r"(sbase), "r"(span), "f"(vy_last));
#endif
#pragma unroll
        for (int t = 0; t < TILE; ++t) inside[t] = acc[t] >> 31;
    }
#elif ASM
    unsigned inside[TILE];
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(s_packed);
    const unsigned zero = 0u;
    const unsigned span = NPACK * 16u;
#if TILE == 1
    asm volatile("{\n" PREDS EXTRA_REGS ".reg .f32 ylo, yhi, sl, ic, x;\n.reg .u32 ptr, end;\n" INIT
                 "mov.u32 ptr, %" BASE_OP ";\nadd.u32 end, ptr, %" END_OP ";\n"
                 "PNPOLY_LOOP:\n" BODY
                 "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_LOOP;\n" OUT_SELP "}\n"
                 : "=r"(inside[0]) : "f"(px[0]), "f"(py[0]), "r"(sbase), "r"(zero), "r"(span));
#elif TILE == 2
    asm volatile("{\n" PREDS EXTRA_REGS ".reg .f32 ylo, yhi, sl, ic, x;\n.reg .u32 ptr, end;\n" INIT
                 "mov.u32 ptr, %" BASE_OP ";\nadd.u32 end, ptr, %" END_OP ";\n"
                 "PNPOLY_LOOP:\n" BODY
                 "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_LOOP;\n" OUT_SELP "}\n"
                 : "=r"(inside[0]), "=r"(inside[1])
                 : "f"(px[0]), "f"(px[1]), "f"(py[0]), "f"(py[1]), "r"(sbase), "r"(zero), "r"(span));
#elif TILE == 4
    asm volatile("{\n" PREDS EXTRA_REGS ".reg .f32 ylo, yhi, sl, ic, x;\n.reg .u32 ptr, end;\n" INIT
                 "mov.u32 ptr, %" BASE_OP ";\nadd.u32 end, ptr, %" END_OP ";\n"
                 "PNPOLY_LOOP:\n" BODY
                 "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_LOOP;\n" OUT_SELP "}\n"
                 : "=r"(inside[0]), "=r"(inside[1]), "=r"(inside[2]), "=r"(inside[3])
                 : "f"(px[0]), "f"(px[1]), "f"(px[2]), "f"(px[3]), "f"(py[0]), "f"(py[1]), "f"(py[2]), "f"(py[3]),
                   "r"(sbase), "r"(zero), "r"(span));
#else
    asm volatile("{\n" PREDS EXTRA_REGS ".reg .f32 ylo, yhi, sl, ic, x;\n.reg .u32 ptr, end;\n" INIT
                 "mov.u32 ptr, %" BASE_OP ";\nadd.u32 end, ptr, %" END_OP ";\n"
                 "PNPOLY_LOOP:\n" BODY
                 "add.u32 ptr, ptr, 64;\nsetp.lt.u32 s, ptr, end;\n@s bra PNPOLY_LOOP;\n" OUT_SELP "}\n"
                 : "=r"(inside[0]), "=r"(inside[1]), "=r"(inside[2]), "=r"(inside[3]), "=r"(inside[4]),
                   "=r"(inside[5])
                 : "f"(px[0]), "f"(px[1]), "f"(px[2]), "f"(px[3]), "f"(px[4]), "f"(px[5]), "f"(py[0]), "f"(py[1]),
                   "f"(py[2]), "f"(py[3]), "f"(py[4]), "f"(py[5]), "r"(sbase), "r"(zero), "r"(span));
#endif
#else
    bool inside[TILE];
#if BETWEEN == 0
    bool prev_above[TILE];
    const float vy_last = edges[VERTICES - 1].x;
#pragma unroll
    for (int t = 0; t < TILE; ++t) prev_above[t] = vy_last > py[t];
#endif
#pragma unroll
    for (int t = 0; t < TILE; ++t) inside[t] = false;

#pragma unroll 4
    for (int k = 0; k < VERTICES; ++k) {
        const float4 e = edges[k];
#if BETWEEN == 1
        const float2 yb = ybounds[k];
#endif
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
#if BETWEEN == 0
            const bool above = e.x > py[t];
            const bool spans = above != prev_above[t];
            prev_above[t] = above;
#else
            const bool spans = (yb.x <= py[t]) & (py[t] < yb.y);
#endif
            // predicated toggle: ptxas folds this into one @P FSETP.LT.XOR
            const float xc = crossing_x(e, py[t]);
            if (spans) inside[t] = inside[t] != (px[t] < xc);
        }
    }

#endif
#pragma unroll
    for (int t = 0; t < TILE; ++t)
        if (idx[t] < n) bitmap[idx[t]] = inside[t] ? 1 : 0;
    }  // tile loop
}
