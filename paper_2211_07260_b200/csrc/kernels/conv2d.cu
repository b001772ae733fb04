// 2D correlation out[y][x] = sum_{i,j} in[y+i][x+j] * f[i][j], sm_100a, per-config NVRTC.
//
// No reference code exists: the paper's Kernel-Tuner
// convolution benchmark rebuilt for B200. The input is pre-padded
// ((H+FH-1) x (W+FW-1), row pitch IN_W floats); the filter lives in
// __constant__ memory so that, with every loop counted at compile time,
// each FFMA takes its coefficient as a constant-bank operand (no load).
//
// Work decomposition: a CTA of BLOCK_X x BLOCK_Y threads computes a
// (BLOCK_X*TILE_X) x (BLOCK_Y*TILE_Y) output tile; each thread owns a
// TILE_X-wide, TILE_Y-tall patch of *contiguous* outputs, so the
// TILE_X + FW - 1 input values of one input row serve TILE_X*FW FFMAs and
// every input row loaded into registers serves all (output row, filter
// row) pairs that need it (fully unrolled: smem traffic per FFMA ~
// (TILE_Y+FH-1)(TILE_X+FW-1) / (FH*FW*TILE_X*TILE_Y) words).
//
// Tunables (-D): BLOCK_X, BLOCK_Y, TILE_X (1,2,4,8), TILE_Y, USE_SMEM (stage
// the input tile in shared memory, else read through L1 with __ldg),
// PAD (extra floats per smem row, multiple of 4), IMAGE_W, IMAGE_H, FW, FH,
// FMA2 (B200 addition): accumulators in x-adjacent pairs; for even filter
// columns j the pair {in[x+j], in[x+j+1]} is an aligned register pair, so one
// packed FFMA2 (filter coefficient as the broadcast operand, held in a uniform
// register) does two FMAs; odd columns stay scalar. Half the issue slots of
// the even-column FMAs, the same fma.rn per output in the same order: the
// result is bit-identical to FMA2 = 0. Needs an even TILE_X. MIN_BLOCKS
// (optional): the __launch_bounds__ minimum-blocks hint.
#ifndef BLOCK_X
#define BLOCK_X 32
#endif
#ifndef BLOCK_Y
#define BLOCK_Y 4
#endif
#ifndef TILE_X
#define TILE_X 4
#endif
#ifndef TILE_Y
#define TILE_Y 4
#endif
#ifndef USE_SMEM
#define USE_SMEM 1
#endif
#ifndef PAD
#define PAD 0
#endif
#ifndef IMAGE_W
#define IMAGE_W 4096
#endif
#ifndef IMAGE_H
#define IMAGE_H 4096
#endif
#ifndef FW
#define FW 17
#endif
#ifndef FH
#define FH 17
#endif
#ifndef FMA2
#define FMA2 0
#endif
#if FMA2 && (TILE_X % 2)
#error "FMA2 needs an even TILE_X"
#endif

#if ((FW - 1) % 4) != 0 || (PAD % 4) != 0
#error "vector loads need FW-1 and PAD to be multiples of 4"
#endif

#define IN_W (IMAGE_W + FW - 1)
#define OUT_TW (BLOCK_X * TILE_X)
#define OUT_TH (BLOCK_Y * TILE_Y)
#define SH_W (OUT_TW + FW - 1 + PAD)
#define SH_H (OUT_TH + FH - 1)
#define SEG (TILE_X + FW - 1)

#if (TILE_X % 4) == 0
#define VW 4
#elif (TILE_X % 2) == 0
#define VW 2
#else
#define VW 1
#endif

__constant__ float d_filter[FH * FW];

template <int W>
struct vec_t;
template <>
struct vec_t<1> { typedef float type; };
template <>
struct vec_t<2> { typedef float2 type; };
template <>
struct vec_t<4> { typedef float4 type; };

// Load SEG consecutive floats starting at p (p is VW-aligned) into r[].
template <bool Global>
__device__ __forceinline__ void load_segment(float (&r)[SEG + 3], const float *p) {
    typedef typename vec_t<VW>::type V;
#pragma unroll
    for (int s = 0; s < (SEG + VW - 1) / VW; ++s) {
        V v;
        if (Global)
            v = __ldg(reinterpret_cast<const V *>(p) + s);
        else
            v = reinterpret_cast<const V *>(p)[s];
        const float *f = reinterpret_cast<const float *>(&v);
#pragma unroll
        for (int q = 0; q < VW; ++q) r[s * VW + q] = f[q];
    }
}

#if FMA2
// {acc.lo, acc.hi} += {x0, x1} * {f, f} as one fma.rn.f32x2
__device__ __forceinline__ void fma2(unsigned long long &acc, float f, float x0, float x1) {
    asm("{\n.reg .b64 ff, xx;\nmov.b64 ff, {%1, %1};\nmov.b64 xx, {%2, %3};\nfma.rn.f32x2 %0, xx, ff, %0;\n}"
        : "+l"(acc)
        : "f"(f), "f"(x0), "f"(x1));
}
// the same two FMAs as scalar fma.rn (x0 / x1 need not form an aligned pair)
__device__ __forceinline__ void fma_split(unsigned long long &acc, float f, float x0, float x1) {
    asm("{\n.reg .f32 lo, hi;\nmov.b64 {lo, hi}, %0;\nfma.rn.f32 lo, %2, %1, lo;\nfma.rn.f32 hi, %3, %1, hi;\n"
        "mov.b64 %0, {lo, hi};\n}"
        : "+l"(acc)
        : "f"(f), "f"(x0), "f"(x1));
}
#endif

#ifdef MIN_BLOCKS  // minimum resident blocks: with 2, ptxas may use up to 64 registers (more loads in
                   // flight) while two 512-thread blocks still fit (scripts/time_conv_minb.py)
extern "C" __global__ void __launch_bounds__(BLOCK_X *BLOCK_Y, MIN_BLOCKS)
#else
extern "C" __global__ void __launch_bounds__(BLOCK_X *BLOCK_Y)
#endif
conv2d(float *__restrict__ out, const float *__restrict__ in) {
    const int x0 = blockIdx.x * OUT_TW;
    const int y0 = blockIdx.y * OUT_TH;
#if USE_SMEM
    __shared__ __align__(16) float tile[SH_H * SH_W + 4];  // +4: vector over-read of the last row
    {
        // cooperative, vectorised copy of the (SH_H x (OUT_TW+FW-1)) input window
        constexpr int COLS = OUT_TW + FW - 1;       // floats per row actually needed
        constexpr int COLS4 = (COLS + 3) / 4;      // float4 per row (over-read <= 3, stays in the padded row)
        const int tid = threadIdx.y * BLOCK_X + threadIdx.x;
        for (int e = tid; e < SH_H * COLS4; e += BLOCK_X * BLOCK_Y) {
            const int r = e / COLS4, c4 = e - r * COLS4;
            const float *src = in + (size_t)(y0 + r) * IN_W + x0 + 4 * c4;
            float4 v;
            if (x0 + 4 * c4 + 3 < IN_W) {
                v = __ldg(reinterpret_cast<const float4 *>(src));
            } else {
                v.x = x0 + 4 * c4 + 0 < IN_W ? src[0] : 0.f;
                v.y = x0 + 4 * c4 + 1 < IN_W ? src[1] : 0.f;
                v.z = x0 + 4 * c4 + 2 < IN_W ? src[2] : 0.f;
                v.w = 0.f;
            }
            if (4 * c4 + 3 < SH_W) {
                *reinterpret_cast<float4 *>(&tile[r * SH_W + 4 * c4]) = v;
            } else {
                float *d = &tile[r * SH_W + 4 * c4];
                if (4 * c4 + 0 < SH_W) d[0] = v.x;
                if (4 * c4 + 1 < SH_W) d[1] = v.y;
                if (4 * c4 + 2 < SH_W) d[2] = v.z;
            }
        }
        __syncthreads();
    }
    const float *base = tile + (threadIdx.y * TILE_Y) * SH_W + threadIdx.x * TILE_X;
    constexpr int PITCH = SH_W;
#else
    const float *base = in + (size_t)(y0 + threadIdx.y * TILE_Y) * IN_W + x0 + threadIdx.x * TILE_X;
    constexpr int PITCH = IN_W;
#endif

#if FMA2
    unsigned long long acc2[TILE_Y][TILE_X / 2];
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty)
#pragma unroll
        for (int tx = 0; tx < TILE_X / 2; ++tx) acc2[ty][tx] = 0ull;
#else
    float acc[TILE_Y][TILE_X];
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty)
#pragma unroll
        for (int tx = 0; tx < TILE_X; ++tx) acc[ty][tx] = 0.f;
#endif

    // Input row r (relative to the thread patch) feeds output rows ty with
    // filter row i = r - ty in [0, FH).
#pragma unroll
    for (int r = 0; r < TILE_Y + FH - 1; ++r) {
        float seg[SEG + 3];
        load_segment<!USE_SMEM>(seg, base + r * PITCH);
#pragma unroll
        for (int ty = 0; ty < TILE_Y; ++ty) {
            const int i = r - ty;
            if (i >= 0 && i < FH) {
#pragma unroll
                for (int j = 0; j < FW; ++j)
#if FMA2
#pragma unroll
                    for (int tx = 0; tx < TILE_X; tx += 2) {
                        if ((j & 1) == 0)
                            fma2(acc2[ty][tx / 2], d_filter[i * FW + j], seg[tx + j], seg[tx + j + 1]);
                        else
                            fma_split(acc2[ty][tx / 2], d_filter[i * FW + j], seg[tx + j], seg[tx + j + 1]);
                    }
#else
#pragma unroll
                    for (int tx = 0; tx < TILE_X; ++tx) acc[ty][tx] = fmaf(seg[tx + j], d_filter[i * FW + j], acc[ty][tx]);
#endif
            }
        }
    }

#if FMA2
    float acc[TILE_Y][TILE_X];
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty)
#pragma unroll
        for (int tx = 0; tx < TILE_X; tx += 2) {
            acc[ty][tx] = __uint_as_float((unsigned)acc2[ty][tx / 2]);
            acc[ty][tx + 1] = __uint_as_float((unsigned)(acc2[ty][tx / 2] >> 32));
        }
#endif
    const int ox = x0 + threadIdx.x * TILE_X;
    const int oy = y0 + threadIdx.y * TILE_Y;
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty) {
        float *dst = out + (size_t)(oy + ty) * IMAGE_W + ox;
#if VW == 4
#pragma unroll
        for (int tx = 0; tx < TILE_X; tx += 4)
            *reinterpret_cast<float4 *>(dst + tx) = make_float4(acc[ty][tx], acc[ty][tx + 1], acc[ty][tx + 2], acc[ty][tx + 3]);
#elif VW == 2
#pragma unroll
        for (int tx = 0; tx < TILE_X; tx += 2) *reinterpret_cast<float2 *>(dst + tx) = make_float2(acc[ty][tx], acc[ty][tx + 1]);
#else
#pragma unroll
        for (int tx = 0; tx < TILE_X; ++tx) dst[tx] = acc[ty][tx];
#endif
    }
}
