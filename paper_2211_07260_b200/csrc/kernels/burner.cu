// Full-load FP32 burner for the P(f) clock sweep, sm_100a.
//
// Replaces the simulator's ConstantSurface(kappa=1, load=1) sweep kernel
// (reference cli.py:144-146): every FP32 lane runs CHAINS independent FFMA
// dependency chains for `iters` iterations, so runtime scales with 1/f_sm and
// the board draws full-load power at each requested clock. With CHAINS >= 8
// and >= 8 warps per SM scheduler the FMA pipe stays saturated (FFMA latency
// 4 cycles). The result is stored only if it equals a value it cannot reach,
// which keeps the arithmetic alive without any memory traffic.
#ifndef CHAINS
#define CHAINS 8
#endif
#ifndef BLOCK
#define BLOCK 256
#endif

extern "C" __global__ void __launch_bounds__(BLOCK)
burner(float *__restrict__ sink, const int iters, const float seed) {
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = seed + 0.001f * (threadIdx.x + c);
    const float a = 0.999999f, b = 1e-7f;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == -12345.678f) sink[blockIdx.x * BLOCK + threadIdx.x] = s;
}
