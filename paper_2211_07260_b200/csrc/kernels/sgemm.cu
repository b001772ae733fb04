// CLBlast-style FP32 SIMT SGEMM for sm_100a, compiled per config by NVRTC.
//
//   C[M][N] = alpha * sum_k A[m][k] * B[k][n] + beta * C[m][n]
//
// Storage (BLAS conventions): A column-major (M contiguous, i.e. a K x M
// row-major buffer "AT"), B row-major (K x N, N contiguous), C row-major.
// This is the layout CLBlast's xgemm kernel works in after its
// pre-processing, so the tunables keep CLBlast's meaning (PAPER.md:309-316,
// fixture analogue pkg/src/jouletune/fixtures/gemm_space.json):
//
//   MWG, NWG, KWG   CTA tile (M, N) and K step staged per iteration
//   MDIMC, NDIMC    threads of the CTA along M / N (CTA = MDIMC*NDIMC)
//   MDIMA, NDIMB    thread shape along M (for A) / N (for B) when loading tiles
//   KWI             unroll factor of the inner k loop
//   VWM, VWN        vector widths along M / N (fragment loads, A/B tile loads)
//   STRM, STRN      0: a thread's MWI (NWI) outputs are contiguous in M (N);
//                   1: strided by MDIMC*VWM (NDIMC*VWN) -> conflict-free smem
//   SA, SB          1: stage the A (B) tile in shared memory (double buffered);
//                   0: read fragments straight from global memory through L1
//   ASYNC           (B200 addition, not a CLBlast knob) 0: CLBlast's staging
//                   through registers (global -> registers -> shared, two
//                   static buffers); 2 or 3: that many shared-memory stages
//                   filled by cp.async (LDGSTS) straight from global memory,
//                   one __syncthreads per k-tile. Frees the KWA*MWA/VWM +
//                   KWB*NWB/VWN staging registers per thread and lets the
//                   copy of tile t+ASYNC-1 overlap the FFMAs of tile t.
//                   Needs SA = SB = 1 (dynamic shared memory, up to 227 KB).
//   FMA2            (B200 addition) 1: the outer product issues packed
//                   FFMA2 on pairs of N-adjacent accumulators with the A
//                   element as a broadcast scalar: half the FFMA issue slots
//                   for the same FMA-pipe work, leaving issue bandwidth for
//                   the fragment loads. Per element the same fma.rn sequence,
//                   so the result is bit-identical to FMA2 = 0. Needs VWN even.
//   GROUP_M         (B200 addition) CTA rasterisation: 1 = launch order (all of
//                   A streams past every B column panel), g = groups of g M-tiles
//                   sweep the N-tiles together, so the resident CTAs' A and B
//                   panels stay in L2 (fewer DRAM re-reads; same result bits).
//   SPLIT_TAIL      (B200 addition) 0: one CTA per C tile (2D grid). s > 1: a 1D
//                   grid in which the tiles that fill whole waves (full_tiles =
//                   a multiple of SMs x resident CTAs, sized by the host) run
//                   whole, and the last partial wave's tiles are split along K
//                   over `split` (<= s) CTAs each. 4096^2 in 128 x 128 tiles is
//                   1024 tiles = 3.46 waves of 296 CTAs: without the split the
//                   4th wave runs at 46% occupancy. Partials go to a workspace;
//                   the last of a tile's CTAs to arrive (per-tile counter, reset
//                   by that CTA) sums them in part order (so the bits do not
//                   depend on arrival order) and runs the epilogue.
//
// Requirements (the tuning-space restrictions, kernels.py):
//   MWG % (MDIMC*VWM) == 0, NWG % (NDIMC*VWN) == 0,
//   MWG % (MDIMA*VWM) == 0, NWG % (NDIMB*VWN) == 0,
//   KWG % (MDIMC*NDIMC/MDIMA) == 0, KWG % (MDIMC*NDIMC/NDIMB) == 0,
//   KWG % KWI == 0, M % MWG == 0, N % NWG == 0, K % KWG == 0.
#ifndef MWG
#define MWG 128
#endif
#ifndef NWG
#define NWG 128
#endif
#ifndef KWG
#define KWG 16
#endif
#ifndef MDIMC
#define MDIMC 16
#endif
#ifndef NDIMC
#define NDIMC 16
#endif
#ifndef MDIMA
#define MDIMA 32
#endif
#ifndef NDIMB
#define NDIMB 32
#endif
#ifndef KWI
#define KWI 2
#endif
#ifndef VWM
#define VWM 4
#endif
#ifndef VWN
#define VWN 4
#endif
#ifndef STRM
#define STRM 1
#endif
#ifndef STRN
#define STRN 1
#endif
#ifndef SA
#define SA 1
#endif
#ifndef SB
#define SB 1
#endif
#ifndef ASYNC
#define ASYNC 0
#endif
#if ASYNC && !(SA && SB)
#error "ASYNC staging needs SA = SB = 1"
#endif
#if ASYNC == 1 || ASYNC > 4
#error "ASYNC must be 0, 2, 3 or 4"
#endif

#ifndef FMA2
#define FMA2 0
#endif
#ifndef GROUP_M  // (B200 addition) CTA rasterisation group along M; 1 = CLBlast's launch order
#define GROUP_M 1
#endif
#ifndef SPLIT_TAIL
#define SPLIT_TAIL 0
#endif
#if FMA2 && (VWN % 2)
#error "FMA2 needs an even VWN (accumulator pairs inside one B vector)"
#endif
#define THREADS (MDIMC * NDIMC)
#define MWI (MWG / MDIMC)
#define NWI (NWG / NDIMC)
#define KDIMA (THREADS / MDIMA)
#define KDIMB (THREADS / NDIMB)
#define MWA (MWG / MDIMA)  // M elements per thread when loading A
#define KWA (KWG / KDIMA)  // K rows per thread when loading A
#define NWB (NWG / NDIMB)
#define KWB (KWG / KDIMB)

#if (MWG % (MDIMC * VWM)) || (NWG % (NDIMC * VWN)) || (MWG % (MDIMA * VWM)) || (NWG % (NDIMB * VWN)) || \
    (KWG % KDIMA) || (KWG % KDIMB) || (KWG % KWI) || (THREADS % MDIMA) || (THREADS % NDIMB)
#error "invalid CLBlast-style SGEMM configuration"
#endif

template <int W>
struct vec;
template <>
struct vec<1> { typedef float t; };
template <>
struct vec<2> { typedef float2 t; };
template <>
struct vec<4> { typedef float4 t; };
// CLBlast's float8 (OpenCL has it, CUDA does not): two float4 halves, 32-byte aligned
struct __align__(32) float8 {
    float4 lo, hi;
};
template <>
struct vec<8> { typedef float8 t; };
typedef typename vec<VWM>::t vm_t;
typedef typename vec<VWN>::t vn_t;

__device__ __forceinline__ float lane(const float &v, int) { return v; }
__device__ __forceinline__ float lane(const float2 &v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ float lane(const float4 &v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ float lane(const float8 &v, int i) { return i < 4 ? lane(v.lo, i) : lane(v.hi, i - 4); }

// read-only global loads of one vector (__ldg has no float8 overload)
template <typename T>
__device__ __forceinline__ T ldg(const T *p) { return __ldg(p); }
template <>
__device__ __forceinline__ float8 ldg(const float8 *p) {
    const float4 *q = reinterpret_cast<const float4 *>(p);
    return float8{__ldg(q), __ldg(q + 1)};
}

// Offset (in vectors of VWM) of this thread's w-th A fragment vector inside the MWG tile.
__device__ __forceinline__ int frag_m(int tm, int w) {
#if STRM == 0
    return tm * (MWI / VWM) + w;
#else
    return w * MDIMC + tm;
#endif
}
__device__ __forceinline__ int frag_n(int tn, int w) {
#if STRN == 0
    return tn * (NWI / VWN) + w;
#else
    return w * NDIMC + tn;
#endif
}

#if ASYNC
// one VW-float vector global -> shared without a register round trip
template <typename T>
__device__ __forceinline__ void cp_async(T *dst, const T *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if constexpr (sizeof(T) == 32) {  // float8: two 16-byte copies
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16), "l"((const char *)src + 16) : "memory");
    } else if constexpr (sizeof(T) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"((int)sizeof(T)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
#endif

#if FMA2
// acc2 = {b0, b1} * {a, a} + acc2 per lane (fma.rn.f32x2): the accumulator pair lives in
// one 64-bit register pair, the A element is the broadcast scalar operand
__device__ __forceinline__ void fma2(unsigned long long &acc2, float a, float b0, float b1) {
    asm("{\n.reg .b64 aa, bb;\nmov.b64 aa, {%1, %1};\nmov.b64 bb, {%2, %3};\nfma.rn.f32x2 %0, bb, aa, %0;\n}"
        : "+l"(acc2)
        : "f"(a), "f"(b0), "f"(b1));
}
#endif

#ifdef MIN_BLOCKS  // (optional) __launch_bounds__ minimum resident blocks (register cap)
extern "C" __global__ void __launch_bounds__(THREADS, MIN_BLOCKS)
#else
extern "C" __global__ void __launch_bounds__(THREADS)
#endif
sgemm(const int M, const int N, const int K, const float alpha, const float beta,
      const float *__restrict__ at, const float *__restrict__ b, float *__restrict__ c
#if SPLIT_TAIL
      , float *__restrict__ ws, unsigned *__restrict__ counters, const int full_tiles, const int split
#endif
) {
    const int tid = threadIdx.x;
    const int tm = tid % MDIMC, tn = tid / MDIMC;
    const int tiles = K / KWG;  // k-tiles
#if SPLIT_TAIL
    // 1D grid: [0, full_tiles) whole tiles, then `split` K-parts of each remaining tile
    const int tiles_m = M / MWG, tiles_n = N / NWG;
    int tile = blockIdx.x, part = 0, parts = 1;
    if (tile >= full_tiles) {
        const int u = tile - full_tiles;
        tile = full_tiles + u / split;
        part = u % split;
        parts = split;
    }
    const int kt0 = part * tiles / parts, kt1 = (part + 1) * tiles / parts;
    int m_tile = tile % tiles_m, n_tile = tile / tiles_m;
#else
    const int kt0 = 0, kt1 = tiles;
    const int tiles_m = gridDim.x, tiles_n = gridDim.y;
    int m_tile = blockIdx.x, n_tile = blockIdx.y;
#endif
    // CTA rasterisation: GROUP_M = 1 is CLBlast's launch order (blockIdx.x walks M with one B
    // column panel); GROUP_M = g walks g M-tiles across all N-tiles before moving on, so the CTAs
    // resident at once share g A panels and a run of B panels in L2 instead of all of A.
#if GROUP_M > 1
    {
        const int pid = m_tile + n_tile * tiles_m;
        const int per_group = GROUP_M * tiles_n;
        const int first = (pid / per_group) * GROUP_M;
        const int rows = min(tiles_m - first, GROUP_M);
        m_tile = first + (pid % per_group) % rows;
        n_tile = (pid % per_group) / rows;
    }
#endif
    const int m0 = m_tile * MWG, n0 = n_tile * NWG;

#if ASYNC
    // ASYNC stages of {A tile, B tile} in dynamic shared memory
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    typedef vm_t a_tile_t[KWG][MWG / VWM];
    typedef vn_t b_tile_t[KWG][NWG / VWN];
    a_tile_t *a_sm = reinterpret_cast<a_tile_t *>(smem_dyn);
    b_tile_t *b_sm = reinterpret_cast<b_tile_t *>(smem_dyn + ASYNC * sizeof(a_tile_t));
    const int ma = tid % MDIMA, ka = tid / MDIMA;
    const int nb = tid % NDIMB, kb = tid / NDIMB;
#else
    // CLBlast's two shared-memory buffers, in dynamic shared memory: the paper's space has
    // configs (KWG 32, 128 x 128, SA = SB = 1: 64 KB double-buffered) above the 48 KB static cap
    extern __shared__ __align__(128) unsigned char smem_dyn[];
#if SA
    typedef vm_t a_tile_t[KWG][MWG / VWM];
    a_tile_t *a_sm = reinterpret_cast<a_tile_t *>(smem_dyn);
    const int ma = tid % MDIMA, ka = tid / MDIMA;
    vm_t a_reg[KWA][MWA / VWM];
#endif
#if SB
    typedef vn_t b_tile_t[KWG][NWG / VWN];
    b_tile_t *b_sm = reinterpret_cast<b_tile_t *>(smem_dyn + (SA ? 2 * KWG * MWG * 4 : 0));
    const int nb = tid % NDIMB, kb = tid / NDIMB;
    vn_t b_reg[KWB][NWB / VWN];
#endif

#endif

#if FMA2
    unsigned long long acc2[MWI][NWI / 2];
#pragma unroll
    for (int i = 0; i < MWI; ++i)
#pragma unroll
        for (int j = 0; j < NWI / 2; ++j) acc2[i][j] = 0ull;
#else
    float acc[MWI][NWI];
#pragma unroll
    for (int i = 0; i < MWI; ++i)
#pragma unroll
        for (int j = 0; j < NWI; ++j) acc[i][j] = 0.f;
#endif

    const vm_t *at_v = reinterpret_cast<const vm_t *>(at);
    const vn_t *b_v = reinterpret_cast<const vn_t *>(b);
    const int lda_v = M / VWM, ldb_v = N / VWN;

    // one KWG-deep k-tile of FFMAs from stage `buf` (SA/SB = 0: fragments from global at k0)
    auto mac_tile = [&](const int buf, const int k0) {
#pragma unroll 1
        for (int kw = 0; kw < KWG; kw += KWI) {
#pragma unroll
            for (int ki = 0; ki < KWI; ++ki) {
                const int k = kw + ki;
                vm_t af[MWI / VWM];
                vn_t bf[NWI / VWN];
#pragma unroll
                for (int w = 0; w < MWI / VWM; ++w) {
#if SA
                    af[w] = a_sm[buf][k][frag_m(tm, w)];
#else
                    af[w] = ldg(at_v + (size_t)(k0 + k) * lda_v + m0 / VWM + frag_m(tm, w));
#endif
                }
#pragma unroll
                for (int w = 0; w < NWI / VWN; ++w) {
#if SB
                    bf[w] = b_sm[buf][k][frag_n(tn, w)];
#else
                    bf[w] = ldg(b_v + (size_t)(k0 + k) * ldb_v + n0 / VWN + frag_n(tn, w));
#endif
                }
#pragma unroll
                for (int i = 0; i < MWI; ++i)
#pragma unroll
#if FMA2
                    for (int j = 0; j < NWI; j += 2)
                        fma2(acc2[i][j / 2], lane(af[i / VWM], i % VWM), lane(bf[j / VWN], j % VWN),
                             lane(bf[j / VWN], j % VWN + 1));
#else
                    for (int j = 0; j < NWI; ++j)
                        acc[i][j] = fmaf(lane(af[i / VWM], i % VWM), lane(bf[j / VWN], j % VWN), acc[i][j]);
#endif
            }
        }
    };
#if ASYNC
    // global -> shared copies of k-tile `tile` into stage `buf`, same thread mapping as CLBlast's loads
    auto issue = [&](int tile, int buf) {
        const int k0 = tile * KWG;
#pragma unroll
        for (int kk = 0; kk < KWA; ++kk)
#pragma unroll
            for (int mv = 0; mv < MWA / VWM; ++mv)
                cp_async(&a_sm[buf][ka + kk * KDIMA][ma + mv * MDIMA],
                         at_v + (size_t)(k0 + ka + kk * KDIMA) * lda_v + m0 / VWM + ma + mv * MDIMA);
#pragma unroll
        for (int kk = 0; kk < KWB; ++kk)
#pragma unroll
            for (int nv = 0; nv < NWB / VWN; ++nv)
                cp_async(&b_sm[buf][kb + kk * KDIMB][nb + nv * NDIMB],
                         b_v + (size_t)(k0 + kb + kk * KDIMB) * ldb_v + n0 / VWN + nb + nv * NDIMB);
    };
#pragma unroll
    for (int s = 0; s < ASYNC - 1; ++s) {
        if (kt0 + s < kt1) issue(kt0 + s, s);
        cp_async_commit();  // empty groups keep the wait_group arithmetic uniform
    }
#pragma unroll 1
    for (int t = kt0; t < kt1; ++t) {
        const int i = t - kt0;
        cp_async_wait<ASYNC - 2>();  // this thread's copies of tile t have landed
        __syncthreads();             // everyone's have; and everyone is done with tile t-1's stage
        if (t + ASYNC - 1 < kt1) issue(t + ASYNC - 1, (i + ASYNC - 1) % ASYNC);  // refill tile t-1's stage
        cp_async_commit();
        mac_tile(i % ASYNC, t * KWG);
    }
#else
    auto fetch = [&](int k0) {
#if SA
#pragma unroll
        for (int kk = 0; kk < KWA; ++kk)
#pragma unroll
            for (int mv = 0; mv < MWA / VWM; ++mv)
                a_reg[kk][mv] = ldg(at_v + (size_t)(k0 + ka + kk * KDIMA) * lda_v + m0 / VWM + ma + mv * MDIMA);
#endif
#if SB
#pragma unroll
        for (int kk = 0; kk < KWB; ++kk)
#pragma unroll
            for (int nv = 0; nv < NWB / VWN; ++nv)
                b_reg[kk][nv] = ldg(b_v + (size_t)(k0 + kb + kk * KDIMB) * ldb_v + n0 / VWN + nb + nv * NDIMB);
#endif
    };
    auto stash = [&](int buf) {
#if SA
#pragma unroll
        for (int kk = 0; kk < KWA; ++kk)
#pragma unroll
            for (int mv = 0; mv < MWA / VWM; ++mv) a_sm[buf][ka + kk * KDIMA][ma + mv * MDIMA] = a_reg[kk][mv];
#endif
#if SB
#pragma unroll
        for (int kk = 0; kk < KWB; ++kk)
#pragma unroll
            for (int nv = 0; nv < NWB / VWN; ++nv) b_sm[buf][kb + kk * KDIMB][nb + nv * NDIMB] = b_reg[kk][nv];
#endif
    };

#if SA || SB
    fetch(kt0 * KWG);
    stash(0);
    __syncthreads();
#endif
#pragma unroll 1
    for (int t = kt0; t < kt1; ++t) {
        const int buf = (t - kt0) & 1;
        const int k0 = t * KWG;
#if SA || SB
        if (t + 1 < kt1) fetch(k0 + KWG);
#endif
        mac_tile(buf, k0);
#if SA || SB
        if (t + 1 < kt1) stash(buf ^ 1);
        __syncthreads();
#endif
    }

#endif

#if FMA2
    float acc[MWI][NWI];
#pragma unroll
    for (int i = 0; i < MWI; ++i)
#pragma unroll
        for (int j = 0; j < NWI; j += 2) {
            acc[i][j] = __uint_as_float((unsigned)acc2[i][j / 2]);
            acc[i][j + 1] = __uint_as_float((unsigned)(acc2[i][j / 2] >> 32));
        }
#endif
#if SPLIT_TAIL
    if (parts > 1) {
        // this part's partial tile -> workspace slot (coalesced: element e of every thread together)
        const int slot0 = (tile - full_tiles) * parts;
        float *mine = ws + (size_t)(slot0 + part) * (MWG * NWG);
#pragma unroll
        for (int i = 0; i < MWI; ++i)
#pragma unroll
            for (int j = 0; j < NWI; ++j) __stcg(mine + (i * NWI + j) * THREADS + tid, acc[i][j]);
        __threadfence();
        __syncthreads();
        __shared__ unsigned arrived;
        if (tid == 0) arrived = atomicAdd(counters + (tile - full_tiles), 1u);
        __syncthreads();
        if (arrived != (unsigned)(parts - 1)) return;  // another part finishes this tile
        if (tid == 0) counters[tile - full_tiles] = 0u;  // every part has arrived: reset for the next launch
        __threadfence();
        // every partial (this CTA's too) is re-read from the workspace and summed in part order,
        // whatever the arrival order, so the bits are reproducible
        const float *w = ws + (size_t)slot0 * (MWG * NWG) + tid;
#pragma unroll
        for (int i = 0; i < MWI; ++i)
#pragma unroll
            for (int j = 0; j < NWI; ++j) {
                const int e = (i * NWI + j) * THREADS;
                float sum = __ldcg(w + e) + __ldcg(w + MWG * NWG + e);
#pragma unroll
                for (int q = 2; q < SPLIT_TAIL; ++q)
                    if (q < parts) sum += __ldcg(w + q * (MWG * NWG) + e);
                acc[i][j] = sum;
            }
    }
#endif
    // epilogue: C = alpha * acc + beta * C, VWN-wide row segments
#pragma unroll
    for (int i = 0; i < MWI; ++i) {
        const int m = m0 + frag_m(tm, i / VWM) * VWM + i % VWM;
#pragma unroll
        for (int w = 0; w < NWI / VWN; ++w) {
            const int n = n0 + frag_n(tn, w) * VWN;
            vn_t *dst = reinterpret_cast<vn_t *>(c + (size_t)m * N + n);
            vn_t old = beta != 0.f ? *dst : vn_t();
            float *o = reinterpret_cast<float *>(&old);
#pragma unroll
            for (int v = 0; v < VWN; ++v) o[v] = fmaf(alpha, acc[i][w * VWN + v], beta * o[v]);
            *dst = old;
        }
    }
}
