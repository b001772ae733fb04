// Persistent TF32 tensor-core SGEMM for sm_100a (tcgen05 + TMA + TMEM).
//
//   C[M][N] = alpha * sum_k A[m][k] * B[k][n] + beta * C[m][n]
//
// Storage and shared-memory operand layout as in sgemm_tf32.cu (A column-
// major / B row-major, both MN-major UMMA operands in the SWIZZLE_128B_BASE32B
// layout that TMA writes with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
//
// What this version adds:
//   * persistent CTAs (grid <= #SMs, one CTA per SM) walking a static list
//     of work units, warp-specialised: warp 0 = TMA producer, warp 1 = MMA
//     issuer, warps 2-5 = epilogue (warp w drains TMEM lanes 32*(w%4)..+31);
//   * two TMEM accumulators (2 x BN columns): the epilogue of unit i runs
//     while the tensor core already accumulates unit i+1
//     (tmem_full / tmem_empty mbarrier pairs);
//   * split-K tail: tiles = q * grid + r; the q full waves run data
//     parallel, and when 2r <= grid the r leftover tiles are split into two
//     K halves (2r units on 2r CTAs instead of r tiles on r CTAs). Each half
//     stores its partial accumulator to a workspace, bumps a per-tile
//     counter, and the second finisher sums both halves and writes C — no
//     CTA ever waits on another.
// Tunables (-D): BN (128, 256), STAGES, SPLIT_TAIL (0/1).
#ifndef BN
#define BN 256
#endif
#ifndef STAGES
#define STAGES 4
#endif
#ifndef SPLIT_TAIL
#define SPLIT_TAIL 1
#endif
#define BM 128
#define BK 32
#define A_STAGE_BYTES (BM * BK * 4)
#define B_STAGE_BYTES (BN * BK * 4)
#define STAGE_BYTES (A_STAGE_BYTES + B_STAGE_BYTES)
#define TMEM_COLS (2 * BN)
#define EPI_THREADS 128

#if BN != 128 && BN != 256
#error "BN must be 128 or 256"
#endif

struct __align__(64) TensorMap {
    unsigned long long opaque[16];
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Wait until the phase with parity `parity` has completed (a fresh barrier
// reports parity 1 as completed, so producers start with parity 1).
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const TensorMap *map, unsigned bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ unsigned long long smem_desc(unsigned addr) {
    // SWIZZLE_128B_BASE32B, MN-major: LBO = BK*128 B (MN groups), SBO = 512 B (4-row K groups)
    return (unsigned long long)((addr >> 4) & 0x3FFF) | ((unsigned long long)((BK * 128) >> 4) << 16) |
           ((unsigned long long)(512 >> 4) << 32) | (1ull << 46) | (1ull << 61);
}
__host__ __device__ constexpr unsigned instr_desc() {
    return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((unsigned)(BN >> 3) << 17) |
           ((unsigned)(BM >> 4) << 24);
}
__device__ __forceinline__ void named_sync(unsigned id, unsigned threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// A work unit: a tile and a K range; part 0 = whole tile, 1/2 = split halves.
struct Unit {
    int tile, k_begin, k_end, part;
};

// The static schedule, computed arithmetically (no per-thread unit list).
struct Schedule {
    int dp_units;    // full tiles this CTA owns: tiles cta, cta + grid, ...
    int split_unit;  // 1 if this CTA also owns one half of a split tail tile
    int dp_tiles, k_tiles, cta;
    __device__ Schedule(int cta_, int grid, int tiles, int k_tiles_) : k_tiles(k_tiles_), cta(cta_) {
        const int full_waves = tiles / grid, rest = tiles - full_waves * grid;
        const bool split = SPLIT_TAIL && rest > 0 && 2 * rest <= grid && k_tiles >= 2;
        dp_tiles = split ? full_waves * grid : tiles;
        dp_units = cta < dp_tiles ? (dp_tiles - 1 - cta) / grid + 1 : 0;
        split_unit = (split && cta < 2 * rest) ? 1 : 0;
    }
    __device__ int count() const { return dp_units + split_unit; }
    __device__ Unit at(int i, int grid) const {
        if (i < dp_units) return Unit{cta + i * grid, 0, k_tiles, 0};
        const int half = cta & 1, mid = k_tiles / 2;
        return Unit{dp_tiles + (cta >> 1), half ? mid : 0, half ? k_tiles : mid, 1 + half};
    }
};

#ifndef GROUP_M  // tile walk: GROUP_M M-tiles sweep every N-tile before the next group (1 = M fastest, all of A per B panel)
#define GROUP_M 1
#endif
// Persistent tile order -> (M tile, N tile). GROUP_M = 1: consecutive tiles share the B column
// panel and walk all of A. GROUP_M = g: g M-tiles x all N-tiles per group, so the tiles in flight
// at once (one per CTA / pair) touch g A panels and a run of B panels that stay in L2.
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int &mt, int &nt) {
#if GROUP_M > 1
    const int per_group = GROUP_M * tiles_n;
    const int first = (tile / per_group) * GROUP_M;
    const int rows = min(tiles_m - first, GROUP_M);
    mt = first + (tile % per_group) % rows;
    nt = (tile % per_group) / rows;
#else
    mt = tile % tiles_m;
    nt = tile / tiles_m;
#endif
}

__device__ __forceinline__ void tile_origin(int tile, int tiles_m, int tiles_n, int &m0, int &n0) {
    int mt, nt;
    tile_coords(tile, tiles_m, tiles_n, mt, nt);
    m0 = mt * BM;
    n0 = nt * BN;
}

#define TMEM_LD32(taddr, v)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "  \
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"               \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),          \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),    \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),  \
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])   \
        : "r"(taddr))

extern "C" __global__ void __launch_bounds__(192, 1)
sgemm_tf32p(const __grid_constant__ TensorMap map_a, const __grid_constant__ TensorMap map_b, float *__restrict__ c,
            float *__restrict__ workspace, unsigned *__restrict__ counters, const int M, const int N, const int K,
            const float alpha, const float beta) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = (unsigned char *)(((unsigned long long)smem_raw + 1023) & ~1023ull);
    unsigned long long *full = (unsigned long long *)(smem + STAGES * STAGE_BYTES);
    unsigned long long *empty = full + STAGES;
    unsigned long long *tmem_full = empty + STAGES;  // [2]
    unsigned long long *tmem_empty = tmem_full + 2;  // [2]
    unsigned *tmem_slot = (unsigned *)(tmem_empty + 2);
    unsigned *reduce_flag = tmem_slot + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_m = M / BM, tiles = tiles_m * (N / BN), k_tiles = K / BK;
    const Schedule sched(blockIdx.x, gridDim.x, tiles, k_tiles);
    const int n_units = sched.count();

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&tmem_full[b]), 1);
            mbar_init(smem_u32(&tmem_empty[b]), EPI_THREADS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: k-steps of all units through the smem ring ----
            int g = 0;
            for (int u = 0; u < n_units; ++u) {
                const Unit unit = sched.at(u, gridDim.x);
                int m0, n0;
                tile_origin(unit.tile, tiles_m, N / BN, m0, n0);
                for (int kt = unit.k_begin; kt < unit.k_end; ++kt, ++g) {
                    const int s = g % STAGES;
                    mbar_wait(smem_u32(&empty[s]), ((g / STAGES) & 1) ^ 1);
                    const unsigned bar = smem_u32(&full[s]);
                    mbar_expect_tx(bar, STAGE_BYTES);
                    const unsigned a_dst = smem_u32(smem + s * STAGE_BYTES), b_dst = a_dst + A_STAGE_BYTES;
#pragma unroll
                    for (int q = 0; q < BM / 32; ++q) tma_load_2d(a_dst + q * (BK * 128), &map_a, bar, m0 + 32 * q, kt * BK);
#pragma unroll
                    for (int q = 0; q < BN / 32; ++q) tma_load_2d(b_dst + q * (BK * 128), &map_b, bar, n0 + 32 * q, kt * BK);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer ----
            const unsigned idesc = instr_desc();
            int g = 0;
            for (int u = 0; u < n_units; ++u) {
                const Unit unit = sched.at(u, gridDim.x);
                const int acc = u & 1;
                mbar_wait(smem_u32(&tmem_empty[acc]), ((u >> 1) & 1) ^ 1);  // epilogue drained this buffer
                asm volatile("tcgen05.fence::after_thread_sync;");
                const unsigned d_tmem = tmem + acc * BN;
                for (int kt = unit.k_begin; kt < unit.k_end; ++kt, ++g) {
                    const int s = g % STAGES;
                    mbar_wait(smem_u32(&full[s]), (g / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const unsigned a_base = smem_u32(smem + s * STAGE_BYTES), b_base = a_base + A_STAGE_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 8; ++kk) {
                        const unsigned accumulate = (kt != unit.k_begin || kk) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
                            "l"(smem_desc(a_base + kk * 1024)), "l"(smem_desc(b_base + kk * 1024)), "r"(idesc),
                            "r"(accumulate));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&empty[s]))
                                 : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&tmem_full[acc]))
                             : "memory");
            }
        }
    } else {
        // ---- epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31 ----
        const int quarter = warp & 3;
        const int epi_tid = threadIdx.x - 64;
        for (int u = 0; u < n_units; ++u) {
            const Unit unit = sched.at(u, gridDim.x);
            const int acc = u & 1;
            int m0, n0;
            tile_origin(unit.tile, tiles_m, N / BN, m0, n0);
            mbar_wait(smem_u32(&tmem_full[acc]), (u >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int row = quarter * 32 + lane;
            float *crow = c + (size_t)(m0 + row) * N + n0;
            const unsigned lane_base = tmem + acc * BN + ((unsigned)(quarter * 32) << 16);
            const int part = unit.part;
            if (part == 0) {
#pragma unroll 1
                for (int col = 0; col < BN; col += 32) {
                    unsigned v[32];
                    TMEM_LD32(lane_base + col, v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    float4 *dst = reinterpret_cast<float4 *>(crow + col);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 o = beta != 0.f ? dst[q] : make_float4(0.f, 0.f, 0.f, 0.f);
                        o.x = fmaf(alpha, __uint_as_float(v[4 * q + 0]), beta * o.x);
                        o.y = fmaf(alpha, __uint_as_float(v[4 * q + 1]), beta * o.y);
                        o.z = fmaf(alpha, __uint_as_float(v[4 * q + 2]), beta * o.z);
                        o.w = fmaf(alpha, __uint_as_float(v[4 * q + 3]), beta * o.w);
                        dst[q] = o;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                mbar_arrive(smem_u32(&tmem_empty[acc]));
            } else {
                // split-K half: publish the partial, the second finisher reduces
                const int slot = unit.tile - sched.dp_tiles;
                const size_t half_stride = (size_t)BM * BN;
                float *h0 = workspace + (size_t)2 * slot * half_stride + (size_t)row * BN;
                float *mine = h0 + (part - 1) * half_stride;
#pragma unroll 1
                for (int col = 0; col < BN; col += 32) {
                    unsigned v[32];
                    TMEM_LD32(lane_base + col, v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    float4 *dst = reinterpret_cast<float4 *>(mine + col);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                mbar_arrive(smem_u32(&tmem_empty[acc]));  // TMEM no longer needed
                __threadfence();
                named_sync(1, EPI_THREADS);
                if (epi_tid == 0) *reduce_flag = atomicAdd(&counters[slot], 1u);
                named_sync(1, EPI_THREADS);
                const unsigned arrived_before = *reduce_flag;
                named_sync(1, EPI_THREADS);  // everyone read the flag before the next unit reuses it
                if (arrived_before & 1u) {   // second finisher (counters only grow: odd = partner done)
                    __threadfence();
                    const float *h1 = h0 + half_stride;
#pragma unroll 1
                    for (int col = 0; col < BN; col += 4) {
                        // fixed summation order (half 0 + half 1): deterministic results
                        const float4 p0 = __ldcg(reinterpret_cast<const float4 *>(h0 + col));
                        const float4 p1 = __ldcg(reinterpret_cast<const float4 *>(h1 + col));
                        float4 *dst = reinterpret_cast<float4 *>(crow + col);
                        float4 o = beta != 0.f ? *dst : make_float4(0.f, 0.f, 0.f, 0.f);
                        o.x = fmaf(alpha, p0.x + p1.x, beta * o.x);
                        o.y = fmaf(alpha, p0.y + p1.y, beta * o.y);
                        o.z = fmaf(alpha, p0.z + p1.z, beta * o.z);
                        o.w = fmaf(alpha, p0.w + p1.w, beta * o.w);
                        *dst = o;
                    }
                }
            }
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}
