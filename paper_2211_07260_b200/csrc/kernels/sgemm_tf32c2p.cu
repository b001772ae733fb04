// Persistent TF32 tensor-core SGEMM on CTA pairs (tcgen05.mma.cta_group::2), sm_100a.
//
//   C[M][N] = alpha * sum_k A[m][k] * B[k][n] + beta * C[m][n]
//
// The CTA-pair kernel (sgemm_tf32c2.cu: one 256 x BN tile per cluster of two
// CTAs, M = 256 MMAs issued by the leader) made persistent and warp
// specialised like sgemm_tf32p.cu:
//
//   * one cluster of 2 CTAs per TPC (grid = 2 x min(#SMs / 2, #tiles)); pair p
//     walks tiles p, p + pairs, ... so the last wave no longer leaves whole
//     TPCs idle while the pair kernel's 3.5 waves finish;
//   * warp 0 of each CTA is its TMA producer (own 128 rows of A, own BN/2
//     columns of B per k-step, completing on the LEADER's full barrier);
//     warp 1 of the leader issues the M = 256 MMAs; warps 2-5 of both CTAs
//     are the epilogue (warp w drains TMEM lanes 32*(w%4)..+31 of its CTA);
//   * two TMEM accumulators (2 x BN columns, pair allocation): the epilogue
//     of tile i overlaps the MMAs of tile i+1. The leader's tmem_empty
//     barrier takes one arrival from each CTA's epilogue (the follower's
//     through its shared::cluster address), so the MMA never overwrites an
//     accumulator either CTA is still reading;
//   * tcgen05.commit ... multicast::cluster frees a stage in both CTAs and
//     signals both epilogues;
//   * SPLIT_TAIL: tiles = q * pairs + r. A static persistent schedule still
//     leaves r pairs with one tile more than the others; when 2r <= pairs
//     the r leftover tiles are split into two K halves run by 2r pairs.
//     Each CTA of a half-pair stores its 128 partial rows to a workspace and
//     bumps a counter per (tile, CTA rank); the second finisher sums the two
//     halves in a fixed order (deterministic) and writes C. No CTA waits on
//     another; counters only grow (odd = partner done), so relaunches need
//     no reset.
//
// Storage and operand layout as sgemm_tf32c2.cu. Tunables (-D): BN (128,
// 256), STAGES, SPLIT_TAIL, BK (32, 64, 128). Requires M % 256 == 0, N % BN == 0, K % BK == 0. Launch:
// grid (2 * pairs, 1, 1), 192 threads, cluster (2, 1, 1).
#ifndef BN
#define BN 256
#endif
#ifndef STAGES
#define STAGES 4
#endif
#define BM 128  // rows per CTA (the pair covers 256)
#ifndef BK  // k-rows per stage (one TMA box per 32 M / N columns; BK / 8 MMAs per stage)
#define BK 32
#endif
#if BK != 32 && BK != 64 && BK != 128
#error "BK must be 32, 64 or 128"
#endif
#define BN_HALF (BN / 2)
#define A_STAGE_BYTES (BM * BK * 4)
#define B_STAGE_BYTES (BN_HALF * BK * 4)
#define STAGE_BYTES (A_STAGE_BYTES + B_STAGE_BYTES)
#define TMEM_COLS (2 * BN)
#define EPI_THREADS 128
#ifndef SPLIT_TAIL
#define SPLIT_TAIL 1
#endif

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
// arrive on a barrier given by its shared::cluster address (possibly in the peer CTA)
__device__ __forceinline__ void mbar_arrive_cluster(unsigned cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// wait until the phase with parity `parity` completed (a fresh barrier reports parity 1 as
// completed, so waits for "free" start with parity 1); acquire at cluster scope, since
// arrivals come from the peer CTA too
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned map_to_rank(unsigned addr, unsigned rank) {
    unsigned out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
    return out;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_sync(unsigned id, unsigned threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(unsigned dst, const TensorMap *map, unsigned bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(dst),
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
           ((unsigned)(256 >> 4) << 24);
}

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

// A work unit: a tile and a K range; part 0 = whole tile, 1/2 = split halves.
struct Unit {
    int tile, k_begin, k_end, part;
};
// The static schedule of one pair, computed arithmetically.
struct Schedule {
    int dp_units, split_unit, dp_tiles, k_tiles, pair;
    __device__ Schedule(int pair_, int pairs, int tiles, int k_tiles_) : k_tiles(k_tiles_), pair(pair_) {
        const int full_waves = tiles / pairs, rest = tiles - full_waves * pairs;
        const bool split = SPLIT_TAIL && rest > 0 && 2 * rest <= pairs && k_tiles >= 2;
        dp_tiles = split ? full_waves * pairs : tiles;
        dp_units = pair < dp_tiles ? (dp_tiles - 1 - pair) / pairs + 1 : 0;
        split_unit = (split && pair < 2 * rest) ? 1 : 0;
    }
    __device__ int count() const { return dp_units + split_unit; }
    __device__ Unit at(int i, int pairs) const {
        if (i < dp_units) return Unit{pair + i * pairs, 0, k_tiles, 0};
        const int half = pair & 1, mid = k_tiles / 2;
        return Unit{dp_tiles + (pair >> 1), half ? mid : 0, half ? k_tiles : mid, 1 + half};
    }
};

#define TMEM_LD32(taddr, v)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, " \
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"              \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),          \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),    \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),  \
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])   \
        : "r"(taddr))

extern "C" __global__ void __launch_bounds__(192, 1)
sgemm_tf32c2p(const __grid_constant__ TensorMap map_a, const __grid_constant__ TensorMap map_b, float *__restrict__ c,
              float *__restrict__ workspace, unsigned *__restrict__ counters, const int M, const int N, const int K,
              const float alpha, const float beta) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = (unsigned char *)(((unsigned long long)smem_raw + 1023) & ~1023ull);
    unsigned long long *full = (unsigned long long *)(smem + STAGES * STAGE_BYTES);
    unsigned long long *empty = full + STAGES;
    unsigned long long *tmem_full = empty + STAGES;  // [2]
    unsigned long long *tmem_empty = tmem_full + 2;  // [2], the leader's counts both CTAs
    unsigned *tmem_slot = (unsigned *)(tmem_empty + 2);
    unsigned *reduce_flag = tmem_slot + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
    const int tiles_m = M / 256, tiles = tiles_m * (N / BN), k_tiles = K / BK;
    const Schedule sched(pair, pairs, tiles, k_tiles);
    const int n_units = sched.count();

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);   // leader only: its arrive.expect_tx (both CTAs' bytes)
            mbar_init(smem_u32(&empty[s]), 1);  // one multicast commit per use
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&tmem_full[b]), 1);   // one multicast commit per tile
            mbar_init(smem_u32(&tmem_empty[b]), 2);  // leader: one arrival per CTA's epilogue
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 0) {  // pair allocation: the same warp of both CTAs
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (both CTAs) ----
            int g = 0;
            for (int u = 0; u < n_units; ++u) {
                const Unit unit = sched.at(u, pairs);
                int mt, nt;
                tile_coords(unit.tile, tiles_m, N / BN, mt, nt);
                const int m0 = mt * 256, n0 = nt * BN;
                const int m_own = m0 + (int)rank * BM, n_own = n0 + (int)rank * BN_HALF;
                for (int kt = unit.k_begin; kt < unit.k_end; ++kt, ++g) {
                    const int s = g % STAGES;
                    mbar_wait(smem_u32(&empty[s]), ((g / STAGES) & 1) ^ 1);
                    const unsigned bar_local = smem_u32(&full[s]);
                    if (leader) mbar_expect_tx(bar_local, 2 * STAGE_BYTES);
                    const unsigned bar = map_to_rank(bar_local, 0);
                    const unsigned a_dst = smem_u32(smem + s * STAGE_BYTES), b_dst = a_dst + A_STAGE_BYTES;
#pragma unroll
                    for (int q = 0; q < BM / 32; ++q)
                        tma_load_2d_pair(a_dst + q * (BK * 128), &map_a, bar, m_own + 32 * q, kt * BK);
#pragma unroll
                    for (int q = 0; q < BN_HALF / 32; ++q)
                        tma_load_2d_pair(b_dst + q * (BK * 128), &map_b, bar, n_own + 32 * q, kt * BK);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {  // ---- MMA issuer (leader only): M = 256 over both SMs ----
            const unsigned idesc = instr_desc();
            int g = 0;
            for (int u = 0; u < n_units; ++u) {
                const Unit unit = sched.at(u, pairs);
                const int acc = u & 1;
                mbar_wait(smem_u32(&tmem_empty[acc]), ((u >> 1) & 1) ^ 1);  // both epilogues drained it
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
                            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
                            "l"(smem_desc(a_base + kk * 1024)), "l"(smem_desc(b_base + kk * 1024)), "r"(idesc),
                            "r"(accumulate));
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                        "%1;" ::"r"(smem_u32(&empty[s])),
                        "h"((unsigned short)3)
                        : "memory");
                }
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                    "%1;" ::"r"(smem_u32(&tmem_full[acc])),
                    "h"((unsigned short)3)
                    : "memory");
            }
        }
    } else {
        // ---- epilogue warps 2..5 of both CTAs: this CTA's 128 rows, TMEM lanes 32*(warp%4).. ----
        const int quarter = warp & 3;
        const int epi_tid = threadIdx.x - 64;
        for (int u = 0; u < n_units; ++u) {
            const Unit unit = sched.at(u, pairs);
            const int acc = u & 1;
            int mt, nt;
            tile_coords(unit.tile, tiles_m, N / BN, mt, nt);
            const int m0 = mt * 256, n0 = nt * BN;
            mbar_wait(smem_u32(&tmem_full[acc]), (u >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int local_row = (int)rank * BM + quarter * 32 + lane;  // row within the 256-row tile
            float *crow = c + (size_t)(m0 + local_row) * N + n0;
            const unsigned lane_base = tmem + acc * BN + ((unsigned)(quarter * 32) << 16);
            if (unit.part) {
                // split-K half: publish this CTA's 128 partial rows, the second finisher reduces
                const int slot = unit.tile - sched.dp_tiles;
                const size_t half_stride = (size_t)256 * BN;
                float *h0 = workspace + (size_t)2 * slot * half_stride + (size_t)local_row * BN;
                float *mine = h0 + (unit.part - 1) * half_stride;
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
                named_sync(1, EPI_THREADS);
                if (epi_tid == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&tmem_empty[acc]), 0));
                __threadfence();
                named_sync(1, EPI_THREADS);
                if (epi_tid == 0) *reduce_flag = atomicAdd(&counters[2 * slot + rank], 1u);
                named_sync(1, EPI_THREADS);
                const unsigned arrived_before = *reduce_flag;
                named_sync(1, EPI_THREADS);  // everyone read the flag before the next unit reuses it
                if (arrived_before & 1u) {   // second finisher: fixed order half 0 + half 1
                    __threadfence();
                    const float *h1 = h0 + half_stride;
#pragma unroll 1
                    for (int col = 0; col < BN; col += 4) {
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
                continue;
            }
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
            named_sync(1, EPI_THREADS);  // all 128 rows of this CTA drained
            if (epi_tid == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&tmem_empty[acc]), 0));
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();  // neither CTA frees the pair's TMEM while the other may still use it
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}
