// TF32 tensor-core SGEMM for sm_100a on a CTA pair: tcgen05.mma.cta_group::2.
//
//   C[M][N] = alpha * sum_k A[m][k] * B[k][n] + beta * C[m][n]
//
// Same storage and operand layout as sgemm_tf32.cu (A column-major = a K x M
// row-major buffer, B row-major K x N, both MN-major for UMMA, TMA boxes of
// 32 k-rows x 128 B in the SWIZZLE_128B_BASE32B layout). What changes is the
// unit of work: a cluster of two CTAs on the two SMs of a TPC computes one
// 256 x BN tile with M=256 MMAs issued by the leader CTA alone:
//
//   * each CTA stages ITS OWN 128 rows of A and ITS OWN BN/2 columns of B per
//     k-step (16 KB + BN*64 B per stage instead of 16 KB + BN*128 B for a
//     single-CTA 128 x BN tile): the pair reads each B byte once for 256 rows
//     of output, halving the L2 -> SM operand traffic per flop for B;
//   * both CTAs' TMA loads complete on the LEADER's full barrier
//     (cp.async.bulk.tensor.cta_group::2, barrier address mapped to rank 0);
//   * the leader's MMA thread issues tcgen05.mma.cta_group::2.kind::tf32
//     (M=256, N=BN, K=8): the tensor cores of both SMs read their own smem
//     halves and each accumulates its 128 x BN rows in its own TMEM;
//   * tcgen05.commit.cta_group::2 ... multicast::cluster frees the stage in
//     both CTAs (empty barriers) and finally signals both epilogues;
//   * each CTA's 4 warps drain their TMEM (rows rank*128 + 32*warp + lane).
//
// Tunables (-D): BN (128, 256) = the pair's N tile, STAGES (2..8).
// Requires M % 256 == 0, N % BN == 0, K % 32 == 0. Launch: grid
// (2 * N / BN, M / 256), 128 threads, cluster (2, 1, 1).
#ifndef BN
#define BN 256
#endif
#ifndef STAGES
#define STAGES 4
#endif
#define BM 128           // rows per CTA (the pair covers 256)
#define BK 32
#define BN_HALF (BN / 2) // B columns staged per CTA
#define A_STAGE_BYTES (BM * BK * 4)
#define B_STAGE_BYTES (BN_HALF * BK * 4)
#define STAGE_BYTES (A_STAGE_BYTES + B_STAGE_BYTES)
#define TMEM_COLS BN

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

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ unsigned map_to_rank(unsigned addr, unsigned rank) {
    unsigned out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
    return out;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// pair TMA: data lands in this CTA's smem, the byte count completes on `bar`
// (the leader's full barrier, a shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(unsigned dst, const TensorMap *map, unsigned bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

// SWIZZLE_128B_BASE32B MN-major shared-memory matrix descriptor (Blackwell version bits = 1)
__device__ __forceinline__ unsigned long long smem_desc(unsigned addr, unsigned lbo, unsigned sbo) {
    unsigned long long d = 0;
    d |= (unsigned long long)((addr >> 4) & 0x3FFF);
    d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
    d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version
    d |= 1ull << 61;  // SWIZZLE_128B_BASE32B
    return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, both MN-major, M = 256 (pair)
__host__ __device__ constexpr unsigned instr_desc() {
    return (1u << 4)                       // c_format = F32
           | (2u << 7)                     // a_format = TF32
           | (2u << 10)                    // b_format = TF32
           | (1u << 15)                    // a_major = MN
           | (1u << 16)                    // b_major = MN
           | ((unsigned)(BN >> 3) << 17)   // n_dim
           | ((unsigned)(256 >> 4) << 24); // m_dim
}

extern "C" __global__ void __launch_bounds__(128, 1)
sgemm_tf32c2(const __grid_constant__ TensorMap map_a, const __grid_constant__ TensorMap map_b, float *__restrict__ c,
             const int M, const int N, const int K, const float alpha, const float beta) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = (unsigned char *)(((unsigned long long)smem_raw + 1023) & ~1023ull);
    unsigned long long *full = (unsigned long long *)(smem + STAGES * STAGE_BYTES);
    unsigned long long *empty = full + STAGES;
    unsigned long long *acc_ready = empty + STAGES;
    unsigned *tmem_slot = (unsigned *)(acc_ready + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned rank = cluster_rank();
    const bool leader = rank == 0;
    const int n0 = (blockIdx.x >> 1) * BN;       // the pair's N tile
    const int m0 = blockIdx.y * 256;             // the pair's M tile
    const int k_tiles = K / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);    // used in the leader only: its own expect_tx arrival
            mbar_init(smem_u32(&empty[s]), 1);   // one multicast commit per round
        }
        mbar_init(smem_u32(acc_ready), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 0) {  // pair allocation: the same warp of both CTAs, same slot offset
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync();  // barriers of both CTAs initialised, TMEM of both allocated
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer (both CTAs): own A rows and own B columns, completing on the leader's barrier ----
        const int m_own = m0 + (int)rank * BM;
        const int n_own = n0 + (int)rank * BN_HALF;
        for (int kt = 0; kt < k_tiles; ++kt) {
            const int s = kt % STAGES;
            if (kt >= STAGES) mbar_wait(smem_u32(&empty[s]), ((kt / STAGES) - 1) & 1);
            const unsigned bar_local = smem_u32(&full[s]);
            if (leader) mbar_expect_tx(bar_local, 2 * STAGE_BYTES);
            const unsigned bar = map_to_rank(bar_local, 0);
            const unsigned a_dst = smem_u32(smem + s * STAGE_BYTES);
            const unsigned b_dst = a_dst + A_STAGE_BYTES;
            const int k0 = kt * BK;
#pragma unroll
            for (int g = 0; g < BM / 32; ++g) tma_load_2d_pair(a_dst + g * (BK * 128), &map_a, bar, m_own + 32 * g, k0);
#pragma unroll
            for (int g = 0; g < BN_HALF / 32; ++g)
                tma_load_2d_pair(b_dst + g * (BK * 128), &map_b, bar, n_own + 32 * g, k0);
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // ---- MMA issuer (leader only): M = 256 over both SMs ----
        const unsigned idesc = instr_desc();
        for (int kt = 0; kt < k_tiles; ++kt) {
            const int s = kt % STAGES;
            mbar_wait(smem_u32(&full[s]), (kt / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const unsigned a_base = smem_u32(smem + s * STAGE_BYTES);
            const unsigned b_base = a_base + A_STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
                const unsigned long long da = smem_desc(a_base + kk * 1024, BK * 128, 512);
                const unsigned long long db = smem_desc(b_base + kk * 1024, BK * 128, 512);
                const unsigned accumulate = (kt | kk) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
            }
            // frees stage s in BOTH CTAs once the tensor cores have read it
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&empty[s])),
                "h"((unsigned short)3)
                : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(acc_ready)),
            "h"((unsigned short)3)
            : "memory");
    }

    // ---- epilogue (both CTAs): this CTA's 128 rows of the 256 x BN tile ----
    mbar_wait(smem_u32(acc_ready), 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = m0 + (int)rank * BM + warp * 32 + lane;
    float *crow = c + (size_t)row * N + n0;
#pragma unroll 1
    for (int col = 0; col < BN; col += 32) {
        unsigned v[32];
        const unsigned taddr = tmem + ((unsigned)(warp * 32) << 16) + col;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float4 *dst = reinterpret_cast<float4 *>(crow + col);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float4 old = beta != 0.f ? dst[q] : make_float4(0.f, 0.f, 0.f, 0.f);
            old.x = fmaf(alpha, __uint_as_float(v[4 * q + 0]), beta * old.x);
            old.y = fmaf(alpha, __uint_as_float(v[4 * q + 1]), beta * old.y);
            old.z = fmaf(alpha, __uint_as_float(v[4 * q + 2]), beta * old.z);
            old.w = fmaf(alpha, __uint_as_float(v[4 * q + 3]), beta * old.w);
            dst[q] = old;
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();  // neither CTA frees the pair's TMEM while the other may still read it
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}
