// TF32 tensor-core SGEMM for sm_100a: TMA -> shared memory -> tcgen05.mma -> TMEM.
//
//   C[M][N] = alpha * sum_k A[m][k] * B[k][n] + beta * C[m][n]
//
// Same storage as the SIMT kernel (sgemm.cu): A column-major (a K x M
// row-major buffer, M contiguous), B row-major (K x N, N contiguous), C
// row-major. Both operands are therefore "MN-major" for UMMA, which TF32
// supports directly: no transposes anywhere.
//
// Structure (one output tile of BM x BN per CTA, 128 threads):
//   * warp 0, one lane: TMA producer. Per k-step of BK=32 it loads the A tile
//     (BK x BM) as BM/32 boxes of 32 k-rows x 128 B and the B tile as BN/32
//     such boxes, 128-byte swizzled, into a STAGES-deep ring of shared
//     memory slots, signalling a full-barrier with the byte count.
//   * warp 1, one lane: MMA issuer. Waits for a slot, issues BK/8
//     `tcgen05.mma.cta_group::1.kind::tf32` (M=BM, N=BN, K=8) accumulating in
//     TMEM, then `tcgen05.commit` arrives on the slot's empty-barrier when the
//     tensor core is done reading it.
//   * all 4 warps: epilogue. After the last commit, each warp reads its 32
//     TMEM lanes (= 32 tile rows) with `tcgen05.ld.32x32b.x32`, applies
//     alpha/beta against C and stores.
//
// Shared-memory operand layout: MN-major TF32 operands must use the
// SWIZZLE_128B_BASE32B canonical layout (32-byte chunks XOR-swizzled within
// each 128-byte row, 4-row period), which TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B. Each 32-element MN group is a block of
// BK rows x 128 B; LBO = BK*128 B between MN groups, SBO = 4 rows x 128 B =
// 512 B between 4-row K groups; one MMA (K=8) spans 8 rows = 1 KB per MN
// group, so the k-th MMA of a stage starts 1 KB further. 1 KB aligned.
//
// Tunables (-D): BN (64, 128, 256), STAGES (2..6). Requires M % 128 == 0,
// N % BN == 0, K % 32 == 0.
#ifndef BN
#define BN 256
#endif
#ifndef STAGES
#define STAGES 4
#endif
#define BM 128
#define BK 32
#define A_STAGE_BYTES (BM * BK * 4)
#define B_STAGE_BYTES (BN * BK * 4)
#define STAGE_BYTES (A_STAGE_BYTES + B_STAGE_BYTES)
#define TMEM_COLS (BN < 32 ? 32 : BN)

#if (BN % 32) || BN > 256 || BN < 32
#error "BN must be a multiple of 32 in [32, 256]"
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

__device__ __forceinline__ void tma_load_2d(unsigned dst, const TensorMap *map, unsigned bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
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

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, both MN-major
__host__ __device__ constexpr unsigned instr_desc() {
    return (1u << 4)                  // c_format = F32
           | (2u << 7)                // a_format = TF32
           | (2u << 10)               // b_format = TF32
           | (1u << 15)               // a_major = MN
           | (1u << 16)               // b_major = MN
           | ((unsigned)(BN >> 3) << 17)  // n_dim
           | ((unsigned)(BM >> 4) << 24); // m_dim
}

extern "C" __global__ void __launch_bounds__(128, 1)
sgemm_tf32(const __grid_constant__ TensorMap map_a, const __grid_constant__ TensorMap map_b, float *__restrict__ c,
           const int M, const int N, const int K, const float alpha, const float beta) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1 KB alignment for the swizzle atoms
    unsigned char *smem = (unsigned char *)(((unsigned long long)smem_raw + 1023) & ~1023ull);
    unsigned long long *full = (unsigned long long *)(smem + STAGES * STAGE_BYTES);
    unsigned long long *empty = full + STAGES;
    unsigned long long *acc_ready = empty + STAGES;
    unsigned *tmem_slot = (unsigned *)(acc_ready + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int k_tiles = K / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        mbar_init(smem_u32(acc_ready), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 0) {  // TMEM accumulator: BN columns x 128 lanes of fp32
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        for (int kt = 0; kt < k_tiles; ++kt) {
            const int s = kt % STAGES;
            if (kt >= STAGES) mbar_wait(smem_u32(&empty[s]), ((kt / STAGES) - 1) & 1);
            const unsigned bar = smem_u32(&full[s]);
            mbar_expect_tx(bar, STAGE_BYTES);
            const unsigned a_dst = smem_u32(smem + s * STAGE_BYTES);
            const unsigned b_dst = a_dst + A_STAGE_BYTES;
            const int k0 = kt * BK;
#pragma unroll
            for (int g = 0; g < BM / 32; ++g) tma_load_2d(a_dst + g * (BK * 128), &map_a, bar, m0 + 32 * g, k0);
#pragma unroll
            for (int g = 0; g < BN / 32; ++g) tma_load_2d(b_dst + g * (BK * 128), &map_b, bar, n0 + 32 * g, k0);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer ----
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
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
            }
            // frees the smem slot once the tensor core has consumed it
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&empty[s]))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(acc_ready))
                     : "memory");
    }

    // ---- epilogue: TMEM -> registers -> C ----
    mbar_wait(smem_u32(acc_ready), 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = m0 + warp * 32 + lane;
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
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}
