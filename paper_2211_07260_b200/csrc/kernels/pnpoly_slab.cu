// PnPoly by y-slab point location, sm_100a, compiled per config by NVRTC.
//
// Same output as the brute-force kernel (pnpoly.cu) at METHOD 2, bit for bit:
// bitmap[i] = parity of #{edges k : (vy_k > py) != (vy_j > py) and
// px < fma(slope_k, py, icpt_k)}. The brute-force loop spends ~3 issue slots
// on each of the 600 edges for every point, although a horizontal line meets
// only ~20 of them. Here the host (libjt jt_pnpoly_slabs) sorts the distinct
// vertex ordinates u[0..nu) once; for a point, r = #{u <= py} names its slab,
// and exactly the edges listed for slab r satisfy the y-test for every py in
// [u[r-1], u[r]) (every other edge fails it for every such py). The x-test
// and the parity are then the brute-force kernel's, edge for edge, on the same
// float32 slope / intercept bits, so the bitmap is identical; only the edges
// whose crossing bit is necessarily 0 are skipped.
//
// Per point: a bucket lookup gives a starting rank, corrected by exact float
// compares (typically 0-2 steps); then one FFMA + FADD per listed edge and
// one LOP3 per two (slab lists are padded to a multiple of 4 with {0, -inf},
// which never toggles).
//
// Tunables (-D):
//   BLOCK_SIZE_X  threads per block (persistent grid: each CTA stages the
//                 table once and strides over point chunks)
//   TILE          points per thread per chunk (chunk = BLOCK_SIZE_X * TILE)
//   SORT          0: each thread walks its own points' slabs (lanes of a warp
//                    sit in random slabs: the warp pays the longest list)
//                 1: counting sort of the chunk by slab in shared memory
//                    (smem histogram + block scan + scatter), so a warp's 32
//                    lanes walk the same or neighbouring slabs (uniform trip
//                    counts, broadcast table reads); results go back through
//                    shared memory for a coalesced store
//   PAIRS_SMEM    1: slab edge lists staged in shared memory; 0: read through
//                 L1 (ld.global.nc)
//   XSEARCH       1: no edge loop at all (SORT / PAIRS_SMEM unused). The
//                 slab's edges come sorted by lo, the smallest computed
//                 crossing abscissa over the slab (fma(slope, py, icpt) is
//                 monotone in py, so lo / hi are its two end values, computed
//                 by the host with the same fmaf). Edges with lo > px cross
//                 for every py of the slab, edges with hi <= px for none, so
//                 parity = (#{lo > px} + crossings among lo <= px < hi) & 1.
//                 pos = #{lo <= px} comes from a per-slab uniform x-bucket
//                 (the table's xbuckets), exact where no lo falls inside the
//                 bucket (flagged by the host), else corrected by compares;
//                 the slab rank likewise comes from a y-bucket
//                 (EXACT_FLAGS=0: ignore the host's exactness flags and
//                 always run the correcting compares); HALF=1 stages lo / pmax
//                 as binary16 rounded down / up (half the shared memory, two
//                 CTAs per SM): a too-small lo or too-large pmax only sends more
//                 edges through the exact re-evaluation, so the bitmap is
//                 unchanged;
//                 the undecided edges (about 0.05 per point on the benchmark
//                 polygon) are found by walking back from pos while the
//                 running max of hi (pmax) exceeds px, jumping along each
//                 record's skip pointer (the next lower edge whose hi exceeds
//                 this edge's lo), and are evaluated with the brute-force
//                 formula.
#ifndef BLOCK_SIZE_X
#define BLOCK_SIZE_X 512
#endif
#ifndef TILE
#define TILE 4
#endif
#ifndef SORT
#define SORT 1
#endif
#ifndef PAIRS_SMEM
#define PAIRS_SMEM 0
#endif
#ifndef XSEARCH
#define XSEARCH 0
#endif
#ifndef EXACT_FLAGS
#define EXACT_FLAGS 1
#endif
#ifndef HALF
#define HALF 0
#endif
#if XSEARCH && (SORT || PAIRS_SMEM)
#error "XSEARCH=1 takes SORT=0 and PAIRS_SMEM=0"
#endif
#define CHUNK (BLOCK_SIZE_X * TILE)
#define NWARPS (BLOCK_SIZE_X / 32)

__device__ __forceinline__ int slab_of(float py, const float *u, const int *guess, int nu, int ng, float ybase,
                                       float yscale) {
    if (!(py == py)) return 0;  // NaN: every y-compare is false, no edge spans
    // any starting rank will do: the two loops below make it exact
    int g = __float2int_rz((py - ybase) * yscale);
    g = min(max(g, 0), ng - 1);
    const int gv = guess[g];  // bit 31: the rank is exact for every py of this bucket
    int r = gv & 0x7fffffff;
    if (gv < 0) return r;
    while (r < nu && u[r] <= py) ++r;
    while (r > 0 && u[r - 1] > py) --r;
    return r;
}

// Parity of the slab's crossings, 4 edges (two 16-byte {slope, icpt} pairs)
// per trip. The compare px < x is taken as the sign bit of the exactly
// rounded difference px' - x with px' = px + 0.0f: rounding keeps the sign of
// a nonzero difference and x - y == +0 iff x == y, and adding +0.0 turns a
// -0.0 abscissa into +0.0, the one case where signbit(px - x) != (px < x).
// (The {0, -inf} fillers give px' - (-inf) = +inf: no toggle.)
__device__ __forceinline__ int slab_parity(float px, float py, const float4 *pairs4, int b, int e) {
    const float pxc = __fadd_rn(px, 0.0f);
    unsigned acc = 0u;
    for (int j = b >> 1; j < (e >> 1); j += 2) {
#if PAIRS_SMEM
        const float4 p = pairs4[j], q = pairs4[j + 1];
#else
        const float4 p = __ldg(pairs4 + j), q = __ldg(pairs4 + j + 1);
#endif
        const unsigned e0 = __float_as_uint(__fsub_rn(pxc, __fmaf_rn(p.x, py, p.y)));
        const unsigned e1 = __float_as_uint(__fsub_rn(pxc, __fmaf_rn(p.z, py, p.w)));
        const unsigned e2 = __float_as_uint(__fsub_rn(pxc, __fmaf_rn(q.x, py, q.y)));
        const unsigned e3 = __float_as_uint(__fsub_rn(pxc, __fmaf_rn(q.z, py, q.w)));
        acc ^= e0 ^ e1 ^ e2 ^ e3;
    }
    return (int)(acc >> 31);
}

#if SORT
// exclusive prefix sum of a[0..m) in place (one block); returns the total
__device__ __forceinline__ int block_exclusive_scan(int *a, int m, int *warp_tot) {
    const int per = (m + BLOCK_SIZE_X - 1) / BLOCK_SIZE_X;
    const int lo = min(m, (int)threadIdx.x * per), hi = min(m, lo + per);
    int sum = 0;
    for (int k = lo; k < hi; ++k) sum += a[k];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < NWARPS ? warp_tot[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += v;
        }
        if (lane < NWARPS) warp_tot[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    int run = incl - sum + (warp ? warp_tot[warp - 1] : 0);
    for (int k = lo; k < hi; ++k) {
        const int c = a[k];
        a[k] = run;
        run += c;
    }
    return warp_tot[NWARPS - 1];
}
#endif

#if XSEARCH
// 32-bit shared-window loads: the tables live at runtime offsets of the
// dynamic shared array, so plain pointers would be generic and re-derive the
// window base at every access.
__device__ __forceinline__ float lds_f32(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_u16(unsigned a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_f16(unsigned a) {
    float v;
    asm volatile("{\n.reg .b16 h;\nld.shared.b16 h, [%1];\ncvt.f32.f16 %0, h;\n}" : "=f"(v) : "r"(a));
    return v;
}
#if HALF
#define LO_AT(i) lds_f16(T.xlo + 4u * (i))
#define PMAX_AT(i) lds_f16(T.xlo + 4u * (i) + 2u)
#else
#define LO_AT(i) lds_f32(T.xlo + 4u * (i))
#define PMAX_AT(i) lds_f32(T.pmax + 4u * (i))
#endif
__device__ __forceinline__ float4 lds_f32x4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

struct XTables {
    unsigned u, guess, band, xpar, xst, xlo, pmax;  // shared-window byte addresses
    int nu, ng, xb;
    float ybase, yscale;
    const float4 *recs;  // {slope, icpt, hi, 0} per slab edge (global, rarely read)
};

// One point: slab by rank, #{lo <= px} by x-bucket + exact correction, then
// the undecided edges. Returns the crossing parity (the brute-force bit).
__device__ __forceinline__ int xsearch_point(float px, float py, const XTables &T) {
    if (!(px == px) || !(py == py)) return 0;  // NaN: every compare is false
    int g = __float2int_rz(__fmul_rn(__fsub_rn(py, T.ybase), T.yscale));
    g = min(max(g, 0), T.ng - 1);
    const int gv = lds_s32(T.guess + 4u * g);  // bit 31: the rank is exact for this bucket
    int r = gv & 0x7fffffff;
    if (!EXACT_FLAGS || gv >= 0) {
        while (r < T.nu && lds_f32(T.u + 4u * r) <= py) ++r;
        while (r > 0 && lds_f32(T.u + 4u * r - 4u) > py) --r;
    }
    if (r == 0 || r >= T.nu) return 0;  // below / above every vertex: no edge spans
    const float4 sr = lds_f32x4(T.xpar + 16u * r);  // {first edge, count, x0, xscale}
    const int b = __float_as_int(sr.x), cnt = __float_as_int(sr.y);
    int k = __float2int_rz(__fmul_rn(__fsub_rn(px, sr.z), sr.w));
    k = min(max(k, 0), T.xb);
    const int w = lds_u16(T.xst + 2u * (r * (T.xb + 1) + k));  // bit 15: pos is exact
    int pos = w & 0x7fff;
    if (!EXACT_FLAGS || !(w & 0x8000)) {
        while (pos < cnt && LO_AT(b + pos) <= px) ++pos;
        while (pos > 0 && LO_AT(b + pos - 1) > px) --pos;
    }
    int in = (cnt - pos) & 1;  // lo > px: crosses for every py of the slab
    // undecided: lo <= px < hi; pmax[j] = max hi over the slab's first j+1 edges
    // (the walk follows each record's skip pointer: the next lower edge whose hi can exceed px)
    for (int j = pos - 1; j >= 0 && PMAX_AT(b + j) > px;) {
        const float4 q = __ldg(T.recs + b + j);  // {slope, icpt, hi, skip}
        if (q.z > px) in ^= (px < __fmaf_rn(q.x, py, q.y)) ? 1 : 0;
        j = __float_as_int(q.w);
    }
    return in;
}
#endif

extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X)
pnpoly_slab(int *__restrict__ bitmap, const float2 *__restrict__ points, int n, const float *__restrict__ table,
            int nu, int ng, int band_off, int pair_off, int staged_words, float ybase, float yscale,
            int xlo_off, int pmax_off, int xpar_off, int xst_off, int xb, int arr_off, int arr_words) {
    // stage table words [0, staged_words), then [arr_off, arr_off + arr_words) right after them
    // (x-search: the lo / pmax arrays of the chosen precision); xlo_off / pmax_off are
    // shared-memory word offsets
    extern __shared__ __align__(16) float smem[];
    for (int i = threadIdx.x; i < staged_words / 4; i += BLOCK_SIZE_X)
        reinterpret_cast<float4 *>(smem)[i] = __ldg(reinterpret_cast<const float4 *>(table) + i);
    for (int i = threadIdx.x; i < arr_words / 4; i += BLOCK_SIZE_X)
        reinterpret_cast<float4 *>(smem)[staged_words / 4 + i] = __ldg(reinterpret_cast<const float4 *>(table) + arr_off / 4 + i);
    const float *u = smem;
    const int *guess = reinterpret_cast<const int *>(smem + ((nu + 3) & ~3));
    const int *band = reinterpret_cast<const int *>(smem + band_off);
#if XSEARCH
    const unsigned s0 = (unsigned)__cvta_generic_to_shared(smem);
    XTables T;
    T.u = s0;
    T.guess = s0 + 4u * ((nu + 3) & ~3);
    T.band = s0 + 4u * band_off;
    T.xpar = s0 + 4u * xpar_off;
    T.xst = s0 + 4u * xst_off;
    T.xlo = s0 + 4u * xlo_off;
    T.pmax = s0 + 4u * pmax_off;
    T.nu = nu;
    T.ng = ng;
    T.xb = xb;
    T.ybase = ybase;
    T.yscale = yscale;
    T.recs = reinterpret_cast<const float4 *>(table + pair_off);
    __syncthreads();
    // 32-bit indices (n < 2^31); the next chunk's points are loaded into
    // registers before this chunk is computed, so the loads overlap the search
    const int n_chunks = (n + CHUNK - 1) / CHUNK;
    float2 q[TILE];
    int c = blockIdx.x;
#pragma unroll
    for (int t = 0; t < TILE; ++t) {
        const int i = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
        q[t] = (c < n_chunks && i < n) ? points[i] : make_float2(0.f, 0.f);
    }
    for (; c < n_chunks; c += gridDim.x) {
        float2 cur[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) cur[t] = q[t];
        const int cn = c + gridDim.x;
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int i = cn * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            q[t] = (cn < n_chunks && i < n) ? points[i] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int i = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            if (i < n) bitmap[i] = xsearch_point(cur[t].x, cur[t].y, T);
        }
    }
#else
#if PAIRS_SMEM
    const float4 *pairs = reinterpret_cast<const float4 *>(smem + pair_off);
#else
    const float4 *pairs = reinterpret_cast<const float4 *>(table + pair_off);
#endif
#if SORT
    __shared__ int warp_tot[32];
    int *hist = reinterpret_cast<int *>(smem + staged_words + arr_words);  // nu + 1 counters
    float4 *sorted = reinterpret_cast<float4 *>(hist + ((nu + 4) & ~3));  // CHUNK records
    int *result = reinterpret_cast<int *>(sorted + CHUNK);                 // CHUNK results
#endif
    __syncthreads();

    const long long n_chunks = ((long long)n + CHUNK - 1) / CHUNK;
    for (long long c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const long long base = c * CHUNK;
        float px[TILE], py[TILE];
        int r[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const long long i = base + t * BLOCK_SIZE_X + threadIdx.x;
            const float2 q = i < n ? points[i] : make_float2(0.f, 0.f);
            px[t] = q.x;
            py[t] = q.y;
            r[t] = i < n ? slab_of(q.y, u, guess, nu, ng, ybase, yscale) : 0;
        }
#if !SORT
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const long long i = base + t * BLOCK_SIZE_X + threadIdx.x;
            if (i < n) bitmap[i] = slab_parity(px[t], py[t], pairs, band[r[t]], band[r[t] + 1]);
        }
#else
        for (int k = threadIdx.x; k <= nu; k += BLOCK_SIZE_X) hist[k] = 0;
        __syncthreads();
        int slot[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) slot[t] = (r[t] > 0 && r[t] < nu) ? atomicAdd(&hist[r[t]], 1) : -1;
        __syncthreads();
        const int total = block_exclusive_scan(hist, nu + 1, warp_tot);
        __syncthreads();
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int local = t * BLOCK_SIZE_X + threadIdx.x;
            if (slot[t] >= 0)
                sorted[hist[r[t]] + slot[t]] = make_float4(px[t], py[t], __int_as_float(local), __int_as_float(r[t]));
            else
                result[local] = 0;  // outside every slab's y-range: no edge spans
        }
        __syncthreads();
        for (int k = threadIdx.x; k < total; k += BLOCK_SIZE_X) {
            const float4 s = sorted[k];
            const int rr = __float_as_int(s.w);
            result[__float_as_int(s.z)] = slab_parity(s.x, s.y, pairs, band[rr], band[rr + 1]);
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const long long i = base + t * BLOCK_SIZE_X + threadIdx.x;
            if (i < n) bitmap[i] = result[t * BLOCK_SIZE_X + threadIdx.x];
        }
        __syncthreads();  // hist / sorted / result are reused by the next chunk
#endif
    }
#endif  // XSEARCH
}
