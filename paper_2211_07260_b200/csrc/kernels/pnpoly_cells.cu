// PnPoly with per-cell edge lists, sm_100a.
//
// Same bitmap as the brute-force kernel at METHOD 2 (pnpoly.cu), bit for bit.
// The host (libjt jt_pnpoly_cells) classifies every edge for every cell of a
// GRID x GRID raster over the polygon's bounding box: its METHOD 2 test is
// false for every point of the cell, true for every point, or undecided. A
// cell whose edges are all decided stores its parity (2 bits per cell, staged
// in shared memory): on the benchmark polygon 92% of the points are answered
// by that one lookup. An undecided cell lists its undecided edges (1.3 on
// average at GRID = 512) with the parity of the always-true ones; its points
// are queued per warp and answered by base ^ their listed tests (two dependent
// L2 reads: the cell head, then its edges). Cells with more than `lmax`
// undecided edges fall back to the exact slab search of pnpoly_slab.cu.
//
// Memory side: two points per 16-byte load and two results per 8-byte store,
// TILE pairs per thread in flight per chunk. The kernel is HBM bound
// when the lookup path issues few enough instructions; 8 bytes read and 4
// written per point are its algorithmic traffic.
//
// Tunables (-D): BLOCK_SIZE_X, TILE (point pairs per thread per chunk), GRID
// (cells per side), GRID_SMEM (1: raster in shared memory; 0: read through L1),
// STREAM (1: points loaded / results stored with the evict-first hints).
#ifndef BLOCK_SIZE_X
#define BLOCK_SIZE_X 1024
#endif
#ifndef TILE
#define TILE 2
#endif
#ifndef GRID
#define GRID 512
#endif
#ifndef GRID_SMEM
#define GRID_SMEM 1
#endif
#ifndef STREAM
#define STREAM 0
#endif
#define CHUNK (BLOCK_SIZE_X * TILE)
// ring slots per warp (a power of two): < 32 left after a drain + 32 pushed per pair step
#define QCAP (TILE <= 3 ? 128 : 256)

#if STREAM
#define LOAD_PAIR(p) __ldcs(p)
#define STORE_PAIR(p, v) __stcs(p, v)
#else
#define LOAD_PAIR(p) __ldg(p)
#define STORE_PAIR(p, v) (*(p) = (v))
#endif

// The exact search of pnpoly_slab.cu (XSEARCH) over the slab / x-search table of
// jt_pnpoly_slabs (xbuckets > 0) in global memory, loads through the read-only path. The
// table fields are the kernel's parameters (constant bank), not registers.
#define SLAB_PARAMS const float *__restrict__ table, int nu, int ng, int xb, float ybase, float yscale, \
    int guess_off, int xpar_off, int xst_off, int xlo_off, int pmax_off, int rec_off
#define SLAB_ARGS table, nu, ng, xb, ybase, yscale, guess_off, xpar_off, xst_off, xlo_off, pmax_off, rec_off
__device__ __forceinline__ int slab_search(float px, float py, SLAB_PARAMS) {
    if (!(px == px) || !(py == py)) return 0;  // NaN: every compare is false, never inside
    const float *u = table;
    int g = __float2int_rz(__fmul_rn(__fsub_rn(py, ybase), yscale));
    g = min(max(g, 0), ng - 1);
    int r = __ldg(reinterpret_cast<const int *>(table + guess_off) + g) & 0x7fffffff;
    while (r < nu && __ldg(u + r) <= py) ++r;
    while (r > 0 && __ldg(u + r - 1) > py) --r;
    if (r == 0 || r >= nu) return 0;
    const float4 sr = __ldg(reinterpret_cast<const float4 *>(table + xpar_off) + r);  // {first, count, x0, xscale}
    const int b = __float_as_int(sr.x), cnt = __float_as_int(sr.y);
    int k = __float2int_rz(__fmul_rn(__fsub_rn(px, sr.z), sr.w));
    k = min(max(k, 0), xb);
    int pos = __ldg(reinterpret_cast<const unsigned short *>(table + xst_off) + r * (xb + 1) + k) & 0x7fff;
    const float *lo = table + xlo_off + b, *pmax = table + pmax_off + b;
    const float4 *recs = reinterpret_cast<const float4 *>(table + rec_off) + b;  // {slope, icpt, hi, skip}
    while (pos < cnt && __ldg(lo + pos) <= px) ++pos;
    while (pos > 0 && __ldg(lo + pos - 1) > px) --pos;
    int in = (cnt - pos) & 1;
    for (int j = pos - 1; j >= 0 && __ldg(pmax + j) > px;) {
        const float4 q = __ldg(recs + j);
        if (q.z > px) in ^= (px < __fmaf_rn(q.x, py, q.y)) ? 1 : 0;
        j = __float_as_int(q.w);
    }
    return in;
}

// A queued point: base parity ^ the listed edges' METHOD 2 tests (ylo <= py < yhi is the
// y-test (vy_k > py) != (vy_j > py)), or the slab search for a code-3 cell.
__device__ __forceinline__ int cell_search(float px, float py, unsigned cell, unsigned code,
                                           const uint2 *__restrict__ heads, const float4 *__restrict__ edges,
                                           SLAB_PARAMS) {
    if (code == 3u) return slab_search(px, py, SLAB_ARGS);
    if (!(px == px) || !(py == py)) return 0;
    const uint2 h = __ldg(heads + cell);
    int in = h.y & 1;
    const int cnt = h.y >> 1;
    for (int k = 0; k < cnt; ++k) {
        const float4 q = __ldg(edges + h.x + k);
        in ^= (q.z <= py && py < q.w && px < __fmaf_rn(q.x, py, q.y)) ? 1 : 0;
    }
    return in;
}

// The host's cell function (jt_pnpoly_cells): min(f2u_rz(fma(v, s, o)), GRID - 1); cvt.rzi.u32
// maps NaN and negatives to 0, so NaN lands in row / column 0 (whose decided cells hold 0).
// The raster holds two bit planes per 32 cells of a row ({code & 1, code >> 1} words), so a
// point's code is one 8-byte lookup and two rotates by cx (mod 32).
struct Code {
    unsigned lo, hi;  // bit 0: code & 1 (the answer, or the fallback flag), code >> 1 (undecided)
};
#if GRID_SMEM
#define GRID_PAIR(i) s_grid[i]
#else
#define GRID_PAIR(i) __ldg(grid + (i))
#endif
#define CODE_OF(px, py, out)                                                                 \
    do {                                                                                     \
        const unsigned cx_ = min(__float2uint_rz(__fmaf_rn(px, gsx, gox)), GRID - 1u);        \
        const unsigned cy_ = min(__float2uint_rz(__fmaf_rn(py, gsy, goy)), GRID - 1u);        \
        const uint2 w_ = GRID_PAIR(cy_ * (GRID / 32) + (cx_ >> 5));                           \
        (out).lo = __funnelshift_r(w_.x, w_.x, cx_);                                          \
        (out).hi = __funnelshift_r(w_.y, w_.y, cx_);                                          \
        cell_ = cy_ * GRID + cx_;                                                            \
    } while (0)

// full occupancy (2048 threads per SM) needs <= 32 registers per thread
extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X, 2048 / BLOCK_SIZE_X)
pnpoly_cells(int *__restrict__ bitmap, const float2 *__restrict__ points, int n, const uint2 *__restrict__ grid,
             const uint2 *__restrict__ heads, const float4 *__restrict__ edges, float gsx, float gox, float gsy,
             float goy, SLAB_PARAMS) {
    extern __shared__ __align__(16) unsigned smem[];
#if GRID_SMEM
    constexpr int GRID_PAIRS = GRID * GRID / 32;
    uint2 *s_grid = reinterpret_cast<uint2 *>(smem);
    int *ring = reinterpret_cast<int *>(smem + 2 * GRID_PAIRS) + (threadIdx.x >> 5) * QCAP;
    for (int i = threadIdx.x; i < GRID_PAIRS / 2; i += BLOCK_SIZE_X)
        reinterpret_cast<uint4 *>(s_grid)[i] = __ldg(reinterpret_cast<const uint4 *>(grid) + i);
    __syncthreads();
#else
    int *ring = reinterpret_cast<int *>(smem) + (threadIdx.x >> 5) * QCAP;
#endif
    const float4 *pairs = reinterpret_cast<const float4 *>(points);
    int2 *out = reinterpret_cast<int2 *>(bitmap);
    const int full = n >> 1, npairs = (n + 1) >> 1;  // pair q = points 2q, 2q + 1; an odd tail pair
    const int lane = threadIdx.x & 31;
    unsigned lanes_below;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lanes_below));
    // Per-warp ring of pairs with an undecided point: pushed at tail during a chunk, drained
    // 32 at a time from head at its end (warp-uniform counters; < 32 left after a drain, so
    // a chunk's <= 32 TILE pushes never reach the slots the last drain read). Nothing but
    // loop counters is live across the drain: the chunk's loads are issued after it.
    unsigned head = 0, tail = 0;
    const int n_chunks = (npairs + CHUNK - 1) / CHUNK;
    auto chunk = [&](int c, const bool FULL) {  // inlined twice with FULL constant
        float4 cur[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            if (FULL || q < full) cur[t] = LOAD_PAIR(pairs + q);
            else if (q < npairs) {
                const float2 p = points[2 * q];
                cur[t] = make_float4(p.x, p.y, 0.f, 0.f);
            } else cur[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            Code k0, k1;
            unsigned cell_;
            CODE_OF(cur[t].x, cur[t].y, k0);
            CODE_OF(cur[t].z, cur[t].w, k1);
            // decided points get their answer here; a pair with an undecided point is queued
            // and both its points are rewritten by a later drain of the same warp
            if (FULL || q < full) STORE_PAIR(out + q, make_int2((int)(k0.lo & 1u), (int)(k1.lo & 1u)));
            else if (q < npairs) bitmap[2 * q] = (int)(k0.lo & 1u);
            const bool slow = (FULL || q < npairs) && ((k0.hi | k1.hi) & 1u);
            const unsigned need = __ballot_sync(0xffffffffu, slow);
            if (slow) ring[(tail + __popc(need & lanes_below)) % QCAP] = q;
            tail += __popc(need);
        }
    };
    // one queued pair: both points redone, the undecided ones searched
    auto drain = [&](int q) {
        float4 v;
        if (q < full) v = __ldg(pairs + q);
        else { const float2 p = points[2 * q]; v = make_float4(p.x, p.y, 0.f, 0.f); }
        Code k;
        unsigned cell_;
        CODE_OF(v.x, v.y, k);
        const int r0 = (k.hi & 1u) ? cell_search(v.x, v.y, cell_, 2u | (k.lo & 1u), heads, edges, SLAB_ARGS)
                                   : (int)(k.lo & 1u);
        if (q < full) {
            CODE_OF(v.z, v.w, k);
            const int r1 = (k.hi & 1u) ? cell_search(v.z, v.w, cell_, 2u | (k.lo & 1u), heads, edges, SLAB_ARGS)
                                       : (int)(k.lo & 1u);
            out[q] = make_int2(r0, r1);
        } else bitmap[2 * q] = r0;
    };
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        if ((c + 1) * CHUNK <= full) chunk(c, true);
        else chunk(c, false);
        __syncwarp();
        while (tail - head >= 32u) {
            const int q = ring[(head + lane) % QCAP];
            head += 32;
            drain(q);
        }
    }
    if (lane < tail - head) drain(ring[(head + lane) % QCAP]);  // the warp's leftovers
}
