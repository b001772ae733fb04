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
// ring slots per warp (a power of two): < 32 left after a drain + 2 x 32 pushed per pair
#define QCAP (TILE <= 1 ? 128 : TILE <= 2 ? 256 : TILE <= 6 ? 512 : 1024)
#define GRID_WORDS ((GRID * GRID + 15) / 16)

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

// the host's cell function (jt_pnpoly_cells): min(f2u_rz(fma(v, s, o)), GRID - 1); cvt.rzi.u32
// maps NaN and negatives to 0, so NaN lands in row / column 0 (whose clean cells hold 0)
__device__ __forceinline__ unsigned cell_of(float px, float py, float gsx, float gox, float gsy, float goy) {
    const unsigned cx = min(__float2uint_rz(__fmaf_rn(px, gsx, gox)), GRID - 1u);
    const unsigned cy = min(__float2uint_rz(__fmaf_rn(py, gsy, goy)), GRID - 1u);
    return cy * GRID + cx;
}

// one undecided point of the drain: reload it (L1 / L2: its line was read moments ago),
// redo its cell and code, answer it
#define DRAIN_ONE(idx)                                                                      \
    do {                                                                                    \
        const float2 p_ = points[idx];                                                      \
        const unsigned cell_ = cell_of(p_.x, p_.y, gsx, gox, gsy, goy);                     \
        const unsigned w_ = GRID_WORD(cell_ >> 4);                                          \
        const unsigned code_ = __funnelshift_r(w_, w_, cell_ * 2u) & 3u;                    \
        bitmap[idx] = cell_search(p_.x, p_.y, cell_, code_, heads, edges, SLAB_ARGS);       \
    } while (0)

// full occupancy (2048 threads per SM) needs <= 32 registers per thread
extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X, 2048 / BLOCK_SIZE_X)
pnpoly_cells(int *__restrict__ bitmap, const float2 *__restrict__ points, int n, const unsigned *__restrict__ grid,
             const uint2 *__restrict__ heads, const float4 *__restrict__ edges, float gsx, float gox, float gsy,
             float goy, SLAB_PARAMS) {
    extern __shared__ __align__(16) unsigned smem[];
#if GRID_SMEM
    unsigned *s_grid = smem;
    int *ring = reinterpret_cast<int *>(smem + ((GRID_WORDS + 3) & ~3)) + (threadIdx.x >> 5) * QCAP;
    for (int i = threadIdx.x; i < GRID_WORDS / 4; i += BLOCK_SIZE_X)
        reinterpret_cast<uint4 *>(s_grid)[i] = __ldg(reinterpret_cast<const uint4 *>(grid) + i);
    for (int i = GRID_WORDS / 4 * 4 + threadIdx.x; i < GRID_WORDS; i += BLOCK_SIZE_X) s_grid[i] = __ldg(grid + i);
    __syncthreads();
#define GRID_WORD(w) s_grid[w]
#else
    int *ring = reinterpret_cast<int *>(smem) + (threadIdx.x >> 5) * QCAP;
#define GRID_WORD(w) __ldg(grid + (w))
#endif
    const float4 *pairs = reinterpret_cast<const float4 *>(points);
    int2 *out = reinterpret_cast<int2 *>(bitmap);
    const int full = n >> 1, npairs = (n + 1) >> 1;  // pair q = points 2q, 2q + 1; an odd tail pair
    const int lane = threadIdx.x & 31;
    const unsigned lanes_below = (1u << lane) - 1u;
    // per-warp ring of undecided point indices: pushed at tail during a chunk, drained 32 at
    // a time from head at its end (warp-uniform counters; < 32 left after a drain, so a
    // chunk's <= 64 TILE pushes never reach the slots the last drain read). Nothing but
    // loop counters is live across the drain: the chunk's loads are issued after it.
    unsigned head = 0, tail = 0;
    const int n_chunks = (npairs + CHUNK - 1) / CHUNK;
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        float4 cur[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            if (q < full) cur[t] = LOAD_PAIR(pairs + q);
            else if (q < npairs) {
                const float2 p = points[2 * q];
                cur[t] = make_float4(p.x, p.y, 0.f, 0.f);
            } else cur[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            const unsigned c0 = cell_of(cur[t].x, cur[t].y, gsx, gox, gsy, goy);
            const unsigned c1 = cell_of(cur[t].z, cur[t].w, gsx, gox, gsy, goy);
            const unsigned w0 = GRID_WORD(c0 >> 4), w1 = GRID_WORD(c1 >> 4);
            const unsigned k0 = __funnelshift_r(w0, w0, c0 * 2u) & 3u, k1 = __funnelshift_r(w1, w1, c1 * 2u) & 3u;
            // codes 0 / 1: the answer; 2: listed edges; 3: slab search. Undecided points get a
            // placeholder here and their answer from a later drain of the same warp.
            if (q < full) STORE_PAIR(out + q, make_int2((int)(k0 & 1u), (int)(k1 & 1u)));
            else if (q < npairs) bitmap[2 * q] = (int)(k0 & 1u);
            const bool s0 = q < npairs && (k0 & 2u), s1 = q < full && (k1 & 2u);
            const unsigned need0 = __ballot_sync(0xffffffffu, s0), need1 = __ballot_sync(0xffffffffu, s1);
            if (need0 | need1) {
                if (s0) ring[(tail + __popc(need0 & lanes_below)) % QCAP] = 2 * q;
                tail += __popc(need0);
                if (s1) ring[(tail + __popc(need1 & lanes_below)) % QCAP] = 2 * q + 1;
                tail += __popc(need1);
            }
        }
        __syncwarp();
        while (tail - head >= 32u) {
            const int idx = ring[(head + lane) % QCAP];
            head += 32;
            DRAIN_ONE(idx);
        }
    }
    if (lane < tail - head) {  // the warp's leftovers
        const int idx = ring[(head + lane) % QCAP];
        DRAIN_ONE(idx);
    }
}
