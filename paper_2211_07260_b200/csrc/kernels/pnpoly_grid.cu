// PnPoly with a uniform-cell fast path in front of the exact slab search, sm_100a.
//
// Same bitmap as the brute-force kernel at METHOD 2 (pnpoly.cu) and the slab
// kernel (pnpoly_slab.cu), bit for bit. The host (libjt jt_pnpoly_grid)
// marks a cell of a GRID x GRID raster over the polygon's bounding box clean
// when every edge spanning any py of the cell is decided for every px of the
// cell by its computed-x range (fma(slope, py, icpt) is monotone in py), and
// the crossing parity is the same in every y-slab the cell meets; clean
// cells store that parity. On the benchmark polygon 95% of the points land in
// a clean cell (GRID = 512): for them the answer is one shared-memory lookup.
//
// The other points take the exact x-search of pnpoly_slab.cu (y-slab rank,
// #{lo <= px}, undecided edges along skip pointers), reading the slab table
// through L1 / L2 (it is touched by ~5% of the points). Because a warp's 32
// points rarely are all clean, those points are not searched in place (the
// whole warp would pay the search): each warp appends them to its own queue in
// shared memory (ballot + popc) and searches them 32 at a time with every
// lane busy.
//
// Tunables (-D): BLOCK_SIZE_X, TILE (points per thread per chunk, loaded one
// chunk ahead), GRID (cells per side), GRID_SMEM (1: the 2-bit raster is
// staged in shared memory, GRID^2 / 4 bytes; 0: it is read through L1 from
// global memory, which allows finer rasters and fewer queued points).
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
#define CHUNK (BLOCK_SIZE_X * TILE)
#define NWARPS (BLOCK_SIZE_X / 32)
#define QCAP 64
#define GRID_WORDS ((GRID * GRID + 15) / 16)

// the slab / x-search table of jt_pnpoly_slabs (xbuckets > 0), in global memory
struct SlabTable {
    const float *u;
    const int *guess;
    const float4 *srec;             // per slab {first edge, count, x0, xscale}
    const unsigned short *xst;      // per slab x-bucket starts (bit 15 = exact, unused here)
    const float *xlo, *pmax;        // per edge, sorted by lo within its slab
    const float4 *recs;             // per edge {slope, icpt, hi, skip}
    int nu, ng, xb;
    float ybase, yscale;
};

// The exact search of pnpoly_slab.cu (XSEARCH), loads through the read-only path.
__device__ __forceinline__ int slab_search(float px, float py, const SlabTable &T) {
    if (!(px == px) || !(py == py)) return 0;  // NaN: every compare is false, never inside
    int g = __float2int_rz(__fmul_rn(__fsub_rn(py, T.ybase), T.yscale));
    g = min(max(g, 0), T.ng - 1);
    int r = __ldg(T.guess + g) & 0x7fffffff;
    while (r < T.nu && __ldg(T.u + r) <= py) ++r;
    while (r > 0 && __ldg(T.u + r - 1) > py) --r;
    if (r == 0 || r >= T.nu) return 0;
    const float4 sr = __ldg(T.srec + r);
    const int b = __float_as_int(sr.x), cnt = __float_as_int(sr.y);
    int k = __float2int_rz(__fmul_rn(__fsub_rn(px, sr.z), sr.w));
    k = min(max(k, 0), T.xb);
    int pos = __ldg(T.xst + r * (T.xb + 1) + k) & 0x7fff;
    const float *lo = T.xlo + b;
    while (pos < cnt && __ldg(lo + pos) <= px) ++pos;
    while (pos > 0 && __ldg(lo + pos - 1) > px) --pos;
    int in = (cnt - pos) & 1;
    for (int j = pos - 1; j >= 0 && __ldg(T.pmax + b + j) > px;) {
        const float4 q = __ldg(T.recs + b + j);
        if (q.z > px) in ^= (px < __fmaf_rn(q.x, py, q.y)) ? 1 : 0;
        j = __float_as_int(q.w);
    }
    return in;
}

extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X)
pnpoly_grid(int *__restrict__ bitmap, const float2 *__restrict__ points, int n, const unsigned *__restrict__ grid,
            float gsx, float gox, float gsy, float goy, const float *__restrict__ table, int nu, int ng, int xb,
            float ybase, float yscale, int guess_off, int xpar_off, int xst_off, int xlo_off, int pmax_off,
            int rec_off) {
    extern __shared__ __align__(16) unsigned smem[];
#if GRID_SMEM
    unsigned *s_grid = smem;
    float4 *queue = reinterpret_cast<float4 *>(smem + ((GRID_WORDS + 3) & ~3)) + (threadIdx.x >> 5) * QCAP;
    for (int i = threadIdx.x; i < GRID_WORDS / 4; i += BLOCK_SIZE_X)
        reinterpret_cast<uint4 *>(s_grid)[i] = __ldg(reinterpret_cast<const uint4 *>(grid) + i);
    for (int i = GRID_WORDS / 4 * 4 + threadIdx.x; i < GRID_WORDS; i += BLOCK_SIZE_X) s_grid[i] = __ldg(grid + i);
#define GRID_WORD(w) s_grid[w]
#else
    float4 *queue = reinterpret_cast<float4 *>(smem) + (threadIdx.x >> 5) * QCAP;
#define GRID_WORD(w) __ldg(grid + (w))
#endif
    SlabTable T;
    T.u = table;
    T.guess = reinterpret_cast<const int *>(table + guess_off);
    T.srec = reinterpret_cast<const float4 *>(table + xpar_off);
    T.xst = reinterpret_cast<const unsigned short *>(table + xst_off);
    T.xlo = table + xlo_off;
    T.pmax = table + pmax_off;
    T.recs = reinterpret_cast<const float4 *>(table + rec_off);
    T.nu = nu;
    T.ng = ng;
    T.xb = xb;
    T.ybase = ybase;
    T.yscale = yscale;
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const unsigned lanes_below = (1u << lane) - 1u;
    int queued = 0;  // warp-uniform
    const int n_chunks = (n + CHUNK - 1) / CHUNK;
    float2 nxt[TILE];
    int c = blockIdx.x;
#pragma unroll
    for (int t = 0; t < TILE; ++t) {
        const int i = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
        nxt[t] = (c < n_chunks && i < n) ? points[i] : make_float2(0.f, 0.f);
    }
    for (; c < n_chunks; c += gridDim.x) {
        float2 cur[TILE];
#pragma unroll
        for (int t = 0; t < TILE; ++t) cur[t] = nxt[t];
        const int cn = c + gridDim.x;
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int i = cn * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            nxt[t] = (cn < n_chunks && i < n) ? points[i] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int i = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            const float px = cur[t].x, py = cur[t].y;
            bool slow = false;
            if (i < n) {
                // the host's cell function (jt_pnpoly_grid): min(f2u_rz(fma(v, s, o)), GRID - 1);
                // cvt.rzi.u32 maps NaN and negatives to 0. A NaN coordinate lands in the first
                // column (px) or row (py): a clean cell there has parity 0 (no edge spans below
                // every vertex; every spanning edge crosses left of every vertex, and a closed
                // polygon has an even number of them), which is the answer for NaN; an unclean
                // one sends the point to slab_search, which returns 0.
                const unsigned cx = min(__float2uint_rz(__fmaf_rn(px, gsx, gox)), GRID - 1u);
                const unsigned cy = min(__float2uint_rz(__fmaf_rn(py, gsy, goy)), GRID - 1u);
                const unsigned cell = cy * GRID + cx;
                const unsigned code = (GRID_WORD(cell >> 4) >> ((cell & 15u) * 2u)) & 3u;
                slow = !(code & 1u);
                if (!slow) bitmap[i] = (int)(code >> 1);
            }
            // queue the undecided points of this warp; search 32 at a time
            const unsigned need = __ballot_sync(0xffffffffu, slow);
            if (need) {
                if (slow)
                    queue[queued + __popc(need & lanes_below)] = make_float4(px, py, __int_as_float(i), 0.f);
                queued += __popc(need);
                __syncwarp();
                if (queued >= 32) {
                    const float4 e = queue[lane];
                    bitmap[__float_as_int(e.z)] = slab_search(e.x, e.y, T);
                    __syncwarp();
                    if (lane < queued - 32) queue[lane] = queue[32 + lane];
                    __syncwarp();
                    queued -= 32;
                }
            }
        }
    }
    if (lane < queued) {  // the warp's leftovers
        const float4 e = queue[lane];
        bitmap[__float_as_int(e.z)] = slab_search(e.x, e.y, T);
    }
}
