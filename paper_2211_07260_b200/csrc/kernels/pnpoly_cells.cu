// PnPoly with per-cell edge lists, sm_100a.
//
// Same bitmap as the brute-force kernel at METHOD 2 (pnpoly.cu), bit for bit.
// The host (libjt jt_pnpoly_cells) classifies every edge for every cell of a
// GRID x GRID raster over the polygon's bounding box: its METHOD 2 test is
// false for every point of the cell, true for every point, or undecided. A
// cell whose edges are all decided stores its parity (2 bits per cell, staged
// in shared memory): on the benchmark polygon 94-95% of the points are
// answered by that one lookup. An undecided cell lists its undecided edges
// (1.3 on average at GRID = 512); its points are queued per warp with their
// coordinates and answered 32 at a time by base ^ their listed tests: one head
// read per point (16 bytes holding one edge in place, or 32 bytes holding two
// with HEAD32), more only for cells with more edges. Cells with more than
// `lmax` undecided edges fall back to the exact slab search of pnpoly_slab.cu.
//
// Memory side: two points per 16-byte load and two results per 8-byte store
// (QUAD: four per 32-byte LDG.E.256 load and 16-byte store), TILE vectors per
// thread per chunk. The raster lookups cost nothing measurable
// (scripts/cells_floor.py); the queued points' dependent head reads are the
// cost above the loop's own floor, hence in-place edges and the split drain.
//
// Tunables (-D): BLOCK_SIZE_X, TILE (point vectors per thread per chunk), QUAD, GRID
// (cells per side), GRID_SMEM (1: raster in shared memory; 0: read through L1),
// STREAM (1: points loaded / results stored with the evict-first hints; 2: points loaded with
// L1::no_allocate), PREFETCH
// (chunks ahead that one thread of the block pulls into L2 with
// cp.async.bulk.prefetch: the block's points are one contiguous span per chunk,
// so the next chunk's HBM latency overlaps this chunk's work without holding
// registers), REGPF (1: the next chunk's vectors are loaded into registers before
// this chunk is classified; 2: the same with two buffers swapping roles, no copies), ADRAIN (1: split drains, the heads fetched by
// cp.async and tested at the next drain), HEAD32 (32-byte heads), HPF (a queued point's
// cell head prefetched into L1, so its drain read hits L1), PUSHV (one warp prefix per point
// vector for the ring pushes), RING16 (16-byte ring records), MIN_BLOCKS. Tried and
// dropped: a 2-4 stage shared-memory ring filled by cp.async.bulk from one
// producer thread (67 us and up: the producer waits for every warp to free a
// stage, which couples the warps).
//
// DEFER (1): no ring. ncu on the ring kernel (profiles/r1_pnpoly_cells_tuned) counts ~56
// thread instructions per point at 71% issue: the per-point ballot / prefix / push and the
// drain bookkeeping cost more than the lookup itself, and the 32-register cap makes the
// compiler re-read constants and thread ids inside the loop. With DEFER every thread keeps
// up to two undecided points of its own pending in registers: their head loads are issued
// when the points are classified and consumed one step later (the next step's point loads
// and lookups cover the L2 latency), so an undecided point costs a divergent head load, a
// test and a 4-byte store, and a decided one nothing beyond its lookup. A third undecided
// point in one step (rare) is resolved on the spot. MIN_BLOCKS (1: one block per SM with
// up to 64 registers) sets the launch bounds.
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
#ifndef PREFETCH
#define PREFETCH 1
#endif
#ifndef REGPF
#define REGPF 0
#endif
#ifndef QUAD
#define QUAD 0  // 1: four points per 32-byte load (LDG.E.256) and four results per 16-byte store
#endif
#define PPV (2 + 2 * QUAD)  // points per vector load
#define CHUNK (BLOCK_SIZE_X * TILE)  // vectors per block per chunk
#ifndef ADRAIN
#define ADRAIN 1
#endif
#ifndef HEAD32
#define HEAD32 0  // 1: 32-byte heads holding up to two undecided edges in place
#endif
#ifndef DEFER
#define DEFER 0
#endif
#ifndef HPF
#define HPF 0  // 1: an undecided point's cell head is prefetched into L1 when it is queued
#endif
#define HW (1 + HEAD32)  // float4s per head
// ring slots per warp (a power of two): < 32 left after a drain, + 32 per point push (split
// drains run after each push) or + 64 per pair step
#ifndef PUSHV
#define PUSHV 0  // 1: one warp prefix (2-3 ballots) per point vector instead of one ballot per point
#endif
#ifndef RING16
#define RING16 0  // 1: ring slots are one 16-byte record {px, py, tag, 0} (one address, one STS.128)
#endif
#define RSLOT (12 + 4 * RING16)  // bytes per ring slot
#if ADRAIN
#define QCAP 64
#elif PUSHV && QUAD
#define QCAP 256  // < 32 left after a drain + 128 per 4-point vector step
#else
#define QCAP 128
#endif
#if PUSHV && ADRAIN
#error "PUSHV drains once per vector: it needs the whole-drain ring (ADRAIN 0)"
#endif

#if STREAM == 2  // the point stream bypasses L1 (keeps L1 for the cell heads and edge lists)
__device__ __forceinline__ float4 ldg_na(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
#define LOAD_PAIR(p) ldg_na(p)
#define STORE_PAIR(p, v) (*(p) = (v))
#define LDQ "ld.global.nc.L1::no_allocate"
#define STQ "st.global"
#elif STREAM
#define LOAD_PAIR(p) __ldcs(p)
#define STORE_PAIR(p, v) __stcs(p, v)
#define LDQ "ld.global.cs"
#define STQ "st.global.cs"
#else
#define LOAD_PAIR(p) __ldg(p)
#define STORE_PAIR(p, v) (*(p) = (v))
#define LDQ "ld.global.nc"
#define STQ "st.global"
#endif

// PPV points {x0, y0, x1, y1, ...} of one vector
struct pvec {
    float v[2 * PPV];
};
__device__ __forceinline__ pvec load_vec(const float *p) {
    pvec r;
#if QUAD
    asm volatile(LDQ ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                   "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
#else
    const float4 q = LOAD_PAIR(reinterpret_cast<const float4 *>(p));
    r.v[0] = q.x, r.v[1] = q.y, r.v[2] = q.z, r.v[3] = q.w;
#endif
    return r;
}
__device__ __forceinline__ void store_vec(int *o, const unsigned *k) {
#if QUAD
    asm volatile(STQ ".v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(o), "r"(k[0] & 1u), "r"(k[1] & 1u), "r"(k[2] & 1u),
                 "r"(k[3] & 1u)
                 : "memory");
#else
    STORE_PAIR(reinterpret_cast<int2 *>(o), make_int2((int)(k[0] & 1u), (int)(k[1] & 1u)));
#endif
}

// The exact search of pnpoly_slab.cu (XSEARCH) over the slab / x-search table of
// jt_pnpoly_slabs (xbuckets > 0) in global memory, loads through the read-only path. The
// table fields are the kernel's parameters (constant bank), not registers.
#define SLAB_PARAMS const float *__restrict__ table, int nu, int ng, int xb, float ybase, float yscale, \
    int guess_off, int xpar_off, int xst_off, int xlo_off, int pmax_off, int rec_off
#define SLAB_ARGS table, nu, ng, xb, ybase, yscale, guess_off, xpar_off, xst_off, xlo_off, pmax_off, rec_off
__device__ __noinline__ int slab_search(float px, float py, SLAB_PARAMS) {  // rare: out of line
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

// A queued undecided point: base parity ^ the METHOD 2 tests of its cell's listed edges
// (ylo <= py < yhi is the y-test (vy_k > py) != (vy_j > py)). The cell's 16-byte head is
// its one listed edge, or {first entry, count, NaN, 0} (count ~0: the slab search).
__device__ __forceinline__ int edge_test(float4 e, float px, float py) {
    return (e.z <= py && py < e.w && px < __fmaf_rn(e.x, py, e.y)) ? 1 : 0;
}
__device__ __forceinline__ int resolve(float px, float py, int base, float4 h, float4 h1,
                                       const float4 *__restrict__ edges, SLAB_PARAMS) {
    if (!(px == px) || !(py == py)) return 0;
    if (h.z == h.z) return base ^ edge_test(h, px, py) ^ (HEAD32 ? edge_test(h1, px, py) : 0);
    const unsigned first = __float_as_uint(h.x), cnt = __float_as_uint(h.y);
    if (cnt == 0xffffffffu) return slab_search(px, py, SLAB_ARGS);
    int in = base;
#pragma unroll 1
    for (unsigned k = 0; k < cnt; ++k) in ^= edge_test(__ldg(edges + first + k), px, py);
    return in;
}
__device__ __forceinline__ int cell_search(float px, float py, unsigned cell, int base,
                                           const float4 *__restrict__ heads, const float4 *__restrict__ edges,
                                           SLAB_PARAMS) {
    if (!(px == px) || !(py == py)) return 0;
    return resolve(px, py, base, __ldg(heads + HW * cell), HEAD32 ? __ldg(heads + HW * cell + 1) : make_float4(0.f, 0.f, 0.f, 0.f),
                   edges, SLAB_ARGS);
}

// The host's cell function (jt_pnpoly_cells): min(f2u_rz(fma(v, s, o)), GRID - 1); cvt.rzi.u32
// maps NaN and negatives to 0, so NaN lands in row / column 0 (whose decided cells hold 0).
// The raster packs 16 cells per 32-bit word: one 4-byte shared load per point (random
// cells: these lookups' bank conflicts are what the L1 pipe spends its wavefronts on, so a
// single 32-bit load beats an 8-byte one) and a rotate by 2 cell (mod 32): bit 0 = code & 1
// (the answer, or the fallback flag), bit 1 = undecided.
#if GRID_SMEM
#define GRID_WORD(i) s_grid[i]
#else
#define GRID_WORD(i) __ldg(grid + (i))
#endif
#define CELL_OF(px, py)                                                                      \
    do {                                                                                     \
        const unsigned cx_ = min(__float2uint_rz(__fmaf_rn(px, gsx, gox)), GRID - 1u);        \
        const unsigned cy_ = min(__float2uint_rz(__fmaf_rn(py, gsy, goy)), GRID - 1u);        \
        cell_ = cy_ * GRID + cx_;                                                            \
    } while (0)
#if PROBE_FLOOR == 1  // measurement probes only (scripts/cells_floor.py): 1 = same loop, no lookup
#define CODE_OF(px, py, out) ((out) = (px) < (py) ? 1u : 0u, cell_ = 0u)
#else
#define CODE_OF(px, py, out)                                                                 \
    do {                                                                                     \
        CELL_OF(px, py);                                                                     \
        const unsigned w_ = GRID_WORD(cell_ >> 4);                                           \
        (out) = __funnelshift_r(w_, w_, cell_ * 2u);                                         \
    } while (0)
#endif

// pull chunk c's vectors (one contiguous span) into L2
__device__ __forceinline__ void prefetch_chunk(const float *pts, int c, int full) {
    const long long q0 = (long long)c * CHUNK;
    if (q0 >= full) return;
    const long long q1 = min((long long)full, q0 + CHUNK);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pts + q0 * 2 * PPV),
                 "r"((unsigned)((q1 - q0) * 8 * PPV))
                 : "memory");
}
// the same from one thread without a branch: predicated on `issue` (and on the chunk
// holding full vectors); the size is clamped to the vectors left
__device__ __forceinline__ void prefetch_chunk_if(bool issue, const float *pts, int c, int full) {
    const int q0 = c * CHUNK;
    const int left = max(min(full - q0, CHUNK), 0);
    const unsigned go = (issue && left > 0) ? 1u : 0u;
    asm volatile("{\n.reg .pred p;\nsetp.ne.u32 p, %2, 0;\n"
                 "@p cp.async.bulk.prefetch.L2.global [%0], %1;\n}" ::"l"(pts + (long long)q0 * 2 * PPV),
                 "r"(left * 8 * PPV), "r"(go)
                 : "memory");
}

// warp ballot of (v != 0)
__device__ __forceinline__ unsigned ballot_nz(unsigned v) {
    unsigned m;
    asm volatile("{\n.reg .pred p;\nsetp.ne.u32 p, %1, 0;\nvote.sync.ballot.b32 %0, p, 0xffffffff;\n}"
                 : "=r"(m) : "r"(v));
    return m;
}

// MIN_BLOCKS resident blocks per SM: the default, full occupancy (2048 threads per SM), caps
// the kernel at 32 registers per thread; fewer blocks leave room for more registers
#ifndef MIN_BLOCKS
#define MIN_BLOCKS (2048 / BLOCK_SIZE_X)
#endif
extern "C" __global__ void __launch_bounds__(BLOCK_SIZE_X, MIN_BLOCKS)
pnpoly_cells(int *__restrict__ bitmap, const float2 *__restrict__ points, int n, const unsigned *__restrict__ grid,
             const float4 *__restrict__ heads, const float4 *__restrict__ edges, float gsx, float gox, float gsy,
             float goy, SLAB_PARAMS) {
    extern __shared__ __align__(16) unsigned smem[];
    const float *pts = reinterpret_cast<const float *>(points);
    // vector q = points PPV q .. PPV q + PPV - 1; a partial tail vector when n % PPV != 0
    const int full = n / PPV, nvec = (n + PPV - 1) / PPV;
#if PREFETCH
    // this block's first chunks head for L2 while the raster is staged
    if (threadIdx.x == 0)
        for (int a = 0; a <= PREFETCH; ++a) prefetch_chunk(pts, blockIdx.x + a * gridDim.x, full);
#endif
#if GRID_SMEM
    constexpr int GRID_WORDS = (GRID * GRID + 15) / 16;
    unsigned *s_grid = smem;
    unsigned *rings = smem + ((GRID_WORDS + 3) & ~3);
    for (int i = threadIdx.x; i < GRID_WORDS / 4; i += BLOCK_SIZE_X)
        reinterpret_cast<uint4 *>(s_grid)[i] = __ldg(reinterpret_cast<const uint4 *>(grid) + i);
    for (int i = GRID_WORDS / 4 * 4 + threadIdx.x; i < GRID_WORDS; i += BLOCK_SIZE_X) s_grid[i] = __ldg(grid + i);
    __syncthreads();
#else
    unsigned *rings = smem;
#endif
#if DEFER
    (void)rings;
    // Up to two undecided points pending per thread: coordinates, tag = index | base << 31
    // (~0u: free) and the cell head, loaded when the point was classified and consumed at the
    // next step, after that step's lookups (its point loads outlast the head's L2 latency).
    float q0x = 0.f, q0y = 0.f, q1x = 0.f, q1y = 0.f;
    unsigned q0t = ~0u, q1t = ~0u;
    float4 h0 = make_float4(0.f, 0.f, 0.f, 0.f), h1 = h0, h0b = h0, h1b = h0;
    auto settle = [&]() {
        if (q0t != ~0u)
            bitmap[q0t & 0x7fffffffu] = resolve(q0x, q0y, (int)(q0t >> 31), h0, h0b, edges, SLAB_ARGS), q0t = ~0u;
        if (q1t != ~0u)
            bitmap[q1t & 0x7fffffffu] = resolve(q1x, q1y, (int)(q1t >> 31), h1, h1b, edges, SLAB_ARGS), q1t = ~0u;
    };
    auto defer = [&](float px, float py, unsigned tag, unsigned cell) {
        const float4 *h = heads + HW * cell;
        if (q0t == ~0u) {
            q0x = px, q0y = py, q0t = tag, h0 = __ldg(h);
            if (HEAD32) h0b = __ldg(h + 1);
        } else if (q1t == ~0u) {
            q1x = px, q1y = py, q1t = tag, h1 = __ldg(h);
            if (HEAD32) h1b = __ldg(h + 1);
        } else {  // a third in one step: on the spot
            bitmap[tag & 0x7fffffffu] =
                resolve(px, py, (int)(tag >> 31), __ldg(h), HEAD32 ? __ldg(h + 1) : make_float4(0.f, 0.f, 0.f, 0.f),
                        edges, SLAB_ARGS);
        }
    };
    const int n_chunks = (nvec + CHUNK - 1) / CHUNK;
    auto load = [&](int c, pvec *v) {
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            if (c < n_chunks && q < full) v[t] = load_vec(pts + (long long)q * 2 * PPV);
            else {
#pragma unroll
                for (int j = 0; j < 2 * PPV; ++j) v[t].v[j] = 0.f;
                if (c < n_chunks && q < nvec)  // the partial tail vector: its points one by one
#pragma unroll
                    for (int j = 0; j < PPV; ++j)
                        if (PPV * q + j < n) {
                            const float2 p = points[PPV * q + j];
                            v[t].v[2 * j] = p.x, v[t].v[2 * j + 1] = p.y;
                        }
            }
        }
    };
    auto chunk = [&](int c, const pvec *cur, const bool FULL) {  // inlined twice with FULL constant
        unsigned k[TILE][PPV], cl[TILE][PPV];
#pragma unroll
        for (int t = 0; t < TILE; ++t)
#pragma unroll
            for (int j = 0; j < PPV; ++j) {
                unsigned cell_;
                CODE_OF(cur[t].v[2 * j], cur[t].v[2 * j + 1], k[t][j]);
                cl[t][j] = cell_;
            }
        settle();  // the previous step's pending points
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            // decided points get their answer here; undecided ones a placeholder, rewritten
            // when the point settles (same thread, later store)
            if (FULL || q < full) store_vec(bitmap + (long long)PPV * q, k[t]);
            else if (q < nvec)
#pragma unroll
                for (int j = 0; j < PPV; ++j)
                    if (PPV * q + j < n) bitmap[PPV * q + j] = (int)(k[t][j] & 1u);
#pragma unroll
            for (int j = 0; j < PPV; ++j)
                if ((FULL || PPV * q + j < n) && (k[t][j] & 2u))
                    defer(cur[t].v[2 * j], cur[t].v[2 * j + 1], (unsigned)(PPV * q + j) | (k[t][j] << 31), cl[t][j]);
        }
    };
#if REGPF == 2
    // register double buffering without the copy: two buffers swap roles every chunk (the loop
    // body is the pair of chunks c, c + grid)
    pvec bufa[TILE], bufb[TILE];
    load(blockIdx.x, bufa);
    for (int c = blockIdx.x; c < n_chunks; c += 2 * gridDim.x) {
#if PREFETCH
        prefetch_chunk_if(threadIdx.x == 0, pts, c + (PREFETCH + 1) * gridDim.x, full);
#endif
        load(c + gridDim.x, bufb);
        if ((c + 1) * CHUNK <= full) chunk(c, bufa, true);
        else chunk(c, bufa, false);
        const int c2 = c + gridDim.x;
        if (c2 >= n_chunks) break;
#if PREFETCH
        prefetch_chunk_if(threadIdx.x == 0, pts, c2 + (PREFETCH + 1) * gridDim.x, full);
#endif
        load(c2 + gridDim.x, bufa);
        if ((c2 + 1) * CHUNK <= full) chunk(c2, bufb, true);
        else chunk(c2, bufb, false);
    }
#else
#if REGPF
    pvec nxt[TILE];  // the next chunk, loaded while this one is classified
    load(blockIdx.x, nxt);
#endif
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
#if PREFETCH
        prefetch_chunk_if(threadIdx.x == 0, pts, c + (PREFETCH + 1) * gridDim.x, full);
#endif
        pvec cur[TILE];
#if REGPF
#pragma unroll
        for (int t = 0; t < TILE; ++t) cur[t] = nxt[t];
        load(c + gridDim.x, nxt);
#else
        load(c, cur);
#endif
        if ((c + 1) * CHUNK <= full) chunk(c, cur, true);
        else chunk(c, cur, false);
    }
#endif
    settle();
}
#else
    // per warp: QCAP undecided points {px, py} and their indices (bit 31: base parity)
#if RING16
    float4 *ring_r = reinterpret_cast<float4 *>(rings) + (threadIdx.x >> 5) * QCAP;
#define RING_PUT(pos, px, py, tag) (ring_r[pos] = make_float4((px), (py), __int_as_float(tag), 0.f))
#define RING_GET(pos, px, py, tag)                                                                   \
    do {                                                                                             \
        const float4 r_ = ring_r[pos];                                                               \
        (px) = r_.x, (py) = r_.y, (tag) = __float_as_int(r_.z);                                      \
    } while (0)
#else
    float2 *ring_p = reinterpret_cast<float2 *>(rings) + (threadIdx.x >> 5) * QCAP;
    int *ring_i = reinterpret_cast<int *>(rings + 2 * (BLOCK_SIZE_X / 32) * QCAP) + (threadIdx.x >> 5) * QCAP;
#define RING_PUT(pos, px, py, tag) (ring_p[pos] = make_float2((px), (py)), ring_i[pos] = (tag))
#define RING_GET(pos, px, py, tag)                                                                   \
    do {                                                                                             \
        const float2 e_ = ring_p[pos];                                                               \
        (px) = e_.x, (py) = e_.y, (tag) = ring_i[pos];                                               \
    } while (0)
#endif
    const int lane = threadIdx.x & 31;
    unsigned lanes_below;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lanes_below));
    // The ring is pushed at tail and drained 32 points at a time from head (warp-uniform
    // counters) after each pair step: < 32 are left after a drain, so a step's <= 64 pushes
    // never reach the slots the last drain read.
    unsigned head = 0, tail = 0;
#if ADRAIN
    // Drains are split in two so the head read's L2 latency overlaps the next chunks: a
    // batch of 32 takes its points into registers and starts a 16-byte cp.async of each
    // point's cell head into a per-lane slot; the batch is finished (test, store) when the
    // next one starts, or at the end. One batch is pending once any has started (head > 0).
    float4 *hslot = reinterpret_cast<float4 *>(rings + RSLOT / 4 * (BLOCK_SIZE_X / 32) * QCAP) + HW * threadIdx.x;
    float apx = 0.f, apy = 0.f;
    int aidx = 0;
    auto finish = [&]() {
        asm volatile("cp.async.wait_all;" ::: "memory");
        bitmap[aidx & 0x7fffffff] = resolve(apx, apy, (int)((unsigned)aidx >> 31), hslot[0], hslot[HW - 1], edges,
                                            SLAB_ARGS);
    };
    auto drain = [&]() {
        __syncwarp();
#if PROBE_FLOOR == 3  // 3 = pushes, the drained points dropped
        while (tail - head >= 32u) head += 32;
        return;
#endif
        while (tail - head >= 32u) {
            if (head) finish();
            RING_GET((head + lane) % QCAP, apx, apy, aidx);
            head += 32;
            unsigned cell_;
            CELL_OF(apx, apy);
            const unsigned slot = (unsigned)__cvta_generic_to_shared(hslot);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot), "l"(heads + HW * cell_) : "memory");
            if (HEAD32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot + 16), "l"(heads + HW * cell_ + 1)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
#else
    auto drain = [&]() {
        __syncwarp();
        while (tail - head >= 32u) {
            float ex, ey;
            int i;
            RING_GET((head + lane) % QCAP, ex, ey, i);
            head += 32;
            unsigned cell_;
            CELL_OF(ex, ey);
            bitmap[i & 0x7fffffff] = cell_search(ex, ey, cell_, (int)((unsigned)i >> 31), heads, edges, SLAB_ARGS);
        }
    };
#endif
    const int n_chunks = (nvec + CHUNK - 1) / CHUNK;
    auto load = [&](int c, pvec *v) {
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            if (c < n_chunks && q < full) v[t] = load_vec(pts + (long long)q * 2 * PPV);
            else {
#pragma unroll
                for (int j = 0; j < 2 * PPV; ++j) v[t].v[j] = 0.f;
                if (c < n_chunks && q < nvec)  // the partial tail vector: its points one by one
#pragma unroll
                    for (int j = 0; j < PPV; ++j)
                        if (PPV * q + j < n) {
                            const float2 p = points[PPV * q + j];
                            v[t].v[2 * j] = p.x, v[t].v[2 * j + 1] = p.y;
                        }
            }
        }
    };
    // one point's push into the warp's ring (u != 0: undecided); k carries the base parity in bit 0
    auto push = [&](float px, float py, int idx, unsigned k, unsigned u) {
        const unsigned need = ballot_nz(u);
        const unsigned pos = (tail + __popc(need & lanes_below)) % QCAP;
        if (u) RING_PUT(pos, px, py, idx | (int)(k << 31));
        tail += __popc(need);
    };
    auto chunk = [&](int c, const pvec *cur, const bool FULL) {  // inlined twice with FULL constant
#pragma unroll
        for (int t = 0; t < TILE; ++t) {
            const int q = c * CHUNK + t * BLOCK_SIZE_X + threadIdx.x;
            unsigned k[PPV], cl[PPV], cell_;
#pragma unroll
            for (int j = 0; j < PPV; ++j) {
                CODE_OF(cur[t].v[2 * j], cur[t].v[2 * j + 1], k[j]);
                cl[j] = cell_;
            }
            // decided points get their answer here; undecided ones a placeholder, rewritten
            // by a later drain of the same warp
            if (FULL || q < full) store_vec(bitmap + (long long)PPV * q, k);
            else if (q < nvec)
#pragma unroll
                for (int j = 0; j < PPV; ++j)
                    if (PPV * q + j < n) bitmap[PPV * q + j] = (int)(k[j] & 1u);
#if PUSHV
            {
                // the vector's undecided points: one warp prefix over their counts (<= PPV, so
                // 2-3 ballots of its bits), then each lane writes its own run of slots
                unsigned um = 0u;
#pragma unroll
                for (int j = 0; j < PPV; ++j)
                    if ((FULL || PPV * q + j < n) && (k[j] & 2u)) um |= 1u << j;
                const unsigned cnt = __popc(um);
                const unsigned b0 = ballot_nz(cnt & 1u), b1 = ballot_nz(cnt & 2u), b2 = PPV > 2 ? ballot_nz(cnt & 4u) : 0u;
                unsigned pos = tail + __popc(b0 & lanes_below) + 2u * __popc(b1 & lanes_below) +
                               4u * __popc(b2 & lanes_below);
#pragma unroll
                for (int j = 0; j < PPV; ++j)
                    if (um & (1u << j)) {
                        RING_PUT(pos % QCAP, cur[t].v[2 * j], cur[t].v[2 * j + 1], (PPV * q + j) | (int)(k[j] << 31));
                        if (HPF) asm volatile("prefetch.global.L1 [%0];" ::"l"(heads + HW * cl[j]));
                        ++pos;
                    }
                tail += __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
                drain();
            }
#else
#pragma unroll
            for (int j = 0; j < PPV; ++j) {
#if PROBE_FLOOR == 2  // 2 = lookups, nothing queued
                const unsigned u = 0u;
#else
                const unsigned u = (FULL || PPV * q + j < n) ? (k[j] & 2u) : 0u;
#endif
                push(cur[t].v[2 * j], cur[t].v[2 * j + 1], PPV * q + j, k[j], u);
                // the head's L2 -> L1 trip overlaps the point's wait in the ring
                if (HPF && u) asm volatile("prefetch.global.L1 [%0];" ::"l"(heads + HW * cl[j]));
                // ring: < 32 left after a drain; split drains after every push (+32), whole
                // drains after every second push (+64)
                if (ADRAIN || (j & 1)) drain();
            }
#endif
        }
    };
#if REGPF == 2
    // register double buffering without the copy: two buffers swap roles every chunk (the loop
    // body is the pair of chunks c, c + grid)
    pvec bufa[TILE], bufb[TILE];
    load(blockIdx.x, bufa);
    for (int c = blockIdx.x; c < n_chunks; c += 2 * gridDim.x) {
#if PREFETCH
        prefetch_chunk_if(threadIdx.x == 0, pts, c + (PREFETCH + 1) * gridDim.x, full);
#endif
        load(c + gridDim.x, bufb);
        if ((c + 1) * CHUNK <= full) chunk(c, bufa, true);
        else chunk(c, bufa, false);
        const int c2 = c + gridDim.x;
        if (c2 >= n_chunks) break;
#if PREFETCH
        prefetch_chunk_if(threadIdx.x == 0, pts, c2 + (PREFETCH + 1) * gridDim.x, full);
#endif
        load(c2 + gridDim.x, bufa);
        if ((c2 + 1) * CHUNK <= full) chunk(c2, bufb, true);
        else chunk(c2, bufb, false);
    }
#else
#if REGPF
    pvec nxt[TILE];  // the next chunk, loaded while this one is classified
    load(blockIdx.x, nxt);
#endif
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
#if PREFETCH
        prefetch_chunk_if(threadIdx.x == 0, pts, c + (PREFETCH + 1) * gridDim.x, full);
#endif
        pvec cur[TILE];
#if REGPF
#pragma unroll
        for (int t = 0; t < TILE; ++t) cur[t] = nxt[t];
        load(c + gridDim.x, nxt);
#else
        load(c, cur);
#endif
        if ((c + 1) * CHUNK <= full) chunk(c, cur, true);
        else chunk(c, cur, false);
    }
#endif
#if ADRAIN
#if PROBE_FLOOR != 3
    if (head) finish();
#endif
#endif
    if (lane < tail - head) {  // the warp's leftovers
        float ex, ey;
        int i;
        RING_GET((head + lane) % QCAP, ex, ey, i);
        unsigned cell_;
        CELL_OF(ex, ey);
        bitmap[i & 0x7fffffff] = cell_search(ex, ey, cell_, (int)((unsigned)i >> 31), heads, edges, SLAB_ARGS);
    }
}
#endif
