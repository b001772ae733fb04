/*
 * jt.h — C-ABI of libjt, the B200 device boundary of paper_2211_07260_b200.
 *
 * The reference package (jouletune) has no FFI: its device boundary is the
 * duck-typed SimulatedDevice (pkg/src/jouletune/device.py:246-382). libjt is
 * what a maintainer binds to replace that simulator with a real GPU; each
 * entry point below names the reference interface it stands in for.
 * Plain C types only (no torch, no CUDA types in signatures); every call
 * returns a jt_status and leaves a message retrievable with jt_last_error().
 *
 * Threading: one jt_ctx per (process, GPU). Calls on one ctx are serialised
 * by the caller (the reference benchmark loop is single threaded,
 * SPEC.md:465). jt_compile() is context free and thread safe, so configs can
 * be compiled on a host thread pool while the GPU is busy. The only thread
 * libjt creates is the NVML sampler inside jt_bench()/jt_sampler_*.
 */
#ifndef JT_H
#define JT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JT_ABI_VERSION 3

/* Status codes and the Python exception each maps to (native.py):         */
typedef enum {
    JT_OK = 0,
    JT_EINVAL = 1,     /* malformed argument            -> ConfigurationError */
    JT_ENOGPU = 2,     /* no driver / device             -> CapabilityError   */
    JT_ECUDA = 3,      /* CUDA driver error              -> DomainError       */
    JT_ECOMPILE = 4,   /* NVRTC rejected the config      -> DomainError       */
    JT_ELAUNCH = 5,    /* launch shape / smem rejected   -> DomainError       */
    JT_ENVML = 6,      /* NVML missing or failed         -> CapabilityError   */
    JT_ENOPERM = 7,    /* NVML refused (clock lock etc.) -> recorded, no raise */
    JT_ENOTSUP = 8     /* not supported on this device   -> CapabilityError   */
} jt_status;

typedef struct jt_ctx jt_ctx;
typedef struct jt_module jt_module;
typedef struct jt_kernel jt_kernel;

/* Static device description; replaces DeviceSpec's inputs
 * (reference device.py:44-78: supported_core_clocks, base/peak clock,
 * power_limit_range, tdp). All clocks in MHz, power in mW. */
typedef struct {
    int ordinal;
    int cc_major, cc_minor;
    int sm_count;
    int max_smem_optin;          /* bytes per block with opt-in            */
    int l2_bytes;
    unsigned long long total_mem;
    char name[128];
    char pci_bus_id[32];
    int nvml_ok;                 /* NVML handle resolved by PCI bus id      */
    int energy_counter_ok;
    int instant_power_ok;
    unsigned n_clocks;           /* supported SM clocks at the top memory clock, ascending */
    unsigned clocks_mhz[512];
    unsigned mem_clock_mhz;
    unsigned max_sm_clock_mhz;
    unsigned default_sm_clock_mhz; /* default applications clock (base)    */
    unsigned power_limit_min_mw, power_limit_max_mw;
    unsigned power_limit_default_mw, power_limit_mw;
    unsigned tdp_mw;             /* enforced default limit                   */
} jt_device_info;

/* One NVML sample. Times are seconds on the jt_now() clock.
 * Replaces the simulator's PowerSample trace (device.py:124-127, 366-378). */
typedef struct {
    double t_s;
    double power_w;              /* NVML_FI_DEV_POWER_INSTANT (NaN if n/a)  */
    double power_avg_w;          /* nvmlDeviceGetPowerUsage (1 s average)   */
    double energy_j;             /* total energy counter (NaN if n/a)       */
    double energy_stamp_s;       /* driver timestamp of the energy field, jt_now() clock */
    unsigned sm_mhz, mem_mhz, temp_c, pad;
    unsigned long long reasons;  /* clocks-event reason bitmask             */
} jt_sample;

/* Kernel argument; replaces nothing in the reference (kernels were simulated
 * by PerformanceSurface, device.py:148-243). */
/* JT_ARG_BLOB: v.ptr is a host pointer to a by-value parameter (e.g. a
 * 128-byte CUtensorMap from jt_tensor_map_2d) passed as __grid_constant__. */
typedef enum { JT_ARG_PTR = 0, JT_ARG_I32 = 1, JT_ARG_F32 = 2, JT_ARG_F64 = 3, JT_ARG_I64 = 4, JT_ARG_BLOB = 5 } jt_arg_kind;
typedef struct {
    int kind;
    int pad;
    union { unsigned long long ptr; long long i64; double f64; float f32; int i32; } v;
} jt_arg;

typedef struct {
    unsigned grid[3];
    unsigned block[3];
    unsigned smem_bytes;         /* dynamic shared memory                   */
    unsigned cluster_x;          /* 0/1 = no cluster                        */
} jt_launch_shape;

/* Result of a device-timed back-to-back loop; replaces the runtime /
 * repetitions / total_duration of Execution (device.py:130-138, 349-382). */
typedef struct {
    double first_launch_s;       /* event time of the untimed probe launch  */
    double per_launch_s;         /* loop time / reps                        */
    double total_s;              /* CUDA-event loop time                    */
    int reps;
    int n_samples;               /* samples written                          */
    double host_t_enqueue;       /* jt_now() before the first timed launch  */
    double host_t_done;          /* jt_now() after the stop event completed */
    double loop_t0;              /* estimated device start = done - total   */
} jt_bench_result;

/* --- context ------------------------------------------------------------ */
int jt_abi_version(void);
double jt_now(void);                           /* CLOCK_MONOTONIC seconds   */
const char *jt_last_error(void);               /* thread-local message      */
int jt_device_count(int *count);
int jt_open(int ordinal, jt_ctx **out);        /* retains the primary context, resolves NVML by PCI id */
int jt_close(jt_ctx *ctx);                     /* resets clocks/limits this ctx changed */
int jt_device_info_get(jt_ctx *ctx, jt_device_info *out);

/* --- memory (Execution inputs; the simulator had none) -------------------- */
int jt_alloc(jt_ctx *ctx, size_t bytes, unsigned long long *dptr);
int jt_free(jt_ctx *ctx, unsigned long long dptr);
int jt_host_alloc(jt_ctx *ctx, size_t bytes, void **hptr);   /* pinned */
int jt_host_free(jt_ctx *ctx, void *hptr);
int jt_h2d(jt_ctx *ctx, unsigned long long dst, const void *src, size_t bytes);
int jt_d2h(jt_ctx *ctx, void *dst, unsigned long long src, size_t bytes);
int jt_memset_d8(jt_ctx *ctx, unsigned long long dst, unsigned char value, size_t bytes);
int jt_synchronize(jt_ctx *ctx);

/* --- kernels: per-config compile + load (Kernel Tuner's compile step) ---- */
int jt_compile(const char *source, const char *program_name, const char *const *options, int n_options,
               void **image, size_t *image_bytes, char *log, size_t log_capacity);
void jt_free_image(void *image);
/* Version and path of the NVRTC jt_compile uses: dlopen'ed by full path from the
 * toolkit (JT_CUDA_HOME / CUDA_HOME / /usr/local/cuda), never whichever
 * libnvrtc.so.12 the host process happened to load first. No reference
 * counterpart (Kernel Tuner reports its compiler through the `compiler`
 * field of its environment record, core.py get_environment). */
int jt_nvrtc_version(int *major, int *minor, char *path, size_t path_capacity);
int jt_module_load(jt_ctx *ctx, const void *image, size_t image_bytes, jt_module **out);
int jt_module_unload(jt_ctx *ctx, jt_module *module);
int jt_kernel_get(jt_ctx *ctx, jt_module *module, const char *name, jt_kernel **out);
int jt_kernel_attributes(jt_ctx *ctx, jt_kernel *kernel, int *regs, int *static_smem, int *local_bytes,
                         int *max_threads);
/* Resident CTAs per SM for `block_threads` threads and `dynamic_smem` bytes
 * (cuOccupancyMaxActiveBlocksPerMultiprocessor; raises the kernel's dynamic
 * shared-memory limit first). Used to size split-tail grids to whole waves. */
int jt_kernel_occupancy(jt_ctx *ctx, jt_kernel *kernel, int block_threads, size_t dynamic_smem, int *blocks_per_sm);

/* --- execution (SimulatedDevice.execute, device.py:349-382) ------------------ */
int jt_launch(jt_ctx *ctx, jt_kernel *kernel, const jt_launch_shape *shape, const jt_arg *args, int n_args);
/* Event-timed loop of exactly `reps` launches; *seconds = total device time. */
int jt_time(jt_ctx *ctx, jt_kernel *kernel, const jt_launch_shape *shape, const jt_arg *args, int n_args,
            int reps, double *seconds);
/* The benchmark primitive: one probe launch, then back-to-back launches
 * between two CUDA events while the NVML sampler records every
 * `sample_period_us` into `samples` (capacity `cap`; may be NULL to skip
 * sampling). The loop lasts >= min_seconds: its first quarter (sized from the
 * probe) is timed on its own and the remaining launch count recomputed from it
 * while a second quarter keeps the GPU busy; reps stays in [min_reps, max_reps]. */
int jt_bench(jt_ctx *ctx, jt_kernel *kernel, const jt_launch_shape *shape, const jt_arg *args, int n_args,
             double min_seconds, int min_reps, int max_reps, int sample_period_us, jt_bench_result *out,
             jt_sample *samples, int cap);
/* jt_bench over `n_sets` argument sets (args holds n_sets x n_args entries):
 * launch i uses set i % n_sets, so a loop can rotate inputs/outputs larger
 * than L2 between launches (bench.py per-kernel loops). n_sets = 1 is
 * jt_bench. */
int jt_bench_sets(jt_ctx *ctx, jt_kernel *kernel, const jt_launch_shape *shape, const jt_arg *args, int n_args,
                  int n_sets, double min_seconds, int min_reps, int max_reps, int sample_period_us,
                  jt_bench_result *out, jt_sample *samples, int cap);
/* CUDA events on the context's stream: an indexed pool of `n` events for
 * timing arbitrary launch/copy sequences (bench.py). */
int jt_events_reserve(jt_ctx *ctx, int n);
int jt_event_record(jt_ctx *ctx, int index);
int jt_event_elapsed(jt_ctx *ctx, int start, int stop, double *seconds);
/* Stream gate for host-independent timed regions: jt_stream_gate makes the
 * active stream wait (cuStreamWaitValue32 on a mapped host word) so a whole
 * sequence -- start event, K launches, stop event -- can be enqueued first;
 * jt_stream_release lets it run back to back, with no host submission (or
 * driver lock held by the NVML sampler) between the events. Replaces nothing
 * in the reference (its simulated device has no launch path); used by
 * bench.py's timed region. */
int jt_stream_gate(jt_ctx *ctx);
int jt_stream_release(jt_ctx *ctx);
/* Streams: index 0 is the context's own; jt_streams_reserve(n) makes 1..n-1.
 * jt_stream_select routes subsequent launches, async copies, memsets, event
 * records and timed loops to that stream (copy/compute overlap for the
 * host-buffer suite entry points); jt_synchronize waits for all of them. */
int jt_streams_reserve(jt_ctx *ctx, int n);
int jt_stream_select(jt_ctx *ctx, int index);
int jt_stream_wait_event(jt_ctx *ctx, int event_index);   /* selected stream waits on event */
/* Async copies on the selected stream (host memory should be pinned). */
int jt_h2d_async(jt_ctx *ctx, unsigned long long dst, const void *src, size_t bytes);
int jt_d2h_async(jt_ctx *ctx, void *dst, unsigned long long src, size_t bytes);
/* Pitched (2D) async copies on the selected stream: `rows` rows of
 * `width_bytes`, row starts `*_pitch` bytes apart. The host-buffer API uses
 * them to place an arbitrary M x N operand inside a buffer padded to the
 * kernel's tile multiples (CLBlast's "indirect" GEMM padding, done by the
 * copy engines) and to read the valid region back. */
int jt_h2d_2d_async(jt_ctx *ctx, unsigned long long dst, size_t dst_pitch, const void *src, size_t src_pitch,
                    size_t width_bytes, size_t rows);
int jt_d2h_2d_async(jt_ctx *ctx, void *dst, size_t dst_pitch, unsigned long long src, size_t src_pitch,
                    size_t width_bytes, size_t rows);
/* Overwrite a scratch buffer larger than L2 (126 MB on B200). */
int jt_l2_flush(jt_ctx *ctx);

/* --- NVML sensors (observers.py:81-124 sensor semantics, real sources) --- */
int jt_sample_now(jt_ctx *ctx, jt_sample *out);
int jt_sampler_start(jt_ctx *ctx, int period_us, int cap);
int jt_sampler_stop(jt_ctx *ctx, jt_sample *out, int cap, int *n);

/* --- clock / power controller (set_core_clock / set_power_limit,
 *     device.py:277-293). JT_ENOPERM is returned, not fatal, when NVML
 *     refuses; callers then record the observed clock. ------------------- */
int jt_clock_lock(jt_ctx *ctx, unsigned min_mhz, unsigned max_mhz);
int jt_clock_reset(jt_ctx *ctx);
/* Fallback knob when locked clocks are refused: NVML applications clocks. */
int jt_app_clocks_set(jt_ctx *ctx, unsigned mem_mhz, unsigned sm_mhz);
int jt_app_clocks_reset(jt_ctx *ctx);
int jt_power_limit_set(jt_ctx *ctx, unsigned milliwatts);
int jt_power_limit_reset(jt_ctx *ctx);

/* --- kernel-suite helpers ------------------------------------------------ */
/* PnPoly edge table for the chosen crossing METHOD (see
 * csrc/kernels/pnpoly.cu): edges[4k..4k+3] = {vy_k, a, b, c},
 * ybounds[2k..2k+1] = {min, max} of the edge's y range. Computed in IEEE
 * float32 with explicit fmaf so the device and the oracle see the same bits. */
int jt_pnpoly_edges(const float *vx, const float *vy, int n, int method, float *edges, float *ybounds);
/* PnPoly slab tables for csrc/kernels/pnpoly_slab.cu (exact point location
 * by y-slab; the bitmap is bit-identical to the brute-force METHOD 2 crossing
 * test). The sorted distinct vertex ordinates u[0..nu) cut the plane into
 * nu+1 slabs; slab r = #{u <= py} holds exactly the edges whose y-range
 * spans every py in [u[r-1], u[r]). `buckets` uniform y-buckets give each
 * point a starting rank that the kernel corrects by exact compares.
 * xbuckets = 0: each slab lists its edges as {slope, icpt} pairs (the
 *   jt_pnpoly_edges METHOD 2 bits), padded to a multiple of `pad` with
 *   never-crossing {0, -inf} fillers; the kernel tests every listed edge.
 * xbuckets > 0: each slab's edges sorted by lo, the smallest computed crossing
 *   abscissa fma(slope, py, icpt) over the slab (fma is monotone in py, so it
 *   is the smaller of the two end values), with pmax = running max of hi; the
 *   kernel counts {lo > px} (certain crossings) from a starting position
 *   (xbuckets uniform x-buckets per slab over [lo_min, lo_max], uint16
 *   positions) corrected by exact compares, and evaluates only edges with
 *   lo <= px < hi. Records {slope, icpt, hi, 0}; {x0, xscale} per slab.
 * Table words (4 B): u at u_off (nu floats), guess at guess_off (buckets
 * int32), slab starts at band_off (nu+2 int32, in edges); x-search only:
 * {x0, xscale} float pairs at xpar_off, uint16 [nu+1][xb+1] bucket starts at
 * xst_off, lo / pmax at xlo_off / pmax_off and their conservatively rounded
 * binary16 copy at half_off; pairs / records at pair_off.
 * table == NULL: fill `info` only (size query). The reference has no PnPoly
 * code; this serves the B200 PnPoly suite. */
typedef struct {
    int nu, ng, ne, max_band;
    int u_off, guess_off, band_off, pair_off, words;
    float ybase, yscale;
    int xlo_off, pmax_off, xpar_off, xst_off, xb;
    int half_off;  /* x-search only: per edge (pmax as binary16 rounded up) << 16 | (lo rounded down) */
} jt_slab_info;
int jt_pnpoly_slabs(const float *vx, const float *vy, int n, int buckets, int pad, int xbuckets, float *table,
                    long long capacity, jt_slab_info *info);
/* PnPoly uniform-cell fast path for csrc/kernels/pnpoly_grid.cu: a gw x gh
 * grid over the polygon's bounding box (cells on the border extend to
 * infinity); cell (cx, cy) = (min(f2u_rz(fma(px, sx, ox)), gw - 1),
 * min(f2u_rz(fma(py, sy, oy)), gh - 1)) in float32. A cell is "clean" when, for every point that maps to it,
 * every edge spanning its py is decided by the computed-x ranges (crosses for
 * all px of the cell or for none) and the crossing count has one parity in
 * all slabs the cell's rows meet; its bits are then 1 | parity << 1 (2 bits
 * per cell, 16 cells per word), else 0 (the kernel runs the exact slab
 * search). params = {sx, ox, sy, oy}. bits == NULL: params only. */
int jt_pnpoly_grid(const float *vx, const float *vy, int n, int gw, int gh, float *params, uint32_t *bits,
                   long long capacity, int *clean_cells);
/* Per-cell edge lists over the same gw x gh raster and cell function as
 * jt_pnpoly_grid, for csrc/kernels/pnpoly_cells.cu. Per cell a 2-bit code
 * (16 cells per word, cell c at bits 2 (c % 16)): 0 / 1 = every edge's METHOD 2
 * test is constant over the cell and the answer is that parity; 2 | base = some
 * tests are undecided, base = the parity of the always-true ones, and the
 * cell's head (head_words = 4 or 8 words at heads + head_words cell) holds the
 * undecided edges in place when there are 1 .. head_words / 4 of them (float
 * {slope, icpt, ylo, yhi} each; an unused slot is {0, 0, NaN, 0}, never true),
 * else {first entry, count, NaN, 0} with the count undecided edges as float4
 * entries in `edges` from that entry on (count 0xffffffff: more than `lmax`,
 * the kernel runs the exact slab search). Border cells (row 0, column 0, where
 * NaN coordinates land) with base 1 are always undecided. stats = {entries,
 * decided cells, listed cells, fallback cells}. bits or heads NULL: params and
 * stats only; edges NULL or too small: sizes only (JT_EINVAL if too small). */
int jt_pnpoly_cells(const float *vx, const float *vy, int n, int gw, int gh, int lmax, int head_words, float *params,
                    uint32_t *bits, long long bits_capacity, uint32_t *heads, long long heads_capacity, float *edges,
                    long long edge_capacity, long long *stats);

/* TMA descriptor (CUtensorMap, 128 bytes written to out128) for a row-major
 * fp32 matrix [rows][cols] at dptr, tiles of box_rows x box_cols elements.
 * `swizzle` is a CUtensorMapSwizzle value: 0 none, 1 32B, 2 64B, 3 128B,
 * 4 128B with 32-byte atoms (the MN-major TF32 UMMA layout), 6 128B/64B atoms
 * (box_cols * 4 must be <= the swizzle span). */
int jt_tensor_map_2d(jt_ctx *ctx, unsigned long long dptr, unsigned long long rows, unsigned long long cols,
                     unsigned box_rows, unsigned box_cols, int swizzle, void *out128);
/* Copy host bytes into a __constant__ / __device__ symbol of a loaded module. */
int jt_module_set_global(jt_ctx *ctx, jt_module *module, const char *name, const void *src, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* JT_H */
