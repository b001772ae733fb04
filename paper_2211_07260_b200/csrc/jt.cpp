// libjt — the B200 device boundary (see include/jt.h for the contract).
//
// Host-side runtime only: CUDA driver API (primary context, one
// non-blocking stream per ctx, CUDA events), NVRTC for per-config kernel
// compilation to sm_100a cubins, and NVML (dlopen'ed, so the library loads on
// machines without a driver) for the sampler thread and the clock / power
// controller. The kernels themselves live in csrc/kernels/*.cu and reach the
// GPU through jt_compile + jt_module_load.
#include "jt.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvml.h>
#include <nvrtc.h>
#include <time.h>

#include <algorithm>
#include <limits>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_error;

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
    return code;
}

double mono_now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

double real_now() {
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}


// ---------------------------------------------------------------------------
// CUDA driver, resolved at runtime through cuGetProcAddress so that libjt
// loads (and its symbols can be inspected) on a machine without a driver.
#define JT_DRIVER_FNS(X) \
    X(cuCtxSetCurrent) \
    X(cuDeviceGet) \
    X(cuDeviceGetAttribute) \
    X(cuDeviceGetCount) \
    X(cuDeviceGetName) \
    X(cuDeviceGetPCIBusId) \
    X(cuDevicePrimaryCtxRelease) \
    X(cuDevicePrimaryCtxRetain) \
    X(cuDeviceTotalMem) \
    X(cuEventCreate) \
    X(cuEventDestroy) \
    X(cuEventElapsedTime) \
    X(cuEventRecord) \
    X(cuEventSynchronize) \
    X(cuFuncGetAttribute) \
    X(cuFuncSetAttribute) \
    X(cuGetErrorName) \
    X(cuGetErrorString) \
    X(cuInit) \
    X(cuLaunchKernel) \
    X(cuLaunchKernelEx) \
    X(cuMemAlloc) \
    X(cuMemFree) \
    X(cuMemFreeHost) \
    X(cuMemHostAlloc) \
    X(cuMemHostGetDevicePointer) \
    X(cuMemcpy2DAsync) \
    X(cuMemcpyDtoHAsync) \
    X(cuMemcpyHtoDAsync) \
    X(cuMemsetD8Async) \
    X(cuModuleGetFunction) \
    X(cuModuleGetGlobal) \
    X(cuModuleLoadData) \
    X(cuModuleUnload) \
    X(cuOccupancyMaxActiveBlocksPerMultiprocessor) \
    X(cuStreamCreate) \
    X(cuStreamDestroy) \
    X(cuStreamSynchronize) \
    X(cuStreamWaitEvent) \
    X(cuStreamWaitValue32) \
    X(cuTensorMapEncodeTiled)

struct Driver {
    bool ok = false;
#define JT_DECL(fn) decltype(&::fn) p_##fn = nullptr;
    JT_DRIVER_FNS(JT_DECL)
#undef JT_DECL
};

Driver D;
std::once_flag g_driver_once;
std::string g_driver_why;

void driver_load() {
    void *lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("libcuda.so", RTLD_NOW | RTLD_LOCAL);
    if (!lib) {
        g_driver_why = "libcuda.so.1 not found (no NVIDIA driver)";
        return;
    }
    using getproc_t = CUresult (*)(const char *, void **, int, cuuint64_t, CUdriverProcAddressQueryResult *);
    auto getproc = reinterpret_cast<getproc_t>(dlsym(lib, "cuGetProcAddress_v2"));
    if (!getproc) {
        g_driver_why = "driver lacks cuGetProcAddress_v2 (needs a CUDA 12 driver)";
        return;
    }
    bool all = true;
#define JT_LOAD(fn)                                                                          \
    {                                                                                        \
        CUdriverProcAddressQueryResult st;                                                   \
        if (getproc(#fn, reinterpret_cast<void **>(&D.p_##fn), CUDA_VERSION, 0, &st) != CUDA_SUCCESS || !D.p_##fn) { \
            all = false;                                                                     \
            g_driver_why = "driver symbol missing: " #fn;                                    \
        }                                                                                    \
    }
    JT_DRIVER_FNS(JT_LOAD)
#undef JT_LOAD
    D.ok = all;
}

bool driver_ready() {
    std::call_once(g_driver_once, driver_load);
    return D.ok;
}

const char *cu_name(CUresult r) {
    const char *s = nullptr;
    if (D.p_cuGetErrorName) D.p_cuGetErrorName(r, &s);
    return s ? s : "CUDA_ERROR_?";
}

int cu_fail(CUresult r, const char *what) {
    const char *desc = nullptr;
    if (D.p_cuGetErrorString) D.p_cuGetErrorString(r, &desc);
    int code = JT_ECUDA;
    switch (r) {
        case CUDA_ERROR_NO_DEVICE:
        case CUDA_ERROR_NOT_INITIALIZED:
        case CUDA_ERROR_INVALID_DEVICE:
        case CUDA_ERROR_STUB_LIBRARY:
            code = JT_ENOGPU;
            break;
        case CUDA_ERROR_INVALID_VALUE:
        case CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES:
        case CUDA_ERROR_INVALID_CLUSTER_SIZE:
        case CUDA_ERROR_NOT_SUPPORTED:
            code = JT_ELAUNCH;
            break;
        default:
            break;
    }
    return fail(code, "%s: %s (%s)", what, cu_name(r), desc ? desc : "");
}

#define CU_TRY(call, what)                          \
    do {                                            \
        CUresult r_ = (call);                       \
        if (r_ != CUDA_SUCCESS) return cu_fail(r_, what); \
    } while (0)

// ---------------------------------------------------------------------------
// NVML, resolved at runtime.
struct Nvml {
    void *lib = nullptr;
    bool ok = false;
    nvmlReturn_t (*Init)() = nullptr;
    const char *(*ErrorString)(nvmlReturn_t) = nullptr;
    nvmlReturn_t (*HandleByPci)(const char *, nvmlDevice_t *) = nullptr;
    nvmlReturn_t (*FieldValues)(nvmlDevice_t, int, nvmlFieldValue_t *) = nullptr;
    nvmlReturn_t (*PowerUsage)(nvmlDevice_t, unsigned *) = nullptr;
    nvmlReturn_t (*TotalEnergy)(nvmlDevice_t, unsigned long long *) = nullptr;
    nvmlReturn_t (*ClockInfo)(nvmlDevice_t, nvmlClockType_t, unsigned *) = nullptr;
    nvmlReturn_t (*MaxClockInfo)(nvmlDevice_t, nvmlClockType_t, unsigned *) = nullptr;
    nvmlReturn_t (*DefaultAppClock)(nvmlDevice_t, nvmlClockType_t, unsigned *) = nullptr;
    nvmlReturn_t (*Temperature)(nvmlDevice_t, nvmlTemperatureSensors_t, unsigned *) = nullptr;
    nvmlReturn_t (*Reasons)(nvmlDevice_t, unsigned long long *) = nullptr;
    nvmlReturn_t (*MemClocks)(nvmlDevice_t, unsigned *, unsigned *) = nullptr;
    nvmlReturn_t (*GrClocks)(nvmlDevice_t, unsigned, unsigned *, unsigned *) = nullptr;
    nvmlReturn_t (*LimitRange)(nvmlDevice_t, unsigned *, unsigned *) = nullptr;
    nvmlReturn_t (*Limit)(nvmlDevice_t, unsigned *) = nullptr;
    nvmlReturn_t (*DefaultLimit)(nvmlDevice_t, unsigned *) = nullptr;
    nvmlReturn_t (*EnforcedLimit)(nvmlDevice_t, unsigned *) = nullptr;
    nvmlReturn_t (*SetLocked)(nvmlDevice_t, unsigned, unsigned) = nullptr;
    nvmlReturn_t (*ResetLocked)(nvmlDevice_t) = nullptr;
    nvmlReturn_t (*SetLimit)(nvmlDevice_t, unsigned) = nullptr;
    nvmlReturn_t (*SetAppClocks)(nvmlDevice_t, unsigned, unsigned) = nullptr;
    nvmlReturn_t (*ResetAppClocks)(nvmlDevice_t) = nullptr;
};

Nvml g_nvml;
std::once_flag g_nvml_once;

template <class F>
void sym(void *lib, F &fn, const char *name) {
    fn = reinterpret_cast<F>(dlsym(lib, name));
}

void nvml_load() {
    const char *names[] = {"libnvidia-ml.so.1", "libnvidia-ml.so"};
    for (const char *n : names) {
        g_nvml.lib = dlopen(n, RTLD_NOW | RTLD_LOCAL);
        if (g_nvml.lib) break;
    }
    if (!g_nvml.lib) return;
    void *l = g_nvml.lib;
    sym(l, g_nvml.Init, "nvmlInit_v2");
    sym(l, g_nvml.ErrorString, "nvmlErrorString");
    sym(l, g_nvml.HandleByPci, "nvmlDeviceGetHandleByPciBusId_v2");
    sym(l, g_nvml.FieldValues, "nvmlDeviceGetFieldValues");
    sym(l, g_nvml.PowerUsage, "nvmlDeviceGetPowerUsage");
    sym(l, g_nvml.TotalEnergy, "nvmlDeviceGetTotalEnergyConsumption");
    sym(l, g_nvml.ClockInfo, "nvmlDeviceGetClockInfo");
    sym(l, g_nvml.MaxClockInfo, "nvmlDeviceGetMaxClockInfo");
    sym(l, g_nvml.DefaultAppClock, "nvmlDeviceGetDefaultApplicationsClock");
    sym(l, g_nvml.Temperature, "nvmlDeviceGetTemperature");
    sym(l, g_nvml.Reasons, "nvmlDeviceGetCurrentClocksEventReasons");
    if (!g_nvml.Reasons) sym(l, g_nvml.Reasons, "nvmlDeviceGetCurrentClocksThrottleReasons");
    sym(l, g_nvml.MemClocks, "nvmlDeviceGetSupportedMemoryClocks");
    sym(l, g_nvml.GrClocks, "nvmlDeviceGetSupportedGraphicsClocks");
    sym(l, g_nvml.LimitRange, "nvmlDeviceGetPowerManagementLimitConstraints");
    sym(l, g_nvml.Limit, "nvmlDeviceGetPowerManagementLimit");
    sym(l, g_nvml.DefaultLimit, "nvmlDeviceGetPowerManagementDefaultLimit");
    sym(l, g_nvml.EnforcedLimit, "nvmlDeviceGetEnforcedPowerLimit");
    sym(l, g_nvml.SetLocked, "nvmlDeviceSetGpuLockedClocks");
    sym(l, g_nvml.ResetLocked, "nvmlDeviceResetGpuLockedClocks");
    sym(l, g_nvml.SetLimit, "nvmlDeviceSetPowerManagementLimit");
    sym(l, g_nvml.SetAppClocks, "nvmlDeviceSetApplicationsClocks");
    sym(l, g_nvml.ResetAppClocks, "nvmlDeviceResetApplicationsClocks");
    g_nvml.ok = g_nvml.Init && g_nvml.HandleByPci && g_nvml.Init() == NVML_SUCCESS;
}

const char *nvml_err(nvmlReturn_t r) {
    return g_nvml.ErrorString ? g_nvml.ErrorString(r) : "nvml error";
}

}  // namespace

// ---------------------------------------------------------------------------
struct jt_module {
    CUmodule mod;
};

struct jt_kernel {
    CUfunction fn;
    unsigned smem_attr = 0;  // dynamic smem limit already raised to this value
};

struct jt_ctx {
    int ordinal = 0;
    CUdevice dev = 0;
    CUcontext cu = nullptr;
    CUstream stream = nullptr;             // stream 0: the context's own
    std::vector<CUstream> lanes;           // streams 1..n (jt_streams_reserve)
    int cur = 0;                           // stream launches / copies / events go to
    CUevent ev_a = nullptr, ev_b = nullptr, ev_m = nullptr;
    CUdeviceptr flush_buf = 0;
    size_t flush_bytes = 0;
    jt_device_info info{};
    nvmlDevice_t nvdev = nullptr;
    bool have_nvml = false;
    double realtime_offset = 0.0;  // real_now() - mono_now() at open
    bool clocks_locked = false;
    bool app_clocks_set = false;
    bool limit_changed = false;
    // sampler
    std::thread sampler;
    std::atomic<bool> sampling{false};
    std::mutex sample_mu;
    std::vector<jt_sample> samples;
    size_t sample_cap = 0;
    int period_us = 1000;
    std::vector<CUevent> events;
    // stream gate (jt_stream_gate / jt_stream_release): a mapped host word the stream waits on
    volatile unsigned *gate_host = nullptr;
    CUdeviceptr gate_dev = 0;
    unsigned gate_value = 0;
    std::vector<jt_module *> modules;
    std::vector<jt_kernel *> kernels;
};

namespace {

inline CUstream active(const jt_ctx *c) { return c->cur == 0 ? c->stream : c->lanes[c->cur - 1]; }

std::mutex g_open_mu;
std::set<jt_ctx *> g_open;
std::once_flag g_atexit_once;

void reset_controls(jt_ctx *c) {
    if (!c->have_nvml) return;
    if (c->clocks_locked && g_nvml.ResetLocked) {
        g_nvml.ResetLocked(c->nvdev);
        c->clocks_locked = false;
    }
    if (c->app_clocks_set && g_nvml.ResetAppClocks) {
        g_nvml.ResetAppClocks(c->nvdev);
        c->app_clocks_set = false;
    }
    if (c->limit_changed && g_nvml.SetLimit && c->info.power_limit_default_mw) {
        g_nvml.SetLimit(c->nvdev, c->info.power_limit_default_mw);
        c->limit_changed = false;
    }
}

void reset_all_at_exit() {
    std::lock_guard<std::mutex> g(g_open_mu);
    for (jt_ctx *c : g_open) reset_controls(c);
}

int bind(jt_ctx *c) {
    if (!c) return fail(JT_EINVAL, "null context");
    CU_TRY(D.p_cuCtxSetCurrent(c->cu), "cuCtxSetCurrent");
    return JT_OK;
}

void read_sample(jt_ctx *c, jt_sample *s) {
    std::memset(s, 0, sizeof *s);
    s->t_s = mono_now();
    s->power_w = NAN;
    s->power_avg_w = NAN;
    s->energy_j = NAN;
    s->energy_stamp_s = NAN;
    if (!c->have_nvml) return;
    nvmlFieldValue_t fv[2];
    std::memset(fv, 0, sizeof fv);
    fv[0].fieldId = NVML_FI_DEV_POWER_INSTANT;
    fv[1].fieldId = NVML_FI_DEV_TOTAL_ENERGY_CONSUMPTION;
    if (g_nvml.FieldValues && g_nvml.FieldValues(c->nvdev, 2, fv) == NVML_SUCCESS) {
        if (fv[0].nvmlReturn == NVML_SUCCESS) {
            double mw = fv[0].valueType == NVML_VALUE_TYPE_UNSIGNED_LONG_LONG ? (double)fv[0].value.ullVal
                                                                               : (double)fv[0].value.uiVal;
            s->power_w = mw * 1e-3;
        }
        if (fv[1].nvmlReturn == NVML_SUCCESS) {
            s->energy_j = (double)fv[1].value.ullVal * 1e-3;
            s->energy_stamp_s = (double)fv[1].timestamp * 1e-6 - c->realtime_offset;
        }
    }
    if (std::isnan(s->energy_j) && g_nvml.TotalEnergy) {
        unsigned long long mj = 0;
        if (g_nvml.TotalEnergy(c->nvdev, &mj) == NVML_SUCCESS) s->energy_j = mj * 1e-3;
    }
    unsigned v = 0;
    if (g_nvml.PowerUsage && g_nvml.PowerUsage(c->nvdev, &v) == NVML_SUCCESS) s->power_avg_w = v * 1e-3;
    if (g_nvml.ClockInfo && g_nvml.ClockInfo(c->nvdev, NVML_CLOCK_SM, &v) == NVML_SUCCESS) s->sm_mhz = v;
    if (g_nvml.ClockInfo && g_nvml.ClockInfo(c->nvdev, NVML_CLOCK_MEM, &v) == NVML_SUCCESS) s->mem_mhz = v;
    if (g_nvml.Temperature && g_nvml.Temperature(c->nvdev, NVML_TEMPERATURE_GPU, &v) == NVML_SUCCESS)
        s->temp_c = v;
    unsigned long long reasons = 0;
    if (g_nvml.Reasons && g_nvml.Reasons(c->nvdev, &reasons) == NVML_SUCCESS) s->reasons = reasons;
}

void sampler_loop(jt_ctx *c) {
    using clk = std::chrono::steady_clock;
    auto next = clk::now();
    const auto period = std::chrono::microseconds(c->period_us);
    while (c->sampling.load(std::memory_order_relaxed)) {
        jt_sample s;
        read_sample(c, &s);
        {
            std::lock_guard<std::mutex> g(c->sample_mu);
            if (c->samples.size() < c->sample_cap) c->samples.push_back(s);
        }
        next += period;
        auto now = clk::now();
        if (next < now) next = now;  // fell behind: do not burst
        std::this_thread::sleep_until(next);
    }
}

int start_sampler(jt_ctx *c, int period_us, int cap) {
    if (c->sampling.load()) return fail(JT_EINVAL, "sampler already running");
    c->period_us = std::max(period_us, 100);
    c->sample_cap = (size_t)std::max(cap, 1);
    c->samples.clear();
    c->samples.reserve(c->sample_cap);
    c->sampling.store(true);
    c->sampler = std::thread(sampler_loop, c);
    return JT_OK;
}

int stop_sampler(jt_ctx *c, jt_sample *out, int cap, int *n) {
    if (!c->sampling.load()) {
        if (n) *n = 0;
        return JT_OK;
    }
    c->sampling.store(false);
    if (c->sampler.joinable()) c->sampler.join();
    // one closing sample so the trace covers the end of the measured region
    jt_sample last;
    read_sample(c, &last);
    std::lock_guard<std::mutex> g(c->sample_mu);
    if (c->samples.size() < c->sample_cap) c->samples.push_back(last);
    int k = (int)std::min<size_t>(c->samples.size(), (size_t)std::max(cap, 0));
    if (out && k) std::memcpy(out, c->samples.data(), k * sizeof(jt_sample));
    if (n) *n = k;
    return JT_OK;
}

int launch_on(jt_ctx *c, jt_kernel *k, const jt_launch_shape *s, void **params) {
    // raised whenever it changes: static + dynamic shared memory above 48 KB needs it even when
    // the dynamic part alone is below (cuLaunchKernel fails with INVALID_VALUE otherwise)
    if (s->smem_bytes > 0 && s->smem_bytes != k->smem_attr) {
        CUresult r = D.p_cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)s->smem_bytes);
        if (r != CUDA_SUCCESS) return cu_fail(r, "raise dynamic shared memory limit");
        k->smem_attr = s->smem_bytes;
    }
    if (s->cluster_x > 1) {
        CUlaunchConfig cfg;
        std::memset(&cfg, 0, sizeof cfg);
        cfg.gridDimX = s->grid[0];
        cfg.gridDimY = s->grid[1];
        cfg.gridDimZ = s->grid[2];
        cfg.blockDimX = s->block[0];
        cfg.blockDimY = s->block[1];
        cfg.blockDimZ = s->block[2];
        cfg.sharedMemBytes = s->smem_bytes;
        cfg.hStream = active(c);
        CUlaunchAttribute attr;
        std::memset(&attr, 0, sizeof attr);
        attr.id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
        attr.value.clusterDim.x = s->cluster_x;
        attr.value.clusterDim.y = 1;
        attr.value.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        CU_TRY(D.p_cuLaunchKernelEx(&cfg, k->fn, params, nullptr), "cuLaunchKernelEx");
        return JT_OK;
    }
    CU_TRY(D.p_cuLaunchKernel(k->fn, s->grid[0], s->grid[1], s->grid[2], s->block[0], s->block[1], s->block[2],
                          s->smem_bytes, active(c), params, nullptr),
           "cuLaunchKernel");
    return JT_OK;
}

int pack_args(const jt_arg *args, int n, std::vector<void *> &params) {
    if (n < 0 || (n > 0 && !args)) return fail(JT_EINVAL, "bad argument list");
    params.resize(n);
    for (int i = 0; i < n; ++i) {
        const jt_arg &a = args[i];
        switch (a.kind) {
            case JT_ARG_PTR: params[i] = (void *)&a.v.ptr; break;
            case JT_ARG_I32: params[i] = (void *)&a.v.i32; break;
            case JT_ARG_F32: params[i] = (void *)&a.v.f32; break;
            case JT_ARG_F64: params[i] = (void *)&a.v.f64; break;
            case JT_ARG_I64: params[i] = (void *)&a.v.i64; break;
            case JT_ARG_BLOB:
                if (!a.v.ptr) return fail(JT_EINVAL, "argument %d: null blob", i);
                params[i] = (void *)a.v.ptr;
                break;
            default: return fail(JT_EINVAL, "argument %d has unknown kind %d", i, a.kind);
        }
    }
    return JT_OK;
}

int check_shape(const jt_launch_shape *s) {
    if (!s) return fail(JT_EINVAL, "null launch shape");
    for (int i = 0; i < 3; ++i)
        if (s->grid[i] == 0 || s->block[i] == 0) return fail(JT_ELAUNCH, "zero grid/block dimension");
    return JT_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

int jt_abi_version(void) { return JT_ABI_VERSION; }

double jt_now(void) { return mono_now(); }

const char *jt_last_error(void) { return g_error.c_str(); }

int jt_device_count(int *count) {
    if (!count) return fail(JT_EINVAL, "null count");
    *count = 0;
    if (!driver_ready()) return fail(JT_ENOGPU, "%s", g_driver_why.c_str());
    CUresult r = D.p_cuInit(0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuInit");
    CU_TRY(D.p_cuDeviceGetCount(count), "cuDeviceGetCount");
    return JT_OK;
}

int jt_open(int ordinal, jt_ctx **out) {
    if (!out) return fail(JT_EINVAL, "null out");
    *out = nullptr;
    if (!driver_ready()) return fail(JT_ENOGPU, "%s", g_driver_why.c_str());
    CUresult r = D.p_cuInit(0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuInit (no usable CUDA driver/GPU)");
    int n = 0;
    CU_TRY(D.p_cuDeviceGetCount(&n), "cuDeviceGetCount");
    if (ordinal < 0 || ordinal >= n) return fail(JT_ENOGPU, "CUDA ordinal %d not present (%d devices)", ordinal, n);
    auto *c = new jt_ctx();
    c->ordinal = ordinal;
    c->realtime_offset = real_now() - mono_now();
    auto bail = [&](int code) {
        delete c;
        return code;
    };
    if ((r = D.p_cuDeviceGet(&c->dev, ordinal)) != CUDA_SUCCESS) return bail(cu_fail(r, "cuDeviceGet"));
    if ((r = D.p_cuDevicePrimaryCtxRetain(&c->cu, c->dev)) != CUDA_SUCCESS) return bail(cu_fail(r, "retain primary ctx"));
    if ((r = D.p_cuCtxSetCurrent(c->cu)) != CUDA_SUCCESS) return bail(cu_fail(r, "cuCtxSetCurrent"));
    if ((r = D.p_cuStreamCreate(&c->stream, CU_STREAM_NON_BLOCKING)) != CUDA_SUCCESS) return bail(cu_fail(r, "stream"));
    if ((r = D.p_cuEventCreate(&c->ev_a, CU_EVENT_DEFAULT)) != CUDA_SUCCESS) return bail(cu_fail(r, "event"));
    if ((r = D.p_cuEventCreate(&c->ev_b, CU_EVENT_DEFAULT)) != CUDA_SUCCESS) return bail(cu_fail(r, "event"));
    if ((r = D.p_cuEventCreate(&c->ev_m, CU_EVENT_DEFAULT)) != CUDA_SUCCESS) return bail(cu_fail(r, "event"));

    jt_device_info &d = c->info;
    d.ordinal = ordinal;
    D.p_cuDeviceGetName(d.name, sizeof d.name, c->dev);
    D.p_cuDeviceGetAttribute(&d.cc_major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, c->dev);
    D.p_cuDeviceGetAttribute(&d.cc_minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, c->dev);
    D.p_cuDeviceGetAttribute(&d.sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, c->dev);
    D.p_cuDeviceGetAttribute(&d.max_smem_optin, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN, c->dev);
    D.p_cuDeviceGetAttribute(&d.l2_bytes, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE, c->dev);
    size_t mem = 0;
    D.p_cuDeviceTotalMem(&mem, c->dev);
    d.total_mem = mem;
    D.p_cuDeviceGetPCIBusId(d.pci_bus_id, sizeof d.pci_bus_id, c->dev);

    std::call_once(g_nvml_once, nvml_load);
    if (g_nvml.ok && g_nvml.HandleByPci(d.pci_bus_id, &c->nvdev) == NVML_SUCCESS) {
        c->have_nvml = true;
        d.nvml_ok = 1;
        jt_sample probe;
        read_sample(c, &probe);
        d.energy_counter_ok = !std::isnan(probe.energy_j);
        d.instant_power_ok = !std::isnan(probe.power_w);
        unsigned mems[64];
        unsigned nm = 64;
        if (g_nvml.MemClocks && g_nvml.MemClocks(c->nvdev, &nm, mems) == NVML_SUCCESS && nm > 0) {
            d.mem_clock_mhz = *std::max_element(mems, mems + nm);
            unsigned ng = 512;
            unsigned grs[512];
            if (g_nvml.GrClocks && g_nvml.GrClocks(c->nvdev, d.mem_clock_mhz, &ng, grs) == NVML_SUCCESS) {
                std::sort(grs, grs + ng);
                ng = (unsigned)(std::unique(grs, grs + ng) - grs);
                d.n_clocks = ng;
                std::memcpy(d.clocks_mhz, grs, ng * sizeof(unsigned));
            }
        }
        unsigned v = 0;
        if (g_nvml.MaxClockInfo && g_nvml.MaxClockInfo(c->nvdev, NVML_CLOCK_SM, &v) == NVML_SUCCESS)
            d.max_sm_clock_mhz = v;
        if (g_nvml.DefaultAppClock && g_nvml.DefaultAppClock(c->nvdev, NVML_CLOCK_SM, &v) == NVML_SUCCESS)
            d.default_sm_clock_mhz = v;
        unsigned lo = 0, hi = 0;
        if (g_nvml.LimitRange && g_nvml.LimitRange(c->nvdev, &lo, &hi) == NVML_SUCCESS) {
            d.power_limit_min_mw = lo;
            d.power_limit_max_mw = hi;
        }
        if (g_nvml.DefaultLimit && g_nvml.DefaultLimit(c->nvdev, &v) == NVML_SUCCESS) d.power_limit_default_mw = v;
        if (g_nvml.Limit && g_nvml.Limit(c->nvdev, &v) == NVML_SUCCESS) d.power_limit_mw = v;
        if (g_nvml.EnforcedLimit && g_nvml.EnforcedLimit(c->nvdev, &v) == NVML_SUCCESS) d.tdp_mw = v;
    }
    {
        std::lock_guard<std::mutex> g(g_open_mu);
        g_open.insert(c);
    }
    std::call_once(g_atexit_once, [] { std::atexit(reset_all_at_exit); });
    *out = c;
    return JT_OK;
}

int jt_close(jt_ctx *c) {
    if (!c) return JT_OK;
    {
        std::lock_guard<std::mutex> g(g_open_mu);
        g_open.erase(c);
    }
    if (c->sampling.load()) stop_sampler(c, nullptr, 0, nullptr);
    reset_controls(c);
    D.p_cuCtxSetCurrent(c->cu);
    D.p_cuStreamSynchronize(c->stream);
    for (CUstream st : c->lanes) {
        D.p_cuStreamSynchronize(st);
        D.p_cuStreamDestroy(st);
    }
    for (jt_kernel *k : c->kernels) delete k;
    for (jt_module *m : c->modules) {
        D.p_cuModuleUnload(m->mod);
        delete m;
    }
    if (c->flush_buf) D.p_cuMemFree(c->flush_buf);
    if (c->gate_host) D.p_cuMemFreeHost((void *)c->gate_host);
    for (CUevent e : c->events) D.p_cuEventDestroy(e);
    D.p_cuEventDestroy(c->ev_a);
    D.p_cuEventDestroy(c->ev_b);
    D.p_cuEventDestroy(c->ev_m);
    D.p_cuStreamDestroy(c->stream);
    D.p_cuDevicePrimaryCtxRelease(c->dev);
    delete c;
    return JT_OK;
}

int jt_device_info_get(jt_ctx *c, jt_device_info *out) {
    if (!c || !out) return fail(JT_EINVAL, "null argument");
    if (c->have_nvml) {
        unsigned v = 0;
        if (g_nvml.Limit && g_nvml.Limit(c->nvdev, &v) == NVML_SUCCESS) c->info.power_limit_mw = v;
    }
    *out = c->info;
    return JT_OK;
}

// --- memory ------------------------------------------------------------------
int jt_alloc(jt_ctx *c, size_t bytes, unsigned long long *dptr) {
    if (int e = bind(c)) return e;
    if (!dptr || bytes == 0) return fail(JT_EINVAL, "bad allocation request");
    CUdeviceptr p = 0;
    CU_TRY(D.p_cuMemAlloc(&p, bytes), "cuMemAlloc");
    *dptr = (unsigned long long)p;
    return JT_OK;
}

int jt_free(jt_ctx *c, unsigned long long dptr) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemFree((CUdeviceptr)dptr), "cuMemFree");
    return JT_OK;
}

int jt_host_alloc(jt_ctx *c, size_t bytes, void **hptr) {
    if (int e = bind(c)) return e;
    if (!hptr || bytes == 0) return fail(JT_EINVAL, "bad host allocation request");
    CU_TRY(D.p_cuMemHostAlloc(hptr, bytes, CU_MEMHOSTALLOC_PORTABLE), "cuMemHostAlloc");
    return JT_OK;
}

int jt_host_free(jt_ctx *c, void *hptr) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemFreeHost(hptr), "cuMemFreeHost");
    return JT_OK;
}

int jt_h2d(jt_ctx *c, unsigned long long dst, const void *src, size_t bytes) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemcpyHtoDAsync((CUdeviceptr)dst, src, bytes, active(c)), "cuMemcpyHtoDAsync");
    CU_TRY(D.p_cuStreamSynchronize(active(c)), "h2d sync");
    return JT_OK;
}

int jt_d2h(jt_ctx *c, void *dst, unsigned long long src, size_t bytes) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemcpyDtoHAsync(dst, (CUdeviceptr)src, bytes, active(c)), "cuMemcpyDtoHAsync");
    CU_TRY(D.p_cuStreamSynchronize(active(c)), "d2h sync");
    return JT_OK;
}

int jt_memset_d8(jt_ctx *c, unsigned long long dst, unsigned char value, size_t bytes) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemsetD8Async((CUdeviceptr)dst, value, bytes, active(c)), "cuMemsetD8Async");
    return JT_OK;
}

int jt_synchronize(jt_ctx *c) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuStreamSynchronize(c->stream), "cuStreamSynchronize");
    for (CUstream st : c->lanes) CU_TRY(D.p_cuStreamSynchronize(st), "cuStreamSynchronize");
    return JT_OK;
}

int jt_streams_reserve(jt_ctx *c, int n) {
    if (int e = bind(c)) return e;
    if (n < 1 || n > 64) return fail(JT_EINVAL, "bad stream count %d", n);
    while ((int)c->lanes.size() + 1 < n) {
        CUstream st;
        CU_TRY(D.p_cuStreamCreate(&st, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
        c->lanes.push_back(st);
    }
    return JT_OK;
}

int jt_stream_select(jt_ctx *c, int index) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (index < 0 || index > (int)c->lanes.size()) return fail(JT_EINVAL, "stream %d not reserved", index);
    c->cur = index;
    return JT_OK;
}

int jt_stream_wait_event(jt_ctx *c, int event_index) {
    if (int e = bind(c)) return e;
    if (event_index < 0 || event_index >= (int)c->events.size())
        return fail(JT_EINVAL, "event %d not reserved", event_index);
    CU_TRY(D.p_cuStreamWaitEvent(active(c), c->events[event_index], 0), "cuStreamWaitEvent");
    return JT_OK;
}

// --- compile / load ------------------------------------------------------------
//
// NVRTC is dlopen'ed by full path from the toolkit the library was built against
// (JT_CUDA_HOME, else CUDA_HOME, else /usr/local/cuda), RTLD_LOCAL. Linking it by
// soname would bind to whichever libnvrtc.so.12 the process loaded first: after
// `import torch` that is torch's bundled 12.8 copy, whose ptxas rejects PTX 8.8
// forms the kernels use (ld.global.v8.f32 = LDG.E.256), and whose code generation
// would silently differ between test processes that did or did not import torch.
namespace {
struct Nvrtc {
    std::once_flag once;
    void *lib = nullptr;
    std::string path;
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) get_log = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) get_cubin = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    decltype(&nvrtcGetErrorString) error_string = nullptr;
    decltype(&nvrtcVersion) version = nullptr;
} g_nvrtc;

int nvrtc_load() {
    std::call_once(g_nvrtc.once, [] {
        std::vector<std::string> tries;
        for (const char *env : {"JT_CUDA_HOME", "CUDA_HOME"})
            if (const char *h = std::getenv(env); h && *h) tries.push_back(std::string(h) + "/lib64/libnvrtc.so.12");
#ifdef JT_CUDA_LIB_DIR
        tries.push_back(JT_CUDA_LIB_DIR "/libnvrtc.so.12");  // the toolkit libjt was built against
#endif
        tries.push_back("/usr/local/cuda/lib64/libnvrtc.so.12");
        tries.push_back("libnvrtc.so.12");  // last resort: whatever the loader finds
        for (const auto &p : tries) {
            if ((g_nvrtc.lib = dlopen(p.c_str(), RTLD_NOW | RTLD_LOCAL))) {
                g_nvrtc.path = p;
                break;
            }
        }
        if (!g_nvrtc.lib) return;
        auto sym = [](auto &fn, const char *name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(g_nvrtc.lib, name)); };
        sym(g_nvrtc.create, "nvrtcCreateProgram");
        sym(g_nvrtc.compile, "nvrtcCompileProgram");
        sym(g_nvrtc.log_size, "nvrtcGetProgramLogSize");
        sym(g_nvrtc.get_log, "nvrtcGetProgramLog");
        sym(g_nvrtc.cubin_size, "nvrtcGetCUBINSize");
        sym(g_nvrtc.get_cubin, "nvrtcGetCUBIN");
        sym(g_nvrtc.destroy, "nvrtcDestroyProgram");
        sym(g_nvrtc.error_string, "nvrtcGetErrorString");
        sym(g_nvrtc.version, "nvrtcVersion");
    });
    if (!g_nvrtc.lib) return fail(JT_ECOMPILE, "libnvrtc.so.12 not found (set JT_CUDA_HOME)");
    if (!g_nvrtc.create || !g_nvrtc.compile || !g_nvrtc.log_size || !g_nvrtc.get_log || !g_nvrtc.cubin_size ||
        !g_nvrtc.get_cubin || !g_nvrtc.destroy || !g_nvrtc.error_string || !g_nvrtc.version)
        return fail(JT_ECOMPILE, "%s lacks an NVRTC entry point", g_nvrtc.path.c_str());
    return JT_OK;
}
}  // namespace

int jt_nvrtc_version(int *major, int *minor, char *path, size_t path_capacity) {
    if (!major || !minor) return fail(JT_EINVAL, "null version argument");
    if (int e = nvrtc_load()) return e;
    g_nvrtc.version(major, minor);
    if (path && path_capacity) {
        std::snprintf(path, path_capacity, "%s", g_nvrtc.path.c_str());
    }
    return JT_OK;
}

int jt_compile(const char *source, const char *program_name, const char *const *options, int n_options,
               void **image, size_t *image_bytes, char *log, size_t log_capacity) {
    if (!source || !image || !image_bytes) return fail(JT_EINVAL, "null compile argument");
    *image = nullptr;
    *image_bytes = 0;
    if (log && log_capacity) log[0] = 0;
    if (int e = nvrtc_load()) return e;
    const Nvrtc &N = g_nvrtc;
    nvrtcProgram prog;
    nvrtcResult r = N.create(&prog, source, program_name ? program_name : "kernel.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return fail(JT_ECOMPILE, "nvrtcCreateProgram: %s", N.error_string(r));
    r = N.compile(prog, n_options, options);
    size_t log_size = 0;
    N.log_size(prog, &log_size);
    if (log && log_capacity && log_size > 1) {
        std::vector<char> buf(log_size + 1);
        N.get_log(prog, buf.data());
        size_t k = std::min(log_capacity - 1, log_size);
        std::memcpy(log, buf.data(), k);
        log[k] = 0;
    }
    if (r != NVRTC_SUCCESS) {
        N.destroy(&prog);
        return fail(JT_ECOMPILE, "nvrtcCompileProgram: %s", N.error_string(r));
    }
    size_t n = 0;
    r = N.cubin_size(prog, &n);
    if (r != NVRTC_SUCCESS || n == 0) {
        N.destroy(&prog);
        return fail(JT_ECOMPILE, "no cubin produced (use --gpu-architecture=sm_100a): %s", N.error_string(r));
    }
    void *buf = std::malloc(n);
    N.get_cubin(prog, (char *)buf);
    N.destroy(&prog);
    *image = buf;
    *image_bytes = n;
    return JT_OK;
}

void jt_free_image(void *image) { std::free(image); }

int jt_module_load(jt_ctx *c, const void *image, size_t image_bytes, jt_module **out) {
    if (int e = bind(c)) return e;
    if (!image || !image_bytes || !out) return fail(JT_EINVAL, "null module image");
    CUmodule m;
    CUresult r = D.p_cuModuleLoadData(&m, image);
    if (r != CUDA_SUCCESS) {
        int code = cu_fail(r, "cuModuleLoadData");
        return code == JT_ECUDA ? JT_ECOMPILE : code;
    }
    auto *jm = new jt_module{m};
    c->modules.push_back(jm);
    *out = jm;
    return JT_OK;
}

int jt_module_unload(jt_ctx *c, jt_module *m) {
    if (int e = bind(c)) return e;
    if (!m) return JT_OK;
    auto it = std::find(c->modules.begin(), c->modules.end(), m);
    if (it == c->modules.end()) return fail(JT_EINVAL, "module not owned by this context");
    D.p_cuModuleUnload(m->mod);
    c->modules.erase(it);
    delete m;
    return JT_OK;
}

int jt_kernel_get(jt_ctx *c, jt_module *m, const char *name, jt_kernel **out) {
    if (int e = bind(c)) return e;
    if (!m || !name || !out) return fail(JT_EINVAL, "null kernel lookup argument");
    CUfunction f;
    CUresult r = D.p_cuModuleGetFunction(&f, m->mod, name);
    if (r != CUDA_SUCCESS) return fail(JT_EINVAL, "kernel %s not in module: %s", name, cu_name(r));
    auto *k = new jt_kernel();
    k->fn = f;
    c->kernels.push_back(k);
    *out = k;
    return JT_OK;
}

int jt_kernel_attributes(jt_ctx *c, jt_kernel *k, int *regs, int *static_smem, int *local_bytes, int *max_threads) {
    if (int e = bind(c)) return e;
    if (!k) return fail(JT_EINVAL, "null kernel");
    if (regs) D.p_cuFuncGetAttribute(regs, CU_FUNC_ATTRIBUTE_NUM_REGS, k->fn);
    if (static_smem) D.p_cuFuncGetAttribute(static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, k->fn);
    if (local_bytes) D.p_cuFuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, k->fn);
    if (max_threads) D.p_cuFuncGetAttribute(max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, k->fn);
    return JT_OK;
}

int jt_kernel_occupancy(jt_ctx *c, jt_kernel *k, int block_threads, size_t dynamic_smem, int *blocks_per_sm) {
    if (int e = bind(c)) return e;
    if (!k || !blocks_per_sm || block_threads < 1) return fail(JT_EINVAL, "bad occupancy arguments");
    if (dynamic_smem > 0 && (unsigned)dynamic_smem != k->smem_attr) {
        CUresult r = D.p_cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)dynamic_smem);
        if (r != CUDA_SUCCESS) return cu_fail(r, "raise dynamic shared memory limit");
        k->smem_attr = (unsigned)dynamic_smem;
    }
    CU_TRY(D.p_cuOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k->fn, block_threads, dynamic_smem),
           "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    return JT_OK;
}

// --- execution -----------------------------------------------------------------
int jt_launch(jt_ctx *c, jt_kernel *k, const jt_launch_shape *s, const jt_arg *args, int n_args) {
    if (int e = bind(c)) return e;
    if (!k) return fail(JT_EINVAL, "null kernel");
    if (int e = check_shape(s)) return e;
    std::vector<void *> params;
    if (int e = pack_args(args, n_args, params)) return e;
    return launch_on(c, k, s, params.data());
}

int jt_time(jt_ctx *c, jt_kernel *k, const jt_launch_shape *s, const jt_arg *args, int n_args, int reps,
            double *seconds) {
    if (int e = bind(c)) return e;
    if (!k || !seconds || reps < 1) return fail(JT_EINVAL, "bad jt_time arguments");
    if (int e = check_shape(s)) return e;
    std::vector<void *> params;
    if (int e = pack_args(args, n_args, params)) return e;
    CU_TRY(D.p_cuEventRecord(c->ev_a, active(c)), "cuEventRecord");
    for (int i = 0; i < reps; ++i)
        if (int e = launch_on(c, k, s, params.data())) return e;
    CU_TRY(D.p_cuEventRecord(c->ev_b, active(c)), "cuEventRecord");
    CU_TRY(D.p_cuEventSynchronize(c->ev_b), "kernel execution");
    float ms = 0.f;
    CU_TRY(D.p_cuEventElapsedTime(&ms, c->ev_a, c->ev_b), "cuEventElapsedTime");
    *seconds = ms * 1e-3;
    return JT_OK;
}

int jt_bench(jt_ctx *c, jt_kernel *k, const jt_launch_shape *s, const jt_arg *args, int n_args, double min_seconds,
             int min_reps, int max_reps, int sample_period_us, jt_bench_result *out, jt_sample *samples, int cap) {
    return jt_bench_sets(c, k, s, args, n_args, 1, min_seconds, min_reps, max_reps, sample_period_us, out, samples,
                         cap);
}

int jt_bench_sets(jt_ctx *c, jt_kernel *k, const jt_launch_shape *s, const jt_arg *args, int n_args, int n_sets,
                  double min_seconds, int min_reps, int max_reps, int sample_period_us, jt_bench_result *out,
                  jt_sample *samples, int cap) {
    if (int e = bind(c)) return e;
    if (!k || !out || n_sets < 1) return fail(JT_EINVAL, "bad jt_bench arguments");
    if (int e = check_shape(s)) return e;
    std::memset(out, 0, sizeof *out);
    // launch i uses argument set i % n_sets (inputs rotate so no launch reads an L2-warm set)
    std::vector<std::vector<void *>> params(n_sets);
    for (int j = 0; j < n_sets; ++j)
        if (int e = pack_args(args + (size_t)j * n_args, n_args, params[j])) return e;
    min_reps = std::max(min_reps, 1);
    max_reps = std::max(max_reps, min_reps);
    const bool sampling = samples && cap > 0;
    if (sampling)
        if (int e = start_sampler(c, sample_period_us, cap)) return e;
    auto finish = [&](int code) {
        if (sampling) {
            int n = 0;
            stop_sampler(c, samples, cap, &n);
            out->n_samples = n;
        }
        return code;
    };
    // probe launch (also the warm-up): untimed by the loop, timed by events
    CUresult r;
    if ((r = D.p_cuEventRecord(c->ev_a, active(c))) != CUDA_SUCCESS) return finish(cu_fail(r, "cuEventRecord"));
    if (int e = launch_on(c, k, s, params[0].data())) return finish(e);
    if ((r = D.p_cuEventRecord(c->ev_b, active(c))) != CUDA_SUCCESS) return finish(cu_fail(r, "cuEventRecord"));
    if ((r = D.p_cuEventSynchronize(c->ev_b)) != CUDA_SUCCESS) return finish(cu_fail(r, "kernel execution"));
    float ms = 0.f;
    D.p_cuEventElapsedTime(&ms, c->ev_a, c->ev_b);
    out->first_launch_s = ms * 1e-3;
    double probe = std::max(out->first_launch_s, 1e-7);
    long want = (long)std::ceil(min_seconds / probe);
    int reps = (int)std::min<long>(std::max<long>(want, min_reps), max_reps);

    // The probe launch (cold clocks, cold caches) usually overestimates a launch, so the loop is
    // sized in three parts without ever idling the GPU: a first quarter timed on its own (ev_m),
    // a second quarter enqueued behind it to keep the GPU busy while the host waits on ev_m, then
    // the remainder recomputed from the measured quarter so the loop lasts >= min_seconds.
    out->host_t_enqueue = mono_now();
    if ((r = D.p_cuEventRecord(c->ev_a, active(c))) != CUDA_SUCCESS) return finish(cu_fail(r, "cuEventRecord"));
    int done = 0;
    const int quarter = std::max(1, reps / 4);
    const bool adaptive = reps >= 8 && min_seconds > 0;
    int first = adaptive ? quarter : reps;
    for (; done < first; ++done)
        if (int e = launch_on(c, k, s, params[done % n_sets].data())) return finish(e);
    if (adaptive) {
        if ((r = D.p_cuEventRecord(c->ev_m, active(c))) != CUDA_SUCCESS) return finish(cu_fail(r, "cuEventRecord"));
        for (int i = 0; i < quarter && done < max_reps; ++i, ++done)
            if (int e = launch_on(c, k, s, params[done % n_sets].data())) return finish(e);
        if ((r = D.p_cuEventSynchronize(c->ev_m)) != CUDA_SUCCESS) return finish(cu_fail(r, "kernel execution"));
        float q_ms = 0.f;
        D.p_cuEventElapsedTime(&q_ms, c->ev_a, c->ev_m);
        const double per = std::max(q_ms * 1e-3 / first, 1e-8);
        // 3% over: launches after the measured quarter run a little faster (clocks and caches
        // settle), and the loop must not end short of min_seconds (reference "at least")
        long total = std::max<long>((long)std::ceil(1.03 * min_seconds / per), min_reps);
        total = std::min<long>(total, max_reps);
        for (; done < total; ++done)
            if (int e = launch_on(c, k, s, params[done % n_sets].data())) return finish(e);
    }
    reps = done;
    if ((r = D.p_cuEventRecord(c->ev_b, active(c))) != CUDA_SUCCESS) return finish(cu_fail(r, "cuEventRecord"));
    if ((r = D.p_cuEventSynchronize(c->ev_b)) != CUDA_SUCCESS) return finish(cu_fail(r, "kernel execution"));
    out->host_t_done = mono_now();
    D.p_cuEventElapsedTime(&ms, c->ev_a, c->ev_b);
    out->total_s = ms * 1e-3;
    out->reps = reps;
    out->per_launch_s = out->total_s / reps;
    out->loop_t0 = out->host_t_done - out->total_s;
    return finish(JT_OK);
}

int jt_events_reserve(jt_ctx *c, int n) {
    if (int e = bind(c)) return e;
    if (n < 0 || n > (1 << 20)) return fail(JT_EINVAL, "bad event count %d", n);
    while ((int)c->events.size() < n) {
        CUevent ev;
        CU_TRY(D.p_cuEventCreate(&ev, CU_EVENT_DEFAULT), "cuEventCreate");
        c->events.push_back(ev);
    }
    return JT_OK;
}

int jt_event_record(jt_ctx *c, int index) {
    if (int e = bind(c)) return e;
    if (index < 0 || index >= (int)c->events.size()) return fail(JT_EINVAL, "event %d not reserved", index);
    CU_TRY(D.p_cuEventRecord(c->events[index], active(c)), "cuEventRecord");
    return JT_OK;
}

int jt_stream_gate(jt_ctx *c) {
    if (int e = bind(c)) return e;
    if (!c->gate_host) {
        void *h = nullptr;
        CU_TRY(D.p_cuMemHostAlloc(&h, 64, CU_MEMHOSTALLOC_PORTABLE | CU_MEMHOSTALLOC_DEVICEMAP), "cuMemHostAlloc");
        CUdeviceptr d = 0;
        CUresult r = D.p_cuMemHostGetDevicePointer(&d, h, 0);
        if (r != CUDA_SUCCESS) {
            D.p_cuMemFreeHost(h);
            return cu_fail(r, "cuMemHostGetDevicePointer");
        }
        c->gate_host = static_cast<volatile unsigned *>(h);
        c->gate_dev = d;
        __atomic_store_n(const_cast<unsigned *>(c->gate_host), 0u, __ATOMIC_SEQ_CST);
        c->gate_value = 0;
    }
    // the stream holds until the host word reaches the next value; work enqueued behind it (events
    // included) starts only at jt_stream_release
    const unsigned want = c->gate_value + 1;
    CU_TRY(D.p_cuStreamWaitValue32(active(c), c->gate_dev, want, CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue32");
    c->gate_value = want;
    return JT_OK;
}

int jt_stream_release(jt_ctx *c) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->gate_host) return fail(JT_EINVAL, "no stream gate armed");
    __atomic_store_n(const_cast<unsigned *>(c->gate_host), c->gate_value, __ATOMIC_SEQ_CST);
    return JT_OK;
}

int jt_event_elapsed(jt_ctx *c, int start, int stop, double *seconds) {
    if (int e = bind(c)) return e;
    const int n = (int)c->events.size();
    if (!seconds || start < 0 || stop < 0 || start >= n || stop >= n) return fail(JT_EINVAL, "bad event index");
    CU_TRY(D.p_cuEventSynchronize(c->events[stop]), "cuEventSynchronize");
    float ms = 0.f;
    CU_TRY(D.p_cuEventElapsedTime(&ms, c->events[start], c->events[stop]), "cuEventElapsedTime");
    *seconds = ms * 1e-3;
    return JT_OK;
}

int jt_h2d_async(jt_ctx *c, unsigned long long dst, const void *src, size_t bytes) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemcpyHtoDAsync((CUdeviceptr)dst, src, bytes, active(c)), "cuMemcpyHtoDAsync");
    return JT_OK;
}

int jt_d2h_async(jt_ctx *c, void *dst, unsigned long long src, size_t bytes) {
    if (int e = bind(c)) return e;
    CU_TRY(D.p_cuMemcpyDtoHAsync(dst, (CUdeviceptr)src, bytes, active(c)), "cuMemcpyDtoHAsync");
    return JT_OK;
}

int jt_h2d_2d_async(jt_ctx *c, unsigned long long dst, size_t dst_pitch, const void *src, size_t src_pitch,
                    size_t width_bytes, size_t rows) {
    if (int e = bind(c)) return e;
    if (width_bytes > dst_pitch || width_bytes > src_pitch) return fail(JT_EINVAL, "row wider than its pitch");
    if (!rows || !width_bytes) return JT_OK;
    CUDA_MEMCPY2D m;
    std::memset(&m, 0, sizeof m);
    m.srcMemoryType = CU_MEMORYTYPE_HOST;
    m.srcHost = src;
    m.srcPitch = src_pitch;
    m.dstMemoryType = CU_MEMORYTYPE_DEVICE;
    m.dstDevice = (CUdeviceptr)dst;
    m.dstPitch = dst_pitch;
    m.WidthInBytes = width_bytes;
    m.Height = rows;
    CU_TRY(D.p_cuMemcpy2DAsync(&m, active(c)), "cuMemcpy2DAsync (H2D)");
    return JT_OK;
}

int jt_d2h_2d_async(jt_ctx *c, void *dst, size_t dst_pitch, unsigned long long src, size_t src_pitch,
                    size_t width_bytes, size_t rows) {
    if (int e = bind(c)) return e;
    if (width_bytes > dst_pitch || width_bytes > src_pitch) return fail(JT_EINVAL, "row wider than its pitch");
    if (!rows || !width_bytes) return JT_OK;
    CUDA_MEMCPY2D m;
    std::memset(&m, 0, sizeof m);
    m.srcMemoryType = CU_MEMORYTYPE_DEVICE;
    m.srcDevice = (CUdeviceptr)src;
    m.srcPitch = src_pitch;
    m.dstMemoryType = CU_MEMORYTYPE_HOST;
    m.dstHost = dst;
    m.dstPitch = dst_pitch;
    m.WidthInBytes = width_bytes;
    m.Height = rows;
    CU_TRY(D.p_cuMemcpy2DAsync(&m, active(c)), "cuMemcpy2DAsync (D2H)");
    return JT_OK;
}

int jt_l2_flush(jt_ctx *c) {
    if (int e = bind(c)) return e;
    if (!c->flush_buf) {
        c->flush_bytes = std::max<size_t>((size_t)c->info.l2_bytes * 2, (size_t)256 << 20);
        CU_TRY(D.p_cuMemAlloc(&c->flush_buf, c->flush_bytes), "alloc L2 flush buffer");
    }
    CU_TRY(D.p_cuMemsetD8Async(c->flush_buf, 0x5a, c->flush_bytes, active(c)), "L2 flush");
    return JT_OK;
}

// --- sensors ---------------------------------------------------------------------
int jt_sample_now(jt_ctx *c, jt_sample *out) {
    if (!c || !out) return fail(JT_EINVAL, "null argument");
    read_sample(c, out);
    return c->have_nvml ? JT_OK : fail(JT_ENVML, "NVML not available for this device");
}

int jt_sampler_start(jt_ctx *c, int period_us, int cap) {
    if (!c) return fail(JT_EINVAL, "null context");
    return start_sampler(c, period_us, cap);
}

int jt_sampler_stop(jt_ctx *c, jt_sample *out, int cap, int *n) {
    if (!c) return fail(JT_EINVAL, "null context");
    return stop_sampler(c, out, cap, n);
}

// --- controller ------------------------------------------------------------------
static int nvml_status(nvmlReturn_t r, const char *what) {
    if (r == NVML_SUCCESS) return JT_OK;
    if (r == NVML_ERROR_NO_PERMISSION) return fail(JT_ENOPERM, "%s: %s", what, nvml_err(r));
    if (r == NVML_ERROR_NOT_SUPPORTED) return fail(JT_ENOTSUP, "%s: %s", what, nvml_err(r));
    if (r == NVML_ERROR_INVALID_ARGUMENT) return fail(JT_EINVAL, "%s: %s", what, nvml_err(r));
    return fail(JT_ENVML, "%s: %s", what, nvml_err(r));
}

int jt_clock_lock(jt_ctx *c, unsigned min_mhz, unsigned max_mhz) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->have_nvml || !g_nvml.SetLocked) return fail(JT_ENVML, "NVML clock control unavailable");
    if (min_mhz > max_mhz) return fail(JT_EINVAL, "min clock above max clock");
    int e = nvml_status(g_nvml.SetLocked(c->nvdev, min_mhz, max_mhz), "nvmlDeviceSetGpuLockedClocks");
    if (e == JT_OK) c->clocks_locked = true;
    return e;
}

int jt_clock_reset(jt_ctx *c) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->have_nvml || !g_nvml.ResetLocked) return fail(JT_ENVML, "NVML clock control unavailable");
    int e = nvml_status(g_nvml.ResetLocked(c->nvdev), "nvmlDeviceResetGpuLockedClocks");
    if (e == JT_OK) c->clocks_locked = false;
    return e;
}

int jt_app_clocks_set(jt_ctx *c, unsigned mem_mhz, unsigned sm_mhz) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->have_nvml || !g_nvml.SetAppClocks) return fail(JT_ENVML, "NVML applications clocks unavailable");
    int e = nvml_status(g_nvml.SetAppClocks(c->nvdev, mem_mhz, sm_mhz), "nvmlDeviceSetApplicationsClocks");
    if (e == JT_OK) c->app_clocks_set = true;
    return e;
}

int jt_app_clocks_reset(jt_ctx *c) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->have_nvml || !g_nvml.ResetAppClocks) return fail(JT_ENVML, "NVML applications clocks unavailable");
    int e = nvml_status(g_nvml.ResetAppClocks(c->nvdev), "nvmlDeviceResetApplicationsClocks");
    if (e == JT_OK) c->app_clocks_set = false;
    return e;
}

int jt_power_limit_set(jt_ctx *c, unsigned mw) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->have_nvml || !g_nvml.SetLimit) return fail(JT_ENVML, "NVML power control unavailable");
    int e = nvml_status(g_nvml.SetLimit(c->nvdev, mw), "nvmlDeviceSetPowerManagementLimit");
    if (e == JT_OK) c->limit_changed = (mw != c->info.power_limit_default_mw);
    return e;
}

int jt_power_limit_reset(jt_ctx *c) {
    if (!c) return fail(JT_EINVAL, "null context");
    if (!c->info.power_limit_default_mw) return fail(JT_ENOTSUP, "default power limit unknown");
    return jt_power_limit_set(c, c->info.power_limit_default_mw);
}

// --- kernel-suite helpers ---------------------------------------------------------
int jt_pnpoly_edges(const float *vx, const float *vy, int n, int method, float *edges, float *ybounds) {
    if (!vx || !vy || !edges || !ybounds || n < 3) return fail(JT_EINVAL, "polygon needs >= 3 vertices");
    if (method < 0 || method > 2) return fail(JT_EINVAL, "unknown PnPoly method %d", method);
    for (int k = 0; k < n; ++k) {
        const int p = (k + n - 1) % n;
        const float dx = vx[p] - vx[k];
        const float dy = vy[p] - vy[k];
        float *e = edges + 4 * k;
        e[0] = vy[k];
        if (method == 0) {
            e[1] = vx[k];
            e[2] = dx;
            e[3] = dy;
        } else {
            volatile float slope = dx / dy;  // IEEE division, never contracted
            e[1] = method == 1 ? vx[k] : std::fmaf(-slope, vy[k], vx[k]);
            e[2] = slope;
            e[3] = 0.f;
        }
        ybounds[2 * k] = std::min(vy[k], vy[p]);
        ybounds[2 * k + 1] = std::max(vy[k], vy[p]);
    }
    return JT_OK;
}

// The kernel's bucket index, op for op: min(max(__float2int_rz((v - base) * scale), 0), hi)
// with cvt.rzi.s32 semantics (NaN -> 0, saturation at the int range). This
// file is built with -ffp-contract=off, so (v - base) * scale rounds twice,
// like __fsub_rn / __fmul_rn on the device.
static int slab_bucket(float v, float base, float scale, int hi) {
    const float f = (v - base) * scale;
    long long k;
    if (std::isnan(f)) k = 0;
    else if (f >= 2147483647.f) k = 2147483647LL;
    else if (f <= -2147483648.f) k = -2147483648LL;
    else k = (long long)std::trunc(f);
    return (int)std::min<long long>(std::max<long long>(k, 0), hi);
}

// float32 -> IEEE binary16 bits, rounded toward -inf (dir < 0) or +inf (dir > 0):
// the result, read back as a float, is <= (resp. >=) v. Overflow goes to +-inf.
static uint16_t half_round(float v, int dir) {
    if (std::isnan(v)) return 0x7e00;
    auto to_float = [](uint16_t h) -> float {
        const int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
        float f = e == 0 ? std::ldexp((float)m, -24) : e == 31 ? (m ? NAN : INFINITY) : std::ldexp(1024.f + m, e - 25);
        return s ? -f : f;
    };
    // nearest-ish candidate by scanning the ordered code space with a binary search on magnitude
    const float a = std::fabs(v);
    uint16_t lo = 0, hi = 0x7c00;  // +0 .. +inf
    while (lo < hi) {  // smallest magnitude code >= a
        const uint16_t mid = (uint16_t)((lo + hi) / 2);
        if (to_float(mid) >= a) hi = mid; else lo = (uint16_t)(mid + 1);
    }
    uint16_t up = lo;                                               // |h| >= a
    uint16_t dn = to_float(up) == a ? up : (uint16_t)(up - 1);      // |h| <= a
    const bool neg = std::signbit(v);
    // magnitude rounding direction flips for negative values
    const uint16_t mag = (dir > 0) != neg ? up : dn;
    return (uint16_t)(mag | (neg ? 0x8000 : 0));
}

static float half_value(uint16_t h) {
    const int e = (h >> 10) & 31, m = h & 1023;
    const float f = e == 0 ? std::ldexp((float)m, -24) : e == 31 ? (m ? NAN : INFINITY) : std::ldexp(1024.f + m, e - 25);
    return (h >> 15) ? -f : f;
}

// Bucket starts with an exactness flag. vals: sorted ascending; bucket(v) is
// monotone in v, so #{vals <= v} is constant over bucket g unless some value
// and its float predecessor share bucket g. Exact buckets get that count and
// `flag`; the others get #{bucket(val) < g} (a start the kernel corrects).
static void slab_bucket_starts(const float *vals, int m, float base, float scale, int hi, unsigned flag,
                               std::vector<unsigned> &out) {
    out.assign(hi + 1, 0u);
    std::vector<char> split(hi + 1, 0);
    std::vector<int> at(m);
    for (int i = 0; i < m; ++i) {
        at[i] = slab_bucket(vals[i], base, scale, hi);
        if (slab_bucket(std::nextafter(vals[i], -INFINITY), base, scale, hi) == at[i]) split[at[i]] = 1;
    }
    int below = 0, upto = 0;  // #{at < g}, #{at <= g}
    for (int g = 0; g <= hi; ++g) {
        while (below < m && at[below] < g) ++below;
        upto = std::max(upto, below);
        while (upto < m && at[upto] <= g) ++upto;
        out[g] = split[g] ? (unsigned)below : ((unsigned)upto | flag);
    }
}

int jt_pnpoly_slabs(const float *vx, const float *vy, int n, int buckets, int pad, int xbuckets, float *table,
                    long long capacity, jt_slab_info *info) {
    if (!vx || !vy || !info || n < 3) return fail(JT_EINVAL, "polygon needs >= 3 vertices");
    if (buckets < 1 || buckets > (1 << 20)) return fail(JT_EINVAL, "bucket count %d out of range", buckets);
    if (pad < 1 || pad > 64) return fail(JT_EINVAL, "band padding %d out of range", pad);
    if (xbuckets < 0 || xbuckets > 4096) return fail(JT_EINVAL, "x-bucket count %d out of range", xbuckets);
    const bool xsearch = xbuckets > 0;
    // METHOD 2 edge records, bit for bit those of jt_pnpoly_edges
    std::vector<float> slope(n), icpt(n), ylo(n), yhi(n);
    for (int k = 0; k < n; ++k) {
        if (std::isnan(vy[k]) || std::isnan(vx[k])) return fail(JT_EINVAL, "vertex %d is NaN", k);
        const int p = (k + n - 1) % n;
        const float dx = vx[p] - vx[k];
        const float dy = vy[p] - vy[k];
        volatile float s = dx / dy;
        slope[k] = s;
        icpt[k] = std::fmaf(-slope[k], vy[k], vx[k]);
        ylo[k] = std::min(vy[k], vy[p]);
        yhi[k] = std::max(vy[k], vy[p]);
    }
    // distinct vertex ordinates (IEEE equality: -0.0 == +0.0)
    std::vector<float> u(vy, vy + n);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end(), [](float a, float b) { return a == b; }), u.end());
    const int nu = (int)u.size();
    // slab r = #{u <= py}: r = 0 and r = nu span nothing; slab r in [1, nu-1]
    // holds every edge with ylo <= u[r-1] and yhi >= u[r], i.e. every edge
    // whose (vy_k > py) != (vy_j > py) for all py in [u[r-1], u[r])
    if (xsearch) pad = 1;
    std::vector<int> off(nu + 2, 0);
    std::vector<int> members;
    std::vector<float> xlo, xhi;
    int max_band = 0;
    for (int r = 0; r <= nu; ++r) {
        off[r] = (int)members.size();
        if (r == 0 || r == nu) continue;
        const size_t first = members.size();
        for (int k = 0; k < n; ++k)
            if (ylo[k] <= u[r - 1] && yhi[k] >= u[r]) members.push_back(k);
        if (xsearch) {
            // fma(slope, py, icpt) is monotone in py (a correctly rounded
            // monotone function), so over the slab's py in [u[r-1], pred(u[r])]
            // each edge's computed crossing abscissa lies in [lo, hi], its two
            // end values. px < lo: the edge certainly crosses; px >= hi: it
            // certainly does not; otherwise the kernel evaluates it. A NaN end
            // value widens the interval to (-inf, +inf).
            const float top = std::nextafter(u[r], -INFINITY);
            std::vector<float> los, his;
            for (size_t i = first; i < members.size(); ++i) {
                const int k = members[i];
                const float a = std::fmaf(slope[k], u[r - 1], icpt[k]);
                const float b = std::fmaf(slope[k], top, icpt[k]);
                const bool nan = std::isnan(a) || std::isnan(b);
                los.push_back(nan ? -INFINITY : std::min(a, b));
                his.push_back(nan ? INFINITY : std::max(a, b));
            }
            std::vector<int> idx(los.size());
            for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
            std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return los[a] < los[b]; });
            std::vector<int> sorted(idx.size());
            for (size_t i = 0; i < idx.size(); ++i) {
                sorted[i] = members[first + idx[i]];
                xlo.push_back(los[idx[i]]);
                xhi.push_back(his[idx[i]]);
            }
            std::copy(sorted.begin(), sorted.end(), members.begin() + first);
        }
        int cnt = (int)(members.size() - first);
        for (; cnt % pad; ++cnt) members.push_back(-1);  // never-crossing filler
        max_band = std::max(max_band, cnt);
    }
    off[nu + 1] = (int)members.size();
    const int ne = (int)members.size();
    auto up4 = [](long long w) { return (w + 3) / 4 * 4; };
    info->nu = nu;
    info->ng = buckets;
    info->ne = ne;
    info->max_band = max_band;
    info->u_off = 0;
    info->guess_off = (int)up4(nu);
    info->band_off = info->guess_off + (int)up4(buckets);
    info->xb = xbuckets;
    if (xsearch) {
        info->xpar_off = info->band_off + (int)up4(nu + 2);                 // {b, cnt, x0, xscale} per slab
        info->xst_off = info->xpar_off + 4 * (nu + 1);                      // uint16 [nu+1][xb+1]
        // compact copy first: one word per edge, lo rounded down | pmax rounded up to binary16
        info->half_off = info->xst_off + (int)up4(((long long)(nu + 1) * (xbuckets + 1) + 1) / 2);
        info->xlo_off = info->half_off + (int)up4(ne);
        info->pmax_off = info->xlo_off + (int)up4(ne);
        info->pair_off = info->pmax_off + (int)up4(ne);  // records {slope, icpt, hi, 0}
        info->words = info->pair_off + 4 * ne;
        if (max_band > 32767) return fail(JT_EINVAL, "slab of %d edges exceeds the 15-bit x-bucket index", max_band);
    } else {
        info->xpar_off = info->xst_off = info->half_off = 0;
        info->xlo_off = info->pmax_off = 0;
        info->pair_off = info->band_off + (int)up4(nu + 2);  // pairs {slope, icpt}
        info->words = info->pair_off + 2 * ne;
    }
    info->ybase = u[0];
    info->yscale = nu > 1 && u[nu - 1] > u[0] ? (float)buckets / (u[nu - 1] - u[0]) : 0.f;
    if (!table) return JT_OK;  // size query
    if (capacity < info->words) return fail(JT_EINVAL, "slab table needs %d words, got %lld", info->words, capacity);
    std::memset(table, 0, sizeof(float) * info->words);
    std::memcpy(table + info->u_off, u.data(), sizeof(float) * nu);
    // rank = #{u <= py} per y-bucket; bit 31 set: exact for every py of the bucket
    std::vector<unsigned> starts;
    slab_bucket_starts(u.data(), nu, info->ybase, info->yscale, buckets - 1, 0x80000000u, starts);
    std::memcpy(table + info->guess_off, starts.data(), sizeof(unsigned) * buckets);
    std::memcpy(table + info->band_off, off.data(), sizeof(int) * (nu + 2));
    if (xsearch) {
        float *lo = table + info->xlo_off, *pm = table + info->pmax_off, *rec = table + info->pair_off;
        float *xpar = table + info->xpar_off;
        uint16_t *xst = reinterpret_cast<uint16_t *>(table + info->xst_off);
        std::vector<unsigned> xs;
        for (int r = 1; r < nu; ++r) {
            float run = -INFINITY;
            for (int i = off[r]; i < off[r + 1]; ++i) {
                run = std::max(run, xhi[i]);
                lo[i] = xlo[i];
                pm[i] = run;  // max hi over the slab's edges up to and including i
            }
            // slab record {first edge, edge count, x0, xscale}; x-buckets: pos = #{lo <= px}
            // per bucket, bit 15 set where it is exact (else a start the kernel corrects)
            const int cnt = off[r + 1] - off[r];
            int32_t *srec = reinterpret_cast<int32_t *>(xpar + 4 * r);
            srec[0] = off[r];
            srec[1] = cnt;
            if (!cnt) continue;
            const float x0 = xlo[off[r]], x1 = xlo[off[r + 1] - 1];
            const float scale = std::isfinite(x0) && std::isfinite(x1) && x1 > x0 ? (float)xbuckets / (x1 - x0) : 0.f;
            const float base = std::isfinite(x0) ? x0 : 0.f;
            xpar[4 * r + 2] = base;
            xpar[4 * r + 3] = scale;
            slab_bucket_starts(xlo.data() + off[r], cnt, base, scale, xbuckets, 0x8000u, xs);
            for (int k = 0; k <= xbuckets; ++k) xst[(size_t)r * (xbuckets + 1) + k] = (uint16_t)xs[k];
        }
        for (int i = 0; i < ne; ++i) {
            const int k = members[i];
            rec[4 * i] = slope[k];
            rec[4 * i + 1] = icpt[k];
            rec[4 * i + 2] = xhi[i];
        }
        uint32_t *half = reinterpret_cast<uint32_t *>(table + info->half_off);
        std::vector<float> lo16(ne);
        for (int i = 0; i < ne; ++i) {  // conservative: lo never above, pmax never below the float32 value
            const uint16_t l = half_round(lo[i], -1);
            half[i] = (uint32_t)l | ((uint32_t)half_round(pm[i], +1) << 16);
            lo16[i] = half_value(l);
        }
        // skip pointer (record word 3): the largest j < i in the slab with hi_j > lo16_i, else -1.
        // The kernel visits undecided candidates (j < pos with hi_j > px) from pos - 1 down; every
        // visited j has lo16_j <= px, so an edge strictly between skip(j) and j (hi <= lo16_j <= px)
        // can never be one. lo16 (<= lo) keeps this valid for both the float32 and the HALF tables.
        int32_t *recw = reinterpret_cast<int32_t *>(rec);
        for (int r = 1; r < nu; ++r)
            for (int i = off[r]; i < off[r + 1]; ++i) {
                int j = i - 1;
                while (j >= off[r] && !(xhi[j] > lo16[i])) --j;
                recw[4 * i + 3] = j >= off[r] ? j - off[r] : -1;
            }
        return JT_OK;
    }
    float *pairs = table + info->pair_off;
    for (int i = 0; i < ne; ++i) {
        const int k = members[i];
        pairs[2 * i] = k < 0 ? 0.f : slope[k];
        pairs[2 * i + 1] = k < 0 ? -INFINITY : icpt[k];  // fma(0, py, -inf) = -inf: px < x never holds
    }
    return JT_OK;
}

// Monotone integer key of a float (total order of the non-NaN floats, -0.0 < +0.0 by bits).
static uint32_t float_key(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
static float key_float(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
// The grid kernel's cell index, op for op: min(cvt.rzi.u32(fma(v, scale, offset)), hi)
// (cvt.rzi.u32: NaN and negatives -> 0, saturating above). fmaf is correctly rounded, so
// the index is monotone in v for scale >= 0.
static int grid_cell(float v, float scale, float offset, int hi) {
    const float f = std::fmaf(v, scale, offset);
    long long k;
    if (std::isnan(f) || f <= 0.f) k = 0;
    else if (f >= 4294967295.f) k = 4294967295LL;
    else k = (long long)std::trunc(f);
    return (int)std::min<long long>(k, hi);
}
// Smallest non-NaN float v with grid_cell(v) >= k (+inf if none).
static float cell_first(int k, float scale, float offset, int hi) {
    uint32_t lo = float_key(-INFINITY), up = float_key(INFINITY);
    if (grid_cell(key_float(up), scale, offset, hi) < k) return INFINITY;
    while (lo < up) {
        const uint32_t mid = lo + (up - lo) / 2;
        if (grid_cell(key_float(mid), scale, offset, hi) >= k) up = mid; else lo = mid + 1;
    }
    return key_float(lo);
}

int jt_pnpoly_grid(const float *vx, const float *vy, int n, int gw, int gh, float *params, uint32_t *bits,
                   long long capacity, int *clean_cells) {
    if (!vx || !vy || !params || n < 3) return fail(JT_EINVAL, "polygon needs >= 3 vertices");
    if (gw < 1 || gh < 1 || (long long)gw * gh > (1LL << 26)) return fail(JT_EINVAL, "bad grid %d x %d", gw, gh);
    const long long words = ((long long)gw * gh + 15) / 16;
    // METHOD 2 edges and y-slabs, bit for bit those of jt_pnpoly_slabs
    std::vector<float> slope(n), icpt(n), ylo(n), yhi(n);
    float xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    for (int k = 0; k < n; ++k) {
        if (std::isnan(vy[k]) || std::isnan(vx[k])) return fail(JT_EINVAL, "vertex %d is NaN", k);
        const int p = (k + n - 1) % n;
        const float dx = vx[p] - vx[k];
        const float dy = vy[p] - vy[k];
        volatile float s = dx / dy;
        slope[k] = s;
        icpt[k] = std::fmaf(-slope[k], vy[k], vx[k]);
        ylo[k] = std::min(vy[k], vy[p]);
        yhi[k] = std::max(vy[k], vy[p]);
        xmin = std::min(xmin, vx[k]), xmax = std::max(xmax, vx[k]);
        ymin = std::min(ymin, vy[k]), ymax = std::max(ymax, vy[k]);
    }
    std::vector<float> u(vy, vy + n);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end(), [](float a, float b) { return a == b; }), u.end());
    const int nu = (int)u.size();
    // the cell of a point: (min(f2u_rz(fma(px, sx, ox)), gw - 1), same in y), as the kernel computes it
    const float sx = xmax > xmin ? (float)gw / (xmax - xmin) : 0.f;
    const float sy = ymax > ymin ? (float)gh / (ymax - ymin) : 0.f;
    const float ox = -xmin * sx, oy = -ymin * sy;
    params[0] = sx, params[1] = ox, params[2] = sy, params[3] = oy;
    if (!bits) return JT_OK;
    if (capacity < words) return fail(JT_EINVAL, "grid needs %lld words, got %lld", words, capacity);
    std::memset(bits, 0, sizeof(uint32_t) * words);
    // exact float ranges of the cells: [first(k), pred(first(k + 1))]
    std::vector<float> cx0(gw + 1), cy0(gh + 1);
    for (int k = 0; k <= gw; ++k) cx0[k] = k == 0 ? -INFINITY : cell_first(k, sx, ox, gw - 1);
    for (int k = 0; k <= gh; ++k) cy0[k] = k == 0 ? -INFINITY : cell_first(k, sy, oy, gh - 1);
    cx0[gw] = cy0[gh] = INFINITY;
    // slab lists
    std::vector<std::vector<int>> slab(nu + 1);
    for (int r = 1; r < nu; ++r)
        for (int k = 0; k < n; ++k)
            if (ylo[k] <= u[r - 1] && yhi[k] >= u[r]) slab[r].push_back(k);
    auto rank = [&](float y) { return (int)(std::upper_bound(u.begin(), u.end(), y) - u.begin()); };
    int clean = 0;
    std::vector<float> elo, ehi;
    for (int cy = 0; cy < gh; ++cy) {
        const float Y0 = cy0[cy], Y1 = cy0[cy + 1] == INFINITY ? INFINITY : std::nextafter(cy0[cy + 1], -INFINITY);
        if (!(Y0 <= Y1)) continue;  // no float maps to this row
        const int r0 = rank(Y0), r1 = rank(Y1);
        // per slab of the row: the py sub-range and every edge's computed-x range over it
        struct Part { int r; float lo_y, hi_y; };
        std::vector<Part> parts;
        for (int r = r0; r <= r1; ++r) {
            const float a = r == r0 ? Y0 : u[r - 1];
            const float b = r == r1 ? Y1 : std::nextafter(u[r], -INFINITY);
            parts.push_back({r, a, b});
        }
        std::vector<std::vector<std::pair<float, float>>> ranges(parts.size());
        bool row_nan = false;
        for (size_t q = 0; q < parts.size(); ++q) {
            const Part &P = parts[q];
            if (P.r <= 0 || P.r >= nu) continue;
            for (int k : slab[P.r]) {
                const float a = std::fmaf(slope[k], P.lo_y, icpt[k]);
                const float b = std::fmaf(slope[k], P.hi_y, icpt[k]);
                if (std::isnan(a) || std::isnan(b)) row_nan = true;
                ranges[q].push_back({std::min(a, b), std::max(a, b)});
            }
        }
        if (row_nan) continue;  // leave the whole row to the exact search
        for (int cx = 0; cx < gw; ++cx) {
            const float X0 = cx0[cx], X1 = cx0[cx + 1] == INFINITY ? INFINITY : std::nextafter(cx0[cx + 1], -INFINITY);
            if (!(X0 <= X1)) continue;
            // every edge of every slab of the row must be decided for all px in [X0, X1]:
            // X1 < lo (crosses for every point of the cell) or X0 >= hi (for none); and the
            // number of crossings must have one parity in every slab the cell's rows span
            int parity = -1;
            bool ok = true;
            for (size_t q = 0; q < parts.size() && ok; ++q) {
                int cnt = 0;
                for (const auto &lh : ranges[q]) {
                    if (X1 < lh.first) ++cnt;
                    else if (!(X0 >= lh.second)) { ok = false; break; }
                }
                if (ok) {
                    if (parity < 0) parity = cnt & 1;
                    else if (parity != (cnt & 1)) ok = false;
                }
            }
            if (!ok) continue;
            const long long cell = (long long)cy * gw + cx;
            bits[cell >> 4] |= (1u | ((uint32_t)parity << 1)) << ((cell & 15) * 2);  // bit 0 clean, bit 1 inside
            ++clean;
        }
    }
    if (clean_cells) *clean_cells = clean;
    return JT_OK;
}

// Per-cell edge lists for csrc/kernels/pnpoly_cells.cu. The METHOD 2 test of edge k,
// spans(py) && px < fma(slope, py, icpt) with spans = ylo <= py < yhi, is decided for a
// whole cell [X0, X1] x [Y0, Y1] when it is false for every point (no py of the cell's
// rows in the span, or X0 >= every computed x over the spanned py) or true for every
// point (the span covers the rows and X1 < every computed x); computed x is monotone in
// py, so its range over a py interval comes from the interval's ends. The always-true
// edges give the cell's base parity, the undecided ones are listed; a point's answer is
// base ^ the XOR of its listed edges' tests, which is the brute-force XOR over all edges.
int jt_pnpoly_cells(const float *vx, const float *vy, int n, int gw, int gh, int lmax, int head_words, float *params,
                    uint32_t *bits, long long bits_capacity, uint32_t *heads, long long heads_capacity, float *edges,
                    long long edge_capacity, long long *stats) {
    if (!vx || !vy || !params || n < 3) return fail(JT_EINVAL, "polygon needs >= 3 vertices");
    if (gw < 1 || gh < 1 || (long long)gw * gh > (1LL << 24)) return fail(JT_EINVAL, "bad grid %d x %d", gw, gh);
    if (lmax < 0 || lmax > (1 << 20)) return fail(JT_EINVAL, "bad list limit %d", lmax);
    if (head_words != 4 && head_words != 8) return fail(JT_EINVAL, "head_words must be 4 or 8, not %d", head_words);
    const int inline_edges = head_words / 4;  // edges a head holds in place
    const long long cells = (long long)gw * gh, words = (cells + 15) / 16;
    std::vector<float> slope(n), icpt(n), ylo(n), yhi(n);
    float xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    for (int k = 0; k < n; ++k) {
        if (std::isnan(vy[k]) || std::isnan(vx[k])) return fail(JT_EINVAL, "vertex %d is NaN", k);
        const int p = (k + n - 1) % n;
        volatile float s = (vx[p] - vx[k]) / (vy[p] - vy[k]);
        slope[k] = s;
        icpt[k] = std::fmaf(-slope[k], vy[k], vx[k]);
        ylo[k] = std::min(vy[k], vy[p]);
        yhi[k] = std::max(vy[k], vy[p]);
        xmin = std::min(xmin, vx[k]), xmax = std::max(xmax, vx[k]);
        ymin = std::min(ymin, vy[k]), ymax = std::max(ymax, vy[k]);
    }
    // the cell function of jt_pnpoly_grid: min(f2u_rz(fma(v, s, o)), g - 1)
    const float sx = xmax > xmin ? (float)gw / (xmax - xmin) : 0.f;
    const float sy = ymax > ymin ? (float)gh / (ymax - ymin) : 0.f;
    const float ox = -xmin * sx, oy = -ymin * sy;
    params[0] = sx, params[1] = ox, params[2] = sy, params[3] = oy;
    const bool fill = bits && heads;
    if (fill && (bits_capacity < words || heads_capacity < head_words * cells))
        return fail(JT_EINVAL, "cell tables need %lld words and %lld head words", words, head_words * cells);
    if (fill) {
        std::memset(bits, 0, sizeof(uint32_t) * words);
        std::memset(heads, 0, sizeof(uint32_t) * head_words * cells);
    }
    std::vector<float> cx0(gw + 1), cy0(gh + 1);
    for (int k = 0; k <= gw; ++k) cx0[k] = k == 0 ? -INFINITY : cell_first(k, sx, ox, gw - 1);
    for (int k = 0; k <= gh; ++k) cy0[k] = k == 0 ? -INFINITY : cell_first(k, sy, oy, gh - 1);
    cx0[gw] = cy0[gh] = INFINITY;
    long long entries = 0, n_clean = 0, n_listed = 0, n_fallback = 0;
    struct Row { int k; bool full, exact; float xl, xh; };
    std::vector<Row> row;
    std::vector<int> list, part;
    std::vector<float> steps;
    for (int cy = 0; cy < gh; ++cy) {
        const float Y0 = cy0[cy], Y1 = cy0[cy + 1] == INFINITY ? INFINITY : std::nextafter(cy0[cy + 1], -INFINITY);
        if (!(Y0 <= Y1)) continue;  // no float maps to this row
        row.clear();
        for (int k = 0; k < n; ++k) {
            if (!(ylo[k] < yhi[k])) continue;  // horizontal: never spans
            const float a = std::max(Y0, ylo[k]), b = std::min(Y1, std::nextafter(yhi[k], -INFINITY));
            if (!(a <= b)) continue;  // spans no py of the row
            Row r{k, ylo[k] <= Y0 && Y1 < yhi[k], false, 0.f, 0.f};
            if (std::isfinite(slope[k]) && std::isfinite(icpt[k])) {
                const float xa = std::fmaf(slope[k], a, icpt[k]), xb = std::fmaf(slope[k], b, icpt[k]);
                if (!std::isnan(xa) && !std::isnan(xb)) r.exact = true, r.xl = std::min(xa, xb), r.xh = std::max(xa, xb);
            }
            row.push_back(r);
        }
        for (int cx = 0; cx < gw; ++cx) {
            const float X0 = cx0[cx], X1 = cx0[cx + 1] == INFINITY ? INFINITY : std::nextafter(cx0[cx + 1], -INFINITY);
            if (!(X0 <= X1)) continue;
            int base = 0;
            list.clear();
            part.clear();
            for (const Row &r : row) {
                if (r.exact && X0 >= r.xh) continue;  // false for every point
                if (r.exact && X1 < r.xl) {           // true wherever the edge spans py
                    if (r.full) base ^= 1;
                    else part.push_back(r.k);
                    continue;
                }
                list.push_back(r.k);
            }
            // the partly spanning always-right edges contribute the parity of #{k: ylo <= py < yhi},
            // a step function of py: constant over the row when every step y inside (Y0, Y1]
            // toggles it an even number of times (e.g. the two edges at a vertex)
            if (!part.empty()) {
                steps.clear();
                int at_y0 = 0;
                for (int k : part) {
                    at_y0 ^= (ylo[k] <= Y0 && Y0 < yhi[k]) ? 1 : 0;
                    if (Y0 < ylo[k] && ylo[k] <= Y1) steps.push_back(ylo[k]);
                    if (Y0 < yhi[k] && yhi[k] <= Y1) steps.push_back(yhi[k]);
                }
                std::sort(steps.begin(), steps.end());
                bool constant = true;
                for (size_t i = 0; i < steps.size() && constant;) {
                    size_t j = i;
                    while (j < steps.size() && steps[j] == steps[i]) ++j;
                    constant = ((j - i) & 1) == 0;
                    i = j;
                }
                if (constant) base ^= at_y0;
                else list.insert(list.end(), part.begin(), part.end());
            }
            const long long cell = (long long)cy * gw + cx;
            // NaN coordinates land in row 0 / column 0 and are never inside: a clean cell
            // there with base parity 1 is listed (with no edges) so the exact path answers
            const bool border = cx == 0 || cy == 0;
            // codes: 0 / 1 decided (the answer); 2 | base undecided, with a 16-byte head: the
            // one listed edge {slope, icpt, ylo, yhi}, or {first entry, count, NaN, 0} for 0 or
            // >= 2 listed edges in `edges` (count 0xffffffff: over lmax, the slab search).
            // No real edge has ylo NaN (NaN vertices are rejected).
            uint32_t code;
            if (list.empty() && !(border && base)) code = (uint32_t)base, ++n_clean;
            else {
                code = 2u | (uint32_t)base;
                const bool over = (int)list.size() > lmax;
                over ? ++n_fallback : ++n_listed;
                uint32_t *h = fill ? heads + (long long)head_words * cell : nullptr;
                const float nan = std::numeric_limits<float>::quiet_NaN();
                if (!over && list.size() >= 1 && (int)list.size() <= inline_edges) {
                    // the edges in place; an unused second slot is a never-true {0, 0, NaN, 0}
                    for (int j = 0; j < inline_edges && h; ++j) {
                        if (j < (int)list.size()) {
                            const int k = list[(size_t)j];
                            const float e[4] = {slope[k], icpt[k], ylo[k], yhi[k]};
                            std::memcpy(h + 4 * j, e, sizeof e);
                        } else {
                            h[4 * j] = h[4 * j + 1] = h[4 * j + 3] = 0, std::memcpy(h + 4 * j + 2, &nan, 4);
                        }
                    }
                } else {
                    if (h) {
                        h[0] = over ? 0u : (uint32_t)entries, h[1] = over ? 0xffffffffu : (uint32_t)list.size();
                        std::memcpy(h + 2, &nan, 4), h[3] = 0;
                    }
                    if (!over) {
                        if (fill && edges && entries + (long long)list.size() <= edge_capacity)
                            for (size_t i = 0; i < list.size(); ++i) {
                                float *e = edges + 4 * (entries + (long long)i);
                                const int k = list[i];
                                e[0] = slope[k], e[1] = icpt[k], e[2] = ylo[k], e[3] = yhi[k];
                            }
                        entries += (long long)list.size();
                    }
                }
            }
            if (fill) bits[cell >> 4] |= code << ((cell & 15) * 2);  // 16 cells per word
        }
    }
    if (entries > (1LL << 31)) return fail(JT_EINVAL, "cell lists need %lld entries", entries);
    if (stats) stats[0] = entries, stats[1] = n_clean, stats[2] = n_listed, stats[3] = n_fallback;
    if (fill && edges && entries > edge_capacity)
        return fail(JT_EINVAL, "cell lists need %lld entries, got %lld", entries, edge_capacity);
    return JT_OK;
}

int jt_tensor_map_2d(jt_ctx *c, unsigned long long dptr, unsigned long long rows, unsigned long long cols,
                     unsigned box_rows, unsigned box_cols, int swizzle, void *out128) {
    if (int e = bind(c)) return e;
    if (!out128 || !dptr || !rows || !cols || !box_rows || !box_cols) return fail(JT_EINVAL, "bad tensor map request");
    if (swizzle < 0 || swizzle > 6) return fail(JT_EINVAL, "unknown swizzle mode %d", swizzle);
    const unsigned span = swizzle == 1 ? 32 : swizzle == 2 ? 64 : 128;
    if (swizzle && box_cols * 4 > span) return fail(JT_EINVAL, "box inner extent exceeds the swizzle span");
    if ((cols * 4) % 16) return fail(JT_EINVAL, "row pitch must be a multiple of 16 bytes");
    CUtensorMap map;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = D.p_cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)dptr, dims, strides, box,
                                            estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            (CUtensorMapSwizzle)swizzle,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled");
    std::memcpy(out128, &map, sizeof map);
    return JT_OK;
}

int jt_module_set_global(jt_ctx *c, jt_module *m, const char *name, const void *src, size_t bytes) {
    if (int e = bind(c)) return e;
    if (!m || !name || !src) return fail(JT_EINVAL, "null argument");
    CUdeviceptr p = 0;
    size_t size = 0;
    CUresult r = D.p_cuModuleGetGlobal(&p, &size, m->mod, name);
    if (r != CUDA_SUCCESS) return fail(JT_EINVAL, "module has no global %s (%s)", name, cu_name(r));
    if (bytes > size) return fail(JT_EINVAL, "global %s holds %zu bytes, got %zu", name, size, bytes);
    CU_TRY(D.p_cuMemcpyHtoDAsync(p, src, bytes, c->stream), "copy to module global");
    CU_TRY(D.p_cuStreamSynchronize(c->stream), "copy to module global");
    return JT_OK;
}

}  // extern "C"
