// api.cu -- extern "C" boundary of libprng_b200.so (include/prng_b200.h).
//
// Host-side validation mirrors the reference's error behaviour
// (distributions.py:47-48, 60-62, 100-101; engine.py:206, 219); the launch
// planners pick the kernel instantiation and grid.  No entry point on the
// device path allocates memory or synchronises the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/prng_b200.h"
#include "common.cuh"
#include "mrg32k3a.cuh"
#include "philox.cuh"

using namespace prng;

static_assert(sizeof(prng_segment_t) == sizeof(PhiloxSegment), "segment layout");

namespace {

typedef unsigned __int128 u128;

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

}  // namespace

// Shared with the other translation units (calo.cu): one error slot per thread.
int prng_detail_fail(int code, const char* msg) { return fail(code, "%s", msg); }

namespace {

int cuda_fail(cudaError_t e, const char* what) {
    return fail(PRNG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define PRNG_CUDA(call)                                     \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// ---- device resolution: the device that owns `ptr` becomes current for the
// duration of the entry point; DeviceGuard (declared first in every extern "C"
// entry that launches) switches the caller's device back on return, so a
// generate into a tensor on cuda:3 never leaves cuda:3 current.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

int bind_output(const void* ptr, void** dev_ptr) {
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(e, "cudaPointerGetAttributes(out)");
    }
    if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
        int cur = -1;
        PRNG_CUDA(cudaGetDevice(&cur));
        if (cur != attr.device) PRNG_CUDA(cudaSetDevice(attr.device));
        *dev_ptr = const_cast<void*>(ptr);
        return PRNG_OK;
    }
    if (attr.type == cudaMemoryTypeHost && attr.devicePointer != nullptr) {
        *dev_ptr = attr.devicePointer;  // mapped pinned host memory (zero-copy)
        return PRNG_OK;
    }
    return fail(PRNG_ERR_INVALID_PARAMETER, "out must be device memory or mapped pinned host memory");
}

struct DeviceInfo {
    int sms = 0;
    std::map<const void*, int> occ;
};
std::mutex g_mu;
std::map<int, DeviceInfo> g_dev;

// SM count of the current device (cached; 148 on B200, queried so that a
// partitioned / MIG device or another part gets a grid sized for it).
int device_sms(int* sms_out) {
    int dev = 0;
    PRNG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceInfo& di = g_dev[dev];
    if (di.sms == 0) PRNG_CUDA(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
    *sms_out = di.sms;
    return PRNG_OK;
}

int resident_ctas(const void* kernel, int threads, int* sms_out, int* occ_out) {
    int dev = 0;
    PRNG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceInfo& di = g_dev[dev];
    if (di.sms == 0) PRNG_CUDA(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
    auto it = di.occ.find(kernel);
    if (it == di.occ.end()) {
        int o = 0;
        PRNG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, threads, 0));
        it = di.occ.emplace(kernel, o < 1 ? 1 : o).first;
    }
    *sms_out = di.sms;
    *occ_out = it->second;
    return PRNG_OK;
}

// ---- parameter validation (reference error behaviour) ----
int check_uniform(double a, double b) {
    if (!(std::isfinite(a) && std::isfinite(b)) || a >= b)
        return fail(PRNG_ERR_INVALID_RANGE, "uniform range requires finite lo < hi, got [%g, %g)", a, b);
    return PRNG_OK;
}

int check_gaussian(double mean, double sd) {
    if (!std::isfinite(mean) || !std::isfinite(sd) || sd <= 0)
        return fail(PRNG_ERR_INVALID_PARAMETER, "gaussian requires finite mean and stddev > 0, got (%g, %g)", mean,
                    sd);
    return PRNG_OK;
}

int check_lognormal(double m, double s, double displ, double scale) {
    if (!std::isfinite(m) || !std::isfinite(s) || s <= 0 || !std::isfinite(displ) || !std::isfinite(scale) ||
        scale <= 0)
        return fail(PRNG_ERR_INVALID_PARAMETER,
                    "lognormal requires finite m, s > 0, finite displ, scale > 0, got (%g, %g, %g, %g)", m, s, displ,
                    scale);
    return PRNG_OK;
}

int check_gauss_method(int method) {
    if (method != PRNG_METHOD_FAST && method != PRNG_METHOD_ACCURATE && method != PRNG_METHOD_EXACT &&
        method != PRNG_METHOD_PRECISE)
        return fail(PRNG_ERR_INVALID_PARAMETER, "method must be PRNG_METHOD_FAST, _ACCURATE, _EXACT or _PRECISE");
    return PRNG_OK;
}

// ---- exact Box-Muller tables (box_muller_exact, common.cuh) ----
// Built once per process from the host libm -- the library the reference's
// compiled core calls (_core.pyx:116-121) -- on every host thread, then
// uploaded once per device.
constexpr size_t kExactN = size_t(1) << 24;
std::mutex g_exact_mu;
std::vector<double> g_exact_log;
std::vector<double2> g_exact_sc;

void build_exact_host_tables() {
    g_exact_log.resize(kExactN);
    g_exact_sc.resize(kExactN);
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt < 1 ? 1 : (nt > 64 ? 64 : nt);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([t, nt] {
            const double two_pi = kTwoPi;  // distributions.py:25 / _core.pyx:17
            for (size_t i = t; i < kExactN; i += nt) {
                volatile double u1p = (double)(i + 1) * 0x1p-24;  // 1 - u1, exact (m = i + 1)
                g_exact_log[i] = std::log((double)u1p);
                volatile double tt = two_pi * ((double)i * 0x1p-24);  // TWO_PI * u2, one rounding
                const double tv = tt;
                g_exact_sc[i] = make_double2(std::sin(tv), std::cos(tv));
            }
        });
    }
    for (auto& x : th) x.join();
}

__global__ void exact_approx_kernel(double* L, double* S, double* C) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (uint32_t)kExactN; i += gridDim.x * blockDim.x) {
        L[i] = log_u1_f64((16777215u - i) << 8);  // m - 1 = i
        double sn, cs;
        sincos_ref_f64(i << 8, sn, cs);  // k = i
        S[i] = sn;
        C[i] = cs;
    }
}

// Worst differences of the short approximations (the fp32 exact route's
// common path) from the full ones over both whole domains: [0] relative for
// the log, [1] absolute for sin / cos (non-negative doubles order like their
// bit patterns, so atomicMax on the bits).
__global__ void exact_short_bounds_kernel(unsigned long long* out) {
    double rl = 0.0, asc = 0.0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (uint32_t)kExactN; i += gridDim.x * blockDim.x) {
        const uint32_t w0 = (16777215u - i) << 8;
        const double a = log_u1_f64(w0), b = log_u1_f64_short(w0);
        if (a != 0.0) rl = fmax(rl, fabs(b - a) / fabs(a));
        else if (b != 0.0) rl = INFINITY;
        double s, c, s2, c2;
        sincos_2pi_k24_f64(i, s, c);
        sincos_f64_short(i << 8, s2, c2);
        double s3, c3;
        sincos_ref_f64(i << 8, s3, c3);  // the full form incl. the argument-rounding term
        asc = fmax(asc, fmax(fabs(s2 - s3), fabs(c2 - c3)));
        (void)s; (void)c;
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(rl));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(asc));
}

struct ExactDevice {
    ExactCorrections corr{};
    size_t escapes = 0;
};
std::map<int, ExactDevice> g_exact_corr;

// Correction of one approximation: 4-bit ulp delta, or 8 (= -8) for an escape.
inline uint8_t nibble(double want, double approx) {
    long long kw, ka;
    memcpy(&kw, &want, 8);
    memcpy(&ka, &approx, 8);
    const long long d = dkey(kw) - dkey(ka);
    if (d >= -7 && d <= 7 && dunkey(dkey(ka) + d) == kw) return (uint8_t)(d & 0xF);
    return 8;
}

// Builds (once per device) and binds the correction tables.  Safe to call
// while a stream of this thread is being captured into a CUDA graph: the
// build switches this thread to relaxed capture mode and works on a private
// non-blocking stream with stream-ordered allocations, so nothing touches
// the legacy stream or synchronises the device.  The host libm tables
// (384 MB) are released after the upload unless prng_exact_tables_host
// asked for them.
bool g_exact_keep_host = false;

int exact_tables_build(ExactDevice& ed, cudaStream_t st) {
    if (g_exact_log.empty()) build_exact_host_tables();
    // 1. the device approximations over both whole domains
    double* dL = nullptr;
    PRNG_CUDA(cudaMallocAsync((void**)&dL, 3 * kExactN * sizeof(double), st));
    double* dS = dL + kExactN;
    double* dC = dS + kExactN;
    exact_approx_kernel<<<1184, 256, 0, st>>>(dL, dS, dC);
    std::vector<double> aL(kExactN), aS(kExactN), aC(kExactN);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(aL.data(), dL, kExactN * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(aS.data(), dS, kExactN * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(aC.data(), dC, kExactN * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dL, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "exact tables: approximations");
    // 2. ulp corrections to the host libm, escapes where they do not fit
    std::vector<uint8_t> lnib(kExactN / 2), scnib(kExactN);
    for (size_t i = 0; i < kExactN; i += 2)
        lnib[i / 2] = (uint8_t)(nibble(g_exact_log[i], aL[i]) | (nibble(g_exact_log[i + 1], aL[i + 1]) << 4));
    for (size_t i = 0; i < kExactN; ++i)
        scnib[i] = (uint8_t)(nibble(g_exact_sc[i].x, aS[i]) | (nibble(g_exact_sc[i].y, aC[i]) << 4));
    // worst approximation errors (the fp32 route's rounding test): relative
    // for the log (0 only at u1' = 1, where both are exactly 0), absolute for
    // sin / cos
    double rel_log = 0.0, abs_sc = 0.0;
    for (size_t i = 0; i < kExactN; ++i) {
        const double w = g_exact_log[i], a = aL[i];
        if (w == 0.0) {
            if (a != 0.0) rel_log = INFINITY;
        } else {
            rel_log = std::max(rel_log, std::fabs(a - w) / std::fabs(w));
        }
        abs_sc = std::max(abs_sc, std::max(std::fabs(aS[i] - g_exact_sc[i].x), std::fabs(aC[i] - g_exact_sc[i].y)));
    }
    // the short forms' bounds: |short - libm| <= |short - full| + |full - libm|
    unsigned long long* dmax = nullptr;
    PRNG_CUDA(cudaMallocAsync((void**)&dmax, 2 * sizeof(unsigned long long), st));
    PRNG_CUDA(cudaMemsetAsync(dmax, 0, 2 * sizeof(unsigned long long), st));
    exact_short_bounds_kernel<<<1184, 256, 0, st>>>(dmax);
    unsigned long long hmax[2] = {0, 0};
    PRNG_CUDA(cudaGetLastError());
    PRNG_CUDA(cudaMemcpyAsync(hmax, dmax, sizeof hmax, cudaMemcpyDeviceToHost, st));
    PRNG_CUDA(cudaFreeAsync(dmax, st));
    PRNG_CUDA(cudaStreamSynchronize(st));
    double rs, as;
    memcpy(&rs, &hmax[0], 8);
    memcpy(&as, &hmax[1], 8);
    const double rel_short = rs * (1.0 + rel_log) + rel_log;
    const double abs_short = as + abs_sc;
    ed.corr.rel_log = rel_short;
    ed.corr.abs_sc = abs_short;
    ed.corr.tol_c = std::isfinite(rel_short)
                        ? nextafterf((float)(2.0 * (0.5 * rel_short + abs_short + 6.0 * 0x1p-53)), INFINITY)
                        : INFINITY;
    std::vector<uint32_t> eidx[3];
    std::vector<double> eval[3];
    for (size_t i = 0; i < kExactN; ++i) {
        if (((lnib[i / 2] >> ((i & 1) * 4)) & 0xF) == 8) {
            eidx[0].push_back((uint32_t)i);
            eval[0].push_back(g_exact_log[i]);
        }
        if ((scnib[i] & 0xF) == 8) {
            eidx[1].push_back((uint32_t)i);
            eval[1].push_back(g_exact_sc[i].x);
        }
        if ((scnib[i] >> 4) == 8) {
            eidx[2].push_back((uint32_t)i);
            eval[2].push_back(g_exact_sc[i].y);
        }
    }
    // 3. upload: one long-lived allocation (nibbles, then each escape list)
    size_t bytes = lnib.size() + scnib.size();
    for (int t = 0; t < 3; ++t) bytes += eidx[t].size() * 12 + 16;
    char* base = nullptr;
    PRNG_CUDA(cudaMalloc(&base, bytes));
    char* q = base;
    PRNG_CUDA(cudaMemcpyAsync(q, lnib.data(), lnib.size(), cudaMemcpyHostToDevice, st));
    ed.corr.log_nib = reinterpret_cast<const uint8_t*>(q);
    q += lnib.size();
    PRNG_CUDA(cudaMemcpyAsync(q, scnib.data(), scnib.size(), cudaMemcpyHostToDevice, st));
    ed.corr.sc_nib = reinterpret_cast<const uint8_t*>(q);
    q += scnib.size();
    for (int t = 0; t < 3; ++t) {
        const size_t ne = eidx[t].size();
        PRNG_CUDA(cudaMemcpyAsync(q, eval[t].data(), ne * 8, cudaMemcpyHostToDevice, st));
        ed.corr.esc_val[t] = reinterpret_cast<const double*>(q);
        q += ne * 8 + 8;
        PRNG_CUDA(cudaMemcpyAsync(q, eidx[t].data(), ne * 4, cudaMemcpyHostToDevice, st));
        ed.corr.esc_idx[t] = reinterpret_cast<const uint32_t*>(q);
        q += (ne * 4 + 8) / 8 * 8;
        ed.corr.esc_n[t] = (uint32_t)ne;
        ed.escapes += ne;
    }
    PRNG_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
    return PRNG_OK;
}

int exact_tables(XformParams& p) {
    int dev = 0;
    PRNG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_exact_mu);
    auto it = g_exact_corr.find(dev);
    if (it == g_exact_corr.end()) {
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        PRNG_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
        cudaStream_t st = nullptr;
        ExactDevice ed;
        cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        int rc = e == cudaSuccess ? exact_tables_build(ed, st) : cuda_fail(e, "cudaStreamCreateWithFlags");
        if (st) cudaStreamDestroy(st);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (rc) return rc;
        if (!g_exact_keep_host) {
            std::vector<double>().swap(g_exact_log);
            std::vector<double2>().swap(g_exact_sc);
        }
        it = g_exact_corr.emplace(dev, ed).first;
    }
    p.exact = it->second.corr;
    return PRNG_OK;
}

// The fast fp32 lognormal takes ex2.approx.ftz: results below FLT_MIN would
// flush to 0.  |z| <= sqrt(-2 ln 2^-24) < 5.78 on the reference's 24-bit
// grid, so when m - 5.78 s can reach the subnormal range (ln FLT_MIN =
// -87.34) the request takes the accurate route instead (fp64 exp, one cast:
// subnormals kept).
bool logn_fast_ok(double m, double s) { return m - 5.78 * s > -87.0; }

int check_method(int method) {
    if (method != PRNG_METHOD_FAST && method != PRNG_METHOD_ACCURATE && method != PRNG_METHOD_PRECISE)
        return fail(PRNG_ERR_INVALID_PARAMETER, "method must be PRNG_METHOD_FAST, _ACCURATE or _PRECISE");
    return PRNG_OK;
}

// Uniform [a, b) plan.  numpy NEP-50 makes the fp32 affine use f32(b - a)
// and f32(a) (distributions.py:102-103 on an fp32 array); fp64 uses b - a, a.
enum UniformPlan { kPlanIdentity, kPlanFolded, kPlanTwoPass };

struct UniformSpec {
    UniformPlan plan;
    XformParams p;
};

UniformSpec uniform_spec_f32(double a, double b) {
    UniformSpec u{};
    const float S = (float)(b - a), off = (float)a;
    u.p.scale_f = S * 5.9604644775390625e-08f;  // exact power-of-two scaling when normal
    u.p.off_f = off;
    if (S == 1.0f && off == 0.0f)
        u.plan = kPlanIdentity;
    else if (std::isinf(S) || S >= 0x1p-102f)
        u.plan = kPlanFolded;
    else
        u.plan = kPlanTwoPass;
    return u;
}

UniformSpec uniform_spec_f64(double a, double b) {
    UniformSpec u{};
    const double S = b - a;
    u.p.scale_d = S * 5.9604644775390625e-08;
    u.p.mag_d = -S * 0x1p28;  // -2^52 * scale_d
    u.p.off_d = a;
    if (S == 1.0 && a == 0.0)
        u.plan = kPlanIdentity;
    else if (std::isfinite(u.p.mag_d) && S >= 0x1p-998)
        u.plan = kPlanFolded;
    else
        u.plan = kPlanTwoPass;
    return u;
}

XformParams gauss_params(double mean, double sd) {
    XformParams p{};
    p.scale_f = (float)sd;
    p.off_f = (float)mean;
    p.scale_d = sd;
    p.off_d = mean;
    return p;
}

XformParams logn_params(double m, double s, double displ, double scale) {
    XformParams p = gauss_params(m, s);
    p.ln_scale = scale;
    p.ln_displ = displ;
    p.ln_scale_f = (float)scale;
    p.ln_displ_f = (float)displ;
    return p;
}

template <typename T>
int launch_range(T* v, uint64_t n, double lo, double hi, void* stream);

// ---- Philox launch ----
// Plan: scalar head (to a 32-byte boundary) + body groups + scalar tail; the
// body is cut into launches inside which c1..c3 are constant (philox.cuh).
template <int X>
int launch_philox(uint32_t k0, uint32_t k1, const uint32_t* ctr, uint32_t lane, uint64_t n, void* out,
                  const XformParams& p, void* stream) {
    using T = typename XformTraits<X>::T;
    constexpr bool kPair = XformTraits<X>::kPair;
    if (n == 0) return PRNG_OK;
    if (ctr == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "ctr must not be NULL");
    if (lane > 3) return fail(PRNG_ERR_INVALID_PARAMETER, "lane must be 0..3, got %u", lane);
    if (out == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "out must not be NULL");
    if (((uintptr_t)out) % sizeof(T)) return fail(PRNG_ERR_INVALID_PARAMETER, "out is not aligned to its element");
    void* dptr = nullptr;
    int rc = bind_output(out, &dptr);
    if (rc) return rc;

    PhiloxScalar s{};
    s.k0 = k0;
    s.k1 = k1;
    s.ctr_lo = (uint64_t)ctr[0] | ((uint64_t)ctr[1] << 32);
    s.ctr_hi = (uint64_t)ctr[2] | ((uint64_t)ctr[3] << 32);
    s.lane = lane;
    s.n = n;
    uint64_t i0 = ((32u - (uint32_t)((uintptr_t)dptr & 31u)) & 31u) / sizeof(T);
    uint64_t ngroups = 0;
    // Pair transforms need groups that start on a pair boundary: with an odd
    // head (an odd-element output view) the body starts one element early,
    // one element below the 32-byte boundary, and each group is stored as
    // element + aligned pair + element (PhiloxBody::mis).
    const uint32_t mis = (kPair && (i0 & 1)) ? 1u : 0u;
    i0 -= mis;
    if (i0 >= n) {
        i0 = n;  // tiny: everything scalar
    } else {
        ngroups = (n - i0) >> 2;
    }
    s.i0 = i0;
    s.tail0 = i0 + 4 * ngroups;
    const int shift = (int)((lane + i0) & 3);
    const void* kern = shift == 0   ? (const void*)philox_kernel<X, 0>
                       : shift == 1 ? (const void*)philox_kernel<X, 1>
                       : shift == 2 ? (const void*)philox_kernel<X, 2>
                                    : (const void*)philox_kernel<X, 3>;
    if constexpr (kPair) {
        if (mis)
            kern = shift == 0   ? (const void*)philox_kernel<X, 0, true>
                   : shift == 1 ? (const void*)philox_kernel<X, 1, true>
                   : shift == 2 ? (const void*)philox_kernel<X, 2, true>
                                : (const void*)philox_kernel<X, 3, true>;
    }
    int sms = 0, occ = 0;
    rc = resident_ctas(kern, kPhiloxThreads, &sms, &occ);
    if (rc) return rc;
    // persistent grid: every SM filled to the kernel's occupancy (2x / 4x and
    // uncapped grids measured no faster at 2^22-2^26, profiles/r2_ab_small_n_grid.txt)
    const uint64_t cap = (uint64_t)sms * occ;

    u128 blk = (((u128)s.ctr_hi << 64) | s.ctr_lo) + ((lane + i0) >> 2);
    T* body = static_cast<T*>(dptr) + i0;
    uint64_t left = ngroups;
    bool first = true;
    do {
        const uint32_t c0 = (uint32_t)blk;
        uint64_t g = (1ull << 32) - c0;
        if (g > left) g = left;
        if (g > (1ull << 31)) g = 1ull << 31;
        // A launch boundary at an odd group leaves the next body 16-byte
        // aligned; emit one single-group launch to restore 32-byte alignment
        // for the 256-bit stores (rare: only at 2^34-word stream boundaries).
        if (left > 0 && ((uintptr_t)(body + mis) & 31u) != 0) g = 1;
        PhiloxBody a{};
        a.k0 = k0;
        a.k1 = k1;
        a.c0 = c0;
        a.c1 = (uint32_t)(blk >> 32);
        a.c2 = (uint32_t)(blk >> 64);
        a.c3 = (uint32_t)(blk >> 96);
        a.ngroups = (uint32_t)g;
        a.mis = mis;
        a.pre = philox_pre(k0, k1, a.c1, a.c2, a.c3);
        a.out = body;
        a.p = p;
        if (first) a.s = s;  // head/tail ride on the first launch
        uint64_t threads = shift == 0 ? (g + PhiloxBpt<T>::kValue - 1) / PhiloxBpt<T>::kValue : (g + 125) / 126 * 32;
        const uint64_t nscalar = first ? s.i0 + (n - s.tail0) : 0;
        if (nscalar > threads) threads = nscalar;
        uint64_t blocks = (threads + kPhiloxThreads - 1) / kPhiloxThreads;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        void* args[] = {&a};
        PRNG_CUDA(cudaLaunchKernel(kern, dim3((unsigned)blocks), dim3(kPhiloxThreads), args, 0, (cudaStream_t)stream));
        blk += g;
        body += 4 * g;
        left -= g;
        first = false;
    } while (left > 0);
    return PRNG_OK;
}

// ---- MRG32k3a host math: jump matrices A^k mod m ----
struct Mat3 {
    uint64_t v[9];
};

Mat3 mat_mul(const Mat3& a, const Mat3& b, uint64_t m) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            u128 s = 0;
            for (int k = 0; k < 3; ++k) s += (u128)a.v[3 * i + k] * b.v[3 * k + j];
            r.v[3 * i + j] = (uint64_t)(s % m);
        }
    return r;
}

void mat_vec(const Mat3& a, uint32_t* x, uint64_t m) {
    uint64_t r[3];
    for (int i = 0; i < 3; ++i) {
        u128 s = 0;
        for (int k = 0; k < 3; ++k) s += (u128)a.v[3 * i + k] * x[k];
        r[i] = (uint64_t)(s % m);
    }
    for (int i = 0; i < 3; ++i) x[i] = (uint32_t)r[i];
}

// Companion matrices on (x_{n-3}, x_{n-2}, x_{n-1}) (engine.py:165-174).
const Mat3 kA1 = {{0, 1, 0, 0, 0, 1, kMrgM1 - kMrgA13N, kMrgA12, 0}};
const Mat3 kA2 = {{0, 1, 0, 0, 0, 1, kMrgM2 - kMrgA23N, 0, kMrgA21}};

Mat3 mat_identity() { return Mat3{{1, 0, 0, 0, 1, 0, 0, 0, 1}}; }

// A^(2^i) cache for i < 128 (shared by skip_ahead and the launch tables).
struct PowCache {
    std::vector<Mat3> p1, p2;
    PowCache() {
        Mat3 a = kA1, b = kA2;
        for (int i = 0; i < 128; ++i) {
            p1.push_back(a);
            p2.push_back(b);
            a = mat_mul(a, a, kMrgM1);
            b = mat_mul(b, b, kMrgM2);
        }
    }
};
const PowCache& pow_cache() {
    static PowCache c;
    return c;
}

void mat_pow_u64(uint64_t k, Mat3* r1, Mat3* r2) {
    const PowCache& c = pow_cache();
    Mat3 a = mat_identity(), b = mat_identity();
    for (int i = 0; i < 64; ++i)
        if ((k >> i) & 1) {
            a = mat_mul(a, c.p1[i], kMrgM1);
            b = mat_mul(b, c.p2[i], kMrgM2);
        }
    *r1 = a;
    *r2 = b;
}

int check_mrg_state(const uint32_t* s1, const uint32_t* s2) {
    if (!s1 || !s2) return fail(PRNG_ERR_INVALID_PARAMETER, "MRG32k3a state must not be NULL");
    for (int i = 0; i < 3; ++i)
        if (s1[i] >= kMrgM1 || s2[i] >= kMrgM2)
            return fail(PRNG_ERR_INVALID_PARAMETER, "MRG32k3a state components must be below their modulus");
    if ((s1[0] | s1[1] | s1[2]) == 0 || (s2[0] | s2[1] | s2[2]) == 0)
        return fail(PRNG_ERR_INVALID_PARAMETER, "MRG32k3a state components must not be all zero");
    return PRNG_OK;
}

struct MrgTables {
    uint32_t nbits;
    uint32_t j1[kMrgMaxBits][9], j2[kMrgMaxBits][9];  // A^(seg * 2^b)
    MrgJump hs1, hs2;                                   // A^(32*chunk/chains), split
    MrgJump b1, b2;                                     // A^(31*seg), split
};
std::mutex g_mrg_mu;
std::map<std::tuple<uint64_t, uint64_t, uint32_t, uint64_t>, MrgTables> g_mrg_tables;

// B = hi*2^16 + lo with B's entries as symmetric residues mod m.
MrgJump split_jump(const Mat3& b, uint64_t m) {
    MrgJump j{};
    for (int e = 0; e < 9; ++e) {
        const int64_t v = b.v[e] > m / 2 ? (int64_t)b.v[e] - (int64_t)m : (int64_t)b.v[e];
        const int64_t hi = (v >= 0 ? v + 32768 : v - 32767) / 65536;  // round to nearest
        j.hi[e] = (double)hi;
        j.lo[e] = (double)(v - hi * 65536);
    }
    return j;
}

// Returned by value: another thread may evict the cache entry right after
// the lock is released.
MrgTables mrg_tables(uint64_t chunk, uint64_t seg, uint32_t nbits, uint64_t chains) {
    std::lock_guard<std::mutex> lk(g_mrg_mu);
    auto key = std::make_tuple(chunk, seg, nbits, chains);
    auto it = g_mrg_tables.find(key);
    if (it != g_mrg_tables.end()) return it->second;
    MrgTables t{};
    t.nbits = nbits;
    Mat3 a, b;
    mat_pow_u64(32 * chunk / chains, &a, &b);
    t.hs1 = split_jump(a, kMrgM1);
    t.hs2 = split_jump(b, kMrgM2);
    mat_pow_u64(31 * seg, &a, &b);
    t.b1 = split_jump(a, kMrgM1);
    t.b2 = split_jump(b, kMrgM2);
    mat_pow_u64(seg, &a, &b);
    for (uint32_t i = 0; i < nbits; ++i) {
        for (int e = 0; e < 9; ++e) {
            t.j1[i][e] = (uint32_t)a.v[e];
            t.j2[i][e] = (uint32_t)b.v[e];
        }
        a = mat_mul(a, a, kMrgM1);
        b = mat_mul(b, b, kMrgM2);
    }
    if (g_mrg_tables.size() > 256) g_mrg_tables.clear();
    return g_mrg_tables.emplace(key, t).first->second;
}

template <int X>
int launch_mrg(const uint32_t* s1, const uint32_t* s2, uint64_t n, void* out, const XformParams& p, void* stream) {
    using T = typename XformTraits<X>::T;
    constexpr uint64_t TW = MrgTile<T>::kWords;
    if (n == 0) return PRNG_OK;
    int rc = check_mrg_state(s1, s2);
    if (rc) return rc;
    if (out == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "out must not be NULL");
    if (((uintptr_t)out) % sizeof(T)) return fail(PRNG_ERR_INVALID_PARAMETER, "out is not aligned to its element");
    void* dptr = nullptr;
    rc = bind_output(out, &dptr);
    if (rc) return rc;
    const void* kern = (const void*)mrg_kernel<X>;
    int sms = 0, occ = 0;
    rc = resident_ctas(kern, kMrgThreads, &sms, &occ);
    if (rc) return rc;
    // A lane's share `chunk` is a whole number of segments per chain, so
    // every chain region is whole rounds (MrgPlan: segments of 4 tiles, or
    // one segment of chunk / kChains words).
    const uint64_t tmax = (uint64_t)sms * occ * kMrgThreads;
    uint64_t chunk = (n + tmax - 1) / tmax;
    constexpr uint64_t NC = MrgPlan<X>::kChains;
    const uint64_t unit = MrgPlan<X>::kSegmented ? NC * 4 * TW : NC * TW;
    chunk = (chunk + unit - 1) / unit * unit;
    const uint64_t seg = MrgPlan<X>::kSegmented ? 4 * TW : chunk / NC;
    const uint64_t tact = (n + chunk - 1) / chunk;
    const uint64_t qmax = ((tact - 1) / 32) * 32 * chunk / seg + 31;  // last lane's first segment
    uint32_t nbits = 0;
    while (nbits < 64 && (qmax >> nbits) != 0) ++nbits;
    if (nbits > (uint32_t)kMrgMaxBits) return fail(PRNG_ERR_INVALID_PARAMETER, "request too large");
    const MrgTables tb = mrg_tables(chunk, seg, nbits, NC);
    MrgLaunch a{};
    for (int i = 0; i < 3; ++i) {
        a.s1[i] = s1[i];
        a.s2[i] = s2[i];
    }
    a.n = n;
    a.chunk = chunk;
    a.seg = seg;
    a.nbits = nbits;
    memcpy(a.j1, tb.j1, sizeof a.j1);
    memcpy(a.j2, tb.j2, sizeof a.j2);
    a.hs1 = tb.hs1;
    a.hs2 = tb.hs2;
    a.b1 = tb.b1;
    a.b2 = tb.b2;
    a.out = dptr;
    a.p = p;
    const uint64_t blocks = (tact + kMrgThreads - 1) / kMrgThreads;
    void* args[] = {&a};
    PRNG_CUDA(cudaLaunchKernel(kern, dim3((unsigned)blocks), dim3(kMrgThreads), args, 0, (cudaStream_t)stream));
    return PRNG_OK;
}

// ---- write-ceiling probe (roofline denominator for write-only kernels) ----
// The same grid shape and store pattern as the aligned Philox 4-byte body
// (256-thread CTAs, every SM filled to the unit kernel's occupancy, thread
// u owning 64 contiguous bytes per grid-stride pass, two 256-bit streaming
// stores) with no generator work: what HBM takes for pure writes issued
// this way.
__global__ void __launch_bounds__(kPhiloxThreads) write_probe_kernel(uint32_t* out, uint64_t groups16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups16; g += stride) {
        const uint32_t v = (uint32_t)g;
        const uint32_t a[4] = {v, v + 1, v + 2, v + 3}, b[4] = {v + 4, v + 5, v + 6, v + 7};
        const uint32_t c[4] = {v + 8, v + 9, v + 10, v + 11}, d[4] = {v + 12, v + 13, v + 14, v + 15};
        st_group2(out + 16 * g, a, b);
        st_group2(out + 16 * g + 8, c, d);
    }
}

// ---- elementwise kernels ----
template <typename T>
__global__ void range_kernel(T* v, uint64_t n, T scale, T off) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if constexpr (sizeof(T) == 4)
            v[i] = __fadd_rn(__fmul_rn(v[i], scale), off);
        else
            v[i] = __dadd_rn(__dmul_rn(v[i], scale), off);
    }
}

__global__ void box_muller_kernel(const double* u1, const double* u2, uint64_t m, double* z0, double* z1,
                                  XformParams p) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        // _core.pyx:116-121 (u1 pre-flipped by the caller).  Inputs on the
        // reference's 24-bit grid (every call the reference makes: u1' =
        // m 2^-24, u2 = k 2^-24) take the exact route -- bit-identical to
        // _core -- anything else the libdevice formula.
        const double a = u1[i], b = u2[i];
        const double ma = __dmul_rn(a, 16777216.0), kb = __dmul_rn(b, 16777216.0);
        if (p.exact.log_nib && ma >= 1.0 && ma <= 16777216.0 && kb >= 0.0 && kb < 16777216.0 && ma == rint(ma) &&
            kb == rint(kb)) {
            const uint32_t w0 = (16777216u - (uint32_t)ma) << 8, w1 = (uint32_t)kb << 8;
            box_muller_exact(w0, w1, p, z0[i], z1[i]);
            continue;
        }
        const double r = sqrt(__dmul_rn(-2.0, log(a)));
        const double t = __dmul_rn(kTwoPi, b);
        double s, c;
        sincos(t, &s, &c);
        z0[i] = __dmul_rn(r, c);
        z1[i] = __dmul_rn(r, s);
    }
}

template <int X>
__global__ void words_kernel(const uint32_t* __restrict__ w, uint64_t n, XformParams p,
                             typename XformTraits<X>::T* __restrict__ out) {
    xform_prologue<X>(p);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;; i += stride) {
        if constexpr (XformTraits<X>::kPair) {
            if (2 * i >= n) break;
            typename XformTraits<X>::T o0, o1;
            xform2k<X>(w[2 * i], w[2 * i + 1], p, o0, o1);
            out[2 * i] = o0;
            if (2 * i + 1 < n) out[2 * i + 1] = o1;
        } else {
            if (i >= n) break;
            out[i] = xform1<X>(w[i], p);
        }
    }
}

template <int X>
int launch_words(const uint32_t* w, uint64_t n, const XformParams& p, void* out, void* stream) {
    using T = typename XformTraits<X>::T;
    if (n == 0) return PRNG_OK;
    if (!w || !out) return fail(PRNG_ERR_INVALID_PARAMETER, "NULL array");
    if (((uintptr_t)out) % sizeof(T)) return fail(PRNG_ERR_INVALID_PARAMETER, "out is not aligned to its element");
    void* d = nullptr;
    int rc = bind_output(out, &d);
    if (rc) return rc;
    int sms = 0;
    if ((rc = device_sms(&sms))) return rc;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
    words_kernel<X><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(w, n, p, (T*)d);
    PRNG_CUDA(cudaGetLastError());
    return PRNG_OK;
}

template <typename T>
int launch_range(T* v, uint64_t n, double lo, double hi, void* stream) {
    int rc = check_uniform(lo, hi);
    if (rc) return rc;
    if (n == 0) return PRNG_OK;
    if (!v) return fail(PRNG_ERR_INVALID_PARAMETER, "values must not be NULL");
    void* d = nullptr;
    rc = bind_output(v, &d);
    if (rc) return rc;
    int sms = 0;
    if ((rc = device_sms(&sms))) return rc;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
    range_kernel<T><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((T*)d, n, (T)(hi - lo), (T)lo);
    PRNG_CUDA(cudaGetLastError());
    return PRNG_OK;
}

// ---- library-owned staging for the host-buffer drop-ins ----
// The plugin drop-ins (prng_kernels_*) hand back ordinary (pageable) host
// arrays like the reference's _core (_core.pyx:44, 81).  They run a
// double-buffered pipeline per device: chunk c is generated into device
// slot c&1 and copied to pinned slot c&1 on a private stream, while the
// host copies chunk c-1 from pinned memory into the caller's array on
// several threads -- PCIe, the kernel and the host copy overlap.
struct Staging {
    void* dev = nullptr;   // 2 slots of kHostChunk words
    void* host = nullptr;  // 2 pinned slots
    size_t slot_bytes = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};
};
std::mutex g_scratch_mu;
std::map<int, Staging> g_staging;

constexpr uint64_t kHostChunk = 1ull << 24;  // words per staged chunk (64 MB)

int staging(size_t slot_bytes, Staging** out) {
    int dev = 0;
    PRNG_CUDA(cudaGetDevice(&dev));
    Staging& sg = g_staging[dev];
    if (!sg.stream) {
        PRNG_CUDA(cudaStreamCreateWithFlags(&sg.stream, cudaStreamNonBlocking));
        for (auto& e : sg.done) PRNG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (sg.slot_bytes < slot_bytes) {
        if (sg.dev) PRNG_CUDA(cudaFree(sg.dev));
        if (sg.host) PRNG_CUDA(cudaFreeHost(sg.host));
        sg.dev = sg.host = nullptr;
        sg.slot_bytes = 0;
        PRNG_CUDA(cudaMalloc(&sg.dev, 2 * slot_bytes));
        PRNG_CUDA(cudaHostAlloc(&sg.host, 2 * slot_bytes, cudaHostAllocDefault));
        sg.slot_bytes = slot_bytes;
    }
    *out = &sg;
    return PRNG_OK;
}

// memcpy on up to 8 host threads (one pageable destination, pinned source).
void host_copy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kMinPart = size_t(4) << 20;
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt < 1 ? 1 : (nt > 8 ? 8 : nt);
    if (bytes / kMinPart < nt) nt = (unsigned)(bytes / kMinPart) > 0 ? (unsigned)(bytes / kMinPart) : 1;
    if (nt == 1) {
        memcpy(dst, src, bytes);
        return;
    }
    const size_t part = (bytes / nt + 63) / 64 * 64;
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) {
        const size_t off = part * t;
        if (off >= bytes) break;
        const size_t len = bytes - off < part ? bytes - off : part;
        th.emplace_back([=] { memcpy((char*)dst + off, (const char*)src + off, len); });
    }
    memcpy(dst, src, part < bytes ? part : bytes);
    for (auto& x : th) x.join();
}

// Runs `gen(done, m, dev_slot, stream)` for consecutive chunks of `n`
// elements of `esize` bytes and lands them in host_out.
template <typename Gen>
int host_pipeline(uint64_t n, size_t esize, void* host_out, Gen&& gen) {
    if (n == 0) return PRNG_OK;
    const uint64_t chunk = n < kHostChunk ? n : kHostChunk;
    Staging* sg = nullptr;
    int rc = staging(chunk * esize, &sg);
    if (rc) return rc;
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    auto land = [&](uint64_t c) -> int {
        const uint64_t m = (c + 1) * chunk <= n ? chunk : n - c * chunk;
        PRNG_CUDA(cudaEventSynchronize(sg->done[c & 1]));
        host_copy((char*)host_out + c * chunk * esize, (char*)sg->host + (c & 1) * sg->slot_bytes, m * esize);
        return PRNG_OK;
    };
    for (uint64_t c = 0; c < nchunks; ++c) {
        const uint64_t m = (c + 1) * chunk <= n ? chunk : n - c * chunk;
        void* d = (char*)sg->dev + (c & 1) * sg->slot_bytes;
        if ((rc = gen(c * chunk, m, d, sg->stream))) return rc;
        PRNG_CUDA(cudaMemcpyAsync((char*)sg->host + (c & 1) * sg->slot_bytes, d, m * esize, cudaMemcpyDeviceToHost,
                                  sg->stream));
        PRNG_CUDA(cudaEventRecord(sg->done[c & 1], sg->stream));
        if (c > 0 && (rc = land(c - 1))) return rc;
    }
    return land(nchunks - 1);
}

}  // namespace

// =====================================================================
extern "C" {

int prng_abi_version(void) { return PRNG_ABI_VERSION; }
const char* prng_last_error(void) { return g_err; }

#define PHILOX_ARGS uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n

int prng_philox4x32x10_bits(PHILOX_ARGS, uint32_t* out, void* stream) {
    DeviceGuard guard_;
    return launch_philox<kBits>(k0, k1, ctr, lane, n, out, XformParams{}, stream);
}

int prng_philox4x32x10_uniform_f32(PHILOX_ARGS, double a, double b, float* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_uniform(a, b);
    if (rc) return rc;
    const UniformSpec u = uniform_spec_f32(a, b);
    if (u.plan == kPlanFolded) return launch_philox<kUniformF32>(k0, k1, ctr, lane, n, out, u.p, stream);
    rc = launch_philox<kUnitF32>(k0, k1, ctr, lane, n, out, u.p, stream);
    return (rc || u.plan == kPlanIdentity) ? rc : launch_range<float>(out, n, a, b, stream);
}

int prng_philox4x32x10_uniform_f64(PHILOX_ARGS, double a, double b, double* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_uniform(a, b);
    if (rc) return rc;
    const UniformSpec u = uniform_spec_f64(a, b);
    if (u.plan == kPlanFolded) return launch_philox<kUniformF64>(k0, k1, ctr, lane, n, out, u.p, stream);
    rc = launch_philox<kUnitF64>(k0, k1, ctr, lane, n, out, u.p, stream);
    return (rc || u.plan == kPlanIdentity) ? rc : launch_range<double>(out, n, a, b, stream);
}

int prng_philox4x32x10_gaussian_f32(PHILOX_ARGS, double mean, double stddev, int method, float* out,
                                    void* stream) {
    DeviceGuard guard_;
    int rc = check_gaussian(mean, stddev);
    if (!rc) rc = check_gauss_method(method);
    if (rc) return rc;
    XformParams p = gauss_params(mean, stddev);
    if (method == PRNG_METHOD_EXACT) {
        if (n == 0) return PRNG_OK;
        void* d = nullptr;
        if (out == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "out must not be NULL");
        if ((rc = bind_output(out, &d)) || (rc = exact_tables(p))) return rc;
        return launch_philox<kGaussF32Exact>(k0, k1, ctr, lane, n, out, p, stream);
    }
    if (method == PRNG_METHOD_PRECISE) return launch_philox<kGaussF32Precise>(k0, k1, ctr, lane, n, out, p, stream);
    return method == PRNG_METHOD_FAST ? launch_philox<kGaussF32Fast>(k0, k1, ctr, lane, n, out, p, stream)
                                      : launch_philox<kGaussF32Accurate>(k0, k1, ctr, lane, n, out, p, stream);
}

int prng_philox4x32x10_gaussian_f64(PHILOX_ARGS, double mean, double stddev, double* out, void* stream) {
    DeviceGuard guard_;
    return prng_philox4x32x10_gaussian_f64_method(k0, k1, ctr, lane, n, mean, stddev, PRNG_METHOD_ACCURATE, out,
                                                  stream);
}

int prng_philox4x32x10_gaussian_f64_method(PHILOX_ARGS, double mean, double stddev, int method, double* out,
                                           void* stream) {
    DeviceGuard guard_;
    int rc = check_gaussian(mean, stddev);
    if (!rc) rc = check_gauss_method(method);
    if (rc) return rc;
    XformParams p = gauss_params(mean, stddev);
    if (method == PRNG_METHOD_EXACT) {
        if (n == 0) return PRNG_OK;
        void* d = nullptr;
        if (out == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "out must not be NULL");
        if ((rc = bind_output(out, &d)) || (rc = exact_tables(p))) return rc;
        return launch_philox<kGaussF64Exact>(k0, k1, ctr, lane, n, out, p, stream);
    }
    return launch_philox<kGaussF64>(k0, k1, ctr, lane, n, out, p, stream);  // FAST == ACCURATE for fp64
}

int prng_philox4x32x10_lognormal_f32(PHILOX_ARGS, double m, double s, double displ, double scale, int method,
                                     float* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_lognormal(m, s, displ, scale);
    if (!rc) rc = check_method(method);
    if (rc) return rc;
    const XformParams p = logn_params(m, s, displ, scale);
    if (!logn_fast_ok(m, s)) method = PRNG_METHOD_ACCURATE;
    if (method == PRNG_METHOD_PRECISE) return launch_philox<kLognF32Precise>(k0, k1, ctr, lane, n, out, p, stream);
    if (method == PRNG_METHOD_FAST && p.ln_scale_f == 1.0f && p.ln_displ_f == 0.0f)  // oneMKL's default form
        return launch_philox<kLognF32FastUnit>(k0, k1, ctr, lane, n, out, p, stream);
    return method == PRNG_METHOD_FAST ? launch_philox<kLognF32Fast>(k0, k1, ctr, lane, n, out, p, stream)
                                      : launch_philox<kLognF32Accurate>(k0, k1, ctr, lane, n, out, p, stream);
}

int prng_philox4x32x10_lognormal_f64(PHILOX_ARGS, double m, double s, double displ, double scale, double* out,
                                     void* stream) {
    DeviceGuard guard_;
    int rc = check_lognormal(m, s, displ, scale);
    return rc ? rc
              : launch_philox<kLognF64>(k0, k1, ctr, lane, n, out, logn_params(m, s, displ, scale), stream);
}

#define MRG_ARGS const uint32_t s1[3], const uint32_t s2[3], uint64_t n

int prng_mrg32k3a_bits(MRG_ARGS, uint32_t* out, void* stream) {
    DeviceGuard guard_;
    return launch_mrg<kBits>(s1, s2, n, out, XformParams{}, stream);
}

int prng_mrg32k3a_uniform_f32(MRG_ARGS, double a, double b, float* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_uniform(a, b);
    if (rc) return rc;
    const UniformSpec u = uniform_spec_f32(a, b);
    if (u.plan == kPlanFolded) return launch_mrg<kUniformF32>(s1, s2, n, out, u.p, stream);
    rc = launch_mrg<kUnitF32>(s1, s2, n, out, u.p, stream);
    return (rc || u.plan == kPlanIdentity) ? rc : launch_range<float>(out, n, a, b, stream);
}

int prng_mrg32k3a_uniform_f64(MRG_ARGS, double a, double b, double* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_uniform(a, b);
    if (rc) return rc;
    const UniformSpec u = uniform_spec_f64(a, b);
    if (u.plan == kPlanFolded) return launch_mrg<kUniformF64>(s1, s2, n, out, u.p, stream);
    rc = launch_mrg<kUnitF64>(s1, s2, n, out, u.p, stream);
    return (rc || u.plan == kPlanIdentity) ? rc : launch_range<double>(out, n, a, b, stream);
}

int prng_mrg32k3a_gaussian_f32(MRG_ARGS, double mean, double stddev, int method, float* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_gaussian(mean, stddev);
    if (!rc) rc = check_gauss_method(method);
    if (rc) return rc;
    XformParams p = gauss_params(mean, stddev);
    if (method == PRNG_METHOD_EXACT) {
        if (n == 0) return PRNG_OK;
        void* d = nullptr;
        if (out == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "out must not be NULL");
        if ((rc = bind_output(out, &d)) || (rc = exact_tables(p))) return rc;
        return launch_mrg<kGaussF32Exact>(s1, s2, n, out, p, stream);
    }
    return method == PRNG_METHOD_FAST ? launch_mrg<kGaussF32Fast>(s1, s2, n, out, p, stream)
                                      : launch_mrg<kGaussF32Accurate>(s1, s2, n, out, p, stream);
}

int prng_mrg32k3a_gaussian_f64(MRG_ARGS, double mean, double stddev, double* out, void* stream) {
    DeviceGuard guard_;
    return prng_mrg32k3a_gaussian_f64_method(s1, s2, n, mean, stddev, PRNG_METHOD_ACCURATE, out, stream);
}

int prng_mrg32k3a_gaussian_f64_method(MRG_ARGS, double mean, double stddev, int method, double* out,
                                      void* stream) {
    DeviceGuard guard_;
    int rc = check_gaussian(mean, stddev);
    if (!rc) rc = check_gauss_method(method);
    if (rc) return rc;
    XformParams p = gauss_params(mean, stddev);
    if (method == PRNG_METHOD_EXACT) {
        if (n == 0) return PRNG_OK;
        void* d = nullptr;
        if (out == nullptr) return fail(PRNG_ERR_INVALID_PARAMETER, "out must not be NULL");
        if ((rc = bind_output(out, &d)) || (rc = exact_tables(p))) return rc;
        return launch_mrg<kGaussF64Exact>(s1, s2, n, out, p, stream);
    }
    return launch_mrg<kGaussF64>(s1, s2, n, out, p, stream);
}

int prng_mrg32k3a_lognormal_f32(MRG_ARGS, double m, double s, double displ, double scale, int method, float* out,
                                void* stream) {
    DeviceGuard guard_;
    int rc = check_lognormal(m, s, displ, scale);
    if (!rc) rc = check_method(method);
    if (rc) return rc;
    const XformParams p = logn_params(m, s, displ, scale);
    if (!logn_fast_ok(m, s)) method = PRNG_METHOD_ACCURATE;
    return method == PRNG_METHOD_FAST ? launch_mrg<kLognF32Fast>(s1, s2, n, out, p, stream)
                                      : launch_mrg<kLognF32Accurate>(s1, s2, n, out, p, stream);
}

int prng_mrg32k3a_lognormal_f64(MRG_ARGS, double m, double s, double displ, double scale, double* out,
                                void* stream) {
    DeviceGuard guard_;
    int rc = check_lognormal(m, s, displ, scale);
    return rc ? rc : launch_mrg<kLognF64>(s1, s2, n, out, logn_params(m, s, displ, scale), stream);
}

int prng_mrg32k3a_skip_ahead(const uint32_t s1[3], const uint32_t s2[3], uint64_t k_lo, uint64_t k_hi,
                             uint32_t s1_out[3], uint32_t s2_out[3]) {
    int rc = check_mrg_state(s1, s2);
    if (rc) return rc;
    if (!s1_out || !s2_out) return fail(PRNG_ERR_INVALID_PARAMETER, "output state must not be NULL");
    uint32_t x1[3] = {s1[0], s1[1], s1[2]}, x2[3] = {s2[0], s2[1], s2[2]};
    const PowCache& c = pow_cache();
    for (int w = 0; w < 2; ++w) {
        const uint64_t k = w ? k_hi : k_lo;
        for (int i = 0; i < 64; ++i)
            if ((k >> i) & 1) {
                mat_vec(c.p1[64 * w + i], x1, kMrgM1);
                mat_vec(c.p2[64 * w + i], x2, kMrgM2);
            }
    }
    for (int i = 0; i < 3; ++i) {
        s1_out[i] = x1[i];
        s2_out[i] = x2[i];
    }
    return PRNG_OK;
}

int prng_words_to_unit_f32(const uint32_t* words, uint64_t n, float* out, void* stream) {
    DeviceGuard guard_;
    return launch_words<kUnitF32>(words, n, XformParams{}, out, stream);
}

int prng_words_to_unit_f64(const uint32_t* words, uint64_t n, double* out, void* stream) {
    DeviceGuard guard_;
    return launch_words<kUnitF64>(words, n, XformParams{}, out, stream);
}

int prng_gaussian_from_words_f32(const uint32_t* words, uint64_t n, double mean, double stddev, int method,
                                 float* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_gaussian(mean, stddev);
    if (!rc) rc = check_gauss_method(method);
    if (rc) return rc;
    XformParams p = gauss_params(mean, stddev);
    if (method == PRNG_METHOD_EXACT) {
        if (n == 0) return PRNG_OK;
        if ((rc = exact_tables(p))) return rc;
        return launch_words<kGaussF32Exact>(words, n, p, out, stream);
    }
    if (method == PRNG_METHOD_PRECISE) return launch_words<kGaussF32Precise>(words, n, p, out, stream);
    return method == PRNG_METHOD_FAST ? launch_words<kGaussF32Fast>(words, n, p, out, stream)
                                      : launch_words<kGaussF32Accurate>(words, n, p, out, stream);
}

int prng_gaussian_from_words_f64(const uint32_t* words, uint64_t n, double mean, double stddev, double* out,
                                 void* stream) {
    DeviceGuard guard_;
    return prng_gaussian_from_words_f64_method(words, n, mean, stddev, PRNG_METHOD_ACCURATE, out, stream);
}

int prng_gaussian_from_words_f64_method(const uint32_t* words, uint64_t n, double mean, double stddev, int method,
                                        double* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_gaussian(mean, stddev);
    if (!rc) rc = check_gauss_method(method);
    if (rc) return rc;
    XformParams p = gauss_params(mean, stddev);
    if (method == PRNG_METHOD_EXACT) {
        if (n == 0) return PRNG_OK;
        if ((rc = exact_tables(p))) return rc;
        return launch_words<kGaussF64Exact>(words, n, p, out, stream);
    }
    return launch_words<kGaussF64>(words, n, p, out, stream);
}

int prng_exact_tables_prepare(void) {
    DeviceGuard guard_;
    XformParams p{};
    return exact_tables(p);
}

int prng_exact_tables_bounds(double bounds[2], uint64_t* escapes) {
    DeviceGuard guard_;
    if (!bounds || !escapes) return fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    XformParams p{};
    int rc = exact_tables(p);
    if (rc) return rc;
    bounds[0] = p.exact.rel_log;
    bounds[1] = p.exact.abs_sc;
    *escapes = (uint64_t)p.exact.esc_n[0] + p.exact.esc_n[1] + p.exact.esc_n[2];
    return PRNG_OK;
}

int prng_exact_tables_host(const double** log_table, const double** sincos_table) {
    if (!log_table || !sincos_table) return fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    std::lock_guard<std::mutex> lk(g_exact_mu);
    g_exact_keep_host = true;  // the caller holds the pointers for the life of the process
    if (g_exact_log.empty()) build_exact_host_tables();
    *log_table = g_exact_log.data();
    *sincos_table = reinterpret_cast<const double*>(g_exact_sc.data());
    return PRNG_OK;
}

int prng_range_transform_f32(float* values, uint64_t n, double lo, double hi, void* stream) {
    DeviceGuard guard_;
    return launch_range<float>(values, n, lo, hi, stream);
}

int prng_range_transform_f64(double* values, uint64_t n, double lo, double hi, void* stream) {
    DeviceGuard guard_;
    return launch_range<double>(values, n, lo, hi, stream);
}

int prng_philox4x32x10_uniform_f32_segments(uint32_t k0, uint32_t k1, const prng_segment_t* segs, uint32_t nseg,
                                            uint64_t max_count, double a, double b, float* out, void* stream) {
    DeviceGuard guard_;
    int rc = check_uniform(a, b);
    if (rc) return rc;
    if (nseg == 0 || max_count == 0) return PRNG_OK;
    if (!segs || !out) return fail(PRNG_ERR_INVALID_PARAMETER, "segs and out must not be NULL");
    if (((uintptr_t)out) % 4) return fail(PRNG_ERR_INVALID_PARAMETER, "out is not aligned to its element");
    void* dptr = nullptr;
    rc = bind_output(out, &dptr);
    if (rc) return rc;
    const void* kern = (const void*)philox_segments_kernel<kUniformF32>;
    int sms = 0, occ = 0;
    rc = resident_ctas(kern, kPhiloxThreads, &sms, &occ);
    if (rc) return rc;
    // blocks per segment: enough threads for 8 elements each, but keep the
    // whole grid within ~4 waves of resident CTAs.
    uint64_t bx = (max_count / 8 + kPhiloxThreads) / kPhiloxThreads;
    if (bx < 1) bx = 1;
    const uint64_t cap = (uint64_t)sms * occ * 4;
    uint64_t by = nseg < 65535u ? nseg : 65535u;
    if (bx * by > cap) bx = (cap + by - 1) / by;
    if (bx < 1) bx = 1;
    const UniformSpec u = uniform_spec_f32(a, b);
    if (u.plan == kPlanTwoPass) return fail(PRNG_ERR_INVALID_RANGE, "segment range too narrow for fp32");
    const XformParams p = u.p;
    philox_segments_kernel<kUniformF32><<<dim3((unsigned)bx, (unsigned)by), kPhiloxThreads, 0, (cudaStream_t)stream>>>(
        k0, k1, reinterpret_cast<const PhiloxSegment*>(segs), nseg, p, (float*)dptr);
    PRNG_CUDA(cudaGetLastError());
    return PRNG_OK;
}

#ifdef PRNG_TRACE_CTA
int prng_diag_cta_trace(unsigned long long* host, int n) {  // diagnostics build only
    return cudaMemcpyFromSymbol(host, prng::g_cta_trace, sizeof(unsigned long long) * 3 * (size_t)n) == cudaSuccess
               ? PRNG_OK
               : PRNG_ERR_CUDA;
}
#endif

int prng_diag_write_probe(void* out, uint64_t bytes, void* stream) {
    DeviceGuard guard_;
    if (!out || ((uintptr_t)out & 31u) || (bytes & 63u))
        return fail(PRNG_ERR_INVALID_PARAMETER, "write probe needs a 32-byte aligned buffer of 64-byte multiples");
    void* d = nullptr;
    int rc = bind_output(out, &d);
    if (rc) return rc;
    int sms = 0, occ = 0;
    if ((rc = resident_ctas((const void*)philox_kernel<kUnitF32, 0>, kPhiloxThreads, &sms, &occ))) return rc;
    const uint64_t groups = bytes / 64;
    uint64_t blocks = (groups + kPhiloxThreads - 1) / kPhiloxThreads;
    if (blocks > (uint64_t)sms * occ) blocks = (uint64_t)sms * occ;
    if (blocks < 1) blocks = 1;
    write_probe_kernel<<<(unsigned)blocks, kPhiloxThreads, 0, (cudaStream_t)stream>>>((uint32_t*)d, groups);
    PRNG_CUDA(cudaGetLastError());
    return PRNG_OK;
}

int prng_kernels_philox_fill(uint32_t k0, uint32_t k1, uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3,
                             uint32_t offset, uint64_t n, uint32_t* host_out) {
    DeviceGuard guard_;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    if (n == 0) return PRNG_OK;
    if (!host_out) return fail(PRNG_ERR_INVALID_PARAMETER, "host_out must not be NULL");
    // _core.pyx:49-62: `lane = offset`; a lane >= 4 emits nothing from the
    // first block, then the counter steps and lane restarts at 0 -- so any
    // offset >= 4 streams from block b + 1, word 0.
    u128 base_blk = ((u128)b3 << 96) | ((u128)b2 << 64) | ((u128)b1 << 32) | b0;
    if (offset > 3) {
        base_blk += 1;
        offset = 0;
    }
    // Each chunk restarts from its own stream offset exactly as the
    // reference's chunk kernels do (rngburn.py:70-73); the block counter
    // wraps mod 2^128 like _core.pyx:63-70.
    return host_pipeline(n, 4, host_out, [&](uint64_t done, uint64_t m, void* d, cudaStream_t s) {
        const uint64_t rel = (uint64_t)offset + done;
        const u128 blk = base_blk + (rel >> 2);
        const uint32_t ctr[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)(blk >> 64), (uint32_t)(blk >> 96)};
        return launch_philox<kBits>(k0, k1, ctr, (uint32_t)(rel & 3), m, d, XformParams{}, s);
    });
}

int prng_kernels_mrg_fill(uint32_t s10, uint32_t s11, uint32_t s12, uint32_t s20, uint32_t s21, uint32_t s22,
                          uint64_t n, uint32_t* host_out, uint32_t s1_out[3], uint32_t s2_out[3]) {
    DeviceGuard guard_;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    uint32_t s1[3] = {s10, s11, s12}, s2[3] = {s20, s21, s22};
    int rc = check_mrg_state(s1, s2);
    if (rc) return rc;
    if (n && !host_out) return fail(PRNG_ERR_INVALID_PARAMETER, "host_out must not be NULL");
    uint32_t c1[3] = {s10, s11, s12}, c2[3] = {s20, s21, s22};
    rc = host_pipeline(n, 4, host_out, [&](uint64_t, uint64_t m, void* d, cudaStream_t s) {
        int r = launch_mrg<kBits>(c1, c2, m, d, XformParams{}, s);
        return r ? r : prng_mrg32k3a_skip_ahead(c1, c2, m, 0, c1, c2);
    });
    if (rc) return rc;
    if (s1_out && s2_out)
        for (int i = 0; i < 3; ++i) {
            s1_out[i] = c1[i];
            s2_out[i] = c2[i];
        }
    return PRNG_OK;
}

int prng_kernels_box_muller(const double* u1, const double* u2, uint64_t m, double* z0, double* z1) {
    DeviceGuard guard_;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    if (m == 0) return PRNG_OK;
    if (!u1 || !u2 || !z0 || !z1) return fail(PRNG_ERR_INVALID_PARAMETER, "NULL array");
    Staging* sg = nullptr;
    int rc = staging(m * 16, &sg);  // two slots: (u1, u2) and (z0, z1)
    if (rc) return rc;
    cudaStream_t s = sg->stream;
    double* du1 = (double*)sg->dev;
    double* du2 = du1 + m;
    double* dz0 = du2 + m;
    double* dz1 = dz0 + m;
    PRNG_CUDA(cudaMemcpyAsync(du1, u1, m * 8, cudaMemcpyHostToDevice, s));
    PRNG_CUDA(cudaMemcpyAsync(du2, u2, m * 8, cudaMemcpyHostToDevice, s));
    int sms = 0;
    if ((rc = device_sms(&sms))) return rc;
    uint64_t blocks = (m + 255) / 256;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    XformParams p{};
    if ((rc = exact_tables(p))) return rc;
    box_muller_kernel<<<(unsigned)blocks, 256, 0, s>>>(du1, du2, m, dz0, dz1, p);
    PRNG_CUDA(cudaGetLastError());
    PRNG_CUDA(cudaMemcpyAsync(z0, dz0, m * 8, cudaMemcpyDeviceToHost, s));
    PRNG_CUDA(cudaMemcpyAsync(z1, dz1, m * 8, cudaMemcpyDeviceToHost, s));
    PRNG_CUDA(cudaStreamSynchronize(s));
    return PRNG_OK;
}

}  // extern "C"
