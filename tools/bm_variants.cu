// bm_variants.cu -- fast fp32 Box-Muller design study (sm_100a): throughput
// at n = 2^30 and exhaustive accuracy in fp32 ulps, per variant.
//
// Variants (template parameters):
//   LOGM 0 = library route (lg2.approx + near-1 series, select)
//        1 = table-driven log over the bits of 1 - u1 (64 buckets per binade,
//            r = 1 - omx * inv_j >= 0, 4-term series): relative accuracy
//            everywhere, no MUFU.LG2
//   TL   0 = library sin/cos (4096-entry table, uncentred, sin x = x, cos x = 1)
//        12/13 = centred table (index rounded to the nearest table angle, the
//            quadrant points are table points), x = (f - c) * 2 pi 2^-9
//   QUAD 1 = keep the cos x = 1 - x^2/2 term
//   LOOP 0 = pipelined with register copies (library), 1 = pipelined, unrolled
//            by two (ping-pong), 2 = not pipelined
// Accuracy: for every k in [0, 2^24): u1 = k (u2 hashed) and u2 = k (u1
// hashed), against the fp64 formula sqrt(-2 log(1 - u1)) * cos/sin(fl(2 pi u2))
// (libdevice; ~1e-16 relative), max error in fp32 ulps of the reference value
// per |z| band, and max |err| / max(1, |z|) in units of 2^-20.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2109_01329_b200/csrc \
//        -o bm_variants bm_variants.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

using namespace prng;

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

constexpr int kLogIdx0 = 103 << 6;           // bits(2^-24) >> 17
constexpr int kLogEntries = (127 << 6) - kLogIdx0 + 1;  // ... bits(1.0) >> 17
constexpr float kLc1 = 1.4426950408889634f, kLc2 = 0.7213475204444817f, kLc3 = 0.48089834696298783f,
                kLc4 = 0.36067376022224085f;

struct GParams {
    uint32_t k0, k1;
    PhiloxPre pre;
    uint32_t ngroups;
    float* out;
    float S, off;
};

template <int TL>
__device__ __forceinline__ float2* dyn_sincos() {
    extern __shared__ float2 dsm[];
    return dsm;
}
template <int TL>
__device__ __forceinline__ float2* dyn_log() {
    extern __shared__ float2 dsm[];
    return dsm + (TL ? (1 << TL) + 1 : 0);
}

__device__ __align__(16) float2 g_tabs[(1 << 13) + 1 + 2048];  // sincos (2^TL + 1) then log (kLogEntries)

template <int LOGM, int TL>
__global__ void kfill(float S);

// LOOP 3 (non-persistent CTAs): copy the tables from global (L2-resident,
// filled once by kfill) instead of recomputing them per CTA.
template <int LOGM, int TL>
__device__ void prologue_copy() {
    extern __shared__ float4 dsm4[];
    constexpr int n2 = (TL ? (1 << TL) + 1 : 0) + (LOGM ? kLogEntries : 0);  // float2 entries
    const float4* src = reinterpret_cast<const float4*>(g_tabs);
    for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) dsm4[i] = src[i];
    if ((n2 & 1) && threadIdx.x == 0) reinterpret_cast<float2*>(dsm4)[n2 - 1] = g_tabs[n2 - 1];
    __syncthreads();
}

template <int LOGM, int TL>
__device__ void prologue(float S) {
    if constexpr (TL == 0) {
        float2* tab = sincos_tab<12>();
        for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
            float sn, cs;
            sincospif((float)i * (2.0f / 4096), &sn, &cs);
            tab[i] = make_float2(sn * S, cs * S);
        }
    } else {
        float2* tab = dyn_sincos<TL>();
        for (int i = threadIdx.x; i <= (1 << TL); i += blockDim.x) {
            // the reference's argument fl64(TWO_PI * u2) at the table angle
            // (quadrant points keep cos(fl(pi/2)) = 6.1e-17 etc.)
            double sn, cs;
            sincos(__dmul_rn(6.283185307179586, (double)i / (double)(1 << TL)), &sn, &cs);
            tab[i] = make_float2((float)(sn * (double)S), (float)(cs * (double)S));
        }
    }
    if constexpr (LOGM == 1) {
        float2* lt = dyn_log<TL>();
        for (int i = threadIdx.x; i < kLogEntries; i += blockDim.x) {
            const uint32_t idx = kLogIdx0 + i;
            const double hi = (double)__uint_as_float((idx + 1) << 17);  // bucket end (exclusive)
            float inv = idx == (127u << 6) ? 1.0f : __double2float_rd(1.0 / hi);
            if (inv < 1.0f) inv = 1.0f;
            lt[i] = make_float2(inv, (float)log2((double)inv));
        }
    }
    __syncthreads();
}

template <int LOGM, int TL>
__global__ void kfill(float S) {
    // one CTA: run the per-CTA prologue, then write the smem tables to global
    prologue<LOGM, TL>(S);
    extern __shared__ float2 dsm[];
    constexpr int n2 = (TL ? (1 << TL) + 1 : 0) + (LOGM ? kLogEntries : 0);
    for (int i = threadIdx.x; i < n2; i += blockDim.x) g_tabs[i] = dsm[i];
}

template <int LOGM, int TL>
__device__ __forceinline__ float neg_lg2_v(uint32_t w0) {
    if constexpr (LOGM == 0) {
        return neg_lg2_1mu(w0);
    } else {
        const float kf = __uint2float_rn(w0 >> 8);
        const float omx = fmaf(kf, -5.9604644775390625e-08f, 1.0f);  // exact
        const float2 e = dyn_log<TL>()[(__float_as_uint(omx) >> 17) - kLogIdx0];
        const float r = fmaf(-omx, e.x, 1.0f);  // >= 0, <= 2^-6
        float p = fmaf(r, kLc4, kLc3);
        p = fmaf(p, r, kLc2);
        p = fmaf(p, r, kLc1);
        return fmaf(r, p, e.y);
    }
}

template <int TL, int QUAD>
__device__ __forceinline__ void sincos_v(uint32_t w1, float& sn, float& cs) {
    if constexpr (TL == 0) {
        sincos_2pi_k24<12>(w1, sn, cs);
    } else {
        constexpr int L = 24 - TL;
        const uint32_t wc = w1 + (1u << (31 - TL));
        const float2 t = dyn_sincos<TL>()[wc >> (32 - TL)];
        uint32_t fb;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(fb) : "r"(wc), "n"(((1u << L) - 1u) << 8), "r"(0x3F800000u));
        constexpr float C = 1.0f + (float)(1u << (L - 1)) * 3.0517578125e-05f;  // 1 + 2^(L-1) 2^-15
        const float d = __fsub_rn(__uint_as_float(fb), C);                      // exact, signed offset
        const float x = __fmul_rn(d, 0.01227184630308513f);                      // 2 pi 2^-9
        if constexpr (QUAD) {
            const float nh = __fmul_rn(x, __fmul_rn(x, -0.5f));
            sn = fmaf(t.y, x, fmaf(t.x, nh, t.x));
            cs = fmaf(-t.x, x, fmaf(t.y, nh, t.y));
        } else {
            sn = fmaf(t.y, x, t.x);
            cs = fmaf(-t.x, x, t.y);
        }
    }
}

template <int LOGM, int TL, int QUAD>
__device__ __forceinline__ void bm(uint32_t w0, uint32_t w1, float off, float& o0, float& o1) {
    const float s = neg_lg2_v<LOGM, TL>(w0);
    float rq;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"(s));
    float sn, cs;
    sincos_v<TL, QUAD>(w1, sn, cs);
    o0 = fmaf(rq, cs, off);
    o1 = fmaf(rq, sn, off);
}

template <int LOGM, int TL, int QUAD>
__device__ __forceinline__ void bm4(const U4& w, float off, float o[4]) {
    bm<LOGM, TL, QUAD>(w.x, w.y, off, o[0], o[1]);
    bm<LOGM, TL, QUAD>(w.z, w.w, off, o[2], o[3]);
}

template <int LOGM, int TL, int QUAD, int LOOP, int MINB, int THREADS>
__global__ void __launch_bounds__(THREADS, MINB) kgauss(const GParams a) {
    if constexpr (LOOP >= 3) {
        static_assert(TL != 0, "non-persistent variants use the dynamic tables");
        prologue_copy<LOGM, TL>();
        constexpr int BPT = 4, ITER = LOOP - 2;  // LOOP 3.. : ITER = 1..
        const uint32_t g0c = blockIdx.x * (THREADS * BPT * ITER);
#pragma unroll 1
        for (int i = 0; i < ITER; ++i) {
            const uint32_t g0 = g0c + (i * THREADS + threadIdx.x) * BPT;
            if (g0 + BPT > a.ngroups) return;
            float o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) bm4<LOGM, TL, QUAD>(philox_block_pre(a.k0, a.k1, g0 + j, a.pre), a.off, o[j]);
#pragma unroll
            for (int j = 0; j < BPT; j += 2) st_group2(a.out + (size_t)4 * (g0 + j), o[j], o[j + 1]);
        }
        return;
    }
    prologue<LOGM, TL>(a.S);
    constexpr int BPT = 4;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    const uint32_t gstep = gstride * BPT;
    const uint32_t gfull = a.ngroups - a.ngroups % BPT;
    float* dst = a.out + (size_t)4 * BPT * gtid;
    const size_t dstep = (size_t)4 * gstep;
    if constexpr (LOOP == 0) {
        U4 w[BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) w[j] = philox_block_pre(a.k0, a.k1, gtid * BPT + j, a.pre);
        for (uint32_t g0 = gtid * BPT; g0 < gfull; g0 += gstep, dst += dstep) {
            U4 nw[BPT];
#pragma unroll
            for (int j = 0; j < BPT; ++j) nw[j] = philox_block_pre(a.k0, a.k1, g0 + gstep + j, a.pre);
            float o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) bm4<LOGM, TL, QUAD>(w[j], a.off, o[j]);
#pragma unroll
            for (int j = 0; j < BPT; j += 2) st_group2(dst + 4 * j, o[j], o[j + 1]);
#pragma unroll
            for (int j = 0; j < BPT; ++j) w[j] = nw[j];
        }
    } else if constexpr (LOOP == 1) {
        U4 wa[BPT], wb[BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) wa[j] = philox_block_pre(a.k0, a.k1, gtid * BPT + j, a.pre);
        uint32_t g0 = gtid * BPT;
        while (g0 < gfull) {
#pragma unroll
            for (int j = 0; j < BPT; ++j) wb[j] = philox_block_pre(a.k0, a.k1, g0 + gstep + j, a.pre);
            {
                float o[BPT][4];
#pragma unroll
                for (int j = 0; j < BPT; ++j) bm4<LOGM, TL, QUAD>(wa[j], a.off, o[j]);
#pragma unroll
                for (int j = 0; j < BPT; j += 2) st_group2(dst + 4 * j, o[j], o[j + 1]);
            }
            g0 += gstep;
            dst += dstep;
            if (g0 >= gfull) break;
#pragma unroll
            for (int j = 0; j < BPT; ++j) wa[j] = philox_block_pre(a.k0, a.k1, g0 + gstep + j, a.pre);
            {
                float o[BPT][4];
#pragma unroll
                for (int j = 0; j < BPT; ++j) bm4<LOGM, TL, QUAD>(wb[j], a.off, o[j]);
#pragma unroll
                for (int j = 0; j < BPT; j += 2) st_group2(dst + 4 * j, o[j], o[j + 1]);
            }
            g0 += gstep;
            dst += dstep;
        }
    } else {
        for (uint32_t g0 = gtid * BPT; g0 < gfull; g0 += gstep, dst += dstep) {
            float o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) bm4<LOGM, TL, QUAD>(philox_block_pre(a.k0, a.k1, g0 + j, a.pre), a.off, o[j]);
#pragma unroll
            for (int j = 0; j < BPT; j += 2) st_group2(dst + 4 * j, o[j], o[j + 1]);
        }
    }
}

// ------------------------------------------------------------ accuracy
__device__ unsigned int g_acc[16];  // [0..6] max ulp per band (float bits), [7] max abs/2^-20, [8] neg r count

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__device__ void acc_err(float got, double ref) {
    const double a = fabs(ref);
    const int band = a < 1e-6 ? 0 : a < 1e-3 ? 1 : a < 0.1 ? 2 : a < 1.0 ? 3 : a < 2.0 ? 4 : a < 4.0 ? 5 : 6;
    const float rf = (float)ref;
    int e;
    frexpf(fabsf(rf) < 1.17549435e-38f ? 1.17549435e-38f : rf, &e);
    const double ulp = ldexp(1.0, e - 24);
    const double err = fabs((double)got - ref);
    const float u = (float)(err / ulp);
    atomicMax(&g_acc[band], __float_as_uint(u));
    const float ab = (float)(err / (a > 1.0 ? a : 1.0) / 9.5367431640625e-07);
    atomicMax(&g_acc[7], __float_as_uint(ab));
}

template <int LOGM, int TL, int QUAD>
__global__ void kacc() {
    prologue<LOGM, TL>(1.1774100225154747f);  // S = sqrt(2 ln 2): table-scaled standard normal
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < (1u << 24); k += gridDim.x * blockDim.x) {
        for (int side = 0; side < 2; ++side) {
            const uint32_t h = hash32(k * 2 + side) & 0xFFFFFF00u;
            const uint32_t w0 = side == 0 ? (k << 8) : h;
            const uint32_t w1 = side == 0 ? h : (k << 8);
            float o0, o1;
            bm<LOGM, TL, QUAD>(w0, w1, 0.0f, o0, o1);
            const double u1 = (double)(w0 >> 8) * 5.9604644775390625e-08;
            const double u2 = (double)(w1 >> 8) * 5.9604644775390625e-08;
            const double r = sqrt(-2.0 * log(1.0 - u1));
            const double t = __dmul_rn(6.283185307179586, u2);
            double sn, cs;
            sincos(t, &sn, &cs);
            acc_err(o0, r * cs);
            acc_err(o1, r * sn);
        }
    }
}

// lognormal m = 0, s = 1: x = ex2(fma(rq, cs', 0)) with the table scaled by
// sqrt(2 ln 2) log2(e) (library route), vs exp(z) in fp64; ulps of x, and
// ulps / max(1, |ln x|) in g_acc[9..10]
template <int LOGM, int TL, int QUAD>
__global__ void kacc_logn() {
    prologue<LOGM, TL>(1.1774100225154747f * 1.4426950408889634f);
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < (1u << 24); k += gridDim.x * blockDim.x) {
        for (int side = 0; side < 2; ++side) {
            const uint32_t h = hash32(k * 2 + side) & 0xFFFFFF00u;
            const uint32_t w0 = side == 0 ? (k << 8) : h;
            const uint32_t w1 = side == 0 ? h : (k << 8);
            float y0, y1;
            bm<LOGM, TL, QUAD>(w0, w1, 0.0f, y0, y1);
            float e0, e1;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(y0));
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(y1));
            const double u1 = (double)(w0 >> 8) * 5.9604644775390625e-08;
            const double u2 = (double)(w1 >> 8) * 5.9604644775390625e-08;
            const double r = sqrt(-2.0 * log(1.0 - u1));
            const double t = __dmul_rn(6.283185307179586, u2);
            double sn, cs;
            sincos(t, &sn, &cs);
            const double x0 = exp(r * cs), x1 = exp(r * sn);
            for (int q = 0; q < 2; ++q) {
                const double x = q ? x1 : x0;
                const float got = q ? e1 : e0;
                int e;
                frexpf((float)x, &e);
                const double ulp = ldexp(1.0, e - 24);
                const float u = (float)(fabs((double)got - x) / ulp);
                atomicMax(&g_acc[9], __float_as_uint(u));
                const double lx = fabs(log(x));
                atomicMax(&g_acc[10], __float_as_uint((float)(u / (lx > 1.0 ? lx : 1.0))));
            }
        }
    }
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(a));
        for (int i = 0; i < 10; ++i) f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms / 10 < best) best = ms / 10;
    }
    CK(cudaGetLastError());
    return best;
}

static float* g_out;
static int g_sms;
static const uint32_t kN = 1u << 30;

template <int LOGM, int TL, int QUAD, int LOOP, int MINB, int THREADS>
void run(const char* tag) {
    auto kern = kgauss<LOGM, TL, QUAD, LOOP, MINB, THREADS>;
    const size_t smem = (TL ? ((1 << TL) + 1) * 8 : 0) + (LOGM ? kLogEntries * 8 : 0);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, smem));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    GParams a{};
    a.k0 = 777;
    a.k1 = 0;
    a.pre = philox_pre(777, 0, 0, 0, 0);
    a.ngroups = kN / 4;
    a.out = g_out;
    a.S = 1.1774100225154747f;
    a.off = 0.0f;
    unsigned grid = g_sms * occ;
    if constexpr (LOOP >= 3) {
        CK(cudaFuncSetAttribute(kfill<LOGM, TL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kfill<LOGM, TL><<<1, 256, smem>>>(a.S);
        grid = (unsigned)((a.ngroups + THREADS * 4 * (LOOP - 2) - 1) / (THREADS * 4 * (LOOP - 2)));
    }
    const float ms = timeit([&] { kern<<<grid, THREADS, smem>>>(a); });
    // accuracy
    unsigned int z[16] = {0};
    CK(cudaMemcpyToSymbol(g_acc, z, sizeof z));
    kacc<LOGM, TL, QUAD><<<g_sms * 2, 256, smem>>>();
    CK(cudaFuncSetAttribute(kacc<LOGM, TL, QUAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaMemcpyToSymbol(g_acc, z, sizeof z));
    kacc<LOGM, TL, QUAD><<<g_sms * 2, 256, smem>>>();
    CK(cudaFuncSetAttribute(kacc_logn<LOGM, TL, QUAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kacc_logn<LOGM, TL, QUAD><<<g_sms * 2, 256, smem>>>();
    CK(cudaDeviceSynchronize());
    unsigned int h[16];
    CK(cudaMemcpyFromSymbol(h, g_acc, sizeof h));
    float f[16];
    memcpy(f, h, sizeof f);
    printf("%-34s regs=%3d occ=%d smem=%6zu  %7.3f ms %7.1f Gs/s %7.1f GB/s | ulp <1e-6 %.3g  <1e-3 %.3g  <.1 %.3g  <1 %.2f  "
           "<2 %.2f  <4 %.2f  >=4 %.2f | abs %.3f x2^-20 | logn ulp %.2f, /max(1,|ln x|) %.2f\n",
           tag, fa.numRegs, occ, smem, ms, kN / ms / 1e6, kN * 4.0 / ms / 1e6, f[0], f[1], f[2], f[3], f[4], f[5], f[6],
           f[7], f[9], f[10]);
    fflush(stdout);
}

int main(int argc, char** argv) {
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaMalloc(&g_out, (size_t)kN * 4));
    run<0, 0, 0, 2, 0, 256>("lib math, loop2");
    run<0, 0, 0, 0, 4, 256>("lib math, loop0 minb4");
    run<0, 12, 0, 2, 0, 256>("lg2, ctr12, loop2");
    run<0, 12, 0, 0, 4, 256>("lg2, ctr12, loop0 minb4");
    run<0, 12, 0, 2, 6, 256>("lg2, ctr12, loop2 minb6");
    run<0, 13, 0, 2, 0, 512>("lg2, ctr13, loop2 512");
    run<1, 12, 1, 2, 0, 256>("ltab, ctr12 quad, loop2");
    run<1, 12, 1, 2, 5, 256>("ltab, ctr12 quad, loop2 minb5");
    run<1, 12, 1, 0, 4, 256>("ltab, ctr12 quad, loop0 minb4");
    run<1, 13, 0, 2, 0, 512>("ltab, ctr13, loop2 512");
    run<1, 12, 0, 2, 0, 256>("ltab, ctr12, loop2");
    run<1, 12, 0, 2, 5, 256>("ltab, ctr12, loop2 minb5");
    run<1, 12, 0, 0, 4, 256>("ltab, ctr12, loop0 minb4");
    CK(cudaFree(g_out));
    return 0;
}
