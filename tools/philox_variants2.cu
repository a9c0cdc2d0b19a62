// philox_variants2.cu -- second round of Philox kernel experiments (sm_100a).
//
// All variants use the library's round-1..3 host folding (PhiloxPre) and write
// n = 2^32 unit fp32 samples (16 GiB).  Compares block-per-thread counts,
// occupancy, store flavours, and compute-only / store-only ceilings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2109_01329_b200/csrc \
//        -o philox_variants2 philox_variants2.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "philox.cuh"

using namespace prng;

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

enum StoreKind { kCs = 0, kWb = 1, kNa = 2, kNone = 3 };

template <int SK>
__device__ __forceinline__ void st8(float* p, const float* a) {
    if constexpr (SK == kCs)
        asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a[0]), "f"(a[1]),
                     "f"(a[2]), "f"(a[3]), "f"(a[4]), "f"(a[5]), "f"(a[6]), "f"(a[7])
                     : "memory");
    if constexpr (SK == kWb)
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]),
                     "f"(a[3]), "f"(a[4]), "f"(a[5]), "f"(a[6]), "f"(a[7])
                     : "memory");
    if constexpr (SK == kNa)
        asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a[0]),
                     "f"(a[1]), "f"(a[2]), "f"(a[3]), "f"(a[4]), "f"(a[5]), "f"(a[6]), "f"(a[7])
                     : "memory");
}

// Generic grid-stride kernel: BPT blocks per thread per pass.
template <int BPT, int SK, int MINB, int THREADS>
__global__ void __launch_bounds__(THREADS, MINB) kgen(float* out, uint32_t k0, uint32_t k1, PhiloxPre pre,
                                                     uint32_t ngroups, uint32_t* sink) {
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    uint32_t acc = 0;
    float* dst = out + (size_t)4 * BPT * gtid;
    for (uint32_t g0 = gtid * BPT; g0 < ngroups; g0 += gstride * BPT, dst += (size_t)4 * BPT * gstride) {
        float o[4 * BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const U4 w = philox_block_pre(k0, k1, g0 + j, pre);
            o[4 * j] = unit_f32(w.x);
            o[4 * j + 1] = unit_f32(w.y);
            o[4 * j + 2] = unit_f32(w.z);
            o[4 * j + 3] = unit_f32(w.w);
            acc ^= w.x ^ w.y ^ w.z ^ w.w;
        }
        if constexpr (SK != kNone) {
#pragma unroll
            for (int j = 0; j < BPT; j += 2) st8<SK>(dst + 4 * j, o + 4 * j);
        }
    }
    if constexpr (SK == kNone) {
        if (acc == 0x12345678u) sink[0] = acc;  // keep the compute alive
    }
}

// Conversion variants: 0 = I2FP + FMUL (library), 1 = I2FP + integer exponent
// adjust (max(bits - 24<<23, 0)), 2 = raw words (no conversion).
template <int CONV>
__device__ __forceinline__ float conv(uint32_t w) {
    if constexpr (CONV == 0) return unit_f32(w);
    if constexpr (CONV == 1) {
        const int b = __float_as_int((float)(w >> 8)) - 0x0C000000;
        return __int_as_float(b > 0 ? b : 0);
    }
    if constexpr (CONV == 3) return (float)(w >> 8);  // I2FP only
    if constexpr (CONV == 4) {
        // no I2FP: f = 0.5 + m 2^-24 from bits, minus 0.5 unless the top bit is set (exact)
        const float f = __uint_as_float(((w >> 8) & 0x7FFFFFu) | 0x3F000000u);
        const float c = __uint_as_float(~((uint32_t)((int)w >> 31)) & 0x3F000000u);
        return __fsub_rn(f, c);
    }
    if constexpr (CONV == 5) return __uint_as_float(w >> 8);  // shift only
    return __uint_as_float(w);
}

template <int CONV>
__global__ void __launch_bounds__(256) kconv(float* out, uint32_t k0, uint32_t k1, PhiloxPre pre, uint32_t ngroups) {
    constexpr int BPT = 4;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    float* dst = out + (size_t)4 * BPT * gtid;
    for (uint32_t g0 = gtid * BPT; g0 < ngroups; g0 += gstride * BPT, dst += (size_t)4 * BPT * gstride) {
        float o[4 * BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const U4 w = philox_block_pre(k0, k1, g0 + j, pre);
            if constexpr (CONV == 6) {  // half I2FP (FMA-heavy), half bit trick (ALU)
                o[4 * j] = conv<0>(w.x);
                o[4 * j + 1] = conv<4>(w.y);
                o[4 * j + 2] = conv<0>(w.z);
                o[4 * j + 3] = conv<4>(w.w);
            } else if constexpr (CONV == 7) {  // 1 of 4 via bit trick
                o[4 * j] = conv<0>(w.x);
                o[4 * j + 1] = conv<0>(w.y);
                o[4 * j + 2] = conv<0>(w.z);
                o[4 * j + 3] = conv<4>(w.w);
            } else {
                o[4 * j] = conv<CONV>(w.x);
                o[4 * j + 1] = conv<CONV>(w.y);
                o[4 * j + 2] = conv<CONV>(w.z);
                o[4 * j + 3] = conv<CONV>(w.w);
            }
        }
#pragma unroll
        for (int j = 0; j < BPT; j += 2) st8<kCs>(dst + 4 * j, o + 4 * j);
    }
}

// Store-only ceiling with the same access pattern.
template <int BPT>
__global__ void __launch_bounds__(256) kstore(float* out, uint32_t ngroups) {
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    float* dst = out + (size_t)4 * BPT * gtid;
    float o[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    for (uint32_t g0 = gtid * BPT; g0 < ngroups; g0 += gstride * BPT, dst += (size_t)4 * BPT * gstride) {
#pragma unroll
        for (int j = 0; j < BPT; j += 2) st8<kCs>(dst + 4 * j, o);
    }
}


// Warp-contiguous layouts: a warp pass covers 32*BPT consecutive blocks.
//  LAYOUT 1: lane l computes block pairs (2l, 2l+1) + 64*i -> each STG.256 instruction = 1 KiB contiguous
//  LAYOUT 2: lane l computes blocks l + 32*i -> each STG.128 instruction = 512 B contiguous
template <int BPT, int LAYOUT, bool STORE, int MINB>
__global__ void __launch_bounds__(256, MINB) kwarp(float* out, uint32_t k0, uint32_t k1, PhiloxPre pre,
                                                   uint32_t ngroups, uint32_t* sink) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (uint32_t base = gw * 32 * BPT; base < ngroups; base += nw * 32 * BPT) {
        float o[4 * BPT];
        uint32_t blk[BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            if (LAYOUT == 1) blk[j] = base + 64 * (j >> 1) + 2 * lane + (j & 1);
            else blk[j] = base + 32 * j + lane;
            const U4 w = philox_block_pre(k0, k1, blk[j], pre);
            o[4 * j] = unit_f32(w.x);
            o[4 * j + 1] = unit_f32(w.y);
            o[4 * j + 2] = unit_f32(w.z);
            o[4 * j + 3] = unit_f32(w.w);
            acc ^= w.x ^ w.y ^ w.z ^ w.w;
        }
        if (STORE) {
            if (LAYOUT == 1) {
#pragma unroll
                for (int j = 0; j < BPT; j += 2) st8<kCs>(out + 4 * (size_t)blk[j], o + 4 * j);
            } else {
#pragma unroll
                for (int j = 0; j < BPT; ++j) {
                    float* p = out + 4 * (size_t)blk[j];
                    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(o[4*j]), "f"(o[4*j+1]),
                                 "f"(o[4*j+2]), "f"(o[4*j+3]) : "memory");
                }
            }
        }
    }
    if (!STORE && acc == 0x12345678u) sink[0] = acc;
}

template <int BPT, int LAYOUT>
__global__ void __launch_bounds__(256) kwstore(float* out, uint32_t ngroups) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    float o[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    for (uint32_t base = gw * 32 * BPT; base < ngroups; base += nw * 32 * BPT) {
        if (LAYOUT == 1) {
#pragma unroll
            for (int j = 0; j < BPT; j += 2) st8<kCs>(out + 4 * (size_t)(base + 64 * (j >> 1) + 2 * lane), o);
        } else {
#pragma unroll
            for (int j = 0; j < BPT; ++j) {
                float* p = out + 4 * (size_t)(base + 32 * j + lane);
                asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                             "f"(o[3]) : "memory");
            }
        }
    }
}

template <typename F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) f();
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

template <typename K>
int occ(K k, int threads) {
    int o = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, threads, 0));
    return o;
}

int main() {
    const uint64_t n = 1ull << 32;
    const uint32_t ngroups = (uint32_t)(n / 4);
    float* out;
    uint32_t* sink;
    CK(cudaMalloc(&out, n * 4));
    CK(cudaMalloc(&sink, 4));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t k0 = 777, k1 = 0;
    const PhiloxPre pre = philox_pre(k0, k1, 0, 0, 0);
    auto report = [&](const char* name, float ms) {
        printf("%-44s %8.3f ms  %8.1f GB/s  %7.1f Gs/s\n", name, ms, n * 4 / ms / 1e6, n / ms / 1e6);
    };
#define RUN(BPT, SK, MINB, THREADS, WAVES)                                                                   \
    {                                                                                                        \
        auto k = kgen<BPT, SK, MINB, THREADS>;                                                               \
        int o = occ(k, THREADS);                                                                             \
        int g = sms * o * WAVES;                                                                             \
        float ms = timeit([&] { kgen<BPT, SK, MINB, THREADS><<<g, THREADS>>>(out, k0, k1, pre, ngroups, sink); }); \
        char nm[96];                                                                                         \
        snprintf(nm, 96, "bpt=%d st=%d minb=%d thr=%d occ=%d waves=%d", BPT, SK, MINB, THREADS, o, WAVES);     \
        report(nm, ms);                                                                                      \
    }
    {
        // the library's own kernel template, launched directly (no Python / C-ABI in the loop)
        PhiloxBody b{};
        b.k0 = k0;
        b.k1 = k1;
        b.ngroups = ngroups;
        b.pre = pre;
        b.out = out;
        auto k = philox_kernel<kUnitF32, 0>;
        int o = occ(k, 256);
        float ms = timeit([&] { philox_kernel<kUnitF32, 0><<<sms * o, 256>>>(b); });
        char nm[96];
        snprintf(nm, 96, "library philox_kernel<kUnitF32,0> occ=%d", o);
        report(nm, ms);
        auto kb = philox_kernel<kBits, 0>;
        o = occ(kb, 256);
        ms = timeit([&] { philox_kernel<kBits, 0><<<sms * o, 256>>>(b); });
        snprintf(nm, 96, "library philox_kernel<kBits,0> occ=%d", o);
        report(nm, ms);
    }
    {
        const char* names[3] = {"conv I2FP+FMUL", "conv I2FP+exp-adjust (ALU)", "conv none (raw bits)"};
        float ms0 = timeit([&] { kconv<0><<<sms * occ(kconv<0>, 256), 256>>>(out, k0, k1, pre, ngroups); });
        report(names[0], ms0);
        float ms1 = timeit([&] { kconv<1><<<sms * occ(kconv<1>, 256), 256>>>(out, k0, k1, pre, ngroups); });
        report(names[1], ms1);
        float ms2 = timeit([&] { kconv<2><<<sms * occ(kconv<2>, 256), 256>>>(out, k0, k1, pre, ngroups); });
        report(names[2], ms2);
        report("conv I2FP only", timeit([&] { kconv<3><<<sms * occ(kconv<3>, 256), 256>>>(out, k0, k1, pre, ngroups); }));
        report("conv bit-trick (no I2FP)", timeit([&] { kconv<4><<<sms * occ(kconv<4>, 256), 256>>>(out, k0, k1, pre, ngroups); }));
        report("conv shift only", timeit([&] { kconv<5><<<sms * occ(kconv<5>, 256), 256>>>(out, k0, k1, pre, ngroups); }));
        report("conv mixed 2 I2FP + 2 bit-trick", timeit([&] { kconv<6><<<sms * occ(kconv<6>, 256), 256>>>(out, k0, k1, pre, ngroups); }));
        report("conv mixed 3 I2FP + 1 bit-trick", timeit([&] { kconv<7><<<sms * occ(kconv<7>, 256), 256>>>(out, k0, k1, pre, ngroups); }));
        report("conv I2FP+FMUL (again)",timeit([&] { kconv<0><<<sms * occ(kconv<0>, 256), 256>>>(out, k0, k1, pre, ngroups); }));
    }
    RUN(4, kCs, 1, 256, 1);  // library shape
    RUN(4, kWb, 1, 256, 1);
    RUN(4, kNa, 1, 256, 1);
    RUN(4, kNone, 1, 256, 1);  // compute-only ceiling
    RUN(2, kCs, 1, 256, 1);
    RUN(8, kCs, 1, 256, 1);
    RUN(8, kNone, 1, 256, 1);
    RUN(4, kCs, 6, 256, 1);
    RUN(4, kCs, 8, 256, 1);
    RUN(4, kCs, 1, 128, 1);
    RUN(4, kCs, 1, 512, 1);
    RUN(4, kCs, 1, 256, 2);
    RUN(4, kCs, 1, 256, 4);

#define RUNW(BPT, LAYOUT, STORE, MINB)                                                                         \
    {                                                                                                        \
        auto k = kwarp<BPT, LAYOUT, STORE, MINB>;                                                            \
        int o = occ(k, 256);                                                                                 \
        int g = sms * o;                                                                                     \
        float ms = timeit([&] { kwarp<BPT, LAYOUT, STORE, MINB><<<g, 256>>>(out, k0, k1, pre, ngroups, sink); }); \
        char nm[96];                                                                                         \
        snprintf(nm, 96, "warp-contig bpt=%d layout=%d store=%d minb=%d occ=%d", BPT, LAYOUT, STORE, MINB, o); \
        report(nm, ms);                                                                                      \
    }
    RUNW(4, 1, true, 1);
    RUNW(4, 2, true, 1);
    RUNW(8, 1, true, 1);
    RUNW(8, 2, true, 1);
    RUNW(4, 1, false, 1);
    RUNW(8, 1, false, 1);
    RUNW(6, 2, true, 1);
    {
        float ms = timeit([&] { kwstore<4, 1><<<sms * 8, 256>>>(out, ngroups); });
        report("store-only warp-contig STG.256 (1KiB/instr)", ms);
        ms = timeit([&] { kwstore<4, 2><<<sms * 8, 256>>>(out, ngroups); });
        report("store-only warp-contig STG.128 (512B/instr)", ms);
        ms = timeit([&] { kwstore<8, 2><<<sms * 8, 256>>>(out, ngroups); });
        report("store-only warp-contig STG.128 bpt8", ms);
    }
    {
        float ms = timeit([&] { kstore<4><<<sms * 8, 256>>>(out, ngroups); });
        report("store-only bpt=4 (same pattern)", ms);
    }
    {
        float ms = timeit([&] { CK(cudaMemsetAsync(out, 0, n * 4)); });
        report("cudaMemset", ms);
    }
    return 0;
}
