// unit_conv.cu -- word -> unit fp32 conversion variants in the headline kernel
// shape (persistent grid, 4 Philox blocks per thread per pass, 256-bit
// streaming stores, round keys from the parameter table), n = 2^32,
// bit-checked against the library kernel.  All variants are exact:
//   0  (float)(w >> 8) * 2^-24                      SHF + I2FP + FMUL (library)
//   1  (float)(w & 0xFFFFFF00) * 2^-32              LOP3 + I2FP + FMUL: <= 24 significant bits, exact
//   2  I2FP-free: f = bits(0x3F000000 | (w>>8 & 0x7FFFFF)), u = f - (w < 2^31 ? 0.5 : 0)
//   3  half the words as 1, half as 2 (spread the work over the FMA and ALU pipes)
//   4  one word in four as 2
//   5  bits only (no conversion): the compute ceiling of the store pattern
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I../paper_2109_01329_b200/csrc -o unit_conv unit_conv.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

template <int C>
__device__ __forceinline__ float conv(uint32_t w) {
    if constexpr (C == 0) return __fmul_rn((float)(w >> 8), 5.9604644775390625e-08f);
    if constexpr (C == 1) return __fmul_rn(__uint2float_rn(w & 0xFFFFFF00u), 2.3283064365386963e-10f);
    if constexpr (C == 2) {
        const float f = __uint_as_float(((w >> 8) & 0x7FFFFFu) | 0x3F000000u);
        const float c = __uint_as_float(~((uint32_t)((int)w >> 31)) & 0x3F000000u);
        return __fsub_rn(f, c);
    }
    return __uint_as_float(w);
}

template <int C>
__device__ __forceinline__ void conv4(const U4& w, float o[4]) {
    if constexpr (C <= 2 || C == 5) {
        constexpr int K = C == 5 ? 9 : C;
        o[0] = conv<K>(w.x); o[1] = conv<K>(w.y); o[2] = conv<K>(w.z); o[3] = conv<K>(w.w);
    } else if constexpr (C == 3) {
        o[0] = conv<1>(w.x); o[1] = conv<2>(w.y); o[2] = conv<1>(w.z); o[3] = conv<2>(w.w);
    } else {
        o[0] = conv<1>(w.x); o[1] = conv<1>(w.y); o[2] = conv<1>(w.z); o[3] = conv<2>(w.w);
    }
}

template <int C, int MINB>
__global__ void __launch_bounds__(256, MINB) kunit(const PhiloxBody a) {
    constexpr int BPT = 4;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    const uint32_t gstep = gstride * BPT;
    const uint32_t gfull = a.ngroups - a.ngroups % BPT;
    float* dst = static_cast<float*>(a.out) + (size_t)4 * BPT * gtid;
    for (uint32_t g0 = gtid * BPT; g0 < gfull; g0 += gstep, dst += (size_t)4 * gstep) {
        float o[BPT][4];
#pragma unroll
        for (int j = 0; j < BPT; ++j) conv4<C>(philox_block_pre<true>(a.k0, a.k1, a.c0 + g0 + j, a.pre), o[j]);
#pragma unroll
        for (int j = 0; j < BPT; j += 2) st_group2(dst + 4 * j, o[j], o[j + 1]);
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
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        for (int i = 0; i < reps; ++i) f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        ts.push_back(ms / reps);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

static const uint64_t kN = 1ull << 32;
static int g_sms;
static uint32_t *g_ref, *g_out;

PhiloxBody body_for(void* out) {
    PhiloxBody b{};
    b.k0 = 777;
    b.ngroups = (uint32_t)(kN / 4);
    b.pre = philox_pre(777, 0, 0, 0, 0);
    b.out = out;
    b.p.scale_f = 1.0f;
    return b;
}

bool same() {
    std::vector<uint32_t> x(1 << 24), y(1 << 24);
    const uint64_t offs[3] = {0ull, kN / 2 - (1ull << 23), kN - (1ull << 24)};
    for (uint64_t off : offs) {
        CK(cudaMemcpy(x.data(), g_out + off, x.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(y.data(), g_ref + off, y.size() * 4, cudaMemcpyDeviceToHost));
        if (x != y) return false;
    }
    return true;
}

template <int C, int MINB>
void run(const char* nm) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kunit<C, MINB>, 256, 0));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kunit<C, MINB>));
    PhiloxBody b = body_for(g_out);
    CK(cudaMemset(g_out, 0, kN * 4));
    const float ms = timeit([&] { kunit<C, MINB><<<g_sms * occ, 256>>>(b); });
    printf("%-34s regs=%2d occ=%d %7.3f ms %8.1f GB/s %7.1f Gs/s %s\n", nm, fa.numRegs, occ, ms, kN * 4 / ms / 1e6,
           kN / ms / 1e6, C == 5 ? "(bits)" : same() ? "ok" : "MISMATCH");
    fflush(stdout);
}

int main() {
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaMalloc(&g_ref, kN * 4));
    CK(cudaMalloc(&g_out, kN * 4));
    {
        PhiloxBody b = body_for(g_ref);
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, philox_kernel<kUnitF32, 0>, 256, 0));
        const float ms = timeit([&] { philox_kernel<kUnitF32, 0><<<g_sms * occ, 256>>>(b); });
        printf("%-34s        occ=%d %7.3f ms %8.1f GB/s %7.1f Gs/s\n", "library philox_kernel<kUnitF32,0>", occ, ms,
               kN * 4 / ms / 1e6, kN / ms / 1e6);
    }
    for (int rep = 0; rep < 2; ++rep) {
        run<0, 5>("0 shf+i2fp+fmul minb5");
        run<1, 5>("1 lop3+i2fp+fmul minb5");
        run<2, 5>("2 no-i2fp minb5");
        run<3, 5>("3 half/half minb5");
        run<4, 5>("4 three-quarter/quarter minb5");
        run<1, 6>("1 lop3+i2fp+fmul minb6");
        run<1, 4>("1 lop3+i2fp+fmul minb4");
        run<5, 5>("5 bits (no conversion) minb5");
        run<5, 0>("5 bits (no conversion) minb0");
    }
    return 0;
}
