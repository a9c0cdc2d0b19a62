// philox_np.cu -- persistent vs non-persistent Philox generate kernels
// (sm_100a).  tools/store_probe.cu showed write-only kernels plateau at
// ~6.4 TB/s with any persistent grid-stride pattern but reach ~7.6 TB/s when
// every CTA writes one small contiguous chunk and exits.  This compares the
// library kernel (persistent) with non-persistent shapes of the same Philox +
// unit-fp32 (and bits) work at n = 2^32, bit-checked against the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I../paper_2109_01329_b200/csrc \
//        -o philox_np philox_np.cu
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

// Non-persistent: CTA b covers groups [b * CH, (b + 1) * CH), CH = THREADS *
// BPT * ITER; within a pass i every thread computes BPT adjacent blocks and
// stores them with 256-bit stores (thread-contiguous 16*BPT bytes, like the
// library), or LAYOUT 1: warp-contiguous (each STG.256 covers 1 KiB).
template <int X, int BPT, int ITER, int THREADS, int MINB, int LAYOUT>
__global__ void __launch_bounds__(THREADS, MINB) knp(const PhiloxBody a) {
    using T = typename XformTraits<X>::T;
    T* __restrict__ body = static_cast<T*>(a.out);
    constexpr uint32_t CH = THREADS * BPT * ITER;
    const uint32_t cbase = blockIdx.x * CH;
#pragma unroll 1
    for (int i = 0; i < ITER; ++i) {
        uint32_t g0;
        if constexpr (LAYOUT == 0) {
            g0 = cbase + (i * THREADS + threadIdx.x) * BPT;
        } else {
            const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            g0 = cbase + (i * THREADS + warp * 32) * BPT + 2 * lane;  // blocks 2l, 2l+1 (+64 for the 2nd pair)
        }
        if (g0 + (LAYOUT ? 64 + 2 : BPT) > a.ngroups) {
            for (int j = 0; j < BPT; ++j) {
                const uint32_t g = LAYOUT ? g0 + 64 * (j >> 1) + (j & 1) : g0 + j;
                if (g < a.ngroups) {
                    T o[4];
                    xform4<X>(philox_block_pre<philox_rk<X>()>(a.k0, a.k1, a.c0 + g, a.pre), a.p, o);
                    st_group(body + (size_t)4 * g, o);
                }
            }
            continue;
        }
        T o[BPT][4];
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const uint32_t g = LAYOUT ? g0 + 64 * (j >> 1) + (j & 1) : g0 + j;
            xform4<X>(philox_block_pre<philox_rk<X>()>(a.k0, a.k1, a.c0 + g, a.pre), a.p, o[j]);
        }
#pragma unroll
        for (int j = 0; j < BPT; j += 2) {
            const uint32_t g = LAYOUT ? g0 + 64 * (j >> 1) : g0 + j;
            st_group2(body + (size_t)4 * g, o[j], o[j + 1]);
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
    for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(a));
        for (int i = 0; i < reps; ++i) f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        ts.push_back(ms / reps);
    }
    CK(cudaGetLastError());
    return *std::min_element(ts.begin(), ts.end());
}

static const uint64_t kN = 1ull << 32;
static int g_sms;
static uint32_t *g_ref, *g_out;

PhiloxBody body_for(void* out) {
    PhiloxBody b{};
    b.k0 = 777;
    b.k1 = 0;
    b.ngroups = (uint32_t)(kN / 4);
    b.pre = philox_pre(777, 0, 0, 0, 0);
    b.out = out;
    b.p.scale_f = 1.0f;
    return b;
}

bool same(const uint32_t* a, const uint32_t* b) {
    // sample compare: 64 MiB window at the start, middle, end
    std::vector<uint32_t> x(1 << 24), y(1 << 24);
    const uint64_t offs[3] = {0ull, kN / 2 - (1ull << 23), kN - (1ull << 24)};
    for (uint64_t off : offs) {
        CK(cudaMemcpy(x.data(), a + off, x.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(y.data(), b + off, y.size() * 4, cudaMemcpyDeviceToHost));
        if (x != y) return false;
    }
    return true;
}

template <int X, int BPT, int ITER, int THREADS, int MINB, int LAYOUT>
void run_np(const char* xname) {
    PhiloxBody b = body_for(g_out);
    constexpr uint32_t CH = THREADS * BPT * ITER;
    const uint32_t grid = (uint32_t)((b.ngroups + CH - 1) / CH);
    CK(cudaMemset(g_out, 0, kN * 4));
    const float ms = timeit([&] { knp<X, BPT, ITER, THREADS, MINB, LAYOUT><<<grid, THREADS>>>(b); });
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, knp<X, BPT, ITER, THREADS, MINB, LAYOUT>));
    printf("%-6s np bpt=%d iter=%2d thr=%4d minb=%d layout=%d regs=%2d  %7.3f ms %8.1f GB/s %7.1f Gs/s %s\n", xname, BPT,
           ITER, THREADS, MINB, LAYOUT, fa.numRegs, ms, kN * 4 / ms / 1e6, kN / ms / 1e6,
           same(g_out, g_ref) ? "ok" : "MISMATCH");
    fflush(stdout);
}

template <int X>
void run_lib(const char* xname) {
    PhiloxBody b = body_for(g_ref);
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, philox_kernel<X, 0>, kPhiloxThreads, 0));
    const float ms = timeit([&] { philox_kernel<X, 0><<<g_sms * occ, kPhiloxThreads>>>(b); });
    printf("%-6s library persistent occ=%d                          %7.3f ms %8.1f GB/s %7.1f Gs/s\n", xname, occ, ms,
           kN * 4 / ms / 1e6, kN / ms / 1e6);
    fflush(stdout);
}

int main() {
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaMalloc(&g_ref, kN * 4));
    CK(cudaMalloc(&g_out, kN * 4));
    run_lib<kUnitF32>("unit");
    run_np<kUnitF32, 4, 1, 256, 0, 0>("unit");
    run_np<kUnitF32, 4, 2, 256, 0, 0>("unit");
    run_np<kUnitF32, 4, 4, 256, 0, 0>("unit");
    run_np<kUnitF32, 4, 8, 256, 0, 0>("unit");
    run_np<kUnitF32, 4, 1, 256, 5, 0>("unit");
    run_np<kUnitF32, 4, 2, 256, 5, 0>("unit");
    run_np<kUnitF32, 4, 4, 256, 5, 0>("unit");
    run_np<kUnitF32, 2, 2, 256, 0, 0>("unit");
    run_np<kUnitF32, 2, 4, 256, 0, 0>("unit");
    run_np<kUnitF32, 4, 2, 128, 0, 0>("unit");
    run_np<kUnitF32, 4, 2, 512, 0, 0>("unit");
    run_np<kUnitF32, 4, 1, 256, 0, 1>("unit");
    run_np<kUnitF32, 4, 2, 256, 0, 1>("unit");
    run_np<kUnitF32, 4, 4, 256, 5, 1>("unit");
    run_lib<kBits>("bits");
    run_np<kBits, 4, 1, 256, 0, 0>("bits");
    run_np<kBits, 4, 2, 256, 0, 0>("bits");
    run_np<kBits, 4, 4, 256, 0, 0>("bits");
    run_np<kBits, 4, 2, 256, 0, 1>("bits");
    CK(cudaFree(g_ref));
    CK(cudaFree(g_out));
    return 0;
}
