// philox_tma.cu -- experiment: Philox unit-fp32 generation with the output
// staged in shared memory and written by per-warp bulk (TMA) stores instead of
// per-thread STG.256.  Compares against the library kernel on n = 2^32.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2109_01329_b200/csrc \
//        -o philox_tma philox_tma.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
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

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// HINT: 0 = none, 1 = L2 evict_first policy.
template <int BPT, int SLOTS, int HINT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) ktma(float* out, uint32_t k0, uint32_t k1, PhiloxPre pre,
                                                   uint32_t nblocks) {
    extern __shared__ __align__(128) float smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kPer = 32 * BPT;  // Philox blocks per warp iteration
    float* wbuf = smem + warp * SLOTS * kPer * 4;
    const uint32_t wstride = gridDim.x * WARPS * kPer;
    uint64_t policy = 0;
    if constexpr (HINT == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int slot = 0, it = 0;
    for (uint32_t b0 = (blockIdx.x * WARPS + warp) * kPer; b0 < nblocks; b0 += wstride) {
        float* s = wbuf + slot * kPer * 4;
        if (it >= SLOTS) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(SLOTS - 1) : "memory");
            __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const U4 w = philox_block_pre(k0, k1, b0 + j * 32 + lane, pre);
            float o[4] = {unit_f32(w.x), unit_f32(w.y), unit_f32(w.z), unit_f32(w.w)};
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(s + (j * 32 + lane) * 4)), "f"(o[0]),
                         "f"(o[1]), "f"(o[2]), "f"(o[3])
                         : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            float* g = out + (size_t)b0 * 4;
            if constexpr (HINT == 1)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(g),
                             "r"(smem_addr(s)), "n"(kPer * 16), "l"(policy)
                             : "memory");
            else
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_addr(s)),
                             "n"(kPer * 16)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        slot = slot + 1 == SLOTS ? 0 : slot + 1;
        ++it;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) f();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> v;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        v.push_back(ms);
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

int main() {
    const uint64_t n = 1ull << 32;
    const uint32_t nblocks = (uint32_t)(n / 4);
    float* out;
    CK(cudaMalloc(&out, n * 4));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t k0 = 777, k1 = 0;
    const PhiloxPre pre = philox_pre(k0, k1, 0, 0, 0);
    std::vector<float> ref(1 << 20), got(1 << 20);
    auto report = [&](const char* name, float ms) {
        printf("%-52s %8.3f ms  %8.1f GB/s  %7.1f Gs/s\n", name, ms, n * 4 / ms / 1e6, n / ms / 1e6);
    };
    {
        PhiloxBody b{};
        b.k0 = k0;
        b.k1 = k1;
        b.ngroups = nblocks;
        b.pre = pre;
        b.out = out;
        int o = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, philox_kernel<kUnitF32, 0>, 256, 0));
        float ms = timeit([&] { philox_kernel<kUnitF32, 0><<<sms * o, 256>>>(b); });
        report("library philox_kernel<kUnitF32,0>", ms);
        CK(cudaMemcpy(ref.data(), out + (n - ref.size()), ref.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(got.data(), out, ref.size() * 4, cudaMemcpyDeviceToHost));
        ref.insert(ref.end(), got.begin(), got.end());  // [tail | head]
    }
#define TMA(BPT, SLOTS, HINT, WARPS, CTAS)                                                                      \
    {                                                                                                           \
        auto k = ktma<BPT, SLOTS, HINT, WARPS>;                                                                 \
        const int sm_bytes = WARPS * SLOTS * 32 * BPT * 16;                                                     \
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));                     \
        int o = 0;                                                                                              \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, WARPS * 32, sm_bytes));                         \
        const int ctas = CTAS ? (CTAS < o ? CTAS : o) : o;                                                      \
        CK(cudaMemset(out, 0, n * 4));                                                                          \
        float ms = timeit([&] { k<<<sms * ctas, WARPS * 32, sm_bytes>>>(out, k0, k1, pre, nblocks); });         \
        std::vector<float> h(1 << 20), t(1 << 20);                                                              \
        CK(cudaMemcpy(t.data(), out + (n - t.size()), t.size() * 4, cudaMemcpyDeviceToHost));                  \
        CK(cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost));                                    \
        t.insert(t.end(), h.begin(), h.end());                                                                  \
        const bool ok = t == ref;                                                                               \
        char nm[128];                                                                                           \
        snprintf(nm, 128, "tma bpt=%d slots=%d hint=%d warps=%d ctas/sm=%d smem=%dK %s", BPT, SLOTS, HINT, WARPS, \
                 ctas, sm_bytes / 1024, ok ? "ok" : "MISMATCH");                                                \
        report(nm, ms);                                                                                         \
    }
    TMA(4, 2, 0, 8, 0);
    TMA(4, 3, 0, 8, 0);
    TMA(4, 4, 0, 8, 0);
    TMA(4, 4, 1, 8, 0);
    TMA(2, 4, 0, 8, 0);
    TMA(2, 6, 0, 8, 0);
    TMA(8, 2, 0, 8, 0);
    TMA(8, 3, 0, 8, 0);
    TMA(4, 4, 0, 4, 0);
    TMA(4, 4, 0, 16, 0);
    TMA(4, 3, 0, 16, 0);
    TMA(2, 4, 0, 16, 0);
    TMA(4, 4, 0, 8, 2);
    TMA(4, 4, 0, 8, 4);
    return 0;
}
