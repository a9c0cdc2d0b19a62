// philox_variants.cu -- microbenchmark of Philox4x32-10 kernel formulations on sm_100a.
//
// Standalone (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pv philox_variants.cu).
// Each variant writes n = 2^30 unit fp32 samples (4 GiB, > L2) and checks its
// output against variant A.  Prints ms and GB/s per variant.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstring>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                   \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;

struct U4 {
    uint32_t x, y, z, w;
};

template <int SPLIT>
__device__ __forceinline__ U4 philox(uint32_t k0, uint32_t k1, U4 c) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        uint32_t hi0, lo0, hi1, lo1;
        if (SPLIT == 2) {
            asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi0) : "r"(c.x), "n"(M0));
            asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo0) : "r"(c.x), "n"(M0));
            asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi1) : "r"(c.z), "n"(M1));
            asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo1) : "r"(c.z), "n"(M1));
        } else if (SPLIT == 1) {
            hi0 = __umulhi(M0, c.x);
            lo0 = M0 * c.x;
            hi1 = __umulhi(M1, c.z);
            lo1 = M1 * c.z;
        } else {
            const uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
            hi0 = (uint32_t)(p0 >> 32);
            lo0 = (uint32_t)p0;
            hi1 = (uint32_t)(p1 >> 32);
            lo1 = (uint32_t)p1;
        }
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += W0;
        k1 += W1;
    }
    return c;
}

__device__ __forceinline__ float unit(uint32_t w) { return __fmul_rn((float)(w >> 8), 5.9604644775390625e-08f); }

__device__ __forceinline__ void st8(float* p, const float* a) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]),
                 "f"(a[3]), "f"(a[4]), "f"(a[5]), "f"(a[6]), "f"(a[7])
                 : "memory");
}
__device__ __forceinline__ void st4(float* p, const float* a) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]), "f"(a[3])
                 : "memory");
}

// A: 64-bit counter add per block (current library kernel shape), 2 blocks/thread, v8 store.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) kA(float* out, uint32_t k0, uint32_t k1, uint64_t clo, uint64_t chi,
                                                 uint64_t nunits) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint64_t l = clo + 2 * u + j;
            const uint64_t h = chi + (l < clo);
            U4 w = philox<0>(k0, k1, U4{(uint32_t)l, (uint32_t)(l >> 32), (uint32_t)h, (uint32_t)(h >> 32)});
            o[4 * j] = unit(w.x);
            o[4 * j + 1] = unit(w.y);
            o[4 * j + 2] = unit(w.z);
            o[4 * j + 3] = unit(w.w);
        }
        st8(out + 8 * u, o);
    }
}

// B: upper counter words uniform (host splits launches at 2^32-block
// boundaries), 32-bit block index; BPT blocks per thread; SPLIT = mul.hi + mul.lo.
template <int SPLIT, int BPT, int MINB>
__global__ void __launch_bounds__(256, MINB) kB(float* out, uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1,
                                                 uint32_t c2, uint32_t c3, uint32_t nunits) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        float o[4 * BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            U4 w = philox<SPLIT>(k0, k1, U4{c0 + BPT * u + j, c1, c2, c3});
            o[4 * j] = unit(w.x);
            o[4 * j + 1] = unit(w.y);
            o[4 * j + 2] = unit(w.z);
            o[4 * j + 3] = unit(w.w);
        }
        float* p = out + (size_t)(4 * BPT) * u;
        if (BPT == 1) st4(p, o);
        if (BPT == 2) st8(p, o);
        if (BPT == 4) {
            st8(p, o);
            st8(p + 8, o + 8);
        }
    }
}

// C: B with the counter words as (c1, c2, c3) uniform and
// a block-contiguous layout: each warp covers 32*BPT consecutive blocks per pass.
template <int BPT, int MINB>
__global__ void __launch_bounds__(256, MINB) kC(float* out, uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1,
                                                 uint32_t c2, uint32_t c3, uint32_t nblk) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t base = gw * 32 * BPT; base < nblk; base += nw * 32 * BPT) {
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const uint32_t b = base + j * 32 + lane;
            U4 w = philox<0>(k0, k1, U4{c0 + b, c1, c2, c3});
            float o[4] = {unit(w.x), unit(w.y), unit(w.z), unit(w.w)};
            if (b < nblk) st4(out + 4 * (size_t)b, o);
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
int occ(K k) {
    int o = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 256, 0));
    return o;
}

int main() {
    const uint64_t n = 1ull << 30;
    const uint64_t nblk = n / 4;
    float *out, *ref;
    CK(cudaMalloc(&out, n * 4));
    CK(cudaMalloc(&ref, n * 4));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t k0 = 777, k1 = 0;
    std::vector<float> h(1 << 20), hr(1 << 20);
    auto check = [&](const char* name, float ms) {
        CK(cudaMemcpy(h.data(), out + (n - (1 << 20)), 4 << 20, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hr.data(), ref + (n - (1 << 20)), 4 << 20, cudaMemcpyDeviceToHost));
        bool ok = memcmp(h.data(), hr.data(), 4 << 20) == 0;
        printf("%-34s %8.3f ms  %8.1f GB/s  %7.1f Gs/s %s\n", name, ms, n * 4 / ms / 1e6, n / ms / 1e6,
               ok ? "ok" : "MISMATCH");
    };
    {
        auto k = kA<1>;
        int g = sms * occ(k);
        kA<1><<<g, 256>>>(ref, k0, k1, 0, 0, nblk / 2);
        CK(cudaDeviceSynchronize());
        float ms = timeit([&] { kA<1><<<g, 256>>>(out, k0, k1, 0, 0, nblk / 2); });
        check("A: 64b ctr, 2 blk/thr (lib shape)", ms);
    }
#define RUNB(SPLIT, BPT, MINB)                                                                          \
    {                                                                                                   \
        auto k = kB<SPLIT, BPT, MINB>;                                                                  \
        int g = sms * occ(k);                                                                           \
        float ms = timeit([&] { kB<SPLIT, BPT, MINB><<<g, 256>>>(out, k0, k1, 0, 0, 0, 0, nblk / BPT); }); \
        char nm[64];                                                                                    \
        snprintf(nm, 64, "B: split=%d bpt=%d minb=%d occ=%d", SPLIT, BPT, MINB, occ(k));               \
        check(nm, ms);                                                                                  \
    }
    RUNB(false, 1, 1);
    RUNB(false, 2, 1);
    RUNB(false, 4, 1);
    RUNB(true, 1, 1);
    RUNB(true, 2, 1);
    RUNB(false, 2, 6);
    RUNB(false, 2, 8);
    RUNB(true, 2, 8);
    RUNB(false, 1, 8);
    RUNB(2, 1, 1);
    RUNB(2, 2, 1);
    RUNB(2, 2, 8);
#define RUNC(BPT, MINB)                                                                          \
    {                                                                                            \
        auto k = kC<BPT, MINB>;                                                                  \
        int g = sms * occ(k);                                                                    \
        float ms = timeit([&] { kC<BPT, MINB><<<g, 256>>>(out, k0, k1, 0, 0, 0, 0, nblk); });    \
        char nm[64];                                                                             \
        snprintf(nm, 64, "C: warp-contig bpt=%d minb=%d occ=%d", BPT, MINB, occ(k));            \
        check(nm, ms);                                                                           \
    }
    RUNC(1, 1);
    RUNC(2, 1);
    RUNC(2, 8);
    {
        float ms = timeit([&] { CK(cudaMemsetAsync(out, 0, n * 4)); });
        printf("%-34s %8.3f ms  %8.1f GB/s\n", "cudaMemset", ms, n * 4 / ms / 1e6);
    }
    return 0;
}
