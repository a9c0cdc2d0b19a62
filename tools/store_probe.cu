// store_probe.cu -- write-only HBM ceilings of different store patterns on
// B200 (no generator work), to find which access pattern a generate kernel
// should use.  16 GiB buffer (far above L2), CUDA-event timed, best of 3
// batches of 5 launches after warm-up.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o store_probe store_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

enum { kCs = 0, kWb = 1 };

template <int SK>
__device__ __forceinline__ void st256(uint32_t* p, uint32_t v) {
    if constexpr (SK == kCs)
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
    else
        asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
}
template <int SK>
__device__ __forceinline__ void st128(uint32_t* p, uint32_t v) {
    if constexpr (SK == kCs)
        asm volatile("st.global.cs.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
    else
        asm volatile("st.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
}

// P1: library pattern -- persistent grid stride, a thread writes 64 B
// contiguous per pass as two 256-bit stores (each instruction: 32 x 32 B at
// a 64 B stride).
template <int SK>
__global__ void __launch_bounds__(256) p1(uint32_t* out, uint64_t units64) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < units64; g += stride) {
        st256<SK>(out + 16 * g, (uint32_t)g);
        st256<SK>(out + 16 * g + 8, (uint32_t)g);
    }
}

// P2: persistent, warp-contiguous: each 256-bit store instruction of a warp
// covers 1 KiB contiguous; a warp pass writes 2 KiB.
template <int SK, int U>
__global__ void __launch_bounds__(256) p2(uint32_t* out, uint64_t units64) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    // a warp pass = 32 * U 32-byte chunks
    const uint64_t nchunk = units64 * 2;
    for (uint64_t base = gw * 32 * U; base < nchunk; base += nw * 32 * U) {
#pragma unroll
        for (int j = 0; j < U; ++j) st256<SK>(out + 8 * (base + 32 * j + lane), (uint32_t)base);
    }
}

// P3: non-persistent, CTA-contiguous chunks: CTA b writes [b*C, (b+1)*C)
// with each instruction 8 KiB contiguous (256 thr x 32 B), grid = total / C.
template <int SK, int ITER>
__global__ void __launch_bounds__(256) p3(uint32_t* out) {
    uint32_t* base = out + (size_t)blockIdx.x * ITER * 256 * 8;
#pragma unroll 4
    for (int i = 0; i < ITER; ++i) st256<SK>(base + (size_t)(i * 256 + threadIdx.x) * 8, (uint32_t)i);
}

// P4: torch-like: 128-bit stores, 4 per thread, block-contiguous, huge grid.
template <int SK>
__global__ void __launch_bounds__(128) p4(uint32_t* out) {
    uint32_t* base = out + (size_t)blockIdx.x * 128 * 4 * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) st128<SK>(base + (size_t)(i * 128 + threadIdx.x) * 4, (uint32_t)i);
}

// P5: persistent, CTA-contiguous segments: CTA b owns a contiguous range and
// sweeps it; each instruction 8 KiB contiguous.
template <int SK>
__global__ void __launch_bounds__(256) p5(uint32_t* out, uint64_t chunks32) {
    const uint64_t per = (chunks32 + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = per * blockIdx.x;
    uint64_t hi = lo + per;
    if (hi > chunks32) hi = chunks32;
    for (uint64_t c = lo + threadIdx.x; c < hi; c += 256) st256<SK>(out + 8 * c, (uint32_t)c);
}

// P6: persistent grid stride, block-contiguous per pass: in each pass the
// CTA writes 256 x 64 B = 16 KiB contiguous (two instructions of 8 KiB each).
template <int SK>
__global__ void __launch_bounds__(256) p6(uint32_t* out, uint64_t units64) {
    const uint64_t cstride = (uint64_t)gridDim.x * 256;
    for (uint64_t b = (uint64_t)blockIdx.x * 256; b < units64; b += cstride) {
        uint32_t* p = out + 16 * b;
        st256<SK>(p + 8 * threadIdx.x, (uint32_t)b);
        st256<SK>(p + 8 * (256 + threadIdx.x), (uint32_t)b);
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
        for (int i = 0; i < 5; ++i) f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms / 5 < best) best = ms / 5;
    }
    CK(cudaGetLastError());
    return best;
}

int main() {
    const uint64_t bytes = 16ull << 30;
    uint32_t* out;
    CK(cudaMalloc(&out, bytes));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t units64 = bytes / 64, chunks32 = bytes / 32;
    auto rep = [&](const char* nm, float ms) {
        printf("%-52s %8.3f ms  %8.1f GB/s\n", nm, ms, bytes / ms / 1e6);
    };
    char nm[128];
    rep("cudaMemset", timeit([&] { cudaMemset(out, 1, bytes); }));
    for (int occ : {2, 4, 5, 6, 8}) {
        snprintf(nm, sizeof nm, "P1 lib pattern .cs occ=%d", occ);
        rep(nm, timeit([&] { p1<kCs><<<sms * occ, 256>>>(out, units64); }));
        snprintf(nm, sizeof nm, "P1 lib pattern .wb occ=%d", occ);
        rep(nm, timeit([&] { p1<kWb><<<sms * occ, 256>>>(out, units64); }));
        snprintf(nm, sizeof nm, "P2 warp-contig U=2 .cs occ=%d", occ);
        rep(nm, timeit([&] { p2<kCs, 2><<<sms * occ, 256>>>(out, units64); }));
        snprintf(nm, sizeof nm, "P2 warp-contig U=4 .cs occ=%d", occ);
        rep(nm, timeit([&] { p2<kCs, 4><<<sms * occ, 256>>>(out, units64); }));
        snprintf(nm, sizeof nm, "P5 cta-segment .cs occ=%d", occ);
        rep(nm, timeit([&] { p5<kCs><<<sms * occ, 256>>>(out, chunks32); }));
        snprintf(nm, sizeof nm, "P6 cta-contig pass .cs occ=%d", occ);
        rep(nm, timeit([&] { p6<kCs><<<sms * occ, 256>>>(out, units64); }));
        snprintf(nm, sizeof nm, "P6 cta-contig pass .wb occ=%d", occ);
        rep(nm, timeit([&] { p6<kWb><<<sms * occ, 256>>>(out, units64); }));
    }
    rep("P3 nonpersistent ITER=4 .cs", timeit([&] { p3<kCs, 4><<<(unsigned)(chunks32 / (4 * 256)), 256>>>(out); }));
    rep("P3 nonpersistent ITER=16 .cs", timeit([&] { p3<kCs, 16><<<(unsigned)(chunks32 / (16 * 256)), 256>>>(out); }));
    rep("P3 nonpersistent ITER=16 .wb", timeit([&] { p3<kWb, 16><<<(unsigned)(chunks32 / (16 * 256)), 256>>>(out); }));
    rep("P3 nonpersistent ITER=64 .cs", timeit([&] { p3<kCs, 64><<<(unsigned)(chunks32 / (64 * 256)), 256>>>(out); }));
    rep("P4 torch-like v4 x4 .wb", timeit([&] { p4<kWb><<<(unsigned)(bytes / (128 * 64)), 128>>>(out); }));
    rep("P4 torch-like v4 x4 .cs", timeit([&] { p4<kCs><<<(unsigned)(bytes / (128 * 64)), 128>>>(out); }));
    CK(cudaFree(out));
    return 0;
}
