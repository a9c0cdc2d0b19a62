// Store-pattern probe for the MRG32k3a kernel (no RNG arithmetic): does the
// per-thread contiguous-run layout (32 runs per warp, one 128-byte line per
// run per store instruction, runs `chunk` words apart) cost DRAM bandwidth
// against a warp-contiguous layout?  Same grid as mrg_kernel<kUniformF64> at
// n = 2^28 (886 x 128 threads, chunk 2368, 16-double tiles, 2 chains).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mrg_pattern tools/mrg_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int TW = 16;  // doubles per tile per lane (128 B)

__device__ __forceinline__ void stcs(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Layout A (current): lane run = [t*chunk, (t+1)*chunk), two halves; each
// instruction writes row 4i + lane>>3, 16-byte chunk lane&7.
__global__ void __launch_bounds__(128) runs_kernel(double* out, uint64_t n, uint64_t chunk, int spin) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t w0 = (t - lane) * chunk;
    if (w0 >= n) return;
    const uint64_t half = chunk / 2;
    uint32_t acc = lane;
    for (uint64_t off = 0; off < half; off += TW) {
        for (int s = 0; s < spin; ++s) acc = acc * 1664525u + 1013904223u;
        const uint32_t x = lane & 7, r0 = lane >> 3;
        for (int h = 0; h < 2; ++h) {
            double* p = out + w0 + h * half + off + r0 * chunk + x * 2;
            if (w0 + h * half + off + 31 * chunk + TW <= n) {
#pragma unroll
                for (int i = 0; i < 8; ++i) stcs(p + i * 4 * chunk, make_uint4(acc, i, h, x));
            }
        }
    }
}

// Layout B: the warp's region [w0, w0 + 32*chunk) is cut into 32-lane tile
// rows; tile row k covers words [w0 + k*32*TW, +32*TW) and lane L owns its
// TW-word tile (so one instruction round writes 4 KB contiguous).
__global__ void __launch_bounds__(128) rows_kernel(double* out, uint64_t n, uint64_t chunk, int spin) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t w0 = (t - lane) * chunk;
    if (w0 >= n) return;
    uint32_t acc = lane;
    const uint64_t rows = chunk / TW;  // 32*chunk words / (32*TW)
    for (uint64_t k = 0; k < rows; ++k) {
        for (int s = 0; s < spin; ++s) acc = acc * 1664525u + 1013904223u;
        double* base = out + w0 + k * 32 * TW;
        if (w0 + (k + 1) * 32 * TW <= n) {
#pragma unroll
            for (int i = 0; i < 8; ++i) stcs(base + (i * 32 + lane) * 2, make_uint4(acc, i, 0, lane));
        }
    }
}

// Layout C: segmented runs.  The warp region is processed in rounds of
// 32*seg words; in each round lane L owns the contiguous segment
// [round*32*seg + L*seg, +seg) (a per-lane jump of 31*seg words between
// rounds in the real kernel).  seg = TW is layout B; seg = chunk is layout A.
__global__ void __launch_bounds__(128) segs_kernel(double* out, uint64_t n, uint64_t chunk, uint64_t seg, int spin) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t w0 = (t - lane) * chunk;
    if (w0 >= n) return;
    uint32_t acc = lane;
    const uint32_t x = lane & 7, r0 = lane >> 3;
    for (uint64_t rb = 0; rb < 32 * chunk; rb += 32 * seg) {
        for (uint64_t off = 0; off < seg; off += TW) {
            for (int s = 0; s < spin; ++s) acc = acc * 1664525u + 1013904223u;
            double* p = out + w0 + rb + off + r0 * seg + x * 2;
            if (w0 + rb + off + 31 * seg + TW <= n) {
#pragma unroll
                for (int i = 0; i < 8; ++i) stcs(p + i * 4 * seg, make_uint4(acc, i, 0, x));
            }
        }
    }
}

int main() {
    const uint64_t n = 1ull << 28;
    const uint64_t chunk = 2368;
    const uint64_t tact = (n + chunk - 1) / chunk;
    const unsigned blocks = (unsigned)((tact + 127) / 128);
    double* out;
    cudaMalloc(&out, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int spin : {0, 8, 32}) {
        for (int layout = 0; layout < 2; ++layout) {
            float best = 1e9, sum = 0;
            for (int r = 0; r < 23; ++r) {
                cudaEventRecord(a);
                if (layout == 0)
                    runs_kernel<<<blocks, 128>>>(out, n, chunk, spin);
                else
                    rows_kernel<<<blocks, 128>>>(out, n, chunk, spin);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) {
                    best = ms < best ? ms : best;
                    sum += ms;
                }
            }
            printf("%s spin %2d: best %.4f ms (%.0f GB/s) mean %.4f ms (%.0f GB/s)\n", layout ? "rows" : "runs", spin, best,
                   n * 8 / best / 1e6, sum / 20, n * 8 / (sum / 20) / 1e6);
        }
    }
    for (uint64_t seg : {16ull, 32ull, 64ull, 128ull, 256ull, 592ull, 1184ull, 2368ull}) {
        float best = 1e9, sum = 0;
        for (int r = 0; r < 23; ++r) {
            cudaEventRecord(a);
            segs_kernel<<<blocks, 128>>>(out, n, chunk, seg, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) {
                best = ms < best ? ms : best;
                sum += ms;
            }
        }
        printf("segs seg %4llu: best %.4f ms (%.0f GB/s) mean %.4f ms (%.0f GB/s)\n", (unsigned long long)seg, best,
               n * 8 / best / 1e6, sum / 20, n * 8 / (sum / 20) / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
