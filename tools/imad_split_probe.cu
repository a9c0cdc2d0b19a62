// Probe: Philox-round throughput with IMAD.WIDE.U32 (fused) versus IMAD.HI.U32 +
// IMAD (lo) against a register copy of the constant (unfusable) -- do the two
// halves use different pipes on sm_100a?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/imad_split_probe tools/imad_split_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t* o, uint32_t a0, uint32_t m0r, uint32_t m1r, int n) {
    uint32_t x[4], y[4], z[4], w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        x[j] = threadIdx.x + a0 + j;
        y[j] = x[j] * 3u;
        z[j] = x[j] ^ 5u;
        w[j] = x[j] + 7u;
    }
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t lo0, hi0, lo1, hi1;
            if (MODE == 0) {
                const uint64_t p0 = (uint64_t)0xD2511F53u * x[j], p1 = (uint64_t)0xCD9E8D57u * z[j];
                lo0 = (uint32_t)p0; hi0 = (uint32_t)(p0 >> 32); lo1 = (uint32_t)p1; hi1 = (uint32_t)(p1 >> 32);
            } else {
                hi0 = __umulhi(x[j], 0xD2511F53u);
                hi1 = __umulhi(z[j], 0xCD9E8D57u);
                lo0 = x[j] * m0r;  // register copy: ptxas cannot fuse with the hi half
                lo1 = z[j] * m1r;
            }
            const uint32_t nx = hi1 ^ y[j] ^ 0x9E3779B9u, nz = hi0 ^ w[j] ^ 0xBB67AE85u;
            y[j] = lo1; w[j] = lo0; x[j] = nx; z[j] = nz;
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) r ^= x[j] ^ y[j] ^ z[j] ^ w[j];
    o[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    const int blocks = 148 * 8, n = 4096;
    uint32_t* o;
    cudaMalloc(&o, blocks * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, 256>>>(o, r, 0xD2511F53u, 0xCD9E8D57u, n);
            else k<1><<<blocks, 256>>>(o, r, 0xD2511F53u, 0xCD9E8D57u, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r) best = ms < best ? ms : best;
        }
        const double rounds = (double)blocks * 256 * n * 4;
        printf("mode %d (%s): %.3f ms, %.1f G rounds/s\n", mode, mode ? "IMAD.HI + IMAD(reg)" : "IMAD.WIDE", best,
               rounds / best / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
