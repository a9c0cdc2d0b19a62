// Probe: Philox-round throughput with IMAD.WIDE.U32 (fused) versus IMAD.HI.U32 +
// IMAD (lo) against a register copy of the constant (unfusable) -- do the two
// halves use different pipes on sm_100a?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/imad_split_probe tools/imad_split_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// x * M as (lo32, hi32) on the FP64 pipe: M = Mh 2^16 + Ml, two exact DFMAs on
// the magic double 2^52 + x (partial products < 2^48), stitched in integers.
__device__ __forceinline__ void mul_f64(uint32_t x, double mh, double ml, double mhm, double mlm, uint32_t& lo,
                                        uint32_t& hi) {
    const double xd = __hiloint2double(0x43300000, (int)x);                 // 2^52 + x
    const double a = __fma_rn(xd, ml, mlm);                                 // 2^52 + x Ml  (mlm = 2^52 - 2^52 Ml)
    const double b = __fma_rn(xd, mh, mhm);                                 // 2^52 + x Mh
    const uint32_t alo = (uint32_t)__double2loint(a), ahi = (uint32_t)__double2hiint(a) & 0xFFFFu;
    const uint32_t blo = (uint32_t)__double2loint(b), bhi = (uint32_t)__double2hiint(b);
    uint32_t l, h;
    const uint32_t bsh = __funnelshift_r(blo, bhi, 16);  // (x Mh) >> 16, low 32 bits
    asm("add.cc.u32 %0, %1, %2;" : "=r"(l) : "r"(alo), "r"(blo << 16));
    asm("addc.u32 %0, %1, %2;" : "=r"(h) : "r"(ahi), "r"(bsh));
    lo = l;
    hi = h;
}

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
            if (MODE == 0 || (MODE == 2 && j >= 1) || (MODE == 3 && j >= 2)) {
                const uint64_t p0 = (uint64_t)0xD2511F53u * x[j], p1 = (uint64_t)0xCD9E8D57u * z[j];
                lo0 = (uint32_t)p0; hi0 = (uint32_t)(p0 >> 32); lo1 = (uint32_t)p1; hi1 = (uint32_t)(p1 >> 32);
            } else if (MODE == 2 || MODE == 3) {
                const uint64_t p0 = (uint64_t)0xD2511F53u * x[j];
                lo0 = (uint32_t)p0; hi0 = (uint32_t)(p0 >> 32);
                // 0xCD9E8D57 = 0xCD9E * 2^16 + 0x8D57
                mul_f64(z[j], 52638.0, 36183.0, 4503599627370496.0 - 52638.0 * 4503599627370496.0,
                        4503599627370496.0 - 36183.0 * 4503599627370496.0, lo1, hi1);
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

__global__ void check(uint32_t* bad) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    x = x * 2654435761u + 12345u;
    uint32_t lo, hi;
    mul_f64(x, 52638.0, 36183.0, 4503599627370496.0 - 52638.0 * 4503599627370496.0,
            4503599627370496.0 - 36183.0 * 4503599627370496.0, lo, hi);
    const uint64_t p = (uint64_t)0xCD9E8D57u * x;
    if (lo != (uint32_t)p || hi != (uint32_t)(p >> 32)) atomicAdd(bad, 1u);
}

int main() {
    uint32_t* bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    check<<<1 << 16, 256>>>(bad);
    uint32_t hb = 0;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("mul_f64 mismatches over 2^24 inputs: %u\n", hb);
    const int blocks = 148 * 8, n = 4096;
    uint32_t* o;
    cudaMalloc(&o, blocks * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, 256>>>(o, r, 0xD2511F53u, 0xCD9E8D57u, n);
            else if (mode == 1) k<1><<<blocks, 256>>>(o, r, 0xD2511F53u, 0xCD9E8D57u, n);
            else if (mode == 2) k<2><<<blocks, 256>>>(o, r, 0xD2511F53u, 0xCD9E8D57u, n);
            else k<3><<<blocks, 256>>>(o, r, 0xD2511F53u, 0xCD9E8D57u, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r) best = ms < best ? ms : best;
        }
        const double rounds = (double)blocks * 256 * n * 4;
        const char* names[] = {"IMAD.WIDE", "IMAD.HI + IMAD(reg)", "1 of 8 multiplies on FP64", "2 of 8 multiplies on FP64"};
        printf("mode %d (%s): %.3f ms, %.1f G rounds/s\n", mode, names[mode], best, rounds / best / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
