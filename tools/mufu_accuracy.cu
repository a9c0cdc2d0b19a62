// mufu_accuracy.cu -- exhaustive accuracy of the SFU approximations the fast
// Box-Muller could use, over the 24-bit input grid (all 2^24 points):
//   lg2.approx.f32(m 2^-24)        vs log2 in fp64  (absolute error)
//   sqrt.approx.f32(s), s = -2 ln(u1') (relative error)
//   sin/cos.approx.f32(2 pi k 2^-24 reduced to [-pi/4, pi/4]) (absolute error)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_accuracy mufu_accuracy.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ float lg2a(float x) { float y; asm("lg2.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ float sqa(float x) { float y; asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ float sina(float x) { float y; asm("sin.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ float cosa(float x) { float y; asm("cos.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__device__ unsigned long long g_max[8];

__device__ void upd(int i, double e) { atomicMax(&g_max[i], __double_as_longlong(e)); }

__global__ void k_all() {
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < (1u << 24); k += gridDim.x * blockDim.x) {
        const unsigned m = (1u << 24) - k;  // u1' = m 2^-24 in (0, 1]
        const float u = (float)m * 5.9604644775390625e-08f;
        const double l2 = log2((double)m) - 24.0;
        const double e_lg = fabs((double)lg2a(u) - l2);
        if (k >= (1u << 20)) upd(0, e_lg);       // u1' <= 1 - 2^-4
        else if (k >= (1u << 21) / 2) upd(1, e_lg);
        if (k >= (1u << 21)) upd(7, e_lg / fabs(l2));  // relative, u1' <= 1 - 2^-3
        const double s = -2.0 * log((double)m * 5.9604644775390625e-08);
        if (s > 0) upd(2, fabs((double)sqa((float)s) - sqrt((double)(float)s)) / sqrt((double)(float)s));
        // angle on the exact quadrant-reduced grid: theta = pi/4 * t, t in [-1, 1)
        const int ti = (int)((k + (1u << 21)) & 0x3FFFFFu) - (1 << 21);
        const float t = (float)ti * 4.76837158203125e-07f;
        const double th = 0.7853981633974483 * (double)ti * 4.76837158203125e-07;
        const float thf = (float)th;
        upd(3, fabs((double)sina(thf) - sin((double)thf)));
        upd(4, fabs((double)cosa(thf) - cos((double)thf)));
        const float full = 6.2831853f * (float)k * 5.9604644775390625e-08f;
        upd(5, fabs((double)sina(full) - sin((double)full)));
        upd(6, fabs((double)cosa(full) - cos((double)full)));
        (void)t;
    }
}

int main() {
    k_all<<<148 * 8, 256>>>();
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, g_max, sizeof h);
    const char* nm[8] = {"lg2.approx abs err, u1' <= 1-2^-4", "lg2.approx abs err, 1-2^-4 < u1' <= 1-2^-5",
                         "sqrt.approx rel err", "sin.approx abs err |x|<=pi/4", "cos.approx abs err |x|<=pi/4",
                         "sin.approx abs err [0,2pi)", "cos.approx abs err [0,2pi)",
                         "lg2.approx REL err, u1' <= 1-2^-3"};
    for (int i = 0; i < 8; ++i) {
        double d;
        memcpy(&d, &h[i], 8);
        printf("%-48s %.3e = 2^%.2f\n", nm[i], d, log2(d));
    }
    return 0;
}
