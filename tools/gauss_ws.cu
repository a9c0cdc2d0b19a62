// gauss_ws.cu -- design study: warp-specialised fast fp32 gaussian (sm_100a).
//
// The library's fast gaussian kernel is issue-bound at ~65% issue-active:
// each warp alternates a Philox section (IMAD.WIDE on the FMA-heavy pipe)
// and a Box-Muller section (FP32 / XU / ALU), and dispatch stalls where the
// two meet.  Here a CTA holds PAIRS producer warps (Philox blocks into a
// double-buffered shared-memory ring) and PAIRS consumer warps (Box-Muller
// + 256-bit stores), one named barrier per pair and step, so every
// scheduler has warps of both kinds to pick from.  Same arithmetic as the
// library (xform4<kGaussF32Fast>), so outputs must be bit-identical; the
// run prints both timings and the comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I../paper_2109_01329_b200/csrc \
//        -o gauss_ws gauss_ws.cu -L../paper_2109_01329_b200 -lprng_b200 -Xlinker -rpath=$PWD/../paper_2109_01329_b200
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "philox.cuh"
#include "../../include/prng_b200.h"

using namespace prng;

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e_ = (x);                                                \
        if (e_ != cudaSuccess) {                                             \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

constexpr int kBpt = 4;

template <int PAIRS, int MINB>
__global__ void __launch_bounds__(64 * PAIRS, MINB) ws_gauss(const PhiloxBody a) {
    xform_prologue<kGaussF32Fast>(a.p);
    __shared__ uint4 ring[PAIRS][2][kBpt][32];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pair = w % PAIRS;
    const bool producer = w < (uint32_t)PAIRS;
    const uint32_t pid = blockIdx.x * PAIRS + pair, npairs = gridDim.x * PAIRS;
    const uint32_t gfull = a.ngroups;
    const uint32_t per_step = npairs * 32 * kBpt;
    const uint32_t nsteps = (gfull + per_step - 1) / per_step;
    float* body = static_cast<float*>(a.out);
    for (uint32_t k = 0; k < nsteps; ++k) {
        const uint32_t g0 = ((k * npairs + pid) * 32 + lane) * kBpt;
        const uint32_t slot = k & 1;
        if (producer) {
#pragma unroll
            for (int j = 0; j < kBpt; ++j) {
                U4 b{0, 0, 0, 0};
                if (g0 + j < gfull) b = philox_block_pre(a.k0, a.k1, a.c0 + g0 + j, a.pre);
                ring[pair][slot][j][lane] = make_uint4(b.x, b.y, b.z, b.w);
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(64) : "memory");
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(64) : "memory");
            float o[kBpt][4];
#pragma unroll
            for (int j = 0; j < kBpt; ++j) {
                const uint4 v = ring[pair][slot][j][lane];
                xform4<kGaussF32Fast>(U4{v.x, v.y, v.z, v.w}, a.p, o[j]);
            }
            float* d = body + (size_t)4 * g0;
            if (g0 + kBpt <= gfull) {
                st_group2(d, o[0], o[1]);
                st_group2(d + 8, o[2], o[3]);
            } else {
#pragma unroll
                for (int j = 0; j < kBpt; ++j)
                    if (g0 + j < gfull) st_group(d + 4 * j, o[j]);
            }
        }
    }
}

template <int PAIRS, int MINB>
float run_ws(float* out, uint64_t n, int ctas_per_sm, int sms) {
    PhiloxBody a{};
    a.k0 = 777;
    a.k1 = 0;
    a.c0 = a.c1 = a.c2 = a.c3 = 0;
    a.ngroups = (uint32_t)(n / 4);
    a.pre = philox_pre(a.k0, a.k1, 0, 0, 0);
    a.out = out;
    a.p.scale_f = 1.0f;
    a.p.off_f = 0.0f;
    a.p.scale_d = 1.0;
    a.p.off_d = 0.0;
    const int grid = sms * ctas_per_sm;
    for (int i = 0; i < 3; ++i) ws_gauss<PAIRS, MINB><<<grid, 64 * PAIRS>>>(a);
    CK(cudaGetLastError());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) ws_gauss<PAIRS, MINB><<<grid, 64 * PAIRS>>>(a);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
}

float run_lib(float* out, uint64_t n) {
    const uint32_t ctr[4] = {0, 0, 0, 0};
    for (int i = 0; i < 3; ++i) prng_philox4x32x10_gaussian_f32(777, 0, ctr, 0, n, 0.0, 1.0, 0, out, nullptr);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) prng_philox4x32x10_gaussian_f32(777, 0, ctr, 0, n, 0.0, 1.0, 0, out, nullptr);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
}

__global__ void cmp_kernel(const uint32_t* a, const uint32_t* b, uint64_t n, unsigned long long* bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (a[i] != b[i]) atomicAdd(bad, 1ull);
}

bool cudaMemcmp_dummy(const float* a, const float* b, uint64_t n) {
    unsigned long long* d;
    CK(cudaMalloc(&d, 8));
    CK(cudaMemset(d, 0, 8));
    cmp_kernel<<<1184, 256>>>(reinterpret_cast<const uint32_t*>(a), reinterpret_cast<const uint32_t*>(b), n, d);
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return h == 0;
}

template <int PAIRS, int MINB>
void variant(const char* name, float* ref, float* out, uint64_t n, int sms, int ctas) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ws_gauss<PAIRS, MINB>, 64 * PAIRS, 0));
    if (ctas > occ) ctas = occ;
    CK(cudaMemset(out, 0, n * 4));
    const float ms = run_ws<PAIRS, MINB>(out, n, ctas, sms);
    const bool same = cudaMemcmp_dummy(ref, out, n);
    printf("%-28s occ=%d ctas/SM=%d  %.4f ms  %7.1f Gs/s  %s\n", name, occ, ctas, ms, n / ms / 1e6,
           same ? "bit-identical" : "DIFFERS");
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t n = 1ull << 30;
    float *ref, *out;
    CK(cudaMalloc(&ref, n * 4));
    CK(cudaMalloc(&out, n * 4));
    const float lms = run_lib(ref, n);
    printf("%-28s                %.4f ms  %7.1f Gs/s\n", "library fast gaussian", lms, n / lms / 1e6);
    variant<4, 1>("ws 4 pairs", ref, out, n, sms, 8);
    variant<4, 2>("ws 4 pairs minb2", ref, out, n, sms, 8);
    variant<2, 1>("ws 2 pairs", ref, out, n, sms, 16);
    variant<2, 4>("ws 2 pairs minb4", ref, out, n, sms, 16);
    return 0;
}
