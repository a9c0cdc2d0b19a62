// mrg32k3a.cuh -- MRG32k3a generate+transform kernel with per-thread
// jump-ahead (sm_100a).
//
// Replaces the strictly sequential reference loop _core.pyx:74-102
// (mrg_fill), which the reference cannot split (rngburn.py:123,
// engine.py:201-202).  Thread t owns words [t*chunk, (t+1)*chunk) of the
// request.  Its start state is A^(t*chunk) s0, assembled from the host-built
// table J_b = A^(chunk * 2^b) mod m (b < nbits), staged in shared memory:
// one 3x3 mod-m mat-vec per set bit of t.  The chunk is run as two halves
// (second start = A^(chunk/2) x first start) whose recurrences are
// interleaved step by step, so every thread carries two independent
// dependency chains.  Each TILE-word tile of both halves is transposed
// through shared memory so the warp stores whole 128-byte lines: store step
// j writes element `lane` of run j (4-byte outputs) or element lane&15 of
// run 2j+(lane>>4) (8-byte outputs), with a running pointer per lane.
#pragma once

#include "common.cuh"

namespace prng {

constexpr int kMrgMaxBits = 32;
constexpr int kMrgThreads = 128;

struct MrgLaunch {
    uint32_t s1[3], s2[3];
    uint64_t n;
    uint64_t chunk;  // words per thread (multiple of 2 tiles)
    uint32_t nbits;
    uint32_t j1[kMrgMaxBits][9];
    uint32_t j2[kMrgMaxBits][9];
    uint32_t h1[9], h2[9];  // A^(chunk/2)
    void* out;
    XformParams p;
};

template <typename T> struct MrgTile { static constexpr int kWords = 32, kPad = 1; };
template <> struct MrgTile<double> { static constexpr int kWords = 16, kPad = 1; };

// Write one staged tile (32 runs of TW elements, run j = lane j's tile) to
// out: run j starts at run0 + j*chunk.
template <typename T, int TW, int ROW>
__device__ __forceinline__ void mrg_store_tile(const T* st, T* __restrict__ run0, uint64_t chunk, uint32_t lane,
                                               uint64_t first_elem, uint64_t n) {
    const bool full = first_elem + 31 * chunk + TW <= n;  // warp-uniform
    if constexpr (TW == 32) {
        T* p = run0 + lane;
        uint64_t e = first_elem + lane;
#pragma unroll 4
        for (int j = 0; j < 32; ++j, p += chunk, e += chunk)
            if (full || e < n) *p = st[j * ROW + lane];
    } else {
        const uint32_t x = lane & 15;
        const uint32_t r = lane >> 4;
        T* p = run0 + r * chunk + x;
        uint64_t e = first_elem + r * chunk + x;
#pragma unroll 4
        for (int j2 = 0; j2 < 16; ++j2, p += 2 * chunk, e += 2 * chunk)
            if (full || e < n) *p = st[(2 * j2 + r) * ROW + x];
    }
}

template <int X>
__global__ void __launch_bounds__(kMrgThreads) mrg_kernel(const MrgLaunch a) {
    using T = typename XformTraits<X>::T;
    constexpr int TW = MrgTile<T>::kWords;
    constexpr int ROW = TW + MrgTile<T>::kPad;
    constexpr int WARPS = kMrgThreads / 32;
    __shared__ T stage[2][WARPS][32 * ROW];
    __shared__ uint32_t sj1[kMrgMaxBits * 9], sj2[kMrgMaxBits * 9];

    for (uint32_t i = threadIdx.x; i < a.nbits * 9; i += blockDim.x) {
        sj1[i] = a.j1[i / 9][i % 9];
        sj2[i] = a.j2[i / 9][i % 9];
    }
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t t_warp0 = t - lane;
    if (t_warp0 * a.chunk >= a.n) return;  // whole warp idle (warp-uniform)

    uint32_t x10 = a.s1[0], x11 = a.s1[1], x12 = a.s1[2], x20 = a.s2[0], x21 = a.s2[1], x22 = a.s2[2];
    for (uint32_t b = 0; b < a.nbits; ++b) {
        if ((t >> b) & 1) {
            mat3_apply<kMrgC1>(&sj1[9 * b], x10, x11, x12);
            mat3_apply<kMrgC2>(&sj2[9 * b], x20, x21, x22);
        }
    }
    MrgStateMixed sa{x10, x11, x12, (double)x20, (double)x21, (double)x22};
    mat3_apply<kMrgC1>(a.h1, x10, x11, x12);
    mat3_apply<kMrgC2>(a.h2, x20, x21, x22);
    MrgStateMixed sb{x10, x11, x12, (double)x20, (double)x21, (double)x22};

    const uint64_t half = a.chunk >> 1;
    T* __restrict__ out = static_cast<T*>(a.out);
    T* sta = stage[0][warp];
    T* stb = stage[1][warp];
    const uint64_t warp_elem0 = t_warp0 * a.chunk;
    for (uint64_t off = 0; off < half; off += TW) {
        if (warp_elem0 + off >= a.n) break;  // warp-uniform
        if constexpr (XformTraits<X>::kPair) {
#pragma unroll
            for (int k = 0; k < TW; k += 2) {
                const uint32_t a0 = mrg_step_mixed(sa);
                const uint32_t b0 = mrg_step_mixed(sb);
                const uint32_t a1 = mrg_step_mixed(sa);
                const uint32_t b1 = mrg_step_mixed(sb);
                T o0, o1;
                xform2<X>(a0, a1, a.p, o0, o1);
                sta[lane * ROW + k] = o0;
                sta[lane * ROW + k + 1] = o1;
                xform2<X>(b0, b1, a.p, o0, o1);
                stb[lane * ROW + k] = o0;
                stb[lane * ROW + k + 1] = o1;
            }
        } else {
#pragma unroll
            for (int k = 0; k < TW; ++k) {
                const uint32_t wa = mrg_step_mixed(sa);
                const uint32_t wb = mrg_step_mixed(sb);
                sta[lane * ROW + k] = xform1<X>(wa, a.p);
                stb[lane * ROW + k] = xform1<X>(wb, a.p);
            }
        }
        __syncwarp();
        mrg_store_tile<T, TW, ROW>(sta, out + warp_elem0 + off, a.chunk, lane, warp_elem0 + off, a.n);
        mrg_store_tile<T, TW, ROW>(stb, out + warp_elem0 + half + off, a.chunk, lane, warp_elem0 + half + off,
                                   a.n);
        __syncwarp();
    }
}

}  // namespace prng
