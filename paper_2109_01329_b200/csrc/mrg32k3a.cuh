// mrg32k3a.cuh -- MRG32k3a generate+transform kernel with per-thread
// jump-ahead (sm_100a).
//
// Replaces the strictly sequential reference loop _core.pyx:74-102
// (mrg_fill), which the reference cannot split (rngburn.py:123,
// engine.py:201-202).  Thread t owns words [t*chunk, (t+1)*chunk) of the
// request.  Its start state is A^(t*chunk) s0, assembled from the host-built
// table J_b = A^(chunk * 2^b) mod m (b < nbits), staged in shared memory:
// one 3x3 mod-m mat-vec per set bit of t.  The thread then runs the
// recurrence for its chunk in TILE-word tiles; each tile is transposed
// through shared memory so the warp stores whole 128-byte lines: lane x of
// store step j writes element x of lane j's tile (4-byte outputs) or
// element x&15 of lane 2j+(x>>4)'s tile (8-byte outputs).
#pragma once

#include "common.cuh"

namespace prng {

constexpr int kMrgMaxBits = 32;
constexpr int kMrgThreads = 128;

struct MrgLaunch {
    uint32_t s1[3], s2[3];
    uint64_t n;
    uint64_t chunk;   // words per thread (multiple of the tile)
    uint32_t nbits;
    uint32_t j1[kMrgMaxBits][9];
    uint32_t j2[kMrgMaxBits][9];
    void* out;
    XformParams p;
};

template <typename T> struct MrgTile { static constexpr int kWords = 32, kPad = 1; };
template <> struct MrgTile<double> { static constexpr int kWords = 16, kPad = 1; };

template <int X>
__global__ void __launch_bounds__(kMrgThreads) mrg_kernel(const MrgLaunch a) {
    using T = typename XformTraits<X>::T;
    constexpr int TW = MrgTile<T>::kWords;
    constexpr int ROW = TW + MrgTile<T>::kPad;
    constexpr int WARPS = kMrgThreads / 32;
    __shared__ T stage[WARPS][32 * ROW];
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
    MrgStateMixed s{x10, x11, x12, (double)x20, (double)x21, (double)x22};

    T* __restrict__ out = static_cast<T*>(a.out);
    T* st = stage[warp];
    for (uint64_t off = 0; off < a.chunk; off += TW) {
        if (t_warp0 * a.chunk + off >= a.n) break;  // warp-uniform
        if constexpr (XformTraits<X>::kPair) {
#pragma unroll
            for (int k = 0; k < TW; k += 2) {
                const uint32_t w0 = mrg_step_mixed(s);
                const uint32_t w1 = mrg_step_mixed(s);
                T o0, o1;
                xform2<X>(w0, w1, a.p, o0, o1);
                st[lane * ROW + k] = o0;
                st[lane * ROW + k + 1] = o1;
            }
        } else {
#pragma unroll
            for (int k = 0; k < TW; ++k) st[lane * ROW + k] = xform1<X>(mrg_step_mixed(s), a.p);
        }
        __syncwarp();
        if constexpr (TW == 32) {
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const uint64_t e = (t_warp0 + j) * a.chunk + off + lane;
                if (e < a.n) out[e] = st[j * ROW + lane];
            }
        } else {
            const int x = lane & 15;
#pragma unroll 4
            for (int j2 = 0; j2 < 16; ++j2) {
                const int j = 2 * j2 + (lane >> 4);
                const uint64_t e = (t_warp0 + j) * a.chunk + off + x;
                if (e < a.n) out[e] = st[j * ROW + x];
            }
        }
        __syncwarp();
    }
}

}  // namespace prng
