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
// dependency chains.  Each 128-byte tile of both halves is transposed
// through an XOR-swizzled shared-memory stage (16-byte chunks) so the warp
// writes four runs' whole 128-byte lines per 128-bit store instruction.
#pragma once

#include "common.cuh"

namespace prng {

constexpr int kMrgMaxBits = 32;
constexpr int kMrgThreads = 128;
#ifndef PRNG_MRG_MINB
#define PRNG_MRG_MINB 6
#endif
constexpr int kMrgMinBlocks = PRNG_MRG_MINB;
#ifndef PRNG_MRG_CHAINS
#define PRNG_MRG_CHAINS 2
#endif
constexpr int kMrgChains = PRNG_MRG_CHAINS;  // interleaved recurrences per thread (1 or 2)

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

template <typename T> struct MrgTile { static constexpr int kWords = 32; };
template <> struct MrgTile<double> { static constexpr int kWords = 16; };

// Shared-memory stage of one warp: 32 rows (one per lane's run) of 8
// 16-byte chunks, chunk c of row r stored at physical chunk c ^ (r & 7)
// (XOR swizzle: the per-lane 128-bit writes and the row-wise 128-bit reads
// are both bank-conflict free within each 8-lane phase).
template <typename T>
__device__ __forceinline__ uint4 pack16(const T* v) {
    if constexpr (sizeof(T) == 4) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(v);
        return make_uint4(u[0], u[1], u[2], u[3]);
    } else {
        return make_uint4((uint32_t)__double2loint(v[0]), (uint32_t)__double2hiint(v[0]),
                          (uint32_t)__double2loint(v[1]), (uint32_t)__double2hiint(v[1]));
    }
}

__device__ __forceinline__ void stage_put(uint4* st, uint32_t lane, int c, uint4 v) {
    st[lane * 8 + (c ^ (lane & 7))] = v;
}

#ifndef PRNG_MRG_ST
#define PRNG_MRG_ST 0
#endif
__device__ __forceinline__ void st_global_cs_v4(void* p, uint4 v) {
#if PRNG_MRG_ST == 0
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
#elif PRNG_MRG_ST == 1
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
#else
    asm volatile("st.global.L1::no_allocate.L2::evict_last.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
#endif
}

// Write one staged tile (row j = run j, starting at run0 + j*chunk).  Each
// instruction moves four runs' 128-byte lines: lane L handles row
// 4i + (L >> 3), chunk L & 7.  The common case (tile entirely inside the
// request, 16-byte aligned output) is a straight-line block of 8 LDS.128 +
// 8 STG.128 with one 64-bit stride add each; the predicated element path
// only runs for the request's last tiles.
template <typename T>
__device__ __forceinline__ void mrg_store_tile(const uint4* st, T* __restrict__ run0, uint64_t chunk, uint32_t lane,
                                               uint64_t first_elem, uint64_t n, bool vec_ok) {
    constexpr int CE = 16 / sizeof(T);
    constexpr int TW = 8 * CE;
    const uint32_t x = lane & 7;
    const uint32_t r0 = lane >> 3;
    T* p = run0 + r0 * chunk + x * CE;
    const uint64_t stride = 4 * chunk;
    if (vec_ok && first_elem + 31 * chunk + TW <= n) {  // warp-uniform
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t j = 4 * i + r0;
            st_global_cs_v4(p + i * stride, st[j * 8 + (x ^ (j & 7))]);
        }
        return;
    }
    uint64_t e = first_elem + r0 * chunk + x * CE;
    for (int i = 0; i < 8; ++i, p += stride, e += stride) {
        const uint32_t j = 4 * i + r0;
        const uint4 v = st[j * 8 + (x ^ (j & 7))];
        const T* vv = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int q = 0; q < CE; ++q)
            if (e + q < n) p[q] = vv[q];
    }
}

template <int X>
__global__ void __launch_bounds__(kMrgThreads, kMrgMinBlocks) mrg_kernel(const MrgLaunch a) {
    using T = typename XformTraits<X>::T;
    constexpr int TW = MrgTile<T>::kWords;
    constexpr int WARPS = kMrgThreads / 32;
    __shared__ uint4 stage[kMrgChains][WARPS][32 * 8];
    __shared__ uint32_t sj1[kMrgMaxBits * 9], sj2[kMrgMaxBits * 9];

    for (uint32_t i = threadIdx.x; i < a.nbits * 9; i += blockDim.x) {
        sj1[i] = a.j1[i / 9][i % 9];
        sj2[i] = a.j2[i / 9][i % 9];
    }
    xform_prologue<X, kMrgTabLog2>();
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
    MrgStateF64 sa{mrg_sym(x10, kMrgM1), mrg_sym(x11, kMrgM1), mrg_sym(x12, kMrgM1),
                   mrg_sym(x20, kMrgM2), mrg_sym(x21, kMrgM2), mrg_sym(x22, kMrgM2)};
    MrgStateF64 sb = sa;
    if constexpr (kMrgChains == 2) {
        mat3_apply<kMrgC1>(a.h1, x10, x11, x12);
        mat3_apply<kMrgC2>(a.h2, x20, x21, x22);
        sb = MrgStateF64{mrg_sym(x10, kMrgM1), mrg_sym(x11, kMrgM1), mrg_sym(x12, kMrgM1),
                         mrg_sym(x20, kMrgM2), mrg_sym(x21, kMrgM2), mrg_sym(x22, kMrgM2)};
    }

    const uint64_t half = a.chunk / kMrgChains;
    T* __restrict__ out = static_cast<T*>(a.out);
    uint4* sta = stage[0][warp];
    uint4* stb = stage[kMrgChains - 1][warp];
    const bool vec_ok = ((uintptr_t)out & 15u) == 0;
    const uint64_t warp_elem0 = t_warp0 * a.chunk;
    constexpr int CE = 16 / sizeof(T);  // elements per 16-byte chunk
    for (uint64_t off = 0; off < half; off += TW) {
        if (warp_elem0 + off >= a.n) break;  // warp-uniform
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            T oa[CE], ob[CE];
            if constexpr (XformTraits<X>::kPair) {
#pragma unroll
                for (int k = 0; k < CE; k += 2) {
                    const uint32_t a0 = mrg_step_f64(sa);
                    const uint32_t a1 = mrg_step_f64(sa);
                    xform2k<X, kMrgTabLog2>(a0, a1, a.p, oa[k], oa[k + 1]);
                    if constexpr (kMrgChains == 2) {
                        const uint32_t b0 = mrg_step_f64(sb);
                        const uint32_t b1 = mrg_step_f64(sb);
                        xform2k<X, kMrgTabLog2>(b0, b1, a.p, ob[k], ob[k + 1]);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < CE; ++k) {
                    oa[k] = xform1<X>(mrg_step_f64(sa), a.p);
                    if constexpr (kMrgChains == 2) ob[k] = xform1<X>(mrg_step_f64(sb), a.p);
                }
            }
            stage_put(sta, lane, c, pack16<T>(oa));
            if constexpr (kMrgChains == 2) stage_put(stb, lane, c, pack16<T>(ob));
        }
        __syncwarp();
        mrg_store_tile<T>(sta, out + warp_elem0 + off, a.chunk, lane, warp_elem0 + off, a.n, vec_ok);
        if constexpr (kMrgChains == 2)
            mrg_store_tile<T>(stb, out + warp_elem0 + half + off, a.chunk, lane, warp_elem0 + half + off, a.n,
                              vec_ok);
        __syncwarp();
    }
}

}  // namespace prng
