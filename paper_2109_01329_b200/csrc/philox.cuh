// philox.cuh -- fused Philox4x32-10 generate+transform kernels (sm_100a).
//
// Replaces the reference hot loop _core.pyx:42-71 (philox_fill) together with
// the passes layered on it: words_to_unit (distributions.py:83-87), the range
// transform (distributions.py:98-104 / rngburn.py:62-64, 94-100), Box-Muller
// (distributions.py:116-131) and the lognormal extension.  Each sample is
// written to HBM exactly once.
//
// Work decomposition.  A request is n elements starting at stream word `lane`
// of the block with 128-bit counter `ctr` (the reference's philox_fill(k0, k1,
// b0..b3, offset, n) arguments, engine.py:222-225).  Output element i consumes
// "virtual word" v = lane + i, i.e. lane v&3 of block ctr + (v>>2).  The
// output is split into
//   * a scalar head [0, i0) that brings out+i0 to a 32-byte boundary,
//   * a body of 4-element groups, group g holding virtual words
//     lane+i0+4g .. +3, stored with 128/256-bit streaming stores,
//   * a scalar tail.
// The host cuts the body into launches inside which the upper 96 counter bits
// are constant (a new launch at every 2^32-block boundary, i.e. every 2^34
// words): c1..c3 are then kernel-uniform, the per-block counter is one 32-bit
// add, and the first two Philox rounds partly fold into uniform registers.
// When (lane + i0) % 4 == 0 every group is exactly one Philox block
// (SHIFT = 0): a thread computes BPT adjacent blocks and issues 256-bit
// stores.  Otherwise (SHIFT = 1..3) a group straddles two blocks: lane t of a
// warp computes blocks 4t..4t+3 and takes block 4t+4 from lane t+1 by
// shuffle; each warp pass emits 126 groups from 128 blocks.
#pragma once

#include "common.cuh"

namespace prng {

constexpr int kPhiloxThreads = 256;

// Scalar (head / tail / fully generic) description of a request.
struct PhiloxScalar {
    uint32_t k0, k1;
    uint64_t ctr_lo, ctr_hi;  // counter of the block holding element 0
    uint32_t lane;            // virtual word of element 0 (0..3)
    uint64_t i0;              // head length
    uint64_t tail0;           // first tail element
    uint64_t n;               // total elements
};

// One body launch: `ngroups` groups whose first block has counter
// (c0, c1, c2, c3), with c0 + ngroups (+1 for SHIFT > 0) <= 2^32.
struct PhiloxBody {
    uint32_t k0, k1;
    uint32_t c0, c1, c2, c3;
    uint32_t ngroups;
    uint32_t mis;  // pair transforms at an odd-element output: body = 32-byte boundary - 1 element
    PhiloxPre pre;  // philox_pre(k0, k1, c1, c2, c3)
    void* out;  // address of group 0
    XformParams p;
    PhiloxScalar s;  // head/tail done by this launch when s.n != 0
};

// Element i computed on its own (head, tail and the fully generic path).
template <int X>
__device__ __forceinline__ typename XformTraits<X>::T philox_scalar(const PhiloxScalar& a, const XformParams& p,
                                                                    uint64_t i) {
    using T = typename XformTraits<X>::T;
    if constexpr (XformTraits<X>::kPair) {
        const uint64_t v0 = a.lane + 2 * (i >> 1);
        const U4 b = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, v0 >> 2));
        const uint32_t w0 = lane_of(b, (uint32_t)(v0 & 3));
        uint32_t w1;
        if ((v0 & 3) == 3) {
            w1 = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, (v0 >> 2) + 1)).x;
        } else {
            w1 = lane_of(b, (uint32_t)(v0 & 3) + 1);
        }
        T o0, o1;
        xform2k<X>(w0, w1, p, o0, o1);
        return (i & 1) ? o1 : o0;
    } else {
        const uint64_t v = a.lane + i;
        const U4 b = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, v >> 2));
        return xform1<X>(lane_of(b, (uint32_t)(v & 3)), p);
    }
}

template <int X>
__device__ __forceinline__ void philox_scalar_range(const PhiloxScalar& a, const XformParams& p, void* out_base,
                                                    uint64_t gtid, uint64_t gstride) {
    using T = typename XformTraits<X>::T;
    T* out = static_cast<T*>(out_base);
    const uint64_t nscalar = a.i0 + (a.n - a.tail0);
    for (uint64_t s = gtid; s < nscalar; s += gstride) {
        const uint64_t i = s < a.i0 ? s : a.tail0 + (s - a.i0);
        out[i] = philox_scalar<X>(a, p, i);
    }
}

template <int SHIFT>
__device__ __forceinline__ U4 funnel(const U4& a, const U4& b) {
    if constexpr (SHIFT == 1) return U4{a.y, a.z, a.w, b.x};
    if constexpr (SHIFT == 2) return U4{a.z, a.w, b.x, b.y};
    if constexpr (SHIFT == 3) return U4{a.w, b.x, b.y, b.z};
    return a;
}

// Blocks per thread per pass on the aligned path: 4 for 4-byte outputs (two
// 256-bit stores of 64 contiguous bytes), 2 for 8-byte outputs.
#ifndef PRNG_PHILOX_BPT
#define PRNG_PHILOX_BPT 4
#endif
#ifndef PRNG_UNIT_MINB
#define PRNG_UNIT_MINB 5
#endif
template <typename T> struct PhiloxBpt { static constexpr int kValue = PRNG_PHILOX_BPT; };
// Round keys from the parameter table (philox_block_pre<true>) for the
// uniform transforms.
template <int X>
constexpr bool philox_rk() {
    return X == kUnitF32 || X == kUniformF32 || X == kUnitF64 || X == kUniformF64;
}
#ifndef PRNG_PHILOX_PIPE
#define PRNG_PHILOX_PIPE 1
#endif
#ifndef PRNG_GAUSS_MINB  // min resident CTAs for the unpipelined fast Box-Muller kernels
#define PRNG_GAUSS_MINB 0
#endif
// Aligned-path software pipelining (Philox of pass i+1 next to the transform
// of pass i): the fast fp32 lognormal (+3% in-library, 4-CTA bound); the
// centred-table fast gaussian is 1.8% faster unpipelined with no bound
// (tools/ab_lib.py, gpurun_out r2_9).
template <int X>
constexpr bool philox_pipelined() {
    return PRNG_PHILOX_PIPE && is_logn_fast(X);
}
template <> struct PhiloxBpt<double> { static constexpr int kValue = 2; };

// Store of one group whose first element sits one element below a 32-byte
// boundary (pair transforms into an odd-element output view, PhiloxBody::mis):
// the pairs keep their natural grouping, and the group goes out as element,
// aligned pair, element.
template <typename T>
__device__ __forceinline__ void st_group_mis(T* p, const T o[4]) {
    if constexpr (sizeof(T) == 4) {
        uint32_t b[4];
        memcpy(b, o, 16);
        asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(b[0]) : "memory");
        asm volatile("st.global.cs.v2.b32 [%0], {%1,%2};" ::"l"(p + 1), "r"(b[1]), "r"(b[2]) : "memory");
        asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p + 3), "r"(b[3]) : "memory");
    } else {
        unsigned long long b[4];
        memcpy(b, o, 32);
        asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(b[0]) : "memory");
        asm volatile("st.global.cs.v2.b64 [%0], {%1,%2};" ::"l"(p + 1), "l"(b[1]), "l"(b[2]) : "memory");
        asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p + 3), "l"(b[3]) : "memory");
    }
}


// Odd-element pair outputs, warp-shifted (PhiloxBody::mis): a lane that holds
// NE consecutive outputs v[0..NE) starting one element below a 32-byte
// boundary writes v[1..NE) plus its right neighbour's v[0] (by shuffle) as
// whole 32-byte sectors; only the first lane stores its v[0] on its own and a
// lane without a right neighbour ends with 16/8/4-byte pieces.  Every element
// is written once, with full-sector stores except at the two ends of a
// warp's run.
template <typename T>
__device__ __forceinline__ void st_bytes32(T* p, const T* e) {
    if constexpr (sizeof(T) == 4) {
        uint32_t b[8];
        memcpy(b, e, 32);
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(b[0]), "r"(b[1]), "r"(b[2]),
                     "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]) : "memory");
    } else {
        unsigned long long b[4];
        memcpy(b, e, 32);
        asm volatile("st.global.cs.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3])
                     : "memory");
    }
}
template <typename T, int BYTES>
__device__ __forceinline__ void st_piece(T* p, const T* e) {
    if constexpr (BYTES == 16 && sizeof(T) == 4) {
        uint32_t b[4];
        memcpy(b, e, 16);
        asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3])
                     : "memory");
    } else if constexpr (BYTES == 16) {
        unsigned long long b[2];
        memcpy(b, e, 16);
        asm volatile("st.global.cs.v2.b64 [%0], {%1,%2};" ::"l"(p), "l"(b[0]), "l"(b[1]) : "memory");
    } else if constexpr (BYTES == 8 && sizeof(T) == 4) {
        uint32_t b[2];
        memcpy(b, e, 8);
        asm volatile("st.global.cs.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(b[0]), "r"(b[1]) : "memory");
    } else if constexpr (BYTES == 8) {
        unsigned long long b;
        memcpy(&b, e, 8);
        asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
    } else {
        uint32_t b;
        memcpy(&b, e, 4);
        asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(b) : "memory");
    }
}

template <typename T, int NG>
__device__ __forceinline__ void st_run_shift1(T* dst, const T (&o)[NG][4], T nxt, bool has_next, bool first) {
    constexpr int NE = 4 * NG;
    constexpr int PER = 32 / (int)sizeof(T);
    const T* v = &o[0][0];
    if (first) st_piece<T, sizeof(T)>(dst, v);
    T* a = dst + 1;  // 32-byte aligned
    if (has_next) {
#pragma unroll
        for (int c = 0; c < NE / PER; ++c) {
            T e[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) e[k] = (1 + c * PER + k < NE) ? v[1 + c * PER + k] : nxt;
            st_bytes32(a + c * PER, e);
        }
    } else {
        constexpr int M = NE - 1, FULL = M / PER;
#pragma unroll
        for (int c = 0; c < FULL; ++c) st_bytes32(a + c * PER, v + 1 + c * PER);
        int off = FULL * PER;  // M - off < PER elements left: 16, 8, 4-byte pieces
        if constexpr ((M - FULL * PER) * sizeof(T) >= 16) {
            st_piece<T, 16>(a + off, v + 1 + off);
            off += 16 / sizeof(T);
        }
        if constexpr (((M - FULL * PER) * sizeof(T)) % 16 >= 8) {
            st_piece<T, 8>(a + off, v + 1 + off);
            off += 8 / sizeof(T);
        }
        if constexpr (((M - FULL * PER) * sizeof(T)) % 8 >= 4) st_piece<T, 4>(a + off, v + 1 + off);
    }
}

// Aligned path (SHIFT = 0) of one body launch; MIS: pair transforms whose
// body starts one element below a 32-byte boundary (a separate instantiation
// so the common loop keeps its register allocation).
template <int X, bool MIS>
__device__ __forceinline__ void philox_body_aligned(const PhiloxBody& a, uint32_t gtid, uint32_t gstride) {
    using T = typename XformTraits<X>::T;
    T* __restrict__ body = static_cast<T*>(a.out);
    constexpr int BPT = PhiloxBpt<T>::kValue;
    // Running group index and output pointer (adds on the ALU pipe; the
    // FMA-heavy pipe is kept for the Philox multiplies).
    // The steady-state loop covers whole units only (no per-iteration
    // bounds branch); the < BPT leftover groups go to one thread after it.
    const uint32_t gstep = gstride * BPT;
    const uint32_t gfull = a.ngroups - a.ngroups % BPT;
    T* dst = body + (size_t)4 * BPT * gtid;
    if constexpr (MIS) {
        // warp-uniform passes (the shuffle needs every lane); a lane's BPT
        // groups follow its left neighbour's, lane 31's right neighbour is
        // in the next warp
        const uint32_t lane = threadIdx.x & 31;
        for (uint32_t base = (gtid - lane) * BPT; base < gfull; base += gstep, dst += (size_t)4 * gstep) {
            const uint32_t g0 = base + lane * BPT;
            const bool valid = g0 < gfull;
            T o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) xform4<X>(philox_block_pre(a.k0, a.k1, a.c0 + g0 + j, a.pre), a.p, o[j]);
            const T nxt = __shfl_down_sync(0xffffffffu, o[0][0], 1);
            if (valid) st_run_shift1<T, BPT>(dst, o, nxt, lane != 31 && g0 + BPT < gfull, lane == 0);
        }
    } else {
    auto store = [&](T* d, T (&o)[BPT][4]) {
        if constexpr (sizeof(T) == 4) {
#pragma unroll
            for (int j = 0; j < BPT; j += 2) st_group2(d + 4 * j, o[j], o[j + 1]);
        } else {
#pragma unroll
            for (int j = 0; j < BPT; ++j) st_group(d + 4 * j, o[j]);
        }
    };
    if constexpr (philox_pipelined<X>()) {
        // Software-pipelined: the next pass's Philox blocks (FMA-heavy
        // IMAD.WIDE + ALU) are computed in the same basic block as this
        // pass's transform (FMA-lite, XU, LSU), so the scheduler can
        // interleave the two instruction mixes.  The blocks computed on
        // the last pass are not used (counter wrap is harmless there).
        U4 w[BPT];
#pragma unroll
        for (int j = 0; j < BPT; ++j) w[j] = philox_block_pre(a.k0, a.k1, a.c0 + gtid * BPT + j, a.pre);
        for (uint32_t g0 = gtid * BPT; g0 < gfull; g0 += gstep, dst += (size_t)4 * gstep) {
            U4 nw[BPT];
#pragma unroll
            for (int j = 0; j < BPT; ++j) nw[j] = philox_block_pre(a.k0, a.k1, a.c0 + g0 + gstep + j, a.pre);
            T o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) xform4<X>(w[j], a.p, o[j]);
            store(dst, o);
#pragma unroll
            for (int j = 0; j < BPT; ++j) w[j] = nw[j];
        }
    } else {
        for (uint32_t g0 = gtid * BPT; g0 < gfull; g0 += gstep, dst += (size_t)4 * gstep) {
            T o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) {
                const U4 w = philox_block_pre<philox_rk<X>()>(a.k0, a.k1, a.c0 + g0 + j, a.pre);
                xform4<X>(w, a.p, o[j]);
            }
            store(dst, o);
        }
    }
    }
    if (gtid == gstride - 1) {
        for (uint32_t g = gfull; g < a.ngroups; ++g) {
            T o[4];
            xform4<X>(philox_block_pre<philox_rk<X>()>(a.k0, a.k1, a.c0 + g, a.pre), a.p, o);
            if constexpr (MIS)
                st_group_mis(body + (size_t)4 * g, o);
            else
                st_group(body + (size_t)4 * g, o);
        }
    }
}

// MIS: the odd-element pair-output variant (PhiloxBody::mis), a separate
// kernel instantiation so the common kernels keep their register counts.
template <int X, int SHIFT, bool MIS = false>
__device__ __forceinline__ void philox_body(const PhiloxBody& a, uint32_t gtid, uint32_t gstride) {
    using T = typename XformTraits<X>::T;
    T* __restrict__ body = static_cast<T*>(a.out);
    if constexpr (SHIFT == 0) {
        philox_body_aligned<X, MIS>(a, gtid, gstride);
    } else {
        // Warp-cooperative funnel.  Lane l of a warp pass computes blocks
        // 4l..4l+3 of the tile and takes block 4l+4 (the first block of lane
        // l+1) by shuffle; group g = words d..3 of block g + words 0..d-1 of
        // block g+1.  A pass covers 126 groups (the 127th needs the next
        // tile's first block; 126 keeps every pass 32-byte aligned).
        constexpr int BPT = 4;
        constexpr uint32_t kTileGroups = 32 * BPT - 2;
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t gwarp = gtid >> 5;
        const uint32_t nwarps = gstride >> 5;
        const uint32_t ntiles = (uint32_t)(((uint64_t)a.ngroups + kTileGroups - 1) / kTileGroups);
        // blocks at index >= lim wrap c0 past 2^32 (only the one block after
        // a launch's last group can be consumed there)
        const uint64_t lim = (1ull << 32) - a.c0;
        for (uint32_t tile = gwarp; tile < ntiles; tile += nwarps) {
            const uint32_t gb = tile * kTileGroups + BPT * lane;
            U4 w[BPT + 1];
            if ((uint64_t)gb + BPT <= lim) {
#pragma unroll
                for (int j = 0; j < BPT; ++j) w[j] = philox_block_pre<philox_rk<X>()>(a.k0, a.k1, a.c0 + gb + j, a.pre);
            } else {
#pragma unroll
                for (int j = 0; j < BPT; ++j) {
                    U4 c{a.c0 + gb + j, a.c1, a.c2, a.c3};
                    if ((uint64_t)gb + j >= lim && ++c.y == 0 && ++c.z == 0) ++c.w;
                    w[j] = philox_block(a.k0, a.k1, c);
                }
            }
            w[BPT].x = __shfl_down_sync(0xffffffffu, w[0].x, 1);
            w[BPT].y = __shfl_down_sync(0xffffffffu, w[0].y, 1);
            w[BPT].z = __shfl_down_sync(0xffffffffu, w[0].z, 1);
            w[BPT].w = __shfl_down_sync(0xffffffffu, w[0].w, 1);
            T o[BPT][4];
#pragma unroll
            for (int j = 0; j < BPT; ++j) xform4<X>(funnel<SHIFT>(w[j], w[j + 1]), a.p, o[j]);
            T* dst = body + (size_t)4 * gb;
            const uint32_t nvalid = lane == 31 ? 2 : BPT;  // groups of this lane inside the pass
            if constexpr (MIS) {
                // odd-element pair output: whole lanes shift their run by one
                // element (st_run_shift1); a lane cut by the end of the data
                // stores group by group (its first element again: same value)
                const T nxt = __shfl_down_sync(0xffffffffu, o[0][0], 1);
                const bool full = gb + nvalid <= a.ngroups;
                const bool has_next = lane < 31 && gb + BPT < a.ngroups;
                if (full && lane < 31) {
                    st_run_shift1<T, BPT>(dst, o, nxt, has_next, lane == 0);
                } else if (full) {
                    const T(&o2)[2][4] = *reinterpret_cast<const T(*)[2][4]>(&o[0][0]);
                    st_run_shift1<T, 2>(dst, o2, nxt, false, false);
                } else {
#pragma unroll
                    for (int j = 0; j < BPT; ++j)
                        if (j < (int)nvalid && gb + j < a.ngroups) st_group_mis(dst + 4 * j, o[j]);
                }
            } else if (nvalid == BPT && gb + BPT <= a.ngroups) {
                if constexpr (sizeof(T) == 4) {
                    st_group2(dst, o[0], o[1]);
                    st_group2(dst + 8, o[2], o[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < BPT; ++j) st_group(dst + 4 * j, o[j]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < BPT; ++j)
                    if (j < (int)nvalid && gb + j < a.ngroups) st_group(dst + 4 * j, o[j]);
            }
        }
    }
}

// Minimum resident CTAs per SM given to ptxas.  For the unit / [a, b) fp32
// kernels (C1/C4) a bound of 5 (4 for the funnel variants) lets ptxas use
// ~48 registers and schedule the four blocks' multiply chains further
// apart: occupancy 5 instead of 6 but +3.5-4% throughput (+6% for the
// funnel), measured; the pipelined fast gaussian takes 4
// (61 registers: +1.4% over no bound, 5 is 2.4% slower), the other
// transforms keep ptxas' default (0 = no bound).  Eight blocks per thread measured 20% slower.
template <int X, int SHIFT>
constexpr int philox_min_blocks() {
    return (X == kUnitF32 || X == kUniformF32) ? (SHIFT == 0 ? PRNG_UNIT_MINB : 4)
           : ((X == kGaussF32Fast || is_logn_fast(X)) && SHIFT == 0) ? (philox_pipelined<X>() ? 4 : PRNG_GAUSS_MINB)
           : (is_precise(X) && SHIFT == 0) ? 5  // 45 KB of tables: at most 5 CTAs per SM
                                           : 0;
}

#ifdef PRNG_TRACE_CTA  // diagnostics build only (tools/cta_residency.py): per-CTA SM id, start, end (ns)
__device__ unsigned long long g_cta_trace[8192][3];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

template <int X, int SHIFT, bool MIS = false>
__global__ void __launch_bounds__(kPhiloxThreads, MIS ? 0 : philox_min_blocks<X, SHIFT>())
    philox_kernel(const PhiloxBody a) {
#ifdef PRNG_TRACE_CTA
    if (threadIdx.x == 0 && blockIdx.x < 8192) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cta_trace[blockIdx.x][0] = smid;
        g_cta_trace[blockIdx.x][1] = gtimer();
    }
#endif
    xform_prologue<X>(a.p);
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    if (a.s.n) {
        using T = typename XformTraits<X>::T;
        philox_scalar_range<X>(a.s, a.p, static_cast<T*>(a.out) - a.s.i0, gtid, gstride);
    }
    if (a.ngroups) philox_body<X, SHIFT, MIS>(a, gtid, gstride);
#ifdef PRNG_TRACE_CTA
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 8192) g_cta_trace[blockIdx.x][2] = gtimer();
#endif
}

// ------------------------------------------------------------- segments
// Many small requests in one launch (FastCaloSim consumer): blockIdx.y
// strides over segments, blockIdx.x over each segment's groups.  Segments
// keep the generic 64-bit counter arithmetic since a segment may straddle a
// 2^32-block boundary.
struct PhiloxSegment {
    uint64_t pos_lo, pos_hi, count, out_offset;
};

template <int X>
__global__ void __launch_bounds__(kPhiloxThreads)
    philox_segments_kernel(uint32_t k0, uint32_t k1, const PhiloxSegment* __restrict__ segs, uint32_t nseg,
                           XformParams p, typename XformTraits<X>::T* out) {
    using T = typename XformTraits<X>::T;
    static_assert(!XformTraits<X>::kPair, "segments carry single-word transforms only");
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    for (uint32_t s = blockIdx.y; s < nseg; s += gridDim.y) {
        const PhiloxSegment sg = segs[s];
        PhiloxBody a;
        a.mis = 0u;
        a.k0 = k0;
        a.k1 = k1;
        a.p = p;
        PhiloxScalar& sc = a.s;
        sc.k0 = k0;
        sc.k1 = k1;
        // block = pos >> 2 (128-bit), lane = pos & 3 (engine.py:221-222)
        sc.ctr_lo = (sg.pos_lo >> 2) | (sg.pos_hi << 62);
        sc.ctr_hi = sg.pos_hi >> 2;
        sc.lane = (uint32_t)(sg.pos_lo & 3);
        sc.n = sg.count;
        T* dst = out + sg.out_offset;
        // same plan as the host launcher: scalar head to a 32-byte boundary,
        // 4-element groups, scalar tail
        uint64_t i0 = ((32u - (uint32_t)((uintptr_t)dst & 31u)) & 31u) / sizeof(T);
        if (i0 > sc.n) i0 = sc.n;
        uint64_t ng = (sc.n - i0) >> 2;
        const uint64_t v0 = sc.lane + i0;
        const uint64_t blk_lo = sc.ctr_lo + (v0 >> 2);
        const uint64_t blk_hi = sc.ctr_hi + (blk_lo < sc.ctr_lo ? 1u : 0u);
        // a segment whose blocks cross a 2^32 boundary of c0 (or is > 2^31
        // groups) takes the all-scalar path; segments are small in practice.
        if ((uint64_t)(uint32_t)blk_lo + ng + 1 > (1ull << 32) || ng > (1ull << 31)) {
            i0 = sc.n;
            ng = 0;
        }
        sc.i0 = i0;
        sc.tail0 = i0 + 4 * ng;
        a.c0 = (uint32_t)blk_lo;
        a.c1 = (uint32_t)(blk_lo >> 32);
        a.c2 = (uint32_t)blk_hi;
        a.c3 = (uint32_t)(blk_hi >> 32);
        a.ngroups = (uint32_t)ng;
        a.pre = philox_pre(k0, k1, a.c1, a.c2, a.c3);
        a.out = dst + i0;
        philox_scalar_range<X>(sc, p, dst, gtid, gstride);
        if (ng) {
            switch ((uint32_t)(v0 & 3)) {
                case 0: philox_body<X, 0>(a, gtid, gstride); break;
                case 1: philox_body<X, 1>(a, gtid, gstride); break;
                case 2: philox_body<X, 2>(a, gtid, gstride); break;
                default: philox_body<X, 3>(a, gtid, gstride); break;
            }
        }
    }
}

}  // namespace prng
