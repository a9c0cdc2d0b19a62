// philox.cuh -- fused Philox4x32-10 generate+transform kernel (sm_100a).
//
// Replaces the reference hot loop _core.pyx:42-71 (philox_fill) together with
// the two passes layered on it: words_to_unit (distributions.py:83-87) and the
// range transform (distributions.py:98-104 / rngburn.py:62-64, 94-100), or
// Box-Muller (distributions.py:116-131) / lognormal.  Each sample is written
// to HBM exactly once.
//
// Work decomposition.  A request is n elements starting at stream word
// `lane` of the block with 128-bit counter `ctr` (the reference's
// philox_fill(k0, k1, b0..b3, offset, n) arguments, engine.py:222-225).
// Output element i consumes "virtual word" v = lane + i, i.e. lane v&3 of
// block ctr + (v>>2).  The output is split into
//   * a scalar head [0, i0) that brings out+i0 to a 32-byte boundary,
//   * a body of `ngroups` 4-element groups, group g holding virtual words
//     lane+i0+4g .. +3, stored with 128/256-bit streaming stores,
//   * a scalar tail.
// When (lane + i0) % 4 == 0 every body group is exactly one Philox block
// (SHIFT = 0): each thread computes two adjacent blocks and issues one
// 256-bit store (fp32/u32) or one 256-bit store per block (fp64), so a warp
// instruction writes 1 KiB of contiguous output.  Otherwise (SHIFT = 1..3) a
// group straddles two blocks: lane t of a warp computes block t and takes the
// first SHIFT words of block t+1 from lane t+1 by shuffle; each warp pass
// emits 31 groups from 32 blocks.
#pragma once

#include "common.cuh"

namespace prng {

struct PhiloxLaunch {
    uint32_t k0, k1;
    uint64_t ctr_lo, ctr_hi;  // counter of the block holding element 0
    uint32_t lane;            // virtual word index of element 0 (0..3)
    uint64_t n;               // elements
    uint64_t i0;              // scalar head length
    uint64_t ngroups;         // vector body groups
    uint64_t body_blk;        // (lane + i0) >> 2
    void* out;
    XformParams p;
};

// Element i computed on its own (head, tail and the fully generic path).
template <int X>
__device__ __forceinline__ typename XformTraits<X>::T philox_scalar(const PhiloxLaunch& a, uint64_t i) {
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
        xform2<X>(w0, w1, a.p, o0, o1);
        return (i & 1) ? o1 : o0;
    } else {
        const uint64_t v = a.lane + i;
        const U4 b = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, v >> 2));
        return xform1<X>(lane_of(b, (uint32_t)(v & 3)), a.p);
    }
}

template <int SHIFT>
__device__ __forceinline__ U4 funnel(const U4& a, const U4& b) {
    if constexpr (SHIFT == 1) return U4{a.y, a.z, a.w, b.x};
    if constexpr (SHIFT == 2) return U4{a.z, a.w, b.x, b.y};
    if constexpr (SHIFT == 3) return U4{a.w, b.x, b.y, b.z};
    return a;
}

constexpr int kPhiloxThreads = 256;

// Split a request into head / body / tail for an output at `out_addr`.
// Returns the body SHIFT ((lane + i0) & 3).  Pair transforms need the body to
// start on a pair boundary (i0 even); if the output is misaligned for that
// (fp32 at an odd 4-byte offset) everything goes through the scalar path.
__host__ __device__ inline int plan_philox(PhiloxLaunch& a, uint64_t out_addr, uint32_t esize, bool pair) {
    const uint64_t i0 = ((32u - (uint32_t)(out_addr & 31u)) & 31u) / esize;
    if ((pair && (i0 & 1)) || i0 >= a.n) {
        a.i0 = a.n;
        a.ngroups = 0;
        a.body_blk = 0;
        return 0;
    }
    a.i0 = i0;
    a.ngroups = (a.n - i0) >> 2;
    a.body_blk = (a.lane + i0) >> 2;
    return (int)((a.lane + i0) & 3);
}

template <int X, int SHIFT>
__device__ __forceinline__ void philox_body(const PhiloxLaunch& a, uint64_t gtid, uint64_t gstride) {
    using T = typename XformTraits<X>::T;
    T* __restrict__ out = static_cast<T*>(a.out);

    // Scalar head/tail (at most 7 + 3 elements unless the request is
    // misaligned for pair transforms, in which case everything is scalar).
    const uint64_t body_end = a.i0 + 4 * a.ngroups;
    const uint64_t nscalar = a.i0 + (a.n - body_end);
    for (uint64_t s = gtid; s < nscalar; s += gstride) {
        const uint64_t i = s < a.i0 ? s : body_end + (s - a.i0);
        out[i] = philox_scalar<X>(a, i);
    }
    if (a.ngroups == 0) return;
    T* __restrict__ body = out + a.i0;

    if constexpr (SHIFT == 0) {
        if constexpr (sizeof(T) == 4) {
            // Two blocks per thread -> one 256-bit store.
            const uint64_t nunits = (a.ngroups + 1) >> 1;
            for (uint64_t u = gtid; u < nunits; u += gstride) {
                const uint64_t g = 2 * u;
                const U4 w0 = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, a.body_blk + g));
                T o0[4];
                xform4<X>(w0, a.p, o0);
                if (g + 1 < a.ngroups) {
                    const U4 w1 = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, a.body_blk + g + 1));
                    T o1[4];
                    xform4<X>(w1, a.p, o1);
                    st_group2(body + 4 * g, o0, o1);
                } else {
                    st_group(body + 4 * g, o0);
                }
            }
        } else {
            for (uint64_t g = gtid; g < a.ngroups; g += gstride) {
                const U4 w = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, a.body_blk + g));
                T o[4];
                xform4<X>(w, a.p, o);
                st_group(body + 4 * g, o);
            }
        }
    } else {
        // Warp-cooperative funnel: 32 blocks -> 31 groups per pass.
        const uint32_t lane = threadIdx.x & 31;
        const uint64_t gwarp = gtid >> 5;
        const uint64_t nwarps = gstride >> 5;
        const uint64_t ntiles = (a.ngroups + 30) / 31;
        for (uint64_t tile = gwarp; tile < ntiles; tile += nwarps) {
            const uint64_t g = tile * 31 + lane;
            const U4 w = philox_block(a.k0, a.k1, counter_add(a.ctr_lo, a.ctr_hi, a.body_blk + g));
            U4 nx;
            nx.x = __shfl_down_sync(0xffffffffu, w.x, 1);
            nx.y = __shfl_down_sync(0xffffffffu, w.y, 1);
            nx.z = __shfl_down_sync(0xffffffffu, w.z, 1);
            nx.w = __shfl_down_sync(0xffffffffu, w.w, 1);
            if (lane < 31 && g < a.ngroups) {
                T o[4];
                xform4<X>(funnel<SHIFT>(w, nx), a.p, o);
                st_group(body + 4 * g, o);
            }
        }
    }
}

template <int X, int SHIFT>
__global__ void __launch_bounds__(kPhiloxThreads) philox_kernel(const PhiloxLaunch a) {
    philox_body<X, SHIFT>(a, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
}

// Segment table (many small batches in one launch): blockIdx.y strides over
// segments, blockIdx.x over each segment's elements.
struct PhiloxSegment {
    uint64_t pos_lo, pos_hi, count, out_offset;
};

template <int X>
__global__ void __launch_bounds__(kPhiloxThreads)
    philox_segments_kernel(uint32_t k0, uint32_t k1, const PhiloxSegment* __restrict__ segs, uint32_t nseg,
                           XformParams p, typename XformTraits<X>::T* out) {
    using T = typename XformTraits<X>::T;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    for (uint32_t s = blockIdx.y; s < nseg; s += gridDim.y) {
        const PhiloxSegment sg = segs[s];
        PhiloxLaunch a;
        a.k0 = k0;
        a.k1 = k1;
        // block = pos >> 2 (128-bit), lane = pos & 3 (engine.py:221-222)
        a.ctr_lo = (sg.pos_lo >> 2) | (sg.pos_hi << 62);
        a.ctr_hi = sg.pos_hi >> 2;
        a.lane = (uint32_t)(sg.pos_lo & 3);
        a.n = sg.count;
        a.out = out + sg.out_offset;
        a.p = p;
        const int shift = plan_philox(a, (uint64_t)(uintptr_t)a.out, sizeof(T), XformTraits<X>::kPair);
        switch (shift) {
            case 0: philox_body<X, 0>(a, gtid, gstride); break;
            case 1: philox_body<X, 1>(a, gtid, gstride); break;
            case 2: philox_body<X, 2>(a, gtid, gstride); break;
            default: philox_body<X, 3>(a, gtid, gstride); break;
        }
    }
}

}  // namespace prng
