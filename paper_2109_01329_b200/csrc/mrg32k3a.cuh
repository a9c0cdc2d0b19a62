// mrg32k3a.cuh -- MRG32k3a generate+transform kernel with per-lane
// jump-ahead (sm_100a).
//
// Replaces the strictly sequential reference loop _core.pyx:74-102
// (mrg_fill), which the reference cannot split (rngburn.py:123,
// engine.py:201-202).
//
// Layout ("segmented rows").  Warp w owns the region [w*32*chunk,
// (w+1)*32*chunk) of the request, cut into kChains regions, one per
// interleaved recurrence ("chain") of every lane.  A chain's region is walked
// in rounds of 32 segments of `seg` words (seg = 4 tiles = 512 bytes of
// output for the plain fp64 transforms, MrgPlan); in each round lane L produces the segment [round*32*seg + L*seg,
// +seg) and then jumps its state 31*seg words ahead (x -> B x mod m, B =
// A^(31 seg) split into 16-bit halves so the 3x3 mat-vec is exact in fp64).
// So at any time a warp writes one 16 KB contiguous window per chain.  The
// earlier layout -- one contiguous chunk per lane, 32 write fronts per warp
// `chunk` words apart -- capped the same stores at 4.5 TB/s on B200 against
// 6.0 TB/s for windows of 512-byte segments (tools/mrg_pattern.cu,
// profiles/r1_mrg_pattern.txt).
//
// Lane start states are A^(q*seg) s0 with q = (region start)/seg + L,
// assembled from host tables J_b = A^(seg*2^b) staged in shared memory (one
// 3x3 mod-m mat-vec per set bit of q); each further chain starts from the
// previous one by the host matrix A^(32*chunk/kChains).  Each 128-byte tile of
// every segment is transposed through an XOR-swizzled shared-memory stage
// (16-byte chunks) so each 128-bit store instruction writes four segments'
// whole 128-byte lines.
#pragma once

#include "common.cuh"

namespace prng {

constexpr int kMrgMaxBits = 32;
constexpr int kMrgThreads = 128;
#ifndef PRNG_MRG_MINB
#define PRNG_MRG_MINB 6
#endif
#ifndef PRNG_MRG_SEG_CHAINS
#define PRNG_MRG_SEG_CHAINS 2
#endif
#ifndef PRNG_MRG_SEG_MINB
#define PRNG_MRG_SEG_MINB 4
#endif

// Segmented rows (seg = 4 tiles, a jump every seg words) pay off where the
// store pattern is the bound: the plain 8-byte transforms.  Elsewhere (4-byte
// outputs at <= 3.6 TB/s, the Box-Muller transforms) the jumps cost more than
// the pattern, and seg = chunk / kChains gives one round per lane (no
// jumps).  kChains interleaved recurrences per lane; the 8-byte kernels take
// a 4-CTA bound (128 registers: no spills with the jump temporaries; 5 CTAs
// spilled 12 bytes and ran 2-5% slower), the others 6.
template <int X>
struct MrgPlan {
    static constexpr bool kSegmented = sizeof(typename XformTraits<X>::T) == 8 && !XformTraits<X>::kPair;
    static constexpr int kChains = kSegmented ? PRNG_MRG_SEG_CHAINS : 2;
    static constexpr int kMinBlocks = kSegmented ? PRNG_MRG_SEG_MINB : PRNG_MRG_MINB;
};

// Jump matrix B (entries as symmetric residues) split as B = hi*2^16 + lo,
// |hi|, |lo| <= 2^15: every product with a symmetric state value is below
// 2^46.1 and every row sum below 2^47.7, exact in fp64.
struct MrgJump {
    double hi[9], lo[9];
};

struct MrgLaunch {
    uint32_t s1[3], s2[3];
    uint64_t n;
    uint64_t chunk;  // words per lane (region of a warp = 32*chunk; multiple of kChains*seg)
    uint64_t seg;    // words per lane segment (4 tiles)
    uint32_t nbits;
    uint32_t j1[kMrgMaxBits][9];  // A^(seg * 2^b)
    uint32_t j2[kMrgMaxBits][9];
    MrgJump hs1, hs2;       // A^(32*chunk/kChains), split: chain c -> chain c+1
    MrgJump b1, b2;         // A^(31*seg): end of a segment -> start of the lane's next one
    void* out;
    XformParams p;
};

// y = B x mod m with B split as hi*2^16 + lo (tables in shared memory).
__device__ __forceinline__ void mrg_jump_p(const double* hi, const double* lo, double m, double inv_m, double& x0,
                                           double& x1, double& x2) {
    double y[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double l = __fma_rn(lo[3 * i + 2], x2, __fma_rn(lo[3 * i + 1], x1, __dmul_rn(lo[3 * i], x0)));
        const double h = __fma_rn(hi[3 * i + 2], x2, __fma_rn(hi[3 * i + 1], x1, __dmul_rn(hi[3 * i], x0)));
        y[i] = mrg_reduce(__fma_rn(mrg_reduce(h, m, inv_m), 65536.0, l), m, inv_m);
    }
    x0 = y[0];
    x1 = y[1];
    x2 = y[2];
}

// split_jump (api.cu) on the device: entry v < m as symmetric residue = hi 2^16 + lo.
__device__ __forceinline__ void split_entry(uint32_t v, uint32_t m, double& hi, double& lo) {
    const double sv = mrg_sym(v, m);
    hi = rint(sv * (1.0 / 65536.0));
    lo = __fma_rn(-hi, 65536.0, sv);
}

__device__ __forceinline__ void mrg_jump(const MrgJump& B, double m, double inv_m, double& x0, double& x1,
                                         double& x2) {
    double y[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double l = __fma_rn(B.lo[3 * i + 2], x2, __fma_rn(B.lo[3 * i + 1], x1, __dmul_rn(B.lo[3 * i], x0)));
        const double h = __fma_rn(B.hi[3 * i + 2], x2, __fma_rn(B.hi[3 * i + 1], x1, __dmul_rn(B.hi[3 * i], x0)));
        y[i] = mrg_reduce(__fma_rn(mrg_reduce(h, m, inv_m), 65536.0, l), m, inv_m);
    }
    x0 = y[0];
    x1 = y[1];
    x2 = y[2];
}

__device__ __forceinline__ void mrg_jump_state(const MrgLaunch& a, MrgStateF64& s) {
    mrg_jump(a.b1, (double)kMrgM1, 1.0 / (double)kMrgM1, s.x10, s.x11, s.x12);
    mrg_jump(a.b2, (double)kMrgM2, 1.0 / (double)kMrgM2, s.x20, s.x21, s.x22);
}

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

// Write one staged tile (row j = lane j's segment, starting at run0 + j*rs).
// Each instruction moves four rows' 128-byte lines: lane L handles row
// 4i + (L >> 3), chunk L & 7.  The common case (tile entirely inside the
// request, 16-byte aligned output) is a straight-line block of 8 LDS.128 +
// 8 STG.128 with one 64-bit stride add each; the predicated element path
// only runs for the request's last tiles.
template <typename T>
__device__ __forceinline__ void mrg_store_tile(const uint4* st, T* __restrict__ run0, uint64_t rs, uint32_t lane,
                                               uint64_t first_elem, uint64_t n, bool vec_ok) {
    constexpr int CE = 16 / sizeof(T);
    constexpr int TW = 8 * CE;
    const uint32_t x = lane & 7;
    const uint32_t r0 = lane >> 3;
    T* p = run0 + r0 * rs + x * CE;
    const uint64_t stride = 4 * rs;
    if (vec_ok && first_elem + 31 * rs + TW <= n) {  // warp-uniform
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t j = 4 * i + r0;
            st_global_cs_v4(p + i * stride, st[j * 8 + (x ^ (j & 7))]);
        }
        return;
    }
    uint64_t e = first_elem + r0 * rs + x * CE;
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
__global__ void __launch_bounds__(kMrgThreads, MrgPlan<X>::kMinBlocks) mrg_kernel(const MrgLaunch a) {
    using T = typename XformTraits<X>::T;
    constexpr int TW = MrgTile<T>::kWords;
    constexpr int WARPS = kMrgThreads / 32;
    constexpr int NC = MrgPlan<X>::kChains;
    __shared__ uint4 stage[NC][WARPS][32 * 8];
    // Start-state tables J_b.  The non-Box-Muller kernels split them for
    // the exact fp64 mat-vec (mrg_jump_p: ~2.5x less pipe time than the
    // integer fold formulation, on the FP64 pipe that is idle during
    // start-up; 9 KB of shared memory), the others (whose Box-Muller table
    // leaves no room) keep the integer walk.
    constexpr bool kF64Walk = !XformTraits<X>::kPair;
    constexpr int kTabN = kF64Walk ? kMrgMaxBits * 9 : 1;
    constexpr int kIntN = kF64Walk ? 1 : kMrgMaxBits * 9;
    __shared__ double sjh1[kTabN], sjl1[kTabN], sjh2[kTabN], sjl2[kTabN];
    __shared__ uint32_t sj1[kIntN], sj2[kIntN];
    for (uint32_t i = threadIdx.x; i < a.nbits * 9; i += blockDim.x) {
        if constexpr (kF64Walk) {
            split_entry(a.j1[i / 9][i % 9], kMrgM1, sjh1[i], sjl1[i]);
            split_entry(a.j2[i / 9][i % 9], kMrgM2, sjh2[i], sjl2[i]);
        } else {
            sj1[i] = a.j1[i / 9][i % 9];
            sj2[i] = a.j2[i / 9][i % 9];
        }
    }
    xform_prologue<X, kMrgTabLog2>(a.p);
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t t_warp0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    const uint64_t w0 = t_warp0 * a.chunk;  // first word of the warp's region
    if (w0 >= a.n) return;                  // whole warp idle (warp-uniform)

    const uint64_t q = w0 / a.seg + lane;  // lane's first segment, in units of seg
    MrgStateF64 x;
    if constexpr (kF64Walk) {
        x = MrgStateF64{mrg_sym(a.s1[0], kMrgM1), mrg_sym(a.s1[1], kMrgM1), mrg_sym(a.s1[2], kMrgM1),
                        mrg_sym(a.s2[0], kMrgM2), mrg_sym(a.s2[1], kMrgM2), mrg_sym(a.s2[2], kMrgM2)};
        for (uint32_t b = 0; b < a.nbits; ++b) {
            if ((q >> b) & 1) {
                mrg_jump_p(&sjh1[9 * b], &sjl1[9 * b], (double)kMrgM1, 1.0 / (double)kMrgM1, x.x10, x.x11, x.x12);
                mrg_jump_p(&sjh2[9 * b], &sjl2[9 * b], (double)kMrgM2, 1.0 / (double)kMrgM2, x.x20, x.x21, x.x22);
            }
        }
    } else {
        uint32_t x10 = a.s1[0], x11 = a.s1[1], x12 = a.s1[2], x20 = a.s2[0], x21 = a.s2[1], x22 = a.s2[2];
        for (uint32_t b = 0; b < a.nbits; ++b) {
            if ((q >> b) & 1) {
                mat3_apply<kMrgC1>(&sj1[9 * b], x10, x11, x12);
                mat3_apply<kMrgC2>(&sj2[9 * b], x20, x21, x22);
            }
        }
        x = MrgStateF64{mrg_sym(x10, kMrgM1), mrg_sym(x11, kMrgM1), mrg_sym(x12, kMrgM1),
                        mrg_sym(x20, kMrgM2), mrg_sym(x21, kMrgM2), mrg_sym(x22, kMrgM2)};
    }
    MrgStateF64 st[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c) {  // chain c starts one chain region (A^(32 chunk / NC)) after chain c-1
            mrg_jump(a.hs1, (double)kMrgM1, 1.0 / (double)kMrgM1, x.x10, x.x11, x.x12);
            mrg_jump(a.hs2, (double)kMrgM2, 1.0 / (double)kMrgM2, x.x20, x.x21, x.x22);
        }
        st[c] = x;
    }

    const uint64_t region = 32 * a.chunk / NC;  // words per chain region
    const uint64_t seg = a.seg;
    T* __restrict__ out = static_cast<T*>(a.out);
    const bool vec_ok = ((uintptr_t)out & 15u) == 0;
    constexpr int CE = 16 / sizeof(T);  // elements per 16-byte chunk
    for (uint64_t rb = 0; rb < region; rb += 32 * seg) {
        if (w0 + rb >= a.n) break;  // warp-uniform
        for (uint64_t off = 0; off < seg; off += TW) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                T o[NC][CE];
                if constexpr (XformTraits<X>::kPair) {
#pragma unroll
                    for (int k = 0; k < CE; k += 2) {
#pragma unroll
                        for (int h = 0; h < NC; ++h) {
                            const uint32_t u0 = mrg_step_f64(st[h]);
                            const uint32_t u1 = mrg_step_f64(st[h]);
                            xform2k<X, kMrgTabLog2>(u0, u1, a.p, o[h][k], o[h][k + 1]);
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < CE; ++k) {
#pragma unroll
                        for (int h = 0; h < NC; ++h) o[h][k] = xform1<X>(mrg_step_f64(st[h]), a.p);
                    }
                }
#pragma unroll
                for (int h = 0; h < NC; ++h) stage_put(stage[h][warp], lane, c, pack16<T>(o[h]));
            }
            __syncwarp();
            const uint64_t ea = w0 + rb + off;
#pragma unroll
            for (int h = 0; h < NC; ++h)
                mrg_store_tile<T>(stage[h][warp], out + ea + h * region, seg, lane, ea + h * region, a.n, vec_ok);
            __syncwarp();
        }
        if constexpr (MrgPlan<X>::kSegmented) {  // otherwise one round (seg = region / 32)
            if (rb + 32 * seg < region) {
#pragma unroll
                for (int h = 0; h < NC; ++h) mrg_jump_state(a, st[h]);
            }
        }
    }
}

}  // namespace prng
