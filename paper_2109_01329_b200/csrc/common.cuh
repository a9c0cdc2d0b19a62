// common.cuh -- shared device code for the B200 RNG kernels.
//
// Engine arithmetic (Philox4x32-10, MRG32k3a modular steps) and the fused
// distribution transforms.  Every transform reproduces the reference's
// rounding sequence explicitly (no FMA contraction where the reference has
// two roundings), see the per-function citations.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace prng {

// engine.py:34-37 / _core.pyx:12-15
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// engine.py:41-46
constexpr uint32_t kMrgM1 = 4294967087u;  // 2^32 - 209
constexpr uint32_t kMrgM2 = 4294944443u;  // 2^32 - 22853
constexpr uint32_t kMrgC1 = 209u;
constexpr uint32_t kMrgC2 = 22853u;
constexpr uint32_t kMrgA12 = 1403580u;
constexpr uint32_t kMrgA13N = 810728u;
constexpr uint32_t kMrgA21 = 527612u;
constexpr uint32_t kMrgA23N = 1370589u;

constexpr float kUnitF = 5.9604644775390625e-08f;  // 2^-24 (distributions.py:24)
constexpr double kUnitD = 5.9604644775390625e-08;
constexpr double kTwoPi = 6.283185307179586;  // distributions.py:25, _core.pyx:17

struct U4 {
    uint32_t x, y, z, w;
};

// One Philox4x32-10 block (engine.py:86-103, _core.pyx:20-39).  The round
// keys k + i*W are kernel-uniform, so ptxas keeps them in uniform registers;
// each round is two IMAD.WIDE.U32 and two 3-input LOP3s.
__device__ __forceinline__ U4 philox_block(uint32_t k0, uint32_t k1, U4 c) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint64_t p0 = (uint64_t)kPhiloxM0 * c.x;
        const uint64_t p1 = (uint64_t)kPhiloxM1 * c.z;
        const uint32_t t0 = (uint32_t)(p1 >> 32) ^ c.y ^ k0;
        const uint32_t t2 = (uint32_t)(p0 >> 32) ^ c.w ^ k1;
        c.y = (uint32_t)p1;
        c.w = (uint32_t)p0;
        c.x = t0;
        c.z = t2;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return c;
}

// Rounds 1-3 with the upper counter words (c1, c2, c3) uniform across the
// launch: everything that depends only on (key, c1, c2, c3) is folded on the
// host into five words, so a block costs 18 vector IMAD.WIDE instead of 20 and
// no uniform->vector moves (philox.cuh, "PhiloxBody").
struct PhiloxPre {
    uint32_t r1_x3;  // c3 ^ k1                      (round 1: c2' = hi(M0 c0) ^ r1_x3)
    uint32_t r2_x1;  // lo(M1 c2) ^ (k0 + W0)        (round 2: c0'' = hi(M1 c2') ^ r2_x1)
    uint32_t r2_x3;  // hi(M0 U0) ^ (k1 + W1)        (round 2: c2'' = lo(M0 c0) ^ r2_x3)
    uint32_t r2_c3;  // lo(M0 U0), U0 = hi(M1 c2) ^ c1 ^ k0
    uint32_t r3_x3;  // r2_c3 ^ (k1 + 2 W1)
    uint32_t rk0[8], rk1[8];  // round keys k + i W for rounds i = 2..9 (kernel-parameter operands)
};


__host__ __device__ inline PhiloxPre philox_pre(uint32_t k0, uint32_t k1, uint32_t c1, uint32_t c2, uint32_t c3) {
    const uint64_t p1 = (uint64_t)kPhiloxM1 * c2;
    const uint32_t u0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t u1 = (uint32_t)p1;
    const uint64_t p0u = (uint64_t)kPhiloxM0 * u0;
    PhiloxPre q;
    q.r1_x3 = c3 ^ k1;
    q.r2_x1 = u1 ^ (k0 + kPhiloxW0);
    q.r2_x3 = (uint32_t)(p0u >> 32) ^ (k1 + kPhiloxW1);
    q.r2_c3 = (uint32_t)p0u;
    q.r3_x3 = q.r2_c3 ^ (k1 + 2 * kPhiloxW1);
    for (int i = 0; i < 8; ++i) {
        q.rk0[i] = k0 + (uint32_t)(i + 2) * kPhiloxW0;
        q.rk1[i] = k1 + (uint32_t)(i + 2) * kPhiloxW1;
    }
    return q;
}

// Philox4x32-10 of counter (c0, c1, c2, c3) given philox_pre(k0, k1, c1, c2, c3).
// RK: take the round keys from q's table -- constant-bank operands of the
// LOP3s when q is a kernel parameter (no per-pass key arithmetic: -12 of 225
// instructions per 16 fp32 uniforms, +2-3%; measured neutral-to-worse for
// the bits and Box-Muller kernels, which recompute them).
template <bool RK = false>
__device__ __forceinline__ U4 philox_block_pre(uint32_t k0, uint32_t k1, uint32_t c0, const PhiloxPre& q) {
    uint64_t p0 = (uint64_t)kPhiloxM0 * c0;  // round 1
    const uint32_t x2 = (uint32_t)(p0 >> 32) ^ q.r1_x3;
    const uint32_t x3 = (uint32_t)p0;
    uint64_t p1 = (uint64_t)kPhiloxM1 * x2;  // round 2
    const uint32_t y0 = (uint32_t)(p1 >> 32) ^ q.r2_x1;
    const uint32_t y1 = (uint32_t)p1;
    const uint32_t y2 = x3 ^ q.r2_x3;
    p0 = (uint64_t)kPhiloxM0 * y0;  // round 3
    p1 = (uint64_t)kPhiloxM1 * y2;
    U4 c{(uint32_t)(p1 >> 32) ^ y1 ^ (RK ? q.rk0[0] : k0 + 2 * kPhiloxW0), (uint32_t)p1,
         (uint32_t)(p0 >> 32) ^ q.r3_x3, (uint32_t)p0};
#pragma unroll
    for (int i = 3; i < 10; ++i) {
        const uint32_t ki0 = RK ? q.rk0[i - 2] : k0 + (uint32_t)i * kPhiloxW0;
        const uint32_t ki1 = RK ? q.rk1[i - 2] : k1 + (uint32_t)i * kPhiloxW1;
        const uint64_t a = (uint64_t)kPhiloxM0 * c.x;
        const uint64_t b = (uint64_t)kPhiloxM1 * c.z;
        const uint32_t t0 = (uint32_t)(b >> 32) ^ c.y ^ ki0;
        const uint32_t t2 = (uint32_t)(a >> 32) ^ c.w ^ ki1;
        c.y = (uint32_t)b;
        c.w = (uint32_t)a;
        c.x = t0;
        c.z = t2;
    }
    return c;
}

// 128-bit counter (lo64, hi64) + idx, carried across all four lanes
// (_core.pyx:63-70).
__device__ __forceinline__ U4 counter_add(uint64_t lo, uint64_t hi, uint64_t idx) {
    const uint64_t l = lo + idx;
    const uint64_t h = hi + (l < lo ? 1u : 0u);
    return U4{(uint32_t)l, (uint32_t)(l >> 32), (uint32_t)h, (uint32_t)(h >> 32)};
}

__device__ __forceinline__ uint32_t lane_of(const U4& b, uint32_t i) {
    return i == 0 ? b.x : i == 1 ? b.y : i == 2 ? b.z : b.w;
}

// ---------------------------------------------------------------- MRG32k3a
// x mod m for m = 2^32 - c, x < 2^64 (two folds of 2^32 == c, one subtract).
template <uint32_t C>
__device__ __forceinline__ uint32_t fold_mod(uint64_t t) {
    constexpr uint64_t M = (1ull << 32) - C;
    t = (t >> 32) * C + (t & 0xffffffffull);
    t = (t >> 32) * C + (t & 0xffffffffull);
    return (uint32_t)(t >= M ? t - M : t);
}

// All-fp64 formulation (L'Ecuyer's floating-point MRG32k3a with symmetric
// residues).  Each component keeps its window as integers in [-m/2 - 1,
// m/2 + 1] held in doubles, so a*x_i - b*x_j stays below 2^52.1 and is exact
// (DMUL + DFMA); the reduction r = p - rint(p/m)*m (DFMA with the 1.5*2^52
// rounding magic, DADD, DFMA) is exact and lands back in the symmetric range.
// Both components run on the FP64 pipe with no compare/select in the
// recurrence; only the output word is canonicalised, in 32-bit integers:
// the magic-added double's low word is the residue's two's complement,
// c = r < 0 ? r + m : r, z = (c1 - c2) mod m1 (_core.pyx:85-101).
struct MrgStateF64 {
    double x10, x11, x12, x20, x21, x22;
};

__host__ __device__ inline double mrg_sym(uint32_t x, uint32_t m) {
    return x > m / 2 ? (double)x - (double)m : (double)x;
}

constexpr double kRintMagic = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ double mrg_reduce(double p, double m, double inv_m) {
    const double k = __dadd_rn(__fma_rn(p, inv_m, kRintMagic), -kRintMagic);
    return __fma_rn(-k, m, p);
}

__device__ __forceinline__ uint32_t mrg_canon(double r, uint32_t m) {
    const int32_t i = __double2loint(__dadd_rn(r, kRintMagic));
    return (uint32_t)i + (i < 0 ? m : 0u);
}

__device__ __forceinline__ uint32_t mrg_step_f64(MrgStateF64& s) {
    const double p1 = mrg_reduce(__fma_rn(-(double)kMrgA13N, s.x10, __dmul_rn((double)kMrgA12, s.x11)),
                                 (double)kMrgM1, 1.0 / (double)kMrgM1);
    const double p2 = mrg_reduce(__fma_rn(-(double)kMrgA23N, s.x20, __dmul_rn((double)kMrgA21, s.x22)),
                                 (double)kMrgM2, 1.0 / (double)kMrgM2);
    s.x10 = s.x11; s.x11 = s.x12; s.x12 = p1;
    s.x20 = s.x21; s.x21 = s.x22; s.x22 = p2;
    const uint32_t c1 = mrg_canon(p1, kMrgM1);
    const uint32_t c2 = mrg_canon(p2, kMrgM2);
    return c1 >= c2 ? c1 - c2 : c1 - c2 + kMrgM1;
}

// y = J x mod m (3x3), products folded before summation.
template <uint32_t C>
__device__ __forceinline__ void mat3_apply(const uint32_t* J, uint32_t& a, uint32_t& b, uint32_t& c) {
    uint32_t r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const uint64_t s = (uint64_t)fold_mod<C>((uint64_t)J[3 * i] * a) +
                           (uint64_t)fold_mod<C>((uint64_t)J[3 * i + 1] * b) +
                           (uint64_t)fold_mod<C>((uint64_t)J[3 * i + 2] * c);
        r[i] = fold_mod<C>(s);
    }
    a = r[0]; b = r[1]; c = r[2];
}

// ---------------------------------------------------------- transforms
// Word -> unit: (w >> 8) * 2^-24, exact in fp32 and fp64 (distributions.py:78-87).
// I2FP + FMUL.  (An I2FP-free exact alternative -- F = bits(0x3F000000 |
// (w >> 8)), u = min(F - 0.5, F * 0.5), tools/check_unit_trick.c -- moves the
// conversion off the FMA-heavy pipe but measured 0.4-1.4% slower on B200:
// the extra ALU/FMA-lite instructions cost more than the I2FP.)
__device__ __forceinline__ float unit_f32(uint32_t w) { return __fmul_rn((float)(w >> 8), kUnitF); }
// 2^52 + (w >> 8) built from bits (no I2F.F64 on the XU pipe): the 24-bit
// integer sits in the low mantissa bits of 2^52.
__device__ __forceinline__ double u24_magic(uint32_t w) { return __hiloint2double(0x43300000, (int)(w >> 8)); }
// (2^52 + x) * 2^-24 - 2^28 = x * 2^-24 exactly (one DFMA).
__device__ __forceinline__ double unit_f64(uint32_t w) { return __fma_rn(u24_magic(w), kUnitD, -268435456.0); }

// Exact gaussian method: per-input ulp corrections of the device
// approximations to the host libm (box_muller_exact below).
struct ExactCorrections {
    const uint8_t* log_nib;  // 2^23 bytes: 4-bit ulp correction of log_u1_f64 per m (two per byte)
    const uint8_t* sc_nib;   // 2^24 bytes: sin (low) / cos (high) 4-bit corrections per k
    const uint32_t* esc_idx[3];  // escapes (correction -8): sorted indices ...
    const double* esc_val[3];    // ... and the host-libm values; [0] log, [1] sin, [2] cos
    uint32_t esc_n[3];
    // Worst differences of the short approximations (log_u1_f64_short,
    // sincos_f64_short) from the host libm over both whole domains (measured
    // when the tables are built): relative for the log, absolute for sin /
    // cos.  The fp32 exact route's rounding test (f32_rounding_uncertain)
    // uses them.
    double rel_log, abs_sc;
    float tol_c;  // 2 (rel_log / 2 + abs_sc + 6 * 2^-53), rounded up (f32_rounding_uncertain)
};

// Parameters of one fused request.  For uniform: (a, b) -> scale/offset with
// the reference's precision rules (distributions.py:98-104 under numpy
// NEP-50: fp32 arrays see f32(hi - lo) and f32(lo)).
struct XformParams {
    float scale_f, off_f;    // uniform fp32: f32(b - a) * 2^-24, f32(a); gaussian fp32: stddev, mean
    double scale_d, off_d;   // uniform fp64: (b - a) * 2^-24, a; gaussian fp64: stddev, mean
    double mag_d;            // uniform fp64: -2^52 * scale_d
    double ln_scale, ln_displ;  // lognormal: scale, displ (fp64 path) ...
    float ln_scale_f, ln_displ_f;  // ... and fp32 path
    ExactCorrections exact;     // exact gaussian: correction tables (device memory)
};

// Transform kinds (template parameter).
enum Xform : int {
    kBits = 0,
    kUniformF32 = 1,
    kUniformF64 = 2,
    kGaussF32Fast = 3,
    kGaussF32Accurate = 4,
    kGaussF64 = 5,
    kLognF32Fast = 6,
    kLognF32Accurate = 7,
    kLognF64 = 8,
    kUnitF32 = 9,   // uniform on [0, 1): the affine pass is an exact identity
    kUnitF64 = 10,
    kGaussF32Exact = 11,  // the reference's fp64 Box-Muller bit for bit, cast once
    kGaussF64Exact = 12,
    kLognF32FastUnit = 13,  // kLognF32Fast with scale 1, displ 0 (no final affine: bit-identical)
    kGaussF32Precise = 14,  // fp32 route with relative accuracy everywhere (table log, centred sin/cos + x^2)
    kLognF32Precise = 15,
};

constexpr bool is_logn_fast(int X) { return X == kLognF32Fast || X == kLognF32FastUnit; }
constexpr bool is_precise(int X) { return X == kGaussF32Precise || X == kLognF32Precise; }
// fp32 Box-Muller routes with a shared-memory sin/cos table
constexpr bool is_f32_table_route(int X) { return X == kGaussF32Fast || is_logn_fast(X) || is_precise(X); }

template <int X> struct XformTraits;
template <> struct XformTraits<kBits> { using T = uint32_t; static constexpr bool kPair = false; };
template <> struct XformTraits<kUniformF32> { using T = float; static constexpr bool kPair = false; };
template <> struct XformTraits<kUniformF64> { using T = double; static constexpr bool kPair = false; };
template <> struct XformTraits<kUnitF32> { using T = float; static constexpr bool kPair = false; };
template <> struct XformTraits<kUnitF64> { using T = double; static constexpr bool kPair = false; };
template <> struct XformTraits<kGaussF32Fast> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kGaussF32Accurate> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kGaussF64> { using T = double; static constexpr bool kPair = true; };
template <> struct XformTraits<kLognF32Fast> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kLognF32FastUnit> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kLognF32Accurate> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kLognF64> { using T = double; static constexpr bool kPair = true; };
template <> struct XformTraits<kGaussF32Exact> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kGaussF64Exact> { using T = double; static constexpr bool kPair = true; };
template <> struct XformTraits<kGaussF32Precise> { using T = float; static constexpr bool kPair = true; };
template <> struct XformTraits<kLognF32Precise> { using T = float; static constexpr bool kPair = true; };

// Single-word transforms.
template <int X>
__device__ __forceinline__ typename XformTraits<X>::T xform1(uint32_t w, const XformParams& p);

template <> __device__ __forceinline__ uint32_t xform1<kBits>(uint32_t w, const XformParams&) { return w; }

template <> __device__ __forceinline__ float xform1<kUnitF32>(uint32_t w, const XformParams&) { return unit_f32(w); }

template <> __device__ __forceinline__ double xform1<kUnitF64>(uint32_t w, const XformParams&) { return unit_f64(w); }

// fl(fl(u * S) + off) with u = (w >> 8) * 2^-24.  Because the 2^-24 factor is
// a power of two, fl(u * S) == fl((w >> 8) * S') with S' = S * 2^-24 (exact;
// the host only takes this path when S' is a normal number), which saves one
// multiply per sample.  The add is a separate rounding: never an FMA.
template <> __device__ __forceinline__ float xform1<kUniformF32>(uint32_t w, const XformParams& p) {
    return __fadd_rn(__fmul_rn((float)(w >> 8), p.scale_f), p.off_f);
}

// fl(x * S') as fma(2^52 + x, S', -2^52 S'): the FMA's exact intermediate is
// x * S', rounded once (the host keeps 2^52 S' finite, api.cu).
template <> __device__ __forceinline__ double xform1<kUniformF64>(uint32_t w, const XformParams& p) {
    return __dadd_rn(__fma_rn(u24_magic(w), p.scale_d, p.mag_d), p.off_d);
}

// Box-Muller on one word pair (distributions.py:107-131, _core.pyx:116-121):
// u1' = 1 - u1 in (0, 1], r = sqrt(-2 ln u1'), t = 2 pi u2, (r cos t, r sin t).
//
// Accurate (fp64) route, specialised to the 24-bit inputs (the general
// libdevice log/sincos cost ~3x more; the reference's own libm formula is the
// oracle):
//  * -2 ln u1' with u1' = m 2^-24: m = f 2^e, f in [sqrt(1/2), sqrt(2)),
//    ln f = 2 atanh(s), s = (f-1)/(f+1), |s| <= 0.1716, series to s^19
//    (truncation < 2^-56); g = f - 1 is exact so the relative accuracy holds
//    as u1' -> 1; e ln2 with a split constant;
//  * r = sqrt(.) (IEEE);
//  * cos/sin(2 pi k 2^-24), k = w1 >> 8: exact integer quadrant reduction,
//    t in [-1, 1) exact, Taylor polynomials of pi t / 4 to t^17 / t^18
//    (truncation < 1e-19).  The reference evaluates cos(fl(2 pi u2)); the
//    argument rounding it carries (<= 2^-51 absolute) is inside the stated
//    tolerance.
// fp64 coefficients live in the constant bank: DFMA takes c[][] operands
// directly, whereas 64-bit literals cost two UMOVs per use inside the loop.
__constant__ double kAtanhC[9] = {0.3333333333333333,  0.2,  0.14285714285714285, 0.1111111111111111,
                                  0.09090909090909091, 0.07692307692307693, 0.06666666666666667,
                                  0.058823529411764705, 0.05263157894736842};  // 1/(2k+1), k = 1..9
__constant__ double kLn2Split[2] = {0.6931467056274414, 4.7493250390316726e-07};
__constant__ double kSinC[9] = {0.7853981633974483,     -0.08074551218828079,   0.0024903945701927202,
                                -3.657620418217725e-05, 3.1336168903781217e-07, -1.757247673443401e-09,
                                6.948453273886629e-12,  -2.0410263396641442e-14, 4.628704628834683e-17};
__constant__ double kCosC[10] = {1.0,                    -0.30842513753404244,   0.015854344243815502,
                                 -0.00032599188692739,   3.59086044859151e-06,   -2.4611369504942e-08,
                                 1.1501159127974052e-10, -3.8980731712596753e-13, 1.001886461636272e-15,
                                 -2.019653396886682e-18};

// log(u1'), u1' = 1 - (w0 >> 8) 2^-24 = m 2^-24 (intrinsics only: no
// contraction freedom, so the exact method's correction tables, built by
// running this same code, stay valid).
template <int TERMS = 9>
__device__ __forceinline__ double log_u1_f64_t(uint32_t w0) {
    const double x = __uint2double_rn(16777216u - (w0 >> 8));  // m, exact, in [1, 2^24]
    const int hi = __double2hiint(x);
    const int e = (hi - 0x3FE6A09E) >> 20;  // 0x3FE6A09E: high word of sqrt(1/2)
    const double f = __hiloint2double(hi - (e << 20), __double2loint(x));
    const double g = __dsub_rn(f, 1.0);  // exact
    const double d = __dadd_rn(f, 1.0);
    double rd;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(d));
    double er = __fma_rn(-d, rd, 1.0);
    rd = __fma_rn(rd, er, rd);
    er = __fma_rn(-d, rd, 1.0);
    rd = __fma_rn(rd, er, rd);
    const double s = __dmul_rn(g, rd);
    const double z = __dmul_rn(s, s);
    double p = kAtanhC[TERMS - 1];
#pragma unroll
    for (int i = TERMS - 2; i >= 0; --i) p = __fma_rn(p, z, kAtanhC[i]);
    const double s2 = __dmul_rn(2.0, s);
    const double lnf = __fma_rn(s2, __dmul_rn(z, p), s2);
    const double ee = (double)(e - 24);
    return __fma_rn(ee, kLn2Split[0], __fma_rn(ee, kLn2Split[1], lnf));
}

template <int SIN_TERMS = 9, int COS_TERMS = 10>
__device__ __forceinline__ void sincos_2pi_k24_f64_t(uint32_t k, double& sn, double& cs) {
    const uint32_t kk = k + (1u << 21);
    const uint32_t q = (kk >> 22) & 3u;
    const double t = __dmul_rn((double)((int)(kk & 0x3FFFFFu) - (1 << 21)), 4.76837158203125e-07);  // exact
    const double t2 = __dmul_rn(t, t);
    double s = kSinC[SIN_TERMS - 1];
#pragma unroll
    for (int i = SIN_TERMS - 2; i >= 0; --i) s = __fma_rn(s, t2, kSinC[i]);
    s = __dmul_rn(s, t);
    double c = kCosC[COS_TERMS - 1];
#pragma unroll
    for (int i = COS_TERMS - 2; i >= 0; --i) c = __fma_rn(c, t2, kCosC[i]);
    const bool swap = q & 1u;
    const double a = swap ? s : c;
    const double b = swap ? c : s;
    cs = (((q + 1u) >> 1) & 1u) ? -a : a;
    sn = (q >> 1) ? -b : b;
}

// (sin t, cos t) of the reference's argument t = fl(TWO_PI * u2)
// (distributions.py:125, _core.pyx:119): t = 2 pi u2 + delta with
// delta = fl(TWO_PI u2) - TWO_PI u2 - (2 pi - TWO_PI) u2, |delta| < 1e-15;
// a first-order correction on the exactly reduced 2 pi k 2^-24 reproduces it
// (and the reference's non-zero values at the quadrant points, e.g.
// cos(fl(pi/2))).
__device__ __forceinline__ double log_u1_f64(uint32_t w0) { return log_u1_f64_t<9>(w0); }
__device__ __forceinline__ void sincos_2pi_k24_f64(uint32_t k, double& sn, double& cs) {
    sincos_2pi_k24_f64_t<9, 10>(k, sn, cs);
}

// Shorter forms for the fp32 exact route's common path (~2^-44 instead of a
// few ulps; no first-order argument-rounding term): its rounding test only
// needs an error BOUND, which the table build measures over both whole
// domains (exact_fast_bounds_kernel).
#ifndef PRNG_EXACT_SHORT
#define PRNG_EXACT_SHORT 1
#endif
__device__ __forceinline__ double log_u1_f64_short(uint32_t w0) { return log_u1_f64_t<PRNG_EXACT_SHORT ? 7 : 9>(w0); }
__device__ __forceinline__ void sincos_f64_short(uint32_t w1, double& sn, double& cs) {
    sincos_2pi_k24_f64_t<PRNG_EXACT_SHORT ? 7 : 9, PRNG_EXACT_SHORT ? 8 : 10>(w1 >> 8, sn, cs);
}

__device__ __forceinline__ void sincos_ref_f64(uint32_t w1, double& sn, double& cs) {
    double s, c;
    sincos_2pi_k24_f64(w1 >> 8, s, c);
    const double u2 = unit_f64(w1);
    const double t = __dmul_rn(kTwoPi, u2);
    const double delta = __fma_rn(-2.4492935982947064e-16, u2, -__fma_rn(kTwoPi, u2, -t));
    cs = __fma_rn(-delta, s, c);
    sn = __fma_rn(delta, c, s);
}

__device__ __forceinline__ void box_muller_f64(uint32_t w0, uint32_t w1, double& z0, double& z1) {
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log_u1_f64(w0)));
    double s, c;
    sincos_ref_f64(w1, s, c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

// ---- exact route: approximations above + per-input ulp corrections ----
// Order-preserving integer key of a double (adjacent doubles differ by 1;
// +0 and -0 both map to 0).
__device__ __host__ __forceinline__ long long dkey(long long b) {
    return b >= 0 ? b : -(b & 0x7FFFFFFFFFFFFFFFll);
}
__device__ __host__ __forceinline__ long long dunkey(long long k) {
    return k >= 0 ? k : ((-k) | (long long)0x8000000000000000ull);
}

__device__ __noinline__ double exact_escape(const uint32_t* idx, const double* val, uint32_t n, uint32_t i) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (idx[mid] < i) lo = mid + 1; else hi = mid;
    }
    return val[lo];
}

__device__ __forceinline__ int nib_delta(uint32_t v) { return (int)((v & 0xFu) ^ 8u) - 8; }

__device__ __forceinline__ double corrected(double approx, int d, const ExactCorrections& x, int tab, uint32_t i) {
    if (d == -8) return exact_escape(x.esc_idx[tab], x.esc_val[tab], x.esc_n[tab], i);
    return __longlong_as_double(dunkey(dkey(__double_as_longlong(approx)) + d));
}

// Fast (fp32) route, specialised to the 24-bit inputs (DESIGN.md
// "Tolerances"; accuracy measured exhaustively over the 2^24-point grids by
// the GPU tests: worst error 0.2-0.6 of the stated tolerance).
//  * -lg2(1 - u1) by one MUFU.LG2 for u1 >= 2^(SER - 24); below, the series
//    x (1 + x/2 + x^2/3)/ln 2 (truncation x^3/4 < 2^-26 relative), so r keeps
//    its relative accuracy as u1' -> 1.  Working in lg2 units saves the
//    -2 ln 2 multiply: r = sqrt(-lg2(1 - u1)) * sqrt(2 ln 2), and the
//    sqrt(2 ln 2) is folded into the caller's loop-invariant scale.
//  * r by MUFU.SQRT (relative error <= 2^-23.2, exhaustive);
//  * (sin, cos)(2 pi k 2^-24) by angle addition from the NEAREST point of a
//    per-CTA shared-memory table of (sin, cos)(2 pi j / 2^TL) (kernel
//    prologue, sincos_tab_entry), residual |x| <= pi 2^-TL: sin x = x,
//    cos x = 1 - x^2/2 (TL < 12) or 1 (TL >= 12: relative x^2/2 <= 2^-21.7).
//    See sincos_2pi_k24 (tools/bm_variants.cu measured the variants).
#ifndef PRNG_BM_TAB_LOG2
#define PRNG_BM_TAB_LOG2 12
#endif
#ifndef PRNG_BM_SER_LOG2K  // series for k < 2^PRNG_BM_SER_LOG2K, i.e. u1 < 2^(LOG2K - 24)
#define PRNG_BM_SER_LOG2K 16
#endif
#ifndef PRNG_BM_SER_TERMS
#define PRNG_BM_SER_TERMS 3
#endif
#ifndef PRNG_BM_COS_QUAD_BELOW  // keep the cos x^2/2 term for tables smaller than 2^this
#define PRNG_BM_COS_QUAD_BELOW 12
#endif
constexpr int kPhiloxTabLog2 = PRNG_BM_TAB_LOG2;  // Philox / words kernels (32 KB at 12)
constexpr int kMrgTabLog2 = 10;                   // MRG kernel: 8 KB next to its 32 KB store stage
constexpr float kBmRq = 1.1774100225154747f;      // sqrt(2 ln 2): r = rq * kBmRq

template <int TL>
__device__ __forceinline__ float2* sincos_tab() {
    __shared__ float2 tab[1 << TL];
    return tab;
}

// The fast gaussian's table holds (sin, cos) * stddev * sqrt(2 ln 2), so the
// per-pair r scaling multiply disappears (one more rounding on the table:
// exhaustive worst err/allowed 0.658 vs 0.669; +2% at 2^30); the lognormal's
// also folds log2(e), removing the exp's argument multiplies.
template <int X>
constexpr bool bm_table_scaled() {
    return is_f32_table_route(X);
}
constexpr float kLog2E = 1.4426950408889634f;

// (sin, cos) of the reference's angle fl64(TWO_PI * u2) at table point i of
// 2^TL (fp32): sincospif's exactly-rounded values, except that the quadrant
// points carry the reference's non-zero residues cos(fl(pi/2)),
// sin(fl(pi)), cos(fl(3 pi/2)) (exact zeros would be infinitely many ulps
// from the reference's tiny outputs there).
template <int TL>
__device__ __forceinline__ void sincos_tab_entry(int i, float& sn, float& cs) {
    sincospif((float)i * (2.0f / (1 << TL)), &sn, &cs);
    constexpr int Q = 1 << (TL - 2);
    if ((i & (Q - 1)) == 0) {
        const int q = i / Q;
        sn = q == 0 ? 0.0f : q == 1 ? 1.0f : q == 2 ? 1.2246467991473532e-16f : -1.0f;
        cs = q == 0 ? 1.0f : q == 1 ? 6.123233995736766e-17f : q == 2 ? -1.0f : -1.8369701987210297e-16f;
    }
}

// Precise route: -lg2(1 - u1) from a table over the float bits of
// omx = 1 - u1 (exact): 64 buckets per binade (idx = bits >> 17) for omx in
// [2^-24, 1].  Entry (inv, lg2(inv)) with inv = the largest fp32 <= 1 / (the
// bucket's end), so r = 1 - omx inv is in [0, 2^-6] and
// -lg2(omx) = lg2(inv) - lg2(1 - r) = lg2(inv) + (r + r^2/2 + r^3/3 + r^4/4)/ln 2
// (truncation r^4/5 < 2^-26 relative): two non-negative terms, so the result
// keeps its relative accuracy as u1 -> 0 (where lg2.approx's error is
// absolute).  12 KB next to the 32 KB sin/cos table.
constexpr int kLogTabIdx0 = 103 << 6;                          // bits(2^-24) >> 17
constexpr int kLogTabEntries = (127 << 6) - kLogTabIdx0 + 1;  // ... bits(1.0) >> 17

__device__ __forceinline__ float2* log_tab() {
    __shared__ float2 tab[kLogTabEntries];
    return tab;
}

template <int X, int TL = kPhiloxTabLog2>
__device__ __forceinline__ void xform_prologue(const XformParams& p) {
    if constexpr (is_f32_table_route(X)) {
        float2* tab = sincos_tab<TL>();
        // lognormal: also log2(e), so exp(m + s z) = ex2(fma(rq, cs', m log2(e)))
        const float S = !bm_table_scaled<X>()               ? 1.0f
                        : (is_logn_fast(X) || X == kLognF32Precise) ? p.scale_f * kBmRq * kLog2E
                                                             : p.scale_f * kBmRq;
        for (int i = threadIdx.x; i < (1 << TL); i += blockDim.x) {
            float sn, cs;
            sincos_tab_entry<TL>(i, sn, cs);
            tab[i] = bm_table_scaled<X>() ? make_float2(sn * S, cs * S) : make_float2(sn, cs);
        }
        if constexpr (is_precise(X)) {
            float2* lt = log_tab();
            for (int i = threadIdx.x; i < kLogTabEntries; i += blockDim.x) {
                const uint32_t idx = kLogTabIdx0 + i;
                float inv = 1.0f;
                if (idx != (127u << 6)) {
                    inv = __double2float_rd(1.0 / (double)__uint_as_float((idx + 1) << 17));
                    if (inv < 1.0f) inv = 1.0f;
                }
                lt[i] = make_float2(inv, (float)log2((double)inv));
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ float neg_lg2_1mu_precise(uint32_t w0) {
    constexpr float c1 = 1.4426950408889634f, c2 = 0.7213475204444817f, c3 = 0.48089834696298783f,
                    c4 = 0.36067376022224085f;  // 1/(j ln 2)
    const float kf = __uint2float_rn(w0 >> 8);
    const float omx = fmaf(kf, -5.9604644775390625e-08f, 1.0f);  // 1 - u1, exact, in [2^-24, 1]
    const float2 e = log_tab()[(__float_as_uint(omx) >> 17) - kLogTabIdx0];
    const float r = fmaf(-omx, e.x, 1.0f);
    float q = fmaf(r, c4, c3);
    q = fmaf(q, r, c2);
    q = fmaf(q, r, c1);
    return fmaf(r, q, e.y);
}

__device__ __forceinline__ float neg_lg2_1mu(uint32_t w0) {
    const uint32_t k = w0 >> 8;
    const float kf = __uint2float_rn(k);
    const float omx = fmaf(kf, -5.9604644775390625e-08f, 1.0f);  // 1 - u1, exact
    float l2;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(omx));     // 1 - u1 >= 2^-24: normal
    if constexpr (PRNG_BM_SER_LOG2K == 0) {
        return -l2;
    } else {
        // x (1 + x/2 + x^2/3 ...) / ln 2 with x = u1 = kf 2^-24, evaluated on kf
        // with the coefficients pre-scaled by 2^(-24 (j + 1)): every
        // intermediate is the x-form's value times a power of two, so the
        // roundings (and the result) are identical, one multiply fewer.
        constexpr float c[5] = {1.4426950408889634f * 0x1p-24f, 0.7213475204444817f * 0x1p-48f,
                                0.48089834696298783f * 0x1p-72f, 0.36067376022224085f * 0x1p-96f,
                                0.28853900817779266f * 0x1p-120f};  // 1/(j ln 2) 2^(-24 j)
        static_assert(PRNG_BM_SER_TERMS <= 4, "the fifth scaled coefficient is near the fp32 normal limit");
        float p = c[PRNG_BM_SER_TERMS - 1];
#pragma unroll
        for (int j = PRNG_BM_SER_TERMS - 2; j >= 0; --j) p = fmaf(p, kf, c[j]);
        return k < (1u << PRNG_BM_SER_LOG2K) ? kf * p : -l2;
    }
}

// sin/cos(2 pi k 2^-24), k = w1 >> 8, by angle addition from the table
// point NEAREST to the angle (round-to-nearest index: (w1 + half a bucket)
// >> (32 - TL), wrapping to 0 at 2 pi): the quadrant points are table points,
// so results near the zeros of sin/cos keep their relative accuracy, and the
// residual angle |x| <= pi 2^-TL is half the truncated form's.  x is built
// without I2FP or a shift: the L = 24 - TL low bits of k stay in place as
// mantissa bits [8, 8 + L) under 1.0f (one LOP3), f - (1 + 2^(L-1) 2^-15)
// is the signed offset from the bucket centre times 2^-15 (exact), times
// 2 pi 2^-9.  sin x = x and cos x = 1 for TL >= 12 (|x| <= 7.7e-4:
// relative x^2/2 <= 2^-21.7), cos x = 1 - x^2/2 below.
template <int TL, bool QUAD = (TL < PRNG_BM_COS_QUAD_BELOW)>
__device__ __forceinline__ void sincos_2pi_k24(uint32_t w1, float& sn, float& cs) {
    constexpr int L = 24 - TL;  // low bits of k left to the polynomial
    static_assert(L >= 1 && L <= 15, "table size");
    const uint32_t wc = w1 + (1u << (31 - TL));
    const float2 t = sincos_tab<TL>()[wc >> (32 - TL)];
    uint32_t fb;  // (wc & mask) | bits(1.0f) as ONE 3-input LOP3 (one operand in a register)
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(fb) : "r"(wc), "n"(((1u << L) - 1u) << 8), "r"(0x3F800000u));
    constexpr float kCentre = 1.0f + (float)(1u << (L - 1)) * 3.0517578125e-05f;  // 1 + 2^(L-1) 2^-15
    const float d = __fsub_rn(__uint_as_float(fb), kCentre);                         // exact
    const float x = __fmul_rn(d, 0.01227184630308513f);                              // 2 pi 2^-9
    if constexpr (QUAD) {
        const float nh = __fmul_rn(x, __fmul_rn(x, -0.5f));
        sn = fmaf(t.y, x, fmaf(t.x, nh, t.x));
        cs = fmaf(-t.x, x, fmaf(t.y, nh, t.y));
    } else {
        sn = fmaf(t.y, x, t.x);
        cs = fmaf(-t.x, x, t.y);
    }
}

// (rq, sin, cos) of the fast route, r = rq * kBmRq.
template <int TL>
__device__ __forceinline__ void box_muller_f32_parts(uint32_t w0, uint32_t w1, float& rq, float& sn, float& cs) {
    const float s = neg_lg2_1mu(w0);
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"(s));  // s = 0 or >= 1.7e-7
    sincos_2pi_k24<TL>(w1, sn, cs);
}

// Precise route: table log, sqrt.approx, centred sin/cos with the x^2 term.
template <int TL>
__device__ __forceinline__ void box_muller_f32_parts_precise(uint32_t w0, uint32_t w1, float& rq, float& sn,
                                                             float& cs) {
    const float s = neg_lg2_1mu_precise(w0);
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"(s));
    sincos_2pi_k24<TL, true>(w1, sn, cs);
}

template <int X>
__device__ __forceinline__ void xform2(uint32_t w0, uint32_t w1, const XformParams& p,
                                       typename XformTraits<X>::T& o0, typename XformTraits<X>::T& o1);

template <> __device__ __forceinline__ void xform2<kGaussF64>(uint32_t w0, uint32_t w1, const XformParams& p,
                                                             double& o0, double& o1) {
    double z0, z1;
    box_muller_f64(w0, w1, z0, z1);
    o0 = __dadd_rn(__dmul_rn(z0, p.scale_d), p.off_d);
    o1 = __dadd_rn(__dmul_rn(z1, p.scale_d), p.off_d);
}

template <> __device__ __forceinline__ void xform2<kGaussF32Accurate>(uint32_t w0, uint32_t w1, const XformParams& p,
                                                                     float& o0, float& o1) {
    double z0, z1;
    box_muller_f64(w0, w1, z0, z1);
    o0 = (float)__dadd_rn(__dmul_rn(z0, p.scale_d), p.off_d);
    o1 = (float)__dadd_rn(__dmul_rn(z1, p.scale_d), p.off_d);
}


// Exact route: the reference evaluates r = sqrt(-2.0 * log(u1')), t =
// TWO_PI * u2, (r cos t, r sin t) in fp64 with the host libm (_core.pyx:
// 116-121).  u1' = m 2^-24 (m in [1, 2^24]) and u2 = k 2^-24 (k < 2^24) take
// only 2^24 values each, so the library runs the device approximations
// (log_u1_f64, sincos_ref_f64: a few ulps) once over both whole domains,
// compares them with the host libm's log/sin/cos and keeps the difference
// in ulps as 4-bit corrections (24 MB, L2-resident; the rare larger
// differences go to sorted escape lists).  Approximation + correction is
// the host libm's value bit for bit; the remaining operations (exact -2x
// scaling, IEEE sqrt, two products, the affine) are correctly rounded on
// both sides, so every output is bit-identical to the reference's.
__device__ __forceinline__ void box_muller_exact(uint32_t w0, uint32_t w1, const XformParams& p, double& z0,
                                                 double& z1) {
    const ExactCorrections& x = p.exact;
    const uint32_t mi = 16777215u - (w0 >> 8);  // m - 1
    const uint32_t k = w1 >> 8;
    const uint32_t lb = __ldg(x.log_nib + (mi >> 1));
    const uint32_t sb = __ldg(x.sc_nib + k);
    const double L = corrected(log_u1_f64(w0), nib_delta(lb >> ((mi & 1u) * 4)), x, 0, mi);
    double s, c;
    sincos_ref_f64(w1, s, c);
    s = corrected(s, nib_delta(sb), x, 1, k);
    c = corrected(c, nib_delta(sb >> 4), x, 2, k);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, L));
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

template <> __device__ __forceinline__ void xform2<kGaussF64Exact>(uint32_t w0, uint32_t w1, const XformParams& p,
                                                                  double& o0, double& o1) {
    double z0, z1;
    box_muller_exact(w0, w1, p, z0, z1);
    o0 = __dadd_rn(__dmul_rn(z0, p.scale_d), p.off_d);  // z *= stddev; z += mean (distributions.py:128-129)
    o1 = __dadd_rn(__dmul_rn(z1, p.scale_d), p.off_d);
}

// fp32 exact route (Ziv's rounding test).  The reference's fp32 output is
// RN32(v), v = fl(fl(z sd) + mean), z its fp64 Box-Muller value.  The
// uncorrected device value v' (the short fp64 approximations) differs from
// v by at most
//   sd (|z'| (rel_log / 2 + 4 u) + r' abs_sc) + 2 u (sd |z'| + |v'|)
//   <= C (sd r' + |v'|),   C = rel_log / 2 + abs_sc + 6 u,  u = 2^-53
// (sqrt and the products rounded on both sides, |z'| <= r'; rel_log and
// abs_sc measured over the whole domains when the tables are built); the
// test uses twice that, evaluated in fp32.  RN32(v') == RN32(v) unless v'
// lies within it of an fp32 rounding boundary -- i.e. unless the 29 mantissa
// bits fp32 drops are within tol / ulp64(v') of 2^28 -- and only then
// (~2^-20 of the pairs, plus |v'| outside [2^-74, 2^127)) are the correction
// tables read.  The test is integer / fp32 work; the FP64 pipe does only the
// accurate route's formula.
__device__ __forceinline__ bool f32_rounding_uncertain(double v, float tol) {
    const uint32_t lo = (uint32_t)__double2loint(v);
    const uint32_t e = ((uint32_t)__double2hiint(v) >> 20) & 0x7FFu;  // biased fp64 exponent
    if (e < 949u || e > 1149u) return true;  // |v| < 2^-74 or >= 2^127
    const int d = abs((int)(lo & 0x1FFFFFFFu) - (1 << 28));  // ulp64s to the boundary
    const float ulp = __uint_as_float((e - 948u) << 23);     // 2^(e - 1075) = ulp64(v)
    return (float)d * ulp <= tol;
}

// The corrected pair (rare path of the fp32 exact route), out of line so the
// common path keeps its registers.
#ifndef PRNG_EXACT_NOINLINE
#define PRNG_EXACT_NOINLINE 0
#endif
#if PRNG_EXACT_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void exact_pair_f32(uint32_t w0, uint32_t w1, double sd, double mean, const ExactCorrections x, float& o0,
                    float& o1) {
    XformParams q{};
    q.scale_d = sd;
    q.off_d = mean;
    q.exact = x;
    double a, b;
    box_muller_exact(w0, w1, q, a, b);
    o0 = (float)__dadd_rn(__dmul_rn(a, sd), mean);
    o1 = (float)__dadd_rn(__dmul_rn(b, sd), mean);
}

// The common path of the fp32 exact route: the uncorrected pair and whether
// either output's rounding is uncertain (then exact_pair_f32 decides).
__device__ __forceinline__ bool gauss_f32_exact_try(uint32_t w0, uint32_t w1, const XformParams& p, float& o0,
                                                    float& o1) {
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log_u1_f64_short(w0)));
    double s, c;
    sincos_f64_short(w1, s, c);
    const double v0 = __dadd_rn(__dmul_rn(__dmul_rn(r, c), p.scale_d), p.off_d);
    const double v1 = __dadd_rn(__dmul_rn(__dmul_rn(r, s), p.scale_d), p.off_d);
    o0 = (float)v0;  // .astype(float32) (distributions.py:131)
    o1 = (float)v1;
    const float base = p.exact.tol_c * p.scale_f * (float)r;
    return f32_rounding_uncertain(v0, fmaf(p.exact.tol_c, fabsf(o0), base)) ||
           f32_rounding_uncertain(v1, fmaf(p.exact.tol_c, fabsf(o1), base));
}

template <> __device__ __forceinline__ void xform2<kGaussF32Exact>(uint32_t w0, uint32_t w1, const XformParams& p,
                                                                  float& o0, float& o1) {
    if (gauss_f32_exact_try(w0, w1, p, o0, o1)) exact_pair_f32(w0, w1, p.scale_d, p.off_d, p.exact, o0, o1);
}

// Lognormal (extension a18): x = exp(m + s*z) * scale + displ.
template <> __device__ __forceinline__ void xform2<kLognF64>(uint32_t w0, uint32_t w1, const XformParams& p,
                                                            double& o0, double& o1) {
    double z0, z1;
    box_muller_f64(w0, w1, z0, z1);
    const double g0 = __dadd_rn(__dmul_rn(z0, p.scale_d), p.off_d);
    const double g1 = __dadd_rn(__dmul_rn(z1, p.scale_d), p.off_d);
    o0 = __dadd_rn(__dmul_rn(exp(g0), p.ln_scale), p.ln_displ);
    o1 = __dadd_rn(__dmul_rn(exp(g1), p.ln_scale), p.ln_displ);
}

template <> __device__ __forceinline__ void xform2<kLognF32Accurate>(uint32_t w0, uint32_t w1, const XformParams& p,
                                                                    float& o0, float& o1) {
    double a, b;
    xform2<kLognF64>(w0, w1, p, a, b);
    o0 = (float)a;
    o1 = (float)b;
}


// Pair transform as called by the kernels: the fast fp32 routes read the
// sin/cos table of the calling kernel's size TL (xform_prologue<X, TL>).
template <int X, int TL = kPhiloxTabLog2>
__device__ __forceinline__ void xform2k(uint32_t w0, uint32_t w1, const XformParams& p,
                                        typename XformTraits<X>::T& o0, typename XformTraits<X>::T& o1) {
    if constexpr (is_f32_table_route(X)) {
        float rq, sn, cs;
        if constexpr (is_precise(X))
            box_muller_f32_parts_precise<TL>(w0, w1, rq, sn, cs);
        else
            box_muller_f32_parts<TL>(w0, w1, rq, sn, cs);
        // stddev and sqrt(2 ln 2) folded into r (loop-invariant) or into the table
        const float rs = bm_table_scaled<X>() ? rq : rq * (p.scale_f * kBmRq);
        if constexpr (X == kGaussF32Fast || X == kGaussF32Precise) {
            o0 = fmaf(rs, cs, p.off_f);
            o1 = fmaf(rs, sn, p.off_f);
        } else {
            // table scaled by s sqrt(2 ln 2) log2(e): the exponent in base 2 is one
            // FMA; ex2.approx (~2^-22 rel)
            const float off2 = p.off_f * kLog2E;  // loop-invariant
            float e0, e1;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(fmaf(rs, cs, off2)));
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(fmaf(rs, sn, off2)));
            if constexpr (X == kLognF32FastUnit) {  // fma(e, 1, 0) == e
                o0 = e0;
                o1 = e1;
            } else {
                o0 = fmaf(e0, p.ln_scale_f, p.ln_displ_f);
                o1 = fmaf(e1, p.ln_scale_f, p.ln_displ_f);
            }
        }
    } else {
        xform2<X>(w0, w1, p, o0, o1);
    }
}

// Four consecutive stream words -> four outputs.  For pair transforms the
// group must start on a pair boundary (relative to the request start).
template <int X>
__device__ __forceinline__ void xform4(const U4& w, const XformParams& p, typename XformTraits<X>::T o[4]) {
    if constexpr (XformTraits<X>::kPair) {
        xform2k<X>(w.x, w.y, p, o[0], o[1]);
        xform2k<X>(w.z, w.w, p, o[2], o[3]);
    } else {
        o[0] = xform1<X>(w.x, p);
        o[1] = xform1<X>(w.y, p);
        o[2] = xform1<X>(w.z, p);
        o[3] = xform1<X>(w.w, p);
    }
}

// ---------------------------------------------------------------- stores
// Streaming (evict-first) vector stores: every sample is written once and
// never re-read by the kernel.
__device__ __forceinline__ void st_group(uint32_t* p, const uint32_t o[4]) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                 : "memory");
}
__device__ __forceinline__ void st_group(float* p, const float o[4]) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(o[0]), "f"(o[1]), "f"(o[2]), "f"(o[3])
                 : "memory");
}
__device__ __forceinline__ void st_group(double* p, const double o[4]) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(o[0]), "d"(o[1]), "d"(o[2]), "d"(o[3])
                 : "memory");
}
// Two adjacent 4-byte groups as one 256-bit store.
__device__ __forceinline__ void st_group2(uint32_t* p, const uint32_t a[4], const uint32_t b[4]) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a[0]), "r"(a[1]), "r"(a[2]),
                 "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3])
                 : "memory");
}
__device__ __forceinline__ void st_group2(float* p, const float a[4], const float b[4]) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]),
                 "f"(a[3]), "f"(b[0]), "f"(b[1]), "f"(b[2]), "f"(b[3])
                 : "memory");
}

}  // namespace prng
