/*
 * prng_b200.h -- C ABI of the B200-native RNG hot path (libprng_b200.so).
 *
 * Drop-in for the portarng kernel plugin (reference seam
 * pkg/src/portarng/_kernels/__init__.py:10-27) and for the fused
 * generate -> transform cycle the reference runs as two passes
 * (rngburn.py:62-151, distributions.py:83-153).
 *
 * Conventions
 *  - Plain pointers and sizes only; no allocation on the device entry points,
 *    no host synchronisation, stream-ordered on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  The device is taken from `out` for the
 *    duration of the call; the caller's current device is restored on
 *    return.  (One exception: the first PRNG_METHOD_EXACT request on a
 *    device builds its correction tables -- see below.)
 *  - `out` is caller-owned device memory (or mapped pinned host memory),
 *    aligned to its element size.
 *  - Philox state arguments are exactly those of the reference kernel
 *    philox_fill(k0, k1, b0, b1, b2, b3, offset, n) (_core.pyx:42):
 *    key (k0, k1), 128-bit block counter ctr[0..3] (lane 0 least
 *    significant) and `lane` = words of that block already consumed (0..3).
 *    From an engine state at stream position p: ctr = p >> 2, lane = p & 3
 *    (engine.py:221-225).
 *  - MRG32k3a state arguments are the two recurrence windows s1[3], s2[3]
 *    (Mrg32k3aState, engine.py:75-80), components < m1 / m2, not all zero.
 *  - Return 0 on success or a negative PRNG_ERR_* code; prng_last_error()
 *    returns the message for the calling thread.
 *  - The word stream consumed by a request is the reference's: n words for
 *    bits/uniform, 2*ceil(n/2) for gaussian/lognormal (fill_gaussian,
 *    distributions.py:146-149), pairs taken relative to the request start.
 */
#ifndef PRNG_B200_H
#define PRNG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRNG_ABI_VERSION 1

/* Status codes: 1:1 with the reference exception types (errors.py). */
#define PRNG_OK 0
#define PRNG_ERR_UNSUPPORTED_ENGINE (-1) /* errors.py:8  UnsupportedEngine */
#define PRNG_ERR_INVALID_RANGE (-2)      /* errors.py:12 InvalidRange      */
#define PRNG_ERR_INVALID_PARAMETER (-3)  /* errors.py:16 InvalidParameter  */
#define PRNG_ERR_VALUE (-4)              /* ValueError (engine.py:206,219) */
#define PRNG_ERR_CUDA (-5)               /* CUDA runtime failure           */

/* Gaussian / lognormal fp32 method.  FAST: fp32 SFU lg2/sqrt with a short
 * series near u1 = 0 and a shared-memory sin/cos table with angle addition
 * (documented tolerance).  ACCURATE: the reference's
 * fp64 formula, then cast (fp64 outputs always use ACCURATE). */
#define PRNG_METHOD_FAST 0
#define PRNG_METHOD_ACCURATE 1
/* Gaussian only (fp32 and fp64): bit-identical to the reference's fp64
 * Box-Muller (_core.pyx:116-121 with the host libm): the device
 * approximations of log(u1') and (sin t, cos t) are corrected to the host
 * libm's values by 4-bit ulp deltas tabulated over their whole 2^24-point
 * domains (~24 MB per device plus short escape lists, built once per
 * device; prng_exact_tables_prepare builds them ahead of the first
 * request).  The build runs on a private stream in relaxed capture mode, so
 * a first exact request inside CUDA-graph capture works; it blocks the
 * calling thread for about a second. */
#define PRNG_METHOD_EXACT 2
/* fp32 gaussian / lognormal: relative accuracy everywhere at ~85% of FAST's
 * throughput -- -lg2(1 - u1) from a 12 KB table over the bits of 1 - u1 plus
 * a 4-term series (no SFU log), sqrt.approx, and sin/cos from the nearest
 * point of a 4096-entry table with the x^2 term.  Gaussian within 5 ulp of
 * the reference for every input (exhaustive over both 24-bit grids),
 * lognormal within 5 ulp * max(1, |ln x|).  MRG32k3a
 * requests take ACCURATE (its kernel's shared memory holds the store stage);
 * fp64 outputs take ACCURATE. */
#define PRNG_METHOD_PRECISE 3

int prng_abi_version(void);
const char *prng_last_error(void);

/* ---- Philox4x32-10: replaces _core.philox_fill (_core.pyx:42-71) + the
 *      words_to_unit / range_transform / Box-Muller passes. ---- */

/* uniform_bits uint32: engine.generate_words (engine.py:212-226) */
int prng_philox4x32x10_bits(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                            uint32_t *out, void *stream);
/* uniform on [a, b): fill_uniform_unit + range_transform (distributions.py:90-104) */
int prng_philox4x32x10_uniform_f32(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                                   double a, double b, float *out, void *stream);
int prng_philox4x32x10_uniform_f64(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                                   double a, double b, double *out, void *stream);
/* gaussian: fill_gaussian (distributions.py:134-153) */
int prng_philox4x32x10_gaussian_f32(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                                    double mean, double stddev, int method, float *out, void *stream);
int prng_philox4x32x10_gaussian_f64(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                                    double mean, double stddev, double *out, void *stream);
int prng_philox4x32x10_gaussian_f64_method(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane,
                                           uint64_t n, double mean, double stddev, int method, double *out,
                                           void *stream);
/* lognormal (extension; oneMKL lognormal(m, s, displ, scale)) */
int prng_philox4x32x10_lognormal_f32(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                                     double m, double s, double displ, double scale, int method, float *out,
                                     void *stream);
int prng_philox4x32x10_lognormal_f64(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t lane, uint64_t n,
                                     double m, double s, double displ, double scale, double *out, void *stream);

/* ---- MRG32k3a: replaces _core.mrg_fill (_core.pyx:74-102), split across
 *      threads by jump-ahead.  The caller advances its state with
 *      prng_mrg32k3a_skip_ahead(s, n) (or 2*ceil(n/2) for pair dists). ---- */
int prng_mrg32k3a_bits(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, uint32_t *out, void *stream);
int prng_mrg32k3a_uniform_f32(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double a, double b,
                              float *out, void *stream);
int prng_mrg32k3a_uniform_f64(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double a, double b,
                              double *out, void *stream);
int prng_mrg32k3a_gaussian_f32(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double mean,
                               double stddev, int method, float *out, void *stream);
int prng_mrg32k3a_gaussian_f64(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double mean,
                               double stddev, double *out, void *stream);
int prng_mrg32k3a_gaussian_f64_method(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double mean,
                                      double stddev, int method, double *out, void *stream);
int prng_mrg32k3a_lognormal_f32(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double m, double s,
                                double displ, double scale, int method, float *out, void *stream);
int prng_mrg32k3a_lognormal_f64(const uint32_t s1[3], const uint32_t s2[3], uint64_t n, double m, double s,
                                double displ, double scale, double *out, void *stream);

/* MRG32k3a jump-ahead by k = k_hi * 2^64 + k_lo words (host only; absent in
 * the reference, engine.py:201-202).  s*_out may alias s*. */
int prng_mrg32k3a_skip_ahead(const uint32_t s1[3], const uint32_t s2[3], uint64_t k_lo, uint64_t k_hi,
                             uint32_t s1_out[3], uint32_t s2_out[3]);

/* In-place affine range transform of unit values (distributions.py:98-104),
 * same two-rounding arithmetic as the fused path. */
int prng_range_transform_f32(float *values, uint64_t n, double lo, double hi, void *stream);
int prng_range_transform_f64(double *values, uint64_t n, double lo, double hi, void *stream);

/* Word-array transforms (distributions.py:83-87, 116-131) on device arrays:
 * words_to_unit maps n words; gaussian_from_words reads 2*ceil(n/2) words. */
int prng_words_to_unit_f32(const uint32_t *words, uint64_t n, float *out, void *stream);
int prng_words_to_unit_f64(const uint32_t *words, uint64_t n, double *out, void *stream);
int prng_gaussian_from_words_f32(const uint32_t *words, uint64_t n, double mean, double stddev, int method,
                                 float *out, void *stream);
int prng_gaussian_from_words_f64(const uint32_t *words, uint64_t n, double mean, double stddev, double *out,
                                 void *stream);
int prng_gaussian_from_words_f64_method(const uint32_t *words, uint64_t n, double mean, double stddev, int method,
                                        double *out, void *stream);

/* Exact-method tables: build (host libm) and upload for the current device
 * now instead of at the first PRNG_METHOD_EXACT request; and the host copies
 * (2^24 doubles log(m 2^-24), m = 1..2^24; 2^24 (sin, cos) pairs of
 * fl(TWO_PI k 2^-24)) for inspection. */
int prng_exact_tables_prepare(void);
int prng_exact_tables_host(const double **log_table, const double **sincos_table);
/* The current device's exact tables (built if needed): worst relative error
 * of the short device log approximation and worst absolute error of its
 * sin/cos against the host libm over both whole domains (bounds[0],
 * bounds[1]) -- the fp32 exact route's rounding test uses them -- and the
 * number of escape-list entries of the corrections. */
int prng_exact_tables_bounds(double bounds[2], uint64_t *escapes);

/* ---- Many small batches (FastCaloSim consumer, calosim.py:269-358). ----
 * One launch generates every segment: segment i writes `count` fp32 uniforms
 * on [a, b) of the Philox stream starting at 128-bit word position
 * (pos_hi:pos_lo) to out + out_offset.  `segs` is device memory. */
typedef struct prng_segment {
    uint64_t pos_lo, pos_hi;
    uint64_t count;
    uint64_t out_offset;
} prng_segment_t;
int prng_philox4x32x10_uniform_f32_segments(uint32_t k0, uint32_t k1, const prng_segment_t *segs, uint32_t nseg,
                                            uint64_t max_count, double a, double b, float *out, void *stream);

/* ---- FastCaloSim-style deposition consumer (calosim.simulate_event,
 *      calosim.py:313-347), bit-identical to the reference's numpy
 *      arithmetic.  All arrays are device memory. ---- */
#define PRNG_CALO_MAX_BINS 16
typedef struct prng_calo_particle {
    uint64_t batch_offset; /* first of its 3*hits uniforms in the packed batch buffer */
    uint64_t hit_offset;   /* first of its hits in the per-hit arrays              */
    uint32_t hits;         /* m (calosim.py:296-300)                                */
    uint32_t region;       /* _particle_region (calosim.py:259-262)                 */
    uint32_t param;        /* index into the parameterization table                 */
    uint32_t pad;
    double target;         /* energy * sampling_fraction                            */
} prng_calo_particle_t;
typedef struct prng_calo_param {
    double bin_edges[PRNG_CALO_MAX_BINS + 1];
    double cumw[PRNG_CALO_MAX_BINS]; /* np.cumsum(weights) */
    uint32_t nbins;
    uint32_t pad;
} prng_calo_param_t;
/* Per hit: cell id and raw energy, then per particle the pairwise-summed
 * normalisation to amounts (in place) and the particle sums. */
int prng_calo_hits(const float *batch, const prng_calo_particle_t *particles, uint32_t nparticles,
                   const uint32_t *region_offsets, const uint32_t *region_cells, const prng_calo_param_t *params,
                   uint32_t *hit_cell, double *hit_amount, double *particle_sums, void *stream);
/* Per event (hits [event_hit_offsets[e], event_hit_offsets[e+1])): unique
 * cells ascending with their sequentially summed amounts (np.unique +
 * np.bincount), packed over all events: event e's deposits are
 * dep_cell/dep_energy[dep_offsets[e] .. dep_offsets[e+1]) (dep_offsets has
 * nevents + 1 entries; dep_offsets[nevents] = total deposits <= total_hits).
 * cell_bits: a bound on the cell ids (< 2^cell_bits; 0 = none): ids < 2^18
 * are ranked in one shared-memory bitmap window per event from 0, wider
 * ranges in several windows over the event's min/max; an id at or above an
 * understated bound is detected and its event redone the wide way, so the
 * result never depends on it.
 * scratch: prng_calo_deposit_scratch_bytes(total_hits, nevents) bytes of
 * device memory (look-back state, zeroed by the call on `stream`, and the
 * bucket arrays of events with more than 8192 hits).  One kernel launch. */
size_t prng_calo_deposit_scratch_bytes(uint64_t total_hits, uint32_t nevents);
int prng_calo_deposit(const uint32_t *hit_cell, const double *hit_amount, uint64_t total_hits,
                      const uint64_t *event_hit_offsets, uint32_t nevents, uint32_t cell_bits, void *scratch,
                      size_t scratch_bytes, uint32_t *dep_cell, double *dep_energy, uint64_t *dep_offsets,
                      void *stream);

/* ---- Host-buffer drop-ins for the reference kernel plugin
 *      (portarng._kernels: philox_fill / mrg_fill / box_muller,
 *      _kernels/__init__.py:24-27).  Synchronous; generate on the current
 *      device into library-owned scratch and copy to the host buffer. ---- */
int prng_kernels_philox_fill(uint32_t k0, uint32_t k1, uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3,
                             uint32_t offset, uint64_t n, uint32_t *host_out);
int prng_kernels_mrg_fill(uint32_t s10, uint32_t s11, uint32_t s12, uint32_t s20, uint32_t s21, uint32_t s22,
                          uint64_t n, uint32_t *host_out, uint32_t s1_out[3], uint32_t s2_out[3]);
int prng_kernels_box_muller(const double *u1, const double *u2, uint64_t m, double *z0, double *z1);

/* ---- Diagnostics. ----
 * Write-only roofline probe: fills `bytes` (a multiple of 64) of 32-byte
 * aligned device memory with the grid shape and 256-bit streaming-store
 * pattern of the aligned Philox 4-byte kernel, and no generator arithmetic;
 * bench.py times it next to the headline kernel as the HBM write ceiling. */
int prng_diag_write_probe(void *out, uint64_t bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PRNG_B200_H */
