// calo.cu -- FastCaloSim-style hit deposition on the GPU.
//
// Consumes the per-event uniform batches the generator wrote (segment
// kernel) and reproduces calosim.simulate_event's deposition arithmetic
// (calosim.py:313-347) bit for bit:
//   * per hit: cell = region_cells[min(int(u0 * ncell), ncell-1)];
//     bin = min(#(cumw <= u1), nbins-1) (searchsorted side='right');
//     raw = edges[bin] + u2 * (edges[bin+1] - edges[bin])   (fp64, no FMA);
//   * per particle: raw_sum = numpy's pairwise sum (PW_BLOCKSIZE 128, 8-way
//     unrolled leaves), amounts = raw * (target / raw_sum) (or target / m),
//     particle_sum = pairwise sum of amounts;
//   * per event: deposits = np.unique + np.bincount over the particles' hits
//     in order, i.e. cells ascending and each cell's amounts summed
//     sequentially in hit order: a shared-memory bitmap of the event's cells
//     ranks them (no sort), one warp adds the amounts in hit order, and a
//     decoupled look-back over the events' deposit counts packs the output
//     in the same launch (calo_deposit_kernel) so the host copies back
//     exactly the deposits.  No library kernels.
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/prng_b200.h"

namespace {

constexpr int kCaloThreads = 256;

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), float64,
// leaf branch (n <= PW_BLOCKSIZE = 128): n < 8 sequential; else eight
// strided accumulators, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then
// the remainder sequentially.  Larger n recurse on (n2, n - n2) with
// n2 = n/2 rounded down to a multiple of 8 (combine_leaves below).
__device__ double np_leaf_sum(const double* a, uint64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (uint64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    uint64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[i + k]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

__global__ void __launch_bounds__(kCaloThreads)
    calo_hits_kernel(const float* __restrict__ batch, const prng_calo_particle_t* __restrict__ parts,
                     const uint32_t* __restrict__ region_offsets, const uint32_t* __restrict__ region_cells,
                     const prng_calo_param_t* __restrict__ params, uint32_t* __restrict__ hit_cell,
                     double* __restrict__ hit_amount) {
    const prng_calo_particle_t pt = parts[blockIdx.x];
    const prng_calo_param_t& pr = params[pt.param];
    const uint32_t c0 = region_offsets[pt.region];
    const uint32_t ncell = region_offsets[pt.region + 1] - c0;
    const uint32_t nb = pr.nbins;
    for (uint32_t j = threadIdx.x; j < pt.hits; j += blockDim.x) {
        const float* u = batch + pt.batch_offset + 3ull * j;
        const double u0 = (double)u[0], u1 = (double)u[1], u2 = (double)u[2];
        uint64_t ci = (uint64_t)__dmul_rn(u0, (double)ncell);  // astype(int64) truncates (u0 >= 0)
        if (ci > ncell - 1) ci = ncell - 1;
        uint32_t b = 0;
        for (uint32_t k = 0; k < nb; ++k) b += pr.cumw[k] <= u1 ? 1u : 0u;
        if (b > nb - 1) b = nb - 1;
        const double lo = pr.bin_edges[b];
        const double raw = __dadd_rn(lo, __dmul_rn(u2, __dsub_rn(pr.bin_edges[b + 1], lo)));
        hit_cell[pt.hit_offset + j] = region_cells[c0 + ci];
        hit_amount[pt.hit_offset + j] = raw;
    }
}

// numpy's pairwise sum evaluated by a warp: the recursion's leaves (runs of
// <= 128 elements, each summed exactly as np_pairwise_sum's leaf branch) are
// independent, so lane 0 lists them once per particle (iterative DFS),
// lane l sums leaves l, l + 32, ..., and lane 0 adds the leaf sums back up the
// same binary tree (iterative post-order walk).  Bit-identical to
// np_pairwise_sum.  All stacks live in shared memory: no local memory, so
// the kernel carries no per-thread stack reservation.
constexpr int kNormWarps = 4;
constexpr int kNormMaxLeaves = 512;  // n <= ~28k per particle in the list; larger: leaves summed by lane 0
constexpr int kNormStack = 48;      // tree depth <= log2(n / 64) + 1 < 48 for any 64-bit n

__device__ __forceinline__ uint64_t pw_split(uint64_t n) {  // numpy: n2 = n / 2; n2 -= n2 % 8
    const uint64_t n2 = n / 2;
    return n2 - n2 % 8;
}

struct NormWarpSmem {
    uint64_t leaf_off[kNormMaxLeaves];
    uint32_t leaf_len[kNormMaxLeaves];
    double leaf_val[kNormMaxLeaves];
    uint64_t st_off[kNormStack], st_n[kNormStack];
    double st_left[kNormStack];
    uint32_t st_stage[kNormStack];
};

// Lane 0: the leaves of np_pairwise_sum(., n) in order; returns their count
// (entries past kNormMaxLeaves are counted, not stored).
__device__ uint32_t list_leaves(NormWarpSmem& m, uint64_t n) {
    int sp = 0;
    uint32_t k = 0;
    m.st_off[0] = 0;
    m.st_n[0] = n;
    sp = 1;
    while (sp) {
        --sp;
        const uint64_t off = m.st_off[sp], len = m.st_n[sp];
        if (len <= 128) {
            if (k < (uint32_t)kNormMaxLeaves) {
                m.leaf_off[k] = off;
                m.leaf_len[k] = (uint32_t)len;
            }
            ++k;
            continue;
        }
        const uint64_t n2 = pw_split(len);
        m.st_off[sp] = off + n2;
        m.st_n[sp] = len - n2;
        ++sp;
        m.st_off[sp] = off;
        m.st_n[sp] = n2;
        ++sp;
    }
    return k;
}

// Lane 0: res = left + right at every internal node of np_pairwise_sum's
// tree over n elements; leaves take leaf_val[] in order (listed) or are
// summed on the fly from a (too many leaves for the list).
__device__ double combine_leaves(NormWarpSmem& m, uint64_t n, const double* a, bool listed) {
    int sp = 0;
    uint32_t kk = 0;
    m.st_off[0] = 0;
    m.st_n[0] = n;
    m.st_stage[0] = 0;
    sp = 1;
    for (;;) {
        const int t = sp - 1;
        if (m.st_n[t] > 128) {
            m.st_stage[t] = 1;
            m.st_off[sp] = m.st_off[t];
            m.st_n[sp] = pw_split(m.st_n[t]);
            m.st_stage[sp] = 0;
            ++sp;
            continue;
        }
        double val = listed ? m.leaf_val[kk++] : np_leaf_sum(a + m.st_off[t], m.st_n[t]);
        --sp;
        for (;;) {  // deliver val to the parents
            if (sp == 0) return val;
            const int q = sp - 1;
            if (m.st_stage[q] == 1) {
                m.st_left[q] = val;
                m.st_stage[q] = 2;
                const uint64_t n2 = pw_split(m.st_n[q]);
                m.st_off[sp] = m.st_off[q] + n2;
                m.st_n[sp] = m.st_n[q] - n2;
                m.st_stage[sp] = 0;
                ++sp;
                break;
            }
            val = __dadd_rn(m.st_left[q], val);
            --sp;
        }
    }
}

__device__ double warp_pairwise_sum(NormWarpSmem& m, const double* a, uint64_t n, uint32_t nleaves, uint32_t lane) {
    const bool listed = nleaves <= (uint32_t)kNormMaxLeaves;
    if (listed) {
        for (uint32_t i = lane; i < nleaves; i += 32) m.leaf_val[i] = np_leaf_sum(a + m.leaf_off[i], m.leaf_len[i]);
        __syncwarp();
    }
    double r = 0.0;
    if (lane == 0) r = combine_leaves(m, n, a, listed);
    __syncwarp();
    return __shfl_sync(0xffffffffu, r, 0);
}

// One warp per particle: raw_sum, in-place scaling to amounts, particle sum.
__global__ void __launch_bounds__(32 * kNormWarps)
    calo_normalize_kernel(const prng_calo_particle_t* __restrict__ parts, uint32_t nparts,
                          double* __restrict__ hit_amount, double* __restrict__ particle_sums) {
    __shared__ NormWarpSmem smem[kNormWarps];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint32_t p = blockIdx.x * kNormWarps + w;
    if (p >= nparts) return;  // warp-uniform
    NormWarpSmem& m = smem[w];
    const prng_calo_particle_t pt = parts[p];
    if (pt.hits == 0) {
        if (lane == 0) particle_sums[p] = 0.0;
        return;
    }
    double* a = hit_amount + pt.hit_offset;
    uint32_t nleaves = lane == 0 ? list_leaves(m, pt.hits) : 0;
    nleaves = __shfl_sync(0xffffffffu, nleaves, 0);
    __syncwarp();
    const double raw_sum = warp_pairwise_sum(m, a, pt.hits, nleaves, lane);
    if (raw_sum > 0.0) {
        const double scale = pt.target / raw_sum;
        for (uint32_t j = lane; j < pt.hits; j += 32) a[j] = __dmul_rn(a[j], scale);
    } else {
        const double each = pt.target / (double)pt.hits;  // np.full(m, target / m)
        for (uint32_t j = lane; j < pt.hits; j += 32) a[j] = each;
    }
    __syncwarp();
    const double sum = warp_pairwise_sum(m, a, pt.hits, nleaves, lane);
    if (lane == 0) particle_sums[p] = sum;
}

// ------------------------------------------------------------- deposits
// Per event e (hits [ev_off[e], ev_off[e+1]) in hit order) the deposits are
// np.unique(cells) ascending with np.bincount(inverse, weights=amounts)
// (calosim.py:340-347): each unique cell's amounts summed sequentially in hit
// order, starting from 0.0.  One CTA per event (events taken by ticket, in
// order), and no sort:
//  1. the event's cells are marked in a shared-memory bitmap over the window
//     [lo, lo + 2^wbits) (atomicOr); a block scan of the 64-bit words'
//     popcounts gives every marked cell its rank among the event's unique
//     cells, i.e. its deposit slot in np.unique's ascending order;
//  2. the event publishes its deposit count and finds its packed output
//     offset by a decoupled look-back over the earlier events' counts (one
//     pass: no separate count, scan and write launches);
//  3. the hits, in stages of 1024, are split stably by slot & 7 into shared
//     memory, and warp b adds bucket b's amounts to their slots' fp64 sums in
//     hit order (eight walkers on disjoint slots); lanes of a step that hit
//     the same cell (__match_any_sync) are added by the group's first lane
//     in lane order, so every sum is the sequential one, bit for bit;
//  4. the sums and the cells (decoded from the bitmap) are written packed.
// A cell range wider than the window is covered by successive windows, each
// starting at the smallest cell not yet covered; more unique cells than the
// sums buffer holds take one walk per slot chunk.
constexpr int kDepThreads = 256;
constexpr int kDepWarps = kDepThreads / 32;
constexpr uint32_t kDepMaxWinLog2 = 18;  // 2^18 cells: 32 KB bitmap + 16 KB ranks
constexpr uint32_t kDepSlots = 4096;     // fp64 sums per walk (32 KB)
constexpr uint32_t kDepStage = 1024;     // hits per split stage (12 KB)
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;

struct DepSmem {
    uint32_t red[2 * kDepWarps];
    uint32_t scan[kDepWarps];
    uint32_t event, total;
    unsigned long long off;
};

// Block-wide min of the event's cells >= floor (0xFFFFFFFF: none) and max of all.
__device__ void dep_minmax(DepSmem& s, const uint32_t* __restrict__ cells, uint64_t beg, uint64_t end,
                           uint64_t floor, uint32_t& mn, uint32_t& mx) {
    uint32_t a = 0xFFFFFFFFu, b = 0;
    for (uint64_t i = beg + threadIdx.x; i < end; i += kDepThreads) {
        const uint32_t c = cells[i];
        if ((uint64_t)c >= floor && c < a) a = c;
        b = c > b ? c : b;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    const uint32_t w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s.red[w] = a;
        s.red[kDepWarps + w] = b;
    }
    __syncthreads();
    a = s.red[0];
    b = s.red[kDepWarps];
#pragma unroll
    for (int k = 1; k < kDepWarps; ++k) {
        a = min(a, s.red[k]);
        b = max(b, s.red[kDepWarps + k]);
    }
    __syncthreads();
    mn = a;
    mx = b;
}

// Marks the cells in [lo, lo + 64 nw) and ranks the words: pref[q] = set bits
// in words < q.  Returns the window's unique-cell count (every thread).
__device__ uint32_t dep_build_window(DepSmem& s, unsigned long long* bm, uint32_t* pref,
                                     const uint32_t* __restrict__ cells, uint64_t beg, uint64_t end, uint32_t lo,
                                     uint32_t nw) {
    for (uint32_t q = threadIdx.x; q < nw; q += kDepThreads) bm[q] = 0ull;
    __syncthreads();
    const uint64_t span = 64ull * nw;
    for (uint64_t i = beg + threadIdx.x; i < end; i += kDepThreads) {
        const uint32_t c = cells[i];
        if (c >= lo && (uint64_t)(c - lo) < span)  // 32-bit halves of the 64-bit words (little-endian)
            atomicOr(reinterpret_cast<unsigned int*>(bm) + ((c - lo) >> 5), 1u << ((c - lo) & 31u));
    }
    __syncthreads();
    // each thread owns a contiguous run of words; block exclusive scan of the runs' popcounts
    const uint32_t per = (nw + kDepThreads - 1) / kDepThreads;
    const uint32_t q0 = threadIdx.x * per, q1 = min(q0 + per, nw);
    uint32_t mine = 0;
    for (uint32_t q = q0; q < q1; ++q) mine += __popcll(bm[q]);
    uint32_t inc = mine;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += v;
    }
    if (lane == 31) s.scan[w] = inc;
    __syncthreads();
    uint32_t base = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kDepWarps; ++k) {
        base += k < (int)w ? s.scan[k] : 0u;
        total += s.scan[k];
    }
    uint32_t r = base + inc - mine;
    for (uint32_t q = q0; q < q1; ++q) {
        pref[q] = r;
        r += __popcll(bm[q]);
    }
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint32_t dep_rank(const unsigned long long* bm, const uint32_t* pref, uint32_t rel) {
    const uint32_t q = rel >> 6;
    return pref[q] + __popcll(bm[q] & ((1ull << (rel & 63u)) - 1ull));
}

// Warp w walks its bucket's entries of a stage in order: sums[rs] += amount.
// Lanes of a step that hit the same slot (__match_any_sync) are added by the
// group's first lane in lane order, so every sum is the sequential one.
__device__ __forceinline__ void dep_walk(double* sums, const uint32_t* st_slot, const double* st_amt, uint32_t cnt) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t t = 0; t < cnt; t += 32) {
        const bool ok = t + lane < cnt;
        const uint32_t rs = ok ? st_slot[t + lane] : 0u;
        const double a = ok ? st_amt[t + lane] : 0.0;
        const uint32_t m = __match_any_sync(0xffffffffu, ok ? rs : (0x80000000u | lane));
        const bool grp = ok && (m & (m - 1u)) != 0u;
        uint32_t dup = __ballot_sync(0xffffffffu, grp);
        if (ok && !grp) sums[rs] = __dadd_rn(sums[rs], a);
        if (dup) {
            const bool lead = grp && (m & ((1u << lane) - 1u)) == 0u;
            double acc = lead ? sums[rs] : 0.0;
            while (dup) {
                const int k = __ffs(dup) - 1;
                dup &= dup - 1u;
                const double ak = __shfl_sync(0xffffffffu, a, k);
                if (lead && ((m >> k) & 1u)) acc = __dadd_rn(acc, ak);
            }
            if (lead) sums[rs] = acc;
        }
        __syncwarp();
    }
}

// sums[slot - s0] += amount over the event's hits in order, for the slots in
// [s0, s0 + nslots) of the window at lo.  The hits go in stages of
// kDepStage (warp w loads tiles 8w..8w+7 of the stage); each stage is split
// stably by bucket = slot & 7 (ballots, per-tile counts, a scan per bucket)
// into shared memory, and warp b walks bucket b: eight walkers on disjoint
// slots, each seeing its hits in hit order.
constexpr uint32_t kDepTilesPerWarp = kDepStage / 32 / kDepWarps;
static_assert(kDepStage == 32 * 32 && kDepWarps == 8 && kDepTilesPerWarp * 8 == 32,
              "the split scans 8 buckets x 32 tiles with 256 threads");

__device__ void dep_sum_slots(double* sums, uint32_t* st_slot, double* st_amt, uint32_t* tcnt,
                              const unsigned long long* bm, const uint32_t* pref, const uint32_t* __restrict__ cells,
                              const double* __restrict__ amts, uint64_t beg, uint64_t end, uint32_t lo,
                              uint64_t span, uint32_t s0, uint32_t nslots) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t j = threadIdx.x; j < nslots; j += kDepThreads) sums[j] = 0.0;
    // tcnt: [bucket][tile] counts (8 x 32), then the per-bucket totals
    uint32_t* wsum = tcnt + kDepWarps * (kDepStage / 32);
    for (uint64_t h0 = beg; h0 < end; h0 += kDepStage) {
        uint32_t rs[kDepTilesPerWarp], rk[kDepTilesPerWarp];
        double av[kDepTilesPerWarp];
#pragma unroll
        for (uint32_t k = 0; k < kDepTilesPerWarp; ++k) {
            const uint64_t i = h0 + (uint64_t)(w * kDepTilesPerWarp + k) * 32 + lane;
            uint32_t r = 0xFFFFFFFFu;
            av[k] = 0.0;
            if (i < end) {
                const uint32_t c = cells[i];
                av[k] = amts[i];
                if (c >= lo && (uint64_t)(c - lo) < span) {
                    const uint32_t q = dep_rank(bm, pref, c - lo) - s0;
                    if (q < nslots) r = q;
                }
            }
            rs[k] = r;
        }
#pragma unroll
        for (uint32_t k = 0; k < kDepTilesPerWarp; ++k) {
            const uint32_t bk = rs[k] == 0xFFFFFFFFu ? 8u : (rs[k] & 7u);
            uint32_t mine = 0;
#pragma unroll
            for (uint32_t b = 0; b < 8; ++b) {
                const uint32_t m = __ballot_sync(0xffffffffu, bk == b);
                if (bk == b) mine = __popc(m & lt);
                if (lane == b) tcnt[b * 32 + w * kDepTilesPerWarp + k] = __popc(m);
            }
            rk[k] = mine;
        }
        __syncthreads();
        // exclusive scan of the counts in [bucket][tile] order (thread t: bucket
        // t / 32 = its warp, tile t % 32): every (bucket, tile) gets its first
        // position, bucket w's run starts where warp w's entries start
        const uint32_t v = tcnt[threadIdx.x];
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
            if ((int)lane >= o) inc += x;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        uint32_t wstart = 0;
#pragma unroll
        for (uint32_t b = 0; b < kDepWarps; ++b) wstart += b < w ? wsum[b] : 0u;
        const uint32_t wcount = wsum[w];
        tcnt[threadIdx.x] = wstart + inc - v;
        __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < kDepTilesPerWarp; ++k) {
            if (rs[k] != 0xFFFFFFFFu) {
                const uint32_t pos = tcnt[(rs[k] & 7u) * 32 + w * kDepTilesPerWarp + k] + rk[k];
                st_slot[pos] = rs[k];
                st_amt[pos] = av[k];
            }
        }
        __syncthreads();
        dep_walk(sums, st_slot + wstart, st_amt + wstart, wcount);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kDepThreads, 1)
    calo_deposit_kernel(const uint32_t* __restrict__ cells, const double* __restrict__ amts,
                        const uint64_t* __restrict__ ev_off, uint32_t nevents, uint32_t cell_bits,
                        uint32_t wbits, unsigned long long* status, unsigned int* ticket, uint32_t* __restrict__ dep_cell,
                        double* __restrict__ dep_energy, uint64_t* __restrict__ dep_offsets) {
    extern __shared__ __align__(16) unsigned char dep_dyn[];
    __shared__ DepSmem s;
    const uint32_t nwords = 1u << (wbits - 6);
    double* sums = reinterpret_cast<double*>(dep_dyn);
    unsigned long long* bm = reinterpret_cast<unsigned long long*>(dep_dyn + kDepSlots * sizeof(double));
    uint32_t* pref = reinterpret_cast<uint32_t*>(bm + nwords);
    double* st_amt = reinterpret_cast<double*>(dep_dyn + kDepSlots * sizeof(double) +
                                               (size_t)nwords * (sizeof(unsigned long long) + sizeof(uint32_t)));
    uint32_t* st_slot = reinterpret_cast<uint32_t*>(st_amt + kDepStage);
    uint32_t* tcnt = st_slot + kDepStage;
    const uint64_t win = 64ull * nwords;
    const bool wide = cell_bits == 0 || cell_bits > wbits;  // ids may lie beyond the first window
    for (;;) {
        if (threadIdx.x == 0) s.event = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t e = s.event;
        if (e >= nevents) return;
        const uint64_t beg = ev_off[e], end = ev_off[e + 1];
        uint32_t lo = 0, cmax = (uint32_t)(win - 1);  // ids < 2^wbits: one window from 0, no min/max pass
        if (end > beg && wide) dep_minmax(s, cells, beg, end, 0, lo, cmax);
        auto words_of = [&](uint32_t wlo) {  // words covering [wlo, min(cmax, wlo + win - 1)]
            const uint64_t top = (uint64_t)cmax - wlo;
            return top >= win ? nwords : (uint32_t)(top >> 6) + 1u;
        };
        const bool single = end == beg || (uint64_t)cmax - lo < win;
        // 1. count (a single window stays built for the walk)
        uint64_t total = 0;
        uint32_t first_u = 0;
        if (end > beg) {
            uint32_t wlo = lo;
            for (;;) {
                const uint32_t u = dep_build_window(s, bm, pref, cells, beg, end, wlo, words_of(wlo));
                if (wlo == lo) first_u = u;
                total += u;
                if (single || (uint64_t)wlo + win > cmax) break;
                uint32_t unused;
                dep_minmax(s, cells, beg, end, (uint64_t)wlo + win, wlo, unused);  // exists: cmax qualifies
            }
        }
        // 2. packed offset: decoupled look-back over the earlier events
        if (threadIdx.x == 0) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(status[e]);
            unsigned long long prefix = 0;
            if (e > 0) {
                me.store(kLbAgg | total, cuda::memory_order_relaxed);
                for (uint32_t j = e - 1;; --j) {
                    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[j]);
                    unsigned long long v;
                    while (((v = st.load(cuda::memory_order_relaxed)) >> 62) == 0ull) __nanosleep(64);
                    prefix += v & kLbVal;
                    if ((v & kLbInc) || j == 0) break;
                }
            }
            me.store(kLbInc | (prefix + total), cuda::memory_order_relaxed);
            dep_offsets[e] = prefix;
            if (e == nevents - 1) dep_offsets[nevents] = prefix + total;
            s.off = prefix;
        }
        __syncthreads();
        const uint64_t off = s.off;
        // 3-4. walks and packed writes, window by window
        if (end > beg) {
            uint64_t base = off;
            uint32_t wlo = lo;
            for (;;) {
                const uint32_t nw = words_of(wlo);
                const uint32_t u = wlo == lo && single ? first_u : dep_build_window(s, bm, pref, cells, beg, end, wlo, nw);
                for (uint32_t s0 = 0; s0 < u; s0 += kDepSlots) {
                    const uint32_t ns = min(kDepSlots, u - s0);
                    dep_sum_slots(sums, st_slot, st_amt, tcnt, bm, pref, cells, amts, beg, end, wlo, 64ull * nw, s0, ns);
                    for (uint32_t j = threadIdx.x; j < ns; j += kDepThreads) dep_energy[base + s0 + j] = sums[j];
                    __syncthreads();
                }
                for (uint32_t q = threadIdx.x; q < nw; q += kDepThreads) {
                    unsigned long long bits = bm[q];
                    uint64_t r = base + pref[q];
                    while (bits) {
                        const int b = __ffsll((long long)bits) - 1;
                        bits &= bits - 1ull;
                        dep_cell[r++] = wlo + 64u * q + (uint32_t)b;
                    }
                }
                base += u;
                __syncthreads();
                if (single || (uint64_t)wlo + win > cmax) break;
                uint32_t unused;
                dep_minmax(s, cells, beg, end, (uint64_t)wlo + win, wlo, unused);  // exists: cmax qualifies
            }
        }
        __syncthreads();  // s.event / s.off are rewritten by the next ticket
    }
}
}  // namespace

int prng_detail_fail(int code, const char* msg);  // api.cu: the prng_last_error() slot

namespace {
int calo_fail(int code, const char* fmt, ...) {
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return prng_detail_fail(code, buf);
}
}  // namespace

extern "C" {

int prng_calo_hits(const float* batch, const prng_calo_particle_t* particles, uint32_t nparticles,
                   const uint32_t* region_offsets, const uint32_t* region_cells, const prng_calo_param_t* params,
                   uint32_t* hit_cell, double* hit_amount, double* particle_sums, void* stream) {
    if (nparticles == 0) return PRNG_OK;
    if (!batch || !particles || !region_offsets || !region_cells || !params || !hit_cell || !hit_amount ||
        !particle_sums)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    cudaStream_t s = (cudaStream_t)stream;
    calo_hits_kernel<<<nparticles, kCaloThreads, 0, s>>>(batch, particles, region_offsets, region_cells, params,
                                                         hit_cell, hit_amount);
    calo_normalize_kernel<<<(nparticles + kNormWarps - 1) / kNormWarps, 32 * kNormWarps, 0, s>>>(
        particles, nparticles, hit_amount, particle_sums);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo hits: %s", cudaGetErrorString(e));
}

namespace {
// Scratch: one look-back status word per event and the ticket counter.
size_t deposit_scratch(uint32_t nevents) { return ((size_t)nevents + 1) * sizeof(unsigned long long); }
}  // namespace

size_t prng_calo_deposit_scratch_bytes(uint64_t total_hits, uint32_t nevents) {
    (void)total_hits;
    return deposit_scratch(nevents);
}

int prng_calo_deposit(const uint32_t* hit_cell, const double* hit_amount, uint64_t total_hits,
                      const uint64_t* event_hit_offsets, uint32_t nevents, uint32_t cell_bits, void* scratch,
                      size_t scratch_bytes, uint32_t* dep_cell, double* dep_energy, uint64_t* dep_offsets,
                      void* stream) {
    if (nevents == 0) return PRNG_OK;
    if ((total_hits && (!hit_cell || !hit_amount)) || !event_hit_offsets || !dep_cell || !dep_energy || !dep_offsets)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    if (cell_bits > 32) return calo_fail(PRNG_ERR_INVALID_PARAMETER, "cell_bits must be <= 32");
    const size_t need = deposit_scratch(nevents);
    if (!scratch || scratch_bytes < need)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "scratch too small: need %zu bytes", need);
    cudaStream_t s = (cudaStream_t)stream;
    // bitmap window: the whole cell-id range when it has <= 2^18 ids
    const uint32_t b = cell_bits == 0 ? 32u : cell_bits;
    const uint32_t wbits = b < 6u ? 6u : (b > kDepMaxWinLog2 ? kDepMaxWinLog2 : b);
    const uint32_t nwords = 1u << (wbits - 6);
    const size_t smem = kDepSlots * sizeof(double) + (size_t)nwords * (sizeof(unsigned long long) + sizeof(uint32_t)) +
                        kDepStage * (sizeof(double) + sizeof(uint32_t)) +
                        (kDepWarps * (kDepStage / 32) + kDepWarps) * sizeof(uint32_t);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(calo_deposit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, calo_deposit_kernel, kDepThreads, smem);
    if (e != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "calo deposit setup: %s", cudaGetErrorString(e));
    const uint64_t slots = (uint64_t)(per_sm > 0 ? per_sm : 1) * (uint64_t)nsm;
    const uint32_t grid = (uint32_t)(slots < nevents ? slots : nevents);
    unsigned long long* status = static_cast<unsigned long long*>(scratch);
    e = cudaMemsetAsync(status, 0, need, s);
    if (e != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(e));
    calo_deposit_kernel<<<grid, kDepThreads, smem, s>>>(hit_cell, hit_amount, event_hit_offsets, nevents, cell_bits,
                                                        wbits, status,
                                                        reinterpret_cast<unsigned int*>(status + nevents), dep_cell,
                                                        dep_energy, dep_offsets);
    e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(e));
}

}  // extern "C"
