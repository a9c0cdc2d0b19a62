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
//     ranks them, a counting sort by rank buckets the hits, each bucket is
//     put back in hit order and summed by one thread, and a decoupled
//     look-back over the events' deposit counts packs the output in the same
//     launch (calo_deposit_kernel) so the host copies back exactly the
//     deposits.  No library kernels.
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <algorithm>
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

// numpy's pairwise sum evaluated by a warp.  The recursion tree of
// np_pairwise_sum(., n) depends only on n: lane 0 walks it once per particle
// (iterative DFS, leaves in order) and records its leaves (runs of <= 128
// elements) and its internal nodes with their children and depth; the leaves
// are summed four at a time, eight lanes per leaf (numpy's eight accumulator
// chains), and the internal nodes are added level by level from the deepest
// (every node is left + right of values already computed, so the order
// across independent nodes changes nothing).  Bit-identical to
// np_pairwise_sum; both sums of a particle reuse the tree.  Trees of more
// than kNormMaxLeaves leaves (particles of > ~16k hits) are summed by lane 0
// on the fly (np_leaf_sum / combine_serial).
constexpr int kNormWarps = 4;
constexpr int kNormMaxLeaves = 256;
constexpr int kNormStack = 48;  // tree depth <= log2(n / 64) + 1 < 48 for any 64-bit n

__device__ __forceinline__ uint64_t pw_split(uint64_t n) {  // numpy: n2 = n / 2; n2 -= n2 % 8
    const uint64_t n2 = n / 2;
    return n2 - n2 % 8;
}

struct NormWarpSmem {
    double val[2 * kNormMaxLeaves];  // leaf k at [k], internal node i at [kNormMaxLeaves + i]
    uint32_t leaf_off[kNormMaxLeaves];
    uint16_t child[kNormMaxLeaves][2];  // ids into val
    uint8_t leaf_len[kNormMaxLeaves];
    uint8_t depth[kNormMaxLeaves];
    uint64_t st_off[kNormStack], st_n[kNormStack];
    uint32_t st_slot[kNormStack];  // DFS: child slot to fill (node * 2 + side, or ~0 for the root)
    uint8_t st_depth[kNormStack];
    double st_left[kNormStack];    // combine_serial
    uint32_t st_stage[kNormStack];
};

struct NormTree {
    uint32_t nleaves, nnodes, maxdepth;
    bool listed;
};

// Lane 0: np_pairwise_sum's tree over n elements.
__device__ NormTree build_tree(NormWarpSmem& m, uint64_t n) {
    NormTree t{0, 0, 0, true};
    int sp = 1;
    m.st_off[0] = 0;
    m.st_n[0] = n;
    m.st_slot[0] = ~0u;
    m.st_depth[0] = 0;
    while (sp) {
        --sp;
        const uint64_t off = m.st_off[sp], len = m.st_n[sp];
        const uint32_t slot = m.st_slot[sp];
        const uint32_t d = m.st_depth[sp];
        uint32_t id;
        if (len <= 128) {
            id = t.nleaves++;
            if (id < (uint32_t)kNormMaxLeaves) {
                m.leaf_off[id] = (uint32_t)off;
                m.leaf_len[id] = (uint8_t)len;
            }
        } else {
            const uint32_t i = t.nnodes++;
            id = kNormMaxLeaves + i;
            const uint64_t n2 = pw_split(len);
            if (i < (uint32_t)kNormMaxLeaves) m.depth[i] = (uint8_t)d;
            t.maxdepth = d > t.maxdepth ? d : t.maxdepth;
            m.st_off[sp] = off + n2;  // right, popped second
            m.st_n[sp] = len - n2;
            m.st_slot[sp] = 2 * i + 1;
            m.st_depth[sp] = (uint8_t)(d + 1);
            ++sp;
            m.st_off[sp] = off;  // left, popped first: leaves come out in order
            m.st_n[sp] = n2;
            m.st_slot[sp] = 2 * i;
            m.st_depth[sp] = (uint8_t)(d + 1);
            ++sp;
        }
        if (slot != ~0u && (slot >> 1) < (uint32_t)kNormMaxLeaves) m.child[slot >> 1][slot & 1u] = (uint16_t)id;
    }
    t.listed = t.nleaves <= (uint32_t)kNormMaxLeaves;
    return t;
}

// Lane 0, trees too large for the lists: res = left + right at every
// internal node, leaves summed on the fly (iterative post-order walk).
__device__ double combine_serial(NormWarpSmem& m, uint64_t n, const double* a) {
    int sp = 1;
    m.st_off[0] = 0;
    m.st_n[0] = n;
    m.st_stage[0] = 0;
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
        double val = np_leaf_sum(a + m.st_off[t], m.st_n[t]);
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

// Four leaves per warp step, eight lanes per leaf: lane k of a group runs
// numpy's accumulator r_k (a[k], then += a[8i + k]) -- the eight chains are
// independent in np_leaf_sum -- and the group combines them by shuffles in
// numpy's order ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)); the group's
// first lane adds the n % 8 remainder (or sums a leaf of < 8 sequentially).
// Bit-identical to np_leaf_sum, with coalesced 64-byte loads per group.
__device__ void warp_leaf_sums(NormWarpSmem& m, const double* a, uint32_t nleaves, uint32_t lane) {
    const uint32_t g = lane >> 3, k = lane & 7u;
    for (uint32_t base = 0; base < nleaves; base += 4) {
        const uint32_t leaf = base + g;
        const bool ok = leaf < nleaves;
        const uint32_t off = ok ? m.leaf_off[leaf] : 0u;
        const uint32_t len = ok ? m.leaf_len[leaf] : 0u;
        const double* p = a + off;
        const uint32_t full = len - len % 8u;
        double r = 0.0;
        if (len >= 8) {  // the chain's <= 16 loads issued together, then the adds in order
            double v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 8u * i < full ? p[8 * i + k] : 0.0;
            r = v[0];
#pragma unroll
            for (int i = 1; i < 16; ++i)
                if (8u * i < full) r = __dadd_rn(r, v[i]);
        }
        const double t = __dadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));  // k even: r_k + r_k+1
        const double u = __dadd_rn(t, __shfl_down_sync(0xffffffffu, t, 2));  // k % 4 == 0
        const double v = __dadd_rn(u, __shfl_down_sync(0xffffffffu, u, 4));  // k == 0
        if (ok && k == 0) {
            double res = len >= 8 ? v : 0.0;
            for (uint32_t i = full; i < len; ++i) res = __dadd_rn(res, p[i]);
            m.val[leaf] = res;
        }
    }
}

__device__ double warp_pairwise_sum(NormWarpSmem& m, const NormTree& t, const double* a, uint64_t n,
                                    uint32_t lane) {
    double r = 0.0;
    if (t.listed) {
        warp_leaf_sums(m, a, t.nleaves, lane);
        __syncwarp();
        for (int d = (int)t.maxdepth; d >= 0 && t.nnodes; --d) {  // deepest internal nodes first
            for (uint32_t i = lane; i < t.nnodes; i += 32)
                if (m.depth[i] == (uint32_t)d)
                    m.val[kNormMaxLeaves + i] = __dadd_rn(m.val[m.child[i][0]], m.val[m.child[i][1]]);
            __syncwarp();
        }
        r = t.nnodes ? m.val[kNormMaxLeaves] : m.val[0];
    } else if (lane == 0) {
        r = combine_serial(m, n, a);
    }
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
    NormTree t{};
    if (lane == 0) t = build_tree(m, pt.hits);
    t.nleaves = __shfl_sync(0xffffffffu, t.nleaves, 0);
    t.nnodes = __shfl_sync(0xffffffffu, t.nnodes, 0);
    t.maxdepth = __shfl_sync(0xffffffffu, t.maxdepth, 0);
    t.listed = t.nleaves <= (uint32_t)kNormMaxLeaves;
    __syncwarp();
    const double raw_sum = warp_pairwise_sum(m, t, a, pt.hits, lane);
    if (raw_sum > 0.0) {
        const double scale = pt.target / raw_sum;
        uint32_t j = lane;
        for (; j + 7 * 32 < pt.hits; j += 8 * 32) {  // eight loads in flight per lane
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = a[j + q * 32];
#pragma unroll
            for (int q = 0; q < 8; ++q) a[j + q * 32] = __dmul_rn(v[q], scale);
        }
        for (; j < pt.hits; j += 32) a[j] = __dmul_rn(a[j], scale);
    } else {
        const double each = pt.target / (double)pt.hits;  // np.full(m, target / m)
        for (uint32_t j = lane; j < pt.hits; j += 32) a[j] = each;
    }
    __syncwarp();
    const double sum = warp_pairwise_sum(m, t, a, pt.hits, lane);
    if (lane == 0) particle_sums[p] = sum;
}

// ------------------------------------------------------------- deposits
// Per event e (hits [ev_off[e], ev_off[e+1]) in hit order) the deposits are
// np.unique(cells) ascending with np.bincount(inverse, weights=amounts)
// (calosim.py:340-347): each unique cell's amounts summed sequentially in hit
// order, starting from 0.0.  One CTA per event (events taken by ticket, in
// order), no sort of the hits and no serial walk:
//  1. the event's cells are marked in a shared-memory bitmap over the window
//     [lo, lo + 2^wbits) (atomicOr); a block scan of the 64-bit words'
//     popcounts ranks every marked cell among the event's unique cells: its
//     deposit slot, in np.unique's ascending order;
//  2. the event publishes its deposit count and finds its packed output
//     offset by a decoupled look-back over the earlier events' counts (one
//     pass: no separate count, scan and write launches);
//  3. a counting sort of the hits by slot (count, block scan, fill) leaves
//     each slot's hit indices in one bucket; the fill's atomics order a
//     bucket arbitrarily, so the slot's thread puts it back in hit order
//     (insertion sort: buckets hold ~1.4 hits here) and adds the amounts
//     sequentially; buckets of more than 32 hits are ordered by the whole
//     CTA (bitonic network) and summed by one thread.  Every sum is the
//     sequential one, bit for bit;
//  4. the sums and the cells are written packed at the event's offset.
// Events of up to 8192 hits keep their counters and indices in shared
// memory (16-bit; each thread's <= 32 slots stay in registers from the count
// to the fill, so the bucket indices overwrite the no longer needed bitmap:
// 56 KB, 4 CTAs per SM), larger ones in the caller's scratch (32-bit).  A cell
// range wider than the window is covered by successive windows, each
// starting at the smallest cell not yet covered.
constexpr int kDepThreads = 256;
constexpr int kDepWarps = kDepThreads / 32;
constexpr uint32_t kDepMaxWinLog2 = 18;  // 2^18 cells: 32 KB bitmap + 8 KB of 16-bit ranks
constexpr uint32_t kDepRankBlock = 256;  // words per 32-bit rank base
constexpr uint32_t kDepCap = 8192;       // hits per event indexed in shared memory
constexpr uint32_t kDepSmall = 32;       // larger buckets are ordered by the whole CTA
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;

struct DepSmem {
    uint32_t red[2 * kDepWarps];
    uint32_t scan[kDepWarps];
    uint32_t event, nbig;
    uint32_t outside;  // a hit outside the window was seen (dep_build_window)
    unsigned long long off;
    uint32_t rbase[(1u << kDepMaxWinLog2) / 64 / kDepRankBlock];
    uint32_t big[kDepCap / (kDepSmall + 1) + 1];  // slots with large buckets (shared-memory path)
};

// Block-wide exclusive scan of one value per thread; *total = the sum.
__device__ uint32_t dep_block_scan(DepSmem& s, uint32_t v, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += x;
    }
    if (lane == 31) s.scan[w] = inc;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kDepWarps; ++k) {
        base += k < (int)w ? s.scan[k] : 0u;
        tot += s.scan[k];
    }
    __syncthreads();
    *total = tot;
    return base + inc - v;
}

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

// Marks the cells in [lo, lo + 64 nw) and ranks the words: the rank of word
// q (set bits in words < q) is rbase[q / 256] plus the 16-bit offset
// (pref[q] - rbase) mod 2^16 (a block of 256 words holds <= 16384 bits).
// Returns the window's unique-cell count.
__device__ uint32_t dep_build_window(DepSmem& s, unsigned long long* bm, uint16_t* pref,
                                     const uint32_t* __restrict__ cells, uint64_t beg, uint64_t end, uint32_t lo,
                                     uint32_t nw) {
    for (uint32_t q = threadIdx.x; q < nw; q += kDepThreads) bm[q] = 0ull;
    if (threadIdx.x == 0) s.outside = 0u;
    __syncthreads();
    const uint64_t span = 64ull * nw;
    bool outside = false;
    for (uint64_t i = beg + threadIdx.x; i < end; i += kDepThreads) {
        const uint32_t c = cells[i];
        if (c >= lo && (uint64_t)(c - lo) < span)  // 32-bit halves of the 64-bit words (little-endian)
            atomicOr(reinterpret_cast<unsigned int*>(bm) + ((c - lo) >> 5), 1u << ((c - lo) & 31u));
        else
            outside = true;
    }
    if (outside) s.outside = 1u;
    __syncthreads();
    const uint32_t per = (nw + kDepThreads - 1) / kDepThreads;
    const uint32_t q0 = min(threadIdx.x * per, nw), q1 = min(q0 + per, nw);
    uint32_t mine = 0;
    for (uint32_t q = q0; q < q1; ++q) mine += __popcll(bm[q]);
    uint32_t total;
    uint32_t r = dep_block_scan(s, mine, &total);
    for (uint32_t q = q0; q < q1; ++q) {
        if ((q & (kDepRankBlock - 1)) == 0) s.rbase[q / kDepRankBlock] = r;
        pref[q] = (uint16_t)r;
        r += __popcll(bm[q]);
    }
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint32_t dep_rank(const DepSmem& s, const unsigned long long* bm, const uint16_t* pref,
                                             uint32_t rel) {
    const uint32_t q = rel >> 6;
    const uint32_t b = s.rbase[q / kDepRankBlock];
    return b + (((uint32_t)pref[q] - b) & 0xFFFFu) + __popcll(bm[q] & ((1ull << (rel & 63u)) - 1ull));
}

// Bucket storage.  Shared memory: 16-bit counters packed in pairs and 16-bit
// hit indices; global (events of more than kDepCap hits): 32-bit, in scratch.
struct DepIdxShared {
    static constexpr bool kRegSlots = true;  // slots in registers from count to fill: lst may alias the bitmap
    uint32_t* cnt2;
    uint16_t* lst;
    uint32_t* big;
    __device__ uint32_t add(uint32_t sl) const {
        const uint32_t sh = (sl & 1u) << 4;
        return (atomicAdd(&cnt2[sl >> 1], 1u << sh) >> sh) & 0xFFFFu;
    }
    __device__ uint32_t get(uint32_t sl) const { return (cnt2[sl >> 1] >> ((sl & 1u) << 4)) & 0xFFFFu; }
    __device__ uint32_t idx(uint32_t p) const { return lst[p]; }
    __device__ void put(uint32_t p, uint32_t h) const { lst[p] = (uint16_t)h; }
    // zero / exclusive-scan the first u counters (whole 32-bit words per thread)
    __device__ void zero(uint32_t u) const {
        for (uint32_t w = threadIdx.x; w < (u + 1) / 2; w += kDepThreads) cnt2[w] = 0u;
    }
    __device__ void scan(DepSmem& s, uint32_t u) const {
        const uint32_t nw = (u + 1) / 2, per = (nw + kDepThreads - 1) / kDepThreads;
        const uint32_t w0 = min(threadIdx.x * per, nw), w1 = min(w0 + per, nw);
        uint32_t mine = 0;
        for (uint32_t w = w0; w < w1; ++w) mine += (cnt2[w] & 0xFFFFu) + (cnt2[w] >> 16);
        uint32_t total;
        uint32_t r = dep_block_scan(s, mine, &total);
        for (uint32_t w = w0; w < w1; ++w) {
            const uint32_t v = cnt2[w];
            const uint32_t a = r, b = r + (v & 0xFFFFu);
            cnt2[w] = a | (b << 16);
            r = b + (v >> 16);
        }
    }
};

struct DepIdxGlobal {
    static constexpr bool kRegSlots = false;
    uint32_t* cnt;
    uint32_t* lst;
    uint32_t* big;
    __device__ uint32_t add(uint32_t sl) const { return atomicAdd(&cnt[sl], 1u); }
    __device__ uint32_t get(uint32_t sl) const { return cnt[sl]; }
    __device__ uint32_t idx(uint32_t p) const { return lst[p]; }
    __device__ void put(uint32_t p, uint32_t h) const { lst[p] = h; }
    __device__ void zero(uint32_t u) const {
        for (uint32_t w = threadIdx.x; w < u; w += kDepThreads) cnt[w] = 0u;
    }
    __device__ void scan(DepSmem& s, uint32_t u) const {
        const uint32_t per = (u + kDepThreads - 1) / kDepThreads;
        const uint32_t w0 = min(threadIdx.x * per, u), w1 = min(w0 + per, u);
        uint32_t mine = 0;
        for (uint32_t w = w0; w < w1; ++w) mine += cnt[w];
        uint32_t total;
        uint32_t r = dep_block_scan(s, mine, &total);
        for (uint32_t w = w0; w < w1; ++w) {
            const uint32_t v = cnt[w];
            cnt[w] = r;
            r += v;
        }
    }
};

// Sequential fp64 sum of the amounts of bucket [st, en) (hit order), with
// the loads issued eight at a time.
template <class IX>
__device__ double dep_bucket_sum(const IX& ix, const double* __restrict__ amts, uint64_t beg, uint32_t st,
                                 uint32_t en) {
    double acc = 0.0;  // np.bincount: 0.0, then += weights in input order
    uint32_t p = st;
    for (; p + 8 <= en; p += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = amts[beg + ix.idx(p + j)];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, v[j]);
    }
    for (; p < en; ++p) acc = __dadd_rn(acc, amts[beg + ix.idx(p)]);
    return acc;
}

// Deposits of the window at lo (u unique cells, ranked in bm/pref) written
// at out + [0, u): counting sort of the hits by slot, then per-slot
// sequential sums in hit order.
template <class IX>
__device__ void dep_window(DepSmem& s, const IX& ix, const unsigned long long* bm, const uint16_t* pref,
                           const uint32_t* __restrict__ cells, const double* __restrict__ amts, uint64_t beg,
                           uint64_t end, uint32_t lo, uint64_t span, uint32_t u, uint32_t* __restrict__ out_cell,
                           double* __restrict__ out_energy) {
    const uint32_t nh = (uint32_t)(end - beg);
    ix.zero(u);
    if (threadIdx.x == 0) s.nbig = 0;
    __syncthreads();
    if constexpr (IX::kRegSlots) {
        // <= 32 hits per thread: their slots (16 bits, 0xFFFF = outside the
        // window) stay in registers from the count to the fill, so the fill
        // needs no ranks and its buckets may overwrite the bitmap
        uint32_t sl2[kDepCap / kDepThreads / 2];
#pragma unroll
        for (int j = 0; j < (int)(kDepCap / kDepThreads); ++j) {
            const uint32_t h = threadIdx.x + j * kDepThreads;
            uint32_t sl = 0xFFFFu;
            if (h < nh) {
                const uint32_t c = cells[beg + h];
                if (c >= lo && (uint64_t)(c - lo) < span) ix.add(sl = dep_rank(s, bm, pref, c - lo));
            }
            if (j & 1) sl2[j / 2] |= sl << 16; else sl2[j / 2] = sl;
        }
        __syncthreads();
        ix.scan(s, u);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < (int)(kDepCap / kDepThreads); ++j) {
            const uint32_t sl = (sl2[j / 2] >> ((j & 1) * 16)) & 0xFFFFu;
            if (sl != 0xFFFFu) ix.put(ix.add(sl), threadIdx.x + j * kDepThreads);
        }
    } else {
        for (uint32_t h = threadIdx.x; h < nh; h += kDepThreads) {
            const uint32_t c = cells[beg + h];
            if (c >= lo && (uint64_t)(c - lo) < span) ix.add(dep_rank(s, bm, pref, c - lo));
        }
        __syncthreads();
        ix.scan(s, u);
        __syncthreads();
        for (uint32_t h = threadIdx.x; h < nh; h += kDepThreads) {
            const uint32_t c = cells[beg + h];
            if (c >= lo && (uint64_t)(c - lo) < span) ix.put(ix.add(dep_rank(s, bm, pref, c - lo)), h);
        }
    }
    __syncthreads();
    // counters now hold each bucket's end; bucket sl = [end(sl - 1), end(sl))
    for (uint32_t sl = threadIdx.x; sl < u; sl += kDepThreads) {
        const uint32_t st = sl ? ix.get(sl - 1) : 0u, en = ix.get(sl);
        if (en - st > kDepSmall) {
            ix.big[atomicAdd(&s.nbig, 1u)] = sl;
            continue;
        }
        for (uint32_t i = st + 1; i < en; ++i) {  // insertion sort back into hit order
            const uint32_t v = ix.idx(i);
            uint32_t j = i;
            for (; j > st && ix.idx(j - 1) > v; --j) ix.put(j, ix.idx(j - 1));
            ix.put(j, v);
        }
        out_energy[sl] = dep_bucket_sum(ix, amts, beg, st, en);
        out_cell[sl] = cells[beg + ix.idx(st)];
    }
    __syncthreads();
    const uint32_t nbig = s.nbig;
    for (uint32_t b = 0; b < nbig; ++b) {
        const uint32_t sl = ix.big[b];
        const uint32_t st = sl ? ix.get(sl - 1) : 0u, en = ix.get(sl), k = en - st;
        uint32_t P = 2;
        while (P < k) P <<= 1;
        // bitonic network with every comparator ascending (the first stage of
        // each merge compares mirrored pairs); positions >= k act as +inf
        for (uint32_t size = 2; size <= P; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                const uint32_t lg = __ffs(stride) - 1;
                for (uint32_t t = threadIdx.x; t < P / 2; t += kDepThreads) {
                    const uint32_t blk = t >> lg, o = t & (stride - 1);
                    const uint32_t i = stride == size >> 1 ? blk * size + o : blk * 2 * stride + o;
                    const uint32_t j = stride == size >> 1 ? blk * size + size - 1 - o : i + stride;
                    if (j < k) {
                        const uint32_t a = ix.idx(st + i), c = ix.idx(st + j);
                        if (a > c) {
                            ix.put(st + i, c);
                            ix.put(st + j, a);
                        }
                    }
                }
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) {
            out_energy[sl] = dep_bucket_sum(ix, amts, beg, st, en);
            out_cell[sl] = cells[beg + ix.idx(st)];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kDepThreads, 4)
    calo_deposit_kernel(const uint32_t* __restrict__ cells, const double* __restrict__ amts,
                        const uint64_t* __restrict__ ev_off, uint32_t nevents, uint32_t cell_bits, uint32_t wbits,
                        unsigned long long* status, unsigned int* ticket, uint32_t* gidx, uint64_t total_hits,
                        uint32_t* __restrict__ dep_cell, double* __restrict__ dep_energy,
                        uint64_t* __restrict__ dep_offsets) {
    extern __shared__ __align__(16) unsigned char dep_dyn[];
    __shared__ DepSmem s;
    const uint32_t nwords = 1u << (wbits - 6);
    unsigned long long* bm = reinterpret_cast<unsigned long long*>(dep_dyn);
    // the bitmap, overwritten by the 16-bit bucket indices once the count
    // has put every hit's slot in registers; then the counters and word ranks
    const uint32_t region = max(nwords * 8u, kDepCap * 2u);
    uint16_t* lst = reinterpret_cast<uint16_t*>(dep_dyn);
    uint32_t* cnt2 = reinterpret_cast<uint32_t*>(dep_dyn + region);
    uint16_t* pref = reinterpret_cast<uint16_t*>(cnt2 + kDepCap / 2);
    const uint64_t win = 64ull * nwords;
    const bool wide = cell_bits == 0 || cell_bits > wbits;  // ids may lie beyond the first window
    for (;;) {
        if (threadIdx.x == 0) s.event = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t e = s.event;
        if (e >= nevents) return;
        const uint64_t beg = ev_off[e], end = ev_off[e + 1];
        // ids < 2^cell_bits <= 2^wbits: one window from 0, no min/max pass --
        // unless a hit outside it shows cell_bits understated the ids, then the
        // event is redone with min/max and windows (results do not depend on it)
        bool ev_wide = wide;
        uint32_t lo = 0, cmax = (uint32_t)(win - 1);
        uint64_t total = 0;
        uint32_t first_u = 0;
        bool single = true;
        auto words_of = [&](uint32_t wlo) {  // words covering [wlo, min(cmax, wlo + win - 1)]
            const uint64_t top = (uint64_t)cmax - wlo;
            return top >= win ? nwords : (uint32_t)(top >> 6) + 1u;
        };
        // 1. count (a single window stays built for step 3)
        for (int attempt = 0; attempt < 2; ++attempt) {
            if (end > beg && ev_wide) dep_minmax(s, cells, beg, end, 0, lo, cmax);
            single = end == beg || (uint64_t)cmax - lo < win;
            total = 0;
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
            if (ev_wide || end == beg || !s.outside) break;
            ev_wide = true;  // an id >= 2^wbits: redo with min/max
            __syncthreads();
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
        // 3-4. per-window counting sort, per-slot sums, packed writes
        if (end > beg) {
            const bool small = end - beg <= kDepCap;
            const DepIdxShared ixs{cnt2, lst, s.big};
            const DepIdxGlobal ixg{gidx + beg, gidx + total_hits + beg, gidx + 2 * total_hits + beg};
            uint64_t base = off;
            uint32_t wlo = lo;
            for (;;) {
                const uint32_t nw = words_of(wlo);
                const uint32_t u =
                    wlo == lo && single ? first_u : dep_build_window(s, bm, pref, cells, beg, end, wlo, nw);
                if (small)
                    dep_window(s, ixs, bm, pref, cells, amts, beg, end, wlo, 64ull * nw, u, dep_cell + base,
                               dep_energy + base);
                else
                    dep_window(s, ixg, bm, pref, cells, amts, beg, end, wlo, 64ull * nw, u, dep_cell + base,
                               dep_energy + base);
                base += u;
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

// The device that owns `ptr` is current for the entry point; the caller's
// device is restored on return (as for the generator entry points, api.cu).
struct CaloDevice {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit CaloDevice(const void* ptr) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        cudaPointerAttributes attr;
        err = cudaPointerGetAttributes(&attr, ptr);
        if (err != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        if ((attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) && attr.device != prev)
            err = cudaSetDevice(attr.device);
    }
    ~CaloDevice() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    CaloDevice(const CaloDevice&) = delete;
    CaloDevice& operator=(const CaloDevice&) = delete;
};
}  // namespace

extern "C" {

int prng_calo_hits(const float* batch, const prng_calo_particle_t* particles, uint32_t nparticles,
                   const uint32_t* region_offsets, const uint32_t* region_cells, const prng_calo_param_t* params,
                   uint32_t* hit_cell, double* hit_amount, double* particle_sums, void* stream) {
    if (nparticles == 0) return PRNG_OK;
    if (!batch || !particles || !region_offsets || !region_cells || !params || !hit_cell || !hit_amount ||
        !particle_sums)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    const CaloDevice on(hit_amount);
    if (on.err != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "calo hits: %s", cudaGetErrorString(on.err));
    cudaStream_t s = (cudaStream_t)stream;
    calo_hits_kernel<<<nparticles, kCaloThreads, 0, s>>>(batch, particles, region_offsets, region_cells, params,
                                                         hit_cell, hit_amount);
    calo_normalize_kernel<<<(nparticles + kNormWarps - 1) / kNormWarps, 32 * kNormWarps, 0, s>>>(
        particles, nparticles, hit_amount, particle_sums);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo hits: %s", cudaGetErrorString(e));
}

namespace {
// Scratch: one look-back status word per event, the ticket counter, and the
// 32-bit bucket arrays of events with more than kDepCap hits (counters,
// hit indices, large-bucket list: total_hits entries each).
size_t deposit_status_bytes(uint32_t nevents) { return ((size_t)nevents + 1) * sizeof(unsigned long long); }
size_t deposit_scratch(uint64_t total_hits, uint32_t nevents) {
    return deposit_status_bytes(nevents) + 3 * (size_t)total_hits * sizeof(uint32_t);
}
}  // namespace

size_t prng_calo_deposit_scratch_bytes(uint64_t total_hits, uint32_t nevents) {
    return deposit_scratch(total_hits, nevents);
}

int prng_calo_deposit(const uint32_t* hit_cell, const double* hit_amount, uint64_t total_hits,
                      const uint64_t* event_hit_offsets, uint32_t nevents, uint32_t cell_bits, void* scratch,
                      size_t scratch_bytes, uint32_t* dep_cell, double* dep_energy, uint64_t* dep_offsets,
                      void* stream) {
    if (nevents == 0) return PRNG_OK;
    if ((total_hits && (!hit_cell || !hit_amount)) || !event_hit_offsets || !dep_cell || !dep_energy || !dep_offsets)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    if (cell_bits > 32) return calo_fail(PRNG_ERR_INVALID_PARAMETER, "cell_bits must be <= 32");
    const size_t need = deposit_scratch(total_hits, nevents);
    if (!scratch || scratch_bytes < need)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "scratch too small: need %zu bytes", need);
    const CaloDevice on(dep_energy);
    if (on.err != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(on.err));
    cudaStream_t s = (cudaStream_t)stream;
    // bitmap window: the whole cell-id range when it has <= 2^18 ids
    const uint32_t b = cell_bits == 0 ? 32u : cell_bits;
    const uint32_t wbits = b < 6u ? 6u : (b > kDepMaxWinLog2 ? kDepMaxWinLog2 : b);
    const uint32_t nwords = 1u << (wbits - 6);
    const size_t smem = std::max<size_t>((size_t)nwords * sizeof(unsigned long long), kDepCap * sizeof(uint16_t)) +
                        kDepCap / 2 * sizeof(uint32_t) + (size_t)nwords * sizeof(uint16_t);  // 56 KB at 2^18
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
    e = cudaMemsetAsync(status, 0, deposit_status_bytes(nevents), s);
    if (e != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(e));
    calo_deposit_kernel<<<grid, kDepThreads, smem, s>>>(hit_cell, hit_amount, event_hit_offsets, nevents, cell_bits,
                                                        wbits, status,
                                                        reinterpret_cast<unsigned int*>(status + nevents),
                                                        reinterpret_cast<uint32_t*>(status + nevents + 1), total_hits,
                                                        dep_cell, dep_energy, dep_offsets);
    e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(e));
}

}  // extern "C"
