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
//     in order, i.e. cells sorted ascending and each cell's amounts summed
//     sequentially in hit order: a stable segmented radix sort (CUB) by cell
//     over the cell-id bits only, then one sequential run-sum per unique
//     cell, compacted with a block scan into one packed array (a count pass,
//     a device scan of the counts, a write pass) so the host copies back
//     exactly the deposits.
#include <cub/cub.cuh>
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

// One CTA per event over its cell-sorted hits.  COUNT pass: number of unique
// cells per event.  WRITE pass: (cell, sequential run sum) compacted at the
// event's packed offset dep_offsets[e] (exclusive scan of the counts).
template <bool WRITE>
__global__ void __launch_bounds__(kCaloThreads)
    calo_reduce_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ vals,
                       const uint64_t* __restrict__ ev_off, uint64_t* __restrict__ counts,
                       const uint64_t* __restrict__ dep_offsets, uint32_t* __restrict__ dep_cell,
                       double* __restrict__ dep_energy) {
    using Scan = cub::BlockScan<uint32_t, kCaloThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t carry;
    const uint64_t beg = ev_off[blockIdx.x], end = ev_off[blockIdx.x + 1];
    const uint64_t out0 = WRITE ? dep_offsets[blockIdx.x] : 0;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = beg; base < end; base += kCaloThreads) {
        const uint64_t i = base + threadIdx.x;
        const uint32_t flag = (i < end && (i == beg || keys[i] != keys[i - 1])) ? 1u : 0u;
        uint32_t idx, total;
        Scan(tmp).ExclusiveSum(flag, idx, total);
        if (WRITE && flag) {
            const uint32_t key = keys[i];
            double s = 0.0;  // np.bincount: 0.0, then += weights in input order
            for (uint64_t k = i; k < end && keys[k] == key; ++k) s = __dadd_rn(s, vals[k]);
            dep_cell[out0 + carry + idx] = key;
            dep_energy[out0 + carry + idx] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (!WRITE && threadIdx.x == 0) counts[blockIdx.x] = carry;
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
struct DepositScratch {
    size_t keys, vals, counts, sort_temp, scan_temp, total;
};

DepositScratch deposit_layout(uint64_t total_hits, uint32_t nevents) {
    size_t sort_temp = 0, scan_temp = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sort_temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                             (const double*)nullptr, (double*)nullptr, (int64_t)total_hits,
                                             (int64_t)nevents, (const uint64_t*)nullptr, (const uint64_t*)nullptr);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_temp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int64_t)nevents + 1);
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    DepositScratch d;
    d.keys = up(total_hits * sizeof(uint32_t));
    d.vals = up(total_hits * sizeof(double));
    d.counts = up(((size_t)nevents + 1) * sizeof(uint64_t));
    d.sort_temp = up(sort_temp);
    d.scan_temp = up(scan_temp);
    d.total = d.keys + d.vals + d.counts + d.sort_temp + d.scan_temp;
    return d;
}
}  // namespace

size_t prng_calo_deposit_scratch_bytes(uint64_t total_hits, uint32_t nevents) {
    return deposit_layout(total_hits, nevents).total;
}

int prng_calo_deposit(const uint32_t* hit_cell, const double* hit_amount, uint64_t total_hits,
                      const uint64_t* event_hit_offsets, uint32_t nevents, uint32_t cell_bits, void* scratch,
                      size_t scratch_bytes, uint32_t* dep_cell, double* dep_energy, uint64_t* dep_offsets,
                      void* stream) {
    if (nevents == 0) return PRNG_OK;
    if (!hit_cell || !hit_amount || !event_hit_offsets || !dep_cell || !dep_energy || !dep_offsets)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    if (cell_bits > 32) return calo_fail(PRNG_ERR_INVALID_PARAMETER, "cell_bits must be <= 32");
    const DepositScratch L = deposit_layout(total_hits, nevents);
    if (!scratch || scratch_bytes < L.total)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "scratch too small: need %zu bytes", L.total);
    cudaStream_t s = (cudaStream_t)stream;
    char* p = static_cast<char*>(scratch);
    uint32_t* keys_out = reinterpret_cast<uint32_t*>(p);
    p += L.keys;
    double* vals_out = reinterpret_cast<double*>(p);
    p += L.vals;
    uint64_t* counts = reinterpret_cast<uint64_t*>(p);
    p += L.counts;
    void* sort_temp = p;
    p += L.sort_temp;
    void* scan_temp = p;
    size_t sort_bytes = L.sort_temp, scan_bytes = L.scan_temp;
    const int end_bit = cell_bits == 0 ? 32 : (int)cell_bits;  // keys < 2^cell_bits: fewer radix passes
    if (total_hits) {
        cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(sort_temp, sort_bytes, hit_cell, keys_out,
                                                                 hit_amount, vals_out, (int64_t)total_hits,
                                                                 (int64_t)nevents, event_hit_offsets,
                                                                 event_hit_offsets + 1, 0, end_bit, s);
        if (e != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "segmented sort: %s", cudaGetErrorString(e));
    }
    cudaMemsetAsync(counts + nevents, 0, sizeof(uint64_t), s);
    calo_reduce_kernel<false><<<nevents, kCaloThreads, 0, s>>>(keys_out, vals_out, event_hit_offsets, counts,
                                                               nullptr, nullptr, nullptr);
    cudaError_t e = cub::DeviceScan::ExclusiveSum(scan_temp, scan_bytes, counts, dep_offsets, (int64_t)nevents + 1, s);
    if (e != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "offset scan: %s", cudaGetErrorString(e));
    calo_reduce_kernel<true><<<nevents, kCaloThreads, 0, s>>>(keys_out, vals_out, event_hit_offsets, nullptr,
                                                              dep_offsets, dep_cell, dep_energy);
    e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(e));
}

}  // extern "C"
