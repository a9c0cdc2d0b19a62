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
//     followed by one sequential run-sum per unique cell, compacted with a
//     block scan.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/prng_b200.h"

namespace {

constexpr int kCaloThreads = 256;

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), float64.
__device__ double np_pairwise_sum(const double* a, uint64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (uint64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
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
    uint64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
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

// One thread per particle: raw_sum, in-place scaling to amounts, particle sum.
__global__ void calo_normalize_kernel(const prng_calo_particle_t* __restrict__ parts, uint32_t nparts,
                                      double* __restrict__ hit_amount, double* __restrict__ particle_sums) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nparts) return;
    const prng_calo_particle_t pt = parts[p];
    if (pt.hits == 0) {
        particle_sums[p] = 0.0;
        return;
    }
    double* a = hit_amount + pt.hit_offset;
    const double raw_sum = np_pairwise_sum(a, pt.hits);
    if (raw_sum > 0.0) {
        const double scale = pt.target / raw_sum;
        for (uint32_t j = 0; j < pt.hits; ++j) a[j] = __dmul_rn(a[j], scale);
    } else {
        const double each = pt.target / (double)pt.hits;  // np.full(m, target / m)
        for (uint32_t j = 0; j < pt.hits; ++j) a[j] = each;
    }
    particle_sums[p] = np_pairwise_sum(a, pt.hits);
}

// One CTA per event over its cell-sorted hits: run starts -> compacted
// (cell, sequential run sum) at the event's offset.
__global__ void __launch_bounds__(kCaloThreads)
    calo_reduce_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ vals,
                       const uint64_t* __restrict__ ev_off, uint32_t* __restrict__ dep_cell,
                       double* __restrict__ dep_energy, uint32_t* __restrict__ dep_count) {
    using Scan = cub::BlockScan<uint32_t, kCaloThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t carry;
    const uint64_t beg = ev_off[blockIdx.x], end = ev_off[blockIdx.x + 1];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = beg; base < end; base += kCaloThreads) {
        const uint64_t i = base + threadIdx.x;
        const uint32_t flag = (i < end && (i == beg || keys[i] != keys[i - 1])) ? 1u : 0u;
        uint32_t idx, total;
        Scan(tmp).ExclusiveSum(flag, idx, total);
        if (flag) {
            const uint32_t key = keys[i];
            double s = 0.0;  // np.bincount: 0.0, then += weights in input order
            for (uint64_t k = i; k < end && keys[k] == key; ++k) s = __dadd_rn(s, vals[k]);
            dep_cell[beg + carry + idx] = key;
            dep_energy[beg + carry + idx] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) dep_count[blockIdx.x] = carry;
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
    calo_normalize_kernel<<<(nparticles + 127) / 128, 128, 0, s>>>(particles, nparticles, hit_amount,
                                                                    particle_sums);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo hits: %s", cudaGetErrorString(e));
}

size_t prng_calo_deposit_scratch_bytes(uint64_t total_hits, uint32_t nevents) {
    size_t temp = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                             (const double*)nullptr, (double*)nullptr, (int64_t)total_hits,
                                             (int64_t)nevents, (const uint64_t*)nullptr, (const uint64_t*)nullptr);
    const size_t align = 256;
    auto up = [&](size_t b) { return (b + align - 1) / align * align; };
    return up(total_hits * sizeof(uint32_t)) + up(total_hits * sizeof(double)) + up(temp);
}

int prng_calo_deposit(const uint32_t* hit_cell, const double* hit_amount, uint64_t total_hits,
                      const uint64_t* event_hit_offsets, uint32_t nevents, void* scratch, size_t scratch_bytes,
                      uint32_t* dep_cell, double* dep_energy, uint32_t* dep_count, void* stream) {
    if (nevents == 0) return PRNG_OK;
    if (!hit_cell || !hit_amount || !event_hit_offsets || !dep_cell || !dep_energy || !dep_count)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "NULL argument");
    const size_t need = prng_calo_deposit_scratch_bytes(total_hits, nevents);
    if (!scratch || scratch_bytes < need)
        return calo_fail(PRNG_ERR_INVALID_PARAMETER, "scratch too small: need %zu bytes", need);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t align = 256;
    auto up = [&](size_t b) { return (b + align - 1) / align * align; };
    char* p = static_cast<char*>(scratch);
    uint32_t* keys_out = reinterpret_cast<uint32_t*>(p);
    p += up(total_hits * sizeof(uint32_t));
    double* vals_out = reinterpret_cast<double*>(p);
    p += up(total_hits * sizeof(double));
    size_t temp = scratch_bytes - (size_t)(p - static_cast<char*>(scratch));
    if (total_hits) {
        cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(p, temp, hit_cell, keys_out, hit_amount, vals_out,
                                                                 (int64_t)total_hits, (int64_t)nevents,
                                                                 event_hit_offsets, event_hit_offsets + 1, 0, 32, s);
        if (e != cudaSuccess) return calo_fail(PRNG_ERR_CUDA, "segmented sort: %s", cudaGetErrorString(e));
    }
    calo_reduce_kernel<<<nevents, kCaloThreads, 0, s>>>(keys_out, vals_out, event_hit_offsets, dep_cell,
                                                        dep_energy, dep_count);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PRNG_OK : calo_fail(PRNG_ERR_CUDA, "calo deposit: %s", cudaGetErrorString(e));
}

}  // extern "C"
