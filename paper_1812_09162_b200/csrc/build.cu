// IVF list construction on the device ("next" row N3): the data-dependent half of IvfIndex::build
// (index.hpp:195-227) given a trained coarse quantizer and residual codebook --
//   assignment: nearest coarse centroid under a DOUBLE accumulator walked serially over the dims,
//               ties to the lowest cell (kmeans.hpp:178-190, detail::sq_dist :41-48);
//   residual:   x - centroid in fp32 (index.hpp:200);
//   encode:     launch_encode (codebook.hpp:94-118) on the residuals.
// Training (k-means) stays on the host: it is out of the hot path.
#include "common.cuh"

namespace qadc {

static constexpr int ASSIGN_VT = 16; // vectors per CTA sharing every centroid load

// grid (ceil(K/256), ceil(n/ASSIGN_VT)).  Thread = cell; the CTA's ASSIGN_VT vectors sit in shared
// memory as [dim][vector] doubles.  Each thread's 16 distances go through a (distance, cell)
// lexicographic reduction, which is the sequential "d < best" rule, and the CTA's winner per
// vector is written to partial[vector][blockIdx.x].
__global__ void __launch_bounds__(256)
assign_partial_kernel(const float* __restrict__ vectors, const float* __restrict__ coarse_t, uint32_t dims,
                      uint32_t k_cells, uint64_t n, double* __restrict__ part_dist, uint32_t* __restrict__ part_cell) {
    extern __shared__ __align__(16) double xs[]; // [dims][ASSIGN_VT]
    __shared__ double red_d[8][ASSIGN_VT];
    __shared__ uint32_t red_c[8][ASSIGN_VT];
    const uint64_t v0 = uint64_t(blockIdx.y) * ASSIGN_VT;
    for (uint32_t u = threadIdx.x; u < dims * ASSIGN_VT; u += blockDim.x) {
        const uint32_t vi = u % ASSIGN_VT, j = u / ASSIGN_VT;
        xs[u] = v0 + vi < n ? double(vectors[(v0 + vi) * dims + j]) : 0.0;
    }
    __syncthreads();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = c < k_cells;
    double acc[ASSIGN_VT];
#pragma unroll
    for (int i = 0; i < ASSIGN_VT; ++i) acc[i] = 0.0;
    if (live) {
        for (uint32_t j = 0; j < dims; ++j) {
            const double ctr = double(coarse_t[size_t(j) * k_cells + c]);
            const double2* xv = reinterpret_cast<const double2*>(xs + j * ASSIGN_VT);
#pragma unroll
            for (int v = 0; v < ASSIGN_VT / 2; ++v) {
                const double2 x = xv[v];
                double d;
                d = __dsub_rn(x.x, ctr); acc[2 * v + 0] = __dadd_rn(acc[2 * v + 0], __dmul_rn(d, d));
                d = __dsub_rn(x.y, ctr); acc[2 * v + 1] = __dadd_rn(acc[2 * v + 1], __dmul_rn(d, d));
            }
        }
    }
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < ASSIGN_VT; ++i) {
        // a NaN or infinite distance never satisfies the reference's "d < best" against best = +inf
        const bool cand = live && acc[i] < inf;
        double d = cand ? acc[i] : inf;
        uint32_t cc = cand ? c : 0xffffffffu;
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, d, o);
            const uint32_t oc = __shfl_xor_sync(0xffffffffu, cc, o);
            if (od < d || (od == d && oc < cc)) {
                d = od;
                cc = oc;
            }
        }
        if (lane == 0) {
            red_d[warp][i] = d;
            red_c[warp][i] = cc;
        }
    }
    __syncthreads();
    if (threadIdx.x < ASSIGN_VT && v0 + threadIdx.x < n) {
        double d = red_d[0][threadIdx.x];
        uint32_t cc = red_c[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) {
            const double od = red_d[w][threadIdx.x];
            const uint32_t oc = red_c[w][threadIdx.x];
            if (od < d || (od == d && oc < cc)) {
                d = od;
                cc = oc;
            }
        }
        part_dist[(v0 + threadIdx.x) * gridDim.x + blockIdx.x] = d;
        part_cell[(v0 + threadIdx.x) * gridDim.x + blockIdx.x] = cc;
    }
}

// One thread per vector: fold the cell-block winners in ascending cell order with a strict "<"
// (NaN distances never win, so an all-NaN vector lands in cell 0 like the reference's loop),
// then the fp32 residual against the winning centroid (row-major coarse).
__global__ void assign_final_kernel(const double* __restrict__ part_dist, const uint32_t* __restrict__ part_cell,
                                    uint32_t n_parts, uint64_t n, uint32_t* __restrict__ assign) {
    const uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (v >= n) return;
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t best_c = 0;
    for (uint32_t p = 0; p < n_parts; ++p) {
        const double d = part_dist[v * n_parts + p];
        if (d < best) {
            best = d;
            best_c = part_cell[v * n_parts + p];
        }
    }
    assign[v] = best_c;
}

__global__ void residual_kernel(const float* __restrict__ vectors, const float* __restrict__ coarse,
                                const uint32_t* __restrict__ assign, uint32_t dims, uint64_t n,
                                float* __restrict__ resid) {
    const uint64_t u = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (u >= n * dims) return;
    const uint64_t v = u / dims;
    const uint32_t j = uint32_t(u - v * dims);
    resid[u] = __fsub_rn(vectors[u], coarse[size_t(assign[v]) * dims + j]);
}

size_t ivf_assign_scratch_bytes(uint32_t k_cells, uint64_t n) {
    const uint64_t parts = (k_cells + 255) / 256;
    return size_t(n) * parts * (sizeof(double) + sizeof(uint32_t)) + 256;
}

void launch_ivf_assign(const float* d_vectors, const float* d_coarse, const float* d_coarse_t, uint32_t dims,
                       uint32_t k_cells, uint64_t n, void* d_scratch, uint32_t* d_assign, float* d_resid,
                       cudaStream_t stream) {
    if (n == 0) return;
    const uint32_t parts = (k_cells + 255) / 256;
    double* pd = static_cast<double*>(d_scratch);
    uint32_t* pc = reinterpret_cast<uint32_t*>(pd + size_t(n) * parts);
    const size_t smem = size_t(dims) * ASSIGN_VT * sizeof(double);
    if (smem > 200 * 1024) throw Error(QADC_ERR_CONFIG, "ivf build: too many dimensions for the assignment tile");
    QADC_CUDA_CHECK(cudaFuncSetAttribute(assign_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const dim3 grid(parts, unsigned((n + ASSIGN_VT - 1) / ASSIGN_VT));
    assign_partial_kernel<<<grid, 256, smem, stream>>>(d_vectors, d_coarse_t, dims, k_cells, n, pd, pc);
    assign_final_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(pd, pc, parts, n, d_assign);
    const uint64_t elems = n * dims;
    residual_kernel<<<unsigned((elems + 255) / 256), 256, 0, stream>>>(d_vectors, d_coarse, d_assign, dims, n, d_resid);
    g_launches += 3;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc

// ------------------------------------------------------------------------------------------------------------------
// Per-list grouping + packing on the device (IvfIndex::build's last step, index.hpp:219-227): every cell's members in
// ascending vector index, one PackedList per cell (layout.hpp:50-68 LSB-first subcode packing, :105-160 transposed
// blocks of block_len codes with all-ones tail padding), ids = vector indices.  Outputs are qadc_ivf_open's arguments.
//   1. histogram of the assignment -> list_count; exclusive scans -> list_id_off (ids) and list_byte_off (whole blocks)
//   2. stable grouping: radix sort of (cell, vector index) pairs.  This one step calls a library (cub::DeviceRadixSort,
//      part of the CUDA toolkit): it is index construction, not the scan path, and a stable sort is exactly the
//      reference's "members in index order" rule.
//   3. pack kernel: one thread per (cell, padded position): LSB-first words, transposed block address, 0xFF padding.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
namespace qadc {

__global__ void ivf_hist_kernel(const uint32_t* __restrict__ assign, uint64_t n, uint32_t k_cells,
                                unsigned long long* __restrict__ counts, int* __restrict__ status) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = assign[i];
    if (c >= k_cells) {
        atomicExch(status, QADC_ERR_CORRUPTION);
        return;
    }
    atomicAdd(&counts[c], 1ull);
}

// single CTA: exclusive scans of the counts (ids) and of the lists' packed sizes (bytes)
__global__ void ivf_offsets_kernel(const unsigned long long* __restrict__ counts, uint32_t k_cells, uint32_t block_len,
                                   uint64_t block_bytes, unsigned long long* __restrict__ id_off,
                                   unsigned long long* __restrict__ byte_off, unsigned long long* __restrict__ totals) {
    __shared__ unsigned long long s_id[1024], s_by[1024];
    __shared__ unsigned long long run_id, run_by;
    if (threadIdx.x == 0) run_id = run_by = 0;
    __syncthreads();
    for (uint32_t base = 0; base < k_cells; base += 1024) {
        const uint32_t c = base + threadIdx.x;
        const unsigned long long cnt = c < k_cells ? counts[c] : 0ull;
        const unsigned long long by = (cnt + block_len - 1) / block_len * block_bytes;
        s_id[threadIdx.x] = cnt;
        s_by[threadIdx.x] = by;
        __syncthreads();
        for (uint32_t o = 1; o < 1024; o <<= 1) { // Hillis-Steele inclusive scan
            unsigned long long a = 0, b = 0;
            if (threadIdx.x >= o) {
                a = s_id[threadIdx.x - o];
                b = s_by[threadIdx.x - o];
            }
            __syncthreads();
            s_id[threadIdx.x] += a;
            s_by[threadIdx.x] += b;
            __syncthreads();
        }
        if (c < k_cells) {
            id_off[c] = run_id + s_id[threadIdx.x] - cnt;
            byte_off[c] = run_by + s_by[threadIdx.x] - by;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            run_id += s_id[1023];
            run_by += s_by[1023];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        totals[0] = run_id;
        totals[1] = run_by;
    }
}

__global__ void ivf_iota_kernel(uint32_t* __restrict__ v, uint64_t n) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = uint32_t(i);
}

// grid.x = cells (grid-stride), threads walk the cell's padded positions
__global__ void ivf_pack_lists_kernel(DevSpec ds, uint32_t g, uint32_t rows, uint32_t block_len, const uint8_t* __restrict__ codes,
                                      const uint32_t* __restrict__ order, const unsigned long long* __restrict__ counts,
                                      const unsigned long long* __restrict__ id_off,
                                      const unsigned long long* __restrict__ byte_off, uint32_t k_cells,
                                      uint8_t* __restrict__ packed) {
    const uint32_t wb = ds.word_width / 8;
    for (uint32_t c = blockIdx.x; c < k_cells; c += gridDim.x) {
        const uint64_t cnt = counts[c], padded = (cnt + block_len - 1) / block_len * block_len;
        uint8_t* out = packed + byte_off[c];
        for (uint64_t p = threadIdx.x; p < padded; p += blockDim.x) {
            const uint64_t b = p / block_len, slot = p % block_len;
            const uint8_t* sub = p < cnt ? codes + size_t(order[id_off[c] + p]) * ds.m : nullptr;
            for (uint32_t r = 0; r < rows; ++r) {
                uint32_t w = ds.word_width == 16 ? 0xFFFFu : 0xFFu; // tail slots: all-ones words (layout.hpp:117)
                if (sub) {
                    w = 0;
                    uint32_t off = 0;
                    for (uint32_t k = 0; k < g; ++k) { // pack_group (layout.hpp:50-60): LSB first
                        w |= uint32_t(sub[r * g + k]) << off;
                        off += ds.bits[r * g + k];
                    }
                }
                uint8_t* dst = out + ((b * rows + r) * block_len + slot) * wb;
                if (wb == 2) *reinterpret_cast<uint16_t*>(dst) = uint16_t(w);
                else *dst = uint8_t(w);
            }
        }
    }
}

// Everything on the device; d_assign [n], d_codes [n * m] come from launch_ivf_assign / launch_encode.
// d_counts / d_id_off / d_byte_off: k_cells u64 each; d_order: n u32; d_totals: 2 u64 {n, packed bytes};
// d_packed must hold ivf_build_packed_bound() bytes.
void launch_ivf_group_pack(const qadc_spec& spec, const DevSpec& ds, const uint32_t* d_assign, const uint8_t* d_codes, uint64_t n,
                           uint32_t k_cells, unsigned long long* d_counts, unsigned long long* d_id_off,
                           unsigned long long* d_byte_off, unsigned long long* d_totals, uint32_t* d_order, uint8_t* d_packed,
                           int* d_status, cudaStream_t stream) {
    QADC_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, size_t(k_cells) * 8, stream));
    if (n) ivf_hist_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(d_assign, n, k_cells, d_counts, d_status);
    const uint64_t block_bytes = uint64_t(spec.groups) * spec.block_len * (spec.word_width / 8);
    ivf_offsets_kernel<<<1, 1024, 0, stream>>>(d_counts, k_cells, spec.block_len, block_bytes, d_id_off, d_byte_off, d_totals);
    g_launches += 2;
    if (n) {
        // stable sort of (cell, index): sorted values = every cell's members in ascending vector index
        uint32_t *keys_in = nullptr, *keys_out = nullptr, *vals_in = nullptr;
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        int end_bit = 1;
        while ((1ull << end_bit) < k_cells && end_bit < 32) ++end_bit;
        QADC_CUDA_CHECK(cudaMalloc(&keys_out, n * 4));
        QADC_CUDA_CHECK(cudaMalloc(&vals_in, n * 4));
        keys_in = const_cast<uint32_t*>(d_assign);
        ivf_iota_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(vals_in, n);
        cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, vals_in, d_order, n, 0, end_bit, stream);
        if (e == cudaSuccess) e = cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 16));
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, d_order, n, 0, end_bit, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        cudaFree(tmp);
        cudaFree(keys_out);
        cudaFree(vals_in);
        QADC_CUDA_CHECK(e);
    }
    ivf_pack_lists_kernel<<<std::min<uint32_t>(std::max<uint32_t>(k_cells, 1u), 148u * 16u), 256, 0, stream>>>(
        ds, spec.g, spec.groups, spec.block_len, d_codes, d_order, d_counts, d_id_off, d_byte_off, k_cells, d_packed);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
