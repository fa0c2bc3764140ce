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
