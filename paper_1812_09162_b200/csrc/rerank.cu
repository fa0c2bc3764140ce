// rerank.cu -- exact re-ranking of the final top-R ("next" row N4).
//
// detail::rerank_by_float (index.hpp:53-67) with FlatIndex::rerank_exact (:148-152) /
// IvfIndex::rerank_exact (:377-386): the R survivors of the quantized search are re-ordered by
// their float ADC distance -- adc_scalar_float (distance.hpp:61-69): fp32 sum of the float table
// entries in table order -- with ties by id; the reported distances become the float ones.  The SET
// of results does not change.  One CTA per query; key = float bits << 32 | id (distances are >= +0,
// so float order == bit order), bitonic sort in shared memory.
#include "select_common.cuh"

namespace qadc {

struct RerankArgs {
    const uint8_t* codes;
    const float* luts;            // flat: [nq][E]; ivf: [nq * a][E]
    uint32_t base_id;             // flat: list position = id - base_id
    const uint32_t* locator;      // ivf: id -> device code position
    const uint64_t* list_code_off; // ivf: first device code of every list (ascending)
    const uint32_t* order;        // ivf: [nq][a] probed cells
    uint32_t k_cells, a;
    uint32_t r;
    uint32_t* ids;                // in/out [nq][r]
    float* dists;                 // in/out [nq][r]
    const uint32_t* counts;       // [nq]
};

__global__ void __launch_bounds__(256) rerank_kernel(DevSpec ds, RerankArgs g, uint32_t pow2) {
    extern __shared__ uint64_t keys[];
    const uint32_t q = blockIdx.x;
    const uint32_t n = min(g.counts[q], g.r);
    for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x) {
        uint64_t key = KEY_INF;
        if (i < n) {
            const uint32_t id = g.ids[size_t(q) * g.r + i];
            uint64_t pos;
            const float* lut;
            if (g.locator) {
                pos = g.locator[id];
                uint32_t lo = 0, hi = g.k_cells; // cell = last list starting at or before pos
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (g.list_code_off[mid] <= pos) lo = mid;
                    else hi = mid;
                }
                uint32_t pi = 0;
                while (pi + 1 < g.a && g.order[size_t(q) * g.a + pi] != lo) ++pi; // std::find over the probe order
                lut = g.luts + (size_t(q) * g.a + pi) * ds.E;
            } else {
                pos = id - g.base_id;
                lut = g.luts + size_t(q) * ds.E;
            }
            const uint8_t* code = g.codes + pos * ds.code_stride;
            float acc = 0.0f;
            for (uint32_t j = 0; j < ds.m; ++j) acc = __fadd_rn(acc, lut[ds.ent_off[j] + code_field(ds, code, j)]);
            key = (uint64_t(__float_as_uint(acc)) << 32) | id;
        }
        keys[i] = key;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= pow2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < pow2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = keys[lo], y = keys[hi];
                if ((x > y) == up) {
                    keys[lo] = y;
                    keys[hi] = x;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        g.ids[size_t(q) * g.r + i] = uint32_t(keys[i]);
        g.dists[size_t(q) * g.r + i] = __uint_as_float(uint32_t(keys[i] >> 32));
    }
}

void launch_rerank(const DevSpec& ds, const uint8_t* d_codes, const float* d_luts, uint32_t base_id,
                   const uint32_t* d_locator, const uint64_t* d_list_code_off, const uint32_t* d_order, uint32_t k_cells,
                   uint32_t a, uint32_t nq, uint32_t r, uint32_t* d_ids, float* d_dists, const uint32_t* d_counts,
                   cudaStream_t stream) {
    if (nq == 0) return;
    uint32_t pow2 = 2;
    while (pow2 < r) pow2 <<= 1;
    RerankArgs g{d_codes, d_luts, base_id, d_locator, d_list_code_off, d_order, k_cells, a, r, d_ids, d_dists, d_counts};
    rerank_kernel<<<nq, 256, size_t(pow2) * 8, stream>>>(ds, g, pow2);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
