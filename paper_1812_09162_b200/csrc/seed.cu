// seed.cu -- dense exact top-R over the HEAD of a list, one CTA per query.
//
// The streaming scan (scan.cu) only appends pairs that beat the query's current R-th
// best key, so it needs a threshold before it starts.  The reference's heap gets one
// implicitly by pushing the first R codes (heap.hpp:41-45).  Here every query's CTA
// evaluates the first S0 (<= 4096) codes exactly -- scan_scalar.hpp:52-58 semantics,
// integer saturating sums from the query's quantized table held in shared memory --
// radix-selects the R smallest (distance, id) keys and stores them as the query's
// running top-R with thr_key = the R-th key.  After S0 codes the admission rate of the
// streaming scan is already R/S0 (2.4 % at R=100), and it falls as 1/n from there.
#include "select_common.cuh"

namespace qadc {

static constexpr int SEED_THREADS = 256;

// dynamic smem: keys[n_head] (u64) | table[E] (u16)
__global__ void __launch_bounds__(SEED_THREADS)
seed_topk_kernel(DevSpec ds, const uint8_t* __restrict__ codes, uint32_t n_head, uint32_t id_base,
                 const uint32_t* __restrict__ ids, const void* __restrict__ qlut, const uint32_t* __restrict__ row_bias,
                 uint32_t r, uint64_t* __restrict__ top, uint32_t* __restrict__ ntop, uint32_t kpad,
                 uint64_t* __restrict__ thr_key) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm_raw);
    uint16_t* table = reinterpret_cast<uint16_t*>(keys + n_head);
    __shared__ SelectScratch sc;

    const uint32_t q = blockIdx.x;
    for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x)
        table[e] = ds.word_width == 8 ? uint16_t(reinterpret_cast<const uint8_t*>(qlut)[size_t(q) * ds.E + e])
                                      : reinterpret_cast<const uint16_t*>(qlut)[size_t(q) * ds.E + e];
    __syncthreads();
    const uint32_t bias = row_bias ? min(row_bias[q], ds.qmax) : 0u;
    for (uint32_t i = threadIdx.x; i < n_head; i += blockDim.x) {
        const uint8_t* code = codes + size_t(i) * ds.code_stride;
        uint32_t acc = bias;
        if (ds.code_stride == 8) {
            const uint2 cw = *reinterpret_cast<const uint2*>(code);
            for (uint32_t j = 0; j < ds.m; ++j) acc += table[ds.ent_off[j] + code_field64(ds, cw.x, cw.y, j)];
        } else {
            for (uint32_t j = 0; j < ds.m; ++j) acc += table[ds.ent_off[j] + code_field(ds, code, j)];
        }
        acc = min(acc, ds.qmax); // == the chain of saturating adds (all terms unsigned)
        keys[i] = make_key(acc, ids ? ids[i] : id_base + i);
    }
    __syncthreads();
    uint64_t* my_top = top + size_t(q) * kpad;
    if (n_head <= r) { // fewer codes than R: the heap just holds them all (heap.hpp:41-45)
        uint64_t mx = 0;
        for (uint32_t i = threadIdx.x; i < n_head; i += blockDim.x) {
            my_top[i] = keys[i];
            mx = max(mx, keys[i]);
        }
        if (n_head == r) {
            __shared__ uint64_t wmax[SEED_THREADS / 32];
            for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 0; w < SEED_THREADS / 32; ++w) mx = max(mx, wmax[w]);
                thr_key[q] = mx;
            }
        }
        if (threadIdx.x == 0) ntop[q] = n_head;
        return;
    }
    auto key_at = [&](uint32_t i) -> uint64_t { return keys[i]; };
    uint32_t eq_needed;
    const uint64_t kth = block_select_kth(key_at, n_head, r, 48, &sc, &eq_needed);
    block_keep_smallest(key_at, n_head, r, kth, eq_needed, &sc, my_top);
    if (threadIdx.x == 0) {
        ntop[q] = r;
        thr_key[q] = kth;
    }
}

void launch_seed_topk(const DevSpec& ds, const uint8_t* d_codes, uint32_t n_head, uint32_t id_base,
                      const uint32_t* d_ids, const void* d_qlut, const uint32_t* d_row_bias, uint32_t nq, uint32_t r,
                      uint64_t* top, uint32_t* ntop, uint32_t kpad, uint64_t* thr_key, cudaStream_t stream) {
    if (nq == 0 || n_head == 0) return;
    const size_t smem = size_t(n_head) * 8 + size_t(ds.E) * 2;
    if (smem > 200 * 1024) throw Error(QADC_ERR_CONFIG, "seed: head + table exceed shared memory");
    QADC_CUDA_CHECK(cudaFuncSetAttribute(seed_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    seed_topk_kernel<<<nq, SEED_THREADS, smem, stream>>>(ds, d_codes, n_head, id_base, d_ids, d_qlut, d_row_bias, r,
                                                         top, ntop, kpad, thr_key);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
