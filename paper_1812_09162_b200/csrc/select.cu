// select.cu -- deterministic top-R selection: the device counterpart of
// CandidateHeap<uint32_t> (heap.hpp:16-71).
//
// The reference keeps "the R lexicographically smallest (distance, id) pairs seen so
// far"; its final content is independent of insertion order (heap.hpp:12-14).  With
// key = distance<<32 | id that set is the R smallest keys, so any selection that
// returns exactly those keys, ascending, is bit-identical to heap.sorted().
//
// Per query the scan appends every pair whose key beats the current R-th smallest
// key (thr_key) to a candidate buffer; between scan segments `tighten` folds the
// buffer into the running top-R with an MSB-first radix select and refreshes thr_key,
// which is what the heap's worst() does continuously on the CPU.  `finalize` sorts
// the survivors (bitonic, shared memory) and applies the affine map
// (unquantize, distance.hpp:158-161 / index.hpp:335-338).
#include "select_common.cuh"

namespace qadc {

__global__ void init_select_kernel(uint64_t* thr_key, uint32_t* cand_count, uint32_t* ntop, uint32_t* overflow,
                                   uint32_t nq) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    thr_key[q] = KEY_INF;
    cand_count[q] = 0;
    ntop[q] = 0;
    overflow[q] = 0;
}

void launch_init_select(uint64_t* thr_key, uint32_t* cand_count, uint32_t* ntop, uint32_t* overflow, uint32_t nq,
                        cudaStream_t stream) {
    if (nq == 0) return;
    init_select_kernel<<<(nq + 255) / 256, 256, 0, stream>>>(thr_key, cand_count, ntop, overflow, nq);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

static constexpr int TIGHTEN_THREADS = 256;

// One CTA per query.  dynamic smem: r keys.
__global__ void __launch_bounds__(TIGHTEN_THREADS)
tighten_kernel(uint64_t* __restrict__ top, uint32_t* __restrict__ ntop, uint32_t kpad, uint64_t* __restrict__ cand,
               uint32_t* __restrict__ cand_count, uint32_t cap, uint64_t* __restrict__ thr_key, uint32_t r,
               unsigned long long* __restrict__ admitted) {
    extern __shared__ uint64_t keep[];
    __shared__ SelectScratch sc;

    const uint32_t q = blockIdx.x;
    const uint32_t n = min(cand_count[q], cap);
    if (n == 0) return;
    if (admitted && threadIdx.x == 0) atomicAdd(admitted, (unsigned long long)n); // statistics only
    const uint32_t nt = ntop[q];
    const uint32_t total = nt + n;
    uint64_t* my_top = top + size_t(q) * kpad;
    const uint64_t* my_cand = cand + size_t(q) * cap;

    if (total <= r) { // heap not over capacity: keep everything (heap.hpp:41-45)
        uint64_t mx = 0;
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) my_top[nt + i] = my_cand[i];
        if (total == r) {
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) mx = max(mx, my_top[i]);
            // block max
            for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            __shared__ uint64_t wmax[TIGHTEN_THREADS / 32];
            if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 0; w < TIGHTEN_THREADS / 32; ++w) mx = max(mx, wmax[w]);
                thr_key[q] = mx;
            }
        }
        if (threadIdx.x == 0) {
            ntop[q] = total;
            cand_count[q] = 0;
        }
        return;
    }

    auto key_at = [&](uint32_t i) -> uint64_t { return i < nt ? my_top[i] : my_cand[i - nt]; };
    // MSB-first radix select of the r-th smallest key (48 significant bits: 16 distance + 32 id)
    uint32_t eq_needed;
    const uint64_t kth = block_select_kth(key_at, total, r, 48, &sc, &eq_needed);
    block_keep_smallest(key_at, total, r, kth, eq_needed, &sc, keep);
    for (uint32_t i = threadIdx.x; i < r; i += blockDim.x) my_top[i] = keep[i];
    if (threadIdx.x == 0) {
        ntop[q] = r;
        cand_count[q] = 0;
        thr_key[q] = kth;
    }
}

void launch_tighten(uint64_t* top, uint32_t* ntop, uint32_t kpad, uint64_t* cand, uint32_t* cand_count, uint32_t cap,
                    uint64_t* thr_key, uint32_t nq, uint32_t r, unsigned long long* admitted, cudaStream_t stream) {
    if (nq == 0) return;
    if (size_t(r) * 8 > 48 * 1024) // R above 6144: opt in to the larger dynamic shared memory (QADC_MAX_R * 8 = 128 KB)
        QADC_CUDA_CHECK(cudaFuncSetAttribute(tighten_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(size_t(r) * 8)));
    tighten_kernel<<<nq, TIGHTEN_THREADS, size_t(r) * 8, stream>>>(top, ntop, kpad, cand, cand_count, cap, thr_key, r,
                                                                   admitted);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// One CTA per query: gather nlists lists of list_len keys, bitonic-sort ascending in
// shared memory, emit the first r.  lists layout: [list][query][list_len].
__global__ void finalize_kernel(const uint64_t* __restrict__ lists, const uint32_t* __restrict__ counts_in,
                                uint32_t list_len, uint32_t nlists, uint32_t nq, uint32_t r, uint32_t pow2,
                                const float* __restrict__ map, uint32_t flags, uint32_t qmax,
                                uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                                uint32_t* __restrict__ out_counts, uint64_t* __restrict__ out_keys) {
    extern __shared__ uint64_t s[];
    const uint32_t q = blockIdx.x;
    const uint32_t total = nlists * list_len;
    for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x) {
        uint64_t k = KEY_INF;
        if (i < total) {
            const uint32_t l = i / list_len, p = i % list_len;
            const bool valid = counts_in ? p < counts_in[size_t(l) * nq + q] : true;
            if (valid) k = lists[(size_t(l) * nq + q) * list_len + p];
        }
        s[i] = k;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= pow2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < pow2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1)); // index with the `stride` bit clear
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = s[lo], b = s[hi];
                if ((a > b) == up) {
                    s[lo] = b;
                    s[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    const float delta = map ? map[size_t(q) * 2] : 1.0f;
    const float d_min = map ? map[size_t(q) * 2 + 1] : 0.0f;
    uint32_t valid = 0;
    for (uint32_t i = threadIdx.x; i < r; i += blockDim.x) {
        const uint64_t k = i < pow2 ? s[i] : KEY_INF;
        const bool ok = k != KEY_INF;
        const uint32_t d = uint32_t(k >> 32);
        float dist = __int_as_float(0x7f800000);
        if (ok) {
            const float fd = float(min(d, qmax));
            dist = (flags & QADC_FLAG_FMA_UNQUANTIZE) ? __fmaf_rn(fd, delta, d_min) : __fadd_rn(__fmul_rn(fd, delta), d_min);
        }
        if (out_ids) out_ids[size_t(q) * r + i] = ok ? uint32_t(k) : 0xFFFFFFFFu;
        if (out_dists) out_dists[size_t(q) * r + i] = dist;
        if (out_keys) out_keys[size_t(q) * r + i] = k;
        valid += ok;
    }
    if (out_counts) {
        __shared__ uint32_t s_valid;
        if (threadIdx.x == 0) s_valid = 0;
        __syncthreads();
        if (valid) atomicAdd(&s_valid, valid);
        __syncthreads();
        if (threadIdx.x == 0) out_counts[q] = s_valid;
    }
}

void launch_finalize(const uint64_t* lists, const uint32_t* counts_in, uint32_t list_len, uint32_t nlists,
                     uint32_t nq, uint32_t r, const float* map, uint32_t flags, uint32_t qmax, uint32_t* out_ids,
                     float* out_dists, uint32_t* out_counts, uint64_t* out_keys, cudaStream_t stream) {
    if (nq == 0) return;
    uint32_t pow2 = 2;
    while (pow2 < nlists * list_len) pow2 <<= 1;
    const size_t smem = size_t(pow2) * 8;
    if (smem > 200 * 1024) throw Error(QADC_ERR_CONFIG, "finalize: too many keys per query for shared memory");
    QADC_CUDA_CHECK(cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int threads = pow2 >= 512 ? 256 : 128;
    finalize_kernel<<<nq, threads, smem, stream>>>(lists, counts_in, list_len, nlists, nq, r, pow2, map, flags, qmax,
                                                   out_ids, out_dists, out_counts, out_keys);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
