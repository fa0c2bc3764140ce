// select_common.cuh -- block-wide MSB-first radix select on 64-bit keys (blockDim.x == 256).
#pragma once
#include "common.cuh"

namespace qadc {

struct SelectScratch {
    uint32_t hist[256];
    uint64_t prefix;
    uint32_t rank;
    uint32_t cnt_less, cnt_eq;
    uint32_t bucket; // population of the bucket the r-th key fell into after the last pass
};

// Finds the r-th smallest (1-based) of key_at(0..total) whose significant bits are
// [0, top_bit).  Returns the key; *eq_needed = how many copies of it belong to the r smallest.
// Every thread of the 256-thread block must call this; all get the same result.
template <class KeyAt>
__device__ uint64_t block_select_kth(KeyAt key_at, uint32_t total, uint32_t r, int top_bit, SelectScratch* sc,
                                     uint32_t* eq_needed) {
    if (threadIdx.x == 0) {
        sc->prefix = 0;
        sc->rank = r;
    }
    for (int shift = top_bit - 8; shift >= 0; shift -= 8) {
        sc->hist[threadIdx.x] = 0;
        __syncthreads();
        const uint64_t prefix = sc->prefix;
        const uint64_t himask = shift + 8 >= 64 ? 0ull : (~0ull << (shift + 8));
        // Keys of one query share their leading bytes, so a plain histogram would hammer one bin with
        // serialised same-address atomics: aggregate equal digits inside the warp first (one atomic per
        // distinct digit per warp).  The loop bound is warp-uniform so that ballot/match are legal.
        for (uint32_t base = 0; base < total; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            uint64_t k = 0;
            bool live = i < total;
            if (live) {
                k = key_at(i);
                live = (k & himask) == (prefix & himask);
            }
            const uint32_t digit = uint32_t(k >> shift) & 255u;
            const uint32_t act = __ballot_sync(0xffffffffu, live);
            if (live) {
                const uint32_t peers = __match_any_sync(act, digit);
                if ((threadIdx.x & 31u) == uint32_t(__ffs(peers) - 1)) atomicAdd(&sc->hist[digit], uint32_t(__popc(peers)));
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) { // lane l owns bins 8l..8l+7
            uint32_t loc[8], sum = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                loc[b] = sc->hist[threadIdx.x * 8 + b];
                sum += loc[b];
            }
            uint32_t incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (int(threadIdx.x) >= o) incl += v;
            }
            uint32_t excl = incl - sum;
            const uint32_t rank = sc->rank;
            if (rank > excl && rank <= incl) {
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (rank > excl && rank <= excl + loc[b]) {
                        sc->prefix = prefix | (uint64_t(threadIdx.x * 8 + b) << shift);
                        sc->rank = rank - excl;
                        sc->bucket = loc[b];
                    }
                    excl += loc[b];
                }
            }
        }
        __syncthreads();
        if (sc->bucket == 1 && shift > 0) {
            // the bucket holds exactly one key: it IS the r-th smallest; fetch its low bits and stop
            const uint64_t pfx = sc->prefix;
            const uint64_t hm = ~0ull << shift;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
                const uint64_t k = key_at(i);
                if ((k & hm) == (pfx & hm)) sc->prefix = k;
            }
            __syncthreads();
            *eq_needed = 1;
            return sc->prefix;
        }
    }
    *eq_needed = sc->rank;
    return sc->prefix;
}

// Copies the r smallest keys (unordered) to out[0..r) given the select result.
template <class KeyAt>
__device__ void block_keep_smallest(KeyAt key_at, uint32_t total, uint32_t r, uint64_t kth, uint32_t eq_needed,
                                    SelectScratch* sc, uint64_t* out) {
    const uint32_t less = r - eq_needed;
    if (threadIdx.x == 0) {
        sc->cnt_less = 0;
        sc->cnt_eq = 0;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
        const uint64_t k = key_at(i);
        if (k < kth) out[atomicAdd(&sc->cnt_less, 1u)] = k;
        else if (k == kth) {
            const uint32_t e = atomicAdd(&sc->cnt_eq, 1u);
            if (e < eq_needed) out[less + e] = k;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t code_field(const DevSpec& ds, const uint8_t* code, uint32_t j) {
    const uint32_t bp = ds.bitpos[j];
    const uint32_t w = reinterpret_cast<const uint32_t*>(code)[bp >> 5];
    return (w >> (bp & 31u)) & ((1u << ds.bits[j]) - 1u);
}

// the same for a 64-bit code already in two registers (one 8-byte load per code instead of one load per field)
__device__ __forceinline__ uint32_t code_field64(const DevSpec& ds, uint32_t lo, uint32_t hi, uint32_t j) {
    const uint32_t bp = ds.bitpos[j];
    const uint32_t w = (bp >> 5) ? hi : lo;
    return (w >> (bp & 31u)) & ((1u << ds.bits[j]) - 1u);
}

} // namespace qadc
