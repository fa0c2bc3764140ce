// scan_common.cuh -- pieces shared by the scan kernels (scan.cu: shared-memory table lookups; scan_tc.cu: one-hot
// int8 GEMM on tcgen05): mbarrier / TMA bulk-copy wrappers, compile-time code geometry and the exact admission test
// (CandidateHeap::push, heap.hpp:40-51).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace qadc {

// ------------------------------------------------------------------ helpers --

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() { // named barrier over the consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(16 * 32) : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier (SASS: UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

// ----------------------------------------------------------------- geometry --

// Compile-time geometry of a 64-bit-or-wider code: ROWS packed words of WW bits, each
// holding the group pattern Ws... LSB-first (layout.hpp:30-36).
template <int WW, int ROWS, int... Ws>
struct GeomCT {
    static constexpr bool RUNTIME = false;
    static constexpr int G = sizeof...(Ws);
    static constexpr int M = G * ROWS;
    static constexpr int WORD = WW;
    using Exact = GeomCT; // geometry of the [row][entry] table used by the exact re-evaluation
    static constexpr int CODE_BYTES = ROWS * WW / 8;
    static constexpr int STRIDE = (CODE_BYTES + 7) / 8 * 8;
    static constexpr int CW = STRIDE / 4; // 32-bit words per code
    __host__ __device__ static constexpr int width_at(int k) {
        const int ws[] = {Ws...};
        return ws[k];
    }
    __host__ __device__ static constexpr int bits(int j) { return width_at(j % G); }
    __host__ __device__ static constexpr int bitpos(int j) {
        int off = 0;
        for (int k = 0; k < j % G; ++k) off += width_at(k);
        return (j / G) * WW + off;
    }
    __host__ __device__ static constexpr int ent_off(int j) {
        int e = 0;
        for (int k = 0; k < j; ++k) e += 1 << bits(k);
        return e;
    }
    static constexpr int E = ent_off(M);
    static bool matches(const DevSpec& ds) {
        if (int(ds.m) != M || int(ds.word_width) != WW || int(ds.code_stride) != STRIDE) return false;
        for (int j = 0; j < M; ++j)
            if (ds.bits[j] != bits(j) || ds.bitpos[j] != bitpos(j)) return false;
        return true;
    }
};
struct GeomRT {
    static constexpr bool RUNTIME = true;
    static constexpr int CW = 2, E = 0, M = 0, STRIDE = 8;
    __host__ __device__ static constexpr int bits(int) { return 0; }
    __host__ __device__ static constexpr int bitpos(int) { return 0; }
    __host__ __device__ static constexpr int ent_off(int) { return 0; }
};

// --------------------------------------------------------- exact admission --

__device__ __forceinline__ uint32_t rt_sub_index(const DevSpec* ds, const uint8_t* code, uint32_t j) {
    const uint32_t bp = ds->bitpos[j];
    const uint32_t w = reinterpret_cast<const uint32_t*>(code)[bp >> 5];
    return (w >> (bp & 31u)) & ((1u << ds->bits[j]) - 1u);
}

// The CandidateHeap::push test (heap.hpp:40-51) for one (row, code): exact saturating
// sum (scan_scalar.hpp:52-58) from the reference-order table, then key < worst key.
__device__ __forceinline__ void exact_admit(const DevSpec* ds, const ScanArgs* a, const uint8_t* code, uint32_t row,
                                         uint32_t id) {
    uint32_t acc = a->row_bias ? min(a->row_bias[row], ds->qmax) : 0u;
    const size_t base = size_t(row) * ds->E;
    if (ds->word_width == 8) {
        const uint8_t* t = reinterpret_cast<const uint8_t*>(a->qlut) + base;
        for (uint32_t j = 0; j < ds->m; ++j) acc += t[ds->ent_off[j] + rt_sub_index(ds, code, j)];
    } else {
        const uint16_t* t = reinterpret_cast<const uint16_t*>(a->qlut) + base;
        for (uint32_t j = 0; j < ds->m; ++j) acc += t[ds->ent_off[j] + rt_sub_index(ds, code, j)];
    }
    acc = min(acc, ds->qmax); // == the chain of saturating adds, all terms being unsigned
    const uint32_t q = a->row_query ? a->row_query[row] : row;
    const uint64_t key = make_key(acc, id);
    if (key < a->thr_key[q]) {
        const uint32_t slot = atomicAdd(&a->cand_count[q], 1u);
        if (slot < a->cap) a->cand[size_t(q) * a->cap + slot] = key;
        else a->overflow[q] = 1u;
    }
}

// The same test with the spec's geometry known at compile time and the code in two registers: the m table
// reads are independent loads issued back to back (the runtime loop above consumes each one before issuing the
// next, i.e. m serialized L2 / HBM round trips per drain -- measured as ~25 % of the IVF scan).
template <class G>
__device__ __forceinline__ void exact_admit_ct(const DevSpec* ds, const ScanArgs* a, uint32_t w0, uint32_t w1,
                                               uint32_t row, uint32_t id) {
    const uint32_t q = a->row_query ? a->row_query[row] : row;
    const uint32_t bias = a->row_bias ? a->row_bias[row] : 0u;
    const uint64_t tk = a->thr_key[q];
    const size_t base = size_t(row) * G::E;
    uint32_t v[G::M];
    static_for<0, G::M>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int bp = G::bitpos(j), nb = G::bits(j);
        const uint32_t w = (bp >> 5) ? w1 : w0;
        const uint32_t idx = (w >> (bp & 31)) & ((1u << nb) - 1u);
        if constexpr (G::WORD == 8) v[j] = reinterpret_cast<const uint8_t*>(a->qlut)[base + G::ent_off(j) + idx];
        else v[j] = reinterpret_cast<const uint16_t*>(a->qlut)[base + G::ent_off(j) + idx];
    });
    uint32_t acc = min(bias, ds->qmax);
#pragma unroll
    for (int j = 0; j < G::M; ++j) acc += v[j];
    acc = min(acc, ds->qmax); // == the chain of saturating adds, all terms being unsigned
    const uint64_t key = make_key(acc, id);
    if (key < tk) {
        const uint32_t slot = atomicAdd(&a->cand_count[q], 1u);
        if (slot < a->cap) a->cand[size_t(q) * a->cap + slot] = key;
        else a->overflow[q] = 1u;
    }
}

} // namespace qadc
