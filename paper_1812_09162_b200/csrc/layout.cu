// layout.cu -- code layout on the device.
//
// The reference stores a list as transposed blocks (layout.hpp:70-144): block b holds
// block_len codes; row r of the block holds the r-th packed word of each of them, rows
// contiguous.  That shape serves one CPU SIMD register per row.  On the GPU every
// warp consumes one WHOLE code at a time (all lanes share the code, each lane owns a
// few queries), so the device layout is the plain array of little-endian codes:
//
//     code i  ->  bytes [i*stride, i*stride + rows*word_bytes),  word r at byte r*word_bytes
//
// stride = rows*word_bytes rounded up to 8 (8 for every 64-bit spec).  Consecutive codes
// are contiguous, so a CTA stages a run of codes with one bulk async copy and a warp
// fetches a code with one broadcast 64/128-bit shared-memory load.  The map is a
// bijection on the occupied slots (tested against unpack_list, layout.hpp:162-176);
// padding slots are written as 0xFF like the reference's (layout.hpp:117).
#include "common.cuh"

namespace qadc {

thread_local unsigned long long g_launches = 0;

__global__ void relayout_kernel(const uint8_t* __restrict__ packed, uint64_t n, uint64_t n_padded, uint32_t rows,
                                uint32_t wb, uint32_t block_len, uint32_t stride, uint8_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n_padded) return;
    uint8_t* dst = out + i * stride;
    if (i >= n) {
        for (uint32_t b = 0; b < stride; ++b) dst[b] = 0xFF;
        return;
    }
    const uint64_t bb = uint64_t(rows) * block_len * wb;
    const uint8_t* blk = packed + (i / block_len) * bb;
    const uint32_t p = uint32_t(i % block_len);
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t b = 0; b < wb; ++b) dst[r * wb + b] = blk[(uint64_t(r) * block_len + p) * wb + b];
    for (uint32_t b = rows * wb; b < stride; ++b) dst[b] = 0xFF;
}

void launch_relayout(const qadc_spec& s, const DevSpec& ds, const uint8_t* d_packed, uint64_t n, uint64_t n_padded,
                     uint8_t* d_codes, cudaStream_t stream) {
    if (n_padded == 0) return;
    const uint32_t rows = ds.code_bytes / (s.word_width / 8);
    const uint64_t blocks = (n_padded + 255) / 256;
    relayout_kernel<<<unsigned(blocks), 256, 0, stream>>>(d_packed, n, n_padded, rows, s.word_width / 8, s.block_len,
                                                          ds.code_stride, d_codes);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

__device__ __forceinline__ uint32_t sub_index(const DevSpec& ds, const uint8_t* code, uint32_t j) {
    const uint32_t bp = ds.bitpos[j];
    const uint32_t byte = bp >> 3;
    uint32_t w = code[byte];
    if (ds.word_width == 16) w = uint32_t(code[byte & ~1u]) | (uint32_t(code[(byte & ~1u) + 1]) << 8);
    const uint32_t sh = ds.word_width == 16 ? (bp & 15u) : (bp & 7u);
    return (w >> sh) & ((1u << ds.bits[j]) - 1u);
}

__global__ void unlayout_kernel(DevSpec ds, const uint8_t* __restrict__ codes, uint64_t first, uint64_t n,
                                uint8_t* __restrict__ sub) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint8_t* code = codes + (first + i) * ds.code_stride;
    for (uint32_t j = 0; j < ds.m; ++j) sub[i * ds.m + j] = uint8_t(sub_index(ds, code, j));
}

void launch_unlayout(const DevSpec& ds, const uint8_t* d_codes, uint64_t first, uint64_t n, uint8_t* d_subcodes,
                     cudaStream_t stream) {
    if (n == 0) return;
    unlayout_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(ds, d_codes, first, n, d_subcodes);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// adc_scalar_quantized (distance.hpp:149-155) for a code range: one thread per code.
// Debug / parity entry point, not the hot path.
__global__ void adc_sums_kernel(DevSpec ds, const uint8_t* __restrict__ codes, const void* __restrict__ qlut,
                                uint32_t acc_init, uint64_t first, uint64_t n, uint32_t* __restrict__ sums) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint8_t* code = codes + (first + i) * ds.code_stride;
    uint32_t acc = min(acc_init, ds.qmax);
    for (uint32_t j = 0; j < ds.m; ++j) {
        const uint32_t e = ds.ent_off[j] + sub_index(ds, code, j);
        const uint32_t v = ds.word_width == 8 ? uint32_t(((const uint8_t*)qlut)[e]) : uint32_t(((const uint16_t*)qlut)[e]);
        acc = min(acc + v, ds.qmax);
    }
    sums[i] = acc;
}

void launch_adc_sums(const DevSpec& ds, const uint8_t* d_codes, const void* d_qlut, uint32_t acc_init,
                     uint64_t first, uint64_t n, uint32_t* d_sums, cudaStream_t stream) {
    if (n == 0) return;
    adc_sums_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(ds, d_codes, d_qlut, acc_init, first, n, d_sums);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// encode (codebook.hpp:94-118): per slice the nearest centroid under a DOUBLE accumulator,
// serial over the slice dims, ties toward the lowest index.  One warp per vector; lanes
// stride over centroids, then a (distance, index) lexicographic warp reduction, which
// reproduces the sequential "acc < best" rule exactly.
__global__ void encode_kernel(DevSpec ds, const float* __restrict__ cb, const float* __restrict__ vec, uint64_t n,
                              uint8_t* __restrict__ codes) {
    const uint64_t v = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (v >= n) return;
    const float* x = vec + v * ds.dims;
    for (uint32_t j = 0; j < ds.m; ++j) {
        const uint32_t dsub = ds.dim_alloc[j];
        const float* q = x + ds.dim_off[j];
        const float* tab = cb + ds.cb_off[j];
        double best = __longlong_as_double(0x7ff0000000000000ll);
        uint32_t best_i = 0;
        for (uint32_t i = lane; i < (1u << ds.bits[j]); i += 32) {
            const float* c = tab + size_t(i) * dsub;
            double acc = 0.0;
            for (uint32_t t = 0; t < dsub; ++t) {
                const double diff = __dsub_rn(double(q[t]), double(c[t]));
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
            if (acc < best) {
                best = acc;
                best_i = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            if (ob < best || (ob == best && oi < best_i)) {
                best = ob;
                best_i = oi;
            }
        }
        if (lane == 0) codes[v * ds.m + j] = uint8_t(best_i);
    }
}

void launch_encode(const DevSpec& ds, const float* d_codebook, const float* d_vectors, uint64_t n, uint8_t* d_codes,
                   cudaStream_t stream) {
    if (n == 0) return;
    const uint64_t threads = n * 32;
    encode_kernel<<<unsigned((threads + 255) / 256), 256, 0, stream>>>(ds, d_codebook, d_vectors, n, d_codes);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
