// tilepack.cu -- quantized tables in the scan kernel's shared-memory layout.
//
// quantize_tables (lut.cu) emits the reference layout [row][entry] at table width.  The scan
// kernel wants, per tile of TQ rows, the transposed image [entry][row] already converted to the
// variant's entry type (fp16 / fp32 / u16 / u8), so that loading a tile is a handful of bulk
// async copies (TMA, UBLKCP) instead of a strided gather.  One CTA transposes a
// (64 entries x TQ rows) panel through shared memory: reads are contiguous along the entry
// axis, writes along the row axis.
#include <cuda_fp16.h>

#include "common.cuh"

namespace qadc {

template <class Entry>
__device__ __forceinline__ Entry tile_convert(uint32_t v, uint32_t width, uint32_t shift);
template <>
__device__ __forceinline__ __half tile_convert<__half>(uint32_t v, uint32_t width, uint32_t shift) {
    return __uint2half_rn(width == 16 ? v >> shift : v); // exact: value <= 2047 whenever a half entry is used
}
template <>
__device__ __forceinline__ float tile_convert<float>(uint32_t v, uint32_t, uint32_t) { return float(v); }
template <>
__device__ __forceinline__ unsigned short tile_convert<unsigned short>(uint32_t v, uint32_t, uint32_t) {
    return (unsigned short)v;
}
template <>
__device__ __forceinline__ unsigned char tile_convert<unsigned char>(uint32_t v, uint32_t width, uint32_t) {
    return (unsigned char)(width == 16 ? v >> 8 : v);
}

static constexpr int PACK_E = 64;

// grid = (ntiles, ceil(E / PACK_E)); block = 256.  rows [tile*TQ, tile*TQ + TQ) clipped to n_rows.
template <class Entry>
__global__ void pack_tiles_kernel(const void* __restrict__ qlut, uint32_t width, uint32_t E, uint32_t n_rows,
                                  uint32_t tq, uint32_t high_byte /* filter shift */, uint32_t copies, uint32_t pair,
                                  Entry* __restrict__ out) {
    extern __shared__ unsigned short panel[]; // [PACK_E][tq + 1]
    const uint32_t tile = blockIdx.x, e0 = blockIdx.y * PACK_E;
    const uint32_t ne = min(uint32_t(PACK_E), E - e0);
    const uint32_t pitch = tq + 1;
    for (uint32_t u = threadIdx.x; u < tq * PACK_E; u += blockDim.x) {
        const uint32_t el = u % PACK_E, r = u / PACK_E;
        const uint32_t row = tile * tq + r;
        uint32_t v = 0;
        if (el < ne && row < n_rows) {
            const size_t gi = size_t(row) * E + e0 + el;
            v = width == 8 ? uint32_t(reinterpret_cast<const uint8_t*>(qlut)[gi])
                           : uint32_t(reinterpret_cast<const uint16_t*>(qlut)[gi]);
        }
        panel[el * pitch + r] = (unsigned short)v;
    }
    __syncthreads();
    // copies == 2: every entry line twice back to back (VAR_F16X4H_C4D)
    // pair: entry lines permuted into the pair-interleaved order (common.cuh: pair_perm)
    Entry* dst = out + size_t(tile) * E * tq * copies;
    for (uint32_t u = threadIdx.x; u < ne * tq; u += blockDim.x) {
        const uint32_t r = u % tq, el = u / tq;
        const Entry v = tile_convert<Entry>(panel[el * pitch + r], width, high_byte);
        const uint32_t line = pair ? pair_perm(e0 + el, pair) : e0 + el;
        for (uint32_t c = 0; c < copies; ++c) dst[(size_t(line) * copies + c) * tq + r] = v;
    }
}

template <class Entry>
static void launch_pack(const void* qlut, uint32_t width, uint32_t E, uint32_t n_rows, uint32_t tq, uint32_t hb,
                        void* out, cudaStream_t stream, uint32_t copies = 1, uint32_t pair = 0) {
    const uint32_t ntiles = (n_rows + tq - 1) / tq;
    if (ntiles == 0) return;
    const dim3 grid(ntiles, (E + PACK_E - 1) / PACK_E);
    const size_t smem = size_t(PACK_E) * (tq + 1) * sizeof(unsigned short);
    pack_tiles_kernel<Entry><<<grid, 256, smem, stream>>>(qlut, width, E, n_rows, tq, hb, copies, pair, static_cast<Entry*>(out));
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// 16x{4,4} merged into 8 byte-indexed tables: entry (j, b) = T[2j][b & 15] + T[2j+1][b >> 4] (VAR_F16X4_C4M).
// grid = (ntiles, 2048 / 64); block = 256; rows [tile*TQ, tile*TQ + TQ) clipped to n_rows; qlut is [row][256] u8.
__global__ void pack_tiles_merged44_kernel(const uint8_t* __restrict__ qlut, uint32_t n_rows, uint32_t tq, uint32_t pair,
                                           __half* __restrict__ out) {
    const uint32_t tile = blockIdx.x, e0 = blockIdx.y * 64;
    __half* base = out + size_t(tile) * 2048 * tq;
    for (uint32_t u = threadIdx.x; u < 64 * tq; u += blockDim.x) {
        const uint32_t r = u % tq, e = e0 + u / tq;
        const uint32_t row = tile * tq + r, j = e >> 8, b = e & 255u;
        uint32_t v = 0;
        if (row < n_rows) {
            const uint8_t* t = qlut + size_t(row) * 256 + 32 * j;
            v = uint32_t(t[b & 15u]) + uint32_t(t[16 + (b >> 4)]);
        }
        base[size_t(pair ? pair_perm(e, pair) : e) * tq + r] = __uint2half_rn(v);
    }
}

uint32_t tile_pair_layout(ScanVariant v, const DevSpec& ds) {
    if (v == VAR_F16X4_C4M) return 256; // the merged view is 8 tables of 256 entries
    if (v != VAR_F16X4H_C4 && v != VAR_F16X4_C4 && v != VAR_F16X4H_C16Q) return 0;
    if (ds.m == 0 || ds.code_stride != 8) return 0;
    bool bytes = ds.m == 8 && ds.E == 2048;
    for (uint32_t j = 0; j < ds.m && bytes; ++j) bytes = ds.bits[j] == 8 && ds.bitpos[j] == 8 * j;
    if (bytes) return 256; // G8 / G88
    // G655 / G664 / G555 on the conservative 32-row variant: four 16-bit words with identical tables
    if ((v == VAR_F16X4H_C4 || v == VAR_F16X4H_C16Q) && ds.word_width == 16 && ds.m == 12 && ds.E % 4 == 0) {
        for (uint32_t j = 0; j < 12; ++j) {
            if (ds.bits[j] != ds.bits[j % 3]) return 0;
            if (ds.bitpos[j] != 16 * (j / 3) + (j % 3 == 0 ? 0 : j % 3 == 1 ? ds.bits[0] : ds.bits[0] + ds.bits[1])) return 0;
        }
        const uint32_t b[3] = {ds.bits[0], ds.bits[1], ds.bits[2]};
        const bool named = (b[0] == 6 && b[1] == 5 && b[2] == 5) || (b[0] == 6 && b[1] == 6 && b[2] == 4) ||
                           (b[0] == 5 && b[1] == 5 && b[2] == 5);
        if (!named) return 0; // the compile-time geometries that implement it
        return v == VAR_F16X4H_C16Q ? (ds.E / 4) | TILE_QUAD : ds.E / 4;
    }
    return 0;
}

// 12x{6,5,5} merged for VAR_F16X4H_C8Q: per tile of 16 rows, 1024 + 64 lines of 128 bytes; line i of the first
// section holds, for each word t = 0..3 (32 bytes = 16 rows each), (T[3t+1][i & 31] >> s) + (T[3t+2][i >> 5] >> s);
// line i of the second section holds T[3t][i] >> s.  qlut is [row][512] u16; s = the plan's filter shift (6).
// b0 / b1 = bits of a word's first / middle subcode ({6,5,5}: 6, 5; {6,6,4}: 6, 6; {5,5,5}: 5, 5); the word's tables
// hold 2^b0, 2^b1 and 2^(10-b1) entries and the tile 1024 + 2^b0 quad lines.
__global__ void pack_tiles_merged655_kernel(const uint16_t* __restrict__ qlut, uint32_t n_rows, uint32_t shift,
                                            uint32_t b0, uint32_t b1, uint32_t E, __half* __restrict__ out) {
    const uint32_t tile = blockIdx.x, lines = 1024u + (1u << b0);
    __half* base = out + size_t(tile) * lines * 64;
    for (uint32_t u = blockIdx.y * blockDim.x + threadIdx.x; u < lines * 64u; u += gridDim.y * blockDim.x) {
        const uint32_t line = u >> 6, t = (u >> 4) & 3u, r = u & 15u;
        const uint32_t row = tile * 16 + r;
        uint32_t v = 0;
        if (row < n_rows) {
            const uint16_t* q = qlut + size_t(row) * E + t * (E / 4);
            const uint32_t n0 = 1u << b0, n1 = 1u << b1;
            v = line < 1024 ? (uint32_t(q[n0 + (line & (n1 - 1u))]) >> shift) + (uint32_t(q[n0 + n1 + (line >> b1)]) >> shift)
                            : uint32_t(q[line - 1024]) >> shift;
        }
        base[u] = __uint2half_rn(v);
    }
}

uint32_t tile_entries(ScanVariant v, uint32_t E) {
    return v == VAR_F16X4_C4M ? 2048u : v == VAR_F16X4H_C8Q ? (E == 384 ? 1056u : 1088u) : E;
}

size_t tile_entry_bytes(ScanVariant v) {
    switch (v) {
    case VAR_F16X4H_C8Q: return 8; // a quad line: four tables x 2 bytes per row
    case VAR_F16X4_C4M:
    case VAR_F16X8:
    case VAR_F16X4H:
    case VAR_F16X4H_C2:
    case VAR_F16X4H_C4:
    case VAR_F16X4H_C16Q:
    case VAR_F16X4_C4: return 2;
    case VAR_F16X4H_C4D: return 4; // two copies of a 2-byte entry
    case VAR_F32X2: return 4;
    case VAR_U16X1: return 2;
    case VAR_U8X1: return 1;
    case VAR_TC8:
    case VAR_TC8S:
    case VAR_TC8P: return 1; // signed bytes e - 128, K-major operand image
    default: return 4;
    }
}

void launch_pack_tiles(ScanVariant v, uint32_t filter_shift, uint32_t pair, const void* qlut, uint32_t width, uint32_t E,
                       uint32_t n_rows, uint32_t tq, void* out, cudaStream_t stream) {
    switch (v) {
    case VAR_TC8:
    case VAR_TC8S:
    case VAR_TC8P:
        if (width != 8 || E != 256 || tq != scan_tc8_tile_rows(tc8_mode(v)))
            throw Error(QADC_ERR_CONFIG, "pack_tiles: the tensor-core layout is for 16x{4,4}");
        launch_pack_tiles_tc8(qlut, n_rows, scan_tc8_pack_rows(tc8_mode(v)), tq / scan_tc8_pack_rows(tc8_mode(v)), out, stream);
        return;
    case VAR_F16X4H_C8Q: {
        if (width != 16 || (E != 512 && E != 576 && E != 384) || tq != 16)
            throw Error(QADC_ERR_CONFIG, "pack_tiles: quad layout is for 12x{6,5,5} / 12x{6,6,4} / 12x{5,5,5}");
        const uint32_t ntiles = (n_rows + tq - 1) / tq;
        if (ntiles == 0) return;
        pack_tiles_merged655_kernel<<<dim3(ntiles, 17), 256, 0, stream>>>(static_cast<const uint16_t*>(qlut), n_rows,
                                                                       filter_shift, E == 384 ? 5u : 6u,
                                                                       E == 576 ? 6u : 5u, E, static_cast<__half*>(out));
        ++g_launches;
        QADC_CUDA_CHECK(cudaGetLastError());
        return;
    }
    case VAR_F16X4_C4M: {
        if (width != 8 || E != 256) throw Error(QADC_ERR_CONFIG, "pack_tiles: merged layout is for 16x{4,4}");
        const uint32_t ntiles = (n_rows + tq - 1) / tq;
        if (ntiles == 0) return;
        pack_tiles_merged44_kernel<<<dim3(ntiles, 2048 / 64), 256, 0, stream>>>(static_cast<const uint8_t*>(qlut), n_rows, tq,
                                                                             pair, static_cast<__half*>(out));
        ++g_launches;
        QADC_CUDA_CHECK(cudaGetLastError());
        return;
    }
    case VAR_F16X8:
    case VAR_F16X4_C4: return launch_pack<__half>(qlut, width, E, n_rows, tq, 0, out, stream, 1, pair);
    case VAR_F16X4H:
    case VAR_F16X4H_C2:
    case VAR_F16X4H_C4:
    case VAR_F16X4H_C16Q:
        return launch_pack<__half>(qlut, width, E, n_rows, tq, filter_shift, out, stream, 1, pair);
    case VAR_F16X4H_C4D: return launch_pack<__half>(qlut, width, E, n_rows, tq, filter_shift, out, stream, 2);
    case VAR_F32X2: return launch_pack<float>(qlut, width, E, n_rows, tq, 0, out, stream);
    case VAR_U16X1: return launch_pack<unsigned short>(qlut, width, E, n_rows, tq, 0, out, stream);
    case VAR_U8X1: return launch_pack<unsigned char>(qlut, width, E, n_rows, tq, 8, out, stream);
    default: throw Error(QADC_ERR_CONFIG, "pack_tiles: bad variant");
    }
}

} // namespace qadc
