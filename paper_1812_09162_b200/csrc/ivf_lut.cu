// ivf_lut.cu -- the table stage of IvfIndex::search at batch scale (index.hpp:282-288, 319-328).
//
// A batch of nq queries x a probes is nq*a independent table sets (6.4e5 of them at C5), i.e. more
// bytes and flops than the probe-order stage.  Two kernels, both keeping the reference's fp32
// operation order per table entry (compute_tables, distance.hpp:35-58; quantize_tables, :102-142):
//
//   ivf_tables_tiled_kernel   thread = table entry, register-tiled over TAB_PT (query, cell) pairs:
//                             the entry's centroid lives in registers (loaded coalesced from the
//                             [sub][dim][entry] transposed codebook), the pairs' residuals sit in
//                             shared memory as [dim][pair] for 128-bit broadcast loads.
//   ivf_quantize_pack_kernel  one CTA per LUT tile: quantizes the tile's rows against their
//                             queries' shared bounds and writes BOTH images the scan uses -- the
//                             [row][entry] table (exact re-evaluation, seeding) and the transposed,
//                             variant-typed [entry][row] tile (tilepack.cu's layout) -- in one pass.
#include <cuda_fp16.h>

#include "common.cuh"

namespace qadc {

static constexpr int TAB_PT = 16;   // pairs per CTA batch
static constexpr int TAB_MAXD = 16; // widest subquantizer slice the register tile holds
static constexpr uint32_t NONE32 = 0xFFFFFFFFu;

__device__ __forceinline__ void fill_sub_of(const DevSpec& ds, uint8_t* sub_of) {
    for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x) {
        uint32_t j = 0;
        while (j + 1 < ds.m && ds.ent_off[j + 1] <= e) ++j;
        sub_of[e] = uint8_t(j);
    }
}

// dynamic smem: res[dims][TAB_PT] | pmin_u[TAB_PT][m] (u32 bit patterns).
// codebook_tp: [sub][TAB_MAXD][entries] zero padded (every entry has TAB_MAXD components at stride `entries`);
// sub_of: entry -> subquantizer (bytes).  Both are built once per index (api.cu).
__global__ void __launch_bounds__(256)
ivf_tables_tiled_kernel(DevSpec ds, const float* __restrict__ codebook_tp, const uint8_t* __restrict__ sub_of,
                        const float* __restrict__ queries, const float* __restrict__ coarse,
                        const uint32_t* __restrict__ order, uint32_t a, uint32_t n_pairs, float* __restrict__ luts,
                        float* __restrict__ pmin_out, float* __restrict__ own_min) {
    extern __shared__ __align__(16) float smf[];
    float* res = smf;
    uint32_t* pmin_u = reinterpret_cast<uint32_t*>(res + size_t(ds.dims) * TAB_PT);
    __shared__ uint32_t s_q[TAB_PT], s_cell[TAB_PT];
    const uint32_t pair0 = blockIdx.x * TAB_PT;
    const uint32_t np = min(uint32_t(TAB_PT), n_pairs - pair0);
    const uint32_t lane = threadIdx.x & 31;
    if (threadIdx.x < TAB_PT) {
        const uint32_t pair = pair0 + threadIdx.x;
        s_q[threadIdx.x] = threadIdx.x < np ? pair / a : 0;
        s_cell[threadIdx.x] = threadIdx.x < np ? order[pair] : 0;
    }
    for (uint32_t u = threadIdx.x; u < ds.m * TAB_PT; u += blockDim.x) pmin_u[u] = 0x7f800000u; // +inf
    __syncthreads();
    // residual = query - centroid (index.hpp:286), one fp32 subtraction per component
    if ((ds.dims & 3u) == 0 && ((reinterpret_cast<uintptr_t>(queries) | reinterpret_cast<uintptr_t>(coarse)) & 15u) == 0) {
        const uint32_t d4 = ds.dims >> 2;
        for (uint32_t u = threadIdx.x; u < d4 * TAB_PT; u += blockDim.x) {
            const uint32_t p = u / d4, j = (u - p * d4) * 4;
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p < np) {
                const float4 q = *reinterpret_cast<const float4*>(queries + size_t(s_q[p]) * ds.dims + j);
                const float4 c = *reinterpret_cast<const float4*>(coarse + size_t(s_cell[p]) * ds.dims + j);
                r = make_float4(__fsub_rn(q.x, c.x), __fsub_rn(q.y, c.y), __fsub_rn(q.z, c.z), __fsub_rn(q.w, c.w));
            }
            res[(j + 0) * TAB_PT + p] = r.x;
            res[(j + 1) * TAB_PT + p] = r.y;
            res[(j + 2) * TAB_PT + p] = r.z;
            res[(j + 3) * TAB_PT + p] = r.w;
        }
    } else {
        for (uint32_t p = 0; p < TAB_PT; ++p) {
            const float* q = queries + size_t(s_q[p]) * ds.dims;
            const float* c = coarse + size_t(s_cell[p]) * ds.dims;
            for (uint32_t d = threadIdx.x; d < ds.dims; d += blockDim.x)
                res[d * TAB_PT + p] = p < np ? __fsub_rn(q[d], c[d]) : 0.0f;
        }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x) {
        const uint32_t j = sub_of[e];
        const uint32_t dsub = ds.dim_alloc[j], nent = 1u << ds.bits[j];
        const float* ct = codebook_tp + size_t(ds.ent_off[j]) * TAB_MAXD + (e - ds.ent_off[j]);
        float c[TAB_MAXD];
#pragma unroll
        for (int t = 0; t < TAB_MAXD; ++t) c[t] = ct[uint32_t(t) * nent]; // zero padded past dsub
        float acc[TAB_PT];
#pragma unroll
        for (int p = 0; p < TAB_PT; ++p) acc[p] = 0.0f;
        const float4* rv = reinterpret_cast<const float4*>(res + size_t(ds.dim_off[j]) * TAB_PT);
#pragma unroll
        for (int t = 0; t < TAB_MAXD; ++t) {
            if (uint32_t(t) < dsub) {
#pragma unroll
                for (int v = 0; v < TAB_PT / 4; ++v) {
                    const float4 x = rv[t * (TAB_PT / 4) + v];
                    float d;
                    d = __fsub_rn(x.x, c[t]); acc[4 * v + 0] = __fadd_rn(acc[4 * v + 0], __fmul_rn(d, d));
                    d = __fsub_rn(x.y, c[t]); acc[4 * v + 1] = __fadd_rn(acc[4 * v + 1], __fmul_rn(d, d));
                    d = __fsub_rn(x.z, c[t]); acc[4 * v + 2] = __fadd_rn(acc[4 * v + 2], __fmul_rn(d, d));
                    d = __fsub_rn(x.w, c[t]); acc[4 * v + 3] = __fadd_rn(acc[4 * v + 3], __fmul_rn(d, d));
                }
            }
        }
        float* out = luts + size_t(pair0) * ds.E + e;
        if (np == TAB_PT) {
#pragma unroll
            for (int p = 0; p < TAB_PT; ++p) out[size_t(p) * ds.E] = acc[p];
        } else {
#pragma unroll
            for (int p = 0; p < TAB_PT; ++p)
                if (uint32_t(p) < np) out[size_t(p) * ds.E] = acc[p];
        }
        // per-table minima (min is order independent; entries are >= +0 or NaN, for which the unsigned order
        // of the bit patterns is the "x < best" rule started from +inf): REDUX over the lanes of this warp that
        // sit in the same table.  With >= TAB_PT such lanes, lane (first + p) keeps pair p's minimum and the
        // group issues ONE shared atomic; smaller groups fall back to one atomic per pair by the group leader.
        const uint32_t peers = __match_any_sync(__activemask(), j);
        const uint32_t first = __ffs(peers) - 1, gsize = __popc(peers);
        const bool wide_group = gsize >= uint32_t(TAB_PT);
        uint32_t keep = 0x7f800000u;
#pragma unroll
        for (int p = 0; p < TAB_PT; ++p) {
            const uint32_t mn = __reduce_min_sync(peers, __float_as_uint(acc[p]));
            if (wide_group) {
                if (lane == first + uint32_t(p)) keep = mn;
            } else if (lane == first) {
                atomicMin(&pmin_u[p * ds.m + j], mn);
            }
        }
        if (wide_group && lane - first < uint32_t(TAB_PT)) atomicMin(&pmin_u[(lane - first) * ds.m + j], keep);
    }
    __syncthreads();
    for (uint32_t u = threadIdx.x; u < np * ds.m; u += blockDim.x)
        pmin_out[size_t(pair0) * ds.m + u] = __uint_as_float(pmin_u[u]);
    if (threadIdx.x < np) { // table-order sum (DistanceTables::min_total, distance.hpp:28-32)
        float s = 0.0f;
        for (uint32_t j = 0; j < ds.m; ++j) s = __fadd_rn(s, __uint_as_float(pmin_u[threadIdx.x * ds.m + j]));
        own_min[pair0 + threadIdx.x] = s;
    }
}

bool ivf_tables_tiled_supported(const DevSpec& ds) {
    for (uint32_t j = 0; j < ds.m; ++j)
        if (ds.dim_alloc[j] > uint32_t(TAB_MAXD)) return false;
    const size_t smem = sizeof(float) * TAB_PT * (size_t(ds.dims) + ds.m);
    return smem <= 160 * 1024;
}

// host side, once per index: zero-padded transposed codebook [sub][TAB_MAXD][entries] and the entry -> sub map
void ivf_tables_tiled_prepare(const DevSpec& ds, const float* codebook, std::vector<float>& cb_tp,
                              std::vector<uint8_t>& sub_of) {
    cb_tp.assign(size_t(ds.E) * TAB_MAXD, 0.0f);
    sub_of.assign(ds.E, 0);
    for (uint32_t j = 0; j < ds.m; ++j) {
        const uint32_t nent = 1u << ds.bits[j], dsub = ds.dim_alloc[j];
        for (uint32_t i = 0; i < nent; ++i) {
            sub_of[ds.ent_off[j] + i] = uint8_t(j);
            for (uint32_t t = 0; t < dsub && t < uint32_t(TAB_MAXD); ++t)
                cb_tp[size_t(ds.ent_off[j]) * TAB_MAXD + size_t(t) * nent + i] = codebook[ds.cb_off[j] + size_t(i) * dsub + t];
        }
    }
}

void launch_ivf_tables_tiled(const DevSpec& ds, const float* d_codebook_tp, const uint8_t* d_sub_of,
                             const float* d_queries, const float* d_coarse, const uint32_t* d_order, uint32_t n_pairs,
                             uint32_t a, float* d_luts, float* d_pmin, float* d_own_min, cudaStream_t stream) {
    if (n_pairs == 0) return;
    const size_t smem = sizeof(float) * TAB_PT * (size_t(ds.dims) + ds.m);
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_tables_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ivf_tables_tiled_kernel<<<(n_pairs + TAB_PT - 1) / TAB_PT, 256, smem, stream>>>(
        ds, d_codebook_tp, d_sub_of, d_queries, d_coarse, d_order, a, n_pairs, d_luts, d_pmin, d_own_min);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------- slot <-> pair map --

__global__ void ivf_slot_map_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ pair_rank,
                                    const uint32_t* __restrict__ cell_tile_base, uint32_t tq, uint32_t n_pairs,
                                    uint32_t* __restrict__ pair_slot, uint32_t* __restrict__ slot_pair) {
    const uint32_t pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= n_pairs) return;
    const uint32_t rank = pair_rank[pair];
    if (rank == NONE32) { // empty list: skipped by the search loop (index.hpp:321)
        pair_slot[pair] = NONE32;
        return;
    }
    const uint32_t slot = cell_tile_base[order[pair]] * tq + rank;
    pair_slot[pair] = slot;
    slot_pair[slot] = pair;
}

// ------------------------------------------------------------ quantize + tile pack --

// quantize_tables' entry rule (distance.hpp:117-124): fp32 saturation test, then
// floor((double(p) - double(pmin)) / double(delta)).  The division is replaced by a multiplication with
// rcp = RN(1/delta) whenever that provably gives the same floor: with Q = RN(x/delta) and y = RN(x*rcp),
// |y - Q| <= 3*2^-53*Q < 2^-34 for Q < 2^17, so when y's fractional part is farther than 2^-30 from an
// integer floor(y) == floor(Q).  Anything else (near-integers, huge or non-finite values) takes the division.
__device__ __forceinline__ uint32_t quantize_entry_fast(float p, float pmin, float d_min, float d_max, float delta,
                                                        double rcp, uint32_t qmax) {
    if (delta <= 0.0f) return p == pmin ? 0u : qmax;
    if (__fsub_rn(p, pmin) >= __fsub_rn(d_max, d_min)) return qmax;
    if (p == pmin) return 0u; // every table's own minimum: x = 0 exactly
    const double x = __dsub_rn(double(p), double(pmin));
    const double y = __dmul_rn(x, rcp);
    if (y >= 0.0 && y < 131072.0) {
        const double k = floor(y);
        const double f = __dsub_rn(y, k); // exact
        if (f > 0x1p-30 && f < 1.0 - 0x1p-30) return k >= double(qmax) ? qmax : uint32_t(k);
    }
    const double q = floor(__ddiv_rn(x, double(delta)));
    if (q >= double(qmax)) return qmax;
    return uint32_t(q);
}

template <class Entry>
__device__ __forceinline__ Entry tile_entry(uint32_t v, uint32_t shift);
template <>
__device__ __forceinline__ __half tile_entry<__half>(uint32_t v, uint32_t shift) {
    return __uint2half_rn(v >> shift); // exact: <= 2047 whenever a half entry is used (ScanPlan::filter_shift)
}
template <>
__device__ __forceinline__ float tile_entry<float>(uint32_t v, uint32_t) { return float(v); }
template <>
__device__ __forceinline__ unsigned short tile_entry<unsigned short>(uint32_t v, uint32_t) { return (unsigned short)v; }
template <>
__device__ __forceinline__ unsigned char tile_entry<unsigned char>(uint32_t v, uint32_t shift) {
    return (unsigned char)(v >> shift);
}

static constexpr uint32_t QP_SLAB = 512; // entries per shared-memory panel

// eight consecutive rows of one entry line, converted to the variant's entry type, as vector stores
template <class Entry>
__device__ __forceinline__ void store_rows8(Entry* dst, const uint32_t (&v)[8], uint32_t shift);
template <>
__device__ __forceinline__ void store_rows8<__half>(__half* dst, const uint32_t (&v)[8], uint32_t shift) {
    __half2 h[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __halves2half2(tile_entry<__half>(v[2 * k], shift), tile_entry<__half>(v[2 * k + 1], shift));
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(h);
}
template <>
__device__ __forceinline__ void store_rows8<float>(float* dst, const uint32_t (&v)[8], uint32_t) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(float(v[0]), float(v[1]), float(v[2]), float(v[3]));
    reinterpret_cast<float4*>(dst)[1] = make_float4(float(v[4]), float(v[5]), float(v[6]), float(v[7]));
}
template <>
__device__ __forceinline__ void store_rows8<unsigned short>(unsigned short* dst, const uint32_t (&v)[8], uint32_t) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
}
template <>
__device__ __forceinline__ void store_rows8<unsigned char>(unsigned char* dst, const uint32_t (&v)[8], uint32_t shift) {
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k >> 2] |= ((v[k] >> shift) & 0xFFu) << (8 * (k & 3));
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
}

// grid = tiles; block = 256.  dynamic smem: panel u16 [min(E, QP_SLAB)][tq + 2] | sub_of[E].
// Phase 1, warp per row: a lane quantizes two adjacent entries at a time (float2 load, one 32-bit store into the
// [row][entry] table, two panel stores), four such pairs in flight.  Phase 2: a thread emits eight consecutive rows
// of one entry line as a 16-byte store (twice for the duplicated-line layout).  E is even and tq a multiple of 8.
template <class Entry>
__global__ void __launch_bounds__(256)
ivf_quantize_pack_kernel(DevSpec ds, const uint32_t* __restrict__ slot_pair, uint32_t a,
                         const float* __restrict__ luts, const float* __restrict__ pmin,
                         const float* __restrict__ own_min, const float* __restrict__ qparams, uint32_t tq,
                         uint32_t filter_shift, uint32_t copies, uint32_t pair_block, void* __restrict__ qluts,
                         Entry* __restrict__ tile_lut,
                         uint32_t* __restrict__ row_query, uint32_t* __restrict__ row_bias) {
    extern __shared__ __align__(16) unsigned short panel[];
    const uint32_t slab_cap = min(ds.E, QP_SLAB), pitch = tq + 2;
    uint8_t* sub_of = reinterpret_cast<uint8_t*>(panel + size_t(slab_cap) * pitch);
    fill_sub_of(ds, sub_of);
    __syncthreads();
    const uint32_t tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const bool wide = ds.word_width == 16;
    for (uint32_t e0 = 0; e0 < ds.E; e0 += slab_cap) {
        const uint32_t ne = min(slab_cap, ds.E - e0);
        for (uint32_t r = warp; r < tq; r += nwarps) {
            const uint32_t slot = tile * tq + r;
            const uint32_t pair = slot_pair[slot];
            uint16_t* q16 = reinterpret_cast<uint16_t*>(qluts) + size_t(slot) * ds.E + e0;
            uint8_t* q8 = reinterpret_cast<uint8_t*>(qluts) + size_t(slot) * ds.E + e0;
            if (pair == NONE32) { // padding row: zero table, no query
                for (uint32_t e = 2 * lane; e < ne; e += 64) {
                    panel[e * pitch + r] = 0;
                    panel[(e + 1) * pitch + r] = 0;
                    if (wide) *reinterpret_cast<uint32_t*>(q16 + e) = 0u;
                    else *reinterpret_cast<uint16_t*>(q8 + e) = 0;
                }
                if (e0 == 0 && lane == 0) {
                    row_query[slot] = NONE32;
                    row_bias[slot] = 0;
                }
                continue;
            }
            const uint32_t qi = pair / a;
            const float d_min = qparams[size_t(qi) * 4 + 0], d_max = qparams[size_t(qi) * 4 + 1];
            const float delta = qparams[size_t(qi) * 4 + 2];
            const double rcp = delta > 0.0f ? __drcp_rn(double(delta)) : 0.0;
            const float* lut = luts + size_t(pair) * ds.E + e0;
            const float* pm = pmin + size_t(pair) * ds.m;
            for (uint32_t eb = 2 * lane; eb < ne; eb += 256) {
                float2 pv[4];
                float pm0[4], pm1[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t e = eb + 64 * k;
                    if (e < ne) {
                        pv[k] = *reinterpret_cast<const float2*>(lut + e);
                        pm0[k] = pm[sub_of[e0 + e]];
                        pm1[k] = pm[sub_of[e0 + e + 1]];
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t e = eb + 64 * k;
                    if (e >= ne) break;
                    const uint32_t q0 = quantize_entry_fast(pv[k].x, pm0[k], d_min, d_max, delta, rcp, ds.qmax);
                    const uint32_t q1 = quantize_entry_fast(pv[k].y, pm1[k], d_min, d_max, delta, rcp, ds.qmax);
                    panel[e * pitch + r] = (unsigned short)q0;
                    panel[(e + 1) * pitch + r] = (unsigned short)q1;
                    if (wide) *reinterpret_cast<uint32_t*>(q16 + e) = q0 | (q1 << 16);
                    else *reinterpret_cast<uint16_t*>(q8 + e) = uint16_t(q0 | (q1 << 8));
                }
            }
            if (e0 == 0 && lane == 0) {
                uint32_t bias = 0;
                if (delta > 0.0f) { // float math, index.hpp:325-327
                    const float b = floorf(__fdiv_rn(__fsub_rn(own_min[pair], d_min), delta));
                    bias = b >= float(ds.qmax) ? ds.qmax : uint32_t(b);
                }
                row_query[slot] = qi;
                row_bias[slot] = bias;
            }
        }
        __syncthreads();
        // copies == 2: every entry line twice back to back (VAR_F16X4H_C4D)
        // pair: entry lines permuted into the pair-interleaved order (common.cuh: pair_perm)
        Entry* dst = tile_lut + size_t(tile) * ds.E * tq * copies;
        const uint32_t groups = tq >> 3, lg = 31 - __clz(groups); // 8-row groups per line (a power of two)
        for (uint32_t u = threadIdx.x; u < ne * groups; u += blockDim.x) {
            const uint32_t el = u >> lg, g = u & (groups - 1);
            const uint32_t* src = reinterpret_cast<const uint32_t*>(panel + el * pitch + g * 8); // 4-byte aligned: pitch even
            uint32_t v[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t w = src[k];
                v[2 * k] = w & 0xFFFFu;
                v[2 * k + 1] = w >> 16;
            }
            const uint32_t line = pair_block ? pair_perm(e0 + el, pair_block) : e0 + el;
            for (uint32_t c = 0; c < copies; ++c)
                store_rows8<Entry>(dst + (size_t(line) * copies + c) * tq + g * 8, v, filter_shift);
        }
        __syncthreads();
    }
}

template <class Entry>
static void launch_qp(const DevSpec& ds, const uint32_t* slot_pair, uint32_t a, const float* luts, const float* pmin,
                      const float* own_min, const float* qparams, uint32_t tq, uint32_t hb, void* qluts, void* tile_lut,
                      uint32_t* row_query, uint32_t* row_bias, uint32_t ntiles, cudaStream_t stream,
                      uint32_t copies = 1, uint32_t pair = 0) {
    const size_t smem = size_t(std::min(ds.E, QP_SLAB)) * (tq + 2) * sizeof(unsigned short) + ds.E;
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_quantize_pack_kernel<Entry>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ivf_quantize_pack_kernel<Entry><<<ntiles, 256, smem, stream>>>(ds, slot_pair, a, luts, pmin, own_min, qparams, tq, hb,
                                                                   copies, pair, qluts, static_cast<Entry*>(tile_lut),
                                                                   row_query, row_bias);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

void launch_ivf_quantize_pack(ScanVariant v, uint32_t filter_shift, uint32_t pair, const DevSpec& ds, const uint32_t* d_order, uint32_t n_pairs, uint32_t a,
                              const float* d_luts, const float* d_pmin, const float* d_own_min,
                              const float* d_qparams, const uint32_t* d_pair_rank, const uint32_t* d_cell_tile_base,
                              uint32_t tq, uint32_t ntiles, void* d_qluts, void* d_tile_lut, uint32_t* d_row_query,
                              uint32_t* d_row_bias, uint32_t* d_pair_slot, uint32_t* d_slot_pair,
                              cudaStream_t stream) {
    if (n_pairs == 0) return;
    if (ntiles) QADC_CUDA_CHECK(cudaMemsetAsync(d_slot_pair, 0xFF, size_t(ntiles) * tq * 4, stream));
    ivf_slot_map_kernel<<<(n_pairs + 255) / 256, 256, 0, stream>>>(d_order, d_pair_rank, d_cell_tile_base, tq, n_pairs,
                                                                   d_pair_slot, d_slot_pair);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
    if (ntiles == 0) return;
    if (tq < 8 || (tq & (tq - 1)) != 0 || (ds.E & 1u))
        throw Error(QADC_ERR_CONFIG, "quantize_pack: tile height must be a power of two >= 8 and E even");
    const uint32_t fs = ds.word_width == 16 ? filter_shift : 0u;
    switch (v) {
    case VAR_F16X8:
    case VAR_F16X4_C4:
        return launch_qp<__half>(ds, d_slot_pair, a, d_luts, d_pmin, d_own_min, d_qparams, tq, 0, d_qluts, d_tile_lut,
                                 d_row_query, d_row_bias, ntiles, stream, 1, pair);
    case VAR_F16X4H:
    case VAR_F16X4H_C2:
    case VAR_F16X4H_C4:
    case VAR_F16X4H_C16Q:
        return launch_qp<__half>(ds, d_slot_pair, a, d_luts, d_pmin, d_own_min, d_qparams, tq, fs, d_qluts, d_tile_lut,
                                 d_row_query, d_row_bias, ntiles, stream, 1, pair);
    case VAR_F16X4H_C4D:
        return launch_qp<__half>(ds, d_slot_pair, a, d_luts, d_pmin, d_own_min, d_qparams, tq, fs, d_qluts, d_tile_lut,
                                 d_row_query, d_row_bias, ntiles, stream, 2);
    case VAR_F32X2:
        return launch_qp<float>(ds, d_slot_pair, a, d_luts, d_pmin, d_own_min, d_qparams, tq, 0, d_qluts, d_tile_lut,
                                d_row_query, d_row_bias, ntiles, stream);
    case VAR_U16X1:
        return launch_qp<unsigned short>(ds, d_slot_pair, a, d_luts, d_pmin, d_own_min, d_qparams, tq, 0, d_qluts,
                                         d_tile_lut, d_row_query, d_row_bias, ntiles, stream);
    case VAR_U8X1:
        return launch_qp<unsigned char>(ds, d_slot_pair, a, d_luts, d_pmin, d_own_min, d_qparams, tq,
                                        ds.word_width == 16 ? 8u : 0u, d_qluts, d_tile_lut, d_row_query, d_row_bias,
                                        ntiles, stream);
    default: throw Error(QADC_ERR_CONFIG, "quantize_pack: bad variant");
    }
}

} // namespace qadc
