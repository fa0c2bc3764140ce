// lut.cu -- per-query distance tables, calibration and quantization on the device.
//
// Exactness contract: the quantized tables must be
// bit-identical to the reference's, and the bin index floor((p - p_min)/delta) can flip on
// a 1-ulp difference, so every float feeding it reproduces the reference's operation
// order with explicitly rounded, never-contracted fp32 ops:
//   compute_tables   distance.hpp:47-55   d = q - c ; acc += d*d   (serial over the slice dims)
//   min_of/min_total distance.hpp:22-32   fp32 min; fp32 sum of minima in table order
//   prefix ADC       scan_scalar.hpp:110-117  fp32 sum in table order over the first t codes
//   calibrate_bounds distance.hpp:74-83   d_max = r-th smallest prefix value
//   quantize_tables  distance.hpp:102-142 delta in fp32; saturation test in fp32; bin in fp64
// The whole file is additionally compiled with --fmad=false.
//
// A dense query x centroid contraction on the tensor cores (|q|^2 - 2 q.c + |c|^2) cannot
// feed the quantizer (different rounding); the work is < 1 GFLOP per 10^4 queries, so
// it runs exactly on the CUDA cores, one CTA per query.
#include "common.cuh"

namespace qadc {

__device__ __forceinline__ uint32_t code_sub_index(const DevSpec& ds, const uint8_t* code, uint32_t j) {
    const uint32_t bp = ds.bitpos[j];
    const uint32_t byte = bp >> 3;
    uint32_t w, sh;
    if (ds.word_width == 16) {
        w = uint32_t(code[byte & ~1u]) | (uint32_t(code[(byte & ~1u) + 1]) << 8);
        sh = bp & 15u;
    } else {
        w = code[byte];
        sh = bp & 7u;
    }
    return (w >> sh) & ((1u << ds.bits[j]) - 1u);
}

// compute_tables (distance.hpp:35-58) for one (residual) query held in shared memory
__device__ void build_tables(const DevSpec& ds, const float* __restrict__ cb, const float* q, float* lut) {
    for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x) {
        uint32_t j = 0;
        while (j + 1 < ds.m && ds.ent_off[j + 1] <= e) ++j;
        const uint32_t i = e - ds.ent_off[j];
        const uint32_t dsub = ds.dim_alloc[j];
        const float* c = cb + ds.cb_off[j] + size_t(i) * dsub;
        const float* qq = q + ds.dim_off[j];
        float acc = 0.0f;
        for (uint32_t t = 0; t < dsub; ++t) {
            const float d = __fsub_rn(qq[t], c[t]);
            acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
        lut[e] = acc;
    }
}

// min_of per table (distance.hpp:22-26); one thread per table, sequential std::min order
__device__ void table_minima(const DevSpec& ds, const float* lut, float* pmin) {
    for (uint32_t j = threadIdx.x; j < ds.m; j += blockDim.x) {
        float mn = __int_as_float(0x7f800000);
        const float* t = lut + ds.ent_off[j];
        for (uint32_t i = 0; i < (1u << ds.bits[j]); ++i) mn = (t[i] < mn) ? t[i] : mn;
        pmin[j] = mn;
    }
}

// quantize_one (distance.hpp:117-124)
__device__ __forceinline__ uint32_t quantize_entry(float p, float pmin, float d_min, float d_max, float delta,
                                                   uint32_t qmax) {
    if (delta <= 0.0f) return p == pmin ? 0u : qmax;
    if (__fsub_rn(p, pmin) >= __fsub_rn(d_max, d_min)) return qmax;
    const double q = floor(__ddiv_rn(__dsub_rn(double(p), double(pmin)), double(delta)));
    if (q >= double(qmax)) return qmax;
    return uint32_t(q);
}

// r-th smallest (1-based) of vals[0..n): rank by counting, O(n^2 / threads).  Only the
// VALUE matters (nth_element semantics, distance.hpp:80-82), so ties are harmless.
__device__ float block_kth_smallest(const float* vals, uint32_t n, uint32_t r, float* result_slot) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float v = vals[i];
        uint32_t less = 0, leq = 0;
        for (uint32_t k = 0; k < n; ++k) {
            const float x = vals[k];
            less += x < v;
            leq += x <= v;
        }
        if (less <= r - 1 && r - 1 < leq) *result_slot = v;
    }
    __syncthreads();
    return *result_slot;
}

// FlatIndex::search up to (and including) quantize_tables, index.hpp:114-129.
// grid = nq, dynamic smem = (dims + E + m + t + 4) floats.
__global__ void flat_tables_kernel(DevSpec ds, LutArgs a) {
    extern __shared__ float sm[];
    float* q = sm;
    float* lut = q + ds.dims;
    float* pmin = lut + ds.E;
    float* prefix = pmin + ds.m;
    float* scal = prefix + a.t; // [0] d_min, [1] d_max
    const uint32_t qi = blockIdx.x;

    for (uint32_t d = threadIdx.x; d < ds.dims; d += blockDim.x) {
        float v = a.queries[size_t(qi) * ds.dims + d];
        if (a.sub) v = __fsub_rn(v, a.sub[size_t(qi) * ds.dims + d]);
        q[d] = v;
    }
    __syncthreads();
    build_tables(ds, a.codebook, q, lut);
    __syncthreads();
    table_minima(ds, lut, pmin);
    // collect_prefix_float (scan_scalar.hpp:96-122): first t codes in list order, table-order sum
    const uint32_t tp = min(a.t, a.calib_count);
    for (uint32_t i = threadIdx.x; i < tp; i += blockDim.x) {
        const uint8_t* code = a.calib_codes + size_t(i) * ds.code_stride;
        float acc = 0.0f;
        for (uint32_t j = 0; j < ds.m; ++j) acc = __fadd_rn(acc, lut[ds.ent_off[j] + code_sub_index(ds, code, j)]);
        prefix[i] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f; // min_total (distance.hpp:28-32)
        for (uint32_t j = 0; j < ds.m; ++j) s = __fadd_rn(s, pmin[j]);
        scal[0] = s;
    }
    const uint32_t r_eff = min(a.r, tp); // index.hpp:127
    const float d_max = block_kth_smallest(prefix, tp, r_eff, &scal[1]);
    const float d_min = scal[0];
    const float delta = __fdiv_rn(__fsub_rn(d_max, d_min), float(ds.qmax)); // distance.hpp:108
    if (threadIdx.x == 0) {
        if (!(d_max >= d_min)) atomicExch(a.status, QADC_ERR_CALIBRATION); // distance.hpp:104
        if (a.calib) {
            float* c = a.calib + size_t(qi) * 4;
            c[0] = d_min;
            c[1] = d_max;
            c[2] = delta;
            c[3] = d_min; // flat: qt.d_min == calibrated d_min (same sum, same order)
        }
        a.map[size_t(qi) * 2 + 0] = delta;
        a.map[size_t(qi) * 2 + 1] = d_min;
    }
    for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x) {
        uint32_t j = 0;
        while (j + 1 < ds.m && ds.ent_off[j + 1] <= e) ++j;
        const float p = lut[e];
        const uint32_t qv = quantize_entry(p, pmin[j], d_min, d_max, delta, ds.qmax);
        if (ds.word_width == 8) ((uint8_t*)a.qluts)[size_t(qi) * ds.E + e] = uint8_t(qv);
        else ((uint16_t*)a.qluts)[size_t(qi) * ds.E + e] = uint16_t(qv);
        if (a.luts) a.luts[size_t(qi) * ds.E + e] = p;
    }
}

void launch_flat_tables(const DevSpec& ds, const LutArgs& a, cudaStream_t stream) {
    if (a.nq == 0) return;
    const size_t smem = sizeof(float) * (size_t(ds.dims) + ds.E + ds.m + a.t + 4);
    if (smem > 200 * 1024) throw Error(QADC_ERR_CONFIG, "tables: dims + entries + t exceed shared memory");
    QADC_CUDA_CHECK(cudaFuncSetAttribute(flat_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    flat_tables_kernel<<<a.nq, 256, smem, stream>>>(ds, a);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
