// ivf_probe_tc.cu -- probe order (index.hpp:247-265) with a tensor-core prefilter.
//
// The reference computes K serial fp32 squared distances per query and keeps the first a by
// (distance, cell).  The exact path (ivf.cu) does the same work on the FP32 pipe: 3 instructions
// per (query, cell, dim), 1.7 ms per 10^4 queries x 16384 cells x 128 dims at best.  Only ~a of the
// K cells matter, so this path first bounds every distance cheaply and then evaluates the
// reference's exact arithmetic only where the bound cannot decide:
//
//   1. approx[q][c] = |c'|^2 - 2 <q', c'> on the tensor cores (bf16 inputs, fp32 accumulate), with
//      q' = q - mean, c' = c - mean (mean of the centroids; a translation leaves distances alone
//      and makes the rounding errors relative to the spread of the data, not its offset).
//   2. With D the real squared distance, D_ref the reference's fp32 value, A = approx + |q'|^2 and
//      S = (|q'| + |c'|)^2 (note |q'||c'| <= S / 4).  bf16 keeps 8 significand bits, so rounding to nearest has
//      unit roundoff u = 2^-8 per input:
//        |<q~,c~> - <q',c'>| <= (2u + u^2) |q'||c'|                  both inputs rounded, Cauchy-Schwarz
//        => the -2<.,.> term is off by <= (2^-6 + 2^-15) |q'||c'| <= (2^-8 + 2^-17) S
//        fp32 accumulation of <= 2048 exact products (truncation allowed): <= 2 * 2048 * 2^-23 |q'||c'| <= 2^-13 S
//        fp32 rounding of |c'|^2 and of the final subtraction:             <= 2^-22 S
//        |D_ref - D| <= (dims + 3) 2^-24 D <= 2^-13 S                      (serial fp32 sum, dims <= 2048)
//      Sum: |A - D_ref| <= 2^-8 (1 + 2^-4 + ...) S < 1.07 * 2^-8 S.  The filter uses
//      eps := 2^-7 (|q'| + max_c |c'|)^2, i.e. a factor ~1.88 above the bound.  (Round 1 used 2^-8 S, derived from
//      u = 2^-9 -- one bit too optimistic; corrected, with an adversarial test whose inputs sit just below bf16
//      rounding midpoints: tests/test_gpu_parity.py::test_probe_order_prefilter_bf16_midpoints.)
//   3. T := the a-th smallest of 256 strided minima of approx (a real value that at least a cells do not
//      exceed).  Those a cells have D_ref <= T + |q'|^2 + eps, hence so does the a-th smallest D_ref, and
//      every cell of the true top-a (ties included) has approx <= T + 2 eps.  Cells passing that test are
//      the candidates (typically 1.5-2 a of them).
//   4. Candidates get the reference's serial fp32 distance; the first a by (distance bits, cell) are the
//      probe order -- bit-identical to the exact path.  A query whose candidate set overflows (massive
//      ties, non-finite input) is flagged and redone by the exact kernels.
#include <cuda_bf16.h>

#include <cstring>

#include "common.cuh"

namespace qadc {

static constexpr uint32_t TC_CAND = 2048;

// ---------------------------------------------------------------- query preparation --

// One warp per query: q' = q - mean in double, bf16 image (zero padded to dpad), eps2 = 2 eps.
__global__ void probe_prep_queries_kernel(const float* __restrict__ queries, const double* __restrict__ mean,
                                          uint32_t dims, uint32_t dpad, uint32_t nq, double cmax,
                                          __nv_bfloat16* __restrict__ qb, double* __restrict__ eps2) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= nq) return;
    double s = 0.0;
    for (uint32_t j = lane; j < dpad; j += 32) {
        double v = 0.0;
        if (j < dims) v = double(queries[size_t(q) * dims + j]) - mean[j];
        qb[size_t(q) * dpad + j] = __float2bfloat16_rn(float(v));
        s += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        const double r = sqrt(s) * (1.0 + 1e-9) + cmax;
        eps2[q] = 2.0 * (r * r) * (1.0 / 128.0) * (1.0 + 1e-9); // 2 eps, eps = 2^-7 r^2; non-finite input -> inf/NaN -> flagged below
    }
}

// ---------------------------------------------------------------- approximate distances --

// C[q][c] = cn[c] - 2 * sum_k A[q][k] B[c][k];  A = queries (bf16, [nq][dpad]), B = centroids (bf16, [K][dpad]).
// 256 threads = 8 warps as 4 (rows) x 2 (cols); CTA tile 128 x 128, k chunks of 64 through shared memory;
// mma.sync.m16n8k16 bf16 -> fp32 (warp tile 32 x 64: 2 x 8 fragments).
static constexpr int GM = 128, GN = 128, GK = 64, GPITCH = GK + 8;

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
    const uint32_t addr = uint32_t(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(256)
probe_approx_gemm_kernel(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ B,
                         const float* __restrict__ cn, uint32_t nq, uint32_t k_cells, uint32_t dpad,
                         float* __restrict__ out) {
    __shared__ __align__(16) __nv_bfloat16 sa[GM * GPITCH];
    __shared__ __align__(16) __nv_bfloat16 sb[GN * GPITCH];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t wm = warp >> 1, wn = warp & 1;
    const uint32_t row0 = blockIdx.y * GM, col0 = blockIdx.x * GN;
    float acc[2][8][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[i][j][k] = 0.0f;
    for (uint32_t k0 = 0; k0 < dpad; k0 += GK) {
        // 128 rows x 64 bf16 = 128 x 8 uint4 per operand; 256 threads x 4 each
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t u = tid + it * 256, r = u >> 3, cseg = u & 7;
            uint4 va = make_uint4(0, 0, 0, 0), vb = make_uint4(0, 0, 0, 0);
            if (k0 + cseg * 8 < dpad) {
                if (row0 + r < nq) va = *reinterpret_cast<const uint4*>(A + size_t(row0 + r) * dpad + k0 + cseg * 8);
                if (col0 + r < k_cells) vb = *reinterpret_cast<const uint4*>(B + size_t(col0 + r) * dpad + k0 + cseg * 8);
            }
            *reinterpret_cast<uint4*>(sa + r * GPITCH + cseg * 8) = va;
            *reinterpret_cast<uint4*>(sb + r * GPITCH + cseg * 8) = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; kk += 16) {
            uint32_t af[2][4];
#pragma unroll
            for (int i = 0; i < 2; ++i) // A fragment: 16 x 16 at rows wm*32 + i*16
                ldmatrix_x4(af[i], sa + (wm * 32 + i * 16 + (lane & 15)) * GPITCH + kk + (lane >> 4) * 8);
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) { // two 8-column B fragments per ldmatrix.x4
                uint32_t bf[4];
                const uint32_t n = wn * 64 + jp * 16 + (lane & 7) + ((lane >> 4) << 3);
                ldmatrix_x4(bf, sb + n * GPITCH + kk + ((lane >> 3) & 1) * 8);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    mma_bf16(acc[i][2 * jp + 0], af[i], bf[0], bf[1]);
                    mma_bf16(acc[i][2 * jp + 1], af[i], bf[2], bf[3]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t c = col0 + wn * 64 + j * 8 + (lane & 3) * 2;
            const uint32_t r = row0 + wm * 32 + i * 16 + (lane >> 2);
            if (c < k_cells) { // K is even or the last column is dropped below
                const float n0 = cn[c], n1 = c + 1 < k_cells ? cn[c + 1] : 0.0f;
                if (r < nq) {
                    out[size_t(r) * k_cells + c] = n0 - 2.0f * acc[i][j][0];
                    if (c + 1 < k_cells) out[size_t(r) * k_cells + c + 1] = n1 - 2.0f * acc[i][j][1];
                }
                if (r + 8 < nq) {
                    out[size_t(r + 8) * k_cells + c] = n0 - 2.0f * acc[i][j][2];
                    if (c + 1 < k_cells) out[size_t(r + 8) * k_cells + c + 1] = n1 - 2.0f * acc[i][j][3];
                }
            }
        }
}

// ---------------------------------------------------------------- candidates -> exact order --

// One CTA (256 threads) per query.  dynamic smem: dims floats (the query).
__global__ void __launch_bounds__(256)
probe_select_tc_kernel(const float* __restrict__ approx, const double* __restrict__ eps2,
                       const float* __restrict__ queries, const float* __restrict__ coarse, uint32_t dims,
                       uint32_t k_cells, uint32_t a, uint32_t* __restrict__ order, uint32_t* __restrict__ redo) {
    extern __shared__ __align__(16) float qs[];
    __shared__ float mins[256];
    __shared__ uint64_t cand[TC_CAND];
    __shared__ uint32_t s_cnt;
    const uint32_t qi = blockIdx.x, tid = threadIdx.x;
    const float* d = approx + size_t(qi) * k_cells;
    for (uint32_t j = tid; j < dims; j += 256) qs[j] = queries[size_t(qi) * dims + j];
    float m = __int_as_float(0x7f800000);
    for (uint32_t c = tid; c < k_cells; c += 256) m = fminf(m, d[c]); // NaN never lowers a minimum
    mins[tid] = m;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (uint32_t size = 2; size <= 256; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            if (tid < 128) {
                const uint32_t lo = 2 * tid - (tid & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const float x = mins[lo], y = mins[hi];
                if ((x > y) == up) {
                    mins[lo] = y;
                    mins[hi] = x;
                }
            }
            __syncthreads();
        }
    // a <= min(256, K) guaranteed by the launcher; rounded UP to fp32 (a superset of candidates is always safe)
    const float limit = __double2float_ru(double(mins[a - 1]) + eps2[qi]);
    for (uint32_t base = 0; base < k_cells; base += 256) {
        const uint32_t c = base + tid;
        const bool take = c < k_cells && !(d[c] > limit); // NaN stays a candidate
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        if (bal) {
            uint32_t start = 0;
            if ((tid & 31) == 0) start = atomicAdd(&s_cnt, uint32_t(__popc(bal)));
            start = __shfl_sync(0xffffffffu, start, 0);
            const uint32_t slot = start + __popc(bal & ((1u << (tid & 31)) - 1u));
            if (take && slot < TC_CAND) cand[slot] = c;
        }
    }
    __syncthreads();
    const uint32_t n = s_cnt;
    if (n > TC_CAND || n < a) { // n < a only if the limit itself is NaN
        if (tid == 0) { // flags[nq] | compact list[nq] | count
            redo[qi] = 1u;
            redo[gridDim.x + atomicAdd(&redo[2 * size_t(gridDim.x)], 1u)] = qi;
        }
        return;
    }
    // the reference's distance (index.hpp:254-258): fp32, serial over the dims, unfused
    for (uint32_t i = tid; i < n; i += 256) {
        const uint32_t c = uint32_t(cand[i]);
        const float* ctr = coarse + size_t(c) * dims;
        float acc = 0.0f;
        if ((dims & 3u) == 0) {
            for (uint32_t j = 0; j < dims; j += 4) {
                const float4 v = *reinterpret_cast<const float4*>(ctr + j);
                float t;
                t = __fsub_rn(qs[j + 0], v.x); acc = __fadd_rn(acc, __fmul_rn(t, t));
                t = __fsub_rn(qs[j + 1], v.y); acc = __fadd_rn(acc, __fmul_rn(t, t));
                t = __fsub_rn(qs[j + 2], v.z); acc = __fadd_rn(acc, __fmul_rn(t, t));
                t = __fsub_rn(qs[j + 3], v.w); acc = __fadd_rn(acc, __fmul_rn(t, t));
            }
        } else {
            for (uint32_t j = 0; j < dims; ++j) {
                const float t = __fsub_rn(qs[j], ctr[j]);
                acc = __fadd_rn(acc, __fmul_rn(t, t));
            }
        }
        cand[i] = (uint64_t(__float_as_uint(acc)) << 32) | c;
    }
    uint32_t pow2 = 2;
    while (pow2 < n) pow2 <<= 1;
    for (uint32_t i = n + tid; i < pow2; i += 256) cand[i] = KEY_INF;
    __syncthreads();
    for (uint32_t size = 2; size <= pow2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < pow2 / 2; i += 256) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = cand[lo], y = cand[hi];
                if ((x > y) == up) {
                    cand[lo] = y;
                    cand[hi] = x;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = tid; i < a; i += 256) order[size_t(qi) * a + i] = uint32_t(cand[i]);
}

// ------------------------------------------------------------------------------ host --

bool ivf_probe_tc_supported(uint32_t dims, uint32_t k_cells, uint32_t a) {
    return a >= 1 && a <= 256 && k_cells >= 512 && a * 4 <= k_cells && dims <= 2048;
}

// d_coarse_bf16 [K][dpad], d_cnorm [K], d_mean [dims] come from ivf_probe_tc_prepare (host, at open).
void launch_ivf_probe_tc(const float* d_queries, const float* d_coarse, const uint16_t* d_coarse_bits,
                         const float* d_cnorm, const double* d_mean, double cmax, uint32_t dims, uint32_t dpad,
                         uint32_t k_cells, uint32_t nq, uint32_t a, uint16_t* d_q_bits, double* d_eps2,
                         float* d_approx, uint32_t* d_redo, uint32_t* d_order, cudaStream_t stream) {
    const __nv_bfloat16* d_coarse_bf16 = reinterpret_cast<const __nv_bfloat16*>(d_coarse_bits);
    __nv_bfloat16* d_qb = reinterpret_cast<__nv_bfloat16*>(d_q_bits);
    QADC_CUDA_CHECK(cudaMemsetAsync(d_redo, 0, (2 * size_t(nq) + 1) * 4, stream)); // flags | list | count
    probe_prep_queries_kernel<<<(nq * 32 + 255) / 256, 256, 0, stream>>>(d_queries, d_mean, dims, dpad, nq, cmax, d_qb,
                                                                        d_eps2);
    const dim3 grid((k_cells + GN - 1) / GN, (nq + GM - 1) / GM);
    probe_approx_gemm_kernel<<<grid, 256, 0, stream>>>(d_qb, d_coarse_bf16, d_cnorm, nq, k_cells, dpad, d_approx);
    probe_select_tc_kernel<<<nq, 256, size_t(dims) * 4, stream>>>(d_approx, d_eps2, d_queries, d_coarse, dims, k_cells, a,
                                                                 d_order, d_redo);
    g_launches += 3;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// Host side of the prefilter, once per index: mean of the centroids, centred bf16 image, |c'|^2, max |c'|.
// Returns false (prefilter off) when a centroid is not finite.
bool ivf_probe_tc_prepare(const float* coarse, uint32_t k_cells, uint32_t dims, uint32_t dpad,
                          std::vector<uint16_t>& bf16_out, std::vector<float>& cnorm, std::vector<double>& mean,
                          double& cmax) {
    mean.assign(dims, 0.0);
    for (uint32_t c = 0; c < k_cells; ++c)
        for (uint32_t j = 0; j < dims; ++j) mean[j] += double(coarse[size_t(c) * dims + j]);
    for (uint32_t j = 0; j < dims; ++j) {
        mean[j] /= double(std::max<uint32_t>(k_cells, 1));
        if (!(mean[j] - mean[j] == 0.0)) return false;
    }
    bf16_out.assign(size_t(k_cells) * dpad, 0);
    cnorm.assign(k_cells, 0.0f);
    cmax = 0.0;
    for (uint32_t c = 0; c < k_cells; ++c) {
        double s = 0.0;
        for (uint32_t j = 0; j < dims; ++j) {
            const double v = double(coarse[size_t(c) * dims + j]) - mean[j];
            s += v * v;
            const float f = float(v);
            uint32_t bits;
            std::memcpy(&bits, &f, 4);
            bits += 0x7FFFu + ((bits >> 16) & 1u); // round to nearest even (finite inputs)
            bf16_out[size_t(c) * dpad + j] = uint16_t(bits >> 16);
        }
        if (!(s - s == 0.0)) return false;
        cnorm[c] = float(s);
        cmax = std::max(cmax, std::sqrt(s));
    }
    cmax *= 1.0 + 1e-9;
    return true;
}

} // namespace qadc
