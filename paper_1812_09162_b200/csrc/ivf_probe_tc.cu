// ivf_probe_tc.cu -- probe order (index.hpp:247-265) with a tensor-core prefilter.
//
// The reference computes K serial fp32 squared distances per query and keeps the first a by
// (distance, cell).  The exact path (ivf.cu) does the same work on the FP32 pipe: 3 instructions
// per (query, cell, dim), 1.7 ms per 10^4 queries x 16384 cells x 128 dims at best.  Only ~a of the
// K cells matter, so this path first bounds every distance cheaply and then evaluates the
// reference's exact arithmetic only where the bound cannot decide:
//
//   1. approx[q][c] = |c'|^2 - 2 <q', c'> on the 5th-generation tensor cores (tcgen05.mma kind::f16: bf16 inputs, fp32
//      accumulators in tensor memory; operands arrive as pre-tiled images through TMA bulk copies), with
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
//   3. The approximate values are never stored: the contraction runs TWICE (it is ~20 us of tensor-core time; a
//      [queries][cells] fp32 image would be 655 MB written and read twice at C5).  Pass 1's epilogue keeps, per query,
//      the minimum of every residue class c mod 256; T := the a-th smallest of those 256 minima (a real value that at
//      least a cells do not exceed).  Those a cells have D_ref <= T + |q'|^2 + eps, hence so does the a-th smallest D_ref, and
//      every cell of the true top-a (ties included) has approx <= T + 2 eps.  Pass 2's epilogue recomputes the same
//      values (bit-identical: same instructions, same data) and appends the cells passing that test to the query's
//      candidate list (typically 1.5-2 a of them).
//   4. Candidates get the reference's serial fp32 distance; the first a by (distance bits, cell) are the
//      probe order -- bit-identical to the exact path.  A query whose candidate set overflows (massive
//      ties, non-finite input) is flagged and redone by the exact kernels.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace qadc {

static constexpr uint32_t TC_CAND = 2048;

// ---------------------------------------------------------------- query preparation --

// Operand images.  The MMA reads its operands from shared memory in the K-major no-swizzle canonical layout (core
// matrices of 8 rows x 16 bytes); both operands are stored in GLOBAL memory already in that order, cut into slabs of
// 128 K-elements, so that a tile slab is one contiguous block a single bulk copy brings in:
//   image[tile][slab][kc = 16][row][8 elements],  rows = 128 (queries, A) or 256 (centroids, B), zero padded.
static constexpr uint32_t PT_M = 128, PT_N = 256, PT_KS = 128; // tile rows (queries), tile columns (cells), K per slab
__host__ __device__ inline size_t probe_image_index(uint32_t row, uint32_t k, uint32_t rows_per_tile, uint32_t nslab) {
    const uint32_t tile = row / rows_per_tile, r = row % rows_per_tile, slab = k / PT_KS, kc = (k % PT_KS) / 8, e = k % 8;
    return ((((size_t(tile) * nslab + slab) * 16 + kc) * rows_per_tile + r) * 8) + e;
}

// One warp per query row of the padded batch: q' = q - mean in double, bf16 image (zero padded), eps2 = 2 eps.
__global__ void probe_prep_queries_kernel(const float* __restrict__ queries, const double* __restrict__ mean,
                                          uint32_t dims, uint32_t dpad, uint32_t nq, uint32_t nq_pad, double cmax,
                                          __nv_bfloat16* __restrict__ qb, double* __restrict__ eps2) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= nq_pad) return;
    const uint32_t nslab = (dpad + PT_KS - 1) / PT_KS;
    double s = 0.0;
    for (uint32_t j = lane; j < nslab * PT_KS; j += 32) {
        double v = 0.0;
        if (j < dims && q < nq) v = double(queries[size_t(q) * dims + j]) - mean[j];
        qb[probe_image_index(q, j, PT_M, nslab)] = __float2bfloat16_rn(float(v));
        s += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && q < nq) {
        const double r = sqrt(s) * (1.0 + 1e-9) + cmax;
        eps2[q] = 2.0 * (r * r) * (1.0 / 128.0) * (1.0 + 1e-9); // 2 eps, eps = 2^-7 r^2; non-finite input -> inf/NaN -> flagged below
    }
}

// ---------------------------------------------------------------- approximate distances --

// out[q][c] = cn[c] - 2 * sum_k A[q][k] B[c][k] on tcgen05: CTA tile 128 queries x 256 cells, K in slabs of 128.
//   warp 0   producer: one bulk copy per operand slab (A 32 KB, B 64 KB) into a 2-stage ring (UBLKCP + mbarrier)
//   warp 1   MMA issuer (one elected lane): 8 x tcgen05.mma kind::f16 (M 128, N 256, K 16) per slab into one of two
//            256-column fp32 accumulators in tensor memory; tcgen05.commit frees the stage / publishes the tile
//   warps 2-9 epilogue (two per TMEM lane quadrant, 128 cells each): tcgen05.ld (thread = query row, 32 cells at a time),
//            cn[c] - 2 acc, eight 16-byte stores = the row's 128 contiguous bytes (a shared-memory transpose so that a
//            whole warp store is one row measured 1.4x slower than the mma.sync kernel it replaced: too few stores in flight)
// Work items are (query tile, group of 16 cell tiles), walked persistently by gridDim.x CTAs.
static constexpr uint32_t PT_THREADS = 320, PT_A_BYTES = 16 * PT_M * 16, PT_B_BYTES = 16 * PT_N * 16, PT_NGROUP = 16;
static constexpr uint32_t PT_SMEM = 2 * (PT_A_BYTES + PT_B_BYTES);

__device__ __forceinline__ uint32_t pt_smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void pt_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(pt_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void pt_mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(pt_smem_u32(bar)), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ uint64_t pt_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) { // K-major, no swizzle, version 1
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) | (uint64_t((sbo >> 4) & 0x3FFFu) << 32) |
           (uint64_t(1) << 46);
}
// instruction descriptor: fp32 accumulate (1 << 4), A = B = bf16 (1 << 7, 1 << 10), K-major, N >> 3 at bit 17, M >> 4 at bit 24
static constexpr uint32_t PT_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((PT_N >> 3) << 17) | ((PT_M >> 4) << 24);

// monotone map float -> uint32 (unsigned order == float order; used for atomicMin on floats of either sign)
__device__ __forceinline__ uint32_t pt_ordered(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float pt_unordered(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// PASS 1: mins_u[q][c mod 256] = min over cells of approx (ordered-uint encoding, atomicMin across work items).
// PASS 2: cand[q][w] = bitmap of the cells 32 w .. 32 w + 31 with !(approx > limit[q])  (ntiles * 8 words per query).
template <int PASS>
__global__ void __launch_bounds__(PT_THREADS, 1)
probe_approx_umma_kernel(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ B,
                         const float* __restrict__ cn, uint32_t nq, uint32_t k_cells, uint32_t dpad,
                         uint32_t* __restrict__ mins_u, const float* __restrict__ limit, uint32_t* __restrict__ cand,
                         uint32_t* __restrict__ cand_count) {
    extern __shared__ __align__(1024) char psm[];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2], s_dfull[2], s_dempty[2];
    __shared__ uint32_t s_tmem;
    char* sA = psm;                                   // [2][PT_A_BYTES]
    char* sB = psm + 2 * PT_A_BYTES;                  // [2][PT_B_BYTES]
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nslab = (dpad + PT_KS - 1) / PT_KS;
    const uint32_t mtiles = (nq + PT_M - 1) / PT_M, ntiles = (k_cells + PT_N - 1) / PT_N;
    const uint32_t ngroups = (ntiles + PT_NGROUP - 1) / PT_NGROUP, n_items = mtiles * ngroups;
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            pt_mbar_init(&s_full[i], 1);
            pt_mbar_init(&s_empty[i], 1);
            pt_mbar_init(&s_dfull[i], 1);
            pt_mbar_init(&s_dempty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(pt_smem_u32(&s_tmem)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        // ---- producer
        uint32_t it = 0;
        for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const uint32_t mt = item / ngroups, g = item % ngroups;
            for (uint32_t nt = g * PT_NGROUP; nt < min(ntiles, (g + 1) * PT_NGROUP); ++nt)
                for (uint32_t sl = 0; sl < nslab; ++sl, ++it) {
                    const uint32_t st = it & 1u;
                    pt_mbar_wait(&s_empty[st], ((it >> 1) & 1u) ^ 1u);
                    if (lane == 0) {
                        const uint32_t bar = pt_smem_u32(&s_full[st]);
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(PT_A_BYTES + PT_B_BYTES) : "memory");
                        const char* srcA = reinterpret_cast<const char*>(A) + (size_t(mt) * nslab + sl) * PT_A_BYTES;
                        const char* srcB = reinterpret_cast<const char*>(B) + (size_t(nt) * nslab + sl) * PT_B_BYTES;
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                         pt_smem_u32(sA + st * PT_A_BYTES)), "l"(srcA), "r"(PT_A_BYTES), "r"(bar) : "memory");
                        for (uint32_t off = 0; off < PT_B_BYTES; off += 32768u)
                            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                             pt_smem_u32(sB + st * PT_B_BYTES + off)), "l"(srcB + off), "r"(32768u), "r"(bar) : "memory");
                    }
                    __syncwarp();
                }
        }
    } else if (warp == 1) {
        // ---- MMA issuer
        uint32_t it = 0, tile = 0;
        for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const uint32_t g = item % ngroups;
            for (uint32_t nt = g * PT_NGROUP; nt < min(ntiles, (g + 1) * PT_NGROUP); ++nt, ++tile) {
                const uint32_t buf = tile & 1u;
                pt_mbar_wait(&s_dempty[buf], ((tile >> 1) & 1u) ^ 1u);
                for (uint32_t sl = 0; sl < nslab; ++sl, ++it) {
                    const uint32_t st = it & 1u;
                    pt_mbar_wait(&s_full[st], (it >> 1) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (lane == 0) {
                        const uint32_t ksteps = min(PT_KS, dpad - sl * PT_KS) / 16;
                        const uint32_t a0 = pt_smem_u32(sA + st * PT_A_BYTES), b0 = pt_smem_u32(sB + st * PT_B_BYTES);
                        for (uint32_t ks = 0; ks < ksteps; ++ks) {
                            const uint64_t da = pt_desc(a0 + ks * 2 * (PT_M * 16), PT_M * 16, 128);
                            const uint64_t db = pt_desc(b0 + ks * 2 * (PT_N * 16), PT_N * 16, 128);
                            const uint32_t acc = (sl | ks) != 0u;
                            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                                         ::"r"(tmem + buf * PT_N), "l"(da), "l"(db), "r"(PT_IDESC), "r"(acc) : "memory");
                        }
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(pt_smem_u32(&s_empty[st])) : "memory");
                        if (sl + 1 == nslab)
                            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(pt_smem_u32(&s_dfull[buf])) : "memory");
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ---- epilogue (warps 2..9: TMEM lane quadrant = warp & 3, column half = (warp - 2) / 4); thread = query row
        const uint32_t quad = warp & 3u, chalf = (warp - 2) >> 2;
        const float INF = __int_as_float(0x7f800000);
        uint32_t tile = 0;
        for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const uint32_t mt = item / ngroups, g = item % ngroups;
            const uint32_t q = mt * PT_M + quad * 32 + lane;
            float mn[PT_N / 2]; // PASS 1: running minimum of each of this thread's 128 residue classes over the item's cell tiles
            float lim = 0.0f;
            const uint32_t bm_words = ntiles * (PT_N / 32); // bitmap words per query (cells padded to whole tiles)
            if (PASS == 1) {
#pragma unroll
                for (int j = 0; j < int(PT_N / 2); ++j) mn[j] = INF;
            } else {
                lim = q < nq ? limit[q] : -INF; // rows past the batch never pass
            }
            for (uint32_t nt = g * PT_NGROUP; nt < min(ntiles, (g + 1) * PT_NGROUP); ++nt, ++tile) {
                const uint32_t buf = tile & 1u;
                pt_mbar_wait(&s_dfull[buf], (tile >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const bool full_tile = (nt + 1) * PT_N <= k_cells; // the last tile's padding columns are zero operands: skip them
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const uint32_t c0 = chalf * (PT_N / 2) + cc * 32;
                    uint32_t v[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
                          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(tmem + buf * PT_N + ((quad * 32u) << 16) + c0));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    const uint32_t c = nt * PT_N + c0; // first of this thread's 32 consecutive cells
                    float val[32];
                    if (full_tile) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 n4 = *reinterpret_cast<const float4*>(cn + c + j); // same address in every lane
                            val[j] = n4.x - 2.0f * __uint_as_float(v[j]);
                            val[j + 1] = n4.y - 2.0f * __uint_as_float(v[j + 1]);
                            val[j + 2] = n4.z - 2.0f * __uint_as_float(v[j + 2]);
                            val[j + 3] = n4.w - 2.0f * __uint_as_float(v[j + 3]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            val[j] = c + j < k_cells ? cn[c + j] - 2.0f * __uint_as_float(v[j]) : INF; // +inf: never a minimum; as a candidate it is dropped by the exact kernel's bound check
                    }
                    if (PASS == 1) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) mn[cc * 32 + j] = fminf(mn[cc * 32 + j], val[j]); // NaN never lowers a minimum
                    } else {
                        // this thread's 32 consecutive cells are exactly one word of the query's candidate bitmap: a plain
                        // store, no atomics, no divergence (appending to a list with atomicAdd was 3x slower than the
                        // whole contraction)
                        uint32_t bits = 0;
#pragma unroll
                        for (int j = 0; j < 32; ++j) bits |= (!(val[j] > lim) ? 1u : 0u) << j; // NaN stays a candidate; padding cells are +inf
                        if (q < nq) cand[size_t(q) * bm_words + (c >> 5)] = bits;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(pt_smem_u32(&s_dempty[buf])) : "memory");
            }
            if (PASS == 1 && q < nq) {
                uint32_t* dst = mins_u + size_t(q) * PT_N + chalf * (PT_N / 2);
#pragma unroll
                for (int j = 0; j < int(PT_N / 2); ++j) atomicMin(dst + j, pt_ordered(mn[j]));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// ---------------------------------------------------------------- candidates -> exact order --

// One CTA (256 threads) per query: T = a-th smallest of the 256 class minima, limit = T + 2 eps rounded UP to fp32
// (a superset of candidates is always safe).  a <= min(256, K) is guaranteed by the launcher.
__global__ void __launch_bounds__(256)
probe_limit_kernel(const uint32_t* __restrict__ mins_u, const double* __restrict__ eps2, uint32_t a,
                   float* __restrict__ limit) {
    __shared__ float mins[256];
    const uint32_t qi = blockIdx.x, tid = threadIdx.x;
    mins[tid] = pt_unordered(mins_u[size_t(qi) * 256 + tid]);
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
    if (tid == 0) limit[qi] = __double2float_ru(double(mins[a - 1]) + eps2[qi]);
}

// One CTA (256 threads) per query: compact the candidate bitmap, evaluate the reference's exact distance for the
// candidates, first a by (distance bits, cell).  dynamic smem: the query (dims floats).
__global__ void __launch_bounds__(256)
probe_exact_kernel(const uint32_t* __restrict__ bitmap, uint32_t bm_words, const float* __restrict__ queries,
                   const float* __restrict__ coarse, uint32_t dims, uint32_t k_cells, uint32_t a,
                   uint32_t* __restrict__ order, uint32_t* __restrict__ redo) {
    extern __shared__ __align__(16) float exs[];
    float* qs = exs;
    __shared__ uint64_t cand[TC_CAND];
    __shared__ uint32_t s_cnt;
    const uint32_t qi = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) s_cnt = 0;
    for (uint32_t j = tid; j < dims; j += 256) qs[j] = queries[size_t(qi) * dims + j];
    __syncthreads();
    for (uint32_t w0 = 0; w0 < bm_words; w0 += 256) { // warp-uniform trip count
        const uint32_t w = w0 + tid;
        uint32_t bits = w < bm_words ? bitmap[size_t(qi) * bm_words + w] : 0u;
        if (w * 32 + 32 > k_cells) bits &= w * 32 >= k_cells ? 0u : (0xFFFFFFFFu >> (32 - (k_cells - w * 32))); // padding cells
        const uint32_t n = __popc(bits);
        uint32_t incl = n;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += t;
        }
        uint32_t base = 0;
        if (lane == 31 && incl) base = atomicAdd(&s_cnt, incl);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - n;
        while (bits) {
            const uint32_t j = __ffs(bits) - 1;
            bits &= bits - 1;
            if (base < TC_CAND) cand[base] = w * 32 + j;
            ++base;
        }
    }
    __syncthreads();
    const uint32_t n = s_cnt;
    if (n > TC_CAND || n < a) { // overflow (massive ties, non-finite input: a NaN limit admits every cell)
        if (tid == 0) {         // flags[nq] | compact list[nq] | count
            redo[qi] = 1u;
            redo[gridDim.x + atomicAdd(&redo[2 * size_t(gridDim.x)], 1u)] = qi;
        }
        return;
    }
    // the reference's distance (index.hpp:254-258): fp32, serial over the dims, unfused.  One thread per candidate,
    // walking its centroid row straight from L2 (staging the rows through shared memory with coalesced loads was
    // measured 2.8x slower: one CTA per SM and a barrier per 128 rows).
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

// d_coarse_bf16 (tiled image), d_cnorm [K], d_mean [dims] come from ivf_probe_tc_prepare (host, at open).
size_t ivf_probe_tc_query_image_elems(uint32_t nq, uint32_t dpad) {
    const uint32_t nslab = (dpad + PT_KS - 1) / PT_KS;
    return size_t((nq + PT_M - 1) / PT_M) * nslab * 16 * PT_M * 8;
}

// workspace of the prefilter: class minima [nq][256] | limit [nq] | candidate bitmaps [nq][ceil(K / 256) * 8]
size_t ivf_probe_tc_scratch_bytes(uint32_t nq, uint32_t k_cells) {
    return size_t(nq) * (256 + 1 + size_t((k_cells + PT_N - 1) / PT_N) * (PT_N / 32)) * 4;
}

void launch_ivf_probe_tc(const float* d_queries, const float* d_coarse, const uint16_t* d_coarse_bits,
                         const float* d_cnorm, const double* d_mean, double cmax, uint32_t dims, uint32_t dpad,
                         uint32_t k_cells, uint32_t nq, uint32_t a, uint16_t* d_q_bits, double* d_eps2,
                         float* d_scratch, uint32_t* d_redo, uint32_t* d_order, cudaStream_t stream) {
    const __nv_bfloat16* d_coarse_bf16 = reinterpret_cast<const __nv_bfloat16*>(d_coarse_bits);
    __nv_bfloat16* d_qb = reinterpret_cast<__nv_bfloat16*>(d_q_bits);
    uint32_t* mins_u = reinterpret_cast<uint32_t*>(d_scratch);
    float* limit = reinterpret_cast<float*>(mins_u + size_t(nq) * 256);
    uint32_t* bitmap = reinterpret_cast<uint32_t*>(limit + nq);
    QADC_CUDA_CHECK(cudaMemsetAsync(d_redo, 0, (2 * size_t(nq) + 1) * 4, stream)); // flags | list | count
    QADC_CUDA_CHECK(cudaMemsetAsync(mins_u, 0xFF, size_t(nq) * 256 * 4, stream));  // ordered encoding of "no value yet"
    const uint32_t nq_pad = (nq + PT_M - 1) / PT_M * PT_M;
    probe_prep_queries_kernel<<<(nq_pad * 32 + 255) / 256, 256, 0, stream>>>(d_queries, d_mean, dims, dpad, nq, nq_pad, cmax,
                                                                            d_qb, d_eps2);
    int dev = 0, sms = 0;
    QADC_CUDA_CHECK(cudaGetDevice(&dev));
    QADC_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint32_t mtiles = nq_pad / PT_M, ntiles = (k_cells + PT_N - 1) / PT_N;
    const uint32_t n_items = mtiles * ((ntiles + PT_NGROUP - 1) / PT_NGROUP);
    const uint32_t grid = std::min<uint32_t>(uint32_t(sms), n_items);
    QADC_CUDA_CHECK(cudaFuncSetAttribute(probe_approx_umma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(PT_SMEM)));
    QADC_CUDA_CHECK(cudaFuncSetAttribute(probe_approx_umma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(PT_SMEM)));
    probe_approx_umma_kernel<1><<<grid, PT_THREADS, PT_SMEM, stream>>>(d_qb, d_coarse_bf16, d_cnorm, nq, k_cells, dpad, mins_u,
                                                                       nullptr, nullptr, nullptr);
    probe_limit_kernel<<<nq, 256, 0, stream>>>(mins_u, d_eps2, a, limit);
    probe_approx_umma_kernel<2><<<grid, PT_THREADS, PT_SMEM, stream>>>(d_qb, d_coarse_bf16, d_cnorm, nq, k_cells, dpad, nullptr,
                                                                       limit, bitmap, nullptr);
    probe_exact_kernel<<<nq, 256, size_t(dims) * 4, stream>>>(bitmap, ntiles * (PT_N / 32), d_queries, d_coarse, dims, k_cells, a, d_order,
                                                     d_redo);
    g_launches += 5;
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
    const uint32_t nslab = (dpad + PT_KS - 1) / PT_KS;
    bf16_out.assign(size_t((k_cells + PT_N - 1) / PT_N) * nslab * 16 * PT_N * 8, 0); // tiled operand image, zero padded
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
            bf16_out[probe_image_index(c, j, PT_N, nslab)] = uint16_t(bits >> 16);
        }
        if (!(s - s == 0.0)) return false;
        cnorm[c] = float(s);
        cmax = std::max(cmax, std::sqrt(s));
    }
    cmax *= 1.0 + 1e-9;
    return true;
}

} // namespace qadc
