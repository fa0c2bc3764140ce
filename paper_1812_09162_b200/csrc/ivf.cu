// ivf.cu -- device stages of IvfIndex::search (index.hpp:276-341) in front of the shared scan kernel.
//
//   probe_order      index.hpp:247-265  K serial fp32 squared distances, first a by (dist, cell)
//   residual tables  index.hpp:282-288  one compute_tables per (query, probed cell)
//   shared map       index.hpp:299-316  d_min_global = min over probed cells of min_total();
//                                       prefix over cells in probe order until t distances;
//                                       d_max = r_eff-th smallest; delta = (d_max - d_min_global)/q_max
//   per cell         index.hpp:319-329  quantize against the SHARED bounds, bias =
//                                       floor((own_d_min - d_min_global)/delta) in fp32, scan with ids
//
// The CPU loops query -> cell -> code.  On the GPU the loop is inverted: all (query, cell)
// pairs that probe the same cell are grouped into tiles of LUT rows, so a cell's codes are
// streamed once per tile and reused by every query probing it -- the same scan kernel as the
// flat index, with per-row bias, a row -> query map and explicit ids.
// Every float that feeds the quantizer follows the reference's operation order with explicitly
// rounded fp32 ops (see lut.cu); the file is compiled with --fmad=false.
#include "select_common.cuh"

namespace qadc {

// ------------------------------------------------------------------ list layout --

// One thread per (padded) device code slot: find its list by binary search over the padded
// offsets and gather its words from the list's transposed blocks (layout.hpp:105-125).
__global__ void ivf_relayout_kernel(const uint8_t* __restrict__ packed, const uint64_t* __restrict__ byte_off,
                                    const uint64_t* __restrict__ code_off, const uint64_t* __restrict__ count,
                                    uint32_t k_cells, uint64_t total_padded, uint32_t rows, uint32_t wb,
                                    uint32_t block_len, uint32_t stride, uint8_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= total_padded) return;
    uint32_t lo = 0, hi = k_cells; // last list with code_off <= i
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (code_off[mid] <= i) lo = mid;
        else hi = mid;
    }
    const uint64_t p = i - code_off[lo];
    uint8_t* dst = out + i * stride;
    if (p >= count[lo]) {
        for (uint32_t b = 0; b < stride; ++b) dst[b] = 0xFF;
        return;
    }
    const uint64_t bb = uint64_t(rows) * block_len * wb;
    const uint8_t* blk = packed + byte_off[lo] + (p / block_len) * bb;
    const uint32_t s = uint32_t(p % block_len);
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t b = 0; b < wb; ++b) dst[r * wb + b] = blk[(uint64_t(r) * block_len + s) * wb + b];
    for (uint32_t b = rows * wb; b < stride; ++b) dst[b] = 0xFF;
}

void launch_ivf_relayout(const qadc_spec& s, const DevSpec& ds, const uint8_t* d_packed, const uint64_t* d_byte_off,
                         const uint64_t* d_code_off, const uint64_t* d_count, uint32_t k_cells, uint64_t total_padded,
                         uint8_t* d_codes, cudaStream_t stream) {
    if (total_padded == 0) return;
    ivf_relayout_kernel<<<unsigned((total_padded + 255) / 256), 256, 0, stream>>>(
        d_packed, d_byte_off, d_code_off, d_count, k_cells, total_padded, s.groups, s.word_width / 8, s.block_len,
        ds.code_stride, d_codes);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------------ probe order --

// Coarse distances, register-tiled: a CTA owns 256 cells (one per thread) x PROBE_QT queries.  Each
// thread walks the dims SERIALLY for every (query, cell) pair -- the reference's operation order,
// index.hpp:254-258 -- but loads each centroid component once for all PROBE_QT queries (from the
// transposed [dims][K] matrix, coalesced across cells), so the 8 MB matrix is read nq/16 times from
// L2 instead of nq times.  Queries sit in shared memory as [dim][query] for 128-bit broadcast loads.
static constexpr int PROBE_QT = 16;

__global__ void __launch_bounds__(256)
ivf_coarse_dist_kernel(const float* __restrict__ queries, const float* __restrict__ coarse_t, uint32_t dims,
                       uint32_t k_cells, uint32_t nq, float* __restrict__ dist /* [nq][K] */,
                       const uint32_t* __restrict__ redo_list /* flags[nq] | list[nq] | count */) {
    extern __shared__ __align__(16) float qs[]; // [dims][PROBE_QT]
    __shared__ uint32_t s_qidx[PROBE_QT];
    // redo pass of the tensor-core prefilter: the undecided queries come as a compact list, a small grid walks it
    const uint32_t n_list = redo_list ? redo_list[2 * size_t(nq)] : nq;
    for (uint32_t q0 = blockIdx.y * PROBE_QT; q0 < n_list; q0 += gridDim.y * PROBE_QT) {
    __syncthreads(); // previous tile's shared data is no longer read
    if (threadIdx.x < PROBE_QT)
        s_qidx[threadIdx.x] = q0 + threadIdx.x < n_list ? (redo_list ? redo_list[nq + q0 + threadIdx.x] : q0 + threadIdx.x)
                                                        : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t u = threadIdx.x; u < dims * PROBE_QT; u += blockDim.x) {
        const uint32_t qi = u % PROBE_QT, j = u / PROBE_QT;
        qs[u] = s_qidx[qi] != 0xFFFFFFFFu ? queries[size_t(s_qidx[qi]) * dims + j] : 0.0f;
    }
    __syncthreads();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k_cells) continue;
    float acc[PROBE_QT];
#pragma unroll
    for (int i = 0; i < PROBE_QT; ++i) acc[i] = 0.0f;
    for (uint32_t j = 0; j < dims; ++j) {
        const float ctr = coarse_t[size_t(j) * k_cells + c];
        const float4* qv = reinterpret_cast<const float4*>(qs + j * PROBE_QT);
#pragma unroll
        for (int v = 0; v < PROBE_QT / 4; ++v) {
            const float4 x = qv[v];
            float d;
            d = __fsub_rn(x.x, ctr); acc[4 * v + 0] = __fadd_rn(acc[4 * v + 0], __fmul_rn(d, d));
            d = __fsub_rn(x.y, ctr); acc[4 * v + 1] = __fadd_rn(acc[4 * v + 1], __fmul_rn(d, d));
            d = __fsub_rn(x.z, ctr); acc[4 * v + 2] = __fadd_rn(acc[4 * v + 2], __fmul_rn(d, d));
            d = __fsub_rn(x.w, ctr); acc[4 * v + 3] = __fadd_rn(acc[4 * v + 3], __fmul_rn(d, d));
        }
    }
#pragma unroll
    for (int i = 0; i < PROBE_QT; ++i)
        if (s_qidx[i] != 0xFFFFFFFFu) dist[size_t(s_qidx[i]) * k_cells + c] = acc[i];
    }
}

// One CTA (256 threads) per query: first a cells by (distance, cell) -- partial_sort on pairs,
// index.hpp:261.  key = float bits << 32 | cell (distance >= +0, so float order == bit order).
// dynamic smem: K keys (u64) + pow2(a) keys.
__global__ void __launch_bounds__(256)
ivf_probe_select_kernel(const float* __restrict__ dist, uint32_t k_cells, uint32_t a, uint32_t* __restrict__ order,
                        const uint32_t* __restrict__ only_flagged) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm_raw);
    uint64_t* best = keys + k_cells;
    __shared__ SelectScratch sc;
    const uint32_t qi = blockIdx.x;
    if (only_flagged && !only_flagged[qi]) return; // the fast kernel already produced this query's order
    for (uint32_t c = threadIdx.x; c < k_cells; c += blockDim.x)
        keys[c] = (uint64_t(__float_as_uint(dist[size_t(qi) * k_cells + c])) << 32) | c;
    __syncthreads();
    auto key_at = [&](uint32_t i) -> uint64_t { return keys[i]; };
    uint32_t pow2 = 1;
    while (pow2 < a) pow2 <<= 1;
    if (a < k_cells) {
        uint32_t eq;
        const uint64_t kth = block_select_kth(key_at, k_cells, a, 64, &sc, &eq);
        block_keep_smallest(key_at, k_cells, a, kth, eq, &sc, best);
    } else {
        for (uint32_t i = threadIdx.x; i < k_cells; i += blockDim.x) best[i] = keys[i];
    }
    for (uint32_t i = a + threadIdx.x; i < pow2; i += blockDim.x) best[i] = KEY_INF;
    __syncthreads();
    for (uint32_t size = 2; size <= pow2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < pow2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = best[lo], y = best[hi];
                if ((x > y) == up) {
                    best[lo] = y;
                    best[hi] = x;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < a; i += blockDim.x) order[size_t(qi) * a + i] = uint32_t(best[i]);
}

// Fast path of the probe selection (a <= 256): threshold-and-compact instead of a full radix select.
// Every thread takes the minimum of its strided share of the K keys; the a-th smallest of those 256
// minima is a real key, hence an upper bound T on the a-th smallest key overall.  A second pass
// compacts the (typically ~a) keys <= T, which are then sorted.  Exact: ties are part of the key
// (distance bits << 32 | cell).  If more than PROBE_CAND keys pass (massive ties), the query is
// flagged and redone by the radix kernel.
static constexpr uint32_t PROBE_CAND = 2048;

__global__ void __launch_bounds__(256)
ivf_probe_select_fast_kernel(const float* __restrict__ dist, uint32_t k_cells, uint32_t a,
                             uint32_t* __restrict__ order, uint32_t* __restrict__ redo) {
    __shared__ uint64_t mins[256];
    __shared__ uint64_t cand[PROBE_CAND];
    __shared__ uint32_t s_cnt;
    const uint32_t qi = blockIdx.x, tid = threadIdx.x;
    const float* d = dist + size_t(qi) * k_cells;
    uint64_t m = KEY_INF;
    for (uint32_t c = tid; c < k_cells; c += 256) m = min(m, (uint64_t(__float_as_uint(d[c])) << 32) | c);
    mins[tid] = m;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (uint32_t size = 2; size <= 256; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            if (tid < 128) {
                const uint32_t lo = 2 * tid - (tid & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = mins[lo], y = mins[hi];
                if ((x > y) == up) {
                    mins[lo] = y;
                    mins[hi] = x;
                }
            }
            __syncthreads();
        }
    const uint64_t T = mins[a - 1]; // a <= min(256, K) guaranteed by the launcher
    for (uint32_t base = 0; base < k_cells; base += 256) {
        const uint32_t c = base + tid;
        const uint64_t k = c < k_cells ? ((uint64_t(__float_as_uint(d[c])) << 32) | c) : KEY_INF;
        const bool take = k <= T;
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        if (bal) {
            uint32_t start = 0;
            if ((tid & 31) == 0) start = atomicAdd(&s_cnt, uint32_t(__popc(bal)));
            start = __shfl_sync(0xffffffffu, start, 0);
            const uint32_t slot = start + __popc(bal & ((1u << (tid & 31)) - 1u));
            if (take && slot < PROBE_CAND) cand[slot] = k;
        }
    }
    __syncthreads();
    const uint32_t n = s_cnt;
    if (n > PROBE_CAND) {
        if (tid == 0) redo[qi] = 1u;
        return;
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

void launch_ivf_probe(const float* d_queries, const float* d_coarse_t, uint32_t dims, uint32_t k_cells, uint32_t nq,
                      uint32_t a, float* d_dist_scratch, uint32_t* d_redo /* [nq] */, uint32_t* d_order,
                      cudaStream_t stream, bool redo_only) {
    // redo_only: d_redo already flags the queries the tensor-core prefilter (ivf_probe_tc.cu) could not
    // decide; only those get exact distances and the radix selection
    if (nq == 0 || a == 0) return;
    uint32_t pow2 = 1;
    while (pow2 < a) pow2 <<= 1;
    const size_t smem_sel = size_t(k_cells) * 8 + size_t(pow2) * 8;
    if (smem_sel > 200 * 1024)
        throw Error(QADC_ERR_CONFIG, "ivf probe: coarse quantizer too large for the shared-memory selection "
                                     "(K*8 + probes*8 bytes must fit 200 KB)");
    const size_t smem_d = size_t(dims) * PROBE_QT * 4;
    if (smem_d > 200 * 1024) throw Error(QADC_ERR_CONFIG, "ivf probe: dims too large");
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_coarse_dist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_d)));
    const uint32_t q_tiles = (nq + PROBE_QT - 1) / PROBE_QT;
    const dim3 grid((k_cells + 255) / 256, redo_only ? std::min<uint32_t>(q_tiles, 8u) : q_tiles);
    ivf_coarse_dist_kernel<<<grid, 256, smem_d, stream>>>(d_queries, d_coarse_t, dims, k_cells, nq, d_dist_scratch,
                                                          redo_only ? d_redo : nullptr);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_probe_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_sel)));
    const bool fast = !redo_only && a <= 256 && a <= k_cells && k_cells >= 256;
    if (fast) {
        QADC_CUDA_CHECK(cudaMemsetAsync(d_redo, 0, size_t(nq) * 4, stream));
        ivf_probe_select_fast_kernel<<<nq, 256, 0, stream>>>(d_dist_scratch, k_cells, a, d_order, d_redo);
        ++g_launches;
        QADC_CUDA_CHECK(cudaGetLastError());
    }
    // radix select: the only path for large a / tiny K, the fallback of flagged queries otherwise
    ivf_probe_select_kernel<<<nq, 256, smem_sel, stream>>>(d_dist_scratch, k_cells, a, d_order,
                                                           fast || redo_only ? d_redo : nullptr);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------- residual tables --

// One CTA walks IVF_PAIRS_PER_CTA consecutive (query, probe) pairs: residual = q - centroid
// (index.hpp:286), compute_tables, per-table minima and their table-order sum
// (DistanceTables::min_total, distance.hpp:28-32).
static constexpr uint32_t IVF_PAIRS_PER_CTA = 8;

__global__ void __launch_bounds__(256)
ivf_tables_kernel(DevSpec ds, const float* __restrict__ codebook, const float* __restrict__ queries,
                  const float* __restrict__ coarse, const uint32_t* __restrict__ order, uint32_t a, uint32_t n_pairs,
                  float* __restrict__ luts, float* __restrict__ pmin_out, float* __restrict__ own_min) {
    extern __shared__ float smf[];
    float* res = smf;
    float* lut = res + ds.dims;
    float* pmin = lut + ds.E;
    for (uint32_t k = 0; k < IVF_PAIRS_PER_CTA; ++k) {
        const uint32_t pair = blockIdx.x * IVF_PAIRS_PER_CTA + k;
        if (pair >= n_pairs) return;
        const uint32_t qi = pair / a;
        const uint32_t cell = order[pair];
        __syncthreads(); // previous pair's shared data is no longer read
        for (uint32_t d = threadIdx.x; d < ds.dims; d += blockDim.x)
            res[d] = __fsub_rn(queries[size_t(qi) * ds.dims + d], coarse[size_t(cell) * ds.dims + d]);
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x) {
            uint32_t j = 0;
            while (j + 1 < ds.m && ds.ent_off[j + 1] <= e) ++j;
            const uint32_t dsub = ds.dim_alloc[j];
            const float* c = codebook + ds.cb_off[j] + size_t(e - ds.ent_off[j]) * dsub;
            const float* qq = res + ds.dim_off[j];
            float acc = 0.0f;
            for (uint32_t t = 0; t < dsub; ++t) {
                const float d = __fsub_rn(qq[t], c[t]);
                acc = __fadd_rn(acc, __fmul_rn(d, d));
            }
            lut[e] = acc;
            luts[size_t(pair) * ds.E + e] = acc;
        }
        __syncthreads();
        // per-table minima, one warp per table (min is order-independent, so a tree is exact)
        for (uint32_t j = threadIdx.x >> 5; j < ds.m; j += blockDim.x >> 5) {
            float mn = __int_as_float(0x7f800000);
            const float* t = lut + ds.ent_off[j];
            for (uint32_t i = threadIdx.x & 31; i < (1u << ds.bits[j]); i += 32) mn = (t[i] < mn) ? t[i] : mn;
            for (int o = 16; o > 0; o >>= 1) {
                const float other = __shfl_xor_sync(0xffffffffu, mn, o);
                mn = (other < mn) ? other : mn;
            }
            if ((threadIdx.x & 31) == 0) {
                pmin[j] = mn;
                pmin_out[size_t(pair) * ds.m + j] = mn;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float s = 0.0f; // table-order fp32 sum (distance.hpp:28-32)
            for (uint32_t j = 0; j < ds.m; ++j) s = __fadd_rn(s, pmin[j]);
            own_min[pair] = s;
        }
    }
}

void launch_ivf_tables(const DevSpec& ds, const float* d_codebook, const float* d_queries, const float* d_coarse,
                       const uint32_t* d_order, uint32_t n_pairs, uint32_t a, float* d_luts, float* d_pmin,
                       float* d_own_min, cudaStream_t stream) {
    if (n_pairs == 0) return;
    const size_t smem = sizeof(float) * (size_t(ds.dims) + ds.E + ds.m);
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ivf_tables_kernel<<<(n_pairs + IVF_PAIRS_PER_CTA - 1) / IVF_PAIRS_PER_CTA, 256, smem, stream>>>(
        ds, d_codebook, d_queries, d_coarse, d_order, a, n_pairs, d_luts, d_pmin, d_own_min);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------------- calibration --

// One CTA per query.  Also counts the (query, cell) pairs per cell for the row grouping and
// records each pair's rank inside its cell.  dynamic smem: t floats + a uint32 (prefix starts).
// qparams[q] = {d_min_global, d_max, delta, n_prefix}
// calib_codes / calib_off / calib_count describe the HEADS of the unsharded lists (first min(count, t_max)
// codes each): for an unsharded index they alias the lists themselves; a shard gets replicated heads so
// that every rank derives the same map.  list_count is the LOCAL length (rows are only grouped for
// lists this rank actually holds codes of).
__global__ void __launch_bounds__(256)
ivf_calib_kernel(DevSpec ds, const uint8_t* __restrict__ codes, const uint64_t* __restrict__ list_code_off,
                 const uint64_t* __restrict__ calib_count, const uint64_t* __restrict__ list_count,
                 const uint32_t* __restrict__ order, uint32_t a,
                 const float* __restrict__ luts, const float* __restrict__ own_min, uint32_t r, uint32_t t,
                 float* __restrict__ qparams, float* __restrict__ map, uint32_t* __restrict__ cell_npairs,
                 uint32_t* __restrict__ pair_rank) {
    extern __shared__ float smf[];
    float* prefix = smf;                                       // t floats, padded to a power of two for the sort
    uint32_t tpow = 1;
    while (tpow < t) tpow <<= 1;
    uint32_t* start = reinterpret_cast<uint32_t*>(prefix + tpow); // a + 1 entries
    __shared__ float s_dmin;
    __shared__ uint32_t s_np;
    __shared__ float w_min[8];
    __shared__ uint32_t w_sum[8];
    const uint32_t qi = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* ord = order + size_t(qi) * a;
    // d_min_global = min over the probed cells of min_total() (index.hpp:301-302), and the prefix budget:
    // cell i contributes min(count_i, t - taken) codes, i.e. taken_i = min(sum_{k<i} count_k, t) (index.hpp:305-306).
    // Probes are walked in chunks of 256 with a block-wide exclusive scan.
    float dmin = __int_as_float(0x7f800000);
    uint32_t carry = 0; // codes taken by earlier chunks (saturated at t)
    for (uint32_t base = 0; base < a; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        uint32_t cnt = 0;
        if (i < a) {
            const float mt = own_min[size_t(qi) * a + i];
            dmin = (mt < dmin) ? mt : dmin;
            cnt = uint32_t(min(calib_count[ord[i]], uint64_t(t)));
        }
        uint32_t incl = cnt; // inclusive warp scan, saturating at t keeps the sums small
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl = min(incl + v, t);
        }
        uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1); // saturated sum of the lanes before this one
        if (lane == 0) excl = 0;
        if (lane == 31) w_sum[warp] = incl;
        __syncthreads();
        uint32_t before = carry;
        for (uint32_t w = 0; w < warp; ++w) before = min(before + w_sum[w], t);
        if (i < a) start[i] = min(before + excl, t);
        uint32_t total = carry;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) total = min(total + w_sum[w], t);
        carry = total;
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float other = __shfl_xor_sync(0xffffffffu, dmin, o);
        dmin = (other < dmin) ? other : dmin;
    }
    if (lane == 0) w_min[warp] = dmin;
    // row grouping: every probed, non-empty cell gets this pair as one LUT row
    for (uint32_t i = threadIdx.x; i < a; i += blockDim.x) {
        const uint32_t cell = ord[i];
        pair_rank[size_t(qi) * a + i] = list_count[cell] ? atomicAdd(&cell_npairs[cell], 1u) : 0xFFFFFFFFu;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = w_min[0];
        for (uint32_t w = 1; w < (blockDim.x >> 5); ++w) m = (w_min[w] < m) ? w_min[w] : m;
        s_dmin = m;
        start[a] = carry;
        s_np = carry;
    }
    __syncthreads();
    const uint32_t np = s_np;
    for (uint32_t p = threadIdx.x; p < np; p += blockDim.x) {
        uint32_t lo = 0, hi = a; // the probe this prefix position falls into: last i with start[i] <= p
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (start[mid] <= p) lo = mid;
            else hi = mid;
        }
        const uint32_t i = lo;
        const uint8_t* code = codes + (list_code_off[ord[i]] + (p - start[i])) * ds.code_stride;
        const float* lut = luts + (size_t(qi) * a + i) * ds.E;
        float acc = 0.0f;
        for (uint32_t j = 0; j < ds.m; ++j) acc = __fadd_rn(acc, lut[ds.ent_off[j] + code_field(ds, code, j)]);
        prefix[p] = acc;
    }
    float d_max = 0.0f;
    if (np) {
        // r_eff-th smallest of the prefix (index.hpp:308, calibrate_bounds): bitonic sort of the bit patterns
        // (sums of non-negative terms: unsigned order == float order), padded with +inf
        const uint32_t r_eff = min(r, np);
        uint32_t npow = 2;
        while (npow < np) npow <<= 1;
        uint32_t* key = reinterpret_cast<uint32_t*>(prefix);
        for (uint32_t i = np + threadIdx.x; i < npow; i += blockDim.x) key[i] = 0xFFFFFFFFu;
        __syncthreads();
        for (uint32_t size = 2; size <= npow; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < npow / 2; i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const uint32_t x = key[lo], y = key[hi];
                    if ((x > y) == up) {
                        key[lo] = y;
                        key[hi] = x;
                    }
                }
                __syncthreads();
            }
        d_max = prefix[r_eff - 1];
    }
    if (threadIdx.x == 0) {
        float* o = qparams + size_t(qi) * 4;
        o[0] = s_dmin;
        o[1] = d_max;
        o[2] = np ? __fdiv_rn(__fsub_rn(d_max, s_dmin), float(ds.qmax)) : 0.0f; // index.hpp:316
        o[3] = __uint_as_float(np);
        map[size_t(qi) * 2 + 0] = o[2];   // unquantize: float(sum) * delta + d_min_global (index.hpp:337)
        map[size_t(qi) * 2 + 1] = s_dmin;
    }
}

void launch_ivf_calib(const DevSpec& ds, const uint8_t* d_codes, const uint64_t* d_list_code_off,
                      const uint64_t* d_calib_count, const uint64_t* d_list_count, const uint32_t* d_order, uint32_t nq,
                      uint32_t a,
                      const float* d_luts, const float* d_own_min, uint32_t r, uint32_t t, float* d_qparams,
                      float* d_map, uint32_t* d_cell_npairs, uint32_t* d_pair_rank, cudaStream_t stream) {
    if (nq == 0) return;
    size_t tpow = 1;
    while (tpow < t) tpow <<= 1;
    const size_t smem = tpow * 4 + size_t(a + 1) * 4;
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_calib_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ivf_calib_kernel<<<nq, 256, smem, stream>>>(ds, d_codes, d_list_code_off, d_calib_count, d_list_count, d_order, a, d_luts,
                                                d_own_min, r, t, d_qparams, d_map, d_cell_npairs, d_pair_rank);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------- threshold seeding --

// One CTA per query: exact quantized sums of the head of the first probed list that holds at
// least r codes; thr_key = (r-th smallest key) + 1.  The codes are real candidates that the
// streaming scan will meet again, so this is a valid (exclusive) upper bound on the final
// r-th key; nothing is kept, only the bound.  dynamic smem: head keys + table (u16).
__global__ void __launch_bounds__(256)
ivf_seed_kernel(DevSpec ds, const uint8_t* __restrict__ codes, const uint32_t* __restrict__ ids,
                const uint64_t* __restrict__ list_code_off, const uint64_t* __restrict__ list_count,
                const uint32_t* __restrict__ order, uint32_t a, const uint32_t* __restrict__ pair_slot,
                const void* __restrict__ qluts, const uint32_t* __restrict__ row_bias, uint32_t r, uint32_t head,
                uint64_t* __restrict__ thr_key) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm_raw);
    uint16_t* table = reinterpret_cast<uint16_t*>(keys + head);
    __shared__ SelectScratch sc;
    __shared__ uint32_t s_probe;
    const uint32_t qi = blockIdx.x;
    if (threadIdx.x == 0) {
        uint32_t pick = 0xFFFFFFFFu;
        for (uint32_t i = 0; i < a; ++i)
            if (list_count[order[size_t(qi) * a + i]] >= r) {
                pick = i;
                break;
            }
        s_probe = pick;
    }
    __syncthreads();
    if (s_probe == 0xFFFFFFFFu) return; // no list with r codes: the scan starts unbounded
    const uint32_t pair = qi * a + s_probe;
    const uint32_t cell = order[pair];
    const uint32_t slot = pair_slot[pair];
    const uint32_t n = uint32_t(min(list_count[cell], uint64_t(head)));
    for (uint32_t e = threadIdx.x; e < ds.E; e += blockDim.x)
        table[e] = ds.word_width == 8 ? uint16_t(reinterpret_cast<const uint8_t*>(qluts)[size_t(slot) * ds.E + e])
                                      : reinterpret_cast<const uint16_t*>(qluts)[size_t(slot) * ds.E + e];
    __syncthreads();
    const uint32_t bias = min(row_bias[slot], ds.qmax);
    const uint64_t base = list_code_off[cell];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint8_t* code = codes + (base + i) * ds.code_stride;
        uint32_t acc = bias;
        if (ds.code_stride == 8) {
            const uint2 cw = *reinterpret_cast<const uint2*>(code);
            for (uint32_t j = 0; j < ds.m; ++j) acc += table[ds.ent_off[j] + code_field64(ds, cw.x, cw.y, j)];
        } else {
            for (uint32_t j = 0; j < ds.m; ++j) acc += table[ds.ent_off[j] + code_field(ds, code, j)];
        }
        keys[i] = make_key(min(acc, ds.qmax), ids[base + i]);
    }
    __syncthreads();
    auto key_at = [&](uint32_t i) -> uint64_t { return keys[i]; };
    uint32_t eq;
    const uint64_t kth = block_select_kth(key_at, n, r, 48, &sc, &eq);
    if (threadIdx.x == 0) thr_key[qi] = kth + 1; // exclusive bound: the seed codes themselves re-enter via the scan
}

void launch_ivf_seed(const DevSpec& ds, const uint8_t* d_codes, const uint32_t* d_ids, const uint64_t* d_list_code_off,
                     const uint64_t* d_list_count, const uint32_t* d_order, uint32_t nq, uint32_t a,
                     const uint32_t* d_pair_slot, const void* d_qluts, const uint32_t* d_row_bias, uint32_t r,
                     uint32_t head, uint64_t* d_thr_key, cudaStream_t stream) {
    if (nq == 0 || head < r) return;
    const size_t smem = size_t(head) * 8 + size_t(ds.E) * 2;
    QADC_CUDA_CHECK(cudaFuncSetAttribute(ivf_seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ivf_seed_kernel<<<nq, 256, smem, stream>>>(ds, d_codes, d_ids, d_list_code_off, d_list_count, d_order, a,
                                               d_pair_slot, d_qluts, d_row_bias, r, head, d_thr_key);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc
