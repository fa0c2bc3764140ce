// common.cuh -- internal declarations shared by the translation units of libqadc_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "qadc.h"

namespace qadc {

// ---- errors: C++ exceptions inside the library, mapped to status codes at the C ABI ----
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

#define QADC_CUDA_CHECK(expr)                                                                        \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess)                                                                       \
            throw ::qadc::Error(QADC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
    } while (0)

// ---- device-side view of a spec (kernel parameter, passed by value) ----
struct DevSpec {
    uint32_t dims, m, E, cb_floats;
    uint32_t word_width; // 8 / 16
    uint32_t qmax;       // 255 / 65535
    uint32_t code_bytes; // rows * word_bytes
    uint32_t code_stride; // bytes between consecutive codes in the device layout (multiple of 8)
    uint8_t bits[QADC_MAX_SUBS];
    uint8_t bitpos[QADC_MAX_SUBS]; // bit position of subquantizer j inside the little-endian code
    uint32_t dim_off[QADC_MAX_SUBS];
    uint32_t dim_alloc[QADC_MAX_SUBS];
    uint32_t ent_off[QADC_MAX_SUBS];
    uint32_t cb_off[QADC_MAX_SUBS];
};

DevSpec make_dev_spec(const qadc_spec& s, uint32_t rows);

// 64-bit candidate key: (quantized distance << 32) | id.  Lexicographic (distance, id)
// order of the reference's CandidateHeap (heap.hpp:21-23) == unsigned order of the key.
__host__ __device__ inline uint64_t make_key(uint32_t dist, uint32_t id) { return (uint64_t(dist) << 32) | id; }
static constexpr uint64_t KEY_INF = ~0ull;

// ---- scan job: one (code range) x (tile of LUT rows) unit of work ----
struct ScanJob {
    uint64_t code_off; // first code (index into the device code array)
    uint64_t ids_off;  // index of the first code's id in the ids array (explicit-id mode)
    uint32_t n_codes;
    uint32_t id_base;  // implicit-id mode: id of the first code
    uint32_t row_begin; // first LUT row of the tile
    uint32_t n_rows;    // rows in the tile (<= TQ of the variant)
};

// ---- scan kernel variants ----
enum ScanVariant : uint32_t {
    VAR_F16X8 = 0,   // u8 tables, fp16 entries in smem, 8 rows per lane (LDS.128), 256-row tile
    VAR_F32X2 = 1,   // u16 tables, fp32 entries in smem, 2 rows per lane (LDS.64), 64-row tile
    VAR_U16X1 = 2,   // any width, u16 entries in smem, 1 row per lane, 32-row tile, int32 accumulate
    VAR_U8X1 = 3,    // any width, u8 (high-byte for u16 tables) conservative filter, 32-row tile
    VAR_F16X4H = 4,  // u16 tables, fp16 HIGH-BYTE conservative filter, 4 rows per lane (LDS.64), 128-row tile
    VAR_F16X4H_C2 = 5, // same, 2 codes per warp step, 64-row tile (short row groups: IVF)
    VAR_F16X4H_C4 = 6, // same, 4 codes per warp step, 32-row tile
    VAR_F16X4_C4 = 7,  // u8 tables exact in fp16, 4 codes per warp step, 32-row tile (large 8-bit tables: 8x{8})
    VAR_F16X4H_C4D = 8, // as C4 with every entry line stored twice (128 B): code groups 0/2 read the low copy,
                        // 1/3 the high copy, so the four groups of a warp never share a bank
    VAR_F16X4_C4M = 9,  // 16x{4,4} scanned as 8x{8}: table j of the tile holds T[2j][b & 15] + T[2j+1][b >> 4] for
                        // every byte b of the code (pair sums <= 510, exact in fp16) -- half the lookups per code
    VAR_F16X4H_C8Q = 10, // 12x{6,5,5} scanned as 8 lookups per code: per 16-bit word one 6-bit table and one 1024-entry
                         // table of (5,5) pair sums; 16-row tile whose 128-byte lines hold the same entry of the four
                         // words' tables (quad-interleaved); code groups walk the words in rotated order
    VAR_F16X4H_C16Q = 11, // irregular 16-bit specs on 16-row tiles: quad lines (the same entry of the four words' tables),
                          // rotated codes, LDS.128, 16 codes per warp step -- the IVF layout with the least row padding
    VAR_TC8 = 12, // 16x{4,4} as a one-hot int8 GEMM on tcgen05 (scan_tc.cu): 128 codes x 256 queries per MMA tile, s32
                  // accumulators in TMEM, the admission threshold folded into a ninth K step (sign bit = admit)
    VAR_TC8S = 13, // the same with 2:4-SPARSE MMAs: a one-hot row has one non-zero per 16 K bytes, so A is stored compressed
                   // (two kept bytes per group of four + 4 metadata bits in tensor memory) and every MMA covers 64 logical K
                   // at the cost of 32: 240-query tiles (24 TMEM columns go to the metadata stages)
    VAR_TC8P = 14, // the sparse form on CTA PAIRS (cta_group::2, clusters of two): M = 256 codes per MMA, each SM holds and
                   // reads only half of the tile's tables (the single-CTA form is bound by those shared-memory reads)
    VAR_COUNT
};

struct ScanArgs {
    const uint8_t* codes;      // device code array, code_stride bytes per code
    const uint32_t* ids;       // explicit ids or nullptr
    const void* qlut;          // [rows][E] at table width, reference table order (exact re-evaluation)
    const void* tile_lut;      // [tile][E][TQ] in the variant's entry type (tilepack.cu); tile = row / TQ
    const uint32_t* row_query; // row -> query index (nullptr: identity)
    const uint32_t* row_bias;  // row -> acc_init (nullptr: 0)
    const ScanJob* jobs;
    uint32_t n_jobs;
    const uint32_t* cta_begin; // optional [grid + 1]: job slice of every CTA (cost-balanced); nullptr = equal counts
    uint64_t* thr_key;         // [nq] current R-th smallest key (KEY_INF while fewer than R)
    uint64_t* cand;            // [nq][cap]
    uint32_t* cand_count;      // [nq]
    uint32_t cap;
    uint32_t* overflow;        // [nq] set to 1 when a candidate did not fit
    uint32_t tile_bufs;        // 1 or 2 LUT tile buffers in shared memory (filled in by launch_scan from the plan)
    uint32_t filter_shift;     // conservative filters on 16-bit tables compare floor(x >> shift) (from the plan)
};

struct ScanPlan {
    ScanVariant variant;
    uint32_t tq;         // rows per tile
    uint32_t smem_bytes;
    uint32_t threads;
    uint32_t tile_bufs;  // 2 when a second LUT tile buffer fits: the next job's tile is prefetched
    // Conservative fp16 filter on 16-bit tables: entries, bias and threshold are compared as floor(x >> shift).
    // fp16 holds integers exactly up to 2048, so shift = 5 (11-bit entries) keeps every partial sum that can still
    // be admitted exact; the shift grows with m so that m * (65535 >> shift) stays below the "admit all" sentinel.
    // 8 for the u8-entry variant, 0 for exact variants and 8-bit tables.
    uint32_t filter_shift;
};

// chooses the variant for a spec (throws config error if nothing fits shared memory)
// allow_merged: the caller packs its tiles with launch_pack_tiles (flat index, scan shim); the IVF batch path
// writes tiles itself and does not produce the merged-pair layout.
ScanPlan plan_scan(const DevSpec& ds, int device, int force_variant, bool allow_merged = false);
void launch_scan(const ScanPlan& plan, const DevSpec& ds, const ScanArgs& args, int grid, cudaStream_t stream);
// tensor-core scan of 16x{4,4} (scan_tc.cu)
inline bool is_tc8(int variant) { return variant == VAR_TC8 || variant == VAR_TC8S || variant == VAR_TC8P; }
inline int tc8_mode(int variant) { return variant - int(VAR_TC8); } // 0 dense, 1 sparse, 2 sparse on CTA pairs
uint32_t scan_tc8_smem_bytes(int mode);
uint32_t scan_tc8_tile_rows(int mode);
uint32_t scan_tc8_pack_rows(int mode);
void launch_scan_tc8(int mode, const DevSpec& ds, const ScanArgs& args, int grid, cudaStream_t stream);
void launch_pack_tiles_tc8(const void* qlut, uint32_t n_rows, uint32_t tq, uint32_t images_per_tile, void* out, cudaStream_t stream);

// ---- LUT / calibration / quantization (lut.cu) ----
struct LutArgs {
    const float* codebook;    // flat codebook on device
    const float* queries;     // [nq][dims]
    const float* sub;         // optional [nq][dims] vectors subtracted first (IVF residual), or nullptr
    const uint8_t* calib_codes; // device layout, first codes of the list
    uint32_t calib_count;     // number of valid calibration codes (<= t)
    uint32_t nq, r, t;
    float* luts;              // optional [nq][E]
    void* qluts;              // [nq][E] at table width
    float* calib;             // [nq][4] {d_min, d_max, delta, own_d_min}
    float* map;               // [nq][2] {delta, d_min} used to unquantize
    int* status;              // device int, set non-zero on calibration errors
};
void launch_flat_tables(const DevSpec& ds, const LutArgs& a, cudaStream_t stream);

// ---- selection (select.cu) ----
void launch_init_select(uint64_t* thr_key, uint32_t* cand_count, uint32_t* ntop, uint32_t* overflow, uint32_t nq,
                        cudaStream_t stream);
// fold the new candidates of every query into its running top-r and refresh thr_key
void launch_tighten(uint64_t* top, uint32_t* ntop, uint32_t kpad, uint64_t* cand, uint32_t* cand_count, uint32_t cap,
                    uint64_t* thr_key, uint32_t nq, uint32_t r, unsigned long long* admitted /* optional counter */,
                    cudaStream_t stream);
// sort each query's top list and emit ids / unquantized distances / counts / keys
void launch_finalize(const uint64_t* lists, const uint32_t* counts_in, uint32_t list_len, uint32_t nlists,
                     uint32_t nq, uint32_t r, const float* map, uint32_t flags, uint32_t qmax, uint32_t* out_ids,
                     float* out_dists, uint32_t* out_counts, uint64_t* out_keys, cudaStream_t stream);

// ---- tile-layout tables (tilepack.cu) ----
size_t tile_entry_bytes(ScanVariant v);
// Pair-interleaved tile layout of the 32-row variants when every table has 256 entries (8x{8,8}, 8x{8}, merged
// 16x{4,4}): tables 2k and 2k+1 share 128-byte lines -- entry i of table 2k in the low half of line k*256 + i,
// entry i of table 2k+1 in the high half.  Odd code groups of a warp walk each table pair in swapped order, so
// at every step two groups read low halves and two read high halves: no bank conflicts (scan.cu).
// The same interleave serves the irregular 16-bit specs on 32-row tiles with the pairing unit = one 16-bit WORD of
// the code (words w and w ^ 1 have identical table sizes; odd code groups see their code with the 16-bit halves of
// every 32-bit word swapped).  `block` = entries of one pairing unit: 256 (a table) or E / 4 (a word's tables).
// Bit 31 of `block` selects the QUAD interleave instead (16-row tiles: four units per 128-byte line).
static constexpr uint32_t TILE_QUAD = 0x80000000u;
__host__ __device__ inline uint32_t pair_perm(uint32_t e, uint32_t block) {
    const uint32_t b = block & ~TILE_QUAD, u = e / b, i = e - u * b;
    if (block & TILE_QUAD) return (i << 2) | u;
    return ((((u >> 1) * b) + i) << 1) | (u & 1u);
}
// 0 = dense lines; otherwise the pairing block of the tile layout the scan kernel expects for (variant, spec)
uint32_t tile_pair_layout(ScanVariant v, const DevSpec& ds);
// entries of one LUT row in the tile image (the spec's E, except for the merged-pair layout)
uint32_t tile_entries(ScanVariant v, uint32_t E);
void launch_pack_tiles(ScanVariant v, uint32_t filter_shift, uint32_t pair, const void* qlut, uint32_t width, uint32_t E, uint32_t n_rows, uint32_t tq,
                       void* out, cudaStream_t stream);

// ---- dense head evaluation (seed.cu) ----
void launch_seed_topk(const DevSpec& ds, const uint8_t* d_codes, uint32_t n_head, uint32_t id_base,
                      const uint32_t* d_ids, const void* d_qlut, const uint32_t* d_row_bias, uint32_t nq, uint32_t r,
                      uint64_t* top, uint32_t* ntop, uint32_t kpad, uint64_t* thr_key, cudaStream_t stream);

// ---- IVF stages (ivf.cu) ----
void launch_ivf_relayout(const qadc_spec& s, const DevSpec& ds, const uint8_t* d_packed, const uint64_t* d_byte_off,
                         const uint64_t* d_code_off, const uint64_t* d_count, uint32_t k_cells, uint64_t total_padded,
                         uint8_t* d_codes, cudaStream_t stream);
void launch_ivf_probe(const float* d_queries, const float* d_coarse_t, uint32_t dims, uint32_t k_cells, uint32_t nq,
                      uint32_t a, float* d_dist_scratch /* [nq][K] */, uint32_t* d_redo /* [nq] */, uint32_t* d_order,
                      cudaStream_t stream, bool redo_only = false);
// tensor-core prefilter of the probe order (ivf_probe_tc.cu)
bool ivf_probe_tc_supported(uint32_t dims, uint32_t k_cells, uint32_t a);
size_t ivf_probe_tc_query_image_elems(uint32_t nq, uint32_t dpad); // bf16 elements of the tiled query operand image
size_t ivf_probe_tc_scratch_bytes(uint32_t nq, uint32_t k_cells);    // class minima, limits, candidate bitmaps
bool ivf_probe_tc_prepare(const float* coarse, uint32_t k_cells, uint32_t dims, uint32_t dpad,
                          std::vector<uint16_t>& bf16_out, std::vector<float>& cnorm, std::vector<double>& mean,
                          double& cmax);
void launch_ivf_probe_tc(const float* d_queries, const float* d_coarse, const uint16_t* d_coarse_bf16 /* bf16 bits */,
                         const float* d_cnorm, const double* d_mean, double cmax, uint32_t dims, uint32_t dpad,
                         uint32_t k_cells, uint32_t nq, uint32_t a, uint16_t* d_qb /* bf16 bits */, double* d_eps2,
                         float* d_scratch, uint32_t* d_redo, uint32_t* d_order, cudaStream_t stream);
void launch_ivf_tables(const DevSpec& ds, const float* d_codebook, const float* d_queries, const float* d_coarse,
                       const uint32_t* d_order, uint32_t n_pairs, uint32_t a, float* d_luts, float* d_pmin,
                       float* d_own_min, cudaStream_t stream);
bool ivf_tables_tiled_supported(const DevSpec& ds);
void ivf_tables_tiled_prepare(const DevSpec& ds, const float* codebook, std::vector<float>& cb_tp,
                              std::vector<uint8_t>& sub_of);
void launch_ivf_tables_tiled(const DevSpec& ds, const float* d_codebook_tp, const uint8_t* d_sub_of,
                             const float* d_queries, const float* d_coarse, const uint32_t* d_order, uint32_t n_pairs,
                             uint32_t a, float* d_luts, float* d_pmin, float* d_own_min, cudaStream_t stream);
void launch_ivf_quantize_pack(ScanVariant v, uint32_t filter_shift, uint32_t pair, const DevSpec& ds, const uint32_t* d_order, uint32_t n_pairs, uint32_t a,
                              const float* d_luts, const float* d_pmin, const float* d_own_min,
                              const float* d_qparams, const uint32_t* d_pair_rank, const uint32_t* d_cell_tile_base,
                              uint32_t tq, uint32_t ntiles, void* d_qluts, void* d_tile_lut, uint32_t* d_row_query,
                              uint32_t* d_row_bias, uint32_t* d_pair_slot, uint32_t* d_slot_pair,
                              cudaStream_t stream);
void launch_ivf_calib(const DevSpec& ds, const uint8_t* d_calib_codes, const uint64_t* d_calib_code_off,
                      const uint64_t* d_calib_count, const uint64_t* d_list_count, const uint32_t* d_order, uint32_t nq,
                      uint32_t a,
                      const float* d_luts, const float* d_own_min, uint32_t r, uint32_t t, float* d_qparams,
                      float* d_map, uint32_t* d_cell_npairs, uint32_t* d_pair_rank, cudaStream_t stream);
void launch_ivf_seed(const DevSpec& ds, const uint8_t* d_codes, const uint32_t* d_ids, const uint64_t* d_list_code_off,
                     const uint64_t* d_list_count, const uint32_t* d_order, uint32_t nq, uint32_t a,
                     const uint32_t* d_pair_slot, const void* d_qluts, const uint32_t* d_row_bias, uint32_t r,
                     uint32_t head, uint64_t* d_thr_key, cudaStream_t stream);

// ---- exact re-ranking of the final top-R (rerank.cu) ----
void launch_rerank(const DevSpec& ds, const uint8_t* d_codes, const float* d_luts, uint32_t base_id,
                   const uint32_t* d_locator, const uint64_t* d_list_code_off, const uint32_t* d_order, uint32_t k_cells,
                   uint32_t a, uint32_t nq, uint32_t r, uint32_t* d_ids, float* d_dists, const uint32_t* d_counts,
                   cudaStream_t stream);

// ---- layout (layout.cu) ----
// reference PackedList bytes (device copy) -> linear device layout, padded with 0xFF codes up to n_padded
void launch_relayout(const qadc_spec& s, const DevSpec& ds, const uint8_t* d_packed, uint64_t n, uint64_t n_padded,
                     uint8_t* d_codes, cudaStream_t stream);
void launch_unlayout(const DevSpec& ds, const uint8_t* d_codes, uint64_t first, uint64_t n, uint8_t* d_subcodes,
                     cudaStream_t stream);
void launch_adc_sums(const DevSpec& ds, const uint8_t* d_codes, const void* d_qlut, uint32_t acc_init,
                     uint64_t first, uint64_t n, uint32_t* d_sums, cudaStream_t stream);
size_t ivf_assign_scratch_bytes(uint32_t k_cells, uint64_t n);
void launch_ivf_assign(const float* d_vectors, const float* d_coarse, const float* d_coarse_t, uint32_t dims,
                       uint32_t k_cells, uint64_t n, void* d_scratch, uint32_t* d_assign, float* d_resid,
                       cudaStream_t stream);
void launch_ivf_group_pack(const qadc_spec& spec, const DevSpec& ds, const uint32_t* d_assign, const uint8_t* d_codes, uint64_t n,
                           uint32_t k_cells, unsigned long long* d_counts, unsigned long long* d_id_off,
                           unsigned long long* d_byte_off, unsigned long long* d_totals, uint32_t* d_order, uint8_t* d_packed,
                           int* d_status, cudaStream_t stream);
void launch_encode(const DevSpec& ds, const float* d_codebook, const float* d_vectors, uint64_t n, uint8_t* d_codes,
                   cudaStream_t stream);

extern thread_local unsigned long long g_launches; // kernels launched by this thread's current call

} // namespace qadc
