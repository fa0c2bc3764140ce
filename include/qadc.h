/*
 * qadc.h -- C ABI of the B200-native Quicker ADC scan path (libqadc_b200.so).
 *
 * This is the drop-in boundary for the reference's scan/search path
 * (reference = header-only C++ library `pqscan`, paths below are relative to
 * /root/reference/proj/include/pqscan/).  Plain pointers and sizes only; the
 * library never throws: every entry point returns a status whose numeric class
 * mirrors the reference's exception taxonomy (errors.hpp:9-46 and the exit codes
 * the CLI maps them to, tools/pqscan_cli.cpp:20-30), and qadc_last_error() holds
 * the message.  There is NO CPU fallback: with no usable CUDA device every
 * compute entry point fails with QADC_ERR_CUDA.
 *
 * Host buffers are owned by the caller; a handle owns its device memory.
 * A handle is immutable after open; calls on one handle serialise on its stream.
 */
#ifndef QADC_H
#define QADC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QADC_MAX_SUBS 64
#define QADC_MAX_GROUP 16
#define QADC_MAX_R 16384 /* results per query supported by the device top-R stage (round 1: 1024) */
#define QADC_MAX_T 16384 /* longest calibration prefix t (the reference bounds neither; beyond these -> config error) */

/* status classes: reference exception -> CLI exit code (errors.hpp, pqscan_cli.cpp:20-30) */
enum {
    QADC_OK = 0,
    QADC_ERR_INVALID_SPEC = 3, /* invalid_spec_error */
    QADC_ERR_TRAINING = 4,     /* training_error (unused by this path) */
    QADC_ERR_INPUT = 5,        /* input_error */
    QADC_ERR_CORRUPTION = 6,   /* corruption_error */
    QADC_ERR_CONFIG = 7,       /* config_error */
    QADC_ERR_IO = 8,           /* io_error (unused by this path) */
    QADC_ERR_CALIBRATION = 9,  /* calibration_error */
    QADC_ERR_CUDA = 20         /* CUDA runtime / no device: new class, no reference analogue */
};

/* Flattened PqSpec (pqspec.hpp:66-113) + PackingScheme (layout.hpp:18-46).
 * Flat float codebooks are the per-subquantizer centroid matrices
 * (codebook.hpp:60, k_j x dim_alloc[j] row-major) concatenated in subquantizer
 * order (cb_off[j] floats in); flat LUTs are the per-subquantizer tables
 * concatenated (ent_off[j] entries in). */
typedef struct qadc_spec {
    uint32_t dims;
    uint32_t m;          /* subquantizers */
    uint32_t g;          /* group size */
    uint32_t groups;     /* m / g = rows of a packed block */
    uint32_t word_width; /* 8 or 16: packing word AND quantized table width */
    uint32_t block_len;  /* 16 / 32 / 64 codes per transposed block */
    uint32_t exact;      /* proportional dim split was integral */
    uint32_t total_entries;
    uint32_t cb_floats;
    uint8_t widths[QADC_MAX_GROUP];
    uint8_t offsets[QADC_MAX_GROUP];
    uint8_t bits[QADC_MAX_SUBS];
    uint32_t dim_alloc[QADC_MAX_SUBS];
    uint32_t dim_off[QADC_MAX_SUBS];
    uint32_t ent_off[QADC_MAX_SUBS];
    uint32_t cb_off[QADC_MAX_SUBS];
} qadc_spec;

/* SearchParams (index.hpp:20-32).  flags: bit 1 = rerank (below); bit 0 = fuse the final q*delta+d_min
 * into one FMA like the reference's default -march=native build does
 * (distance.hpp:158-161); default 0 = unfused, matching the pinned oracle. */
typedef struct qadc_search_params {
    uint32_t probes; /* IVF only */
    uint32_t r;
    uint32_t t;
    uint32_t flags;
} qadc_search_params;
#define QADC_FLAG_FMA_UNQUANTIZE 1u
/* SearchParams::rerank (index.hpp:24): re-order the final top-R by exact float ADC (index.hpp:53-67, 148-152,
 * 377-386).  Only for unsharded handles (ids must address this handle's own codes); incompatible with d_out_keys. */
#define QADC_FLAG_RERANK 2u

/* counters of the last search on a handle (bench.py's gpu_launches comes from here) */
typedef struct qadc_stats {
    uint64_t kernel_launches; /* kernels of this library launched by the last call */
    uint64_t scan_launches;
    uint64_t pairs_scanned;   /* (query, code) pairs evaluated by the scan kernels */
    uint64_t candidates;      /* pairs that passed the exact admission test */
    uint64_t overflow_retries;
    uint64_t segments;
    uint32_t scan_variant;    /* which scan kernel variant ran (see qadc_variant_name) */
    uint32_t query_tile;      /* queries (LUT rows) resident in shared memory per CTA */
    float ms_lut, ms_scan, ms_select; /* CUDA-event time of the stages of the last search */
} qadc_stats;

typedef struct qadc_index qadc_index;

const char* qadc_version(void);
const char* qadc_last_error(void);
const char* qadc_variant_name(uint32_t variant);
/* number of CUDA devices visible, or a negative QADC_ERR_CUDA-class failure */
int qadc_device_count(void);

/* parse_spec_string + allocate_dims + PackingScheme::for_spec
 * (pqspec.hpp:24-55, 119-171; layout.hpp:27-43) */
int qadc_spec_parse(uint32_t dims, const char* text, qadc_spec* out);

/* bytes of a PackedList holding n codes (layout.hpp:135-144) */
uint64_t qadc_packed_bytes(const qadc_spec* spec, uint64_t n);

/* ---- FlatIndex (index.hpp:73-157) ---------------------------------------
 * packed/count: the reference PackedList bytes of this shard (layout.hpp:135-160).
 * base_id: id of the shard's first code (ids are base_id + position,
 *          scan_scalar.hpp:60); 0 for an unsharded index.
 * calib_packed/calib_count: PackedList of the first codes of the WHOLE list
 *          (>= the largest t that will be used), needed only by shards whose
 *          own head is not the global head (index.hpp:124-129 calibrates on the
 *          global prefix); NULL/0 = use this shard's own head.
 * global_count: length of the WHOLE list the shard belongs to (ignored without
 *          calib_packed).  The reference calibrates on min(t, global_count) codes; when the
 *          replicated head is shorter than the whole list (calib_count < global_count, or
 *          global_count = 0 = unknown) a search with t > calib_count cannot reproduce that
 *          and fails with QADC_ERR_CONFIG instead of silently calibrating on fewer codes.
 * device: CUDA ordinal. */
int qadc_flat_open(const qadc_spec* spec, const float* codebook, const uint8_t* packed, uint64_t count,
                   uint32_t base_id, const uint8_t* calib_packed, uint64_t calib_count, uint64_t global_count,
                   int device, qadc_index** out);

/* ---- IvfIndex (index.hpp:166-177, 276-341) ------------------------------
 * Lists are concatenated: list c has list_count[c] codes, PackedList bytes at
 * packed + list_byte_off[c], ids at ids + list_id_off[c].
 * calib_*: per-list PackedList of the first min(count_global, t_max) codes of the
 * unsharded list (same convention as the flat index), or NULL to use own heads;
 * calib_count[c] = codes held by head c; global_list_count[c] = length of the unsharded list c
 * (required with calib_*).  A search whose t exceeds the shortest TRUNCATED head
 * (calib_count[c] < global_list_count[c]) fails with QADC_ERR_CONFIG: the reference's prefix
 * (index.hpp:304-306) could ask that list for more codes than the head holds. */
int qadc_ivf_open(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                  const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                  const uint64_t* list_count, const uint32_t* ids, const uint8_t* calib_packed,
                  const uint64_t* calib_byte_off, const uint64_t* calib_count, const uint64_t* global_list_count,
                  int device, qadc_index** out);

/* Open a QFLT (flat) or QIVF (IVF) container written by the reference (io.hpp:276-326) directly: headers are parsed on
 * the host, the packed blocks go to the device as they are and are re-laid there.  load_flat_index / load_ivf_index
 * + the FlatIndex / IvfIndex constructors in one call; same error classes (io 8, corruption 6, invalid_spec 3). */
int qadc_open_file(const char* path, int device, qadc_index** out);
/* kind: 0 flat, 1 ivf; count = total codes; cells = K (0 for flat).  Any output may be NULL. */
int qadc_index_info(const qadc_index* h, int* kind, qadc_spec* spec, uint64_t* count, uint32_t* cells);

void qadc_close(qadc_index* h);

/* FlatIndex::search / IvfIndex::search over a batch (index.hpp:110, 276), host buffers.
 * out_ids/out_dists: nq*r, ascending (distance, id); rows shorter than r are
 * padded (id 0xFFFFFFFF, dist +inf) and out_counts[q] < r says so
 * (reference returns shorter vectors, T/test_index.cpp:33-44). */
int qadc_search_batch(qadc_index* h, const float* queries, uint32_t nq, const qadc_search_params* params,
                      uint32_t* out_ids, float* out_dists, uint32_t* out_counts);

/* Same with DEVICE buffers on `stream` (a cudaStream_t, NULL = the handle's own).
 * d_out_keys (optional, nq*r u64): (quantized distance << 32 | id), padded with
 * ~0, the per-shard lists exchanged by the multi-GPU merge.
 * d_out_map (optional, nq*2 floats): {delta, d_min} of each query's affine map. */
int qadc_search_batch_device(qadc_index* h, const float* d_queries, uint32_t nq, const qadc_search_params* params,
                             uint32_t* d_out_ids, float* d_out_dists, uint32_t* d_out_counts,
                             uint64_t* d_out_keys, float* d_out_map, void* stream);

/* Multi-GPU exchange step: merge `nshards` per-shard key lists (layout
 * [shard][nq][r], as gathered by NCCL all_gather) into the global top-r and
 * unquantize with the (replicated) map.  Device buffers. */
int qadc_merge_topk_device(const uint64_t* d_keys, uint32_t nshards, uint32_t nq, uint32_t r, const float* d_map,
                           uint32_t flags, uint32_t* d_out_ids, float* d_out_dists, uint32_t* d_out_counts,
                           int device, void* stream);

/* ---- one process, several GPUs ----------------------------
 * The reference is single-process; its multi-GPU drop-in is ONE handle that owns a shard per device: contiguous
 * block-aligned code ranges scanned with base_id = range start (the chunked-scan contract, T/test_kernels.cpp:107-133),
 * the whole list's calibration head replicated on every device (index.hpp:124-129), one ncclAllGather of the per-shard
 * (distance << 32 | id) key lists and the merge kernel on devices[0].  NCCL is bound at run time (dlopen of
 * libnccl.so.2); ndev = 1 works without it.  devices = NULL means ordinals 0..ndev-1. */
typedef struct qadc_multi qadc_multi;
int qadc_flat_open_sharded(const qadc_spec* spec, const float* codebook, const uint8_t* packed, uint64_t count, int ndev,
                           const int* devices, qadc_multi** out);
/* The same for IvfIndex (index.hpp:166-177, 276-341; arguments as qadc_ivf_open): EVERY list is split evenly on
 * packed-block boundaries (ids are explicit, so any split is legal: scan_scalar.hpp:60) and the first
 * min(count, QADC_MAX_T) codes of every unsharded list are replicated as calibration heads, so probe order, tables,
 * d_min_global, d_max, delta and the biases come out identical on every device. */
int qadc_ivf_open_sharded(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                          const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                          const uint64_t* list_count, const uint32_t* ids, int ndev, const int* devices, qadc_multi** out);
/* FlatIndex::search / IvfIndex::search over a batch (index.hpp:110, 276), host buffers, same output convention as
 * qadc_search_batch */
int qadc_multi_search_batch(qadc_multi* h, const float* queries, uint32_t nq, const qadc_search_params* params,
                            uint32_t* out_ids, float* out_dists, uint32_t* out_counts);
int qadc_multi_info(const qadc_multi* h, int* ndev, uint64_t* count, int* uses_nccl);
void qadc_multi_close(qadc_multi* h);

/* ---- debug / parity entry points ----------------------- */
/* float LUTs (compute_tables, distance.hpp:35-58), calibration and quantized
 * LUTs (quantize_tables, distance.hpp:102-142) of a flat index.  Any output may
 * be NULL.  luts: nq*total_entries floats; qluts: nq*total_entries at table
 * width; calib: nq*4 floats {d_min, d_max, delta, own_d_min}. */
int qadc_flat_tables(qadc_index* h, const float* queries, uint32_t nq, const qadc_search_params* params,
                     float* luts, void* qluts, float* calib);

/* raw saturating ADC sums (adc_scalar_quantized, distance.hpp:149-155) of codes
 * [first, first+n) of a flat index under a caller-supplied quantized LUT */
int qadc_flat_adc_sums(qadc_index* h, const void* qlut, uint32_t width, uint32_t acc_init, uint64_t first,
                       uint64_t n, uint32_t* sums);

/* IvfIndex::probe_order (index.hpp:247-265) for a batch: order is nq*min(a,K) */
int qadc_ivf_probe_order(qadc_index* h, const float* queries, uint32_t nq, uint32_t a, uint32_t* order);

/* QuantizedScanFn (simd/kernels.hpp:49-50; normative body scan_scalar.hpp:34-64):
 * scan one PackedList with caller-supplied quantized tables into a bounded
 * (distance, id) heap.  heap_in_*: n_in pre-seeded entries; outputs: the heap's
 * sorted() contents (heap.hpp:61-65), *n_out <= cap entries. */
int qadc_scan_list(const qadc_spec* spec, const uint8_t* packed, uint64_t count, uint32_t rows, const void* qlut,
                   uint32_t width, const uint32_t* ids, uint32_t base_id, uint32_t acc_init, uint32_t cap,
                   const uint32_t* heap_in_dist, const uint32_t* heap_in_id, uint32_t n_in, uint32_t* out_dist,
                   uint32_t* out_id, uint32_t* n_out, int device);

/* encode (codebook.hpp:94-118) on the GPU: codes is n*m bytes ("next" row N2) */
int qadc_encode(const qadc_spec* spec, const float* codebook, const float* vectors, uint64_t n, uint8_t* codes,
                int device);

/* IVF list construction given trained centroids and a residual codebook -- the data-dependent half of
 * IvfIndex::build (index.hpp:195-227; "next" row N3): nearest coarse centroid under a double accumulator, ties to
 * the lowest cell (kmeans.hpp:178-190), fp32 residual (index.hpp:200), encode (codebook.hpp:94-118).
 * assign: n u32 cells; codes: n*m subcodes.  The caller groups vectors by cell in index order and packs each list
 * (index.hpp:219-227; paper_1812_09162_b200.index.build_ivf_lists does). */
int qadc_ivf_assign_encode(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                           const float* vectors, uint64_t n, uint32_t* assign, uint8_t* codes, int device);

/* The whole data-dependent half of IvfIndex::build on the GPU (index.hpp:195-227): assignment, residuals, encode AND
 * the per-list grouping + packing (:219-227: every cell's members in ascending vector index, one PackedList per cell,
 * ids = vector indices).  Outputs are exactly qadc_ivf_open's arguments: list_count / list_byte_off / list_id_off
 * (k_cells each), ids (n), packed (caller buffer of packed_cap >= qadc_ivf_build_packed_bound(spec, n, k_cells) bytes;
 * *packed_bytes = bytes written).  assign (optional, n u32) receives the cells. */
uint64_t qadc_ivf_build_packed_bound(const qadc_spec* spec, uint64_t n, uint32_t k_cells);
int qadc_ivf_build_lists(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                         const float* vectors, uint64_t n, uint64_t* list_count, uint64_t* list_byte_off,
                         uint64_t* list_id_off, uint32_t* ids, uint8_t* packed, uint64_t packed_cap, uint64_t* packed_bytes,
                         uint32_t* assign, int device);

/* Guard-zone check of every device buffer (enabled by the environment variable QADC_DEBUG_CANARY; returns 1 when on):
 * buffers verified so far and guard bytes found overwritten (must stay 0).  Stands in for compute-sanitizer memcheck,
 * which the GPU pool refuses. */
int qadc_debug_canary(uint64_t* buffers_checked, uint64_t* bytes_corrupted);

int qadc_get_stats(const qadc_index* h, qadc_stats* out);
/* tuning knobs for experiments: name in {"cand_cap","seg0","seg_growth","force_variant","threads"} */
int qadc_set_option(qadc_index* h, const char* name, int64_t value);
/* device pointer / stride of the re-laid code array (for tests of the layout bijection) */
int qadc_flat_download_codes(qadc_index* h, uint64_t first, uint64_t n, uint8_t* codes_out /* n*m subquantizer indices */);

#ifdef __cplusplus
}
#endif
#endif
