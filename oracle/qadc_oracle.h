/*
 * qadc_oracle.h -- CPU oracle for the Quicker ADC scan path (TEST INFRASTRUCTURE ONLY).
 *
 * This is a plain-C restatement of the reference's algorithm for the hot path
 * (distance tables -> calibration -> table quantization -> packed-code scan with
 * saturating integer accumulation -> top-R by (distance, id)), written from the
 * reference's published semantics.  Every function cites the reference
 * file:line it follows (paths relative to /root/reference/proj/include/pqscan).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  The product (libqadc_b200.so) never
 * links, loads or calls it.
 *
 * Parity status: PINNED.  tests/test_oracle_pins.py checks this restatement
 * against (a) the known-answer vectors held inline by the reference's own
 * tests (transcribed with file:line in tests/test_oracle_pins.py), (b) golden
 * input/output fixtures produced by running the unmodified reference headers
 * (oracle/_ref, built by oracle/Makefile from the sources where they lie), and
 * (c) when oracle/_ref is present, live differential runs against it.
 *
 * The same C API (prefix orc_) is exported by oracle/_ref/libpqscan_ref.so
 * (ref_shim.cpp, which *calls* the reference headers), so tests can swap the
 * two libraries.
 *
 * Build: gcc -O2 -ffp-contract=off  (no FMA contraction: SURVEY.md section 0.3).
 */
#ifndef QADC_ORACLE_H
#define QADC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_SUBS 64
#define ORC_MAX_GROUP 16

/* status codes mirror the reference's error taxonomy (errors.hpp:9-46) and the
 * CLI exit codes it maps them to (tools/pqscan_cli.cpp:20-30). */
enum {
    ORC_OK = 0,
    ORC_ERR_INVALID_SPEC = 3,
    ORC_ERR_TRAINING = 4,
    ORC_ERR_INPUT = 5,
    ORC_ERR_CORRUPTION = 6,
    ORC_ERR_CONFIG = 7,
    ORC_ERR_IO = 8,
    ORC_ERR_CALIBRATION = 9
};

/* PqSpec + PackingScheme flattened (pqspec.hpp:66-113, layout.hpp:18-46). */
typedef struct orc_spec {
    uint32_t dims;       /* total_dims */
    uint32_t m;          /* subquantizers */
    uint32_t g;          /* group size */
    uint32_t groups;     /* m / g == rows of a packed block */
    uint32_t word_width; /* 8 or 16 */
    uint32_t block_len;  /* 16 / 32 / 64 */
    uint32_t exact;      /* proportional split was integral */
    uint32_t total_entries; /* sum_j 2^bits_j */
    uint32_t cb_floats;     /* sum_j 2^bits_j * dim_alloc_j */
    uint8_t widths[ORC_MAX_GROUP];  /* group pattern */
    uint8_t offsets[ORC_MAX_GROUP]; /* LSB-first bit offsets */
    uint8_t bits[ORC_MAX_SUBS];     /* per subquantizer */
    uint32_t dim_alloc[ORC_MAX_SUBS];
    uint32_t dim_off[ORC_MAX_SUBS];
    uint32_t ent_off[ORC_MAX_SUBS]; /* start of table j in a flat LUT */
    uint32_t cb_off[ORC_MAX_SUBS];  /* start of table j in a flat codebook */
} orc_spec;

const char* orc_impl_name(void); /* "port" or "reference" */
const char* orc_last_error(void);

/* parse_spec_string + allocate_dims (pqspec.hpp:24-55, 119-167) */
int orc_spec_parse(uint32_t dims, const char* text, orc_spec* out);

/* pack_list / unpack_list (layout.hpp:146-176).  codes: n*m bytes, one
 * centroid index per subquantizer.  packed: orc_packed_bytes(spec, n). */
uint64_t orc_packed_bytes(const orc_spec* s, uint64_t n);
int orc_pack_list(const orc_spec* s, const uint8_t* codes, uint64_t n, uint8_t* packed);
int orc_unpack_list(const orc_spec* s, const uint8_t* packed, uint64_t n, uint8_t* codes);

/* encode (codebook.hpp:94-118): nearest centroid per slice, double accumulators, lowest-index ties */
int orc_encode(const orc_spec* s, const float* codebook, const float* vectors, uint64_t n, uint8_t* codes);

/* compute_tables (distance.hpp:35-58): flat LUT of total_entries floats */
int orc_compute_tables(const orc_spec* s, const float* codebook, const float* query, float* lut);
/* DistanceTables::min_of / min_total (distance.hpp:22-32) */
float orc_min_total(const orc_spec* s, const float* lut, float* p_min /* m floats or NULL */);

/* collect_prefix_float (scan_scalar.hpp:96-122); returns number appended */
uint64_t orc_prefix_float(const orc_spec* s, const uint8_t* packed, uint64_t count, const float* lut, uint64_t limit,
                          float* out);
/* calibrate_bounds (distance.hpp:74-83) */
int orc_calibrate(const orc_spec* s, const float* lut, const float* prefix, uint64_t n_prefix, uint32_t r,
                  float* d_min, float* d_max);
/* quantize_tables (distance.hpp:102-142).  qlut: total_entries of u8 (width 8) or u16 (width 16). */
int orc_quantize(const orc_spec* s, const float* lut, float d_min, float d_max, uint32_t width, void* qlut,
                 float* p_min /* m */, float* delta, float* own_d_min);

/* scan_list_scalar_quantized (scan_scalar.hpp:34-64) into a CandidateHeap (heap.hpp:16-71).
 * heap_* in: n_in pre-seeded entries; out: sorted() contents, *n_out entries (<= cap).
 * family: 0 = scalar-quantized (normative); 1 = natural vector family (only
 * honoured by the reference build; the port ignores it). */
int orc_scan_quantized(const orc_spec* s, const uint8_t* packed, uint64_t count, uint32_t rows, const void* qlut,
                       uint32_t width, const uint32_t* ids, uint32_t base_id, uint32_t acc_init, uint32_t cap,
                       const uint32_t* heap_in_dist, const uint32_t* heap_in_id, uint32_t n_in, uint32_t* out_dist,
                       uint32_t* out_id, uint32_t* n_out, int family);

/* raw quantized ADC sums of codes [first, first+n) (adc_scalar_quantized, distance.hpp:149-155) */
int orc_adc_sums(const orc_spec* s, const uint8_t* packed, uint64_t count, const void* qlut, uint32_t width,
                 uint32_t acc_init, uint64_t first, uint64_t n, uint32_t* sums);

/* FlatIndex::search (index.hpp:110-145), batched over nq queries with `threads`
 * query-parallel workers (tools/pqscan_cli.cpp:141-166).  out_ids/out_dists:
 * nq*r, out_counts: nq.  Optional debug outputs may be NULL:
 *   dbg_qlut: nq*total_entries at table width; dbg_params: nq*4 floats
 *   {d_min, d_max, delta, own_d_min}.  family as in orc_scan_quantized. */
int orc_flat_search(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count,
                    const float* queries, uint32_t nq, uint32_t r, uint32_t t, int family, int threads,
                    uint32_t* out_ids, float* out_dists, uint32_t* out_counts, void* dbg_qlut, float* dbg_params);

/* IvfIndex::probe_order (index.hpp:247-265) */
int orc_probe_order(uint32_t dims, const float* coarse, uint32_t k_cells, const float* query, uint32_t a,
                    uint32_t* order);

/* IvfIndex::search (index.hpp:276-341).  Lists are concatenated: list c holds
 * list_count[c] codes whose packed bytes start at packed + list_byte_off[c] and
 * whose ids start at ids + list_id_off[c]. */
int orc_ivf_search(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                   const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                   const uint64_t* list_count, const uint32_t* ids, const float* queries, uint32_t nq,
                   uint32_t probes, uint32_t r, uint32_t t, int family, int threads, uint32_t* out_ids,
                   float* out_dists, uint32_t* out_counts);

/* IVF list construction given a trained coarse quantizer and residual codebook (the data-dependent half of
 * IvfIndex::build, index.hpp:195-227): nearest coarse centroid under a DOUBLE accumulator, ties to the lowest index
 * (kmeans.hpp:178-190, detail::sq_dist :41-48); residual = x - centroid in fp32 (index.hpp:200); encode
 * (codebook.hpp:94-118).  assign: n u32; codes: n*m bytes. */
int orc_ivf_assign_encode(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                          const float* vectors, uint64_t n, uint32_t* assign, uint8_t* codes);

/* Handle-based variants for timing (bench.py cpu_baseline): the index is built once, searches reuse it.
 * The port keeps pointers into the caller's arrays (they must stay alive); the reference shim builds a
 * pqscan::FlatIndex / pqscan::IvfIndex once. */
void* orc_flat_create(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count);
int orc_flat_search_h(void* h, const float* queries, uint32_t nq, uint32_t r, uint32_t t, int family, int threads,
                      uint32_t* out_ids, float* out_dists, uint32_t* out_counts);
void orc_flat_destroy(void* h);
void* orc_ivf_create(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                     const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                     const uint64_t* list_count, const uint32_t* ids);
int orc_ivf_search_h(void* h, const float* queries, uint32_t nq, uint32_t probes, uint32_t r, uint32_t t, int family,
                     int threads, uint32_t* out_ids, float* out_dists, uint32_t* out_counts);
void orc_ivf_destroy(void* h);

#ifdef __cplusplus
}
#endif
#endif
