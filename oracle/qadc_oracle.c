/*
 * qadc_oracle.c -- plain-C CPU restatement of the Quicker ADC scan path.
 * TEST INFRASTRUCTURE ONLY (see qadc_oracle.h).  Parity status: PINNED against
 * the reference's known-answer vectors and golden fixtures generated from the
 * unmodified reference headers (tests/test_oracle_pins.py).
 *
 * Citations are reference file:line under proj/include/pqscan/.
 * Build with -ffp-contract=off: the float tables must not be FMA-contracted.
 */
#include "qadc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char* orc_impl_name(void) { return "port"; }
const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ------------------------------------------------------------------ spec -- */

/* pqspec.hpp:24-55 (grammar <m>x{<w>(,<w>)*}) and :119-167 (allocate_dims) */
int orc_spec_parse(uint32_t dims, const char* text, orc_spec* out) {
    memset(out, 0, sizeof *out);
    const char* x = strchr(text, 'x');
    if (!x || x == text) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: missing 'x'");
    uint64_t m = 0;
    for (const char* p = text; p < x; ++p) {
        if (*p < '0' || *p > '9') return fail(ORC_ERR_INVALID_SPEC, "bad spec string: bad subquantizer count");
        m = m * 10 + (uint64_t)(*p - '0');
        if (m > 0xffffffffull) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: bad subquantizer count");
    }
    if (m == 0) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: bad subquantizer count");
    const char* rest = x + 1;
    size_t len = strlen(rest);
    if (len < 3 || rest[0] != '{' || rest[len - 1] != '}')
        return fail(ORC_ERR_INVALID_SPEC, "bad spec string: missing {...}");
    uint32_t g = 0;
    const char* p = rest + 1;
    const char* end = rest + len - 1;
    while (p < end) {
        const char* comma = memchr(p, ',', (size_t)(end - p));
        const char* tok_end = comma ? comma : end;
        if (tok_end == p) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: bad width");
        unsigned w = 0;
        for (const char* c = p; c < tok_end; ++c) {
            if (*c < '0' || *c > '9') return fail(ORC_ERR_INVALID_SPEC, "bad spec string: bad width");
            w = w * 10 + (unsigned)(*c - '0');
            if (w > 1000) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: bad width");
        }
        if (w < 1 || w > 8) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: widths must be in [1,8]");
        if (g >= ORC_MAX_GROUP) return fail(ORC_ERR_INVALID_SPEC, "group too large for the oracle");
        out->widths[g++] = (uint8_t)w;
        if (!comma) break;
        p = comma + 1;
        if (p >= end) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: trailing comma");
    }
    if (g == 0) return fail(ORC_ERR_INVALID_SPEC, "bad spec string: empty width list");

    /* allocate_dims, pqspec.hpp:119-167 */
    if (m % g != 0) return fail(ORC_ERR_INVALID_SPEC, "subquantizer count is not a multiple of the group size");
    uint32_t sum = 0;
    for (uint32_t i = 0; i < g; ++i) sum += out->widths[i];
    if (sum != 8 && sum != 16 && sum != 15)
        return fail(ORC_ERR_INVALID_SPEC, "group bit widths must sum to 8, 15 or 16");
    if (dims < m) return fail(ORC_ERR_INVALID_SPEC, "cannot split dimensions across subquantizers");
    if (m > ORC_MAX_SUBS) return fail(ORC_ERR_INVALID_SPEC, "too many subquantizers for the oracle");

    out->dims = dims;
    out->m = (uint32_t)m;
    out->g = g;
    out->groups = (uint32_t)m / g;
    out->word_width = (sum <= 8) ? 8 : 16;
    const uint64_t total_bits = (uint64_t)sum * out->groups;
    uint64_t assigned = 0;
    for (uint32_t j = 0; j < m; ++j) {
        uint8_t w = out->widths[j % g];
        out->bits[j] = w;
        out->dim_alloc[j] = (uint32_t)((uint64_t)dims * w / total_bits);
        assigned += out->dim_alloc[j];
    }
    uint64_t leftover = dims - assigned;
    out->exact = (leftover == 0);
    for (uint32_t j = 0; leftover > 0; j = (j + 1) % (uint32_t)m, --leftover) out->dim_alloc[j] += 1;
    for (uint32_t j = 0; j < m; ++j)
        if (out->dim_alloc[j] == 0)
            return fail(ORC_ERR_INVALID_SPEC, "dimension allocation left a subquantizer empty");
    uint32_t off = 0, eoff = 0, coff = 0;
    for (uint32_t j = 0; j < m; ++j) {
        out->dim_off[j] = off;
        off += out->dim_alloc[j];
        out->ent_off[j] = eoff;
        eoff += 1u << out->bits[j];
        out->cb_off[j] = coff;
        coff += (1u << out->bits[j]) * out->dim_alloc[j];
    }
    out->total_entries = eoff;
    out->cb_floats = coff;
    /* PackingScheme::for_spec, layout.hpp:27-43 */
    uint8_t o = 0;
    for (uint32_t i = 0; i < g; ++i) {
        out->offsets[i] = o;
        o = (uint8_t)(o + out->widths[i]);
    }
    if (out->word_width == 16) out->block_len = 32;
    else out->block_len = (g == 1) ? 64 : 16;
    return ORC_OK;
}

/* ---------------------------------------------------------------- layout -- */

static inline uint32_t word_bytes(const orc_spec* s) { return s->word_width / 8; }
static inline uint64_t block_bytes(const orc_spec* s, uint32_t rows) {
    return (uint64_t)rows * s->block_len * word_bytes(s);
}
static inline uint64_t block_count(const orc_spec* s, uint64_t n) {
    return n == 0 ? 0 : (n + s->block_len - 1) / s->block_len;
}

uint64_t orc_packed_bytes(const orc_spec* s, uint64_t n) { return block_count(s, n) * block_bytes(s, s->groups); }

/* detail::load_word, scan_scalar.hpp:16-21 (little-endian 16-bit words) */
static inline uint32_t load_word(const uint8_t* p, uint32_t wb) {
    if (wb == 1) return *p;
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8);
}

/* pack_group (layout.hpp:50-60) + transpose_block (:105-125) + pack_list (:146-160) */
int orc_pack_list(const orc_spec* s, const uint8_t* codes, uint64_t n, uint8_t* packed) {
    const uint32_t wb = word_bytes(s), rows = s->groups, g = s->g;
    const uint64_t bb = block_bytes(s, rows);
    memset(packed, 0xFF, (size_t)orc_packed_bytes(s, n)); /* padding slots stay all-ones */
    for (uint64_t i = 0; i < n; ++i) {
        uint8_t* blk = packed + (i / s->block_len) * bb;
        const uint64_t p = i % s->block_len;
        for (uint32_t r = 0; r < rows; ++r) {
            uint32_t w = 0;
            for (uint32_t k = 0; k < g; ++k) {
                uint32_t idx = codes[i * s->m + r * g + k];
                if (idx >= (1u << s->widths[k])) return fail(ORC_ERR_CORRUPTION, "pack_group: index exceeds bit width");
                w |= idx << s->offsets[k];
            }
            uint8_t* dst = blk + ((uint64_t)r * s->block_len + p) * wb;
            dst[0] = (uint8_t)w;
            if (wb == 2) dst[1] = (uint8_t)(w >> 8);
        }
    }
    return ORC_OK;
}

/* unpack_group (layout.hpp:62-68) + untranspose_block (:128-140) + unpack_list (:162-176) */
int orc_unpack_list(const orc_spec* s, const uint8_t* packed, uint64_t n, uint8_t* codes) {
    const uint32_t wb = word_bytes(s), rows = s->groups, g = s->g;
    const uint64_t bb = block_bytes(s, rows);
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t* blk = packed + (i / s->block_len) * bb;
        const uint64_t p = i % s->block_len;
        for (uint32_t r = 0; r < rows; ++r) {
            uint32_t w = load_word(blk + ((uint64_t)r * s->block_len + p) * wb, wb);
            for (uint32_t k = 0; k < g; ++k)
                codes[i * s->m + r * g + k] = (uint8_t)((w >> s->offsets[k]) & ((1u << s->widths[k]) - 1u));
        }
    }
    return ORC_OK;
}

/* ----------------------------------------------------------- codec / LUT -- */

/* encode, codebook.hpp:94-118 */
int orc_encode(const orc_spec* s, const float* codebook, const float* vectors, uint64_t n, uint8_t* codes) {
    for (uint64_t v = 0; v < n; ++v) {
        const float* vec = vectors + v * s->dims;
        for (uint32_t j = 0; j < s->m; ++j) {
            const uint32_t dsub = s->dim_alloc[j];
            const float* q = vec + s->dim_off[j];
            const float* tab = codebook + s->cb_off[j];
            double best = INFINITY;
            uint32_t best_i = 0;
            for (uint32_t i = 0; i < (1u << s->bits[j]); ++i) {
                const float* c = tab + (size_t)i * dsub;
                double acc = 0.0;
                for (uint32_t t = 0; t < dsub; ++t) {
                    double diff = (double)q[t] - (double)c[t];
                    acc += diff * diff;
                }
                if (acc < best) {
                    best = acc;
                    best_i = i;
                }
            }
            codes[v * s->m + j] = (uint8_t)best_i;
        }
    }
    return ORC_OK;
}

/* compute_tables, distance.hpp:35-58: fp32, serial over the slice dims */
int orc_compute_tables(const orc_spec* s, const float* codebook, const float* query, float* lut) {
    for (uint32_t j = 0; j < s->m; ++j) {
        const uint32_t dsub = s->dim_alloc[j];
        const float* q = query + s->dim_off[j];
        const float* tab = codebook + s->cb_off[j];
        float* out = lut + s->ent_off[j];
        for (uint32_t i = 0; i < (1u << s->bits[j]); ++i) {
            const float* c = tab + (size_t)i * dsub;
            float acc = 0.0f;
            for (uint32_t t = 0; t < dsub; ++t) {
                float d = q[t] - c[t];
                acc += d * d;
            }
            out[i] = acc;
        }
    }
    return ORC_OK;
}

/* min_of (distance.hpp:22-26) and min_total (:28-32): fp32 sum in table order */
float orc_min_total(const orc_spec* s, const float* lut, float* p_min) {
    float sum = 0.0f;
    for (uint32_t j = 0; j < s->m; ++j) {
        float m = INFINITY;
        const float* t = lut + s->ent_off[j];
        for (uint32_t i = 0; i < (1u << s->bits[j]); ++i) m = (t[i] < m) ? t[i] : m; /* std::min(m, v) */
        if (p_min) p_min[j] = m;
        sum += m;
    }
    return sum;
}

/* one code's subquantizer index, straight from the packed layout (scan_scalar.hpp:53-57) */
static inline uint32_t packed_index(const orc_spec* s, const uint8_t* packed, uint32_t rows, uint64_t pos, uint32_t r,
                                    uint32_t k) {
    const uint32_t wb = word_bytes(s);
    const uint8_t* blk = packed + (pos / s->block_len) * block_bytes(s, rows);
    uint32_t w = load_word(blk + ((uint64_t)r * s->block_len + pos % s->block_len) * wb, wb);
    return (w >> s->offsets[k]) & ((1u << s->widths[k]) - 1u);
}

/* collect_prefix_float, scan_scalar.hpp:96-122: first `limit` codes in list order, sum in table order */
uint64_t orc_prefix_float(const orc_spec* s, const uint8_t* packed, uint64_t count, const float* lut, uint64_t limit,
                          float* out) {
    uint64_t taken = 0;
    for (uint64_t pos = 0; pos < count && taken < limit; ++pos, ++taken) {
        float acc = 0.0f;
        for (uint32_t r = 0; r < s->groups; ++r)
            for (uint32_t k = 0; k < s->g; ++k) {
                uint32_t j = r * s->g + k;
                acc += lut[s->ent_off[j] + packed_index(s, packed, s->groups, pos, r, k)];
            }
        out[taken] = acc;
    }
    return taken;
}

static int cmp_float(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

/* calibrate_bounds, distance.hpp:74-83.  nth_element(r-1) == (r)-th order statistic. */
int orc_calibrate(const orc_spec* s, const float* lut, const float* prefix, uint64_t n_prefix, uint32_t r,
                  float* d_min, float* d_max) {
    if (r == 0) return fail(ORC_ERR_CALIBRATION, "calibrate_bounds: R must be at least 1");
    if (n_prefix < r) return fail(ORC_ERR_CALIBRATION, "calibrate_bounds: prefix is shorter than R");
    float* tmp = (float*)malloc(sizeof(float) * n_prefix);
    memcpy(tmp, prefix, sizeof(float) * n_prefix);
    qsort(tmp, n_prefix, sizeof(float), cmp_float);
    *d_max = tmp[r - 1];
    free(tmp);
    *d_min = orc_min_total(s, lut, NULL);
    return ORC_OK;
}

/* quantize_tables, distance.hpp:102-142 */
int orc_quantize(const orc_spec* s, const float* lut, float d_min, float d_max, uint32_t width, void* qlut,
                 float* p_min, float* delta_out, float* own_d_min) {
    if (width != 8 && width != 16) return fail(ORC_ERR_CONFIG, "quantize_tables: width must be 8 or 16");
    if (!(d_max >= d_min)) return fail(ORC_ERR_CALIBRATION, "quantize_tables: d_max < d_min");
    const uint32_t q_max = width == 8 ? 255u : 65535u;
    const float delta = (d_max - d_min) / (float)q_max;
    float pm[ORC_MAX_SUBS];
    const float own = orc_min_total(s, lut, pm);
    for (uint32_t j = 0; j < s->m; ++j) {
        const float pmin = pm[j];
        const float* t = lut + s->ent_off[j];
        for (uint32_t i = 0; i < (1u << s->bits[j]); ++i) {
            const float p = t[i];
            uint32_t q;
            if (delta <= 0.0f) q = (p == pmin) ? 0u : q_max;
            else if (p - pmin >= d_max - d_min) q = q_max;
            else {
                double b = floor(((double)p - pmin) / (double)delta);
                q = (b >= (double)q_max) ? q_max : (uint32_t)b;
            }
            if (width == 8) ((uint8_t*)qlut)[s->ent_off[j] + i] = (uint8_t)q;
            else ((uint16_t*)qlut)[s->ent_off[j] + i] = (uint16_t)q;
        }
        if (p_min) p_min[j] = pmin;
    }
    if (delta_out) *delta_out = delta;
    if (own_d_min) *own_d_min = own;
    return ORC_OK;
}

/* ------------------------------------------------------------------ heap -- */

/* CandidateHeap<uint32_t>, heap.hpp:16-71: bounded max-heap on lexicographic (dist, id). */
typedef struct {
    uint32_t dist, id;
} hent;
typedef struct {
    hent* e;
    uint32_t n, cap;
} heap_t;

static inline int ent_less(hent a, hent b) { return a.dist < b.dist || (a.dist == b.dist && a.id < b.id); }

static void heap_sift_up(heap_t* h, uint32_t i) {
    while (i > 0) {
        uint32_t p = (i - 1) / 2;
        if (!ent_less(h->e[p], h->e[i])) break;
        hent t = h->e[p];
        h->e[p] = h->e[i];
        h->e[i] = t;
        i = p;
    }
}
static void heap_sift_down(heap_t* h, uint32_t i) {
    for (;;) {
        uint32_t l = 2 * i + 1, r = l + 1, big = i;
        if (l < h->n && ent_less(h->e[big], h->e[l])) big = l;
        if (r < h->n && ent_less(h->e[big], h->e[r])) big = r;
        if (big == i) break;
        hent t = h->e[big];
        h->e[big] = h->e[i];
        h->e[i] = t;
        i = big;
    }
}
/* push, heap.hpp:40-51 */
static inline void heap_push(heap_t* h, uint32_t dist, uint32_t id) {
    if (h->n < h->cap) {
        h->e[h->n].dist = dist;
        h->e[h->n].id = id;
        heap_sift_up(h, h->n++);
        return;
    }
    hent top = h->e[0];
    if (dist > top.dist || (dist == top.dist && id >= top.id)) return;
    h->e[0].dist = dist;
    h->e[0].id = id;
    heap_sift_down(h, 0);
}
static int cmp_ent(const void* a, const void* b) {
    hent x = *(const hent*)a, y = *(const hent*)b;
    if (ent_less(x, y)) return -1;
    if (ent_less(y, x)) return 1;
    return 0;
}
/* sorted(), heap.hpp:61-65 */
static void heap_sort_out(heap_t* h) { qsort(h->e, h->n, sizeof(hent), cmp_ent); }

/* ------------------------------------------------------------------ scan -- */

static inline uint32_t qentry(const void* qlut, uint32_t width, uint32_t i) {
    return width == 8 ? ((const uint8_t*)qlut)[i] : ((const uint16_t*)qlut)[i];
}

/* scan_list_scalar_quantized, scan_scalar.hpp:34-64 */
static int scan_into_heap(const orc_spec* s, const uint8_t* packed, uint64_t count, uint32_t rows, const void* qlut,
                          uint32_t width, const uint32_t* ids, uint32_t base_id, uint32_t acc_init, heap_t* heap) {
    if (count != 0 && (uint64_t)rows * s->g != s->m)
        return fail(ORC_ERR_CONFIG, "scan: packed rows do not match the table count for this scheme");
    if (width != s->word_width) return fail(ORC_ERR_CONFIG, "scan: table width does not match the packing word width");
    const uint32_t q_max = width == 8 ? 255u : 65535u;
    const uint32_t init = acc_init < q_max ? acc_init : q_max;
    for (uint64_t pos = 0; pos < count; ++pos) {
        uint32_t acc = init;
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t k = 0; k < s->g; ++k) {
                uint32_t j = r * s->g + k;
                uint32_t v = acc + qentry(qlut, width, s->ent_off[j] + packed_index(s, packed, rows, pos, r, k));
                acc = v < q_max ? v : q_max; /* saturating_add, distance.hpp:144 */
            }
        uint32_t id = ids ? ids[pos] : base_id + (uint32_t)pos;
        heap_push(heap, acc, id);
    }
    return ORC_OK;
}

int orc_scan_quantized(const orc_spec* s, const uint8_t* packed, uint64_t count, uint32_t rows, const void* qlut,
                       uint32_t width, const uint32_t* ids, uint32_t base_id, uint32_t acc_init, uint32_t cap,
                       const uint32_t* heap_in_dist, const uint32_t* heap_in_id, uint32_t n_in, uint32_t* out_dist,
                       uint32_t* out_id, uint32_t* n_out, int family) {
    (void)family;
    if (cap == 0) return fail(ORC_ERR_CONFIG, "candidate heap capacity must be positive");
    heap_t h = {(hent*)malloc(sizeof(hent) * cap), 0, cap};
    for (uint32_t i = 0; i < n_in; ++i) heap_push(&h, heap_in_dist[i], heap_in_id[i]);
    int rc = scan_into_heap(s, packed, count, rows, qlut, width, ids, base_id, acc_init, &h);
    if (rc == ORC_OK) {
        heap_sort_out(&h);
        for (uint32_t i = 0; i < h.n; ++i) {
            out_dist[i] = h.e[i].dist;
            out_id[i] = h.e[i].id;
        }
        *n_out = h.n;
    }
    free(h.e);
    return rc;
}

int orc_adc_sums(const orc_spec* s, const uint8_t* packed, uint64_t count, const void* qlut, uint32_t width,
                 uint32_t acc_init, uint64_t first, uint64_t n, uint32_t* sums) {
    if (first + n > count) return fail(ORC_ERR_INPUT, "adc_sums: range exceeds list");
    const uint32_t q_max = width == 8 ? 255u : 65535u;
    const uint32_t init = acc_init < q_max ? acc_init : q_max;
    for (uint64_t pos = first; pos < first + n; ++pos) {
        uint32_t acc = init;
        for (uint32_t r = 0; r < s->groups; ++r)
            for (uint32_t k = 0; k < s->g; ++k) {
                uint32_t j = r * s->g + k;
                uint32_t v = acc + qentry(qlut, width, s->ent_off[j] + packed_index(s, packed, s->groups, pos, r, k));
                acc = v < q_max ? v : q_max;
            }
        sums[pos - first] = acc;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- search -- */

/* SearchParams::validate, index.hpp:27-31 */
static int validate_params(uint32_t probes, uint32_t r, uint32_t t) {
    if (r < 1) return fail(ORC_ERR_INPUT, "search: R must be at least 1");
    if (t < r) return fail(ORC_ERR_INPUT, "search: calibration prefix t must be at least R");
    if (probes < 1) return fail(ORC_ERR_INPUT, "search: probes must be at least 1");
    return ORC_OK;
}

/* FlatIndex::search for one query, index.hpp:110-145 */
/* detail::rerank_by_float, index.hpp:53-67: order the final set by (exact float ADC, id) */
typedef struct {
    float d;
    uint32_t id;
} fent;
static int cmp_fent(const void* a, const void* b) {
    fent x = *(const fent*)a, y = *(const fent*)b;
    if (x.d < y.d) return -1;
    if (x.d > y.d) return 1;
    return (x.id > y.id) - (x.id < y.id);
}
/* adc_scalar_float of the code at list position pos, distance.hpp:61-69 via FlatIndex::code_at (index.hpp:93-108) */
static float float_adc_at(const orc_spec* s, const uint8_t* packed, uint64_t pos, const float* lut) {
    float acc = 0.0f;
    for (uint32_t r = 0; r < s->groups; ++r)
        for (uint32_t k = 0; k < s->g; ++k) {
            uint32_t j = r * s->g + k;
            acc += lut[s->ent_off[j] + packed_index(s, packed, s->groups, pos, r, k)];
        }
    return acc;
}

static int flat_search_one(const orc_spec* s, const float* cb, const uint8_t* packed, uint64_t count,
                           const float* query, uint32_t r, uint32_t t, int rerank, uint32_t* out_ids, float* out_dists,
                           uint32_t* out_count, void* dbg_qlut, float* dbg_params) {
    *out_count = 0;
    if (count == 0) return ORC_OK;
    int rc = ORC_OK;
    float* lut = (float*)malloc(sizeof(float) * s->total_entries);
    const uint64_t tp = t < count ? t : count;
    float* prefix = (float*)malloc(sizeof(float) * (tp ? tp : 1));
    void* qlut = malloc((size_t)s->total_entries * 2);
    heap_t h = {(hent*)malloc(sizeof(hent) * r), 0, r};
    orc_compute_tables(s, cb, query, lut);
    uint64_t taken = orc_prefix_float(s, packed, count, lut, t, prefix);
    uint32_t r_eff = (uint32_t)(r < taken ? r : taken);
    float d_min, d_max, delta, own;
    rc = orc_calibrate(s, lut, prefix, taken, r_eff, &d_min, &d_max);
    if (rc == ORC_OK) rc = orc_quantize(s, lut, d_min, d_max, s->word_width, qlut, NULL, &delta, &own);
    if (rc == ORC_OK) rc = scan_into_heap(s, packed, count, s->groups, qlut, s->word_width, NULL, 0, 0, &h);
    if (rc == ORC_OK) {
        heap_sort_out(&h);
        for (uint32_t i = 0; i < h.n; ++i) {
            out_ids[i] = h.e[i].id;
            out_dists[i] = (float)h.e[i].dist * delta + own; /* unquantize, distance.hpp:158-161 */
        }
        *out_count = h.n;
        if (rerank) { /* FlatIndex::rerank_exact, index.hpp:148-152 (ids are list positions) */
            fent* fe = (fent*)malloc(sizeof(fent) * (h.n ? h.n : 1));
            for (uint32_t i = 0; i < h.n; ++i) {
                fe[i].id = out_ids[i];
                fe[i].d = float_adc_at(s, packed, out_ids[i], lut);
            }
            qsort(fe, h.n, sizeof(fent), cmp_fent);
            for (uint32_t i = 0; i < h.n; ++i) {
                out_ids[i] = fe[i].id;
                out_dists[i] = fe[i].d;
            }
            free(fe);
        }
        if (dbg_qlut) memcpy(dbg_qlut, qlut, (size_t)s->total_entries * (s->word_width / 8));
        if (dbg_params) {
            dbg_params[0] = d_min;
            dbg_params[1] = d_max;
            dbg_params[2] = delta;
            dbg_params[3] = own;
        }
    }
    free(h.e);
    free(qlut);
    free(prefix);
    free(lut);
    return rc;
}

typedef struct {
    /* shared */
    const orc_spec* s;
    const float* cb;
    const uint8_t* packed;
    uint64_t count;
    const float* queries;
    uint32_t nq, r, t;
    int rerank;
    const uint32_t* loc_cell; /* ivf locator: id -> cell, id -> position (index.hpp:366-375) */
    const uint32_t* loc_pos;
    uint32_t* out_ids;
    float* out_dists;
    uint32_t* out_counts;
    void* dbg_qlut;
    float* dbg_params;
    /* ivf */
    const float* coarse;
    uint32_t k_cells, probes;
    const uint64_t *list_byte_off, *list_id_off, *list_count;
    const uint32_t* ids;
    int is_ivf;
    /* pool: one query per claim, atomic counter (tools/pqscan_cli.cpp:141-166) */
    volatile uint32_t next;
    volatile int rc;
    char err[256];
} job_t;

static int ivf_search_one(const job_t* J, const float* query, uint32_t* out_ids, float* out_dists,
                          uint32_t* out_count);

static void* worker(void* arg) {
    job_t* J = (job_t*)arg;
    for (;;) {
        uint32_t q = __sync_fetch_and_add(&J->next, 1);
        if (q >= J->nq) break;
        const float* query = J->queries + (size_t)q * J->s->dims;
        int rc;
        if (J->is_ivf)
            rc = ivf_search_one(J, query, J->out_ids + (size_t)q * J->r, J->out_dists + (size_t)q * J->r,
                                J->out_counts + q);
        else
            rc = flat_search_one(J->s, J->cb, J->packed, J->count, query, J->r, J->t, J->rerank, J->out_ids + (size_t)q * J->r,
                                 J->out_dists + (size_t)q * J->r, J->out_counts + q,
                                 J->dbg_qlut ? (uint8_t*)J->dbg_qlut + (size_t)q * J->s->total_entries *
                                                                          (J->s->word_width / 8)
                                             : NULL,
                                 J->dbg_params ? J->dbg_params + (size_t)q * 4 : NULL);
        if (rc != ORC_OK && __sync_bool_compare_and_swap(&J->rc, 0, rc)) snprintf(J->err, sizeof J->err, "%s", g_err);
    }
    return NULL;
}

static int run_pool(job_t* J, int threads) {
    if (threads < 1) threads = 1;
    if ((uint32_t)threads > J->nq) threads = (int)(J->nq ? J->nq : 1);
    J->next = 0;
    J->rc = 0;
    if (threads == 1) {
        worker(J);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
        for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, J);
        for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    if (J->rc) return fail(J->rc, J->err);
    return ORC_OK;
}

int orc_flat_search(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count,
                    const float* queries, uint32_t nq, uint32_t r, uint32_t t, int family, int threads,
                    uint32_t* out_ids, float* out_dists, uint32_t* out_counts, void* dbg_qlut, float* dbg_params) {
    int rc = validate_params(1, r, t);
    if (rc) return rc;
    job_t J;
    memset(&J, 0, sizeof J);
    J.rerank = (family & 0x100) != 0; /* bit 8 of `family` = SearchParams::rerank */
    J.s = s;
    J.cb = codebook;
    J.packed = packed;
    J.count = count;
    J.queries = queries;
    J.nq = nq;
    J.r = r;
    J.t = t;
    J.out_ids = out_ids;
    J.out_dists = out_dists;
    J.out_counts = out_counts;
    J.dbg_qlut = dbg_qlut;
    J.dbg_params = dbg_params;
    return run_pool(&J, threads);
}

/* ------------------------------------------------------------------- IVF -- */

typedef struct {
    float d;
    uint32_t c;
} dc_t;
static int cmp_dc(const void* a, const void* b) {
    dc_t x = *(const dc_t*)a, y = *(const dc_t*)b;
    if (x.d < y.d) return -1;
    if (x.d > y.d) return 1;
    return (x.c > y.c) - (x.c < y.c);
}

/* probe_order, index.hpp:247-265: fp32 serial squared distance; ascending (dist, cell) */
int orc_probe_order(uint32_t dims, const float* coarse, uint32_t k_cells, const float* query, uint32_t a,
                    uint32_t* order) {
    if (a > k_cells) a = k_cells;
    dc_t* ds = (dc_t*)malloc(sizeof(dc_t) * (k_cells ? k_cells : 1));
    for (uint32_t c = 0; c < k_cells; ++c) {
        const float* ctr = coarse + (size_t)c * dims;
        float acc = 0.0f;
        for (uint32_t j = 0; j < dims; ++j) {
            float diff = query[j] - ctr[j];
            acc += diff * diff;
        }
        ds[c].d = acc;
        ds[c].c = c;
    }
    qsort(ds, k_cells, sizeof(dc_t), cmp_dc);
    for (uint32_t i = 0; i < a; ++i) order[i] = ds[i].c;
    free(ds);
    return ORC_OK;
}

/* IvfIndex::search for one query, index.hpp:276-341 */
static int ivf_search_one(const job_t* J, const float* query, uint32_t* out_ids, float* out_dists,
                          uint32_t* out_count) {
    const orc_spec* s = J->s;
    *out_count = 0;
    const uint32_t a = J->probes < J->k_cells ? J->probes : J->k_cells;
    const uint32_t E = s->total_entries;
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (a ? a : 1));
    float* tables = (float*)malloc(sizeof(float) * (size_t)E * (a ? a : 1));
    float* residual = (float*)malloc(sizeof(float) * s->dims);
    float* prefix = (float*)malloc(sizeof(float) * (J->t ? J->t : 1));
    void* qlut = malloc((size_t)E * 2);
    heap_t h = {(hent*)malloc(sizeof(hent) * J->r), 0, J->r};
    int rc = ORC_OK;

    orc_probe_order(s->dims, J->coarse, J->k_cells, query, a, order);
    /* residual tables for every probed cell, index.hpp:282-288 */
    for (uint32_t i = 0; i < a; ++i) {
        const float* ctr = J->coarse + (size_t)order[i] * s->dims;
        for (uint32_t j = 0; j < s->dims; ++j) residual[j] = query[j] - ctr[j];
        orc_compute_tables(s, J->cb, residual, tables + (size_t)i * E);
    }
    /* shared affine map, index.hpp:299-316 */
    float d_min_global = INFINITY;
    for (uint32_t i = 0; i < a; ++i) {
        float mt = orc_min_total(s, tables + (size_t)i * E, NULL);
        d_min_global = mt < d_min_global ? mt : d_min_global;
    }
    uint64_t np = 0;
    for (uint32_t i = 0; i < a && np < J->t; ++i) {
        uint32_t c = order[i];
        np += orc_prefix_float(s, J->packed + J->list_byte_off[c], J->list_count[c], tables + (size_t)i * E,
                               J->t - np, prefix + np);
    }
    if (np == 0) goto done; /* index.hpp:307 */
    {
        const uint32_t r_eff = (uint32_t)(J->r < np ? J->r : np);
        qsort(prefix, np, sizeof(float), cmp_float);
        const float d_max = prefix[r_eff - 1];
        const uint32_t q_max = s->word_width == 8 ? 255u : 65535u;
        const float delta = (d_max - d_min_global) / (float)q_max;
        for (uint32_t i = 0; i < a && rc == ORC_OK; ++i) {
            uint32_t c = order[i];
            if (J->list_count[c] == 0) continue;
            float own;
            rc = orc_quantize(s, tables + (size_t)i * E, d_min_global, d_max, s->word_width, qlut, NULL, NULL, &own);
            if (rc) break;
            uint32_t bias = 0; /* index.hpp:324-328: float math */
            if (delta > 0.0f) {
                float b = floorf((own - d_min_global) / delta);
                bias = b >= (float)q_max ? q_max : (uint32_t)b;
            }
            rc = scan_into_heap(s, J->packed + J->list_byte_off[c], J->list_count[c], s->groups, qlut, s->word_width,
                                J->ids + J->list_id_off[c], 0, bias, &h);
        }
        if (rc == ORC_OK) {
            heap_sort_out(&h);
            for (uint32_t i = 0; i < h.n; ++i) {
                out_ids[i] = h.e[i].id;
                out_dists[i] = (float)h.e[i].dist * delta + d_min_global; /* index.hpp:337 */
            }
            *out_count = h.n;
            if (J->rerank) { /* IvfIndex::rerank_exact, index.hpp:377-386 */
                fent* fe = (fent*)malloc(sizeof(fent) * (h.n ? h.n : 1));
                for (uint32_t i = 0; i < h.n; ++i) {
                    const uint32_t id = out_ids[i], cell = J->loc_cell[id];
                    uint32_t pi = 0;
                    while (pi < a && order[pi] != cell) ++pi;
                    fe[i].id = id;
                    fe[i].d = float_adc_at(s, J->packed + J->list_byte_off[cell], J->loc_pos[id], tables + (size_t)pi * E);
                }
                qsort(fe, h.n, sizeof(fent), cmp_fent);
                for (uint32_t i = 0; i < h.n; ++i) {
                    out_ids[i] = fe[i].id;
                    out_dists[i] = fe[i].d;
                }
                free(fe);
            }
        }
    }
done:
    free(h.e);
    free(qlut);
    free(prefix);
    free(residual);
    free(tables);
    free(order);
    return rc;
}

int orc_ivf_search(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                   const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                   const uint64_t* list_count, const uint32_t* ids, const float* queries, uint32_t nq,
                   uint32_t probes, uint32_t r, uint32_t t, int family, int threads, uint32_t* out_ids,
                   float* out_dists, uint32_t* out_counts) {
    int rc = validate_params(probes, r, t);
    if (rc) return rc;
    /* IvfIndex constructor (index.hpp:169-177, 366-375): every id must be < total; build the locator */
    uint64_t total = 0;
    for (uint32_t c = 0; c < k_cells; ++c) total += list_count[c];
    uint32_t* loc_cell = (uint32_t*)malloc(sizeof(uint32_t) * (total ? total : 1));
    uint32_t* loc_pos = (uint32_t*)malloc(sizeof(uint32_t) * (total ? total : 1));
    for (uint32_t c = 0; c < k_cells; ++c)
        for (uint64_t p = 0; p < list_count[c]; ++p) {
            uint32_t id = ids[list_id_off[c] + p];
            if (id >= total) {
                free(loc_cell);
                free(loc_pos);
                return fail(ORC_ERR_CORRUPTION, "ivf: vector id out of range");
            }
            loc_cell[id] = c;
            loc_pos[id] = (uint32_t)p;
        }
    job_t J;
    memset(&J, 0, sizeof J);
    J.rerank = (family & 0x100) != 0;
    J.loc_cell = loc_cell;
    J.loc_pos = loc_pos;
    J.s = s;
    J.cb = codebook;
    J.packed = packed;
    J.queries = queries;
    J.nq = nq;
    J.r = r;
    J.t = t;
    J.out_ids = out_ids;
    J.out_dists = out_dists;
    J.out_counts = out_counts;
    J.coarse = coarse;
    J.k_cells = k_cells;
    J.probes = probes;
    J.list_byte_off = list_byte_off;
    J.list_id_off = list_id_off;
    J.list_count = list_count;
    J.ids = ids;
    J.is_ivf = 1;
    rc = run_pool(&J, threads);
    free(loc_cell);
    free(loc_pos);
    return rc;
}

/* ---------------------------------------------------------- handle variants -- */

typedef struct {
    int is_ivf;
    orc_spec s;
    const float* cb;
    const uint8_t* packed;
    uint64_t count;
    const float* coarse;
    uint32_t k_cells;
    const uint64_t *lbo, *lio, *lc;
    const uint32_t* ids;
} handle_t;

void* orc_flat_create(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count) {
    handle_t* h = (handle_t*)calloc(1, sizeof *h);
    h->s = *s;
    h->cb = codebook;
    h->packed = packed;
    h->count = count;
    return h;
}
int orc_flat_search_h(void* hv, const float* queries, uint32_t nq, uint32_t r, uint32_t t, int family, int threads,
                      uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    handle_t* h = (handle_t*)hv;
    return orc_flat_search(&h->s, h->cb, h->packed, h->count, queries, nq, r, t, family, threads, out_ids, out_dists,
                           out_counts, NULL, NULL);
}
void orc_flat_destroy(void* h) { free(h); }

void* orc_ivf_create(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                     const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                     const uint64_t* list_count, const uint32_t* ids) {
    handle_t* h = (handle_t*)calloc(1, sizeof *h);
    h->is_ivf = 1;
    h->s = *s;
    h->cb = codebook;
    h->coarse = coarse;
    h->k_cells = k_cells;
    h->packed = packed;
    h->lbo = list_byte_off;
    h->lio = list_id_off;
    h->lc = list_count;
    h->ids = ids;
    return h;
}
int orc_ivf_search_h(void* hv, const float* queries, uint32_t nq, uint32_t probes, uint32_t r, uint32_t t, int family,
                     int threads, uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    handle_t* h = (handle_t*)hv;
    return orc_ivf_search(&h->s, h->cb, h->coarse, h->k_cells, h->packed, h->lbo, h->lio, h->lc, h->ids, queries, nq,
                          probes, r, t, family, threads, out_ids, out_dists, out_counts);
}
void orc_ivf_destroy(void* h) { free(h); }

/* -------------------------------------------------- IVF list construction -- */

int orc_ivf_assign_encode(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                          const float* vectors, uint64_t n, uint32_t* assign, uint8_t* codes) {
    if (k_cells == 0) return fail(ORC_ERR_TRAINING, "ivf: no coarse centroids");
    float* resid = (float*)malloc(sizeof(float) * s->dims);
    for (uint64_t v = 0; v < n; ++v) {
        const float* x = vectors + v * s->dims;
        double best = INFINITY; /* kmeans.hpp:178-190: final assignment, ties go to the lowest centroid index */
        uint32_t best_c = 0;
        for (uint32_t c = 0; c < k_cells; ++c) {
            const float* ctr = coarse + (size_t)c * s->dims;
            double acc = 0.0; /* detail::sq_dist, kmeans.hpp:41-48 */
            for (uint32_t j = 0; j < s->dims; ++j) {
                double d = (double)x[j] - (double)ctr[j];
                acc += d * d;
            }
            if (acc < best) {
                best = acc;
                best_c = c;
            }
        }
        assign[v] = best_c;
        const float* ctr = coarse + (size_t)best_c * s->dims;
        for (uint32_t j = 0; j < s->dims; ++j) resid[j] = x[j] - ctr[j]; /* index.hpp:200 */
        orc_encode(s, codebook, resid, 1, codes + v * s->m);
    }
    free(resid);
    return ORC_OK;
}
