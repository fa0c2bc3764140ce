// ref_shim.cpp -- exports the oracle C API (qadc_oracle.h) by CALLING the
// unmodified reference headers (/root/reference/proj/include/pqscan).  TEST
// INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ when the
// reference tree is present; no reference source is copied into this repo.
//
// It is used (1) to pin oracle/qadc_oracle.c (the plain-C restatement),
// (2) to generate tests/golden fixtures (oracle/make_golden.py) and
// (3) as the CPU baseline ("kind": "reference") in bench.py.
//
// Build: g++ -std=c++20 -O2 -march=native -ffp-contract=off -I<reference>/proj/include

#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pqscan/pqscan.hpp"
#include "qadc_oracle.h"

using namespace pqscan;

static thread_local std::string g_err;

extern "C" const char* orc_impl_name(void) { return "reference"; }
extern "C" const char* orc_last_error(void) { return g_err.c_str(); }

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return ORC_OK;
    } catch (const invalid_spec_error& e) {
        g_err = e.what();
        return ORC_ERR_INVALID_SPEC;
    } catch (const training_error& e) {
        g_err = e.what();
        return ORC_ERR_TRAINING;
    } catch (const input_error& e) {
        g_err = e.what();
        return ORC_ERR_INPUT;
    } catch (const corruption_error& e) {
        g_err = e.what();
        return ORC_ERR_CORRUPTION;
    } catch (const config_error& e) {
        g_err = e.what();
        return ORC_ERR_CONFIG;
    } catch (const calibration_error& e) {
        g_err = e.what();
        return ORC_ERR_CALIBRATION;
    } catch (const io_error& e) {
        g_err = e.what();
        return ORC_ERR_IO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

SpecPattern pattern_of(const orc_spec* s) {
    SpecPattern p;
    p.m = s->m;
    p.widths.assign(s->widths, s->widths + s->g);
    return p;
}
PqSpec spec_of(const orc_spec* s) { return allocate_dims(s->dims, pattern_of(s)); }

Codebook codebook_of(const orc_spec* s, const float* cb) {
    PqSpec spec = spec_of(s);
    std::vector<std::vector<float>> tables(spec.num_subs());
    for (size_t j = 0; j < spec.num_subs(); ++j) {
        size_t n = size_t{spec.centroid_count(j)} * spec.dim_alloc(j);
        tables[j].assign(cb + s->cb_off[j], cb + s->cb_off[j] + n);
    }
    return Codebook(spec, std::move(tables));
}

PackedList list_of(const orc_spec* s, const uint8_t* packed, uint64_t count, uint32_t rows) {
    PackedList l;
    l.count = count;
    l.rows = count ? rows : 0;
    if (count) {
        PackingScheme sc = PackingScheme::for_spec(spec_of(s));
        size_t bytes = l.block_count(sc) * l.block_bytes(sc);
        l.data.assign(packed, packed + bytes);
    }
    return l;
}

DistanceTables tables_of(const orc_spec* s, const float* lut) {
    DistanceTables dt;
    dt.tables.resize(s->m);
    for (uint32_t j = 0; j < s->m; ++j) dt.tables[j].assign(lut + s->ent_off[j], lut + s->ent_off[j] + (1u << s->bits[j]));
    return dt;
}

QuantizedTables qtables_of(const orc_spec* s, const void* qlut, uint32_t width) {
    QuantizedTables qt;
    qt.width = width;
    qt.delta = 1.0f;
    qt.d_min = 0.0f;
    qt.p_min.assign(s->m, 0.0f);
    if (width == 8) {
        qt.t8.resize(s->m);
        const uint8_t* q = static_cast<const uint8_t*>(qlut);
        for (uint32_t j = 0; j < s->m; ++j) qt.t8[j].assign(q + s->ent_off[j], q + s->ent_off[j] + (1u << s->bits[j]));
    } else {
        qt.t16.resize(s->m);
        const uint16_t* q = static_cast<const uint16_t*>(qlut);
        for (uint32_t j = 0; j < s->m; ++j)
            qt.t16[j].assign(q + s->ent_off[j], q + s->ent_off[j] + (1u << s->bits[j]));
    }
    return qt;
}

void flatten_q(const orc_spec* s, const QuantizedTables& qt, void* out) {
    for (uint32_t j = 0; j < s->m; ++j)
        for (uint32_t i = 0; i < (1u << s->bits[j]); ++i) {
            if (qt.width == 8) static_cast<uint8_t*>(out)[s->ent_off[j] + i] = qt.t8[j][i];
            else static_cast<uint16_t*>(out)[s->ent_off[j] + i] = qt.t16[j][i];
        }
}

std::optional<KernelFamily> family_of(const PqSpec& spec, int family) {
    if ((family & 0xFF) == 0) return KernelFamily::scalar_quantized;
    return std::nullopt; // auto: natural vector family when the host has it
}
bool rerank_of(int family) { return (family & 0x100) != 0; } // bit 8 of `family` = SearchParams::rerank

template <class F>
void parallel_queries(uint32_t nq, int threads, F&& per_query) {
    // one query per claim, atomic counter: tools/pqscan_cli.cpp:141-166
    if (threads < 1) threads = 1;
    std::atomic<uint32_t> next{0};
    auto work = [&] {
        for (;;) {
            uint32_t q = next.fetch_add(1);
            if (q >= nq) break;
            per_query(q);
        }
    };
    if (threads == 1) {
        work();
        return;
    }
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(work);
    for (auto& t : pool) t.join();
}

} // namespace

extern "C" {

int orc_spec_parse(uint32_t dims, const char* text, orc_spec* out) {
    return guarded([&] {
        std::memset(out, 0, sizeof *out);
        SpecPattern pat = parse_spec_string(text);
        PqSpec spec = allocate_dims(dims, pat);
        if (spec.num_subs() > ORC_MAX_SUBS || spec.group_size() > ORC_MAX_GROUP)
            throw invalid_spec_error("spec too large for the oracle ABI");
        PackingScheme sc = PackingScheme::for_spec(spec);
        out->dims = spec.total_dims();
        out->m = static_cast<uint32_t>(spec.num_subs());
        out->g = static_cast<uint32_t>(spec.group_size());
        out->groups = static_cast<uint32_t>(spec.num_groups());
        out->word_width = spec.word_width();
        out->block_len = sc.block_len;
        out->exact = spec.exact_allocation();
        uint32_t eoff = 0, coff = 0;
        for (uint32_t i = 0; i < out->g; ++i) {
            out->widths[i] = sc.widths[i];
            out->offsets[i] = sc.offsets[i];
        }
        for (uint32_t j = 0; j < out->m; ++j) {
            out->bits[j] = spec.bits(j);
            out->dim_alloc[j] = spec.dim_alloc(j);
            out->dim_off[j] = spec.dim_offset(j);
            out->ent_off[j] = eoff;
            eoff += spec.centroid_count(j);
            out->cb_off[j] = coff;
            coff += spec.centroid_count(j) * spec.dim_alloc(j);
        }
        out->total_entries = eoff;
        out->cb_floats = coff;
    });
}

uint64_t orc_packed_bytes(const orc_spec* s, uint64_t n) {
    PackingScheme sc = PackingScheme::for_spec(spec_of(s));
    PackedList l;
    l.count = n;
    l.rows = s->groups;
    return l.block_count(sc) * l.block_bytes(sc);
}

int orc_pack_list(const orc_spec* s, const uint8_t* codes, uint64_t n, uint8_t* packed) {
    return guarded([&] {
        PackingScheme sc = PackingScheme::for_spec(spec_of(s));
        std::vector<Code> cs(n);
        for (uint64_t i = 0; i < n; ++i) cs[i].assign(codes + i * s->m, codes + (i + 1) * s->m);
        PackedList l = pack_list(cs, sc);
        std::memcpy(packed, l.data.data(), l.data.size());
    });
}

int orc_unpack_list(const orc_spec* s, const uint8_t* packed, uint64_t n, uint8_t* codes) {
    return guarded([&] {
        PackingScheme sc = PackingScheme::for_spec(spec_of(s));
        PackedList l = list_of(s, packed, n, s->groups);
        auto cs = unpack_list(l, sc);
        for (uint64_t i = 0; i < n; ++i) std::memcpy(codes + i * s->m, cs[i].data(), s->m);
    });
}

int orc_encode(const orc_spec* s, const float* codebook, const float* vectors, uint64_t n, uint8_t* codes) {
    return guarded([&] {
        Codebook cb = codebook_of(s, codebook);
        for (uint64_t i = 0; i < n; ++i) {
            Code c = encode({vectors + i * s->dims, s->dims}, cb);
            std::memcpy(codes + i * s->m, c.data(), s->m);
        }
    });
}

int orc_compute_tables(const orc_spec* s, const float* codebook, const float* query, float* lut) {
    return guarded([&] {
        Codebook cb = codebook_of(s, codebook);
        DistanceTables dt = compute_tables({query, s->dims}, cb);
        for (uint32_t j = 0; j < s->m; ++j)
            std::memcpy(lut + s->ent_off[j], dt.tables[j].data(), dt.tables[j].size() * sizeof(float));
    });
}

float orc_min_total(const orc_spec* s, const float* lut, float* p_min) {
    DistanceTables dt = tables_of(s, lut);
    if (p_min)
        for (uint32_t j = 0; j < s->m; ++j) p_min[j] = dt.min_of(j);
    return dt.min_total();
}

uint64_t orc_prefix_float(const orc_spec* s, const uint8_t* packed, uint64_t count, const float* lut, uint64_t limit,
                          float* out) {
    PackingScheme sc = PackingScheme::for_spec(spec_of(s));
    PackedList l = list_of(s, packed, count, s->groups);
    DistanceTables dt = tables_of(s, lut);
    std::vector<float> v;
    size_t taken = collect_prefix_float(l, sc, dt, limit, v);
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return taken;
}

int orc_calibrate(const orc_spec* s, const float* lut, const float* prefix, uint64_t n_prefix, uint32_t r,
                  float* d_min, float* d_max) {
    return guarded([&] {
        DistanceTables dt = tables_of(s, lut);
        auto [a, b] = calibrate_bounds(dt, {prefix, n_prefix}, r);
        *d_min = a;
        *d_max = b;
    });
}

int orc_quantize(const orc_spec* s, const float* lut, float d_min, float d_max, uint32_t width, void* qlut,
                 float* p_min, float* delta, float* own_d_min) {
    return guarded([&] {
        DistanceTables dt = tables_of(s, lut);
        QuantizedTables qt = quantize_tables(dt, d_min, d_max, width);
        flatten_q(s, qt, qlut);
        if (p_min) std::memcpy(p_min, qt.p_min.data(), s->m * sizeof(float));
        if (delta) *delta = qt.delta;
        if (own_d_min) *own_d_min = qt.d_min;
    });
}

int orc_scan_quantized(const orc_spec* s, const uint8_t* packed, uint64_t count, uint32_t rows, const void* qlut,
                       uint32_t width, const uint32_t* ids, uint32_t base_id, uint32_t acc_init, uint32_t cap,
                       const uint32_t* heap_in_dist, const uint32_t* heap_in_id, uint32_t n_in, uint32_t* out_dist,
                       uint32_t* out_id, uint32_t* n_out, int family) {
    return guarded([&] {
        PqSpec spec = spec_of(s);
        PackingScheme sc = PackingScheme::for_spec(spec);
        PackedList l = list_of(s, packed, count, rows);
        QuantizedTables qt = qtables_of(s, qlut, width);
        CandidateHeap<uint32_t> heap(cap);
        for (uint32_t i = 0; i < n_in; ++i) heap.push(heap_in_dist[i], heap_in_id[i]);
        KernelFamily fam = select_kernel(spec, SimdCaps::available(), family_of(spec, family));
        QuantizedScanFn fn = quantized_scan_fn(spec, fam);
        if (!fn) throw config_error("no quantized scan routine for this family");
        fn(l, sc, qt, ids, base_id, acc_init, heap);
        auto sorted = heap.sorted();
        for (size_t i = 0; i < sorted.size(); ++i) {
            out_dist[i] = sorted[i].dist;
            out_id[i] = sorted[i].id;
        }
        *n_out = static_cast<uint32_t>(sorted.size());
    });
}

int orc_adc_sums(const orc_spec* s, const uint8_t* packed, uint64_t count, const void* qlut, uint32_t width,
                 uint32_t acc_init, uint64_t first, uint64_t n, uint32_t* sums) {
    return guarded([&] {
        if (first + n > count) throw input_error("adc_sums: range exceeds list");
        PackingScheme sc = PackingScheme::for_spec(spec_of(s));
        PackedList l = list_of(s, packed, count, s->groups);
        QuantizedTables qt = qtables_of(s, qlut, width);
        auto codes = unpack_list(l, sc);
        for (uint64_t i = 0; i < n; ++i) sums[i] = adc_scalar_quantized(codes[first + i], qt, acc_init);
    });
}

int orc_flat_search(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count,
                    const float* queries, uint32_t nq, uint32_t r, uint32_t t, int family, int threads,
                    uint32_t* out_ids, float* out_dists, uint32_t* out_counts, void* dbg_qlut, float* dbg_params) {
    return guarded([&] {
        PqSpec spec = spec_of(s);
        FlatIndex index(codebook_of(s, codebook), list_of(s, packed, count, s->groups));
        SearchParams params;
        params.r = r;
        params.t = t;
        params.forced_kernel = family_of(spec, family);
        params.rerank = rerank_of(family);
        params.validate();
        std::atomic<int> failed{0};
        std::string err;
        parallel_queries(nq, threads, [&](uint32_t q) {
            try {
                std::span<const float> query{queries + size_t{q} * s->dims, s->dims};
                SearchResult res = index.search(query, params);
                out_counts[q] = static_cast<uint32_t>(res.ids.size());
                std::copy(res.ids.begin(), res.ids.end(), out_ids + size_t{q} * r);
                std::copy(res.dists.begin(), res.dists.end(), out_dists + size_t{q} * r);
                if ((dbg_qlut || dbg_params) && count) {
                    // the intermediate state search() derives, by the same calls (index.hpp:114-129)
                    DistanceTables dt = compute_tables(query, index.codebook());
                    std::vector<float> prefix;
                    collect_prefix_float(index.list(), index.scheme(), dt, t, prefix);
                    uint32_t r_eff = static_cast<uint32_t>(std::min<size_t>(r, prefix.size()));
                    auto [d_min, d_max] = calibrate_bounds(dt, prefix, r_eff);
                    QuantizedTables qt = quantize_tables(dt, d_min, d_max, index.scheme().word_width);
                    if (dbg_qlut)
                        flatten_q(s, qt, static_cast<uint8_t*>(dbg_qlut) + size_t{q} * s->total_entries * (qt.width / 8));
                    if (dbg_params) {
                        float* p = dbg_params + size_t{q} * 4;
                        p[0] = d_min;
                        p[1] = d_max;
                        p[2] = qt.delta;
                        p[3] = qt.d_min;
                    }
                }
            } catch (const std::exception& e) {
                if (!failed.exchange(1)) err = e.what();
            }
        });
        if (failed) throw calibration_error(err);
    });
}

int orc_probe_order(uint32_t dims, const float* coarse, uint32_t k_cells, const float* query, uint32_t a,
                    uint32_t* order) {
    return guarded([&] {
        // IvfIndex needs a codebook; probe_order only reads dims and the coarse centroids
        PqSpec spec = allocate_dims(dims, parse_spec_string("1x{8}"));
        std::vector<std::vector<float>> tables(1, std::vector<float>(size_t{256} * dims, 0.0f));
        std::vector<PackedList> lists(k_cells);
        std::vector<std::vector<uint32_t>> ids(k_cells);
        IvfIndex idx(Codebook(spec, std::move(tables)), std::vector<float>(coarse, coarse + size_t{k_cells} * dims),
                     std::move(lists), std::move(ids));
        auto o = idx.probe_order({query, dims}, a);
        std::copy(o.begin(), o.end(), order);
    });
}

int orc_ivf_search(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                   const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                   const uint64_t* list_count, const uint32_t* ids, const float* queries, uint32_t nq,
                   uint32_t probes, uint32_t r, uint32_t t, int family, int threads, uint32_t* out_ids,
                   float* out_dists, uint32_t* out_counts) {
    return guarded([&] {
        PqSpec spec = spec_of(s);
        std::vector<PackedList> lists(k_cells);
        std::vector<std::vector<uint32_t>> lids(k_cells);
        for (uint32_t c = 0; c < k_cells; ++c) {
            lists[c] = list_of(s, packed + list_byte_off[c], list_count[c], s->groups);
            lids[c].assign(ids + list_id_off[c], ids + list_id_off[c] + list_count[c]);
        }
        IvfIndex index(codebook_of(s, codebook), std::vector<float>(coarse, coarse + size_t{k_cells} * s->dims),
                       std::move(lists), std::move(lids));
        SearchParams params;
        params.probes = probes;
        params.r = r;
        params.t = t;
        params.forced_kernel = family_of(spec, family);
        params.rerank = rerank_of(family);
        params.validate();
        std::atomic<int> failed{0};
        std::string err;
        parallel_queries(nq, threads, [&](uint32_t q) {
            try {
                SearchResult res = index.search({queries + size_t{q} * s->dims, s->dims}, params);
                out_counts[q] = static_cast<uint32_t>(res.ids.size());
                std::copy(res.ids.begin(), res.ids.end(), out_ids + size_t{q} * r);
                std::copy(res.dists.begin(), res.dists.end(), out_dists + size_t{q} * r);
            } catch (const std::exception& e) {
                if (!failed.exchange(1)) err = e.what();
            }
        });
        if (failed) throw calibration_error(err);
    });
}

// ---- handle variants: build the reference index once, search many times ----

struct RefFlat {
    PqSpec spec;
    FlatIndex index;
    uint32_t dims;
};
struct RefIvf {
    PqSpec spec;
    IvfIndex index;
    uint32_t dims;
};

void* orc_flat_create(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count) {
    try {
        return new RefFlat{spec_of(s), FlatIndex(codebook_of(s, codebook), list_of(s, packed, count, s->groups)), s->dims};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int orc_flat_search_h(void* hv, const float* queries, uint32_t nq, uint32_t r, uint32_t t, int family, int threads,
                      uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return guarded([&] {
        RefFlat* h = static_cast<RefFlat*>(hv);
        SearchParams params;
        params.r = r;
        params.t = t;
        params.forced_kernel = family_of(h->spec, family);
        params.rerank = rerank_of(family);
        params.validate();
        std::atomic<int> failed{0};
        std::string err;
        parallel_queries(nq, threads, [&](uint32_t q) {
            try {
                SearchResult res = h->index.search({queries + size_t{q} * h->dims, h->dims}, params);
                out_counts[q] = static_cast<uint32_t>(res.ids.size());
                std::copy(res.ids.begin(), res.ids.end(), out_ids + size_t{q} * r);
                std::copy(res.dists.begin(), res.dists.end(), out_dists + size_t{q} * r);
            } catch (const std::exception& e) {
                if (!failed.exchange(1)) err = e.what();
            }
        });
        if (failed) throw calibration_error(err);
    });
}
void orc_flat_destroy(void* h) { delete static_cast<RefFlat*>(h); }

void* orc_ivf_create(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                     const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                     const uint64_t* list_count, const uint32_t* ids) {
    try {
        std::vector<PackedList> lists(k_cells);
        std::vector<std::vector<uint32_t>> lids(k_cells);
        for (uint32_t c = 0; c < k_cells; ++c) {
            lists[c] = list_of(s, packed + list_byte_off[c], list_count[c], s->groups);
            lids[c].assign(ids + list_id_off[c], ids + list_id_off[c] + list_count[c]);
        }
        return new RefIvf{spec_of(s),
                          IvfIndex(codebook_of(s, codebook), std::vector<float>(coarse, coarse + size_t{k_cells} * s->dims),
                                   std::move(lists), std::move(lids)),
                          s->dims};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int orc_ivf_search_h(void* hv, const float* queries, uint32_t nq, uint32_t probes, uint32_t r, uint32_t t, int family,
                     int threads, uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return guarded([&] {
        RefIvf* h = static_cast<RefIvf*>(hv);
        SearchParams params;
        params.probes = probes;
        params.r = r;
        params.t = t;
        params.forced_kernel = family_of(h->spec, family);
        params.rerank = rerank_of(family);
        params.validate();
        std::atomic<int> failed{0};
        std::string err;
        parallel_queries(nq, threads, [&](uint32_t q) {
            try {
                SearchResult res = h->index.search({queries + size_t{q} * h->dims, h->dims}, params);
                out_counts[q] = static_cast<uint32_t>(res.ids.size());
                std::copy(res.ids.begin(), res.ids.end(), out_ids + size_t{q} * r);
                std::copy(res.dists.begin(), res.dists.end(), out_dists + size_t{q} * r);
            } catch (const std::exception& e) {
                if (!failed.exchange(1)) err = e.what();
            }
        });
        if (failed) throw calibration_error(err);
    });
}
void orc_ivf_destroy(void* h) { delete static_cast<RefIvf*>(h); }

// ---- reference-only helpers (fixture generation; not part of the port) ----

// train_codebook (codebook.hpp:66-91) -> flat codebook of s->cb_floats floats
int ref_train_codebook(const orc_spec* s, const float* vectors, uint64_t n, uint32_t iters, uint64_t seed,
                       float* codebook_out) {
    return guarded([&] {
        PqSpec spec = spec_of(s);
        TrainConfig cfg;
        cfg.kmeans_iters = iters;
        cfg.seed = seed;
        Codebook cb = train_codebook({vectors, n * s->dims}, n, spec, cfg);
        for (uint32_t j = 0; j < s->m; ++j)
            std::memcpy(codebook_out + s->cb_off[j], cb.sub_table(j).data(), cb.sub_table(j).size() * sizeof(float));
    });
}

// kmeans (kmeans.hpp:54-192) -> centroids (k*dim) and assignment (n)
int ref_kmeans(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed,
               float* centroids_out, uint32_t* assignment_out) {
    return guarded([&] {
        KMeansConfig cfg;
        cfg.max_iters = iters;
        cfg.seed = seed;
        KMeansResult res = kmeans({points, n * dim}, n, dim, k, cfg);
        std::memcpy(centroids_out, res.centroids.data(), res.centroids.size() * sizeof(float));
        if (assignment_out) std::memcpy(assignment_out, res.assignment.data(), n * sizeof(uint32_t));
    });
}

// The data-dependent half of IvfIndex::build given trained centroids + codebook.  The reference only exposes it
// inside build(); the port's restatement is exported under the common name, and ref_ivf_build below runs the REAL
// build so that tests can feed its centroids/codebook back and demand byte-identical lists.
int orc_ivf_assign_encode(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells,
                          const float* vectors, uint64_t n, uint32_t* assign, uint8_t* codes) {
    return guarded([&] {
        Codebook cb = codebook_of(s, codebook);
        std::vector<float> residual(s->dims);
        for (uint64_t v = 0; v < n; ++v) {
            const float* x = vectors + v * s->dims;
            double best = std::numeric_limits<double>::infinity();
            uint32_t best_c = 0;
            for (uint32_t c = 0; c < k_cells; ++c) {
                double d = detail::sq_dist(x, coarse + size_t{c} * s->dims, s->dims); // kmeans.hpp:41-48
                if (d < best) {
                    best = d;
                    best_c = c;
                }
            }
            assign[v] = best_c;
            for (uint32_t j = 0; j < s->dims; ++j) residual[j] = x[j] - coarse[size_t{best_c} * s->dims + j];
            Code c = encode(residual, cb);
            std::memcpy(codes + v * s->m, c.data(), s->m);
        }
    });
}

// IvfIndex::build (index.hpp:179-230), the real thing, behind a handle with getters.
struct RefBuilt {
    IvfIndex index;
};
void* ref_ivf_build(const float* vectors, uint64_t n, uint32_t dims, const char* spec_text, uint32_t k_coarse,
                    uint32_t iters, uint64_t seed) {
    try {
        IvfBuildConfig cfg;
        cfg.k_coarse = k_coarse;
        cfg.train.kmeans_iters = iters;
        cfg.train.seed = seed;
        return new RefBuilt{IvfIndex::build({vectors, n * dims}, n, parse_spec_string(spec_text), cfg)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
// sizes: [0] codebook floats, [1] total packed bytes, [2] total ids
void ref_ivf_built_sizes(void* hv, uint64_t* sizes) {
    const IvfIndex& ix = static_cast<RefBuilt*>(hv)->index;
    uint64_t cbf = 0, pb = 0, ni = 0;
    for (size_t j = 0; j < ix.codebook().spec().num_subs(); ++j) cbf += ix.codebook().sub_table(j).size();
    for (const auto& l : ix.lists()) pb += l.data.size();
    for (const auto& v : ix.list_ids()) ni += v.size();
    sizes[0] = cbf;
    sizes[1] = pb;
    sizes[2] = ni;
}
void ref_ivf_built_get(void* hv, float* codebook, float* coarse, uint8_t* packed, uint64_t* byte_off, uint64_t* id_off,
                       uint64_t* counts, uint32_t* ids) {
    const IvfIndex& ix = static_cast<RefBuilt*>(hv)->index;
    size_t o = 0;
    for (size_t j = 0; j < ix.codebook().spec().num_subs(); ++j) {
        const auto& t = ix.codebook().sub_table(j);
        std::memcpy(codebook + o, t.data(), t.size() * 4);
        o += t.size();
    }
    std::memcpy(coarse, ix.coarse_centroids().data(), ix.coarse_centroids().size() * 4);
    uint64_t b = 0, i = 0;
    for (uint32_t c = 0; c < ix.cells(); ++c) {
        byte_off[c] = b;
        id_off[c] = i;
        counts[c] = ix.lists()[c].count;
        std::memcpy(packed + b, ix.lists()[c].data.data(), ix.lists()[c].data.size());
        std::memcpy(ids + i, ix.list_ids()[c].data(), ix.list_ids()[c].size() * 4);
        b += ix.lists()[c].data.size();
        i += ix.list_ids()[c].size();
    }
}
void ref_ivf_built_free(void* hv) { delete static_cast<RefBuilt*>(hv); }

// save_flat_index / save_ivf_index (io.hpp:276-307): container fixtures written BY the reference
int ref_save_flat(const orc_spec* s, const float* codebook, const uint8_t* packed, uint64_t count, const char* path) {
    return guarded([&] {
        FlatIndex index(codebook_of(s, codebook), list_of(s, packed, count, s->groups));
        io::save_flat_index(path, index);
    });
}

int ref_save_ivf(const orc_spec* s, const float* codebook, const float* coarse, uint32_t k_cells, const uint8_t* packed,
                 const uint64_t* list_byte_off, const uint64_t* list_id_off, const uint64_t* list_count,
                 const uint32_t* ids, const char* path) {
    return guarded([&] {
        std::vector<PackedList> lists(k_cells);
        std::vector<std::vector<uint32_t>> lids(k_cells);
        for (uint32_t c = 0; c < k_cells; ++c) {
            lists[c] = list_of(s, packed + list_byte_off[c], list_count[c], s->groups);
            lids[c].assign(ids + list_id_off[c], ids + list_id_off[c] + list_count[c]);
        }
        IvfIndex index(codebook_of(s, codebook), std::vector<float>(coarse, coarse + size_t{k_cells} * s->dims),
                       std::move(lists), std::move(lids));
        io::save_ivf_index(path, index);
    });
}

// which family select_kernel picks on this host for the spec (kernels.hpp:114-129)
const char* ref_auto_family(const orc_spec* s) {
    static thread_local std::string name;
    try {
        name = to_string(select_kernel(spec_of(s), SimdCaps::available()));
    } catch (...) {
        name = "?";
    }
    return name.c_str();
}

const char* ref_simd_caps(void) {
    static thread_local std::string d;
    d = SimdCaps::available().describe();
    return d.c_str();
}

} // extern "C"
