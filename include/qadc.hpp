// qadc.hpp -- C++ adapter that drops the B200 path behind the reference's own interfaces.
//
// Header-only; needs the reference headers on the include path (pqscan/pqscan.hpp) and links
// libqadc_b200.so (C ABI, include/qadc.h).  It is the binding a maintainer of the reference
// would add:
//
//   qadc::gpu_scan_list          a pqscan::QuantizedScanFn (simd/kernels.hpp:49-50): same signature,
//                                same heap semantics as scan_list_scalar_quantized (scan_scalar.hpp:34-64)
//   qadc::GpuFlatIndex           FlatIndex::search (index.hpp:110-145) + a batched search
//   qadc::GpuIvfIndex            IvfIndex::search  (index.hpp:276-341) + a batched search
//
// Status codes of the C ABI are rethrown as the matching pqscan exception (errors.hpp:9-46).
#pragma once

#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "pqscan/pqscan.hpp"
#include "qadc.h"

namespace qadc {

inline void rethrow(int rc) {
    if (rc == QADC_OK) return;
    const std::string msg = qadc_last_error();
    switch (rc) {
    case QADC_ERR_INVALID_SPEC: throw pqscan::invalid_spec_error(msg);
    case QADC_ERR_TRAINING: throw pqscan::training_error(msg);
    case QADC_ERR_INPUT: throw pqscan::input_error(msg);
    case QADC_ERR_CORRUPTION: throw pqscan::corruption_error(msg);
    case QADC_ERR_CONFIG: throw pqscan::config_error(msg);
    case QADC_ERR_CALIBRATION: throw pqscan::calibration_error(msg);
    case QADC_ERR_IO: throw pqscan::io_error(msg);
    default: throw pqscan::error("qadc (cuda): " + msg);
    }
}

// PqSpec (pqspec.hpp:66-113) + PackingScheme (layout.hpp:18-46) -> the flattened ABI struct
inline qadc_spec to_abi(const pqscan::PqSpec& spec) {
    qadc_spec s;
    std::memset(&s, 0, sizeof s);
    if (spec.num_subs() > QADC_MAX_SUBS || spec.group_size() > QADC_MAX_GROUP)
        throw pqscan::invalid_spec_error("spec exceeds the qadc ABI limits");
    const pqscan::PackingScheme sc = pqscan::PackingScheme::for_spec(spec);
    s.dims = spec.total_dims();
    s.m = static_cast<uint32_t>(spec.num_subs());
    s.g = static_cast<uint32_t>(spec.group_size());
    s.groups = static_cast<uint32_t>(spec.num_groups());
    s.word_width = spec.word_width();
    s.block_len = sc.block_len;
    s.exact = spec.exact_allocation();
    for (uint32_t i = 0; i < s.g; ++i) {
        s.widths[i] = sc.widths[i];
        s.offsets[i] = sc.offsets[i];
    }
    uint32_t e = 0, c = 0;
    for (uint32_t j = 0; j < s.m; ++j) {
        s.bits[j] = spec.bits(j);
        s.dim_alloc[j] = spec.dim_alloc(j);
        s.dim_off[j] = spec.dim_offset(j);
        s.ent_off[j] = e;
        e += spec.centroid_count(j);
        s.cb_off[j] = c;
        c += spec.centroid_count(j) * spec.dim_alloc(j);
    }
    s.total_entries = e;
    s.cb_floats = c;
    return s;
}

inline std::vector<float> flatten(const pqscan::Codebook& cb) {
    std::vector<float> out;
    for (size_t j = 0; j < cb.spec().num_subs(); ++j)
        out.insert(out.end(), cb.sub_table(j).begin(), cb.sub_table(j).end());
    return out;
}

// ---- QuantizedScanFn ---------------------------------------------------------------------
// Drop-in for the functions quantized_scan_fn() returns (simd/kernels.hpp:133-153).  The
// final heap is "the R smallest of (old entries U scanned candidates)" (heap.hpp:12-14), so the
// GPU returns the list's own top-R and those R entries are pushed into the caller's heap.
// The function-pointer type has no room for a device argument: the CUDA ordinal comes from
// gpu_scan_device() (per thread, default 0).  This is the CORRECTNESS seam (the reference's differential
// methodology runs through it): list and tables are uploaded on every call; throughput lives in the
// batched GpuFlatIndex / GpuIvfIndex below, which keep the database resident.
inline int& gpu_scan_device() {
    thread_local int device = 0;
    return device;
}
inline void gpu_scan_list(const pqscan::PackedList& list, const pqscan::PackingScheme& scheme,
                          const pqscan::QuantizedTables& qt, const uint32_t* ids, uint32_t base_id,
                          uint32_t acc_init, pqscan::CandidateHeap<uint32_t>& heap) {
    pqscan::detail::check_scan_config(list, scheme, qt.num_subs());
    if (qt.width != scheme.word_width)
        throw pqscan::config_error("scan: table width does not match the packing word width");
    if (list.count == 0) return;
    const uint32_t m = static_cast<uint32_t>(qt.num_subs());
    pqscan::SpecPattern pat{m, scheme.widths};
    const qadc_spec s = to_abi(pqscan::allocate_dims(16 * m, pat)); // dims are irrelevant to the scan (selftest.hpp:57)
    std::vector<uint8_t> q8;
    std::vector<uint16_t> q16;
    const void* qptr;
    if (qt.width == 8) {
        for (const auto& t : qt.t8) q8.insert(q8.end(), t.begin(), t.end());
        qptr = q8.data();
    } else {
        for (const auto& t : qt.t16) q16.insert(q16.end(), t.begin(), t.end());
        qptr = q16.data();
    }
    const uint32_t cap = static_cast<uint32_t>(heap.capacity());
    std::vector<uint32_t> od(cap), oi(cap);
    uint32_t n = 0;
    rethrow(qadc_scan_list(&s, list.data.data(), list.count, list.rows, qptr, qt.width, ids, base_id, acc_init, cap,
                           nullptr, nullptr, 0, od.data(), oi.data(), &n, gpu_scan_device()));
    for (uint32_t i = 0; i < n; ++i) heap.push(od[i], oi[i]);
}

inline pqscan::QuantizedScanFn gpu_scan_fn() { return &gpu_scan_list; }

namespace detail {
inline std::vector<pqscan::SearchResult> split(uint32_t nq, uint32_t r, const std::vector<uint32_t>& ids,
                                               const std::vector<float>& dists, const std::vector<uint32_t>& counts) {
    std::vector<pqscan::SearchResult> out(nq);
    for (uint32_t q = 0; q < nq; ++q) {
        out[q].ids.assign(ids.begin() + size_t{q} * r, ids.begin() + size_t{q} * r + counts[q]);
        out[q].dists.assign(dists.begin() + size_t{q} * r, dists.begin() + size_t{q} * r + counts[q]);
        out[q].kernel = pqscan::KernelFamily::scalar_quantized; // results are the normative kernel's, bit for bit
        out[q].scalar_fallback = false;
    }
    return out;
}
inline qadc_search_params params_of(const pqscan::SearchParams& p) {
    p.validate();
    if (p.forced_kernel == pqscan::KernelFamily::scalar_float)
        throw pqscan::config_error("qadc: the float-table scan is not part of the GPU path");
    return qadc_search_params{p.probes, p.r, p.t, p.rerank ? QADC_FLAG_RERANK : 0u};
}
} // namespace detail

// ---- FlatIndex ---------------------------------------------------------------------------
class GpuFlatIndex {
public:
    explicit GpuFlatIndex(const pqscan::FlatIndex& ref, int device = 0) : dims_(ref.codebook().spec().total_dims()) {
        const qadc_spec s = to_abi(ref.codebook().spec());
        const std::vector<float> cb = flatten(ref.codebook());
        rethrow(qadc_flat_open(&s, cb.data(), ref.list().data.data(), ref.list().count, 0, nullptr, 0, 0, device, &h_));
    }
    // the same index sharded over ndev GPUs of this process (devices = nullptr: ordinals 0..ndev-1): contiguous
    // block-aligned shards, replicated calibration head, one NCCL all_gather + merge per batch
    GpuFlatIndex(const pqscan::FlatIndex& ref, int ndev, const int* devices) : dims_(ref.codebook().spec().total_dims()) {
        const qadc_spec s = to_abi(ref.codebook().spec());
        const std::vector<float> cb = flatten(ref.codebook());
        rethrow(qadc_flat_open_sharded(&s, cb.data(), ref.list().data.data(), ref.list().count, ndev, devices, &m_));
    }
    GpuFlatIndex(const GpuFlatIndex&) = delete;
    GpuFlatIndex& operator=(const GpuFlatIndex&) = delete;
    ~GpuFlatIndex() {
        qadc_close(h_);
        qadc_multi_close(m_);
    }

    pqscan::SearchResult search(std::span<const float> query, const pqscan::SearchParams& params) const {
        if (query.size() != dims_) throw pqscan::input_error("search: query has wrong dimension");
        return search_batch(query, 1, params)[0];
    }
    std::vector<pqscan::SearchResult> search_batch(std::span<const float> queries, uint32_t nq,
                                                   const pqscan::SearchParams& params) const {
        if (queries.size() != size_t{nq} * dims_) throw pqscan::input_error("search: query has wrong dimension");
        const qadc_search_params p = detail::params_of(params);
        std::vector<uint32_t> ids(size_t{nq} * p.r), counts(nq);
        std::vector<float> dists(size_t{nq} * p.r);
        if (m_) rethrow(qadc_multi_search_batch(m_, queries.data(), nq, &p, ids.data(), dists.data(), counts.data()));
        else rethrow(qadc_search_batch(h_, queries.data(), nq, &p, ids.data(), dists.data(), counts.data()));
        return detail::split(nq, p.r, ids, dists, counts);
    }

private:
    qadc_index* h_ = nullptr;
    qadc_multi* m_ = nullptr;
    uint32_t dims_;
};

// ---- IvfIndex ----------------------------------------------------------------------------
class GpuIvfIndex {
public:
    explicit GpuIvfIndex(const pqscan::IvfIndex& ref, int device = 0) : dims_(ref.dims()), cells_(ref.cells()) {
        open(ref, device, 0, nullptr);
    }
    // every list split over `ndev` GPUs of this process (devices = nullptr: ordinals 0..ndev-1): qadc_ivf_open_sharded
    GpuIvfIndex(const pqscan::IvfIndex& ref, int ndev, const int* devices) : dims_(ref.dims()), cells_(ref.cells()) {
        open(ref, 0, ndev, devices);
    }
    GpuIvfIndex(const GpuIvfIndex&) = delete;
    GpuIvfIndex& operator=(const GpuIvfIndex&) = delete;
    ~GpuIvfIndex() {
        qadc_close(h_);
        qadc_multi_close(m_);
    }

    pqscan::SearchResult search(std::span<const float> query, const pqscan::SearchParams& params) const {
        if (query.size() != dims_) throw pqscan::input_error("search: query has wrong dimension");
        return search_batch(query, 1, params)[0];
    }
    std::vector<pqscan::SearchResult> search_batch(std::span<const float> queries, uint32_t nq,
                                                   const pqscan::SearchParams& params) const {
        if (queries.size() != size_t{nq} * dims_) throw pqscan::input_error("search: query has wrong dimension");
        const qadc_search_params p = detail::params_of(params);
        std::vector<uint32_t> ids(size_t{nq} * p.r), counts(nq);
        std::vector<float> dists(size_t{nq} * p.r);
        if (m_) rethrow(qadc_multi_search_batch(m_, queries.data(), nq, &p, ids.data(), dists.data(), counts.data()));
        else rethrow(qadc_search_batch(h_, queries.data(), nq, &p, ids.data(), dists.data(), counts.data()));
        return detail::split(nq, p.r, ids, dists, counts);
    }
    std::vector<uint32_t> probe_order(std::span<const float> query, uint32_t a) const {
        if (query.size() != dims_) throw pqscan::input_error("probe_order: query has wrong dimension");
        if (!h_) throw pqscan::config_error("probe_order: not available on a sharded index");
        std::vector<uint32_t> order(std::min(a, cells_)); // index.hpp:250
        rethrow(qadc_ivf_probe_order(h_, query.data(), 1, a, order.data()));
        return order;
    }

private:
    void open(const pqscan::IvfIndex& ref, int device, int ndev, const int* devices) {
        const qadc_spec s = to_abi(ref.codebook().spec());
        const std::vector<float> cb = flatten(ref.codebook());
        std::vector<uint8_t> packed;
        std::vector<uint32_t> ids;
        std::vector<uint64_t> boff, ioff, cnt;
        for (uint32_t c = 0; c < ref.cells(); ++c) {
            boff.push_back(packed.size());
            ioff.push_back(ids.size());
            cnt.push_back(ref.lists()[c].count);
            packed.insert(packed.end(), ref.lists()[c].data.begin(), ref.lists()[c].data.end());
            ids.insert(ids.end(), ref.list_ids()[c].begin(), ref.list_ids()[c].end());
        }
        if (ndev > 0)
            rethrow(qadc_ivf_open_sharded(&s, cb.data(), ref.coarse_centroids().data(), ref.cells(), packed.data(), boff.data(),
                                          ioff.data(), cnt.data(), ids.data(), ndev, devices, &m_));
        else
            rethrow(qadc_ivf_open(&s, cb.data(), ref.coarse_centroids().data(), ref.cells(), packed.data(), boff.data(),
                                  ioff.data(), cnt.data(), ids.data(), nullptr, nullptr, nullptr, nullptr, device, &h_));
    }
    qadc_index* h_ = nullptr;
    qadc_multi* m_ = nullptr;
    uint32_t dims_, cells_;
};

} // namespace qadc
