// api.cu -- the C ABI (include/qadc.h): index handles, search orchestration, error mapping.
//
// Host-side mirror of FlatIndex::search (index.hpp:110-145), IvfIndex::search
// (index.hpp:276-341) and the QuantizedScanFn plugin point (simd/kernels.hpp:49-50),
// batched over queries.  Everything that touches data runs in CUDA kernels of this
// library; there is no CPU fallback.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace qadc {

void parse_spec(uint32_t dims, const std::string& text, qadc_spec& out);
void validate_spec(const qadc_spec& s);
int open_index_file(const char* path, int device, qadc_index** out);
const char* variant_name(uint32_t v);

static thread_local std::string g_error;

template <class F>
static int guarded(F&& f) {
    try {
        g_launches = 0;
        f();
        return QADC_OK;
    } catch (const Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "out of host memory";
        return QADC_ERR_INPUT;
    } catch (const std::exception& e) {
        g_error = e.what();
        return QADC_ERR_CUDA;
    }
}

// the same status mapping for the other translation units' entry points (multi.cu)
int multi_guarded(const std::function<void()>& f) { return guarded(f); }

// Memory-safety evidence without compute-sanitizer (closed on this pool): with QADC_DEBUG_CANARY set, every device
// buffer of the library is allocated at EXACTLY the requested size between two 1 KiB guard zones filled with 0xA5, and
// the guards are verified whenever a buffer is released or regrown (qadc_debug_canary reports the totals).  An
// out-of-bounds write of any kernel next to any workspace, table image, code array or candidate list shows up there.
static bool canary_mode() {
    static const bool on = std::getenv("QADC_DEBUG_CANARY") != nullptr;
    return on;
}
static std::atomic<unsigned long long> g_canary_checked{0}, g_canary_failures{0};
static constexpr size_t CANARY_GUARD = 1024;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void verify_guards() {
        unsigned char host[2 * CANARY_GUARD];
        char* base = static_cast<char*>(p) - CANARY_GUARD;
        if (cudaMemcpy(host, base, CANARY_GUARD, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(host + CANARY_GUARD, static_cast<char*>(p) + cap, CANARY_GUARD, cudaMemcpyDeviceToHost) != cudaSuccess) {
            g_canary_failures += 1;
            return;
        }
        unsigned long long bad = 0;
        for (unsigned char b : host) bad += b != 0xA5;
        g_canary_checked += 1;
        g_canary_failures += bad;
    }
    void release() {
        if (p) {
            if (canary_mode()) {
                verify_guards();
                cudaFree(static_cast<char*>(p) - CANARY_GUARD);
            } else {
                cudaFree(p);
            }
        }
        p = nullptr;
        cap = 0;
    }
    void ensure(size_t bytes) {
        if (canary_mode() ? bytes == cap && p : bytes <= cap) return; // canary mode: exact size, guard right behind the last byte
        release();
        if (bytes == 0) return;
        if (canary_mode()) {
            char* base = nullptr;
            cudaError_t e = cudaMalloc(&base, bytes + 2 * CANARY_GUARD);
            if (e != cudaSuccess)
                throw Error(QADC_ERR_CUDA, "cudaMalloc(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
            cudaMemset(base, 0xA5, CANARY_GUARD);
            cudaMemset(base + CANARY_GUARD + bytes, 0xA5, CANARY_GUARD);
            p = base + CANARY_GUARD;
            cap = bytes;
            return;
        }
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess)
            throw Error(QADC_ERR_CUDA, "cudaMalloc(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
        cap = bytes;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

static void set_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Error(QADC_ERR_CUDA, std::string("no usable CUDA device (this library has no CPU fallback): ") +
                                       (e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0"));
    if (device < 0 || device >= n) throw Error(QADC_ERR_INPUT, "device ordinal out of range");
    QADC_CUDA_CHECK(cudaSetDevice(device));
}

static void validate_params(const qadc_search_params& p, bool ivf) {
    // SearchParams::validate, index.hpp:27-31
    if (p.r < 1) throw Error(QADC_ERR_INPUT, "search: R must be at least 1");
    if (p.t < p.r) throw Error(QADC_ERR_INPUT, "search: calibration prefix t must be at least R");
    if (ivf && p.probes < 1) throw Error(QADC_ERR_INPUT, "search: probes must be at least 1");
    if (p.r > QADC_MAX_R) throw Error(QADC_ERR_CONFIG, "search: R exceeds QADC_MAX_R supported by the device top-R stage");
    if (p.t > QADC_MAX_T) throw Error(QADC_ERR_CONFIG, "search: calibration prefix t exceeds QADC_MAX_T");
}

// Per-query selection state on the device.
struct SelectBufs {
    DevBuf thr_key, cand, cand_count, top, ntop, overflow;
    uint32_t cap = 0, kpad = 0;
    void ensure(uint32_t nq, uint32_t r, uint32_t cap_) {
        cap = cap_;
        kpad = r;
        thr_key.ensure(size_t(nq) * 8);
        cand.ensure(size_t(nq) * cap * 8);
        cand_count.ensure(size_t(nq) * 4);
        top.ensure(size_t(nq) * kpad * 8);
        ntop.ensure(size_t(nq) * 4);
        overflow.ensure(size_t(nq) * 4);
    }
};

// Stage timing with CUDA events recorded on the launching stream (no extra syncs: the events are
// read after the call's own final synchronisation).  stage: 0 tables, 1 scan, 2 select.
struct StageTimer {
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, std::pair<size_t, size_t>>> spans; // stage -> (begin, end) event index
    size_t used = 0;
    ~StageTimer() {
        for (auto e : pool) cudaEventDestroy(e);
    }
    void reset() {
        used = 0;
        spans.clear();
        tags.clear();
    }
    size_t mark(cudaStream_t st) {
        if (used == pool.size()) {
            cudaEvent_t e;
            QADC_CUDA_CHECK(cudaEventCreate(&e));
            pool.push_back(e);
        }
        QADC_CUDA_CHECK(cudaEventRecord(pool[used], st));
        return used++;
    }
    std::vector<uint64_t> tags;
    void span(int stage, size_t b, size_t e, uint64_t tag = 0) {
        spans.push_back({stage, {b, e}});
        tags.push_back(tag);
    }
    void collect(float* ms /* [3] */) {
        const bool trace = std::getenv("QADC_TRACE") != nullptr;
        for (size_t i = 0; i < spans.size(); ++i) {
            auto& sp = spans[i];
            float t = 0.f;
            if (cudaEventElapsedTime(&t, pool[sp.second.first], pool[sp.second.second]) == cudaSuccess) ms[sp.first] += t;
            if (trace) fprintf(stderr, "[qadc trace] stage %d tag %llu: %.3f ms\n", sp.first, (unsigned long long)tags[i], t);
        }
    }
};

} // namespace qadc

using namespace qadc;

struct qadc_index {
    // The handle is immutable after open, but every call uses its workspaces and stream: concurrent calls on one
    // handle serialise here (the reference lets any number of threads call search on one index).
    std::recursive_mutex mu;
    int kind = 0; // 0 flat, 1 ivf
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    qadc_spec spec{};
    DevSpec ds{};
    DevBuf codebook, codebook_t, sub_of, codes, calib, ids, slot_pair;
    DevBuf coarse_bf16, coarse_norm, coarse_mean, q_bf16, probe_eps; // tensor-core probe prefilter (ivf_probe_tc.cu)
    double coarse_rmax = 0.0;
    uint32_t dpad = 0;
    bool probe_tc_ready = false;
    int probe_tc = 1; // option: 0 = always the exact FP32 probe kernels
    uint64_t count = 0, count_padded = 0;
    uint32_t base_id = 0;
    uint32_t calib_count = 0;
    // A shard calibrates on a replicated head of the WHOLE list (index.hpp:124-129).  When that head is shorter than
    // the whole list, a search with t beyond it would silently calibrate on fewer codes than the reference does:
    // such a t is a config error.  calib_limit = longest t the head can serve exactly (~0 = the head is complete).
    uint64_t calib_limit = ~0ull;
    // ivf
    uint32_t k_cells = 0;
    DevBuf coarse, coarse_t, list_code_off, list_count_dev, calib_code_off, calib_count_dev;
    bool own_heads = true; // calibration heads alias the lists themselves (unsharded index)
    DevBuf locator;        // ivf, unsharded: id -> device code position (IvfIndex::build_locator, index.hpp:366-375)
    std::vector<uint64_t> list_code_off_h, list_count_h;
    uint64_t total_codes = 0;
    uint32_t ivf_round0 = 4096; // list positions scanned in the first round (then x seg_growth per round)
    // ivf workspace
    DevBuf order, pmin, own_min, qparams, cell_npairs, pair_rank, pair_slot, tile_base, row_query, row_bias, cta_begin, round_begin;
    // options
    uint32_t cand_cap = 8192;
    uint32_t seg0 = 4096;
    uint32_t seg_growth = 8;
    uint32_t seg_growth_pct = 0; // experiment: non-integer growth of the flat schedule, in percent (0 = use seg_growth)
    bool seg_growth_set = false; // set_option("seg_growth") was called: the per-variant default below no longer applies
    int force_variant = -1;
    uint32_t tc_debug = 0; // timing experiments on the tensor-core scan (results are wrong when non-zero)
    // workspace
    SelectBufs sel;
    DevBuf qlut, tile_lut, luts, calib_out, map, status, jobs, queries, out_ids, out_dists, out_counts, counters, scratch;
    qadc_stats stats{};
    StageTimer timer;

    ~qadc_index() {
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace qadc {

static constexpr uint64_t CODE_PAD = 1024; // device code arrays are padded to this many codes

// nq = queries of the batch about to be scanned (0 = unknown / one list with one table set).
// The tensor-core scan (scan_tc.cu) works on 256-query tiles and wants long code streams: it takes over from the
// shared-memory kernel's 32-row tiles once a batch fills a good part of a tile and the list is long enough for its
// segments to amortise its tile loads (measured: C4 3.1x faster; C1 -- 1e6 codes x 1e3 queries, launch bound -- 2 %
// faster; a single query over 2e8 codes 2.2x slower: a 256-query tile for one query wastes the tensor core).
static ScanPlan plan_for(const qadc_index* h, bool allow_merged = true, uint32_t nq = 0) {
    int force = h->force_variant;
    if (force < 0) {
        if (const char* e = std::getenv("QADC_FORCE_VARIANT")) force = std::atoi(e); // tests: every entry point, one variant
    }
    if (force < 0 && allow_merged && h->kind == 0 && nq >= 96 && h->count >= (uint64_t(1) << 18)) {
        try {
            // dense (256-query tiles) or 2:4 sparse (240-query tiles; a tile step costs ~4/5 of a dense one -- C4 242 vs
            // 305 ms -- and its admission path is the cheaper one): whichever needs less tensor time for this batch (C1, 1000
            // queries: 5 sparse tiles 0.92 ms, 4 dense ones 1.10).  From 8 Mi codes and ten tiles on, the sparse form runs
            // on CTA pairs with two tiles per job (measured, 1e4 queries: 4e6 codes 11.46 vs 11.39 ms, 1.25e7 22.5 vs 23.0,
            // 2.5e7 36.6 vs 38.4, 5e7 62.5 vs 68.2, 2e8 204 vs 240; 2e7 codes x 2000 queries = 9 tiles: 7.26 vs 6.79)
            const uint64_t t_dense = (nq + 255) / 256, t_sparse = (nq + 239) / 240;
            const bool sparse = t_sparse * 4 <= t_dense * 5;
            const int v = !sparse ? int(VAR_TC8) : (h->count >= (8ull << 20) && t_sparse >= 10) ? int(VAR_TC8P) : int(VAR_TC8S);
            ScanPlan p = plan_scan(h->ds, h->device, v, true);
            p.filter_shift = h->tc_debug;
            return p;
        } catch (const Error&) { // not 16x{4,4}
        }
    }
    ScanPlan p = plan_scan(h->ds, h->device, force, allow_merged);
    if (is_tc8(p.variant)) p.filter_shift = h->tc_debug;
    return p;
}

// Geometric segment schedule: after n codes the R-th best of n bounds the admission
// rate of the next codes by R/n, so each segment admits O(R * growth) candidates.
// (growth in percent: 200 = every segment twice as long as the one before; lengths stay multiples of 256 codes)
static std::vector<uint64_t> segment_bounds(uint64_t count, uint64_t seg0, uint64_t growth, uint64_t growth_pct = 0) {
    std::vector<uint64_t> b{0};
    uint64_t len = std::max<uint64_t>(seg0, 256);
    const uint64_t pct = growth_pct ? std::max<uint64_t>(growth_pct, 110) : std::max<uint64_t>(growth, 2) * 100;
    while (b.back() < count) {
        uint64_t next = std::min(count, b.back() + len);
        if (count - next < len / 2) next = count; // do not leave a tiny tail segment
        b.push_back(next);
        len = (len * pct / 100 + 255) / 256 * 256;
    }
    return b;
}

// Jobs of one segment of a flat list: tile-major so that a CTA's contiguous slice of the
// job list mostly stays on one LUT tile.
static void flat_segment_jobs(std::vector<ScanJob>& jobs, uint64_t seg_begin, uint64_t seg_end, uint32_t nq,
                              uint32_t tq, uint32_t base_id, int grid) {
    const uint32_t tiles = (nq + tq - 1) / tq;
    const uint64_t n = seg_end - seg_begin;
    uint64_t chunk = (n * tiles + uint64_t(grid) * 16 - 1) / (uint64_t(grid) * 16);
    chunk = std::max<uint64_t>(256, (chunk + 255) / 256 * 256);
    chunk = std::min<uint64_t>(chunk, 1u << 22);
    for (uint32_t t = 0; t < tiles; ++t)
        for (uint64_t c = seg_begin; c < seg_end; c += chunk) {
            ScanJob j{};
            j.code_off = c;
            j.ids_off = c;
            j.n_codes = uint32_t(std::min(chunk, seg_end - c));
            j.id_base = base_id + uint32_t(c);
            j.row_begin = t * tq;
            j.n_rows = std::min(tq, nq - t * tq);
            jobs.push_back(j);
        }
}

struct RowSet {
    const void* qlut;          // device [rows][E]
    const void* tile_lut;      // device [tile][E][TQ] (tilepack.cu)
    const uint32_t* row_query; // device or nullptr
    const uint32_t* row_bias;  // device or nullptr
};

// Scan `count` codes for nq queries (rows == queries) segment by segment, tightening the
// per-query thresholds in between; leaves the unsorted top-r in h->sel.top / ntop.
// Returns false if some query overflowed its candidate buffer (caller retries with a
// larger cap).
static bool scan_select_flat(qadc_index* h, const ScanPlan& plan, const uint8_t* d_codes, uint64_t count,
                             uint32_t base_id, const RowSet& rows, uint32_t nq, uint32_t r, uint32_t cap,
                             bool keep_state, cudaStream_t st) {
    h->sel.ensure(nq, r, cap);
    if (!keep_state)
        launch_init_select(h->sel.thr_key.as<uint64_t>(), h->sel.cand_count.as<uint32_t>(), h->sel.ntop.as<uint32_t>(),
                           h->sel.overflow.as<uint32_t>(), nq, st);
    const int grid = h->num_sms;
    // dense exact top-r over the head: seeds every query's threshold before the streaming scan
    const uint64_t head = keep_state ? 0 : std::min<uint64_t>(count, h->seg0);
    if (head) {
        const size_t s0e = h->timer.mark(st);
        launch_seed_topk(h->ds, d_codes, uint32_t(head), base_id, nullptr, rows.qlut, rows.row_bias, nq, r,
                         h->sel.top.as<uint64_t>(), h->sel.ntop.as<uint32_t>(), h->sel.kpad,
                         h->sel.thr_key.as<uint64_t>(), st);
        h->timer.span(2, s0e, h->timer.mark(st));
    }
    // growth of the segment schedule: an admitted pair costs the tensor-core scan far more than the shared-memory
    // kernel (hit path per flagged column vs a ballot), so it prefers more, smaller segments -- fewer candidates per
    // query between two threshold updates (C4: x8 332 ms, x4 320, x3 316, x2 315 per step)
    // (small searches are launch-latency bound and take x4: C1, 1e6 codes x 1e3 queries, 0.84 vs 0.92 ms; 4e6 x 1e4: 9.77 vs 9.42)
    const uint32_t growth = (is_tc8(plan.variant) && !h->seg_growth_set) ? (uint64_t(nq) * count < 10000000000ull ? 4u : 2u) : h->seg_growth;
    std::vector<uint64_t> bounds = segment_bounds(count - head, uint64_t(h->seg0) * growth, growth, h->seg_growth_pct);
    for (auto& b : bounds) b += head;
    std::vector<ScanJob> jobs;
    std::vector<std::pair<size_t, size_t>> seg_jobs;
    for (size_t s = 0; s + 1 < bounds.size(); ++s) {
        const size_t first = jobs.size();
        flat_segment_jobs(jobs, bounds[s], bounds[s + 1], nq, plan.tq, base_id, grid);
        seg_jobs.emplace_back(first, jobs.size() - first);
    }
    h->jobs.ensure(jobs.size() * sizeof(ScanJob));
    if (!jobs.empty())
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->jobs.p, jobs.data(), jobs.size() * sizeof(ScanJob), cudaMemcpyHostToDevice, st));
    for (size_t si = 0; si < seg_jobs.size(); ++si) {
        const size_t first = seg_jobs[si].first, n = seg_jobs[si].second;
        ScanArgs a{};
        a.codes = d_codes;
        a.ids = nullptr;
        a.qlut = rows.qlut;
        a.tile_lut = rows.tile_lut;
        a.row_query = rows.row_query;
        a.row_bias = rows.row_bias;
        a.jobs = h->jobs.as<ScanJob>() + first;
        a.n_jobs = uint32_t(n);
        a.thr_key = h->sel.thr_key.as<uint64_t>();
        a.cand = h->sel.cand.as<uint64_t>();
        a.cand_count = h->sel.cand_count.as<uint32_t>();
        a.cap = cap;
        a.overflow = h->sel.overflow.as<uint32_t>();
        const size_t e0 = h->timer.mark(st);
        launch_scan(plan, h->ds, a, std::min<int>(grid, int(n)), st);
        const size_t e1 = h->timer.mark(st);
        launch_tighten(h->sel.top.as<uint64_t>(), h->sel.ntop.as<uint32_t>(), h->sel.kpad, h->sel.cand.as<uint64_t>(),
                       h->sel.cand_count.as<uint32_t>(), cap, h->sel.thr_key.as<uint64_t>(), nq, r, h->counters.as<unsigned long long>(), st);
        const size_t e2 = h->timer.mark(st);
        h->timer.span(1, e0, e1, bounds[si + 1] - bounds[si]);
        h->timer.span(2, e1, e2);
        h->stats.scan_launches += 1;
        h->stats.segments += 1;
    }
    h->stats.pairs_scanned += count * nq;
    // overflow check (one small D2H; the only host sync of a batch)
    std::vector<uint32_t> ov(nq);
    QADC_CUDA_CHECK(cudaMemcpyAsync(ov.data(), h->sel.overflow.p, size_t(nq) * 4, cudaMemcpyDeviceToHost, st));
    QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    for (uint32_t v : ov)
        if (v) return false;
    return true;
}

static void fill_empty_results(uint32_t nq, uint32_t r, uint32_t* d_ids, float* d_dists, uint32_t* d_counts,
                               uint64_t* d_keys, float* d_map, cudaStream_t st) {
    // empty database: every query returns an empty result (index.hpp:113)
    if (d_ids) QADC_CUDA_CHECK(cudaMemsetAsync(d_ids, 0xFF, size_t(nq) * r * 4, st));
    if (d_dists) {
        std::vector<float> inf(size_t(nq) * r, __builtin_inff());
        QADC_CUDA_CHECK(cudaMemcpyAsync(d_dists, inf.data(), inf.size() * 4, cudaMemcpyHostToDevice, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    if (d_counts) QADC_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, size_t(nq) * 4, st));
    if (d_keys) QADC_CUDA_CHECK(cudaMemsetAsync(d_keys, 0xFF, size_t(nq) * r * 8, st));
    if (d_map) QADC_CUDA_CHECK(cudaMemsetAsync(d_map, 0, size_t(nq) * 2 * 4, st));
}

static void check_status(qadc_index* h, cudaStream_t st) {
    int status = 0;
    unsigned long long admitted = 0;
    QADC_CUDA_CHECK(cudaMemcpyAsync(&status, h->status.p, 4, cudaMemcpyDeviceToHost, st));
    if (h->counters.p) QADC_CUDA_CHECK(cudaMemcpyAsync(&admitted, h->counters.p, 8, cudaMemcpyDeviceToHost, st));
    QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    h->stats.candidates = admitted;
    if (status == QADC_ERR_CALIBRATION) throw Error(QADC_ERR_CALIBRATION, "quantize_tables: d_max < d_min");
    if (status) throw Error(status, "device-side failure");
}

static void check_rerank_args(const qadc_index* h, const qadc_search_params& p, const uint32_t* d_ids,
                              const float* d_dists, const uint32_t* d_counts, const uint64_t* d_keys) {
    if (!(p.flags & QADC_FLAG_RERANK)) return;
    if (d_keys) throw Error(QADC_ERR_CONFIG, "rerank: re-ranking applies to a final result list, not to per-shard key lists");
    if (!d_ids || !d_dists || !d_counts) throw Error(QADC_ERR_INPUT, "rerank: ids, dists and counts outputs are required");
    if (h->kind == 0 && h->base_id != 0) throw Error(QADC_ERR_CONFIG, "rerank: not available on a database shard");
    if (h->kind == 1 && !h->locator.p) throw Error(QADC_ERR_CONFIG, "rerank: not available on an IVF shard");
}

static void flat_search_device(qadc_index* h, const float* d_queries, uint32_t nq, const qadc_search_params& p,
                               uint32_t* d_ids, float* d_dists, uint32_t* d_counts, uint64_t* d_keys, float* d_map,
                               cudaStream_t st) {
    validate_params(p, false);
    check_rerank_args(h, p, d_ids, d_dists, d_counts, d_keys);
    const bool rerank = (p.flags & QADC_FLAG_RERANK) != 0;
    h->stats = qadc_stats{};
    h->timer.reset();
    if (nq == 0) return;
    if (h->calib_count == 0) { // the whole list is empty
        fill_empty_results(nq, p.r, d_ids, d_dists, d_counts, d_keys, d_map, st);
        h->stats.kernel_launches = g_launches;
        return;
    }
    if (uint64_t(p.t) > h->calib_limit)
        throw Error(QADC_ERR_CONFIG, "search: t = " + std::to_string(p.t) + " exceeds the replicated calibration head (" +
                                         std::to_string(h->calib_limit) + " codes of a longer list): open the shard with a longer head");
    const ScanPlan plan = plan_for(h, true, nq);
    h->stats.scan_variant = plan.variant;
    h->stats.query_tile = plan.tq;
    const DevSpec& ds = h->ds;
    const size_t wb = ds.word_width / 8;
    h->status.ensure(4);
    h->counters.ensure(16);
    QADC_CUDA_CHECK(cudaMemsetAsync(h->counters.p, 0, 16, st));
    QADC_CUDA_CHECK(cudaMemsetAsync(h->status.p, 0, 4, st));

    // query batches bound the candidate-buffer footprint
    uint32_t cap = h->cand_cap;
    const size_t budget = size_t(4) << 30;
    for (uint32_t q0 = 0; q0 < nq;) {
        const uint32_t qb_max = uint32_t(std::max<size_t>(1, budget / (size_t(cap) * 8)));
        const uint32_t nb = std::min<uint32_t>(nq - q0, std::min<uint32_t>(qb_max, 1u << 16));
        h->qlut.ensure(size_t(nb) * ds.E * wb);
        h->map.ensure(size_t(nb) * 2 * 4);
        LutArgs la{};
        la.codebook = h->codebook.as<float>();
        la.queries = d_queries + size_t(q0) * ds.dims;
        la.calib_codes = h->calib.as<uint8_t>();
        la.calib_count = h->calib_count;
        la.nq = nb;
        la.r = p.r;
        la.t = p.t;
        la.qluts = h->qlut.p;
        la.map = h->map.as<float>();
        la.status = h->status.as<int>();
        if (rerank) {
            h->luts.ensure(size_t(nb) * ds.E * 4);
            la.luts = h->luts.as<float>();
        }
        const size_t t0 = h->timer.mark(st);
        launch_flat_tables(ds, la, st);
        const uint32_t ntiles = (nb + plan.tq - 1) / plan.tq;
        h->tile_lut.ensure(size_t(ntiles) * tile_entries(plan.variant, ds.E) * plan.tq * tile_entry_bytes(plan.variant));
        launch_pack_tiles(plan.variant, plan.filter_shift, tile_pair_layout(plan.variant, ds), h->qlut.p, ds.word_width, ds.E, nb,
                          plan.tq, h->tile_lut.p, st);
        h->timer.span(0, t0, h->timer.mark(st));
        RowSet rows{h->qlut.p, h->tile_lut.p, nullptr, nullptr};
        const bool ok = scan_select_flat(h, plan, h->codes.as<uint8_t>(), h->count, h->base_id, rows, nb, p.r, cap,
                                         false, st);
        if (!ok) { // some query admitted more candidates than fit: redo this batch with a larger buffer
            if (uint64_t(cap) >= h->count + p.r) throw Error(QADC_ERR_CUDA, "internal: candidate overflow at full capacity");
            cap = uint32_t(std::min<uint64_t>(uint64_t(cap) * 8, h->count + p.r));
            h->stats.overflow_retries += 1;
            continue;
        }
        const size_t f0 = h->timer.mark(st);
        launch_finalize(h->sel.top.as<uint64_t>(), h->sel.ntop.as<uint32_t>(), h->sel.kpad, 1, nb, p.r, h->map.as<float>(),
                        p.flags, ds.qmax, d_ids ? d_ids + size_t(q0) * p.r : nullptr,
                        d_dists ? d_dists + size_t(q0) * p.r : nullptr, d_counts ? d_counts + q0 : nullptr,
                        d_keys ? d_keys + size_t(q0) * p.r : nullptr, st);
        if (rerank)
            launch_rerank(ds, h->codes.as<uint8_t>(), h->luts.as<float>(), h->base_id, nullptr, nullptr, nullptr, 0, 0, nb,
                          p.r, d_ids + size_t(q0) * p.r, d_dists + size_t(q0) * p.r, d_counts + q0, st);
        h->timer.span(2, f0, h->timer.mark(st));
        if (d_map)
            QADC_CUDA_CHECK(cudaMemcpyAsync(d_map + size_t(q0) * 2, h->map.p, size_t(nb) * 8, cudaMemcpyDeviceToDevice, st));
        q0 += nb;
        cap = h->cand_cap;
    }
    check_status(h, st);
    float ms[3] = {0.f, 0.f, 0.f};
    h->timer.collect(ms);
    h->stats.ms_lut = ms[0];
    h->stats.ms_scan = ms[1];
    h->stats.ms_select = ms[2];
    h->stats.kernel_launches = g_launches;
}

// ------------------------------------------------------------------ IVF search --

// probe order of nb queries into h->order; h->scratch holds the [nb][K] distance image
static void ivf_probe_order_device(qadc_index* h, const float* dq, uint32_t nb, uint32_t a, cudaStream_t st) {
    const DevSpec& ds = h->ds;
    const uint32_t K = h->k_cells;
    h->scratch.ensure(std::max(size_t(nb) * K * 4, ivf_probe_tc_scratch_bytes(nb, K))); // exact path: [nb][K] distances
    h->cta_begin.ensure((2 * size_t(nb) + 1) * 4); // reused as the probe-selection redo flags | list | count
    if (h->probe_tc && h->probe_tc_ready && ivf_probe_tc_supported(ds.dims, K, a)) {
        h->q_bf16.ensure(ivf_probe_tc_query_image_elems(nb, h->dpad) * 2);
        h->probe_eps.ensure(size_t(nb) * 8);
        launch_ivf_probe_tc(dq, h->coarse.as<float>(), h->coarse_bf16.as<uint16_t>(),
                            h->coarse_norm.as<float>(), h->coarse_mean.as<double>(), h->coarse_rmax, ds.dims, h->dpad, K,
                            nb, a, h->q_bf16.as<uint16_t>(), h->probe_eps.as<double>(),
                            h->scratch.as<float>(), h->cta_begin.as<uint32_t>(), h->order.as<uint32_t>(), st);
        // queries the prefilter could not decide (candidate overflow, non-finite input): exact kernels
        launch_ivf_probe(dq, h->coarse_t.as<float>(), ds.dims, K, nb, a, h->scratch.as<float>(),
                         h->cta_begin.as<uint32_t>(), h->order.as<uint32_t>(), st, true);
    } else {
        launch_ivf_probe(dq, h->coarse_t.as<float>(), ds.dims, K, nb, a, h->scratch.as<float>(),
                         h->cta_begin.as<uint32_t>(), h->order.as<uint32_t>(), st);
    }
}

static void ivf_search_device(qadc_index* h, const float* d_queries, uint32_t nq, const qadc_search_params& p,
                              uint32_t* d_ids, float* d_dists, uint32_t* d_counts, uint64_t* d_keys, float* d_map,
                              cudaStream_t st) {
    validate_params(p, true);
    check_rerank_args(h, p, d_ids, d_dists, d_counts, d_keys);
    const bool rerank = (p.flags & QADC_FLAG_RERANK) != 0;
    h->stats = qadc_stats{};
    h->timer.reset();
    if (nq == 0) return;
    const DevSpec& ds = h->ds;
    const uint32_t K = h->k_cells;
    const uint32_t a = std::min(p.probes, K); // index.hpp:250
    if (K == 0 || h->total_codes == 0) {
        fill_empty_results(nq, p.r, d_ids, d_dists, d_counts, d_keys, d_map, st);
        h->stats.kernel_launches = g_launches;
        return;
    }
    if (uint64_t(p.t) > h->calib_limit)
        throw Error(QADC_ERR_CONFIG, "search: t = " + std::to_string(p.t) + " exceeds the shortest truncated calibration head (" +
                                         std::to_string(h->calib_limit) + " codes): open the shard with longer list heads");
    ScanPlan plan = plan_for(h, false);
    const size_t wb = ds.word_width / 8;
    uint32_t tq = plan.tq;
    h->status.ensure(4);
    h->counters.ensure(16);
    QADC_CUDA_CHECK(cudaMemsetAsync(h->counters.p, 0, 16, st));
    QADC_CUDA_CHECK(cudaMemsetAsync(h->status.p, 0, 4, st));
    const int grid = h->num_sms;

    uint32_t cap = h->cand_cap;
    // query batches bound the float-table and candidate footprints (~2 GB each)
    const size_t pair_bytes = size_t(a) * ds.E * 4;
    for (uint32_t q0 = 0; q0 < nq;) {
        uint32_t nb = uint32_t(std::min<size_t>(nq - q0, std::max<size_t>(1, (size_t(2) << 30) / pair_bytes)));
        nb = uint32_t(std::min<size_t>(nb, std::max<size_t>(1, (size_t(4) << 30) / (size_t(cap) * 8))));
        const uint32_t n_pairs = nb * a;
        const float* dq = d_queries + size_t(q0) * ds.dims;
        h->order.ensure(size_t(n_pairs) * 4);
        h->luts.ensure(size_t(n_pairs) * ds.E * 4);
        h->pmin.ensure(size_t(n_pairs) * ds.m * 4);
        h->own_min.ensure(size_t(n_pairs) * 4);
        h->qparams.ensure(size_t(nb) * 16);
        h->map.ensure(size_t(nb) * 8);
        h->cell_npairs.ensure(size_t(K) * 4);
        h->pair_rank.ensure(size_t(n_pairs) * 4);
        h->pair_slot.ensure(size_t(n_pairs) * 4);
        h->tile_base.ensure(size_t(K) * 4);
        QADC_CUDA_CHECK(cudaMemsetAsync(h->cell_npairs.p, 0, size_t(K) * 4, st));

        const size_t t0 = h->timer.mark(st);
        ivf_probe_order_device(h, dq, nb, a, st);
        const size_t t1 = h->timer.mark(st);
        if (ivf_tables_tiled_supported(ds))
            launch_ivf_tables_tiled(ds, h->codebook_t.as<float>(), h->sub_of.as<uint8_t>(), dq, h->coarse.as<float>(),
                                    h->order.as<uint32_t>(), n_pairs, a, h->luts.as<float>(), h->pmin.as<float>(),
                                    h->own_min.as<float>(), st);
        else
            launch_ivf_tables(ds, h->codebook.as<float>(), dq, h->coarse.as<float>(), h->order.as<uint32_t>(), n_pairs, a,
                              h->luts.as<float>(), h->pmin.as<float>(), h->own_min.as<float>(), st);
        const size_t t2 = h->timer.mark(st);
        launch_ivf_calib(ds, h->own_heads ? h->codes.as<uint8_t>() : h->calib.as<uint8_t>(),
                         h->own_heads ? h->list_code_off.as<uint64_t>() : h->calib_code_off.as<uint64_t>(),
                         h->own_heads ? h->list_count_dev.as<uint64_t>() : h->calib_count_dev.as<uint64_t>(),
                         h->list_count_dev.as<uint64_t>(), h->order.as<uint32_t>(), nb, a, h->luts.as<float>(), h->own_min.as<float>(), p.r, p.t,
                         h->qparams.as<float>(), h->map.as<float>(), h->cell_npairs.as<uint32_t>(),
                         h->pair_rank.as<uint32_t>(), st);
        const size_t t3 = h->timer.mark(st);
        // rows are grouped by cell: the host lays the cells' tiles out back to back
        std::vector<uint32_t> npairs(K), tile_base(K);
        QADC_CUDA_CHECK(cudaMemcpyAsync(npairs.data(), h->cell_npairs.p, size_t(K) * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
        if (h->force_variant < 0 && plan.variant >= VAR_F16X4H && plan.variant <= VAR_F16X4H_C4) {
            // rows per cell are known now: pick the tile height (128 / 64 / 32 rows, i.e. 1 / 2 / 4 codes per
            // warp step) that minimises padded work = sum over cells of tiles * tile_rows * list_length
            // 32-row tiles: the duplicated-line layout when two tile buffers of it fit, else the dense one
            ScanVariant c32 = VAR_F16X4H_C4;
            double rate32 = 0.93;
            if (tile_pair_layout(VAR_F16X4H_C4, ds)) rate32 = 1.25; // pair-interleaved lines: conflict free, no copies
            else
            try {
                if (plan_scan(ds, h->device, int(VAR_F16X4H_C4D)).tile_bufs == 2) {
                    c32 = VAR_F16X4H_C4D;
                    rate32 = 1.25;
                }
            } catch (const Error&) {
            }
            // 16-row tiles (quad lines) exist for the named irregular specs; every tile is also one more pass over its
            // cell's codes and one more job, hence the larger per-tile constant below
            const bool have16 = tile_pair_layout(VAR_F16X4H_C16Q, ds) != 0;
            const ScanVariant cand[4] = {VAR_F16X4H, VAR_F16X4H_C2, c32, VAR_F16X4H_C16Q};
            const uint32_t rows[4] = {128, 64, 32, 16};
            const double per_pair[4] = {1.0 / 1.13, 1.0 / 1.30, 1.0 / rate32, 1.0 / 1.25}; // measured flat-scan rates (T pairs/s)
            // one pass over the cells for all tile heights (this runs on the host between two kernels)
            const int ncand = have16 ? 4 : 3;
            double cost[4] = {0.0, 0.0, 0.0, 0.0};
            for (uint32_t c = 0; c < K; ++c) {
                const uint32_t np_c = npairs[c];
                if (!np_c) continue;
                const double w = double(h->list_count_h[c]) + 2048.0;
                for (int v = 0; v < ncand; ++v) cost[v] += double((np_c + rows[v] - 1) & ~(rows[v] - 1)) * w;
            }
            double best = -1.0;
            int pick = int(plan.variant) - int(VAR_F16X4H);
            for (int v = 0; v < ncand; ++v) {
                try {
                    (void)plan_scan(ds, h->device, int(cand[v])); // does this tile height fit shared memory?
                } catch (const Error&) {
                    continue;
                }
                const double cst = cost[v] * per_pair[v];
                if (best < 0.0 || cst < best) {
                    best = cst;
                    pick = v;
                }
            }
            plan = plan_scan(ds, h->device, int(cand[pick]));
            tq = plan.tq;
        }
        h->stats.scan_variant = plan.variant;
        h->stats.query_tile = plan.tq;
        uint32_t ntiles = 0;
        for (uint32_t c = 0; c < K; ++c) {
            tile_base[c] = ntiles;
            ntiles += (npairs[c] + tq - 1) / tq;
        }
        const size_t nslots = size_t(ntiles) * tq;
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->tile_base.p, tile_base.data(), size_t(K) * 4, cudaMemcpyHostToDevice, st));
        h->qlut.ensure(std::max<size_t>(nslots * ds.E * wb, 16));
        h->row_query.ensure(std::max<size_t>(nslots * 4, 16));
        h->row_bias.ensure(std::max<size_t>(nslots * 4, 16));
        h->tile_lut.ensure(std::max<size_t>(nslots * ds.E * tile_entry_bytes(plan.variant), 16));
        h->slot_pair.ensure(std::max<size_t>(nslots * 4, 16));
        const size_t t4 = h->timer.mark(st);
        // quantize every tile's rows (padding rows: zero table, no query) and emit the scan's tile image
        launch_ivf_quantize_pack(plan.variant, plan.filter_shift, tile_pair_layout(plan.variant, ds), ds, h->order.as<uint32_t>(), n_pairs, a, h->luts.as<float>(),
                                 h->pmin.as<float>(), h->own_min.as<float>(), h->qparams.as<float>(),
                                 h->pair_rank.as<uint32_t>(), h->tile_base.as<uint32_t>(), tq, ntiles, h->qlut.p,
                                 h->tile_lut.p, h->row_query.as<uint32_t>(), h->row_bias.as<uint32_t>(),
                                 h->pair_slot.as<uint32_t>(), h->slot_pair.as<uint32_t>(), st);
        const size_t t5 = h->timer.mark(st);
        const size_t t6 = t5;
        h->timer.span(0, t0, t1, 101); // probe order
        h->timer.span(0, t1, t2, 102); // residual tables
        h->timer.span(0, t2, t3, 103); // calibration + grouping
        h->timer.span(0, t3, t4, 104); // host: tile layout, memsets
        h->timer.span(0, t4, t5, 105); // quantize + tile pack
        (void)t6;

        h->sel.ensure(nb, p.r, cap);
        launch_init_select(h->sel.thr_key.as<uint64_t>(), h->sel.cand_count.as<uint32_t>(), h->sel.ntop.as<uint32_t>(),
                           h->sel.overflow.as<uint32_t>(), nb, st);
        const size_t s0 = h->timer.mark(st);
        launch_ivf_seed(ds, h->codes.as<uint8_t>(), h->ids.as<uint32_t>(), h->list_code_off.as<uint64_t>(),
                        h->list_count_dev.as<uint64_t>(), h->order.as<uint32_t>(), nb, a, h->pair_slot.as<uint32_t>(),
                        h->qlut.p, h->row_bias.as<uint32_t>(), p.r, std::max<uint32_t>(std::min<uint32_t>(h->seg0, 2048), p.r), 
                        h->sel.thr_key.as<uint64_t>(), st);
        h->timer.span(2, s0, h->timer.mark(st));

        // rounds over list positions [lo, hi): the thresholds tighten between rounds.  All rounds' jobs are
        // built before the first launch and uploaded once (a pageable async copy would otherwise stall the host
        // behind the previous round's kernels).
        uint64_t longest = 0;
        for (uint32_t c = 0; c < K; ++c)
            if (npairs[c]) longest = std::max(longest, h->list_count_h[c]);
        struct Round {
            size_t job_first, n_jobs, begin_first;
            int grid;
        };
        std::vector<Round> rounds;
        std::vector<ScanJob> jobs;
        std::vector<uint32_t> begins;
        std::vector<uint64_t> cost;
        uint64_t pairs_scanned = 0;
        {
            uint64_t lo = 0, len = std::max<uint32_t>(h->ivf_round0, 64);
            const uint64_t max_chunk = 32768;
            while (lo < longest) {
                uint64_t hi = lo + len;
                if (longest - hi < len) hi = longest; // fold a short tail into this round
                if (hi >= longest) hi = ~0ull;
                const size_t first = jobs.size();
                cost.clear();
                for (uint32_t c = 0; c < K; ++c) {
                    const uint64_t cnt = h->list_count_h[c];
                    if (!npairs[c] || cnt <= lo) continue;
                    const uint64_t end = std::min(cnt, hi);
                    const uint32_t tiles = (npairs[c] + tq - 1) / tq;
                    for (uint32_t t = 0; t < tiles; ++t)
                        for (uint64_t bpos = lo; bpos < end; bpos += max_chunk) {
                            ScanJob j{};
                            j.code_off = h->list_code_off_h[c] + bpos;
                            j.ids_off = j.code_off;
                            j.n_codes = uint32_t(std::min(max_chunk, end - bpos));
                            j.id_base = 0;
                            j.row_begin = (tile_base[c] + t) * tq;
                            j.n_rows = std::min(tq, npairs[c] - t * tq);
                            jobs.push_back(j);
                            cost.push_back(uint64_t(j.n_codes) + 1024); // + the tile load
                            pairs_scanned += uint64_t(j.n_codes) * j.n_rows;
                        }
                }
                const size_t n = jobs.size() - first;
                if (n) {
                    // cost-balanced contiguous slices of the round's job list, one per CTA
                    const int g = int(std::min<size_t>(size_t(grid), n));
                    uint64_t total = 0;
                    for (uint64_t cst : cost) total += cst;
                    const size_t bfirst = begins.size();
                    begins.resize(bfirst + size_t(g) + 1, uint32_t(n));
                    uint64_t acc = 0;
                    int cta = 0;
                    begins[bfirst] = 0;
                    for (size_t j = 0; j < n; ++j) {
                        while (cta + 1 < g && acc >= total * uint64_t(cta + 1) / uint64_t(g)) begins[bfirst + size_t(++cta)] = uint32_t(j);
                        acc += cost[j];
                    }
                    while (cta + 1 < g) begins[bfirst + size_t(++cta)] = uint32_t(n);
                    begins[bfirst + size_t(g)] = uint32_t(n);
                    rounds.push_back(Round{first, n, bfirst, g});
                    if (std::getenv("QADC_TRACE")) {
                        uint64_t padded = 0, real = 0, mx = 0;
                        for (size_t j = first; j < jobs.size(); ++j) {
                            padded += uint64_t(jobs[j].n_codes) * tq;
                            real += uint64_t(jobs[j].n_codes) * jobs[j].n_rows;
                        }
                        for (int c = 0; c < g; ++c) {
                            uint64_t cs = 0;
                            for (uint32_t j = begins[bfirst + c]; j < begins[bfirst + c + 1]; ++j) cs += cost[j];
                            mx = std::max(mx, cs);
                        }
                        fprintf(stderr, "[qadc trace] round lo=%llu: %zu jobs, %.3e padded pairs, %.3e real, max CTA cost / mean = %.3f\n",
                                (unsigned long long)lo, n, double(padded), double(real), double(mx) * g / double(total));
                    }
                }
                if (hi == ~0ull) break;
                lo = hi;
                len *= std::max<uint32_t>(h->seg_growth, 2);
            }
        }
        h->jobs.ensure(std::max<size_t>(jobs.size() * sizeof(ScanJob), 16));
        h->round_begin.ensure(std::max<size_t>(begins.size() * 4, 16));
        if (!jobs.empty()) {
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->jobs.p, jobs.data(), jobs.size() * sizeof(ScanJob), cudaMemcpyHostToDevice, st));
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->round_begin.p, begins.data(), begins.size() * 4, cudaMemcpyHostToDevice, st));
        }
        for (const Round& rd : rounds) {
            ScanArgs sa{};
            sa.codes = h->codes.as<uint8_t>();
            sa.ids = h->ids.as<uint32_t>();
            sa.qlut = h->qlut.p;
            sa.tile_lut = h->tile_lut.p;
            sa.row_query = h->row_query.as<uint32_t>();
            sa.row_bias = h->row_bias.as<uint32_t>();
            sa.jobs = h->jobs.as<ScanJob>() + rd.job_first;
            sa.n_jobs = uint32_t(rd.n_jobs);
            sa.cta_begin = h->round_begin.as<uint32_t>() + rd.begin_first;
            sa.thr_key = h->sel.thr_key.as<uint64_t>();
            sa.cand = h->sel.cand.as<uint64_t>();
            sa.cand_count = h->sel.cand_count.as<uint32_t>();
            sa.cap = cap;
            sa.overflow = h->sel.overflow.as<uint32_t>();
            const size_t e0 = h->timer.mark(st);
            launch_scan(plan, ds, sa, rd.grid, st);
            const size_t e1 = h->timer.mark(st);
            launch_tighten(h->sel.top.as<uint64_t>(), h->sel.ntop.as<uint32_t>(), h->sel.kpad, h->sel.cand.as<uint64_t>(),
                           h->sel.cand_count.as<uint32_t>(), cap, h->sel.thr_key.as<uint64_t>(), nb, p.r, h->counters.as<unsigned long long>(), st);
            const size_t e2 = h->timer.mark(st);
            h->timer.span(1, e0, e1, rd.n_jobs);
            h->timer.span(2, e1, e2);
            h->stats.scan_launches += 1;
            h->stats.segments += 1;
        }
        std::vector<uint32_t> ov(nb);
        QADC_CUDA_CHECK(cudaMemcpyAsync(ov.data(), h->sel.overflow.p, size_t(nb) * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
        bool overflowed = false;
        for (uint32_t v : ov) overflowed |= v != 0;
        if (overflowed) {
            if (uint64_t(cap) >= h->total_codes + p.r) throw Error(QADC_ERR_CUDA, "internal: candidate overflow at full capacity");
            cap = uint32_t(std::min<uint64_t>(uint64_t(cap) * 8, h->total_codes + p.r));
            h->stats.overflow_retries += 1;
            continue;
        }
        h->stats.pairs_scanned += pairs_scanned;
        const size_t f0 = h->timer.mark(st);
        launch_finalize(h->sel.top.as<uint64_t>(), h->sel.ntop.as<uint32_t>(), h->sel.kpad, 1, nb, p.r, h->map.as<float>(),
                        p.flags, ds.qmax, d_ids ? d_ids + size_t(q0) * p.r : nullptr,
                        d_dists ? d_dists + size_t(q0) * p.r : nullptr, d_counts ? d_counts + q0 : nullptr,
                        d_keys ? d_keys + size_t(q0) * p.r : nullptr, st);
        if (rerank)
            launch_rerank(ds, h->codes.as<uint8_t>(), h->luts.as<float>(), 0, h->locator.as<uint32_t>(),
                          h->list_code_off.as<uint64_t>(), h->order.as<uint32_t>(), K, a, nb, p.r,
                          d_ids + size_t(q0) * p.r, d_dists + size_t(q0) * p.r, d_counts + q0, st);
        h->timer.span(2, f0, h->timer.mark(st));
        if (d_map)
            QADC_CUDA_CHECK(cudaMemcpyAsync(d_map + size_t(q0) * 2, h->map.p, size_t(nb) * 8, cudaMemcpyDeviceToDevice, st));
        q0 += nb;
        cap = h->cand_cap;
    }
    check_status(h, st);
    float ms[3] = {0.f, 0.f, 0.f};
    h->timer.collect(ms);
    h->stats.ms_lut = ms[0];
    h->stats.ms_scan = ms[1];
    h->stats.ms_select = ms[2];
    h->stats.kernel_launches = g_launches;
}

// Host -> device in plain async copies of at most 256 MiB: the source may be pageable or a file mapping
// (qadc_open_file), where one chunk is what the driver stages at a time anyway.
static void copy_h2d_chunked(void* dst, const void* src, uint64_t bytes, cudaStream_t st) {
    const uint64_t chunk = uint64_t(256) << 20;
    for (uint64_t off = 0; off < bytes; off += chunk)
        QADC_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                                        size_t(std::min(chunk, bytes - off)), cudaMemcpyHostToDevice, st));
}

static void upload_list(qadc_index* h, const qadc_spec& s, const DevSpec& ds, const uint8_t* packed, uint64_t count,
                        DevBuf& out, uint64_t& padded, cudaStream_t st) {
    padded = (count + CODE_PAD - 1) / CODE_PAD * CODE_PAD + CODE_PAD;
    out.ensure(size_t(padded) * ds.code_stride);
    if (count > 0xFFFFFFFFull) throw Error(QADC_ERR_INPUT, "list: more than 2^32 - 1 codes (ids are 32-bit)");
    const uint64_t bytes = qadc_packed_bytes(&s, count);
    DevBuf tmp;
    tmp.ensure(bytes);
    copy_h2d_chunked(tmp.p, packed, bytes, st);
    launch_relayout(s, ds, tmp.as<uint8_t>(), count, padded, out.as<uint8_t>(), st);
    QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    (void)h;
}

} // namespace qadc

// =============================================================== C ABI ======

extern "C" {

const char* qadc_version(void) { return "qadc-b200 0.1 (sm_100a)"; }
const char* qadc_last_error(void) { return g_error.c_str(); }
const char* qadc_variant_name(uint32_t v) { return variant_name(v); }

int qadc_device_count(void) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        g_error = cudaGetErrorString(e);
        cudaGetLastError();
        return -QADC_ERR_CUDA;
    }
    return n;
}

int qadc_spec_parse(uint32_t dims, const char* text, qadc_spec* out) {
    return guarded([&] {
        if (!text || !out) throw Error(QADC_ERR_INPUT, "null argument");
        parse_spec(dims, text, *out);
    });
}

uint64_t qadc_packed_bytes(const qadc_spec* s, uint64_t n) {
    if (n == 0) return 0;
    // ids are uint32 and the product must not wrap: counts from an untrusted container are checked by the caller
    // against this (UINT64_MAX = "does not fit")
    if (n > 0xFFFFFFFFull) return ~0ull;
    const uint64_t blocks = (n + s->block_len - 1) / s->block_len;
    return blocks * s->groups * s->block_len * (s->word_width / 8);
}

int qadc_flat_open(const qadc_spec* spec, const float* codebook, const uint8_t* packed, uint64_t count,
                   uint32_t base_id, const uint8_t* calib_packed, uint64_t calib_count, uint64_t global_count,
                   int device, qadc_index** out) {
    return guarded([&] {
        if (!spec || !codebook || !out || (count && !packed)) throw Error(QADC_ERR_INPUT, "null argument");
        validate_spec(*spec);
        set_device(device);
        std::unique_ptr<qadc_index> h(new qadc_index);
        h->kind = 0;
        h->device = device;
        h->spec = *spec;
        h->ds = make_dev_spec(*spec, spec->groups);
        if (h->ds.code_stride > 32) throw Error(QADC_ERR_CONFIG, "codes wider than 256 bits are not supported");
        QADC_CUDA_CHECK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
        QADC_CUDA_CHECK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        for (uint32_t i = 0; i < spec->cb_floats; ++i)
            if (!(codebook[i] - codebook[i] == 0.0f)) // codebook.hpp:45-46
                throw Error(QADC_ERR_CORRUPTION, "codebook: non-finite centroid component");
        h->codebook.ensure(size_t(spec->cb_floats) * 4);
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->codebook.p, codebook, size_t(spec->cb_floats) * 4, cudaMemcpyHostToDevice, h->stream));
        h->count = count;
        h->base_id = base_id;
        upload_list(h.get(), *spec, h->ds, packed, count, h->codes, h->count_padded, h->stream);
        if (calib_packed && calib_count) {
            uint64_t pad = 0;
            const uint64_t n = std::min<uint64_t>(calib_count, QADC_MAX_T);
            upload_list(h.get(), *spec, h->ds, calib_packed, n, h->calib, pad, h->stream);
            h->calib_count = uint32_t(n);
            // the head is complete only if the caller says the whole list is no longer than it
            if (global_count == 0 || global_count > calib_count) h->calib_limit = n;
        } else {
            const uint64_t n = std::min<uint64_t>(count, QADC_MAX_T);
            h->calib.ensure(std::max<size_t>(size_t(n) * h->ds.code_stride, 16));
            if (n) QADC_CUDA_CHECK(cudaMemcpyAsync(h->calib.p, h->codes.p, size_t(n) * h->ds.code_stride, cudaMemcpyDeviceToDevice, h->stream));
            h->calib_count = uint32_t(n);
        }
        QADC_CUDA_CHECK(cudaStreamSynchronize(h->stream));
        *out = h.release();
    });
}

int qadc_open_file(const char* path, int device, qadc_index** out) {
    int inner = QADC_OK;
    const int rc = guarded([&] {
        if (!path || !out) throw Error(QADC_ERR_INPUT, "null argument");
        inner = open_index_file(path, device, out); // parse errors throw; open errors come back as a status
    });
    return rc != QADC_OK ? rc : inner;
}

int qadc_index_info(const qadc_index* h, int* kind, qadc_spec* spec, uint64_t* count, uint32_t* cells) {
    if (!h) return QADC_ERR_INPUT;
    if (kind) *kind = h->kind;
    if (spec) *spec = h->spec;
    if (count) *count = h->kind == 0 ? h->count : h->total_codes;
    if (cells) *cells = h->k_cells;
    return QADC_OK;
}

void qadc_close(qadc_index* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    delete h;
}

int qadc_search_batch_device(qadc_index* h, const float* d_queries, uint32_t nq, const qadc_search_params* params,
                             uint32_t* d_out_ids, float* d_out_dists, uint32_t* d_out_counts,
                             uint64_t* d_out_keys, float* d_out_map, void* stream) {
    return guarded([&] {
        if (!h || !params || (nq && !d_queries)) throw Error(QADC_ERR_INPUT, "null argument");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        set_device(h->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        if (h->kind == 0)
            flat_search_device(h, d_queries, nq, *params, d_out_ids, d_out_dists, d_out_counts, d_out_keys, d_out_map, st);
        else
            ivf_search_device(h, d_queries, nq, *params, d_out_ids, d_out_dists, d_out_counts, d_out_keys, d_out_map, st);
    });
}

int qadc_search_batch(qadc_index* h, const float* queries, uint32_t nq, const qadc_search_params* params,
                      uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return guarded([&] {
        if (!h || !params || (nq && (!queries || !out_ids || !out_dists || !out_counts)))
            throw Error(QADC_ERR_INPUT, "null argument");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        validate_params(*params, h->kind == 1);
        set_device(h->device);
        cudaStream_t st = h->stream;
        const size_t nr = size_t(nq) * params->r;
        h->queries.ensure(size_t(nq) * h->ds.dims * 4);
        h->out_ids.ensure(nr * 4);
        h->out_dists.ensure(nr * 4);
        h->out_counts.ensure(size_t(nq) * 4);
        if (nq == 0) return;
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->queries.p, queries, size_t(nq) * h->ds.dims * 4, cudaMemcpyHostToDevice, st));
        const unsigned long long before = g_launches;
        if (h->kind == 0)
            flat_search_device(h, h->queries.as<float>(), nq, *params, h->out_ids.as<uint32_t>(), h->out_dists.as<float>(),
                               h->out_counts.as<uint32_t>(), nullptr, nullptr, st);
        else
            ivf_search_device(h, h->queries.as<float>(), nq, *params, h->out_ids.as<uint32_t>(), h->out_dists.as<float>(),
                              h->out_counts.as<uint32_t>(), nullptr, nullptr, st);
        (void)before;
        QADC_CUDA_CHECK(cudaMemcpyAsync(out_ids, h->out_ids.p, nr * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaMemcpyAsync(out_dists, h->out_dists.p, nr * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaMemcpyAsync(out_counts, h->out_counts.p, size_t(nq) * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int qadc_merge_topk_device(const uint64_t* d_keys, uint32_t nshards, uint32_t nq, uint32_t r, const float* d_map,
                           uint32_t flags, uint32_t* d_out_ids, float* d_out_dists, uint32_t* d_out_counts,
                           int device, void* stream) {
    return guarded([&] {
        if (!d_keys || nshards == 0 || r == 0) throw Error(QADC_ERR_INPUT, "merge: bad arguments");
        set_device(device);
        launch_finalize(d_keys, nullptr, r, nshards, nq, r, d_map, flags, 0xFFFFFFFFu, d_out_ids, d_out_dists,
                        d_out_counts, nullptr, static_cast<cudaStream_t>(stream));
    });
}

int qadc_flat_tables(qadc_index* h, const float* queries, uint32_t nq, const qadc_search_params* params,
                     float* luts, void* qluts, float* calib) {
    return guarded([&] {
        if (!h || h->kind != 0 || !params || !queries) throw Error(QADC_ERR_INPUT, "tables: bad arguments");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        validate_params(*params, false);
        set_device(h->device);
        if (nq == 0) return;
        if (h->calib_count == 0) throw Error(QADC_ERR_INPUT, "tables: empty index");
        cudaStream_t st = h->stream;
        const DevSpec& ds = h->ds;
        const size_t wb = ds.word_width / 8;
        h->queries.ensure(size_t(nq) * ds.dims * 4);
        h->qlut.ensure(size_t(nq) * ds.E * wb);
        h->luts.ensure(size_t(nq) * ds.E * 4);
        h->calib_out.ensure(size_t(nq) * 16);
        h->map.ensure(size_t(nq) * 8);
        h->status.ensure(4);
        QADC_CUDA_CHECK(cudaMemsetAsync(h->status.p, 0, 4, st));
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->queries.p, queries, size_t(nq) * ds.dims * 4, cudaMemcpyHostToDevice, st));
        LutArgs la{};
        la.codebook = h->codebook.as<float>();
        la.queries = h->queries.as<float>();
        la.calib_codes = h->calib.as<uint8_t>();
        la.calib_count = h->calib_count;
        la.nq = nq;
        la.r = params->r;
        la.t = params->t;
        la.luts = h->luts.as<float>();
        la.qluts = h->qlut.p;
        la.calib = h->calib_out.as<float>();
        la.map = h->map.as<float>();
        la.status = h->status.as<int>();
        launch_flat_tables(ds, la, st);
        if (luts) QADC_CUDA_CHECK(cudaMemcpyAsync(luts, h->luts.p, size_t(nq) * ds.E * 4, cudaMemcpyDeviceToHost, st));
        if (qluts) QADC_CUDA_CHECK(cudaMemcpyAsync(qluts, h->qlut.p, size_t(nq) * ds.E * wb, cudaMemcpyDeviceToHost, st));
        if (calib) QADC_CUDA_CHECK(cudaMemcpyAsync(calib, h->calib_out.p, size_t(nq) * 16, cudaMemcpyDeviceToHost, st));
        check_status(h, st);
    });
}

int qadc_flat_adc_sums(qadc_index* h, const void* qlut, uint32_t width, uint32_t acc_init, uint64_t first,
                       uint64_t n, uint32_t* sums) {
    return guarded([&] {
        if (!h || h->kind != 0 || !qlut || !sums) throw Error(QADC_ERR_INPUT, "adc_sums: bad arguments");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        if (width != h->ds.word_width) throw Error(QADC_ERR_CONFIG, "scan: table width does not match the packing word width");
        if (first + n > h->count) throw Error(QADC_ERR_INPUT, "adc_sums: range exceeds list");
        set_device(h->device);
        cudaStream_t st = h->stream;
        const size_t wb = width / 8;
        h->qlut.ensure(size_t(h->ds.E) * wb);
        h->scratch.ensure(size_t(n) * 4);
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->qlut.p, qlut, size_t(h->ds.E) * wb, cudaMemcpyHostToDevice, st));
        launch_adc_sums(h->ds, h->codes.as<uint8_t>(), h->qlut.p, acc_init, first, n, h->scratch.as<uint32_t>(), st);
        if (n) QADC_CUDA_CHECK(cudaMemcpyAsync(sums, h->scratch.p, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int qadc_flat_download_codes(qadc_index* h, uint64_t first, uint64_t n, uint8_t* codes_out) {
    return guarded([&] {
        if (!h || h->kind != 0 || !codes_out) throw Error(QADC_ERR_INPUT, "download_codes: bad arguments");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        if (first + n > h->count) throw Error(QADC_ERR_INPUT, "download_codes: range exceeds list");
        set_device(h->device);
        cudaStream_t st = h->stream;
        h->scratch.ensure(size_t(n) * h->ds.m);
        launch_unlayout(h->ds, h->codes.as<uint8_t>(), first, n, h->scratch.as<uint8_t>(), st);
        if (n) QADC_CUDA_CHECK(cudaMemcpyAsync(codes_out, h->scratch.p, size_t(n) * h->ds.m, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int qadc_scan_list(const qadc_spec* spec, const uint8_t* packed, uint64_t count, uint32_t rows, const void* qlut,
                   uint32_t width, const uint32_t* ids, uint32_t base_id, uint32_t acc_init, uint32_t cap,
                   const uint32_t* heap_in_dist, const uint32_t* heap_in_id, uint32_t n_in, uint32_t* out_dist,
                   uint32_t* out_id, uint32_t* n_out, int device) {
    return guarded([&] {
        if (!spec || !qlut || !out_dist || !out_id || !n_out) throw Error(QADC_ERR_INPUT, "scan_list: null argument");
        validate_spec(*spec);
        if (cap == 0) throw Error(QADC_ERR_CONFIG, "candidate heap capacity must be positive"); // heap.hpp:27-28
        // check_scan_config (scan_scalar.hpp:23-27) and the width check (:38-39)
        if (count != 0 && uint64_t(rows) * spec->g != spec->m)
            throw Error(QADC_ERR_CONFIG, "scan: packed rows do not match the table count for this scheme");
        if (width != spec->word_width) throw Error(QADC_ERR_CONFIG, "scan: table width does not match the packing word width");
        // n_in may exceed cap: the reference pushes every seed through the bounded heap (selftest.hpp:104-109)
        // CandidateHeap<uint32_t> takes any distance, but every distance this path produces is <= q_max <= 65535 and the
        // device select ranks 48 key bits (16 distance + 32 id): larger seed distances are refused, not mis-ranked
        for (uint32_t i = 0; i < n_in; ++i)
            if (heap_in_dist[i] > 0xFFFFu) throw Error(QADC_ERR_CONFIG, "scan_list: pre-seeded heap distance exceeds 65535");
        if (cap > QADC_MAX_R) throw Error(QADC_ERR_CONFIG, "scan_list: heap capacity exceeds QADC_MAX_R");
        set_device(device);
        qadc_index h;
        h.device = device;
        h.spec = *spec;
        h.ds = make_dev_spec(*spec, spec->groups);
        QADC_CUDA_CHECK(cudaDeviceGetAttribute(&h.num_sms, cudaDevAttrMultiProcessorCount, device));
        QADC_CUDA_CHECK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
        cudaStream_t st = h.stream;
        const DevSpec& ds = h.ds;
        h.count = count;
        upload_list(&h, *spec, ds, packed, count, h.codes, h.count_padded, st);
        const size_t wb = width / 8;
        h.qlut.ensure(size_t(ds.E) * wb);
        QADC_CUDA_CHECK(cudaMemcpyAsync(h.qlut.p, qlut, size_t(ds.E) * wb, cudaMemcpyHostToDevice, st));
        DevBuf bias;
        bias.ensure(4);
        QADC_CUDA_CHECK(cudaMemcpyAsync(bias.p, &acc_init, 4, cudaMemcpyHostToDevice, st));
        h.counters.ensure(16);
        // explicit ids: translate positions -> ids at the end (keys carry positions during the scan
        // would break the (distance,id) order), so give the kernel the id array directly
        if (ids && count) {
            h.ids.ensure(size_t(count) * 4);
            QADC_CUDA_CHECK(cudaMemcpyAsync(h.ids.p, ids, size_t(count) * 4, cudaMemcpyHostToDevice, st));
        }
        const ScanPlan plan = plan_for(&h);
        // pre-seeded heap entries are just earlier candidates (heap.hpp:12-14: order-independent)
        uint32_t buf_cap = std::max<uint32_t>(h.cand_cap, n_in + 16);
        for (;;) {
            h.sel.ensure(1, cap, buf_cap);
            launch_init_select(h.sel.thr_key.as<uint64_t>(), h.sel.cand_count.as<uint32_t>(), h.sel.ntop.as<uint32_t>(),
                               h.sel.overflow.as<uint32_t>(), 1, st);
            if (n_in) {
                std::vector<uint64_t> seed(n_in);
                for (uint32_t i = 0; i < n_in; ++i) seed[i] = make_key(heap_in_dist[i], heap_in_id[i]);
                QADC_CUDA_CHECK(cudaMemcpyAsync(h.sel.cand.p, seed.data(), size_t(n_in) * 8, cudaMemcpyHostToDevice, st));
                QADC_CUDA_CHECK(cudaMemcpyAsync(h.sel.cand_count.p, &n_in, 4, cudaMemcpyHostToDevice, st));
                launch_tighten(h.sel.top.as<uint64_t>(), h.sel.ntop.as<uint32_t>(), h.sel.kpad, h.sel.cand.as<uint64_t>(),
                               h.sel.cand_count.as<uint32_t>(), buf_cap, h.sel.thr_key.as<uint64_t>(), 1, cap, nullptr, st);
                QADC_CUDA_CHECK(cudaStreamSynchronize(st)); // seed vector goes out of scope
            }
            h.tile_lut.ensure(size_t(tile_entries(plan.variant, ds.E)) * plan.tq * tile_entry_bytes(plan.variant));
            launch_pack_tiles(plan.variant, plan.filter_shift, tile_pair_layout(plan.variant, ds), h.qlut.p, ds.word_width, ds.E, 1,
                              plan.tq, h.tile_lut.p, st);
            RowSet rs{h.qlut.p, h.tile_lut.p, nullptr, bias.as<uint32_t>()};
            bool ok = true;
            if (count) {
                // same machinery as the flat search; explicit ids ride in ScanArgs::ids
                h.sel.cap = buf_cap;
                ok = [&] {
                    const int grid = h.num_sms;
                    const uint64_t s0 = std::min<uint64_t>(h.seg0, std::max<uint32_t>(buf_cap / 2, 256)) / 16 * 16;
                    const std::vector<uint64_t> bounds = segment_bounds(count, s0, h.seg_growth);
                    for (size_t s = 0; s + 1 < bounds.size(); ++s) {
                        std::vector<ScanJob> jobs;
                        flat_segment_jobs(jobs, bounds[s], bounds[s + 1], 1, plan.tq, base_id, grid);
                        h.jobs.ensure(jobs.size() * sizeof(ScanJob));
                        QADC_CUDA_CHECK(cudaMemcpyAsync(h.jobs.p, jobs.data(), jobs.size() * sizeof(ScanJob), cudaMemcpyHostToDevice, st));
                        ScanArgs a{};
                        a.codes = h.codes.as<uint8_t>();
                        a.ids = ids ? h.ids.as<uint32_t>() : nullptr;
                        a.qlut = rs.qlut;
                        a.tile_lut = rs.tile_lut;
                        a.row_bias = rs.row_bias;
                        a.jobs = h.jobs.as<ScanJob>();
                        a.n_jobs = uint32_t(jobs.size());
                        a.thr_key = h.sel.thr_key.as<uint64_t>();
                        a.cand = h.sel.cand.as<uint64_t>();
                        a.cand_count = h.sel.cand_count.as<uint32_t>();
                        a.cap = buf_cap;
                        a.overflow = h.sel.overflow.as<uint32_t>();
                        launch_scan(plan, ds, a, std::min<int>(grid, int(jobs.size())), st);
                        launch_tighten(h.sel.top.as<uint64_t>(), h.sel.ntop.as<uint32_t>(), h.sel.kpad,
                                       h.sel.cand.as<uint64_t>(), h.sel.cand_count.as<uint32_t>(), buf_cap,
                                       h.sel.thr_key.as<uint64_t>(), 1, cap, nullptr, st);
                        QADC_CUDA_CHECK(cudaStreamSynchronize(st)); // jobs vector goes out of scope
                    }
                    uint32_t ov = 0;
                    QADC_CUDA_CHECK(cudaMemcpy(&ov, h.sel.overflow.p, 4, cudaMemcpyDeviceToHost));
                    return ov == 0;
                }();
            }
            if (ok) break;
            if (uint64_t(buf_cap) >= count + n_in + 16) throw Error(QADC_ERR_CUDA, "internal: candidate overflow at full capacity");
            buf_cap = uint32_t(std::min<uint64_t>(uint64_t(buf_cap) * 8, count + n_in + 16));
        }
        DevBuf keys, cnt;
        keys.ensure(size_t(cap) * 8);
        cnt.ensure(4);
        launch_finalize(h.sel.top.as<uint64_t>(), h.sel.ntop.as<uint32_t>(), h.sel.kpad, 1, 1, cap, nullptr, 0, ds.qmax,
                        nullptr, nullptr, cnt.as<uint32_t>(), keys.as<uint64_t>(), st);
        std::vector<uint64_t> hk(cap);
        uint32_t n = 0;
        QADC_CUDA_CHECK(cudaMemcpyAsync(hk.data(), keys.p, size_t(cap) * 8, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaMemcpyAsync(&n, cnt.p, 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
        for (uint32_t i = 0; i < n; ++i) {
            out_dist[i] = uint32_t(hk[i] >> 32);
            out_id[i] = uint32_t(hk[i]);
        }
        *n_out = n;
    });
}

int qadc_encode(const qadc_spec* spec, const float* codebook, const float* vectors, uint64_t n, uint8_t* codes,
                int device) {
    return guarded([&] {
        if (!spec || !codebook || (n && (!vectors || !codes))) throw Error(QADC_ERR_INPUT, "encode: null argument");
        validate_spec(*spec);
        set_device(device);
        const DevSpec ds = make_dev_spec(*spec, spec->groups);
        DevBuf cb, v, c;
        cb.ensure(size_t(spec->cb_floats) * 4);
        QADC_CUDA_CHECK(cudaMemcpy(cb.p, codebook, size_t(spec->cb_floats) * 4, cudaMemcpyHostToDevice));
        const uint64_t batch = 1u << 20;
        v.ensure(size_t(std::min(batch, std::max<uint64_t>(n, 1))) * spec->dims * 4);
        c.ensure(size_t(std::min(batch, std::max<uint64_t>(n, 1))) * spec->m);
        for (uint64_t i = 0; i < n; i += batch) {
            const uint64_t nb = std::min(batch, n - i);
            QADC_CUDA_CHECK(cudaMemcpy(v.p, vectors + i * spec->dims, size_t(nb) * spec->dims * 4, cudaMemcpyHostToDevice));
            launch_encode(ds, cb.as<float>(), v.as<float>(), nb, c.as<uint8_t>(), nullptr);
            QADC_CUDA_CHECK(cudaMemcpy(codes + i * spec->m, c.p, size_t(nb) * spec->m, cudaMemcpyDeviceToHost));
        }
    });
}

int qadc_ivf_assign_encode(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                           const float* vectors, uint64_t n, uint32_t* assign, uint8_t* codes, int device) {
    return guarded([&] {
        if (!spec || !codebook || !coarse || (n && (!vectors || !assign || !codes)))
            throw Error(QADC_ERR_INPUT, "ivf build: null argument");
        if (k_cells == 0) throw Error(QADC_ERR_INPUT, "ivf build: no coarse centroids");
        validate_spec(*spec);
        set_device(device);
        const DevSpec ds = make_dev_spec(*spec, spec->groups);
        const uint32_t dims = spec->dims;
        std::vector<float> ct(size_t(dims) * k_cells);
        for (uint32_t c = 0; c < k_cells; ++c)
            for (uint32_t j = 0; j < dims; ++j) ct[size_t(j) * k_cells + c] = coarse[size_t(c) * dims + j];
        const uint64_t batch = std::min<uint64_t>(1u << 17, std::max<uint64_t>(n, 1));
        DevBuf cb, co, cot, v, resid, scratch, asg, c;
        cb.ensure(size_t(spec->cb_floats) * 4);
        co.ensure(ct.size() * 4);
        cot.ensure(ct.size() * 4);
        v.ensure(size_t(batch) * dims * 4);
        resid.ensure(size_t(batch) * dims * 4);
        scratch.ensure(ivf_assign_scratch_bytes(k_cells, batch));
        asg.ensure(size_t(batch) * 4);
        c.ensure(size_t(batch) * spec->m);
        QADC_CUDA_CHECK(cudaMemcpy(cb.p, codebook, size_t(spec->cb_floats) * 4, cudaMemcpyHostToDevice));
        QADC_CUDA_CHECK(cudaMemcpy(co.p, coarse, ct.size() * 4, cudaMemcpyHostToDevice));
        QADC_CUDA_CHECK(cudaMemcpy(cot.p, ct.data(), ct.size() * 4, cudaMemcpyHostToDevice));
        for (uint64_t i = 0; i < n; i += batch) {
            const uint64_t nb = std::min(batch, n - i);
            QADC_CUDA_CHECK(cudaMemcpy(v.p, vectors + i * dims, size_t(nb) * dims * 4, cudaMemcpyHostToDevice));
            launch_ivf_assign(v.as<float>(), co.as<float>(), cot.as<float>(), dims, k_cells, nb, scratch.p,
                              asg.as<uint32_t>(), resid.as<float>(), nullptr);
            launch_encode(ds, cb.as<float>(), resid.as<float>(), nb, c.as<uint8_t>(), nullptr);
            QADC_CUDA_CHECK(cudaMemcpy(assign + i, asg.p, size_t(nb) * 4, cudaMemcpyDeviceToHost));
            QADC_CUDA_CHECK(cudaMemcpy(codes + i * spec->m, c.p, size_t(nb) * spec->m, cudaMemcpyDeviceToHost));
        }
    });
}

uint64_t qadc_ivf_build_packed_bound(const qadc_spec* s, uint64_t n, uint32_t k_cells) {
    const uint64_t block_bytes = uint64_t(s->groups) * s->block_len * (s->word_width / 8);
    return (n / s->block_len + k_cells) * block_bytes; // every list wastes less than one block
}

int qadc_ivf_build_lists(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                         const float* vectors, uint64_t n, uint64_t* list_count, uint64_t* list_byte_off,
                         uint64_t* list_id_off, uint32_t* ids, uint8_t* packed, uint64_t packed_cap, uint64_t* packed_bytes,
                         uint32_t* assign, int device) {
    return guarded([&] {
        if (!spec || !codebook || !coarse || !list_count || !list_byte_off || !list_id_off || !packed_bytes ||
            (n && (!vectors || !ids || !packed)))
            throw Error(QADC_ERR_INPUT, "ivf build: null argument");
        if (k_cells == 0) throw Error(QADC_ERR_INPUT, "ivf build: no coarse centroids");
        if (n > 0xFFFFFFFFull) throw Error(QADC_ERR_INPUT, "ivf build: more than 2^32 - 1 vectors (ids are 32-bit)");
        validate_spec(*spec);
        if (packed_cap < qadc_ivf_build_packed_bound(spec, n, k_cells))
            throw Error(QADC_ERR_INPUT, "ivf build: packed buffer smaller than qadc_ivf_build_packed_bound()");
        set_device(device);
        const DevSpec ds = make_dev_spec(*spec, spec->groups);
        const uint32_t dims = spec->dims;
        std::vector<float> ct(size_t(dims) * k_cells);
        for (uint32_t c = 0; c < k_cells; ++c)
            for (uint32_t j = 0; j < dims; ++j) ct[size_t(j) * k_cells + c] = coarse[size_t(c) * dims + j];
        const uint64_t batch = std::min<uint64_t>(1u << 17, std::max<uint64_t>(n, 1));
        DevBuf cb, co, cot, v, resid, scratch, asg, codes, counts, id_off, byte_off, totals, order, pk, status;
        cb.ensure(size_t(spec->cb_floats) * 4);
        co.ensure(ct.size() * 4);
        cot.ensure(ct.size() * 4);
        v.ensure(size_t(batch) * dims * 4);
        resid.ensure(size_t(batch) * dims * 4);
        scratch.ensure(ivf_assign_scratch_bytes(k_cells, batch));
        asg.ensure(std::max<size_t>(size_t(n) * 4, 16));
        codes.ensure(std::max<size_t>(size_t(n) * spec->m, 16));
        counts.ensure(size_t(k_cells) * 8);
        id_off.ensure(size_t(k_cells) * 8);
        byte_off.ensure(size_t(k_cells) * 8);
        totals.ensure(16);
        order.ensure(std::max<size_t>(size_t(n) * 4, 16));
        pk.ensure(std::max<uint64_t>(packed_cap, 16));
        status.ensure(4);
        QADC_CUDA_CHECK(cudaMemset(status.p, 0, 4));
        QADC_CUDA_CHECK(cudaMemcpy(cb.p, codebook, size_t(spec->cb_floats) * 4, cudaMemcpyHostToDevice));
        QADC_CUDA_CHECK(cudaMemcpy(co.p, coarse, ct.size() * 4, cudaMemcpyHostToDevice));
        QADC_CUDA_CHECK(cudaMemcpy(cot.p, ct.data(), ct.size() * 4, cudaMemcpyHostToDevice));
        for (uint64_t i = 0; i < n; i += batch) { // vectors stream through; assignments and codes stay on the device
            const uint64_t nb = std::min(batch, n - i);
            QADC_CUDA_CHECK(cudaMemcpy(v.p, vectors + i * dims, size_t(nb) * dims * 4, cudaMemcpyHostToDevice));
            launch_ivf_assign(v.as<float>(), co.as<float>(), cot.as<float>(), dims, k_cells, nb, scratch.p,
                              asg.as<uint32_t>() + i, resid.as<float>(), nullptr);
            launch_encode(ds, cb.as<float>(), resid.as<float>(), nb, codes.as<uint8_t>() + i * spec->m, nullptr);
        }
        launch_ivf_group_pack(*spec, ds, asg.as<uint32_t>(), codes.as<uint8_t>(), n, k_cells,
                              counts.as<unsigned long long>(), id_off.as<unsigned long long>(),
                              byte_off.as<unsigned long long>(), totals.as<unsigned long long>(), order.as<uint32_t>(),
                              pk.as<uint8_t>(), status.as<int>(), nullptr);
        unsigned long long tot[2] = {0, 0};
        int st = 0;
        QADC_CUDA_CHECK(cudaMemcpy(tot, totals.p, 16, cudaMemcpyDeviceToHost));
        QADC_CUDA_CHECK(cudaMemcpy(&st, status.p, 4, cudaMemcpyDeviceToHost));
        if (st) throw Error(st, "ivf build: assignment out of range");
        if (tot[0] != n || tot[1] > packed_cap) throw Error(QADC_ERR_CUDA, "ivf build: internal size mismatch");
        static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "u64");
        QADC_CUDA_CHECK(cudaMemcpy(list_count, counts.p, size_t(k_cells) * 8, cudaMemcpyDeviceToHost));
        QADC_CUDA_CHECK(cudaMemcpy(list_id_off, id_off.p, size_t(k_cells) * 8, cudaMemcpyDeviceToHost));
        QADC_CUDA_CHECK(cudaMemcpy(list_byte_off, byte_off.p, size_t(k_cells) * 8, cudaMemcpyDeviceToHost));
        if (n) {
            QADC_CUDA_CHECK(cudaMemcpy(ids, order.p, size_t(n) * 4, cudaMemcpyDeviceToHost));
            QADC_CUDA_CHECK(cudaMemcpy(packed, pk.p, size_t(tot[1]), cudaMemcpyDeviceToHost));
            if (assign) QADC_CUDA_CHECK(cudaMemcpy(assign, asg.p, size_t(n) * 4, cudaMemcpyDeviceToHost));
        }
        *packed_bytes = tot[1];
    });
}

int qadc_debug_canary(uint64_t* buffers_checked, uint64_t* bytes_corrupted) {
    if (buffers_checked) *buffers_checked = g_canary_checked.load();
    if (bytes_corrupted) *bytes_corrupted = g_canary_failures.load();
    return canary_mode() ? 1 : 0;
}

int qadc_get_stats(const qadc_index* h, qadc_stats* out) {
    if (!h || !out) return QADC_ERR_INPUT;
    *out = h->stats;
    return QADC_OK;
}

int qadc_set_option(qadc_index* h, const char* name, int64_t value) {
    return guarded([&] {
        if (!h || !name) throw Error(QADC_ERR_INPUT, "set_option: null argument");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        const std::string n(name);
        if (n == "cand_cap") h->cand_cap = uint32_t(std::max<int64_t>(value, 16));
        else if (n == "seg0") h->seg0 = uint32_t(std::min<int64_t>(std::max<int64_t>(value, 256), 16384)) / 16u * 16u; // bulk copies: 16-byte aligned
        else if (n == "seg_growth_pct") h->seg_growth_pct = uint32_t(std::max<int64_t>(value, 0));
        else if (n == "seg_growth") {
            h->seg_growth = uint32_t(std::max<int64_t>(value, 2));
            h->seg_growth_set = true;
        }
        else if (n == "force_variant") h->force_variant = int(value);
        else if (n == "probe_tc") h->probe_tc = int(value);
        else if (n == "tc_debug") h->tc_debug = uint32_t(value);
        else if (n == "ivf_round0") h->ivf_round0 = uint32_t(std::min<int64_t>(std::max<int64_t>(value, 64), 1 << 30)) / 16u * 16u;
        else throw Error(QADC_ERR_CONFIG, "set_option: unknown option " + n);
    });
}

int qadc_ivf_open(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                  const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                  const uint64_t* list_count, const uint32_t* ids, const uint8_t* calib_packed,
                  const uint64_t* calib_byte_off, const uint64_t* calib_count, const uint64_t* global_list_count,
                  int device, qadc_index** out) {
    return guarded([&] {
        if (!spec || !codebook || !out || (k_cells && (!coarse || !list_byte_off || !list_id_off || !list_count)))
            throw Error(QADC_ERR_INPUT, "null argument");
        const bool have_heads = calib_packed || calib_byte_off || calib_count;
        if (have_heads && (!calib_byte_off || !calib_count || !global_list_count))
            throw Error(QADC_ERR_INPUT, "ivf: calib_byte_off, calib_count and global_list_count must be given together");
        validate_spec(*spec);
        set_device(device);
        std::unique_ptr<qadc_index> h(new qadc_index);
        h->kind = 1;
        h->device = device;
        h->spec = *spec;
        h->ds = make_dev_spec(*spec, spec->groups);
        h->k_cells = k_cells;
        if (h->ds.code_stride > 32) throw Error(QADC_ERR_CONFIG, "codes wider than 256 bits are not supported");
        QADC_CUDA_CHECK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
        QADC_CUDA_CHECK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        cudaStream_t st = h->stream;
        for (uint32_t i = 0; i < spec->cb_floats; ++i)
            if (!(codebook[i] - codebook[i] == 0.0f)) throw Error(QADC_ERR_CORRUPTION, "codebook: non-finite centroid component");
        h->codebook.ensure(size_t(spec->cb_floats) * 4);
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->codebook.p, codebook, size_t(spec->cb_floats) * 4, cudaMemcpyHostToDevice, st));
        if (ivf_tables_tiled_supported(h->ds)) { // transposed codebook + entry map of the tiled table kernel (ivf_lut.cu)
            std::vector<float> cbt;
            std::vector<uint8_t> sub_of;
            ivf_tables_tiled_prepare(h->ds, codebook, cbt, sub_of);
            h->codebook_t.ensure(cbt.size() * 4);
            h->sub_of.ensure(sub_of.size());
            QADC_CUDA_CHECK(cudaMemcpy(h->codebook_t.p, cbt.data(), cbt.size() * 4, cudaMemcpyHostToDevice));
            QADC_CUDA_CHECK(cudaMemcpy(h->sub_of.p, sub_of.data(), sub_of.size(), cudaMemcpyHostToDevice));
        }
        const uint32_t d = spec->dims;
        // coarse centroids: row-major for the residuals, transposed [dims][K] for the probe kernel
        std::vector<float> ct(size_t(k_cells) * d);
        for (uint32_t c = 0; c < k_cells; ++c)
            for (uint32_t j = 0; j < d; ++j) ct[size_t(j) * k_cells + c] = coarse[size_t(c) * d + j];
        h->coarse.ensure(std::max<size_t>(ct.size() * 4, 16));
        h->coarse_t.ensure(std::max<size_t>(ct.size() * 4, 16));
        if (k_cells) {
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->coarse.p, coarse, ct.size() * 4, cudaMemcpyHostToDevice, st));
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->coarse_t.p, ct.data(), ct.size() * 4, cudaMemcpyHostToDevice, st));
        }
        if (k_cells >= 512) { // tensor-core probe prefilter: centred bf16 image of the centroids, |c'|^2, max |c'|
            h->dpad = (d + 15) / 16 * 16;
            std::vector<uint16_t> cb16;
            std::vector<float> cn;
            std::vector<double> mean;
            h->probe_tc_ready = ivf_probe_tc_prepare(coarse, k_cells, d, h->dpad, cb16, cn, mean, h->coarse_rmax);
            if (h->probe_tc_ready) {
                h->coarse_bf16.ensure(cb16.size() * 2);
                h->coarse_norm.ensure(cn.size() * 4);
                h->coarse_mean.ensure(mean.size() * 8);
                QADC_CUDA_CHECK(cudaMemcpy(h->coarse_bf16.p, cb16.data(), cb16.size() * 2, cudaMemcpyHostToDevice));
                QADC_CUDA_CHECK(cudaMemcpy(h->coarse_norm.p, cn.data(), cn.size() * 4, cudaMemcpyHostToDevice));
                QADC_CUDA_CHECK(cudaMemcpy(h->coarse_mean.p, mean.data(), mean.size() * 8, cudaMemcpyHostToDevice));
            }
        }
        // every list starts on a 16-code boundary of the device array (bulk copies need 16-byte alignment)
        const uint64_t LIST_ALIGN = 16;
        h->list_code_off_h.resize(k_cells);
        h->list_count_h.assign(list_count, list_count + k_cells);
        uint64_t run = 0, packed_total = 0, n_ids = 0;
        for (uint32_t c = 0; c < k_cells; ++c) {
            if (list_count[c] > 0xFFFFFFFFull) throw Error(QADC_ERR_INPUT, "ivf: a list holds more than 2^32 - 1 codes");
            h->list_code_off_h[c] = run;
            run += (list_count[c] + LIST_ALIGN - 1) / LIST_ALIGN * LIST_ALIGN;
            packed_total = std::max<uint64_t>(packed_total, list_byte_off[c] + qadc_packed_bytes(spec, list_count[c]));
            n_ids += list_count[c];
        }
        h->total_codes = n_ids;
        if (n_ids && (!packed || !ids)) throw Error(QADC_ERR_INPUT, "null argument");
        const uint64_t total_padded = run + CODE_PAD;
        h->count_padded = total_padded;
        h->codes.ensure(size_t(total_padded) * h->ds.code_stride);
        h->list_code_off.ensure(std::max<size_t>(size_t(k_cells) * 8, 16));
        h->list_count_dev.ensure(std::max<size_t>(size_t(k_cells) * 8, 16));
        DevBuf tmp, boff;
        tmp.ensure(std::max<uint64_t>(packed_total, 16));
        boff.ensure(std::max<size_t>(size_t(k_cells) * 8, 16));
        if (k_cells) {
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->list_code_off.p, h->list_code_off_h.data(), size_t(k_cells) * 8, cudaMemcpyHostToDevice, st));
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->list_count_dev.p, list_count, size_t(k_cells) * 8, cudaMemcpyHostToDevice, st));
            QADC_CUDA_CHECK(cudaMemcpyAsync(boff.p, list_byte_off, size_t(k_cells) * 8, cudaMemcpyHostToDevice, st));
        }
        copy_h2d_chunked(tmp.p, packed, packed_total, st);
        if (k_cells)
            launch_ivf_relayout(*spec, h->ds, tmp.as<uint8_t>(), boff.as<uint64_t>(), h->list_code_off.as<uint64_t>(),
                                h->list_count_dev.as<uint64_t>(), k_cells, total_padded, h->codes.as<uint8_t>(), st);
        if (have_heads) {
            // replicated heads of the unsharded lists (first min(count, t_max) codes each): calibration input
            h->own_heads = false;
            std::vector<uint64_t> coff(k_cells);
            uint64_t crun = 0, cbytes = 0;
            for (uint32_t c = 0; c < k_cells; ++c) {
                if (calib_count[c] > global_list_count[c] || list_count[c] > global_list_count[c])
                    throw Error(QADC_ERR_INPUT, "ivf: a list head or shard is longer than its whole list");
                if (calib_count[c] < global_list_count[c]) h->calib_limit = std::min<uint64_t>(h->calib_limit, calib_count[c]);
                coff[c] = crun;
                crun += (calib_count[c] + LIST_ALIGN - 1) / LIST_ALIGN * LIST_ALIGN;
                if (calib_count[c]) cbytes = std::max<uint64_t>(cbytes, calib_byte_off[c] + qadc_packed_bytes(spec, calib_count[c]));
            }
            if (cbytes && !calib_packed) throw Error(QADC_ERR_INPUT, "null argument");
            const uint64_t cpad = crun + CODE_PAD;
            h->calib.ensure(size_t(cpad) * h->ds.code_stride);
            h->calib_code_off.ensure(std::max<size_t>(size_t(k_cells) * 8, 16));
            h->calib_count_dev.ensure(std::max<size_t>(size_t(k_cells) * 8, 16));
            DevBuf ctmp, cboff;
            ctmp.ensure(std::max<uint64_t>(cbytes, 16));
            cboff.ensure(std::max<size_t>(size_t(k_cells) * 8, 16));
            if (k_cells) {
                QADC_CUDA_CHECK(cudaMemcpyAsync(h->calib_code_off.p, coff.data(), size_t(k_cells) * 8, cudaMemcpyHostToDevice, st));
                QADC_CUDA_CHECK(cudaMemcpyAsync(h->calib_count_dev.p, calib_count, size_t(k_cells) * 8, cudaMemcpyHostToDevice, st));
                QADC_CUDA_CHECK(cudaMemcpyAsync(cboff.p, calib_byte_off, size_t(k_cells) * 8, cudaMemcpyHostToDevice, st));
            }
            if (cbytes) QADC_CUDA_CHECK(cudaMemcpyAsync(ctmp.p, calib_packed, cbytes, cudaMemcpyHostToDevice, st));
            if (k_cells)
                launch_ivf_relayout(*spec, h->ds, ctmp.as<uint8_t>(), cboff.as<uint64_t>(), h->calib_code_off.as<uint64_t>(),
                                    h->calib_count_dev.as<uint64_t>(), k_cells, cpad, h->calib.as<uint8_t>(), st);
            QADC_CUDA_CHECK(cudaStreamSynchronize(st)); // coff / temporaries go out of scope
        }
        // ids ride in the same index space as the device codes
        std::vector<uint32_t> ids_padded(total_padded, 0xFFFFFFFFu);
        for (uint32_t c = 0; c < k_cells; ++c)
            std::copy(ids + list_id_off[c], ids + list_id_off[c] + list_count[c], ids_padded.begin() + h->list_code_off_h[c]);
        h->ids.ensure(size_t(total_padded) * 4);
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->ids.p, ids_padded.data(), size_t(total_padded) * 4, cudaMemcpyHostToDevice, st));
        std::vector<uint32_t> loc;
        if (!have_heads && total_padded < (uint64_t(1) << 32)) {
            // IvfIndex::build_locator (index.hpp:366-375): ids must be < total ("vector id out of range" otherwise);
            // the locator maps an id to its device code position for exact re-ranking.  Shards carry global ids and
            // skip both.
            loc.assign(std::max<uint64_t>(n_ids, 1), 0u);
            for (uint32_t c = 0; c < k_cells; ++c)
                for (uint64_t pp = 0; pp < list_count[c]; ++pp) {
                    const uint32_t id = ids[list_id_off[c] + pp];
                    if (id >= n_ids) throw Error(QADC_ERR_CORRUPTION, "ivf: vector id out of range");
                    loc[id] = uint32_t(h->list_code_off_h[c] + pp);
                }
            h->locator.ensure(loc.size() * 4);
            QADC_CUDA_CHECK(cudaMemcpyAsync(h->locator.p, loc.data(), loc.size() * 4, cudaMemcpyHostToDevice, st));
        }
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
        *out = h.release();
    });
}

int qadc_ivf_probe_order(qadc_index* h, const float* queries, uint32_t nq, uint32_t a, uint32_t* order) {
    return guarded([&] {
        if (!h || h->kind != 1 || (nq && (!queries || !order))) throw Error(QADC_ERR_INPUT, "probe_order: bad arguments");
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        set_device(h->device);
        a = std::min(a, h->k_cells);
        if (nq == 0 || a == 0) return;
        cudaStream_t st = h->stream;
        h->queries.ensure(size_t(nq) * h->ds.dims * 4);
        h->order.ensure(size_t(nq) * a * 4);
        QADC_CUDA_CHECK(cudaMemcpyAsync(h->queries.p, queries, size_t(nq) * h->ds.dims * 4, cudaMemcpyHostToDevice, st));
        ivf_probe_order_device(h, h->queries.as<float>(), nq, a, st);
        QADC_CUDA_CHECK(cudaMemcpyAsync(order, h->order.p, size_t(nq) * a * 4, cudaMemcpyDeviceToHost, st));
        QADC_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

} // extern "C"
