// integration_test.cpp -- the reference's own C++ types driving the B200 path through include/qadc.hpp.
//
// Compiled IN THE BUILD CONTAINER against the unmodified reference headers (oracle/Makefile, target
// `integration`; output oracle/_ref/integration_test, which travels to the GPU box).  It follows the
// methodology of the reference's differential self-test (selftest.hpp:40-127: random tables, occupancies,
// pre-seeded heaps, bias, both id modes; heaps must match entry by entry) with the GPU scan function in
// the place of the SIMD kernels, then compares FlatIndex::search / IvfIndex::search with their GPU
// counterparts on indexes BUILT BY THE REFERENCE (k-means training, encode, pack).  Exit code 0 = all equal.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "qadc.hpp"

using namespace pqscan;

static void cudaGetDeviceCount_shim(int* n) { *n = qadc_device_count(); } // the ABI's own device probe (no CUDA headers here)

static int g_fail = 0;
#define EXPECT(cond, ...)                      \
    do {                                       \
        if (!(cond)) {                         \
            ++g_fail;                          \
            std::fprintf(stderr, "FAIL: ");    \
            std::fprintf(stderr, __VA_ARGS__); \
            std::fprintf(stderr, "\n");        \
        }                                      \
    } while (0)

static std::vector<float> blobs(size_t n, size_t d, size_t clusters, uint64_t seed) {
    std::mt19937_64 rng(seed);
    auto uni = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
    auto gauss = [&] { // Box-Muller on raw draws: portable across standard libraries
        double u1 = uni(), u2 = uni();
        if (u1 < 1e-300) u1 = 1e-300;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    };
    std::vector<float> centres(clusters * d), out(n * d);
    for (auto& v : centres) v = static_cast<float>(uni() * 100.0);
    for (size_t i = 0; i < n; ++i) {
        const size_t c = rng() % clusters;
        for (size_t j = 0; j < d; ++j) out[i * d + j] = centres[c * d + j] + static_cast<float>(3.0 * gauss());
    }
    return out;
}

static bool same(const SearchResult& a, const SearchResult& b) {
    return a.ids == b.ids && a.dists.size() == b.dists.size() &&
           std::memcmp(a.dists.data(), b.dists.data(), a.dists.size() * sizeof(float)) == 0;
}

static void scan_fn_trials(uint64_t trials, uint64_t seed) {
    const std::vector<std::pair<std::string, std::vector<uint32_t>>> fams = {
        {"{4,4}", {2, 4, 6, 8, 10, 16, 32}}, {"{6,6,4}", {3, 6, 12, 24}}, {"{6,5,5}", {3, 6, 12, 24}},
        {"{5,5,5}", {3, 6, 12, 24}},         {"{8,8}", {2, 4, 8, 16}},    {"{8}", {1, 2, 4, 8, 16}}};
    std::mt19937_64 rng(seed);
    QuantizedScanFn gpu = qadc::gpu_scan_fn();
    for (const auto& [pattern, ms] : fams)
        for (uint64_t t = 0; t < trials; ++t) {
            const uint32_t m = ms[rng() % ms.size()];
            PqSpec spec = allocate_dims(16 * m, parse_spec_string(std::to_string(m) + "x" + pattern));
            PackingScheme scheme = PackingScheme::for_spec(spec);
            QuantizedTables qt;
            qt.width = scheme.word_width;
            qt.delta = 1.0f;
            qt.p_min.assign(spec.num_subs(), 0.0f);
            const uint32_t q_max = qt.q_max();
            const bool sat = rng() % 4 == 0;
            auto draw = [&]() -> uint32_t { return sat ? q_max - rng() % (q_max / 4 + 1) : rng() % (q_max + 1); };
            if (qt.width == 8) {
                qt.t8.resize(spec.num_subs());
                for (size_t j = 0; j < spec.num_subs(); ++j) {
                    qt.t8[j].resize(spec.centroid_count(j));
                    for (auto& e : qt.t8[j]) e = static_cast<uint8_t>(draw());
                }
            } else {
                qt.t16.resize(spec.num_subs());
                for (size_t j = 0; j < spec.num_subs(); ++j) {
                    qt.t16[j].resize(spec.centroid_count(j));
                    for (auto& e : qt.t16[j]) e = static_cast<uint16_t>(draw());
                }
            }
            const size_t n = 1 + rng() % (size_t{scheme.block_len} * 3 + (t % 5 == 0 ? 5000 : 0));
            std::vector<Code> codes(n, Code(spec.num_subs()));
            for (auto& c : codes)
                for (size_t j = 0; j < spec.num_subs(); ++j) c[j] = static_cast<uint8_t>(rng() % spec.centroid_count(j));
            PackedList list = pack_list(codes, scheme);
            const uint32_t r = 1 + rng() % 24;
            const uint32_t init = (rng() % 4 == 0) ? static_cast<uint32_t>(rng() % (q_max + 2)) : 0;
            std::vector<uint32_t> ids;
            const uint32_t* idp = nullptr;
            const uint32_t base = static_cast<uint32_t>(rng() % 100000);
            if (rng() % 2) {
                ids.resize(n);
                for (auto& id : ids) id = static_cast<uint32_t>(rng() % 1000000);
                idp = ids.data();
            }
            CandidateHeap<uint32_t> ref(r), dev(r);
            const uint32_t preseed = rng() % 4;
            for (uint32_t i = 0; i < preseed; ++i) {
                uint32_t d = rng() % (q_max + 1), id = 2000000 + i;
                ref.push(d, id);
                dev.push(d, id);
            }
            scan_list_scalar_quantized(list, scheme, qt, idp, base, init, ref);
            gpu(list, scheme, qt, idp, base, init, dev);
            auto a = ref.sorted(), b = dev.sorted();
            bool ok = a.size() == b.size();
            for (size_t i = 0; ok && i < a.size(); ++i) ok = a[i] == b[i];
            EXPECT(ok, "scan fn mismatch: %ux%s n=%zu R=%u trial=%llu", m, pattern.c_str(), n, r, (unsigned long long)t);
        }
    std::printf("scan-fn differential: %llu trials x %zu families done\n", (unsigned long long)trials, fams.size());
}

static void flat_checks() {
    for (const char* text : {"16x{4,4}", "12x{6,5,5}", "8x{8,8}", "8x{8}"}) {
        const uint32_t d = 64;
        PqSpec spec = allocate_dims(d, parse_spec_string(text));
        auto train = blobs(2500, d, 20, 1);
        TrainConfig tc;
        tc.kmeans_iters = spec.max_centroid_count() > 64 ? 4 : 10;
        tc.seed = 7;
        Codebook cb = train_codebook(train, 2500, spec, tc);
        auto db = blobs(20000, d, 20, 2);
        FlatIndex ref = FlatIndex::encode_database(db, 20000, cb);
        qadc::GpuFlatIndex gpu(ref);
        auto queries = blobs(40, d, 20, 3);
        SearchParams p;
        auto batch = gpu.search_batch(queries, 40, p);
        for (uint32_t q = 0; q < 40; ++q) {
            SearchResult want = ref.search({queries.data() + size_t{q} * d, d}, p);
            EXPECT(same(want, batch[q]), "flat %s query %u differs", text, q);
        }
        SearchResult one = gpu.search({queries.data(), d}, p);
        EXPECT(same(one, batch[0]), "flat %s single vs batch", text);
        SearchParams pr = p; // exact re-ranking of the final set (index.hpp:148-152)
        pr.rerank = true;
        auto rr = gpu.search_batch(queries, 40, pr);
        for (uint32_t q = 0; q < 40; ++q)
            EXPECT(same(ref.search({queries.data() + size_t{q} * d, d}, pr), rr[q]), "flat %s rerank query %u differs", text, q);
        bool threw = false;
        try {
            SearchParams bad;
            bad.t = 5;
            gpu.search({queries.data(), d}, bad);
        } catch (const input_error&) { threw = true; }
        EXPECT(threw, "flat %s: t < R must be an input_error", text);
        // the one-process multi-GPU handle (qadc_flat_open_sharded) on the devices this box has: shards + replicated
        // head + NCCL all_gather + merge must give the same lists
        {
            int ndev = 0;
            cudaGetDeviceCount_shim(&ndev);
            const char* same_env = std::getenv("QADC_MULTI_SAME_DEVICE_TEST"); // three shards on one device (test hook)
            const int three[3] = {0, 0, 0};
            const bool dup = same_env && same_env[0] == '1';
            qadc::GpuFlatIndex multi(ref, dup ? 3 : (ndev > 0 ? ndev : 1), dup ? three : nullptr);
            auto mb = multi.search_batch(queries, 40, p);
            for (uint32_t q = 0; q < 40; ++q) EXPECT(same(batch[q], mb[q]), "flat %s sharded(%d) query %u differs", text, ndev, q);
        }
        std::printf("flat %s: 40 queries identical to FlatIndex::search\n", text);
    }
}

static void ivf_checks() {
    const uint32_t d = 48;
    auto db = blobs(30000, d, 30, 11);
    IvfBuildConfig cfg;
    cfg.k_coarse = 48;
    cfg.train.kmeans_iters = 6;
    cfg.train.seed = 3;
    IvfIndex ref = IvfIndex::build(db, 30000, parse_spec_string("12x{6,5,5}"), cfg);
    qadc::GpuIvfIndex gpu(ref);
    auto queries = blobs(30, d, 30, 12);
    for (uint32_t probes : {1u, 6u, 48u}) {
        SearchParams p;
        p.probes = probes;
        auto batch = gpu.search_batch(queries, 30, p);
        for (uint32_t q = 0; q < 30; ++q) {
            SearchResult want = ref.search({queries.data() + size_t{q} * d, d}, p);
            EXPECT(same(want, batch[q]), "ivf probes=%u query %u differs", probes, q);
        }
        EXPECT(ref.probe_order({queries.data(), d}, probes) == gpu.probe_order({queries.data(), d}, probes),
               "probe order differs at a=%u", probes);
        p.rerank = true; // index.hpp:377-386
        auto rr = gpu.search_batch(queries, 30, p);
        for (uint32_t q = 0; q < 30; ++q)
            EXPECT(same(ref.search({queries.data() + size_t{q} * d, d}, p), rr[q]), "ivf rerank probes=%u query %u differs",
                   probes, q);
    }
    { // the one-process multi-GPU handle for IVF (qadc_ivf_open_sharded): every list split over the devices of this box
      // (three shards on one device under QADC_MULTI_SAME_DEVICE_TEST=1, which the Python test sets)
        int ndev = 0;
        cudaGetDeviceCount_shim(&ndev);
        const char* same_env = std::getenv("QADC_MULTI_SAME_DEVICE_TEST");
        const int three[3] = {0, 0, 0};
        const bool dup = same_env && same_env[0] == '1';
        qadc::GpuIvfIndex multi(ref, dup ? 3 : (ndev > 0 ? ndev : 1), dup ? three : nullptr);
        SearchParams p;
        p.probes = 6;
        auto mb = multi.search_batch(queries, 30, p);
        for (uint32_t q = 0; q < 30; ++q)
            EXPECT(same(ref.search({queries.data() + size_t{q} * d, d}, p), mb[q]), "ivf sharded query %u differs", q);
    }
    std::printf("ivf 12x{6,5,5} K=48: identical to IvfIndex::search at probes 1/6/48 (+ sharded handle)\n");
}

int main(int argc, char** argv) {
    const uint64_t trials = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 40;
    try {
        scan_fn_trials(trials, 0xC0FFEE);
        flat_checks();
        ivf_checks();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    if (g_fail) {
        std::fprintf(stderr, "%d check(s) failed\n", g_fail);
        return 1;
    }
    std::printf("INTEGRATION OK\n");
    return 0;
}
