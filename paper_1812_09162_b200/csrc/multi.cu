// multi.cu -- one host process driving a FlatIndex sharded over several GPUs.
//
// The reference is single-process (its only concurrency is the CLI's query-parallel pool, pqscan_cli.cpp:141-166), so
// the drop-in multi-GPU form is one handle that owns N shards: the code array is split into contiguous block-aligned
// ranges, shard s scans with base_id = start_s exactly like the reference's chunked-scan contract
// (T/test_kernels.cpp:107-133), every shard is opened with the whole list's calibration head so that all of them
// derive bit-identical quantization maps with no communication (index.hpp:124-129), and ONE exchange step -- an
// ncclAllGather of the per-shard key lists (nq x R u64 per rank) over NVLink / NVSwitch -- is followed by the merge
// kernel (qadc_merge_topk_device) on device 0.  Exact because the heap is order-independent (heap.hpp:12-14).
//
// NCCL is bound at run time (dlopen of libnccl.so.2: the copy the process already uses, e.g. PyTorch's, or the
// system's), so libqadc_b200.so has no link-time dependency on it; a single-device handle works without NCCL.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace qadc {

namespace {

// the slice of nccl.h this file uses (ncclResult_t 0 = success; ncclUint64 = 5)
using ncclComm_t = void*;
struct NcclApi {
    void* lib = nullptr;
    int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok() const { return CommInitAll && CommDestroy && AllGather && GroupStart && GroupEnd && GetErrorString; }
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (a.lib) break;
        }
        if (a.lib) {
            a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(a.lib, "ncclCommInitAll"));
            a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.lib, "ncclCommDestroy"));
            a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.lib, "ncclAllGather"));
            a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.lib, "ncclGroupStart"));
            a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.lib, "ncclGroupEnd"));
            a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.lib, "ncclGetErrorString"));
        }
        return a;
    }();
    return api;
}

void nccl_check(int rc, const char* what) {
    if (rc != 0) throw Error(QADC_ERR_CUDA, std::string("NCCL ") + what + ": " + nccl().GetErrorString(rc));
}

struct DevMem {
    void* p = nullptr;
    size_t cap = 0;
    int device = 0;
    ~DevMem() {
        if (p) {
            cudaSetDevice(device);
            cudaFree(p);
        }
    }
    void ensure(int dev, size_t bytes) {
        if (bytes <= cap) return;
        QADC_CUDA_CHECK(cudaSetDevice(dev));
        if (p) cudaFree(p);
        p = nullptr;
        device = dev;
        QADC_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        cap = bytes;
    }
};

} // namespace

} // namespace qadc

using namespace qadc;

struct qadc_multi {
    int ndev = 0;
    qadc_spec spec{};
    uint64_t count = 0;
    std::vector<int> devices;
    std::vector<qadc_index*> shards;
    std::vector<cudaStream_t> streams;
    std::vector<ncclComm_t> comms; // empty: single device without NCCL, or the same-device test mode
    bool local_gather = false;     // QADC_MULTI_SAME_DEVICE_TEST: the shards share a device, the exchange is device-to-device copies
    std::vector<DevMem> queries, keys, map, gathered;
    DevMem out_ids, out_dists, out_counts; // on devices[0]
    std::string error;

    ~qadc_multi() {
        for (size_t i = 0; i < comms.size(); ++i)
            if (comms[i]) nccl().CommDestroy(comms[i]);
        for (size_t i = 0; i < streams.size(); ++i)
            if (streams[i]) {
                cudaSetDevice(devices[i]);
                cudaStreamDestroy(streams[i]);
            }
        for (qadc_index* s : shards) qadc_close(s);
    }
};

// Test hook: with QADC_MULTI_SAME_DEVICE_TEST=1 a device may be listed several times, so that the sharding arithmetic of
// this host (ranges, base ids, replicated heads, gather order, merge) runs with ndev > 1 on a one-GPU box; the exchange
// is then a device-to-device copy instead of ncclAllGather (NCCL refuses two ranks on one device).
static bool same_device_test() {
    const char* e = std::getenv("QADC_MULTI_SAME_DEVICE_TEST");
    return e && e[0] == '1';
}

// devices[] -> m->devices, streams, NCCL communicators
static void multi_setup_devices(qadc_multi* m, int ndev, const int* devices) {
    int visible = 0;
    if (cudaGetDeviceCount(&visible) != cudaSuccess || visible == 0)
        throw Error(QADC_ERR_CUDA, "no usable CUDA device (this library has no CPU fallback)");
    m->ndev = ndev;
    for (int i = 0; i < ndev; ++i) {
        const int d = devices ? devices[i] : i;
        if (d < 0 || d >= visible) throw Error(QADC_ERR_INPUT, "open_sharded: device ordinal out of range");
        if (std::find(m->devices.begin(), m->devices.end(), d) != m->devices.end()) {
            if (!same_device_test()) throw Error(QADC_ERR_INPUT, "open_sharded: a device is listed twice (one shard per GPU)");
            m->local_gather = true;
        }
        m->devices.push_back(d);
    }
}

static void multi_setup_exchange(qadc_multi* m) {
    const int ndev = m->ndev;
    m->streams.assign(ndev, nullptr);
    for (int i = 0; i < ndev; ++i) {
        QADC_CUDA_CHECK(cudaSetDevice(m->devices[i]));
        QADC_CUDA_CHECK(cudaStreamCreateWithFlags(&m->streams[i], cudaStreamNonBlocking));
    }
    if (m->local_gather) {
        // (test mode: no communicator)
    } else if (nccl().ok()) {
        m->comms.assign(ndev, nullptr);
        nccl_check(nccl().CommInitAll(m->comms.data(), ndev, m->devices.data()), "ncclCommInitAll");
    } else if (ndev > 1) {
        throw Error(QADC_ERR_CUDA, "open_sharded: libnccl.so.2 could not be loaded; the multi-GPU exchange needs NCCL");
    }
    m->queries.resize(ndev);
    m->keys.resize(ndev);
    m->map.resize(ndev);
    m->gathered.resize(ndev);
}

namespace qadc {
int multi_guarded(const std::function<void()>& f); // api.cu: maps exceptions to status codes + qadc_last_error
}

extern "C" {

int qadc_flat_open_sharded(const qadc_spec* spec, const float* codebook, const uint8_t* packed, uint64_t count, int ndev,
                           const int* devices, qadc_multi** out) {
    return multi_guarded([&] {
        if (!spec || !codebook || !out || (count && !packed)) throw Error(QADC_ERR_INPUT, "null argument");
        if (ndev < 1) throw Error(QADC_ERR_INPUT, "open_sharded: ndev must be at least 1");
        std::unique_ptr<qadc_multi> m(new qadc_multi);
        m->spec = *spec;
        m->count = count;
        multi_setup_devices(m.get(), ndev, devices);
        // contiguous block-aligned shards (the partition of paper_1812_09162_b200/dist.py::shard_ranges)
        const uint64_t bl = spec->block_len, blocks = (count + bl - 1) / bl;
        const uint64_t block_bytes = uint64_t(spec->groups) * bl * (spec->word_width / 8);
        const uint64_t head_n = std::min<uint64_t>(count, QADC_MAX_T);
        m->shards.assign(ndev, nullptr);
        for (int i = 0; i < ndev; ++i) {
            const uint64_t b0 = blocks * uint64_t(i) / uint64_t(ndev), b1 = blocks * uint64_t(i + 1) / uint64_t(ndev);
            const uint64_t start = std::min(b0 * bl, count), end = std::min(b1 * bl, count);
            if (start > 0xFFFFFFFFull) throw Error(QADC_ERR_INPUT, "open_sharded: more than 2^32 codes (ids are 32-bit)");
            const int rc = qadc_flat_open(spec, codebook, packed + b0 * block_bytes, end - start, uint32_t(start),
                                          ndev > 1 ? packed : nullptr, ndev > 1 ? head_n : 0, count, m->devices[i], &m->shards[i]);
            if (rc != QADC_OK) throw Error(rc, qadc_last_error());
        }
        multi_setup_exchange(m.get());
        *out = m.release();
    });
}

// IvfIndex over several GPUs behind one handle: EVERY list is split evenly on packed-block boundaries (ids are explicit,
// so any split is legal: scan_scalar.hpp:60) and the first min(count, QADC_MAX_T) codes of every unsharded list are
// replicated as calibration heads, so that probe order, tables, d_min_global, d_max, delta and the biases come out
// identical on every shard (index.hpp:276-341) -- the partition of paper_1812_09162_b200/dist.py::shard_ivf_lists.
int qadc_ivf_open_sharded(const qadc_spec* spec, const float* codebook, const float* coarse, uint32_t k_cells,
                          const uint8_t* packed, const uint64_t* list_byte_off, const uint64_t* list_id_off,
                          const uint64_t* list_count, const uint32_t* ids, int ndev, const int* devices, qadc_multi** out) {
    return multi_guarded([&] {
        if (!spec || !codebook || !out || (k_cells && (!coarse || !list_byte_off || !list_id_off || !list_count)))
            throw Error(QADC_ERR_INPUT, "null argument");
        if (ndev < 1) throw Error(QADC_ERR_INPUT, "open_sharded: ndev must be at least 1");
        std::unique_ptr<qadc_multi> m(new qadc_multi);
        m->spec = *spec;
        multi_setup_devices(m.get(), ndev, devices);
        const uint64_t bl = spec->block_len;
        const uint64_t block_bytes = uint64_t(spec->groups) * bl * (spec->word_width / 8);
        uint64_t total = 0;
        for (uint32_t c = 0; c < k_cells; ++c) total += list_count[c];
        m->count = total;
        if (total && (!packed || !ids)) throw Error(QADC_ERR_INPUT, "null argument");
        // the replicated heads (only needed when the lists are really split)
        std::vector<uint8_t> head_packed;
        std::vector<uint64_t> head_off(k_cells), head_cnt(k_cells), global_cnt(list_count, list_count + k_cells);
        if (ndev > 1)
            for (uint32_t c = 0; c < k_cells; ++c) {
                const uint64_t hn = std::min<uint64_t>(list_count[c], QADC_MAX_T);
                const uint64_t hb = (hn + bl - 1) / bl * block_bytes;
                head_off[c] = head_packed.size();
                head_cnt[c] = hn;
                head_packed.insert(head_packed.end(), packed + list_byte_off[c], packed + list_byte_off[c] + hb);
            }
        m->shards.assign(ndev, nullptr);
        for (int i = 0; i < ndev; ++i) {
            std::vector<uint8_t> sp;
            std::vector<uint32_t> sid;
            std::vector<uint64_t> boff(k_cells), ioff(k_cells), cnt(k_cells);
            for (uint32_t c = 0; c < k_cells; ++c) {
                const uint64_t n = list_count[c], blocks = (n + bl - 1) / bl;
                const uint64_t b0 = blocks * uint64_t(i) / uint64_t(ndev), b1 = blocks * uint64_t(i + 1) / uint64_t(ndev);
                const uint64_t start = std::min(b0 * bl, n), end = std::min(b1 * bl, n);
                boff[c] = sp.size();
                ioff[c] = sid.size();
                cnt[c] = end - start;
                const uint8_t* src = packed + list_byte_off[c];
                sp.insert(sp.end(), src + b0 * block_bytes, src + b1 * block_bytes);
                sid.insert(sid.end(), ids + list_id_off[c] + start, ids + list_id_off[c] + end);
            }
            const int rc = qadc_ivf_open(spec, codebook, coarse, k_cells, sp.data(), boff.data(), ioff.data(), cnt.data(), sid.data(),
                                         ndev > 1 ? head_packed.data() : nullptr, ndev > 1 ? head_off.data() : nullptr,
                                         ndev > 1 ? head_cnt.data() : nullptr, ndev > 1 ? global_cnt.data() : nullptr,
                                         m->devices[i], &m->shards[i]);
            if (rc != QADC_OK) throw Error(rc, qadc_last_error());
        }
        multi_setup_exchange(m.get());
        *out = m.release();
    });
}

int qadc_multi_search_batch(qadc_multi* m, const float* queries, uint32_t nq, const qadc_search_params* params,
                            uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    return multi_guarded([&] {
        if (!m || !params || (nq && (!queries || !out_ids || !out_dists || !out_counts)))
            throw Error(QADC_ERR_INPUT, "null argument");
        if (params->flags & QADC_FLAG_RERANK) throw Error(QADC_ERR_CONFIG, "rerank: not available on a sharded index");
        if (nq == 0) return;
        const int ndev = m->ndev;
        const uint32_t r = params->r;
        const size_t nr = size_t(nq) * std::max<uint32_t>(r, 1);
        for (int i = 0; i < ndev; ++i) {
            m->queries[i].ensure(m->devices[i], size_t(nq) * m->spec.dims * 4);
            m->keys[i].ensure(m->devices[i], nr * 8);
            m->map[i].ensure(m->devices[i], size_t(nq) * 8);
            m->gathered[i].ensure(m->devices[i], nr * 8 * ndev);
        }
        m->out_ids.ensure(m->devices[0], nr * 4);
        m->out_dists.ensure(m->devices[0], nr * 4);
        m->out_counts.ensure(m->devices[0], size_t(nq) * 4);
        // shard searches: one host thread per GPU (a search synchronises its own stream for its overflow check)
        std::vector<int> rcs(ndev, QADC_OK);
        std::vector<std::string> errs(ndev);
        auto work = [&](int i) {
            cudaSetDevice(m->devices[i]);
            cudaError_t e = cudaMemcpyAsync(m->queries[i].p, queries, size_t(nq) * m->spec.dims * 4, cudaMemcpyHostToDevice,
                                            m->streams[i]);
            if (e != cudaSuccess) {
                rcs[i] = QADC_ERR_CUDA;
                errs[i] = cudaGetErrorString(e);
                return;
            }
            rcs[i] = qadc_search_batch_device(m->shards[i], static_cast<const float*>(m->queries[i].p), nq, params, nullptr,
                                              nullptr, nullptr, static_cast<uint64_t*>(m->keys[i].p),
                                              static_cast<float*>(m->map[i].p), m->streams[i]);
            if (rcs[i] != QADC_OK) errs[i] = qadc_last_error();
        };
        if (ndev == 1) work(0);
        else {
            std::vector<std::thread> th;
            for (int i = 0; i < ndev; ++i) th.emplace_back(work, i);
            for (auto& t : th) t.join();
        }
        for (int i = 0; i < ndev; ++i)
            if (rcs[i] != QADC_OK) throw Error(rcs[i], "shard " + std::to_string(i) + ": " + errs[i]);
        // the exchange: one all_gather of nq x R keys per rank, ordered behind each shard's search on its own stream
        if (!m->comms.empty()) {
            nccl_check(nccl().GroupStart(), "ncclGroupStart");
            for (int i = 0; i < ndev; ++i)
                nccl_check(nccl().AllGather(m->keys[i].p, m->gathered[i].p, nr, /*ncclUint64*/ 5, m->comms[i], m->streams[i]),
                           "ncclAllGather");
            nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
        } else { // one device (or the same-device test mode): the "gather" is device-to-device copies in rank order
            for (int i = 1; i < ndev; ++i) {
                QADC_CUDA_CHECK(cudaSetDevice(m->devices[i]));
                QADC_CUDA_CHECK(cudaStreamSynchronize(m->streams[i]));
            }
            QADC_CUDA_CHECK(cudaSetDevice(m->devices[0]));
            for (int i = 0; i < ndev; ++i)
                QADC_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(m->gathered[0].p) + size_t(i) * nr * 8, m->keys[i].p, nr * 8,
                                                cudaMemcpyDeviceToDevice, m->streams[0]));
        }
        // merge on device 0 (every rank holds the gathered lists; the reference's caller wants ONE result)
        const int rc = qadc_merge_topk_device(static_cast<const uint64_t*>(m->gathered[0].p), uint32_t(ndev), nq, r,
                                              static_cast<const float*>(m->map[0].p), params->flags & QADC_FLAG_FMA_UNQUANTIZE,
                                              static_cast<uint32_t*>(m->out_ids.p), static_cast<float*>(m->out_dists.p),
                                              static_cast<uint32_t*>(m->out_counts.p), m->devices[0], m->streams[0]);
        if (rc != QADC_OK) throw Error(rc, qadc_last_error());
        QADC_CUDA_CHECK(cudaSetDevice(m->devices[0]));
        QADC_CUDA_CHECK(cudaMemcpyAsync(out_ids, m->out_ids.p, nr * 4, cudaMemcpyDeviceToHost, m->streams[0]));
        QADC_CUDA_CHECK(cudaMemcpyAsync(out_dists, m->out_dists.p, nr * 4, cudaMemcpyDeviceToHost, m->streams[0]));
        QADC_CUDA_CHECK(cudaMemcpyAsync(out_counts, m->out_counts.p, size_t(nq) * 4, cudaMemcpyDeviceToHost, m->streams[0]));
        for (int i = 0; i < ndev; ++i) { // the other ranks' collectives must have completed before the buffers are reused
            QADC_CUDA_CHECK(cudaSetDevice(m->devices[i]));
            QADC_CUDA_CHECK(cudaStreamSynchronize(m->streams[i]));
        }
    });
}

int qadc_multi_info(const qadc_multi* m, int* ndev, uint64_t* count, int* uses_nccl) {
    if (!m) return QADC_ERR_INPUT;
    if (ndev) *ndev = m->ndev;
    if (count) *count = m->count;
    if (uses_nccl) *uses_nccl = m->comms.empty() ? 0 : 1;
    return QADC_OK;
}

void qadc_multi_close(qadc_multi* m) { delete m; }

} // extern "C"
