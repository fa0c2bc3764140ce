// io.cu -- "next" row N1: open the reference's on-disk index containers directly.
//
// The reference's containers (io.hpp:17-22, all little-endian, format version 1):
//   QADC  codebook            magic, version, spec, per-subquantizer centroid matrices     io.hpp:204-223
//   QPKD  packed code lists   magic, version, spec hash (FNV-1a of the spec bytes), word width,
//                             block length, list count, then per list: u64 count + blocks   io.hpp:239-272
//   QFLT  flat index          magic, version, QADC, QPKD with exactly one list              io.hpp:276-295
//   QIVF  IVF index           magic, version, QADC, u32 K, K*dims floats, QPKD with K lists,
//                             then the per-list u32 id arrays                                io.hpp:297-326
// The packed blocks inside a QPKD section ARE the PackedList byte streams the C ABI consumes, so the
// loader only parses headers and passes pointers into the file image to qadc_flat_open / qadc_ivf_open;
// the re-layout into the device format happens on the GPU (layout.cu / ivf.cu).  No host re-pack.
// Error classes follow io.hpp: bad magic / version / truncation -> io_error (8); spec structure,
// allocation, hash, scheme or list-count mismatch -> corruption_error (6); bad widths -> invalid_spec (3).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace qadc {

void parse_spec(uint32_t dims, const std::string& text, qadc_spec& out);

namespace {

struct Reader {
    const uint8_t* p;
    size_t n, at = 0;
    template <class T>
    T get() {
        if (at + sizeof(T) > n) throw Error(QADC_ERR_IO, "unexpected end of file");
        T v;
        std::memcpy(&v, p + at, sizeof(T));
        at += sizeof(T);
        return v;
    }
    const uint8_t* bytes(size_t k) {
        if (k > n - at) throw Error(QADC_ERR_IO, "unexpected end of file");
        const uint8_t* r = p + at;
        at += k;
        return r;
    }
    void magic(const char m[4], const char* what) {
        if (std::memcmp(bytes(4), m, 4) != 0) throw Error(QADC_ERR_IO, std::string("bad magic: not a ") + what + " file");
    }
};

uint64_t fnv1a(const uint8_t* p, size_t n) { // io.hpp:60-67
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

// read_spec (io.hpp:180-195); also returns the serialized spec bytes' hash (spec_hash, io.hpp:197-202)
qadc_spec read_spec(Reader& r, uint64_t* hash) {
    const size_t begin = r.at;
    const uint32_t dims = r.get<uint32_t>();
    const uint32_t ngroups = r.get<uint32_t>();
    const uint32_t g = r.get<uint32_t>();
    if (g == 0 || ngroups == 0 || g > 16) throw Error(QADC_ERR_CORRUPTION, "spec: bad group structure");
    const uint8_t* widths = r.bytes(g);
    std::string text = std::to_string(uint64_t(ngroups) * g) + "x{";
    for (uint32_t i = 0; i < g; ++i) text += (i ? "," : "") + std::to_string(unsigned(widths[i]));
    text += "}";
    qadc_spec s;
    parse_spec(dims, text, s); // allocate_dims: invalid_spec on bad widths / sums / too few dims
    for (uint32_t j = 0; j < s.m; ++j)
        if (r.get<uint32_t>() != s.dim_alloc[j]) throw Error(QADC_ERR_CORRUPTION, "spec: dimension allocation mismatch");
    *hash = fnv1a(r.p + begin, r.at - begin);
    return s;
}

struct Codebook {
    qadc_spec spec;
    uint64_t hash;
    const float* data;
};

Codebook read_codebook(Reader& r) { // load_codebook, io.hpp:212-223
    r.magic("QADC", "codebook");
    if (r.get<uint32_t>() != 1) throw Error(QADC_ERR_IO, "codebook: unsupported format version");
    Codebook cb;
    cb.spec = read_spec(r, &cb.hash);
    cb.data = reinterpret_cast<const float*>(r.bytes(size_t(cb.spec.cb_floats) * 4));
    return cb;
}

struct PackedSection {
    std::vector<uint64_t> count, byte_off; // byte_off relative to `base`
    const uint8_t* base;
};

PackedSection read_packed(Reader& r, const Codebook& cb) { // read_packed_section, io.hpp:253-272
    r.magic("QPKD", "packed-codes");
    if (r.get<uint32_t>() != 1) throw Error(QADC_ERR_IO, "packed section: unsupported format version");
    if (r.get<uint64_t>() != cb.hash)
        throw Error(QADC_ERR_CORRUPTION, "packed section: spec hash mismatch (codes were built for another spec)");
    const uint32_t ww = r.get<uint32_t>(), bl = r.get<uint32_t>();
    if (ww != cb.spec.word_width || bl != cb.spec.block_len)
        throw Error(QADC_ERR_CORRUPTION, "packed section: packing scheme mismatch");
    const uint32_t nlists = r.get<uint32_t>();
    PackedSection ps;
    ps.base = r.p;
    ps.count.resize(nlists);
    ps.byte_off.resize(nlists);
    // A count is untrusted input: it must fit the bytes that are actually left in the file (this also keeps the
    // size arithmetic from wrapping -- a crafted count like 2^62 would otherwise multiply to a small number) and ids
    // are uint32.  The reference fails with io_error on the truncated read (io.hpp:262-268).
    const uint64_t block_bytes = uint64_t(cb.spec.groups) * cb.spec.block_len * (cb.spec.word_width / 8);
    for (uint32_t l = 0; l < nlists; ++l) {
        ps.count[l] = r.get<uint64_t>();
        ps.byte_off[l] = r.at;
        const uint64_t max_blocks = (r.n - r.at) / block_bytes;
        if (ps.count[l] > 0xFFFFFFFFull || (ps.count[l] + cb.spec.block_len - 1) / cb.spec.block_len > max_blocks)
            throw Error(QADC_ERR_IO, "unexpected end of file");
        r.bytes(size_t(qadc_packed_bytes(&cb.spec, ps.count[l])));
    }
    return ps;
}

// Read-only mapping of the container: the packed blocks go from the page cache to the device in the open
// functions' chunked copies, without a second host copy of the whole file (a C5-size QIVF is ~6 GB).
struct Mapping {
    const uint8_t* p = nullptr;
    size_t n = 0;
    explicit Mapping(const char* path) {
        const int fd = ::open(path, O_RDONLY);
        if (fd < 0) throw Error(QADC_ERR_IO, std::string("cannot open ") + path);
        struct stat sb;
        if (::fstat(fd, &sb) != 0 || !S_ISREG(sb.st_mode)) {
            ::close(fd);
            throw Error(QADC_ERR_IO, std::string("cannot stat ") + path);
        }
        n = size_t(sb.st_size);
        if (n) {
            void* m = ::mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
            if (m == MAP_FAILED) {
                ::close(fd);
                throw Error(QADC_ERR_IO, std::string("cannot map ") + path);
            }
            ::madvise(m, n, MADV_SEQUENTIAL);
            p = static_cast<const uint8_t*>(m);
        }
        ::close(fd);
    }
    Mapping(const Mapping&) = delete;
    Mapping& operator=(const Mapping&) = delete;
    ~Mapping() {
        if (p) ::munmap(const_cast<uint8_t*>(p), n);
    }
};

} // namespace

// Returns through the ordinary open functions; the mapping only has to live until they return.
int open_index_file(const char* path, int device, qadc_index** out) {
    const Mapping img(path);
    Reader r{img.p, img.n};
    if (img.n < 4) throw Error(QADC_ERR_IO, "bad magic: not an index file");
    const bool flat = std::memcmp(img.p, "QFLT", 4) == 0;
    const bool ivf = std::memcmp(img.p, "QIVF", 4) == 0;
    if (!flat && !ivf) throw Error(QADC_ERR_IO, "bad magic: not an index file"); // peek_index_kind, io.hpp:330-338
    r.bytes(4);
    if (r.get<uint32_t>() != 1) throw Error(QADC_ERR_IO, flat ? "flat index: unsupported format version" : "ivf index: unsupported format version");
    const Codebook cb = read_codebook(r);
    if (flat) {
        const PackedSection ps = read_packed(r, cb);
        if (ps.count.size() != 1) throw Error(QADC_ERR_CORRUPTION, "flat index: expected exactly one list");
        return qadc_flat_open(&cb.spec, cb.data, ps.base + ps.byte_off[0], ps.count[0], 0, nullptr, 0, 0, device, out);
    }
    const uint32_t k = r.get<uint32_t>();
    const float* coarse = reinterpret_cast<const float*>(r.bytes(size_t(k) * cb.spec.dims * 4));
    const PackedSection ps = read_packed(r, cb);
    if (ps.count.size() != k) throw Error(QADC_ERR_CORRUPTION, "ivf index: list count does not match K");
    std::vector<uint64_t> id_off(k);
    uint64_t total = 0;
    for (uint32_t c = 0; c < k; ++c) {
        id_off[c] = total;
        total += ps.count[c];
    }
    if (total > 0xFFFFFFFFull) throw Error(QADC_ERR_CORRUPTION, "ivf index: more than 2^32 vectors (ids are 32-bit)");
    const uint32_t* ids = reinterpret_cast<const uint32_t*>(r.bytes(size_t(total) * 4));
    return qadc_ivf_open(&cb.spec, cb.data, coarse, k, ps.base, ps.byte_off.data(), id_off.data(), ps.count.data(), ids,
                         nullptr, nullptr, nullptr, nullptr, device, out);
}

} // namespace qadc
