// spec.cu -- host-side quantizer-structure handling: the spec grammar, the
// proportional dimension split and the packing scheme, flattened into qadc_spec.
// Mirrors parse_spec_string (pqspec.hpp:24-55), allocate_dims (pqspec.hpp:119-167)
// and PackingScheme::for_spec (layout.hpp:27-43): same accepted strings, same
// numbers, same error class (invalid_spec_error -> QADC_ERR_INVALID_SPEC).
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace qadc {

static Error bad_spec(const std::string& text, const char* why) {
    return Error(QADC_ERR_INVALID_SPEC, "bad spec string '" + text + "': " + why +
                                            " (expected <m>x{<w>(,<w>)*}, e.g. 16x{4,4}, 12x{6,6,4}, 8x{8,8}, 8x{8})");
}

static bool parse_uint(const std::string& tok, uint64_t limit, uint64_t& value) {
    if (tok.empty()) return false;
    value = 0;
    for (char c : tok) {
        if (c < '0' || c > '9') return false;
        value = value * 10 + uint64_t(c - '0');
        if (value > limit) return false;
    }
    return true;
}

void parse_spec(uint32_t dims, const std::string& text, qadc_spec& out) {
    std::memset(&out, 0, sizeof out);
    const size_t x = text.find('x');
    if (x == std::string::npos || x == 0) throw bad_spec(text, "missing 'x'");
    uint64_t m = 0;
    if (!parse_uint(text.substr(0, x), 0xffffffffull, m) || m == 0) throw bad_spec(text, "bad subquantizer count");
    const std::string body = text.substr(x + 1);
    if (body.size() < 3 || body.front() != '{' || body.back() != '}') throw bad_spec(text, "missing {...}");
    std::vector<uint8_t> widths;
    size_t pos = 1;
    const size_t end = body.size() - 1;
    while (pos < end) {
        size_t comma = body.find(',', pos);
        if (comma == std::string::npos || comma > end) comma = end;
        uint64_t w = 0;
        if (!parse_uint(body.substr(pos, comma - pos), 1000, w)) throw bad_spec(text, "bad width");
        if (w < 1 || w > 8) throw bad_spec(text, "widths must be in [1,8]");
        widths.push_back(uint8_t(w));
        if (comma == end) break;
        pos = comma + 1;
        if (pos >= end) throw bad_spec(text, "trailing comma");
    }
    if (widths.empty()) throw bad_spec(text, "empty width list");

    const size_t g = widths.size();
    if (m % g != 0)
        throw Error(QADC_ERR_INVALID_SPEC, "subquantizer count " + std::to_string(m) +
                                               " is not a multiple of the group size " + std::to_string(g));
    uint32_t sum = 0;
    for (uint8_t w : widths) sum += w;
    if (sum != 8 && sum != 16 && sum != 15) // 15 = padded triple-5 word
        throw Error(QADC_ERR_INVALID_SPEC,
                    "group bit widths of " + text + " sum to " + std::to_string(sum) +
                        "; supported packings are 8-bit bytes and 16-bit words");
    if (dims < m)
        throw Error(QADC_ERR_INVALID_SPEC, "cannot split " + std::to_string(dims) + " dimensions across " +
                                               std::to_string(m) + " subquantizers");
    if (m > QADC_MAX_SUBS || g > QADC_MAX_GROUP)
        throw Error(QADC_ERR_INVALID_SPEC, "spec exceeds the ABI limits (64 subquantizers, 16 per group)");

    out.dims = dims;
    out.m = uint32_t(m);
    out.g = uint32_t(g);
    out.groups = uint32_t(m / g);
    out.word_width = sum <= 8 ? 8 : 16;
    const uint64_t total_bits = uint64_t(sum) * out.groups;
    uint64_t assigned = 0;
    for (uint32_t j = 0; j < out.m; ++j) {
        out.bits[j] = widths[j % g];
        out.dim_alloc[j] = uint32_t(uint64_t(dims) * out.bits[j] / total_bits);
        assigned += out.dim_alloc[j];
    }
    uint64_t leftover = dims - assigned;
    out.exact = leftover == 0;
    for (uint32_t j = 0; leftover > 0; j = (j + 1) % out.m, --leftover) out.dim_alloc[j] += 1;
    for (uint32_t j = 0; j < out.m; ++j)
        if (out.dim_alloc[j] == 0)
            throw Error(QADC_ERR_INVALID_SPEC, "dimension allocation left a subquantizer empty");
    uint32_t doff = 0, eoff = 0, coff = 0;
    for (uint32_t j = 0; j < out.m; ++j) {
        out.dim_off[j] = doff;
        doff += out.dim_alloc[j];
        out.ent_off[j] = eoff;
        eoff += 1u << out.bits[j];
        out.cb_off[j] = coff;
        coff += (1u << out.bits[j]) * out.dim_alloc[j];
    }
    out.total_entries = eoff;
    out.cb_floats = coff;
    uint8_t o = 0;
    for (size_t i = 0; i < g; ++i) {
        out.widths[i] = widths[i];
        out.offsets[i] = o;
        o = uint8_t(o + widths[i]);
    }
    out.block_len = out.word_width == 16 ? 32 : (g == 1 ? 64 : 16);
}

// Structural sanity of a caller-filled qadc_spec (the ABI lets callers build one by hand).
void validate_spec(const qadc_spec& s) {
    if (s.m == 0 || s.g == 0 || s.m > QADC_MAX_SUBS || s.g > QADC_MAX_GROUP || s.m % s.g != 0 ||
        s.groups != s.m / s.g)
        throw Error(QADC_ERR_INVALID_SPEC, "spec: inconsistent m / g / groups");
    if (s.word_width != 8 && s.word_width != 16) throw Error(QADC_ERR_INVALID_SPEC, "spec: word width must be 8 or 16");
    uint32_t sum = 0, eoff = 0, coff = 0, doff = 0;
    for (uint32_t i = 0; i < s.g; ++i) {
        if (s.widths[i] < 1 || s.widths[i] > 8 || s.offsets[i] != sum)
            throw Error(QADC_ERR_INVALID_SPEC, "spec: bad group widths / offsets");
        sum += s.widths[i];
    }
    if (sum > s.word_width) throw Error(QADC_ERR_INVALID_SPEC, "spec: group does not fit its word");
    for (uint32_t j = 0; j < s.m; ++j) {
        if (s.bits[j] != s.widths[j % s.g] || s.ent_off[j] != eoff || s.cb_off[j] != coff || s.dim_off[j] != doff ||
            s.dim_alloc[j] == 0)
            throw Error(QADC_ERR_INVALID_SPEC, "spec: per-subquantizer arrays are inconsistent");
        eoff += 1u << s.bits[j];
        coff += (1u << s.bits[j]) * s.dim_alloc[j];
        doff += s.dim_alloc[j];
    }
    if (eoff != s.total_entries || coff != s.cb_floats || doff != s.dims)
        throw Error(QADC_ERR_INVALID_SPEC, "spec: totals are inconsistent");
    const uint32_t bl = s.word_width == 16 ? 32 : (s.g == 1 ? 64 : 16);
    if (s.block_len != bl) throw Error(QADC_ERR_INVALID_SPEC, "spec: block length does not match the packing family");
}

DevSpec make_dev_spec(const qadc_spec& s, uint32_t rows) {
    DevSpec d;
    std::memset(&d, 0, sizeof d);
    d.dims = s.dims;
    d.m = rows * s.g;
    d.E = 0;
    d.cb_floats = s.cb_floats;
    d.word_width = s.word_width;
    d.qmax = s.word_width == 8 ? 255u : 65535u;
    d.code_bytes = rows * (s.word_width / 8);
    d.code_stride = (d.code_bytes + 7u) & ~7u;
    if (d.code_stride == 0) d.code_stride = 8;
    for (uint32_t j = 0; j < d.m; ++j) {
        d.bits[j] = s.widths[j % s.g];
        d.bitpos[j] = uint8_t((j / s.g) * s.word_width + s.offsets[j % s.g]);
        d.ent_off[j] = d.E;
        d.E += 1u << d.bits[j];
        if (j < s.m) {
            d.dim_off[j] = s.dim_off[j];
            d.dim_alloc[j] = s.dim_alloc[j];
            d.cb_off[j] = s.cb_off[j];
        }
    }
    return d;
}

} // namespace qadc
