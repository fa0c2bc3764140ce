// scan.cu -- the ADC scan kernels (the hot path).
//
// Reference semantics (scan_scalar.hpp:34-64): for every occupied code, fold the m
// quantized table entries selected by its subcodes with saturating adds at table
// width, starting from min(acc_init, q_max), and push (sum, id) into the bounded heap.
// The CPU kernels (scan_x86.hpp) put 16/32/64 CODES in the lanes of one register and
// shuffle one query's tables.  On the GPU the batch dimension is the QUERY:
//
//   * a CTA keeps the quantized tables of a TILE of queries ("LUT rows") resident in
//     shared memory, transposed to [entry][row] so that the 32 lanes of a warp, each
//     owning 1..8 rows, read one conflict-free 64..512-byte line per lookup;
//   * codes stream through a double-buffered shared-memory stage filled by bulk async
//     copies (cp.async.bulk + mbarrier); a warp takes one whole code at a time with a
//     broadcast load, so the code is read once per (warp, tile), not once per query;
//   * sums are accumulated WITHOUT per-step saturation in a wider type and compared
//     once: min(min(S,q)+x,q) == min(S+x,q) for unsigned terms.  u8
//     tables accumulate as packed fp16 pairs (HADD2; integers are exact up to 2048 and
//     every rounded value is far above any 8-bit threshold), u16 tables as fp32
//     (exact below 2^24) or int32;
//   * the accumulator starts at (bias - threshold - 1/2), so "sum <= threshold" is the
//     sign bit: one OR over a lane's accumulators decides whether ANY of its rows
//     admits the code;
//   * the rare admitted (row, code) pair is re-evaluated exactly in integers against
//     the reference-order table in global memory and appended to the query's candidate
//     list iff its (distance, id) key beats the query's current R-th best key -- the
//     CandidateHeap::push test (heap.hpp:46-47).  The in-loop test is only a filter
//     (it never drops a pair the exact test would admit), so results are exact by
//     construction whatever the filter's arithmetic.
#include <cuda_fp16.h>

#include <type_traits>

#include "scan_common.cuh"

namespace qadc {

// 12x{6,5,5} seen as 4 words x {6-bit table, 1024-entry table of (5,5) pair sums}: 1088 quad lines per tile
// (VAR_F16X4H_C8Q).  The hot loop has its own branch; exact re-evaluation uses the original geometry.
// (12x{6,6,4} has the same merged view: 6 bits, then 10 bits = the 6-bit and the 4-bit subcode; 12x{5,5,5}: 5 bits,
// then 10 bits.)  B0 = bits of a word's first subcode.
template <class ExactG, int B0_>
struct GeomQ6_10 {
    static constexpr bool RUNTIME = false;
    static constexpr int B0 = B0_;
    static constexpr int CW = 2, E = 1024 + (1 << B0), M = 8, STRIDE = 8, WORD = 16;
    using Exact = ExactG;
    __host__ __device__ static constexpr int bits(int) { return 0; }
    __host__ __device__ static constexpr int bitpos(int) { return 0; }
    __host__ __device__ static constexpr int ent_off(int) { return 0; }
};

using GeomQ655 = GeomQ6_10<GeomCT<16, 4, 6, 5, 5>, 6>;
using GeomQ664 = GeomQ6_10<GeomCT<16, 4, 6, 6, 4>, 6>;
using GeomQ555 = GeomQ6_10<GeomCT<16, 4, 5, 5, 5>, 5>;

// ------------------------------------------------------------------ policies --
// A policy fixes how table entries live in shared memory and how a lane accumulates.
//   QPL    rows (queries) owned by one lane;   TQ = 32*QPL rows per tile
//   ROWB   bytes of one [entry] line in shared memory = TQ * sizeof(entry)

// fp16 entries, 8 rows per lane (LDS.128).  CPW = 1: the 256-row tile of the u8 16x{4,4} scan.  CPW = 8: eight
// code groups of 4 lanes against a 32-row tile -- the same tile image as the 4-rows-per-lane variants, but one
// LDS.128 + 4 HADD2 per 8 rows instead of two LDS.64 + 4 HADD2, i.e. ~30 % fewer instructions per pair for the
// 2048-entry specs, which are issue bound once the pair layout has removed their bank conflicts.
// HIGH: conservative filter on the top bits of 16-bit tables (see PolF16x4H_T).  PAIR: pair-interleaved lines.
template <int CPW_, bool HIGH, bool PAIR_, bool DUP_ = false>
struct PolF16x8_T {
    static constexpr int CPW = CPW_;
    static constexpr bool PAIR = PAIR_;
    static constexpr bool DUP = DUP_; // every entry line twice, odd code groups read the second copy (see PolF16x4H_T)
    static constexpr int QPL = 8, TQ = 256 / CPW, ROWB = (512 / CPW) * (DUP ? 2 : 1),
                         LOG_ROWB = (CPW == 1 ? 9 : CPW == 2 ? 8 : CPW == 4 ? 7 : 6) + (DUP ? 1 : 0), LANE_B = 16;
    static constexpr bool EXACT_FILTER = !HIGH;
    using Entry = __half;
    struct Acc {
        __half2 h[4];
    };
    __device__ static void init(Acc& a, const float* t) { // t[s] = bias - thr - 0.5 (or +-BIG)
#pragma unroll
        for (int k = 0; k < 4; ++k) a.h[k] = __floats2half2_rn(t[2 * k], t[2 * k + 1]);
    }
    __device__ static void add(Acc& a, const char* p) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        a.h[0] = __hadd2(a.h[0], *reinterpret_cast<const __half2*>(&v.x));
        a.h[1] = __hadd2(a.h[1], *reinterpret_cast<const __half2*>(&v.y));
        a.h[2] = __hadd2(a.h[2], *reinterpret_cast<const __half2*>(&v.z));
        a.h[3] = __hadd2(a.h[3], *reinterpret_cast<const __half2*>(&v.w));
    }
    __device__ static bool any(const Acc& a) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(a.h);
        return ((u[0] | u[1] | u[2] | u[3]) & 0x80008000u) != 0;
    }
    __device__ static bool hit(const Acc& a, int s) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(a.h);
        return (u[s >> 1] >> ((s & 1) * 16 + 15)) & 1u;
    }
    // exact accumulator value of slot s as fp32 (only meaningful when the slot admits, i.e. |v| < 1024)
    __device__ static float value(const Acc& a, int s) {
        return (s & 1) ? __high2float(a.h[s >> 1]) : __low2float(a.h[s >> 1]);
    }
    static constexpr float BIG = 30000.0f, HALF = HIGH ? 1.0f : 0.5f;
};
using PolF16x8 = PolF16x8_T<1, false, false>;
using PolF16x8_C8P = PolF16x8_T<8, false, true>;   // exact, 8-bit tables of 256 entries (8x{8}, merged 16x{4,4})
using PolF16x8H_C8P = PolF16x8_T<8, true, true>;   // conservative, 16-bit tables of 256 entries (8x{8,8})
using PolF16x8H_C8D = PolF16x8_T<8, true, false, true>; // conservative, duplicated lines (E <= 512: IVF 12x{6,5,5})

struct PolF32x2 { // u16 (or u8) tables, fp32 exact below 2^24
    static constexpr int CPW = 1;
    static constexpr int QPL = 2, TQ = 64, ROWB = 256, LOG_ROWB = 8, LANE_B = 8;
    static constexpr bool EXACT_FILTER = true;
    using Entry = float;
    struct Acc {
        float f[2];
    };
    __device__ static void init(Acc& a, const float* t) {
        a.f[0] = t[0];
        a.f[1] = t[1];
    }
    __device__ static void add(Acc& a, const char* p) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        a.f[0] = __fadd_rn(a.f[0], v.x);
        a.f[1] = __fadd_rn(a.f[1], v.y);
    }
    __device__ static bool any(const Acc& a) { return (__float_as_uint(a.f[0]) | __float_as_uint(a.f[1])) >> 31; }
    __device__ static bool hit(const Acc& a, int s) { return __float_as_uint(a.f[s]) >> 31; }
    __device__ static float value(const Acc& a, int s) { return a.f[s]; }
    static constexpr float BIG = 1.0e9f, HALF = 0.5f;
};

// u16 tables: fp16 image of the HIGH byte of every entry; conservative filter.  CPW = codes per warp
// step: the warp's lanes split into CPW groups, each group walks a DIFFERENT code of the same list
// against a tile of 128/CPW rows.  Bytes per wavefront and instructions per pair are unchanged, but
// short row groups (IVF: ~40 (query, cell) pairs per cell) waste far fewer padded rows.
// HIGH = false is the exact twin for 8-bit tables (entries <= 255 are exact in fp16, as in f16x8).
// DUP: every entry line is stored twice back to back (ROWB doubles); odd code groups read the second copy.
// With four groups of 8 lanes x 8 B, groups 0/2 then only touch banks 0-15 and groups 1/3 banks 16-31: a warp
// load is exactly two conflict-free wavefronts, where the dense layout needs 2.75 on average (the bank half
// is the parity of a data-dependent entry index).
// PAIR (32-row tiles, every table 256 entries): tables 2k / 2k+1 share 128-byte lines (low / high half) and the
// odd code groups of a warp walk each table pair in swapped order (their code bytes are swapped pairwise once per
// code), so at every step groups 0/2 and groups 1/3 read opposite bank halves: two conflict-free wavefronts per
// warp load with NO extra shared memory -- what DUP buys with doubled lines, for the specs whose tables are too
// large to double (8x{8,8}, 8x{8}, merged 16x{4,4}).
template <int CPW_, bool HIGH = true, bool DUP_ = false, bool PAIR_ = false>
struct PolF16x4H_T {
    static constexpr int CPW = CPW_;
    static constexpr bool DUP = DUP_;
    static constexpr bool PAIR = PAIR_;
    static constexpr int QPL = 4, TQ = 128 / CPW, ROWB = (256 / CPW) * (DUP ? 2 : 1),
                         LOG_ROWB = (CPW == 1 ? 8 : CPW == 2 ? 7 : 6) + (DUP ? 1 : 0), LANE_B = 8;
    static constexpr bool EXACT_FILTER = !HIGH;
    using Entry = __half;
    struct Acc {
        __half2 h[2];
    };
    __device__ static void init(Acc& a, const float* t) {
        a.h[0] = __floats2half2_rn(t[0], t[1]);
        a.h[1] = __floats2half2_rn(t[2], t[3]);
    }
    __device__ static void add(Acc& a, const char* p) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        a.h[0] = __hadd2(a.h[0], *reinterpret_cast<const __half2*>(&v.x));
        a.h[1] = __hadd2(a.h[1], *reinterpret_cast<const __half2*>(&v.y));
    }
    __device__ static bool any(const Acc& a) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(a.h);
        return ((u[0] | u[1]) & 0x80008000u) != 0;
    }
    __device__ static bool hit(const Acc& a, int s) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(a.h);
        return (u[s >> 1] >> ((s & 1) * 16 + 15)) & 1u;
    }
    // only used when the filter is exact (HIGH == false)
    __device__ static float value(const Acc& a, int s) {
        return (s & 1) ? __high2float(a.h[s >> 1]) : __low2float(a.h[s >> 1]);
    }
    // HIGH: all terms are integers up to 2047, the start is bias' - thr' - 1 (sum' <= thr' <=> negative), every
    // value in [-2048, 2047] is exact in fp16 and anything larger stays positive.  Exact twin: the usual - 1/2.
    static constexpr float BIG = 30000.0f, HALF = HIGH ? 1.0f : 0.5f;
};
// Quad-interleaved 16-row tile of the merged 12x{6,5,5} scan: a 128-byte line holds one entry of the four words'
// tables (32 bytes = 16 rows each); 16 code groups of 2 lanes, 8 rows per lane (LDS.128).  Group g sees its code
// rotated by g mod 4 words, so at step k it reads word (k + g) mod 4's table, i.e. bank quarter (k + g) mod 4:
// every quarter serves exactly four groups -- 512 bytes in four conflict-free wavefronts.  (The 4-rows-per-lane
// twin measured 1.53 T pairs/s on C2, this one 1.78: with 16-row tiles the per-code work dominates the issue slots.)
template <class P, class = void>
struct quad_of : std::false_type {};
template <class P>
struct quad_of<P, std::void_t<decltype(P::QUAD)>> : std::bool_constant<P::QUAD> {};

struct PolQ655 : PolF16x8_T<16, true, false> {
    static constexpr bool QUAD = true;
    static constexpr int TQ = 16, ROWB = 128, LOG_ROWB = 7, LANE_B = 16;
};

// The unmerged sibling for the IVF path (tiles of the merged view are 139 KB, far too much per (query, cell) row):
// the same quad lines and rotated codes with the spec's own 12 tables -- a 16-row tile is E/4 lines of 128 bytes
// (16 KB for 12x{6,5,5}), so a cell's last, partly filled tile wastes at most 15 rows instead of 31.
struct PolQU : PolF16x8_T<16, true, false> {
    static constexpr bool QUADU = true;
    static constexpr int TQ = 16, ROWB = 128, LOG_ROWB = 7, LANE_B = 16;
};
template <class P, class = void>
struct quadu_of : std::false_type {};
template <class P>
struct quadu_of<P, std::void_t<decltype(P::QUADU)>> : std::bool_constant<P::QUADU> {};
// geometry view: a quarter of the entries per line set; the exact re-evaluation keeps the spec's geometry
template <class Gx>
struct GeomQU : Gx {
    static constexpr int E = Gx::E / 4;
    using Exact = Gx;
};

using PolF16x4H = PolF16x4H_T<1>;
using PolF16x4H_C2 = PolF16x4H_T<2>;
using PolF16x4H_C4 = PolF16x4H_T<4>;
using PolF16x4_C4 = PolF16x4H_T<4, false>;
using PolF16x4H_C4D = PolF16x4H_T<4, true, true>;

template <class P, class = void>
struct pair_of : std::false_type {};
template <class P>
struct pair_of<P, std::void_t<decltype(P::PAIR)>> : std::bool_constant<P::PAIR> {};

template <class P, class = void>
struct dup_of : std::false_type {};
template <class P>
struct dup_of<P, std::void_t<decltype(P::DUP)>> : std::bool_constant<P::DUP> {};

struct PolU16x1 { // any width, u16 entries, int32 accumulate
    static constexpr int CPW = 1;
    static constexpr int QPL = 1, TQ = 32, ROWB = 64, LOG_ROWB = 6, LANE_B = 2;
    static constexpr bool EXACT_FILTER = true;
    using Entry = unsigned short;
    struct Acc {
        int v;
    };
    __device__ static void init(Acc& a, const float* t) { a.v = int(floorf(t[0])); } // bias - thr - 1
    __device__ static void add(Acc& a, const char* p) { a.v += int(*reinterpret_cast<const unsigned short*>(p)); }
    __device__ static bool any(const Acc& a) { return a.v < 0; }
    __device__ static bool hit(const Acc& a, int) { return a.v < 0; }
    __device__ static float value(const Acc& a, int) { return float(a.v) + 0.5f; } // init was floor(t) = t - 1/2
    static constexpr float BIG = 1.0e9f, HALF = 0.5f;
};

struct PolU8x1 { // any width; u16 tables keep only the HIGH byte: a conservative filter
    static constexpr int CPW = 1;
    static constexpr int QPL = 1, TQ = 32, ROWB = 32, LOG_ROWB = 5, LANE_B = 1;
    static constexpr bool EXACT_FILTER = false;
    using Entry = unsigned char;
    struct Acc {
        int v;
    };
    __device__ static void init(Acc& a, const float* t) { a.v = int(floorf(t[0])); }
    __device__ static void add(Acc& a, const char* p) { a.v += int(*reinterpret_cast<const unsigned char*>(p)); }
    __device__ static bool any(const Acc& a) { return a.v < 0; }
    __device__ static bool hit(const Acc& a, int) { return a.v < 0; }
    __device__ static float value(const Acc& a, int) { return float(a.v) + 0.5f; }
    // floor(bias/256) + sum floor(e/256) <= floor(thr/256) is necessary for bias + sum e <= thr
    static constexpr float BIG = 1.0e9f, HALF = 0.5f;
};

static constexpr int SCAN_WARPS = 16;                      // consumer warps
static constexpr int SCAN_CONSUMERS = SCAN_WARPS * 32;     // consumer threads
static constexpr int SCAN_THREADS = SCAN_CONSUMERS + 32;   // + one producer warp (TMA issue)
static constexpr int STAGE_BYTES = 8192;                   // one code stage buffer
static constexpr int NSTAGE = 4;
static constexpr int WQ_CAP = 64;                          // per-warp queue of flagged (row, code) pairs
static constexpr int WQ_ENTRY = 28;                        // ref (8) + code copy (8) + row, stage index, value (4 each)
static constexpr int WQ_BYTES = SCAN_WARPS * WQ_CAP * WQ_ENTRY;

// --------------------------------------------------------- exact admission --
// (exact_admit / exact_admit_ct live in scan_common.cuh)

// Admission of one flagged (row, code), run by one lane of a warp-wide flush (32 entries
// resolved at once, all lanes active).  When the in-loop filter is exact and the row has
// a finite, unsaturated threshold, the accumulator itself is exact (it is < 0, far
// inside the exactly representable range): bias + sum = acc + thr + 1/2, no re-evaluation.
// Otherwise (no threshold yet, saturated threshold, or the high-byte filter) fall back to
// the integer re-evaluation above.
template <class P>
__device__ __forceinline__ void admit_entry(const DevSpec* ds, const ScanArgs* a, float val, const uint8_t* code,
                                            uint32_t row, uint32_t id) {
    const uint32_t q = a->row_query ? a->row_query[row] : row;
    const uint64_t tk = a->thr_key[q];
    const uint32_t thr = uint32_t(tk >> 32);
    if (!P::EXACT_FILTER || tk == KEY_INF || thr >= ds->qmax) {
        exact_admit(ds, a, code, row, id);
        return;
    }
    const uint32_t d = uint32_t(val + float(thr) + 0.5f);
    const uint64_t key = make_key(d, id);
    if (key < tk) {
        const uint32_t slot = atomicAdd(&a->cand_count[q], 1u);
        if (slot < a->cap) a->cand[size_t(q) * a->cap + slot] = key;
        else a->overflow[q] = 1u;
    }
}

// ------------------------------------------------------------------- kernel --

template <class P, class G, int EARLY>
__global__ void __launch_bounds__(SCAN_THREADS, 1) scan_kernel(DevSpec ds_param, ScanArgs args_param) {
    constexpr int CIF = 2; // codes in flight per lane group (4 was measured slower on every workload)
    extern __shared__ __align__(1024) char smem[];
    // dynamic smem: tile_bufs x [E*ROWB) LUT tile | NSTAGE code stage buffers | per-warp queues
    __shared__ DevSpec s_ds;
    __shared__ ScanArgs s_args;
    __shared__ __align__(8) uint64_t s_full[NSTAGE], s_empty[NSTAGE];
    __shared__ __align__(8) uint64_t s_tfull[2], s_tempty[2]; // LUT tile buffers: arrival / release
    __shared__ float s_thr[2][P::TQ];                          // per tile buffer: accumulator start of every row

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_ds = ds_param;
        s_args = args_param;
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&s_full[i], 1);           // the producer's arrive.expect_tx
            mbar_init(&s_empty[i], SCAN_WARPS); // one arrival per consumer warp
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_tfull[i], 2); // the tile's expect_tx + the accumulator starts' arrive
            mbar_init(&s_tempty[i], SCAN_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const DevSpec* ds = &s_ds;
    const ScanArgs* a = &s_args;

    const uint32_t E = G::RUNTIME ? ds->E : uint32_t(G::E);
    const uint32_t stride = ds->code_stride;
    const uint32_t tile_bytes = E * P::ROWB;
    const uint32_t tile_bufs = a->tile_bufs == 2 ? 2u : 1u;
    char* stage = smem + size_t(tile_bufs) * tile_bytes;
    const uint32_t stage_codes = STAGE_BYTES / stride;

    // contiguous slice of the job list for this CTA
    const uint32_t j_begin = a->cta_begin ? a->cta_begin[blockIdx.x] : uint32_t(uint64_t(a->n_jobs) * blockIdx.x / gridDim.x);
    const uint32_t j_end = a->cta_begin ? a->cta_begin[blockIdx.x + 1] : uint32_t(uint64_t(a->n_jobs) * (blockIdx.x + 1) / gridDim.x);

    // ============================ producer warp: stream codes with TMA bulk copies ==========
    // Lane 0 issues the copies; at a tile switch all 32 lanes gather the rows' accumulator starts
    // (row -> query -> threshold is a chain of dependent global loads: done here, one tile ahead, it
    // is off the consumers' critical path).
    if (warp == SCAN_WARPS) {
        uint32_t it = 0; // running stage-fill counter, mirrored by the consumers
        uint32_t tseq = 0, prev_rb = 0xFFFFFFFFu, prev_nr = 0; // LUT tiles issued so far
        ScanJob cur{};
        if (j_begin < j_end) cur = a->jobs[j_begin];
        for (uint32_t ji = j_begin; ji < j_end; ++ji) {
            const ScanJob job = cur;
            if (ji + 1 < j_end) cur = a->jobs[ji + 1]; // in flight while this job is issued
            if (job.n_codes == 0 || job.n_rows == 0) continue;
            if (job.row_begin != prev_rb || job.n_rows != prev_nr) {
                // next LUT tile: the image [entry][row] was prepared up front (tilepack.cu / ivf_lut.cu), so it
                // is a few bulk copies.  With two buffers it lands while the consumers still scan the
                // previous job; with one, the wait below is the hand-over.
                prev_rb = job.row_begin;
                prev_nr = job.n_rows;
                const uint32_t tb = tile_bufs == 2 ? (tseq & 1u) : 0u, use = tile_bufs == 2 ? (tseq >> 1) : tseq;
                mbar_wait(&s_tempty[tb], (use & 1u) ^ 1u); // first use passes immediately
                if (lane == 0) {
                    const char* src = reinterpret_cast<const char*>(a->tile_lut) + size_t(job.row_begin / P::TQ) * tile_bytes;
                    char* dst = smem + size_t(tb) * tile_bytes;
                    mbar_expect_tx(&s_tfull[tb], tile_bytes);
                    for (uint32_t off = 0; off < tile_bytes; off += 32768u)
                        bulk_g2s(dst + off, src + off, min(32768u, tile_bytes - off), &s_tfull[tb]);
                }
                __syncwarp(); // the buffer (and its s_thr row) is free: gather while the tile is in flight
                // accumulator start per row: bias - threshold - 1/2 (sign bit <=> admitted)
                for (uint32_t r = lane; r < uint32_t(P::TQ); r += 32) {
                    float t = P::BIG; // rows past the tile / padding rows never admit
                    if (r < job.n_rows) {
                        const uint32_t row = job.row_begin + r;
                        const uint32_t q = a->row_query ? a->row_query[row] : row;
                        if (q != 0xFFFFFFFFu) {
                            const uint64_t tk = a->thr_key[q];
                            uint32_t thr = uint32_t(tk >> 32);
                            uint32_t bias = a->row_bias ? min(a->row_bias[row], ds->qmax) : 0u;
                            if (tk == KEY_INF || thr >= ds->qmax) t = -P::BIG; // heap not full / worst saturated: admit all
                            else {
                                if (!P::EXACT_FILTER && ds->word_width == 16) {
                                    thr >>= a->filter_shift;
                                    bias >>= a->filter_shift;
                                }
                                t = float(bias) - float(thr) - P::HALF;
                            }
                        }
                    }
                    s_thr[tb][r] = t;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_tfull[tb]); // release: the s_thr stores above are visible to waiters
                ++tseq;
            }
            // the whole warp walks the stages in lockstep, all lanes polling the barrier; lane 0 alone issues the
            // copies.  Measured on the 8x{8,8} scan: a long-lived split (lane 0 in the stage loop, 31 lanes
            // parked at the next __syncwarp) costs 5 % of the kernel, a lane-0 poll + shuffle broadcast as much.
            const uint8_t* gcodes = a->codes + job.code_off * stride;
            const uint32_t n_sub = (job.n_codes + stage_codes - 1) / stage_codes;
            for (uint32_t sub = 0; sub < n_sub; ++sub, ++it) {
                const uint32_t b = it % NSTAGE;
                mbar_wait(&s_empty[b], ((it / NSTAGE) & 1u) ^ 1u); // first lap passes immediately
                if (lane == 0) {
                    const uint32_t first = sub * stage_codes;
                    const uint32_t cnt = min(stage_codes, job.n_codes - first);
                    const uint32_t bytes = (cnt * stride + 15u) & ~15u;
                    mbar_expect_tx(&s_full[b], bytes);
                    bulk_g2s(stage + size_t(b) * STAGE_BYTES, gcodes + size_t(first) * stride, bytes, &s_full[b]);
                }
                __syncwarp();
            }
        }
        return;
    }

    // ============================ consumer warps ==============================================
    uint32_t cur_row_begin = 0xFFFFFFFFu, cur_n_rows = 0;
    uint32_t tseq = 0, it = 0;
    const char* tile = smem;
    typename P::Acc acc0;
    {
        float t[P::QPL];
#pragma unroll
        for (int s = 0; s < P::QPL; ++s) t[s] = P::BIG;
        P::init(acc0, t);
    }
    constexpr uint32_t LPC = 32 / P::CPW;             // lanes per code
    const uint32_t lane_in = lane % LPC, lane_code = lane / LPC;
    const uint32_t lane_off = lane_in * P::LANE_B + (dup_of<P>::value ? (lane_code & 1u) * (P::ROWB / 2) : 0u);
    // pair layout: even tables sit in the half (group parity), odd tables in the other one; odd groups see their
    // code with adjacent bytes swapped
    constexpr bool PAIR = pair_of<P>::value && !G::RUNTIME;
    const uint32_t lane_off_a = lane_in * P::LANE_B + (lane_code & 1u) * P::ROWB;
    const uint32_t lane_off_b = lane_in * P::LANE_B + ((lane_code & 1u) ^ 1u) * P::ROWB;
    // pairing unit: a 256-entry table (all-8-bit specs: odd groups swap adjacent code bytes) or one 16-bit word of an
    // irregular spec (odd groups swap the 16-bit halves of every 32-bit code word)
    constexpr bool PAIR_BYTES = G::RUNTIME || G::bits(0) == 8;
    const uint32_t swap_sel = (lane_code & 1u) ? (PAIR_BYTES ? 0x2301u : 0x1032u) : 0x3210u;
    // quad layout (merged 12x{6,5,5}): rotation of this code group and the bank quarter it reads at step k
    constexpr bool QUAD = quad_of<P>::value;
    constexpr bool QUADU = quadu_of<P>::value && !G::RUNTIME;
    const uint32_t quad_r = lane_code & 3u;
    uint32_t quad_off[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) quad_off[k] = ((uint32_t(k) + quad_r) & 3u) * 32u + lane_in * P::LANE_B;
    // per-warp queue of flagged pairs: ballot-compacted in the hot loop, resolved 32 at a time
    // 64-bit codes with a compile-time geometry (every named spec): the queue entry carries a copy of the code
    // and a global id reference, so it outlives its stage buffer and job -- the queue is drained only when 32
    // entries are waiting (full-warp admission) and once at the end.  Other shapes keep an index into the stage
    // buffer and drain at every stage end.
    // (Exact-filter variants admit straight from the accumulator value and rarely need the code: they keep the
    // cheaper stage-indexed entries; measured 4 % faster on the small-N 16x{4,4} workload.)
    constexpr bool COPY = !G::RUNTIME && G::CW == 2 && !P::EXACT_FILTER;
    char* wq_base = stage + NSTAGE * STAGE_BYTES + size_t(warp) * (WQ_CAP * WQ_ENTRY);
    uint64_t* wq_ref = reinterpret_cast<uint64_t*>(wq_base);
    uint2* wq_code = reinterpret_cast<uint2*>(wq_ref + WQ_CAP);
    uint32_t* wq_row = reinterpret_cast<uint32_t*>(wq_code + WQ_CAP);
    uint32_t* wq_idx = wq_row + WQ_CAP;
    float* wq_val = reinterpret_cast<float*>(wq_idx + WQ_CAP);
    uint32_t qn = 0; // warp-uniform fill level
    const uint32_t lanemask_lt = (1u << lane) - 1u;
    auto flush_copy = [&]() {
        __syncwarp();
        for (uint32_t base = 0; base < qn; base += 32) {
            const uint32_t e = base + lane;
            if (e < qn) {
                const uint64_t ref = wq_ref[e];
                const uint32_t id = a->ids ? a->ids[ref] : uint32_t(ref);
                const uint2 code = wq_code[e];
                if constexpr (COPY) exact_admit_ct<typename G::Exact>(ds, a, code.x, code.y, wq_row[e], id); // COPY implies a conservative filter
                else admit_entry<P>(ds, a, wq_val[e], reinterpret_cast<const uint8_t*>(&wq_code[e]), wq_row[e], id);
            }
        }
        __syncwarp();
        qn = 0;
    };

    ScanJob cur{};
    if (j_begin < j_end) cur = a->jobs[j_begin];
    for (uint32_t ji = j_begin; ji < j_end; ++ji) {
        const ScanJob job = cur;
        if (ji + 1 < j_end) cur = a->jobs[ji + 1]; // the next descriptor loads while this job is scanned
        if (job.n_codes == 0 || job.n_rows == 0) continue;

        // ---- switch to the next LUT tile when the row range changes ----
        if (job.row_begin != cur_row_begin || job.n_rows != cur_n_rows) {
            if (tseq > 0) { // this warp is done with the previous tile's buffer
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_tempty[tile_bufs == 2 ? ((tseq - 1) & 1u) : 0u]);
            }
            cur_row_begin = job.row_begin;
            cur_n_rows = job.n_rows;
            const uint32_t tb = tile_bufs == 2 ? (tseq & 1u) : 0u, use = tile_bufs == 2 ? (tseq >> 1) : tseq;
            mbar_wait(&s_tfull[tb], use & 1u); // every thread observes the tile's arrival itself
            tile = smem + size_t(tb) * tile_bytes;
            ++tseq;
            float t[P::QPL]; // per-lane accumulator starts, gathered by the producer warp
#pragma unroll
            for (int sl = 0; sl < P::QPL; ++sl) t[sl] = s_thr[tb][lane_in * P::QPL + sl];
            P::init(acc0, t);
        }

        // ---- consume the job's codes stage by stage ----
        const uint32_t n_sub = (job.n_codes + stage_codes - 1) / stage_codes;
        for (uint32_t sub = 0; sub < n_sub; ++sub, ++it) {
            const uint32_t b = it % NSTAGE;
            mbar_wait(&s_full[b], (it / NSTAGE) & 1u);
            const uint32_t first = sub * stage_codes;
            const uint32_t cnt = min(stage_codes, job.n_codes - first);
            const char* sb = stage + size_t(b) * STAGE_BYTES;
            auto flush = [&]() {
                __syncwarp();
                for (uint32_t base = 0; base < qn; base += 32) {
                    const uint32_t e = base + lane;
                    if (e < qn) {
                        const uint32_t i = wq_idx[e];
                        const uint32_t pos = first + i;
                        const uint32_t id = a->ids ? a->ids[job.ids_off + pos] : job.id_base + pos;
                        admit_entry<P>(ds, a, wq_val[e], reinterpret_cast<const uint8_t*>(sb + size_t(i) * stride),
                                       wq_row[e], id);
                    }
                }
                __syncwarp();
                qn = 0;
            };
            auto flag = [&](const typename P::Acc& acc, bool live, uint32_t i, uint32_t c0, uint32_t c1) {
                const bool h = live && P::any(acc);
                if (__any_sync(0xffffffffu, h)) {
                    // sparse flags: one OR-reduction tells which of the lane's QPL slots is flagged anywhere in
                    // the warp, and only those (typically one) pay a ballot
                    uint32_t hits = 0;
#pragma unroll
                    for (int sl = 0; sl < P::QPL; ++sl) hits |= (h && P::hit(acc, sl)) ? (1u << sl) : 0u;
                    uint32_t live_slots = __reduce_or_sync(0xffffffffu, hits);
                    while (live_slots) {
                        const uint32_t sl = __ffs(live_slots) - 1;
                        live_slots &= live_slots - 1;
                        const bool hs = (hits >> sl) & 1u;
                        const uint32_t m = __ballot_sync(0xffffffffu, hs);
                        if (qn + 32 > WQ_CAP) {
                            if constexpr (COPY) flush_copy();
                            else flush();
                        }
                        if (hs) {
                            const uint32_t slot = qn + __popc(m & lanemask_lt);
                            wq_row[slot] = job.row_begin + lane_in * P::QPL + sl;
                            if constexpr (COPY) { // the drain re-evaluates from the code: no accumulator value needed
                                wq_code[slot] = make_uint2(c0, c1);
                                wq_ref[slot] = a->ids ? job.ids_off + first + i : uint64_t(job.id_base + first + i);
                            } else {
                                float v = 0.0f;
#pragma unroll
                                for (int k = 0; k < P::QPL; ++k)
                                    if (uint32_t(k) == sl) v = P::value(acc, k);
                                wq_val[slot] = v;
                                wq_idx[slot] = i;
                            }
                        }
                        qn += __popc(m);
                    }
                }
            };

            if constexpr (!G::RUNTIME) {
                for (uint32_t i0 = warp * P::CPW + lane_code; i0 < cnt + lane_code; i0 += SCAN_WARPS * P::CPW * CIF) {
                    // (the loop bound is warp-uniform: i0 - lane_code is; lanes past the end are clamped + masked)
                    uint32_t cw[CIF][G::CW];
                    typename P::Acc acc[CIF];
#pragma unroll
                    for (int c = 0; c < CIF; ++c) {
                        const uint32_t i = min(i0 + c * SCAN_WARPS * P::CPW, cnt - 1); // clamp: duplicates are ignored below
                        const uint32_t* src = reinterpret_cast<const uint32_t*>(sb + size_t(i) * G::STRIDE);
                        if constexpr (G::CW == 2) {
                            const uint2 v = *reinterpret_cast<const uint2*>(src);
                            cw[c][0] = v.x;
                            cw[c][1] = v.y;
                        } else {
#pragma unroll
                            for (int k = 0; k < G::CW; ++k) cw[c][k] = src[k];
                        }
                        if constexpr (PAIR) {
#pragma unroll
                            for (int k = 0; k < G::CW; ++k) cw[c][k] = __byte_perm(cw[c][k], 0u, swap_sel);
                        }
                        acc[c] = acc0;
                    }
                    uint32_t orig[CIF][2]; // QUADU: the code as stored (the lookups use the rotated words)
                    if constexpr (QUADU) {
#pragma unroll
                        for (int c = 0; c < CIF; ++c) {
                            orig[c][0] = cw[c][0];
                            orig[c][1] = cw[c][1];
                            const uint32_t lo = (quad_r & 2u) ? cw[c][1] : cw[c][0];
                            const uint32_t hi = (quad_r & 2u) ? cw[c][0] : cw[c][1];
                            const uint32_t sh = (quad_r & 1u) * 16u;
                            cw[c][0] = __funnelshift_r(lo, hi, sh);
                            cw[c][1] = __funnelshift_r(hi, lo, sh);
                        }
                    }
                    if constexpr (QUAD) {
                        // word k of the rotated code = word (k + r) mod 4 of the stored one; per word the (5,5) pair
                        // index (bits 6..15) into the 1024-line section and the 6-bit index into the 64-line section
#pragma unroll
                        for (int c = 0; c < CIF; ++c) {
                            const uint32_t lo = (quad_r & 2u) ? cw[c][1] : cw[c][0];
                            const uint32_t hi = (quad_r & 2u) ? cw[c][0] : cw[c][1];
                            const uint32_t sh = (quad_r & 1u) * 16u;
                            const uint32_t wa = __funnelshift_r(lo, hi, sh), wb = __funnelshift_r(hi, lo, sh);
                            constexpr int b0 = G::RUNTIME ? 6 : (G::E - 1024 == 32 ? 5 : 6); // bits of a word's first subcode
                            constexpr uint32_t m10 = 1023u << 7, m6 = ((1u << b0) - 1u) << 7, base6 = 1024u * 128u;
                            P::add(acc[c], tile + (((wa << (7 - b0)) & m10) | quad_off[0]));
                            P::add(acc[c], tile + (((wa >> (9 + b0)) & m10) | quad_off[1]));
                            P::add(acc[c], tile + (((wb << (7 - b0)) & m10) | quad_off[2]));
                            P::add(acc[c], tile + (((wb >> (9 + b0)) & m10) | quad_off[3]));
                            P::add(acc[c], tile + base6 + (((wa << 7) & m6) | quad_off[0]));
                            P::add(acc[c], tile + base6 + (((wa >> 9) & m6) | quad_off[1]));
                            P::add(acc[c], tile + base6 + (((wb << 7) & m6) | quad_off[2]));
                            P::add(acc[c], tile + base6 + (((wb >> 9) & m6) | quad_off[3]));
                        }
                    } else
                    static_for<0, G::M>([&](auto J) {
                        constexpr int j = decltype(J)::value;
                        constexpr int bp = G::bitpos(j), nb = G::bits(j);
                        constexpr int logl = P::LOG_ROWB + (PAIR ? 1 : 0); // bytes per entry line (pair: two tables per line; quad: LOG_ROWB is the line)
                        constexpr int word = bp >> 5, sh = (bp & 31) - logl;
                        constexpr uint32_t mask = ((1u << nb) - 1u) << logl;
                        // pair layout: unit u = table (8-bit specs) or code word; line = (u >> 1) * block + offset in unit
                        constexpr int pblock = PAIR_BYTES ? 256 : G::ent_off(G::M / 4);
                        constexpr int unit = G::ent_off(j) / pblock, within = G::ent_off(j) - unit * pblock;
                        constexpr uint32_t imm = PAIR    ? uint32_t((unit >> 1) * pblock + within) * 2u * P::ROWB
                                                 : QUADU ? uint32_t(within) * P::ROWB // line = offset inside the word's tables
                                                         : uint32_t(G::ent_off(j)) * P::ROWB;
                        static_assert(!PAIR || PAIR_BYTES ? true : (G::M % 8 == 4 || G::M % 4 == 0), "pair layout: four code words");
                        static_assert(!PAIR || !PAIR_BYTES || (nb == 8 && (G::M & 1) == 0 && bp == 8 * j), "pair layout: 8-bit tables");
#pragma unroll
                        for (int c = 0; c < CIF; ++c) {
                            const uint32_t x = sh >= 0 ? (cw[c][word] >> (sh >= 0 ? sh : 0)) : (cw[c][word] << (sh < 0 ? -sh : 0));
                            const uint32_t off = (x & mask) | (PAIR    ? ((unit & 1) ? lane_off_b : lane_off_a)
                                                               : QUADU ? quad_off[unit & 3]
                                                                       : lane_off);
                            P::add(acc[c], tile + imm + off);
                        }
                    });
#pragma unroll
                    for (int c = 0; c < CIF; ++c) {
                        // the queue keeps the code as stored (the byte swap is an involution)
                        const uint32_t o0 = QUADU ? orig[c][0] : PAIR ? __byte_perm(cw[c][0], 0u, swap_sel) : cw[c][0];
                        const uint32_t o1 = QUADU  ? orig[c][1]
                                            : PAIR ? __byte_perm(cw[c][G::CW > 1 ? 1 : 0], 0u, swap_sel)
                                                   : cw[c][G::CW > 1 ? 1 : 0];
                        flag(acc[c], i0 + c * SCAN_WARPS * P::CPW < cnt, i0 + c * SCAN_WARPS * P::CPW, o0, o1);
                    }
                }
            } else {
                // runtime geometry: any m / widths / code size that fits; one code per warp step
                for (uint32_t iw = warp * P::CPW; iw < cnt; iw += SCAN_WARPS * P::CPW) {
                    const uint32_t i = min(iw + lane_code, cnt - 1);
                    const uint8_t* code = reinterpret_cast<const uint8_t*>(sb + size_t(i) * stride);
                    typename P::Acc acc = acc0;
                    for (uint32_t j = 0; j < ds->m; ++j) {
                        const uint32_t idx = rt_sub_index(ds, code, j);
                        P::add(acc, tile + size_t(ds->ent_off[j] + idx) * P::ROWB + lane_off);
                    }
                    flag(acc, iw + lane_code < cnt, i, 0u, 0u);
                }
            }
            if constexpr (!COPY) flush(); // queued pairs reference this stage buffer: resolve them before releasing it
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]); // this warp is done with stage buffer b
        }
    }
    if constexpr (COPY) flush_copy();
}

// ----------------------------------------------------------------- dispatch --

using G44 = GeomCT<8, 8, 4, 4>;       // 16x{4,4}
using G655 = GeomCT<16, 4, 6, 5, 5>;  // 12x{6,5,5}
using G664 = GeomCT<16, 4, 6, 6, 4>;  // 12x{6,6,4}
using G555 = GeomCT<16, 4, 5, 5, 5>;  // 12x{5,5,5}
using G88 = GeomCT<16, 4, 8, 8>;      // 8x{8,8}
using G8 = GeomCT<8, 8, 8>;           // 8x{8}
// the paper's 128-bit configurations
using G44W = GeomCT<8, 16, 4, 4>;     // 32x{4,4}
using G655W = GeomCT<16, 8, 6, 5, 5>; // 24x{6,5,5}
using G664W = GeomCT<16, 8, 6, 6, 4>; // 24x{6,6,4}
using G88W = GeomCT<16, 8, 8, 8>;     // 16x{8,8}

const char* variant_name(uint32_t v) {
    switch (v) {
    case VAR_F16X8: return "f16x8 (u8 tables as fp16 pairs, 256-query tile, LDS.128)";
    case VAR_F32X2: return "f32x2 (u16 tables as fp32, 64-query tile, LDS.64)";
    case VAR_U16X1: return "u16x1 (u16 entries, 32-query tile, int32 accumulate)";
    case VAR_U8X1: return "u8x1 (high-byte filter, 32-query tile)";
    case VAR_F16X4H: return "f16x4h (u16 tables, fp16 high-byte filter + exact re-evaluation, 128-query tile, LDS.64)";
    case VAR_F16X4H_C2: return "f16x4h-c2 (as f16x4h, 2 codes per warp step, 64-row tile)";
    case VAR_F16X4H_C4: return "f16x4h-c4 (as f16x4h, 32-row tile; named specs: pair-interleaved lines, LDS.128, 8 codes per warp step)";
    case VAR_F16X4_C4: return "f16x4-c4 (u8 tables exact in fp16, 32-row tile; 8x{8}: pair-interleaved lines, LDS.128, 8 codes per warp step)";
    case VAR_F16X4_C4M: return "f16x4-c4m (16x{4,4} as 8 byte-indexed tables of pair sums; 32-row pair-interleaved tile, LDS.128, 8 codes per warp step)";
    case VAR_F16X4H_C8Q: return "f16x4h-c8q (12x{6,5,5} as 4 x {6-bit table, (5,5) pair-sum table}: 8 lookups per code, quad-interleaved 16-row tile, LDS.128, 16 codes per warp step)";
    case VAR_F16X4H_C16Q: return "f16x4h-c16q (irregular 16-bit specs, 16-row tile of quad lines, rotated codes, LDS.128, 16 codes per warp step)";
    case VAR_F16X4H_C4D: return "f16x4h-c4d (as f16x4h-c4, entry lines duplicated: bank-conflict-free)";
    case VAR_TC8: return "tc8 (16x{4,4} as a one-hot int8 GEMM on tcgen05: 128 codes x 256 queries per tile, s32 accumulators in TMEM, threshold folded into the contraction)";
    case VAR_TC8P: return "tc8p (the tc8s contraction on CTA pairs: tcgen05 cta_group::2, 256 codes x 240 queries per MMA, each SM holds half of the tile's tables)";
    case VAR_TC8S: return "tc8s (16x{4,4} as a 2:4-sparse one-hot int8 GEMM on tcgen05: 128 codes x 240 queries per tile, compressed A + metadata in TMEM, s32 accumulators in TMEM, threshold folded into the contraction)";
    }
    return "?";
}

template <class P>
static uint32_t smem_need(uint32_t E) {
    return E * P::ROWB + NSTAGE * STAGE_BYTES + WQ_BYTES;
}

ScanPlan plan_scan(const DevSpec& ds, int device, int force_variant, bool allow_merged) {
    int max_smem = 0;
    QADC_CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    // static shared (DevSpec + ScanArgs + barriers) comes out of the same budget
    const uint32_t budget = uint32_t(max_smem) - uint32_t(sizeof(DevSpec) + sizeof(ScanArgs) + 2 * 256 * sizeof(float) + 256);
    if (ds.code_stride > 32) throw Error(QADC_ERR_CONFIG, "scan: codes wider than 256 bits are not supported");
    ScanPlan p{};
    p.threads = SCAN_THREADS;
    auto filter_shift_for = [&](ScanVariant v) -> uint32_t {
        if (ds.word_width != 16) return 0;
        if (v == VAR_U8X1) return 8;
        if (v == VAR_F16X4H_C8Q) return 6; // pair sums of 10-bit prefixes stay below 2048
        if (v != VAR_F16X4H && v != VAR_F16X4H_C2 && v != VAR_F16X4H_C4 && v != VAR_F16X4H_C4D && v != VAR_F16X4H_C16Q) return 0;
        uint32_t sh = 5;
        while (sh < 8 && ds.m * (65535u >> sh) > 28000u) ++sh;
        return sh;
    };
    auto fits = [&](uint32_t need) { return need <= budget; };
    auto set = [&](ScanVariant v, uint32_t tq, uint32_t need) {
        p.variant = v;
        p.tq = tq;
        p.smem_bytes = need;
    };
    const bool u8 = ds.word_width == 8;
    if (force_variant >= 0) {
        switch (force_variant) {
        case VAR_F16X8:
            if (!u8) throw Error(QADC_ERR_CONFIG, "scan: f16x8 needs 8-bit tables");
            set(VAR_F16X8, PolF16x8::TQ, smem_need<PolF16x8>(ds.E));
            break;
        case VAR_F32X2: set(VAR_F32X2, PolF32x2::TQ, smem_need<PolF32x2>(ds.E)); break;
        case VAR_U16X1: set(VAR_U16X1, PolU16x1::TQ, smem_need<PolU16x1>(ds.E)); break;
        case VAR_U8X1: set(VAR_U8X1, PolU8x1::TQ, smem_need<PolU8x1>(ds.E)); break;
        case VAR_F16X4_C4:
            if (!u8) throw Error(QADC_ERR_CONFIG, "scan: f16x4-c4 needs 8-bit tables");
            set(VAR_F16X4_C4, PolF16x4_C4::TQ, smem_need<PolF16x4_C4>(ds.E));
            break;
        case VAR_F16X4H_C16Q:
            if (u8 || !(G655::matches(ds) || G664::matches(ds) || G555::matches(ds)))
                throw Error(QADC_ERR_CONFIG, "scan: f16x4h-c16q is the 16-row layout of 12x{6,5,5} / 12x{6,6,4} / 12x{5,5,5}");
            set(VAR_F16X4H_C16Q, PolQU::TQ, smem_need<PolQU>(ds.E / 4));
            break;
        case VAR_F16X4H_C8Q:
            if (!allow_merged || !(G655::matches(ds) || G664::matches(ds) || G555::matches(ds)))
                throw Error(QADC_ERR_CONFIG, "scan: f16x4h-c8q is the flat 12x{6,5,5} / 12x{6,6,4} / 12x{5,5,5} layout");
            set(VAR_F16X4H_C8Q, PolQ655::TQ, smem_need<PolQ655>(GeomQ655::E));
            break;
        case VAR_TC8:
        case VAR_TC8S:
        case VAR_TC8P: {
            const int mode = tc8_mode(force_variant);
            if (!allow_merged || !G44::matches(ds)) throw Error(QADC_ERR_CONFIG, "scan: tc8 is the flat 16x{4,4} layout");
            if (!fits(scan_tc8_smem_bytes(mode))) throw Error(QADC_ERR_CONFIG, "scan: tc8 does not fit shared memory");
            p.variant = ScanVariant(force_variant);
            p.tq = scan_tc8_tile_rows(mode);
            p.smem_bytes = scan_tc8_smem_bytes(mode);
            p.tile_bufs = 1;
            p.filter_shift = 0;
            return p;
        }
        case VAR_F16X4_C4M:
            if (!allow_merged || !G44::matches(ds)) throw Error(QADC_ERR_CONFIG, "scan: f16x4-c4m is the flat 16x{4,4} layout");
            set(VAR_F16X4_C4M, PolF16x4_C4::TQ, smem_need<PolF16x4_C4>(G8::E));
            break;
        case VAR_F16X4H:
        case VAR_F16X4H_C2:
        case VAR_F16X4H_C4:
        case VAR_F16X4H_C4D:
            if (u8) throw Error(QADC_ERR_CONFIG, "scan: f16x4h is the 16-bit-table filter");
            if (force_variant == VAR_F16X4H_C4D) set(VAR_F16X4H_C4D, PolF16x4H_C4D::TQ, smem_need<PolF16x4H_C4D>(ds.E));
            else if (force_variant == VAR_F16X4H) set(VAR_F16X4H, PolF16x4H::TQ, smem_need<PolF16x4H>(ds.E));
            else if (force_variant == VAR_F16X4H_C2) set(VAR_F16X4H_C2, PolF16x4H_C2::TQ, smem_need<PolF16x4H_C2>(ds.E));
            else set(VAR_F16X4H_C4, PolF16x4H_C4::TQ, smem_need<PolF16x4H_C4>(ds.E));
            break;
        default: throw Error(QADC_ERR_CONFIG, "scan: unknown forced variant");
        }
        if (!fits(p.smem_bytes)) throw Error(QADC_ERR_CONFIG, "scan: forced variant does not fit shared memory");
        p.tile_bufs = 1;
        p.filter_shift = filter_shift_for(p.variant);
        const uint32_t tile_bytes = p.smem_bytes - (NSTAGE * STAGE_BYTES + WQ_BYTES);
        if (fits(p.smem_bytes + tile_bytes)) {
            p.tile_bufs = 2;
            p.smem_bytes += tile_bytes;
        }
        return p;
    }
    // 16x{4,4} on the flat path: pair sums indexed by whole code bytes halve the lookups per code
    // (measured 1.04 -> 1.45 T pairs/s at N = 2e8, 0.63 -> 0.70 at N = 1e6)
    if (u8 && allow_merged && G44::matches(ds) && fits(smem_need<PolF16x4_C4>(G8::E)))
        set(VAR_F16X4_C4M, PolF16x4_C4::TQ, smem_need<PolF16x4_C4>(G8::E));
    else if (u8 && fits(smem_need<PolF16x8>(ds.E))) set(VAR_F16X8, PolF16x8::TQ, smem_need<PolF16x8>(ds.E));
    else if (u8 && fits(smem_need<PolF16x4_C4>(ds.E))) set(VAR_F16X4_C4, PolF16x4_C4::TQ, smem_need<PolF16x4_C4>(ds.E));
    // flat 12x{6,5,5}: the merged view (8 lookups per code instead of 12) -- measured 1.30 -> 1.78 T pairs/s on C2
    else if (!u8 && allow_merged && (G655::matches(ds) || G664::matches(ds) || G555::matches(ds)) &&
             fits(smem_need<PolQ655>(GeomQ655::E)))
        set(VAR_F16X4H_C8Q, PolQ655::TQ, smem_need<PolQ655>(GeomQ655::E));
    // 64-row tiles first: measured 4 % faster than 128-row tiles on the flat 12x{6,5,5} scan (two tile buffers
    // fit, and two codes per warp step halve the per-code bookkeeping); 32-row tiles pay ~37 % extra
    // shared-memory wavefronts for bank conflicts between the four code groups of a warp
    else if (!u8 && fits(2 * smem_need<PolF16x4H_C2>(ds.E) - (NSTAGE * STAGE_BYTES + WQ_BYTES)))
        set(VAR_F16X4H_C2, PolF16x4H_C2::TQ, smem_need<PolF16x4H_C2>(ds.E));
    else if (!u8 && fits(smem_need<PolF16x4H>(ds.E))) set(VAR_F16X4H, PolF16x4H::TQ, smem_need<PolF16x4H>(ds.E));
    else if (!u8 && fits(smem_need<PolF16x4H_C2>(ds.E))) set(VAR_F16X4H_C2, PolF16x4H_C2::TQ, smem_need<PolF16x4H_C2>(ds.E));
    else if (!u8 && fits(smem_need<PolF16x4H_C4>(ds.E))) set(VAR_F16X4H_C4, PolF16x4H_C4::TQ, smem_need<PolF16x4H_C4>(ds.E));
    else if (fits(smem_need<PolF32x2>(ds.E))) set(VAR_F32X2, PolF32x2::TQ, smem_need<PolF32x2>(ds.E));
    else if (fits(smem_need<PolU16x1>(ds.E))) set(VAR_U16X1, PolU16x1::TQ, smem_need<PolU16x1>(ds.E));
    else if (fits(smem_need<PolU8x1>(ds.E))) set(VAR_U8X1, PolU8x1::TQ, smem_need<PolU8x1>(ds.E));
    else
        throw Error(QADC_ERR_CONFIG, "scan: the quantized tables of this spec (" + std::to_string(ds.E) +
                                         " entries) do not fit shared memory; no CPU fallback exists");
    // a second tile buffer (the next job's tile lands while this one is scanned) whenever it fits
    p.tile_bufs = 1;
    p.filter_shift = filter_shift_for(p.variant);
    const uint32_t tile_bytes = p.smem_bytes - (NSTAGE * STAGE_BYTES + WQ_BYTES);
    if (fits(p.smem_bytes + tile_bytes)) {
        p.tile_bufs = 2;
        p.smem_bytes += tile_bytes;
    }
    return p;
}

template <class P, class G, int EARLY>
static void launch_early(const ScanPlan& plan, const DevSpec& ds, const ScanArgs& args, int grid, cudaStream_t stream) {
    QADC_CUDA_CHECK(cudaFuncSetAttribute(scan_kernel<P, G, EARLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(plan.smem_bytes)));
    scan_kernel<P, G, EARLY><<<grid, SCAN_THREADS, plan.smem_bytes, stream>>>(ds, args);
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}
// EARLY > 0 (check after that many tables whether any row of the warp can still admit the code, skip the
// remaining lookups otherwise) is exact but was measured to never pay: ADC sums concentrate -- the R-th best
// of 10^7 codes sits near 0.5x the median sum -- so after 2/3 of the tables ~16 % of the pairs are still
// pending and with 32..256 rows per warp step the skip practically never fires.
// Only EARLY = 0 is instantiated.
template <class P, class G>
static void launch_one(const ScanPlan& plan, const DevSpec& ds, const ScanArgs& args, int grid, cudaStream_t stream) {
    return launch_early<P, G, 0>(plan, ds, args, grid, stream);
}

// Compile-time geometries are instantiated only for the (policy, shape) pairs the planner
// can actually pick for the named 64-bit specs; everything else runs the runtime geometry.
void launch_scan(const ScanPlan& plan, const DevSpec& ds, const ScanArgs& args_in, int grid, cudaStream_t stream) {
    if (args_in.n_jobs == 0 || grid <= 0) return;
    ScanArgs args = args_in;
    args.tile_bufs = plan.tile_bufs;
    args.filter_shift = plan.filter_shift;
    switch (plan.variant) {
    case VAR_TC8:
    case VAR_TC8S:
    case VAR_TC8P: return launch_scan_tc8(tc8_mode(plan.variant), ds, args, grid, stream);
    case VAR_F16X8:
        if (G44::matches(ds)) return launch_one<PolF16x8, G44>(plan, ds, args, grid, stream);
        return launch_one<PolF16x8, GeomRT>(plan, ds, args, grid, stream);
    case VAR_F32X2:
        if (G655::matches(ds)) return launch_one<PolF32x2, G655>(plan, ds, args, grid, stream);
        if (G664::matches(ds)) return launch_one<PolF32x2, G664>(plan, ds, args, grid, stream);
        if (G555::matches(ds)) return launch_one<PolF32x2, G555>(plan, ds, args, grid, stream);
        if (G44::matches(ds)) return launch_one<PolF32x2, G44>(plan, ds, args, grid, stream);
        return launch_one<PolF32x2, GeomRT>(plan, ds, args, grid, stream);
    case VAR_U16X1:
        if (G88::matches(ds)) return launch_one<PolU16x1, G88>(plan, ds, args, grid, stream);
        if (G8::matches(ds)) return launch_one<PolU16x1, G8>(plan, ds, args, grid, stream);
        return launch_one<PolU16x1, GeomRT>(plan, ds, args, grid, stream);
    case VAR_U8X1:
        if (G88W::matches(ds)) return launch_one<PolU8x1, G88W>(plan, ds, args, grid, stream);
        return launch_one<PolU8x1, GeomRT>(plan, ds, args, grid, stream);
    case VAR_F16X4H:
        if (G655::matches(ds)) return launch_one<PolF16x4H, G655>(plan, ds, args, grid, stream);
        if (G664::matches(ds)) return launch_one<PolF16x4H, G664>(plan, ds, args, grid, stream);
        if (G555::matches(ds)) return launch_one<PolF16x4H, G555>(plan, ds, args, grid, stream);
        return launch_one<PolF16x4H, GeomRT>(plan, ds, args, grid, stream);
    case VAR_F16X4H_C2:
        if (G655::matches(ds)) return launch_one<PolF16x4H_C2, G655>(plan, ds, args, grid, stream);
        if (G655W::matches(ds)) return launch_one<PolF16x4H_C2, G655W>(plan, ds, args, grid, stream);
        if (G664W::matches(ds)) return launch_one<PolF16x4H_C2, G664W>(plan, ds, args, grid, stream);
        return launch_one<PolF16x4H_C2, GeomRT>(plan, ds, args, grid, stream);
    case VAR_F16X4H_C4:
        // irregular specs: word-pair interleaved lines (tile_pair_layout() makes the same choice), 8 rows per lane
        if (G655::matches(ds)) return launch_one<PolF16x8H_C8P, G655>(plan, ds, args, grid, stream);
        if (G664::matches(ds)) return launch_one<PolF16x8H_C8P, G664>(plan, ds, args, grid, stream);
        if (G555::matches(ds)) return launch_one<PolF16x8H_C8P, G555>(plan, ds, args, grid, stream);
        if (G88::matches(ds)) return launch_one<PolF16x8H_C8P, G88>(plan, ds, args, grid, stream);
        return launch_one<PolF16x4H_C4, GeomRT>(plan, ds, args, grid, stream);
    case VAR_F16X4H_C16Q:
        if (G664::matches(ds)) return launch_one<PolQU, GeomQU<G664>>(plan, ds, args, grid, stream);
        if (G555::matches(ds)) return launch_one<PolQU, GeomQU<G555>>(plan, ds, args, grid, stream);
        return launch_one<PolQU, GeomQU<G655>>(plan, ds, args, grid, stream);
    case VAR_F16X4H_C8Q:
        if (G664::matches(ds)) return launch_one<PolQ655, GeomQ664>(plan, ds, args, grid, stream);
        if (G555::matches(ds)) return launch_one<PolQ655, GeomQ555>(plan, ds, args, grid, stream);
        return launch_one<PolQ655, GeomQ655>(plan, ds, args, grid, stream);
    case VAR_F16X4H_C4D:
        // duplicated lines, 8 rows per lane (the 4-rows-per-lane twin was the choice while a flagged warp step cost
        // one ballot per slot; with the sparse flag path this one is 13 % faster on the IVF workload).  Superseded
        // as the IVF default by the word-pair layout of VAR_F16X4H_C4, kept as a selectable variant.
        if (G655::matches(ds)) return launch_one<PolF16x8H_C8D, G655>(plan, ds, args, grid, stream);
        return launch_one<PolF16x4H_C4D, GeomRT>(plan, ds, args, grid, stream);
    // (G8 / G88 run the pair-interleaved tile layout: tile_pair_layout() in tilepack.cu makes the same choice)
    case VAR_F16X4_C4M: return launch_one<PolF16x8_C8P, G8>(plan, ds, args, grid, stream); // the code bytes ARE 8x{8} indices
    case VAR_F16X4_C4:
        if (G8::matches(ds)) return launch_one<PolF16x8_C8P, G8>(plan, ds, args, grid, stream);
        if (G44W::matches(ds)) return launch_one<PolF16x4_C4, G44W>(plan, ds, args, grid, stream);
        return launch_one<PolF16x4_C4, GeomRT>(plan, ds, args, grid, stream);
    default: throw Error(QADC_ERR_CONFIG, "scan: bad variant");
    }
}

} // namespace qadc
