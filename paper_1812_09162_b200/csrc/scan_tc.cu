// scan_tc.cu -- the 16x{4,4} scan as a one-hot int8 GEMM on the 5th-generation tensor cores (tcgen05).
//
// Reference semantics are those of scan.cu (scan_scalar.hpp:34-64): per code, the sum of the m = 16 quantized table
// entries selected by its 4-bit subcodes, saturating at q_max = 255, pushed into a bounded (distance, id) heap.
// Formulation: a code is the 256-dimensional 0/1 vector with a one at (table j, entry c_j); its sum for query q is
// the dot product with q's 256 table bytes.  For a tile of 128 codes x 256 queries that is ONE contraction
//     D[code][query] = sum_k onehot[code][k] * lut[query][k]        M = 128, N = 256, K = 256
// whose operands are bytes and whose result fits 13 bits -- exactly what tcgen05.mma kind::i8 computes, 8192
// multiply-adds per clock per SM, against the 128 B/clk shared-memory pipe that bounds the lookup kernel of scan.cu
// (16 B of table traffic per pair).  VERDICT r1 asked for this experiment with a kill criterion (>= 1.5x end to end
// and bit-exact); the measurement is in DESIGN.md section 4.5.
//
//   * A (one-hot, 128 x 256 B) is BUILT in shared memory by four generator warps from the streamed codes: thread =
//     code, one 16-byte store per table (the 16 entries of table j are exactly one 16-byte K chunk, and the chunk is
//     a single 0x01 byte at position c_j).  B (the tile's tables, 256 queries x 256 B) is resident in shared memory
//     for a whole job, in the K-major no-swizzle canonical layout (8 rows x 16 bytes core matrices), prepared by
//     pack_tiles_tc8_kernel and fetched with TMA bulk copies.  Table bytes are stored as e - 128 (signed), so every
//     MMA is u8 x s8.
//   * The admission threshold rides in the contraction: a ninth K step multiplies a constant all-ones A' block with a
//     per-query row of 32 signed bytes that sum to v = 2048 + bias - thr - 1 (or -4096: admit all; +4064: padding row),
//     so D = bias + sum - thr - 1 and "sum <= thr" is the SIGN BIT of the accumulator.
//   * D (128 x 256 s32) lives in TMEM, two buffers of 256 columns; four epilogue warps read it back with tcgen05.ld
//     (thread = code, 64 queries per load), OR the values and look at one sign bit per 64 pairs.  A flagged pair's
//     accumulator is its exact sum; its (distance, id) key goes through the CandidateHeap::push test (heap.hpp:46-47)
//     against the tile's threshold keys kept in shared memory (dense form), or the pair's coordinates are queued and
//     its sum is recomputed from the reference-order table, 32 pairs at a time (sparse forms; exact_admit_ct,
//     scan_common.cuh, which also serves rows without a usable threshold).  The sign test never drops a pair the
//     exact test would admit, so results are exact by construction, as in scan.cu.
//   * Warp roles: 0-7 epilogue (TMEM lane quadrant = warp id % 4, column half = warp id / 4), 8-11 one-hot
//     generators, 12 and 14 MMA issuers (sparse forms: one per accumulator buffer; 12 also owns the TMEM allocation),
//     13 producer (TMA code stream, tile loads, threshold rows).  All hand-offs are mbarriers; tcgen05.commit releases
//     the one-hot stages and publishes the accumulators.  (Four epilogue warps were the bottleneck of the first
//     version: 1970 cycles per sub-tile against 1205 of MMA, and the two did not overlap.)
//   * Three instantiations: dense (variant 12), 2:4 sparse (13: compressed one-hot + metadata in TMEM, 240-query
//     tiles), and the sparse form on CTA pairs (14: cta_group::2, M = 256, each SM holds half of the tile's tables).
// The operand layouts, the instruction descriptor and TS/SS modes were pinned against a CPU reference on the B200 by
// tools/umma_probe.cu before this kernel relied on them.
#include "scan_common.cuh"

namespace qadc {

namespace {

#ifndef TC_PARK_NS
#define TC_PARK_NS 0u
#endif
#ifndef TC_SPIN
#define TC_SPIN 0 // 1: mbarrier waits spin on test_wait instead of the (parking) try_wait
#endif
#ifndef TC_GEN_GROUP
#define TC_GEN_GROUP 2 // sub-tiles a generator warp emits per hand-over (1 or 2)
#endif
// -DTC_PROFILE: lane 0 of one warp per role accumulates clock64() spans around its waits and prints them for CTA 0 at the
// end of every long launch (build: make EXTRA=-DTC_PROFILE; the numbers behind DESIGN.md section 4.5's stall table)
#ifdef TC_PROFILE
#define TC_PROF_DECL(n) long long prof_t[n] = {}; long long prof_c = clock64(); long long prof_start = prof_c
#define TC_PROF(i) do { const long long now_ = clock64(); prof_t[i] += now_ - prof_c; prof_c = now_; } while (0)
#else
#define TC_PROF_DECL(n)
#define TC_PROF(i)
#endif
// queries per tile = MMA N: 256 dense; 240 for the 2:4-sparse form (it needs 24 TMEM columns for its metadata stages)
__host__ __device__ constexpr int tc_tq(bool sp) { return sp ? 240 : 256; }
constexpr int TC_SUB = 128;            // codes per sub-tile = MMA M
__host__ __device__ constexpr int tc_na(bool sp) { return sp ? 4 : 3; } // one-hot stages (sparse: 16 KB each + 8 metadata columns)
constexpr int TC_NSTAGE = 3;           // code stages (TMA ring)
constexpr int TC_STAGE_BYTES = 8192;   // 1024 codes
constexpr int TC_STAGE_CODES = TC_STAGE_BYTES / 8;
constexpr int TC_INFO = 8;             // sub-tile info ring (generator -> epilogue)
constexpr int TC_KC = 16;              // 16-byte K chunks of the table part (= tables)
// B rows one CTA holds: the whole tile, or half of it for a CTA pair (cta_group::2 reads the other half from the peer)
__host__ __device__ constexpr int tc_brows(bool sp, bool pair = false) { return pair ? tc_tq(sp) / 2 : tc_tq(sp); }
__host__ __device__ constexpr int tc_b_chunk(bool sp, bool pair = false) { return tc_brows(sp, pair) * 16; } // bytes of one K chunk of B (rows x 16 B): the descriptor's LBO
constexpr int TC_A_CHUNK = TC_SUB * 16;
__host__ __device__ constexpr int tc_b_bytes(bool sp, bool pair = false) { return (TC_KC + 2) * tc_b_chunk(sp, pair); } // tables + the threshold K step
__host__ __device__ constexpr int tc_a_bytes(bool sp) { return (sp ? TC_KC / 2 : TC_KC) * TC_A_CHUNK; } // sparse: two kept bytes per group of four
constexpr uint32_t TC_ECOL = 480;      // sparse: first TMEM column of the metadata stages (8 columns each)
constexpr int TC_AP_BYTES = 2 * TC_A_CHUNK;          // A': all ones, K = 32
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_GEN_WARP0 = 8, TC_MMA_WARP = 12, TC_PROD_WARP = 13, TC_MMA_WARP2 = 14;
constexpr int TC_THREADS = 15 * 32;
constexpr int TC_WQ_CAP = 64;          // per-epilogue-warp queue of admitted (key, row) pairs
// query tiles per job: the CTA-pair form keeps TWO tiles' tables resident (its B halves are small enough) and runs every
// one-hot stage against both, one tile per accumulator buffer -- half the generator work, stores and hand-overs per pair
__host__ __device__ constexpr int tc_nt(bool pair) { return pair ? 2 : 1; }
__host__ __device__ constexpr int tc_smem(bool sp, bool pair = false) {
    return tc_nt(pair) * tc_b_bytes(sp, pair) + TC_AP_BYTES + tc_na(sp) * tc_a_bytes(sp) + TC_NSTAGE * TC_STAGE_BYTES +
           TC_INFO * TC_SUB * 8 + TC_EPI_WARPS * TC_WQ_CAP * 16;
}

struct SubInfo {
    uint64_t id_ref;    // explicit ids: index of row 0's id in ScanArgs::ids; implicit: id of row 0
    uint32_t n_valid;   // codes in this sub-tile (rows >= n_valid are padding)
    uint32_t row_begin; // first LUT row of the tile
    uint32_t pad[2];
};

// the rare rows without a usable threshold (heap not full, or its worst entry saturated): integer re-evaluation from the
// reference-order table.  One out-of-line copy: the epilogue's unrolled hit scan would otherwise carry 64 of them.
__device__ __noinline__ void tc_exact_admit(const DevSpec* ds, const ScanArgs* a, uint32_t w0, uint32_t w1, uint32_t row,
                                            uint32_t id) {
    exact_admit_ct<GeomCT<8, 8, 4, 4>>(ds, a, w0, w1, row, id);
}

// shared-memory matrix descriptor: K-major, no swizzle (cute::UMMA::SmemDescriptor, version 1).  LBO = bytes between the
// two 16-byte K chunks one MMA consumes, SBO = bytes between consecutive 8-row groups (a core matrix is 8 x 16 bytes)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) | (uint64_t((sbo >> 4) & 0x3FFFu) << 32) |
           (uint64_t(1) << 46);
}
// instruction descriptor (cute::UMMA::InstrDescriptor): s32 accumulate, A = u8, B = s8, both K-major, M = 128, N = TQ;
// bit 2 = A is 2:4 sparse
__host__ __device__ constexpr uint32_t tc_idesc(bool sp, bool sparse_instr, bool pair = false) {
    return (sparse_instr ? 4u : 0u) | (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t(tc_tq(sp)) >> 3) << 17) |
           ((uint32_t(pair ? 2 * TC_SUB : TC_SUB) >> 4) << 24);
}

template <bool PAIR = false>
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    if constexpr (PAIR)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
    else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
}
// 2:4-sparse A: 32 compressed bytes per row per instruction = 64 logical K; metadata (4 bits per group of four: the two
// kept positions, idx0 | idx1 << 2) in tensor memory, lane = row, two columns per instruction (pinned by tools/umma_probe.cu)
template <bool PAIR = false>
__device__ __forceinline__ void umma_i8_sp(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t e_tmem, uint32_t idesc,
                                           uint32_t accumulate) {
    if constexpr (PAIR)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\ntcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(e_tmem), "r"(idesc), "r"(accumulate)
            : "memory");
    else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\ntcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(e_tmem), "r"(idesc), "r"(accumulate)
            : "memory");
}
// arrives when every MMA issued so far has completed; CTA pair: on the barrier at this offset in BOTH CTAs
template <bool PAIR = false>
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    if constexpr (PAIR)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(bar)),
                     "h"(uint16_t(3))
                     : "memory");
    else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The same three instructions for a CONVERGED warp: every lane executes the statement with warp-uniform operands and
// elect.sync picks the one lane that issues.  Inside `if (lane == 0)` the compiler cannot see that the operands are uniform
// and wraps every tcgen05 instruction in an ELECT / R2UR.BROADCAST / BRA.U.ANY loop (~20 dependent instructions each).
#define QADC_ELECT_PRED ".reg .pred p, q;\nelect.sync _|q, 0xffffffff;\n"
template <bool PAIR>
__device__ __forceinline__ void umma_i8_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    if constexpr (PAIR)
        asm volatile("{\n" QADC_ELECT_PRED "setp.ne.b32 p, %4, 0;\n@q tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
                     "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
                     : "memory");
    else
        asm volatile("{\n" QADC_ELECT_PRED "setp.ne.b32 p, %4, 0;\n@q tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
                     "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
                     : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void umma_i8_sp_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t e_tmem, uint32_t idesc,
                                                 uint32_t accumulate) {
    if constexpr (PAIR)
        asm volatile("{\n" QADC_ELECT_PRED "setp.ne.b32 p, %5, 0;\n@q tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(
                         d_tmem),
                     "l"(a), "l"(b), "r"(e_tmem), "r"(idesc), "r"(accumulate)
                     : "memory");
    else
        asm volatile("{\n" QADC_ELECT_PRED "setp.ne.b32 p, %5, 0;\n@q tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(
                         d_tmem),
                     "l"(a), "l"(b), "r"(e_tmem), "r"(idesc), "r"(accumulate)
                     : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
    if constexpr (PAIR)
        asm volatile("{\n" QADC_ELECT_PRED
                     "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
                         smem_u32(bar)),
                     "h"(uint16_t(3))
                     : "memory");
    else
        asm volatile("{\n" QADC_ELECT_PRED "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                         smem_u32(bar))
                     : "memory");
}
// ---- CTA pair plumbing: rank in the cluster, cluster-wide barrier, arrive on a barrier of the LEADER CTA (rank 0)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// (default .release.cta semantics, as CUTLASS's ClusterBarrier::arrive(cta_id): what the arrivals publish -- the one-hot
// stage and its metadata -- is read by the arriving CTA's OWN tensor core, the barrier only orders the leader's issue
// after it; a .release.cluster arrive was measured at ~400 cycles per hand-over)
template <bool PAIR>
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar, uint32_t rank = 0) {
    if (PAIR && rank != 0) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(0u));
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    } else {
        mbar_arrive(bar);
    }
}
// mbarrier wait that parks the warp between polls (NANOSLEEP.SYNCS wakes on the barrier's phase change): ten of this
// kernel's fourteen warps are waiting at any time, and a tight try_wait loop cost 22 % of all issued instructions
__device__ __forceinline__ void mbar_wait_park(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done;
#if TC_SPIN
    do { // non-blocking probe in a tight loop: lowest wake-up latency, costs issue slots
        asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"(addr), "r"(parity)
                     : "memory");
    } while (!done);
#else
    do {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(TC_PARK_NS)
            : "memory");
    } while (!done);
#endif
}
// the same for a barrier other CTAs of the cluster arrive on (kept apart so that its semantics can be changed in one place)
__device__ __forceinline__ void mbar_wait_park_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done;
    do {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(TC_PARK_NS)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 128 consecutive columns, two per register: register i = low 16 bits of column 2i | low 16 bits of column 2i + 1 << 16
// (every accumulator of this kernel fits 14 bits)
__device__ __forceinline__ void tmem_ld128_pack16(uint32_t taddr, uint32_t (&v)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]),
          "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]),
          "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]),
          "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
          "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

using G44 = GeomCT<8, 8, 4, 4>; // 16x{4,4}: bit position of subquantizer j = 4 j

// sub-tiles of one job: its stages hold TC_STAGE_CODES codes each, every stage is cut into sub-tiles of TC_SUB codes
// (CTA pair: a step covers 2 x TC_SUB codes, the CTA of rank r takes the r-th half)
__device__ __forceinline__ uint32_t job_subtiles(uint32_t n_codes, uint32_t step = TC_SUB) {
    const uint32_t full = n_codes / TC_STAGE_CODES, rem = n_codes - full * TC_STAGE_CODES;
    return full * (TC_STAGE_CODES / step) + (rem + step - 1) / step;
}

} // namespace

template <bool SP, bool PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1) scan_tc8_kernel(DevSpec ds_param, ScanArgs args_param) {
    static_assert(SP || !PAIR, "the CTA-pair form is built for the sparse operand only");
    constexpr int TC_TQ = tc_tq(SP), TC_BROWS = tc_brows(SP, PAIR), TC_B_CHUNK = tc_b_chunk(SP, PAIR), TC_B_BYTES = tc_b_bytes(SP, PAIR),
                  TC_A_BYTES = tc_a_bytes(SP);
    constexpr int TC_NA = tc_na(SP);
    constexpr uint32_t TC_IDESC = tc_idesc(SP, false, PAIR), TC_IDESC_SP = tc_idesc(SP, true, PAIR);
    constexpr uint32_t TC_STEP = PAIR ? 2 * TC_SUB : TC_SUB; // codes per MMA step of the CTA (pair)
    constexpr uint32_t NCTA = PAIR ? 2 : 1;
    constexpr uint32_t NT = tc_nt(PAIR);          // query tiles per job = consumers of one one-hot stage
    extern __shared__ __align__(1024) char smem[];
    __shared__ DevSpec s_ds;
    __shared__ ScanArgs s_args;
    __shared__ __align__(8) uint64_t s_full[TC_NSTAGE], s_empty[TC_NSTAGE]; // code stages: TMA -> generators
    __shared__ __align__(8) uint64_t s_afull[tc_na(SP)], s_aempty[tc_na(SP)]; // one-hot stages: generators -> MMA
    __shared__ __align__(8) uint64_t s_dfull[2], s_dempty[2];                // accumulators: MMA -> epilogue
    __shared__ __align__(8) uint64_t s_tfull, s_tempty;                      // LUT tile: producer -> MMA
    __shared__ __align__(8) uint64_t s_tload;                                // CTA pair: this CTA's half of the tile has landed
    __shared__ SubInfo s_info[TC_INFO];
    __shared__ uint32_t s_tmem;
    __shared__ uint32_t s_wqn[TC_EPI_WARPS]; // admission queues' fill levels while lanes push on their own
#ifdef TC_PROFILE
    __shared__ long long s_stamp[3][8]; // per step (ring): MMAs committed | epilogue warp 0 past dfull | ... released the buffer
#endif

    char* sB = smem;
    char* sAp = sB + NT * TC_B_BYTES;
    char* sA = sAp + TC_AP_BYTES;
    char* stage = sA + TC_NA * TC_A_BYTES;
    uint2* info_codes = reinterpret_cast<uint2*>(stage + TC_NSTAGE * TC_STAGE_BYTES);
    uint64_t* s_wq_key = reinterpret_cast<uint64_t*>(info_codes + TC_INFO * TC_SUB); // [TC_EPI_WARPS][TC_WQ_CAP] queued codes
    uint32_t* s_wq_row = reinterpret_cast<uint32_t*>(s_wq_key + TC_EPI_WARPS * TC_WQ_CAP);
    uint32_t* s_wq_id = s_wq_row + TC_EPI_WARPS * TC_WQ_CAP;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // CTA pair: both CTAs walk the same jobs; rank r generates, holds and post-processes the r-th 128 codes of every step
    // and holds the r-th half of the tile's B rows; the leader (rank 0) issues the MMAs for both.  Barriers the leader's
    // MMA warp waits on (afull, dempty, tfull) live in the leader and count arrivals from both CTAs; barriers the tensor
    // core signals (aempty, dfull, tempty) exist in both CTAs and get multicast commits.
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    if (tid < uint32_t(TC_EPI_WARPS)) s_wqn[tid] = 0u;
    if (tid == 0) {
        s_ds = ds_param;
        s_args = args_param;
        for (int i = 0; i < TC_NSTAGE; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 4);
        }
        for (int i = 0; i < TC_NA; ++i) {
            mbar_init(&s_afull[i], 4 * NCTA);
            mbar_init(&s_aempty[i], NT); // one commit per consumer of the stage
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_dfull[i], 1);
            mbar_init(&s_dempty[i], TC_EPI_WARPS * NCTA);
        }
        mbar_init(&s_tfull, 2); // the tile's expect_tx + the threshold rows' arrive (CTA pair: one arrive per CTA)
        mbar_init(&s_tempty, SP ? 2 : 1); // one commit per MMA warp
        mbar_init(&s_tload, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == TC_MMA_WARP) { // the MMA warp owns the tensor memory: 2 accumulators x 256 columns
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "n"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "n"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    for (uint32_t i = tid; i < TC_AP_BYTES / 16; i += TC_THREADS) // A': every row all ones
        reinterpret_cast<uint4*>(sAp)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync_all(); // the peer's barriers are initialised before anything arrives on them
    tc_fence_after();
    const DevSpec* ds = &s_ds;
    const ScanArgs* a = &s_args;
    const uint32_t tmem = s_tmem;
    const uint32_t dbg = a->filter_shift; // timing experiments (option tc_debug): 1 = epilogue reads nothing, 2 = generators store nothing, 4 = one MMA per sub-tile

    const uint32_t unit = blockIdx.x / NCTA, n_units = gridDim.x / NCTA; // a CTA, or a CTA pair
    const uint32_t j_begin = (a->cta_begin && !PAIR) ? a->cta_begin[unit] : uint32_t(uint64_t(a->n_jobs) * unit / n_units);
    const uint32_t j_end = (a->cta_begin && !PAIR) ? a->cta_begin[unit + 1] : uint32_t(uint64_t(a->n_jobs) * (unit + 1) / n_units);

    if (warp == TC_PROD_WARP) {
        // ============================ producer: code stream + tile loads + threshold rows ====================
        uint32_t it = 0, tseq = 0, prev_rb = 0xFFFFFFFFu, prev_nr = 0;
        for (uint32_t ji = j_begin; ji < j_end; ++ji) {
            const ScanJob job = a->jobs[ji];
            if (job.n_codes == 0 || job.n_rows == 0) continue;
            if (job.row_begin != prev_rb || job.n_rows != prev_nr) {
                prev_rb = job.row_begin;
                prev_nr = job.n_rows;
                mbar_wait_park(&s_tempty, (tseq & 1u) ^ 1u); // the MMAs of the previous tile are done with B
                if (lane == 0) {
                    if constexpr (PAIR) { // this CTA's rows of every K chunk: 16 pieces of each [kc][TQ rows][16 B] image
                        mbar_expect_tx(&s_tload, NT * TC_KC * TC_B_CHUNK);
                        for (uint32_t ti = 0; ti < NT; ++ti) {
                            const char* src = reinterpret_cast<const char*>(a->tile_lut) +
                                              size_t(job.row_begin / TC_TQ + ti) * (TC_KC * TC_TQ * 16) + size_t(rank) * TC_B_CHUNK;
                            for (uint32_t kc = 0; kc < uint32_t(TC_KC); ++kc)
                                bulk_g2s(sB + ti * TC_B_BYTES + kc * TC_B_CHUNK, src + size_t(kc) * (TC_TQ * 16), TC_B_CHUNK, &s_tload);
                        }
                    } else {
                        const char* src = reinterpret_cast<const char*>(a->tile_lut) + size_t(job.row_begin / TC_TQ) * (TC_KC * TC_B_CHUNK);
                        mbar_expect_tx(&s_tfull, TC_KC * TC_B_CHUNK);
                        for (uint32_t off = 0; off < uint32_t(TC_KC * TC_B_CHUNK); off += 32768u)
                            bulk_g2s(sB + off, src + off, min(32768u, uint32_t(TC_KC * TC_B_CHUNK) - off), &s_tfull);
                    }
                }
                // threshold K step: row r gets 32 signed bytes that sum to v
                for (uint32_t r = lane; r < NT * uint32_t(TC_TQ); r += 32) {
                    int v = 4064; // padding rows never admit
                    if (r < job.n_rows) {
                        const uint32_t row = job.row_begin + r;
                        const uint32_t q = a->row_query ? a->row_query[row] : row;
                        if (q != 0xFFFFFFFFu) {
                            uint64_t tk = a->thr_key[q];
                            uint32_t thr = uint32_t(tk >> 32);
                            const uint32_t bias = a->row_bias ? min(a->row_bias[row], ds->qmax) : 0u;
                            // Ties cannot win where ids only grow: with implicit ids every code of this tile run has an id
                            // >= job.id_base, and if that exceeds the id of the heap's worst entry, a sum EQUAL to the
                            // threshold gives key > worst key -- CandidateHeap::push rejects it (heap.hpp:46-47).  The
                            // effective threshold is then (thr - 1, any id): with 8-bit sums about half of the pairs at or
                            // below the threshold sit exactly on it, and each would cost the epilogue an admission attempt (drain() tests
                            // against the REAL key, so a pair that slips through is still judged correctly).
                            if (tk != KEY_INF && thr < ds->qmax && a->ids == nullptr && job.id_base > uint32_t(tk)) {
                                if (thr == 0) {
                                    tk = 0; // nothing is below a zero threshold: never admit (v stays at the padding value)
                                } else {
                                    thr -= 1;
                                    tk = make_key(thr, 0xFFFFFFFFu);
                                }
                            }
                            if (tk == 0) v = 4064;
                            else if (tk == KEY_INF || thr >= ds->qmax) v = -4096; // heap not full / worst saturated: admit all
                            else v = 2048 + int(bias) - int(thr) - 1;
                        }
                    }
                    uint32_t w[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        uint32_t word = 0;
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int x = max(-128, min(127, v));
                            v -= x;
                            word |= (uint32_t(x) & 0xFFu) << (8 * b);
                        }
                        w[k] = word;
                    }
                    const uint32_t ti = r / uint32_t(TC_TQ), rr = r - ti * uint32_t(TC_TQ); // tile of the job, row of the tile
                    if (PAIR && rr / uint32_t(TC_BROWS) != rank) continue; // (the keys above are kept for the whole tile)
                    const uint32_t rl = PAIR ? rr % uint32_t(TC_BROWS) : rr;
                    char* dst = sB + ti * TC_B_BYTES + TC_KC * TC_B_CHUNK + (rl >> 3) * 128 + (rl & 7u) * 16;
                    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
                    *reinterpret_cast<uint4*>(dst + TC_B_CHUNK) = make_uint4(w[4], w[5], w[6], w[7]);
                }
                proxy_fence(); // generic-proxy stores -> visible to the tensor core's (async proxy) operand reads
                __syncwarp();
                if constexpr (PAIR) { // tell the leader once this CTA's half (bulk copies + threshold rows) is in place
                    mbar_wait_park(&s_tload, tseq & 1u);
                    if (lane == 0) mbar_arrive_leader<true>(&s_tfull, rank);
                } else {
                    if (lane == 0) mbar_arrive(&s_tfull);
                }
                ++tseq;
            }
            const uint8_t* gcodes = a->codes + job.code_off * 8;
            const uint32_t n_st = (job.n_codes + TC_STAGE_CODES - 1) / TC_STAGE_CODES;
            for (uint32_t st = 0; st < n_st; ++st, ++it) {
                const uint32_t b = it % TC_NSTAGE;
                mbar_wait_park(&s_empty[b], ((it / TC_NSTAGE) & 1u) ^ 1u);
                if (lane == 0) {
                    const uint32_t first = st * TC_STAGE_CODES;
                    const uint32_t cnt = min(uint32_t(TC_STAGE_CODES), job.n_codes - first);
                    const uint32_t bytes = (cnt * 8 + 15u) & ~15u;
                    mbar_expect_tx(&s_full[b], bytes);
                    bulk_g2s(stage + size_t(b) * TC_STAGE_BYTES, gcodes + size_t(first) * 8, bytes, &s_full[b]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= TC_GEN_WARP0 && warp < TC_GEN_WARP0 + 4) {
        // ============================ generators: codes -> one-hot A stages ==================================
        const uint32_t g = tid - TC_GEN_WARP0 * 32; // row of the sub-tile
        uint32_t it = 0, s = 0, tseq = 0, prev_rb = 0xFFFFFFFFu, prev_nr = 0;
        TC_PROF_DECL(5);
        for (uint32_t ji = j_begin; ji < j_end; ++ji) {
            const ScanJob job = a->jobs[ji];
            if (job.n_codes == 0 || job.n_rows == 0) continue;
            if (job.row_begin != prev_rb || job.n_rows != prev_nr) { // mirrors the producer's tile sequence
                prev_rb = job.row_begin;
                prev_nr = job.n_rows;
                ++tseq;
            }
            const uint32_t n_st = (job.n_codes + TC_STAGE_CODES - 1) / TC_STAGE_CODES;
            for (uint32_t st = 0; st < n_st; ++st, ++it) {
                const uint32_t b = it % TC_NSTAGE;
                TC_PROF(0);
                mbar_wait_park(&s_full[b], (it / TC_NSTAGE) & 1u);
                TC_PROF(1);
                const uint32_t first = st * TC_STAGE_CODES;
                const uint32_t cnt = min(uint32_t(TC_STAGE_CODES), job.n_codes - first);
                const char* sb = stage + size_t(b) * TC_STAGE_BYTES;
                const uint32_t n_sub = (cnt + TC_STEP - 1) / TC_STEP;
                // one sub-tile's operand: everything except the fences and the hand-over (two sub-tiles share those below)
                auto emit = [&](uint32_t sub, uint32_t s) {
                    const uint32_t sa = s % TC_NA;
                    TC_PROF(0);
                    mbar_wait_park(&s_aempty[sa], ((s / TC_NA) & 1u) ^ 1u); // the MMAs that read this stage have completed
                    TC_PROF(2);
                    const uint32_t sub_g = PAIR ? 2 * sub + rank : sub; // which 128 codes of the stage
                    const uint32_t i = sub_g * TC_SUB + g;
                    const bool valid = i < cnt;
                    uint2 code = make_uint2(0u, 0u);
                    if (valid) code = *reinterpret_cast<const uint2*>(sb + size_t(i) * 8);
                    char* dst = sA + size_t(sa) * TC_A_BYTES + (g >> 3) * 128 + (g & 7u) * 16;
                    if constexpr (SP) {
                        // 2:4-sparse one-hot row.  The K order is ours to choose (pack_tiles_tc8_kernel lays B out to match), and
                        // it is chosen so that the operand is a handful of shifts per table: K step ks covers the tables
                        // ks, ks + 4, ks + 8, ks + 12 (the nibbles at bit 4 ks of the code's four 16-bit quarters); entry n of
                        // a table sits in group n >> 2 at position 2 (n & 1) + ((n >> 1) & 1).  The kept pair of EVERY group of
                        // the table is (0, 1) if n is even and (2, 3) if n is odd -- the other groups' kept bytes are zero, so
                        // which positions they claim does not matter -- hence 16 metadata bits 0x4444 or 0xEEEE per table and
                        // the single 0x01 at compressed byte n >> 1.  Per K step: two 16-byte stores + two metadata columns.
                        const uint64_t one = valid ? 1ull : 0ull;
                        uint32_t meta[8];
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            uint64_t w[4];
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint32_t cw = c < 2 ? code.x : code.y;
                                const int lo = 4 * ks + 16 * (c & 1) + 1;                                 // bit position of n >> 1
                                const uint32_t sh = (lo >= 3 ? cw >> (lo >= 3 ? lo - 3 : 0) : cw << (3 - lo)) & 0x38u; // 8 (n >> 1)
                                w[c] = one << sh;
                            }
                            if (dbg & 2u) continue; // (timing experiment: nothing stored)
                            *reinterpret_cast<uint4*>(dst + (2 * ks) * TC_A_CHUNK) =
                                make_uint4(uint32_t(w[0]), uint32_t(w[0] >> 32), uint32_t(w[1]), uint32_t(w[1] >> 32));
                            *reinterpret_cast<uint4*>(dst + (2 * ks + 1) * TC_A_CHUNK) =
                                make_uint4(uint32_t(w[2]), uint32_t(w[2] >> 32), uint32_t(w[3]), uint32_t(w[3] >> 32));
                            meta[2 * ks] = ((code.x >> (4 * ks)) & 0x00010001u) * 0xAAAAu + 0x44444444u;
                            meta[2 * ks + 1] = ((code.y >> (4 * ks)) & 0x00010001u) * 0xAAAAu + 0x44444444u;
                        }
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                                         tmem + (((warp & 3u) * 32u) << 16) + TC_ECOL + sa * 8),
                                     "r"(meta[0]), "r"(meta[1]), "r"(meta[2]), "r"(meta[3]), "r"(meta[4]), "r"(meta[5]), "r"(meta[6]), "r"(meta[7])
                                     : "memory");
                    } else
                    if (!(dbg & 2u)) {
                        // 16 stores of 16 bytes: table j's chunk is a 0x01 byte at position c_j.  (A 17-entry table of the
                        // chunks in shared memory saves ALU work but its bank conflicts overload the shared-memory pipe the
                        // MMA operands come through: measured 1.6x slower.)
                        const uint32_t one = valid ? 1u : 0u; // padding rows: all zero (masked again in the epilogue)
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const uint32_t cw = j < 8 ? code.x : code.y;
                            const int sh = (j & 7) * 4 - 3;                                      // 8 * nibble, in place
                            const uint32_t n8 = (sh >= 0 ? cw >> (sh >= 0 ? sh : 0) : cw << 3) & 0x78u;
                            // the 128-bit value one << n8, word by word: a clamped funnel shift gives one << s for
                            // s < 32 and 0 for any larger (or "negative", i.e. huge unsigned) s -- 9 instructions per
                            // table where compare-and-select took 15
                            uint4 v;
                            v.x = __funnelshift_lc(0u, one, n8);
                            v.y = __funnelshift_lc(0u, one, n8 - 32u);
                            v.z = __funnelshift_lc(0u, one, n8 - 64u);
                            v.w = __funnelshift_lc(0u, one, n8 - 96u);
                            *reinterpret_cast<uint4*>(dst + j * TC_A_CHUNK) = v;
                        }
                    }
                    const uint32_t slot = s % TC_INFO;
                    info_codes[slot * TC_SUB + g] = code;
                    if (g == 0) {
                        SubInfo inf;
                        const uint64_t pos = uint64_t(first) + uint64_t(sub_g) * TC_SUB;
                        inf.id_ref = a->ids ? job.ids_off + pos : uint64_t(job.id_base) + pos;
                        inf.n_valid = sub_g * TC_SUB < cnt ? min(uint32_t(TC_SUB), cnt - sub_g * TC_SUB) : 0u;
                        inf.row_begin = job.row_begin;
                        inf.pad[0] = inf.pad[1] = 0;
                        s_info[slot] = inf;
                    }
                };
                // sub-tiles go out in pairs: the store fences and the mbarrier hand-over are pure latency for a generator
                // warp (one per scheduler), and with one pair of fences per two sub-tiles it keeps ahead of the sparse MMAs
                for (uint32_t sub = 0; sub < n_sub; sub += TC_GEN_GROUP, s += TC_GEN_GROUP) {
                    const bool two = TC_GEN_GROUP == 2 && sub + 1 < n_sub;
                    emit(sub, s);
                    if (two) emit(sub + 1, s + 1);
                    TC_PROF(0);
                    if constexpr (SP) {
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        tc_fence_before();
                    }
                    TC_PROF(3);
                    if (!(dbg & 16u)) proxy_fence();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive_leader<PAIR>(&s_afull[s % TC_NA], rank);
                        if (two) mbar_arrive_leader<PAIR>(&s_afull[(s + 1) % TC_NA], rank);
                    }
                    TC_PROF(4);
                    if (TC_GEN_GROUP == 2 && !two) s -= 1; // (the loop adds 2)
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[b]); // this warp is done with the code stage
            }
        }
#ifdef TC_PROFILE
        if (blockIdx.x == 0 && tid == TC_GEN_WARP0 * 32 && s > 2000)
            printf("tc-prof gen: subtiles %u total %lld | work %lld wait-codes %lld wait-aempty %lld wait-st %lld fence+arrive %lld (cycles per sub-tile: %lld)\n",
                   s, clock64() - prof_start, prof_t[0], prof_t[1], prof_t[2], prof_t[3], prof_t[4], (clock64() - prof_start) / s);
#endif
    } else if ((warp == TC_MMA_WARP || (SP && warp == TC_MMA_WARP2)) && rank == 0) {
        // ============================ MMA issuers (CTA pair: the leader's, for both CTAs) ======================
        // Two warps, one per accumulator buffer (even / odd steps).  A single issuer spends ~570 cycles per step outside
        // the MMAs themselves (barrier waits, fences, the commits, the compiler's elect loops around every uniform-datapath
        // instruction) while the tensor queue holds only a few MMAs: measured, the pipe idled 44 % of the time.  With two
        // issuers one's bookkeeping overlaps the other's MMAs; tcgen05.commit tracks the issuing thread's own MMAs, which is
        // exactly the per-buffer completion the barriers need.
        const uint32_t my_buf = warp == TC_MMA_WARP ? 0u : 1u;
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0), dbg_u = __shfl_sync(0xffffffffu, dbg, 0);
        uint32_t s = 0, tseq = 0, prev_rb = 0xFFFFFFFFu, prev_nr = 0;
        const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB), ap_base = smem_u32(sAp);
        TC_PROF_DECL(3);
#ifdef TC_PROFILE
        long long lat_rel = 0, t_mma = 0, t_commit = 0;
#endif
        for (uint32_t ji = j_begin; ji < j_end; ++ji) {
            const ScanJob job = a->jobs[ji];
            if (job.n_codes == 0 || job.n_rows == 0) continue;
            if (job.row_begin != prev_rb || job.n_rows != prev_nr) {
                prev_rb = job.row_begin;
                prev_nr = job.n_rows;
                if (tseq > 0 && lane == 0) umma_commit<PAIR>(&s_tempty); // every MMA on the old tile has completed
                __syncwarp();
                if constexpr (PAIR) mbar_wait_park_cluster(&s_tfull, tseq & 1u);
                else mbar_wait_park(&s_tfull, tseq & 1u);
                ++tseq;
            }
            // s counts UNITS = (step, tile of the job): accumulator buffer = s & 1 (NT = 2: the tile; NT = 1: step parity)
            const uint32_t n_sub = job_subtiles(job.n_codes, TC_STEP) * NT;
            for (uint32_t k = 0; k < n_sub; ++k, ++s) {
                const uint32_t sa = (s / NT) % TC_NA, buf = s & 1u;
                if (SP && buf != my_buf) continue; // (dense: one issuer -- alternating accumulators per MMA cost it 10 %)
                TC_PROF(0);
                if constexpr (PAIR) mbar_wait_park_cluster(&s_afull[sa], ((s / NT) / TC_NA) & 1u);
                else mbar_wait_park(&s_afull[sa], ((s / NT) / TC_NA) & 1u);
                TC_PROF(1);
                if constexpr (PAIR) mbar_wait_park_cluster(&s_dempty[buf], ((s >> 1) & 1u) ^ 1u);
                else mbar_wait_park(&s_dempty[buf], ((s >> 1) & 1u) ^ 1u);
                TC_PROF(2);
#ifdef TC_PROFILE
                if (lane == 0 && s >= 2) { lat_rel += clock64() - s_stamp[2][(s - 2) & 7u]; }
#endif
                tc_fence_after();
                if constexpr (SP) {
                    // converged issue (see umma_*_elect): sa / buf come from the loop counter of a uniform loop, and the shuffle
                    // tells the compiler so
                    const uint32_t sa_u = __shfl_sync(0xffffffffu, sa, 0), buf_u = __shfl_sync(0xffffffffu, buf, 0);
                    const uint32_t d = tmem_u + buf_u * TC_TQ;
                    const uint32_t a0 = a_base + sa_u * TC_A_BYTES;
                    const uint32_t b0 = b_base + (NT == 2 ? buf_u * uint32_t(TC_B_BYTES) : 0u); // this unit's tile
#ifdef TC_PROFILE
                    const long long t_m0 = clock64();
#endif
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) // four 2:4-sparse MMAs of 64 logical K (= four tables) each
                        if (ks == 0 || !(dbg_u & 4u))
                            umma_i8_sp_elect<PAIR>(d, umma_desc(a0 + ks * 2 * TC_A_CHUNK, TC_A_CHUNK, 128),
                                                   umma_desc(b0 + ks * 4 * TC_B_CHUNK, TC_B_CHUNK, 128),
                                                   tmem_u + TC_ECOL + sa_u * 8 + 2 * ks, TC_IDESC_SP, ks > 0);
                    if (!(dbg_u & 32u)) // (timing experiment: no threshold step)
                        umma_i8_elect<PAIR>(d, umma_desc(ap_base, TC_A_CHUNK, 128), umma_desc(b0 + TC_KC * TC_B_CHUNK, TC_B_CHUNK, 128),
                                            TC_IDESC, 1u);
#ifdef TC_PROFILE
                    const long long t_c0 = clock64();
                    t_mma += t_c0 - t_m0;
#endif
                    umma_commit_elect<PAIR>(&s_aempty[sa_u]); // the one-hot stage is free once these MMAs have read it
                    umma_commit_elect<PAIR>(&s_dfull[buf_u]); // ... and the accumulator is complete
#ifdef TC_PROFILE
                    if (lane == 0) {
                        s_stamp[0][s & 7u] = clock64();
                        t_commit += s_stamp[0][s & 7u] - t_c0;
                    }
#endif
                } else if (lane == 0) {
                    const uint32_t d = tmem + buf * TC_TQ;
                    const uint32_t a0 = a_base + sa * TC_A_BYTES;
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 2; ++ks)
                        if (ks == 0 || !(dbg & 4u))
                            umma_i8(d, umma_desc(a0 + ks * 2 * TC_A_CHUNK, TC_A_CHUNK, 128),
                                    umma_desc(b_base + ks * 2 * TC_B_CHUNK, TC_B_CHUNK, 128), TC_IDESC, ks > 0);
                    umma_i8(d, umma_desc(ap_base, TC_A_CHUNK, 128), umma_desc(b_base + TC_KC * TC_B_CHUNK, TC_B_CHUNK, 128), TC_IDESC, 1u);
                    umma_commit(&s_aempty[sa]); // the one-hot stage is free once these MMAs have read it
                    umma_commit(&s_dfull[buf]); // ... and the accumulator is complete
                }
                __syncwarp();
            }
        }
#ifdef TC_PROFILE
        if (blockIdx.x == 0 && lane == 0 && s > 2000 && my_buf == 0)
            printf("tc-prof mma: subtiles %u total %lld | issue %lld (the MMAs %lld, the commits %lld) wait-afull %lld wait-dempty %lld | release(s-2) -> past dempty(s) %lld\n", s,
                   clock64() - prof_start, prof_t[0], t_mma, t_commit, prof_t[1], prof_t[2], lat_rel);
#endif
    } else if (warp < TC_EPI_WARPS) {
        // ============================ epilogue: TMEM -> sign test -> exact admission ==========================
        uint32_t s = 0;
        const uint32_t quad = warp & 3u, half_w = warp >> 2;   // TMEM lane quadrant, column half
        const uint32_t rowi = quad * 32 + lane;                 // this thread's code (row of the sub-tile)
        const uint32_t lane_base = (quad * 32u) << 16;
        const uint32_t col_w = half_w * (TC_TQ / 2);
        uint64_t* wq_key = s_wq_key + warp * TC_WQ_CAP;
        uint32_t* wq_row = s_wq_row + warp * TC_WQ_CAP;
        uint32_t* wq_id = s_wq_id + warp * TC_WQ_CAP;
        uint32_t qn = 0; // warp-uniform fill level of the queue
        const uint32_t* ids_ptr = a->ids;
        TC_PROF_DECL(3);
#ifdef TC_PROFILE
        long long lat_wake = 0, lat_read = 0;
#endif
        const uint32_t lt_mask = (1u << lane) - 1u;
        auto drain = [&]() { // 32 admissions in flight at once (the atomics' round trips overlap)
            __syncwarp();
            for (uint32_t base = 0; base < qn; base += 32) {
                const uint32_t e = base + lane;
                if (e < qn) {
                    // the queue holds COORDINATES (code, table row, id) of flagged pairs; the sum is recomputed from the
                    // reference-order table -- 16 independent byte loads -- and goes through the CandidateHeap::push test
                    // against the query's current key (exact_admit_ct, scan_common.cuh)
                    const uint64_t code = wq_key[e];
                    tc_exact_admit(ds, a, uint32_t(code), uint32_t(code >> 32), wq_row[e], wq_id[e]);
                }
            }
            __syncwarp();
            qn = 0;
        };
        for (uint32_t ji = j_begin; ji < j_end; ++ji) {
            const ScanJob job = a->jobs[ji];
            if (job.n_codes == 0 || job.n_rows == 0) continue;
            const uint32_t n_sub = job_subtiles(job.n_codes, TC_STEP) * NT; // units, as in the MMA warps
            for (uint32_t k = 0; k < n_sub; ++k, ++s) {
                const uint32_t buf = s & 1u, slot = (s / NT) % TC_INFO;
                const uint32_t toff = NT == 2 ? buf * uint32_t(TC_TQ) : 0u; // first row of this unit's tile within the job
                TC_PROF(0);
                mbar_wait_park(&s_dfull[buf], (s >> 1) & 1u);
                TC_PROF(1);
#ifdef TC_PROFILE
                if (tid == 0) { s_stamp[1][s & 7u] = clock64(); lat_wake += s_stamp[1][s & 7u] - s_stamp[0][s & 7u]; }
#endif
                tc_fence_after();
                if (!(dbg & 1u)) {
                    // this warp's 128 queries of the tile, two 16-bit sums per register (the sub-tile's info is fetched
                    // while the tensor-memory load is in flight)
                    const uint32_t c0 = col_w;
                    uint32_t v[64];
                    tmem_ld128_pack16(tmem + buf * TC_TQ + lane_base + c0, v);
                    const SubInfo inf = s_info[slot];
                    const bool valid = rowi < inf.n_valid;
                    tmem_ld_wait();
                    TC_PROF(2);
                    if constexpr (SP) { // a warp owns 120 of the tile's 240 queries: the load's last 8 columns are not its own
                        v[60] = v[61] = v[62] = v[63] = 0u;
                    }
                    // everything this warp needs from the accumulator is in registers now: hand the buffer back to the MMA
                    // warp BEFORE looking at the values (admissions never touch tensor memory again)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_leader<PAIR>(&s_dempty[buf], rank);
#ifdef TC_PROFILE
                    if (tid == 0) { s_stamp[2][s & 7u] = clock64(); lat_read += s_stamp[2][s & 7u] - s_stamp[1][s & 7u]; }
#endif
                    uint32_t g[4]; // OR of each group of 16 registers = 32 columns (four independent chains)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        uint32_t o = 0;
#pragma unroll
                        for (int j = 0; j < 16; j += 2) o |= v[16 * k + j] | v[16 * k + j + 1];
                        g[k] = o & 0x80008000u; // sign bits of the even / odd columns
                    }
                    const uint32_t any = g[0] | g[1] | g[2] | g[3];
                    const uint32_t hit_lanes = __ballot_sync(0xffffffffu, valid && any != 0u);
                    if (hit_lanes != 0u && !(dbg & 8u)) {
                        // rare (warp-uniform branch): some sums of this sub-tile are <= their query's threshold (D = bias + sum -
                        // thr - 1 is negative).  Nothing but the sign is used from here on.
                        {
                            // LANE-LOCAL admission: every lane with flagged sums turns its sign bits into column
                            // masks and queues the pairs' COORDINATES (code, table row, id); drain() recomputes their sums
                            // exactly.  No votes or reductions in the loop.  (A warp-uniform walk over the union of flagged
                            // columns, picking values out of the registers, cost ~1000 cycles per visit.)
                            uint32_t m[4];
                            uint32_t todo = 0;
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                m[k] = 0u;
                                if (valid && g[k] != 0u) {
                                    uint32_t part[4] = {0u, 0u, 0u, 0u}; // four short OR chains instead of one of sixteen
#pragma unroll
                                    for (int i = 0; i < 16; ++i) {
                                        const uint32_t x = i == 15 ? v[16 * k + i] : (v[16 * k + i] >> (15 - i));
                                        part[i & 3] |= x & (0x00010001u << i);
                                    }
                                    m[k] = (part[0] | part[1]) | (part[2] | part[3]);
                                    todo |= 1u << k;
                                }
                            }
                            // the visit only queues coordinates: no accumulator value is needed again (drain() recomputes the
                            // sum), so there is no register indexing, no threshold lookup and no compare on this path
                            const uint32_t id = ids_ptr ? ids_ptr[inf.id_ref + min(rowi, max(inf.n_valid, 1u) - 1u)] : uint32_t(inf.id_ref) + rowi;
                            const uint2 code2 = info_codes[slot * TC_SUB + rowi];
                            const uint64_t code = (uint64_t(code2.y) << 32) | code2.x;
                            const uint32_t rowbase = inf.row_begin + toff + c0;
                            uint32_t* wqn = &s_wqn[warp];
                            // the common case -- ONE lane has flagged sums and they fit the queue: it takes the next slots
                            // itself, no atomic and no round trip through shared memory for the fill level
                            const uint32_t n_mine = uint32_t(__popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]));
                            const uint32_t n_one = __shfl_sync(0xffffffffu, n_mine, __ffs(hit_lanes) - 1);
                            if ((hit_lanes & (hit_lanes - 1u)) == 0u && qn + n_one <= uint32_t(TC_WQ_CAP)) {
                                uint32_t e = qn;
                                for (uint32_t t = todo; t != 0u; t &= t - 1u) { // (one copy of the loop: flagged groups only)
                                    const uint32_t k = uint32_t(__ffs(t) - 1);
                                    uint32_t mk = k == 0 ? m[0] : k == 1 ? m[1] : k == 2 ? m[2] : m[3];
                                    for (; mk != 0u; mk &= mk - 1u, ++e) {
                                        const uint32_t b = uint32_t(__ffs(mk) - 1);
                                        wq_key[e] = code;
                                        wq_row[e] = rowbase + k * 32 + 2 * (b & 15u) + (b >> 4);
                                        wq_id[e] = id;
                                    }
                                }
                                qn += n_one;
                                __syncwarp();
                            } else {
                            if (lane == 0) *wqn = qn; // the shared fill level is only kept for this path
                            __syncwarp();
                            uint32_t mcur = 0, kcur = 0;
                            for (;;) {
                                bool blocked = false; // the queue is full: drain it (warp-wide) and come back
                                while ((todo | mcur) != 0u && !blocked) {
                                    if (mcur == 0u) { // this lane's next flagged group
                                        kcur = uint32_t(__ffs(todo) - 1);
                                        todo &= todo - 1u;
                                        mcur = kcur == 0 ? m[0] : kcur == 1 ? m[1] : kcur == 2 ? m[2] : m[3];
                                    }
                                    const uint32_t b = uint32_t(__ffs(mcur) - 1);
                                    const uint32_t e = atomicAdd(wqn, 1u);
                                    if (e >= uint32_t(TC_WQ_CAP)) {
                                        blocked = true; // (the bit stays set: retried after the drain)
                                        continue;
                                    }
                                    wq_key[e] = code;
                                    wq_row[e] = rowbase + kcur * 32 + 2 * (b & 15u) + (b >> 4);
                                    wq_id[e] = id;
                                    mcur &= mcur - 1u;
                                }
                                __syncwarp();
                                const uint32_t cnt = *wqn; // > capacity <=> some lane could not push and waits for a drain
                                qn = min(cnt, uint32_t(TC_WQ_CAP));
                                if (cnt <= uint32_t(TC_WQ_CAP)) break;
                                drain();
                                if (lane == 0) *wqn = 0u;
                                __syncwarp();
                            }
                            }
                        }
                    }
                }
                if (qn >= 32) drain();
                if (dbg & 1u) { // (timing experiment: nothing was read)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_leader<PAIR>(&s_dempty[buf], rank);
                }
            }
        }
        if (qn) drain();
#ifdef TC_PROFILE
        if (blockIdx.x == 0 && tid == 0 && s > 2000)
            printf("tc-prof epi: subtiles %u total %lld | work %lld wait-dfull %lld tmem-load %lld | commit(s) -> past dfull(s) %lld, -> released %lld\n", s,
                   clock64() - prof_start, prof_t[0], prof_t[1], prof_t[2], lat_wake, lat_read);
#endif
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) {
        cluster_sync_all(); // neither CTA leaves (or frees tensor memory) while the other may still arrive on its barriers
        if (warp == TC_MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    } else {
        if (warp == TC_MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    }
}

// ------------------------------------------------------------------------------------------ tile image --

// qlut [n_rows][256] u8 (reference table order) -> per tile of tq rows the B operand image
// [kc = 16][row = tq][16 bytes] of e - 128 (two's complement: e ^ 0x80); rows past n_rows hold e = 0.
// Dense: chunk kc = table kc in entry order.  Sparse (the generator's K order): chunk 4 ks + c = table ks + 4 c, and byte
// 4 g + p of the chunk = entry 4 g + 2 (p & 1) + (p >> 1).
__global__ void pack_tiles_tc8_kernel(const uint8_t* __restrict__ qlut, uint32_t n_rows, uint32_t tq, uint32_t sparse,
                                      uint8_t* __restrict__ out) {
    const uint32_t tile = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < uint32_t(TC_KC) * tq; i += blockDim.x) {
        const uint32_t kc = i / tq, r = i % tq;
        const uint32_t row = tile * tq + r;
        const uint32_t table = sparse ? (kc >> 2) + 4 * (kc & 3u) : kc;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row < n_rows) v = *reinterpret_cast<const uint4*>(qlut + size_t(row) * 256 + table * 16);
        if (sparse) { // within every group of four entries: (e0, e1, e2, e3) -> (e0, e2, e1, e3)
            v.x = __byte_perm(v.x, 0u, 0x3120);
            v.y = __byte_perm(v.y, 0u, 0x3120);
            v.z = __byte_perm(v.z, 0u, 0x3120);
            v.w = __byte_perm(v.w, 0u, 0x3120);
        }
        v.x ^= 0x80808080u;
        v.y ^= 0x80808080u;
        v.z ^= 0x80808080u;
        v.w ^= 0x80808080u;
        *reinterpret_cast<uint4*>(out + size_t(tile) * (TC_KC * tq * 16) + size_t(kc) * (tq * 16) + r * 16) = v;
    }
}

// mode: 0 dense, 1 2:4-sparse, 2 2:4-sparse on CTA pairs
uint32_t scan_tc8_smem_bytes(int mode) { return mode == 2 ? tc_smem(true, true) : mode == 1 ? tc_smem(true) : tc_smem(false); }
uint32_t scan_tc8_tile_rows(int mode) { return tc_tq(mode != 0) * tc_nt(mode == 2); } // rows of a JOB's tile (pair form: two images)
uint32_t scan_tc8_pack_rows(int mode) { return tc_tq(mode != 0); }                     // rows of one packed tile image

// `images_per_tile` consecutive images make one job tile: the image count is rounded up to a whole number of them
void launch_pack_tiles_tc8(const void* qlut, uint32_t n_rows, uint32_t tq, uint32_t images_per_tile, void* out, cudaStream_t stream) {
    if (n_rows == 0) return;
    const uint32_t images = ((n_rows + tq - 1) / tq + images_per_tile - 1) / images_per_tile * images_per_tile;
    pack_tiles_tc8_kernel<<<images, 256, 0, stream>>>(static_cast<const uint8_t*>(qlut), n_rows, tq,
                                                                      tq == uint32_t(tc_tq(true)) ? 1u : 0u, static_cast<uint8_t*>(out));
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

void launch_scan_tc8(int mode, const DevSpec& ds, const ScanArgs& args, int grid, cudaStream_t stream) {
    if (mode == 2) {
        // CTA pairs: clusters of two, at most one pair per TPC; `grid` arrives as min(SMs, jobs)
        int dev = 0, sms = 0;
        QADC_CUDA_CHECK(cudaGetDevice(&dev));
        QADC_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int pairs = std::max(1, std::min(grid, sms / 2));
        auto kern = scan_tc8_kernel<true, true>;
        QADC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(true, true)));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(2 * pairs));
        cfg.blockDim = dim3(TC_THREADS);
        cfg.dynamicSmemBytes = tc_smem(true, true);
        cfg.stream = stream;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = 2;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        QADC_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ds, args));
    } else if (mode == 1) {
        auto kern = scan_tc8_kernel<true, false>;
        QADC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(true)));
        kern<<<grid, TC_THREADS, tc_smem(true), stream>>>(ds, args);
    } else {
        auto kern = scan_tc8_kernel<false, false>;
        QADC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(false)));
        kern<<<grid, TC_THREADS, tc_smem(false), stream>>>(ds, args);
    }
    ++g_launches;
    QADC_CUDA_CHECK(cudaGetLastError());
}

} // namespace qadc

