// umma_probe.cu -- stand-alone validation + micro-benchmark of the tcgen05 building blocks the product kernels use
// (NOT part of libqadc_b200.so).  There is no PTX manual in this image, so the operand layouts are pinned here
// against a CPU reference before a product kernel relies on them:
//   1. kind::i8  SS MMA, K-major no-swizzle canonical layout (core matrix = 8 rows x 16 bytes), u8 x u8 and u8 x s8,
//      accumulation over several K steps, D read back with tcgen05.ld.32x32b;
//   2. kind::f16 (bf16 -> f32) the same way;
//   3. rates: back-to-back MMAs per SM (tensor pipe), tcgen05.ld bandwidth.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe tools/umma_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(2);                                                                      \
        }                                                                                 \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!done);
}
// shared-memory matrix descriptor, no swizzle, K-major: LBO = bytes between the two 16-byte K chunks of one MMA,
// SBO = bytes between consecutive 8-row groups (cute::UMMA::SmemDescriptor, version 1)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
           (uint64_t(1) << 46);
}
// instruction descriptor (cute::UMMA::InstrDescriptor): c_format [4,6) a_format [7,10) b_format [10,13) n>>3 [17,23) m>>4 [24,29)
__host__ __device__ constexpr uint32_t idesc(uint32_t cfmt, uint32_t afmt, uint32_t bfmt, uint32_t M, uint32_t N) {
    return (cfmt << 4) | (afmt << 7) | (bfmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&v)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
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

// ---------------------------------------------------------------------------------------------------------------
// Test 1/2: D[128 x N] = A[128 x K] * B[N x K]^T with operands given row-major (K contiguous) in global memory.
// ELT = bytes per element (1: i8 kinds, 2: bf16).  K bytes per MMA = 32.  Operand tile in smem:
//   addr(row, kbyte) = (kbyte / 16) * (ROWS * 16) + (row / 8) * 128 + (row % 8) * 16 + kbyte % 16
// i.e. LBO = ROWS * 16, SBO = 128.
template <int ELT>
__global__ void __launch_bounds__(128) mma_check_kernel(const uint8_t* A, const uint8_t* B, uint32_t N, uint32_t Kbytes,
                                                        uint32_t id, uint32_t* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    uint8_t* sa = sm;
    uint8_t* sb = sm + 128 * Kbytes;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid; i < 128 * Kbytes; i += 128) {
        const uint32_t row = i / Kbytes, kb = i % Kbytes;
        sa[(kb / 16) * (128 * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = A[i];
    }
    for (uint32_t i = tid; i < N * Kbytes; i += 128) {
        const uint32_t row = i / Kbytes, kb = i % Kbytes;
        sb[(kb / 16) * (N * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // generic-proxy smem writes -> visible to the MMA (async proxy)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base;
    if (tid == 0) {
        for (uint32_t ks = 0; ks < Kbytes / 32; ++ks) {
            const uint64_t da = smem_desc(smem_u32(sa) + ks * 2 * (128 * 16), 128 * 16, 128);
            const uint64_t db = smem_desc(smem_u32(sb) + ks * 2 * (N * 16), N * 16, 128);
            if (ELT == 1) mma_i8(tb, da, db, id, ks > 0);
            else mma_f16(tb, da, db, id, ks > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (uint32_t c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tb + ((warp * 32u) << 16) + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j)
            if (c0 + j < N) D[size_t(tid) * N + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(256));
}


__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(d), "r"(a_tmem), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
// Test 1b: A in TMEM.  Hypothesis: row r of A lives in lane r; byte k of the row is byte (k % 4) of column a_col0 + k / 4.
__global__ void __launch_bounds__(128) mma_ts_check_kernel(const uint8_t* A, const uint8_t* B, uint32_t N, uint32_t Kbytes,
                                                           uint32_t id, uint32_t* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    uint8_t* sb = sm;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid; i < N * Kbytes; i += 128) {
        const uint32_t row = i / Kbytes, kb = i % Kbytes;
        sb[(kb / 16) * (N * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base, a_col0 = 256;
    // thread = row: write its K bytes, 8 columns (32 bytes) at a time
    for (uint32_t k0 = 0; k0 < Kbytes; k0 += 32) {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = *reinterpret_cast<const uint32_t*>(A + size_t(tid) * Kbytes + k0 + 4 * j);
        tmem_st8(tb + ((warp * 32u) << 16) + a_col0 + k0 / 4, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        for (uint32_t ks = 0; ks < Kbytes / 32; ++ks) {
            const uint64_t db = smem_desc(smem_u32(sb) + ks * 2 * (N * 16), N * 16, 128);
            mma_i8_ts(tb, tb + a_col0 + ks * 8, db, id, ks > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (uint32_t c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tb + ((warp * 32u) << 16) + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j)
            if (c0 + j < N) D[size_t(tid) * N + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}


// ---------------------------------------------------------------------------------------------------------------
// Test 1c: 2:4-sparse kind::i8.  Logical A [128][64] with at most two non-zeros per group of four K elements is
// stored compressed (32 bytes per row, the dense K = 32 tile layout) + 4 metadata bits per group in tensor memory
// (lane = row, two columns = 64 bits per row per instruction).  `hyp` selects the metadata encoding under test.
__device__ __forceinline__ void mma_i8_sp(uint32_t d, uint64_t a, uint64_t b, uint32_t e_tmem, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\ntcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(e_tmem), "r"(id), "r"(acc) : "memory");
}
__global__ void __launch_bounds__(128) mma_sp_check_kernel(const uint8_t* Ac, const uint32_t* meta /* [128][2] */, const uint8_t* B,
                                                           uint32_t N, uint32_t id, uint32_t* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    uint8_t* sa = sm;             // 128 x 32 B
    uint8_t* sb = sm + 128 * 32;  // N x 64 B
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid; i < 128 * 32; i += 128) {
        const uint32_t row = i / 32, kb = i % 32;
        sa[(kb / 16) * (128 * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = Ac[i];
    }
    for (uint32_t i = tid; i < N * 64; i += 128) {
        const uint32_t row = i / 64, kb = i % 64;
        sb[(kb / 16) * (N * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base, e_col = 256;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(tb + ((warp * 32u) << 16) + e_col),
                 "r"(meta[tid * 2]), "r"(meta[tid * 2 + 1]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        mma_i8_sp(tb, smem_desc(smem_u32(sa), 128 * 16, 128), smem_desc(smem_u32(sb), N * 16, 128), tb + e_col, id, 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (uint32_t c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tb + ((warp * 32u) << 16) + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j)
            if (c0 + j < N) D[size_t(tid) * N + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}

// ---------------------------------------------------------------------------------------------------------------
// Rates.  mode 0: one thread issues `iters` x 8 MMAs (M=128, N, K=32 B each, i8) into two alternating accumulators,
// nobody reads them (tensor pipe + operand fetch only).  mode 1: additionally 4 warps read the 128 x N s32
// accumulator after every 8 MMAs (the product kernel's epilogue traffic), double-buffered through 2 mbarrier pairs.
// EW epilogue warps (4 or 8: warp w reads lane quadrant w % 4 and column half w / 4), batches of BATCH columns
// (32, 64 or 128 = two x64 loads) per tcgen05.wait::ld.  KSTEPS MMAs of K = 32 bytes per tile.
template <int N, int EW, int BATCH, int KSTEPS>
__global__ void __launch_bounds__(EW * 32 + 32) mma_rate_kernel(uint32_t iters, int mode, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[2], empty[2];
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid; i < (128 + N) * 32 * KSTEPS / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 1);
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], EW * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base;
    const uint32_t id = idesc(2, 0, 0, 128, N);
    if (warp == EW) { // MMA issuer
        if ((tid & 31) == 0) {
            const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 32 * KSTEPS);
            for (uint32_t it = 0; it < iters; ++it) {
                const uint32_t buf = it & 1;
                if (mode == 1) mbar_wait(&empty[buf], ((it >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (uint32_t ks = 0; ks < KSTEPS; ++ks)
                    mma_i8(tb + buf * 256, smem_desc(a0 + ks * 2 * 2048, 2048, 128), smem_desc(b0 + ks * 2 * (N * 16), N * 16, 128), id, ks > 0);
                mma_commit(&full[buf]);
            }
            if (mode == 0) mbar_wait(&full[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
        }
    } else if (warp < EW && mode == 1) {
        uint32_t acc = 0;
        constexpr uint32_t COLS = N / (EW / 4);
        const uint32_t col0 = (warp / 4) * COLS, lane_base = ((warp & 3u) * 32u) << 16;
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t buf = it & 1;
            mbar_wait(&full[buf], (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (uint32_t c0 = 0; c0 < COLS; c0 += BATCH) {
                const uint32_t t0 = tb + buf * 256 + lane_base + col0 + c0;
                if constexpr (BATCH == 32) {
                    uint32_t v[32];
                    tmem_ld32(t0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; j += 2) acc |= v[j] | v[j + 1];
                } else if constexpr (BATCH == 64) {
                    uint32_t v[64];
                    tmem_ld64(t0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 64; j += 2) acc |= v[j] | v[j + 1];
                } else {
                    uint32_t v[64], w[64];
                    tmem_ld64(t0, v);
                    tmem_ld64(t0 + 64, w);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 64; j += 2) acc |= v[j] | v[j + 1];
#pragma unroll
                    for (int j = 0; j < 64; j += 2) acc |= w[j] | w[j + 1];
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[buf])) : "memory");
        }
        if (acc == 0x12345678u) sink[tid] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}

template <int EW, int BATCH, int KSTEPS>
static void run_rate(int sms, int clock_khz, int mode, uint32_t* sink) {
    const uint32_t iters = 4000;
    const size_t smem = (128 + 256) * 32 * KSTEPS;
    auto k = mma_rate_kernel<256, EW, BATCH, KSTEPS>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k<<<sms, EW * 32 + 32, smem>>>(100, mode, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    k<<<sms, EW * 32 + 32, smem>>>(iters, mode, sink);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double macs = double(iters) * KSTEPS * 128 * 256 * 32 * sms;
    printf("rate M=128 N=256 K=%d %-34s: %.3f ms, %6.1f TOP/s, %7.1f cycles/tile, %.3e pairs/s\n", KSTEPS * 32,
           mode ? (EW == 4 ? (BATCH == 32 ? "4 epi warps, 32 cols/wait" : BATCH == 64 ? "4 epi warps, 64 cols/wait" : "4 epi warps, 128 cols/wait")
                           : (BATCH == 32 ? "8 epi warps, 32 cols/wait" : BATCH == 64 ? "8 epi warps, 64 cols/wait" : "8 epi warps, 128 cols/wait"))
                : "MMA only",
           ms, 2 * macs / ms / 1e9, ms * 1e-3 * clock_khz * 1e3 / iters, double(iters) * 128 * 256 * sms / (ms * 1e-3));
}


// Rate of the sparse form: per tile NSP sparse MMAs (K = 64 logical each) + one dense K = 32 MMA into alternating
// accumulators of N columns (N = 240 leaves 32 TMEM columns for two metadata stages), nobody reads them.
template <int N, int NSP>
__global__ void __launch_bounds__(64) mma_sp_rate_kernel(uint32_t iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[2];
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid; i < (128 * 32 + N * 64) * NSP / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 1);
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base;
    for (int c = 0; c < 32; c += 2) // metadata: every group keeps positions (0, 1): nibble 0x4
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(tb + ((warp * 32u) << 16) + 480 + c), "r"(0x44444444u), "r"(0x44444444u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 32) {
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 32 * NSP);
        const uint32_t id_sp = idesc(2, 0, 1, 128, N) | (1u << 2), id_d = idesc(2, 0, 1, 128, N);
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t buf = it & 1;
            for (uint32_t ks = 0; ks < NSP; ++ks)
                mma_i8_sp(tb + buf * N, smem_desc(a0 + ks * 2 * 2048, 2048, 128), smem_desc(b0 + ks * 4 * (N * 16), N * 16, 128),
                          tb + 480 + (ks & 7) * 2, id_sp, ks > 0);
            mma_i8(tb + buf * N, smem_desc(a0, 2048, 128), smem_desc(b0, N * 16, 128), id_d, 1);
            mma_commit(&full[buf]);
        }
        mbar_wait(&full[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}

static float bf16_to_f(uint16_t b) {
    uint32_t u = uint32_t(b) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    printf("device %s, %d SMs, clock %d MHz\n", prop.name, sms, prop.clockRate / 1000);
    srand(1);
    int fails = 0, ts_fails = 0;
    // ---- i8 checks
    for (int sgn = 0; sgn < 2; ++sgn)
        for (uint32_t N : {64u, 128u, 256u})
            for (uint32_t Kb : {32u, 64u, 256u}) {
                std::vector<uint8_t> A(128 * Kb), B(N * Kb);
                for (auto& x : A) x = rand() & 255;
                for (auto& x : B) x = rand() & 255;
                uint8_t *dA, *dB;
                uint32_t* dD;
                CK(cudaMalloc(&dA, A.size()));
                CK(cudaMalloc(&dB, B.size()));
                CK(cudaMalloc(&dD, 128 * N * 4));
                CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
                const size_t smem = (128 + N) * Kb;
                CK(cudaFuncSetAttribute(mma_check_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                mma_check_kernel<1><<<1, 128, smem>>>(dA, dB, N, Kb, idesc(2, 0, sgn, 128, N), dD);
                CK(cudaDeviceSynchronize());
                std::vector<int32_t> D(128 * N);
                CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
                long bad = 0;
                for (uint32_t r = 0; r < 128; ++r)
                    for (uint32_t c = 0; c < N; ++c) {
                        int32_t s = 0;
                        for (uint32_t k = 0; k < Kb; ++k)
                            s += int32_t(A[r * Kb + k]) * (sgn ? int32_t(int8_t(B[c * Kb + k])) : int32_t(B[c * Kb + k]));
                        bad += s != D[r * N + c];
                    }
                printf("i8 %s N=%3u Kbytes=%3u: %s (%ld mismatches)\n", sgn ? "u8 x s8" : "u8 x u8", N, Kb, bad ? "FAIL" : "ok", bad);
                fails += bad != 0;
                cudaFree(dA); cudaFree(dB); cudaFree(dD);
            }

    // ---- i8 TS-mode check (A in TMEM)
    for (uint32_t N : {128u, 256u})
        for (uint32_t Kb : {32u, 256u}) {
            std::vector<uint8_t> A(128 * Kb), B(N * Kb);
            for (auto& x : A) x = rand() & 255;
            for (auto& x : B) x = rand() & 255;
            uint8_t *dA, *dB;
            uint32_t* dD;
            CK(cudaMalloc(&dA, A.size()));
            CK(cudaMalloc(&dB, B.size()));
            CK(cudaMalloc(&dD, 128 * N * 4));
            CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
            CK(cudaMemset(dD, 0xEE, 128 * N * 4));
            const size_t smem = N * Kb;
            CK(cudaFuncSetAttribute(mma_ts_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            mma_ts_check_kernel<<<1, 128, smem>>>(dA, dB, N, Kb, idesc(2, 0, 1, 128, N), dD);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("i8 TS N=%3u Kbytes=%3u: CUDA error %s\n", N, Kb, cudaGetErrorString(e));
                return 3;
            }
            std::vector<int32_t> D(128 * N);
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            long bad = 0;
            for (uint32_t r = 0; r < 128; ++r)
                for (uint32_t c = 0; c < N; ++c) {
                    int32_t s2 = 0;
                    for (uint32_t k = 0; k < Kb; ++k) s2 += int32_t(A[r * Kb + k]) * int32_t(int8_t(B[c * Kb + k]));
                    bad += s2 != D[r * N + c];
                }
            printf("i8 TS (A in TMEM) u8 x s8 N=%3u Kbytes=%3u: %s (%ld mismatches)\n", N, Kb, bad ? "FAIL" : "ok", bad);
            ts_fails += bad != 0;
            cudaFree(dA); cudaFree(dB); cudaFree(dD);
        }

    // ---- 2:4 sparse i8 check, several metadata encodings
    for (int hyp = 0; hyp < 4; ++hyp)
        for (uint32_t N : {64u, 240u}) {
            std::vector<uint8_t> A(128 * 64, 0), Ac(128 * 32), B(N * 64);
            std::vector<uint32_t> meta(128 * 2, 0);
            for (auto& x : B) x = rand() & 255;
            for (uint32_t r = 0; r < 128; ++r)
                for (uint32_t g = 0; g < 16; ++g) {
                    uint32_t i0 = rand() % 3, i1 = i0 + 1 + rand() % (3 - i0);
                    const uint8_t v0 = rand() & 255, v1 = rand() & 255;
                    A[r * 64 + 4 * g + i0] = v0;
                    A[r * 64 + 4 * g + i1] = v1;
                    Ac[r * 32 + 2 * g] = v0;
                    Ac[r * 32 + 2 * g + 1] = v1;
                    const uint32_t nib = (hyp & 1) ? (i1 | (i0 << 2)) : (i0 | (i1 << 2));
                    const uint32_t gg = (hyp & 2) ? (g ^ 8) : g;
                    meta[r * 2 + gg / 8] |= nib << (4 * (gg % 8));
                }
            uint8_t *dA, *dB;
            uint32_t *dD, *dM;
            CK(cudaMalloc(&dA, Ac.size()));
            CK(cudaMalloc(&dB, B.size()));
            CK(cudaMalloc(&dM, meta.size() * 4));
            CK(cudaMalloc(&dD, 128 * N * 4));
            CK(cudaMemcpy(dA, Ac.data(), Ac.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dM, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(dD, 0xEE, 128 * N * 4));
            const size_t smem = 128 * 32 + N * 64;
            CK(cudaFuncSetAttribute(mma_sp_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            mma_sp_check_kernel<<<1, 128, smem>>>(dA, dM, dB, N, idesc(2, 0, 1, 128, N) | (1u << 2), dD);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("i8 SPARSE hyp %d N=%3u: CUDA error %s\n", hyp, N, cudaGetErrorString(e));
                return 3;
            }
            std::vector<int32_t> D(128 * N);
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            long bad = 0;
            for (uint32_t r = 0; r < 128; ++r)
                for (uint32_t c = 0; c < N; ++c) {
                    int32_t s2 = 0;
                    for (uint32_t k = 0; k < 64; ++k) s2 += int32_t(A[r * 64 + k]) * int32_t(int8_t(B[c * 64 + k]));
                    bad += s2 != D[r * N + c];
                }
            printf("i8 SPARSE 2:4 (K=64) hyp %d N=%3u: %s (%ld mismatches; D[0][0]=%d D[5][7]=%d)\n", hyp, N, bad ? "no" : "MATCH", bad, D[0], D[5 * N + 7]);
            cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dM);
        }
    // ---- bf16 checks (K elements = Kbytes / 2)
    for (uint32_t N : {64u, 256u})
        for (uint32_t Kb : {32u, 256u}) {
            const uint32_t K = Kb / 2;
            std::vector<uint16_t> A(128 * K), B(N * K);
            for (auto& x : A) x = uint16_t(0x3c00 + (rand() & 0x3ff) + ((rand() & 1) << 15)); // +-[0.0078, 0.0156..)
            for (auto& x : B) x = uint16_t(0x3c00 + (rand() & 0x3ff) + ((rand() & 1) << 15));
            uint8_t *dA, *dB;
            uint32_t* dD;
            CK(cudaMalloc(&dA, A.size() * 2));
            CK(cudaMalloc(&dB, B.size() * 2));
            CK(cudaMalloc(&dD, 128 * N * 4));
            CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
            const size_t smem = (128 + N) * Kb;
            CK(cudaFuncSetAttribute(mma_check_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            mma_check_kernel<2><<<1, 128, smem>>>(dA, dB, N, Kb, idesc(1, 1, 1, 128, N), dD); // f32 accum, bf16 x bf16
            CK(cudaDeviceSynchronize());
            std::vector<float> D(128 * N);
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            long bad = 0;
            double maxrel = 0;
            for (uint32_t r = 0; r < 128; ++r)
                for (uint32_t c = 0; c < N; ++c) {
                    double s = 0, sa = 0;
                    for (uint32_t k = 0; k < K; ++k) {
                        const double p = double(bf16_to_f(A[r * K + k])) * double(bf16_to_f(B[c * K + k]));
                        s += p;
                        sa += p < 0 ? -p : p;
                    }
                    const double err = (double(D[r * N + c]) - s) / (sa + 1e-30);
                    maxrel = err < 0 ? (-err > maxrel ? -err : maxrel) : (err > maxrel ? err : maxrel);
                    bad += !(err < 1e-5 && err > -1e-5);
                }
            printf("bf16 N=%3u K=%3u: %s (%ld off, max |err| / sum|terms| = %.3g)\n", N, K, bad ? "FAIL" : "ok", bad, maxrel);
            fails += bad != 0;
            cudaFree(dA); cudaFree(dB); cudaFree(dD);
        }
    // ---- rates
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4096));
    run_rate<4, 32, 8>(sms, prop.clockRate, 0, sink);
    run_rate<4, 32, 9>(sms, prop.clockRate, 0, sink);
    run_rate<4, 32, 8>(sms, prop.clockRate, 1, sink);
    run_rate<4, 64, 8>(sms, prop.clockRate, 1, sink);
    run_rate<4, 128, 8>(sms, prop.clockRate, 1, sink);
    run_rate<8, 32, 8>(sms, prop.clockRate, 1, sink);
    run_rate<8, 64, 8>(sms, prop.clockRate, 1, sink);
    run_rate<8, 128, 8>(sms, prop.clockRate, 1, sink);
    run_rate<8, 128, 9>(sms, prop.clockRate, 1, sink);
    run_rate<8, 128, 4>(sms, prop.clockRate, 1, sink);
    {
        const uint32_t iters = 4000;
        const size_t smem = (128 * 32 + 240 * 64) * 4;
        auto k = mma_sp_rate_kernel<240, 4>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        k<<<sms, 64, smem>>>(100);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        k<<<sms, 64, smem>>>(iters);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("rate SPARSE M=128 N=240 K=256 (4 sparse K=64 MMAs) + dense K=32: %.3f ms, %7.1f cycles/tile, %.3e pairs/s\n", ms,
               ms * 1e-3 * prop.clockRate * 1e3 / iters, double(iters) * 128 * 240 * sms / (ms * 1e-3));
    }
    printf("TS-mode hypothesis: %s\n", ts_fails ? "WRONG" : "confirmed");
    printf(fails ? "UMMA PROBE: %d FAILURES\n" : "UMMA PROBE: all checks ok\n", fails);
    return fails ? 1 : 0;
}
