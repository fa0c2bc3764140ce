// umma2_probe.cu -- stand-alone check + rate of the CTA-PAIR form (cta_group::2) of the 2:4-sparse kind::i8 MMA the
// tensor-core scan uses (NOT part of libqadc_b200.so; companion of umma_probe.cu).  A cluster of two CTAs computes
//     D[256 x N] = A[256 x 64 (2:4 sparse)] * B[N x 64]^T  (+ a dense K = 32 step)
// with M = 256 split by rows (CTA r holds A rows 128 r .. 128 r + 127, their metadata and their accumulator rows) and B
// split by rows too (CTA r holds B rows N/2 r .. N/2 r + N/2 - 1 at the SAME shared-memory offset): each SM then reads
// half of B per instruction, which is what the single-CTA form is bound by (69 KB of B per 128 x 240 tile).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma2_probe tools/umma2_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
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
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
           (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(uint32_t cfmt, uint32_t afmt, uint32_t bfmt, uint32_t M, uint32_t N) {
    return (cfmt << 4) | (afmt << 7) | (bfmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma2_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_i8_sp(uint32_t d, uint64_t a, uint64_t b, uint32_t e_tmem, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\ntcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(e_tmem), "r"(id), "r"(acc) : "memory");
}
// arrives on the barrier at this shared-memory offset in BOTH CTAs of the pair once every MMA issued so far is complete
__device__ __forceinline__ void mma2_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"(uint16_t(3)) : "memory");
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
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// ---- check: one sparse K = 64 step + one dense K = 32 step, M = 256, N columns
// Ac [256][32] compressed A, meta [256][2], B [N][64] (s8), A2 [256][32] dense (u8), B2 [N][32] (s8)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    mma2_check_kernel(const uint8_t* Ac, const uint32_t* meta, const uint8_t* B, const uint8_t* A2, const uint8_t* B2, uint32_t N,
                      uint32_t id_sp, uint32_t id_d, uint32_t* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, rank = cta_rank(), NH = N / 2;
    uint8_t* sa = sm;                 // 128 x 32 B  (this CTA's rows)
    uint8_t* sb = sa + 128 * 32;      // NH x 64 B   (this CTA's half of B)
    uint8_t* sa2 = sb + NH * 64;      // 128 x 32 B
    uint8_t* sb2 = sa2 + 128 * 32;    // NH x 32 B
    for (uint32_t i = tid; i < 128 * 32; i += 128) {
        const uint32_t row = i / 32, kb = i % 32;
        const uint32_t o = (kb / 16) * (128 * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16;
        sa[o] = Ac[(rank * 128 + row) * 32 + kb];
        sa2[o] = A2[(rank * 128 + row) * 32 + kb];
    }
    for (uint32_t i = tid; i < NH * 64; i += 128) {
        const uint32_t row = i / 64, kb = i % 64;
        sb[(kb / 16) * (NH * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = B[(rank * NH + row) * 64 + kb];
    }
    for (uint32_t i = tid; i < NH * 32; i += 128) {
        const uint32_t row = i / 32, kb = i % 32;
        sb2[(kb / 16) * (NH * 16) + (row / 8) * 128 + (row % 8) * 16 + kb % 16] = B2[(rank * NH + row) * 32 + kb];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base, e_col = 480;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(tb + ((warp * 32u) << 16) + e_col),
                 "r"(meta[(rank * 128 + tid) * 2]), "r"(meta[(rank * 128 + tid) * 2 + 1]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 0 && tid == 0) {
        mma2_i8_sp(tb, smem_desc(smem_u32(sa), 128 * 16, 128), smem_desc(smem_u32(sb), NH * 16, 128), tb + e_col, id_sp, 0);
        mma2_i8(tb, smem_desc(smem_u32(sa2), 128 * 16, 128), smem_desc(smem_u32(sb2), NH * 16, 128), id_d, 1);
        mma2_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (uint32_t c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tb + ((warp * 32u) << 16) + c0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j)
            if (c0 + j < N) D[size_t(rank * 128 + tid) * N + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}

// ---- rate: per tile NSP sparse K = 64 MMAs + one dense K = 32 MMA into alternating accumulators, nobody reads them
template <int N, int NSP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64) mma2_rate_kernel(uint32_t iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[2];
    __shared__ uint32_t tmem_base;
    constexpr int NH = N / 2;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, rank = cta_rank();
    for (uint32_t i = tid; i < (128 * 32 + NH * 64) * NSP / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 1);
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base;
    for (int c = 0; c < 32; c += 2) // (rows 64..127 keep whatever metadata the tensor memory holds: this is a rate test)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(tb + ((warp * 32u) << 16) + 480 + c),
                     "r"(0x44444444u), "r"(0x44444444u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 0 && tid == 32) {
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 32 * NSP);
        const uint32_t id_sp = idesc(2, 0, 1, 256, N) | (1u << 2), id_d = idesc(2, 0, 1, 256, N);
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t buf = it & 1;
            for (uint32_t ks = 0; ks < NSP; ++ks)
                mma2_i8_sp(tb + buf * N, smem_desc(a0 + ks * 2 * 2048, 2048, 128), smem_desc(b0 + ks * 4 * (NH * 16), NH * 16, 128),
                           tb + 480 + (ks & 7) * 2, id_sp, ks > 0);
            mma2_i8(tb + buf * N, smem_desc(a0, 2048, 128), smem_desc(b0, NH * 16, 128), id_d, 1);
            mma2_commit(&full[buf]);
        }
    }
    if (tid == 32) mbar_wait(&full[(iters - 1) & 1], ((iters - 1) >> 1) & 1); // both CTAs get the multicast arrive
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512));
}

int main() {
    int sms = 0;
    cudaDeviceProp prop;
    CK(cudaSetDevice(0));
    CK(cudaGetDeviceProperties(&prop, 0));
    sms = prop.multiProcessorCount;
    printf("device: %s, %d SMs, %d MHz\n", prop.name, sms, prop.clockRate / 1000);
    int fails = 0;
    srand(7);
    for (uint32_t N : {64u, 240u}) {
        const uint32_t M = 256;
        std::vector<uint8_t> A(M * 64, 0), Ac(M * 32), B(N * 64), A2(M * 32), B2(N * 32);
        std::vector<uint32_t> meta(M * 2, 0);
        for (auto& x : B) x = rand() & 255;
        for (auto& x : A2) x = rand() & 255;
        for (auto& x : B2) x = rand() & 255;
        for (uint32_t r = 0; r < M; ++r)
            for (uint32_t g = 0; g < 16; ++g) {
                uint32_t i0 = rand() % 3, i1 = i0 + 1 + rand() % (3 - i0);
                const uint8_t v0 = rand() & 255, v1 = rand() & 255;
                A[r * 64 + 4 * g + i0] = v0;
                A[r * 64 + 4 * g + i1] = v1;
                Ac[r * 32 + 2 * g] = v0;
                Ac[r * 32 + 2 * g + 1] = v1;
                meta[r * 2 + g / 8] |= (i0 | (i1 << 2)) << (4 * (g % 8));
            }
        uint8_t *dA, *dB, *dA2, *dB2;
        uint32_t *dD, *dM;
        CK(cudaMalloc(&dA, Ac.size()));
        CK(cudaMalloc(&dB, B.size()));
        CK(cudaMalloc(&dA2, A2.size()));
        CK(cudaMalloc(&dB2, B2.size()));
        CK(cudaMalloc(&dM, meta.size() * 4));
        CK(cudaMalloc(&dD, M * N * 4));
        CK(cudaMemcpy(dA, Ac.data(), Ac.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dA2, A2.data(), A2.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB2, B2.data(), B2.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dM, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(dD, 0xEE, M * N * 4));
        const size_t smem = 2 * 128 * 32 + (N / 2) * 96;
        CK(cudaFuncSetAttribute(mma2_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        mma2_check_kernel<<<2, 128, smem>>>(dA, dM, dB, dA2, dB2, N, idesc(2, 0, 1, M, N) | (1u << 2), idesc(2, 0, 1, M, N), dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("2-CTA sparse N=%3u: CUDA error %s\n", N, cudaGetErrorString(e));
            return 3;
        }
        std::vector<int32_t> D(M * N);
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        long bad = 0, bad_lo = 0;
        for (uint32_t r = 0; r < M; ++r)
            for (uint32_t c = 0; c < N; ++c) {
                int32_t s2 = 0;
                for (uint32_t k = 0; k < 64; ++k) s2 += int32_t(A[r * 64 + k]) * int32_t(int8_t(B[c * 64 + k]));
                for (uint32_t k = 0; k < 32; ++k) s2 += int32_t(A2[r * 32 + k]) * int32_t(int8_t(B2[c * 32 + k]));
                bad += s2 != D[r * N + c];
                bad_lo += (s2 != D[r * N + c]) && r < 128;
            }
        printf("2-CTA (M=256) sparse K=64 + dense K=32, N=%3u: %s (%ld mismatches, %ld in rows < 128; D[0][0]=%d D[200][7]=%d)\n", N,
               bad ? "FAIL" : "ok", bad, bad_lo, D[0], D[200 * N + 7]);
        fails += bad != 0;
        cudaFree(dA); cudaFree(dB); cudaFree(dA2); cudaFree(dB2); cudaFree(dD); cudaFree(dM);
    }
    {
        const uint32_t iters = 4000;
        const size_t smem = (128 * 32 + 120 * 64) * 4;
        auto k = mma2_rate_kernel<240, 4>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        const int grid = sms / 2 * 2;
        k<<<grid, 64, smem>>>(100);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        k<<<grid, 64, smem>>>(iters);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("rate 2-CTA SPARSE M=256 N=240 K=256 (4 sparse K=64 MMAs) + dense K=32: %.3f ms, %7.1f cycles per 256 x 240 tile, %.3e pairs/s\n", ms,
               ms * 1e-3 * prop.clockRate * 1e3 / iters, double(iters) * 256 * 240 * (grid / 2) / (ms * 1e-3));
    }
    printf(fails ? "UMMA2 PROBE: %d FAILURES\n" : "UMMA2 PROBE: all checks ok\n", fails);
    return fails ? 1 : 0;
}
