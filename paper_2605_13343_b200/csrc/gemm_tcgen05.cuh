// tcgen05 GEMM for the toy-network inference (sm_100a): C[M x N] = epi(A[M x K] * W[K x N]).
//
//  * A: activations, fp32 row-major (K contiguous) — K-major UMMA operand.
//  * B: W^T, fp32 row-major N x K (weights pre-transposed once at load) — K-major.
//  * kind::tf32 MMA (fp32 operands in smem, tf32 products, fp32 accumulation in TMEM).
//  * Tiles of 128 x BN, K blocks of 32 fp32 (one 128-byte SWIZZLE_128B row) loaded by TMA
//    (cp.async.bulk.tensor.2d, SASS UTMALDG) into a 4-stage ring; one elected thread of warp 4
//    produces, one elected thread of warp 5 issues tcgen05.mma (4 x K=8 per block) and commits to
//    the stage's "empty" mbarrier; warps 0-3 drain TMEM (tcgen05.ld 32x32b) through the
//    epilogue functor.
//  * OOB rows/columns of A and B (M, N, K tails) are zero-filled by TMA; the epilogue skips
//    rows >= M and columns >= N.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"

namespace hfpg {

constexpr int kGemmBM = 128, kGemmBK = 32, kGemmStages = 3;  // 3 stages: two CTAs per SM
constexpr int kGemmThreads = 192;  // warps 0-3 epilogue, warp 4 TMA, warp 5 MMA + TMEM

template <int BN>
struct GemmSmem {
    alignas(1024) float A[kGemmStages][kGemmBM * kGemmBK];
    alignas(1024) float B[kGemmStages][BN * kGemmBK];
    uint64_t full[kGemmStages], empty[kGemmStages], done;
    uint32_t tmem_base;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// K-major SWIZZLE_128B smem operand descriptor: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a & 0x3FFFFull) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = BN.
template <int BN>
__host__ __device__ constexpr uint32_t idesc_tf32() {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers (thread t: lane base + t)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Epilogue functor interface: void apply4(int row, int col, float4 v, int nvalid) const —
// columns col .. col + nvalid - 1 (nvalid <= 4, col a multiple of 4) of one output row. The
// accumulator tile is staged through shared memory first, so consecutive lanes get consecutive
// columns of the same row and the functors' global accesses coalesce.
template <int BN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 2)
    k_gemm_tf32(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                int M, int N, int K, Epi epi) {
    extern __shared__ __align__(1024) unsigned char graw[];
    GemmSmem<BN>& sm = *reinterpret_cast<GemmSmem<BN>*>(
        (reinterpret_cast<uintptr_t>(graw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kGemmBM, n0 = blockIdx.y * BN;
    const int nk = (K + kGemmBK - 1) / kGemmBK;
    constexpr uint32_t kCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kGemmStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.done, 1);
        fence_mbar_init();
    }
    if (warp == 5) {  // TMEM allocation (whole warp), address published through smem
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&sm.tmem_base)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 4) {
        if (lane == 0) {  // TMA producer
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kGemmStages;
                const uint32_t use = kb / kGemmStages;
                mbar_wait(&sm.empty[s], (use & 1) ^ 1);
                mbar_expect_tx(&sm.full[s], (kGemmBM + BN) * kGemmBK * 4);
                tma_load_2d(sm.A[s], &tmA, kb * kGemmBK, m0, &sm.full[s]);
                tma_load_2d(sm.B[s], &tmB, kb * kGemmBK, n0, &sm.full[s]);
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = idesc_tf32<BN>();
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kGemmStages;
                mbar_wait(&sm.full[s], (kb / kGemmStages) & 1);
                tc_fence_after();
                const uint64_t da = umma_desc_sw128(sm.A[s]), db = umma_desc_sw128(sm.B[s]);
#pragma unroll
                for (int k = 0; k < kGemmBK / 8; ++k)  // K = 8 tf32 = 32 B per MMA
                    mma_tf32(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) ? 1u : 0u);
                mma_commit(&sm.empty[s]);  // frees the stage once these MMAs retire
            }
            mma_commit(&sm.done);
        }
    } else {  // epilogue: warp w owns TMEM lanes (rows) 32w..32w+31
        mbar_wait(&sm.done, 0);
        tc_fence_after();
        // 1. TMEM -> shared memory, row-major (padded), into the idle stage buffers
        float* S = &sm.A[0][0];
        constexpr int kLd = BN + 4;
        static_assert(sizeof(float) * kGemmBM * (BN + 4) <= sizeof(sm.A) + sizeof(sm.B), "staging");
        const int r = warp * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
            float v[16];
            tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c), v);
            float4* d4 = reinterpret_cast<float4*>(S + r * kLd + c);
#pragma unroll
            for (int q = 0; q < 4; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the four epilogue warps
        // 2. whole rows, coalesced: lane l owns columns 4l .. 4l+3 (+128 per pass); rows in
        //    batches of 8 so a read-modify-write epilogue has 8 row reads in flight
#pragma unroll 1
        for (int c = 4 * lane; c < BN; c += 128) {
            const int col = n0 + c;
            if (col >= N) break;
            const int nv = N - col < 4 ? N - col : 4;
#pragma unroll 1
            for (int i0 = 0; i0 < 32; i0 += 8) {
                const int rr0 = warp * 32 + i0;
                if (m0 + rr0 >= M) break;
                if (m0 + rr0 + 8 <= M) {
                    epi.apply4x8(m0 + rr0, col, S + rr0 * kLd + c, kLd, nv);
                } else {
                    for (int i = 0; i < 8 && m0 + rr0 + i < M; ++i)
                        epi.apply4(m0 + rr0 + i, col, *reinterpret_cast<const float4*>(S + (rr0 + i) * kLd + c), nv);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
    }
}

template <int BN>
constexpr size_t gemm_smem_bytes() {
    return sizeof(GemmSmem<BN>) + 1024;
}

}  // namespace hfpg
