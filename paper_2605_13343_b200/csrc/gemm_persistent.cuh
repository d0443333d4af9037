// Persistent tcgen05 GEMM for the toy-network inference (sm_100a):
//   C[M x N] = epi( [A_0 | A_1 | A_2](M x K) * W(K x N) )
//
//  * A: up to three fp32 row-major activation sources laid side by side along K ("K-sliced":
//    the FFN input [LN(t) | row_hw | col_hw] is read from its three buffers, never concatenated
//    in memory). Source s covers K blocks [kb_end[s-1], kb_end[s]). K-major UMMA operand.
//  * B: W^T, fp32 row-major N x K (pre-transposed once at load), K-major.
//  * kind::tf32 MMA (tf32 products, fp32 accumulation in TMEM), tiles 128 x BN, K blocks of 32
//    fp32 (one 128-byte SWIZZLE_128B row), TMA (cp.async.bulk.tensor.2d) into a ring.
//  * Persistent: one CTA per SM walks tiles t = blockIdx.x + i * gridDim.x (the N tiles of a row
//    block consecutive, so A comes from L2 the second time). Two TMEM accumulators: the
//    epilogue of tile i overlaps the MMAs of tile i+1 (warp 9, one elected thread) while warp 8
//    streams the operands ahead.
//  * Epilogue, eight warps: warp e reads TMEM lanes 32 (e mod 4) .. +31 and every other 32-column
//    chunk; each 32 x 32 chunk is transposed through shared memory so the functor's stores are
//    coalesced rows (Epi::apply8(row0, col, v[8], ncols, M): lane = 4 columns of rows row0 + 4 i,
//    eight rows at once so read-modify-write functors keep all their loads in flight). Epi::kWholeRow (BN = N = 128):
//    residual add + LayerNorm of the new row; a warp pair splits each row's columns, the residual
//    rows arrive by cp.async while the MMAs run, the row statistics meet in shared memory.
#pragma once

#include "gemm_tcgen05.cuh"

namespace hfpg {

constexpr int kPgEpiWarps = 8;
constexpr int kPgThreads = (kPgEpiWarps + 2) * 32;  // + TMA producer + MMA issuer

template <int BN, bool WHOLE>
struct PgCfg {
    static constexpr int kABytes = kGemmBM * kGemmBK * 4, kBBytes = BN * kGemmBK * 4;
    static constexpr int kStgFloats = WHOLE ? kPgEpiWarps * 32 * 65 + 2 * 4 * 2 * 32 : kPgEpiWarps * 32 * 32;
    static constexpr int kBudget = 200 * 1024 - kStgFloats * 4;
    static constexpr int kStages0 = kBudget / (kABytes + kBBytes);
    static constexpr int kStages = kStages0 > 6 ? 6 : kStages0;
    static constexpr uint32_t kAccCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    static constexpr uint32_t kTmemCols = 2 * kAccCols <= 64 ? 64 : 2 * kAccCols <= 128 ? 128 : 2 * kAccCols <= 256 ? 256 : 512;
    static_assert(kStages >= 2, "shared memory");
};

struct PgA {
    CUtensorMap map[3];
    int kb_end[3];  // exclusive end K block of each source
    int nsrc;
};

template <int BN, bool WHOLE>
struct PgSmem {
    using Cfg = PgCfg<BN, WHOLE>;
    alignas(1024) float A[Cfg::kStages][kGemmBM * kGemmBK];
    alignas(1024) float B[Cfg::kStages][BN * kGemmBK];
    float stg[Cfg::kStgFloats];
    uint64_t full[Cfg::kStages], empty[Cfg::kStages], tfull[2], tempty[2];
    uint32_t tmem_base;
};
template <int BN, bool WHOLE>
constexpr size_t pgemm_smem_bytes() {
    return sizeof(PgSmem<BN, WHOLE>) + 1024;
}

// 32 lanes x 32 bit x 16 columns, no wait (the caller waits once for a batch of loads)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int BN, class Epi>
__global__ void __launch_bounds__(kPgThreads, 1)
    k_pgemm_tf32(const __grid_constant__ PgA pa, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                 Epi epi) {
    constexpr bool WHOLE = Epi::kWholeRow;
    using Cfg = PgCfg<BN, WHOLE>;
    constexpr int S = Cfg::kStages;
    constexpr int kEpiActive = kPgEpiWarps;  // warps arriving on tempty
    extern __shared__ __align__(1024) unsigned char praw[];
    // 1024-byte alignment by an offset into the shared array (a uintptr_t round trip would turn
    // every shared-memory access into a generic one)
    PgSmem<BN, WHOLE>& sm = *reinterpret_cast<PgSmem<BN, WHOLE>*>(praw + ((1024u - (smem_u32(praw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (K + kGemmBK - 1) / kGemmBK;
    const int mt = (M + kGemmBM - 1) / kGemmBM, ntl = (N + BN - 1) / BN, tiles = mt * ntl;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.tfull[b], 1);
            mbar_init(&sm.tempty[b], kEpiActive);
        }
        fence_mbar_init();
    }
    if (warp == kPgEpiWarps + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                     "n"(Cfg::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == kPgEpiWarps) {
        if (lane == 0) {  // TMA producer
            for (int s = 0; s < pa.nsrc; ++s) asm volatile("prefetch.tensormap [%0];" ::"l"(&pa.map[s]) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            uint32_t it = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = (t / ntl) * kGemmBM, n0 = (t % ntl) * BN;
                int src = 0, kb0 = 0;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    while (src + 1 < pa.nsrc && kb >= pa.kb_end[src]) kb0 = pa.kb_end[src++];
                    const int s = it % S;
                    mbar_wait(&sm.empty[s], ((it / S) & 1) ^ 1);
                    mbar_expect_tx(&sm.full[s], Cfg::kABytes + Cfg::kBBytes);
                    tma_load_2d(sm.A[s], &pa.map[src], (kb - kb0) * kGemmBK, m0, &sm.full[s]);
                    tma_load_2d(sm.B[s], &tmB, kb * kGemmBK, n0, &sm.full[s]);
                }
            }
        }
    } else if (warp == kPgEpiWarps + 1) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = idesc_tf32<BN>();
            uint32_t it = 0, tl = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
                const uint32_t b = tl & 1, use = tl >> 1;
                mbar_wait(&sm.tempty[b], (use & 1) ^ 1);  // epilogue drained this accumulator
                tc_fence_after();
                const uint32_t tacc = tmem + b * Cfg::kAccCols;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % S;
                    mbar_wait(&sm.full[s], (it / S) & 1);
                    tc_fence_after();
                    const uint64_t da = umma_desc_sw128(sm.A[s]), db = umma_desc_sw128(sm.B[s]);
#pragma unroll
                    for (int k = 0; k < kGemmBK / 8; ++k) mma_tf32(tacc, da + 2 * k, db + 2 * k, idesc, (kb | k) ? 1u : 0u);
                    mma_commit(&sm.empty[s]);
                }
                mma_commit(&sm.tfull[b]);
            }
        }
    } else {
        // epilogue: warp e owns TMEM lanes (rows) 32 (e mod 4) .. +31; chunked: column chunks
        // e / 4 + 2 i; whole-row: columns [64 (e / 4), +64)
        const int quad = warp & 3, half = warp >> 2;
        float* stg = sm.stg + (WHOLE ? warp * 32 * 65 : warp * 32 * 32);
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
            const uint32_t b = tl & 1, use = tl >> 1;
            const int m0 = (t / ntl) * kGemmBM, n0 = (t % ntl) * BN;
            const int rbase = m0 + quad * 32;  // first row of this warp's 32
            const uint32_t tacc = tmem + b * Cfg::kAccCols + (uint32_t(quad * 32) << 16);
            if constexpr (WHOLE) {
                static_assert(BN == 128, "whole-row epilogues need the full 128-column row in one tile");
                // the warp pair (quad, half 0 / 1) splits each row's 128 columns; row statistics
                // are combined through `red` with a 64-thread named barrier per quad
                float* red = sm.stg + kPgEpiWarps * 32 * 65 + quad * 2 * 2 * 32;  // [stat][half][row]
                const int c0 = 64 * half;
                // residual rows of this tile -> staging, asynchronously (cp.async 4 B, coalesced),
                // while the accumulator is still being computed
                for (int rr = 0; rr < 32; ++rr) {
                    const int row = rbase + rr;
                    if (row < M) {
#pragma unroll
                        for (int q = 0; q < 2; ++q)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(stg + rr * 65 + 32 * q + lane)),
                                         "l"(epi.x + uint64_t(row) * 128 + c0 + 32 * q + lane)
                                         : "memory");
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                mbar_wait(&sm.tfull[b], use & 1);
                tc_fence_after();
                float v[64];  // thread = row rbase + lane, columns c0 .. c0 + 63
#pragma unroll
                for (int c = 0; c < 64; c += 32) {
                    uint32_t u0[16], u1[16];
                    tmem_ld16_nowait(tacc + uint32_t(c0 + c), u0);
                    tmem_ld16_nowait(tacc + uint32_t(c0 + c + 16), u1);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        v[c + j] = __uint_as_float(u0[j]);
                        v[c + 16 + j] = __uint_as_float(u1[j]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.tempty[b]);
                if (epi.gelu) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) v[j] = epi.act(v[j]);
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                float s = 0.f;
#pragma unroll
                for (int j = 0; j < 64; j += 4) {
                    v[j] += stg[lane * 65 + j];
                    v[j + 1] += stg[lane * 65 + j + 1];
                    v[j + 2] += stg[lane * 65 + j + 2];
                    v[j + 3] += stg[lane * 65 + j + 3];
                    s += (v[j] + v[j + 1]) + (v[j + 2] + v[j + 3]);
                }
                red[half * 32 + lane] = s;
                named_bar_sync(1 + quad, 64);
                const float mean = (red[lane] + red[32 + lane]) * (1.f / 128.f);
                float qs = 0.f;
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    const float cdev = v[j] - mean;
                    qs = fmaf(cdev, cdev, qs);
                    stg[lane * 65 + j] = v[j];
                }
                red[64 + half * 32 + lane] = qs;
                named_bar_sync(1 + quad, 64);
                const float inv = 1.f / sqrtf((red[64 + lane] + red[96 + lane]) * (1.f / 128.f) + 1e-5f);
                __syncwarp();
                // new rows and their LayerNorm out, coalesced
#pragma unroll 4
                for (int rr = 0; rr < 32; ++rr) {
                    const int row = rbase + rr;
                    const float mr = __shfl_sync(0xffffffffu, mean, rr), ir = __shfl_sync(0xffffffffu, inv, rr);
                    if (row < M) {
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const float xv = stg[rr * 65 + 32 * q + lane];
                            epi.x[uint64_t(row) * 128 + c0 + 32 * q + lane] = xv;
                            epi.ln[uint64_t(row) * 128 + c0 + 32 * q + lane] = (xv - mr) * ir;
                        }
                    }
                }
                named_bar_sync(1 + quad, 64);  // red[] reads done before the next tile writes it
            } else {
                mbar_wait(&sm.tfull[b], use & 1);
                tc_fence_after();
                constexpr int nch = (BN + 31) / 32;
#pragma unroll 1
                for (int ch = half; ch < nch; ch += 2) {
                    const int c = ch * 32;
                    uint32_t u0[16], u1[16];
                    tmem_ld16_nowait(tacc + uint32_t(c), u0);
                    if (c + 16 < BN) tmem_ld16_nowait(tacc + uint32_t(c + 16), u1);
                    tmem_wait_ld();
                    if (ch + 2 >= nch) {  // this warp's last loads of the accumulator are complete
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&sm.tempty[b]);
                    }
                    // 32 x 32 chunk through shared memory, 16-byte granules XOR-swizzled by row
                    // (conflict-free float4 writes by rows and reads by columns): thread = row
                    // writes its 32 columns; lane l then holds columns 4 (l mod 8) .. +3 of rows
                    // l / 8 + 4 i, so each warp store covers four full 128-byte row segments
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        *reinterpret_cast<float4*>(stg + lane * 32 + ((q ^ (lane & 7)) << 2)) =
                            make_float4(__uint_as_float(u0[4 * q]), __uint_as_float(u0[4 * q + 1]),
                                        __uint_as_float(u0[4 * q + 2]), __uint_as_float(u0[4 * q + 3]));
                        *reinterpret_cast<float4*>(stg + lane * 32 + (((q + 4) ^ (lane & 7)) << 2)) =
                            c + 16 < BN ? make_float4(__uint_as_float(u1[4 * q]), __uint_as_float(u1[4 * q + 1]),
                                                      __uint_as_float(u1[4 * q + 2]), __uint_as_float(u1[4 * q + 3]))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    __syncwarp();
                    const int cq = lane & 7, r0 = lane >> 3;
                    float4 cv[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int rr = r0 + 4 * i;
                        cv[i] = *reinterpret_cast<const float4*>(stg + rr * 32 + ((cq ^ (rr & 7)) << 2));
                    }
                    __syncwarp();
                    const int col = n0 + c + 4 * cq;
                    const int ncv = min(min(N - col, BN - (c + 4 * cq)), 4);  // valid columns of the float4
                    if (ncv > 0) epi.apply8(rbase + r0, col, cv, ncv, M);
                }
                if (half >= nch) {  // no chunk of this parity (BN <= 32): still release the buffer
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.tempty[b]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kPgEpiWarps + 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::kTmemCols));
    }
}

}  // namespace hfpg
