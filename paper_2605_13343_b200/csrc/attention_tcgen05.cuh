// Windowed attention on the 5th-generation tensor cores (sm_100a): toy_net.cpp:78-125 for the
// leaf windows (T = 128 tokens) and the strip-pooled tile windows (T = 32 tokens, four windows
// packed into one 128-row MMA), head dim 16, 8 heads. One CTA per group of 128 token rows:
//
//   S = Q K^T            tcgen05.mma kind::tf32, M = 128 rows, N = 128 keys, K = 16 (2 x K=8).
//                        For T = 32 the four 32 x 32 diagonal blocks are the four windows' logits
//                        (the off-diagonal blocks are computed and ignored).
//   P = softmax(S/4 + B) thread = TMEM lane = query row, 32 keys per thread: T = 128 splits the
//                        row's keys over four warp quads (max / sum combined through shared
//                        memory), T = 32 gives each row's window to one thread. The logits stay
//                        in registers between the max and the exponentials. The fp16 edge bias
//                        (query-major as the reference indexes it, pre-scaled by log2 e) is
//                        prefetched one head ahead. P goes to shared memory in the UMMA
//                        SWIZZLE_128B K-major layout; for T = 32 only the row's own window block
//                        is written — the off-diagonal blocks stay zero (block-diagonal mask).
//   O_h = P V_h          tcgen05.mma kind::tf32, M = 128, N = 16, K = 128, into TMEM columns
//                        128 + 16 h; it runs while head h+1 is staged and its logits computed.
//   out = O_h / rowsum   all eight heads at the end, contiguous 16-float runs per thread.
//
// Operands are staged by the threads from the fp32 qkv rows (Q, K zero-padded to 32 columns —
// one 128-byte swizzle row, only the first two K=8 steps are issued), V transposed into a 16-row
// B operand. Pipelined over the heads: Q, K and S are double-buffered (smem, TMEM columns
// 0 / 128), so head h+1's S MMA is issued with head h's PV MMA and is ready when its softmax
// starts; operands are fetched two heads ahead. One block barrier + one named barrier per head.
// TMEM: 512 columns (S 2 x 128 + O 8 x 16), one CTA per SM; T = 128: 512 threads, T = 32: 128.
#pragma once

#include <cuda_fp16.h>
#include <math_constants.h>

#include "gemm_tcgen05.cuh"

namespace hfpg {

constexpr int kAttRows = 128, kAttHD = 16, kAttHeads = 8;
constexpr float kAttLog2e = 1.4426950408889634f;

struct AttSmem {
    alignas(1024) float Q[2][kAttRows * 32]; // 128 x 32 SW128 (cols 16..31 zero), by head parity
    alignas(1024) float K[2][kAttRows * 32];
    alignas(1024) float P[4][kAttRows * 32]; // 4 K-blocks of 128 x 32 SW128
    alignas(1024) float VT[4][16 * 32];      // V^T: 4 K-blocks of 16 x 32
    float part[4][kAttRows];                 // T = 128: per-quad row max (trace: row sums)
    float psum[4][kAttRows];                 // T = 128: per-quad row sum
    uint64_t bar_s, bar_o;
    uint32_t tmem;
};
constexpr size_t att_smem_bytes() { return sizeof(AttSmem) + 1024; }
template <int T>
__host__ __device__ constexpr int att_quads() {
    return T == 128 ? 4 : 1;
}
template <int T>
__host__ __device__ constexpr int att_threads() {
    return att_quads<T>() * 128;
}

// Byte offset of element (row, col < 32) in a SW128 K-major tile of 32-float rows.
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t col) {
    const uint32_t chunk = (col >> 2) ^ (row & 7);
    return (row >> 3) * 1024 + (row & 7) * 128 + chunk * 16 + (col & 3) * 4;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// qkv: rows of [q | k | v] (3 d = 384 wide); bias: fp16 [window][head][query][key] in log2
// units (b log2 e); head_out: rows x d. nwin windows of T tokens (rows = nwin * T).
template <int T>
__global__ void __launch_bounds__(att_threads<T>(), 1)
    k_tn_attn_tc(uint64_t nwin, const float* __restrict__ qkv, const __half* __restrict__ bias,
                 float* __restrict__ head_out, unsigned int* rowsum_err_bits) {
    static_assert(T == 128 || T == 32, "windows of 128 (leaf) or 32 (tile) tokens");
    constexpr int NQ = att_quads<T>();
    constexpr int d = kAttHeads * kAttHD;  // 128
    extern __shared__ __align__(1024) unsigned char araw[];
    // 1024-byte alignment by an offset into the shared array (a uintptr_t round trip would turn
    // every shared-memory access into a generic one)
    AttSmem& sm = *reinterpret_cast<AttSmem*>(araw + ((1024u - (smem_u32(araw) & 1023u)) & 1023u));
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t row = tid & (kAttRows - 1), quad = tid >> 7;
    const uint64_t grow = uint64_t(blockIdx.x) * kAttRows + row;  // global token row
    const uint64_t win = grow / T;                                  // window of this row
    const uint32_t wrow = uint32_t(grow % T);                        // query index inside it
    const bool valid = win < nwin;
    // this thread's 32 keys: window-local [key0, key0 + 32) = S columns [scol0, scol0 + 32) =
    // P K-block kb (T = 128: quad q owns keys 32q..; T = 32: the row's own window)
    const uint32_t key0 = T == 128 ? 32 * quad : 0;
    const uint32_t scol0 = T == 128 ? key0 : (row & ~31u);
    const uint32_t kb = scol0 >> 5;
    // stagers: T = 128 quad 0 -> Q, 1 -> K, 2 -> V^T; T = 32 the single quad stages all three
    const bool stage_q = quad == 0, stage_k = T == 128 ? quad == 1 : true, stage_v = T == 128 ? quad == 2 : true;

    if (tid == 0) {
        mbar_init(&sm.bar_s, 1);
        mbar_init(&sm.bar_o, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (quad == 0) {  // Q, K padding columns 16..31 and (T = 32) every P block: zero once
#pragma unroll
        for (int bq = 0; bq < 2; ++bq)
#pragma unroll
            for (int c = 16; c < 32; c += 4) {
                *reinterpret_cast<float4*>(reinterpret_cast<unsigned char*>(sm.Q[bq]) + sw128_off(row, c)) = make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(reinterpret_cast<unsigned char*>(sm.K[bq]) + sw128_off(row, c)) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        if (T == 32) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                    *reinterpret_cast<float4*>(reinterpret_cast<unsigned char*>(sm.P[b]) + sw128_off(row, c)) =
                        make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem, tO = tmem + 256;  // S(h) in columns 128 (h & 1) .. +127
    constexpr uint32_t idS = idesc_tf32<128>(), idO = idesc_tf32<16>();
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;

    const float* rowp = qkv + grow * 3 * d;
    // next head's operands of this thread (T = 128: one of q / k / v in n0; T = 32: all three)
    struct Ops {
        float4 q[4], k[4], v[4];  // T = 128 uses q only (this quad's one of q / k / v)
    };
    Ops cur, nxt;
    auto fetch = [&](uint32_t h, Ops& o) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if constexpr (T == 128) {
                if (quad < 3) o.q[c] = valid ? reinterpret_cast<const float4*>(rowp + quad * d + h * kAttHD)[c] : z;
            } else {
                o.q[c] = valid ? reinterpret_cast<const float4*>(rowp + h * kAttHD)[c] : z;
                o.k[c] = valid ? reinterpret_cast<const float4*>(rowp + d + h * kAttHD)[c] : z;
                o.v[c] = valid ? reinterpret_cast<const float4*>(rowp + 2 * d + h * kAttHD)[c] : z;
            }
        }
    };
    auto stage_qk = [&](const Ops& o, int bq) {  // Q_h, K_h into buffer bq
        if (stage_q) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<float4*>(reinterpret_cast<unsigned char*>(sm.Q[bq]) + sw128_off(row, 4 * c)) = o.q[c];
        }
        if (stage_k) {
            const float4* kk = T == 128 ? o.q : o.k;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<float4*>(reinterpret_cast<unsigned char*>(sm.K[bq]) + sw128_off(row, 4 * c)) = kk[c];
        }
    };
    auto issue_s = [&](int bq) {  // S = Q K^T into TMEM columns 128 bq
        const uint64_t da = umma_desc_sw128(sm.Q[bq]), db = umma_desc_sw128(sm.K[bq]);
        mma_tf32(tmem + 128 * bq, da, db, idS, 0u);
        mma_tf32(tmem + 128 * bq, da + 2, db + 2, idS, 1u);
        mma_commit(&sm.bar_s);
    };
    uint4 bcur[4], bnext[4];  // 32 fp16 bias values of this thread's keys
    auto fetch_bias = [&](uint32_t h, uint4 (&dst)[4]) {
        const __half* b = bias + ((win * kAttHeads + h) * T + wrow) * T + key0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            dst[i] = valid ? __ldg(reinterpret_cast<const uint4*>(b) + i) : make_uint4(0u, 0u, 0u, 0u);
    };
    // prologue: head 0's S in flight, head 1's operands loading
    fetch(0, cur);
    fetch_bias(0, bcur);
    stage_qk(cur, 0);
    fetch(1, nxt);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) issue_s(0);
    float inv[kAttHeads];
    float rs_err = 0.f;

#pragma unroll 1
    for (uint32_t h = 0; h < kAttHeads; ++h) {
        const uint32_t tS = tmem + 128 * (h & 1);
        if (h + 1 < kAttHeads) {
            fetch_bias(h + 1, bnext);
            // the next head's Q, K into the other buffer now (its last reader, head h-1's S MMA,
            // completed before head h-1's softmax), so S(h+1) can be issued ahead of PV(h)
            stage_qk(nxt, (h + 1) & 1);
        }
        mbar_wait(&sm.bar_s, h & 1);
        tc_fence_after();
        // ---- logits l = s log2(e) / 4 + b' (b' = b log2 e) of this thread's 32 keys, row max
        float lg[32];
        {
            uint32_t u0[16], u1[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(u0[0]), "=r"(u0[1]), "=r"(u0[2]), "=r"(u0[3]), "=r"(u0[4]), "=r"(u0[5]), "=r"(u0[6]),
                  "=r"(u0[7]), "=r"(u0[8]), "=r"(u0[9]), "=r"(u0[10]), "=r"(u0[11]), "=r"(u0[12]), "=r"(u0[13]),
                  "=r"(u0[14]), "=r"(u0[15])
                : "r"(tS + lane_off + scol0));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(u1[0]), "=r"(u1[1]), "=r"(u1[2]), "=r"(u1[3]), "=r"(u1[4]), "=r"(u1[5]), "=r"(u1[6]),
                  "=r"(u1[7]), "=r"(u1[8]), "=r"(u1[9]), "=r"(u1[10]), "=r"(u1[11]), "=r"(u1[12]), "=r"(u1[13]),
                  "=r"(u1[14]), "=r"(u1[15])
                : "r"(tS + lane_off + scol0 + 16));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                lg[j] = __uint_as_float(u0[j]);
                lg[16 + j] = __uint_as_float(u1[j]);
            }
        }
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __half2* b2 = reinterpret_cast<const __half2*>(&bcur[i]);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float2 bf = __half22float2(b2[t]);
                const int j = 8 * i + 2 * t;
                lg[j] = fmaf(lg[j], 0.25f * kAttLog2e, bf.x);
                lg[j + 1] = fmaf(lg[j + 1], 0.25f * kAttLog2e, bf.y);
                mx = fmaxf(mx, fmaxf(lg[j], lg[j + 1]));
            }
        }
        if constexpr (NQ > 1) {
            sm.part[quad][row] = mx;
            named_bar_sync(1, NQ * 128);
            mx = fmaxf(fmaxf(sm.part[0][row], sm.part[1][row]), fmaxf(sm.part[2][row], sm.part[3][row]));
        }
        // ---- after head h-1's PV MMA: V_h^T into its buffer, P = 2^(l - max) into the operand
        if (h > 0) mbar_wait(&sm.bar_o, (h - 1) & 1);
        if (stage_v) {
            const float4* nv = T == 128 ? cur.q : cur.v;
            unsigned char* vb = reinterpret_cast<unsigned char*>(sm.VT[row >> 5]);
            const uint32_t key = row & 31;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 0, key)) = nv[c].x;
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 1, key)) = nv[c].y;
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 2, key)) = nv[c].z;
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 3, key)) = nv[c].w;
            }
        }
        float sum = 0.f;
        unsigned char* pb = reinterpret_cast<unsigned char*>(sm.P[kb]);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
            float pp[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                pp[t] = ex2_approx(lg[4 * q4 + t] - mx);
                sum += pp[t];
            }
            *reinterpret_cast<float4*>(pb + sw128_off(row, 4 * q4)) = make_float4(pp[0], pp[1], pp[2], pp[3]);
        }
        if constexpr (NQ > 1) sm.psum[quad][row] = sum;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();  // P, V^T, the partial sums and the next Q, K complete
        tc_fence_after();
        if (tid == 0) {  // S for head h+1 first (the next softmax waits on it), then O_h = P V_h
            if (h + 1 < kAttHeads) issue_s((h + 1) & 1);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint64_t da = umma_desc_sw128(sm.P[b]), db = umma_desc_sw128(sm.VT[b]);
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_tf32(tO + h * kAttHD, da + 2 * k, db + 2 * k, idO, (b | k) ? 1u : 0u);
            }
            mma_commit(&sm.bar_o);
        }
        if (h + 1 < kAttHeads) {
            cur = nxt;
            if (h + 2 < kAttHeads) fetch(h + 2, nxt);  // two heads ahead, in flight over a whole head
        }
        float tot = sum;
        if constexpr (NQ > 1) tot = (sm.psum[0][row] + sm.psum[1][row]) + (sm.psum[2][row] + sm.psum[3][row]);
        inv[h] = 1.f / tot;
        if (rowsum_err_bits) {  // trace (toy_net.cpp:108-113): row sum of the normalised probabilities
            float rs = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) rs += ex2_approx(lg[j] - mx) * inv[h];
            if constexpr (NQ > 1) {
                sm.part[quad][row] = rs;  // the maxima were read before the block barrier
                named_bar_sync(1, NQ * 128);
                rs = (sm.part[0][row] + sm.part[1][row]) + (sm.part[2][row] + sm.part[3][row]);
                named_bar_sync(1, NQ * 128);
            }
            if (valid) rs_err = fmaxf(rs_err, fabsf(rs - 1.f));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) bcur[i] = bnext[i];
    }
    // ---- out = O_h / rowsum: T = 128 quad q writes heads 2q, 2q+1; T = 32 all eight
    mbar_wait(&sm.bar_o, (kAttHeads - 1) & 1);
    tc_fence_after();
    constexpr int HPQ = kAttHeads / NQ;
    float* dst = head_out + grow * d + quad * HPQ * kAttHD;
#pragma unroll
    for (int hh = 0; hh < HPQ; hh += 2) {
        const uint32_t hg = quad * HPQ + hh;
        uint32_t u0[16], u1[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(u0[0]), "=r"(u0[1]), "=r"(u0[2]), "=r"(u0[3]), "=r"(u0[4]), "=r"(u0[5]), "=r"(u0[6]),
              "=r"(u0[7]), "=r"(u0[8]), "=r"(u0[9]), "=r"(u0[10]), "=r"(u0[11]), "=r"(u0[12]), "=r"(u0[13]),
              "=r"(u0[14]), "=r"(u0[15])
            : "r"(tO + lane_off + hg * kAttHD));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(u1[0]), "=r"(u1[1]), "=r"(u1[2]), "=r"(u1[3]), "=r"(u1[4]), "=r"(u1[5]), "=r"(u1[6]),
              "=r"(u1[7]), "=r"(u1[8]), "=r"(u1[9]), "=r"(u1[10]), "=r"(u1[11]), "=r"(u1[12]), "=r"(u1[13]),
              "=r"(u1[14]), "=r"(u1[15])
            : "r"(tO + lane_off + (hg + 1) * kAttHD));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (valid) {
            const float i0 = inv[hg], i1 = inv[hg + 1];
            float4* o4 = reinterpret_cast<float4*>(dst + hh * kAttHD);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                o4[c] = make_float4(__uint_as_float(u0[4 * c]) * i0, __uint_as_float(u0[4 * c + 1]) * i0,
                                    __uint_as_float(u0[4 * c + 2]) * i0, __uint_as_float(u0[4 * c + 3]) * i0);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                o4[4 + c] = make_float4(__uint_as_float(u1[4 * c]) * i1, __uint_as_float(u1[4 * c + 1]) * i1,
                                        __uint_as_float(u1[4 * c + 2]) * i1, __uint_as_float(u1[4 * c + 3]) * i1);
        }
    }
    if (rowsum_err_bits && quad == 0 && valid) atomicMax(rowsum_err_bits, __float_as_uint(rs_err));
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

}  // namespace hfpg
