// Leaf-window attention on the 5th-generation tensor cores (sm_100a): toy_net.cpp:78-125 for
// windows of T = 128 tokens, head dim 16, per (block, head):
//
//   S = Q K^T            tcgen05.mma kind::tf32, M = 128 queries, N = 128 keys, K = 16 (2 x K=8)
//   P = softmax(S/4 + B) fp32 in registers: each of the 128 threads owns one TMEM lane = one
//                        query row (tcgen05.ld 32x32b), the key-major edge bias is read
//                        coalesced across the rows; P is written back to shared memory in the
//                        UMMA SWIZZLE_128B K-major layout
//   O = P V              tcgen05.mma kind::tf32, M = 128, N = 16, K = 128 (4 blocks x 4 x K=8)
//   out = O / rowsum
//
// Operands are staged by the 128 threads from the fp32 qkv rows: Q and K zero-padded to 32
// columns (one 128-byte swizzle row; only the first two K=8 steps are issued), V transposed into
// a 16-row B operand. One CTA per window loops over the heads; TMEM holds S (128 columns) and O
// (16 columns). The f32->tf32 operand rounding matches the inference GEMMs (kind::tf32).
#pragma once

#include <math_constants.h>

#include "gemm_tcgen05.cuh"

namespace hfpg {

constexpr int kAttT = 128, kAttHD = 16, kAttThreads = 256;

struct AttSmem {
    alignas(1024) float Q[kAttT * 32];       // 128 x 32 SW128 (cols 16..31 zero)
    alignas(1024) float K[kAttT * 32];
    alignas(1024) float P[4][kAttT * 32];    // 4 K-blocks of 128 x 32 SW128
    alignas(1024) float VT[4][16 * 32];      // V^T: 4 K-blocks of 16 x 32 SW128
    float part[2][kAttT];                    // per-half row max, then row sum
    uint64_t bar;
    uint32_t tmem;
};

// Byte offset of element (row, col < 32) in a SW128 K-major tile of 32-float rows.
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t col) {
    const uint32_t chunk = (col >> 2) ^ (row & 7);
    return (row >> 3) * 1024 + (row & 7) * 128 + chunk * 16 + (col & 3) * 4;
}

// Two warp quads per window: quad q (warps 4q..4q+3) owns keys [64q, 64q+64) of every query row
// (TMEM lane = row, warp w reads lanes 32 (w mod 4)..); row max and sum are combined through
// shared memory. Two CTAs per SM.
__global__ void __launch_bounds__(kAttThreads, 2)
    k_tn_attention_tc(uint32_t d, uint32_t heads, const float* qkv, const float* bias,
                      float* head_out, unsigned int* rowsum_err_bits) {
    extern __shared__ __align__(1024) unsigned char araw[];
    AttSmem& sm = *reinterpret_cast<AttSmem*>((reinterpret_cast<uintptr_t>(araw) + 1023) & ~uintptr_t(1023));
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t row = tid & (kAttT - 1), quad = tid >> 7, key0 = 64 * quad;
    const uint64_t blk = blockIdx.x;
    unsigned char* Qb = reinterpret_cast<unsigned char*>(sm.Q);
    unsigned char* Kb = reinterpret_cast<unsigned char*>(sm.K);
    constexpr float kLog2e = 1.4426950408889634f;
    if (tid == 0) {
        mbar_init(&sm.bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&sm.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (quad == 0) {  // zero the padding columns 16..31 of Q and K once (never rewritten)
#pragma unroll
        for (int c = 16; c < 32; c += 4) {
            *reinterpret_cast<float4*>(Qb + sw128_off(row, c)) = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(Kb + sw128_off(row, c)) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem, tS = tmem, tO = tmem + 128;
    constexpr uint32_t idS = idesc_tf32<128>(), idO = idesc_tf32<16>();
    uint32_t phase = 0;
    const float* rowp = qkv + (blk * kAttT + row) * 3 * d;
    float4 n0[4], n1[4];  // next head's operands of row `row`: quad 0 q, k; quad 1 v
    auto fetch = [&](uint32_t h) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (quad == 0) {
                n0[c] = reinterpret_cast<const float4*>(rowp + h * kAttHD)[c];
                n1[c] = reinterpret_cast<const float4*>(rowp + d + h * kAttHD)[c];
            } else {
                n0[c] = reinterpret_cast<const float4*>(rowp + 2 * d + h * kAttHD)[c];
            }
        }
    };
    fetch(0);
    const uint32_t trow = tS + (uint32_t((warp & 3) * 32) << 16);
    for (uint32_t h = 0; h < heads; ++h) {
        // ---- stage Q, K (quad 0, row `row`) and V^T (quad 1, key `row`)
        if (quad == 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                *reinterpret_cast<float4*>(Qb + sw128_off(row, 4 * c)) = n0[c];
                *reinterpret_cast<float4*>(Kb + sw128_off(row, 4 * c)) = n1[c];
            }
        } else {
            unsigned char* vb = reinterpret_cast<unsigned char*>(sm.VT[row >> 5]);
            const uint32_t key = row & 31;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 0, key)) = n0[c].x;
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 1, key)) = n0[c].y;
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 2, key)) = n0[c].z;
                *reinterpret_cast<float*>(vb + sw128_off(4 * c + 3, key)) = n0[c].w;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (tid == 0) {  // S = Q K^T
            const uint64_t da = umma_desc_sw128(sm.Q), db = umma_desc_sw128(sm.K);
            mma_tf32(tS, da, db, idS, 0u);
            mma_tf32(tS, da + 2, db + 2, idS, 1u);
            mma_commit(&sm.bar);
        }
        if (h + 1 < heads) fetch(h + 1);
        // the bias column of this query row (key-major: b[j * T]), keys of this quad; logits in
        // base-2 units: l = (s / 4 + b) log2(e)
        const float* b = bias + (blk * heads + h) * kAttT * kAttT + row + key0 * kAttT;
        float bn[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) bn[j] = __ldg(b + j * kAttT);
        mbar_wait(&sm.bar, phase);
        phase ^= 1;
        tc_fence_after();
        // pass 1: max over this quad's 64 keys (bias chunk c+1 in flight while c computes)
        float mx = -CUDART_INF_F;
#pragma unroll 1
        for (int c = 0; c < 64; c += 16) {
            float s[16], bc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) bc[j] = bn[j];
            if (c + 16 < 64) {
#pragma unroll
                for (int j = 0; j < 16; ++j) bn[j] = __ldg(b + (c + 16 + j) * kAttT);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) bn[j] = __ldg(b + j * kAttT);  // pass 2 restarts
            }
            tmem_ld16(trow + key0 + c, s);
#pragma unroll
            for (int j = 0; j < 16; ++j) mx = fmaxf(mx, fmaf(s[j], 0.25f, bc[j]));
        }
        sm.part[quad][row] = mx;
        __syncthreads();
        mx = fmaxf(sm.part[0][row], sm.part[1][row]);
        const float mx2 = mx * kLog2e;
        // pass 2: p = 2^(l - max), the quad's partial sum, P into the swizzled A operand
        float sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < 64; c += 16) {
            float s[16], bc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) bc[j] = bn[j];
            if (c + 16 < 64) {
#pragma unroll
                for (int j = 0; j < 16; ++j) bn[j] = __ldg(b + (c + 16 + j) * kAttT);
            }
            tmem_ld16(trow + key0 + c, s);
            const uint32_t kk = key0 + c;
            unsigned char* pb = reinterpret_cast<unsigned char*>(sm.P[kk >> 5]);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
                float p[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int j = 4 * j4 + t;
                    p[t] = exp2f(fmaf(fmaf(s[j], 0.25f, bc[j]), kLog2e, -mx2));
                    sum += p[t];
                }
                *reinterpret_cast<float4*>(pb + sw128_off(row, (kk & 31) + 4 * j4)) = make_float4(p[0], p[1], p[2], p[3]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();  // P complete; part[] max reads done
        tc_fence_after();
        if (tid == 0) {  // O = P V
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
                const uint64_t da = umma_desc_sw128(sm.P[kb]), db = umma_desc_sw128(sm.VT[kb]);
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_tf32(tO, da + 2 * k, db + 2 * k, idO, (kb | k) ? 1u : 0u);
            }
            mma_commit(&sm.bar);
        }
        sm.part[quad][row] = sum;
        float rs_trace = 0.f;
        if (rowsum_err_bits) {  // trace: row sum of the normalised probabilities (this quad)
            for (int c = 0; c < 64; c += 16) {
                float s2[16];
                tmem_ld16(trow + key0 + c, s2);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    rs_trace += exp2f(fmaf(fmaf(s2[j], 0.25f, __ldg(b + (c + j) * kAttT)), kLog2e, -mx2));
            }
        }
        mbar_wait(&sm.bar, phase);
        phase ^= 1;
        tc_fence_after();
        __syncthreads();  // partial sums visible
        const float tot = sm.part[0][row] + sm.part[1][row];
        const float inv = 1.f / tot;
        if (quad == 0) {
            float o[16];
            tmem_ld16(tO + (uint32_t((warp & 3) * 32) << 16), o);
            float4* dst = reinterpret_cast<float4*>(head_out + (blk * kAttT + row) * d + h * kAttHD);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                dst[c] = make_float4(o[4 * c] * inv, o[4 * c + 1] * inv, o[4 * c + 2] * inv, o[4 * c + 3] * inv);
        }
        if (rowsum_err_bits) {
            __syncthreads();  // both quads have read part[] for the row total
            sm.part[quad][row] = rs_trace * inv;
            __syncthreads();
            if (quad == 0) atomicMax(rowsum_err_bits, __float_as_uint(fabsf(sm.part[0][row] + sm.part[1][row] - 1.f)));
        }
        tc_fence_before();
        __syncthreads();  // TMEM S / O and smem reused by the next head
        tc_fence_after();
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

constexpr size_t att_smem_bytes() { return sizeof(AttSmem) + 1024; }

}  // namespace hfpg
