// Persistent whole-solve kernel (fast path, L = 128, L_s = 32): pcg_solve (pcg.cpp:53-126)
// with the factor preconditioner (apply.cpp:79-174) as ONE cooperative launch, one CTA of 512
// threads per SM, phases separated by grid barriers instead of kernel boundaries:
//
//   init   x = 0, p_prev = 0 | leaf(r = b) | r0 | coarse | prolong | rz
//   loop   spmv: p = z + beta p, Ap, p.Ap, p.p                          | breakdown, alpha
//          leaf: x += alpha p, r -= alpha Ap, |r|^2, F^T r, F c, Ũ^T r, Ṽ^T r | rel, stop?
//          coarse: strip sums + tile couplings over the whole bisection tree
//          prolong: ancestor gather, Ũ g_r + Ṽ g_c, gate, z, r.z         | beta
//
// Four barriers per iteration (~1.25 us each, measured); each carries its reduction: every CTA
// publishes a partial, and after the barrier every CTA sums all partials in the same fixed
// order, so all CTAs take identical branches and the result is run-to-run deterministic.
//
// Shared memory is two 96 KB leaf stages (F_k + Ũ_k|Ṽ_k, bulk-copied by TMA). The leaf phase
// double-buffers them; when it ends, the next iteration's first leaf is already in flight to one
// stage and the other is the scratch of the coarse, prolongation and SpMV phases (the SpMV
// streams its SELL-32 slices through a 2-stage TMA ring there).
//
// Measured constraints that shape the code (tools/microbench.cu on B200): f32->f64 conversion
// runs at 15.6/clk/SM and f64 shuffles at 0.5 warp-op/clk/SM, so the leaf's F^T r chains use
// vector smem loads (2 columns per lane), the prolongation reduces with a transpose-reduce (7
// shuffles per 16 rows instead of 24) and leaves are dealt across SMs first.
//
// Arithmetic is the per-kernel path's (kernels.cuh): the same operation order for every fp32
// chain (bit-identical c, restrictions and tile coefficients to the reference's matvec_t) and
// exact f64 products with f64 accumulation where the reference accumulates in double.
//
// Data written inside the kernel by other CTAs is read with ld.global.cg (L2; SM L1s are not
// coherent); constant data (factors, CSR, diagonal) goes through the read-only path or TMA.
#pragma once

#include "kernels.cuh"

namespace hfpg {

constexpr int kPThreads = 512;
constexpr int kPWarps = kPThreads / 32;
constexpr int kPMaxGrid = 256;        // grid_reduce reads <= 8 partials per lane
constexpr uint32_t kPSpmvSlices = 16; // SELL-32 slices per SpMV chunk (one per warp)

struct PStage {              // one leaf in flight: 96 KB, reused as phase scratch when free
    float F[kL * kL];
    float B[2 * kL * kLs];
};
struct PSmem {
    PStage st[2];
    double vec[2][4][kL];    // r_k, Ap_k, p_k, x_k of the staged leaf (or b_k at init)
    float rin[kL];
    float c[kL];
    float rin2[2][kL];       // p_leaf_phase_pipe: double-buffered by leaf parity
    float c2[2][kL];
    double red[4][kPWarps];
    double bc[4];
    uint64_t full[2];        // factors of stage s landed
    uint64_t vfull[2];       // vectors of stage s landed
    uint64_t sfull[2];       // SpMV ring stages landed
    int last;
    int probe;
};
static_assert(sizeof(PSmem) <= 227 * 1024, "persistent solve smem");

struct PScratchProlong {
    double su[kPWarps][kL], sv[kPWarps][kL];
};
static_assert(sizeof(PScratchProlong) <= sizeof(PStage), "prolong scratch");

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Intra-phase probe (CTA 0, thread 0) into the last 64 trace slots, in the probed iteration.
#define PROBE_T(id, thr)                                                                       \
    do {                                                                                       \
        if (s.trace && sm.probe && blockIdx.x == 0 && threadIdx.x == (thr))                    \
            s.trace[s.trace_cap - 64 + (id)] = globaltimer();                                  \
    } while (0)
#define PROBE(id) PROBE_T(id, 0)

struct PBar {
    unsigned* count;  // monotonic arrival counter, zeroed before the launch
    unsigned epoch;
};

// Lane 0 of warp 0: arrive and wait. A barrier stuck for ~30 s traps instead of hanging.
__device__ __forceinline__ void bar_arrive_wait(const DevSys& s, PBar& bar) {
    const unsigned target = bar.epoch * gridDim.x;
    red_release_gpu(bar.count, 1u);
    const long long t0 = clock64();
    while (ld_acquire_gpu(bar.count) < target)
        if (clock64() - t0 > (1LL << 36)) __trap();
    if (s.trace && blockIdx.x == 0 && bar.epoch < s.trace_cap) s.trace[bar.epoch] = globaltimer();
}

__device__ __forceinline__ void grid_barrier(const DevSys& s, PBar& bar) {
    __syncthreads();
    ++bar.epoch;
    if (threadIdx.x == 0) bar_arrive_wait(s, bar);
    __syncthreads();
}

// Barrier + deterministic grid reduction of NV values. All threads call it. Each CTA's total
// goes to partials[blockIdx * NV + i]; after the barrier every CTA sums all partials (lane j
// takes partials j, j+32, ... in order, then a fixed butterfly) and returns the same totals.
template <int NV>
__device__ __forceinline__ void grid_reduce(const DevSys& s, PSmem& sm, PBar& bar,
                                            const double (&v)[NV], double* partials,
                                            double (&tot)[NV]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const double t = warp_sum(v[i]);
        if (lane == 0) sm.red[i][warp] = t;
    }
    __syncthreads();  // orders every thread's phase writes before warp 0's release below
    ++bar.epoch;
    if (warp == 0) {
        double cta[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) cta[i] = warp_sum(lane < kPWarps ? sm.red[i][lane] : 0.0);
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < NV; ++i) __stcg(&partials[blockIdx.x * NV + i], cta[i]);
            bar_arrive_wait(s, bar);
        }
        __syncwarp();
        const unsigned G = gridDim.x;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x[kPMaxGrid / 32];
#pragma unroll
            for (int q = 0; q < kPMaxGrid / 32; ++q) {
                const unsigned j = lane + 32u * q;
                x[q] = j < G ? __ldcg(&partials[j * NV + i]) : 0.0;
            }
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < kPMaxGrid / 32; ++q) t += x[q];
            t = warp_sum(t);
            if (lane == 0) sm.bc[i] = t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] = sm.bc[i];
}

struct PLeafSched {
    uint64_t first, count;  // this CTA's leaves: first, first + grid, ...
    uint32_t it;            // ring counter (continues across iterations)
};

// Factors of `leaf` -> stage st (one elected thread): F_k (64 KB) and Ũ_k|Ṽ_k (32 KB, contiguous).
__device__ __forceinline__ void p_issue_factors(const DevSys& s, PSmem& sm, uint64_t leaf, int st,
                                                uint64_t pol_f, uint64_t pol_b) {
    fence_proxy_async_smem();
    mbar_expect_tx(&sm.full[st], kFBytes + kBBytes);
    tma_load_1d(sm.st[st].F, s.F + leaf * (kL * kL), kFBytes, &sm.full[st], pol_f);
    tma_load_1d(sm.st[st].B, s.F + s.bridge_base + leaf * (2 * kL * kLs), kBBytes, &sm.full[st], pol_b);
}
// The leaf's PCG vector slices -> stage st (written earlier in this kernel by other CTAs: the
// caller has passed a grid barrier and a global proxy fence).
__device__ __forceinline__ void p_issue_vectors(const DevSys& s, PSmem& sm, uint64_t leaf, int st,
                                                int mode, const double* b, const double* pcur,
                                                uint64_t pol) {
    const uint64_t o = leaf * kL;
    if (mode == kInit) {
        mbar_expect_tx(&sm.vfull[st], kL * 8);
        tma_load_1d(sm.vec[st][0], b + o, kL * 8, &sm.vfull[st], pol);
    } else {
        mbar_expect_tx(&sm.vfull[st], 4 * kL * 8);
        tma_load_1d(sm.vec[st][0], s.r + o, kL * 8, &sm.vfull[st], pol);
        tma_load_1d(sm.vec[st][1], s.ap + o, kL * 8, &sm.vfull[st], pol);
        tma_load_1d(sm.vec[st][2], pcur + o, kL * 8, &sm.vfull[st], pol);
        tma_load_1d(sm.vec[st][3], s.x + o, kL * 8, &sm.vfull[st], pol);
    }
}


// Two sequential fp32 FMA chains (columns M[., j], M[., j+1]) over the 128 rows in order:
// acc_t = fma(M[i][j+t], r[i], acc_t), i = 0..127 — the exact operation order of matvec_t. The
// loads are software-pipelined one 4-row block ahead (ptxas otherwise places each shared load
// right before its FMA and the chain pays the 29-cycle LDS latency every step).
template <int LD>
__device__ __forceinline__ float2 chain2(const float* M, const float4* r4) {
    float a0 = 0.f, a1 = 0.f;
    float2 fa[4], fb[4];
    float4 ra, rb;
    auto load = [&](int i4, float2 (&f)[4], float4& r) {
#pragma unroll
        for (int t = 0; t < 4; ++t) f[t] = *reinterpret_cast<const float2*>(&M[(4 * i4 + t) * LD]);
        r = r4[i4];
    };
    auto step = [&](const float2 (&f)[4], const float4& r) {
        a0 = fmaf(f[0].x, r.x, a0);
        a1 = fmaf(f[0].y, r.x, a1);
        a0 = fmaf(f[1].x, r.y, a0);
        a1 = fmaf(f[1].y, r.y, a1);
        a0 = fmaf(f[2].x, r.z, a0);
        a1 = fmaf(f[2].y, r.z, a1);
        a0 = fmaf(f[3].x, r.w, a0);
        a1 = fmaf(f[3].y, r.w, a1);
    };
    load(0, fa, ra);
#pragma unroll
    for (int i4 = 0; i4 < kL / 4; i4 += 2) {
        load(i4 + 1, fb, rb);
        step(fa, ra);
        if (i4 + 2 < kL / 4) load(i4 + 2, fa, ra);
        step(fb, rb);
    }
    return make_float2(a0, a1);
}

// Leaf phase (apply stages 1-3 + the fused x/r update). On entry the first leaf's factors are
// in flight to stage it & 1; on exit the NEXT iteration's first leaf is in flight to the new
// stage it & 1 and stage (it & 1) ^ 1 is free. Returns this thread's |r|^2 part.
//
// Per leaf: warps 0-3 update x, r and cast r to fp32; barrier; warps 0-1 run the 128 F^T r
// chains (2 columns per lane, float2 smem loads), warp 2 the 64 restriction chains, warp 15
// issues the next leaf's bulk copies; barrier; all warps y = F c.
__device__ __forceinline__ double p_leaf_phase(const DevSys& s, PSmem& sm, PLeafSched& ls, int mode,
                                               const double* b, const double* pcur, double alpha,
                                               uint64_t pol_f, uint64_t pol_b, uint64_t pol_v) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t G = gridDim.x;
    double rr = 0.0;
    if (ls.count == 0) return rr;
    if (tid == 0) {
        fence_proxy_async_global();
        p_issue_vectors(s, sm, ls.first, int(ls.it & 1), mode, b, pcur, pol_v);
    }
    for (uint64_t j = 0; j < ls.count; ++j, ++ls.it) {
        const uint64_t leaf = ls.first + j * G;
        const int st = int(ls.it & 1);
        const uint32_t par = (ls.it >> 1) & 1;
        if (j < 4) PROBE(j * 4 + 0);
        if (tid < kL) {
            mbar_wait(&sm.vfull[st], par);
            const uint64_t i = leaf * kL + tid;
            double rv = sm.vec[st][0][tid];
            if (mode == kLoop) {  // pcg.cpp:97-98, fused
                s.x[i] = fma(alpha, sm.vec[st][2][tid], sm.vec[st][3][tid]);
                rv = fma(-alpha, sm.vec[st][1][tid], rv);
            }
            s.r[i] = rv;
            rr = fma(rv, rv, rr);
            sm.rin[tid] = static_cast<float>(rv);  // apply.cpp:90
        }
        mbar_wait(&sm.full[st], par);
        __syncthreads();  // rin + stage st ready; every warp is past the previous leaf's F c
        if (j < 4) PROBE(j * 4 + 1);
        const float* F = sm.st[st].F;
        const float* B = sm.st[st].B;
        const float4* r4 = reinterpret_cast<const float4*>(sm.rin);
        if (warp < 2) {
            // c = F^T r: lane owns columns j0, j0 + 1; two sequential fp32 FMA chains over the
            // 128 rows in order — the reference's matvec_t (apply.cpp:25-35), bit for bit
            const int j0 = 64 * warp + 2 * lane;
            long long ck0 = 0;
            if (j == 1 && s.trace && sm.probe && blockIdx.x == 0 && tid == 0) {
                volatile float probe_dep = sm.rin[0];  // forces the deferred barrier to resolve
                (void)probe_dep;
                ck0 = clock64();
            }
            *reinterpret_cast<float2*>(&sm.c[j0]) = chain2<kL>(F + j0, r4);
            if (j == 0) PROBE_T(30, 0);
            if (j == 1 && s.trace && sm.probe && blockIdx.x == 0 && tid == 0) {
                volatile float probe_dep = sm.c[0];
                (void)probe_dep;
                s.trace[s.trace_cap - 64 + 40] = clock64() - ck0;
            }
        } else if (warp == 2) {
            // restrictions Ũ^T r (lanes 0-15) and Ṽ^T r (lanes 16-31), 2 columns per lane
            const int o = lane < 16 ? 2 * lane : kLs + 2 * (lane - 16);
            const float* Bo = B + (lane < 16 ? 0 : kL * kLs) + 2 * (lane & 15);
            __stcg(reinterpret_cast<float2*>(&s.restrict_[leaf * (2 * kLs) + o]), chain2<kLs>(Bo, r4));
            if (j == 0) PROBE_T(34, 64);
        } else if (warp == kPWarps - 1 && lane == 0) {
            // next leaf of the cyclic sequence (wraps to the next iteration's first); stage st^1
            // held the previous leaf, consumed before the barrier above
            const bool wrap = j + 1 == ls.count;
            const uint64_t nxt = wrap ? ls.first : leaf + G;
            if (j == 0) PROBE_T(31, kPThreads - 32);
            p_issue_factors(s, sm, nxt, st ^ 1, pol_f, pol_b);
            if (j == 0) PROBE_T(32, kPThreads - 32);
            if (!wrap) p_issue_vectors(s, sm, nxt, st ^ 1, mode, b, pcur, pol_v);
            if (j == 0) PROBE_T(33, kPThreads - 32);
        }
        __syncthreads();  // c ready
        if (j < 4) PROBE(j * 4 + 2);
        {   // y = F c with exact f64 products (matvec_add_double); 16 warps x 8 rows
            const float4 c4 = reinterpret_cast<const float4*>(sm.c)[lane];
            const double c0 = c4.x, c1 = c4.y, c2 = c4.z, c3 = c4.w;
            double v[8];
#pragma unroll
            for (int rI = 0; rI < 8; ++rI) {
                const float4 f4 = reinterpret_cast<const float4*>(F + (8 * warp + rI) * kL)[lane];
                v[rI] = fma(double(f4.w), c3, fma(double(f4.z), c2, fma(double(f4.y), c1, double(f4.x) * c0)));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool hi = lane & 16;
                const double send = hi ? v[q] : v[q + 4];
                const double keep = hi ? v[q + 4] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const bool hi = lane & 8;
                const double send = hi ? v[q] : v[q + 2];
                const double keep = hi ? v[q + 2] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            {
                const bool hi = lane & 4;
                const double send = hi ? v[0] : v[1];
                const double keep = hi ? v[1] : v[0];
                v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            if ((lane & 3) == 0) {
                const int row = 8 * warp + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                __stcg(&s.y_loc[leaf * kL + row], v[0]);
            }
        }
        if (j < 4) PROBE(j * 4 + 3);
    }
    __syncthreads();  // the last leaf's stage becomes scratch
    return rr;
}

// Leaf phase, pipelined across the CTA's leaves (>= 2 of them): warps 0-3 (the chain group:
// x/r update, the F^T r chains on warps 0-1, the restrictions on warp 2) run leaf j+1 while warps
// 8-15 (the F c group, two 8-row blocks each) finish leaf j, so a leaf costs max(chains, F c)
// instead of their sum. Stage handoff: leaf j lives in stage st_j = (it + j) & 1; the F c group
// issues leaf j+2 (factors + vectors; for j+2 = count the next iteration's first leaf, factors
// only) into st_j once its F c of leaf j is done; at entry leaf 1 (or, with one leaf, the wrap)
// goes into the other stage, which the entry contract leaves free. Same entry / exit contract
// and the same arithmetic per leaf as p_leaf_phase (rr summed by the same threads in the same
// leaf order), so the result is bit-identical.
//   named barriers 3 / 6 (384, by leaf parity): the chain group arrives when c(j) is written,
//   the F c group syncs
//   named barrier 4 (256): the F c group, after its F c of leaf j (then one thread issues)
//   named barrier 5 (128): the chain group, rin(j) complete before the chains
__device__ __forceinline__ double p_leaf_phase_pipe(const DevSys& s, PSmem& sm, PLeafSched& ls, int mode,
                                                    const double* b, const double* pcur, double alpha,
                                                    uint64_t pol_f, uint64_t pol_b, uint64_t pol_v) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t G = gridDim.x, n = ls.count;
    double rr = 0.0;
    const uint32_t it0 = ls.it;
    if (tid == 0) {
        fence_proxy_async_global();
        p_issue_vectors(s, sm, ls.first, int(it0 & 1), mode, b, pcur, pol_v);
        // item 1 into the other (free) stage: leaf 1 (n >= 2 here)
        p_issue_factors(s, sm, ls.first + G, int((it0 + 1) & 1), pol_f, pol_b);
        p_issue_vectors(s, sm, ls.first + G, int((it0 + 1) & 1), mode, b, pcur, pol_v);
    }
    __syncthreads();
    if (warp < 4) {  // ---- chain group
        for (uint64_t j = 0; j < n; ++j) {
            const uint64_t leaf = ls.first + j * G;
            const uint32_t itj = it0 + uint32_t(j);
            const int st = int(itj & 1), pb = int(j & 1);
            const uint32_t par = (itj >> 1) & 1;
            {
                mbar_wait(&sm.vfull[st], par);
                const uint64_t i = leaf * kL + tid;
                double rv = sm.vec[st][0][tid];
                if (mode == kLoop) {  // pcg.cpp:97-98, fused
                    s.x[i] = fma(alpha, sm.vec[st][2][tid], sm.vec[st][3][tid]);
                    rv = fma(-alpha, sm.vec[st][1][tid], rv);
                }
                s.r[i] = rv;
                rr = fma(rv, rv, rr);
                sm.rin2[pb][tid] = static_cast<float>(rv);  // apply.cpp:90
            }
            mbar_wait(&sm.full[st], par);
            named_bar_sync(5, 128);
            const float* F = sm.st[st].F;
            const float* B = sm.st[st].B;
            const float4* r4 = reinterpret_cast<const float4*>(sm.rin2[pb]);
            if (warp < 2) {
                const int j0 = 64 * warp + 2 * lane;
                *reinterpret_cast<float2*>(&sm.c2[pb][j0]) = chain2<kL>(F + j0, r4);
            } else if (warp == 2) {
                const int o = lane < 16 ? 2 * lane : kLs + 2 * (lane - 16);
                const float* Bo = B + (lane < 16 ? 0 : kL * kLs) + 2 * (lane & 15);
                __stcg(reinterpret_cast<float2*>(&s.restrict_[leaf * (2 * kLs) + o]), chain2<kLs>(Bo, r4));
            }
            // c(j) written (warps 0-1), restrictions out. Two barriers by leaf parity: the chain
            // group may reach leaf j+1 before the F c group has synchronised on leaf j (leaf 1
            // is staged at entry), and a hardware barrier counts arrivals, not leaves
            if (j & 1) asm volatile("bar.arrive 6, 384;" ::: "memory");
            else asm volatile("bar.arrive 3, 384;" ::: "memory");
        }
    } else if (warp >= 8) {  // ---- F c group
        const int fw = warp - 8;
        for (uint64_t j = 0; j < n; ++j) {
            const uint64_t leaf = ls.first + j * G;
            const uint32_t itj = it0 + uint32_t(j);
            const int st = int(itj & 1), pb = int(j & 1);
            named_bar_sync((j & 1) ? 6 : 3, 384);  // c(j) complete
            const float* F = sm.st[st].F;
            const float4 c4 = reinterpret_cast<const float4*>(sm.c2[pb])[lane];
            const double c0 = c4.x, c1 = c4.y, c2 = c4.z, c3 = c4.w;
#pragma unroll 1
            for (int blk = fw; blk < 16; blk += 8) {  // two 8-row blocks: rows 8 blk .. 8 blk + 7
                double v[8];
#pragma unroll
                for (int rI = 0; rI < 8; ++rI) {
                    const float4 f4 = reinterpret_cast<const float4*>(F + (8 * blk + rI) * kL)[lane];
                    v[rI] = fma(double(f4.w), c3, fma(double(f4.z), c2, fma(double(f4.y), c1, double(f4.x) * c0)));
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool hi = lane & 16;
                    const double send = hi ? v[q] : v[q + 4];
                    const double keep = hi ? v[q + 4] : v[q];
                    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const bool hi = lane & 8;
                    const double send = hi ? v[q] : v[q + 2];
                    const double keep = hi ? v[q + 2] : v[q];
                    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                }
                {
                    const bool hi = lane & 4;
                    const double send = hi ? v[0] : v[1];
                    const double keep = hi ? v[1] : v[0];
                    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
                v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
                v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
                if ((lane & 3) == 0) {
                    const int row = 8 * blk + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                    __stcg(&s.y_loc[leaf * kL + row], v[0]);
                }
            }
            named_bar_sync(4, 256);  // every F c read of stage st done
            if (fw == 0 && lane == 0 && j + 2 <= n) {
                if (j + 2 < n) {
                    fence_proxy_async_global();
                    p_issue_factors(s, sm, leaf + 2 * G, st, pol_f, pol_b);
                    p_issue_vectors(s, sm, leaf + 2 * G, st, mode, b, pcur, pol_v);
                } else {  // the next iteration's first leaf: factors only (its vectors are not out yet)
                    p_issue_factors(s, sm, ls.first, st, pol_f, pol_b);
                }
            }
        }
    }
    ls.it = it0 + uint32_t(n);
    __syncthreads();  // the last leaf's stage becomes scratch
    return rr;
}

// One tile (L_s = 32, rank 16) per warp:
// lanes q < 16 read column q of U_m (lanes 16 + q: of V_m) straight from L2 (64 contiguous
// bytes per half-warp per row) and run the fp32 chain coef = sum_p U[p][q] float(s_r[p]) in p
// order (matvec_t); lane j then forms coupled_col[j] = float(sum_q V[j][q] coef_r[q]) and
// coupled_row[j] = float(sum_q U[j][q] coef_c[q]) with exact f64 products summed in q order
// (matvec, apply.cpp:121-138) — bit-identical to the reference. f32<->f64 conversions run at
// 15.6/clk/SM (measured), so the strip sums are cast once per tile (lane p casts s_r[p],
// s_c[p]) and each lane converts its coefficient once and broadcasts it through shared memory.
struct alignas(16) PTileScratch {
    float fr[32], fc[32];
    double coef[32];
};
static_assert(kPWarps * sizeof(PTileScratch) + 64 * 32 * sizeof(double) <= sizeof(PStage), "tile scratch");
__device__ __forceinline__ void p_tile(const DevSys& s, uint64_t m, double sr_p, double sc_p,
                                       PTileScratch& ws, int lane, uint64_t pol) {
    const float* T = s.F + s.tile_base + m * (kLs * kLs);
    const float* colp = T + (lane < 16 ? 0 : kLs * 16) + (lane & 15);
    float cv[32];
#pragma unroll
    for (int p = 0; p < 32; ++p) cv[p] = ldg_f32_hint(colp + p * 16, pol);
    float4 u4[4], v4[4];
    const float4* U = reinterpret_cast<const float4*>(T) + lane * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        u4[i] = ldg_hint(U + i, pol);
        v4[i] = ldg_hint(U + 128 + i, pol);
    }
    ws.fr[lane] = float(sr_p);  // apply.cpp:121-124 strip_cast
    ws.fc[lane] = float(sc_p);
    __syncwarp();
    const float4* st4 = reinterpret_cast<const float4*>(lane < 16 ? ws.fr : ws.fc);
    float coef = 0.f;
#pragma unroll
    for (int p4 = 0; p4 < 8; ++p4) {
        const float4 sv = st4[p4];
        coef = fmaf(cv[4 * p4 + 0], sv.x, coef);
        coef = fmaf(cv[4 * p4 + 1], sv.y, coef);
        coef = fmaf(cv[4 * p4 + 2], sv.z, coef);
        coef = fmaf(cv[4 * p4 + 3], sv.w, coef);
    }
    ws.coef[lane] = double(coef);  // [0,16): U^T s_r, [16,32): V^T s_c
    __syncwarp();
    double acc_c = 0.0, acc_r = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float uu[4] = {u4[i].x, u4[i].y, u4[i].z, u4[i].w};
        const float vv[4] = {v4[i].x, v4[i].y, v4[i].z, v4[i].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int qq = 4 * i + t;
            acc_c += double(vv[t]) * ws.coef[qq];
            acc_r += double(uu[t]) * ws.coef[16 + qq];
        }
    }
    __stcg(&s.coupled[m * 64 + 32 + lane], float(acc_c));
    __stcg(&s.coupled[m * 64 + lane], float(acc_r));
    __syncwarp();
}

// Strip sums (apply.cpp:110-120) over the whole bisection tree in one pass. A CTA takes an
// aligned subtree of S <= 32 leaves: warp w owns 4 of the 64 sum columns (u: 0-31, v: 32-63),
// lane q holds leaf q, and a shuffle butterfly builds the pairwise f64 up-sweep (after the step
// of distance d every lane holds its (2d)-group's sum = left child + right child, exactly the
// heap sums node[u] = node[2u+1] + node[2u+2]); the first lane of each group writes the node.
// No shared memory, no block barrier, no arrival hop: the levels above the group roots are never
// materialised (R <= 32 groups in the persistent regime); the tiles phase sums the roots it needs.
__device__ __forceinline__ void p_sums_phase(const DevSys& s, PSmem& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t K = s.K, D = s.D;
    const uint64_t S = K < kCoarseS0 ? K : kCoarseS0, R = K / S;
    int logS = 0;
    while ((1ULL << logS) < S) ++logS;
    const uint64_t dr = D - logS;
    const int side = warp >> 3, c0 = 4 * (warp & 7);  // side 0: u columns, 1: v columns
    double* node = side ? s.node_v : s.node_u;
    (void)sm;
    for (uint64_t task = blockIdx.x; task < R; task += gridDim.x) {
        const bool pr = task == blockIdx.x;
        if (pr) PROBE(44);
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        if (uint64_t(lane) < S) {
            const float4 f = __ldcg(reinterpret_cast<const float4*>(&s.restrict_[(task * S + lane) * 64 + 32 * side + c0]));
            v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        }
        for (int l2 = 0; l2 < logS; ++l2) {  // step 2^l2 -> nodes at local depth logS-1-l2
            const int d = 1 << l2;
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] += __shfl_xor_sync(0xffffffffu, v[c], d);
            const int ld = logS - 1 - l2;
            if (uint64_t(lane) < S && (lane & (2 * d - 1)) == 0) {
                const uint64_t g = (1ULL << (dr + ld)) - 1 + task * (1ULL << ld) + uint64_t(lane >> (l2 + 1));
                __stcg(reinterpret_cast<double2*>(&node[g * 32 + c0]), make_double2(v[0], v[1]));
                __stcg(reinterpret_cast<double2*>(&node[g * 32 + c0 + 2]), make_double2(v[2], v[3]));
            }
        }
        if (pr) PROBE(45);
    }
}

// Pairwise (heap-order) sum of W (a power of two) consecutive group roots at depth dr, lane =
// column: the value the up-sweep would have stored in their common ancestor. Blocks of 8 are
// summed in registers; block sums merge through a binary-counter stack (the same tree).
__device__ __forceinline__ double p_root_sum(const double* node, uint64_t dr, uint64_t g0, uint64_t W, int lane) {
    const double* base = node + ((1ULL << dr) - 1 + g0) * 32 + lane;
    if (W <= 8) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (uint64_t(i) < W) v[i] = __ldcg(base + i * 32);
#pragma unroll
        for (int w = 1; w < 8; w *= 2)
#pragma unroll
            for (int i = 0; i + w < 8; i += 2 * w)
                if (uint64_t(i + w) < W) v[i] = v[i] + v[i + w];
        return v[0];
    }
    double stack[24];
    int top = 0;
    for (uint64_t b = 0; b < W / 8; ++b) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldcg(base + (b * 8 + i) * 32);
#pragma unroll
        for (int w = 1; w < 8; w *= 2)
#pragma unroll
            for (int i = 0; i + w < 8; i += 2 * w) v[i] = v[i] + v[i + w];
        double x = v[0];
        for (uint64_t c = b + 1; (c & 1) == 0; c >>= 1) x = stack[--top] + x;  // merge equal subtrees
        stack[top++] = x;
    }
    return stack[0];
}

// Tile couplings (apply.cpp:121-138): every tile in parallel, one warp each, dealt across CTAs
// first (tile order t -> CTA t mod grid). Children sums come from the node arrays (leaf children:
// the restrictions themselves); tiles above the 32-leaf groups sum their children's group roots
// pairwise themselves (p_root_sum), so the strip-sum phase needs no arrival hop.
__device__ __forceinline__ void p_tiles_phase(const DevSys& s, PSmem& sm, PTileScratch* ws, uint64_t pol) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t K = s.K, G = gridDim.x;
    const uint64_t S0 = K < kCoarseS0 ? K : kCoarseS0, R = K / S0;
    int logS0 = 0;
    while ((1ULL << logS0) < S0) ++logS0;
    const uint64_t dr = s.D - logS0;  // depth of the group roots (R <= 32 in the persistent regime)
    for (uint64_t m = uint64_t(wid) * G + blockIdx.x; m < K - 1; m += G * kPWarps) {
        if (m == 0) PROBE(56);
        const uint64_t l = 2 * m + 1, r = 2 * m + 2;  // children (heap)
        double a, bb;
        if (l >= K - 1) {
            a = double(__ldcg(&s.restrict_[(l - (K - 1)) * 64 + lane]));
            bb = double(__ldcg(&s.restrict_[(r - (K - 1)) * 64 + 32 + lane]));
        } else if (m + 1 < R) {  // above the 32-leaf groups: the children's sums from the group roots
            int d = 0;
            while ((2ULL << d) <= m + 1) ++d;
            const uint64_t wg = R >> d, g0 = (m + 1 - (1ULL << d)) * wg, W = wg / 2;
            a = p_root_sum(s.node_u, dr, g0, W, lane);
            bb = p_root_sum(s.node_v, dr, g0 + W, W, lane);
        } else {
            a = __ldcg(&s.node_u[l * 32 + lane]);
            bb = __ldcg(&s.node_v[r * 32 + lane]);
        }
        p_tile(s, m, a, bb, ws[wid], lane, pol);
        if (m == 0) PROBE(57);
    }
}

// The coarse stage (apply.cpp:110-138) in ONE phase — no strip-sum pass and one grid barrier
// less per iteration. Nothing below the group roots is stored any more:
//   * a tile above the 32-leaf groups (m < R - 1 <= 31: one per CTA) has its CTA's 16 warps sum
//     its children's groups straight from the restrictions, in half-groups of 16 leaves
//     (leaf_run_sum<16>: the up-sweep's tree), then warp 0 forms each group root as the two
//     halves' sum and the child's strip sum as the pairwise tree over its W groups — the values
//     the up-sweep + p_root_sum produced;
//   * a group-internal tile sums its children's <= 16 leaves itself (child_strip_sum).
// Bit-identical couplings to p_sums_phase + p_tiles_phase (same trees, same tile arithmetic).
__device__ __forceinline__ void p_coarse_phase(const DevSys& s, PSmem& sm, unsigned char* scr, uint64_t pol) {
    PTileScratch* ws = reinterpret_cast<PTileScratch*>(scr);
    double* hs = reinterpret_cast<double*>(scr + kPWarps * sizeof(PTileScratch));  // [64][32]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t K = s.K, G = gridDim.x, b = blockIdx.x;
    const uint64_t S0 = K < kCoarseS0 ? K : kCoarseS0, R = K / S0;
    if (R > 1 && b + 1 < R) {  // R <= 32 (the caller's condition): at most one such tile per CTA
        const uint64_t m = b;
        if (m == 0) PROBE(56);
        int d = 0;
        while ((2ULL << d) <= m + 1) ++d;
        const uint64_t wg = R >> d, g0 = (m + 1 - (1ULL << d)) * wg, W = wg / 2;
        for (uint64_t u = uint64_t(wid); u < 4 * W; u += kPWarps) {  // (group, half) units
            const uint64_t gi = u >> 1, side = gi < W ? 0 : 1;
            const float* p = s.restrict_ + ((g0 + gi) * 32 + 16 * (u & 1)) * 64 + 32 * side + lane;
            hs[u * 32 + lane] = leaf_run_sum<16>(p);
        }
        __syncthreads();
        if (wid == 0) {
            double ga[16], gb[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                ga[i] = gb[i] = 0.0;
                if (uint64_t(i) < W) {
                    ga[i] = hs[(2 * i) * 32 + lane] + hs[(2 * i + 1) * 32 + lane];
                    gb[i] = hs[(2 * (W + i)) * 32 + lane] + hs[(2 * (W + i) + 1) * 32 + lane];
                }
            }
#pragma unroll
            for (int w = 1; w < 16; w *= 2)
#pragma unroll
                for (int i = 0; i + w < 16; i += 2 * w)
                    if (uint64_t(i + w) < W) {
                        ga[i] = ga[i] + ga[i + w];
                        gb[i] = gb[i] + gb[i + w];
                    }
            p_tile(s, m, ga[0], gb[0], ws[0], lane, pol);
        }
        if (m == 0) PROBE(57);
    }
    for (uint64_t m = (R - 1) + uint64_t(wid) * G + b; m < K - 1; m += G * kPWarps) {
        const double a = child_strip_sum(s, 2 * m + 1, 0, lane);
        const double bb = child_strip_sum(s, 2 * m + 2, 1, lane);
        p_tile(s, m, a, bb, ws[wid], lane, pol);
    }
}

// Prolongation + gate (apply stages 5-7), one warp per leaf; leaves are dealt across CTAs first
// (leaf order w -> CTA w mod grid) so small systems spread over every SM, in reverse leaf order
// (the bridges read last by the leaf phase may still be in L2). Returns this thread's r.z part.
__device__ __forceinline__ double p_prolong_phase(const DevSys& s, PSmem& sm, PScratchProlong& ps,
                                                  double shift) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t K = s.K, D = s.D, G = gridDim.x;
    const int l8 = lane & 7, rsub = lane >> 3;
    // a leaf's 128 rows are split over P warps (128 / P rows each) when the grid has the warps
    // for it: at small K one warp per leaf walked its 8 bridge chunks in 4-5 dependent L2 round
    // trips while most warps idled (8K: 64 leaves on 2,368 warps). The rows' arithmetic is
    // unchanged; r.z is summed in another (valid) order.
    uint32_t P = 1;
    while (P < 8 && uint64_t(2 * P) * K <= G * kPWarps) P *= 2;
    const uint32_t rows_per = kL / P, nch = rows_per / 16;
    double rz = 0.0;
    for (uint64_t item = uint64_t(wid) * G + blockIdx.x; item < K * P; item += G * kPWarps) {
        const uint64_t w = item / P, leaf = K - 1 - w;
        const uint32_t part = uint32_t(item % P), row0 = part * rows_per, c0 = row0 / 16;
        const uint64_t base = leaf * kL;
        if (item == 0) PROBE(20);
        const uint32_t hl = uint32_t(K + leaf), lf = uint32_t(leaf), Du = uint32_t(D);
        float ga[kMaxDepth];
#pragma unroll
        for (int d = 0; d < kMaxDepth; ++d) {
            ga[d] = 0.f;
            if (uint32_t(d) < Du) {
                const uint32_t m = (hl >> (Du - d)) - 1u, right = (lf >> (Du - 1 - d)) & 1u;
                ga[d] = __ldcg(&s.coupled[m * 64u + right * 32u + lane]);
            }
        }
        // f64 gathers in tile order, root first (apply.cpp:140-154)
        double gr = 0.0, gc = 0.0;
#pragma unroll
        for (int d = 0; d < kMaxDepth; ++d)
            if (uint32_t(d) < Du) {
                if ((lf >> (Du - 1 - d)) & 1u) gc += double(ga[d]);
                else gr += double(ga[d]);
            }
        const float grf = float(gr), gcf = float(gc);
        double g4[4], h4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            g4[q] = double(__shfl_sync(0xffffffffu, grf, 4 * l8 + q));
            h4[q] = double(__shfl_sync(0xffffffffu, gcf, 4 * l8 + q));
        }
        // bridges: chunk c = rows 16c..16c+15; lane (rsub, l8) covers rows 16c + 4i + rsub,
        // columns 4 l8 .. 4 l8 + 3; two chunks in flight. Exact f64 products summed in f64.
        const float4* Bu = reinterpret_cast<const float4*>(s.F + s.bridge_base + leaf * (2 * kL * kLs));
        const float4* Bv = Bu + kL * kLs / 4;
        float4 ua[4], va[4], ub[4], vb[4];
        auto load_chunk = [&](uint32_t c, float4 (&u)[4], float4 (&v)[4]) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = 16 * c + 4 * i + rsub;
                u[i] = ldg_stream(Bu + row * (kLs / 4) + l8);
                v[i] = ldg_stream(Bv + row * (kLs / 4) + l8);
            }
        };
        auto do_chunk = [&](uint32_t c, const float4 (&u)[4], const float4 (&v)[4]) {
            double val[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                val[i] = fma(double(u[i].w), g4[3], fma(double(u[i].z), g4[2],
                         fma(double(u[i].y), g4[1], double(u[i].x) * g4[0])));
                val[4 + i] = fma(double(v[i].w), h4[3], fma(double(v[i].z), h4[2],
                             fma(double(v[i].y), h4[1], double(v[i].x) * h4[0])));
            }
            // transpose-reduce over the 8 lanes of a row group: lane l8 ends with value l8
            // (l8 < 4: Ũ row 16c + 4 l8 + rsub, else Ṽ), 7 shuffles instead of 24
            double t4[4], t2[2];
            const bool h4b = l8 & 4, h2b = l8 & 2, h1b = l8 & 1;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                t4[q] = (h4b ? val[4 + q] : val[q]) + __shfl_xor_sync(0xffffffffu, h4b ? val[q] : val[4 + q], 4);
#pragma unroll
            for (int q = 0; q < 2; ++q)
                t2[q] = (h2b ? t4[2 + q] : t4[q]) + __shfl_xor_sync(0xffffffffu, h2b ? t4[q] : t4[2 + q], 2);
            const double t1 = (h1b ? t2[1] : t2[0]) + __shfl_xor_sync(0xffffffffu, h1b ? t2[0] : t2[1], 1);
            const int row = 16 * c + 4 * (l8 & 3) + rsub;
            if (l8 < 4) ps.su[wid][row] = t1;
            else ps.sv[wid][row] = t1;
        };
        load_chunk(c0, ua, va);
        if (nch == 1) {
            do_chunk(c0, ua, va);
        } else {
#pragma unroll 1
            for (uint32_t c = c0; c < c0 + nch; c += 2) {
                load_chunk(c + 1, ub, vb);
                do_chunk(c, ua, va);
                if (c + 2 < c0 + nch) load_chunk(c + 2, ua, va);
                do_chunk(c + 1, ub, vb);
            }
        }
        if (item == 0) PROBE(21);
        double yl[4], rv[4], ad[4];
        float gt[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t r = lane + 32 * t;
            if (r < rows_per) {
                const uint64_t i = base + row0 + r;
                yl[t] = __ldcg(&s.y_loc[i]);
                rv[t] = __ldcg(&s.r[i]);
                ad[t] = __ldg(&s.a_diag[i]);
                gt[t] = __ldg(&s.F[s.gate_base + i]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t r = lane + 32 * t;
            if (r < rows_per) {
                const uint32_t row = row0 + r;
                double y = yl[t];
                y += ps.su[wid][row];
                y += ps.sv[wid][row];
                y += double(gt[t]) * rv[t] / ad[t] + shift * rv[t];
                s.z[base + row] = y;
                rz = fma(rv[t], y, rz);
            }
        }
        __syncwarp();
        if (item == 0) PROBE(22);
    }
    return rz;
}

// SpMV phase: p = z + beta p_prev (pcg.cpp:118), Ap (csr.cpp:70-79, bit-identical: sequential
// per-row f64 sum in column order, unfused products), p.Ap and p.p parts. A warp owns a SELL-32
// slice (one row per lane). With s.pspmv_stage_bytes > 0 the CTA's chunks of 16 slices stream
// through a 2-stage TMA ring in the scratch stage; else values/columns are loaded directly.
__device__ __forceinline__ void p_spmv_phase(const DevSys& s, PSmem& sm, unsigned char* ring,
                                             uint32_t& spit, double beta, const double* pprev,
                                             double* pcur, double (&v)[2]) {
    const double* z = s.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t nsl = (s.n + 31) >> 5;
    const uint32_t cap = s.pspmv_stage_bytes;
    auto row_work = [&](uint64_t sl, const double* vals, const uint32_t* cols, uint64_t w) {
        const uint64_t row = sl * 32 + lane;
        double zr = 0.0, pr = 0.0;
        if (row < s.n) {
            zr = __ldcg(&z[row]);
            pr = __ldcg(&pprev[row]);
        }
        const double acc = sell_row<true, true>(vals, cols, w, lane, z, pprev, beta);
        if (row < s.n) {
            s.ap[row] = acc;
            const double pi = fma(beta, pr, zr);
            pcur[row] = pi;
            v[0] = fma(pi, acc, v[0]);
            v[1] = fma(pi, pi, v[1]);
        }
    };
    if (cap == 0) {
        for (uint64_t sl = uint64_t(blockIdx.x) * kPWarps + warp; sl < nsl; sl += uint64_t(gridDim.x) * kPWarps) {
            const uint64_t base = __ldg(&s.slice_off[sl]), w = (__ldg(&s.slice_off[sl + 1]) - base) >> 5;
            row_work(sl, s.sell_vals + base, s.sell_cols + base, w);
        }
        return;
    }
    const uint64_t nch = (nsl + kPSpmvSlices - 1) / kPSpmvSlices;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](uint64_t ch, int st) {
        const uint64_t s0 = ch * kPSpmvSlices, s1 = s0 + kPSpmvSlices < nsl ? s0 + kPSpmvSlices : nsl;
        const uint64_t e0 = __ldg(&s.slice_off[s0]), ne = __ldg(&s.slice_off[s1]) - e0;
        unsigned char* bb = ring + size_t(st) * cap;
        fence_proxy_async_smem();
        mbar_expect_tx(&sm.sfull[st], uint32_t(ne * 12));
        tma_load_1d(bb, s.sell_vals + e0, uint32_t(ne * 8), &sm.sfull[st], pol);
        tma_load_1d(bb + ne * 8, s.sell_cols + e0, uint32_t(ne * 4), &sm.sfull[st], pol);
    };
    const uint64_t G = gridDim.x;
    // spit counts this CTA's ring steps over the whole solve (stage = spit & 1)
    if (tid == 0) {
        if (blockIdx.x < nch) issue(blockIdx.x, int(spit & 1));
        if (blockIdx.x + G < nch) issue(blockIdx.x + G, int((spit + 1) & 1));
    }
    for (uint64_t ch = blockIdx.x; ch < nch; ch += G, ++spit) {
        const int st = int(spit & 1);
        mbar_wait(&sm.sfull[st], (spit >> 1) & 1);
        const uint64_t s0 = ch * kPSpmvSlices, sl = s0 + warp;
        if (sl < nsl) {
            const uint64_t s1 = s0 + kPSpmvSlices < nsl ? s0 + kPSpmvSlices : nsl;
            const uint64_t e0 = __ldg(&s.slice_off[s0]), ne = __ldg(&s.slice_off[s1]) - e0;
            const uint64_t o0 = __ldg(&s.slice_off[sl]), o1 = __ldg(&s.slice_off[sl + 1]);
            const unsigned char* bb = ring + size_t(st) * cap;
            row_work(sl, reinterpret_cast<const double*>(bb) + (o0 - e0),
                     reinterpret_cast<const uint32_t*>(bb + ne * 8) + (o0 - e0), (o1 - o0) >> 5);
        }
        __syncthreads();  // stage st consumed
        if (tid == 0 && ch + 2 * G < nch) issue(ch + 2 * G, st);
    }
}

// The whole solve. Scalars in s.sc carry the configuration in (rtol, max_iters, breakdown_tol,
// shift) and the report out. bar_count = grid-barrier counter (zeroed before the launch);
// s.partials holds 3 x gridDim.x x 2 doubles. The loop-carried state is kept to a handful of
// registers (rz, r0, beta, k, the leaf/ring counters): every phase gets the rest of the 128.
__global__ void __launch_bounds__(kPThreads, 1) k_solve(DevSys s, const double* b, unsigned* bar_count) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PSmem& sm = *reinterpret_cast<PSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const Scalars* cfg = s.sc;
    PBar bar{bar_count, 0u};

    PLeafSched ls;
    ls.first = blockIdx.x;
    ls.count = blockIdx.x < s.K ? (s.K - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    ls.it = 0;
    uint32_t spit = 0;
    if (tid == 0) {
        for (int q = 0; q < 2; ++q) {
            mbar_init(&sm.full[q], 1);
            mbar_init(&sm.vfull[q], 1);
            mbar_init(&sm.sfull[q], 1);
        }
        fence_mbar_init();
        sm.probe = 0;
    }
    __syncthreads();
    if (tid == 0 && ls.count)
        p_issue_factors(s, sm, ls.first, 0, s.l2_resident ? policy_evict_last() : policy_evict_first(),
                        policy_evict_last());
    if (s.trace && blockIdx.x == 0 && tid == 0) s.trace[0] = globaltimer();
    auto scratch = [&]() -> unsigned char* {
        return reinterpret_cast<unsigned char*>(&sm.st[ls.count ? ((ls.it & 1) ^ 1) : 0]);
    };
    auto leaf = [&](int mode, const double* pcur, double alpha) -> double {
        const uint64_t keep = policy_evict_last();
        const uint64_t pf = s.l2_resident ? keep : policy_evict_first();
        double v[1] = {ls.count >= 2 && s.ksolve_pipe ? p_leaf_phase_pipe(s, sm, ls, mode, b, pcur, alpha, pf, keep, keep)
                                                      : p_leaf_phase(s, sm, ls, mode, b, pcur, alpha, pf, keep, keep)};
        double t[1];
        grid_reduce<1>(s, sm, bar, v, s.partials + 2 * gridDim.x, t);
        return t[0];
    };
    auto apply_tail = [&]() -> double {  // apply stages 4-7 after the leaf phase's barrier
        if (s.K <= 32 * kCoarseS0) {  // R <= 32 group roots: one phase (p_coarse_phase)
            p_coarse_phase(s, sm, scratch(), policy_evict_last());
        } else {  // larger (forced persistent): strip sums, then every tile
            p_sums_phase(s, sm);
            grid_barrier(s, bar);
            p_tiles_phase(s, sm, reinterpret_cast<PTileScratch*>(scratch()), policy_evict_last());
        }
        grid_barrier(s, bar);
        double v[1] = {p_prolong_phase(s, sm, *reinterpret_cast<PScratchProlong*>(scratch()), __ldg(&cfg->shift))};
        double t[1];
        grid_reduce<1>(s, sm, bar, v, s.partials + 4 * gridDim.x, t);
        return t[0];
    };

    // ---- init (pcg.cpp:65-84): x = 0, r = b, p_prev = 0, r0, z = M r, rz
    for (uint64_t i = uint64_t(blockIdx.x) * kPThreads + tid; i < s.n; i += uint64_t(gridDim.x) * kPThreads) {
        s.x[i] = 0.0;
        s.p0[i] = 0.0;
    }
    // exit reasons: 0 converged, 1 max_iters, 2 breakdown
    int reason = 1;
    unsigned long long k = 0;
    double rz = 0.0, beta = 0.0, rel = 0.0;
    const double r0 = sqrt(leaf(kInit, nullptr, 0.0));
    if (r0 == 0.0) {  // pcg.cpp:73-79: converged in 0 iterations
        reason = 0;
    } else {
        rz = apply_tail();  // pcg.cpp:82-84
        k = 1;
        if (__ldg(&cfg->max_iters) == 0) k = 0;  // max_iters after 0 iterations
    }
    // ---- loop (pcg.cpp:86-119)
    while (k > 0) {
        if (tid == 0) sm.probe = (k == (unsigned long long)s.trace_probe);
        double* pcur = (k & 1ULL) ? s.p1 : s.p0;
        double pap, p2;
        {
            double v[2] = {0.0, 0.0};
            p_spmv_phase(s, sm, scratch(), spit, beta, (k & 1ULL) ? s.p0 : s.p1, pcur, v);
            double t[2];
            grid_reduce<2>(s, sm, bar, v, s.partials, t);
            pap = t[0];
            p2 = t[1];
        }
        if (pap < -__ldg(&cfg->breakdown_tol) * p2 || pap == 0.0) {  // pcg.cpp:90-95
            reason = 2;
            break;
        }
        rel = sqrt(leaf(kLoop, pcur, rz / pap)) / r0;
        if (blockIdx.x == 0 && tid == 0 && s.history) s.history[k - 1] = rel;
        if (rel <= __ldg(&cfg->rtol)) {
            reason = 0;
            break;
        }
        if (k == __ldg(&cfg->max_iters)) break;
        const double rz_new = apply_tail();
        beta = rz_new / rz;  // pcg.cpp:115-117
        rz = rz_new;
        k += 1;
    }
    // drain the prefetched leaf before the CTA's shared memory goes away
    if (ls.count) mbar_wait(&sm.full[ls.it & 1], (ls.it >> 1) & 1);
    if (blockIdx.x == 0 && tid == 0) {
        Scalars* out = s.sc;
        out->rz = rz;
        out->beta = beta;
        out->r0 = r0;
        out->rel = rel;
        out->k = k;
        out->iterations = k;
        out->hist_len = reason == 2 ? (k ? k - 1 : 0) : k;
        out->breakdown_iter = reason == 2 ? k : 0;
        out->status = reason;
        out->converged = reason == 0;
        out->done = 1;
    }
}

}  // namespace hfpg
