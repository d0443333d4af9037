// EXPERIMENTAL, opt-in (HFPG_LEAF_COARSE=1; not the product path): apply stages 1-4 in one
// persistent kernel (single-rank fast path, L = 128, L_s = 32). Parity-green, but measured
// slower than k_leaf_fast + k_coarse_coop (232 vs 171 us at 3D 1M: its F phase is compute-
// latency bound); kept as the A/B arm behind that finding, with a per-CTA phase
// trace (hfpg_set_trace, tools/lc_trace.py).
//
//   phase 1  every CTA streams the bridge pairs Ũ_k | Ṽ_k (and the leaf's PCG vector slices)
//            of its static share of leaves: x += alpha p, r' = r - alpha Ap, |r'|^2
//            (pcg.cpp:97-101), the restrictions û = Ũ_k^T r'_k, v̂ = Ṽ_k^T r'_k (apply.cpp:102-108)
//            -> restrict_. r itself is left alone: the prolongation stores r' (it re-forms it
//            with the same fused multiply-add), so no unit below depends on another CTA's
//            phase-1 output except the coarse ones.
//   phase 2  the CTA's F leaves (the same static share): c = F_k^T r'_k, y_k = F_k c
//            (apply.cpp:93-100) -> y_loc, r'_k re-formed from r_k and Ap_k; between two F
//            leaves, once every CTA has finished phase 1, coarse units taken with tickets: the
//            residual bookkeeping of pcg.cpp:97-112 (one unit), the 32-leaf strip-sum sweeps
//            (apply.cpp:110-120), then — once all sweeps are done — the tiles (V(U^T s_r),
//            U(V^T s_c), apply.cpp:121-138). The coarse stage (latency-bound on its own:
//            k_sums_tree + k_tiles_all) so runs inside the F stream instead of after it.
//            Nothing waits on a CTA that may not be resident: a CTA whose F leaves are done
//            leaves unless every CTA has finished phase 1 and tickets are still open (those
//            units only wait on units running CTAs hold); the CTA that completes phase 1 always
//            sees the open tickets. The last CTA to leave resets the tickets for the next launch.
//
// The arithmetic is k_leaf_fast's / k_sums_tree's / k_tiles_all's unchanged (same chains, same
// orders): the factor path stays bit-identical to the staged kernels.
#pragma once

namespace hfpg {

constexpr int kLcStages1 = 5;  // phase 1 ring: bridges + vector slices (36 KB stages)
constexpr int kLcStages2 = 3;  // phase 2 ring: F_k + r_k, Ap_k (66 KB stages): two in flight while one computes
struct LcSmem {
    union {
        struct {
            float B[kLcStages1][2 * kL * kLs];
            double vec[kLcStages1][4][kL];
        } p1;
        struct {
            float F[kLcStages2][kL * kL];
            double r[kLcStages2][2][kL];  // r_k, Ap_k of the staged leaf
        } p2;
    } u;
    float rin[kL];
    float c[kL];
    TileScratch ws[kLeafThreads / 32];
    uint64_t full[kLcStages1 > kLcStages2 ? kLcStages1 : kLcStages2];
};

// Tickets / arrivals of one launch (DevSys::counters[4 ..]): zero between launches.
enum LcCounter { kLcP1 = 0, kLcSumT, kLcSumD, kLcTileT, kLcEpi, kLcExit, kLcN };

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_relaxed(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long lc_clock() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kLeafThreads, 1) k_leaf_coarse(DevSys s, int mode, const double* rin_ext) {
    if (mode != kApply && s.sc->done) return;
    // hfpg_set_trace(h, >= 4 grid): per-CTA %globaltimer at start / end of phase 1 / end, units
    // (>= 8 grid: + ns spent in F / sum / tile / wait units)
    unsigned long long* tr = (s.trace && s.trace_cap >= 4 * gridDim.x) ? s.trace + (s.trace_cap >= 12 * gridDim.x ? 12 : s.trace_cap >= 8 * gridDim.x ? 8 : 4) * blockIdx.x : nullptr;
    const bool tr8 = tr && s.trace_cap >= 8 * gridDim.x;
    unsigned long long t_unit[4] = {0, 0, 0, 0}, t_mark = 0;
    const bool tr12 = tr && s.trace_cap >= 12 * gridDim.x;  // + F-unit sub-phase clock64 cycles
    long long t_sub[3] = {0, 0, 0};
    const long long clk0 = clock64();
    if (tr && threadIdx.x == 0) tr[0] = lc_clock();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    LcSmem& sm = *reinterpret_cast<LcSmem*>(smem_raw);
    unsigned* ctr = s.counters + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double alpha = 0.0;
    const double* rsrc = mode == kApply ? rin_ext : s.r;
    const double* pcur = mode == kLoop ? p_cur(s, s.sc->k) : nullptr;
    const uint64_t K = s.K;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const int nvec = mode == kLoop ? 4 : 1;
    const uint32_t stage1_bytes = kBBytes + nvec * kL * 8;
    const unsigned grid = gridDim.x;

    if (tid == 0) {
        for (int q = 0; q < kLcStages1; ++q) mbar_init(&sm.full[q], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue1 = [&](uint64_t leaf, int st) {
        mbar_expect_tx(&sm.full[st], stage1_bytes);
        const float* b = s.F + s.bridge_base + leaf * (2 * kL * kLs);
        // bridges evict_last: the prolongation walks the leaves in reverse and finds the most
        // recently streamed ones in L2
        tma_load_1d(&sm.u.p1.B[st][0], b, kBBytes / 2, &sm.full[st], pol_keep);
        tma_load_1d(&sm.u.p1.B[st][kL * kLs], b + kL * kLs, kBBytes / 2, &sm.full[st], pol_keep);
        tma_load_1d(sm.u.p1.vec[st][0], rsrc + leaf * kL, kL * 8, &sm.full[st], pol_keep);
        if (mode == kLoop) {
            tma_load_1d(sm.u.p1.vec[st][1], s.ap + leaf * kL, kL * 8, &sm.full[st], pol_stream);
            tma_load_1d(sm.u.p1.vec[st][2], pcur + leaf * kL, kL * 8, &sm.full[st], pol_stream);
            tma_load_1d(sm.u.p1.vec[st][3], s.x + leaf * kL, kL * 8, &sm.full[st], pol_stream);
        }
    };
    // ---- prologue: first leaves in flight; alpha from the SpMV's partials (pcg.cpp:88-96)
    if (tid == 0)
        for (int q = 0; q < kLcStages1; ++q)
            if (blockIdx.x + uint64_t(q) * grid < K) issue1(blockIdx.x + uint64_t(q) * grid, q);
    if (mode == kLoop) {
        __shared__ double sa;
        __shared__ int sbrk;
        if (tid >= 32 && tid < 64) {
            double t[2];
            sum_partials<2>(s.dpart + kPartSpmv, s.grid_spmv, t);
            if (tid == 32) {
                Scalars* sc = s.sc;
                const unsigned long long k = sc->k;
                const bool brk = t[0] < -sc->breakdown_tol * t[1] || t[0] == 0.0;  // pcg.cpp:90-95
                sa = sc->rzs[k & 1] / t[0];
                sbrk = brk;
                if (blockIdx.x == 0) {
                    sc->pap = t[0];
                    sc->pp = t[1];
                    sc->alpha = sa;
                    if (brk) {
                        sc->status = 2;
                        sc->breakdown_iter = k;
                        sc->iterations = k;
                        sc->done = 1;
                    }
                }
            }
        }
        __syncthreads();
        alpha = sa;
        if (sbrk) {  // no update; let the issued copies land before the CTA exits
            for (int q = 0; q < kLcStages1; ++q)
                if (blockIdx.x + uint64_t(q) * grid < K) mbar_wait(&sm.full[q], 0);
            return;
        }
    }

    // ---- phase 1: update + restrictions of this CTA's leaves
    double rr = 0.0;
    uint32_t it = 0;
    for (uint64_t leaf = blockIdx.x; leaf < K; leaf += grid, ++it) {
        const int st = int(it % kLcStages1);
        mbar_wait(&sm.full[st], (it / kLcStages1) & 1);
        if (tid < kL) {
            const uint64_t i = leaf * kL + tid;
            double rv = sm.u.p1.vec[st][0][tid];
            if (mode == kLoop) {  // pcg.cpp:97-98, fused (r' is stored by the prolongation)
                s.x[i] = fma(alpha, sm.u.p1.vec[st][2][tid], sm.u.p1.vec[st][3][tid]);
                rv = fma(-alpha, sm.u.p1.vec[st][1][tid], rv);
            }
            rr = fma(rv, rv, rr);
            sm.rin[tid] = static_cast<float>(rv);  // apply.cpp:90
        }
        __syncthreads();
        if (tid >= kL && tid < kL + 2 * kLs) {  // matvec_t order (apply.cpp:25-35)
            const int o = tid - kL;
            const float* Bo = sm.u.p1.B[st] + (o >> 5) * (kL * kLs) + (o & 31);
            float acc = 0.f;
#pragma unroll 16
            for (int i = 0; i < kL; ++i) acc = fmaf(Bo[i * kLs], sm.rin[i], acc);
            __stcg(&s.restrict_[leaf * (2 * kLs) + o], acc);
        }
        __syncthreads();
        const uint64_t nxt = leaf + uint64_t(kLcStages1) * grid;
        if (tid == 0 && nxt < K) issue1(nxt, st);
    }
    if (mode != kApply) {  // |r|^2 partial: summed by the coarse epilogue unit
        double v[1] = {rr};
        publish_partials<1>(v, s.dpart + kPartLeaf);
    }
    __shared__ int is_last_p1;
    if (tr && threadIdx.x == 0) tr[1] = lc_clock();
    __syncthreads();  // restrictions / partials of this CTA before its release
    if (tid == 0) is_last_p1 = atom_add_acq_rel_gpu(&ctr[kLcP1], 1u) == grid - 1;
    // the phase-1 ring's last copies have all been consumed (every issued stage was waited on)

    // ---- phase 2: this CTA's F leaves (the same static share as phase 1) with coarse units
    // taken between them through tickets, once every CTA has been through phase 1
    const uint64_t S0 = K < kCoarseS0 ? K : kCoarseS0, R = K / S0;
    int logS0 = 0;
    while ((1ULL << logS0) < S0) ++logS0;
    const uint64_t dr = s.D - logS0;
    const uint64_t n_upper = R - 1;                               // CTA-wide tiles
    const uint64_t n_inner_units = (K - 1 - n_upper + 15) / 16;  // 16 tiles (one per warp) per unit
    const uint64_t n_tile_units = n_upper + n_inner_units;
    const bool want_epi = s.defer && mode != kApply;
    __shared__ int action;
    __shared__ uint64_t unit;
    // tid 0's view of the tickets (once true, stays true)
    __shared__ int p1_done, epi_taken, sums_out, sums_ready, tiles_out;
    enum { kActF = 0, kActSum, kActTile, kActEpi, kActWait, kActExit };
    auto issue2 = [&](uint64_t leaf, int st) {
        mbar_expect_tx(&sm.full[st], kFBytes + (mode == kLoop ? 2 : 1) * kL * 8);
        const float* f = s.F + leaf * (kL * kL);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            tma_load_1d(&sm.u.p2.F[st][q * kL * kL / 4], f + q * kL * kL / 4, kFBytes / 4, &sm.full[st], pol_stream);
        tma_load_1d(sm.u.p2.r[st][0], rsrc + leaf * kL, kL * 8, &sm.full[st], pol_keep);
        if (mode == kLoop) tma_load_1d(sm.u.p2.r[st][1], s.ap + leaf * kL, kL * 8, &sm.full[st], pol_keep);
    };
    // the F ring reuses two of the phase-1 barriers: every phase-1 stage was consumed, nothing is
    // in flight, so they are simply re-initialised
    __syncthreads();
    if (tid == 0) {
        for (int q = 0; q < kLcStages2; ++q) {
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&sm.full[q])) : "memory");
            mbar_init(&sm.full[q], 1);
        }
        fence_mbar_init();
        for (int q = 0; q < kLcStages2; ++q)
            if (blockIdx.x + uint64_t(q) * grid < K) issue2(blockIdx.x + uint64_t(q) * grid, q);
        p1_done = epi_taken = sums_out = sums_ready = tiles_out = 0;
        epi_taken = want_epi ? 0 : 1;
    }
    __syncthreads();
    uint64_t fleaf = blockIdx.x;  // next F leaf of this CTA
    uint32_t fit = 0;
    unsigned peek_p1 = 0, peek_sums = 0;  // relaxed loads issued a unit ahead of their use
    int last_act = -1;
    if (tr8 && tid == 0) t_mark = lc_clock();
    for (;;) {
        if (tid == 0) {
            if (tr8) {
                const unsigned long long now = lc_clock();
                if (last_act == kActF) t_unit[0] += now - t_mark;
                else if (last_act == kActSum) t_unit[1] += now - t_mark;
                else if (last_act == kActTile) t_unit[2] += now - t_mark;
                // (other units' time is not recorded: slot 3 holds the F units' mbarrier waits)
                t_mark = now;
            }
            // the loads issued at the end of the previous unit have landed by now
            if (!p1_done && peek_p1 == grid) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                p1_done = 1;
            }
            if (!sums_ready && sums_out && peek_sums == R) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                sums_ready = 1;
            }
            int act = -1;
            uint64_t u = 0;
            if (p1_done) {
                if (!epi_taken) {
                    epi_taken = 1;
                    if (atomicCAS(&ctr[kLcEpi], 0u, 1u) == 0u) act = kActEpi;
                }
                if (act < 0 && !sums_out) {
                    u = atom_add_relaxed(&ctr[kLcSumT], 1u);
                    if (u < R) act = kActSum;
                    else sums_out = 1;
                }
                if (act < 0 && sums_ready && !tiles_out) {
                    u = atom_add_relaxed(&ctr[kLcTileT], 1u);
                    if (u < n_tile_units) act = kActTile;
                    else tiles_out = 1;
                }
            }
            if (act < 0) {
                if (fleaf < K) act = kActF;
                else if (!p1_done) act = kActExit;  // the CTA that completes phase 1 sees p1_done
                else if (tiles_out && sums_out) act = kActExit;  // every ticket taken (units finish on running CTAs)
                else act = kActWait;  // tiles still blocked on sums held by running CTAs
            }
            action = act;
            last_act = act;
            unit = u;
            // peek ahead: overlapped with the unit about to run
            if (!p1_done) peek_p1 = *reinterpret_cast<volatile unsigned*>(&ctr[kLcP1]);
            if (!sums_ready) peek_sums = *reinterpret_cast<volatile unsigned*>(&ctr[kLcSumD]);
        }
        __syncthreads();
        const int act = action;
        if (act == kActExit) break;
        if (act == kActWait) {
            __nanosleep(200);
            continue;
        }
        if (act == kActF) {
            const int st = int(fit % kLcStages2);
            const uint64_t leaf = fleaf;
            if (tr8 && tid == 0) {
                const unsigned long long w0 = lc_clock();
                mbar_wait(&sm.full[st], (fit / kLcStages2) & 1);
                t_unit[3] += lc_clock() - w0;
            }
            mbar_wait(&sm.full[st], (fit / kLcStages2) & 1);
            if (tid < kL) {  // r'_k exactly as phase 1 formed it
                double rv = sm.u.p2.r[st][0][tid];
                if (mode == kLoop) rv = fma(-alpha, sm.u.p2.r[st][1][tid], rv);
                sm.rin[tid] = static_cast<float>(rv);
            }
            long long c0 = clock64();
            __syncthreads();
            long long c1 = clock64();
            const float* F = sm.u.p2.F[st];
            if (tid < kL) {  // c = F^T r: matvec_t order (apply.cpp:25-35)
                float acc = 0.f;
#pragma unroll 16
                for (int i = 0; i < kL; ++i) acc = fmaf(F[i * kL + tid], sm.rin[i], acc);
                sm.c[tid] = acc;
            }
            __syncthreads();
            long long c2 = clock64();
            {   // y = F c with f64 accumulation (k_leaf_fast's transpose-reduce)
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
                    s.y_loc[leaf * kL + row] = v[0];
                }
            }
            __syncthreads();  // stage consumed
            if (tr12 && tid == 0) {
                const long long c3 = clock64();
                (void)c0;
                t_sub[1] += c2 - c1;
                t_sub[2] += c3 - c2;
            }
            ++fit;
            fleaf += grid;
            const uint64_t nxt = fleaf + uint64_t(kLcStages2 - 1) * grid;  // kLcStages2 leaves ahead
            if (tid == 0 && nxt < K) {
                const long long i0 = clock64();
                issue2(nxt, st);
                if (tr12) t_sub[0] += clock64() - i0;
            }
            continue;
        }
        if (act == kActEpi) {  // |r|^2 over every CTA's phase-1 partial -> r0 / rel / history / stop
            if (warp == 0) {
                double rr2[1];
                sum_partials<1>(s.dpart + kPartLeaf, s.grid_leaf, rr2);
                if (lane == 0) leaf_epilogue(s, mode, rr2[0]);
            }
            __syncthreads();
            continue;
        }
        if (act == kActSum) {  // one 32-leaf group's up-sweep (k_sums_tree level 0)
            sweep_leaves(s, s.D, unit, S0);
            __syncthreads();
            if (tid == 0) atom_add_acq_rel_gpu(&ctr[kLcSumD], 1u);
            continue;
        }
        // kActTile
        const uint64_t pol = policy_evict_last();
        if (unit < n_upper) {  // a tile above the groups: children sums from the group roots
            __shared__ double up_sr[32], up_sc[32];
            const uint64_t m = unit;
            tile_root_sums(s, m, R, dr, up_sr, up_sc);
            if (warp == 0)
                tile_couple(s.F + s.tile_base + m * (kLs * kLs), up_sr[lane], up_sc[lane], sm.ws[0], lane, pol,
                            s.coupled + m * 64);
        } else {  // 16 group-internal tiles, one per warp
            const uint64_t m = n_upper + (unit - n_upper) * 16 + uint64_t(warp);
            if (m < K - 1) {
                const uint64_t l = 2 * m + 1, r = 2 * m + 2;  // heap children
                double a, bb;
                if (l >= K - 1) {
                    a = double(__ldcg(&s.restrict_[(l - (K - 1)) * 64 + lane]));
                    bb = double(__ldcg(&s.restrict_[(r - (K - 1)) * 64 + 32 + lane]));
                } else {
                    a = __ldcg(&s.node_u[l * 32 + lane]);
                    bb = __ldcg(&s.node_v[r * 32 + lane]);
                }
                tile_couple(s.F + s.tile_base + m * (kLs * kLs), a, bb, sm.ws[warp], lane, pol, s.coupled + m * 64);
            }
        }
        __syncthreads();
    }
    if (tr && threadIdx.x == 0) {
        tr[2] = lc_clock();
        tr[3] = fit;
        if (tr8)
            for (int q = 0; q < 4; ++q) tr[4 + q] = t_unit[q];
        if (tr12)
            for (int q = 0; q < 3; ++q) tr[8 + q] = t_sub[q];
        if (tr12) tr[11] = clock64() - clk0;
    }
    // leaving: the last CTA out resets the tickets for the next launch
    if (tid == 0 && atom_add_acq_rel_gpu(&ctr[kLcExit], 1u) == grid - 1)
        for (int q = 0; q < kLcN; ++q) ctr[q] = 0u;
}

}  // namespace hfpg
