// sm_100a kernels of the hot path. One PCG iteration (pcg.cpp:86-119) with the factor
// preconditioner (apply.cpp:79-174) is four launches, all inside one CUDA graph:
//
//   k_spmv    p = z + beta p (fused), Ap = A p on SELL-32, p.Ap and p.p       (csr.cpp:70-79)
//   k_leaf    x += alpha p, r -= alpha Ap, |r|^2; then per leaf: F_k^T r_k, F_k c,
//             Ũ_k^T r_k, Ṽ_k^T r_k (apply stages 1-3) from TMA-staged factors
//   k_coarse  bisection-tree strip sums, tile couplings V(U^T s_r), U(V^T s_c) (stage 4)
//   k_prolong ancestor gather + Ũ_k g_r + Ṽ_k g_c + gate, z, r.z, beta      (stages 5-7)
//
// Accumulator precisions follow the reference apply: F^T r and the restrictions accumulate in
// fp32 (matvec_t, apply.cpp:25-35), F c and the prolongation in f64 (apply.cpp:11-22, 39-50),
// strip sums and gathers in f64; every PCG scalar is f64 (pcg.hpp:14-16).
#pragma once

#include "device_common.cuh"
#include "comm.cuh"

namespace hfpg {

// Device view of the loaded system and factors (pointers fixed at graph build time).
struct DevSys {
    // factors (packed layout, factor_tensor.hpp:18-48)
    const float* F;
    uint64_t n, l, ls, rk, K, D;  // D = log2 K
    uint64_t tile_base, bridge_base, gate_base;
    // operator
    const double* a_diag;
    const unsigned long long* slice_off;  // SELL-32 slices (element offsets, n_slices + 1)
    const uint32_t* sell_cols;
    const double* sell_vals;
    // PCG vectors
    double *x, *r, *z, *ap, *p0, *p1, *y_loc;
    // apply workspace
    float* restrict_;        // K x 2 L_s  (û_k | v̂_k), fp32 as in the reference
    float* coupled;          // M_H x 2 L_s: tile m = [coupled_row (L_s) | coupled_col (L_s)]
    double *node_u, *node_v; // heap-indexed strip sums of subtree roots (2K x L_s)
    unsigned* tree_counters; // 2K arrival counters for the coarse tree
    uint64_t coarse_S;       // subtree width per k_coarse task (power of two)
    uint32_t spmv_stage_bytes; // k_spmv_tma stage capacity (0: use k_spmv)
    uint32_t pspmv_stage_bytes; // k_solve SpMV ring stage (16 slices; 0: direct loads)
    uint32_t spmv_stages;      // k_spmv_tma ring depth (<= 8)
    // reductions / state
    double* partials;
    unsigned* counters;  // [0] spmv, [1] leaf, [2] prolong, [3] simple
    Scalars* sc;
    double* history;
    cudaGraphConditionalHandle cond;
    int use_cond;
    int l2_resident;  // factor tensor small enough to keep in L2 across iterations
    unsigned long long* trace;  // k_solve: %globaltimer at every grid barrier (CTA 0), or null
    unsigned trace_cap;
    int trace_probe;
    // row partition over G ranks (G == 1: the whole system). n, K, D above are this rank's.
    uint32_t G, rank, glog;
    uint64_t n_ghost;               // ghost entries of z, p0, p1 after the n owned rows
    const float* top_tiles;         // the G-1 tiles above the rank subtrees (global heap order)
    float* top_coupled;             // (G-1) x 64: [coupled_row | coupled_col]
    Mailbox* mbox;                  // this rank's mailbox
    Mailbox* const* peer_mbox;      // G mailboxes (device array of pointers)
    double* const* peer_z;          // G z vectors (their ghost regions start at n)
    const uint32_t* send_rows;      // halo: local rows pushed to peers, grouped by peer
    const uint32_t* send_slot;      //       destination ghost slot in that peer
    const unsigned long long* send_off;  // G + 1
    unsigned long long* seq;        // 3 message sequence counters (monotonic across solves)
    // deferred reductions (single-rank factor path): per-CTA partials of the SpMV (p.Ap, p.p),
    // the leaf kernel (|r|^2) and the prolongation (r.z), summed by the next kernel
    int defer;
    double* dpart;
    uint32_t grid_spmv, grid_leaf, grid_prol;
    // k_leaf_coarse (leaf_coarse.cuh) runs apply stages 1-4: r' = r - alpha Ap is then stored by
    // the prolongation (which re-forms it with the same fma) instead of the leaf kernel
    int fused_leaf;
    int bridge_first;  // HFPG_BRIDGE_FIRST=1: the leaf kernel streams the bridges evict_first (A/B)
    int ksolve_pipe;   // k_solve pipelines a CTA's leaves (default; HFPG_KSOLVE_PIPE=0: sequential, A/B)
};
constexpr uint32_t kPartSpmv = 0, kPartLeaf = 2048, kPartProl = 3072, kPartLen = 4096;

enum Mode { kInit = 0, kLoop = 1, kApply = 2 };

__device__ __forceinline__ double* p_cur(const DevSys& s, unsigned long long k) {
    return (k & 1ULL) ? s.p1 : s.p0;
}
__device__ __forceinline__ double* p_prev(const DevSys& s, unsigned long long k) {
    return (k & 1ULL) ? s.p0 : s.p1;
}

// pcg.cpp:97-110 after |r|^2 is known: history, convergence, max_iters.
__device__ __forceinline__ void finish_residual(Scalars* sc, double* history, double rr) {
    const unsigned long long k = sc->k;
    const double rel = sqrt(rr) / sc->r0;
    sc->rel = rel;
    if (history) history[k - 1] = rel;
    sc->hist_len = k;
    if (rel <= sc->rtol) {
        sc->converged = 1;
        sc->status = 0;
        sc->iterations = k;
        sc->done = 1;
    } else if (k == sc->max_iters) {
        sc->iterations = k;
        sc->status = 1;
        sc->done = 1;
    }
}


// ---- row partition (G > 1) helpers -------------------------------------------------------
// SpMV prologue: wait for the last M3 (its z halo rows), beta = rz_{k-1} / rz_{k-2} (k >= 2;
// beta = 0 at k = 1) —
// the same division the single-rank prolong epilogue does (pcg.cpp:115-117) — and the ghost
// entries of the new p (peers' rows this rank reads), p = z + beta p_prev like owned rows.
__device__ __forceinline__ double part_spmv_beta(const DevSys& s, unsigned long long k, const double* pprev,
                                                 double* pnew) {
    __shared__ double sb;
    if (threadIdx.x == 0) {
        // always wait: even at k = 1 (beta = 0) the SpMV reads the z halo rows the peers pushed
        // before their M3 (the init apply's)
        const unsigned long long q3 = s.seq[2];
        mb_wait<2>(s.mbox, s.G, q3);
        sb = k >= 2 ? mb_sum<2>(s.mbox, s.G, q3, 0) / s.sc->rz : 0.0;
    }
    __syncthreads();
    const double beta = sb;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s.n_ghost;
         i += uint64_t(gridDim.x) * blockDim.x)
        pnew[s.n + i] = fma(beta, pprev[s.n + i], s.z[s.n + i]);
    return beta;
}

// The last CTA of a partitioned SpMV: send M1 = {p.Ap, p.p} partials (warp 0).
__device__ __forceinline__ void part_send_m1(const DevSys& s, double pap, double pp) {
    if (threadIdx.x >= 32) return;
    __shared__ double pay[2];
    unsigned long long seq = 0;
    if (threadIdx.x == 0) {
        seq = ++s.seq[0];
        pay[0] = pap;
        pay[1] = pp;
    }
    seq = __shfl_sync(0xffffffffu, seq, 0);
    __syncwarp();
    mb_send<0>(s.peer_mbox, s.G, s.rank, seq, pay, 2);
}

// Single-rank SpMV epilogue (last CTA, thread 0): breakdown test and alpha (pcg.cpp:88-96).
__device__ __forceinline__ void spmv_epilogue(const DevSys& s, unsigned long long k, double pap, double p2) {
    Scalars* sc = s.sc;
    sc->pap = pap;
    sc->pp = p2;
    if (pap < -sc->breakdown_tol * p2 || pap == 0.0) {  // pcg.cpp:90-95
        sc->status = 2;
        sc->breakdown_iter = k;
        sc->iterations = k;
        sc->done = 1;
    } else {
        sc->alpha = sc->rz / pap;
    }
}

// One SELL-32 row: acc += a_q * p(c_q) over W slots in slot (= the reference's column) order,
// products and sums rounded separately (csr.cpp:76 is not FMA-contracted). p(c) = z[c] or, in
// PCG mode, fma(beta, p_prev[c], z[c]) (pcg.cpp:118 recomputed at the gather). Every load of the
// W slots is issued before the first arithmetic, with a fixed trip count: with predicated slots
// ptxas reused one register pair for every gather and serialised the row into W dependent round
// trips to L2 (ncu: 40 us for the 3D 1M SpMV, DFMA stalls on each gather in turn).
template <int W, bool LOOP, bool CG>
__device__ __forceinline__ double sell_row_w(const double* vals, const uint32_t* cols, int lane, const double* z,
                                             const double* pprev, double beta, double acc) {
    uint32_t c[W];
    double zv[W], pv[W], a[W];
#pragma unroll
    for (int q = 0; q < W; ++q) c[q] = cols[q * 32 + lane];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        zv[q] = CG ? __ldcg(&z[c[q]]) : z[c[q]];
        if (LOOP) pv[q] = CG ? __ldcg(&pprev[c[q]]) : pprev[c[q]];
    }
#pragma unroll
    for (int q = 0; q < W; ++q) a[q] = vals[q * 32 + lane];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const double pc = LOOP ? fma(beta, pv[q], zv[q]) : zv[q];
        acc = __dadd_rn(acc, __dmul_rn(a[q], pc));
    }
    return acc;
}
template <bool LOOP, bool CG>
__device__ __forceinline__ double sell_row(const double* vals, const uint32_t* cols, uint64_t w, int lane,
                                           const double* z, const double* pprev, double beta) {
    double acc = 0.0;
    uint64_t j = 0;
    for (; j + 8 <= w; j += 8) acc = sell_row_w<8, LOOP, CG>(vals + j * 32, cols + j * 32, lane, z, pprev, beta, acc);
    vals += j * 32;
    cols += j * 32;
    switch (w - j) {  // uniform per slice
        case 1: return sell_row_w<1, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        case 2: return sell_row_w<2, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        case 3: return sell_row_w<3, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        case 4: return sell_row_w<4, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        case 5: return sell_row_w<5, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        case 6: return sell_row_w<6, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        case 7: return sell_row_w<7, LOOP, CG>(vals, cols, lane, z, pprev, beta, acc);
        default: return acc;
    }
}

// Deferred: beta_k = rz_{k-1} / rz_{k-2} (pcg.cpp:115-117; 0 at k = 1) from the previous
// prolongation's r.z partials. One warp; CTA 0 records rz_{k-1} in the parity slot k & 1 (the
// slot this iteration's leaf kernel reads for alpha, while slot (k-1) & 1 stays readable).
__device__ __forceinline__ double defer_beta(const DevSys& s, unsigned long long k) {
    double rz[1];
    sum_partials<1>(s.dpart + kPartProl, s.grid_prol, rz);
    const double beta = k >= 2 ? rz[0] / s.sc->rzs[(k - 1) & 1] : 0.0;
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
        s.sc->rzs[k & 1] = rz[0];
        s.sc->rz = rz[0];
        s.sc->beta = beta;
    }
    return beta;
}

// ============================================================================================
// SpMV on SELL-32 (slices of 32 rows, column-major inside a slice, padded with (row, 0.0)).
// One thread per row: every load is coalesced and each row accumulates sequentially in the
// reference's column order (csr.cpp:74-77), so ap is bit-identical to the reference spmv.
// PCG mode fuses p = z + beta p_prev (pcg.cpp:118) into the gathers and reduces p.Ap, p.p.
// ============================================================================================
template <int MODE>  // kInit unused; kLoop = PCG, kApply = plain y = A x
__global__ void __launch_bounds__(256) k_spmv(DevSys s, const double* xin, double* yout) {
    if (MODE == kLoop && s.sc->done) return;
    const unsigned long long k = MODE == kLoop ? s.sc->k : 0ULL;
    const double* z = MODE == kLoop ? s.z : xin;
    const double* pp_ = MODE == kLoop ? p_prev(s, k) : nullptr;
    double* pnew = MODE == kLoop ? p_cur(s, k) : nullptr;
    double* y = MODE == kLoop ? s.ap : yout;
    double beta = MODE != kLoop ? 0.0 : s.G > 1 ? part_spmv_beta(s, k, pp_, pnew) : s.sc->beta;
    if (MODE == kLoop && s.defer) {
        __shared__ double sb;
        if (threadIdx.x < 32) sb = defer_beta(s, k);
        __syncthreads();
        beta = sb;
    }
    double v[2] = {0.0, 0.0};
    // persistent grid-stride over rows: one CTA partial (and one fence) per CTA, not per row
    for (uint64_t row = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < s.n;
         row += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t sl = row >> 5, lane = row & 31;
        const uint64_t base = s.slice_off[sl], w = (s.slice_off[sl + 1] - base) >> 5;
        double zr = 0.0, pr = 0.0;
        if (MODE == kLoop) {
            zr = z[row];
            pr = pp_[row];
        }
        const double acc = sell_row<MODE == kLoop, false>(s.sell_vals + base, s.sell_cols + base, w, int(lane), z,
                                                          pp_, beta);
        y[row] = acc;
        if (MODE == kLoop) {
            const double pi = fma(beta, pr, zr);
            pnew[row] = pi;
            v[0] = fma(pi, acc, v[0]);
            v[1] = fma(pi, pi, v[1]);
        }
    }
    if (MODE != kLoop) return;
    if (s.defer) {
        publish_partials<2>(v, s.dpart + kPartSpmv);
        return;
    }
    double tot[2];
    if (grid_reduce_last<2>(v, s.partials, &s.counters[0], tot)) {
        if (s.G > 1) part_send_m1(s, tot[0], tot[1]);
        else if (threadIdx.x == 0) spmv_epilogue(s, k, tot[0], tot[1]);
    }
}

// SpMV, streaming variant: persistent CTAs walk chunks of 8 SELL slices (256 rows), warp-
// specialised. Warp 8 (the producer) reads the chunk's 9 slice offsets into the stage header and
// bulk-copies the chunk's values and column indices (contiguous in SELL order) into a 3-stage
// ring; warps 0-7 (one slice each) copy their slots from the stage into registers, release the
// stage (mbarrier arrive, so the next chunk's copy starts while this one's gathers are still in
// flight), then gather z / p_prev (L1/L2-resident neighbours) and accumulate. No CTA-wide
// barrier inside the loop. Same arithmetic as k_spmv (bit-identical to the reference spmv).
// Used when every chunk fits a stage (host-checked); k_spmv covers the general case.
#ifndef HFPG_SPMV_MINB
#define HFPG_SPMV_MINB 3
#endif
constexpr int kSpmvStages = 3;
constexpr int kSpmvThreads = 288;  // 8 consumer warps + 1 producer warp
constexpr uint32_t kSpmvHdr = 128; // per stage: 9 slice offsets (u64)

// Consumer half of a fixed-width row: slots from the stage into registers, release the stage,
// then the gathers (all issued before the first product) and the exact-order accumulation.
template <int W, bool LOOP>
__device__ __forceinline__ double sell_row_release(const double* vals, const uint32_t* cols, int lane,
                                                   const double* z, const double* pprev, double beta,
                                                   uint64_t* empty) {
    uint32_t c[W];
    double a[W], zv[W], pv[W];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        c[q] = cols[q * 32 + lane];
        a[q] = vals[q * 32 + lane];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty);
#pragma unroll
    for (int q = 0; q < W; ++q) {
        zv[q] = z[c[q]];
        if (LOOP) pv[q] = pprev[c[q]];
    }
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const double pc = LOOP ? fma(beta, pv[q], zv[q]) : zv[q];
        acc = __dadd_rn(acc, __dmul_rn(a[q], pc));
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(kSpmvThreads, HFPG_SPMV_MINB) k_spmv_tma(DevSys s, const double* xin, double* yout) {
    pdl_enter();  // programmatic dependent launch: see device_common.cuh
    if (MODE == kLoop && s.sc->done) return;
    extern __shared__ __align__(128) unsigned char sraw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sraw);
    const uint32_t NS = s.spmv_stages;
    uint64_t* empty = full + NS;
    unsigned char* ring = sraw + 128;
    const uint32_t cap = s.spmv_stage_bytes, stride = cap + kSpmvHdr;
    const unsigned long long k = MODE == kLoop ? s.sc->k : 0ULL;
    const double* z = MODE == kLoop ? s.z : xin;
    const double* pp_ = MODE == kLoop ? p_prev(s, k) : nullptr;
    double* pnew = MODE == kLoop ? p_cur(s, k) : nullptr;
    double* y = MODE == kLoop ? s.ap : yout;
    const bool defer = MODE == kLoop && s.defer;
    double beta = MODE != kLoop || defer ? 0.0 : s.G > 1 ? part_spmv_beta(s, k, pp_, pnew) : s.sc->beta;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t nsl = (s.n + 31) >> 5, nch = (nsl + 7) >> 3;
    if (tid == 0) {
        for (uint32_t q = 0; q < NS; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], 8);
        }
        fence_mbar_init();
    }
    __syncthreads();
    double v[2] = {0.0, 0.0};
    if (warp == 8) {  // producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            uint32_t it = 0;
            for (uint64_t ch = blockIdx.x; ch < nch; ch += gridDim.x, ++it) {
                const int st = int(it % NS);
                if (it >= NS) mbar_wait(&empty[st], ((it / NS) - 1) & 1);
                unsigned char* b = ring + size_t(st) * stride;
                unsigned long long* off = reinterpret_cast<unsigned long long*>(b);
                const uint64_t s0 = ch * 8;
                unsigned long long o[9];
#pragma unroll
                for (int q = 0; q < 9; ++q) o[q] = __ldg(&s.slice_off[s0 + q < nsl ? s0 + q : nsl]);
#pragma unroll
                for (int q = 0; q < 9; ++q) off[q] = o[q];
                const uint64_t ne = o[8] - o[0];
                mbar_expect_tx(&full[st], uint32_t(ne * 12));
                tma_load_1d(b + kSpmvHdr, s.sell_vals + o[0], uint32_t(ne * 8), &full[st], pol);
                tma_load_1d(b + kSpmvHdr + ne * 8, s.sell_cols + o[0], uint32_t(ne * 4), &full[st], pol);
            }
        }
    } else {  // consumers: warp w takes slice 8 ch + w
        if (defer) {  // beta from the previous prolongation's r.z partials, while the producer streams
            __shared__ double sb;
            if (warp == 0) sb = defer_beta(s, k);
            named_bar_sync(1, 256);
            beta = sb;
        }
        uint32_t it = 0;
        for (uint64_t ch = blockIdx.x; ch < nch; ch += gridDim.x, ++it) {
            const int st = int(it % NS);
            const uint64_t sl = ch * 8 + warp, row = sl * 32 + lane;
            double zr = 0.0, pr = 0.0;
            if (MODE == kLoop && row < s.n) {
                zr = z[row];
                pr = pp_[row];
            }
            mbar_wait(&full[st], (it / NS) & 1);
            const unsigned char* b = ring + size_t(st) * stride;
            const unsigned long long* off = reinterpret_cast<const unsigned long long*>(b);
            double acc = 0.0;
            if (sl < nsl) {
                const uint64_t e0 = off[0], ne = off[8] - e0, b0 = off[warp] - e0, w = (off[warp + 1] - off[warp]) >> 5;
                const double* vals = reinterpret_cast<const double*>(b + kSpmvHdr) + b0;
                const uint32_t* cols = reinterpret_cast<const uint32_t*>(b + kSpmvHdr + ne * 8) + b0;
                constexpr bool LP = MODE == kLoop;
                switch (w) {  // uniform per slice
                    case 1: acc = sell_row_release<1, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 2: acc = sell_row_release<2, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 3: acc = sell_row_release<3, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 4: acc = sell_row_release<4, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 5: acc = sell_row_release<5, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 6: acc = sell_row_release<6, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 7: acc = sell_row_release<7, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    case 8: acc = sell_row_release<8, LP>(vals, cols, lane, z, pp_, beta, &empty[st]); break;
                    default:
                        acc = sell_row<LP, false>(vals, cols, w, lane, z, pp_, beta);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[st]);
                }
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            }
            if (row < s.n) {
                y[row] = acc;
                if (MODE == kLoop) {
                    const double pi = fma(beta, pr, zr);
                    pnew[row] = pi;
                    v[0] = fma(pi, acc, v[0]);
                    v[1] = fma(pi, pi, v[1]);
                }
            }
        }
    }
    if (MODE != kLoop) return;
    if (s.defer) {
        publish_partials<2>(v, s.dpart + kPartSpmv);
        return;
    }
    double tot[2];
    if (grid_reduce_last<2>(v, s.partials, &s.counters[0], tot)) {
        if (s.G > 1) part_send_m1(s, tot[0], tot[1]);
        else if (threadIdx.x == 0) spmv_epilogue(s, k, tot[0], tot[1]);
    }
}

// x += alpha p, r -= alpha Ap for one row (pcg.cpp:97-98); returns the updated r.
__device__ __forceinline__ double update_row(const DevSys& s, const double* p, double alpha,
                                             uint64_t i) {
    s.x[i] = fma(alpha, p[i], s.x[i]);
    const double rn = fma(-alpha, s.ap[i], s.r[i]);
    s.r[i] = rn;
    return rn;
}

// Last-CTA epilogue of the leaf kernels: |r|^2 -> r0 (init) or rel/history/stop (loop).
__device__ __forceinline__ void leaf_epilogue(const DevSys& s, int mode, double rr) {
    Scalars* sc = s.sc;
    if (mode == kInit) {
        sc->r0 = sqrt(rr);
        if (sc->r0 == 0.0) {  // pcg.cpp:73-79
            sc->converged = 1;
            sc->status = 0;
            sc->iterations = 0;
            sc->done = 1;
        }
    } else {
        finish_residual(sc, s.history, rr);
    }
}

// ============================================================================================
// Leaf kernel, fast path (L = 128, L_s = 32): persistent, one CTA of 512 threads per SM.
// Per leaf the 64 KB F_k and the 32 KB bridge pair (Ũ_k | Ṽ_k, contiguous in the packed
// layout) arrive by cp.async.bulk into a 2-stage shared-memory ring (192 KB); the next leaf's
// copy is in flight while this one computes, so the kernel streams the factor tensor at HBM
// rate. F_k is read from HBM once and from shared memory twice (F^T r, then F c).
// ============================================================================================
constexpr int kL = 128, kLs = 32;
constexpr int kLeafThreads = 512;
constexpr uint32_t kFBytes = kL * kL * 4, kBBytes = 2 * kL * kLs * 4;
struct LeafSmem {
    float F[2][kL * kL];
    float B[2][2 * kL * kLs];
    double vec[2][4][kL];  // r_k, Ap_k, p_k, x_k of the staged leaf (the fused PCG update)
    float rin[kL];
    float c[kL];
    uint64_t full[2];
};


// Partitioned leaf prologue: wait for every rank's M1, alpha = rz_{k-1} / p.Ap with the rank-
// ordered totals, breakdown test (pcg.cpp:88-96). Every CTA computes the same; CTA 0 records
// the scalars. Returns false (all CTAs) on breakdown.
__device__ __forceinline__ bool part_leaf_alpha(const DevSys& s, double& alpha) {
    __shared__ double sa;
    __shared__ int sok;
    if (threadIdx.x == 0) {
        const unsigned long long q1 = s.seq[0], q3 = s.seq[2];
        mb_wait<0>(s.mbox, s.G, q1);
        const double pap = mb_sum<0>(s.mbox, s.G, q1, 0), p2 = mb_sum<0>(s.mbox, s.G, q1, 1);
        const double rz = mb_sum<2>(s.mbox, s.G, q3, 0);  // rz_{k-1}: awaited by the SpMV
        Scalars* sc = s.sc;
        const bool brk = pap < -sc->breakdown_tol * p2 || pap == 0.0;
        sok = !brk;
        sa = rz / pap;
        if (blockIdx.x == 0) {
            sc->pap = pap;
            sc->pp = p2;
            sc->alpha = sa;
            sc->rz = rz;  // the next SpMV's beta denominator
            if (brk) {
                sc->status = 2;
                sc->breakdown_iter = sc->k;
                sc->iterations = sc->k;
                sc->done = 1;
            }
        }
    }
    __syncthreads();
    alpha = sa;
    return sok != 0;
}

constexpr uint64_t kCoarseS0 = 32;  // leaves per bottom subtree (group) of the up-sweep

__global__ void __launch_bounds__(kLeafThreads, 1) k_leaf_fast(DevSys s, int mode,
                                                               const double* rin_ext) {
    pdl_enter();  // programmatic dependent launch: see device_common.cuh
    if (mode != kApply && s.sc->done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    LeafSmem& sm = *reinterpret_cast<LeafSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const bool defer = mode == kLoop && s.defer;
    double alpha = mode == kLoop && !defer ? s.sc->alpha : 0.0;
    if (s.G > 1 && mode == kLoop && !part_leaf_alpha(s, alpha)) return;
    const double* rsrc = mode == kApply ? rin_ext : s.r;
    const double* pcur = mode == kLoop ? p_cur(s, s.sc->k) : nullptr;
    const uint64_t K = s.K;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const int nvec = mode == kLoop ? 4 : 1;
    const uint32_t stage_bytes = kFBytes + kBBytes + nvec * kL * 8;

    if (tid == 0) {
        mbar_init(&sm.full[0], 1);
        mbar_init(&sm.full[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // One elected thread streams a whole leaf: F_k (4 x 16 KB), Ũ_k|Ṽ_k (2 x 16 KB) and the
    // leaf's slices of the PCG vectors, all completing on the stage's mbarrier.
    auto issue = [&](uint64_t leaf, int st) {
        mbar_expect_tx(&sm.full[st], stage_bytes);
        const float* f = s.F + leaf * (kL * kL);
        const float* b = s.F + s.bridge_base + leaf * (2 * kL * kLs);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            tma_load_1d(&sm.F[st][q * kL * kL / 4], f + q * kL * kL / 4, kFBytes / 4,
                        &sm.full[st], pol_stream);
        // bridges: evict_last, meant for the prolongation's reverse walk to find the last-
        // streamed ones in L2. Measured (r02): no reuse — the prolongation reads all 268 MB of
        // bridges from DRAM, and the solve time is the same with evict_first (HFPG_BRIDGE_FIRST=1,
        // 224.9 vs 223.6 ms); an 80 MB persisting carve-out plus an access-policy window over
        // the bridge tail did not help either (229-230 ms: the carve-out slows the SpMV).
        const uint64_t pol_b = s.bridge_first ? pol_stream : pol_keep;
        tma_load_1d(&sm.B[st][0], b, kBBytes / 2, &sm.full[st], pol_b);
        tma_load_1d(&sm.B[st][kL * kLs], b + kL * kLs, kBBytes / 2, &sm.full[st], pol_b);
        tma_load_1d(sm.vec[st][0], rsrc + leaf * kL, kL * 8, &sm.full[st], pol_keep);
        if (mode == kLoop) {
            tma_load_1d(sm.vec[st][1], s.ap + leaf * kL, kL * 8, &sm.full[st], pol_stream);
            tma_load_1d(sm.vec[st][2], pcur + leaf * kL, kL * 8, &sm.full[st], pol_stream);
            tma_load_1d(sm.vec[st][3], s.x + leaf * kL, kL * 8, &sm.full[st], pol_stream);
        }
    };
    if (tid == 0 && blockIdx.x < K) issue(blockIdx.x, 0);
    if (defer) {  // alpha from the SpMV's partials while the first leaf streams in
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
        if (sbrk) {  // no update; let the issued copy land before the CTA exits
            if (blockIdx.x < K) mbar_wait(&sm.full[0], 0);
            return;
        }
    }

    double rr = 0.0;
    const int lane = tid & 31, warp = tid >> 5;
    uint32_t it = 0;
    for (uint64_t leaf = blockIdx.x; leaf < K; leaf += gridDim.x, ++it) {
        const int st = it & 1;
        if (tid == 0 && leaf + gridDim.x < K) issue(leaf + gridDim.x, st ^ 1);
        mbar_wait(&sm.full[st], (it >> 1) & 1);
        if (tid < kL) {
            const uint64_t i = leaf * kL + tid;
            double rv = sm.vec[st][0][tid];
            if (mode == kLoop) {  // pcg.cpp:97-98, fused
                s.x[i] = fma(alpha, sm.vec[st][2][tid], sm.vec[st][3][tid]);
                rv = fma(-alpha, sm.vec[st][1][tid], rv);
                s.r[i] = rv;
            }
            rr = fma(rv, rv, rr);
            sm.rin[tid] = static_cast<float>(rv);  // apply.cpp:90
        }
        __syncthreads();
        const float* F = sm.F[st];
        const float* B = sm.B[st];
        // c = F^T r and the restrictions Ũ^T r, Ṽ^T r: one thread per output, a sequential
        // fp32 FMA chain over the 128 rows — the exact operation order of the reference's
        // vectorised matvec_t (apply.cpp:25-35), so c and û, v̂ are bit-identical to it.
        if (tid < kL) {
            const int j = tid;
            float acc = 0.f;
#pragma unroll 16
            for (int i = 0; i < kL; ++i) acc = fmaf(F[i * kL + j], sm.rin[i], acc);
            sm.c[j] = acc;
        } else if (tid < kL + 2 * kLs) {
            const int o = tid - kL;
            const float* Bo = B + (o >> 5) * (kL * kLs) + (o & 31);
            float acc = 0.f;
#pragma unroll 16
            for (int i = 0; i < kL; ++i) acc = fmaf(Bo[i * kLs], sm.rin[i], acc);
            s.restrict_[leaf * (2 * kLs) + o] = acc;
        }
        __syncthreads();
        {   // y = F c: products of two floats are exact in f64 and the reference accumulates
            // them in f64 (matvec_add_double, apply.cpp:39-50); warp w owns rows 8w..8w+7, lane
            // l columns 4l..4l+3, then a transpose-reduce across lanes (order differs only at
            // the f64 rounding level)
            const float4 c4 = reinterpret_cast<const float4*>(sm.c)[lane];
            const double c0 = c4.x, c1 = c4.y, c2 = c4.z, c3 = c4.w;
            double v[8];
#pragma unroll
            for (int rI = 0; rI < 8; ++rI) {
                const float4 f4 = reinterpret_cast<const float4*>(F + (8 * warp + rI) * kL)[lane];
                v[rI] = fma(double(f4.w), c3, fma(double(f4.z), c2, fma(double(f4.y), c1, double(f4.x) * c0)));
            }
            // transpose-reduce 8 rows x 32 lanes: after xor 16/8/4 each lane holds one row's
            // partial over 4 lanes; xor 2/1 finish it.
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
        __syncthreads();
    }
    if (mode == kApply) return;
    double v[1] = {rr}, tot[1];
    if (s.defer) {  // |r|^2 is finished by k_tiles_all's CTA 0 (rel, history, stop)
        publish_partials<1>(v, s.dpart + kPartLeaf);
        return;
    }
    if (grid_reduce_last<1>(v, s.partials, &s.counters[1], tot) && tid == 0) {
        if (s.G > 1) s.sc->rr_loc = tot[0];  // reduced across ranks after the strip sums (M2)
        else leaf_epilogue(s, mode, tot[0]);
    }
}

// Leaf kernel, generic path (any L, L_s): one CTA per leaf, factors read from global.
__global__ void __launch_bounds__(256) k_leaf_generic(DevSys s, int mode, const double* rin_ext) {
    if (mode != kApply && s.sc->done) return;
    extern __shared__ float gsm[];
    const uint64_t L = s.l, ls = s.ls, leaf = blockIdx.x;
    float* rin = gsm;
    float* c = gsm + L;
    const double alpha = mode == kLoop ? s.sc->alpha : 0.0;
    const double* rsrc = mode == kApply ? rin_ext : s.r;
    const double* pcur = mode == kLoop ? p_cur(s, s.sc->k) : nullptr;
    double rr = 0.0;
    for (uint64_t t = threadIdx.x; t < L; t += blockDim.x) {
        const uint64_t i = leaf * L + t;
        const double rv = mode == kLoop ? update_row(s, pcur, alpha, i) : rsrc[i];
        rr = fma(rv, rv, rr);
        rin[t] = static_cast<float>(rv);
    }
    __syncthreads();
    const float* F = s.F + leaf * L * L;
    for (uint64_t j = threadIdx.x; j < L; j += blockDim.x) {  // c = F^T r (fp32)
        float acc = 0.f;
        for (uint64_t i = 0; i < L; ++i) acc = fmaf(F[i * L + j], rin[i], acc);
        c[j] = acc;
    }
    for (uint64_t o = threadIdx.x; o < 2 * ls; o += blockDim.x) {  // restriction (fp32)
        const float* B = s.F + s.bridge_base + leaf * 2 * L * ls + (o >= ls ? L * ls : 0);
        const uint64_t col = o % ls;
        float acc = 0.f;
        for (uint64_t i = 0; i < L; ++i) acc = fmaf(B[i * ls + col], rin[i], acc);
        s.restrict_[leaf * 2 * ls + o] = acc;
    }
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < L; i += blockDim.x) {  // y = F c (f64)
        double acc = 0.0;
        for (uint64_t j = 0; j < L; ++j) acc = fma(double(F[i * L + j]), double(c[j]), acc);
        s.y_loc[leaf * L + i] = acc;
    }
    if (mode == kApply) return;
    double v[1] = {rr}, tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[1], tot) && threadIdx.x == 0)
        leaf_epilogue(s, mode, tot[0]);
}

// ============================================================================================
// Coarse stage (apply stage 4, apply.cpp:110-138) over the bisection tree in heap order
// (tile m = heap node m; its rows are the left child's leaves, its columns the right child's).
// s_r(m) = Σ û over the left child, s_c(m) = Σ v̂ over the right child: an f64 up-sweep. Each
// CTA owns an aligned subtree of up to 32 leaves (or of 32 subtree roots at higher levels),
// computes its internal tiles, publishes its root sums, and the last-arriving CTA of each
// group of siblings carries on one level up — one launch covers the whole tree (k_coarse, the
// generic path, below); the fast path splits it into k_sums_tree and k_tiles_all.
// ============================================================================================

// ============================================================================================
// Coarse stage, graph path (also the row-partitioned solve): strip sums, then every tile.
// ============================================================================================
// One tile (L_s = 32, rank 16) per warp, without shared staging of the factors: lanes q < 16
// read column q of U (lanes 16 + q: of V) from L2 and run the fp32 chain
// coef = sum_p U[p][q] float(s_r[p]) in p order (matvec_t); lane j then forms
// coupled_col[j] = float(sum_q V[j][q] coef_r[q]) and coupled_row[j] = float(sum_q U[j][q]
// coef_c[q]) with exact f64 products summed in q order (matvec, apply.cpp:121-138) — bit-
// identical to the reference. f32<->f64 conversions run at 15.6/clk/SM (measured), so the strip
// sums are cast once per tile and each coefficient is converted once and broadcast through
// shared memory. T = the tile's U (V = T + 512); out = [coupled_row (32) | coupled_col (32)].
struct alignas(16) TileScratch {
    float fr[32], fc[32];
    double coef[32];
};
// `sums(sr_p, sc_p)` yields the strip sums; it runs after the tile's loads are issued, so loads
// it makes itself (k_coarse_coop) are in flight together with the tile's.
struct TileRegs {
    float cv[32];
    float4 u4[4], v4[4];
};
__device__ __forceinline__ void tile_load(const float* T, int lane, uint64_t pol, TileRegs& t) {
    const float* colp = T + (lane < 16 ? 0 : kLs * 16) + (lane & 15);
#pragma unroll
    for (int p = 0; p < 32; ++p) t.cv[p] = ldg_f32_hint(colp + p * 16, pol);
    const float4* U = reinterpret_cast<const float4*>(T) + lane * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        t.u4[i] = ldg_hint(U + i, pol);
        t.v4[i] = ldg_hint(U + 128 + i, pol);
    }
}
__device__ __forceinline__ void tile_finish(const TileRegs& t, double sr_p, double sc_p, TileScratch& ws, int lane,
                                            float* out);
template <class Sums>
__device__ __forceinline__ void tile_couple_f(const float* T, Sums sums, TileScratch& ws, int lane, uint64_t pol,
                                              float* out) {
    TileRegs t;
    tile_load(T, lane, pol, t);
    double sr_p, sc_p;
    sums(sr_p, sc_p);
    tile_finish(t, sr_p, sc_p, ws, lane, out);
}
__device__ __forceinline__ void tile_finish(const TileRegs& t, double sr_p, double sc_p, TileScratch& ws, int lane,
                                            float* out) {
    const float* cv = t.cv;
    const float4* u4 = t.u4;
    const float4* v4 = t.v4;
    ws.fr[lane] = float(sr_p);  // apply.cpp:121-124 (strip sums cast to T)
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
    __stcg(&out[32 + lane], float(acc_c));
    __stcg(&out[lane], float(acc_r));
    __syncwarp();
}
__device__ __forceinline__ void tile_couple(const float* T, double sr_p, double sc_p, TileScratch& ws,
                                            int lane, uint64_t pol, float* out) {
    tile_couple_f(T, [&](double& a, double& b) { a = sr_p; b = sc_p; }, ws, lane, pol, out);
}
// Row-only variant (k_coarse_coop): a tile's 1,024 floats are loaded once, lane = row (8
// float4 loads instead of 8 + 32 scalar column loads), and the coefficient chains read the
// column view from a per-warp shared copy. The copy is XOR-swizzled by 16-byte chunk
// (chunk ^ ((row >> 1) & 3)), so both the row stores and the column reads are conflict-free;
// V sits 16 floats after U's 512 so the two half-warps' columns use different banks. Same
// arithmetic as tile_finish, so the couplings are bit-identical.
struct TileRows {
    float4 u4[4], v4[4];
};
constexpr int kTileColFloats = 2 * 512 + 16;
__device__ __forceinline__ int tile_sw(int row, int col) {  // swizzled offset of (row, col < 16)
    return row * 16 + 4 * ((col >> 2) ^ ((row >> 1) & 3)) + (col & 3);
}
__device__ __forceinline__ void tile_load_rows(const float* T, int lane, uint64_t pol, TileRows& t) {
    const float4* U = reinterpret_cast<const float4*>(T) + lane * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        t.u4[i] = ldg_hint(U + i, pol);
        t.v4[i] = ldg_hint(U + 128 + i, pol);
    }
}
__device__ __forceinline__ void tile_finish_rows(const TileRows& t, double sr_p, double sc_p, TileScratch& ws,
                                                 float* col, int lane, float* out) {
    float* cu = col;
    float* cvv = col + 512 + 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        *reinterpret_cast<float4*>(cu + tile_sw(lane, 4 * i)) = t.u4[i];
        *reinterpret_cast<float4*>(cvv + tile_sw(lane, 4 * i)) = t.v4[i];
    }
    ws.fr[lane] = float(sr_p);  // apply.cpp:121-124 (strip sums cast to T)
    ws.fc[lane] = float(sc_p);
    __syncwarp();
    const float* cb = lane < 16 ? cu : cvv;
    const int q = lane & 15;
    const float4* st4 = reinterpret_cast<const float4*>(lane < 16 ? ws.fr : ws.fc);
    float coef = 0.f;
#pragma unroll
    for (int p4 = 0; p4 < 8; ++p4) {
        const float4 sv = st4[p4];
        coef = fmaf(cb[tile_sw(4 * p4 + 0, q)], sv.x, coef);
        coef = fmaf(cb[tile_sw(4 * p4 + 1, q)], sv.y, coef);
        coef = fmaf(cb[tile_sw(4 * p4 + 2, q)], sv.z, coef);
        coef = fmaf(cb[tile_sw(4 * p4 + 3, q)], sv.w, coef);
    }
    ws.coef[lane] = double(coef);  // [0,16): U^T s_r, [16,32): V^T s_c
    __syncwarp();
    double acc_c = 0.0, acc_r = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float uu[4] = {t.u4[i].x, t.u4[i].y, t.u4[i].z, t.u4[i].w};
        const float vv[4] = {t.v4[i].x, t.v4[i].y, t.v4[i].z, t.v4[i].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int qq = 4 * i + k;
            acc_c += double(vv[k]) * ws.coef[qq];
            acc_r += double(uu[k]) * ws.coef[16 + qq];
        }
    }
    __stcg(&out[32 + lane], float(acc_c));
    __stcg(&out[lane], float(acc_r));
    __syncwarp();
}

// Strip sums (apply.cpp:110-120) over this rank's bisection tree in one launch.
// Level 0: a CTA takes an aligned subtree of S0 = min(K, 32) leaves; warp w owns 4 of the 64 sum
// columns (u: 0-31, v: 32-63), lane q holds leaf q, and a shuffle butterfly builds the pairwise
// f64 up-sweep (after the step of distance d every lane holds its 2d-group's sum = left + right
// child, the heap sums node[u] = node[2u+1] + node[2u+2]); the first lane of each group writes
// the node. Upper levels: the last CTA to finish (one arrival counter) sweeps groups of up to 512
// subtree roots — lane q first sums its 16 contiguous roots pairwise in registers, then the same
// butterfly — so the tree costs two dependent steps, not one per 32-ary level. (Groups of 512
// chain through further arrival counters only above K = 16384 leaves.) Partitioned: the CTA that
// finishes the rank's root sends M2 = {|r|^2 partial, root sums}.
constexpr int kSumsThreads = 512;
constexpr uint64_t kSumsGroup = 512;  // upper-level group: 32 lanes x 16 nodes

// Pairwise up-sweep of M = 2^m nodes at depth dlo, positions [t M, (t+1) M), by one CTA
// (V = max(1, M / 32) nodes per lane): writes every internal node (depths dlo-1 .. dlo-m).
// Level 0 (leaves, V = 1): all 4 columns of the lane's leaf in one float4 load.
__device__ __forceinline__ void sweep_leaves(const DevSys& s, uint64_t dlo, uint64_t t, uint64_t M) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int side = warp >> 3, c0 = 4 * (warp & 7);
    double* node = side ? s.node_v : s.node_u;
    const int lanes = int(M);
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (lane < lanes) {
        const float4 f = __ldcg(reinterpret_cast<const float4*>(&s.restrict_[(t * M + lane) * 64 + 32 * side + c0]));
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    }
    for (int l2 = 0; (1 << l2) < lanes; ++l2) {
        const int d = 1 << l2;
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] += __shfl_xor_sync(0xffffffffu, v[c], d);
        if (lane < lanes && (lane & (2 * d - 1)) == 0) {
            const uint64_t dd = dlo - (l2 + 1);
            const uint64_t p = ((t * M) >> (l2 + 1)) + uint64_t(lane >> (l2 + 1));
            double* o = &node[((1ULL << dd) - 1 + p) * 32 + c0];
            __stcg(reinterpret_cast<double2*>(o), make_double2(v[0], v[1]));
            __stcg(reinterpret_cast<double2*>(o + 2), make_double2(v[2], v[3]));
        }
    }
}

// Upper levels, coalesced: lane = column (256-byte rows of node sums per load / store). A block
// of B consecutive nodes is summed pairwise in one lane's registers, one column per lane;
// the <= 16 block roots of a group meet in shared memory for the last levels. (The previous
// lane-per-node layout issued 32-sector loads and stores and took 10 us for 256 roots on the
// single SM that runs the upper levels.)
template <int B>
__device__ __forceinline__ double sweep_block(double* node, uint64_t dlo, uint64_t p0, int lane) {
    double v[B];
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = __ldcg(&node[((1ULL << dlo) - 1 + p0 + i) * 32 + lane]);
#pragma unroll
    for (int l2 = 0; (1 << l2) < B; ++l2) {
#pragma unroll
        for (int i = 0; i < (B >> (l2 + 1)); ++i) {
            v[i] = v[2 * i] + v[2 * i + 1];  // heap sum: left child + right child
            const uint64_t d = dlo - (l2 + 1), pos = (p0 >> (l2 + 1)) + i;
            __stcg(&node[((1ULL << d) - 1 + pos) * 32 + lane], v[i]);
        }
    }
    return v[0];
}
// All internal nodes above M (a power of two <= kSumsGroup) nodes at depth dlo, positions
// [t M, (t+1) M). Called by every thread of a kSumsThreads CTA: warps 0-7 the u sums, 8-15 v.
__device__ __forceinline__ void sweep_group(const DevSys& s, uint64_t dlo, uint64_t t, uint64_t M) {
    __shared__ double roots[2][16][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int side = warp >> 3, j = warp & 7;
    double* node = side ? s.node_v : s.node_u;
    const uint64_t B = M >= 256 ? 32 : (M >= 8 ? M / 8 : 1), nb = M / B;
    int logB = 0;
    while ((1ULL << logB) < B) ++logB;
    for (uint64_t b = j; b < nb; b += 8) {
        const uint64_t p0 = t * M + b * B;
        double r;
        switch (B) {
            case 1: r = sweep_block<1>(node, dlo, p0, lane); break;
            case 2: r = sweep_block<2>(node, dlo, p0, lane); break;
            case 4: r = sweep_block<4>(node, dlo, p0, lane); break;
            case 8: r = sweep_block<8>(node, dlo, p0, lane); break;
            case 16: r = sweep_block<16>(node, dlo, p0, lane); break;
            default: r = sweep_block<32>(node, dlo, p0, lane); break;
        }
        roots[side][b][lane] = r;
    }
    __syncthreads();
    if (j == 0 && nb > 1) {  // the levels above the blocks (nb <= 16 block roots)
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = uint64_t(i) < nb ? roots[side][i][lane] : 0.0;
        const uint64_t dblk = dlo - logB, q0 = t * nb;  // block roots: depth dblk, positions q0 + i
        uint64_t cnt = nb;
#pragma unroll
        for (int l2 = 0; l2 < 4; ++l2) {
            if (cnt < 2) break;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (uint64_t(i) < cnt / 2) {
                    v[i] = v[2 * i] + v[2 * i + 1];
                    const uint64_t d = dblk - (l2 + 1), pos = (q0 >> (l2 + 1)) + i;
                    __stcg(&node[((1ULL << d) - 1 + pos) * 32 + lane], v[i]);
                }
            }
            cnt /= 2;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSumsThreads) k_sums_tree(DevSys s, int mode) {
    if (mode != kApply && s.sc->done) return;
    __shared__ int last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t K = s.K, D = s.D;
    const uint64_t S0 = K < kCoarseS0 ? K : kCoarseS0, R = K / S0;
    int logS0 = 0;
    while ((1ULL << logS0) < S0) ++logS0;
    // level 0: subtrees of S0 leaves, dealt round-robin
    for (uint64_t task = blockIdx.x; task < R; task += gridDim.x) sweep_leaves(s, D, task, S0);
    // single rank: no levels above the group roots — k_tiles_all's upper tiles sum the roots
    // they need themselves (tile_root_sums), so there is no arrival hop or serial sweep here
    if (s.G == 1) return;
    // upper levels: groups of up to 512 nodes; the last CTA of each level continues
    uint64_t dlo = D - logS0, cnt = R;  // current level: cnt nodes at depth dlo
    unsigned* counter = s.tree_counters;
    unsigned arrivals = gridDim.x;  // CTAs that report into this level's counter
    uint64_t t = blockIdx.x;
    while (true) {
        // the CTA's node writes are ordered before thread 0's release by the barrier; thread 0's
        // acq_rel arrival also acquires the other CTAs' writes for the whole CTA (no SC fences:
        // MEMBAR.SC.GPU from every warp cost more than the sweep itself)
        __syncthreads();
        if (dlo == 0) break;  // the rank's root is done
        if (tid == 0) {
            const unsigned old = atom_add_acq_rel_gpu(counter, 1u);
            last = (old == arrivals - 1);
            if (last) *counter = 0u;
        }
        __syncthreads();
        if (!last) return;
        // this CTA is the last of its level: sweep the next level's groups (all of them if
        // they fit one group, else chain once more per group of 512)
        const uint64_t M = cnt < kSumsGroup ? cnt : kSumsGroup, ng = cnt / M;
        int logM = 0;
        while ((1ULL << logM) < M) ++logM;
        for (uint64_t g = 0; g < ng; ++g) sweep_group(s, dlo, g, M);
        dlo -= logM;
        cnt = ng;
        ++counter;
        arrivals = 1;
        t = 0;
    }
    (void)t;
    // partitioned: the CTA that wrote the root sends M2 (rank root = node 0)
    if (s.G > 1) {
        if (warp == 0) {
            __shared__ double pay[kM2Len];
            unsigned long long seq = 0;
            if (lane == 0) {
                seq = ++s.seq[1];
                pay[0] = mode == kApply ? 0.0 : s.sc->rr_loc;
                pay[1] = 0.0;
            }
            pay[2 + lane] = __ldcg(&s.node_u[lane]);
            pay[34 + lane] = __ldcg(&s.node_v[lane]);
            seq = __shfl_sync(0xffffffffu, seq, 0);
            __syncwarp();
            mb_send<1>(s.peer_mbox, s.G, s.rank, seq, pay, kM2Len);
        }
    }
}

// Tile couplings (apply.cpp:121-138): every tile of the rank's tree in parallel, one warp each,
// dealt across CTAs first (tile t -> CTA t mod grid); children sums from the node arrays (leaf
// children: the restrictions). Partitioned: CTA 0 first waits for every rank's M2, finishes the
// residual bookkeeping with the rank-ordered |r|^2 (r0 at init, rel / history / stop in the
// loop — pcg.cpp:73-112) and computes the G-1 top tiles from the rank-root sums (same pairwise
// order as a single-rank up-sweep), identically on every rank.
// Pairwise (heap-order) sum of n (a power of two) consecutive nodes at depth d, lane = column:
// blocks of 8 in registers, block sums merged through a binary-counter stack (the same tree).
__device__ __forceinline__ double pairwise_nodes(const double* node, uint64_t d, uint64_t p0, uint64_t n, int lane) {
    const double* base = node + ((1ULL << d) - 1 + p0) * 32 + lane;
    if (n <= 8) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (uint64_t(i) < n) v[i] = __ldcg(base + i * 32);
#pragma unroll
        for (int w = 1; w < 8; w *= 2)
#pragma unroll
            for (int i = 0; i + w < 8; i += 2 * w)
                if (uint64_t(i + w) < n) v[i] = v[i] + v[i + w];
        return v[0];
    }
    double stack[24];
    int top = 0;
    for (uint64_t b = 0; b < n / 8; ++b) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldcg(base + (b * 8 + i) * 32);
#pragma unroll
        for (int w = 1; w < 8; w *= 2)
#pragma unroll
            for (int i = 0; i + w < 8; i += 2 * w) v[i] = v[i] + v[i + w];
        double x = v[0];
        for (uint64_t c = b + 1; (c & 1) == 0; c >>= 1) x = stack[--top] + x;
        stack[top++] = x;
    }
    return stack[0];
}
// The strip sums of tile m < R - 1 (above the 32-leaf groups) from the group roots, by all 8
// warps of the CTA: each sums an aligned eighth of each child's roots pairwise, warp 0 merges the
// eight partials pairwise — the heap-order tree of the up-sweep, so the sums equal the node sums
// a full sweep would have stored. All threads call it (contains block barriers).
constexpr int kTileRootWarps = 8;
__device__ __forceinline__ void tile_root_sums(const DevSys& s, uint64_t m, uint64_t R, uint64_t dr,
                                               double* sr_out, double* sc_out) {
    __shared__ double part[2][kTileRootWarps][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int d = 0;
    while ((2ULL << d) <= m + 1) ++d;
    const uint64_t wg = R >> d, g0 = (m + 1 - (1ULL << d)) * wg, W = wg / 2;  // W roots per child
    const uint64_t per = W >= kTileRootWarps ? W / kTileRootWarps : 1;
    const uint64_t nw = W >= kTileRootWarps ? kTileRootWarps : 1;
    if (uint64_t(wid) < nw) {
        part[0][wid][lane] = pairwise_nodes(s.node_u, dr, g0 + wid * per, nw == 1 ? W : per, lane);
        part[1][wid][lane] = pairwise_nodes(s.node_v, dr, g0 + W + wid * per, nw == 1 ? W : per, lane);
    }
    __syncthreads();
    if (wid == 0) {
        double u[kTileRootWarps], v[kTileRootWarps];
#pragma unroll
        for (int q = 0; q < kTileRootWarps; ++q) {
            u[q] = uint64_t(q) < nw ? part[0][q][lane] : 0.0;
            v[q] = uint64_t(q) < nw ? part[1][q][lane] : 0.0;
        }
#pragma unroll
        for (int w = 1; w < kTileRootWarps; w *= 2)
#pragma unroll
            for (int q = 0; q + w < kTileRootWarps; q += 2 * w)
                if (uint64_t(q + w) < nw) {
                    u[q] = u[q] + u[q + w];
                    v[q] = v[q] + v[q + w];
                }
        sr_out[lane] = u[0];
        sc_out[lane] = v[0];
    }
    __syncthreads();
}

constexpr int kTilesThreads = 256;
// MINB = resident CTAs per SM the register budget is fitted to (2: 98 registers; 4: 64)
template <int MINB>
__global__ void __launch_bounds__(kTilesThreads, MINB) k_tiles_all(DevSys s, int mode) {
    if (mode != kApply && s.sc->done) return;
    __shared__ TileScratch ws[kTilesThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t pol = policy_evict_last();
    if (s.defer && mode != kApply && blockIdx.x == 0 && wid == 0) {  // |r|^2 of the leaf kernel
        double rr[1];
        sum_partials<1>(s.dpart + kPartLeaf, s.grid_leaf, rr);
        if (lane == 0) leaf_epilogue(s, mode, rr[0]);  // r0 (init) or rel / history / stop
    }
    if (s.G > 1 && blockIdx.x == 0) {
        __shared__ int stop;
        __shared__ unsigned long long q2s;
        if (threadIdx.x == 0) {
            const unsigned long long q2 = s.seq[1];
            mb_wait<1>(s.mbox, s.G, q2);
            q2s = q2;
            stop = 0;
            if (mode != kApply) {
                const double rr = mb_sum<1>(s.mbox, s.G, q2, 0);
                if (mode == kInit) leaf_epilogue(s, kInit, rr);
                else finish_residual(s.sc, s.history, rr);
                stop = s.sc->done;
            }
        }
        __syncthreads();
        for (unsigned t = unsigned(wid); !stop && t + 1 < s.G; t += kTilesThreads / 32) {
            // top tile t over the rank-root tree (its leaves: heap nodes G-1 .. 2G-2 = ranks);
            // strip sums of its children: pairwise sums of the covered ranks' roots
            const unsigned G = s.G;
            const int par = int(q2s & 1);
            double sum[2];
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
                const unsigned c = 2 * t + 1 + sd;  // left child (u sums) / right child (v sums)
                unsigned dc = 0;
                while ((2u << dc) <= c + 1) ++dc;
                const unsigned span = G >> dc, a = (c + 1 - (1u << dc)) * span;
                double acc[kMaxRanksDev];
                for (unsigned i = 0; i < span; ++i) acc[i] = __ldcg(&s.mbox->m2[par][a + i][2 + 32 * sd + lane]);
                for (unsigned w2 = 1; w2 < span; w2 *= 2)
                    for (unsigned i = 0; i + w2 < span; i += 2 * w2) acc[i] += acc[i + w2];
                sum[sd] = acc[0];
            }
            tile_couple(s.top_tiles + uint64_t(t) * (kLs * kLs), sum[0], sum[1], ws[wid], lane, pol,
                        s.top_coupled + uint64_t(t) * 64);
        }
    }
    const uint64_t K = s.K, G = gridDim.x;
    const uint64_t S0 = K < kCoarseS0 ? K : kCoarseS0, R = K / S0;
    int logS0 = 0;
    while ((1ULL << logS0) < S0) ++logS0;
    const uint64_t dr = s.D - logS0;  // depth of the group roots
    // single rank: the R - 1 tiles above the 32-leaf groups first, one per CTA at a time, their
    // children's sums from the group roots by all 8 warps (tile_root_sums); then the group-internal
    // tiles, one per warp. Partitioned ranks: every tile from the node sums of k_sums_tree.
    const uint64_t first = s.G == 1 ? R - 1 : 0;
    if (s.G == 1) {
        __shared__ double up_sr[32], up_sc[32];
        for (uint64_t m = blockIdx.x; m + 1 < R; m += G) {
            TileRegs t;  // warp 0's tile loads in flight during the root sums
            if (wid == 0) tile_load(s.F + s.tile_base + m * (kLs * kLs), lane, pol, t);
            tile_root_sums(s, m, R, dr, up_sr, up_sc);
            if (wid == 0) tile_finish(t, up_sr[lane], up_sc[lane], ws[0], lane, s.coupled + m * 64);
        }
    }
    for (uint64_t m = first + uint64_t(wid) * G + blockIdx.x; m < K - 1; m += G * (kTilesThreads / 32)) {
        const uint64_t l = 2 * m + 1, r = 2 * m + 2;  // children (heap)
        double a, bb;
        if (l >= K - 1) {
            a = double(__ldcg(&s.restrict_[(l - (K - 1)) * 64 + lane]));
            bb = double(__ldcg(&s.restrict_[(r - (K - 1)) * 64 + 32 + lane]));
        } else {
            a = __ldcg(&s.node_u[l * 32 + lane]);
            bb = __ldcg(&s.node_v[r * 32 + lane]);
        }
        tile_couple(s.F + s.tile_base + m * (kLs * kLs), a, bb, ws[wid], lane, pol, s.coupled + m * 64);
    }
}

// Coarse stage in one cooperative launch (single rank, K >= 64): replaces k_sums_tree +
// k_tiles_all and the launch between them.
//   A. CTA t < R sums group t's 32 restrictions pairwise into the group roots (the up-sweep's
//      depth-dr nodes; nothing below them is stored — nothing reads it), then every CTA arrives
//      on one counter (release).
//   B. the group-internal tiles, one per warp: their children's strip sums are pairwise sums of
//      at most 16 consecutive leaves' restrictions, read directly (the same left + right tree
//      as the up-sweep, so bit-identical to the node sums k_sums_tree stores).
//   C. the R - 1 tiles above the groups, after waiting for the counter to reach the grid size
//      (acquire; the launch is cooperative, so every CTA is resident and the wait cannot hang),
//      exactly as k_tiles_all does them (tile_root_sums + tile_couple).
// CTA 0 finishes |r|^2 (deferred mode) only after the wait, i.e. after every CTA has read
// sc->done at entry, so all CTAs agree on whether to run. The last CTA out resets the counters.
template <int N>
__device__ __forceinline__ double leaf_run_sum(const float* p) {  // p: first leaf's column, stride 64
    double v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = double(__ldcg(p + i * 64));
#pragma unroll
    for (int w = 1; w < N; w *= 2)
#pragma unroll
        for (int i = 0; i + w < N; i += 2 * w) v[i] = v[i] + v[i + w];  // heap sum: left + right
    return v[0];
}
__device__ __forceinline__ double child_strip_sum(const DevSys& s, uint64_t c, int side, int lane) {
    const uint64_t K = s.K, D = s.D;
    if (c >= K - 1) return double(__ldcg(&s.restrict_[(c - (K - 1)) * 64 + 32 * side + lane]));
    int dc = 0;
    while ((2ULL << dc) <= c + 1) ++dc;
    const uint64_t n = 1ULL << (D - dc), leaf0 = (c + 1 - (1ULL << dc)) * n;
    const float* p = s.restrict_ + leaf0 * 64 + 32 * side + lane;
    switch (n) {
        case 2: return leaf_run_sum<2>(p);
        case 4: return leaf_run_sum<4>(p);
        case 8: return leaf_run_sum<8>(p);
        default: return leaf_run_sum<16>(p);
    }
}

__global__ void __launch_bounds__(kTilesThreads, 2) k_coarse_coop(DevSys s, int mode) {
    pdl_enter();  // programmatic dependent launch: see device_common.cuh
    if (mode != kApply && s.sc->done) return;  // every CTA reads the same value (see above)
    __shared__ TileScratch ws[kTilesThreads / 32];
    __shared__ double half[2][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t pol = policy_evict_last();
    const uint64_t K = s.K, G = gridDim.x, R = K / kCoarseS0;
    const uint64_t dr = s.D - 5;  // depth of the group roots (32 = 2^5 leaves per group)
    unsigned* ctr = s.counters + 12;
    // hfpg_set_trace(h, >= 8 grid): %globaltimer at entry / after A / after B / after the wait /
    // after C / exit, thread 0 of every CTA (tools/coarse_trace.py)
    unsigned long long* tr = (s.trace && s.trace_cap >= 8 * gridDim.x) ? s.trace + 8 * blockIdx.x : nullptr;
    auto stamp = [&](int q) {
        if (tr && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            tr[q] = t;
        }
    };
    stamp(0);
    // A. group roots: warps 0-3 = (side, half of the group), lane = column; warps 4-7 go
    // straight to their tiles (B), so part of the tile-factor burst starts at entry
    if (wid < 4) {
        for (uint64_t g = blockIdx.x; g < R; g += G) {
            const int side = wid >> 1, h = wid & 1;
            const double r = leaf_run_sum<16>(s.restrict_ + (g * 32 + 16 * h) * 64 + 32 * side + lane);
            if (h) half[side][lane] = r;
            named_bar_sync(1, 128);
            if (!h) (side ? s.node_v : s.node_u)[((1ULL << dr) - 1 + g) * 32 + lane] = r + half[side][lane];
            named_bar_sync(1, 128);  // the roots are stored (and half[] free) before the next group / the release
        }
        if (threadIdx.x == 0) atom_add_acq_rel_gpu(&ctr[0], 1u);
    }
    stamp(1);
    // B. group-internal tiles
    __shared__ __align__(16) float colv[kTilesThreads / 32][kTileColFloats];
    for (uint64_t m = (R - 1) + uint64_t(wid) * G + blockIdx.x; m < K - 1; m += G * (kTilesThreads / 32)) {
        TileRows t;  // the tile's loads and its children's sums in flight together
        tile_load_rows(s.F + s.tile_base + m * (kLs * kLs), lane, pol, t);
        const double a = child_strip_sum(s, 2 * m + 1, 0, lane);
        const double bb = child_strip_sum(s, 2 * m + 2, 1, lane);
        tile_finish_rows(t, a, bb, ws[wid], colv[wid], lane, s.coupled + m * 64);
    }
    // C. the tiles above the groups (and CTA 0's |r|^2 epilogue) once every group root is out
    stamp(2);
    if (blockIdx.x + 1 < R || blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&ctr[0]) : "memory");
            } while (v < G);
        }
        __syncthreads();
        stamp(3);
        __shared__ double up_sr[32], up_sc[32];
        for (uint64_t m = blockIdx.x; m + 1 < R; m += G) {
            TileRegs t;  // warp 0's tile loads in flight during the root sums
            if (wid == 0) tile_load(s.F + s.tile_base + m * (kLs * kLs), lane, pol, t);
            tile_root_sums(s, m, R, dr, up_sr, up_sc);
            if (wid == 0) tile_finish(t, up_sr[lane], up_sc[lane], ws[0], lane, s.coupled + m * 64);
        }
        if (s.defer && mode != kApply && blockIdx.x == 0 && wid == 0) {  // |r|^2 of the leaf kernel
            double rr[1];
            sum_partials<1>(s.dpart + kPartLeaf, s.grid_leaf, rr);
            if (lane == 0) leaf_epilogue(s, mode, rr[0]);  // r0 (init) or rel / history / stop
        }
    }
    stamp(4);
    __syncthreads();
    stamp(5);
    if (threadIdx.x == 0 && atom_add_acq_rel_gpu(&ctr[1], 1u) == G - 1) {
        ctr[0] = 0u;
        ctr[1] = 0u;
    }
}

constexpr int kCoarseThreads = 256;

// Shared-memory bytes of k_coarse for a given L_s and subtree width Smax.
__host__ __device__ inline size_t coarse_smem_bytes(uint64_t ls, uint64_t Smax) {
    return (2 * (2 * Smax - 1) * ls) * sizeof(double) + (Smax - 1) * ls * ls * sizeof(float) +
           Smax * 2 * ls * sizeof(float) + (kCoarseThreads / 32) * ls * sizeof(float);
}

__global__ void __launch_bounds__(kCoarseThreads) k_coarse(DevSys s, int mode) {
    if (mode != kApply && s.sc->done) return;
    extern __shared__ __align__(128) unsigned char craw[];
    const uint64_t ls = s.ls, rk = s.rk, Smax = s.coarse_S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* SU = reinterpret_cast<double*>(craw);        // (2Smax-1) x ls, local heap order
    double* SV = SU + (2 * Smax - 1) * ls;
    float* T = reinterpret_cast<float*>(SV + (2 * Smax - 1) * ls);  // tile slot u: U|V
    float* Rst = T + (Smax - 1) * ls * ls;                // bottom restrictions (level 0)
    float* coef = Rst + Smax * 2 * ls;                    // per warp: rk + rk
    __shared__ uint64_t bar;
    __shared__ int last;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol_keep = policy_evict_last();  // tiles + restrictions are re-read every iteration
    uint32_t phase = 0;

    uint64_t task = blockIdx.x;
    uint64_t dlo = s.D;  // depth of this task's bottom layer
    for (int level = 0;; ++level) {
        const uint64_t cnt = 1ULL << dlo;
        const uint64_t S = cnt < Smax ? cnt : Smax;
        int logS = 0;
        while ((1ULL << logS) < S) ++logS;
        const uint64_t dr = dlo - logS;  // depth of this task's root
        const uint64_t g0 = (1ULL << dlo) - 1 + task * S;  // heap index of the first bottom node
        // Stage the subtree's tile factors (one bulk copy per depth: the 2^ld tiles of a depth
        // are contiguous in heap order) and its bottom layer, on one mbarrier.
        const bool tiles_tma = (s.tile_base & 3) == 0;  // 16-byte aligned tile section
        if (tid == 0) {
            uint32_t bytes = 0;
            if (tiles_tma)
                for (int ld = 0; ld < logS; ++ld) bytes += (1u << ld) * uint32_t(ls * ls * 4);
            bytes += level == 0 ? uint32_t(S * 2 * ls * 4) : uint32_t(2 * S * ls * 8);
            mbar_expect_tx(&bar, bytes);
            for (int ld = 0; tiles_tma && ld < logS; ++ld) {
                const uint64_t m0 = (1ULL << (dr + ld)) - 1 + task * (1ULL << ld);
                tma_load_1d(T + ((1ULL << ld) - 1) * ls * ls, s.F + s.tile_base + m0 * ls * ls,
                            uint32_t((1ULL << ld) * ls * ls * 4), &bar, pol_keep);
            }
            if (level == 0) {
                tma_load_1d(Rst, s.restrict_ + task * S * 2 * ls, uint32_t(S * 2 * ls * 4), &bar,
                            pol_keep);
            } else {
                tma_load_1d(SU + (S - 1) * ls, s.node_u + g0 * ls, uint32_t(S * ls * 8), &bar, pol_keep);
                tma_load_1d(SV + (S - 1) * ls, s.node_v + g0 * ls, uint32_t(S * ls * 8), &bar, pol_keep);
            }
        }
        if (!tiles_tma)
            for (int ld = 0; ld < logS; ++ld) {
                const uint64_t m0 = (1ULL << (dr + ld)) - 1 + task * (1ULL << ld);
                for (uint64_t e = tid; e < (1ULL << ld) * ls * ls; e += blockDim.x)
                    T[((1ULL << ld) - 1) * ls * ls + e] = s.F[s.tile_base + m0 * ls * ls + e];
            }
        mbar_wait(&bar, phase);
        phase ^= 1;
        if (level == 0) {
            for (uint64_t e = tid; e < S * ls; e += blockDim.x) {
                const uint64_t q = e / ls, j = e % ls, u = S - 1 + q;
                SU[u * ls + j] = double(Rst[q * 2 * ls + j]);
                SV[u * ls + j] = double(Rst[q * 2 * ls + ls + j]);
            }
        }
        __syncthreads();
        for (int ld = logS - 1; ld >= 0; --ld) {  // f64 up-sweep inside the subtree
            const uint64_t u0 = (1ULL << ld) - 1, nu = 1ULL << ld;
            for (uint64_t e = tid; e < nu * ls; e += blockDim.x) {
                const uint64_t u = u0 + e / ls, j = e % ls;
                SU[u * ls + j] = SU[(2 * u + 1) * ls + j] + SU[(2 * u + 2) * ls + j];
                SV[u * ls + j] = SV[(2 * u + 1) * ls + j] + SV[(2 * u + 2) * ls + j];
            }
            __syncthreads();
        }
        // Internal tiles, one warp each: coupled_col = V (U^T float(s_r)) and
        // coupled_row = U (V^T float(s_c)); U^T / V^T accumulate in fp32 over p ascending
        // (matvec_t), V c / U c' in f64 then cast (matvec), as apply.cpp:125-137.
        float* cr_ = coef + warp * 2 * rk;
        float* cc_ = cr_ + rk;
        for (uint64_t u = warp; u + 1 < S; u += blockDim.x / 32) {
            int ld = 0;
            while ((2ULL << ld) <= u + 1) ++ld;
            const uint64_t m = (1ULL << (dr + ld)) - 1 + task * (1ULL << ld) + (u + 1 - (1ULL << ld));
            const float* U = T + u * ls * ls;
            const float* V = U + ls * rk;
            const double* sr = SU + (2 * u + 1) * ls;
            const double* sc = SV + (2 * u + 2) * ls;
            for (uint64_t q = lane; q < rk; q += 32) {
                float a = 0.f, b = 0.f;
                for (uint64_t p = 0; p < ls; ++p) {
                    a = fmaf(U[p * rk + q], float(sr[p]), a);
                    b = fmaf(V[p * rk + q], float(sc[p]), b);
                }
                cr_[q] = a;
                cc_[q] = b;
            }
            __syncwarp();
            for (uint64_t j = lane; j < ls; j += 32) {
                double a = 0.0, b = 0.0;
                for (uint64_t q = 0; q < rk; ++q) {
                    a = fma(double(V[j * rk + q]), double(cr_[q]), a);
                    b = fma(double(U[j * rk + q]), double(cc_[q]), b);
                }
                s.coupled[m * 2 * ls + ls + j] = float(a);
                s.coupled[m * 2 * ls + j] = float(b);
            }
            __syncwarp();
        }
        if (dr == 0) return;  // the root tile is done
        {   // publish the subtree root's sums for the next level
            const uint64_t g = (1ULL << dr) - 1 + task;
            for (uint64_t j = tid; j < ls; j += blockDim.x) {
                s.node_u[g * ls + j] = SU[j];
                s.node_v[g * ls + j] = SV[j];
            }
        }
        const uint64_t cnt2 = 1ULL << dr;
        const uint64_t S2 = cnt2 < Smax ? cnt2 : Smax;
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            int logS2 = 0;
            while ((1ULL << logS2) < S2) ++logS2;
            const uint64_t parent = (1ULL << (dr - logS2)) - 1 + task / S2;
            const unsigned t = atomicAdd(&s.tree_counters[parent], 1u);
            last = (t == S2 - 1);
            if (last) s.tree_counters[parent] = 0u;
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        // generic-proxy writes of other CTAs (node sums) must be visible to the async proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        task /= S2;
        dlo = dr;
    }
}

// ============================================================================================
// Prolongation kernels: apply stages 5-7. The f64 gather of leaf k sums coupled_row over the
// ancestors whose left half holds k and coupled_col over those whose right half holds it, in
// tile order (root first), exactly the order of apply.cpp:140-154.
// ============================================================================================
__device__ __forceinline__ void prolong_epilogue(const DevSys& s, int mode, double rz) {
    Scalars* sc = s.sc;
    if (mode == kInit) {
        sc->rz = rz;  // pcg.cpp:84
        sc->beta = 0.0;
        sc->k = 1;
        if (sc->max_iters == 0) {
            sc->iterations = 0;
            sc->status = 1;
            sc->done = 1;
        }
    } else {
        sc->beta = rz / sc->rz;  // pcg.cpp:115-117
        sc->rz = rz;
        sc->k += 1;
    }
    if (s.use_cond) cudaGraphSetConditional(s.cond, sc->done ? 0u : 1u);
}

__device__ __forceinline__ bool prolong_skip(const DevSys& s, int mode) {
    if (mode == kApply || !s.sc->done) return false;
    if (blockIdx.x == 0 && threadIdx.x == 0 && s.use_cond) cudaGraphSetConditional(s.cond, 0u);
    return true;
}


// Partitioned prolong epilogue (last CTA, all threads): push the halo rows of z into the
// peers' ghost slots, send M3 = {r.z partial}, then the iteration bookkeeping (beta is formed by
// the next SpMV from the rank-ordered r.z totals).
__device__ __forceinline__ void part_prolong_epilogue(const DevSys& s, int mode, double rz_loc) {
    const uint64_t nsend = s.send_off[s.G];
    for (uint64_t i = threadIdx.x; i < nsend; i += blockDim.x) {
        unsigned q = 0;
        while (s.send_off[q + 1] <= i) ++q;
        s.peer_z[q][s.n + s.send_slot[i]] = __ldcg(&s.z[s.send_rows[i]]);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < 32) {
        __shared__ double pay[2];
        unsigned long long seq = 0;
        if (threadIdx.x == 0) {
            seq = ++s.seq[2];
            pay[0] = rz_loc;
            pay[1] = 0.0;
        }
        seq = __shfl_sync(0xffffffffu, seq, 0);
        __syncwarp();
        mb_send<2>(s.peer_mbox, s.G, s.rank, seq, pay, 2);
    }
    if (threadIdx.x == 0) {
        Scalars* sc = s.sc;
        if (mode == kInit) {
            sc->beta = 0.0;
            sc->k = 1;
            if (sc->max_iters == 0) {
                sc->iterations = 0;
                sc->status = 1;
                sc->done = 1;
            }
        } else {
            sc->k += 1;
        }
        if (s.use_cond) cudaGraphSetConditional(s.cond, sc->done ? 0u : 1u);
    }
}

// Prolongation, fast path: one warp per leaf, no shared-memory staging and no block
// barriers. Leaves are walked in REVERSE order: the leaf kernel streamed the bridges with an
// evict_last policy, so the ones it read last are still in L2 here. Per leaf a warp
//   1. loads the epilogue operands of its 128 rows (lane L: rows L + 32t) and the ancestor
//      gather (lane j: coupled_row / coupled_col component j of every ancestor),
//   2. streams Ũ_k | Ṽ_k as 128-bit loads, two 16-row chunks in flight, 8 lanes per row,
//      exact f64 products summed in f64 (matvec_add_double, apply.cpp:156-166),
//   3. finishes z = y_loc + Ũ g_r + Ṽ g_c + gate r / a + shift r (apply.cpp:169-173).
constexpr int kMaxDepth = 20;  // K <= 2^20 leaves (N <= 134M at L = 128)
constexpr int kProlWarps = 8;

__global__ void __launch_bounds__(256, 2) k_prolong_fast(DevSys s, int mode, const double* rin_ext,
                                                         double* zout) {
    if (prolong_skip(s, mode)) return;
    __shared__ double su[kProlWarps][kL], sv[kProlWarps][kL];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t K = s.K, D = s.D;
    const double* rsrc = mode == kApply ? rin_ext : s.r;
    double* zdst = mode == kApply ? zout : s.z;
    const double shift = s.sc->shift;
    const int l8 = lane & 7, rsub = lane >> 3;
    double rz = 0.0;
    for (uint64_t w = uint64_t(blockIdx.x) * kProlWarps + wid; w < K; w += uint64_t(gridDim.x) * kProlWarps) {
        const uint64_t leaf = K - 1 - w;
        const uint64_t base = leaf * kL;
        // (1) ancestor gather, all loads issued up front
        // ancestor at depth d: heap node (K + leaf) >> (D - d), minus one; the leaf sits in its
        // column half iff bit D-1-d of the leaf index is set -> offset 32 in the tile's pair
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
        // f64 gathers in tile order, root first (apply.cpp:140-154): lane j ends with
        // g_r[j] (rows halves) and g_c[j] (column halves). Partitioned: the top tiles (depth <
        // log2 G) come first and are the same for every leaf of the rank.
        double gr = 0.0, gc = 0.0;
        for (uint32_t d = 0; d < s.glog; ++d) {
            const uint32_t t = ((s.G + s.rank) >> (s.glog - d)) - 1u, right = (s.rank >> (s.glog - 1 - d)) & 1u;
            const double gv = double(__ldcg(&s.top_coupled[t * 64u + right * 32u + lane]));
            if (right) gc += gv;
            else gr += gv;
        }
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
        // (2) bridges: chunk c = rows 16c..16c+15; lane (rsub, l8) covers rows 16c + 4i + rsub;
        //     two chunks (8 KB per warp) in flight
        const float4* Bu = reinterpret_cast<const float4*>(s.F + s.bridge_base + leaf * (2 * kL * kLs));
        const float4* Bv = Bu + kL * kLs / 4;
        float4 ua[4], va[4], ub[4], vb[4];
        auto load_chunk = [&](int c, float4 (&u)[4], float4 (&v)[4]) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = 16 * c + 4 * i + rsub;
                u[i] = ldg_stream(Bu + row * (kLs / 4) + l8);
                v[i] = ldg_stream(Bv + row * (kLs / 4) + l8);
            }
        };
        auto do_chunk = [&](int c, const float4 (&u)[4], const float4 (&v)[4]) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double au = fma(double(u[i].w), g4[3], fma(double(u[i].z), g4[2],
                            fma(double(u[i].y), g4[1], double(u[i].x) * g4[0])));
                double av = fma(double(v[i].w), h4[3], fma(double(v[i].z), h4[2],
                            fma(double(v[i].y), h4[1], double(v[i].x) * h4[0])));
                au += __shfl_xor_sync(0xffffffffu, au, 4);
                au += __shfl_xor_sync(0xffffffffu, au, 2);
                au += __shfl_xor_sync(0xffffffffu, au, 1);
                av += __shfl_xor_sync(0xffffffffu, av, 4);
                av += __shfl_xor_sync(0xffffffffu, av, 2);
                av += __shfl_xor_sync(0xffffffffu, av, 1);
                if (l8 == 0) {
                    su[wid][16 * c + 4 * i + rsub] = au;
                    sv[wid][16 * c + 4 * i + rsub] = av;
                }
            }
        };
        load_chunk(0, ua, va);
#pragma unroll 1
        for (int c = 0; c < 8; c += 2) {
            load_chunk(c + 1, ub, vb);
            do_chunk(c, ua, va);
            if (c + 2 < 8) load_chunk(c + 2, ua, va);
            do_chunk(c + 1, ub, vb);
        }
        double yl[4], rv[4], ad[4];
        float gt[4];
        const bool form_r = mode == kLoop && s.fused_leaf;  // r' = r - alpha Ap (pcg.cpp:98) lands here
        const double alpha = form_r ? s.sc->alpha : 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint64_t i = base + lane + 32 * t;
            yl[t] = __ldcg(&s.y_loc[i]);
            rv[t] = __ldcg(&rsrc[i]);
            if (form_r) {
                rv[t] = fma(-alpha, __ldcg(&s.ap[i]), rv[t]);
                s.r[i] = rv[t];
            }
            ad[t] = __ldg(&s.a_diag[i]);
            gt[t] = __ldg(&s.F[s.gate_base + i]);
        }
        __syncwarp();
        // (3) epilogue, lane L owns rows L + 32t (coalesced)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int row = lane + 32 * t;
            double y = yl[t];
            y += su[wid][row];
            y += sv[wid][row];
            y += double(gt[t]) * rv[t] / ad[t] + shift * rv[t];
            zdst[base + row] = y;
            rz = fma(rv[t], y, rz);
        }
        __syncwarp();
    }
    if (mode == kApply) return;
    double v[1] = {rz}, tot[1];
    if (s.defer) {  // r.z is summed by the next SpMV (beta); CTA 0 keeps the books
        publish_partials<1>(v, s.dpart + kPartProl);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            Scalars* sc = s.sc;
            if (mode == kInit) {
                sc->beta = 0.0;
                sc->k = 1;
                if (sc->max_iters == 0) {
                    sc->iterations = 0;
                    sc->status = 1;
                    sc->done = 1;
                }
            } else {
                sc->k += 1;
            }
            if (s.use_cond) cudaGraphSetConditional(s.cond, sc->done ? 0u : 1u);
        }
        return;
    }
    if (grid_reduce_last<1>(v, s.partials, &s.counters[2], tot)) {
        if (s.G > 1) part_prolong_epilogue(s, mode, tot[0]);
        else if (threadIdx.x == 0) prolong_epilogue(s, mode, tot[0]);
    }
}


// Prolongation, TMA ring (the default fast path): one persistent CTA per SM, four producer warps
// and sixteen consumer warps. Per leaf a producer streams Ũ_k | Ṽ_k (32 KB) and the leaf's
// epilogue operands (y_loc, r, diag(A), Ap, gate: 4.5 KB) by cp.async.bulk into a 6-stage
// shared-memory ring, then gathers the leaf's ancestor corrections g_r | g_c into the stage
// (one L2 round trip; the four producers keep four gathers in flight, one producer alone was
// gather-latency bound at 1.9 us per leaf) and arrives on the stage's full barrier; five leaves
// stay in flight while the consumers compute one, which is what
// k_prolong_fast's register-staged loads (two 4 KB chunks per warp) could not sustain; sixteen
// consumer warps (eight rows each) hide the F2F / f64 / shuffle latencies (eight were issue-
// latency bound at 0.34 IPC per scheduler). The
// consumer arithmetic is k_prolong_fast's, lane for lane (same 8-lanes-per-row float4 split, same
// f64 fma order and xor tree), so z is bit-identical to it; only the r.z partial's summation
// order differs (rows are owned per warp here).
constexpr int kPtStages = 6;
constexpr int kPtCons = 16;  // consumer warps: warp w owns rows kPtRows w .. kPtRows w + kPtRows - 1
constexpr int kPtRows = kL / kPtCons;
constexpr int kPtProd = 4;  // producer warps: warp kPtCons + j stages the leaves k = j (mod kPtProd)
constexpr int kPtThreads = (kPtCons + kPtProd) * 32;
struct ProlSmem {
    float B[kPtStages][2 * kL * kLs];  // Ũ_k | Ṽ_k
    double vec[kPtStages][4][kL];       // y_loc, r, diag(A), Ap (form_r only)
    float gate[kPtStages][kL];
    double g[kPtStages][2 * kLs];       // g_r | g_c, rounded to fp32 as apply.cpp:154 does
    uint64_t full[kPtStages], empty[kPtStages];
};

__global__ void __launch_bounds__(kPtThreads, 1) k_prolong_tma(DevSys s, int mode, const double* rin_ext,
                                                               double* zout) {
    pdl_enter();  // programmatic dependent launch: see device_common.cuh
    if (prolong_skip(s, mode)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    ProlSmem& sm = *reinterpret_cast<ProlSmem*>(smem_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t K = s.K, D = s.D, grid = gridDim.x;
    const double* rsrc = mode == kApply ? rin_ext : s.r;
    double* zdst = mode == kApply ? zout : s.z;
    const bool form_r = mode == kLoop && s.fused_leaf;  // r' = r - alpha Ap (pcg.cpp:98) lands here
    if (threadIdx.x == 0) {
        for (int q = 0; q < kPtStages; ++q) {
            mbar_init(&sm.full[q], 1 + 32);  // the producer's expect_tx arrival + one per gathering lane
            mbar_init(&sm.empty[q], kPtCons);
        }
        fence_mbar_init();
    }
    __syncthreads();
    double rz = 0.0;
    if (wid >= kPtCons) {  // ---- producer warps: several ancestor gathers in flight at once
        const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
        const uint32_t bytes = 2 * kL * kLs * 4 + (form_r ? 4 : 3) * kL * 8 + kL * 4;
        const uint32_t Du = uint32_t(D);
        uint32_t k = uint32_t(wid - kPtCons);
        for (uint64_t w = blockIdx.x + uint64_t(k) * grid; w < K; w += kPtProd * grid, k += kPtProd) {
            const int st = int(k % kPtStages);
            if (k >= kPtStages) mbar_wait(&sm.empty[st], (k / kPtStages - 1) & 1);
            const uint64_t leaf = K - 1 - w, base = leaf * kL;  // reverse walk: see k_prolong_fast
            if (lane == 0) {
                mbar_expect_tx(&sm.full[st], bytes);
                const float* b = s.F + s.bridge_base + leaf * (2 * kL * kLs);
                tma_load_1d(&sm.B[st][0], b, kL * kLs * 4, &sm.full[st], pol_stream);
                tma_load_1d(&sm.B[st][kL * kLs], b + kL * kLs, kL * kLs * 4, &sm.full[st], pol_stream);
                tma_load_1d(sm.vec[st][0], s.y_loc + base, kL * 8, &sm.full[st], pol_stream);
                tma_load_1d(sm.vec[st][1], rsrc + base, kL * 8, &sm.full[st], pol_keep);
                tma_load_1d(sm.vec[st][2], s.a_diag + base, kL * 8, &sm.full[st], pol_keep);
                if (form_r) tma_load_1d(sm.vec[st][3], s.ap + base, kL * 8, &sm.full[st], pol_stream);
                tma_load_1d(sm.gate[st], s.F + s.gate_base + base, kL * 4, &sm.full[st], pol_keep);
            }
            // ancestor gather (apply.cpp:140-154), exactly k_prolong_fast's: all loads up front,
            // partitioned top tiles first, then root -> leaf in f64
            const uint32_t hl = uint32_t(K + leaf), lf = uint32_t(leaf);
            float ga[kMaxDepth];
#pragma unroll
            for (int d = 0; d < kMaxDepth; ++d) {
                ga[d] = 0.f;
                if (uint32_t(d) < Du) {
                    const uint32_t m = (hl >> (Du - d)) - 1u, right = (lf >> (Du - 1 - d)) & 1u;
                    ga[d] = __ldcg(&s.coupled[m * 64u + right * 32u + lane]);
                }
            }
            double gr = 0.0, gc = 0.0;
            for (uint32_t d = 0; d < s.glog; ++d) {
                const uint32_t t = ((s.G + s.rank) >> (s.glog - d)) - 1u, right = (s.rank >> (s.glog - 1 - d)) & 1u;
                const double gv = double(__ldcg(&s.top_coupled[t * 64u + right * 32u + lane]));
                if (right) gc += gv;
                else gr += gv;
            }
#pragma unroll
            for (int d = 0; d < kMaxDepth; ++d)
                if (uint32_t(d) < Du) {
                    if ((lf >> (Du - 1 - d)) & 1u) gc += double(ga[d]);
                    else gr += double(ga[d]);
                }
            sm.g[st][lane] = double(float(gr));
            sm.g[st][kLs + lane] = double(float(gc));
            mbar_arrive(&sm.full[st]);  // every lane releases its own gather writes
        }
    } else {  // ---- consumer warps
        const int l8 = lane & 7, rsub = lane >> 3;
        const double shift = s.sc->shift;
        const double alpha = form_r ? s.sc->alpha : 0.0;
        uint32_t k = 0;
        for (uint64_t w = blockIdx.x; w < K; w += grid, ++k) {
            const int st = int(k % kPtStages);
            mbar_wait(&sm.full[st], (k / kPtStages) & 1);
            const uint64_t base = (K - 1 - w) * kL;
            double g4[4], h4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                g4[q] = sm.g[st][4 * l8 + q];
                h4[q] = sm.g[st][kLs + 4 * l8 + q];
            }
            const float4* Bu = reinterpret_cast<const float4*>(sm.B[st]);
            const float4* Bv = Bu + kL * kLs / 4;
            // rows 8w + rsub (i = 0) and 8w + 4 + rsub (i = 1): four partial dot products per lane
            // (Ũ, Ṽ x two rows), reduced over the row's 8 lanes by a transpose-reduce — 4 f64
            // shuffles instead of 12, and the same pairing tree as the xor butterfly
            // ((a0+a4)+(a2+a6))+((a1+a5)+(a3+a7)), so each sum is bit-identical to k_prolong_fast's
            static_assert(kPtRows == 8, "two 4-row passes per warp");
            double v[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int row = kPtRows * wid + 4 * i + rsub;
                const float4 u = Bu[row * (kLs / 4) + l8], w4 = Bv[row * (kLs / 4) + l8];
                v[2 * i] = fma(double(u.w), g4[3], fma(double(u.z), g4[2], fma(double(u.y), g4[1], double(u.x) * g4[0])));
                v[2 * i + 1] = fma(double(w4.w), h4[3], fma(double(w4.z), h4[2], fma(double(w4.y), h4[1], double(w4.x) * h4[0])));
            }
            {
                const bool hi = lane & 4;  // bit 2 keeps row pass i = 1
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double send = hi ? v[q] : v[q + 2];
                    const double keep = hi ? v[q + 2] : v[q];
                    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
            }
            {
                const bool hi = lane & 2;  // bit 1 keeps the Ṽ sum
                const double send = hi ? v[0] : v[1];
                const double keep = hi ? v[1] : v[0];
                v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            const double vsum = __shfl_xor_sync(0xffffffffu, v[0], 2);  // lanes with bit 1 clear: + the Ṽ sum
            if ((lane & 3) == 0) {  // epilogue (apply.cpp:169-173): row 8w + 4 (bit 2) + rsub
                const int row = kPtRows * wid + ((lane >> 2) & 1) * 4 + rsub;
                double rv = sm.vec[st][1][row];
                if (form_r) {
                    rv = fma(-alpha, sm.vec[st][3][row], rv);
                    s.r[base + row] = rv;
                }
                double y = sm.vec[st][0][row];
                y += v[0];
                y += vsum;
                y += double(sm.gate[st][row]) * rv / sm.vec[st][2][row] + shift * rv;
                zdst[base + row] = y;
                rz = fma(rv, y, rz);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[st]);
        }
    }
    if (mode == kApply) return;
    double v[1] = {rz}, tot[1];
    if (s.defer) {  // r.z is summed by the next SpMV (beta); CTA 0 keeps the books
        publish_partials<1>(v, s.dpart + kPartProl);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            Scalars* sc = s.sc;
            if (mode == kInit) {
                sc->beta = 0.0;
                sc->k = 1;
                if (sc->max_iters == 0) {
                    sc->iterations = 0;
                    sc->status = 1;
                    sc->done = 1;
                }
            } else {
                sc->k += 1;
            }
            if (s.use_cond) cudaGraphSetConditional(s.cond, sc->done ? 0u : 1u);
        }
        return;
    }
    if (grid_reduce_last<1>(v, s.partials, &s.counters[2], tot)) {
        if (s.G > 1) part_prolong_epilogue(s, mode, tot[0]);
        else if (threadIdx.x == 0) prolong_epilogue(s, mode, tot[0]);
    }
}

__global__ void __launch_bounds__(256) k_prolong_generic(DevSys s, int mode,
                                                         const double* rin_ext, double* zout) {
    if (prolong_skip(s, mode)) return;
    extern __shared__ float psm[];
    const uint64_t L = s.l, ls = s.ls, leaf = blockIdx.x, K = s.K, D = s.D;
    for (uint64_t t = threadIdx.x; t < 2 * ls; t += blockDim.x) {
        const uint64_t side = t / ls, j = t % ls;
        const float* src = s.coupled + side * ls;
        double acc = 0.0;
        for (uint64_t d = 0; d < D; ++d) {
            const uint64_t m = ((K + leaf) >> (D - d)) - 1;
            if (((leaf >> (D - 1 - d)) & 1ULL) == side) acc += double(__ldcg(&src[m * 2 * ls + j]));
        }
        psm[t] = float(acc);
    }
    __syncthreads();
    const float* Bu = s.F + s.bridge_base + leaf * 2 * L * ls;
    const float* Bv = Bu + L * ls;
    double rz = 0.0;
    for (uint64_t t = threadIdx.x; t < L; t += blockDim.x) {
        double au = 0.0, av = 0.0;
        for (uint64_t j = 0; j < ls; ++j) au = fma(double(Bu[t * ls + j]), double(psm[j]), au);
        for (uint64_t j = 0; j < ls; ++j) av = fma(double(Bv[t * ls + j]), double(psm[ls + j]), av);
        const uint64_t i = leaf * L + t;
        const double rv = mode == kApply ? rin_ext[i] : s.r[i];
        double y = s.y_loc[i];
        y += au;
        y += av;
        y += double(s.F[s.gate_base + i]) * rv / s.a_diag[i] + s.sc->shift * rv;
        (mode == kApply ? zout : s.z)[i] = y;
        rz = fma(rv, y, rz);
    }
    if (mode == kApply) return;
    double v[1] = {rz}, tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[2], tot) && threadIdx.x == 0)
        prolong_epilogue(s, mode, tot[0]);
}

// ============================================================================================
// Identity / Jacobi preconditioners (pcg.cpp:28-42) on the same graph: update, |r|^2,
// z = r (/ a_ii), r.z in one pass.
// ============================================================================================
__global__ void __launch_bounds__(256) k_simple(DevSys s, int mode, int jacobi) {
    if (s.sc->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && s.use_cond) cudaGraphSetConditional(s.cond, 0u);
        return;
    }
    const double alpha = mode == kLoop ? s.sc->alpha : 0.0;
    const double* pcur = mode == kLoop ? p_cur(s, s.sc->k) : nullptr;
    double v[2] = {0.0, 0.0};
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double rv = mode == kLoop ? update_row(s, pcur, alpha, i) : s.r[i];
        const double zv = jacobi ? rv / s.a_diag[i] : rv;
        s.z[i] = zv;
        v[0] = fma(rv, rv, v[0]);
        v[1] = fma(rv, zv, v[1]);
    }
    double tot[2];
    if (grid_reduce_last<2>(v, s.partials, &s.counters[3], tot) && threadIdx.x == 0) {
        Scalars* sc = s.sc;
        if (mode == kInit) {
            leaf_epilogue(s, kInit, tot[0]);
            if (!sc->done) prolong_epilogue(s, kInit, tot[1]);
            else if (s.use_cond) cudaGraphSetConditional(s.cond, 0u);
        } else {
            finish_residual(sc, s.history, tot[0]);
            if (!sc->done) prolong_epilogue(s, kLoop, tot[1]);
            else if (s.use_cond) cudaGraphSetConditional(s.cond, 0u);
        }
    }
}

// pcg.cpp:28-42 standalone: z = r / a_ii (jacobi) or z = r (identity), IEEE division.
__global__ void k_diag_apply(uint64_t n, const double* __restrict__ r, const double* __restrict__ a_diag,
                             double* __restrict__ z, int jacobi) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        z[i] = jacobi ? r[i] / a_diag[i] : r[i];
}

// Solve initialisation: x = 0, r = b, p_prev = 0 and the state words (pcg.cpp:65-80).
__global__ void k_init(DevSys s, const double* b) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        s.x[i] = 0.0;
        s.r[i] = b[i];
        s.p0[i] = 0.0;  // p_prev of iteration 1 (k = 1 -> p_prev = p0)
    }
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s.n_ghost;
         i += uint64_t(gridDim.x) * blockDim.x)
        s.p0[s.n + i] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Scalars* sc = s.sc;
        sc->k = 0;
        sc->iterations = 0;
        sc->breakdown_iter = 0;
        sc->hist_len = 0;
        sc->status = 1;
        sc->converged = 0;
        sc->done = 0;
        sc->beta = 0.0;
        sc->alpha = 0.0;
    }
}

}  // namespace hfpg

#include "leaf_coarse.cuh"

