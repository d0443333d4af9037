// IC(0) preconditioner apply on sm_100a (ic0.cpp:72-99, ic0_applier): z = (L L^T)^{-1} r by a
// forward sweep L y = r and a backward sweep L^T z = y, each a sync-free triangular solve.
//
// One thread per row, rows handed out in dependency-level order (fperm / bperm,
// ic0_levels_host). A row polls its dependencies' values until they are no longer pending (the
// value word is the ready flag, see kIc0Pending), then accumulates exactly as the reference:
//   forward   y_i = (r_i - sum_p L_ip y_p) / L_ii, p ascending          (ic0.cpp:80-86)
//   backward  z_j = (y_j - sum_i L_ij z_i) / L_jj, i DESCENDING          (ic0.cpp:88-95)
// with the pinned reference build's rounding (oracle/_ref: vmulsd + vsubsd in the forward loop,
// vfnmadd in the backward scatter) and IEEE division, so y and z are bit-identical to it.
// Deadlock freedom: every dependency of a row sits earlier in the level order, so in a CTA of
// lower (or the same) index, and CTAs are dispatched in index order.
// For a 7-point stencil in Morton order the dependency depth is nx + ny + nz - 2 levels.
#pragma once

#include "kernels.cuh"

namespace hfpg {

struct Ic0Dev {
    const unsigned long long* lro;  // L, lower CSR, diagonal last (n + 1)
    const uint32_t* lci;
    const double* lv;
    const unsigned long long* tro;  // strictly-lower L transposed, rows in decreasing order
    const uint32_t* tci;
    const double* tv;
    double* y;                      // forward-sweep result
    const uint32_t* fperm;          // rows in forward / backward dependency-level order
    const uint32_t* bperm;
    // chunked sweeps: rows in chunks of kIc0Threads consecutive (Morton) rows, one CTA each
    const uint16_t* flev;           // level of a row among its chunk's rows (forward / backward)
    const uint16_t* blev;
    const uint16_t* fmax;           // deepest level per chunk
    const uint16_t* bmax;
    int chunked;
};
constexpr int kIc0Threads = 128;
// "Not yet computed": a NaN payload no arithmetic produces (a computed value with these bits is
// stored as the canonical NaN instead). The value word is its own ready flag: one relaxed 64-bit
// store publishes it, one polled load receives it — no separate flag, fence or second load.
constexpr unsigned long long kIc0Pending = 0x7FF4DEAD0C0FFEE1ULL;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double x) {
    unsigned long long v = __double_as_longlong(x);
    if (v == kIc0Pending) v = 0x7FFFFFFFFFFFFFFFULL;
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ic0_get(const double* p) {
    unsigned long long v = ld_relaxed_u64(p);
    while (v == kIc0Pending) v = ld_relaxed_u64(p);
    return __longlong_as_double(v);
}
// Gather up to 8 dependency values at once (one round trip when they are ready), in order.
template <class Idx>
__device__ __forceinline__ int ic0_gather8(const double* src, Idx idx, int cnt, double (&v)[8]) {
    unsigned long long raw[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < cnt) raw[k] = ld_relaxed_u64(src + idx(k));
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < cnt) {
            while (raw[k] == kIc0Pending) raw[k] = ld_relaxed_u64(src + idx(k));
            v[k] = __longlong_as_double(raw[k]);
        }
    return cnt;
}

// Forward sweep: y = L^{-1} rin.
__device__ __forceinline__ void ic0_forward_row(const Ic0Dev& d, const double* rin, uint64_t i) {
    const uint64_t beg = d.lro[i], end = d.lro[i + 1] - 1;
    double s = rin[i];
    for (uint64_t p0 = beg; p0 < end; p0 += 8) {
        const int cnt = int(end - p0 < 8 ? end - p0 : 8);
        double v[8];
        ic0_gather8(d.y, [&](int k) { return d.lci[p0 + k]; }, cnt, v);
        for (int k = 0; k < cnt; ++k)
            s = __dsub_rn(s, __dmul_rn(d.lv[p0 + k], v[k]));  // the reference build does not contract this one
    }
    st_relaxed_f64(&d.y[i], s / d.lv[end]);
}
// Backward sweep: z = L^{-T} y.
__device__ __forceinline__ double ic0_backward_row(const Ic0Dev& d, double* z, uint64_t j) {
    double s = __ldcg(&d.y[j]);
    const uint64_t q0 = d.tro[j], q1 = d.tro[j + 1];
    for (uint64_t q = q0; q < q1; q += 8) {
        const int cnt = int(q1 - q < 8 ? q1 - q : 8);
        double v[8];
        ic0_gather8(z, [&](int k) { return d.tci[q + k]; }, cnt, v);
        for (int k = 0; k < cnt; ++k) s = fma(-d.tv[q + k], v[k], s);
    }
    const double zj = s / d.lv[d.lro[j + 1] - 1];
    st_relaxed_f64(&z[j], zj);
    return zj;
}

// Mark y and z pending (before a pair of sweeps).
__device__ __forceinline__ void ic0_mark_pending(const Ic0Dev& d, double* z, uint64_t n) {
    const double pend = __longlong_as_double((long long)kIc0Pending);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        d.y[i] = pend;
        z[i] = pend;
    }
}
__global__ void k_ic0_pending(Ic0Dev d, double* z, uint64_t n) { ic0_mark_pending(d, z, n); }


// PCG with IC(0), stage 1: x += alpha p, r -= alpha Ap and |r|^2 (pcg.cpp:97-101; k_simple's
// arithmetic), r0 at init, y and z marked pending; the last CTA finishes the residual
// bookkeeping.
__global__ void __launch_bounds__(256) k_ic0_update(DevSys s, Ic0Dev d, int mode) {
    if (s.sc->done) return;
    const double alpha = mode == kLoop ? s.sc->alpha : 0.0;
    const double* pcur = mode == kLoop ? p_cur(s, s.sc->k) : nullptr;
    double v[1] = {0.0};
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double rv = mode == kLoop ? update_row(s, pcur, alpha, i) : s.r[i];
        v[0] = fma(rv, rv, v[0]);
    }
    ic0_mark_pending(d, s.z, s.n);
    double tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[3], tot) && threadIdx.x == 0)
        leaf_epilogue(s, mode, tot[0]);  // r0 (init) or rel / history / stop
}

// Chunked sweeps (the default): CTA c owns the kIc0Threads consecutive rows of chunk c (a Morton
// brick), one thread per row, plus one helper warp. Every row thread loads its row's (up to 8)
// off-diagonal columns and values, right-hand side and diagonal into registers and registers each
// dependency outside the chunk (earlier chunks forward; later chunks backward, whose CTAs are
// numbered from the end) in a shared slot list. The helper warp polls all slots from global
// memory concurrently and drops each value into shared memory as soon as it is published; the
// row threads meanwhile resolve the chunk level by level (flev / blev, ic0_chunk_levels_host),
// one named barrier per level, reading in-chunk values and external slots from shared memory.
// The global hand-off latency thus overlaps the chunk's own levels: the wavefront pipelines
// across bricks and pays about one L2 round trip per brick crossing. Accumulation order and
// rounding are the per-row kernels' (bit-identical to the reference).
constexpr int kIc0ChunkThreads = kIc0Threads + 32;
constexpr int kIc0Slots = 256;  // external dependencies per chunk served by the helper warp
// Two register budgets: 4 CTAs per SM (96 registers, no spills) and 6 (64 registers). When the
// chunks far outnumber the resident slots the sweep is a wavefront over CTAs dispatched in index
// order and the number of chunks in flight bounds it (3D 1M: 1.38 -> 1.21 ms per IC(0)-PCG
// iteration with 6); on the 2D grids the per-level latency dominates and the larger budget wins
// (2D 65K: 0.65 vs 0.71 ms; 2D 262K: 1.42 vs 1.47 ms).
constexpr int kIc0MinBlocksWide = 6, kIc0MinBlocksResident = 4;

__device__ __forceinline__ unsigned long long ld_volatile_shared_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

template <bool FWD>
__device__ __forceinline__ double ic0_chunk_sweep(const Ic0Dev& d, const double* rhs, double* out, uint64_t n,
                                                  uint64_t ch) {
    __shared__ double sh[kIc0Threads];
    __shared__ unsigned long long ext[kIc0Slots];
    __shared__ uint32_t ext_col[kIc0Slots];
    __shared__ int nslot;
    const uint64_t c0 = ch * kIc0Threads, c1 = c0 + kIc0Threads, i = c0 + threadIdx.x;
    const bool helper = threadIdx.x >= kIc0Threads;
    if (threadIdx.x == 0) nslot = 0;
    __syncthreads();
    uint64_t beg = 0, end = 0;
    uint32_t col[8];
    double val[8];
    int slot[8];
    double rv = 0.0, diag = 1.0;
    int lev = -1;
    if (!helper && i < n) {
        if (FWD) {
            beg = d.lro[i];
            end = d.lro[i + 1] - 1;
            lev = d.flev[i];
            diag = d.lv[end];
        } else {
            beg = d.tro[i];
            end = d.tro[i + 1];
            lev = d.blev[i];
            diag = d.lv[d.lro[i + 1] - 1];
        }
        rv = FWD ? rhs[i] : __ldcg(&rhs[i]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            slot[k] = -1;
            if (beg + k < end) {
                col[k] = FWD ? d.lci[beg + k] : d.tci[beg + k];
                val[k] = FWD ? d.lv[beg + k] : d.tv[beg + k];
                if (FWD ? col[k] < c0 : col[k] >= c1) {
                    const int t = atomicAdd(&nslot, 1);
                    if (t < kIc0Slots) {  // beyond kIc0Slots the row polls global memory itself
                        slot[k] = t;
                        ext_col[t] = col[k];
                        ext[t] = kIc0Pending;
                    } else {
                        slot[k] = -2;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (helper) {  // poll every registered slot until all are published
        const int ns = min(nslot, kIc0Slots), lane = threadIdx.x & 31;
        for (int base = 0; base < ns; base += 32 * 8) {
            unsigned long long raw[8];
            bool pend = true;
            while (pend) {
                pend = false;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int t = base + k * 32 + lane;
                    if (t < ns && ext[t] == kIc0Pending) raw[k] = ld_relaxed_u64(&out[ext_col[t]]);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int t = base + k * 32 + lane;
                    if (t < ns && ext[t] == kIc0Pending) {
                        if (raw[k] != kIc0Pending) *reinterpret_cast<volatile unsigned long long*>(&ext[t]) = raw[k];
                        else pend = true;
                    }
                }
            }
        }
        return 0.0;
    }
    const int maxl = FWD ? d.fmax[ch] : d.bmax[ch];
    double res = 0.0;
    for (int l = 0; l <= maxl; ++l) {
        if (lev == l) {
            double acc = rv;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (beg + k < end) {
                    double v;
                    if (slot[k] == -1) {
                        v = sh[col[k] - c0];
                    } else if (slot[k] >= 0) {
                        unsigned long long r = ld_volatile_shared_u64(&ext[slot[k]]);
                        while (r == kIc0Pending) r = ld_volatile_shared_u64(&ext[slot[k]]);
                        v = __longlong_as_double(r);
                    } else {
                        v = ic0_get(&out[col[k]]);
                    }
                    // forward: vmulsd + vsubsd as the reference build; backward: its vfnmadd
                    acc = FWD ? __dsub_rn(acc, __dmul_rn(val[k], v)) : fma(-val[k], v, acc);
                }
            for (uint64_t p = beg + 8; p < end; ++p) {  // rows with more than 8 couplings
                const uint32_t j = FWD ? d.lci[p] : d.tci[p];
                const double a = FWD ? d.lv[p] : d.tv[p];
                const double v = (FWD ? j >= c0 : j < c1) ? sh[j - c0] : ic0_get(&out[j]);
                acc = FWD ? __dsub_rn(acc, __dmul_rn(a, v)) : fma(-a, v, acc);
            }
            res = acc / diag;
            sh[threadIdx.x] = res;
            st_relaxed_f64(&out[i], res);
        }
        named_bar_sync(1, kIc0Threads);
    }
    return res;
}

template <int MINB>
__global__ void __launch_bounds__(kIc0ChunkThreads, MINB) k_ic0_forward_chunk(DevSys s, Ic0Dev d, const double* rin,
                                                                        int mode) {
    if (mode != kApply && s.sc->done) return;
    ic0_chunk_sweep<true>(d, rin, d.y, s.n, blockIdx.x);
}

template <int MINB>
__global__ void __launch_bounds__(kIc0ChunkThreads, MINB) k_ic0_backward_chunk(DevSys s, Ic0Dev d, const double* rin,
                                                                         double* zout, int mode) {
    if (prolong_skip(s, mode)) return;
    const uint64_t nch = (s.n + kIc0Threads - 1) / kIc0Threads, ch = nch - 1 - blockIdx.x;
    const double zj = ic0_chunk_sweep<false>(d, d.y, zout, s.n, ch);
    const uint64_t j = ch * kIc0Threads + threadIdx.x;
    double v[1] = {threadIdx.x < kIc0Threads && j < s.n ? rin[j] * zj : 0.0};
    if (mode == kApply) return;
    double tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[2], tot) && threadIdx.x == 0)
        prolong_epilogue(s, mode, tot[0]);
}

__global__ void __launch_bounds__(kIc0Threads) k_ic0_forward(DevSys s, Ic0Dev d, const double* rin, int mode) {
    if (mode != kApply && s.sc->done) return;
    const uint64_t t = uint64_t(blockIdx.x) * kIc0Threads + threadIdx.x;
    if (t < s.n) ic0_forward_row(d, rin, d.fperm[t]);
}

// Stage 3 (and the standalone apply): the backward sweep into z, then r.z, beta and the
// iteration's bookkeeping (pcg.cpp:114-119) in the last CTA.
__global__ void __launch_bounds__(kIc0Threads) k_ic0_backward(DevSys s, Ic0Dev d, const double* rin, double* zout,
                                                              int mode) {
    if (prolong_skip(s, mode)) return;
    const uint64_t t = uint64_t(blockIdx.x) * kIc0Threads + threadIdx.x;
    double v[1] = {0.0};
    if (t < s.n) {
        const uint64_t j = d.bperm[t];
        const double zj = ic0_backward_row(d, zout, j);
        v[0] = rin[j] * zj;
    }
    if (mode == kApply) return;
    double tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[2], tot) && threadIdx.x == 0)
        prolong_epilogue(s, mode, tot[0]);
}

}  // namespace hfpg
