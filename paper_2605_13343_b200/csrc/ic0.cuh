// IC(0) preconditioner apply on sm_100a (ic0.cpp:72-99, ic0_applier): z = (L L^T)^{-1} r by a
// forward sweep L y = r and a backward sweep L^T z = y, each a sync-free triangular solve.
//
// One thread per row. A row waits, per dependency, for that row's ready flag (ld.acquire, the
// writer publishes value then flag with st.release), then accumulates exactly as the reference:
//   forward   y_i = (r_i - sum_p L_ip y_p) / L_ii, p ascending          (ic0.cpp:80-86)
//   backward  z_j = (y_j - sum_i L_ij z_i) / L_jj, i DESCENDING          (ic0.cpp:88-95)
// with the reference build's rounding of each product and difference and IEEE division, so y and z are
// bit-identical to the reference's (the pinned reference build, oracle/_ref: vmulsd + vsubsd in
// the forward loop, vfnmadd in the backward scatter). Flags carry an epoch (bumped once per apply), so they are
// never reset. Deadlock freedom: every dependency of a row lives in a CTA of lower index (the
// backward sweep numbers its CTAs from the last row), and CTAs are dispatched in index order.
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
    double* y;         // forward-sweep result
    unsigned* fflag;   // per-row ready epochs, forward / backward
    unsigned* bflag;
    unsigned* epoch;   // current apply's epoch (device word)
};
constexpr int kIc0Threads = 128;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void ic0_wait(const unsigned* flag, unsigned e) {
    while (ld_acquire_u32(flag) != e) __nanosleep(20);
}

// Forward sweep: y = L^{-1} rin.
__device__ __forceinline__ void ic0_forward_row(const Ic0Dev& d, const double* rin, uint64_t i, unsigned e) {
    const uint64_t beg = d.lro[i], end = d.lro[i + 1] - 1;
    double s = rin[i];
    for (uint64_t p = beg; p < end; ++p) {
        const uint32_t j = d.lci[p];
        ic0_wait(&d.fflag[j], e);
        s = __dsub_rn(s, __dmul_rn(d.lv[p], __ldcg(&d.y[j])));  // the reference build does not contract this one
    }
    const double yi = s / d.lv[end];
    __stcg(&d.y[i], yi);
    st_release_u32(&d.fflag[i], e);
}
// Backward sweep: z = L^{-T} y.
__device__ __forceinline__ double ic0_backward_row(const Ic0Dev& d, double* z, uint64_t j, unsigned e) {
    double s = __ldcg(&d.y[j]);
    for (uint64_t q = d.tro[j]; q < d.tro[j + 1]; ++q) {
        const uint32_t i = d.tci[q];
        ic0_wait(&d.bflag[i], e);
        s = fma(-d.tv[q], __ldcg(&z[i]), s);
    }
    const double zj = s / d.lv[d.lro[j + 1] - 1];
    __stcg(&z[j], zj);
    st_release_u32(&d.bflag[j], e);
    return zj;
}

__global__ void k_ic0_bump(Ic0Dev d) { *d.epoch += 1u; }

// PCG with IC(0), stage 1: x += alpha p, r -= alpha Ap and |r|^2 (pcg.cpp:97-101; k_simple's
// arithmetic), r0 at init; the last CTA finishes the residual bookkeeping and opens the next
// apply's epoch.
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
    double tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[3], tot) && threadIdx.x == 0) {
        leaf_epilogue(s, mode, tot[0]);  // r0 (init) or rel / history / stop
        *d.epoch += 1u;
    }
}

__global__ void __launch_bounds__(kIc0Threads) k_ic0_forward(DevSys s, Ic0Dev d, const double* rin, int mode) {
    if (mode != kApply && s.sc->done) return;
    const unsigned e = *d.epoch;
    const uint64_t i = uint64_t(blockIdx.x) * kIc0Threads + threadIdx.x;
    if (i < s.n) ic0_forward_row(d, rin, i, e);
}

// Stage 3 (and the standalone apply): the backward sweep into z, then r.z, beta and the
// iteration's bookkeeping (pcg.cpp:114-119) in the last CTA.
__global__ void __launch_bounds__(kIc0Threads) k_ic0_backward(DevSys s, Ic0Dev d, const double* rin, double* zout,
                                                              int mode) {
    if (prolong_skip(s, mode)) return;
    const unsigned e = *d.epoch;
    const uint64_t t = uint64_t(blockIdx.x) * kIc0Threads + threadIdx.x;
    double v[1] = {0.0};
    if (t < s.n) {
        const uint64_t j = s.n - 1 - t;
        const double zj = ic0_backward_row(d, zout, j, e);
        v[0] = rin[j] * zj;
    }
    if (mode == kApply) return;
    double tot[1];
    if (grid_reduce_last<1>(v, s.partials, &s.counters[2], tot) && threadIdx.x == 0)
        prolong_epilogue(s, mode, tot[0]);
}

}  // namespace hfpg
