// The reference's PCG bit for bit (pcg.cpp:53-126 as its pinned build computes it): every dot
// product as its sequential loop, every vector update with its rounding, so x, the residual
// history, the iteration count and the stopping status are identical to the reference's.
//
// The pinned build (oracle/_ref, read from its object code) vectorises `s += a[i] * c[i]` as
// packed products added to s one by one in index order (vmulpd + four in-order vaddsd) over the
// first n & ~3 elements; the (n & 3) remainder is a pair (products, in-order sums) then a fused
// last element (vfmadd231sd) — except the first |r0|^2, whose remainder is fused element by
// element. The sum over the products is the sequential sum the frame generator already emulates
// exactly in parallel (seq_sum, framegen.cuh); the products are materialised once per dot.
// Updates: x = fma(alpha, p, x), r = fma(-alpha, ap, r), p = fma(beta, p, z) (vfmadd213pd /
// vfnmadd213pd). SpMV and the preconditioners are the solve path's own (bit-identical) kernels.
#pragma once

#include "train.cuh"  // each(), tile_span()

namespace hfpg {

// apply<float> (apply.cpp:80-173) exactly as the pinned build computes it: r cast to float; the
// transposed matvecs (F^T r, the restrictions, U^T s / V^T s) accumulate in float with fused
// multiply-adds in row order (vfmadd...ss/ps); the matvecs with a double accumulator add the
// exact float products in column order and round once (to float for the couplings); strip and
// gather sums are double, in span / tile order; the gate term is y + fma(shift, r, (g r) / d).
// One thread per output of each stage — a verification path, not the solve path's kernels.
struct ExApplyWs {
    float *rin, *coef, *rr, *rc, *scr, *scc, *cc1, *cc2, *crow, *ccol, *gr, *gc;
};
inline void apply_exact_f32(cudaStream_t st, const Layout L, const float* P, const double* a_diag, double shift,
                            const double* r, double* y, const ExApplyWs w) {
    const uint64_t n = L.n, l = L.l, ls = L.ls, rk = L.rk, K = L.k, M = K - 1, D = L.depth;
    const uint64_t tb = L.tile_base, bb = L.bridge_base;  // Layout's offsets (host-only methods)
    each(st, n, [=] __device__(uint64_t i) { w.rin[i] = __double2float_rn(r[i]); });
    each(st, K * l, [=] __device__(uint64_t t) {  // leaf_coef = F_k^T r_k (matvec_t)
        const uint64_t k = t / l, j = t % l;
        const float* f = P + k * l * l;
        float c = 0.f;
        for (uint64_t i = 0; i < l; ++i) c = __fmaf_rn(f[i * l + j], w.rin[k * l + i], c);
        w.coef[t] = c;
    });
    each(st, n, [=] __device__(uint64_t t) {  // y_k = F_k leaf_coef (matvec_add_double)
        const uint64_t k = t / l, i = t % l;
        const float* f = P + k * l * l + i * l;
        double acc = 0.0;
        for (uint64_t j = 0; j < l; ++j) acc = __fma_rn(double(f[j]), double(w.coef[k * l + j]), acc);
        y[t] = __dadd_rn(0.0, acc);
    });
    each(st, K * ls, [=] __device__(uint64_t t) {  // restrictions (matvec_t)
        const uint64_t k = t / ls, c = t % ls;
        const float *bu = P + bb + k * 2 * l * ls, *bv = P + bb + k * 2 * l * ls + l * ls;
        float u = 0.f, v = 0.f;
        for (uint64_t i = 0; i < l; ++i) u = __fmaf_rn(bu[i * ls + c], w.rin[k * l + i], u);
        for (uint64_t i = 0; i < l; ++i) v = __fmaf_rn(bv[i * ls + c], w.rin[k * l + i], v);
        w.rr[t] = u;
        w.rc[t] = v;
    });
    each(st, M * ls, [=] __device__(uint64_t t) {  // strip sums (double, span order), cast
        const uint64_t m = t / ls, j = t % ls;
        uint64_t span, rb, cb;
        tile_span(K, m, span, rb, cb);
        double sr = 0.0, sc = 0.0;
        uint64_t q = 0;
        for (; q + 8 <= span; q += 8) {  // 8 loads in flight, then the in-order adds
            float a[8], b[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                a[e] = w.rr[(rb + q + e) * ls + j];
                b[e] = w.rc[(cb + q + e) * ls + j];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                sr = __dadd_rn(sr, double(a[e]));
                sc = __dadd_rn(sc, double(b[e]));
            }
        }
        for (; q < span; ++q) {
            sr = __dadd_rn(sr, double(w.rr[(rb + q) * ls + j]));
            sc = __dadd_rn(sc, double(w.rc[(cb + q) * ls + j]));
        }
        w.scr[t] = __double2float_rn(sr);
        w.scc[t] = __double2float_rn(sc);
    });
    each(st, M * rk, [=] __device__(uint64_t t) {  // coarse_coef = U^T s_r, V^T s_c (matvec_t)
        const uint64_t m = t / rk, q = t % rk;
        const float *u = P + tb + m * ls * ls, *v = P + tb + m * ls * ls + ls * rk;
        float a = 0.f, b = 0.f;
        for (uint64_t p = 0; p < ls; ++p) a = __fmaf_rn(u[p * rk + q], w.scr[m * ls + p], a);
        for (uint64_t p = 0; p < ls; ++p) b = __fmaf_rn(v[p * rk + q], w.scc[m * ls + p], b);
        w.cc1[t] = a;
        w.cc2[t] = b;
    });
    each(st, M * ls, [=] __device__(uint64_t t) {  // coupled_col = V cc1, coupled_row = U cc2 (matvec)
        const uint64_t m = t / ls, c = t % ls;
        const float *u = P + tb + m * ls * ls + c * rk, *v = P + tb + m * ls * ls + ls * rk + c * rk;
        double a = 0.0, b = 0.0;
        for (uint64_t q = 0; q < rk; ++q) a = __fma_rn(double(v[q]), double(w.cc1[m * rk + q]), a);
        for (uint64_t q = 0; q < rk; ++q) b = __fma_rn(double(u[q]), double(w.cc2[m * rk + q]), b);
        w.ccol[t] = __double2float_rn(a);
        w.crow[t] = __double2float_rn(b);
    });
    each(st, K * ls, [=] __device__(uint64_t t) {  // gathers (double, tile order = root first), cast
        const uint64_t k = t / ls, j = t % ls;
        double gr = 0.0, gc = 0.0;
        for (uint64_t d = 0; d < D; ++d) {
            const uint64_t m = ((K + k) >> (D - d)) - 1;
            if ((k >> (D - 1 - d)) & 1) gc = __dadd_rn(gc, double(w.ccol[m * ls + j]));
            else gr = __dadd_rn(gr, double(w.crow[m * ls + j]));
        }
        w.gr[t] = __double2float_rn(gr);
        w.gc[t] = __double2float_rn(gc);
    });
    const float* gate = P + L.gate_base;
    each(st, n, [=] __device__(uint64_t t) {  // prolongation (matvec_add_double x2), gate + shift
        const uint64_t k = t / l, i = t % l;
        const float *bu = P + bb + k * 2 * l * ls + i * ls, *bv = P + bb + k * 2 * l * ls + l * ls + i * ls;
        double acc = 0.0;
        for (uint64_t j = 0; j < ls; ++j) acc = __fma_rn(double(bu[j]), double(w.gr[k * ls + j]), acc);
        double yv = __dadd_rn(y[t], acc);
        acc = 0.0;
        for (uint64_t j = 0; j < ls; ++j) acc = __fma_rn(double(bv[j]), double(w.gc[k * ls + j]), acc);
        yv = __dadd_rn(yv, acc);
        const double g = __ddiv_rn(__dmul_rn(double(gate[t]), r[t]), a_diag[t]);
        y[t] = __dadd_rn(yv, __fma_rn(shift, r[t], g));
    });
}

__global__ void k_ex_prod(const double* __restrict__ a, const double* __restrict__ c, uint64_t n,
                          double* __restrict__ out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = __dmul_rn(a[i], c[i]);
}
// The remainder after the vectorised body (one thread). fused_each: the |r0|^2 site's form.
__global__ void k_ex_tail(const double* __restrict__ a, const double* __restrict__ c, uint64_t n, uint64_t n4,
                          int fused_each, double* sum) {
    double s = *sum;
    uint64_t i = n4;
    if (fused_each) {
        for (; i < n; ++i) s = __fma_rn(a[i], c[i], s);
    } else {
        if (n - i >= 2) {
            s = __dadd_rn(s, __dmul_rn(a[i], c[i]));
            s = __dadd_rn(s, __dmul_rn(a[i + 1], c[i + 1]));
            i += 2;
        }
        if (i < n) s = __fma_rn(a[i], c[i], s);
    }
    *sum = s;
}
__global__ void k_ex_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                        const double* __restrict__ ap, double alpha, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        x[i] = __fma_rn(alpha, p[i], x[i]);
        r[i] = __fma_rn(-alpha, ap[i], r[i]);
    }
}
__global__ void k_ex_p(double* __restrict__ p, const double* __restrict__ z, double beta, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = __fma_rn(beta, p[i], z[i]);
}
__global__ void k_ex_jacobi(const double* __restrict__ r, const double* __restrict__ d, double* __restrict__ z,
                            uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        z[i] = __ddiv_rn(r[i], d[i]);
}

// Device-resident loop state for the captured iteration (hfpg_pcg_solve_exact without a
// residual callback): the scalar decisions of pcg.cpp:86-119 taken on the device, so one CUDA
// graph per iteration runs without host round trips; once `stop` is set every later step is a
// no-op for x, r, p and the history.
struct ExState {
    double rz, alpha, beta, r0, tol_bd, rtol;
    unsigned long long k, iters;  // current iteration (1-based); the stopping iteration
    int stop, pad;                // 0 running, 1 converged, 2 breakdown
};
__global__ void k_exg_alpha(ExState* S, const double* dsum) {  // pcg.cpp:88-96
    if (S->stop) return;
    const double pap = dsum[0], p2 = dsum[1];
    if (pap < -S->tol_bd * p2 || pap == 0.0) {
        S->stop = 2;
        S->iters = S->k;
        return;
    }
    S->alpha = S->rz / pap;
}
__global__ void k_exg_xr(const ExState* S, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ ap, uint64_t n) {
    if (S->stop) return;
    const double alpha = S->alpha;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        x[i] = __fma_rn(alpha, p[i], x[i]);
        r[i] = __fma_rn(-alpha, ap[i], r[i]);
    }
}
__global__ void k_exg_rel(ExState* S, const double* rr, double* hist) {  // pcg.cpp:100-107
    if (S->stop) return;
    const double rel = sqrt(*rr) / S->r0;
    hist[S->k - 1] = rel;
    if (rel <= S->rtol) {
        S->stop = 1;
        S->iters = S->k;
    }
}
__global__ void k_exg_beta(ExState* S, const double* rzn) {  // pcg.cpp:115-117
    if (!S->stop) {
        S->beta = *rzn / S->rz;
        S->rz = *rzn;
    }
    S->k += 1;
}
__global__ void k_exg_p(const ExState* S, double* __restrict__ p, const double* __restrict__ z, uint64_t n) {
    if (S->stop) return;
    const double beta = S->beta;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = __fma_rn(beta, p[i], z[i]);
}

}  // namespace hfpg
