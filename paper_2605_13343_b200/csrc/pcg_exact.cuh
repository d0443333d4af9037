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

namespace hfpg {

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

}  // namespace hfpg
