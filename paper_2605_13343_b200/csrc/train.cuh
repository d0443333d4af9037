// Training of the factor tensor on the GPU: the double-precision batched
// apply with every stage stashed (adjoint.cpp:44-127, factor_apply_batch), its adjoint
// (adjoint.cpp:129-248, factor_apply_batch_adjoint), the probe losses (adjoint.cpp:250-292,
// loss_gradient; loss.cpp) and the AdamW step (train.cpp:136-160).
//
// A batch is kz probe columns, row-major (element (i, j) at i kz + j). Every stage is a batch of
// small GEMMs (128 x 128 leaf blocks, 128 x 32 bridges, 32 x 16 tiles) and runs one thread per
// output element, accumulating over the reduction index in ascending order — fused multiply-adds
// where the reference build fuses (the axpy-shaped gemm_nn / gemm_tn, dense.cpp:34-64), separate
// products and sums where it vectorises a dot product (gemm_nt, the gate adjoint; dot_ref) — and
// in the order of its strip / gather / gate loops, so the stashes, Y and the gradient are
// bit-identical to the reference's for the same inputs.
#pragma once

#include <cstdint>

namespace hfpg {

template <class F>
__global__ void __launch_bounds__(256) k_each(uint64_t n, F f) {
    for (uint64_t t = uint64_t(blockIdx.x) * 256 + threadIdx.x; t < n; t += uint64_t(gridDim.x) * 256) f(t);
}
template <class F>
void each(cudaStream_t st, uint64_t n, F f) {
    if (!n) return;
    const uint64_t g = std::min<uint64_t>((n + 255) / 256, 148 * 32);
    k_each<<<unsigned(g), 256, 0, st>>>(n, f);
}

// Device views of the batch state (all f64). L = 128, Ls = 32, rank 16 (the fast layout).
struct TrainDev {
    uint64_t n, K, D, M, kz;
    uint64_t tile_base, bridge_base, gate_base;
    const double* a_diag;
    double shift;
    // forward stashes
    double *X, *H, *Rr, *Rc, *Sr, *Sc, *Pu, *Qv, *Crow, *Ccol, *Gr, *Gc, *Y;
    // adjoint scratch
    double *W, *BGr, *BGc, *BCr, *BCc, *Bc1, *Bc2, *BSr, *BSc, *BRr, *BRc;
};

// The reference build's dot-product loops (gemm_nt, the gate adjoint: `acc += a[j] * b[j]`) are
// vectorised by GCC as packed products added one by one in order (vmulpd + vaddsd) with a scalar
// fused tail for an odd last element (vfmadd231sd) — read from the pinned build's object code.
__device__ __forceinline__ double dot_ref(const double* a, const double* b, uint64_t kz) {
    double acc = 0.0;
    const uint64_t body = kz & ~uint64_t(1);
    for (uint64_t j = 0; j < body; ++j) acc = __dadd_rn(acc, __dmul_rn(a[j], b[j]));
    if (kz & 1) acc = fma(a[body], b[body], acc);
    return acc;
}

__device__ __forceinline__ void tile_span(uint64_t K, uint64_t m, uint64_t& span, uint64_t& rb, uint64_t& cb) {
    uint64_t d = 0;
    while ((2ULL << d) <= m + 1) ++d;
    const uint64_t i = m + 1 - (1ULL << d), width = K >> d;
    span = width / 2;
    rb = i * width;
    cb = rb + span;
}

// factor_apply_batch: Y = M X (X already in T.X).
inline void train_forward(cudaStream_t st, const TrainDev T, const double* P) {
    const uint64_t kz = T.kz, K = T.K, M = T.M, D = T.D;
    // diagonal blocks: H_k = F_k^T X_k (gemm_tn), Y_k = F_k H_k (gemm_nn)
    each(st, T.n * kz, [=] __device__(uint64_t t) {
        const uint64_t row = t / kz, j = t % kz, k = row >> 7, r = row & 127;
        const double* F = P + k * 16384;
        const double* Xk = T.X + k * 128 * kz + j;
        double acc = 0.0;
        for (int p = 0; p < 128; ++p) acc = fma(F[p * 128 + r], Xk[p * kz], acc);
        T.H[t] = acc;
    });
    each(st, T.n * kz, [=] __device__(uint64_t t) {
        const uint64_t row = t / kz, j = t % kz, k = row >> 7, r = row & 127;
        const double* F = P + k * 16384 + r * 128;
        const double* Hk = T.H + k * 128 * kz + j;
        double acc = 0.0;
        for (int p = 0; p < 128; ++p) acc = fma(F[p], Hk[p * kz], acc);
        T.Y[t] = acc;
    });
    // restriction (gemm_tn with the bridges)
    each(st, K * 32 * kz, [=] __device__(uint64_t t) {
        const uint64_t row = t / kz, j = t % kz, k = row >> 5, c = row & 31;
        const double* Bu = P + T.bridge_base + k * 8192;
        const double* Xk = T.X + k * 128 * kz + j;
        double au = 0.0, av = 0.0;
        for (int p = 0; p < 128; ++p) au = fma(Bu[p * 32 + c], Xk[p * kz], au);
        for (int p = 0; p < 128; ++p) av = fma(Bu[4096 + p * 32 + c], Xk[p * kz], av);
        T.Rr[t] = au;
        T.Rc[t] = av;
    });
    // strip aggregation (leaf order)
    each(st, M * 32 * kz, [=] __device__(uint64_t t) {
        const uint64_t m = t / (32 * kz), e = t % (32 * kz);
        uint64_t span, rb, cb;
        tile_span(K, m, span, rb, cb);
        double sr = 0.0, sc = 0.0;
        for (uint64_t s = 0; s < span; ++s) {
            sr += T.Rr[(rb + s) * 32 * kz + e];
            sc += T.Rc[(cb + s) * 32 * kz + e];
        }
        T.Sr[t] = sr;
        T.Sc[t] = sc;
    });
    // coarse coupling: pu = U^T s_r, qv = V^T s_c (gemm_tn), then V pu, U qv (gemm_nn)
    each(st, M * 16 * kz, [=] __device__(uint64_t t) {
        const uint64_t m = t / (16 * kz), e = t % (16 * kz), q = e / kz, j = e % kz;
        const double* U = P + T.tile_base + m * 1024;
        const double* sr = T.Sr + m * 32 * kz + j;
        const double* sc = T.Sc + m * 32 * kz + j;
        double pu = 0.0, qv = 0.0;
        for (int p = 0; p < 32; ++p) pu = fma(U[p * 16 + q], sr[p * kz], pu);
        for (int p = 0; p < 32; ++p) qv = fma(U[512 + p * 16 + q], sc[p * kz], qv);
        T.Pu[t] = pu;
        T.Qv[t] = qv;
    });
    each(st, M * 32 * kz, [=] __device__(uint64_t t) {
        const uint64_t m = t / (32 * kz), e = t % (32 * kz), c = e / kz, j = e % kz;
        const double* U = P + T.tile_base + m * 1024;
        const double* pu = T.Pu + m * 16 * kz + j;
        const double* qv = T.Qv + m * 16 * kz + j;
        double cc = 0.0, cr = 0.0;
        for (int q = 0; q < 16; ++q) cc = fma(U[512 + c * 16 + q], pu[q * kz], cc);
        for (int q = 0; q < 16; ++q) cr = fma(U[c * 16 + q], qv[q * kz], cr);
        T.Ccol[t] = cc;
        T.Crow[t] = cr;
    });
    // gather tile outputs back to leaves (tile order = root first)
    each(st, K * 32 * kz, [=] __device__(uint64_t t) {
        const uint64_t k = t / (32 * kz), e = t % (32 * kz);
        double gr = 0.0, gc = 0.0;
        for (uint64_t d = 0; d < D; ++d) {
            const uint64_t m = ((K + k) >> (D - d)) - 1;
            if ((k >> (D - 1 - d)) & 1) gc += T.Ccol[m * 32 * kz + e];
            else gr += T.Crow[m * 32 * kz + e];
        }
        T.Gr[t] = gr;
        T.Gc[t] = gc;
    });
    // prolongation (gemm_nn accumulate: Ũ then Ṽ), then gate and shift
    each(st, T.n * kz, [=] __device__(uint64_t t) {
        const uint64_t row = t / kz, j = t % kz, k = row >> 7, r = row & 127;
        const double* Bu = P + T.bridge_base + k * 8192 + r * 32;
        const double* gr = T.Gr + k * 32 * kz + j;
        const double* gc = T.Gc + k * 32 * kz + j;
        double y = T.Y[t];
        for (int p = 0; p < 32; ++p) y = fma(Bu[p], gr[p * kz], y);
        for (int p = 0; p < 32; ++p) y = fma(Bu[4096 + p], gc[p * kz], y);
        const double g = P[T.gate_base + row] / T.a_diag[row] + T.shift;
        T.Y[t] = fma(g, T.X[t], y);
    });
}

// factor_apply_batch_adjoint: G (zeroed by the caller) += d(loss)/d(params) for bar_y = BY.
inline void train_adjoint(cudaStream_t st, const TrainDev T, const double* P, const double* BY, double* G) {
    const uint64_t kz = T.kz, K = T.K, M = T.M, D = T.D;
    each(st, T.n, [=] __device__(uint64_t i) {  // gate
        const double acc = dot_ref(BY + i * kz, T.X + i * kz, kz);
        G[T.gate_base + i] += acc / T.a_diag[i];
    });
    each(st, T.n * kz, [=] __device__(uint64_t t) {  // W = F^T bar_Y
        const uint64_t row = t / kz, j = t % kz, k = row >> 7, c = row & 127;
        const double* F = P + k * 16384;
        const double* by = BY + k * 128 * kz + j;
        double acc = 0.0;
        for (int p = 0; p < 128; ++p) acc = fma(F[p * 128 + c], by[p * kz], acc);
        T.W[t] = acc;
    });
    each(st, K * 16384, [=] __device__(uint64_t t) {  // bar_F += bar_Y H^T; bar_F += X W^T
        const uint64_t k = t >> 14, r = (t >> 7) & 127, c = t & 127;
        const double* by = BY + (k * 128 + r) * kz;
        const double* h = T.H + (k * 128 + c) * kz;
        const double* x = T.X + (k * 128 + r) * kz;
        const double* w = T.W + (k * 128 + c) * kz;
        const double a1 = dot_ref(by, h, kz), a2 = dot_ref(x, w, kz);
        double g = G[t];
        g = g + a1;
        G[t] = g + a2;
    });
    each(st, K * 128 * 32, [=] __device__(uint64_t t) {  // bridges: bar_Y G^T (prolongation)
        const uint64_t k = t >> 12, r = (t >> 5) & 127, c = t & 31;
        const double* by = BY + (k * 128 + r) * kz;
        const double* gr = T.Gr + (k * 32 + c) * kz;
        const double* gc = T.Gc + (k * 32 + c) * kz;
        const double a1 = dot_ref(by, gr, kz), a2 = dot_ref(by, gc, kz);
        double* gb = G + T.bridge_base + k * 8192 + r * 32 + c;
        gb[0] = gb[0] + a1;
        gb[4096] = gb[4096] + a2;
    });
    each(st, K * 32 * kz, [=] __device__(uint64_t t) {  // bar_gather = bridge^T bar_Y
        const uint64_t row = t / kz, j = t % kz, k = row >> 5, c = row & 31;
        const double* Bu = P + T.bridge_base + k * 8192;
        const double* by = BY + k * 128 * kz + j;
        double au = 0.0, av = 0.0;
        for (int p = 0; p < 128; ++p) au = fma(Bu[p * 32 + c], by[p * kz], au);
        for (int p = 0; p < 128; ++p) av = fma(Bu[4096 + p * 32 + c], by[p * kz], av);
        T.BGr[t] = au;
        T.BGc[t] = av;
    });
    each(st, M * 32 * kz, [=] __device__(uint64_t t) {  // gather adjoint: member leaves' bar-gathers
        const uint64_t m = t / (32 * kz), e = t % (32 * kz);
        uint64_t span, rb, cb;
        tile_span(K, m, span, rb, cb);
        double br = 0.0, bc = 0.0;
        for (uint64_t s = 0; s < span; ++s) {
            br += T.BGr[(rb + s) * 32 * kz + e];
            bc += T.BGc[(cb + s) * 32 * kz + e];
        }
        T.BCr[t] = br;
        T.BCc[t] = bc;
    });
    each(st, M * 16 * kz, [=] __device__(uint64_t t) {  // bar_coef: U^T btr, V^T btc
        const uint64_t m = t / (16 * kz), e = t % (16 * kz), q = e / kz, j = e % kz;
        const double* U = P + T.tile_base + m * 1024;
        const double* btr = T.BCr + m * 32 * kz + j;
        const double* btc = T.BCc + m * 32 * kz + j;
        double b1 = 0.0, b2 = 0.0;
        for (int p = 0; p < 32; ++p) b1 = fma(U[p * 16 + q], btr[p * kz], b1);
        for (int p = 0; p < 32; ++p) b2 = fma(U[512 + p * 16 + q], btc[p * kz], b2);
        T.Bc1[t] = b1;
        T.Bc2[t] = b2;
    });
    each(st, M * 32 * 16, [=] __device__(uint64_t t) {  // tile grads (reference order)
        const uint64_t m = t >> 9, c = (t >> 4) & 31, q = t & 15;
        const double* btr = T.BCr + (m * 32 + c) * kz;
        const double* btc = T.BCc + (m * 32 + c) * kz;
        const double* sr = T.Sr + (m * 32 + c) * kz;
        const double* sc = T.Sc + (m * 32 + c) * kz;
        const double* qv = T.Qv + (m * 16 + q) * kz;
        const double* pu = T.Pu + (m * 16 + q) * kz;
        const double* b1 = T.Bc1 + (m * 16 + q) * kz;
        const double* b2 = T.Bc2 + (m * 16 + q) * kz;
        const double u1 = dot_ref(btr, qv, kz), v1 = dot_ref(sc, b1, kz), v2 = dot_ref(btc, pu, kz),
                     u2 = dot_ref(sr, b2, kz);
        double* gu = G + T.tile_base + m * 1024 + c * 16 + q;
        double a = gu[0];
        a = a + u1;
        gu[0] = a + u2;
        double b = gu[512];
        b = b + v1;
        gu[512] = b + v2;
    });
    each(st, M * 32 * kz, [=] __device__(uint64_t t) {  // bar strips: V bar_coef1, U bar_coef2
        const uint64_t m = t / (32 * kz), e = t % (32 * kz), c = e / kz, j = e % kz;
        const double* U = P + T.tile_base + m * 1024;
        const double* b1 = T.Bc1 + m * 16 * kz + j;
        const double* b2 = T.Bc2 + m * 16 * kz + j;
        double bsc = 0.0, bsr = 0.0;
        for (int q = 0; q < 16; ++q) bsc = fma(U[512 + c * 16 + q], b1[q * kz], bsc);
        for (int q = 0; q < 16; ++q) bsr = fma(U[c * 16 + q], b2[q * kz], bsr);
        T.BSc[t] = bsc;
        T.BSr[t] = bsr;
    });
    each(st, K * 32 * kz, [=] __device__(uint64_t t) {  // strip adjoint back to leaves (tile order)
        const uint64_t k = t / (32 * kz), e = t % (32 * kz);
        double rr = 0.0, rc = 0.0;
        for (uint64_t d = 0; d < D; ++d) {
            const uint64_t m = ((K + k) >> (D - d)) - 1;
            if ((k >> (D - 1 - d)) & 1) rc += T.BSc[m * 32 * kz + e];
            else rr += T.BSr[m * 32 * kz + e];
        }
        T.BRr[t] = rr;
        T.BRc[t] = rc;
    });
    each(st, K * 128 * 32, [=] __device__(uint64_t t) {  // restriction adjoint: X bar_r^T
        const uint64_t k = t >> 12, r = (t >> 5) & 127, c = t & 31;
        const double* x = T.X + (k * 128 + r) * kz;
        const double* br = T.BRr + (k * 32 + c) * kz;
        const double* bc = T.BRc + (k * 32 + c) * kz;
        const double a1 = dot_ref(x, br, kz), a2 = dot_ref(x, bc, kz);
        double* gb = G + T.bridge_base + k * 8192 + r * 32 + c;
        gb[0] = gb[0] + a1;
        gb[4096] = gb[4096] + a2;
    });
}

}  // namespace hfpg
