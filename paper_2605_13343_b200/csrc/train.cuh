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

// Batched small GEMMs through shared memory: out(r, j) = sum_p a(r, p) b(p, j) per batch entry
// (blockIdx.z), 4 x 4 outputs per thread, p staged 16 at a time through shared memory.
// Each output still accumulates over p in ascending order with the reference's rounding — fused
// (DOT = false: gemm_nn / gemm_tn) or dot_ref's products-then-sums with a fused odd tail
// (DOT = true: gemm_nt, the parameter gradients) — so tiling changes only the data reuse. NP = 2
// runs a second operand pair over the same output index (two accumulators, one epilogue).
struct BgOp {
    const double* a;
    uint64_t sa, ar, ap;  // a(r, p) = a[batch sa + r ar + p ap]
    const double* b;
    uint64_t sb, bp, bj;  // b(p, j) = b[batch sb + p bp + j bj]
};
constexpr int kBgP = 16;

// TM x TN output tile per CTA (TM * TN = 4096): 64 x 64, or 128 x 32 / 32 x 128 when one output
// dimension is 32 (the bridge and restriction stages), so no thread idles on padding.
template <bool DOT, int NP, int TM, int TN, class Epi>
__global__ void __launch_bounds__(256) k_bgemm(uint64_t R, uint64_t J, uint64_t P, BgOp o0, BgOp o1, Epi epi) {
    constexpr int TX = TN / 4, TY = 256 / TX;
    static_assert(TY * 4 == TM, "tile shape");
    __shared__ double As[NP][kBgP][TM + 1], Bs[NP][kBgP][TN + 1];
    const uint64_t bz = blockIdx.z, r0 = uint64_t(blockIdx.y) * TM, j0 = uint64_t(blockIdx.x) * TN;
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    double acc[NP][4][4];
#pragma unroll
    for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[n][i][q] = 0.0;
    for (uint64_t p0 = 0; p0 < P; p0 += kBgP) {
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            const BgOp& o = n ? o1 : o0;
#pragma unroll
            for (int e = 0; e < TM * kBgP / 256; ++e) {
                const int idx = tid + 256 * e;
                int r, pp;
                if (o.ap == 1) { pp = idx % kBgP; r = idx / kBgP; } else { r = idx % TM; pp = idx / TM; }
                const uint64_t gr = r0 + r, gp = p0 + pp;
                As[n][pp][r] = gr < R && gp < P ? o.a[bz * o.sa + gr * o.ar + gp * o.ap] : 0.0;
            }
#pragma unroll
            for (int e = 0; e < TN * kBgP / 256; ++e) {
                const int idx = tid + 256 * e;
                int j, pp;
                if (o.bj == 1) { j = idx % TN; pp = idx / TN; } else { pp = idx % kBgP; j = idx / kBgP; }
                const uint64_t gj = j0 + j, gq = p0 + pp;
                Bs[n][pp][j] = gj < J && gq < P ? o.b[bz * o.sb + gq * o.bp + gj * o.bj] : 0.0;
            }
        }
        __syncthreads();
        const int pl = int(P - p0 < kBgP ? P - p0 : kBgP);
        const bool odd_tail = DOT && (P & 1) && p0 + kBgP >= P;  // the fused last element
        for (int pp = 0; pp < pl; ++pp) {
            const bool fused = !DOT || (odd_tail && pp == pl - 1);
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = As[n][pp][ty + TY * i];
#pragma unroll
                for (int q = 0; q < 4; ++q) b[q] = Bs[n][pp][tx + TX * q];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        acc[n][i][q] = fused ? fma(a[i], b[q], acc[n][i][q])
                                             : __dadd_rn(acc[n][i][q], __dmul_rn(a[i], b[q]));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t r = r0 + ty + TY * i, j = j0 + tx + TX * q;
            if (r < R && j < J) epi(bz, r, j, acc[0][i][q], acc[NP - 1][i][q]);
        }
}
template <bool DOT, int NP, int TM, int TN, class Epi>
void bgemm_shape(cudaStream_t st, uint64_t batch, uint64_t R, uint64_t J, uint64_t P, BgOp o0, BgOp o1, Epi epi) {
    const dim3 g(unsigned((J + TN - 1) / TN), unsigned((R + TM - 1) / TM), unsigned(batch));
    k_bgemm<DOT, NP, TM, TN><<<g, 256, 0, st>>>(R, J, P, o0, o1, epi);
}
template <bool DOT, int NP, class Epi>
void bgemm(cudaStream_t st, uint64_t batch, uint64_t R, uint64_t J, uint64_t P, BgOp o0, BgOp o1, Epi epi) {
    if (!batch || !R || !J) return;
    if (J <= 32) bgemm_shape<DOT, NP, 128, 32>(st, batch, R, J, P, o0, o1, epi);
    else if (R <= 32) bgemm_shape<DOT, NP, 32, 128>(st, batch, R, J, P, o0, o1, epi);
    else bgemm_shape<DOT, NP, 64, 64>(st, batch, R, J, P, o0, o1, epi);
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
    const BgOp ft{P, 16384, 1, 128, T.X, 128 * kz, kz, 1};  // F^T X
    bgemm<false, 1>(st, K, 128, kz, 128, ft, ft, [=] __device__(uint64_t k, uint64_t r, uint64_t j, double a, double) {
        T.H[(k * 128 + r) * kz + j] = a;
    });
    const BgOp fh{P, 16384, 128, 1, T.H, 128 * kz, kz, 1};  // F H
    bgemm<false, 1>(st, K, 128, kz, 128, fh, fh, [=] __device__(uint64_t k, uint64_t r, uint64_t j, double a, double) {
        T.Y[(k * 128 + r) * kz + j] = a;
    });
    // restriction (gemm_tn with the bridges)
    const BgOp ru{P + T.bridge_base, 8192, 1, 32, T.X, 128 * kz, kz, 1}, rv{P + T.bridge_base + 4096, 8192, 1, 32,
                                                                          T.X, 128 * kz, kz, 1};
    bgemm<false, 2>(st, K, 32, kz, 128, ru, rv, [=] __device__(uint64_t k, uint64_t c, uint64_t j, double au, double av) {
        T.Rr[(k * 32 + c) * kz + j] = au;
        T.Rc[(k * 32 + c) * kz + j] = av;
    });
    // strip aggregation (leaf order)
    each(st, M * 32 * kz, [=] __device__(uint64_t t) {
        const uint64_t m = t / (32 * kz), e = t % (32 * kz);
        uint64_t span, rb, cb;
        tile_span(K, m, span, rb, cb);
        double sr = 0.0, sc = 0.0;
        uint64_t s = 0;
        for (; s + 8 <= span; s += 8) {  // 8 loads in flight, then the in-order adds
            double a[8], b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                a[q] = T.Rr[(rb + s + q) * 32 * kz + e];
                b[q] = T.Rc[(cb + s + q) * 32 * kz + e];
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sr += a[q];
                sc += b[q];
            }
        }
        for (; s < span; ++s) {
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
    const BgOp fb{P, 16384, 1, 128, BY, 128 * kz, kz, 1};  // W = F^T bar_Y
    bgemm<false, 1>(st, K, 128, kz, 128, fb, fb, [=] __device__(uint64_t k, uint64_t c, uint64_t j, double a, double) {
        T.W[(k * 128 + c) * kz + j] = a;
    });
    // bar_F += bar_Y H^T; bar_F += X W^T (dot products over the probes)
    const BgOp yh{BY, 128 * kz, kz, 1, T.H, 128 * kz, 1, kz}, xw{T.X, 128 * kz, kz, 1, T.W, 128 * kz, 1, kz};
    bgemm<true, 2>(st, K, 128, 128, kz, yh, xw, [=] __device__(uint64_t k, uint64_t r, uint64_t c, double a1, double a2) {
        double* g = G + k * 16384 + r * 128 + c;
        const double t = *g + a1;
        *g = t + a2;
    });
    // bridges: bar_Y G^T (prolongation)
    const BgOp yr{BY, 128 * kz, kz, 1, T.Gr, 32 * kz, 1, kz}, yc{BY, 128 * kz, kz, 1, T.Gc, 32 * kz, 1, kz};
    bgemm<true, 2>(st, K, 128, 32, kz, yr, yc, [=] __device__(uint64_t k, uint64_t r, uint64_t c, double a1, double a2) {
        double* gb = G + T.bridge_base + k * 8192 + r * 32 + c;
        gb[0] = gb[0] + a1;
        gb[4096] = gb[4096] + a2;
    });
    // bar_gather = bridge^T bar_Y
    const BgOp gu{P + T.bridge_base, 8192, 1, 32, BY, 128 * kz, kz, 1}, gv{P + T.bridge_base + 4096, 8192, 1, 32,
                                                                           BY, 128 * kz, kz, 1};
    bgemm<false, 2>(st, K, 32, kz, 128, gu, gv, [=] __device__(uint64_t k, uint64_t c, uint64_t j, double au, double av) {
        T.BGr[(k * 32 + c) * kz + j] = au;
        T.BGc[(k * 32 + c) * kz + j] = av;
    });
    each(st, M * 32 * kz, [=] __device__(uint64_t t) {  // gather adjoint: member leaves' bar-gathers
        const uint64_t m = t / (32 * kz), e = t % (32 * kz);
        uint64_t span, rb, cb;
        tile_span(K, m, span, rb, cb);
        double br = 0.0, bc = 0.0;
        uint64_t s = 0;
        for (; s + 8 <= span; s += 8) {
            double a[8], b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                a[q] = T.BGr[(rb + s + q) * 32 * kz + e];
                b[q] = T.BGc[(cb + s + q) * 32 * kz + e];
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                br += a[q];
                bc += b[q];
            }
        }
        for (; s < span; ++s) {
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
    // restriction adjoint: X bar_r^T
    const BgOp xr{T.X, 128 * kz, kz, 1, T.BRr, 32 * kz, 1, kz}, xc{T.X, 128 * kz, kz, 1, T.BRc, 32 * kz, 1, kz};
    bgemm<true, 2>(st, K, 128, 32, kz, xr, xc, [=] __device__(uint64_t k, uint64_t r, uint64_t c, double a1, double a2) {
        double* gb = G + T.bridge_base + k * 8192 + r * 32 + c;
        gb[0] = gb[0] + a1;
        gb[4096] = gb[4096] + a2;
    });
}

}  // namespace hfpg
