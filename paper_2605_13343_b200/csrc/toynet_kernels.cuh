// Toy-network inference kernels (toy_net.cpp:225-586) other than the tcgen05 GEMMs:
// features, D^-1 A graph aggregation, layer norm, edge-bias MLP, windowed attention,
// strip pooling, highway scatter / chunk means, FFN input assembly. fp32 activations.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace hfpg {

struct TnDims {
    uint64_t n, L, Ls, rk, K, M, D;  // nodes, leaf, coarse, rank, leaves, tiles, log2 K
    uint32_t width, height, d, heads, dglob, eh, feat_pad;
};

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
// GELU with erf from Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7 absolute, below the fp32
// rounding of the GELU's inputs after tf32 products): one reciprocal, one exp2 and a degree-5
// polynomial instead of erff's branchy evaluation. The GEMM epilogues and the edge-bias MLPs use it.
__device__ __forceinline__ float gelu_fast(float x) {
    const float z = fabsf(x) * 0.70710678118654752f;
    float t, e;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.f)));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
    float p = fmaf(1.061405429f, t, -1.453152027f);
    p = fmaf(p, t, 1.421413741f);
    p = fmaf(p, t, -0.284496736f);
    p = fmaf(p, t, 0.254829592f);
    p *= t;
    const float erf_abs = fmaf(-p, e, 1.f);  // erf(|x| / sqrt 2)
    return 0.5f * x * (1.f + copysignf(erf_abs, x));
}

// Tile heap index m -> (span in leaves, row0 node, col0 node, chunk rows per token)
struct TileGeom {
    uint64_t span, row0, col0, chunk;
};
__device__ __forceinline__ TileGeom tile_geom(const TnDims& g, uint64_t m) {
    int d = 0;
    while ((2ULL << d) <= m + 1) ++d;
    const uint64_t i = m + 1 - (1ULL << d), width = g.K >> d, span = width / 2;
    TileGeom t;
    t.span = span;
    t.row0 = i * width * g.L;
    t.col0 = (i * width + span) * g.L;
    t.chunk = span * g.L / g.Ls;
    return t;
}


// sum_{s < cnt} p[s * stride], eight interleaved fp32 partial sums combined in a fixed order
// (deterministic; eight loads in flight per thread instead of one dependent chain).
__device__ __forceinline__ float strided_sum(const float* p, uint64_t cnt, uint64_t stride) {
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint64_t s = 0;
    for (; s + 8 <= cnt; s += 8)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] += p[(s + q) * stride];
    for (int q = 0; s < cnt; ++s, ++q) a[q] += p[s * stride];
    return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// toy_net.cpp:270-293 per-node features [rho, x^, y^, 4 absent-neighbour flags, glob]; the
// flags come from the operator's off-diagonal pattern (a present neighbour always couples).
__global__ void k_tn_features(TnDims g, const uint32_t* order, const double* rho,
                              const unsigned long long* ro, const uint32_t* ci, const float* glob,
                              float* feat) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const uint32_t id = order[i], x = id % g.width, y = id / g.width;
    float* f = feat + i * g.feat_pad;
    bool present[4] = {false, false, false, false};
    for (unsigned long long p = ro[i]; p < ro[i + 1]; ++p) {
        const uint32_t j = ci[p];
        if (j == i) continue;
        const uint32_t jd = order[j], xj = jd % g.width, yj = jd / g.width;
        if (xj + 1 == x && yj == y) present[0] = true;
        if (xj == x + 1 && yj == y) present[1] = true;
        if (xj == x && yj + 1 == y) present[2] = true;
        if (xj == x && yj == y + 1) present[3] = true;
    }
    f[0] = float(rho[i]);
    f[1] = float((double(x) + 0.5) / double(g.width));
    f[2] = float((double(y) + 0.5) / double(g.height));
    for (int b = 0; b < 4; ++b) f[3 + b] = present[b] ? 0.f : 1.f;
    for (uint32_t q = 0; q < g.dglob; ++q) f[7 + q] = glob[q];
    for (uint32_t q = 7 + g.dglob; q < g.feat_pad; ++q) f[q] = 0.f;
}

// toy_net.cpp:305-313 msg_i = sum_p (A_ip / A_ii) x_j: one warp per row, lane owns 4 channels
// (d = 128). f64 weights, fp32 accumulation of the channel sums.
__global__ void k_tn_gcn_msg(TnDims g, const unsigned long long* ro, const uint32_t* ci,
                             const double* v, const double* diag, const float* x, float* msg) {
    const uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= g.n) return;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const unsigned long long p0 = ro[row], p1 = ro[row + 1];
    const double rdiag = 1.0 / diag[row];  // A_ij / A_ii to within an f64 ulp, then cast to fp32
    for (unsigned long long pb = p0; pb < p1; pb += 8) {  // the row's (<= 8) gathers in flight together
        float w[8];
        float4 xj[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            w[q] = 0.f;
            xj[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (pb + q < p1) {
                w[q] = float(v[pb + q] * rdiag);
                xj[q] = reinterpret_cast<const float4*>(x + uint64_t(ci[pb + q]) * g.d)[lane];
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // the row's entries in CSR order (toy_net.cpp:305-313)
            acc.x = fmaf(w[q], xj[q].x, acc.x);
            acc.y = fmaf(w[q], xj[q].y, acc.y);
            acc.z = fmaf(w[q], xj[q].z, acc.z);
            acc.w = fmaf(w[q], xj[q].w, acc.w);
        }
    }
    reinterpret_cast<float4*>(msg + row * g.d)[lane] = acc;
}

// toy_net.cpp:28-41 layer norm without affine, eps 1e-5, two-pass (mean, then centred
// variance) so huge token magnitudes stay accurate. One warp per row of d = 128.
// out may be a wider matrix (row stride ld_out).
__global__ void k_tn_layernorm(uint64_t rows, uint32_t d, const float* x, float* out, uint32_t ld_out) {
    const uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float4 v = reinterpret_cast<const float4*>(x + row * d)[lane];
    float s = (v.x + v.y) + (v.z + v.w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / float(d);
    const float a = v.x - mean, b = v.y - mean, c = v.z - mean, e = v.w - mean;
    float q = (a * a + b * b) + (c * c + e * e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.f / sqrtf(q / float(d) + 1e-5f);
    reinterpret_cast<float4*>(out + row * ld_out)[lane] = make_float4(a * inv, b * inv, c * inv, e * inv);
}

// toy_net.cpp:55-74 edge-bias MLP [dx, dy, dist, c] -> GELU(8) -> heads.
struct EdgeMlp {
    float w1[4 * 8], b1[8], w2[8 * 8], b2[8];
};
// Fixed-size form (the production config: edge_hidden = heads = 8): fully unrolled, so the
// hidden layer and outputs stay in registers (the runtime-bounded loops below put them, and the
// indexed weights, in local memory — 374 us for the 8.4 M leaf pairs at N=65,536).
template <int EH, int HD>
__device__ __forceinline__ void edge_mlp_t(const EdgeMlp& m, float dx, float dy, float dist, float c,
                                           float (&out)[8]) {
    float hid[EH];
#pragma unroll
    for (int k = 0; k < EH; ++k) {
        float a = m.b1[k];
        a = fmaf(dx, m.w1[0 * EH + k], a);
        a = fmaf(dy, m.w1[1 * EH + k], a);
        a = fmaf(dist, m.w1[2 * EH + k], a);
        a = fmaf(c, m.w1[3 * EH + k], a);
        hid[k] = gelu_fast(a);
    }
#pragma unroll
    for (int h = 0; h < HD; ++h) {
        float a = m.b2[h];
#pragma unroll
        for (int k = 0; k < EH; ++k) a = fmaf(hid[k], m.w2[k * HD + h], a);
        out[h] = a;
    }
}
__device__ __forceinline__ void edge_mlp(const EdgeMlp& m, uint32_t eh, uint32_t heads, float dx,
                                         float dy, float dist, float c, float* out) {
    if (eh == 8 && heads == 8) {
        float o[8];
        edge_mlp_t<8, 8>(m, dx, dy, dist, c, o);
#pragma unroll
        for (int h = 0; h < 8; ++h) out[h] = o[h];
        return;
    }
    float hid[8];
    for (uint32_t k = 0; k < eh; ++k) {
        float a = m.b1[k];
        a = fmaf(dx, m.w1[0 * eh + k], a);
        a = fmaf(dy, m.w1[1 * eh + k], a);
        a = fmaf(dist, m.w1[2 * eh + k], a);
        a = fmaf(c, m.w1[3 * eh + k], a);
        hid[k] = gelu_fast(a);
    }
    for (uint32_t h = 0; h < heads; ++h) {
        float a = m.b2[h];
        for (uint32_t k = 0; k < eh; ++k) a = fmaf(hid[k], m.w2[k * heads + h], a);
        out[h] = a;
    }
}

// Leaf-pair edge biases (toy_net.cpp:371-381), once per forward (reused by every layer), stored
// as the reference indexes them — bias[k][h][i][j], query i, key j (toy_net.cpp:95) — in fp16
// (10-bit mantissa like the tf32 products; the MLP outputs are O(1e3) at most, far inside the
// fp16 range), pre-multiplied by log2(e) for the attention kernels' exp2 softmax: half the bytes
// of fp32, one query row's keys contiguous. Coupling = A_{base+i, base+j} looked up in the sorted CSR row.
__device__ __forceinline__ void leaf_bias_pair(TnDims g, uint32_t lL, uint64_t k, uint64_t base, uint32_t idx,
                                               const float* cx, const float* cy, const uint32_t* order,
                                               const unsigned long long* ro, const uint32_t* ci, const double* v,
                                               const EdgeMlp& mlp, __half* bias) {
    const uint32_t i = idx >> lL, j = idx & ((1u << lL) - 1u);
    float xa, ya, xb, yb;
    if (g.L <= 128) {
        xa = cx[i]; ya = cy[i]; xb = cx[j]; yb = cy[j];
    } else {
        const uint32_t a = order[base + i], b = order[base + j];
        xa = float((double(a % g.width) + 0.5) / double(g.width)); ya = float((double(a / g.width) + 0.5) / double(g.height));
        xb = float((double(b % g.width) + 0.5) / double(g.width)); yb = float((double(b / g.width) + 0.5) / double(g.height));
    }
    const float dx = xa - xb, dy = ya - yb, dist = sqrtf(dx * dx + dy * dy);
    double c = 0.0;
    const uint32_t col = uint32_t(base) + j;
    for (unsigned long long p = ro[base + i], pe = ro[base + i + 1]; p < pe; ++p)
        if (ci[p] == col) c = v[p];
    float out[8];
    const uint64_t L2 = uint64_t(1) << (2 * lL);
    __half* bk = bias + (k * g.heads) * L2 + idx;  // + h L^2: [k][h][i][j]
    if (g.eh == 8 && g.heads == 8) {
        edge_mlp_t<8, 8>(mlp, dx, dy, dist, float(c), out);
#pragma unroll
        for (int h = 0; h < 8; ++h) bk[h * L2] = __float2half_rn(out[h] * 1.4426950408889634f);
        return;
    }
    edge_mlp(mlp, g.eh, g.heads, dx, dy, dist, float(c), out);
    for (uint32_t h = 0; h < g.heads; ++h) bk[h * L2] = __float2half_rn(out[h] * 1.4426950408889634f);
}

// One CTA per leaf. Production shape (L = 128, edge_hidden = heads = 8): a pair's descriptors
// are its cell offset (dx, dy) = (Δcol / width, Δrow / height), |d| and the coupling A_ij, and
// A_ij = 0 for every pair but the row's few stencil neighbours. So the MLP runs once per distinct
// offset inside the leaf's bounding box (a 16 x 8 Morton block has 31 x 15 = 465 of them, against
// 16,384 pairs) into a shared-memory table of the 8 fp16 outputs, every pair copies its entry
// (one 16-byte shared load, coalesced fp16 stores), and the A_ij != 0 pairs are then recomputed
// with their coupling and overwritten (after a barrier, so the later store wins). The offsets are
// formed as Δ/width rounded once from f64 — the reference's f64 difference of the two centres,
// correctly rounded — instead of the difference of two rounded fp32 centres. Other shapes, or a
// box whose table would not fit, take the per-pair path below. (Per pair, 452 instructions
// issued at 0.83 IPC held this kernel at 151 us for the 8.4 M pairs at N = 65,536.)
constexpr int kBiasLutCap = 2048;  // 32 KB of fp16 x 8 entries
__global__ void __launch_bounds__(256) k_tn_leaf_bias(TnDims g, uint32_t lL, const uint32_t* order,
                                                      const unsigned long long* ro, const uint32_t* ci,
                                                      const double* v, EdgeMlp mlp, __half* bias) {
    const uint64_t k = blockIdx.x;
    const uint64_t base = k << lL;
    __shared__ float cx[128], cy[128];
    __shared__ int ax[128], ay[128];
    __shared__ uint4 lut[kBiasLutCap];
    __shared__ int box[4];
    const bool fast = lL == 7 && g.eh == 8 && g.heads == 8;
    if (threadIdx.x < 4) box[threadIdx.x] = (threadIdx.x & 1) ? -1 : 0x7fffffff;
    __syncthreads();
    for (uint64_t q = threadIdx.x; q < g.L && q < 128; q += blockDim.x) {
        const uint32_t a = order[base + q];
        // the leaf's node coordinates (frame.cpp cell centres, rounded once from f64) for the
        // per-pair path; its cell indices for the table
        cx[q] = float((double(a % g.width) + 0.5) / double(g.width));
        cy[q] = float((double(a / g.width) + 0.5) / double(g.height));
        ax[q] = int(a % g.width);
        ay[q] = int(a / g.width);
        if (fast) {
            atomicMin(&box[0], ax[q]);
            atomicMax(&box[1], ax[q]);
            atomicMin(&box[2], ay[q]);
            atomicMax(&box[3], ay[q]);
        }
    }
    __syncthreads();
    const int ex = box[1] - box[0], ey = box[3] - box[2], W = 2 * ex + 1, H = 2 * ey + 1;
    if (!fast || W * H > kBiasLutCap) {
        for (uint32_t idx = threadIdx.x; idx < (1u << (2 * lL)); idx += blockDim.x)  // i * L + j (L = 2^lL)
            leaf_bias_pair(g, lL, k, base, idx, cx, cy, order, ro, ci, v, mlp, bias);
        return;
    }
    auto mlp8 = [&](int ddx, int ddy, float c) {  // the 8 outputs x log2(e), packed fp16
        const float dx = float(double(ddx) / double(g.width)), dy = float(double(ddy) / double(g.height));
        const float dist = sqrtf(dx * dx + dy * dy);
        float out[8];
        edge_mlp_t<8, 8>(mlp, dx, dy, dist, c, out);
        uint4 p;
        __half2 h2[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
            h2[t] = __floats2half2_rn(out[2 * t] * 1.4426950408889634f, out[2 * t + 1] * 1.4426950408889634f);
        p.x = *reinterpret_cast<uint32_t*>(&h2[0]);
        p.y = *reinterpret_cast<uint32_t*>(&h2[1]);
        p.z = *reinterpret_cast<uint32_t*>(&h2[2]);
        p.w = *reinterpret_cast<uint32_t*>(&h2[3]);
        return p;
    };
    for (int e = threadIdx.x; e < W * H; e += blockDim.x) lut[e] = mlp8(e % W - ex, e / W - ey, 0.f);
    __syncthreads();
    constexpr uint64_t L2 = 1u << 14;
    __half* bk = bias + (k * 8) * L2;  // [k][h][i][j]
    for (uint32_t idx = 8 * threadIdx.x; idx < L2; idx += 8 * blockDim.x) {  // keys j .. j + 7 of query i
        const uint32_t i = idx >> 7, j0 = idx & 127u;
        __half hv[8][8];  // [key][head]
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint4 p = lut[(ax[i] - ax[j0 + t] + ex) + (ay[i] - ay[j0 + t] + ey) * W];
            const __half* hp = reinterpret_cast<const __half*>(&p);
#pragma unroll
            for (int h = 0; h < 8; ++h) hv[t][h] = hp[h];
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {  // one 16-byte store per head: the 8 keys' fp16 biases
            __half o[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) o[t] = hv[t][h];
            *reinterpret_cast<uint4*>(bk + h * L2 + idx) = *reinterpret_cast<const uint4*>(o);
        }
    }
    __syncthreads();  // the coupled pairs below overwrite their table entries
    if (threadIdx.x < 128) {
        const uint32_t i = threadIdx.x;
        for (unsigned long long p = ro[base + i], pe = ro[base + i + 1]; p < pe; ++p) {
            const uint32_t col = ci[p];
            if (col < base || col >= base + 128) continue;
            const uint32_t j = col - uint32_t(base);
            const uint4 q = mlp8(ax[i] - ax[j], ay[i] - ay[j], float(v[p]));
            const __half* hp = reinterpret_cast<const __half*>(&q);
#pragma unroll
            for (int h = 0; h < 8; ++h) bk[h * L2 + i * 128 + j] = hp[h];
        }
    }
}

// Chunk positions of every tile (toy_net.cpp:382-414 descriptors): pos[m][side][chunk] =
// (sum x, sum y) over the chunk's nodes (side 0: row chunks, 1: column chunks), f64. One CTA per
// (tile, side), one warp per chunk, lanes over the chunk's nodes, fixed-order reduction.
__global__ void k_tn_tile_pos(TnDims g, const uint32_t* order, double* pos) {
    const uint64_t m = blockIdx.x, side = blockIdx.y;
    const TileGeom t = tile_geom(g, m);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t base = side ? t.col0 : t.row0;
    for (uint64_t c = w; c < g.Ls; c += nw) {
        double sx = 0.0, sy = 0.0;
        for (uint64_t s = lane; s < t.chunk; s += 32) {
            const uint32_t id = order[base + c * t.chunk + s];
            sx += (double(id % g.width) + 0.5) / double(g.width);
            sy += (double(id / g.width) + 0.5) / double(g.height);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        if (lane == 0) {
            pos[((m * 2 + side) * g.Ls + c) * 2 + 0] = sx;
            pos[((m * 2 + side) * g.Ls + c) * 2 + 1] = sy;
        }
    }
}

// Tile-pair edge biases (toy_net.cpp:382-414): chunk-mean positions and the mean coupling over
// each (row chunk a, column chunk b) pair, stored query-major fp16 bias[m][h][a][b]. One CTA (64
// threads) per (tile, a): the a-chunk's CSR rows are split over the threads, each bins its
// column-band entries into a private column of partial sums, combined per bin in thread order.
__global__ void __launch_bounds__(64) k_tn_tile_bias(TnDims g, const double* pos, const unsigned long long* ro,
                                                    const uint32_t* ci, const double* v, EdgeMlp mlp,
                                                    __half* bias) {
    const uint64_t m = blockIdx.x, a = blockIdx.y;
    const TileGeom t = tile_geom(g, m);
    __shared__ double part[64][33];
    const int tid = threadIdx.x;
    for (uint32_t b = 0; b < g.Ls; ++b) part[tid][b] = 0.0;
    const uint64_t cbase = t.col0, cend = t.col0 + g.Ls * t.chunk;
    for (uint64_t s = tid; s < t.chunk; s += 64) {
        const uint64_t r = t.row0 + a * t.chunk + s;
        for (unsigned long long p = ro[r]; p < ro[r + 1]; ++p)
            if (ci[p] >= cbase && ci[p] < cend) part[tid][(ci[p] - cbase) / t.chunk] += v[p];
    }
    __syncthreads();
    if (tid < int(g.Ls)) {
        double c = 0.0;
        for (int q = 0; q < 64; ++q) c += part[q][tid];
        const double ch = double(t.chunk);
        const double* rp = pos + ((m * 2 + 0) * g.Ls + a) * 2;
        const double* cp = pos + ((m * 2 + 1) * g.Ls + tid) * 2;
        const double dx = (rp[0] - cp[0]) / ch, dy = (rp[1] - cp[1]) / ch;
        const double dist = sqrt(dx * dx + dy * dy);
        c /= ch * ch;
        float out[8];
        edge_mlp(mlp, g.eh, g.heads, float(dx), float(dy), float(dist), float(c), out);
        for (uint32_t h = 0; h < g.heads; ++h)  // query a (row chunk), key tid (column chunk)
            bias[((m * g.heads + h) * g.Ls + a) * g.Ls + tid] = __float2half_rn(out[h] * 1.4426950408889634f);
    }
}

// toy_net.cpp:348-365 tile tokens: mean over each token's chunk of (row_emb + col_emb) / 2.
__global__ void k_tn_tile_pool(TnDims g, const float* emb, float* tile_tok) {
    const uint64_t m = blockIdx.x, tok = blockIdx.y;
    const TileGeom t = tile_geom(g, m);
    for (uint32_t c = threadIdx.x; c < g.d; c += blockDim.x) {
        const float rs = strided_sum(emb + (t.row0 + tok * t.chunk) * g.d + c, t.chunk, g.d);
        const float cs = strided_sum(emb + (t.col0 + tok * t.chunk) * g.d + c, t.chunk, g.d);
        tile_tok[(m * g.Ls + tok) * g.d + c] = 0.5f * (rs + cs) / float(t.chunk);
    }
}

// Windowed multi-head attention core (toy_net.cpp:78-125) for one (block, head): T tokens,
// head dim 16. qkv rows hold [q | k | v] (3d wide). One thread per query row; K/V of the block
// head staged in shared memory; the thread's fp16 bias row read along the keys; softmax in fp32 with an online (rescaled) running max, i.e. one pass over the
// keys. Writes head_out[row, h*16..]. With rowsum_err_bits (trace) a second pass audits
// max |row sum - 1| of the normalised probabilities.
template <int T>
__global__ void __launch_bounds__(T) k_tn_attention(uint32_t d, uint32_t heads, const float* qkv,
                                                    const __half* bias, float* head_out,
                                                    unsigned int* rowsum_err_bits) {
    const uint64_t blk = blockIdx.x;
    const uint32_t h = blockIdx.y, i = threadIdx.x;
    constexpr int HD = 16;
    __shared__ float4 ks[T][HD / 4], vs[T][HD / 4];
    const float4* rowp = reinterpret_cast<const float4*>(qkv + (blk * T + i) * 3 * d);
    float4 q4[HD / 4];
#pragma unroll
    for (int c = 0; c < HD / 4; ++c) {
        q4[c] = rowp[(h * HD) / 4 + c];
        ks[i][c] = rowp[(d + h * HD) / 4 + c];
        vs[i][c] = rowp[(2 * d + h * HD) / 4 + c];
    }
    __syncthreads();
    const __half* b = bias + ((blk * heads + h) * T + i) * T;  // query row i of the bias
    const float scale = 0.25f;  // 1/sqrt(16)
    auto logit = [&](int j) {
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < HD / 4; ++c) {
            const float4 k = ks[j][c];
            dot = fmaf(q4[c].x, k.x, dot);
            dot = fmaf(q4[c].y, k.y, dot);
            dot = fmaf(q4[c].z, k.z, dot);
            dot = fmaf(q4[c].w, k.w, dot);
        }
        return fmaf(dot, scale, __half2float(b[j]) * 0.69314718055994531f);  // bias stored x log2(e)
    };
    float mx = -CUDART_INF_F, sum = 0.f;
    float4 acc[HD / 4];
#pragma unroll
    for (int c = 0; c < HD / 4; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < T; ++j) {
        const float sj = logit(j);
        if (sj > mx) {  // rescale the running sums to the new max
            const float r = expf(mx - sj);
            sum *= r;
#pragma unroll
            for (int c = 0; c < HD / 4; ++c) {
                acc[c].x *= r; acc[c].y *= r; acc[c].z *= r; acc[c].w *= r;
            }
            mx = sj;
        }
        const float p = expf(sj - mx);
        sum += p;
#pragma unroll
        for (int c = 0; c < HD / 4; ++c) {
            const float4 v = vs[j][c];
            acc[c].x = fmaf(p, v.x, acc[c].x);
            acc[c].y = fmaf(p, v.y, acc[c].y);
            acc[c].z = fmaf(p, v.z, acc[c].z);
            acc[c].w = fmaf(p, v.w, acc[c].w);
        }
    }
    const float inv = 1.f / sum;
    float4* o = reinterpret_cast<float4*>(head_out + (blk * T + i) * d + h * HD);
#pragma unroll
    for (int c = 0; c < HD / 4; ++c) o[c] = make_float4(acc[c].x * inv, acc[c].y * inv, acc[c].z * inv, acc[c].w * inv);
    if (rowsum_err_bits) {  // row sum of the normalised probabilities, as the trace audits
        float rs = 0.f;
        for (int j = 0; j < T; ++j) rs += expf(logit(j) - mx) * inv;
        atomicMax(rowsum_err_bits, __float_as_uint(fabsf(rs - 1.f)));
    }
}

// Highway scatter (toy_net.cpp:451-476) as an ancestor gather: row_hw[i] = leaf_tok[i] + the
// tile token covering i in the row half of every ancestor tile; col_hw likewise for column
// halves. One warp per node, lane owns 4 channels.
__global__ void k_tn_highway(TnDims g, const float* leaf_tok, const float* tile_tok, float* row_hw,
                             float* col_hw) {
    constexpr int kMaxD = 20;
    const uint32_t i = uint32_t((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= g.n) return;
    // all sizes are powers of two: leaf = i >> log L; the depth-dd ancestor's chunk holds
    // 2^(D-dd-1) * L / L_s rows, so the covering token is (i mod 2^(D-dd) L) >> log chunk, less
    // L_s in the column half
    int lL = 0, lLs = 0;
    while ((1u << lL) < g.L) ++lL;
    while ((1u << lLs) < g.Ls) ++lLs;
    const uint32_t D = uint32_t(g.D), K = uint32_t(g.K), leaf = i >> lL;
    float4 e[kMaxD];
#pragma unroll
    for (int dd = 0; dd < kMaxD; ++dd) {  // every ancestor's covering tile token, loads first
        e[dd] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (uint32_t(dd) < D) {
            const uint32_t m = ((K + leaf) >> (D - dd)) - 1u;
            const uint32_t within = i & ((1u << (D - dd + lL)) - 1u);  // offset inside the tile
            const uint32_t tok = (within >> (D - dd - 1 + lL - lLs)) & (uint32_t(g.Ls) - 1u);
            e[dd] = __ldg(reinterpret_cast<const float4*>(tile_tok + (uint64_t(m) * g.Ls + tok) * g.d) + lane);
        }
    }
    const float4 lt = reinterpret_cast<const float4*>(leaf_tok + uint64_t(i) * g.d)[lane];
    float4 r = lt, c = lt;
#pragma unroll
    for (int dd = 0; dd < kMaxD; ++dd)
        if (uint32_t(dd) < D) {
            float4& dst = ((leaf >> (D - 1 - dd)) & 1u) ? c : r;
            dst.x += e[dd].x; dst.y += e[dd].y; dst.z += e[dd].z; dst.w += e[dd].w;
        }
    reinterpret_cast<float4*>(row_hw + uint64_t(i) * g.d)[lane] = r;
    reinterpret_cast<float4*>(col_hw + uint64_t(i) * g.d)[lane] = c;
}

// The same scatter by level-0 chunks (c0 = L / L_s nodes share every ancestor's covering tile
// token): one warp per chunk sums the D ancestors' tokens into a row-side and a column-side
// accumulator (depth dd: the chunk's tile m, half and token from the chunk index at level
// l = D - 1 - dd), then writes t + acc for each of its c0 nodes — D gathers per c0 nodes instead
// of per node.
// Also the leaf half of glob_hw (toy_net.cpp:458): the CTA's column sums of the leaf tokens it
// reads anyway, one fixed-order partial per CTA in colsum_part (finished by k_tn_colsum_finish).
__global__ void __launch_bounds__(256) k_tn_highway_chunks(TnDims g, uint32_t c0, const float* leaf_tok,
                                                           const float* tile_tok, float* row_hw, float* col_hw,
                                                           float* colsum_part) {
    __shared__ float4 wsum[8][32];
    const uint64_t j0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float4 ts = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j0 * c0 < g.n) {
    const uint32_t D = uint32_t(g.D);
    float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ac = ar;
#pragma unroll 4
    for (uint32_t l = 0; l < D; ++l) {  // all gathers independent
        const uint64_t jl = j0 >> l, it = jl / (2 * g.Ls), a = jl % g.Ls;
        const uint32_t dd = D - 1 - l;
        const uint64_t m = ((uint64_t(1) << dd) - 1) + it;
        const float4 e = __ldg(reinterpret_cast<const float4*>(tile_tok + (m * g.Ls + a) * g.d) + lane);
        float4& dst = ((jl / g.Ls) & 1) ? ac : ar;
        dst.x += e.x; dst.y += e.y; dst.z += e.z; dst.w += e.w;
    }
    for (uint32_t q = 0; q < c0; ++q) {
        const uint64_t i = j0 * c0 + q;
        const float4 t = reinterpret_cast<const float4*>(leaf_tok + i * g.d)[lane];
        reinterpret_cast<float4*>(row_hw + i * g.d)[lane] = make_float4(t.x + ar.x, t.y + ar.y, t.z + ar.z, t.w + ar.w);
        reinterpret_cast<float4*>(col_hw + i * g.d)[lane] = make_float4(t.x + ac.x, t.y + ac.y, t.z + ac.z, t.w + ac.w);
        ts.x += t.x; ts.y += t.y; ts.z += t.z; ts.w += t.w;
    }
    }
    wsum[warp][lane] = ts;
    __syncthreads();
    if (threadIdx.x < 32) {
        float4 a = wsum[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) {
            const float4 b = wsum[w][threadIdx.x];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        reinterpret_cast<float4*>(colsum_part + uint64_t(blockIdx.x) * g.d)[threadIdx.x] = a;
    }
}

// glob_hw = sum of every leaf token + every tile token (toy_net.cpp:458, 474). Column sums via
// per-block partials (deterministic), then a single-block finish.
__global__ void k_tn_colsum_partial(uint64_t rows, uint32_t d, const float* x, float* partial) {
    const uint32_t c = threadIdx.x;  // blockDim.x == d; block b sums rows b, b + grid, ...
    const uint64_t cnt = rows > blockIdx.x ? (rows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    partial[uint64_t(blockIdx.x) * d + c] = strided_sum(x + uint64_t(blockIdx.x) * d + c, cnt, uint64_t(gridDim.x) * d);
}
// Tile-token column sums weighted by each token's chunk length (the number of highway rows it
// is scattered to), for the conservation audit.
__global__ void k_tn_colsum_tiles_weighted(TnDims g, const float* tile_tok, float* partial) {
    const uint32_t c = threadIdx.x;
    float s = 0.f;
    for (uint64_t r = blockIdx.x; r < g.M * g.Ls; r += gridDim.x)
        s += tile_tok[r * g.d + c] * float(tile_geom(g, r / g.Ls).chunk);
    partial[uint64_t(blockIdx.x) * g.d + c] = s;
}
// Highway conservation (toy_net.cpp:478-512) from column sums: sums[0..5] = row_hw, col_hw,
// leaf tokens, tile tokens, chunk-weighted tile tokens, glob_hw -> dev / scale.
__global__ void k_tn_highway_audit(uint32_t d, const float* sums, float* out_layer) {
    __shared__ float dev[128], sc[128];
    const uint32_t c = threadIdx.x;
    const float gr = sums[c], gc = sums[d + c], lt = sums[2 * d + c], tt = sums[3 * d + c],
                ttw = sums[4 * d + c], gg = sums[5 * d + c];
    const float er = lt + ttw, eg = lt + tt;
    dev[c] = fmaxf(fmaxf(fabsf(gr - er), fabsf(gc - er)), fabsf(gg - eg));
    sc[c] = fmaxf(fmaxf(fabsf(er), fabsf(eg)), 1.f);
    __syncthreads();
    if (c == 0) {
        float dm = 0.f, sm = 0.f;
        for (uint32_t i = 0; i < d; ++i) {
            dm = fmaxf(dm, dev[i]);
            sm = fmaxf(sm, sc[i]);
        }
        *out_layer = dm / sm;
    }
}

// Column totals of the per-block partials (f64, fixed order): block c sums column c, each of
// its 32 lanes a strided share, then a butterfly.
__global__ void k_tn_colsum_finish(uint32_t nparts, uint32_t d, const float* partial, float* out) {
    const uint32_t c = blockIdx.x, lane = threadIdx.x;
    double s = 0.0;
    for (uint32_t b = lane; b < nparts; b += 32) s += partial[uint64_t(b) * d + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = float(s);
}

// Tile FFN strip means walked chunk by chunk (toy_net.cpp:519-532), for partitions whose chunks
// do not nest as powers of two (L < L_s); the production shapes use k_tn_tile_means_pyr.
__global__ void k_tn_tile_means_walk(TnDims g, const float* row_hw, const float* col_hw, float* rmean,
                                     float* cmean) {
    const uint64_t m = blockIdx.x, tok = blockIdx.y;
    const TileGeom t = tile_geom(g, m);
    for (uint32_t c = threadIdx.x; c < g.d; c += blockDim.x) {
        const float rs = strided_sum(row_hw + (t.row0 + tok * t.chunk) * g.d + c, t.chunk, g.d);
        const float cs = strided_sum(col_hw + (t.col0 + tok * t.chunk) * g.d + c, t.chunk, g.d);
        rmean[(m * g.Ls + tok) * g.d + c] = rs / float(t.chunk);
        cmean[(m * g.Ls + tok) * g.d + c] = cs / float(t.chunk);
    }
}

// ---- chunk-sum pyramids: O(N d) strip pooling and chunk means --------------------------
// Every tile of span s leaves splits its row and column halves into L_s chunks of c = s L / L_s
// consecutive nodes (toy_net.cpp:352-353). Chunk sizes are c0 2^l (c0 = L / L_s, l = log2 s) and
// chunks nest: level l of a pyramid holds the sums of c0 2^l consecutive rows, level l + 1 the
// pairwise sums of level l. Tile pooling (toy_net.cpp:348-365), the tile FFN's strip means
// (:519-537) and the tile descriptors' chunk positions (:382-414) then read one pyramid entry per
// (tile, token) instead of walking the chunk: O(N d) per pyramid instead of O(N d log K).
template <class T>
struct PyrLevels {
    T* lev[24];
};
// One launch produces levels l0 .. l0 + q: block b of (group << q) <= 32 source rows; a thread
// owns VW consecutive channels of one block, loads all its rows first (up to 32 vector loads in
// flight), then forms level l0 (sums of `group` rows) and each level above as pairwise sums.
__device__ __forceinline__ float4 vadd(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ double2 vadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
template <class T, class V, uint32_t group>
__global__ void __launch_bounds__(128) k_tn_pyramid(const T* __restrict__ src, uint64_t nblocks, uint32_t C,
                                                    uint32_t q, PyrLevels<T> out, uint32_t l0) {
    constexpr uint32_t VW = sizeof(V) / sizeof(T);
    const uint32_t cv = C / VW;
    const uint64_t gid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t blk = gid / cv;
    const uint32_t c = uint32_t(gid % cv);
    if (blk >= nblocks) return;
    const uint32_t rows = group << q;
    const V* s = reinterpret_cast<const V*>(src) + blk * rows * cv + c;
    V r[32];
#pragma unroll
    for (uint32_t i = 0; i < 32; ++i)
        if (i < rows) r[i] = s[uint64_t(i) * cv];
    // level l0: r[j] = sum of rows j*group .. j*group+group-1 (in order), in place
    const uint32_t n0 = 1u << q;
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) {
        if (j < n0) {
            V a = r[j * group];
#pragma unroll
            for (uint32_t gg = 1; gg < group; ++gg) a = vadd(a, r[j * group + gg]);
            r[j] = a;  // j * group >= j: reads ahead of the writes
        }
    }
    for (uint32_t l = 0; l <= q; ++l) {
        const uint32_t cnt = n0 >> l;
        V* o = reinterpret_cast<V*>(out.lev[l0 + l]) + ((blk << q) >> l) * cv + c;
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < cnt) o[uint64_t(j) * cv] = r[j];
        if (l < q) {
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j)
                if (j < cnt / 2) r[j] = vadd(r[2 * j], r[2 * j + 1]);
        }
    }
}

// Tile token (m, a) from the embedding pyramid: 0.5 (row chunk sum + column chunk sum) / c
// (toy_net.cpp:356-364). lev_shift = log2(L / L_s).
// One warp per tile token (d = 128: a float4 per lane).
__global__ void k_tn_tile_pool_pyr(TnDims g, PyrLevels<float> P, uint32_t lev_shift, float* tile_tok) {
    const uint64_t tok = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (tok >= g.M * g.Ls) return;
    const uint64_t m = tok / g.Ls, a = tok % g.Ls;
    const TileGeom t = tile_geom(g, m);
    int l = 0;
    while ((uint64_t(1) << (l + lev_shift)) < t.chunk) ++l;
    const float4 r = reinterpret_cast<const float4*>(P.lev[l] + (t.row0 / t.chunk + a) * g.d)[lane];
    const float4 c = reinterpret_cast<const float4*>(P.lev[l] + (t.col0 / t.chunk + a) * g.d)[lane];
    const float inv = 1.f / float(t.chunk);  // a power of two: exact
    reinterpret_cast<float4*>(tile_tok + tok * g.d)[lane] =
        make_float4(0.5f * (r.x + c.x) * inv, 0.5f * (r.y + c.y) * inv, 0.5f * (r.z + c.z) * inv, 0.5f * (r.w + c.w) * inv);
}

// Tile FFN strip means (toy_net.cpp:519-532): rmean = row_hw chunk sum / c over the token's row
// chunk, cmean = col_hw chunk sum / c over its column chunk; rows of the tile FFN's K-sliced
// input (sources 1 and 2).
__global__ void k_tn_tile_means_pyr(TnDims g, PyrLevels<float> Pr, PyrLevels<float> Pc, uint32_t lev_shift,
                                    float* rmean, float* cmean) {
    const uint64_t tok = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // warp per tile token
    const int lane = threadIdx.x & 31;
    if (tok >= g.M * g.Ls) return;
    const uint64_t m = tok / g.Ls, a = tok % g.Ls;
    const TileGeom t = tile_geom(g, m);
    int l = 0;
    while ((uint64_t(1) << (l + lev_shift)) < t.chunk) ++l;
    const float4 r = reinterpret_cast<const float4*>(Pr.lev[l] + (t.row0 / t.chunk + a) * g.d)[lane];
    const float4 c = reinterpret_cast<const float4*>(Pc.lev[l] + (t.col0 / t.chunk + a) * g.d)[lane];
    const float inv = 1.f / float(t.chunk);
    reinterpret_cast<float4*>(rmean + tok * g.d)[lane] = make_float4(r.x * inv, r.y * inv, r.z * inv, r.w * inv);
    reinterpret_cast<float4*>(cmean + tok * g.d)[lane] = make_float4(c.x * inv, c.y * inv, c.z * inv, c.w * inv);
}

// Node positions (frame.cpp cell centres, toy_net.cpp:333-338) as f64 pairs, the input of the
// position pyramid.
__global__ void k_tn_positions(TnDims g, const uint32_t* order, double* pos) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const uint32_t id = order[i];
    pos[2 * i] = (double(id % g.width) + 0.5) / double(g.width);
    pos[2 * i + 1] = (double(id / g.width) + 0.5) / double(g.height);
}
// Chunk position sums of every tile from the position pyramid, in k_tn_tile_bias's layout
// pos[m][side][chunk][x|y].
__global__ void k_tn_tile_pos_pyr(TnDims g, PyrLevels<double> P, uint32_t lev_shift, double* pos) {
    const uint64_t m = blockIdx.x;
    const TileGeom t = tile_geom(g, m);
    int l = 0;
    while ((uint64_t(1) << (l + lev_shift)) < t.chunk) ++l;
    for (uint32_t q = threadIdx.x; q < 2 * g.Ls; q += blockDim.x) {
        const uint32_t side = q / g.Ls, a = q % g.Ls;
        const double* e = P.lev[l] + ((side ? t.col0 : t.row0) / t.chunk + a) * 2;
        pos[((m * 2 + side) * g.Ls + a) * 2 + 0] = e[0];
        pos[((m * 2 + side) * g.Ls + a) * 2 + 1] = e[1];
    }
}

// The FFN's glob slice as a bias (toy_net.cpp:428-430: every row of a layer's FFN input carries
// the same glob_hw in columns [3d, 4d)): bias[o] = sum_i glob[i] W1[3d + i][o], once per layer
// and stream instead of a K = d slice of every row's product. w1t is W1^T (4d x 4d, out x in).
__global__ void k_tn_glob_bias(uint32_t d, const float* glob, const float* w1t_leaf, const float* w1t_tile,
                               float* bias_leaf, float* bias_tile) {
    const uint32_t o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;  // warp per output
    if (o >= 4 * d) return;
    const float* w = (blockIdx.y ? w1t_tile : w1t_leaf) + uint64_t(o) * 4 * d + 3 * d;
    double a = 0.0;
    for (uint32_t i = lane; i < d; i += 32) a = fma(double(glob[i]), double(w[i]), a);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) a += __shfl_xor_sync(0xffffffffu, a, s);
    if (lane == 0) (blockIdx.y ? bias_tile : bias_leaf)[o] = float(a);
}

// ---- global statistics of a device frame (toy_net.cpp:232-268) --------------------------
// Fixed partition into kStatParts blocks, fixed-order combination: deterministic.
constexpr int kStatParts = 296, kStatFields = 7;  // rho sum, diag sum/min/max, |offdiag| sum/count, rho sq dev
__device__ __forceinline__ double block_reduce_d(double v, int op, double* sh) {  // op 0 sum, 1 min, 2 max
    for (int o = 16; o; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, v, o);
        v = op == 0 ? v + t : (op == 1 ? fmin(v, t) : fmax(v, t));
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = sh[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) r = op == 0 ? r + sh[w] : (op == 1 ? fmin(r, sh[w]) : fmax(r, sh[w]));
    __syncthreads();
    return r;
}
__global__ void __launch_bounds__(256) k_tn_frame_stats(uint64_t n, const double* __restrict__ rho,
                                                        const unsigned long long* __restrict__ ro,
                                                        const uint32_t* __restrict__ ci, const double* __restrict__ v,
                                                        const double* __restrict__ diag, double* __restrict__ part) {
    __shared__ double sh[8];
    const uint64_t per = (n + kStatParts - 1) / kStatParts, r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double rs = 0.0, ds = 0.0, dmn = INFINITY, dmx = -INFINITY, os = 0.0, oc = 0.0;
    for (uint64_t i = r0 + threadIdx.x; i < r1; i += 256) {
        rs += rho[i];
        const double dd = diag[i];
        ds += dd;
        dmn = fmin(dmn, dd);
        dmx = fmax(dmx, dd);
        for (unsigned long long p = ro[i]; p < ro[i + 1]; ++p)
            if (ci[p] != i) {
                os += fabs(v[p]);
                oc += 1.0;
            }
    }
    double* o = part + uint64_t(blockIdx.x) * kStatFields;
    rs = block_reduce_d(rs, 0, sh);
    ds = block_reduce_d(ds, 0, sh);
    dmn = block_reduce_d(dmn, 1, sh);
    dmx = block_reduce_d(dmx, 2, sh);
    os = block_reduce_d(os, 0, sh);
    oc = block_reduce_d(oc, 0, sh);
    if (threadIdx.x == 0) {
        o[0] = rs;
        o[1] = ds;
        o[2] = dmn;
        o[3] = dmx;
        o[4] = os;
        o[5] = oc;
    }
}
__global__ void __launch_bounds__(256) k_tn_frame_var(uint64_t n, const double* __restrict__ rho, double* __restrict__ part) {
    __shared__ double sh[8];
    double tot = 0.0;  // every block recombines the rho partial sums in the same order
    for (int b = 0; b < kStatParts; ++b) tot += part[uint64_t(b) * kStatFields];
    const double mean = tot / double(n);
    const uint64_t per = (n + kStatParts - 1) / kStatParts, r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    double q = 0.0;
    for (uint64_t i = r0 + threadIdx.x; i < r1; i += 256) q += (rho[i] - mean) * (rho[i] - mean);
    q = block_reduce_d(q, 0, sh);
    if (threadIdx.x == 0) part[uint64_t(blockIdx.x) * kStatFields + 6] = q;
}
__global__ void k_tn_frame_finish(uint64_t n, uint64_t nnz, uint64_t width, uint64_t height, double rho_heavy,
                                  const double* __restrict__ part, uint32_t dglob, float* __restrict__ glob) {
    if (threadIdx.x != 0) return;
    double a[kStatFields] = {0, 0, INFINITY, -INFINITY, 0, 0, 0};
    for (int b = 0; b < kStatParts; ++b) {
        const double* o = part + uint64_t(b) * kStatFields;
        a[0] += o[0];
        a[1] += o[1];
        a[2] = fmin(a[2], o[2]);
        a[3] = fmax(a[3], o[3]);
        a[4] += o[4];
        a[5] += o[5];
        a[6] += o[6];
    }
    const double dn = double(n);
    const double stats[12] = {log(dn), a[0] / dn, sqrt(a[6] / dn), log(fmax(rho_heavy, 1.0)), a[1] / dn, a[3], a[2],
                              a[5] > 0.0 ? a[4] / a[5] : 0.0, double(nnz) / dn, double(width) / double(height),
                              a[3] / fmax(a[2], 1e-30), 1.0};
    for (uint32_t i = 0; i < (dglob > 0 ? dglob : 1u); ++i) glob[i] = i < 12 && i < dglob ? float(stats[i]) : 0.f;
}

}  // namespace hfpg
