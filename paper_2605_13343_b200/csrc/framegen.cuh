// GPU frame generator: make_frame (frame.cpp:161-181) and the 3D analogue, written straight
// into device memory and loaded as the handle's system (SELL-32 operator, diagonal, |A|_F, b).
//
// Integer work is bit-identical to the host generator (Morton order, CSR structure). Floating
// values are bit-identical to the host generator built on a correctly rounded libm
// (HFPG_FRAME_CRMATH=1, crmath.cuh) — glibc's log/cos are off by one ulp on ~0.16% of draws, so
// against the default host build the normals differ there by one ulp (tests/test_gpu_framegen.py).
//
// Kernels, in stream order:
//   k_fg_rank      cell id -> Morton rank by counting the grid cells in the quadrants/octants
//                  that precede it at every level (no sort); cell_order[rank] = id, rank_of[id]
//   k_fg_cells     per retained cell: rho (barriers + noise normal), row length, rhs normal
//   scan           row lengths -> row_offsets (exclusive, u64)
//   k_fg_assemble  per row: harmonic-mean weights in neighbour order, diagonal, column sort
//   k_fg_chain     the reference's two sequential sums (sum b, sum v^2), one thread each on two
//                  side streams, overlapping the rest; associativity-sensitive, so they stay serial
//   k_fg_center    b -= mean
//   SELL-32        slice widths -> scan -> fill (csr -> the layout k_spmv / k_solve read)
#pragma once
#include "crmath.cuh"

namespace hfpg {

struct FgBarrier {
    int axis, gap;
    double center, thickness;
};
struct FgParams {
    int dims, nb;
    uint32_t levels;  // Morton levels: 2^levels >= max(W, H, D)
    unsigned long long n, W, H, D;
    double rho_heavy;
    unsigned long long density_key, c0, rhs_key;
    FgBarrier bars[3];
};

constexpr uint32_t kFgNone = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long fg_mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long fg_ext(unsigned long long lim, unsigned long long o,
                                                     unsigned long long s) {
    return o >= lim ? 0ULL : (lim - o < s ? lim - o : s);
}

// Number of grid cells whose Morton key is below (x, y, z)'s: at each level the cell's
// quadrant/octant q (x bit 0, y bit 1, z bit 2, as spread2/spread3 interleave) is preceded by the
// sibling blocks q' < q, each contributing its clipped extent.
__device__ __forceinline__ unsigned long long fg_morton_rank(const FgParams& P, uint32_t x, uint32_t y,
                                                             uint32_t z) {
    unsigned long long rank = 0, ox = 0, oy = 0, oz = 0;
    for (int b = int(P.levels) - 1; b >= 0; --b) {
        const unsigned long long s = 1ULL << b;
        const uint32_t q = ((x >> b) & 1u) | (((y >> b) & 1u) << 1) | (((z >> b) & 1u) << 2);
        for (uint32_t qq = 0; qq < q; ++qq) {
            const unsigned long long ex = fg_ext(P.W, ox + (qq & 1u) * s, s);
            const unsigned long long ey = fg_ext(P.H, oy + ((qq >> 1) & 1u) * s, s);
            const unsigned long long ez = P.dims == 3 ? fg_ext(P.D, oz + (qq >> 2) * s, s) : 1ULL;
            rank += ex * ey * ez;
        }
        ox += (q & 1u) * s;
        oy += ((q >> 1) & 1u) * s;
        oz += (q >> 2) * s;
    }
    return rank;
}

__global__ void k_fg_rank(FgParams P, uint32_t* __restrict__ cell_order, uint32_t* __restrict__ rank_of) {
    const unsigned long long cells = P.W * P.H * P.D;
    for (unsigned long long id = blockIdx.x * 256ULL + threadIdx.x; id < cells; id += gridDim.x * 256ULL) {
        const uint32_t x = uint32_t(id % P.W), y = uint32_t((id / P.W) % P.H), z = uint32_t(id / (P.W * P.H));
        const unsigned long long r = fg_morton_rank(P, x, y, z);
        if (r < P.n) {
            cell_order[r] = uint32_t(id);
            rank_of[id] = uint32_t(r);
        } else {
            rank_of[id] = kFgNone;
        }
    }
}

// Neighbour ranks of cell id in the reference's order (x-1, x+1, y-1, y+1[, z-1, z+1]); kFgNone
// where the neighbour is off the grid or not retained.
__device__ __forceinline__ void fg_neighbours(const FgParams& P, const uint32_t* __restrict__ rank_of,
                                              uint32_t id, uint32_t nb[6]) {
    const unsigned long long W = P.W, H = P.H, D = P.D;
    const uint32_t x = uint32_t(id % W), y = uint32_t((id / W) % H), z = uint32_t(id / (W * H));
    nb[0] = x > 0 ? rank_of[id - 1] : kFgNone;
    nb[1] = x + 1 < W ? rank_of[id + 1] : kFgNone;
    nb[2] = y > 0 ? rank_of[id - W] : kFgNone;
    nb[3] = y + 1 < H ? rank_of[id + W] : kFgNone;
    if (P.dims == 3) {
        nb[4] = z > 0 ? rank_of[id - W * H] : kFgNone;
        nb[5] = z + 1 < D ? rank_of[id + W * H] : kFgNone;
    } else {
        nb[4] = nb[5] = kFgNone;
    }
}

// frame.cpp:60-79 in_heavy_region
__device__ __forceinline__ bool fg_heavy_at(double cross, double along, const FgBarrier& b) {
    if (fabs(__dsub_rn(cross, b.center)) > __dmul_rn(0.5, b.thickness)) return false;
    switch (b.gap) {
        case 0: return along < 0.8;
        case 1: return along > 0.2;
        case 2: return along < 0.4 || along > 0.6;
        default: return true;
    }
}

// rho (frame.cpp:171-179 / the 3D slabs), row length, and the uncentred rhs normal.
__global__ void k_fg_cells(FgParams P, const uint32_t* __restrict__ cell_order,
                           const uint32_t* __restrict__ rank_of, double* __restrict__ rho,
                           uint32_t* __restrict__ len, double* __restrict__ b) {
    for (unsigned long long i = blockIdx.x * 256ULL + threadIdx.x; i < P.n; i += gridDim.x * 256ULL) {
        const uint32_t id = cell_order[i];
        const unsigned long long W = P.W, H = P.H;
        const double c[3] = {__ddiv_rn(__dadd_rn(double(id % W), 0.5), double(W)),
                             __ddiv_rn(__dadd_rn(double((id / W) % H), 0.5), double(H)),
                             __ddiv_rn(__dadd_rn(double(id / (W * H)), 0.5), double(P.D))};
        bool heavy = false;
        for (int k = 0; k < P.nb && !heavy; ++k) {
            const FgBarrier& br = P.bars[k];
            heavy = fg_heavy_at(c[br.axis], c[(br.axis + 1) % P.dims], br);
        }
        // 1.0 + 0.05 * normal: the host build (-march=x86-64-v3, -ffp-contract=fast) fuses it
        const double g = crm::normal_of_cr(fg_mix64(P.density_key ^ (P.c0 + i)));
        const double t = __fma_rn(0.05, g, 1.0);
        const double noise = 0.5 < t ? t : 0.5;
        rho[i] = __dmul_rn(heavy ? P.rho_heavy : 1.0, noise);
        uint32_t nb[6];
        fg_neighbours(P, rank_of, id, nb);
        uint32_t l = 1;
        for (int q = 0; q < 6; ++q) l += nb[q] != kFgNone;
        len[i] = l;
        b[i] = crm::normal_of_cr(fg_mix64(P.rhs_key ^ i));
    }
}

// frame.cpp:100-145 assemble_operator: w = 2 rho_i rho_j / (rho_i + rho_j) in neighbour order,
// diagonal = sum of w (same order), columns sorted.
__global__ void k_fg_assemble(FgParams P, const uint32_t* __restrict__ cell_order,
                              const uint32_t* __restrict__ rank_of, const double* __restrict__ rho,
                              const unsigned long long* __restrict__ ro, uint32_t* __restrict__ ci,
                              double* __restrict__ vals, double* __restrict__ a_diag,
                              unsigned* __restrict__ nonpositive) {
    for (unsigned long long i = blockIdx.x * 256ULL + threadIdx.x; i < P.n; i += gridDim.x * 256ULL) {
        uint32_t nb[6];
        fg_neighbours(P, rank_of, cell_order[i], nb);
        const double ri = rho[i];
        uint32_t col[7];
        double val[7];
        int cnt = 0;
        double diag = 0.0;
        for (int q = 0; q < 6; ++q) {
            if (nb[q] == kFgNone) continue;
            const double rj = rho[nb[q]];
            const double w = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, ri), rj), __dadd_rn(ri, rj));
            diag = __dadd_rn(diag, w);
            col[cnt] = nb[q];
            val[cnt] = -w;
            ++cnt;
        }
        col[cnt] = uint32_t(i);
        val[cnt] = diag;
        ++cnt;
        for (int a = 1; a < cnt; ++a)  // insertion sort by column (distinct)
            for (int k = a; k > 0 && col[k - 1] > col[k]; --k) {
                const uint32_t tc = col[k];
                col[k] = col[k - 1];
                col[k - 1] = tc;
                const double tv = val[k];
                val[k] = val[k - 1];
                val[k - 1] = tv;
            }
        const unsigned long long p0 = ro[i];
        for (int k = 0; k < cnt; ++k) {
            ci[p0 + k] = col[k];
            vals[p0 + k] = val[k];
        }
        a_diag[i] = diag;
        if (!(diag > 0.0)) atomicAdd(nonpositive, 1u);
    }
}

// One of the reference's sequential sums, by one thread (launched as a single CTA on a side
// stream): sum of b (frame.cpp:147-152) or sum of v*v over the CSR values (csr.cpp:64-68, fused
// multiply-add as the host build contracts it). Associativity-sensitive, so it stays serial; the
// CTA's other threads stage 2 x 2048 values through shared memory ahead of the summing thread.
constexpr int kFgChainThreads = 256, kFgChainTile = 2048;
__global__ void __launch_bounds__(kFgChainThreads) k_fg_chain(const double* __restrict__ src,
                                                              unsigned long long cnt,
                                                              const unsigned long long* __restrict__ cnt_dev,
                                                              int squares, double* __restrict__ out) {
    __shared__ double buf[2][kFgChainTile];
    if (cnt_dev) cnt = *cnt_dev;
    double acc = 0.0;
    const unsigned long long tiles = (cnt + kFgChainTile - 1) / kFgChainTile;
    auto load = [&](unsigned long long t, int s) {
        for (int j = threadIdx.x; j < kFgChainTile; j += kFgChainThreads) {
            const unsigned long long e = t * kFgChainTile + j;
            buf[s][j] = e < cnt ? src[e] : 0.0;
        }
    };
    if (tiles) load(0, 0);
    __syncthreads();
    for (unsigned long long t = 0; t < tiles; ++t) {
        const int s = int(t & 1);
        if (t + 1 < tiles) load(t + 1, s ^ 1);
        if (threadIdx.x == 0) {
            const int m = int(cnt - t * kFgChainTile < kFgChainTile ? cnt - t * kFgChainTile : kFgChainTile);
            const double* x = buf[s];
            if (squares) {
#pragma unroll 16
                for (int j = 0; j < m; ++j) acc = __fma_rn(x[j], x[j], acc);
            } else {
#pragma unroll 16
                for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, x[j]);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = acc;
}

__global__ void k_fg_center(double* __restrict__ b, unsigned long long n, const double* __restrict__ sums) {
    const double mean = __ddiv_rn(sums[0], double(n));
    for (unsigned long long i = blockIdx.x * 256ULL + threadIdx.x; i < n; i += gridDim.x * 256ULL)
        b[i] = __dsub_rn(b[i], mean);
}

// ---- exclusive scan of u32 counts into u64 offsets (out[n] = total) -------------------------
constexpr int kScanThreads = 1024, kScanPer = 4, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                    unsigned long long* warp_tot,
                                                                    unsigned long long& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long x = lane < int(blockDim.x >> 5) ? warp_tot[lane] : 0ULL, xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        warp_tot[lane] = xi - x;  // exclusive warp offsets
        if (lane == 31) warp_tot[32] = xi;
    }
    __syncthreads();
    total = warp_tot[32];
    const unsigned long long r = warp_tot[w] + inc - v;
    __syncthreads();
    return r;
}

// Pass 1: per-tile exclusive scan, tile totals into tot[].
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint32_t* __restrict__ in, unsigned long long n,
                                                             unsigned long long* __restrict__ out,
                                                             unsigned long long* __restrict__ tot) {
    __shared__ unsigned long long wt[33];
    const unsigned long long base = blockIdx.x * (unsigned long long)kScanTile + threadIdx.x * kScanPer;
    unsigned long long v[kScanPer], s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        v[k] = base + k < n ? in[base + k] : 0u;
        s += v[k];
    }
    unsigned long long total;
    unsigned long long run = block_exclusive_scan(s, wt, total);
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = total;
}
// Pass 2: one CTA scans the tile totals in place (carry across chunks); out[n] = grand total.
__global__ void __launch_bounds__(kScanThreads) k_scan_totals(unsigned long long* __restrict__ tot, unsigned long long m,
                                                              unsigned long long* __restrict__ out_end) {
    __shared__ unsigned long long wt[33];
    unsigned long long carry = 0;
    for (unsigned long long c = 0; c < m; c += kScanThreads) {
        const unsigned long long i = c + threadIdx.x;
        const unsigned long long v = i < m ? tot[i] : 0ULL;
        unsigned long long total;
        const unsigned long long ex = block_exclusive_scan(v, wt, total);
        if (i < m) tot[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) *out_end = carry;
}
// Pass 3: add the tile offsets.
__global__ void __launch_bounds__(kScanThreads) k_scan_add(unsigned long long* __restrict__ out, unsigned long long n,
                                                           const unsigned long long* __restrict__ tot) {
    const unsigned long long base = blockIdx.x * (unsigned long long)kScanTile + threadIdx.x * kScanPer;
    const unsigned long long add = tot[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanPer; ++k)
        if (base + k < n) out[base + k] += add;
}

// ---- SELL-32 from the device CSR (the layout upload_csr builds on the host) ------------------
// Slice s: rows 32s..32s+31, width = longest row, column-major; padding = (own row, 0.0).
__global__ void k_sell_widths(const uint32_t* __restrict__ len, unsigned long long n, unsigned long long ns,
                              uint32_t* __restrict__ slice_len) {
    const unsigned long long s = blockIdx.x * 8ULL + (threadIdx.x >> 5);
    if (s >= ns) return;
    const unsigned long long r = s * 32 + (threadIdx.x & 31);
    uint32_t w = r < n ? len[r] : 0u;
    for (int o = 16; o; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    if ((threadIdx.x & 31) == 0) slice_len[s] = 32u * w;
}
__global__ void k_sell_fill(const unsigned long long* __restrict__ ro, const uint32_t* __restrict__ ci,
                            const double* __restrict__ vals, unsigned long long n, unsigned long long ns,
                            const unsigned long long* __restrict__ slice_off, uint32_t* __restrict__ sc,
                            double* __restrict__ sv) {
    const unsigned long long s = blockIdx.x * 8ULL + (threadIdx.x >> 5);
    if (s >= ns) return;
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long r = s * 32 + lane, off = slice_off[s];
    const uint32_t w = uint32_t((slice_off[s + 1] - off) / 32);
    const unsigned long long p0 = r < n ? ro[r] : 0ULL, l = r < n ? ro[r + 1] - p0 : 0ULL;
    const uint32_t pad = uint32_t(r < n ? r : n - 1);
    for (uint32_t j = 0; j < w; ++j) {
        const unsigned long long idx = off + j * 32ULL + lane;
        if (j < l) {
            sc[idx] = ci[p0 + j];
            sv[idx] = vals[p0 + j];
        } else {
            sc[idx] = pad;
            sv[idx] = 0.0;
        }
    }
}
// Largest 8-slice and 16-slice chunks in bytes (12 per entry): the TMA stage sizes of k_spmv_tma
// and k_solve's ring.
__global__ void k_sell_chunks(const unsigned long long* __restrict__ slice_off, unsigned long long ns,
                              unsigned long long* __restrict__ maxch) {
    const unsigned long long g = blockIdx.x * 256ULL + threadIdx.x;
    if (g * 8 < ns) {
        const unsigned long long e = g * 8 + 8 < ns ? g * 8 + 8 : ns;
        atomicMax(&maxch[0], (slice_off[e] - slice_off[g * 8]) * 12ULL);
    }
    if (g * 16 < ns) {
        const unsigned long long e = g * 16 + 16 < ns ? g * 16 + 16 : ns;
        atomicMax(&maxch[1], (slice_off[e] - slice_off[g * 16]) * 12ULL);
    }
}

}  // namespace hfpg
