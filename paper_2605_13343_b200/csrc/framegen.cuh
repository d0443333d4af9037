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

// ---- the same sequential sums, emulated exactly in parallel ---------------------------------
// While the running sum s stays inside one binade [2^e, 2^(e+1)) (one sign), every step rounds on
// the fixed grid u = 2^(e-52): RN(s + x) = s + RN_u(x). In units of u the sum is an integer T
// with |T| in [2^52, 2^53), and the increment d = RN_u(x) does not depend on s — except at an
// exact tie (x/u = m + 1/2), where round-to-even takes m or m + 1 by the parity of T. So:
//
//   k_seq_tsum / k_seq_guess  an approximate (any-order) prefix sum guesses the binade at every
//                             4096-element tile start;
//   k_seq_summ                all SMs summarise each tile under its guessed grid, for either
//                             parity of the incoming T: total, min/max partial sum, outgoing
//                             parity (ties resolved exactly through the parity) — an ordered
//                             reduction over the (parity -> ...) monoid;
//   k_seq_sum                 one CTA walks the tiles: a tile whose guess matches s's binade and
//                             whose partial sums provably stay inside it (|T| in [2^52 + 1,
//                             2^53 - 1]) is applied in O(1); any other tile is scanned element by
//                             element (block scan of the increments, first element that leaves
//                             the binade / is a tie / is out of range done by thread 0 with the
//                             real rounding: RN(s + x), or fma(x, x, s) for the sum of squares).
//
// Every accepted value is the serial loop's, bit for bit (tests/test_gpu_framegen.py stresses
// ties, cancellation, crossings and overflow against the serial oracle). The source must be
// readable up to the next 16-byte boundary past cnt (TMA chunks).
constexpr int kSeqW = 4096;
constexpr int kSeqThreads = 1024, kSeqPer = kSeqW / kSeqThreads;
constexpr int kSeqSumThreads = 256, kSeqSumPer = kSeqW / kSeqSumThreads;
constexpr int kSeqSerialRun = 256, kSeqSerialBelow = 64;
constexpr size_t kSeqSmem = 2 * size_t(kSeqW) * sizeof(double);
constexpr int kSeqNoGuess = -100000;

struct SeqTile {
    long long tot[2], mn[2], mx[2];  // by incoming parity of T: sum of d, min/max partial sum
    int pout[2];                     // outgoing parity
    int ex;                          // frexp exponent of the guessed start sum (kSeqNoGuess: none)
    int ok;                          // 0: an element needs the detailed path
};

__device__ __forceinline__ double pow2_dev(int k) {  // 2^k, k in [-1022, 1023]
    return __longlong_as_double((long long)(1023 + k) << 52);
}

// x's increment on the grid 2^(ex-53) (scale = 2^(53-ex)): floor part + round-up bit; a tie is
// settled by the parity of the running T (seq_d). ok = 0: exact handling needed (out of range).
struct SeqInc {
    long long fl;
    int up, tie, ok;
};
template <bool Squares>
__device__ __forceinline__ SeqInc seq_inc(double x, double scale) {
    SeqInc r{0, 0, 0, 1};
    double qh, ql = 0.0;
    if (Squares) {
        const double th = __dmul_rn(x, x), tl = __fma_rn(x, x, -th);
        qh = __dmul_rn(th, scale);
        ql = __dmul_rn(tl, scale);
        r.ok = th == 0.0 || fabs(th) > 0x1p-900;
    } else {
        qh = __dmul_rn(x, scale);
        r.ok = x == 0.0 || fabs(x) > 0x1p-960;
    }
    // |d| < 2^50: a 4096-element partial sum stays below 2^62 (no 64-bit overflow)
    r.ok = r.ok && fabs(qh) < 0x1p50;
    if (r.ok) {
        const double fl = floor(qh), fr = __dsub_rn(qh, fl);
        r.fl = (long long)fl;
        r.tie = fr == 0.5 && ql == 0.0;
        r.up = fr > 0.5 || (fr == 0.5 && ql > 0.0);
    }
    return r;
}
__device__ __forceinline__ long long seq_d(const SeqInc& a, long long t_prev) {
    return a.fl + (a.tie ? ((t_prev + a.fl) & 1) : a.up);
}

// Approximate tile sums (any order) -> per-tile guessed start exponent.
template <bool Squares>
__global__ void __launch_bounds__(kSeqSumThreads) k_seq_tsum(const double* __restrict__ src, unsigned long long cnt,
                                                             const unsigned long long* __restrict__ cnt_dev,
                                                             double* __restrict__ tsum) {
    if (cnt_dev) cnt = *cnt_dev;
    const unsigned long long t = blockIdx.x, e0 = t * kSeqW;
    if (e0 >= cnt) return;
    double a = 0.0;
    for (int k = 0; k < kSeqSumPer; ++k) {
        const unsigned long long j = e0 + threadIdx.x + (unsigned long long)k * kSeqSumThreads;
        if (j < cnt) {
            const double x = src[j];
            a = Squares ? fma(x, x, a) : a + x;
        }
    }
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    __shared__ double w[kSeqSumThreads / 32];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kSeqSumThreads / 32; ++i) s += w[i];
        tsum[t] = s;
    }
}
__global__ void __launch_bounds__(1024) k_seq_guess(const double* __restrict__ tsum, unsigned long long tiles_max,
                                                    unsigned long long cnt, const unsigned long long* __restrict__ cnt_dev,
                                                    int* __restrict__ guess) {
    if (cnt_dev) cnt = *cnt_dev;
    const unsigned long long tiles = (cnt + kSeqW - 1) / kSeqW < tiles_max ? (cnt + kSeqW - 1) / kSeqW : tiles_max;
    __shared__ double wt[33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double carry = 0.0;
    for (unsigned long long c = 0; c < tiles; c += 1024) {
        const unsigned long long i = c + threadIdx.x;
        const double v = i < tiles ? tsum[i] : 0.0;
        double inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wt[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const double x = wt[lane];
            double xi = x;
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += t;
            }
            wt[lane] = xi - x;
            if (lane == 31) wt[32] = xi;
        }
        __syncthreads();
        const double P = carry + wt[wid] + (inc - v);  // approximate sum before tile i
        if (i < tiles) {
            int ex = kSeqNoGuess;
            if (P != 0.0 && isfinite(P)) frexp(P, &ex);
            guess[i] = ex;
        }
        carry += wt[32];
        __syncthreads();
    }
}

// (parity -> total, min, max, parity out) of a run of increments; empty = identity.
struct SeqRun {
    long long tot[2], mn[2], mx[2];
    int pout[2];
    bool empty;
};
__device__ __forceinline__ SeqRun seq_combine(const SeqRun& A, const SeqRun& B) {
    if (A.empty) return B;
    if (B.empty) return A;
    SeqRun R;
    R.empty = false;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const bool q = A.pout[p] != 0;  // selects, not indexing: keeps the runs in registers
        R.tot[p] = A.tot[p] + (q ? B.tot[1] : B.tot[0]);
        R.mn[p] = min(A.mn[p], A.tot[p] + (q ? B.mn[1] : B.mn[0]));
        R.mx[p] = max(A.mx[p], A.tot[p] + (q ? B.mx[1] : B.mx[0]));
        R.pout[p] = q ? B.pout[1] : B.pout[0];
    }
    return R;
}
__device__ __forceinline__ SeqRun seq_shfl_down(const SeqRun& a, int off) {
    SeqRun r;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        r.tot[p] = __shfl_down_sync(0xffffffffu, a.tot[p], off);
        r.mn[p] = __shfl_down_sync(0xffffffffu, a.mn[p], off);
        r.mx[p] = __shfl_down_sync(0xffffffffu, a.mx[p], off);
        r.pout[p] = __shfl_down_sync(0xffffffffu, a.pout[p], off);
    }
    r.empty = __shfl_down_sync(0xffffffffu, int(a.empty), off) != 0;
    return r;
}

template <bool Squares>
__global__ void __launch_bounds__(kSeqSumThreads) k_seq_summ(const double* __restrict__ src, unsigned long long cnt,
                                                             const unsigned long long* __restrict__ cnt_dev,
                                                             const int* __restrict__ guess, SeqTile* __restrict__ tiles) {
    if (cnt_dev) cnt = *cnt_dev;
    const unsigned long long t = blockIdx.x, e0 = t * kSeqW;
    if (e0 >= cnt) return;
    const int ex = guess[t], sh = 53 - ex;
    const bool usable = ex != kSeqNoGuess && sh <= 1000 && sh >= -1000;
    const double scale = usable ? pow2_dev(sh) : 1.0;
    SeqRun run;
    run.empty = true;
    int ok = usable ? 1 : 0;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        run.tot[p] = 0;
        run.mn[p] = 0;
        run.mx[p] = 0;
        run.pout[p] = p;
    }
    if (usable) {
        const unsigned long long j0 = e0 + (unsigned long long)threadIdx.x * kSeqSumPer;
        SeqInc inc[kSeqSumPer];
        int m = 0;
#pragma unroll
        for (int k = 0; k < kSeqSumPer; ++k) {
            if (j0 + k < cnt) {
                inc[k] = seq_inc<Squares>(src[j0 + k], scale);
                ok &= inc[k].ok;
                m = k + 1;
            }
        }
        if (m > 0) {
            run.empty = false;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                long long T = p, mn = 0, mx = 0;  // T carries the parity; partial sums relative
#pragma unroll
                for (int k = 0; k < kSeqSumPer; ++k) {
                    if (k < m) {
                        T += seq_d(inc[k], T);
                        const long long rel = T - p;
                        mn = k == 0 ? rel : min(mn, rel);
                        mx = k == 0 ? rel : max(mx, rel);
                    }
                }
                run.tot[p] = T - p;
                run.mn[p] = mn;
                run.mx[p] = mx;
                run.pout[p] = int(T & 1);
            }
        }
    }
    ok = __syncthreads_and(ok);
    // ordered reduction: lower lanes first
    for (int off = 1; off < 32; off <<= 1) {
        const SeqRun o = seq_shfl_down(run, off);
        if ((threadIdx.x & (2 * off - 1)) == 0) run = seq_combine(run, o);
    }
    __shared__ SeqRun wr[kSeqSumThreads / 32];
    if ((threadIdx.x & 31) == 0) wr[threadIdx.x >> 5] = run;
    __syncthreads();
    if (threadIdx.x == 0) {
        SeqRun r = wr[0];
        for (int i = 1; i < kSeqSumThreads / 32; ++i) r = seq_combine(r, wr[i]);
        SeqTile out;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            out.tot[p] = r.tot[p];
            out.mn[p] = r.mn[p];
            out.mx[p] = r.mx[p];
            out.pout[p] = r.pout[p];
        }
        out.ex = ex;
        // a usable tile keeps |partial sums| <= 2^54 (a binade spans 2^53 units): the walk's
        // 32-tile scan and S + mn / mx then stay far from overflow
        bool small = true;
        for (int p = 0; p < 2; ++p) {
            const long long lim = 1LL << 54;
            small = small && r.tot[p] <= lim && r.tot[p] >= -lim && r.mn[p] <= lim && r.mn[p] >= -lim &&
                    r.mx[p] <= lim && r.mx[p] >= -lim;
        }
        out.ok = ok && !r.empty && small;
        tiles[t] = out;
    }
}

// The walk: one CTA. Whole tiles through their summaries (warp 0, 32 checked per warp scan),
// else detailed windows (4 elements per thread) that never cross a tile, read from a 2-chunk
// TMA ring (the chunk, and the next one prefetched).
template <bool Squares>
__global__ void __launch_bounds__(kSeqThreads, 1) k_seq_sum(const double* __restrict__ src, unsigned long long cnt,
                                                            const unsigned long long* __restrict__ cnt_dev,
                                                            const SeqTile* __restrict__ tiles, double* __restrict__ out) {
    extern __shared__ __align__(128) double ring[];
    __shared__ uint64_t bar[2];
    __shared__ unsigned long long wtot[64];
    __shared__ int wpar[32];
    __shared__ int wmin[32];
    __shared__ long long t_last;
    __shared__ double s_sh;
    __shared__ unsigned long long pos_sh;
    __shared__ int buf_sh, par_sh;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (cnt_dev) cnt = *cnt_dev;
    const unsigned long long ntiles = (cnt + kSeqW - 1) / kSeqW;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    long long loaded[2] = {-1, -1};  // thread 0: chunk in each buffer
    unsigned nload[2] = {0, 0};      // thread 0: loads issued per buffer
    double s = 0.0;                  // block-uniform at the top of every iteration
    unsigned long long pos = 0;
    const long long lo = (1LL << 52) + 1, hi = (1LL << 53) - 1;
    for (;;) {
        // fast path (warp 0): whole tiles whose summaries provably apply
        if (wid == 0 && tiles && pos % kSeqW == 0 && s != 0.0 && isfinite(s)) {
            int ex = 0;
            const double fs = frexp(s, &ex);
            long long S = (long long)(fs * 9007199254740992.0);
            const bool neg = S < 0;
            unsigned long long t = pos / kSeqW;
            bool moved = false;
            for (;;) {
                const unsigned long long k = t + lane;
                SeqRun r;
                r.empty = true;
                bool okk = false;
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    r.tot[p] = r.mn[p] = r.mx[p] = 0;
                    r.pout[p] = p;
                }
                if (k < ntiles) {
                    const SeqTile T = tiles[k];
                    okk = T.ok && T.ex == ex;
                    r.empty = false;
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        r.tot[p] = T.tot[p];
                        r.mn[p] = T.mn[p];
                        r.mx[p] = T.mx[p];
                        r.pout[p] = T.pout[p];
                    }
                }
                for (int off = 1; off < 32; off <<= 1) {
                    SeqRun o;
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        o.tot[p] = __shfl_up_sync(0xffffffffu, r.tot[p], off);
                        o.mn[p] = __shfl_up_sync(0xffffffffu, r.mn[p], off);
                        o.mx[p] = __shfl_up_sync(0xffffffffu, r.mx[p], off);
                        o.pout[p] = __shfl_up_sync(0xffffffffu, r.pout[p], off);
                    }
                    o.empty = __shfl_up_sync(0xffffffffu, int(r.empty), off) != 0;
                    if (lane >= off) r = seq_combine(o, r);
                }
                const unsigned okmask = __ballot_sync(0xffffffffu, okk);
                const int okrun = okmask == 0xffffffffu ? 32 : __ffs(~okmask) - 1;
                const bool p0 = (S & 1) != 0;
                const long long a = S + (p0 ? r.mn[1] : r.mn[0]), b2 = S + (p0 ? r.mx[1] : r.mx[0]);
                const bool inb = neg ? (b2 <= -lo && a >= -hi) : (a >= lo && b2 <= hi);
                const unsigned vmask = __ballot_sync(0xffffffffu, lane < okrun && !r.empty && inb);
                const int acc = vmask == 0xffffffffu ? 32 : __ffs(~vmask) - 1;
                if (acc > 0) {
                    S += __shfl_sync(0xffffffffu, p0 ? r.tot[1] : r.tot[0], acc - 1);
                    t += acc;
                    moved = true;
                }
                if (acc < 32 || t >= ntiles) break;
            }
            if (moved) {
                s = __dmul_rn(double(S), pow2_dev(ex - 53));
                pos = t * kSeqW < cnt ? t * kSeqW : cnt;
            }
        }
        if (tid == 0) {
            int b = 0, par = 0;
            if (pos < cnt) {
                const unsigned long long c0 = pos / kSeqW;
                b = int(c0 & 1);
                for (unsigned long long cc = c0; cc <= c0 + 1 && cc < ntiles; ++cc) {
                    const int bb = int(cc & 1);
                    if (loaded[bb] == (long long)cc) continue;
                    const unsigned long long e0 = cc * kSeqW, m = cnt - e0 < kSeqW ? cnt - e0 : kSeqW;
                    const uint32_t bytes = uint32_t((m * 8 + 15) & ~15ULL);
                    mbar_expect_tx(&bar[bb], bytes);
                    tma_load_1d(ring + bb * kSeqW, src + e0, bytes, &bar[bb], pol);
                    loaded[bb] = (long long)cc;
                    ++nload[bb];
                }
                par = int((nload[b] - 1) & 1);
            }
            s_sh = s;
            pos_sh = pos;
            buf_sh = b;
            par_sh = par;
        }
        __syncthreads();
        s = s_sh;
        pos = pos_sh;
        if (pos >= cnt) break;
        const int b = buf_sh;
        mbar_wait(&bar[b], uint32_t(par_sh));
        const double* chunk = ring + b * kSeqW;  // chunk[i - base] = element i
        const unsigned long long base = (pos / kSeqW) * kSeqW, tend = base + kSeqW < cnt ? base + kSeqW : cnt;
        const unsigned long long span = tend - pos;
        int ex = 0;
        const double fr_s = frexp(s, &ex);
        const int sh = 53 - ex;
        const bool parallel_ok = s != 0.0 && isfinite(s) && sh <= 1000 && sh >= -1000;
        int bad = 0;
        if (parallel_ok) {
            const long long S = (long long)(fr_s * 9007199254740992.0);
            const double scale = pow2_dev(sh);
            SeqInc in[kSeqPer];
#pragma unroll
            for (int k = 0; k < kSeqPer; ++k) {
                const unsigned long long j = (unsigned long long)tid * kSeqPer + k;
                in[k] = SeqInc{0, 0, 0, 1};
                if (j < span) in[k] = seq_inc<Squares>(chunk[pos + j - base], scale);
            }
            // this thread's run for either incoming parity (ties settle by parity), then an
            // inclusive warp scan of runs, lower lanes first
            unsigned long long it[2];
            int ip[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                long long T = p;
#pragma unroll
                for (int k = 0; k < kSeqPer; ++k) T += seq_d(in[k], T);
                it[p] = (unsigned long long)(T - p);
                ip[p] = int(T & 1);
            }
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long ot0 = __shfl_up_sync(0xffffffffu, it[0], o), ot1 = __shfl_up_sync(0xffffffffu, it[1], o);
                const int op0 = __shfl_up_sync(0xffffffffu, ip[0], o), op1 = __shfl_up_sync(0xffffffffu, ip[1], o);
                if (lane >= o) {
                    const unsigned long long n0 = ot0 + (op0 ? it[1] : it[0]), n1 = ot1 + (op1 ? it[1] : it[0]);
                    const int q0 = op0 ? ip[1] : ip[0], q1 = op1 ? ip[1] : ip[0];
                    it[0] = n0;
                    it[1] = n1;
                    ip[0] = q0;
                    ip[1] = q1;
                }
            }
            if (lane == 31) {
                wtot[2 * wid] = it[0];
                wtot[2 * wid + 1] = it[1];
                wpar[wid] = ip[0] | (ip[1] << 1);
            }
            __syncthreads();
            if (wid == 0) {  // exclusive scan of the warp runs
                unsigned long long xt[2] = {wtot[2 * lane], wtot[2 * lane + 1]};
                int xp[2] = {wpar[lane] & 1, (wpar[lane] >> 1) & 1};
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long ot0 = __shfl_up_sync(0xffffffffu, xt[0], o), ot1 = __shfl_up_sync(0xffffffffu, xt[1], o);
                    const int op0 = __shfl_up_sync(0xffffffffu, xp[0], o), op1 = __shfl_up_sync(0xffffffffu, xp[1], o);
                    if (lane >= o) {
                        const unsigned long long n0 = ot0 + (op0 ? xt[1] : xt[0]), n1 = ot1 + (op1 ? xt[1] : xt[0]);
                        const int q0 = op0 ? xp[1] : xp[0], q1 = op1 ? xp[1] : xp[0];
                        xt[0] = n0;
                        xt[1] = n1;
                        xp[0] = q0;
                        xp[1] = q1;
                    }
                }
                const unsigned long long e0 = __shfl_up_sync(0xffffffffu, xt[0], 1), e1 = __shfl_up_sync(0xffffffffu, xt[1], 1);
                const int f0 = __shfl_up_sync(0xffffffffu, xp[0], 1), f1 = __shfl_up_sync(0xffffffffu, xp[1], 1);
                __syncwarp();
                wtot[2 * lane] = lane ? e0 : 0ULL;
                wtot[2 * lane + 1] = lane ? e1 : 0ULL;
                wpar[lane] = lane ? (f0 | (f1 << 1)) : 2;  // identity: parity p -> p
            }
            __syncthreads();
            // this thread's start: the warps before it, then the lanes before it (at the parity
            // reached there); wrapping is harmless: only the valid prefix is used
            const bool p0 = (S & 1) != 0;
            const bool wp = ((wpar[wid] >> (p0 ? 1 : 0)) & 1) != 0;
            unsigned long long T = (unsigned long long)S + (p0 ? wtot[2 * wid + 1] : wtot[2 * wid]);
            {
                const unsigned long long lt0 = __shfl_up_sync(0xffffffffu, it[0], 1), lt1 = __shfl_up_sync(0xffffffffu, it[1], 1);
                if (lane > 0) T += wp ? lt1 : lt0;
            }
            const unsigned long long T0 = T;
            int my_bad = int(span);
#pragma unroll
            for (int k = 0; k < kSeqPer; ++k) {
                const unsigned long long j = (unsigned long long)tid * kSeqPer + k;
                if (j < span && my_bad == int(span)) {
                    T += (unsigned long long)seq_d(in[k], (long long)T);
                    const long long av = S > 0 ? (long long)T : -(long long)T;
                    if (!in[k].ok || av < lo || av > hi) my_bad = int(j);
                }
            }
            int wb = int(__reduce_min_sync(0xffffffffu, unsigned(my_bad)));
            if (lane == 0) wmin[wid] = wb;
            __syncthreads();
            if (wid == 0) {
                wb = int(__reduce_min_sync(0xffffffffu, unsigned(wmin[lane])));
                if (lane == 0) wmin[0] = wb;
            }
            __syncthreads();
            bad = wmin[0];
            if (bad > 0 && (bad - 1) / kSeqPer == tid) {
                unsigned long long Tb = T0;
                const int last = (bad - 1) % kSeqPer;
#pragma unroll
                for (int k = 0; k < kSeqPer; ++k)
                    if (k <= last) Tb += (unsigned long long)seq_d(in[k], (long long)Tb);
                t_last = (long long)Tb;
            }
            __syncthreads();
        }
        if (tid == 0) {
            double sn = s;
            if (bad > 0) sn = __dmul_rn(double(t_last), pow2_dev(-sh));  // T u, exact
            unsigned long long p = pos + (unsigned long long)bad;
            if ((unsigned long long)bad < span) {
                // the event itself; a serial run when the fast path keeps failing early
                const unsigned long long end =
                    bad < kSeqSerialBelow ? (tend < p + kSeqSerialRun ? tend : p + kSeqSerialRun) : p + 1;
                for (; p < end; ++p) {
                    const double x = chunk[p - base];
                    sn = Squares ? __fma_rn(x, x, sn) : __dadd_rn(sn, x);
                }
            }
            s_sh = sn;
            pos_sh = p;
        }
        __syncthreads();  // every thread (warp 0's fast path in particular) sees the new state
        s = s_sh;
        pos = pos_sh;
        __syncthreads();
    }
    if (tid == 0) *out = s;
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
