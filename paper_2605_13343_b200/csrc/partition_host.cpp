// Row partition of one system over G ranks (host side): the rank's local CSR with ghost
// columns, the halo send lists, and its slice of the packed factor tensor.
//
// The split follows the bisection tree (partition.cpp:9-46): rank r owns the subtree rooted at
// heap node G-1+r, i.e. leaves [r K/G, (r+1) K/G) and rows [r N/G, (r+1) N/G). Every tile at
// depth >= log2 G lies inside one rank's subtree; the G-1 tiles above ("top tiles") are the only
// ones whose strips span ranks. Index values are preserved: local column c - row0 for owned
// columns, n_loc + i for the i-th distinct external column in ascending global order (ghosts
// owned by one peer are therefore contiguous), and the order of entries within a row is the
// reference's, so the local SpMV is bit-identical to csr.cpp:70-79 on the owned rows.
#include "internal.hpp"
#include "partition_host.hpp"

#include <algorithm>
#include <cstring>
#include <thread>

namespace hfpg {

static uint64_t ilog2(uint64_t v) {
    uint64_t l = 0;
    while ((1ULL << l) < v) ++l;
    return l;
}

static void check_part(uint64_t n, uint64_t leaf, uint64_t G, uint64_t rank) {
    check_partition(n, leaf);
    if (G == 0 || (G & (G - 1)) != 0) throw InvalidArgument("partition: rank count must be a power of two");
    if (G > kMaxRanks) throw InvalidArgument("partition: at most 16 ranks");
    if (rank >= G) throw InvalidArgument("partition: rank out of range");
    const uint64_t K = n / leaf;
    if (K / G < 2) throw InvalidArgument("partition: need at least two leaves per rank");
}

// Sorted distinct columns of rows [a, b) that fall outside [a, b).
static std::vector<uint32_t> ghosts_of(const uint64_t* ro, const uint32_t* ci, uint64_t a, uint64_t b) {
    std::vector<uint32_t> g;
    for (uint64_t i = a; i < b; ++i)
        for (uint64_t p = ro[i]; p < ro[i + 1]; ++p)
            if (ci[p] < a || ci[p] >= b) g.push_back(ci[p]);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    return g;
}

PartPlan plan_partition(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                        uint64_t leaf, uint64_t G, uint64_t rank) {
    check_part(n, leaf, G, rank);
    PartPlan P;
    P.n_global = n;
    P.G = G;
    P.rank = rank;
    P.glog = ilog2(G);
    P.n_loc = n / G;
    P.row0 = rank * P.n_loc;
    const uint64_t r0 = P.row0, r1 = r0 + P.n_loc;
    if (ro[0] != 0) throw InvalidArgument("csr: row_offsets[0] != 0");
    for (uint64_t i = 0; i < n; ++i)
        if (ro[i] > ro[i + 1]) throw InvalidArgument("csr: row_offsets not nondecreasing");
    for (uint64_t p = 0; p < ro[n]; ++p)
        if (ci[p] >= n) throw InvalidArgument("csr: column index out of range");
    // global |A|_F (csr.cpp:64-68, sequential) for the breakdown tolerance
    double fro = 0.0;
    for (uint64_t p = 0; p < ro[n]; ++p) fro += v[p] * v[p];
    P.fro = std::sqrt(fro);

    P.ghost_cols = ghosts_of(ro, ci, r0, r1);
    const uint64_t ng = P.ghost_cols.size();
    P.recv_off.assign(G + 1, 0);
    for (uint64_t q = 0, j = 0; q < G; ++q) {
        P.recv_off[q] = j;
        while (j < ng && P.ghost_cols[j] < (q + 1) * P.n_loc) ++j;
        P.recv_off[q + 1] = j;
    }
    // local CSR, columns remapped
    P.local.n = P.n_loc;
    P.local.row_offsets.resize(P.n_loc + 1);
    const uint64_t p0 = ro[r0];
    for (uint64_t i = 0; i <= P.n_loc; ++i) P.local.row_offsets[i] = ro[r0 + i] - p0;
    const uint64_t nnz = ro[r1] - p0;
    P.local.cols.resize(nnz);
    P.local.vals.assign(v + p0, v + p0 + nnz);
    for (uint64_t p = 0; p < nnz; ++p) {
        const uint32_t c = ci[p0 + p];
        if (c >= r0 && c < r1) {
            P.local.cols[p] = uint32_t(c - r0);
        } else {
            const auto it = std::lower_bound(P.ghost_cols.begin(), P.ghost_cols.end(), c);
            P.local.cols[p] = uint32_t(P.n_loc + (it - P.ghost_cols.begin()));
        }
    }
    // send lists: for every peer q, my rows q reads (its ghosts in my range, ascending), each
    // landing at q's ghost slot recv_off_q[rank] + j
    P.send_off.assign(G + 1, 0);
    for (uint64_t q = 0; q < G; ++q) {
        P.send_off[q] = P.send_rows.size();
        if (q == rank) continue;
        const std::vector<uint32_t> gq = ghosts_of(ro, ci, q * P.n_loc, (q + 1) * P.n_loc);
        const auto lo = std::lower_bound(gq.begin(), gq.end(), uint32_t(r0));
        const auto hi = std::lower_bound(gq.begin(), gq.end(), uint32_t(r1));
        const uint64_t base = uint64_t(lo - gq.begin());
        for (auto it = lo; it != hi; ++it) {
            P.send_rows.push_back(uint32_t(*it - r0));
            P.send_slot.push_back(uint32_t(base + uint64_t(it - lo)));
        }
    }
    P.send_off[G] = P.send_rows.size();
    return P;
}

// Global packed-tensor element index of every local element (rank's slice), plus the top tiles.
template <class Fn>
static void for_slice(const Layout& Lg, uint64_t G, uint64_t rank, Fn&& fn) {
    const Layout Ll = make_layout(Lg.n / G, Lg.l, Lg.ls);
    const uint64_t Kl = Ll.k, glog = ilog2(G), LL = Lg.l * Lg.l, TT = Lg.ls * Lg.ls;
    // leaves
    fn(Ll.leaf(0), Lg.leaf(rank * Kl), Kl * LL);
    // local tiles: local heap node u at local depth ld <-> global tile 2^(glog+ld)-1 + rank 2^ld + j
    for (uint64_t ld = 0; (1ULL << ld) < Kl; ++ld) {
        const uint64_t cnt = 1ULL << ld;
        fn(Ll.tile_base + (cnt - 1) * TT, Lg.tile_base + ((1ULL << (glog + ld)) - 1 + rank * cnt) * TT, cnt * TT);
    }
    // bridges, gate
    fn(Ll.bridge_base, Lg.bridge_u(rank * Kl), Kl * 2 * Lg.l * Lg.ls);
    fn(Ll.gate_base, Lg.gate_base + rank * Ll.n, Ll.n);
}

void slice_factors(const Layout& Lg, const float* global, uint64_t G, uint64_t rank, float* local,
                   float* top) {
    for_slice(Lg, G, rank, [&](uint64_t dst, uint64_t src, uint64_t cnt) {
        std::memcpy(local + dst, global + src, cnt * 4);
    });
    std::memcpy(top, global + Lg.tile_base, (G - 1) * Lg.ls * Lg.ls * 4);
}

void init_factors_slice(const Layout& Lg, uint64_t G, uint64_t rank, double sigma, uint64_t seed,
                        uint64_t frame, float* local, float* top) {
    // init_factors (factor_tensor.cpp:30-39) draws element e from counter e of
    // RngStream(seed, frame, factor_init); gate = 1. Generate only this rank's elements.
    const Rng s(seed, frame, kFactorInit);
    auto val = [&](uint64_t e) -> float {
        if (e >= Lg.gate_base) return 1.0f;
        return static_cast<float>(sigma == 0.0 ? 0.0 : sigma * Rng::normal_of(s.bits_at(e)));
    };
    std::vector<std::thread> th;
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    for_slice(Lg, G, rank, [&](uint64_t dst, uint64_t src, uint64_t cnt) {
        if (cnt < (1u << 16)) {
            for (uint64_t i = 0; i < cnt; ++i) local[dst + i] = val(src + i);
            return;
        }
        th.clear();
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                const uint64_t b = cnt * t / nt, e = cnt * (t + 1) / nt;
                for (uint64_t i = b; i < e; ++i) local[dst + i] = val(src + i);
            });
        for (auto& x : th) x.join();
    });
    for (uint64_t i = 0; i < (G - 1) * Lg.ls * Lg.ls; ++i) top[i] = val(Lg.tile_base + i);
}

}  // namespace hfpg

using namespace hfpg;

extern "C" {

int hfpg_part_plan(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                   uint64_t leaf, uint32_t G, uint32_t rank, uint64_t* counts,
                   uint32_t* ghost_cols, uint32_t* send_rows, uint32_t* send_slot,
                   uint64_t* send_off, uint32_t* local_cols) {
    return guarded([&] {
        const PartPlan P = plan_partition(n, ro, ci, v, leaf, G, rank);
        counts[0] = P.n_loc;
        counts[1] = P.ghost_cols.size();
        counts[2] = P.send_rows.size();
        counts[3] = P.local.cols.size();
        if (ghost_cols) std::copy(P.ghost_cols.begin(), P.ghost_cols.end(), ghost_cols);
        if (send_rows) std::copy(P.send_rows.begin(), P.send_rows.end(), send_rows);
        if (send_slot) std::copy(P.send_slot.begin(), P.send_slot.end(), send_slot);
        if (send_off) std::copy(P.send_off.begin(), P.send_off.end(), send_off);
        if (local_cols) std::copy(P.local.cols.begin(), P.local.cols.end(), local_cols);
    });
}

int hfpg_part_factors(uint64_t n, uint64_t leaf, uint64_t ls, uint32_t G, uint32_t rank,
                      const float* packed, double sigma, uint64_t seed, uint64_t frame,
                      float* local, float* top) {
    return guarded([&] {
        check_part(n, leaf, G, rank);
        const Layout Lg = make_layout(n, leaf, ls);
        if (packed) slice_factors(Lg, packed, G, rank, local, top);
        else init_factors_slice(Lg, G, rank, sigma, seed, frame, local, top);
    });
}

}  // extern "C"
