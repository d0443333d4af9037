// TEST INFRASTRUCTURE ONLY — the oracle side of the 3D benchmark frame (BASELINE configs[2],
// SURVEY.md §8(d) item 3), compiled into oracle/_ref/libhfpref.so next to the unmodified
// reference sources and never linked into the product.
//
// The reference has no 3D generator; SURVEY §8(d) defines one as make_frame (frame.cpp:161-181)
// lifted to a 3D grid. This file builds it from the reference's own pieces so the reference
// arm of bench.py gets its inputs without the product library:
//   * hfp::RngStream (rng.hpp:37-87) drawn in make_frame's order: density stream
//     (rho_heavy, 1-3 barriers — sample_density, frame.cpp:81-98, with the slab normal drawn
//     from {x, y, z}), then one noise normal per cell in Morton order (density_from_barriers,
//     frame.cpp:60-79); rhs = hfp::sample_rhs (frame.cpp:154-159) on the rhs stream;
//   * the barrier test of frame.cpp:44-56 with cross = the slab normal's coordinate and
//     along = the next axis's;
//   * 3D Morton order (x -> bit 3i, y -> 3i+1, z -> 3i+2) of all nx*ny*nz cells;
//   * assemble_operator's 5-point rule (frame.cpp:100-145) extended to 7 points, neighbour
//     order (x-1, x+1, y-1, y+1, z-1, z+1), harmonic-mean weights, columns sorted per row.
#include "hfp/frame.hpp"
#include "hfp/rng.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

using namespace hfp;

namespace {
thread_local std::string g_err3;

uint64_t spread3(uint64_t v) {
    uint64_t out = 0;
    for (int b = 0; b < 21; ++b) out |= ((v >> b) & 1ull) << (3 * b);
    return out;
}

struct Frame3 {
    uint64_t n = 0, nx = 0, ny = 0, nz = 0;
    double rho_heavy = 0.0;
    std::vector<uint32_t> order;
    std::vector<double> rho, b;
    CsrMatrix A;
};

bool heavy(double cross, double along, double center, double thickness, uint64_t gap) {
    if (std::fabs(cross - center) > 0.5 * thickness) return false;
    switch (gap) {  // frame.cpp:48-53
        case 0: return along < 0.8;
        case 1: return along > 0.2;
        case 2: return along < 0.4 || along > 0.6;
        default: return true;
    }
}

Frame3* make3(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed, uint64_t fidx) {
    if (nx < 2 || ny < 2 || nz < 2) throw std::invalid_argument("frame_3d: each dimension must be >= 2");
    auto* f = new Frame3;
    const uint64_t n = nx * ny * nz;
    f->n = n;
    f->nx = nx;
    f->ny = ny;
    f->nz = nz;
    std::vector<std::pair<uint64_t, uint32_t>> keyed(n);
    for (uint64_t id = 0; id < n; ++id) {
        const uint64_t x = id % nx, y = (id / nx) % ny, z = id / (nx * ny);
        keyed[id] = {spread3(x) | (spread3(y) << 1) | (spread3(z) << 2), uint32_t(id)};
    }
    std::sort(keyed.begin(), keyed.end());
    f->order.resize(n);
    for (uint64_t i = 0; i < n; ++i) f->order[i] = keyed[i].second;

    RngStream ds(seed, fidx, RngPurpose::density);
    f->rho_heavy = std::exp(ds.next_uniform(std::log(5.0), std::log(100.0)));
    struct Bar {
        uint64_t axis, gap;
        double center, thickness;
    };
    std::vector<Bar> bars;
    const uint64_t nb = 1 + ds.next_below(3);
    for (uint64_t i = 0; i < nb; ++i) {
        Bar b;
        b.axis = ds.next_below(3);
        b.center = ds.next_uniform(0.2, 0.8);
        b.thickness = ds.next_uniform(0.05, 0.20);
        b.gap = ds.next_below(4);
        bars.push_back(b);
    }
    f->rho.resize(n);
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t id = f->order[i];
        const double c[3] = {(double(id % nx) + 0.5) / double(nx), (double((id / nx) % ny) + 0.5) / double(ny),
                             (double(id / (nx * ny)) + 0.5) / double(nz)};
        bool h = false;
        for (const Bar& b : bars)
            if (heavy(c[b.axis], c[(b.axis + 1) % 3], b.center, b.thickness, b.gap)) {
                h = true;
                break;
            }
        const double noise = std::max(0.5, 1.0 + 0.05 * ds.next_normal());
        f->rho[i] = (h ? f->rho_heavy : 1.0) * noise;
    }

    std::vector<int64_t> rank_of(n);
    for (uint64_t i = 0; i < n; ++i) rank_of[f->order[i]] = int64_t(i);
    CsrMatrix& A = f->A;
    A.n_rows = A.n_cols = n;
    A.row_offsets.reserve(n + 1);
    A.row_offsets.push_back(0);
    std::vector<std::pair<uint32_t, double>> row;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t id = f->order[i];
        const int64_t x = id % nx, y = (id / nx) % ny, z = id / (nx * ny);
        const int64_t nbr[6][3] = {{x - 1, y, z}, {x + 1, y, z}, {x, y - 1, z},
                                   {x, y + 1, z}, {x, y, z - 1}, {x, y, z + 1}};
        row.clear();
        double diag = 0.0;
        for (const auto& c : nbr) {
            if (c[0] < 0 || c[0] >= int64_t(nx) || c[1] < 0 || c[1] >= int64_t(ny) || c[2] < 0 ||
                c[2] >= int64_t(nz))
                continue;
            const int64_t j = rank_of[uint64_t(c[2]) * nx * ny + uint64_t(c[1]) * nx + uint64_t(c[0])];
            const double w = 2.0 * f->rho[i] * f->rho[j] / (f->rho[i] + f->rho[j]);
            diag += w;
            row.emplace_back(uint32_t(j), -w);
        }
        row.emplace_back(uint32_t(i), diag);
        std::sort(row.begin(), row.end());
        for (const auto& [c, v] : row) {
            A.col_indices.push_back(c);
            A.values.push_back(v);
        }
        A.row_offsets.push_back(A.col_indices.size());
    }
    RngStream rs(seed, fidx, RngPurpose::rhs);
    f->b = sample_rhs(n, rs);
    return f;
}
}  // namespace

extern "C" {

const char* ref_frame3d_last_error() { return g_err3.c_str(); }

void* ref_frame3d_create(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed, uint64_t frame_index) {
    try {
        return make3(nx, ny, nz, seed, frame_index);
    } catch (const std::exception& e) {
        g_err3 = e.what();
        return nullptr;
    }
}
void ref_frame3d_sizes(void* h, uint64_t* n, uint64_t* nnz, double* rho_heavy) {
    auto* f = static_cast<Frame3*>(h);
    *n = f->n;
    *nnz = f->A.col_indices.size();
    *rho_heavy = f->rho_heavy;
}
void ref_frame3d_fill(void* h, uint32_t* cell_order, double* rho, uint64_t* row_offsets, uint32_t* cols,
                      double* vals, double* b) {
    auto* f = static_cast<Frame3*>(h);
    if (cell_order) std::memcpy(cell_order, f->order.data(), f->n * 4);
    if (rho) std::memcpy(rho, f->rho.data(), f->n * 8);
    if (row_offsets) std::memcpy(row_offsets, f->A.row_offsets.data(), (f->n + 1) * 8);
    if (cols) std::memcpy(cols, f->A.col_indices.data(), f->A.col_indices.size() * 4);
    if (vals) std::memcpy(vals, f->A.values.data(), f->A.values.size() * 8);
    if (b) std::memcpy(b, f->b.data(), f->n * 8);
}
void ref_frame3d_free(void* h) { delete static_cast<Frame3*>(h); }

}  // extern "C"
