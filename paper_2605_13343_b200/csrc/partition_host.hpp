// Host-side row partition of a system over G ranks (partition_host.cpp).
#pragma once

#include "internal.hpp"

namespace hfpg {

constexpr uint64_t kMaxRanks = 16;

struct PartPlan {
    uint64_t n_global = 0, n_loc = 0, G = 1, rank = 0, glog = 0, row0 = 0;
    double fro = 0.0;                  // global |A|_F
    Csr local;                         // n_loc rows; columns in [0, n_loc + n_ghost)
    std::vector<uint32_t> ghost_cols;  // global ids of the ghost columns, ascending
    std::vector<uint64_t> recv_off;    // G+1: ghosts owned by rank q = [recv_off[q], recv_off[q+1])
    std::vector<uint32_t> send_rows;   // local rows pushed to peers, grouped by peer
    std::vector<uint32_t> send_slot;   // destination slot in that peer's ghost region
    std::vector<uint64_t> send_off;    // G+1
};

PartPlan plan_partition(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                        uint64_t leaf, uint64_t G, uint64_t rank);
// Local packed tensor of the rank (layout of size n/G) + the G-1 top tiles (global heap order).
void slice_factors(const Layout& Lg, const float* global, uint64_t G, uint64_t rank, float* local,
                   float* top);
void init_factors_slice(const Layout& Lg, uint64_t G, uint64_t rank, double sigma, uint64_t seed,
                        uint64_t frame, float* local, float* top);

}  // namespace hfpg
