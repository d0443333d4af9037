// Internal host-side declarations shared by the C ABI, the generators and the CUDA driver.
#pragma once

#include "../../include/hfpg.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hfpg {

// Error classes mirroring the reference's exception split.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);

// The reference hands zlib a whole payload / section with its byte length cast to uInt
// (checkpoint.cpp:28-30, 79-81; mppf.cpp:21-24), so its stored crc32 covers only the first
// (bytes mod 2^32) bytes. Every HFTC / MPPF checksum here covers the same prefix.
inline uint64_t ref_crc_len(uint64_t bytes) { return bytes & 0xFFFFFFFFull; }

// ic0_host.cpp (ic0.cpp:10-69): lower IC(0) factor of A (policy 0 none, 1 scaled); its transpose.
void ic0_factorize_host(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v, int policy,
                        std::vector<uint64_t>& lro, std::vector<uint32_t>& lci, std::vector<double>& lv,
                        double& shift);
void ic0_transpose_host(uint64_t n, const std::vector<uint64_t>& lro, const std::vector<uint32_t>& lci,
                        const std::vector<double>& lv, std::vector<uint64_t>& tro, std::vector<uint32_t>& tci,
                        std::vector<double>& tv);
void ic0_levels_host(uint64_t n, const std::vector<uint64_t>& lro, const std::vector<uint32_t>& lci,
                     const std::vector<uint64_t>& tro, const std::vector<uint32_t>& tci,
                     std::vector<uint32_t>& fperm, std::vector<uint32_t>& bperm, uint32_t& flevels,
                     uint32_t& blevels);
void ic0_chunk_levels_host(uint64_t n, uint64_t chunk, const std::vector<uint64_t>& lro,
                           const std::vector<uint32_t>& lci, const std::vector<uint64_t>& tro,
                           const std::vector<uint32_t>& tci, std::vector<uint16_t>& flev,
                           std::vector<uint16_t>& blev, std::vector<uint16_t>& fmax, std::vector<uint16_t>& bmax);

// Runs f(), maps exceptions to status codes and records the message.
template <class F>
int guarded(F&& f) {
    try {
        f();
        set_error("");
        return HFPG_OK;
    } catch (const InvalidArgument& e) {
        set_error(e.what());
        return HFPG_EINVAL;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return HFPG_EINVAL;
    } catch (const IoError& e) {
        set_error(e.what());
        return HFPG_EIO;
    } catch (const CudaError& e) {
        set_error(e.what());
        return HFPG_ECUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return HFPG_EIO;
    }
}

// ---- counter-based RNG: same key schedule and draws as rng.hpp:25-70 -------------------
inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
enum Purpose : uint64_t { kDensity = 1, kRhs = 2, kFactorInit = 4 };

struct Rng {
    uint64_t key, counter = 0;
    Rng(uint64_t seed, uint64_t frame, uint64_t purpose)
        : key(mix64(mix64(mix64(seed) ^ frame) ^ purpose)) {}
    // Value at an explicit counter: the stream is a pure function of (key, counter), which is
    // what lets the generators below fill large arrays in parallel and stay bit-identical.
    uint64_t bits_at(uint64_t c) const { return mix64(key ^ c); }
    static double normal_of(uint64_t bits) {
        const double u1 = (static_cast<double>(bits >> 32) + 1.0) * 0x1.0p-32;
        const double u2 = static_cast<double>(bits & 0xFFFFFFFFULL) * 0x1.0p-32;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
    }
    uint64_t bits() { return bits_at(counter++); }
    double uniform() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t below(uint64_t n) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(bits()) * n) >> 64);
    }
    double normal() { return normal_of(bits()); }
};

// ---- frame parameters (frame.cpp:45-98, :161-181): everything a frame draws before its
// per-cell arrays, shared by the host generator and the GPU generator (framegen.cuh) ----------
struct FrameBarrier {
    uint64_t axis = 0;  // 2D: 0 vertical (cross = x), 1 horizontal (cross = y); 3D: slab normal
    double center = 0.5, thickness = 0.1;
    uint64_t gap = 3;   // frame.hpp:15 top/bottom/middle_hole/closed
};
struct FrameParams {
    int dims = 2;
    uint64_t n = 0, W = 0, H = 0, D = 1;  // 2D: the first n cells of W x H in Morton order
    double rho_heavy = 0.0;
    uint64_t density_key = 0, c0 = 0;  // noise of retained cell i = normal(density stream @ c0+i)
    uint64_t rhs_key = 0;              // b_i = normal(rhs stream @ i) before centring
    std::vector<FrameBarrier> bars;
};
FrameParams frame_params_2d(uint64_t n, uint64_t seed, uint64_t fidx);
FrameParams frame_params_3d(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed, uint64_t fidx);
// HFPG_FRAME_CRMATH=1: the host generator draws its normals with crmath.cuh's correctly
// rounded log/cos (what the GPU generator computes) instead of libm's.
bool frame_crmath();

// ---- partition / layout: partition.cpp:9-53, factor_tensor.cpp:7-28 ---------------------
struct Layout {
    uint64_t n = 0, l = 0, ls = 0, rk = 0, k = 0, m = 0, depth = 0;  // depth = log2 K
    uint64_t tile_base = 0, bridge_base = 0, gate_base = 0, total = 0;
    uint64_t leaf(uint64_t kk) const { return kk * l * l; }
    uint64_t tile_u(uint64_t t) const { return tile_base + t * ls * ls; }
    uint64_t tile_v(uint64_t t) const { return tile_u(t) + ls * rk; }
    uint64_t bridge_u(uint64_t kk) const { return bridge_base + kk * 2 * l * ls; }
    uint64_t bridge_v(uint64_t kk) const { return bridge_u(kk) + l * ls; }
};
void check_partition(uint64_t n, uint64_t leaf);
Layout make_layout(uint64_t n, uint64_t leaf, uint64_t ls);
hfpg_layout to_c(const Layout& L);

// ---- synthetic systems ---------------------------------------------------------------------
struct Csr {
    uint64_t n = 0;
    std::vector<uint64_t> row_offsets;
    std::vector<uint32_t> cols;
    std::vector<double> vals;
};
void init_factors_host(const Layout& L, double sigma, uint64_t seed, uint64_t frame, float* out);

// toynet.cu: device-resident toy-network model (weights once per config/seed) and the GPU
// forward of one frame into a device buffer of the packed layout.
struct ToynetModel;
ToynetModel* toynet_model_create(const hfpg_toynet_config& cfg, uint64_t L, uint64_t Ls, uint64_t seed);
void toynet_model_destroy(ToynetModel* m);
bool toynet_model_matches(const ToynetModel* m, const hfpg_toynet_config& cfg, uint64_t L, uint64_t Ls,
                          uint64_t seed);
void toynet_forward_device(ToynetModel* m, cudaStream_t st, const hfpg_frame_view& fr, float* out,
                           hfpg_toynet_trace* trace);
// A frame resident on the device (the GPU frame generator's arrays).
struct ToynetDeviceFrame {
    uint64_t n, width, height, nnz;
    double rho_heavy;
    const uint32_t* order;
    const double* rho;
    const unsigned long long* ro;
    const uint32_t* ci;
    const double* v;
    const double* diag;
};
void toynet_forward_device_frame(ToynetModel* m, cudaStream_t st, const ToynetDeviceFrame& f, float* out,
                                 hfpg_toynet_trace* trace);

// HFTC / MPPF headers (host_structure.cpp), for the device loaders in hfpg_device.cu.
struct HftcHeader {
    Layout L;
    int spd_enabled = 0;
    double spd_raw = 0.0;
    uint32_t crc = 0;
    uint64_t payload_offset = 0;
};
HftcHeader hftc_read_header(const char* path);
struct MppfSection {
    std::string name;
    uint64_t offset = 0, bytes = 0;
    uint32_t crc = 0;
};
struct MppfHeader {
    uint64_t n = 0, width = 0, height = 0, seed = 0, frame = 0;
    double rho_heavy = 0.0;
    std::vector<FrameBarrier> bars;
    std::vector<MppfSection> sections;
    uint64_t payload_offset = 0;
};
MppfHeader mppf_read_header(const char* path);

}  // namespace hfpg

struct hfpg_frame {
    uint64_t n = 0, width = 0, height = 0, depth = 1;
    double rho_heavy = 0.0;
    uint64_t master_seed = 0, frame_index = 0;
    std::vector<hfpg::FrameBarrier> bars;  // frame.hpp:37 (MPPF header)
    std::vector<uint32_t> cell_order;
    std::vector<double> rho, b;
    hfpg::Csr A;
};
