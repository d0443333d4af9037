// hfp_gpu.hpp — C++ drop-in for the reference `hfp` solve path, backed by libhfpg (sm_100a).
//
// Header-only; links against libhfpg.so (C ABI in hfpg.h). Works with the reference's own
// types by duck typing, so a reference build switches with one line:
//
//   #include "hfp/pcg.hpp"        // reference
//   #include "hfp_gpu.hpp"        // this
//   hfp::PrecondApplier M = hfp::gpu::factor_applier(factors, A);   // was hfp::factor_applier
//   hfp::SolveReport rep  = hfp::pcg_solve(A, b, M, cfg);            // reference PCG, GPU apply
//   hfp::SolveReport rep2 = hfp::gpu::pcg_solve<hfp::SolveReport>(A, b, hfp::gpu::Precond::factor(factors, A), cfg);
//                                                                    // whole loop on the GPU
//
// Error behaviour follows the reference: contract violations throw std::invalid_argument,
// I/O/format problems std::runtime_error; breakdown / max_iters are reported, never thrown.
#pragma once

#include "hfpg.h"

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace hfp::gpu {

inline void check(int rc) {
    if (rc == HFPG_OK) return;
    const std::string msg = hfpg_last_error();
    if (rc == HFPG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// One device-resident context: operator, factors, workspace and a CUDA stream (pcg.cpp:44-51
// takes owning copies of the tensor and diag(A); so does this).
class Device {
  public:
    explicit Device(int device = 0) {
        hfpg_handle* h = nullptr;
        check(hfpg_create(device, &h));
        h_.reset(h);
    }
    hfpg_handle* get() const { return h_.get(); }

    template <class Csr>
    void load_csr(const Csr& A) {  // csr.hpp:11-16 fields
        check(hfpg_load_csr(get(), A.n_rows, A.row_offsets.data(), A.col_indices.data(),
                            A.values.data(), HFPG_HOST));
    }
    template <class Factors>
    void load_factors(const Factors& f) {  // factor_tensor.hpp:57-112 fields
        check(hfpg_load_factors(get(), f.layout.n, f.layout.leaf_size, f.layout.coarse_size,
                                f.data.data(), f.data.size(), f.spd_shift_enabled ? 1 : 0,
                                f.spd_shift_raw, HFPG_HOST));
    }
    void set_precond(int kind) { check(hfpg_set_precond(get(), kind)); }

  private:
    struct Del {
        void operator()(hfpg_handle* h) const { hfpg_destroy(h); }
    };
    std::unique_ptr<hfpg_handle, Del> h_;
};

// pcg.hpp:36 PrecondApplier-compatible GPU applier (apply.cpp:79-174 on the device). Each call
// copies r in and z out — the plug-compatible path for the reference's own pcg_solve,
// spectrum and CLI. For speed use gpu::pcg_solve, which keeps the loop on the device.
template <class Factors, class Csr>
std::function<void(std::span<const double>, std::span<double>)> factor_applier(
    const Factors& factors, const Csr& A) {
    auto dev = std::make_shared<Device>();
    dev->load_csr(A);
    dev->load_factors(factors);
    const std::size_t n = A.n_rows;
    return [dev, n](std::span<const double> r, std::span<double> z) {
        if (r.size() != n || z.size() != n) throw std::invalid_argument("apply: length mismatch");
        check(hfpg_apply(dev->get(), r.data(), z.data(), HFPG_HOST));
    };
}

// 64-bit content fingerprint of a CSR operator (structure and value bits), so gpu::pcg_solve can
// tell whether the device operator is still the A it is handed (pcg.cpp:53 always uses its A).
template <class Csr>
uint64_t csr_fingerprint(const Csr& A) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t(A.n_rows) * 0x100000001B3ull);
    auto mix = [&h](const void* p, std::size_t bytes) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        std::size_t i = 0;
        for (; i + 8 <= bytes; i += 8) {
            uint64_t w;
            std::memcpy(&w, c + i, 8);
            h = (h ^ w) * 0x100000001B3ull;
            h ^= h >> 29;
        }
        for (; i < bytes; ++i) h = (h ^ c[i]) * 0x100000001B3ull;
        h ^= bytes;
    };
    mix(A.row_offsets.data(), A.row_offsets.size() * sizeof(A.row_offsets[0]));
    mix(A.col_indices.data(), A.col_indices.size() * sizeof(A.col_indices[0]));
    mix(A.values.data(), A.values.size() * sizeof(A.values[0]));
    return h;
}

// Device-side description of the preconditioner for gpu::pcg_solve (pcg.cpp:28-51).
struct Precond {
    std::shared_ptr<Device> dev;
    int kind = HFPG_PRECOND_FACTOR;
    std::string method;
    std::shared_ptr<uint64_t> operator_fp = std::make_shared<uint64_t>(0);  // A on the device

    // Make the device operator A (reload it when A's content differs from what was loaded).
    template <class Csr>
    void bind(const Csr& A) const {
        const uint64_t fp = csr_fingerprint(A);
        if (fp == *operator_fp) return;
        dev->load_csr(A);
        dev->set_precond(kind);
        *operator_fp = fp;
    }

    template <class Csr>
    static Precond identity(const Csr& A) {
        return make(A, HFPG_PRECOND_IDENTITY, "none");
    }
    template <class Csr>
    static Precond jacobi(const Csr& A) {
        return make(A, HFPG_PRECOND_JACOBI, "jacobi");
    }
    template <class Factors, class Csr>
    static Precond factor(const Factors& f, const Csr& A) {
        Precond p = make(A, HFPG_PRECOND_FACTOR, "hfactor-gpu");
        p.dev->load_factors(f);
        return p;
    }

  private:
    template <class Csr>
    static Precond make(const Csr& A, int kind, const char* method) {
        Precond p;
        p.dev = std::make_shared<Device>();
        p.dev->load_csr(A);
        p.dev->set_precond(kind);
        p.kind = kind;
        p.method = method;
        *p.operator_fp = csr_fingerprint(A);
        return p;
    }
};

// Field-compatible mirror of pcg.hpp:21-33 SolveReport (used when the reference header is not
// included; pass hfp::SolveReport as Report to get the reference type back).
struct SolveReport {
    enum class Status { converged, max_iters, breakdown };
    std::string method;
    std::size_t n = 0;
    std::size_t iterations = 0;
    bool converged = false;
    Status status = Status::max_iters;
    std::vector<double> residual_history;
    double wall_ms = 0.0;
    std::string frame_id;
    std::size_t breakdown_iter = 0;
};

// pcg.cpp:53-126 with the whole loop captured in one CUDA graph (conditional WHILE node).
// Config: any type with .rtol and .max_iters (pcg.hpp:12-17).
template <class Report = SolveReport, class Csr, class Config>
Report pcg_solve(const Csr& A, std::span<const double> b, const Precond& M, const Config& cfg,
                 std::vector<double>* x_out = nullptr) {
    if (!(cfg.rtol > 0.0)) throw std::invalid_argument("pcg_solve: rtol must be positive");
    if (b.size() != A.n_rows) throw std::invalid_argument("pcg_solve: rhs length mismatch");
    M.bind(A);  // solve with the A handed in, as pcg.cpp:53 does
    std::vector<double> x(A.n_rows), hist(cfg.max_iters ? cfg.max_iters : 1);
    hfpg_solve_config c{cfg.rtol, static_cast<uint64_t>(cfg.max_iters)};
    hfpg_report r{};
    check(hfpg_pcg_solve(M.dev->get(), b.data(), &c, x.data(), hist.data(), &r, HFPG_HOST));
    Report rep;
    rep.method = M.method;
    rep.n = r.n;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.status = static_cast<decltype(rep.status)>(r.status);  // same enumerator order
    rep.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
    rep.wall_ms = r.wall_ms;
    rep.breakdown_iter = r.breakdown_iter;
    if (x_out) *x_out = std::move(x);
    return rep;
}

}  // namespace hfp::gpu
