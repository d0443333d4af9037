// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/src/*.cpp,
// compiled in place by oracle/Makefile into oracle/_ref/libhfpref.so). It lets the Python
// tests, the golden-fixture generator and bench.py's reference arm call the reference's own
// functions with plain pointers. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it.
//
// Every entry point forwards to the reference symbol named in its comment; no arithmetic of
// the path is restated here.

#include "hfp/apply.hpp"
#include "hfp/checkpoint.hpp"
#include "hfp/csr.hpp"
#include "hfp/factor_tensor.hpp"
#include "hfp/frame.hpp"
#include "hfp/ic0.hpp"
#include "hfp/mppf.hpp"
#include "hfp/adjoint.hpp"
#include "hfp/morton.hpp"
#include "hfp/partition.hpp"
#include "hfp/pcg.hpp"
#include "hfp/rng.hpp"
#include "hfp/toy_net.hpp"
#include "hfp/train.hpp"

#include "../include/hfpg.h"  // plain C structs of the training run (layout only)

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

using namespace hfp;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

CsrMatrix make_csr(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v) {
    CsrMatrix A;
    A.n_rows = A.n_cols = n;
    A.row_offsets.assign(ro, ro + n + 1);
    const uint64_t nnz = ro[n];
    A.col_indices.assign(ci, ci + nnz);
    A.values.assign(v, v + nnz);
    return A;
}

template <typename T>
PackedFactors<T> make_factors(uint64_t n, uint64_t leaf, uint64_t ls, const T* packed,
                              int spd_enabled, double spd_raw) {
    PackedFactors<T> f(make_factor_layout(build_partition(n, leaf), ls));
    std::memcpy(f.data.data(), packed, f.data.size() * sizeof(T));
    f.spd_shift_enabled = spd_enabled != 0;
    f.spd_shift_raw = spd_raw;
    return f;
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// partition.cpp:48 packed_width(build_partition(n, leaf), ls)
int ref_packed_width(uint64_t n, uint64_t leaf, uint64_t ls, uint64_t* out) {
    return guard([&] { *out = packed_width(build_partition(n, leaf), ls); });
}

// partition.cpp:9 build_partition; tiles as rows {id, span, row_begin, col_begin, depth}
int ref_partition(uint64_t n, uint64_t leaf, uint64_t* tiles_out /* (K-1) x 5 */) {
    return guard([&] {
        HPartition p = build_partition(n, leaf);
        for (const TileSpec& t : p.tiles) {
            uint64_t* o = tiles_out + 5 * t.id;
            o[0] = t.id; o[1] = t.span; o[2] = t.row_begin; o[3] = t.col_begin; o[4] = t.depth;
        }
    });
}

uint32_t ref_morton_encode(uint32_t x, uint32_t y) { return morton_encode(x, y); }

// rng.hpp:37-70 RngStream draws
int ref_rng_draws(uint64_t seed, uint64_t frame, uint64_t purpose, uint64_t count,
                  uint64_t* bits_out, double* normal_out) {
    return guard([&] {
        RngStream a(seed, frame, static_cast<RngPurpose>(purpose));
        RngStream b(seed, frame, static_cast<RngPurpose>(purpose));
        for (uint64_t i = 0; i < count; ++i) {
            if (bits_out) bits_out[i] = a.next_bits();
            if (normal_out) normal_out[i] = b.next_normal();
        }
    });
}

// factor_tensor.cpp:30 init_factors<float> with RngStream(seed, frame, factor_init)
int ref_init_factors_f32(uint64_t n, uint64_t leaf, uint64_t ls, double sigma, uint64_t seed,
                         uint64_t frame, float* out) {
    return guard([&] {
        RngStream s(seed, frame, RngPurpose::factor_init);
        FactorTensor f = init_factors<float>(build_partition(n, leaf), ls,
                                             FactorInit::jacobi_seed, sigma, s);
        std::memcpy(out, f.data.data(), f.data.size() * sizeof(float));
    });
}

int ref_init_factors_f64(uint64_t n, uint64_t leaf, uint64_t ls, double sigma, uint64_t seed,
                         uint64_t frame, double* out) {
    return guard([&] {
        RngStream s(seed, frame, RngPurpose::factor_init);
        auto f = init_factors<double>(build_partition(n, leaf), ls, FactorInit::jacobi_seed,
                                      sigma, s);
        std::memcpy(out, f.data.data(), f.data.size() * sizeof(double));
    });
}

// frame.cpp:161 make_frame. Two calls: sizes, then fill (any pointer may be null).
struct RefFrame {
    Frame f;
};
void* ref_frame_create(uint64_t n, uint64_t seed, uint64_t frame_index) {
    RefFrame* r = nullptr;
    int rc = guard([&] { r = new RefFrame{make_frame(n, seed, frame_index)}; });
    return rc == 0 ? r : nullptr;
}
void ref_frame_sizes(void* h, uint64_t* n, uint64_t* nnz, uint64_t* width, uint64_t* height,
                     double* rho_heavy) {
    auto* r = static_cast<RefFrame*>(h);
    *n = r->f.n;
    *nnz = r->f.A.nnz();
    *width = r->f.width;
    *height = r->f.height;
    *rho_heavy = r->f.rho_heavy;
}
void ref_frame_fill(void* h, uint32_t* cell_order, double* rho, uint64_t* row_offsets,
                    uint32_t* cols, double* vals, double* b) {
    auto* r = static_cast<RefFrame*>(h);
    const Frame& f = r->f;
    if (cell_order) std::memcpy(cell_order, f.cell_order.data(), f.n * 4);
    if (rho) std::memcpy(rho, f.rho.data(), f.n * 8);
    if (row_offsets) std::memcpy(row_offsets, f.A.row_offsets.data(), (f.n + 1) * 8);
    if (cols) std::memcpy(cols, f.A.col_indices.data(), f.A.nnz() * 4);
    if (vals) std::memcpy(vals, f.A.values.data(), f.A.nnz() * 8);
    if (b) std::memcpy(b, f.b.data(), f.n * 8);
}
void ref_frame_free(void* h) { delete static_cast<RefFrame*>(h); }

// mppf.cpp:48 write_mppf of make_frame(n, seed, frame_index); mppf.cpp:102 read_mppf -> a frame
// handle for ref_frame_sizes / ref_frame_fill / ref_frame_barriers.
int ref_write_mppf(uint64_t n, uint64_t seed, uint64_t frame_index, const char* path) {
    return guard([&] { write_mppf(make_frame(n, seed, frame_index), path); });
}
void* ref_read_mppf(const char* path) {
    RefFrame* r = nullptr;
    int rc = guard([&] { r = new RefFrame{read_mppf(path)}; });
    return rc == 0 ? r : nullptr;
}
void ref_frame_meta(void* h, uint64_t* seed, uint64_t* frame_index, uint32_t* nbar, double* bars) {
    auto* r = static_cast<RefFrame*>(h);
    *seed = r->f.master_seed;
    *frame_index = r->f.frame_index;
    *nbar = uint32_t(r->f.barriers.size());
    for (size_t i = 0; i < r->f.barriers.size() && i < 3; ++i) {
        bars[4 * i + 0] = double(static_cast<int>(r->f.barriers[i].orientation));
        bars[4 * i + 1] = r->f.barriers[i].center;
        bars[4 * i + 2] = r->f.barriers[i].thickness;
        bars[4 * i + 3] = double(static_cast<int>(r->f.barriers[i].gap));
    }
}

// csr.cpp:70 spmv
int ref_spmv(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
             const double* x, double* y) {
    return guard([&] {
        CsrMatrix A = make_csr(n, ro, ci, v);
        spmv(A, std::span<const double>(x, n), std::span<double>(y, n));
    });
}

// apply.cpp:79 apply<float>
int ref_apply_f32(uint64_t n, uint64_t leaf, uint64_t ls, const float* packed,
                  int spd_enabled, double spd_raw, const double* a_diag, const double* r,
                  double* y) {
    return guard([&] {
        auto f = make_factors<float>(n, leaf, ls, packed, spd_enabled, spd_raw);
        ApplyWorkspace<float> ws(f.layout);
        apply(f, std::span<const double>(a_diag, n), std::span<const double>(r, n), ws,
              std::span<double>(y, n));
    });
}

// apply.cpp:79 apply<double> on factors.cast<double>() — the parity gate's reference
int ref_apply_f64_of_f32(uint64_t n, uint64_t leaf, uint64_t ls, const float* packed,
                         int spd_enabled, double spd_raw, const double* a_diag,
                         const double* r, double* y) {
    return guard([&] {
        auto f = make_factors<float>(n, leaf, ls, packed, spd_enabled, spd_raw).template cast<double>();
        ApplyWorkspace<double> ws(f.layout);
        apply(f, std::span<const double>(a_diag, n), std::span<const double>(r, n), ws,
              std::span<double>(y, n));
    });
}

// Timing helper for the CPU baseline: mean ms of `reps` apply<float> calls (factor copy and
// workspace built once, outside the timed loop — as factor_applier does, pcg.cpp:44-51).
int ref_time_apply_f32(uint64_t n, uint64_t leaf, uint64_t ls, const float* packed,
                       const double* a_diag, const double* r, uint64_t reps, double* ms) {
    return guard([&] {
        auto f = make_factors<float>(n, leaf, ls, packed, 0, 0.0);
        ApplyWorkspace<float> ws(f.layout);
        std::vector<double> y(n);
        auto t0 = std::chrono::steady_clock::now();
        for (uint64_t i = 0; i < reps; ++i)
            apply(f, std::span<const double>(a_diag, n), std::span<const double>(r, n), ws, y);
        *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count() / double(reps);
    });
}

// apply.cpp:184 assemble_dense<float> (n <= 4096)
int ref_assemble_dense_f32(uint64_t n, uint64_t leaf, uint64_t ls, const float* packed,
                           int spd_enabled, double spd_raw, const double* a_diag,
                           double* out) {
    return guard([&] {
        auto f = make_factors<float>(n, leaf, ls, packed, spd_enabled, spd_raw);
        DenseMat M = assemble_dense(f, std::span<const double>(a_diag, n));
        std::memcpy(out, M.data.data(), n * n * 8);
    });
}

// adjoint.cpp:44 factor_apply_batch then :129 factor_apply_batch_adjoint on the same context.
int ref_apply_batch_adjoint(uint64_t n, uint64_t leaf, uint64_t ls, const double* packed, int spd_enabled,
                            double spd_raw, const double* a_diag, const double* x, uint64_t kz,
                            const double* bar_y, double* y_out, double* grad_out) {
    return guard([&] {
        PackedFactors<double> f = make_factors<double>(n, leaf, ls, packed, spd_enabled, spd_raw);
        BatchApplyContext ctx(f.layout, kz);
        std::vector<double> y(n * kz), grad(f.layout.total, 0.0);
        factor_apply_batch(f, std::span<const double>(a_diag, n), std::span<const double>(x, n * kz), ctx, y);
        std::memcpy(y_out, y.data(), n * kz * 8);
        if (bar_y) {
            factor_apply_batch_adjoint(f, std::span<const double>(a_diag, n), std::span<const double>(bar_y, n * kz),
                                       ctx, grad);
            std::memcpy(grad_out, grad.data(), grad.size() * 8);
        }
    });
}

// adjoint.cpp:250 loss_gradient (kind 0 cosine, 1 sai).
int ref_loss_gradient(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v, uint64_t leaf,
                      uint64_t ls, const double* packed, const double* z, uint64_t kz, int kind, double norm_a,
                      double* loss, int* degenerate, double* grad_out) {
    return guard([&] {
        CsrMatrix A = make_csr(n, ro, ci, v);
        PackedFactors<double> f = make_factors<double>(n, leaf, ls, packed, 0, 0.0);
        BatchApplyContext ctx(f.layout, kz);
        LossGradResult r = loss_gradient(f, A, std::span<const double>(z, n * kz), kz,
                                         kind ? LossKind::sai : LossKind::cosine, norm_a, ctx);
        *loss = r.loss;
        *degenerate = r.degenerate ? 1 : 0;
        std::memcpy(grad_out, r.grad.data(), r.grad.size() * 8);
    });
}

// ic0.cpp:10 ic0_factorize (policy 0 none, 1 scaled) -> the lower factor as CSR.
int ref_ic0_factorize(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v, int policy,
                      uint64_t* lro, uint32_t* lci, double* lv, uint64_t cap, uint64_t* nnz_out,
                      double* shift_out) {
    return guard([&] {
        Ic0Factor f = ic0_factorize(make_csr(n, ro, ci, v), policy ? Ic0Shift::scaled : Ic0Shift::none);
        *nnz_out = f.lower.col_indices.size();
        *shift_out = f.shift;
        if (cap < *nnz_out) throw std::invalid_argument("ref_ic0_factorize: capacity");
        std::memcpy(lro, f.lower.row_offsets.data(), (n + 1) * 8);
        std::memcpy(lci, f.lower.col_indices.data(), *nnz_out * 4);
        std::memcpy(lv, f.lower.values.data(), *nnz_out * 8);
    });
}

// ic0.cpp:72 ic0_applier(ic0_factorize(A, policy)) applied to r.
int ref_ic0_apply(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v, int policy,
                  const double* r, double* z) {
    return guard([&] {
        PrecondApplier pa = ic0_applier(ic0_factorize(make_csr(n, ro, ci, v),
                                                      policy ? Ic0Shift::scaled : Ic0Shift::none));
        pa(std::span<const double>(r, n), std::span<double>(z, n));
    });
}

// pcg.cpp:53 pcg_solve with identity (0) / jacobi (1) / factor (2) applier (pcg.cpp:28-51),
// or (3) ic0_applier(ic0_factorize(A)) as hfp solve --method ic0 (hfp_cli.cpp:80).
// report_out: {iterations, converged, status(0 conv,1 max,2 breakdown), breakdown_iter,
//              history_len, wall_ms}
int ref_pcg_solve(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                  const double* b, int kind, uint64_t leaf, uint64_t ls, const float* packed,
                  int spd_enabled, double spd_raw, double rtol, uint64_t max_iters,
                  double* x_out, double* history_out, double* report_out) {
    return guard([&] {
        CsrMatrix A = make_csr(n, ro, ci, v);
        PrecondApplier pa;
        if (kind == 0) pa = identity_applier();
        else if (kind == 1) pa = jacobi_applier(A);
        else if (kind == 3) pa = ic0_applier(ic0_factorize(A));
        else pa = factor_applier(make_factors<float>(n, leaf, ls, packed, spd_enabled, spd_raw), A);
        SolveConfig cfg;
        cfg.rtol = rtol;
        cfg.max_iters = max_iters;
        std::vector<double> x;
        SolveReport rep = pcg_solve(A, std::span<const double>(b, n), pa, cfg, &x);
        if (x_out) std::memcpy(x_out, x.data(), n * 8);
        if (history_out)
            std::memcpy(history_out, rep.residual_history.data(),
                        rep.residual_history.size() * 8);
        report_out[0] = double(rep.iterations);
        report_out[1] = rep.converged ? 1.0 : 0.0;
        report_out[2] = rep.status == SolveStatus::converged   ? 0.0
                        : rep.status == SolveStatus::max_iters ? 1.0
                                                               : 2.0;
        report_out[3] = double(rep.breakdown_iter);
        report_out[4] = double(rep.residual_history.size());
        report_out[5] = rep.wall_ms;
    });
}

// Bounded-sample CPU baseline: the reference PCG loop (pcg.cpp:86-119 body, same calls:
// spmv + dots + axpys + factor_applier) run for exactly `iters` iterations; returns ms.
int ref_pcg_time_iters(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                       const double* b, uint64_t leaf, uint64_t ls, const float* packed,
                       uint64_t iters, double* ms_out) {
    return guard([&] {
        CsrMatrix A = make_csr(n, ro, ci, v);
        PrecondApplier pa = factor_applier(make_factors<float>(n, leaf, ls, packed, 0, 0.0), A);
        SolveConfig cfg;
        cfg.rtol = 1e-300; // never converges inside the sample; runs exactly `iters`
        cfg.max_iters = iters;
        SolveReport rep = pcg_solve(A, std::span<const double>(b, n), pa, cfg);
        *ms_out = rep.wall_ms;
    });
}

// checkpoint.cpp:17 / :45 HFTC I/O
int ref_write_checkpoint(const char* path, uint64_t n, uint64_t leaf, uint64_t ls,
                         const float* packed, int spd_enabled, double spd_raw,
                         const char* metadata_json) {
    return guard([&] {
        auto f = make_factors<float>(n, leaf, ls, packed, spd_enabled, spd_raw);
        write_checkpoint(f, path, metadata_json ? metadata_json : "{}");
    });
}
int ref_read_checkpoint(const char* path, uint64_t* n, uint64_t* leaf, uint64_t* ls,
                        uint64_t* total, float* packed /* may be null: sizes only */) {
    return guard([&] {
        Checkpoint ck = read_checkpoint(path);
        *n = ck.factors.layout.n;
        *leaf = ck.factors.layout.leaf_size;
        *ls = ck.factors.layout.coarse_size;
        *total = ck.factors.layout.total;
        if (packed) std::memcpy(packed, ck.factors.data.data(), ck.factors.data.size() * 4);
    });
}

// toy_net.cpp:170 init_weights + :322 forward on make_frame(n, seed, frame_index).
// trace_out: {max_attention_row_sum_error, highway_max_deviation, leaf_dispatches,
//             tile_dispatches}
int ref_toynet_forward(uint64_t n, uint64_t seed, uint64_t frame_index, uint64_t leaf,
                       uint64_t ls, uint64_t d, uint64_t layers, uint64_t heads,
                       uint64_t gcn_layers, uint64_t d_global, uint64_t edge_hidden,
                       uint64_t weight_seed, float* out, double* trace_out, double* ms_out) {
    return guard([&] {
        Frame fr = make_frame(n, seed, frame_index);
        HPartition p = build_partition(n, leaf);
        toynet::Config cfg;
        cfg.d = d; cfg.layers = layers; cfg.heads = heads; cfg.gcn_layers = gcn_layers;
        cfg.d_global = d_global; cfg.edge_hidden = edge_hidden;
        toynet::Weights w = toynet::init_weights(cfg, make_factor_layout(p, ls), weight_seed);
        toynet::Trace tr;
        auto t0 = std::chrono::steady_clock::now();
        FactorTensor f = toynet::forward(fr, p, ls, cfg, w, &tr);
        if (ms_out)
            *ms_out = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0).count();
        std::memcpy(out, f.data.data(), f.data.size() * 4);
        if (trace_out) {
            trace_out[0] = tr.max_attention_row_sum_error;
            trace_out[1] = tr.highway_max_deviation;
            trace_out[2] = double(tr.leaf_attention_dispatches);
            trace_out[3] = double(tr.tile_attention_dispatches);
        }
    });
}

// train.cpp:29 train_factors on make_frame(n, frame_seed, idx[i]) (eval: make_frame(n, frame_seed,
// eval_index)); the same hfpg_train_config / log / summary layout as the product's ABI.
int ref_train_factors(uint64_t n, uint64_t frame_seed, const uint64_t* idx, uint64_t nframes,
                      uint64_t eval_index, const hfpg_train_config* c, uint64_t seed, float* factors_out,
                      hfpg_train_log* log_out, uint64_t log_cap, hfpg_train_summary* summary) {
    return guard([&] {
        std::vector<Frame> fr;
        for (uint64_t i = 0; i < nframes; ++i) fr.push_back(make_frame(n, frame_seed, idx[i]));
        Frame ev = make_frame(n, frame_seed, eval_index);
        std::vector<const Frame*> fp;
        for (auto& f : fr) fp.push_back(&f);
        TrainConfig cfg;
        cfg.lr = c->lr;
        cfg.weight_decay = c->weight_decay;
        cfg.clip_norm = c->clip_norm;
        cfg.plateau.factor = c->plateau_factor;
        cfg.plateau.patience = c->plateau_patience;
        cfg.plateau.rel_threshold = c->plateau_rel_threshold;
        cfg.max_steps = c->max_steps;
        cfg.autostop_window = c->autostop_window;
        cfg.probe_omega = c->probe_omega;
        cfg.probe_smooth_steps = c->probe_smooth_steps;
        cfg.contexts_per_step = c->contexts_per_step;
        cfg.loss = c->loss == 1 ? LossKind::sai : LossKind::cosine;
        cfg.log_every = c->log_every;
        cfg.init_sigma = c->init_sigma;
        cfg.leaf_size = c->leaf_size;
        cfg.coarse_size = c->coarse_size;
        cfg.eval_every_logs = c->eval_every_logs;
        cfg.solve_rtol = c->solve_rtol;
        cfg.solve_max_iters = c->solve_max_iters;
        cfg.stop_at_iters = c->stop_at_iters;
        TrainResult r = train_factors(fp, cfg, seed, &ev);
        if (factors_out) std::memcpy(factors_out, r.factors.data.data(), r.factors.data.size() * 4);
        const auto& E = r.history.entries;
        for (size_t i = 0; i < E.size() && i < log_cap; ++i) {
            log_out[i].step = E[i].step;
            log_out[i].train_loss = E[i].train_loss;
            log_out[i].sai_heldout = E[i].sai_heldout;
            log_out[i].pcg_iters_heldout = E[i].pcg_iters_heldout;
            log_out[i].lr = E[i].lr;
            log_out[i].wall_s = E[i].wall_s;
        }
        summary->total_steps = r.history.total_steps;
        summary->auto_stopped = r.history.auto_stopped;
        summary->aborted_divergence = r.history.aborted_divergence;
        summary->reached_target = r.history.reached_target;
        summary->n_entries = E.size();
        summary->leaf_size = r.factors.layout.leaf_size;
        summary->packed_width = r.factors.data.size();
    });
}

} // extern "C"
