// train_factors (train.cpp:29-217) on the GPU: direct self-supervised optimisation of the packed
// factor tensor — the only source of convergent, better-than-Jacobi tensors.
//
// The device does the work that scales: per context the smoothed probe batch goes up once and
// hfpg_loss_gradient (batched apply + hand adjoint, train.cuh) runs on the frame's handle;
// gradients accumulate and AdamW updates the f64 master parameters on the device
// (hfpg_adamw_step); the held-out evaluation solves with the reference's exact PCG semantics
// (hfpg_pcg_solve_exact) and the batched apply. The host keeps what the reference keeps on its
// single thread — the counter-based draws (probes, the frame choice), the probe smoothing and the
// power iteration, written as the reference's loops and compiled with the same contraction
// settings so they round alike — plus the scalar schedule (plateau, auto-stop, divergence abort,
// target exit) and the log.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace hfpg {
namespace {

#define TLCK(call)                                                                        \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

void abi(int rc) {
    if (rc != HFPG_OK) {
        const std::string msg = hfpg_last_error();
        if (rc == HFPG_EINVAL) throw InvalidArgument(msg);
        throw IoError(msg);
    }
}

constexpr uint64_t kProbesPurpose = 3, kPowerIterPurpose = 6, kFactorInitPurpose = 4;
// probe batches up to this many entries are drawn and smoothed on the host exactly as the
// reference does (libm log / cos); larger ones on the device (hfpg_probes_device)
constexpr uint64_t kHostProbeMax = uint64_t(1) << 22;

struct HostCsr {
    uint64_t n = 0;
    const uint64_t* ro = nullptr;
    const uint32_t* ci = nullptr;
    const double* v = nullptr;
    std::vector<double> diag() const {  // csr.cpp:52-58
        std::vector<double> d(n, 0.0);
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t p = ro[i]; p < ro[i + 1]; ++p)
                if (ci[p] == i) d[i] = v[p];
        return d;
    }
};

template <class Fn>
void par_rows(uint64_t n, Fn fn) {
    uint64_t nt = std::max(1u, std::thread::hardware_concurrency());
    nt = std::min<uint64_t>(nt, std::max<uint64_t>(1, n / 256));
    if (nt <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < nt; ++t) th.emplace_back([=] { fn(n * t / nt, n * (t + 1) / nt); });
    for (auto& x : th) x.join();
}

// csr.cpp:87-100 spmm, rows split over threads (each row's sums keep the reference's order)
void spmm_host(const HostCsr& A, const double* X, uint64_t k, double* Y) {
    par_rows(A.n, [&](uint64_t r0, uint64_t r1) {
        for (uint64_t i = r0; i < r1; ++i) {
            double* yi = Y + i * k;
            for (uint64_t j = 0; j < k; ++j) yi[j] = 0.0;
            for (uint64_t p = A.ro[i]; p < A.ro[i + 1]; ++p) {
                const double a = A.v[p];
                const double* xr = X + uint64_t(A.ci[p]) * k;
                for (uint64_t j = 0; j < k; ++j) yi[j] += a * xr[j];
            }
        }
    });
}
// csr.cpp:70-79 spmv
void spmv_host(const HostCsr& A, const double* x, double* y) {
    for (uint64_t i = 0; i < A.n; ++i) {
        double acc = 0.0;
        for (uint64_t p = A.ro[i]; p < A.ro[i + 1]; ++p) acc += A.v[p] * x[A.ci[p]];
        y[i] = acc;
    }
}

// probes.cpp:8-12
uint64_t probe_count(uint64_t n) {
    const auto root = static_cast<uint64_t>(std::ceil(std::sqrt(static_cast<double>(n))));
    return std::max<uint64_t>(64, root);
}
// probes.cpp:14-21 sample_probes: the stream's next n kz normals (counter advanced)
void sample_probes(Rng& s, uint64_t count, double* z) {
    const uint64_t c0 = s.counter;
    par_rows(count, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) z[i] = Rng::normal_of(s.bits_at(c0 + i));
    });
    s.counter = c0 + count;
}
// probes.cpp:23-44 smooth_probes (diag checked positive by the caller)
void smooth_probes(const HostCsr& A, const std::vector<double>& diag, double* z, uint64_t k, double omega,
                   uint64_t steps, std::vector<double>& az) {
    az.resize(A.n * k);
    for (uint64_t s = 0; s < steps; ++s) {
        spmm_host(A, z, k, az.data());
        par_rows(A.n, [&](uint64_t r0, uint64_t r1) {
            for (uint64_t i = r0; i < r1; ++i) {
                const double scale = omega / diag[i];
                double* zi = z + i * k;
                const double* ai = az.data() + i * k;
                for (uint64_t j = 0; j < k; ++j) zi[j] -= scale * ai[j];
            }
        });
    }
}
// loss.cpp:37-55 power_iteration_norm
double power_iteration_norm(const HostCsr& A, Rng& s, uint64_t steps = 50) {
    const uint64_t n = A.n;
    std::vector<double> v(n), av(n);
    for (double& x : v) x = s.normal();
    double norm = 0.0;
    for (double x : v) norm += x * x;
    norm = std::sqrt(norm);
    for (double& x : v) x /= norm;
    double sigma = 0.0;
    for (uint64_t st = 0; st < steps; ++st) {
        spmv_host(A, v.data(), av.data());
        sigma = 0.0;
        for (double x : av) sigma += x * x;
        sigma = std::sqrt(sigma);
        if (sigma == 0.0) return 0.0;
        for (uint64_t i = 0; i < n; ++i) v[i] = av[i] / sigma;
    }
    return sigma;
}
// loss.cpp:22-35 sai_loss
double sai_loss(const HostCsr& A, const double* mz, const double* z, uint64_t kz, double norm_a) {
    std::vector<double> amz(A.n * kz);
    spmm_host(A, mz, kz, amz.data());
    double acc = 0.0;
    for (uint64_t i = 0; i < amz.size(); ++i) {
        const double q = amz[i] / norm_a - z[i];
        acc += q * q;
    }
    return acc;
}

__global__ void k_axpy1(double* __restrict__ g, const double* __restrict__ x, uint64_t n) {  // g += x
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        g[i] += x[i];
}
__global__ void k_scale(double* __restrict__ g, double s, uint64_t n) {  // g *= s (train.cpp:130)
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        g[i] *= s;
}
__global__ void k_to_float(const double* __restrict__ p, float* __restrict__ f, uint64_t n) {  // params.cast<float>()
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        f[i] = static_cast<float>(p[i]);
}
__global__ void k_to_double(const float* __restrict__ f, double* __restrict__ p, uint64_t n) {  // f.cast<double>()
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = static_cast<double>(f[i]);
}

struct Handle {
    hfpg_handle* h = nullptr;
    ~Handle() {
        if (h) hfpg_destroy(h);
    }
};
template <class T>
struct DBuf {
    T* p = nullptr;
    explicit DBuf(uint64_t n) { TLCK(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T))); }
    ~DBuf() { cudaFree(p); }
};

}  // namespace
}  // namespace hfpg

extern "C" int hfpg_train_factors(const hfpg_train_frame* frames, uint64_t nframes, const hfpg_train_frame* eval,
                                  const hfpg_train_config* cfg, uint64_t seed, int device, float* factors_out,
                                  hfpg_train_log* log_out, uint64_t log_cap, hfpg_train_summary* summary) {
    using namespace hfpg;
    return guarded([&] {
        if (!frames || nframes == 0) throw InvalidArgument("train_factors: no frames");
        if (!cfg || !summary) throw InvalidArgument("train_factors: null config / summary");
        const uint64_t n = frames[0].view.n;
        for (uint64_t i = 0; i < nframes; ++i)
            if (frames[i].view.n != n) throw InvalidArgument("train_factors: frames must share N");
        if (!eval) eval = &frames[0];
        if (eval->view.n != n) throw InvalidArgument("train_factors: eval frame size");
        const hfpg_train_config& C = *cfg;
        const uint64_t leaf = (n < 2 * C.leaf_size) ? n / 2 : C.leaf_size;  // partition.hpp:48-50
        const Layout L = make_layout(n, leaf, C.coarse_size);
        const uint64_t kz = probe_count(n), P = L.total, nk = n * kz;

        auto csr_of = [&](const hfpg_train_frame& f) {
            HostCsr A;
            A.n = f.view.n;
            A.ro = f.view.row_offsets;
            A.ci = f.view.col_indices;
            A.v = f.view.values;
            return A;
        };
        // ---- per-frame device handles (operator + training workspace), diagonals, norms
        std::vector<std::unique_ptr<Handle>> hs;
        std::vector<std::vector<double>> diags;
        std::vector<double> norms(nframes, 0.0);
        for (uint64_t i = 0; i < nframes; ++i) {
            auto hd = std::make_unique<Handle>();
            abi(hfpg_create(device, &hd->h));
            const HostCsr A = csr_of(frames[i]);
            abi(hfpg_load_csr(hd->h, n, A.ro, A.ci, A.v, HFPG_HOST));
            diags.push_back(A.diag());
            for (double d : diags.back())
                if (!(d > 0.0)) throw InvalidArgument("smooth_probes: nonpositive diagonal");
            if (C.loss == 1) {
                Rng ps(seed, frames[i].frame_index, kPowerIterPurpose);
                norms[i] = power_iteration_norm(A, ps);
            }
            hs.push_back(std::move(hd));
        }
        const HostCsr EA = csr_of(*eval);
        Rng eval_power(seed, eval->frame_index, kPowerIterPurpose);
        const double eval_norm = power_iteration_norm(EA, eval_power);
        const std::vector<double> eval_diag = EA.diag();
        for (double d : eval_diag)
            if (!(d > 0.0)) throw InvalidArgument("smooth_probes: nonpositive diagonal");
        // fixed, pre-smoothed evaluation probes (train.cpp:64-69)
        std::vector<double> az, eval_z(nk);
        {
            Rng es(seed ^ 0x5eedULL, eval->frame_index, kProbesPurpose);
            sample_probes(es, nk, eval_z.data());
            smooth_probes(EA, eval_diag, eval_z.data(), kz, C.probe_omega, C.probe_smooth_steps, az);
        }
        Handle eh;  // evaluation: operator, snapshot factors, exact PCG, batched apply
        abi(hfpg_create(device, &eh.h));
        abi(hfpg_load_csr(eh.h, n, EA.ro, EA.ci, EA.v, HFPG_HOST));
        abi(hfpg_set_precond(eh.h, HFPG_PRECOND_FACTOR));

        // ---- parameters: init_factors<double>(jacobi_seed, init_sigma) (factor_tensor.cpp:30-39)
        std::vector<double> hp(P);
        {
            const Rng s(seed, 0, kFactorInitPurpose);
            for (uint64_t i = 0; i < L.gate_base; ++i)
                hp[i] = C.init_sigma == 0.0 ? 0.0 : C.init_sigma * Rng::normal_of(s.bits_at(i));
            for (uint64_t i = L.gate_base; i < P; ++i) hp[i] = 1.0;
        }
        DBuf<double> params(P), m1(P), m2(P), grad(P), gctx(P), pd(P), zdev(nk), wdev(nk), b_eval(n), x_eval(n);
        DBuf<float> snap(P);
        cudaStream_t st = nullptr;  // every device step below is ordered on the first frame's handle stream
        TLCK(cudaMemcpy(params.p, hp.data(), P * 8, cudaMemcpyHostToDevice));
        TLCK(cudaMemset(m1.p, 0, P * 8));
        TLCK(cudaMemset(m2.p, 0, P * 8));
        DBuf<double> eval_zd(nk);
        TLCK(cudaMemcpy(eval_zd.p, eval_z.data(), nk * 8, cudaMemcpyHostToDevice));
        TLCK(cudaMemcpy(b_eval.p, eval->b, n * 8, cudaMemcpyHostToDevice));
        const unsigned eg = unsigned(std::min<uint64_t>((P + 255) / 256, 4096));

        double lr = C.lr;
        const double min_lr = std::max(C.lr * 1e-3, 1e-6);
        double sched_best = std::numeric_limits<double>::infinity(), stop_best = sched_best;
        uint64_t sched_bad = 0, stop_bad = 0, diverged_logs = 0, logs_emitted = 0, n_log = 0;
        Rng train_stream(seed, 1, kProbesPurpose);
        double window_loss = 0.0;
        uint64_t window_count = 0;
        bool auto_stopped = false, aborted = false, reached = false;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<double> z(nk <= kHostProbeMax ? nk : 0), w(nk);

        auto eval_now = [&](hfpg_train_log& e) {
            k_to_float<<<eg, 256, 0, st>>>(params.p, snap.p, P);
            TLCK(cudaGetLastError());
            TLCK(cudaStreamSynchronize(st));
            abi(hfpg_load_factors(eh.h, n, leaf, C.coarse_size, snap.p, P, 0, 0.0, HFPG_DEVICE));
            hfpg_solve_config sc{C.solve_rtol, C.solve_max_iters};
            hfpg_report rep{};
            abi(hfpg_pcg_solve_exact(eh.h, b_eval.p, &sc, x_eval.p, nullptr, &rep, HFPG_DEVICE));
            e.pcg_iters_heldout = rep.iterations;
            k_to_double<<<eg, 256, 0, st>>>(snap.p, pd.p, P);
            TLCK(cudaGetLastError());
            TLCK(cudaStreamSynchronize(st));
            abi(hfpg_batch_apply(eh.h, pd.p, leaf, C.coarse_size, 0.0, eval_zd.p, kz, wdev.p, HFPG_DEVICE));
            TLCK(cudaMemcpy(w.data(), wdev.p, nk * 8, cudaMemcpyDeviceToHost));
            e.sai_heldout = sai_loss(EA, w.data(), eval_z.data(), kz, eval_norm);
        };

        uint64_t step = 0;
        for (step = 1; step <= C.max_steps; ++step) {
            TLCK(cudaMemset(grad.p, 0, P * 8));
            double step_loss = 0.0;
            uint64_t valid = 0;
            for (uint64_t c = 0; c < C.contexts_per_step; ++c) {
                const uint64_t fi = nframes == 1 ? 0 : train_stream.below(nframes);
                if (nk <= kHostProbeMax) {  // libm normals and host sweeps, as the reference rounds them
                    sample_probes(train_stream, nk, z.data());
                    smooth_probes(csr_of(frames[fi]), diags[fi], z.data(), kz, C.probe_omega, C.probe_smooth_steps, az);
                    TLCK(cudaMemcpy(zdev.p, z.data(), nk * 8, cudaMemcpyHostToDevice));
                } else {  // large batches: drawn and smoothed on the device
                    abi(hfpg_probes_device(hs[fi]->h, train_stream.key, train_stream.counter, kz, C.probe_omega,
                                           C.probe_smooth_steps, zdev.p));
                    train_stream.counter += nk;
                }
                double loss = 0.0;
                int32_t deg = 0;
                abi(hfpg_loss_gradient(hs[fi]->h, params.p, leaf, C.coarse_size, 0.0, zdev.p, kz, C.loss, norms[fi],
                                       &loss, &deg, gctx.p, HFPG_DEVICE));
                if (deg) continue;  // adjoint.cpp: a degenerate context is skipped
                k_axpy1<<<eg, 256, 0, st>>>(grad.p, gctx.p, P);
                TLCK(cudaGetLastError());
                TLCK(cudaStreamSynchronize(st));  // gctx is rewritten on the handle's (non-blocking) stream
                step_loss += loss;
                ++valid;
            }
            if (valid == 0) continue;  // fully degenerate step, skipped
            const double inv = 1.0 / static_cast<double>(valid);
            k_scale<<<eg, 256, 0, st>>>(grad.p, inv, P);
            TLCK(cudaGetLastError());
            TLCK(cudaStreamSynchronize(st));
            step_loss *= inv;
            window_loss += step_loss;
            ++window_count;
            double gnorm = 0.0;  // global clip + AdamW (train.cpp:136-160)
            abi(hfpg_adamw_step(hs[0]->h, params.p, grad.p, m1.p, m2.p, P, step, lr, 0.9, 0.999, 1e-8, C.weight_decay,
                                C.clip_norm, &gnorm));
            if (step % C.log_every != 0) continue;

            const double metric = window_loss / static_cast<double>(window_count);
            window_loss = 0.0;
            window_count = 0;
            ++logs_emitted;
            hfpg_train_log e{};
            e.step = step;
            e.train_loss = metric;
            e.lr = lr;
            e.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (C.eval_every_logs != 0 && logs_emitted % C.eval_every_logs == 0) eval_now(e);
            if (log_out && n_log < log_cap) log_out[n_log] = e;
            ++n_log;
            // plateau schedule (relative threshold, min mode)
            if (metric < sched_best * (1.0 - C.plateau_rel_threshold)) {
                sched_best = metric;
                sched_bad = 0;
            } else if (++sched_bad > C.plateau_patience) {
                lr = std::max(lr * C.plateau_factor, min_lr);
                sched_bad = 0;
            }
            // auto-stop (its window does not reset on LR drops)
            if (metric < stop_best * (1.0 - C.plateau_rel_threshold)) {
                stop_best = metric;
                stop_bad = 0;
            } else {
                ++stop_bad;
            }
            if (lr <= min_lr && stop_bad >= C.autostop_window) {
                auto_stopped = true;
                break;
            }
            if (C.loss == 0) {  // divergence abort: cosine objective only
                diverged_logs = (metric > 1.9) ? diverged_logs + 1 : 0;
                if (diverged_logs >= 20) {
                    aborted = true;
                    break;
                }
            }
            if (C.stop_at_iters != 0 && e.pcg_iters_heldout != 0 && e.pcg_iters_heldout <= C.stop_at_iters) {
                reached = true;
                break;
            }
        }
        k_to_float<<<eg, 256, 0, st>>>(params.p, snap.p, P);
        TLCK(cudaGetLastError());
        TLCK(cudaStreamSynchronize(st));
        if (factors_out) TLCK(cudaMemcpy(factors_out, snap.p, P * 4, cudaMemcpyDeviceToHost));
        summary->total_steps = std::min(step, C.max_steps);
        summary->auto_stopped = auto_stopped;
        summary->aborted_divergence = aborted;
        summary->reached_target = reached;
        summary->n_entries = n_log;
        summary->leaf_size = leaf;
        summary->packed_width = P;
    });
}
