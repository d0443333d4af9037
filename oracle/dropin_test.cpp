// TEST INFRASTRUCTURE ONLY — the drop-in check from the reference's side.
//
// Links the UNMODIFIED reference library (oracle/_ref objects) together with include/hfp_gpu.hpp
// + libhfpg.so and runs, on the same make_frame / init_factors inputs:
//   (1) the reference pcg_solve with the reference factor_applier (CPU),
//   (2) the reference pcg_solve with hfp::gpu::factor_applier — the one-line drop-in,
//   (3) hfp::gpu::pcg_solve<hfp::SolveReport> — the whole loop as one CUDA graph,
// and compares one apply bit-for-bit-ish. Prints one JSON line; exit 0 iff (2) and (3) stay
// within +-2 iterations of (1). Built by oracle/Makefile; run by tests/test_gpu_dropin.py.
#include "hfp/apply.hpp"
#include "hfp/frame.hpp"
#include "hfp/pcg.hpp"
#include "hfp_gpu.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
    using namespace hfp;
    const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 8192;
    Frame fr = make_frame(n, 2024, 0);
    HPartition p = build_partition(n, 128);
    RngStream rng(2024, 0, RngPurpose::factor_init);
    FactorTensor f = init_factors<float>(p, 32, FactorInit::jacobi_seed, 1e-2, rng);
    SolveConfig cfg;

    // one apply: reference apply<float> vs the drop-in applier
    ApplyWorkspace<float> ws(f.layout);
    const auto diag = fr.A.diagonal();
    std::vector<double> yr(n), yg(n);
    apply(f, diag, fr.b, ws, yr);
    auto gpu_apply = gpu::factor_applier(f, fr.A);
    gpu_apply(fr.b, yg);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < n; ++i) {
        num += (yg[i] - yr[i]) * (yg[i] - yr[i]);
        den += yr[i] * yr[i];
    }

    SolveReport ref = pcg_solve(fr.A, fr.b, factor_applier(f, fr.A), cfg);
    SolveReport mix = pcg_solve(fr.A, fr.b, gpu_apply, cfg);
    SolveReport dev = gpu::pcg_solve<SolveReport>(fr.A, fr.b, gpu::Precond::factor(f, fr.A), cfg);
    // a Precond bound to A must solve the A it is handed: an edited operator (values of A
    // scaled) gives the same report as a Precond built from the edited operator itself
    CsrMatrix A2 = fr.A;
    for (double& v : A2.values) v *= 3.0;
    const gpu::Precond pj = gpu::Precond::jacobi(fr.A);
    SolveReport stale = gpu::pcg_solve<SolveReport>(A2, fr.b, pj, cfg);
    SolveReport fresh = gpu::pcg_solve<SolveReport>(A2, fr.b, gpu::Precond::jacobi(A2), cfg);
    const bool rebind_ok = stale.iterations == fresh.iterations &&
                           stale.residual_history == fresh.residual_history;
    const bool ok = rebind_ok && ref.converged && mix.converged && dev.converged &&
                    std::llabs((long long)mix.iterations - (long long)ref.iterations) <= 2 &&
                    std::llabs((long long)dev.iterations - (long long)ref.iterations) <= 2;
    std::printf("{\"n\": %zu, \"apply_rel_l2_vs_ref_f32\": %.3e, \"ref_iterations\": %zu, "
                "\"ref_wall_ms\": %.2f, \"dropin_applier_iterations\": %zu, "
                "\"dropin_applier_wall_ms\": %.2f, \"gpu_pcg_iterations\": %zu, "
                "\"gpu_pcg_wall_ms\": %.3f, \"rebind_ok\": %s, \"ok\": %s}\n",
                n, std::sqrt(num / den), ref.iterations, ref.wall_ms, mix.iterations,
                mix.wall_ms, dev.iterations, dev.wall_ms, rebind_ok ? "true" : "false", ok ? "true" : "false");
    return ok ? 0 : 1;
}
