"""include/hfp_gpu.hpp compiles against reference-shaped types (duck-typed drop-in), CPU only."""
import os
import subprocess
import tempfile

from conftest import ROOT

SRC = r'''
#include "hfp_gpu.hpp"
#include <cstdint>
#include <vector>
namespace hfp {
struct CsrMatrix { std::size_t n_rows = 0, n_cols = 0; std::vector<std::uint64_t> row_offsets;
                   std::vector<std::uint32_t> col_indices; std::vector<double> values; };
struct FactorLayout { std::size_t n = 0, leaf_size = 0, coarse_size = 0; };
struct FactorTensor { FactorLayout layout; std::vector<float> data; bool spd_shift_enabled = false;
                      double spd_shift_raw = 0.0; };
enum class SolveStatus { converged, max_iters, breakdown };
struct SolveReport { std::string method; std::size_t n = 0, iterations = 0; bool converged = false;
                     SolveStatus status = SolveStatus::max_iters; std::vector<double> residual_history;
                     double wall_ms = 0.0; std::string frame_id; std::size_t breakdown_iter = 0; };
struct SolveConfig { double rtol = 1e-8; std::size_t max_iters = 20000; };
}
void use(const hfp::CsrMatrix& A, const hfp::FactorTensor& f, std::vector<double>& b) {
    std::function<void(std::span<const double>, std::span<double>)> M = hfp::gpu::factor_applier(f, A);
    hfp::SolveReport r = hfp::gpu::pcg_solve<hfp::SolveReport>(A, b, hfp::gpu::Precond::factor(f, A),
                                                               hfp::SolveConfig{});
    (void)M; (void)r;
}
'''


def test_header_compiles_with_reference_shaped_types():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.cpp")
        open(src, "w").write(SRC)
        r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                            src], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_c_header_is_plain_c():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        open(src, "w").write('#include "hfpg.h"\nint main(void){hfpg_handle* h = 0; (void)h; return 0;}\n')
        r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I",
                            os.path.join(ROOT, "include"), src], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
