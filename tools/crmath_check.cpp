// Host check of crmath.cuh on the frame generator's own inputs: every 16th draw against the
// __float128 log/cos rounded once (must agree: exit 1 otherwise), and all draws against glibc's
// libm (reported: glibc 2.39's log/cos are not correctly rounded, ~0.1% of draws are 1 ulp off).
// Build: g++ -O3 -march=x86-64-v3 -ffp-contract=fast -fopenmp tools/crmath_check.cpp -lquadmath
// Usage: crmath_check [log2 samples] [key]
#include "../paper_2605_13343_b200/csrc/crmath.cuh"
#include <quadmath.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 24;
    const uint64_t key = argc > 2 ? strtoull(argv[2], 0, 0) : mix64(mix64(mix64(0) ^ 0) ^ 2);
    const uint64_t n = 1ULL << lg;
    unsigned long long bad_log = 0, bad_cos = 0, bad_norm = 0, bad_q = 0, nq = 0;
#pragma omp parallel for reduction(+ : bad_log, bad_cos, bad_norm, bad_q, nq) schedule(static, 65536)
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t bits = mix64(key ^ i);
        const double u1 = (double(bits >> 32) + 1.0) * 0x1.0p-32;
        const double u2 = double(bits & 0xFFFFFFFFULL) * 0x1.0p-32;
        const double y = 2.0 * 3.14159265358979323846 * u2;
        const double lg_ = std::log(u1), lc = crm::log_cr(u1);
        const double cg = std::cos(y), cc = crm::cos_cr(y);
        if (!same(lg_, lc)) bad_log++;
        if (!same(cg, cc)) bad_cos++;
        const double ng = std::sqrt(-2.0 * lg_) * cg;
        if (!same(ng, crm::normal_of_cr(bits))) bad_norm++;
        if ((i & 15) == 0) {
            nq++;
            const double ql = (double)logq((__float128)u1), qc = (double)cosq((__float128)y);
            if (!same(ql, lc) || !same(qc, cc)) bad_q++;
        }
    }
    std::printf("{\"samples\": %llu, \"log_mismatch\": %llu, \"cos_mismatch\": %llu, "
                "\"normal_mismatch\": %llu, \"quad_checked\": %llu, \"quad_mismatch\": %llu}\n",
                (unsigned long long)n, bad_log, bad_cos, bad_norm, nq, bad_q);
    return bad_q ? 1 : 0;  // glibc itself is not correctly rounded: its mismatches are reported only
}
