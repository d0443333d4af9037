/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the hfp solve-time hot path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj, C++20 library
 * `hfp`). Each function cites the reference file:line it restates. It is pinned against the
 * reference itself (oracle/_ref/libhfpref.so, built from the unmodified sources by
 * oracle/Makefile) and against the committed golden fixtures in tests/golden/ — see
 * tests/test_oracle.py. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it; the product library never does.
 */
#ifndef HFP_ORACLE_H
#define HFP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:12-20 */
enum { ORC_DENSITY = 1, ORC_RHS = 2, ORC_PROBES = 3, ORC_FACTOR_INIT = 4, ORC_NET_WEIGHTS = 5 };

typedef struct {
    uint64_t key;
    uint64_t counter;
} orc_rng;

void orc_rng_init(orc_rng* s, uint64_t seed, uint64_t frame, uint64_t purpose);
uint64_t orc_rng_bits(orc_rng* s);
double orc_rng_normal(orc_rng* s);

/* partition.cpp:9-53 — tiles as rows {id, span, row_begin, col_begin, depth} */
int orc_partition(uint64_t n, uint64_t leaf, uint64_t* tiles_out);
int orc_packed_width(uint64_t n, uint64_t leaf, uint64_t ls, uint64_t* out);

/* factor_tensor.cpp:30-39 */
int orc_init_factors_f32(uint64_t n, uint64_t leaf, uint64_t ls, double sigma, uint64_t seed,
                         uint64_t frame, float* out);

/* csr.cpp:70-79 */
void orc_spmv(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
              const double* x, double* y);

/* apply.cpp:79-174; returns 0 or -1 on a contract violation */
int orc_apply_f32(uint64_t n, uint64_t leaf, uint64_t ls, const float* packed, int spd_enabled,
                  double spd_raw, const double* a_diag, const double* r, double* y);
int orc_apply_f64(uint64_t n, uint64_t leaf, uint64_t ls, const double* packed,
                  int spd_enabled, double spd_raw, const double* a_diag, const double* r,
                  double* y);

/* pcg.cpp:53-126 with identity (0) / jacobi (1) / factor (2) appliers (pcg.cpp:28-51).
 * report_out: {iterations, converged, status(0 conv, 1 max_iters, 2 breakdown),
 *              breakdown_iter, history_len} */
int orc_pcg_solve(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                  const double* b, int kind, uint64_t leaf, uint64_t ls, const float* packed,
                  int spd_enabled, double spd_raw, double rtol, uint64_t max_iters,
                  double* x_out, double* history_out, double* report_out);

/* frame.cpp:147-152 / csr.cpp:64-68 sequential sums (squares: s = fma(x, x, s)) */
double orc_seq_sum(const double* x, uint64_t n, int squares);

#ifdef __cplusplus
}
#endif
#endif
