/* TEST INFRASTRUCTURE ONLY — see hfp_oracle.h. Plain-C restatement of the reference's
 * solve-time hot path. Citations are relative to /root/reference/proj. The accumulator
 * precisions and summation orders follow the reference exactly (the tests assert bit
 * equality against oracle/_ref where the reference is deterministic), so this file is also
 * compiled with FMA contraction on, like the reference's gnu++20 -O3 build. */
#include "hfp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:25-30 SplitMix64 finaliser ---------------------------------------------- */
static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.hpp:39-41: key = mix(mix(mix(seed) ^ frame) ^ purpose) */
void orc_rng_init(orc_rng* s, uint64_t seed, uint64_t frame, uint64_t purpose) {
    s->key = mix64(mix64(mix64(seed) ^ frame) ^ purpose);
    s->counter = 0;
}

/* rng.hpp:43 */
uint64_t orc_rng_bits(orc_rng* s) { return mix64(s->key ^ s->counter++); }

/* rng.hpp:61-70: Box-Muller, one normal per 64-bit draw; u1 from the high word (0,1],
 * u2 from the low word [0,1). */
double orc_rng_normal(orc_rng* s) {
    const uint64_t bits = orc_rng_bits(s);
    const double u1 = ((double)(bits >> 32) + 1.0) * 0x1.0p-32;
    const double u2 = (double)(bits & 0xFFFFFFFFULL) * 0x1.0p-32;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* ---- partition.cpp:9-46 ------------------------------------------------------------------ */
static int valid_partition(uint64_t n, uint64_t leaf) {
    if (leaf == 0 || n % leaf != 0) return 0;
    const uint64_t k = n / leaf;
    return k >= 2 && (k & (k - 1)) == 0;
}

/* Breadth-first bisection: depth d has 2^d nodes of width K/2^d leaves; node i emits the
 * tile (rows [i*w, i*w+w/2), cols [i*w+w/2, (i+1)*w)). */
int orc_partition(uint64_t n, uint64_t leaf, uint64_t* tiles_out) {
    if (!valid_partition(n, leaf)) return -1;
    const uint64_t k = n / leaf;
    uint64_t id = 0;
    for (uint64_t depth = 0, nodes = 1, width = k; width >= 2; ++depth, nodes *= 2, width /= 2)
        for (uint64_t i = 0; i < nodes; ++i, ++id) {
            uint64_t* t = tiles_out + 5 * id;
            t[0] = id;
            t[1] = width / 2;
            t[2] = i * width;
            t[3] = i * width + width / 2;
            t[4] = depth;
        }
    return 0;
}

/* partition.cpp:48-53, factor_tensor.cpp:7-28 (L_s | L and L_s even) */
int orc_packed_width(uint64_t n, uint64_t leaf, uint64_t ls, uint64_t* out) {
    if (!valid_partition(n, leaf) || ls == 0 || leaf % ls != 0) return -1;
    const uint64_t k = n / leaf;
    *out = k * leaf * leaf + (k - 1) * ls * ls + 2 * n * ls + n;
    return 0;
}

typedef struct {
    uint64_t n, l, ls, rk, k, m;
    uint64_t tile_base, bridge_base, gate_base, total;
} layout_t;

/* factor_tensor.hpp:34-47 section offsets */
static int make_layout(uint64_t n, uint64_t leaf, uint64_t ls, layout_t* L) {
    if (!valid_partition(n, leaf) || ls == 0 || leaf % ls != 0 || ls % 2 != 0) return -1;
    L->n = n; L->l = leaf; L->ls = ls; L->rk = ls / 2;
    L->k = n / leaf; L->m = L->k - 1;
    L->tile_base = L->k * leaf * leaf;
    L->bridge_base = L->tile_base + L->m * ls * ls;
    L->gate_base = L->bridge_base + 2 * n * ls;
    L->total = L->gate_base + n;
    return 0;
}
#define LEAF_F(L, k) ((k) * (L)->l * (L)->l)
#define TILE_U(L, t) ((L)->tile_base + (t) * (L)->ls * (L)->ls)
#define TILE_V(L, t) (TILE_U(L, t) + (L)->ls * (L)->rk)
#define BRIDGE_U(L, k) ((L)->bridge_base + (k) * 2 * (L)->l * (L)->ls)
#define BRIDGE_V(L, k) (BRIDGE_U(L, k) + (L)->l * (L)->ls)

/* ---- factor_tensor.cpp:30-39: sigma * N(0,1) below the gate, gate = 1 -------------------- */
int orc_init_factors_f32(uint64_t n, uint64_t leaf, uint64_t ls, double sigma, uint64_t seed,
                         uint64_t frame, float* out) {
    layout_t L;
    if (make_layout(n, leaf, ls, &L)) return -1;
    orc_rng s;
    orc_rng_init(&s, seed, frame, ORC_FACTOR_INIT);
    for (uint64_t i = 0; i < L.gate_base; ++i)
        out[i] = (float)(sigma == 0.0 ? 0.0 : sigma * orc_rng_normal(&s));
    for (uint64_t i = L.gate_base; i < L.total; ++i) out[i] = 1.0f;
    return 0;
}

/* ---- csr.cpp:70-79: per-row sequential f64 sum ----------------------------------------- */
void orc_spmv(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
              const double* x, double* y) {
    for (uint64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (uint64_t p = ro[i]; p < ro[i + 1]; ++p) acc += v[p] * x[ci[p]];
        y[i] = acc;
    }
}

/* ---- apply.cpp:79-174 ------------------------------------------------------------------ *
 * Generated twice: T=float (the solve path) and T=double (the parity gate's reference).
 * Accumulators as in the reference helpers (apply.cpp:11-50):
 *   MV_T   (matvec_t):           y_j = sum_i M_ij x_i, accumulated in T, i ascending;
 *   MV     (matvec):             y_i = T(sum_j M_ij x_j) with a double accumulator;
 *   MV_ADD (matvec_add_double):  y_i += sum_j M_ij x_j with a double accumulator.        */
#define DEFINE_APPLY(NAME, T)                                                                \
    static void NAME##_mv_t(const T* M, uint64_t rows, uint64_t cols, const T* x, T* y) {    \
        for (uint64_t j = 0; j < cols; ++j) y[j] = (T)0;                                     \
        for (uint64_t i = 0; i < rows; ++i) {                                                \
            const T xi = x[i];                                                               \
            const T* mi = M + i * cols;                                                      \
            for (uint64_t j = 0; j < cols; ++j) y[j] += mi[j] * xi;                          \
        }                                                                                    \
    }                                                                                        \
    static void NAME##_mv(const T* M, uint64_t rows, uint64_t cols, const T* x, T* y) {      \
        for (uint64_t i = 0; i < rows; ++i) {                                                \
            double acc = 0.0;                                                                \
            const T* mi = M + i * cols;                                                      \
            for (uint64_t j = 0; j < cols; ++j) acc += (double)mi[j] * (double)x[j];         \
            y[i] = (T)acc;                                                                   \
        }                                                                                    \
    }                                                                                        \
    static void NAME##_mv_add(const T* M, uint64_t rows, uint64_t cols, const T* x,          \
                              double* y) {                                                   \
        for (uint64_t i = 0; i < rows; ++i) {                                                \
            double acc = 0.0;                                                                \
            const T* mi = M + i * cols;                                                      \
            for (uint64_t j = 0; j < cols; ++j) acc += (double)mi[j] * (double)x[j];         \
            y[i] += acc;                                                                     \
        }                                                                                    \
    }                                                                                        \
    int NAME(uint64_t n, uint64_t leaf, uint64_t ls, const T* f, int spd_enabled,            \
             double spd_raw, const double* a_diag, const double* r, double* y) {             \
        layout_t L;                                                                          \
        if (make_layout(n, leaf, ls, &L)) return -1;                                         \
        const uint64_t l = L.l, rk = L.rk, K = L.k, M = L.m;                                 \
        T* rin = malloc(n * sizeof(T));                                                      \
        T* coef = malloc(l * sizeof(T));                                                     \
        T* rrow = malloc(K * ls * sizeof(T));                                                \
        T* rcol = malloc(K * ls * sizeof(T));                                                \
        T* cast = malloc(ls * sizeof(T));                                                    \
        T* ccoef = malloc(rk * sizeof(T));                                                   \
        T* crow = malloc(M * ls * sizeof(T));                                                \
        T* ccol = malloc(M * ls * sizeof(T));                                                \
        double* srow = malloc(ls * sizeof(double));                                          \
        double* scol = malloc(ls * sizeof(double));                                          \
        double* grow = calloc(K * ls, sizeof(double));                                       \
        double* gcol = calloc(K * ls, sizeof(double));                                       \
        uint64_t* tiles = malloc(5 * M * sizeof(uint64_t));                                  \
        orc_partition(n, leaf, tiles);                                                       \
        /* (1) cast, :90 */                                                                  \
        for (uint64_t i = 0; i < n; ++i) rin[i] = (T)r[i];                                   \
        /* (2) block diagonal y_k = F_k (F_k^T r_k), :93-100 */                              \
        for (uint64_t i = 0; i < n; ++i) y[i] = 0.0;                                         \
        for (uint64_t k = 0; k < K; ++k) {                                                   \
            NAME##_mv_t(f + LEAF_F(&L, k), l, l, rin + k * l, coef);                         \
            NAME##_mv_add(f + LEAF_F(&L, k), l, l, coef, y + k * l);                         \
        }                                                                                    \
        /* (3) restriction, :102-108 */                                                      \
        for (uint64_t k = 0; k < K; ++k) {                                                   \
            NAME##_mv_t(f + BRIDGE_U(&L, k), l, ls, rin + k * l, rrow + k * ls);             \
            NAME##_mv_t(f + BRIDGE_V(&L, k), l, ls, rin + k * l, rcol + k * ls);             \
        }                                                                                    \
        /* (4) strips (double) and coarse coupling V(U^T s_r), U(V^T s_c), :110-138 */       \
        for (uint64_t t = 0; t < M; ++t) {                                                   \
            const uint64_t span = tiles[5 * t + 1], rb = tiles[5 * t + 2],                   \
                           cb = tiles[5 * t + 3];                                            \
            for (uint64_t j = 0; j < ls; ++j) srow[j] = scol[j] = 0.0;                       \
            for (uint64_t s = 0; s < span; ++s)                                              \
                for (uint64_t j = 0; j < ls; ++j) {                                          \
                    srow[j] += (double)rrow[(rb + s) * ls + j];                              \
                    scol[j] += (double)rcol[(cb + s) * ls + j];                              \
                }                                                                            \
            const T* u = f + TILE_U(&L, t);                                                  \
            const T* v = f + TILE_V(&L, t);                                                  \
            for (uint64_t j = 0; j < ls; ++j) cast[j] = (T)srow[j];                          \
            NAME##_mv_t(u, ls, rk, cast, ccoef);                                             \
            NAME##_mv(v, ls, rk, ccoef, ccol + t * ls);                                      \
            for (uint64_t j = 0; j < ls; ++j) cast[j] = (T)scol[j];                          \
            NAME##_mv_t(v, ls, rk, cast, ccoef);                                             \
            NAME##_mv(u, ls, rk, ccoef, crow + t * ls);                                      \
        }                                                                                    \
        /* (5) gather to member leaves (double), :140-154 */                                 \
        for (uint64_t t = 0; t < M; ++t) {                                                   \
            const uint64_t span = tiles[5 * t + 1], rb = tiles[5 * t + 2],                   \
                           cb = tiles[5 * t + 3];                                            \
            for (uint64_t s = 0; s < span; ++s)                                              \
                for (uint64_t j = 0; j < ls; ++j) {                                          \
                    grow[(rb + s) * ls + j] += (double)crow[t * ls + j];                     \
                    gcol[(cb + s) * ls + j] += (double)ccol[t * ls + j];                     \
                }                                                                            \
        }                                                                                    \
        /* (6) prolongation, :156-166 */                                                     \
        for (uint64_t k = 0; k < K; ++k) {                                                   \
            for (uint64_t j = 0; j < ls; ++j) cast[j] = (T)grow[k * ls + j];                 \
            NAME##_mv_add(f + BRIDGE_U(&L, k), l, ls, cast, y + k * l);                      \
            for (uint64_t j = 0; j < ls; ++j) cast[j] = (T)gcol[k * ls + j];                 \
            NAME##_mv_add(f + BRIDGE_V(&L, k), l, ls, cast, y + k * l);                      \
        }                                                                                    \
        /* (7) gated Jacobi term + optional softplus shift, :168-173, factor_tensor.hpp:64 */ \
        const T* gate = f + L.gate_base;                                                     \
        const double shift = spd_enabled ? log1p(exp(spd_raw)) : 0.0;                        \
        for (uint64_t i = 0; i < n; ++i)                                                     \
            y[i] += (double)gate[i] * r[i] / a_diag[i] + shift * r[i];                       \
        free(rin); free(coef); free(rrow); free(rcol); free(cast); free(ccoef);              \
        free(crow); free(ccol); free(srow); free(scol); free(grow); free(gcol);              \
        free(tiles);                                                                         \
        return 0;                                                                            \
    }

DEFINE_APPLY(orc_apply_f32, float)
DEFINE_APPLY(orc_apply_f64, double)

/* ---- pcg.cpp:53-126 --------------------------------------------------------------------- */
/* Sequential as the reference (pcg.cpp dot). ORC_DOT_MODE (sensitivity experiments only):
 * 1 = blocked tree (128-element sequential blocks, pairwise combine, like a GPU reduction),
 * 2 = compensated (Neumaier) — near the exact dot. */
static int dot_mode = -1;
static double dot(uint64_t n, const double* a, const double* c) {
    if (dot_mode < 0) {
        const char* e = getenv("ORC_DOT_MODE");
        dot_mode = e ? atoi(e) : 0;
    }
    if (dot_mode == 1) {
        uint64_t nb = (n + 127) / 128;
        double* part = (double*)malloc(nb * sizeof(double));
        for (uint64_t b = 0; b < nb; ++b) {
            double t = 0.0;
            for (uint64_t i = 128 * b; i < n && i < 128 * b + 128; ++i) t += a[i] * c[i];
            part[b] = t;
        }
        for (uint64_t w = 1; w < nb; w *= 2)
            for (uint64_t b = 0; b + w < nb; b += 2 * w) part[b] += part[b + w];
        double r = part[0];
        free(part);
        return r;
    }
    if (dot_mode == 2) {
        double s = 0.0, comp = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double p = a[i] * c[i];
            const double pe = fma(a[i], c[i], -p);
            const double t = s + p;
            comp += (fabs(s) >= fabs(p)) ? (s - t) + p : (p - t) + s;
            comp += pe;
            s = t;
        }
        return s + comp;
    }
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += a[i] * c[i];
    return s;
}

typedef struct {
    int kind;
    uint64_t n, leaf, ls;
    const float* packed;
    int spd_enabled;
    double spd_raw;
    const double* diag;
} applier_t;

/* pcg.cpp:28-51: identity, jacobi (r_i / A_ii), factor (apply<float>) */
static void run_applier(const applier_t* a, const double* r, double* z) {
    if (a->kind == 0)
        for (uint64_t i = 0; i < a->n; ++i) z[i] = r[i];
    else if (a->kind == 1)
        for (uint64_t i = 0; i < a->n; ++i) z[i] = r[i] / a->diag[i];
    else
        orc_apply_f32(a->n, a->leaf, a->ls, a->packed, a->spd_enabled, a->spd_raw, a->diag, r,
                      z);
}

int orc_pcg_solve(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v,
                  const double* b, int kind, uint64_t leaf, uint64_t ls, const float* packed,
                  int spd_enabled, double spd_raw, double rtol, uint64_t max_iters,
                  double* x_out, double* history_out, double* report_out) {
    if (!(rtol > 0.0)) return -1;
    /* csr.cpp:52-58 diagonal, csr.cpp:64-68 Frobenius norm */
    double* diag = calloc(n, sizeof(double));
    double fro = 0.0;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t p = ro[i]; p < ro[i + 1]; ++p)
            if (ci[p] == i) diag[i] = v[p];
    for (uint64_t p = 0; p < ro[n]; ++p) fro += v[p] * v[p];
    fro = sqrt(fro);
    if (kind == 1)
        for (uint64_t i = 0; i < n; ++i)
            if (!(diag[i] > 0.0)) { free(diag); return -1; }
    applier_t ap = {kind, n, leaf, ls, packed, spd_enabled, spd_raw, diag};

    double *x = calloc(n, 8), *r = malloc(n * 8), *z = malloc(n * 8), *p = malloc(n * 8),
           *q = malloc(n * 8);
    memcpy(r, b, n * 8);
    uint64_t iterations = 0, breakdown_iter = 0, hist = 0;
    int status = 1, converged = 0;

    const double r0 = sqrt(dot(n, r, r));
    if (r0 == 0.0) {
        status = 0; converged = 1;
    } else {
        const double breakdown_tol = 1e-12 * fro;
        run_applier(&ap, r, z);
        memcpy(p, z, n * 8);
        double rz = dot(n, r, z);
        for (uint64_t k = 1; k <= max_iters; ++k) {
            orc_spmv(n, ro, ci, v, p, q);
            const double pap = dot(n, p, q);
            const double p2 = dot(n, p, p);
            if (pap < -breakdown_tol * p2 || pap == 0.0) {
                status = 2; breakdown_iter = k; iterations = k;
                break;
            }
            const double alpha = rz / pap;
            for (uint64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
            for (uint64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
            const double rel = sqrt(dot(n, r, r)) / r0;
            if (history_out) history_out[hist] = rel;
            ++hist;
            if (rel <= rtol) { status = 0; converged = 1; iterations = k; break; }
            if (k == max_iters) { iterations = k; break; }
            run_applier(&ap, r, z);
            const double rz_next = dot(n, r, z);
            const double beta = rz_next / rz;
            rz = rz_next;
            for (uint64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
    }
    if (x_out) memcpy(x_out, x, n * 8);
    report_out[0] = (double)iterations;
    report_out[1] = converged;
    report_out[2] = status;
    report_out[3] = (double)breakdown_iter;
    report_out[4] = (double)hist;
    free(diag); free(x); free(r); free(z); free(p); free(q);
    return 0;
}

/* frame.cpp:147-152 (the rhs mean's sum) and csr.cpp:64-68 (|A|_F^2, one fused multiply-add per
 * entry as the reference's -march=native build contracts `fro += v * v`): the sequential sums the
 * GPU frame generator reproduces bit for bit. */
double orc_seq_sum(const double* x, uint64_t n, int squares) {
    double s = 0.0;
    if (squares)
        for (uint64_t i = 0; i < n; ++i) s = fma(x[i], x[i], s);
    else
        for (uint64_t i = 0; i < n; ++i) s = s + x[i];
    return s;
}
