/* hfpg — B200-native (sm_100a) solve-time hot path of the hierarchical-factor preconditioner.
 *
 * C ABI: plain pointers and sizes, no torch or C++ types. Each entry point names the
 * reference interface (path:line under /root/reference/proj) it replaces. The C++ drop-in
 * wrappers (hfp::gpu::pcg_solve, hfp::gpu::factor_applier, ...) live in hfp_gpu.hpp; the
 * Python mirror in paper_2605_13343_b200/.
 *
 * Error model (mirrors the reference's exception split):
 *   HFPG_EINVAL  <-> std::invalid_argument  (contract violations: lengths, layout, partition)
 *   HFPG_EIO     <-> std::runtime_error     (HFTC format / checksum / file errors)
 *   HFPG_ECUDA / HFPG_ENCCL                 (device / communicator failures)
 * Numerical outcomes (breakdown, max_iters) are never errors: they are reported in
 * hfpg_report, as pcg.cpp:90-112 does. hfpg_last_error() returns the message of the last
 * failing call on the calling thread.
 *
 * Threading: one handle = one device + one CUDA stream + one workspace; a handle is not
 * thread-safe, any number of handles may coexist (pcg.hpp:35, pcg.cpp:44-51).
 */
#ifndef HFPG_H
#define HFPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HFPG_ABI_VERSION 1

enum hfpg_status { HFPG_OK = 0, HFPG_EINVAL = 1, HFPG_EIO = 2, HFPG_ECUDA = 3, HFPG_ENCCL = 4 };
enum hfpg_where { HFPG_HOST = 0, HFPG_DEVICE = 1 };
/* pcg.cpp:28-51 identity_applier / jacobi_applier / factor_applier */
enum hfpg_precond { HFPG_PRECOND_IDENTITY = 0, HFPG_PRECOND_JACOBI = 1, HFPG_PRECOND_FACTOR = 2,
                     HFPG_PRECOND_IC0 = 3 };
/* How hfpg_pcg_solve runs the loop. GRAPH: one CUDA graph, a conditional WHILE node over the
 * per-stage kernels (any layout / preconditioner). PERSISTENT: one cooperative kernel for the
 * whole solve, phases separated by grid barriers (factor preconditioner, L=128, L_s=32).
 * AUTO picks PERSISTENT where it applies. */
enum hfpg_solver { HFPG_SOLVER_AUTO = 0, HFPG_SOLVER_GRAPH = 1, HFPG_SOLVER_PERSISTENT = 2 };
/* pcg.hpp:19 SolveStatus */
enum hfpg_solve_status { HFPG_CONVERGED = 0, HFPG_MAX_ITERS = 1, HFPG_BREAKDOWN = 2 };

/* partition.hpp:11-17 TileSpec */
typedef struct {
    uint64_t id, span, row_begin, col_begin, depth;
} hfpg_tile;

/* factor_tensor.hpp:18-48 FactorLayout (section bases in elements) */
typedef struct {
    uint64_t n, leaf_size, coarse_size, coupling_rank, leaf_count, tile_count;
    uint64_t leaf_base, tile_base, bridge_base, gate_base, total;
} hfpg_layout;

/* pcg.hpp:12-17 SolveConfig */
typedef struct {
    double rtol;        /* default 1e-8 */
    uint64_t max_iters; /* default 20000 */
} hfpg_solve_config;

/* pcg.hpp:21-33 SolveReport (residual_history is returned through a caller buffer) */
typedef struct {
    uint64_t n;
    uint64_t iterations;     /* first k with |r_k|/|r_0| <= rtol, or the stopping k */
    int32_t converged;
    int32_t status;          /* hfpg_solve_status */
    uint64_t breakdown_iter;
    uint64_t history_len;    /* entries of residual_history produced */
    double wall_ms;          /* device time of the solve (CUDA events around the graph) */
} hfpg_report;

/* toy_net.hpp:12-19 Config */
typedef struct {
    uint64_t d, layers, heads, gcn_layers, d_global, edge_hidden;
} hfpg_toynet_config;

/* toy_net.hpp:64-74 Trace, plus the host wall time of the call */
typedef struct {
    double max_attention_row_sum_error;
    double highway_max_deviation;
    uint64_t leaf_attention_dispatches, tile_attention_dispatches;
    double ms;           /* out: device time of the forward (CUDA events) */
    int32_t timing_only; /* in: 1 = fill only ms (no row-sum / conservation audits, which add
                            work to the forward); 0 = the full trace, as toy_net.hpp:64-74 */
} hfpg_toynet_trace;

/* frame.hpp:26-40 — the fields toynet::encode / forward consume (host pointers) */
typedef struct {
    uint64_t n, width, height;
    const uint32_t* cell_order;
    const double* rho;
    double rho_heavy;
    const uint64_t* row_offsets;
    const uint32_t* col_indices;
    const double* values;
} hfpg_frame_view;

typedef struct hfpg_handle hfpg_handle;
typedef struct hfpg_frame hfpg_frame;

const char* hfpg_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* hfpg_last_error(void);

/* ---- host-side structure (no GPU needed) ------------------------------------------------ */
/* partition.cpp:48-53 packed_width(build_partition(n, leaf), coarse) */
int hfpg_packed_width(uint64_t n, uint64_t leaf_size, uint64_t coarse_size, uint64_t* out);
/* partition.cpp:9-46 build_partition; writes min(K-1, cap) tiles, *count = K-1 */
int hfpg_build_partition(uint64_t n, uint64_t leaf_size, hfpg_tile* tiles, uint64_t cap,
                         uint64_t* count);
/* factor_tensor.cpp:7-28 make_factor_layout */
int hfpg_factor_layout(uint64_t n, uint64_t leaf_size, uint64_t coarse_size, hfpg_layout* out);
/* factor_tensor.cpp:30-39 init_factors<float>(..., sigma, RngStream(seed, frame, factor_init));
 * out has hfpg_packed_width elements. Bit-identical to the reference (multi-threaded). */
int hfpg_init_factors(uint64_t n, uint64_t leaf_size, uint64_t coarse_size, double sigma,
                      uint64_t seed, uint64_t frame, float* out);
/* checkpoint.cpp:45-85 read_checkpoint. Call with packed == NULL to get the layout first.
 * metadata (may be NULL) receives the JSON metadata object, truncated to meta_cap bytes. */
int hfpg_read_checkpoint(const char* path, hfpg_layout* layout, float* packed,
                         int32_t* spd_enabled, double* spd_raw, char* metadata,
                         uint64_t meta_cap);
/* checkpoint.cpp:17-43 write_checkpoint */
int hfpg_write_checkpoint(const char* path, uint64_t n, uint64_t leaf_size,
                          uint64_t coarse_size, const float* packed, int32_t spd_enabled,
                          double spd_raw, const char* metadata_json);

/* ---- synthetic systems (the path's input side) ------------------------------------------ */
/* frame.cpp:161-181 make_frame(n, seed, frame_index): 2D Morton-ordered 5-point Neumann
 * Laplacian, bit-identical to the reference (ordering, CSR, values, rhs). */
int hfpg_frame_2d(uint64_t n, uint64_t seed, uint64_t frame_index, hfpg_frame** out);
/* New (no reference counterpart): nx x ny x nz 7-point harmonic-mean Neumann Laplacian in 3D
 * Morton order (x -> bit 3i, y -> 3i+1, z -> 3i+2), barrier slabs drawn with frame.cpp:45-98's
 * parameter laws from RngStream(seed, frame, density); rhs = sample_rhs (frame.cpp:154-159). */
int hfpg_frame_3d(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed, uint64_t frame_index,
                  hfpg_frame** out);
int hfpg_frame_info(const hfpg_frame* f, uint64_t* n, uint64_t* nnz, uint64_t* width,
                    uint64_t* height, uint64_t* depth, double* rho_heavy);
/* Copy out (any pointer may be NULL). */
int hfpg_frame_copy(const hfpg_frame* f, uint32_t* cell_order, double* rho,
                    uint64_t* row_offsets, uint32_t* col_indices, double* values, double* b);
void hfpg_frame_free(hfpg_frame* f);

/* ---- GPU frame generator (new; framegen.cuh) ---------------------------------------------
 * make_frame (frame.cpp:161-181) / hfpg_frame_3d generated on the handle's device and loaded as
 * its system (operator, diagonal, |A|_F): no host round trip. Morton order and CSR structure
 * are bit-identical to hfpg_frame_2d/3d; floating values are bit-identical to them under
 * HFPG_FRAME_CRMATH=1 (correctly rounded log/cos) and within one ulp of the glibc draws on the
 * ~0.16% of normals glibc rounds incorrectly. The arrays stay valid until the next frame. */
typedef struct {
    uint64_t n, nnz, width, height, depth;
    double rho_heavy;
    const uint32_t* cell_order; /* device pointers */
    const double* rho;
    const uint64_t* row_offsets;
    const uint32_t* col_indices;
    const double* values;
    const double* b;
    const double* a_diag;
    float generate_ms; /* device time of the generation (events on the handle's stream) */
    double frobenius;  /* |A|_F = sqrt of the sequential fused sum of squares (csr.cpp:64-68) */
} hfpg_frame_device;
int hfpg_frame_gpu_2d(hfpg_handle* h, uint64_t n, uint64_t seed, uint64_t frame_index);
int hfpg_frame_gpu_3d(hfpg_handle* h, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed,
                      uint64_t frame_index);
int hfpg_frame_gpu_view(hfpg_handle* h, hfpg_frame_device* out);
/* The generator's sequential sums as a primitive: *out = (((0 + x0) + x1) + ...) in exactly the
 * rounding order of the one-thread loop (squares != 0: s = fma(x_i, x_i, s), csr.cpp:64-68 as the
 * host build contracts it), computed by the exact parallel emulation (framegen.cuh k_seq_sum).
 * x is a host (HFPG_HOST) or device pointer. */
int hfpg_seq_sum(hfpg_handle* h, const double* x, uint64_t n, int32_t squares, int where, double* out);
/* Copy the GPU frame to host arrays (any pointer may be NULL). */
int hfpg_frame_gpu_copy(hfpg_handle* h, uint32_t* cell_order, double* rho, uint64_t* row_offsets,
                        uint32_t* col_indices, double* values, double* b);

/* Pinned host memory for the end-to-end path (cudaMallocHost). */
int hfpg_host_alloc(uint64_t bytes, void** out);
int hfpg_host_free(void* p);

/* ---- device handle ------------------------------------------------------------------------ */
int hfpg_create(int device, hfpg_handle** out);
int hfpg_destroy(hfpg_handle* h);
/* The handle's CUDA stream (cudaStream_t), for callers timing with events. */
int hfpg_get_stream(hfpg_handle* h, void** stream);

/* System load: csr.hpp:11-16 CsrMatrix fields. Index values are preserved bit-exactly; the
 * device copy is re-laid out as SELL-32 (slices of 32 rows, column-major within a slice).
 * Computes diagonal() (csr.cpp:52-58) and frobenius_norm() (csr.cpp:64-68). */
int hfpg_load_csr(hfpg_handle* h, uint64_t n, const uint64_t* row_offsets,
                  const uint32_t* col_indices, const double* values, int where);
/* Model load: the packed factor tensor (factor_tensor.hpp:57-112) for (n, leaf, coarse),
 * `total` must equal the packed width. Host or device pointer; copied (owning, as
 * factor_applier does, pcg.cpp:46). */
int hfpg_load_factors(hfpg_handle* h, uint64_t n, uint64_t leaf_size, uint64_t coarse_size,
                      const float* packed, uint64_t total, int32_t spd_enabled, double spd_raw,
                      int where);
/* apply.hpp:41-43 takes a_diag explicitly: override diag(A) (e.g. to apply with a diagonal
 * that has no matrix, as test_apply.cpp does). Loading a CSR resets it to diag(A). */
int hfpg_set_diag(hfpg_handle* h, uint64_t n, const double* a_diag, int where);
/* Select the preconditioner used by hfpg_pcg_solve. JACOBI throws EINVAL on a nonpositive
 * diagonal entry like jacobi_applier (pcg.cpp:34-42). */
int hfpg_set_precond(hfpg_handle* h, int kind);

/* Select the solve driver (hfpg_solver); the one that will run is reported by
 * hfpg_solver_in_use. Iterates are identical up to the order of the f64 dot-product sums. */
int hfpg_set_solver(hfpg_handle* h, int kind);
int hfpg_solver_in_use(hfpg_handle* h, int32_t* out);
/* Phase trace of the persistent solver: with cap > 0, every later solve records %globaltimer
 * (ns) at its start (entry 0) and after each grid barrier e (entry e, e < cap), from CTA 0.
 * Barrier sequence: init = [leaf, sums, tiles, prolong], then per iteration [spmv, leaf, sums,
 * tiles, prolong]. cap = 0 turns tracing off. */
int hfpg_set_trace(hfpg_handle* h, uint32_t cap);
int hfpg_get_trace(hfpg_handle* h, uint64_t* out, uint32_t cap);

/* apply.cpp:79-174 apply<float>: z = M r with the loaded factors and diag(A). */
int hfpg_apply(hfpg_handle* h, const double* r, double* z, int where);
/* pcg.cpp:28-51 PrecondApplier of the handle's current kind (hfpg_set_precond): identity
 * (z = r), jacobi (z = r / a_ii, IEEE division, pcg.cpp:34-42), factor (hfpg_apply) or IC(0)
 * (hfpg_ic0_apply), on the device. */
int hfpg_precond_apply(hfpg_handle* h, const double* r, double* z, int where);
/* ---- on-disk formats (mppf.hpp / checkpoint.hpp) ----
 * zlib crc32 of `bytes` at data: HFPG_DEVICE computes it on the GPU (parallel CRC by
 * polynomial combination, bit-identical to zlib), HFPG_HOST with zlib. */
int hfpg_crc32(hfpg_handle* h, const void* data, uint64_t bytes, int where, uint32_t* out);
/* The checksum an HFTC payload / MPPF section stores (checkpoint.cpp:28-30, mppf.cpp:21-24):
 * the reference casts the byte length to zlib's uInt, so it covers the first (bytes mod 2^32)
 * bytes. Host memory. */
int hfpg_payload_crc32(const void* data, uint64_t bytes, uint32_t* out);
/* checkpoint.cpp:45-85 read_checkpoint straight into the handle's factor tensor: the payload is
 * streamed through pinned buffers into device memory and its crc32 checked on the GPU. Same
 * errors as hfpg_read_checkpoint; afterwards as hfpg_load_factors. */
int hfpg_load_checkpoint(hfpg_handle* h, const char* path);
/* A host frame from arrays (e.g. to write one): barriers as in hfpg_frame_meta; cell_order may
 * be NULL. Free with hfpg_frame_free. */
int hfpg_frame_create(uint64_t n, uint64_t width, uint64_t height, uint64_t depth, uint64_t master_seed,
                      uint64_t frame_index, double rho_heavy, uint32_t nbarriers, const double* barriers,
                      const uint32_t* cell_order, const double* rho, const uint64_t* row_offsets,
                      const uint32_t* col_indices, const double* values, const double* b, hfpg_frame** out);
/* mppf.cpp:48-100 write_mppf of a host frame (2D frames only, as MPPF v1). */
int hfpg_write_mppf(const hfpg_frame* f, const char* path);
/* mppf.cpp:102-177 read_mppf into a host frame: checksums, CSR invariants incl. symmetry
 * (std::invalid_argument -> HFPG_EINVAL), section sizes, Morton cell order. */
int hfpg_read_mppf(const char* path, hfpg_frame** out);
/* The frame's seeds and barriers (frame.hpp:34-37): barriers[4i..4i+3] = orientation, center,
 * thickness, gap for i < min(*nbarriers, cap). */
int hfpg_frame_meta(const hfpg_frame* f, uint64_t* master_seed, uint64_t* frame_index, uint32_t* nbarriers,
                    double* barriers, uint32_t cap);
/* read_mppf on the device: sections streamed into device memory through pinned buffers, every
 * checksum and the CSR invariants (symmetry included) checked on the GPU, Morton order on the GPU;
 * the frame becomes the handle's system and GPU frame (hfpg_frame_gpu_view / _copy). */
int hfpg_load_mppf(hfpg_handle* h, const char* path);

/* ---- training of the factor tensor (adjoint.hpp, loss.hpp, train.cpp) ----
 * Double-precision parameters (PackedFactors<double>, packed width of make_factor_layout(n, 128,
 * 32)); batches are kz columns, row-major n x kz; diag(A) is the loaded system's. shift = the
 * tensor's spd_shift() (0 when disabled). where = HFPG_HOST / HFPG_DEVICE for every pointer.
 * adjoint.cpp:44-127 factor_apply_batch: y = M x, every stage stashed on the handle. */
int hfpg_batch_apply(hfpg_handle* h, const double* params, uint64_t leaf, uint64_t ls, double shift,
                     const double* x, uint64_t kz, double* y, int where);
/* adjoint.cpp:129-248 factor_apply_batch_adjoint for the handle's last forward batch:
 * grad = d(loss)/d(params) for the upstream adjoint bar_y (grad is overwritten). */
int hfpg_batch_adjoint(hfpg_handle* h, const double* params, const double* bar_y, double* grad, int where);
/* adjoint.cpp:250-292 loss_gradient on the loaded system: kind 0 cosine (Y = M A Z, 1 - cos),
 * 1 sai (|(1/norm_a) A M Z - Z|_F^2). A zero image sets *degenerate and a zero gradient. */
int hfpg_loss_gradient(hfpg_handle* h, const double* params, uint64_t leaf, uint64_t ls, double shift,
                       const double* z, uint64_t kz, int32_t kind, double norm_a, double* loss,
                       int32_t* degenerate, double* grad, int where);
/* train.cpp:136-160: global clip of grad to clip_norm, then AdamW with decoupled weight decay;
 * device pointers; updates params, m1, m2 (and grad, clipped) in place. */
int hfpg_adamw_step(hfpg_handle* h, double* params, double* grad, double* m1, double* m2, uint64_t count,
                    uint64_t step, double lr, double beta1, double beta2, double eps, double weight_decay,
                    double clip_norm, double* gnorm_out);

/* probes.cpp:14-44 on the device for large batches: z (device, n * kz) = the normals of draws
 * counter0 .. of the RngStream with key `key` (rng.hpp; correctly rounded log / cos), then
 * `steps` damped-Jacobi sweeps with omega on the handle's operator. */
int hfpg_probes_device(hfpg_handle* h, uint64_t key, uint64_t counter0, uint64_t kz, double omega, uint64_t steps,
                       double* z);
/* train.hpp:12-52 — a training frame (frame.hpp fields + rhs + its frame index, which keys the
 * power-iteration and evaluation-probe streams), TrainConfig, one log entry, the run summary. */
typedef struct {
    hfpg_frame_view view;
    const double* b;
    uint64_t frame_index;
} hfpg_train_frame;
typedef struct {
    double lr, weight_decay, clip_norm;
    double plateau_factor;
    uint64_t plateau_patience;
    double plateau_rel_threshold;
    uint64_t max_steps, autostop_window;
    double probe_omega;
    uint64_t probe_smooth_steps, contexts_per_step;
    int32_t loss; /* 0 cosine, 1 sai */
    uint64_t log_every;
    double init_sigma;
    uint64_t leaf_size, coarse_size, eval_every_logs;
    double solve_rtol;
    uint64_t solve_max_iters, stop_at_iters;
} hfpg_train_config;
typedef struct {
    uint64_t step;
    double train_loss, sai_heldout;
    uint64_t pcg_iters_heldout;
    double lr, wall_s;
} hfpg_train_log;
typedef struct {
    uint64_t total_steps;
    int32_t auto_stopped, aborted_divergence, reached_target;
    uint64_t n_entries;  /* log entries produced (entries beyond log_cap are not stored) */
    uint64_t leaf_size;  /* after clamp_leaf_size (partition.hpp:48-50) */
    uint64_t packed_width;
} hfpg_train_summary;
/* train.cpp:29-217 train_factors on `device`: frames share N; eval NULL = frames[0]. Writes the
 * final float tensor (packed_width floats, may be NULL) and up to log_cap log entries. The
 * held-out PCG iterations use hfpg_pcg_solve_exact (the reference's count exactly). */
int hfpg_train_factors(const hfpg_train_frame* frames, uint64_t nframes, const hfpg_train_frame* eval,
                       const hfpg_train_config* cfg, uint64_t seed, int device, float* factors_out,
                       hfpg_train_log* log_out, uint64_t log_cap, hfpg_train_summary* summary);

/* ---- IC(0) baseline (ic0.hpp / ic0.cpp) ----
 * ic0.cpp:10-69 ic0_factorize on the host (no device needed): the lower factor L of A (pattern =
 * lower triangle of A, diagonal last; policy 0 = Ic0Shift::none, 1 = Ic0Shift::scaled, shift
 * 1e-8 max diag), bit-identical to the reference. lro: n + 1, lci / lv: cap >= nnz(A) + n
 * entries; *nnz_out = nnz(L). A nonpositive pivot is HFPG_EIO (std::runtime_error). */
int hfpg_ic0_factor_host(uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                         const double* values, int32_t policy, uint64_t* lro, uint32_t* lci, double* lv,
                         uint64_t cap, uint64_t* nnz_out, double* shift_out);
/* ic0.cpp:72 ic0_applier: loads the factor (host pointers) for hfpg_ic0_apply and for
 * hfpg_pcg_solve with HFPG_PRECOND_IC0. */
int hfpg_load_ic0(hfpg_handle* h, uint64_t n, const uint64_t* lro, const uint32_t* lci, const double* lv);
/* ic0.cpp:75-98: z = (L L^T)^{-1} r by two sync-free triangular sweeps on the device,
 * bit-identical to the reference applier. */
int hfpg_ic0_apply(hfpg_handle* h, const double* r, double* z, int where);

/* csr.cpp:70-79 spmv: y = A x. */
int hfpg_spmv(hfpg_handle* h, const double* x, double* y, int where);
/* pcg.cpp:53-126 pcg_solve, the whole loop as one CUDA graph (conditional WHILE node).
 * x (n) and history (max_iters entries, may be NULL) are written in `where` memory. */
int hfpg_pcg_solve(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg, double* x,
                   double* history, hfpg_report* report, int where);
/* pcg.cpp:53-126 pcg_solve bit for bit: the same loop driven from the host with every dot
 * product evaluated exactly as the reference's sequential loop (its pinned build: in-order sums
 * of the products, fused remainder), so x, the residual history, the iteration count and the
 * status are identical to the reference's for the loaded preconditioner (factor, IC(0), Jacobi,
 * identity). A verification mode: several host round trips per iteration. */
int hfpg_pcg_solve_exact(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg, double* x,
                         double* history, hfpg_report* report, int where);
/* pcg.cpp:56,102 residual_vectors: hfpg_pcg_solve_exact calls fn(user, k, r_k, n) after every
 * iteration's residual update (r_k in host memory, valid during the call). NULL disables. */
typedef void (*hfpg_residual_fn)(void* user, uint64_t k, const double* r, uint64_t n);
int hfpg_set_residual_callback(hfpg_handle* h, hfpg_residual_fn fn, void* user);
/* apply.cpp:80-173 apply<float> bit for bit (the pinned build's float accumulation and
 * contractions, stage by stage): the factor preconditioner of hfpg_pcg_solve_exact. */
int hfpg_apply_exact(hfpg_handle* h, const double* r, double* z, int where);

/* ---- row-partitioned solve (north star: N=16.7M over 8 GPUs) ------------------------------
 * The system is split along the bisection tree (partition.cpp:9-46): rank r of G (a power of
 * two, <= 16, >= 2 leaves per rank) owns leaves [r K/G, (r+1) K/G) and rows [r N/G, (r+1) N/G),
 * with every tile inside its subtree; the G-1 tiles above the rank subtrees are recomputed by
 * every rank from the exchanged subtree-root strip sums. Per iteration each rank sends three
 * small f64 messages to every rank (p.Ap/p.p, |r|^2 + root sums, r.z after pushing its z halo
 * rows into the peers' ghost slots) through device mailboxes over peer memory, and reduces
 * them in rank order, so all ranks take identical decisions. A partitioned handle solves with
 * hfpg_pcg_solve on its local slices (b, x: n/G entries) once connected; hfpg_apply /
 * hfpg_spmv are refused (use hfpg_group_apply). */
/* Rank `rank`'s share of the GLOBAL system (host pointers): local CSR with ghost columns,
 * halo lists, and the factor slice — sliced from `packed` (the global packed tensor) or, when
 * packed == NULL, drawn directly as init_factors(sigma, RngStream(seed, frame, factor_init))
 * would draw those elements (factor_tensor.cpp:30-39). L = 128, L_s = 32 required. */
int hfpg_part_load(hfpg_handle* h, uint32_t G, uint32_t rank, uint64_t n, const uint64_t* row_offsets,
                   const uint32_t* col_indices, const double* values, uint64_t leaf_size,
                   uint64_t coarse_size, const float* packed, double sigma, uint64_t seed,
                   uint64_t frame, int32_t spd_enabled, double spd_raw);
/* out[6] = {n_local, row_begin, n_ghost, halo rows sent, G, rank} */
int hfpg_part_info(hfpg_handle* h, uint64_t* out);
/* Device addresses peers write into (mailbox, z) — for ranks sharing a process. */
int hfpg_part_mailbox(hfpg_handle* h, void** mailbox, void** z);
/* Peer tables: G device pointers each, valid in h's context (own slot = own buffers). */
int hfpg_part_connect(hfpg_handle* h, void* const* mailboxes, void* const* zs);
/* Multi-process: 128 bytes of CUDA IPC handles (mailbox, z) to all-gather, then connect with
 * the G x 128-byte table (own entry ignored). */
int hfpg_part_ipc_get(hfpg_handle* h, void* out);
int hfpg_part_ipc_connect(hfpg_handle* h, const void* all);
/* All G ranks in this process on one device (e.g. to check a partitioning on one GPU): one
 * graph over every rank, b / x / r / z are GLOBAL host vectors. */
int hfpg_group_pcg_solve(hfpg_handle* const* hs, uint32_t G, const double* b,
                         const hfpg_solve_config* cfg, double* x, double* history,
                         hfpg_report* report);
int hfpg_group_apply(hfpg_handle* const* hs, uint32_t G, const double* r, double* z);
/* Host-only: the partition plan (no GPU). counts[4] = {n_local, n_ghost, halo rows sent,
 * local nnz}; any array may be NULL (ghost_cols: n_ghost, send_rows/send_slot: halo rows,
 * send_off: G+1, local_cols: local nnz). */
int hfpg_part_plan(uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                   const double* values, uint64_t leaf_size, uint32_t G, uint32_t rank,
                   uint64_t* counts, uint32_t* ghost_cols, uint32_t* send_rows, uint32_t* send_slot,
                   uint64_t* send_off, uint32_t* local_cols);
/* Host-only: rank's factor slice (local packed tensor of size n/G + (G-1) x L_s^2 top tiles),
 * sliced from `packed` or drawn from (sigma, seed, frame) when packed == NULL. */
int hfpg_part_factors(uint64_t n, uint64_t leaf_size, uint64_t coarse_size, uint32_t G, uint32_t rank,
                      const float* packed, double sigma, uint64_t seed, uint64_t frame,
                      float* local, float* top);

/* Asynchronous form of hfpg_pcg_solve: enqueue on the handle's stream and return; wait for it
 * (and fill history / report) with hfpg_pcg_solve_wait. Lets independent systems on separate
 * handles run concurrently on one GPU (the batched-frames configuration). With HFPG_HOST
 * buffers the copies are only asynchronous for pinned memory (hfpg_host_alloc). */
int hfpg_pcg_solve_async(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg, double* x,
                         int where);
int hfpg_pcg_solve_wait(hfpg_handle* h, double* history, hfpg_report* report, int where);

/* ---- network inference + factor assembly ------------------------------------------------ */
/* toy_net.cpp:170-223 init_weights(cfg, make_factor_layout(build_partition(n, leaf), coarse),
 * weight_seed) and :322-586 forward(frame, ...) on the GPU (tcgen05 tf32 GEMMs + fp32 kernels;
 * d = 128, head dim 16). Writes the packed factor tensor to `out` (host, packed-width floats;
 * may be NULL); if `load` != 0 it also becomes the handle's factor tensor (no host round trip),
 * ready for hfpg_apply / hfpg_pcg_solve. */
int hfpg_toynet_forward(hfpg_handle* h, const hfpg_frame_view* frame, uint64_t leaf_size,
                        uint64_t coarse_size, const hfpg_toynet_config* cfg, uint64_t weight_seed,
                        float* out, int32_t load, hfpg_toynet_trace* trace);
/* The same forward from the handle's GPU frame (hfpg_frame_gpu_2d): inputs stay on the device,
 * the global statistics (toy_net.cpp:232-268) are reduced on the device. With load, the factors
 * go straight into the handle: generate -> infer -> solve without a host round trip. */
int hfpg_toynet_forward_gpu_frame(hfpg_handle* h, uint64_t leaf_size, uint64_t coarse_size,
                                  const hfpg_toynet_config* cfg, uint64_t weight_seed, float* out,
                                  int32_t load, hfpg_toynet_trace* trace);

/* ---- introspection for tests / bench ---------------------------------------------------- */
/* Number of kernels one PCG iteration launches, and one apply. */
int hfpg_launch_counts(hfpg_handle* h, uint32_t* per_iteration, uint32_t* per_apply);
/* Per-kernel device time of one factor-preconditioned PCG iteration, measured with CUDA events
 * between standalone launches of the iteration's kernels on the handle's stream (state left by
 * the last solve; alpha = beta = 0 so the traffic is a real iteration's but x, r stay fixed).
 * ms_out[4] = {spmv, leaf, coarse, prolong}, averaged over `reps`. */
int hfpg_profile_iteration(hfpg_handle* h, uint32_t reps, float* ms_out);
/* C = A (M x K) * Bt^T (Bt: N x K), fp32 in/out, through the inference path's tcgen05 kind::tf32
 * GEMM (host pointers; test hook). */
int hfpg_gemm_tf32(uint64_t M, uint64_t N, uint64_t K, const float* A, const float* Bt, float* C);
/* 1 if the fast sm_100a TMA path (L=128, L_s=32) is selected for the loaded layout. */
int hfpg_fast_path(hfpg_handle* h, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* HFPG_H */
