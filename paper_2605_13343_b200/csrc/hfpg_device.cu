// Device handle, CUDA-graph PCG driver and the device half of the C ABI (include/hfpg.h).
#include <atomic>

#include "internal.hpp"
#include "kernels.cuh"
#include "solve_persistent.cuh"
#include "partition_host.hpp"
#include "framegen.cuh"
#include "ic0.cuh"
#include "crc32.cuh"
#include "io_device.cuh"
#include "train.cuh"
#include "pcg_exact.cuh"

#include <algorithm>
#include <cstdio>
#include <memory>
#include <zlib.h>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace hfpg {

static thread_local std::string g_last_error;
void set_error(const std::string& m) { g_last_error = m; }

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

template <class T>
static void dfree(T*& p) {
    if (p) cudaFree(const_cast<void*>(static_cast<const void*>(p)));
    p = nullptr;
}
// Runs its callable when the scope ends, on every exit path.
template <class F>
struct ScopeExit {
    F f;
    ~ScopeExit() { f(); }
};
template <class F>
ScopeExit<F> on_scope_exit(F f) {
    return ScopeExit<F>{f};
}
template <class T>
static void dalloc(T*& p, size_t count) {
    dfree(p);
    if (count == 0) count = 1;
    CK(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T)));
}


// Scratch of one exact sequential sum (per-tile approximate sums, guesses, summaries).
struct SeqScratch {
    double* tsum = nullptr;
    int* guess = nullptr;
    SeqTile* tiles = nullptr;
    uint64_t cap = 0;
    void reserve(uint64_t tiles_max) {
        if (tiles_max <= cap && tsum) return;
        dalloc(tsum, tiles_max);
        dalloc(guess, tiles_max);
        dalloc(tiles, tiles_max);
        cap = tiles_max;
    }
    void release() {
        dfree(tsum);
        dfree(guess);
        dfree(tiles);
        cap = 0;
    }
};

}  // namespace hfpg

using namespace hfpg;

struct hfpg_handle {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t lstream = nullptr;  // stream the launch_* helpers use (a group capture redirects it)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // file -> device streaming (HFTC / MPPF loaders): two pinned staging buffers + their events
    unsigned char* pin[2] = {nullptr, nullptr};
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    uint32_t* crc_scratch = nullptr;
    uint64_t crc_cap = 0;
    // training batch state (train.cuh): stashes for (n, kz), params / grad / bar_y staging
    struct Train {
        uint64_t n = 0, kz = 0;
        std::vector<double*> bufs;
        TrainDev T{};
        double *P = nullptr, *G = nullptr, *BY = nullptr, *Z = nullptr, *part = nullptr;
        uint64_t pcap = 0;
        bool have_fwd = false;
    } tr;

    // factors
    bool have_factors = false;
    Layout L;
    float* F = nullptr;
    int spd_enabled = 0;
    hfpg_residual_fn res_fn = nullptr;  // pcg.cpp:102 residual_vectors (exact loop only)
    void* res_user = nullptr;
    double spd_raw = 0.0;
    bool fast = false;

    // operator
    bool have_csr = false;
    uint64_t n = 0;  // system size (CSR, else factors)
    double fro = 0.0;
    bool diag_positive = false;
    // IC(0) preconditioner (hfpg_load_ic0): lower factor, its transpose, sweep state
    struct Ic0 {
        bool have = false;
        uint64_t n = 0;
        unsigned long long *lro = nullptr, *tro = nullptr;
        uint32_t *lci = nullptr, *tci = nullptr;
        double *lv = nullptr, *tv = nullptr, *y = nullptr;
        uint32_t *fperm = nullptr, *bperm = nullptr;
        uint32_t flevels = 0, blevels = 0;
        uint16_t *flev = nullptr, *blev = nullptr, *fmax = nullptr, *bmax = nullptr;
    } ic0;
    unsigned long long* slice_off = nullptr;
    uint32_t* sell_cols = nullptr;
    double* sell_vals = nullptr;
    double* a_diag = nullptr;
    bool have_diag = false;
    uint32_t spmv_stage_bytes = 0;  // >0: slices streamed by k_spmv_tma
    uint32_t pspmv_stage_bytes = 0; // >0: k_solve streams 16-slice chunks through a TMA ring

    // vectors / workspace (sized for vec_n / ws layout)
    uint64_t vec_n = 0;
    double *x = nullptr, *r = nullptr, *z = nullptr, *ap = nullptr, *p0 = nullptr, *p1 = nullptr,
           *y_loc = nullptr, *b = nullptr, *scratch = nullptr;
    Layout ws_layout;
    bool have_ws = false;
    float *restrict_ = nullptr, *coupled = nullptr;
    double *node_u = nullptr, *node_v = nullptr;
    unsigned* tree_counters = nullptr;
    double* partials = nullptr;
    double* dpart = nullptr;  // deferred-reduction partials (kPartLen)
    uint64_t partials_cap = 0;
    unsigned* counters = nullptr;
    Scalars* sc = nullptr;
    double* history = nullptr;
    uint64_t history_cap = 0;

    int precond = HFPG_PRECOND_FACTOR;
    int solver = HFPG_SOLVER_AUTO;
    Scalars* sc_host = nullptr;  // pinned copy of the solve's scalars (async solves)
    bool pending = false;
    unsigned* gbar = nullptr;  // grid-barrier counter of k_solve
    unsigned long long* trace = nullptr;  // k_solve barrier timestamps (hfpg_set_trace)
    unsigned trace_cap = 0;
    int l2_bytes = 0;

    // graph
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool graph_valid = false;

    DevSys sys{};
    ToynetModel* toynet = nullptr;
    // exact-mode apply<float> scratch (apply_exact_f32's stage arrays), grown once, reused
    float* exbuf = nullptr;
    uint64_t exbuf_cap = 0;
    // probe smoothing scratch (hfpg_probes_device): A z of one batch
    double* probe_tmp = nullptr;
    uint64_t probe_cap = 0;

    // row partition (G > 1): this handle holds rank `rank`'s share of a system
    struct Part {
        uint32_t G = 1, rank = 0, glog = 0;
        uint64_t n_ghost = 0, row0 = 0, n_global = 0, halo_send = 0;
        float* top_tiles = nullptr;
        float* top_coupled = nullptr;
        Mailbox* mbox = nullptr;
        Mailbox** peer_mbox = nullptr;  // device array of G
        double** peer_z = nullptr;      // device array of G
        uint32_t *send_rows = nullptr, *send_slot = nullptr;
        unsigned long long* send_off = nullptr;
        unsigned long long* seq = nullptr;
        bool connected = false;
        std::vector<void*> ipc_opened;
    } part;
    uint64_t vec_ng = 0;  // ghost entries the z/p vectors were sized for

    // operator storage capacities (a GPU frame per step reuses them)
    uint64_t sell_cap = 0, slice_cap = 0, diag_cap = 0;

    // GPU-generated frame (framegen.cuh), resident and loaded as the system
    struct FrameDev {
        bool valid = false;
        FgParams P{};
        uint64_t nnz = 0, cap_cells = 0, cap_n = 0, cap_nnz = 0;
        uint32_t *order = nullptr, *rank_of = nullptr, *len = nullptr, *ci = nullptr, *slice_len = nullptr;
        double *rho = nullptr, *b = nullptr, *vals = nullptr, *sums = nullptr;
        unsigned long long *ro = nullptr, *tot = nullptr, *tail = nullptr;  // tail: nnz, nonpos, maxch8, maxch16
        unsigned long long* tail_host = nullptr;
        cudaStream_t side[2] = {nullptr, nullptr};
        cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
        float gen_ms = 0.f;
        SeqScratch seq[2];  // the two sequential sums' scratch
    } fr;
};

namespace {

void set_device(hfpg_handle* h) { CK(cudaSetDevice(h->device)); }

void invalidate_graph(hfpg_handle* h) {
    if (h->exec) cudaGraphExecDestroy(h->exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    h->exec = nullptr;
    h->graph = nullptr;
    h->graph_valid = false;
}

// Kernel launch with programmatic stream serialisation (PDL, see pdl_enter in device_common.cuh)
// for the fast path's solve kernels when HFPG_PDL=1. Off by default: measured (r02, 3D 1M, same
// box, A/B twice) 222.7 ms per solve with PDL vs 220.9 ms without — the graph's kernel-to-kernel
// gaps are not launch-bound. `coop` adds the cooperative attribute (k_coarse_coop).
bool pdl_on() {
    static const bool v = std::getenv("HFPG_PDL") && std::getenv("HFPG_PDL")[0] == '1';
    return v;
}
template <class... KArgs, class... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool coop,
              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned na = 0;
    if (pdl_on()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

uint64_t leaf_grid(const hfpg_handle* h) {
    return h->fast ? std::min<uint64_t>(h->L.k, uint64_t(h->num_sms)) : h->L.k;
}
// k_prolong_tma is the fast path's prolongation; HFPG_PROLONG_WARP=1 selects the register-
// staged k_prolong_fast (A/B), which also serves apply calls whose vectors are not 16-byte
// aligned (cp.async.bulk needs 16-byte aligned sources).
bool prolong_tma_on() {
    static const bool v = std::getenv("HFPG_PROLONG_WARP") == nullptr;
    return v;
}
bool prolong_tma(const hfpg_handle* h, const double* rin, const double* zout) {
    return h->fast && prolong_tma_on() && (reinterpret_cast<uintptr_t>(rin) & 15u) == 0 &&
           (reinterpret_cast<uintptr_t>(zout) & 15u) == 0;
}
uint64_t prolong_grid(const hfpg_handle* h, bool tma = true) {
    if (!h->fast) return h->L.k;
    if (tma && prolong_tma_on()) return std::min<uint64_t>(h->L.k, uint64_t(h->num_sms));
    return std::min<uint64_t>((h->L.k + kProlWarps - 1) / kProlWarps, uint64_t(h->num_sms) * 2);
}
void launch_prolong(hfpg_handle* h, const DevSys& s, cudaStream_t st, int mode, const double* rin, double* zout) {
    if (prolong_tma(h, rin, zout))
        launch_k(k_prolong_tma, dim3(unsigned(prolong_grid(h))), dim3(kPtThreads), sizeof(ProlSmem), st, false, s,
                 mode, rin, zout);
    else
        k_prolong_fast<<<unsigned(prolong_grid(h, false)), 256, 0, st>>>(s, mode, rin, zout);
}
uint32_t spmv_stages() {
    static const uint32_t v = [] {
        const char* e = std::getenv("HFPG_SPMV_STAGES");
        const int n = e ? std::atoi(e) : kSpmvStages;
        return uint32_t(n >= 2 && n <= 8 ? n : kSpmvStages);
    }();
    return v;
}
size_t spmv_smem(const hfpg_handle* h) {
    return h->spmv_stage_bytes ? 128 + size_t(h->spmv_stage_bytes + kSpmvHdr) * spmv_stages() : 0;
}
uint64_t spmv_grid(const hfpg_handle* h) {
    if (h->spmv_stage_bytes) {
        const uint64_t per_sm = std::max<uint64_t>(1, (227 * 1024) / (spmv_smem(h) + 1024));
        const uint64_t nch = ((h->n + 31) / 32 + 7) / 8;
        return std::max<uint64_t>(1, std::min<uint64_t>(nch, uint64_t(h->num_sms) * std::min<uint64_t>(per_sm, 4)));
    }
    return std::max<uint64_t>(1, std::min<uint64_t>((h->n + 255) / 256, uint64_t(h->num_sms) * 4));
}
template <int MODE>
void launch_spmv(hfpg_handle* h, const DevSys& s, const double* x, double* y) {
    if (h->spmv_stage_bytes)
        launch_k(k_spmv_tma<MODE>, dim3(unsigned(spmv_grid(h))), dim3(kSpmvThreads), spmv_smem(h), h->lstream, false,
                 s, x, y);
    else
        k_spmv<MODE><<<unsigned(spmv_grid(h)), 256, 0, h->lstream>>>(s, x, y);
}
uint64_t simple_grid(const hfpg_handle* h) {
    return std::max<uint64_t>(1, std::min<uint64_t>((h->n + 255) / 256, uint64_t(h->num_sms) * 8));
}

// (Re)allocate the per-n vectors and the per-layout apply workspace.
void ensure_workspace(hfpg_handle* h) {
    const uint64_t n = h->n;
    if (h->vec_n != n || h->vec_ng != h->part.n_ghost) {
        invalidate_graph(h);
        const uint64_t ng = h->part.n_ghost;  // peers' rows read by this rank's SpMV
        dalloc(h->x, n);
        dalloc(h->r, n);
        dalloc(h->z, n + ng);
        dalloc(h->ap, n);
        dalloc(h->p0, n + ng);
        dalloc(h->p1, n + ng);
        h->vec_ng = ng;
        if (ng) {
            CK(cudaMemset(h->z, 0, (n + ng) * 8));
            CK(cudaMemset(h->p1, 0, (n + ng) * 8));
        }
        dalloc(h->y_loc, n);
        dalloc(h->b, n);
        dalloc(h->scratch, n);
        h->vec_n = n;
    }
    if (h->have_factors &&
        (!h->have_ws || h->ws_layout.n != h->L.n || h->ws_layout.l != h->L.l ||
         h->ws_layout.ls != h->L.ls)) {
        invalidate_graph(h);
        const Layout& L = h->L;
        dalloc(h->restrict_, L.k * 2 * L.ls);
        dalloc(h->coupled, L.m * 2 * L.ls);
        dalloc(h->node_u, 2 * L.k * L.ls);
        dalloc(h->node_v, 2 * L.k * L.ls);
        dalloc(h->tree_counters, 2 * L.k);
        CK(cudaMemsetAsync(h->tree_counters, 0, 2 * L.k * sizeof(unsigned), h->stream));
        h->ws_layout = L;
        h->have_ws = true;
    }
    const uint64_t need = 2 * std::max<uint64_t>({(n + 255) / 256, h->have_factors ? 2 * h->L.k : 1,
                                                   uint64_t(h->num_sms) * 8});
    if (h->partials_cap < need) {
        invalidate_graph(h);
        dalloc(h->partials, need);
        h->partials_cap = need;
    }
    if (!h->dpart) {
        dalloc(h->dpart, kPartLen);
        CK(cudaMemsetAsync(h->dpart, 0, kPartLen * sizeof(double), h->stream));
    }
    if (!h->counters) {
        dalloc(h->counters, 16);  // [0..3] grid reductions, [4..11] k_leaf_coarse tickets
        CK(cudaMemsetAsync(h->counters, 0, 16 * sizeof(unsigned), h->stream));
    }
    if (!h->gbar) dalloc(h->gbar, 1);
    if (!h->sc) {
        dalloc(h->sc, 1);
        CK(cudaMemsetAsync(h->sc, 0, sizeof(Scalars), h->stream));
    }
}

// Subtree width of k_coarse: 32 leaves when the staged tiles fit, else fewer.
uint64_t coarse_width(const Layout& L) {
    uint64_t S = 32;
    while (S > 2 && coarse_smem_bytes(L.ls, S) > 200 * 1024) S /= 2;
    return S;
}
size_t coarse_smem(const Layout& L) { return coarse_smem_bytes(L.ls, coarse_width(L)); }

void fill_sys(hfpg_handle* h) {
    DevSys& s = h->sys;
    s = DevSys{};
    const Layout& L = h->L;
    s.F = h->F;
    s.n = h->n;
    s.l = L.l;
    s.ls = L.ls;
    s.rk = L.rk;
    s.K = L.k;
    s.D = L.depth;
    s.tile_base = L.tile_base;
    s.bridge_base = L.bridge_base;
    s.gate_base = L.gate_base;
    s.a_diag = h->a_diag;
    s.slice_off = h->slice_off;
    s.sell_cols = h->sell_cols;
    s.sell_vals = h->sell_vals;
    s.x = h->x;
    s.r = h->r;
    s.z = h->z;
    s.ap = h->ap;
    s.p0 = h->p0;
    s.p1 = h->p1;
    s.y_loc = h->y_loc;
    s.restrict_ = h->restrict_;
    s.coupled = h->coupled;
    s.node_u = h->node_u;
    s.node_v = h->node_v;
    s.tree_counters = h->tree_counters;
    s.coarse_S = coarse_width(L);
    s.spmv_stage_bytes = h->spmv_stage_bytes;
    s.pspmv_stage_bytes = h->pspmv_stage_bytes;
    s.spmv_stages = spmv_stages();
    s.partials = h->partials;
    s.counters = h->counters;
    s.dpart = h->dpart;
    s.grid_spmv = uint32_t(spmv_grid(h));
    s.grid_leaf = uint32_t(leaf_grid(h));
    s.grid_prol = uint32_t(prolong_grid(h));
    // deferred reductions on the single-rank factor fast path (HFPG_NO_DEFER=1: last-CTA tails)
    s.defer = h->part.G == 1 && h->precond == HFPG_PRECOND_FACTOR && h->fast && h->have_factors &&
              !std::getenv("HFPG_NO_DEFER");
    // apply stages 1-4 in one kernel (leaf_coarse.cuh) with HFPG_LEAF_COARSE=1 — measured slower
    // than the staged kernels, so opt-in only
    s.fused_leaf = s.defer && std::getenv("HFPG_LEAF_COARSE") && std::getenv("HFPG_LEAF_COARSE")[0] == '1';
    s.bridge_first = std::getenv("HFPG_BRIDGE_FIRST") && std::getenv("HFPG_BRIDGE_FIRST")[0] == '1';
    s.ksolve_pipe = !(std::getenv("HFPG_KSOLVE_PIPE") && std::getenv("HFPG_KSOLVE_PIPE")[0] == '0');
    s.sc = h->sc;
    s.history = h->history;
    s.use_cond = 0;
    s.trace = h->trace;
    s.trace_cap = h->trace_cap;
    s.G = h->part.G;
    s.rank = h->part.rank;
    s.glog = h->part.glog;
    s.n_ghost = h->part.n_ghost;
    s.top_tiles = h->part.top_tiles;
    s.top_coupled = h->part.top_coupled;
    s.mbox = h->part.mbox;
    s.peer_mbox = h->part.peer_mbox;
    s.peer_z = h->part.peer_z;
    s.send_rows = h->part.send_rows;
    s.send_slot = h->part.send_slot;
    s.send_off = h->part.send_off;
    s.seq = h->part.seq;
    s.trace_probe = h->trace_cap > 64 ? 3 : 0;  // intra-phase probes in iteration 3
    // keep the factors L2-resident across iterations when they fit comfortably (65K: 53 MB)
    s.l2_resident = h->have_factors && double(h->L.total) * 4.0 < 0.6 * double(h->l2_bytes);
}


// Coarse-stage launch shapes. The tile kernel keeps its free register budget (98 registers,
// two CTAs per SM); HFPG_COARSE_MINB=4 is the 64-register variant (four CTAs per SM, spills) kept
// for A/B runs. The strip-sum sweep: up to two CTAs per SM, one 32-leaf group each.
int tiles_minb() {
    static const int v = [] {
        const char* e = std::getenv("HFPG_COARSE_MINB");
        return (e && e[0] == '4') ? 4 : 1;
    }();
    return v;
}
uint64_t sums_ctas_per_sm() { return 2; }
void launch_tiles(hfpg_handle* h, const DevSys& s, int mode, uint64_t tw) {
    const uint64_t cap = uint64_t(h->num_sms) * uint64_t(tiles_minb() == 4 ? 4 : 2);
    const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(tw, cap)));
    if (tiles_minb() == 4) k_tiles_all<4><<<g, kTilesThreads, 0, h->lstream>>>(s, mode);
    else k_tiles_all<1><<<g, kTilesThreads, 0, h->lstream>>>(s, mode);
}

// Apply stage 4: subtree kernel + (above 32 leaves) the parallel top-of-tree kernel.
// k_coarse_coop (one cooperative launch) is the single-rank fast path's coarse stage for K >= 64;
// HFPG_COARSE_SPLIT=1 selects k_sums_tree + k_tiles_all (A/B; also the partitioned path).
bool coarse_coop(const hfpg_handle* h, const DevSys& s) {
    static const bool split = std::getenv("HFPG_COARSE_SPLIT") != nullptr;
    return h->fast && !split && s.G == 1 && h->L.k >= 64 && h->L.ls == 32;
}
unsigned coarse_coop_grid(const hfpg_handle* h) {
    static const int occ = [] {
        int o = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_coarse_coop, kTilesThreads, 0));
        return o;
    }();
    if (occ < 1) throw CudaError("k_coarse_coop: no resident CTA fits an SM");
    return unsigned(h->num_sms) * unsigned(std::min(occ, 2));
}
void launch_coarse(hfpg_handle* h, const DevSys& s, int mode) {
    const Layout& L = h->L;
    if (coarse_coop(h, s)) {
        launch_k(k_coarse_coop, dim3(coarse_coop_grid(h)), dim3(kTilesThreads), 0, h->lstream, true, s, mode);
    } else if (h->fast) {
        const uint64_t R = L.k / std::min<uint64_t>(L.k, kCoarseS0);
        k_sums_tree<<<unsigned(std::min<uint64_t>(R, uint64_t(h->num_sms) * sums_ctas_per_sm())), kSumsThreads, 0, h->lstream>>>(s, mode);
        CK(cudaGetLastError());
        const uint64_t tw = (L.k - 1 + kTilesThreads / 32 - 1) / (kTilesThreads / 32);
        launch_tiles(h, s, mode, tw);
    } else {
        const uint64_t S0 = std::min<uint64_t>(L.k, coarse_width(L));
        k_coarse<<<unsigned(L.k / S0), kCoarseThreads, coarse_smem(L), h->lstream>>>(s, mode);
    }
    CK(cudaGetLastError());
}

// The apply launches (stages 1-3, 4, 5-7) in a given mode.
void launch_apply(hfpg_handle* h, int mode, const double* rin, double* zout) {
    const DevSys& s = h->sys;
    const Layout& L = h->L;
    if (h->fast && s.fused_leaf) {  // stages 1-4 in one launch
        k_leaf_coarse<<<unsigned(leaf_grid(h)), kLeafThreads, sizeof(LcSmem), h->lstream>>>(s, mode, rin);
    } else if (h->fast) {
        launch_k(k_leaf_fast, dim3(unsigned(leaf_grid(h))), dim3(kLeafThreads), sizeof(LeafSmem), h->lstream, false, s,
                 mode, rin);
    } else {
        k_leaf_generic<<<unsigned(L.k), 256, 2 * L.l * sizeof(float), h->lstream>>>(s, mode, rin);
    }
    CK(cudaGetLastError());
    if (!(h->fast && s.fused_leaf)) launch_coarse(h, s, mode);
    if (h->fast)
        launch_prolong(h, s, h->lstream, mode, rin, zout);
    else
        k_prolong_generic<<<unsigned(L.k), 256, 2 * L.ls * sizeof(float), h->lstream>>>(s, mode, rin, zout);
    CK(cudaGetLastError());
}

Ic0Dev ic0_dev(const hfpg_handle* h) {
    const auto& c = h->ic0;
    static const bool rows = std::getenv("HFPG_IC0_ROWS") != nullptr;  // A/B: per-row sweeps
    return Ic0Dev{c.lro, c.lci, c.lv, c.tro, c.tci, c.tv, c.y, c.fperm, c.bperm, c.flev, c.blev, c.fmax, c.bmax,
                  rows ? 0 : 1};
}
// The two sync-free sweeps (ic0.cuh): z = (L L^T)^{-1} rin; mode kApply leaves the scalars alone.
void launch_ic0_sweeps(hfpg_handle* h, const DevSys& s, int mode, const double* rin, double* zout) {
    const unsigned g = unsigned((h->n + kIc0Threads - 1) / kIc0Threads);
    const Ic0Dev d = ic0_dev(h);
    // the larger register budget wins while the wavefront is short next to the chunk count
    // (2D 65K / 262K: 512 / 2,048 chunks); the higher residency once chunks far outnumber the
    // slots (3D 1M: 8,192 chunks)
    if (d.chunked && g <= unsigned(h->num_sms) * kIc0MinBlocksResident * 4) {
        k_ic0_forward_chunk<kIc0MinBlocksResident><<<g, kIc0ChunkThreads, 0, h->lstream>>>(s, d, rin, mode);
        CK(cudaGetLastError());
        k_ic0_backward_chunk<kIc0MinBlocksResident><<<g, kIc0ChunkThreads, 0, h->lstream>>>(s, d, rin, zout, mode);
    } else if (d.chunked) {
        k_ic0_forward_chunk<kIc0MinBlocksWide><<<g, kIc0ChunkThreads, 0, h->lstream>>>(s, d, rin, mode);
        CK(cudaGetLastError());
        k_ic0_backward_chunk<kIc0MinBlocksWide><<<g, kIc0ChunkThreads, 0, h->lstream>>>(s, d, rin, zout, mode);
    } else {
        k_ic0_forward<<<g, kIc0Threads, 0, h->lstream>>>(s, d, rin, mode);
        CK(cudaGetLastError());
        k_ic0_backward<<<g, kIc0Threads, 0, h->lstream>>>(s, d, rin, zout, mode);
    }
    CK(cudaGetLastError());
}
void launch_ic0_step(hfpg_handle* h, const DevSys& s, int mode) {
    k_ic0_update<<<unsigned(simple_grid(h)), 256, 0, h->lstream>>>(s, ic0_dev(h), mode);
    CK(cudaGetLastError());
    launch_ic0_sweeps(h, s, mode, h->r, h->z);
}

void launch_iteration(hfpg_handle* h) {
    const DevSys& s = h->sys;
    launch_spmv<kLoop>(h, s, nullptr, nullptr);
    CK(cudaGetLastError());
    if (h->precond == HFPG_PRECOND_FACTOR) {
        launch_apply(h, kLoop, nullptr, nullptr);
    } else if (h->precond == HFPG_PRECOND_IC0) {
        launch_ic0_step(h, s, kLoop);
    } else {
        k_simple<<<unsigned(simple_grid(h)), 256, 0, h->lstream>>>(s, kLoop, h->precond == HFPG_PRECOND_JACOBI);
        CK(cudaGetLastError());
    }
}

void launch_init(hfpg_handle* h) {
    const DevSys& s = h->sys;
    k_init<<<unsigned(simple_grid(h)), 256, 0, h->lstream>>>(s, h->b);
    CK(cudaGetLastError());
    if (h->precond == HFPG_PRECOND_FACTOR) {
        launch_apply(h, kInit, nullptr, nullptr);
    } else if (h->precond == HFPG_PRECOND_IC0) {
        launch_ic0_step(h, s, kInit);
    } else {
        k_simple<<<unsigned(simple_grid(h)), 256, 0, h->lstream>>>(s, kInit, h->precond == HFPG_PRECOND_JACOBI);
        CK(cudaGetLastError());
    }
}

void configure_kernels() {
    static std::once_flag once;
    std::call_once(once, [] {
        CK(cudaFuncSetAttribute(k_leaf_fast, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(LeafSmem))));
        CK(cudaFuncSetAttribute(k_leaf_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(LcSmem))));
        CK(cudaFuncSetAttribute(k_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CK(cudaFuncSetAttribute(k_prolong_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(ProlSmem))));
        CK(cudaFuncSetAttribute(k_spmv_tma<kLoop>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
        CK(cudaFuncSetAttribute(k_spmv_tma<kApply>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
        CK(cudaFuncSetAttribute(k_leaf_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        CK(cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PSmem))));
    });
}

// One graph per handle: [k_init, precond init] -> WHILE(cond) { spmv, precond iteration }.
void build_graph(hfpg_handle* h) {
    invalidate_graph(h);
    fill_sys(h);
    CK(cudaGraphCreate(&h->graph, 0));
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, h->graph, 1, cudaGraphCondAssignDefault));
    h->sys.cond = cond;
    h->sys.use_cond = 1;

    CK(cudaStreamBeginCaptureToGraph(h->stream, h->graph, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    launch_init(h);
    CK(cudaStreamEndCapture(h->stream, &h->graph));

    size_t nn = 0;
    CK(cudaGraphGetNodes(h->graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(h->graph, nodes.data(), &nn));
    cudaGraphNode_t sink = nullptr;
    for (auto nd : nodes) {
        size_t nout = 0;
        CK(cudaGraphNodeGetDependentNodes(nd, nullptr, &nout));
        if (nout == 0) sink = nd;
    }
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, h->graph, &sink, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    launch_iteration(h);
    CK(cudaStreamEndCapture(h->stream, &body));
    CK(cudaGraphInstantiate(&h->exec, h->graph, 0));
    h->graph_valid = true;
}

// The persistent whole-solve kernel serves the factor preconditioner on the fast layout.
constexpr uint64_t kPersistentMaxLeaves = 1024;  // N <= 131072 at L = 128
bool use_persistent(const hfpg_handle* h) {
    int solver = h->solver;
    if (solver == HFPG_SOLVER_AUTO) {  // HFPG_SOLVER=graph|persistent overrides AUTO (experiments)
        const char* e = std::getenv("HFPG_SOLVER");
        if (e && std::strcmp(e, "graph") == 0) solver = HFPG_SOLVER_GRAPH;
        if (e && std::strcmp(e, "persistent") == 0) solver = HFPG_SOLVER_PERSISTENT;
    }
    if (solver == HFPG_SOLVER_GRAPH) return false;
    const bool ok = h->fast && h->precond == HFPG_PRECOND_FACTOR && h->part.G == 1;
    // AUTO: the persistent kernel wins where a solve is latency-bound (measured: 65K leaves it
    // 5% ahead); for HBM-bound systems the per-stage kernels keep their own register budgets
    if (solver == HFPG_SOLVER_AUTO && ok && h->L.k > kPersistentMaxLeaves) return false;
    if (solver == HFPG_SOLVER_PERSISTENT && !ok && h->solver == HFPG_SOLVER_PERSISTENT)
        throw InvalidArgument("persistent solver needs the factor preconditioner on L=128, L_s=32");
    return ok;
}

void launch_persistent(hfpg_handle* h) {
    fill_sys(h);
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, kPThreads, sizeof(PSmem)));
    if (per_sm < 1) throw CudaError("k_solve does not fit on an SM");
    const unsigned grid = unsigned(h->num_sms);
    CK(cudaMemsetAsync(h->gbar, 0, sizeof(unsigned), h->stream));
    const double* bptr = h->b;
    unsigned* gb = h->gbar;
    void* args[] = {&h->sys, &bptr, &gb};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_solve), dim3(grid), dim3(kPThreads), args,
                                   sizeof(PSmem), h->stream));
}

void require_apply_ready(hfpg_handle* h) {
    if (!h->have_factors) throw InvalidArgument("apply: no factor tensor loaded");
    if (!h->have_diag) throw InvalidArgument("apply: no diagonal (load a CSR or set_diag)");
    if (h->n != h->L.n) throw InvalidArgument("apply: length mismatch");
}

// Copy `count` doubles between caller memory (`where`) and device memory.
void copy_in(hfpg_handle* h, double* dst, const double* src, uint64_t count, int where) {
    CK(cudaMemcpyAsync(dst, src, count * 8, where == HFPG_HOST ? cudaMemcpyHostToDevice
                                                                  : cudaMemcpyDeviceToDevice,
                       h->stream));
}
void copy_out(hfpg_handle* h, double* dst, const double* src, uint64_t count, int where) {
    CK(cudaMemcpyAsync(dst, src, count * 8, where == HFPG_HOST ? cudaMemcpyDeviceToHost
                                                                  : cudaMemcpyDeviceToDevice,
                       h->stream));
}

// Device copy of a (local) CSR with n rows: diagonal, |A|_F (fro < 0: computed here, else the
// global value of a partitioned system), SELL-32 layout. Columns are < n + n_ghost.
void upload_csr(hfpg_handle* h, uint64_t n, const std::vector<uint64_t>& ro,
                const std::vector<uint32_t>& ci, const std::vector<double>& vv, double fro_in) {
        // csr.cpp:52-58 diagonal, csr.cpp:64-68 Frobenius norm (sequential, as the reference)
    std::vector<double> diag(n, 0.0);
    double fro = 0.0;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t p = ro[i]; p < ro[i + 1]; ++p)
            if (ci[p] == i) diag[i] = vv[p];
    for (double v : vv) fro += v * v;
    h->fro = fro_in < 0.0 ? std::sqrt(fro) : fro_in;
    h->diag_positive = std::all_of(diag.begin(), diag.end(), [](double d) { return d > 0.0; });
    // SELL-32: slice s holds rows 32s..32s+31, width = longest row, column-major inside;
    // padding = (own row, 0.0) so padded FMAs add exactly +0.
    const uint64_t ns = (n + 31) / 32;
    std::vector<unsigned long long> off(ns + 1, 0);
    for (uint64_t s = 0; s < ns; ++s) {
        uint64_t w = 0;
        for (uint64_t r = 32 * s; r < std::min(n, 32 * s + 32); ++r) w = std::max(w, ro[r + 1] - ro[r]);
        off[s + 1] = off[s] + 32 * w;
    }
    std::vector<uint32_t> sc(off[ns]);
    std::vector<double> sv(off[ns]);
    for (uint64_t s = 0; s < ns; ++s) {
        const uint64_t w = (off[s + 1] - off[s]) / 32;
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const uint64_t r = 32 * s + lane;
            for (uint64_t j = 0; j < w; ++j) {
                const uint64_t idx = off[s] + j * 32 + lane;
                if (r < n && j < ro[r + 1] - ro[r]) {
                    sc[idx] = ci[ro[r] + j];
                    sv[idx] = vv[ro[r] + j];
                } else {
                    sc[idx] = uint32_t(std::min(r, n - 1));
                    sv[idx] = 0.0;
                }
            }
        }
    }
    if (h->n != n) {
        h->n = n;
    }
    // k_spmv_tma stage capacity: the largest 8-slice chunk, if three stages leave room for
    // at least two CTAs per SM
    uint64_t maxch = 0;
    for (uint64_t s0 = 0; s0 < ns; s0 += 8)
        maxch = std::max<uint64_t>(maxch, (off[std::min(ns, s0 + 8)] - off[s0]) * 12);
    maxch = (maxch + 1023) & ~uint64_t(1023);
    h->spmv_stage_bytes = (maxch > 0 && (maxch + kSpmvHdr) * spmv_stages() + 128 <= 110 * 1024) ? uint32_t(maxch) : 0;
    if (std::getenv("HFPG_NO_SPMV_TMA")) h->spmv_stage_bytes = 0;
    // k_solve's ring: two stages of 16-slice chunks inside a free 96 KB leaf stage
    uint64_t maxch16 = 0;
    for (uint64_t s0 = 0; s0 < ns; s0 += kPSpmvSlices)
        maxch16 = std::max<uint64_t>(maxch16, (off[std::min<uint64_t>(ns, s0 + kPSpmvSlices)] - off[s0]) * 12);
    maxch16 = (maxch16 + 127) & ~uint64_t(127);
    h->pspmv_stage_bytes = (maxch16 > 0 && 2 * maxch16 <= sizeof(PStage)) ? uint32_t(maxch16) : 0;
    if (std::getenv("HFPG_NO_SPMV_TMA")) h->pspmv_stage_bytes = 0;
    invalidate_graph(h);
    dalloc(h->slice_off, ns + 1);
    dalloc(h->sell_cols, sc.size());
    dalloc(h->sell_vals, sv.size());
    dalloc(h->a_diag, n);
    h->sell_cap = sc.size();
    h->slice_cap = ns + 1;
    h->diag_cap = n;
    CK(cudaMemcpy(h->slice_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->sell_cols, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->sell_vals, sv.data(), sv.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->a_diag, diag.data(), n * 8, cudaMemcpyHostToDevice));
    h->have_csr = true;
    h->have_diag = true;
    ensure_workspace(h);
}



// ---- row partition (G > 1) ---------------------------------------------------------------
void reset_partition(hfpg_handle* h) {
    auto& P = h->part;
    for (void* q : P.ipc_opened) cudaIpcCloseMemHandle(q);
    P.ipc_opened.clear();
    dfree(P.top_tiles); dfree(P.top_coupled); dfree(P.mbox); dfree(P.peer_mbox); dfree(P.peer_z);
    dfree(P.send_rows); dfree(P.send_slot); dfree(P.send_off); dfree(P.seq);
    P = hfpg_handle::Part{};
    invalidate_graph(h);
}

void require_part_ready(hfpg_handle* h) {
    if (h->part.G > 1 && !h->part.connected)
        throw InvalidArgument("partition: rank not connected to its peers (hfpg_part_connect)");
}

// The apply's stages for stage-ordered multi-rank launches (one stream, rank after rank).
void stage_leaf(hfpg_handle* h, int mode, const double* rin) {
    k_leaf_fast<<<unsigned(leaf_grid(h)), kLeafThreads, sizeof(LeafSmem), h->lstream>>>(h->sys, mode, rin);
    CK(cudaGetLastError());
}
void stage_prolong(hfpg_handle* h, int mode, const double* rin, double* zout) {
    launch_prolong(h, h->sys, h->lstream, mode, rin, zout);
    CK(cudaGetLastError());
}
void stage_sums(hfpg_handle* h, int mode) {
    const uint64_t R = h->L.k / std::min<uint64_t>(h->L.k, kCoarseS0);
    k_sums_tree<<<unsigned(std::min<uint64_t>(R, uint64_t(h->num_sms) * sums_ctas_per_sm())), kSumsThreads, 0, h->lstream>>>(h->sys, mode);
    CK(cudaGetLastError());
}
void stage_tiles(hfpg_handle* h, int mode) {
    const uint64_t tw = (h->L.k - 1 + kTilesThreads / 32 - 1) / (kTilesThreads / 32);
    launch_tiles(h, h->sys, mode, tw);
    CK(cudaGetLastError());
}

// Per-solve state words (the loop-invariant part of Scalars).
Scalars solve_scalars(const hfpg_handle* h, const hfpg_solve_config& cfg) {
    Scalars init{};
    init.rtol = cfg.rtol;
    init.max_iters = cfg.max_iters;
    init.breakdown_tol = 1e-12 * h->fro;  // pcg.cpp:80
    init.shift = (h->precond == HFPG_PRECOND_FACTOR && h->spd_enabled) ? std::log1p(std::exp(h->spd_raw)) : 0.0;
    init.status = 1;
    return init;
}

void check_group(hfpg_handle* const* hs, uint32_t G) {
    if (G < 2 || G > kMaxRanks) throw InvalidArgument("group: rank count must be in [2, 16]");
    for (uint32_t r = 0; r < G; ++r) {
        hfpg_handle* h = hs[r];
        if (!h || h->part.G != G || h->part.rank != r)
            throw InvalidArgument("group: handle " + std::to_string(r) + " is not rank " + std::to_string(r) + " of " + std::to_string(G));
        if (h->device != hs[0]->device) throw InvalidArgument("group: all ranks must share a device");
        require_part_ready(h);
        require_apply_ready(h);
        if (!h->fast) throw InvalidArgument("group: fast layout (L=128, L_s=32) required");
    }
}

unsigned fg_blocks(const hfpg_handle* h, uint64_t items) {
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((items + 255) / 256, uint64_t(h->num_sms) * 16)));
}

// u32 counts -> u64 exclusive offsets, out[n] = total (three passes, framegen.cuh).
void scan_counts(hfpg_handle* h, cudaStream_t st, const uint32_t* in, uint64_t n, unsigned long long* out) {
    auto& F = h->fr;
    const uint64_t tiles = std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
    k_scan_tiles<<<unsigned(tiles), kScanThreads, 0, st>>>(in, n, out, F.tot);
    k_scan_totals<<<1, kScanThreads, 0, st>>>(F.tot, tiles, out + n);
    k_scan_add<<<unsigned(tiles), kScanThreads, 0, st>>>(out, n, F.tot);
    CK(cudaGetLastError());
}

// One of the reference's sequential sums on `st` (cnt elements, or *cnt_dev when given, at most
// cnt_max): the exact parallel emulation (framegen.cuh), HFPG_FG_SERIAL=1 the literal one-thread
// loop, HFPG_FG_NOSUMM=1 the emulation without tile summaries (A/B checks).
void seq_sum(cudaStream_t st, const double* src, uint64_t cnt, const unsigned long long* cnt_dev,
             uint64_t cnt_max, bool squares, double* out, SeqScratch& sc) {
    static std::atomic<uint64_t> attr_set{0};  // one bit per device (function attributes are per device)
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const uint64_t bit = 1ULL << (dev & 63);
    if (!(attr_set.load() & bit)) {
        CK(cudaFuncSetAttribute(k_seq_sum<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSeqSmem)));
        CK(cudaFuncSetAttribute(k_seq_sum<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSeqSmem)));
        attr_set.fetch_or(bit);
    }
    if (std::getenv("HFPG_FG_SERIAL")) {
        k_fg_chain<<<1, kFgChainThreads, 0, st>>>(src, cnt, cnt_dev, squares ? 1 : 0, out);
        CK(cudaGetLastError());
        return;
    }
    const uint64_t tiles_max = std::max<uint64_t>(1, (cnt_max + kSeqW - 1) / kSeqW);
    const bool summ = std::getenv("HFPG_FG_NOSUMM") == nullptr;
    if (summ) {
        sc.reserve(tiles_max);
        const unsigned g = unsigned(tiles_max);
        if (squares) k_seq_tsum<true><<<g, kSeqSumThreads, 0, st>>>(src, cnt, cnt_dev, sc.tsum);
        else k_seq_tsum<false><<<g, kSeqSumThreads, 0, st>>>(src, cnt, cnt_dev, sc.tsum);
        k_seq_guess<<<1, 1024, 0, st>>>(sc.tsum, tiles_max, cnt, cnt_dev, sc.guess);
        if (squares) k_seq_summ<true><<<g, kSeqSumThreads, 0, st>>>(src, cnt, cnt_dev, sc.guess, sc.tiles);
        else k_seq_summ<false><<<g, kSeqSumThreads, 0, st>>>(src, cnt, cnt_dev, sc.guess, sc.tiles);
    }
    const SeqTile* tl = summ ? sc.tiles : nullptr;
    if (squares) k_seq_sum<true><<<1, kSeqThreads, kSeqSmem, st>>>(src, cnt, cnt_dev, tl, out);
    else k_seq_sum<false><<<1, kSeqThreads, kSeqSmem, st>>>(src, cnt, cnt_dev, tl, out);
    CK(cudaGetLastError());
}

// make_frame / frame_3d on the GPU, loaded as the handle's system (framegen.cuh).
void frame_gpu(hfpg_handle* h, const FrameParams& FP) {
    set_device(h);
    if (h->part.G > 1) reset_partition(h);
    auto& F = h->fr;
    FgParams P{};
    P.dims = FP.dims;
    P.nb = int(FP.bars.size());
    P.n = FP.n;
    P.W = FP.W;
    P.H = FP.H;
    P.D = FP.D;
    P.rho_heavy = FP.rho_heavy;
    P.density_key = FP.density_key;
    P.c0 = FP.c0;
    P.rhs_key = FP.rhs_key;
    for (int k = 0; k < P.nb; ++k)
        P.bars[k] = {int(FP.bars[k].axis), int(FP.bars[k].gap), FP.bars[k].center, FP.bars[k].thickness};
    const uint64_t big = std::max(P.W, std::max(P.H, P.D));
    P.levels = 0;
    while ((1ULL << P.levels) < big) ++P.levels;
    const uint64_t n = P.n, cells = P.W * P.H * P.D, ns = (n + 31) / 32;
    const uint64_t nnz_max = n * uint64_t(1 + 2 * P.dims), sell_max = ns * 32 * uint64_t(1 + 2 * P.dims);

    if (!F.side[0]) {
        for (auto& st : F.side) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        for (auto& e : F.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaMallocHost(reinterpret_cast<void**>(&F.tail_host), 8 * sizeof(unsigned long long)));
        dalloc(F.sums, 2);
        dalloc(F.tail, 8);
    }
    // per-frame arrays: every per-row array is sized n + 1, every per-entry array nnz_max
    if (cells > F.cap_cells || !F.rank_of) {
        dalloc(F.rank_of, cells);
        F.cap_cells = cells;
    }
    if (n + 1 > F.cap_n || !F.order) {
        for (uint32_t** p : {&F.order, &F.len, &F.slice_len}) dalloc(*p, n + 1);
        for (double** p : {&F.rho, &F.b}) dalloc(*p, n + 1);
        for (unsigned long long** p : {&F.ro, &F.tot}) dalloc(*p, n + 1);
        F.cap_n = n + 1;
    }
    if (nnz_max > F.cap_nnz || !F.ci) {
        dalloc(F.ci, nnz_max);
        dalloc(F.vals, nnz_max);
        F.cap_nnz = nnz_max;
    }
    F.valid = false;

    // the handle's operator arrays: reuse when large enough (pointers stay put -> graph stays valid)
    const bool realloc_op = sell_max > h->sell_cap || ns + 1 > h->slice_cap || n > h->diag_cap ||
                            !h->sell_cols || !h->slice_off || !h->a_diag;
    if (realloc_op) {
        invalidate_graph(h);
        dalloc(h->sell_cols, sell_max);
        dalloc(h->sell_vals, sell_max);
        dalloc(h->slice_off, ns + 1);
        dalloc(h->a_diag, n);
        h->sell_cap = sell_max;
        h->slice_cap = ns + 1;
        h->diag_cap = n;
    }

    cudaStream_t st = h->stream;
    cudaEvent_t t0 = h->ev0, t1 = h->ev1;
    CK(cudaEventRecord(t0, st));
    CK(cudaMemsetAsync(F.tail, 0, 8 * sizeof(unsigned long long), st));
    k_fg_rank<<<fg_blocks(h, cells), 256, 0, st>>>(P, F.order, F.rank_of);
    k_fg_cells<<<fg_blocks(h, n), 256, 0, st>>>(P, F.order, F.rank_of, F.rho, F.len, F.b);
    CK(cudaGetLastError());
    // sum of b on side stream 0 (overlaps assembly and SELL), then b -= mean
    CK(cudaEventRecord(F.ev[0], st));
    CK(cudaStreamWaitEvent(F.side[0], F.ev[0], 0));
    seq_sum(F.side[0], F.b, n, nullptr, n, false, F.sums, F.seq[0]);
    k_fg_center<<<fg_blocks(h, n), 256, 0, F.side[0]>>>(F.b, n, F.sums);
    CK(cudaGetLastError());
    scan_counts(h, st, F.len, n, F.ro);
    k_fg_assemble<<<fg_blocks(h, n), 256, 0, st>>>(P, F.order, F.rank_of, F.rho, F.ro, F.ci, F.vals,
                                                   h->a_diag, reinterpret_cast<unsigned*>(F.tail + 1));
    CK(cudaGetLastError());
    // sum of v^2 on side stream 1
    CK(cudaEventRecord(F.ev[1], st));
    CK(cudaStreamWaitEvent(F.side[1], F.ev[1], 0));
    seq_sum(F.side[1], F.vals, 0, F.ro + n, nnz_max, true, F.sums + 1, F.seq[1]);
    CK(cudaGetLastError());
    // SELL-32
    k_sell_widths<<<unsigned((ns + 7) / 8), 256, 0, st>>>(F.len, n, ns, F.slice_len);
    scan_counts(h, st, F.slice_len, ns, h->slice_off);
    k_sell_fill<<<unsigned((ns + 7) / 8), 256, 0, st>>>(F.ro, F.ci, F.vals, n, ns, h->slice_off,
                                                         h->sell_cols, h->sell_vals);
    k_sell_chunks<<<unsigned((ns + 8 * 256 - 1) / (8 * 256)), 256, 0, st>>>(h->slice_off, ns, F.tail + 2);
    CK(cudaGetLastError());
    CK(cudaEventRecord(F.ev[0], F.side[0]));
    CK(cudaEventRecord(F.ev[1], F.side[1]));
    CK(cudaStreamWaitEvent(st, F.ev[0], 0));
    CK(cudaStreamWaitEvent(st, F.ev[1], 0));
    CK(cudaMemcpyAsync(F.tail, F.ro + n, 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(F.tail + 4, F.sums, 16, cudaMemcpyDeviceToDevice, st));
    CK(cudaEventRecord(t1, st));
    CK(cudaMemcpyAsync(F.tail_host, F.tail, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaEventElapsedTime(&F.gen_ms, t0, t1));

    const unsigned long long* T = F.tail_host;
    F.nnz = T[0];
    double sums[2];
    std::memcpy(sums, T + 4, 16);
    F.P = P;
    F.valid = true;

    // the state upload_csr leaves (csr.cpp:52-68; stage sizes as upload_csr computes them)
    h->fro = std::sqrt(sums[1]);
    h->diag_positive = (T[1] & 0xFFFFFFFFULL) == 0;
    uint64_t maxch = (T[2] + 1023) & ~uint64_t(1023);
    const uint32_t sb = (maxch > 0 && (maxch + kSpmvHdr) * spmv_stages() + 128 <= 110 * 1024) ? uint32_t(maxch) : 0;
    const uint64_t maxch16 = (T[3] + 127) & ~uint64_t(127);
    const uint32_t psb = (maxch16 > 0 && 2 * maxch16 <= sizeof(PStage)) ? uint32_t(maxch16) : 0;
    const bool no_tma = std::getenv("HFPG_NO_SPMV_TMA") != nullptr;
    const uint32_t sb2 = no_tma ? 0 : sb, psb2 = no_tma ? 0 : psb;
    if (h->n != n || sb2 != h->spmv_stage_bytes || psb2 != h->pspmv_stage_bytes) invalidate_graph(h);
    h->spmv_stage_bytes = sb2;
    h->pspmv_stage_bytes = psb2;
    h->n = n;
    h->have_csr = true;
    h->have_diag = true;
    ensure_workspace(h);
}

// ---- file -> device ------------------------------------------------------
constexpr uint64_t kPinBytes = 32ull << 20;
// Copy `bytes` of the open file starting at `off` into device memory `dst`: 32 MB pieces through
// two pinned buffers, the read of one piece overlapping the H2D copy of the other.
void stream_to_device(hfpg_handle* h, std::FILE* fp, uint64_t off, uint64_t bytes, void* dst, const char* what) {
    for (int q = 0; q < 2; ++q)
        if (!h->pin[q]) {
            CK(cudaMallocHost(reinterpret_cast<void**>(&h->pin[q]), kPinBytes));
            CK(cudaEventCreateWithFlags(&h->pin_ev[q], cudaEventDisableTiming));
            CK(cudaEventRecord(h->pin_ev[q], h->stream));
        }
    if (std::fseek(fp, long(off), SEEK_SET) != 0) throw IoError(std::string(what) + ": seek failed");
    unsigned char* d = static_cast<unsigned char*>(dst);
    for (uint64_t done = 0, k = 0; done < bytes; ++k) {
        const int q = int(k & 1);
        const uint64_t piece = std::min<uint64_t>(kPinBytes, bytes - done);
        CK(cudaEventSynchronize(h->pin_ev[q]));  // this buffer's previous copy has landed
        if (std::fread(h->pin[q], 1, piece, fp) != piece) throw IoError(std::string(what) + ": truncated payload");
        CK(cudaMemcpyAsync(d + done, h->pin[q], piece, cudaMemcpyHostToDevice, h->stream));
        CK(cudaEventRecord(h->pin_ev[q], h->stream));
        done += piece;
    }
}
// zlib crc32 of device memory, on the handle's stream (crc32.cuh); synchronous.
uint32_t device_crc(hfpg_handle* h, const void* d, uint64_t bytes) {
    const uint64_t need = crc_scratch_words(bytes);
    if (h->crc_cap < need) {
        dalloc(h->crc_scratch, need);
        h->crc_cap = need;
    }
    crc32_device(d, bytes, h->crc_scratch, h->stream);
    CK(cudaGetLastError());
    uint32_t out = 0;
    CK(cudaMemcpyAsync(&out, h->crc_scratch, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return out;
}
struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};

// mppf.cpp:102-177 read_mppf on the device: sections streamed into the handle's GPU-frame arrays,
// every checksum computed on the GPU, the CSR validated on the GPU with the reference's rules,
// Morton order by k_fg_rank, then the operator state upload_csr leaves (SELL-32, diagonal,
// exact |A|_F) — the frame is the handle's system, as after hfpg_frame_gpu_2d.
void frame_from_mppf(hfpg_handle* h, const char* path) {
    set_device(h);
    if (h->part.G > 1) reset_partition(h);
    const MppfHeader m = mppf_read_header(path);
    uint64_t nnz = 0, got = 0;
    for (const MppfSection& sc : m.sections) {
        if (sc.name == "col_indices") nnz = sc.bytes / 4;
        got |= sc.name == "rho" ? 1 : sc.name == "row_offsets" ? 2 : sc.name == "col_indices" ? 4 : sc.name == "values" ? 8 : 16;
    }
    if (got != 31) throw IoError(std::string("read_mppf: missing section in ") + path);
    const uint64_t n = m.n;
    if (n < 1 || m.width * m.height < n || m.width >= (1u << 16) || m.height >= (1u << 16))
        throw InvalidArgument("morton_cell_order: grid does not hold n cells");
    auto& F = h->fr;
    FgParams P{};
    P.dims = 2;
    P.nb = int(std::min<size_t>(m.bars.size(), 3));
    for (int k = 0; k < P.nb; ++k) P.bars[k] = {int(m.bars[k].axis), int(m.bars[k].gap), m.bars[k].center, m.bars[k].thickness};
    P.n = n;
    P.W = m.width;
    P.H = m.height;
    P.D = 1;
    P.rho_heavy = m.rho_heavy;
    const uint64_t big = std::max(P.W, P.H);
    P.levels = 0;
    while ((1ULL << P.levels) < big) ++P.levels;
    const uint64_t cells = P.W * P.H, ns = (n + 31) / 32;
    if (!F.side[0]) {
        for (auto& st : F.side) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        for (auto& e : F.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaMallocHost(reinterpret_cast<void**>(&F.tail_host), 8 * sizeof(unsigned long long)));
        dalloc(F.sums, 2);
        dalloc(F.tail, 8);
    }
    if (cells > F.cap_cells || !F.rank_of) {
        dalloc(F.rank_of, cells);
        F.cap_cells = cells;
    }
    if (n + 1 > F.cap_n || !F.order) {
        for (uint32_t** p : {&F.order, &F.len, &F.slice_len}) dalloc(*p, n + 1);
        for (double** p : {&F.rho, &F.b}) dalloc(*p, n + 1);
        for (unsigned long long** p : {&F.ro, &F.tot}) dalloc(*p, n + 1);
        F.cap_n = n + 1;
    }
    if (nnz + 1 > F.cap_nnz || !F.ci) {
        dalloc(F.ci, nnz + 1);
        dalloc(F.vals, nnz + 1);
        F.cap_nnz = nnz + 1;
    }
    F.valid = false;
    // stream the sections, then check every checksum on the device (mppf.cpp:139-141)
    std::unique_ptr<std::FILE, FileCloser> fp(std::fopen(path, "rb"));
    if (!fp) throw IoError(std::string("read_mppf: cannot open ") + path);
    struct Dst { void* p; uint64_t cap; };
    auto dst_of = [&](const std::string& nm) -> Dst {
        if (nm == "rho") return {F.rho, n * 8};
        if (nm == "row_offsets") return {F.ro, (n + 1) * 8};
        if (nm == "col_indices") return {F.ci, nnz * 4};
        if (nm == "values") return {F.vals, nnz * 8};
        return {F.b, n * 8};
    };
    for (const MppfSection& sc : m.sections) {
        const Dst d = dst_of(sc.name);
        if (sc.bytes > d.cap) {
            if (sc.name == "rho" || sc.name == "b") throw IoError("read_mppf: section sizes inconsistent with n");
            throw InvalidArgument(sc.name == "row_offsets" ? "csr: row_offsets length != n_rows+1" : "csr: nnz mismatch");
        }
        stream_to_device(h, fp.get(), m.payload_offset + sc.offset, sc.bytes, d.p, "read_mppf");
    }
    for (const MppfSection& sc : m.sections)
        if (device_crc(h, dst_of(sc.name).p, ref_crc_len(sc.bytes)) != sc.crc)
            throw IoError("read_mppf: checksum mismatch in section " + sc.name);
    // csr.cpp:9-53 in the reference's order of checks
    for (const MppfSection& sc : m.sections) {
        if (sc.name == "row_offsets" && sc.bytes != (n + 1) * 8) throw InvalidArgument("csr: row_offsets length != n_rows+1");
        if (sc.name == "values" && sc.bytes != nnz * 8) throw InvalidArgument("csr: nnz mismatch");
    }
    const bool realloc_op = ns * 32 * 8 > h->sell_cap || ns + 1 > h->slice_cap || n > h->diag_cap ||
                            !h->sell_cols || !h->slice_off || !h->a_diag;
    cudaStream_t st = h->stream;
    CK(cudaMemsetAsync(F.tail, 0, 8 * sizeof(unsigned long long), st));
    if (n > h->diag_cap || !h->a_diag) {
        invalidate_graph(h);
        dalloc(h->a_diag, n);
        h->diag_cap = n;
    }
    k_mppf_rows<<<unsigned((n + 255) / 256), 256, 0, st>>>(F.ro, F.ci, F.vals, n, nnz, F.len, h->a_diag,
                                                          reinterpret_cast<unsigned*>(F.tail + 1));
    CK(cudaGetLastError());
    unsigned err = 0;
    CK(cudaMemcpyAsync(&err, F.tail + 1, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err & kCsrFirst) throw InvalidArgument("csr: row_offsets[0] != 0");
    if (err & kCsrLast) throw InvalidArgument("csr: nnz mismatch");
    if (err & kCsrNondecreasing) throw InvalidArgument("csr: row_offsets not nondecreasing");
    if (err & kCsrColRange) throw InvalidArgument("csr: column index out of range");
    if (err & kCsrColOrder) throw InvalidArgument("csr: column indices not strictly increasing");
    if (err & kCsrSymmetric) throw InvalidArgument("csr: values not symmetric");
    // SELL-32 width per slice, then the operator arrays (sized by this frame's widest slice)
    if (realloc_op && (ns + 1 > h->slice_cap || !h->slice_off)) {
        invalidate_graph(h);
        dalloc(h->slice_off, ns + 1);
        h->slice_cap = ns + 1;
    }
    k_sell_widths<<<unsigned((ns + 7) / 8), 256, 0, st>>>(F.len, n, ns, F.slice_len);
    scan_counts(h, st, F.slice_len, ns, h->slice_off);
    unsigned long long sell_n = 0;
    CK(cudaMemcpyAsync(&sell_n, h->slice_off + ns, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (sell_n > h->sell_cap || !h->sell_cols || !h->sell_vals) {
        invalidate_graph(h);
        dalloc(h->sell_cols, std::max<uint64_t>(sell_n, 1));
        dalloc(h->sell_vals, std::max<uint64_t>(sell_n, 1));
        h->sell_cap = std::max<uint64_t>(sell_n, 1);
    }
    k_sell_fill<<<unsigned((ns + 7) / 8), 256, 0, st>>>(F.ro, F.ci, F.vals, n, ns, h->slice_off, h->sell_cols,
                                                         h->sell_vals);
    k_sell_chunks<<<unsigned((ns + 8 * 256 - 1) / (8 * 256)), 256, 0, st>>>(h->slice_off, ns, F.tail + 2);
    k_fg_rank<<<fg_blocks(h, cells), 256, 0, st>>>(P, F.order, F.rank_of);  // frame.cpp:24-41 order
    CK(cudaGetLastError());
    seq_sum(st, F.vals, nnz, nullptr, nnz, true, F.sums + 1, F.seq[1]);  // csr.cpp:64-68, exactly
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(F.tail + 4, F.sums, 16, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(F.tail_host, F.tail, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const unsigned long long* T = F.tail_host;
    double sums[2];
    std::memcpy(sums, T + 4, 16);
    F.nnz = nnz;
    F.P = P;
    F.gen_ms = 0.f;
    F.valid = true;
    h->fro = std::sqrt(sums[1]);
    std::vector<double> dg(n);
    CK(cudaMemcpy(dg.data(), h->a_diag, n * 8, cudaMemcpyDeviceToHost));
    h->diag_positive = std::all_of(dg.begin(), dg.end(), [](double d) { return d > 0.0; });
    uint64_t maxch = (T[2] + 1023) & ~uint64_t(1023);
    const uint32_t sb = (maxch > 0 && (maxch + kSpmvHdr) * spmv_stages() + 128 <= 110 * 1024) ? uint32_t(maxch) : 0;
    const uint64_t maxch16 = (T[3] + 127) & ~uint64_t(127);
    const uint32_t psb = (maxch16 > 0 && 2 * maxch16 <= sizeof(PStage)) ? uint32_t(maxch16) : 0;
    const bool no_tma = std::getenv("HFPG_NO_SPMV_TMA") != nullptr;
    const uint32_t sb2 = no_tma ? 0 : sb, psb2 = no_tma ? 0 : psb;
    if (h->n != n || sb2 != h->spmv_stage_bytes || psb2 != h->pspmv_stage_bytes) invalidate_graph(h);
    h->spmv_stage_bytes = sb2;
    h->pspmv_stage_bytes = psb2;
    h->n = n;
    h->have_csr = true;
    h->have_diag = true;
    ensure_workspace(h);
}

// ---- training (train.cuh) ---------------------------------------------------------------------
// Size the batch state for (n, kz) and the packed width; point T at the loaded system.
void train_prepare(hfpg_handle* h, uint64_t leaf, uint64_t ls, uint64_t kz, double shift) {
    if (!h->have_diag || h->n == 0) throw InvalidArgument("factor_apply_batch: no system loaded (diag(A))");
    if (leaf != 128 || ls != 32) throw InvalidArgument("factor_apply_batch: the GPU path implements L = 128, L_s = 32");
    if (kz == 0) throw InvalidArgument("factor_apply_batch: kz must be positive");
    const Layout L = make_layout(h->n, leaf, ls);
    auto& R = h->tr;
    if (R.n != h->n || R.kz != kz) {
        for (double* b : R.bufs) dfree(b);
        R.bufs.clear();
        const uint64_t nk = h->n * kz, kk = L.k * 32 * kz, mk = L.m * 32 * kz, mq = L.m * 16 * kz;
        auto mk_buf = [&](uint64_t cnt) {
            double* p = nullptr;
            dalloc(p, std::max<uint64_t>(cnt, 1));
            R.bufs.push_back(p);
            return p;
        };
        TrainDev& T = R.T;
        T.X = mk_buf(nk); T.H = mk_buf(nk); T.Y = mk_buf(nk); T.W = mk_buf(nk);
        T.Rr = mk_buf(kk); T.Rc = mk_buf(kk); T.Gr = mk_buf(kk); T.Gc = mk_buf(kk);
        T.BGr = mk_buf(kk); T.BGc = mk_buf(kk); T.BRr = mk_buf(kk); T.BRc = mk_buf(kk);
        T.Sr = mk_buf(mk); T.Sc = mk_buf(mk); T.Crow = mk_buf(mk); T.Ccol = mk_buf(mk);
        T.BCr = mk_buf(mk); T.BCc = mk_buf(mk); T.BSr = mk_buf(mk); T.BSc = mk_buf(mk);
        T.Pu = mk_buf(mq); T.Qv = mk_buf(mq); T.Bc1 = mk_buf(mq); T.Bc2 = mk_buf(mq);
        dfree(R.BY); dfree(R.Z);
        dalloc(R.BY, nk);
        dalloc(R.Z, nk);
        R.n = h->n;
        R.kz = kz;
        R.have_fwd = false;
    }
    if (R.pcap < L.total) {
        dfree(R.P); dfree(R.G);
        dalloc(R.P, L.total);
        dalloc(R.G, L.total);
        R.pcap = L.total;
    }
    if (!R.part) dalloc(R.part, 4096 * 3);
    TrainDev& T = R.T;
    T.n = h->n; T.K = L.k; T.D = L.depth; T.M = L.m; T.kz = kz;
    T.tile_base = L.tile_base; T.bridge_base = L.bridge_base; T.gate_base = L.gate_base;
    T.a_diag = h->a_diag;
    T.shift = shift;
}
const double* train_params(hfpg_handle* h, const double* params, uint64_t total, int where) {
    if (where == HFPG_DEVICE) return params;
    CK(cudaMemcpyAsync(h->tr.P, params, total * 8, cudaMemcpyHostToDevice, h->stream));
    return h->tr.P;
}
// Y = A X for a kz-wide row-major batch (csr.cpp:87-100 spmm; SELL slots in column order).
void train_spmm(hfpg_handle* h, const double* X, double* Y, uint64_t kz) {
    const unsigned long long* so = h->slice_off;
    const uint32_t* sc = h->sell_cols;
    const double* sv = h->sell_vals;
    const uint64_t n = h->n;
    each(h->stream, n * kz, [=] __device__(uint64_t t) {
        const uint64_t row = t / kz, j = t % kz, sl = row >> 5, lane = row & 31;
        const uint64_t b = so[sl], w = (so[sl + 1] - b) >> 5;
        double y = 0.0;
        for (uint64_t q = 0; q < w; ++q) {
            const uint64_t idx = b + q * 32 + lane;
            y = fma(sv[idx], X[uint64_t(sc[idx]) * kz + j], y);
        }
        Y[t] = y;
    });
}
// Deterministic sums of NV per-element functions over cnt elements: a fixed grid of 256-thread
// CTAs, each thread a fixed strided subset, a fixed shared-memory tree per CTA, then the CTAs'
// partials added in CTA order on the host — the same bits on every run.
template <int NV, class F>
__global__ void __launch_bounds__(256) k_train_sums(uint64_t cnt, F f, double* part) {
    __shared__ double red[NV][256];
    double acc[NV];
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    for (uint64_t t = uint64_t(blockIdx.x) * 256 + threadIdx.x; t < cnt; t += uint64_t(gridDim.x) * 256) {
        double e[NV];
        f(t, e);
        for (int v = 0; v < NV; ++v) acc[v] += e[v];
    }
    for (int v = 0; v < NV; ++v) red[v][threadIdx.x] = acc[v];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w)
            for (int v = 0; v < NV; ++v) red[v][threadIdx.x] += red[v][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < NV) part[blockIdx.x * NV + threadIdx.x] = red[threadIdx.x][0];
}
template <int NV, class F>
void train_sums(hfpg_handle* h, uint64_t cnt, F f, double (&out)[NV]) {
    const unsigned blocks = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((cnt + 255) / 256, 4096 / NV)));
    double* part = h->tr.part;
    k_train_sums<NV><<<blocks, 256, 0, h->stream>>>(cnt, f, part);
    CK(cudaGetLastError());
    std::vector<double> hp(size_t(blocks) * NV);
    CK(cudaMemcpyAsync(hp.data(), part, hp.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int v = 0; v < NV; ++v) {
        out[v] = 0.0;
        for (unsigned b = 0; b < blocks; ++b) out[v] += hp[size_t(b) * NV + v];
    }
}

}  // namespace

extern "C" {

const char* hfpg_version(void) { return "hfpg 0.1 (sm_100a)"; }
const char* hfpg_last_error(void) { return g_last_error.c_str(); }

int hfpg_host_alloc(uint64_t bytes, void** out) {
    return guarded([&] { CK(cudaMallocHost(out, bytes ? bytes : 1)); });
}
int hfpg_host_free(void* p) {
    return guarded([&] { CK(cudaFreeHost(p)); });
}

int hfpg_create(int device, hfpg_handle** out) {
    return guarded([&] {
        auto* h = new hfpg_handle;
        try {
            h->device = device;
            CK(cudaSetDevice(device));
            CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
            CK(cudaDeviceGetAttribute(&h->l2_bytes, cudaDevAttrL2CacheSize, device));
            int major = 0, minor = 0;
            CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
            CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
            if (major != 10 || minor != 0)
                throw CudaError("hfpg is built for sm_100a (B200); device is sm_" +
                                std::to_string(major) + std::to_string(minor));
            CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->lstream = h->stream;
            CK(cudaEventCreate(&h->ev0));
            CK(cudaEventCreate(&h->ev1));
            configure_kernels();
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int hfpg_destroy(hfpg_handle* h) {
    return guarded([&] {
        if (!h) return;
        cudaSetDevice(h->device);
        invalidate_graph(h);
        dfree(h->F); dfree(h->slice_off); dfree(h->sell_cols); dfree(h->sell_vals);
        dfree(h->a_diag); dfree(h->x); dfree(h->r); dfree(h->z); dfree(h->ap); dfree(h->p0);
        dfree(h->p1); dfree(h->y_loc); dfree(h->b); dfree(h->scratch); dfree(h->restrict_);
        dfree(h->coupled); dfree(h->node_u); dfree(h->node_v);
        dfree(h->tree_counters); dfree(h->partials); dfree(h->dpart); dfree(h->counters); dfree(h->sc);
        dfree(h->history); dfree(h->gbar); dfree(h->trace);
        dfree(h->ic0.lro); dfree(h->ic0.lci); dfree(h->ic0.lv); dfree(h->ic0.tro); dfree(h->ic0.tci);
        dfree(h->ic0.tv); dfree(h->ic0.y);
        dfree(h->ic0.fperm); dfree(h->ic0.bperm);
        dfree(h->ic0.flev); dfree(h->ic0.blev); dfree(h->ic0.fmax); dfree(h->ic0.bmax);
        if (h->sc_host) cudaFreeHost(h->sc_host);
        {
            auto& F = h->fr;
            dfree(F.order); dfree(F.rank_of); dfree(F.len); dfree(F.ci); dfree(F.slice_len);
            dfree(F.rho); dfree(F.b); dfree(F.vals); dfree(F.sums); dfree(F.ro); dfree(F.tot); dfree(F.tail);
            if (F.tail_host) cudaFreeHost(F.tail_host);
            for (auto& st : F.side) if (st) cudaStreamDestroy(st);
            for (auto& e : F.ev) if (e) cudaEventDestroy(e);
            for (auto& q : F.seq) q.release();
        }
        reset_partition(h);
        if (h->toynet) toynet_model_destroy(h->toynet);
        if (h->ev0) cudaEventDestroy(h->ev0);
        if (h->ev1) cudaEventDestroy(h->ev1);
        for (int q = 0; q < 2; ++q) {
            if (h->pin[q]) cudaFreeHost(h->pin[q]);
            if (h->pin_ev[q]) cudaEventDestroy(h->pin_ev[q]);
        }
        dfree(h->crc_scratch);
        dfree(h->exbuf);
        dfree(h->probe_tmp);
        for (double* b : h->tr.bufs) dfree(b);
        dfree(h->tr.P); dfree(h->tr.G); dfree(h->tr.BY); dfree(h->tr.Z); dfree(h->tr.part);
        if (h->stream) cudaStreamDestroy(h->stream);
        delete h;
    });
}

int hfpg_get_stream(hfpg_handle* h, void** stream) {
    return guarded([&] { *stream = h->stream; });
}

int hfpg_load_csr(hfpg_handle* h, uint64_t n, const uint64_t* ro_in, const uint32_t* ci_in,
                  const double* v_in, int where) {
    return guarded([&] {
        set_device(h);
        if (n == 0) throw InvalidArgument("csr: empty matrix");
        std::vector<uint64_t> ro(n + 1);
        std::vector<uint32_t> ci;
        std::vector<double> vv;
        if (where == HFPG_DEVICE) {
            CK(cudaMemcpy(ro.data(), ro_in, (n + 1) * 8, cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(ro.data(), ro_in, (n + 1) * 8);
        }
        // csr.cpp:9-25 structural checks that keep device reads in bounds
        if (ro[0] != 0) throw InvalidArgument("csr: row_offsets[0] != 0");
        for (uint64_t i = 0; i < n; ++i)
            if (ro[i] > ro[i + 1]) throw InvalidArgument("csr: row_offsets not nondecreasing");
        const uint64_t nnz = ro[n];
        ci.resize(nnz);
        vv.resize(nnz);
        if (where == HFPG_DEVICE) {
            CK(cudaMemcpy(ci.data(), ci_in, nnz * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(vv.data(), v_in, nnz * 8, cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(ci.data(), ci_in, nnz * 4);
            std::memcpy(vv.data(), v_in, nnz * 8);
        }
        for (uint64_t p = 0; p < nnz; ++p)
            if (ci[p] >= n) throw InvalidArgument("csr: column index out of range");
        if (h->part.G > 1) reset_partition(h);
        upload_csr(h, n, ro, ci, vv, -1.0);
    });
}

int hfpg_frame_gpu_2d(hfpg_handle* h, uint64_t n, uint64_t seed, uint64_t frame_index) {
    return guarded([&] { frame_gpu(h, frame_params_2d(n, seed, frame_index)); });
}

int hfpg_frame_gpu_3d(hfpg_handle* h, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed,
                      uint64_t frame_index) {
    return guarded([&] { frame_gpu(h, frame_params_3d(nx, ny, nz, seed, frame_index)); });
}

int hfpg_seq_sum(hfpg_handle* h, const double* x, uint64_t n, int32_t squares, int where, double* out) {
    return guarded([&] {
        set_device(h);
        double* d = nullptr;
        dalloc(d, n + 2);  // k_seq_sum may read to the next 16-byte boundary
        if (n) CK(cudaMemcpyAsync(d, x, n * 8, where == HFPG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
        double* r = nullptr;
        dalloc(r, 1);
        SeqScratch sc;
        seq_sum(h->stream, d, n, nullptr, n, squares != 0, r, sc);
        CK(cudaMemcpyAsync(out, r, 8, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        dfree(d);
        dfree(r);
        sc.release();
    });
}

int hfpg_frame_gpu_view(hfpg_handle* h, hfpg_frame_device* out) {
    return guarded([&] {
        const auto& F = h->fr;
        if (!F.valid) throw InvalidArgument("frame_gpu: no GPU frame generated on this handle");
        out->n = F.P.n;
        out->nnz = F.nnz;
        out->width = F.P.W;
        out->height = F.P.H;
        out->depth = F.P.D;
        out->rho_heavy = F.P.rho_heavy;
        out->cell_order = F.order;
        out->rho = F.rho;
        out->row_offsets = reinterpret_cast<uint64_t*>(F.ro);
        out->col_indices = F.ci;
        out->values = F.vals;
        out->b = F.b;
        out->a_diag = h->a_diag;
        out->generate_ms = F.gen_ms;
        out->frobenius = h->fro;
    });
}

int hfpg_frame_gpu_copy(hfpg_handle* h, uint32_t* cell_order, double* rho, uint64_t* row_offsets,
                        uint32_t* col_indices, double* values, double* b) {
    return guarded([&] {
        set_device(h);
        const auto& F = h->fr;
        if (!F.valid) throw InvalidArgument("frame_gpu: no GPU frame generated on this handle");
        const uint64_t n = F.P.n;
        auto d2h = [&](void* dst, const void* src, size_t bytes) {
            if (dst) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
        };
        d2h(cell_order, F.order, n * 4);
        d2h(rho, F.rho, n * 8);
        d2h(row_offsets, F.ro, (n + 1) * 8);
        d2h(col_indices, F.ci, F.nnz * 4);
        d2h(values, F.vals, F.nnz * 8);
        d2h(b, F.b, n * 8);
        CK(cudaStreamSynchronize(h->stream));
    });
}

int hfpg_set_diag(hfpg_handle* h, uint64_t n, const double* a_diag, int where) {
    return guarded([&] {
        set_device(h);
        if (h->have_csr && n != h->n) throw InvalidArgument("set_diag: length mismatch");
        if (!h->have_csr) h->n = n;
        invalidate_graph(h);
        dalloc(h->a_diag, n);
        h->diag_cap = n;
        copy_in(h, h->a_diag, a_diag, n, where);
        CK(cudaStreamSynchronize(h->stream));
        h->have_diag = true;
        ensure_workspace(h);
    });
}

int hfpg_load_factors(hfpg_handle* h, uint64_t n, uint64_t leaf, uint64_t ls, const float* packed,
                      uint64_t total, int32_t spd_enabled, double spd_raw, int where) {
    return guarded([&] {
        set_device(h);
        const Layout L = make_layout(n, leaf, ls);
        if (total != L.total) throw InvalidArgument("load_factors: packed width mismatch");
        if (h->have_csr && h->n != n) throw InvalidArgument("load_factors: length mismatch");
        invalidate_graph(h);
        if (!h->have_factors || h->L.total != L.total) dalloc(h->F, L.total);
        CK(cudaMemcpyAsync(h->F, packed, L.total * 4,
                           where == HFPG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                           h->stream));
        h->L = L;
        h->have_factors = true;
        h->spd_enabled = spd_enabled;
        h->spd_raw = spd_raw;
        h->fast = (L.l == kL && L.ls == kLs && std::getenv("HFPG_FORCE_GENERIC") == nullptr);
        if (!h->have_csr && !h->have_diag) h->n = n;
        ensure_workspace(h);
        const double shift = spd_enabled ? std::log1p(std::exp(spd_raw)) : 0.0;  // factor_tensor.hpp:64
        CK(cudaMemcpyAsync(&h->sc->shift, &shift, 8, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int hfpg_set_precond(hfpg_handle* h, int kind) {
    return guarded([&] {
        if (kind < 0 || kind > 3) throw InvalidArgument("set_precond: unknown kind");
        if (kind == HFPG_PRECOND_IC0 && (!h->ic0.have || h->ic0.n != h->n || !h->have_csr))
            throw InvalidArgument("ic0_applier: no IC(0) factor of the loaded matrix (hfpg_load_ic0)");
        if (kind == HFPG_PRECOND_JACOBI) {
            if (!h->have_csr) throw InvalidArgument("jacobi_applier: no matrix loaded");
            if (!h->diag_positive)
                throw InvalidArgument("jacobi_applier: nonpositive diagonal entry");
        }
        if (kind != h->precond) invalidate_graph(h);
        h->precond = kind;
    });
}

int hfpg_apply(hfpg_handle* h, const double* r, double* z, int where) {
    return guarded([&] {
        set_device(h);
        if (h->part.G > 1) throw InvalidArgument("apply: partitioned handle (use hfpg_group_apply)");
        require_apply_ready(h);
        ensure_workspace(h);
        fill_sys(h);
        const double* rin = r;
        double* zout = z;
        // the leaf kernel bulk-copies r slices: it needs a 16-byte aligned source
        if (where == HFPG_HOST || (reinterpret_cast<uintptr_t>(r) & 15)) {
            copy_in(h, h->scratch, r, h->n, where);
            rin = h->scratch;
        }
        if (where == HFPG_HOST) zout = h->z;
        launch_apply(h, kApply, rin, zout);
        if (where == HFPG_HOST) copy_out(h, z, h->z, h->n, HFPG_HOST);
        CK(cudaStreamSynchronize(h->stream));
    });
}

int hfpg_precond_apply(hfpg_handle* h, const double* r, double* z, int where) {
    if (h && h->precond == HFPG_PRECOND_FACTOR) return hfpg_apply(h, r, z, where);
    if (h && h->precond == HFPG_PRECOND_IC0) return hfpg_ic0_apply(h, r, z, where);
    return guarded([&] {
        set_device(h);
        if (h->part.G > 1) throw InvalidArgument("precond_apply: partitioned handle");
        if (!h->have_csr) throw InvalidArgument("precond_apply: no matrix loaded");
        ensure_workspace(h);
        const double* rin = r;
        double* zout = z;
        if (where == HFPG_HOST) {
            copy_in(h, h->scratch, r, h->n, HFPG_HOST);
            rin = h->scratch;
            zout = h->z;
        }
        k_diag_apply<<<unsigned(simple_grid(h)), 256, 0, h->stream>>>(h->n, rin, h->a_diag, zout,
                                                                      h->precond == HFPG_PRECOND_JACOBI);
        CK(cudaGetLastError());
        if (where == HFPG_HOST) copy_out(h, z, h->z, h->n, HFPG_HOST);
        CK(cudaStreamSynchronize(h->stream));
    });
}

// probes.cpp:14-44 on the device, for batches too large to draw and smooth on the host: z_i is
// the normal of draw counter0 + i of the stream `key` (rng.hpp, with correctly rounded log / cos —
// crmath.cuh; libm differs by <= 1 ulp on ~0.2% of draws), then `steps` damped-Jacobi sweeps
// z -= (omega / a_ii) (A z) with the reference build's fused update (probes.cpp:36-41).
int hfpg_probes_device(hfpg_handle* h, uint64_t key, uint64_t counter0, uint64_t kz, double omega, uint64_t steps,
                       double* z) {
    return guarded([&] {
        set_device(h);
        if (!h->have_csr) throw InvalidArgument("smooth_probes: no matrix loaded");
        if (!h->diag_positive) throw InvalidArgument("smooth_probes: nonpositive diagonal");
        const uint64_t n = h->n, nk = n * kz;
        each(h->stream, nk, [=] __device__(uint64_t i) { z[i] = crm::normal_of_cr(fg_mix64(key ^ (counter0 + i))); });
        if (steps) {
            if (h->probe_cap < nk) {
                dalloc(h->probe_tmp, nk);
                h->probe_cap = nk;
            }
            double* az = h->probe_tmp;
            const double* d = h->a_diag;
            for (uint64_t s = 0; s < steps; ++s) {
                train_spmm(h, z, az, kz);
                each(h->stream, nk, [=] __device__(uint64_t t) {
                    const uint64_t i = t / kz;
                    const double scale = omega / d[i];
                    z[t] = fma(-scale, az[t], z[t]);
                });
            }
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
    });
}

int hfpg_spmv(hfpg_handle* h, const double* x, double* y, int where) {
    return guarded([&] {
        set_device(h);
        if (h->part.G > 1) throw InvalidArgument("spmv: partitioned handle");
        if (!h->have_csr) throw InvalidArgument("spmv: no matrix loaded");
        ensure_workspace(h);
        fill_sys(h);
        const double* xin = x;
        double* yout = y;
        if (where == HFPG_HOST) {
            copy_in(h, h->scratch, x, h->n, HFPG_HOST);
            xin = h->scratch;
            yout = h->ap;
        }
        launch_spmv<kApply>(h, h->sys, xin, yout);
        CK(cudaGetLastError());
        if (where == HFPG_HOST) copy_out(h, y, h->ap, h->n, HFPG_HOST);
        CK(cudaStreamSynchronize(h->stream));
    });
}

// Enqueue a solve on the handle's stream (no host synchronisation). The scalars land in the
// handle's pinned report buffer; x (n) is copied to `where` memory.
static void solve_enqueue(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg_in, double* x, int where) {
    set_device(h);
    // the report buffer doubles as the config staging buffer: a second solve before the first
    // one's report is collected would read back that solve's scalars as its config
    if (h->pending) throw InvalidArgument("pcg_solve: a solve is in flight (hfpg_pcg_solve_wait first)");
    hfpg_solve_config cfg = cfg_in ? *cfg_in : hfpg_solve_config{1e-8, 20000};
    if (!(cfg.rtol > 0.0)) throw InvalidArgument("pcg_solve: rtol must be positive");
    if (!h->have_csr) throw InvalidArgument("pcg_solve: no matrix loaded");
    if (h->precond == HFPG_PRECOND_FACTOR) require_apply_ready(h);
    require_part_ready(h);
    ensure_workspace(h);
    const uint64_t n = h->n;
    const uint64_t hcap = std::max<uint64_t>(cfg.max_iters, 1);
    if (h->history_cap < hcap) {
        invalidate_graph(h);
        dalloc(h->history, hcap);
        h->history_cap = hcap;
    }
    if (!h->sc_host) CK(cudaMallocHost(reinterpret_cast<void**>(&h->sc_host), sizeof(Scalars)));
    const bool persistent = use_persistent(h);
    if (!persistent && !h->graph_valid) build_graph(h);
    *h->sc_host = solve_scalars(h, cfg);
    CK(cudaMemcpyAsync(h->sc, h->sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, h->stream));
    copy_in(h, h->b, b, n, where);
    CK(cudaEventRecord(h->ev0, h->stream));
    if (persistent)
        launch_persistent(h);
    else
        CK(cudaGraphLaunch(h->exec, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
    if (x) copy_out(h, x, h->x, n, where);
    h->pending = true;
}

static void solve_finish(hfpg_handle* h, double* history, hfpg_report* report, int where) {
    set_device(h);
    if (!h->pending) throw InvalidArgument("pcg_solve_wait: no solve in flight");
    h->pending = false;
    CK(cudaStreamSynchronize(h->stream));
    const Scalars out = *h->sc_host;
    if (history && out.hist_len) {
        copy_out(h, history, h->history, out.hist_len, where);
        CK(cudaStreamSynchronize(h->stream));
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (report) {
        report->n = h->n;
        report->iterations = out.iterations;
        report->converged = out.converged;
        report->status = out.status;
        report->breakdown_iter = out.breakdown_iter;
        report->history_len = out.hist_len;
        report->wall_ms = ms;
    }
}

int hfpg_pcg_solve(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg_in, double* x,
                   double* history, hfpg_report* report, int where) {
    return guarded([&] {
        solve_enqueue(h, b, cfg_in, x, where);
        solve_finish(h, history, report, where);
    });
}

int hfpg_pcg_solve_async(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg, double* x, int where) {
    return guarded([&] { solve_enqueue(h, b, cfg, x, where); });
}

int hfpg_pcg_solve_wait(hfpg_handle* h, double* history, hfpg_report* report, int where) {
    return guarded([&] { solve_finish(h, history, report, where); });
}

int hfpg_set_residual_callback(hfpg_handle* h, hfpg_residual_fn fn, void* user) {
    return guarded([&] {
        h->res_fn = fn;
        h->res_user = fn ? user : nullptr;
    });
}

// Device scratch for apply_exact_f32: one float buffer on the handle, carved into the stage
// arrays; allocated on first use and kept (apply allocates nothing per call, test_apply.cpp:262).
ExApplyWs exact_ws(hfpg_handle* h) {
    const Layout& L = h->L;
    const uint64_t n = L.n, K = L.k, M = K ? K - 1 : 0, ls = L.ls, rk = L.rk;
    const uint64_t sizes[12] = {n, n, K * ls, K * ls, M * ls, M * ls, M * rk, M * rk, M * ls, M * ls, K * ls, K * ls};
    uint64_t tot = 0;
    for (uint64_t v : sizes) tot += v + 4;
    if (h->exbuf_cap < tot) {
        dalloc(h->exbuf, tot);
        h->exbuf_cap = tot;
    }
    ExApplyWs w{};
    float** dst[12] = {&w.rin, &w.coef, &w.rr, &w.rc, &w.scr, &w.scc, &w.cc1, &w.cc2, &w.crow, &w.ccol, &w.gr, &w.gc};
    uint64_t off = 0;
    for (int i = 0; i < 12; ++i) {
        *dst[i] = h->exbuf + off;
        off += sizes[i] + 4;
    }
    return w;
}
double factor_shift(const hfpg_handle* h) {
    return h->spd_enabled ? std::log1p(std::exp(h->spd_raw)) : 0.0;  // factor_tensor.hpp:64
}

// apply<float> bit for bit (pcg_exact.cuh): z = M r.
int hfpg_apply_exact(hfpg_handle* h, const double* r, double* z, int where) {
    return guarded([&] {
        set_device(h);
        if (h->part.G > 1) throw InvalidArgument("apply: partitioned handle");
        require_apply_ready(h);
        const uint64_t n = h->n;
        ensure_workspace(h);
        double *dr = h->scratch, *dz = h->z;  // handle-owned (no allocation per call)
        const ExApplyWs ws = exact_ws(h);
        CK(cudaMemcpyAsync(dr, r, n * 8, where == HFPG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
        apply_exact_f32(h->stream, h->L, h->F, h->a_diag, factor_shift(h), dr, dz, ws);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(z, dz, n * 8, where == HFPG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

// pcg.cpp:53-126 bit for bit (pcg_exact.cuh): a host-driven loop over the solve path's SpMV and
// preconditioner kernels with every dot product as the reference's sequential loop.
int hfpg_pcg_solve_exact(hfpg_handle* h, const double* b, const hfpg_solve_config* cfg_in, double* x,
                         double* history, hfpg_report* report, int where) {
    return guarded([&] {
        set_device(h);
        if (h->part.G > 1) throw InvalidArgument("pcg_solve_exact: partitioned handle");
        if (!h->have_csr) throw InvalidArgument("pcg_solve: no matrix loaded");
        if (h->pending) throw InvalidArgument("pcg_solve_exact: a solve is in flight");
        if (h->precond == HFPG_PRECOND_FACTOR) require_apply_ready(h);
        if (h->precond == HFPG_PRECOND_IC0 && (!h->ic0.have || h->ic0.n != h->n))
            throw InvalidArgument("pcg_solve: no IC(0) factor loaded");
        const hfpg_solve_config cfg = cfg_in ? *cfg_in : hfpg_solve_config{1e-8, 20000};
        ensure_workspace(h);
        fill_sys(h);
        h->lstream = h->stream;
        cudaStream_t st = h->stream;
        const uint64_t n = h->n, n4 = n & ~uint64_t(3);
        double *dx = h->x, *dr = h->r, *dz = h->z, *dp = h->p0, *dap = h->ap, *prod = nullptr, *dsum = nullptr,
               *hsum = nullptr;
        dalloc(prod, n + 2);  // seq_sum reads to the next 16-byte boundary
        dalloc(dsum, 4);
        CK(cudaMallocHost(&hsum, 4 * sizeof(double)));
        SeqScratch sc;
        ExApplyWs ews{};
        if (h->precond == HFPG_PRECOND_FACTOR) ews = exact_ws(h);
        auto cleanup = [&] {
            dfree(prod);
            dfree(dsum);
            if (hsum) cudaFreeHost(hsum);
            sc.release();
        };
        try {
            const unsigned g = unsigned(simple_grid(h));
            // one dot into dsum[slot] (device); fused_each: the |r0|^2 site's remainder form
            auto dot = [&](const double* a, const double* c, int slot, int fused_each) {
                if (n4 >= 4) {
                    k_ex_prod<<<g, 256, 0, st>>>(a, c, n4, prod);
                    seq_sum(st, prod, n4, nullptr, n4, false, dsum + slot, sc);
                } else {
                    CK(cudaMemsetAsync(dsum + slot, 0, 8, st));
                }
                // n <= 2: the whole vector is the remainder (the vector body needs n > 2)
                k_ex_tail<<<1, 1, 0, st>>>(a, c, n, n <= 2 ? 0 : n4, fused_each, dsum + slot);
                CK(cudaGetLastError());
            };
            auto fetch = [&](int cnt) {
                CK(cudaMemcpyAsync(hsum, dsum, cnt * 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
            };
            auto precond = [&] {  // z = M r
                if (h->precond == HFPG_PRECOND_FACTOR) {
                    apply_exact_f32(st, h->L, h->F, h->a_diag, factor_shift(h), dr, dz, ews);
                } else if (h->precond == HFPG_PRECOND_IC0) {
                    k_ic0_pending<<<g, 256, 0, st>>>(ic0_dev(h), dz, n);
                    launch_ic0_sweeps(h, h->sys, kApply, dr, dz);
                } else if (h->precond == HFPG_PRECOND_JACOBI) {
                    k_ex_jacobi<<<g, 256, 0, st>>>(dr, h->a_diag, dz, n);
                } else {
                    CK(cudaMemcpyAsync(dz, dr, n * 8, cudaMemcpyDeviceToDevice, st));
                }
                CK(cudaGetLastError());
            };
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            auto ev_guard = on_scope_exit([&] {
                if (e0) cudaEventDestroy(e0);
                if (e1) cudaEventDestroy(e1);
            });
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, st));
            CK(cudaMemsetAsync(dx, 0, n * 8, st));
            copy_in(h, dr, b, n, where);
            std::vector<double> hist, rbuf;
            uint64_t iterations = 0, breakdown_iter = 0;
            int status = HFPG_MAX_ITERS, converged = 0;
            dot(dr, dr, 0, 1);
            fetch(1);
            const double r0 = std::sqrt(hsum[0]);
            if (r0 == 0.0) {
                status = HFPG_CONVERGED;
                converged = 1;
            } else {
                const double breakdown_tol = 1e-12 * h->fro;
                precond();
                CK(cudaMemcpyAsync(dp, dz, n * 8, cudaMemcpyDeviceToDevice, st));
                dot(dr, dz, 0, 0);
                fetch(1);
                double rz = hsum[0];
                if (!h->res_fn && cfg.max_iters > 0 && !std::getenv("HFPG_EXACT_HOSTLOOP")) {
                    // one captured CUDA graph per iteration, the scalar decisions on the device
                    // (ExState); the host polls the state every kBatch iterations
                    constexpr uint64_t kBatch = 8;
                    ExState* S = nullptr;
                    double* dhist = nullptr;
                    cudaGraph_t gr = nullptr;
                    cudaGraphExec_t ge = nullptr;
                    auto loop_guard = on_scope_exit([&] {  // every exit path, throws included
                        if (ge) cudaGraphExecDestroy(ge);
                        if (gr) cudaGraphDestroy(gr);
                        dfree(S);
                        dfree(dhist);
                    });
                    dalloc(S, 1);
                    dalloc(dhist, cfg.max_iters);
                    ExState hs{rz, 0.0, 0.0, r0, breakdown_tol, cfg.rtol, 1ULL, 0ULL, 0, 0};
                    CK(cudaMemcpyAsync(S, &hs, sizeof(ExState), cudaMemcpyHostToDevice, st));
                    CK(cudaStreamSynchronize(st));
                    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                    try {
                        launch_spmv<kApply>(h, h->sys, dp, dap);
                        dot(dp, dap, 0, 0);
                        dot(dp, dp, 1, 0);
                        k_exg_alpha<<<1, 1, 0, st>>>(S, dsum);
                        k_exg_xr<<<g, 256, 0, st>>>(S, dx, dr, dp, dap, n);
                        dot(dr, dr, 2, 0);
                        k_exg_rel<<<1, 1, 0, st>>>(S, dsum + 2, dhist);
                        precond();
                        dot(dr, dz, 3, 0);
                        k_exg_beta<<<1, 1, 0, st>>>(S, dsum + 3);
                        k_exg_p<<<g, 256, 0, st>>>(S, dp, dz, n);
                        CK(cudaGetLastError());
                    } catch (...) {
                        cudaStreamEndCapture(st, &gr);  // gr (if any) freed by loop_guard
                        throw;
                    }
                    CK(cudaStreamEndCapture(st, &gr));
                    CK(cudaGraphInstantiate(&ge, gr, 0));
                    uint64_t launched = 0;
                    while (launched < cfg.max_iters) {
                        const uint64_t batch = std::min<uint64_t>(kBatch, cfg.max_iters - launched);
                        for (uint64_t q = 0; q < batch; ++q) CK(cudaGraphLaunch(ge, st));
                        launched += batch;
                        CK(cudaMemcpyAsync(&hs, S, sizeof(ExState), cudaMemcpyDeviceToHost, st));
                        CK(cudaStreamSynchronize(st));
                        if (hs.stop) break;
                    }
                    uint64_t hlen = cfg.max_iters;
                    if (hs.stop == 1) {
                        status = HFPG_CONVERGED;
                        converged = 1;
                        iterations = hlen = hs.iters;
                    } else if (hs.stop == 2) {
                        status = HFPG_BREAKDOWN;
                        breakdown_iter = iterations = hs.iters;
                        hlen = hs.iters - 1;
                    } else {
                        iterations = cfg.max_iters;
                    }
                    hist.resize(hlen);
                    if (hlen) CK(cudaMemcpyAsync(hist.data(), dhist, hlen * 8, cudaMemcpyDeviceToHost, st));
                    CK(cudaStreamSynchronize(st));
                } else
                for (uint64_t k = 1; k <= cfg.max_iters; ++k) {
                    launch_spmv<kApply>(h, h->sys, dp, dap);
                    CK(cudaGetLastError());
                    dot(dp, dap, 0, 0);
                    dot(dp, dp, 1, 0);
                    fetch(2);
                    const double pap = hsum[0], p2 = hsum[1];
                    if (pap < -breakdown_tol * p2 || pap == 0.0) {
                        status = HFPG_BREAKDOWN;
                        breakdown_iter = k;
                        iterations = k;
                        break;
                    }
                    const double alpha = rz / pap;
                    k_ex_xr<<<g, 256, 0, st>>>(dx, dr, dp, dap, alpha, n);
                    dot(dr, dr, 0, 0);
                    fetch(1);
                    const double rel = std::sqrt(hsum[0]) / r0;
                    hist.push_back(rel);
                    if (h->res_fn) {  // residual_vectors->push_back(r) (pcg.cpp:102)
                        if (rbuf.size() != n) rbuf.resize(n);
                        CK(cudaMemcpyAsync(rbuf.data(), dr, n * 8, cudaMemcpyDeviceToHost, st));
                        CK(cudaStreamSynchronize(st));
                        h->res_fn(h->res_user, k, rbuf.data(), n);
                    }
                    if (rel <= cfg.rtol) {
                        status = HFPG_CONVERGED;
                        converged = 1;
                        iterations = k;
                        break;
                    }
                    if (k == cfg.max_iters) {
                        iterations = k;
                        break;
                    }
                    precond();
                    dot(dr, dz, 0, 0);
                    fetch(1);
                    const double rz_next = hsum[0];
                    const double beta = rz_next / rz;
                    rz = rz_next;
                    k_ex_p<<<g, 256, 0, st>>>(dp, dz, beta, n);
                    CK(cudaGetLastError());
                }
            }
            CK(cudaEventRecord(e1, st));
            copy_out(h, x, dx, n, where);
            if (history && !hist.empty())
                CK(cudaMemcpyAsync(history, hist.data(), hist.size() * 8,
                                   where == HFPG_HOST ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (report) {
                report->n = n;
                report->iterations = iterations;
                report->converged = converged;
                report->status = status;
                report->breakdown_iter = breakdown_iter;
                report->history_len = hist.size();
                report->wall_ms = ms;
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

int hfpg_launch_counts(hfpg_handle* h, uint32_t* per_iteration, uint32_t* per_apply) {
    return guarded([&] {
        fill_sys(h);
        const uint32_t apply = (h->have_factors && h->fast)
                                   ? (h->sys.fused_leaf ? 2 : coarse_coop(h, h->sys) ? 3 : 4)
                                   : 3;
        *per_apply = apply;
        *per_iteration = h->precond == HFPG_PRECOND_FACTOR ? apply + 1 : h->precond == HFPG_PRECOND_IC0 ? 4 : 2;
        if (use_persistent(h)) {  // one k_solve launch per solve
            *per_apply = 0;
            *per_iteration = 0;
        }
    });
}

int hfpg_set_trace(hfpg_handle* h, uint32_t cap) {
    return guarded([&] {
        set_device(h);
        dfree(h->trace);
        h->trace_cap = 0;
        if (cap) {
            dalloc(h->trace, cap);
            CK(cudaMemset(h->trace, 0, cap * sizeof(unsigned long long)));
            h->trace_cap = cap;
        }
    });
}

int hfpg_get_trace(hfpg_handle* h, uint64_t* out, uint32_t cap) {
    return guarded([&] {
        set_device(h);
        if (!h->trace) throw InvalidArgument("get_trace: tracing is off");
        CK(cudaMemcpy(out, h->trace, std::min(cap, h->trace_cap) * 8, cudaMemcpyDeviceToHost));
    });
}

int hfpg_set_solver(hfpg_handle* h, int kind) {
    return guarded([&] {
        if (kind < HFPG_SOLVER_AUTO || kind > HFPG_SOLVER_PERSISTENT)
            throw InvalidArgument("set_solver: unknown kind");
        h->solver = kind;
    });
}

int hfpg_solver_in_use(hfpg_handle* h, int32_t* out) {
    return guarded([&] { *out = use_persistent(h) ? HFPG_SOLVER_PERSISTENT : HFPG_SOLVER_GRAPH; });
}

int hfpg_profile_iteration(hfpg_handle* h, uint32_t reps, float* ms_out) {
    return guarded([&] {
        set_device(h);
        if (h->precond != HFPG_PRECOND_FACTOR || !h->have_csr) throw InvalidArgument("profile: factor solve required");
        require_apply_ready(h);
        ensure_workspace(h);
        fill_sys(h);
        // every rep enqueued before one synchronisation (a per-rep host sync let the first
        // kernel's interval absorb the host's launch latency: ~4 us per kernel at 3D 1M), the
        // first rep a warm-up
        const uint32_t R = std::max(reps, 1u) + 1;
        std::vector<cudaEvent_t> evs(5 * size_t(R));
        for (auto& e : evs) CK(cudaEventCreate(&e));
        double acc[4] = {0, 0, 0, 0};
        Scalars prof{};
        prof.rtol = 0.0;
        prof.max_iters = ~0ULL >> 1;
        prof.rz = 1.0;
        prof.r0 = 1.0;
        prof.k = 1;
        prof.breakdown_tol = 1e-12 * h->fro;
        prof.shift = h->spd_enabled ? std::log1p(std::exp(h->spd_raw)) : 0.0;
        const Layout& L = h->L;
        const uint64_t S0 = std::min<uint64_t>(L.k, coarse_width(L));
        for (uint32_t rep = 0; rep < R; ++rep) {
            cudaEvent_t* ev = evs.data() + 5 * size_t(rep);
            CK(cudaMemcpyAsync(h->sc, &prof, sizeof(Scalars), cudaMemcpyHostToDevice, h->stream));
            CK(cudaEventRecord(ev[0], h->stream));
            launch_spmv<kLoop>(h, h->sys, nullptr, nullptr);
            CK(cudaEventRecord(ev[1], h->stream));
            if (h->fast && h->sys.fused_leaf)  // leaf + coarse in one kernel: "coarse" reads 0
                k_leaf_coarse<<<unsigned(leaf_grid(h)), kLeafThreads, sizeof(LcSmem), h->stream>>>(h->sys, kLoop, nullptr);
            else if (h->fast)
                k_leaf_fast<<<unsigned(leaf_grid(h)), kLeafThreads, sizeof(LeafSmem), h->stream>>>(h->sys, kLoop, nullptr);
            else
                k_leaf_generic<<<unsigned(L.k), 256, 2 * L.l * sizeof(float), h->stream>>>(h->sys, kLoop, nullptr);
            CK(cudaEventRecord(ev[2], h->stream));
            if (!(h->fast && h->sys.fused_leaf)) launch_coarse(h, h->sys, kLoop);
            CK(cudaEventRecord(ev[3], h->stream));
            if (h->fast)
                launch_prolong(h, h->sys, h->stream, kLoop, nullptr, nullptr);
            else
                k_prolong_generic<<<unsigned(L.k), 256, 2 * L.ls * sizeof(float), h->stream>>>(h->sys, kLoop, nullptr, nullptr);
            CK(cudaEventRecord(ev[4], h->stream));
            CK(cudaGetLastError());
        }
        CK(cudaEventSynchronize(evs.back()));
        for (uint32_t rep = 1; rep < R; ++rep)
            for (int i = 0; i < 4; ++i) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, evs[5 * size_t(rep) + i], evs[5 * size_t(rep) + i + 1]));
                acc[i] += ms;
            }
        for (int i = 0; i < 4; ++i) ms_out[i] = float(acc[i] / (R - 1));
        for (auto& e : evs) cudaEventDestroy(e);
    });
}

}  // extern "C"

namespace {
// toynet forward of an n-node frame into a fresh buffer (out != NULL: copied to the host) or,
// with load, straight into the handle's factor tensor. `run(dst)` launches the forward.
template <class Run>
void toynet_into(hfpg_handle* h, uint64_t n, uint64_t leaf, uint64_t ls, const hfpg_toynet_config& cfg,
                 uint64_t seed, float* out, int32_t load, Run&& run) {
    set_device(h);
    const Layout L = make_layout(n, leaf, ls);
    float* dst = nullptr;
    if (load) {
        if (h->have_csr && h->n != n) throw InvalidArgument("toynet: length mismatch");
        invalidate_graph(h);
        if (!h->have_factors || h->L.total != L.total) dalloc(h->F, L.total);
        dst = h->F;
    } else {
        CK(cudaMalloc(&dst, L.total * 4));
    }
    CK(cudaMemsetAsync(dst, 0, L.total * 4, h->stream));
    try {
        if (!toynet_model_matches(h->toynet, cfg, leaf, ls, seed)) {
            if (h->toynet) toynet_model_destroy(h->toynet);
            h->toynet = nullptr;
            h->toynet = toynet_model_create(cfg, leaf, ls, seed);
        }
        run(dst);
        if (out) CK(cudaMemcpy(out, dst, L.total * 4, cudaMemcpyDeviceToHost));
    } catch (...) {
        if (!load) cudaFree(dst);
        throw;
    }
    if (!load) {
        CK(cudaFree(dst));
        return;
    }
    h->L = L;
    h->have_factors = true;
    h->spd_enabled = 0;
    h->spd_raw = 0.0;
    h->fast = (L.l == kL && L.ls == kLs && std::getenv("HFPG_FORCE_GENERIC") == nullptr);
    if (!h->have_csr && !h->have_diag) h->n = n;
    ensure_workspace(h);
    const double shift = 0.0;
    CK(cudaMemcpyAsync(&h->sc->shift, &shift, 8, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
}
}  // namespace

extern "C" {

int hfpg_toynet_forward(hfpg_handle* h, const hfpg_frame_view* frame, uint64_t leaf, uint64_t ls,
                        const hfpg_toynet_config* cfg, uint64_t seed, float* out, int32_t load,
                        hfpg_toynet_trace* trace) {
    return guarded([&] {
        if (!frame || !cfg) throw InvalidArgument("toynet: null frame or config");
        toynet_into(h, frame->n, leaf, ls, *cfg, seed, out, load,
                    [&](float* dst) { toynet_forward_device(h->toynet, h->stream, *frame, dst, trace); });
    });
}

int hfpg_toynet_forward_gpu_frame(hfpg_handle* h, uint64_t leaf, uint64_t ls, const hfpg_toynet_config* cfg,
                                  uint64_t seed, float* out, int32_t load, hfpg_toynet_trace* trace) {
    return guarded([&] {
        if (!cfg) throw InvalidArgument("toynet: null config");
        const auto& F = h->fr;
        if (!F.valid) throw InvalidArgument("toynet: no GPU frame generated on this handle");
        if (F.P.dims != 2) throw InvalidArgument("toynet: 2D frames only (frame.hpp)");
        const ToynetDeviceFrame df{F.P.n, F.P.W, F.P.H, F.nnz, F.P.rho_heavy, F.order, F.rho, F.ro, F.ci, F.vals, h->a_diag};
        toynet_into(h, F.P.n, leaf, ls, *cfg, seed, out, load,
                    [&](float* dst) { toynet_forward_device_frame(h->toynet, h->stream, df, dst, trace); });
    });
}

int hfpg_fast_path(hfpg_handle* h, int32_t* out) {
    return guarded([&] { *out = h->have_factors && h->fast ? 1 : 0; });
}


// ---- row partition ------------------------------------------------------------------------
int hfpg_part_load(hfpg_handle* h, uint32_t G, uint32_t rank, uint64_t n, const uint64_t* ro,
                   const uint32_t* ci, const double* v, uint64_t leaf, uint64_t ls,
                   const float* packed, double sigma, uint64_t seed, uint64_t frame,
                   int32_t spd_enabled, double spd_raw) {
    return guarded([&] {
        set_device(h);
        if (leaf != uint64_t(kL) || ls != uint64_t(kLs))
            throw InvalidArgument("partition: fast layout (L=128, L_s=32) required");
        PartPlan P = plan_partition(n, ro, ci, v, leaf, G, rank);
        reset_partition(h);
        auto& S = h->part;
        S.G = G;
        S.rank = rank;
        S.glog = uint32_t(P.glog);
        S.n_ghost = P.ghost_cols.size();
        S.row0 = P.row0;
        S.n_global = n;
        S.halo_send = P.send_rows.size();
        h->have_factors = false;
        h->n = 0;
        upload_csr(h, P.n_loc, P.local.row_offsets, P.local.cols, P.local.vals, P.fro);
        // factor slice: the rank's leaves, subtree tiles, bridges and gate + the G-1 top tiles
        const Layout Lg = make_layout(n, leaf, ls), Ll = make_layout(P.n_loc, leaf, ls);
        std::vector<float> loc(Ll.total), top((G - 1) * ls * ls);
        if (packed) slice_factors(Lg, packed, G, rank, loc.data(), top.data());
        else init_factors_slice(Lg, G, rank, sigma, seed, frame, loc.data(), top.data());
        dalloc(h->F, Ll.total);
        CK(cudaMemcpy(h->F, loc.data(), Ll.total * 4, cudaMemcpyHostToDevice));
        h->L = Ll;
        h->have_factors = true;
        h->spd_enabled = spd_enabled;
        h->spd_raw = spd_raw;
        h->fast = true;
        h->precond = HFPG_PRECOND_FACTOR;
        ensure_workspace(h);
        dalloc(S.top_tiles, top.size());
        CK(cudaMemcpy(S.top_tiles, top.data(), top.size() * 4, cudaMemcpyHostToDevice));
        dalloc(S.top_coupled, (G - 1) * 64);
        dalloc(S.send_rows, P.send_rows.size());
        dalloc(S.send_slot, P.send_slot.size());
        dalloc(S.send_off, G + 1);
        if (!P.send_rows.empty()) {
            CK(cudaMemcpy(S.send_rows, P.send_rows.data(), P.send_rows.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(S.send_slot, P.send_slot.data(), P.send_slot.size() * 4, cudaMemcpyHostToDevice));
        }
        std::vector<unsigned long long> so(P.send_off.begin(), P.send_off.end());
        CK(cudaMemcpy(S.send_off, so.data(), so.size() * 8, cudaMemcpyHostToDevice));
        dalloc(S.mbox, 1);
        CK(cudaMemset(S.mbox, 0, sizeof(Mailbox)));
        dalloc(S.seq, 3);
        CK(cudaMemset(S.seq, 0, 3 * 8));
        dalloc(S.peer_mbox, G);
        dalloc(S.peer_z, G);
        const double shift = spd_enabled ? std::log1p(std::exp(spd_raw)) : 0.0;
        CK(cudaMemcpy(&h->sc->shift, &shift, 8, cudaMemcpyHostToDevice));
        CK(cudaDeviceSynchronize());
    });
}

int hfpg_part_info(hfpg_handle* h, uint64_t* out) {
    return guarded([&] {
        out[0] = h->part.G > 1 ? h->n : h->n;
        out[1] = h->part.row0;
        out[2] = h->part.n_ghost;
        out[3] = h->part.halo_send;
        out[4] = h->part.G;
        out[5] = h->part.rank;
    });
}

int hfpg_part_mailbox(hfpg_handle* h, void** mailbox, void** z) {
    return guarded([&] {
        if (h->part.G < 2) throw InvalidArgument("partition: handle holds no partition");
        *mailbox = h->part.mbox;
        *z = h->z;
    });
}

int hfpg_part_connect(hfpg_handle* h, void* const* mailboxes, void* const* zs) {
    return guarded([&] {
        set_device(h);
        auto& S = h->part;
        if (S.G < 2) throw InvalidArgument("partition: handle holds no partition");
        if (mailboxes[S.rank] != S.mbox || zs[S.rank] != h->z)
            throw InvalidArgument("partition: own slot of the peer table is not this rank");
        CK(cudaMemcpy(S.peer_mbox, mailboxes, S.G * sizeof(void*), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(S.peer_z, zs, S.G * sizeof(void*), cudaMemcpyHostToDevice));
        S.connected = true;
        invalidate_graph(h);
    });
}

int hfpg_part_ipc_get(hfpg_handle* h, void* out) {
    return guarded([&] {
        set_device(h);
        if (h->part.G < 2) throw InvalidArgument("partition: handle holds no partition");
        cudaIpcMemHandle_t a, b;
        CK(cudaIpcGetMemHandle(&a, h->part.mbox));
        CK(cudaIpcGetMemHandle(&b, h->z));
        std::memcpy(out, &a, sizeof(a));
        std::memcpy(static_cast<char*>(out) + 64, &b, sizeof(b));
    });
}

int hfpg_part_ipc_connect(hfpg_handle* h, const void* all) {
    return guarded([&] {
        set_device(h);
        auto& S = h->part;
        if (S.G < 2) throw InvalidArgument("partition: handle holds no partition");
        std::vector<void*> mb(S.G), zz(S.G);
        for (uint32_t q = 0; q < S.G; ++q) {
            if (q == S.rank) {
                mb[q] = S.mbox;
                zz[q] = h->z;
                continue;
            }
            cudaIpcMemHandle_t a, b;
            std::memcpy(&a, static_cast<const char*>(all) + 128 * q, sizeof(a));
            std::memcpy(&b, static_cast<const char*>(all) + 128 * q + 64, sizeof(b));
            CK(cudaIpcOpenMemHandle(&mb[q], a, cudaIpcMemLazyEnablePeerAccess));
            S.ipc_opened.push_back(mb[q]);
            CK(cudaIpcOpenMemHandle(&zz[q], b, cudaIpcMemLazyEnablePeerAccess));
            S.ipc_opened.push_back(zz[q]);
        }
        CK(cudaMemcpy(S.peer_mbox, mb.data(), S.G * sizeof(void*), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(S.peer_z, zz.data(), S.G * sizeof(void*), cudaMemcpyHostToDevice));
        S.connected = true;
        invalidate_graph(h);
    });
}

// In-process group: every rank's kernels in ONE graph on rank 0's stream, stage by stage, so a
// stage's messages are complete before any rank's next stage waits on them.
int hfpg_group_pcg_solve(hfpg_handle* const* hs, uint32_t G, const double* b,
                         const hfpg_solve_config* cfg_in, double* x, double* history,
                         hfpg_report* report) {
    return guarded([&] {
        check_group(hs, G);
        hfpg_handle* h0 = hs[0];
        set_device(h0);
        hfpg_solve_config cfg = cfg_in ? *cfg_in : hfpg_solve_config{1e-8, 20000};
        if (!(cfg.rtol > 0.0)) throw InvalidArgument("pcg_solve: rtol must be positive");
        const uint64_t nl = h0->n, hcap = std::max<uint64_t>(cfg.max_iters, 1);
        for (uint32_t r = 0; r < G; ++r) {
            hfpg_handle* h = hs[r];
            ensure_workspace(h);
            if (h->history_cap < hcap) {
                dalloc(h->history, hcap);
                h->history_cap = hcap;
            }
            const Scalars init = solve_scalars(h, cfg);
            CK(cudaMemcpyAsync(h->sc, &init, sizeof(Scalars), cudaMemcpyHostToDevice, h0->stream));
            CK(cudaMemcpyAsync(h->b, b + r * nl, nl * 8, cudaMemcpyHostToDevice, h0->stream));
        }
        cudaGraph_t graph;
        CK(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle cond;
        CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
        for (uint32_t r = 0; r < G; ++r) {
            fill_sys(hs[r]);
            hs[r]->sys.cond = cond;
            hs[r]->sys.use_cond = 1;
            hs[r]->lstream = h0->stream;
        }
        auto each = [&](auto&& fn) { for (uint32_t r = 0; r < G; ++r) fn(hs[r]); };
        CK(cudaStreamBeginCaptureToGraph(h0->stream, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        each([&](hfpg_handle* h) { k_init<<<unsigned(simple_grid(h)), 256, 0, h0->stream>>>(h->sys, h->b); });
        each([&](hfpg_handle* h) { stage_leaf(h, kInit, nullptr); });
        each([&](hfpg_handle* h) { stage_sums(h, kInit); });
        each([&](hfpg_handle* h) { stage_tiles(h, kInit); });
        each([&](hfpg_handle* h) { stage_prolong(h, kInit, nullptr, nullptr); });
        CK(cudaStreamEndCapture(h0->stream, &graph));
        size_t nn = 0;
        CK(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
        cudaGraphNode_t sink = nullptr;
        for (auto nd : nodes) {
            size_t nout = 0;
            CK(cudaGraphNodeGetDependentNodes(nd, nullptr, &nout));
            if (nout == 0) sink = nd;
        }
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        CK(cudaGraphAddNode(&cnode, graph, &sink, 1, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(h0->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        each([&](hfpg_handle* h) { launch_spmv<kLoop>(h, h->sys, nullptr, nullptr); CK(cudaGetLastError()); });
        each([&](hfpg_handle* h) { stage_leaf(h, kLoop, nullptr); });
        each([&](hfpg_handle* h) { stage_sums(h, kLoop); });
        each([&](hfpg_handle* h) { stage_tiles(h, kLoop); });
        each([&](hfpg_handle* h) { stage_prolong(h, kLoop, nullptr, nullptr); });
        CK(cudaStreamEndCapture(h0->stream, &body));
        for (uint32_t r = 0; r < G; ++r) hs[r]->lstream = hs[r]->stream;
        cudaGraphExec_t exec;
        CK(cudaGraphInstantiate(&exec, graph, 0));
        CK(cudaEventRecord(h0->ev0, h0->stream));
        CK(cudaGraphLaunch(exec, h0->stream));
        CK(cudaEventRecord(h0->ev1, h0->stream));
        Scalars out{};
        CK(cudaMemcpyAsync(&out, h0->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, h0->stream));
        if (x)
            for (uint32_t r = 0; r < G; ++r)
                CK(cudaMemcpyAsync(x + r * nl, hs[r]->x, nl * 8, cudaMemcpyDeviceToHost, h0->stream));
        CK(cudaStreamSynchronize(h0->stream));
        if (history && out.hist_len) {
            CK(cudaMemcpy(history, h0->history, out.hist_len * 8, cudaMemcpyDeviceToHost));
        }
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h0->ev0, h0->ev1));
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
        if (report) {
            report->n = nl * G;
            report->iterations = out.iterations;
            report->converged = out.converged;
            report->status = out.status;
            report->breakdown_iter = out.breakdown_iter;
            report->history_len = out.hist_len;
            report->wall_ms = ms;
        }
    });
}

int hfpg_group_apply(hfpg_handle* const* hs, uint32_t G, const double* r_in, double* z_out) {
    return guarded([&] {
        check_group(hs, G);
        hfpg_handle* h0 = hs[0];
        set_device(h0);
        const uint64_t nl = h0->n;
        for (uint32_t r = 0; r < G; ++r) {
            ensure_workspace(hs[r]);
            fill_sys(hs[r]);
            hs[r]->lstream = h0->stream;
            CK(cudaMemcpyAsync(hs[r]->scratch, r_in + r * nl, nl * 8, cudaMemcpyHostToDevice, h0->stream));
        }
        for (uint32_t r = 0; r < G; ++r) stage_leaf(hs[r], kApply, hs[r]->scratch);
        for (uint32_t r = 0; r < G; ++r) stage_sums(hs[r], kApply);
        for (uint32_t r = 0; r < G; ++r) stage_tiles(hs[r], kApply);
        for (uint32_t r = 0; r < G; ++r) stage_prolong(hs[r], kApply, hs[r]->scratch, hs[r]->z);
        for (uint32_t r = 0; r < G; ++r) {
            hs[r]->lstream = hs[r]->stream;
            CK(cudaMemcpyAsync(z_out + r * nl, hs[r]->z, nl * 8, cudaMemcpyDeviceToHost, h0->stream));
        }
        CK(cudaStreamSynchronize(h0->stream));
    });
}


// ---- IC(0) (ic0.cpp) ------------------------------------------------------------------------
int hfpg_ic0_factor_host(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v, int32_t policy,
                         uint64_t* lro, uint32_t* lci, double* lv, uint64_t cap, uint64_t* nnz_out,
                         double* shift_out) {
    return guarded([&] {
        std::vector<uint64_t> r;
        std::vector<uint32_t> c;
        std::vector<double> x;
        double shift = 0.0;
        ic0_factorize_host(n, ro, ci, v, policy, r, c, x, shift);
        *nnz_out = c.size();
        if (shift_out) *shift_out = shift;
        if (cap < c.size()) throw InvalidArgument("ic0_factor_host: output capacity below nnz(L)");
        std::memcpy(lro, r.data(), (n + 1) * 8);
        std::memcpy(lci, c.data(), c.size() * 4);
        std::memcpy(lv, x.data(), x.size() * 8);
    });
}

int hfpg_load_ic0(hfpg_handle* h, uint64_t n, const uint64_t* lro, const uint32_t* lci, const double* lv) {
    return guarded([&] {
        set_device(h);
        if (h->part.G > 1) throw InvalidArgument("load_ic0: partitioned handle");
        if (n == 0 || lro[0] != 0) throw InvalidArgument("load_ic0: bad lower factor");
        for (uint64_t i = 0; i < n; ++i)  // rows nonempty, diagonal last, strictly lower before it
            if (lro[i + 1] <= lro[i] || lci[lro[i + 1] - 1] != i)
                throw InvalidArgument("load_ic0: row " + std::to_string(i) + " does not end with its diagonal");
        const uint64_t nnz = lro[n];
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t p = lro[i]; p + 1 < lro[i + 1]; ++p)
                if (lci[p] >= i) throw InvalidArgument("load_ic0: entry above the diagonal");
        std::vector<uint64_t> vr(lro, lro + n + 1), tro;
        std::vector<uint32_t> vc(lci, lci + nnz), tci;
        std::vector<double> vv(lv, lv + nnz), tv;
        ic0_transpose_host(n, vr, vc, vv, tro, tci, tv);
        std::vector<uint32_t> fperm, bperm;
        uint32_t fl = 0, bl = 0;
        ic0_levels_host(n, vr, vc, tro, tci, fperm, bperm, fl, bl);
        std::vector<uint16_t> flev, blev, fmx, bmx;
        ic0_chunk_levels_host(n, kIc0Threads, vr, vc, tro, tci, flev, blev, fmx, bmx);
        invalidate_graph(h);
        auto& c = h->ic0;
        dalloc(c.lro, n + 1);
        dalloc(c.lci, nnz);
        dalloc(c.lv, nnz);
        dalloc(c.tro, n + 1);
        dalloc(c.tci, std::max<uint64_t>(tci.size(), 1));
        dalloc(c.tv, std::max<uint64_t>(tv.size(), 1));
        dalloc(c.y, n);
        dalloc(c.fperm, n);
        dalloc(c.bperm, n);
        dalloc(c.flev, n);
        dalloc(c.blev, n);
        dalloc(c.fmax, fmx.size());
        dalloc(c.bmax, bmx.size());
        CK(cudaMemcpy(c.flev, flev.data(), n * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.blev, blev.data(), n * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.fmax, fmx.data(), fmx.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.bmax, bmx.data(), bmx.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.fperm, fperm.data(), n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.bperm, bperm.data(), n * 4, cudaMemcpyHostToDevice));
        c.flevels = fl;
        c.blevels = bl;
        CK(cudaMemcpy(c.lro, vr.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.lci, vc.data(), nnz * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.lv, vv.data(), nnz * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.tro, tro.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
        if (!tci.empty()) {
            CK(cudaMemcpy(c.tci, tci.data(), tci.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(c.tv, tv.data(), tv.size() * 8, cudaMemcpyHostToDevice));
        }
        c.n = n;
        c.have = true;
    });
}

int hfpg_ic0_apply(hfpg_handle* h, const double* r, double* z, int where) {
    return guarded([&] {
        set_device(h);
        if (!h->ic0.have || !h->have_csr || h->ic0.n != h->n) throw InvalidArgument("ic0_apply: no IC(0) factor loaded");
        ensure_workspace(h);
        fill_sys(h);
        const double* rin = r;
        double* zout = z;
        if (where == HFPG_HOST) {
            copy_in(h, h->scratch, r, h->n, HFPG_HOST);
            rin = h->scratch;
            zout = h->z;
        }
        h->lstream = h->stream;
        k_ic0_pending<<<unsigned(simple_grid(h)), 256, 0, h->stream>>>(ic0_dev(h), zout, h->n);
        CK(cudaGetLastError());
        launch_ic0_sweeps(h, h->sys, kApply, rin, zout);
        if (where == HFPG_HOST) copy_out(h, z, h->z, h->n, HFPG_HOST);
        CK(cudaStreamSynchronize(h->stream));
    });
}


// ---- on-disk formats on the device --------------------------------------
int hfpg_crc32(hfpg_handle* h, const void* data, uint64_t bytes, int where, uint32_t* out) {
    return guarded([&] {
        set_device(h);
        if (where == HFPG_DEVICE) {
            *out = device_crc(h, data, bytes);
        } else {
            uLong c = ::crc32(0L, Z_NULL, 0);
            const Bytef* b = static_cast<const Bytef*>(data);
            for (uint64_t left = bytes; left;) {
                const uInt chunk = static_cast<uInt>(std::min<uint64_t>(left, 1u << 30));
                c = ::crc32(c, b, chunk);
                b += chunk;
                left -= chunk;
            }
            *out = uint32_t(c);
        }
    });
}

// checkpoint.cpp:45-85 read_checkpoint straight into the handle's factor tensor: header on the
// host, payload streamed through pinned buffers into device memory, crc32 on the GPU.
int hfpg_load_checkpoint(hfpg_handle* h, const char* path) {
    return guarded([&] {
        set_device(h);
        const HftcHeader H = hftc_read_header(path);
        const Layout& L = H.L;
        if (h->have_csr && h->n != L.n) throw InvalidArgument("load_factors: length mismatch");
        std::unique_ptr<std::FILE, FileCloser> fp(std::fopen(path, "rb"));
        if (!fp) throw IoError(std::string("read_checkpoint: cannot open ") + path);
        invalidate_graph(h);
        if (!h->have_factors || h->L.total != L.total) dalloc(h->F, L.total);
        h->have_factors = false;
        stream_to_device(h, fp.get(), H.payload_offset, L.total * 4, h->F, "read_checkpoint");
        if (device_crc(h, h->F, ref_crc_len(L.total * 4)) != H.crc) throw IoError("read_checkpoint: payload checksum mismatch");
        h->L = L;
        h->have_factors = true;
        h->spd_enabled = H.spd_enabled;
        h->spd_raw = H.spd_raw;
        h->fast = (L.l == kL && L.ls == kLs && std::getenv("HFPG_FORCE_GENERIC") == nullptr);
        if (!h->have_csr && !h->have_diag) h->n = L.n;
        ensure_workspace(h);
        const double shift = H.spd_enabled ? std::log1p(std::exp(H.spd_raw)) : 0.0;  // factor_tensor.hpp:64
        CK(cudaMemcpyAsync(&h->sc->shift, &shift, 8, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int hfpg_load_mppf(hfpg_handle* h, const char* path) {
    return guarded([&] { frame_from_mppf(h, path); });
}


// ---- training (adjoint.cpp, loss.cpp, train.cpp) ---------------------------
int hfpg_batch_apply(hfpg_handle* h, const double* params, uint64_t leaf, uint64_t ls, double shift,
                     const double* x, uint64_t kz, double* y, int where) {
    return guarded([&] {
        set_device(h);
        train_prepare(h, leaf, ls, kz, shift);
        const Layout L = make_layout(h->n, leaf, ls);
        const double* P = train_params(h, params, L.total, where);
        auto& T = h->tr.T;
        CK(cudaMemcpyAsync(T.X, x, h->n * kz * 8, where == HFPG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                           h->stream));
        train_forward(h->stream, T, P);
        CK(cudaGetLastError());
        if (y) CK(cudaMemcpyAsync(y, T.Y, h->n * kz * 8, where == HFPG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                  h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->tr.have_fwd = true;
    });
}

int hfpg_batch_adjoint(hfpg_handle* h, const double* params, const double* bar_y, double* grad, int where) {
    return guarded([&] {
        set_device(h);
        auto& R = h->tr;
        if (!R.have_fwd) throw InvalidArgument("factor_apply_batch_adjoint: no forward batch on this handle");
        const Layout L = make_layout(h->n, 128, 32);
        const double* P = train_params(h, params, L.total, where);
        const uint64_t nk = h->n * R.kz;
        const double* BY = bar_y;
        if (where == HFPG_HOST) {
            CK(cudaMemcpyAsync(R.BY, bar_y, nk * 8, cudaMemcpyHostToDevice, h->stream));
            BY = R.BY;
        }
        double* G = where == HFPG_HOST ? R.G : grad;
        CK(cudaMemsetAsync(G, 0, L.total * 8, h->stream));
        train_adjoint(h->stream, R.T, P, BY, G);
        CK(cudaGetLastError());
        if (where == HFPG_HOST) CK(cudaMemcpyAsync(grad, R.G, L.total * 8, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

// adjoint.cpp:250-292 loss_gradient (kind 0 cosine, 1 sai) on the handle's system.
int hfpg_loss_gradient(hfpg_handle* h, const double* params, uint64_t leaf, uint64_t ls, double shift,
                       const double* z, uint64_t kz, int32_t kind, double norm_a, double* loss,
                       int32_t* degenerate, double* grad, int where) {
    return guarded([&] {
        set_device(h);
        if (kind != 0 && kind != 1) throw InvalidArgument("loss_gradient: unknown loss kind");
        if (kind == 1 && !(norm_a > 0.0)) throw InvalidArgument("sai_loss: norm_a must be positive");
        train_prepare(h, leaf, ls, kz, shift);
        const Layout L = make_layout(h->n, leaf, ls);
        const double* P = train_params(h, params, L.total, where);
        auto& R = h->tr;
        auto& T = R.T;
        const uint64_t nk = h->n * kz;
        double* Z = R.Z;
        CK(cudaMemcpyAsync(Z, z, nk * 8, where == HFPG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
        double* G = where == HFPG_HOST ? R.G : grad;
        CK(cudaMemsetAsync(G, 0, L.total * 8, h->stream));
        double* BY = R.BY;
        *degenerate = 0;
        if (kind == 0) {  // Y = M (A Z), 1 - cos(Z, Y)
            train_spmm(h, Z, T.X, kz);
            train_forward(h->stream, T, P);
            const double* Y = T.Y;
            double s3[3];
            train_sums<3>(h, nk, [=] __device__(uint64_t i, double (&e)[3]) {
                e[0] = Z[i] * Y[i];
                e[1] = Z[i] * Z[i];
                e[2] = Y[i] * Y[i];
            }, s3);
            const double zy = s3[0], zz = s3[1], yy = s3[2];
            if (zz == 0.0 || yy == 0.0) {
                *degenerate = 1;
                *loss = 0.0;
            } else {
                const double nz = std::sqrt(zz), ny = std::sqrt(yy);
                *loss = 1.0 - zy / (nz * ny);
                const double c1 = 1.0 / (nz * ny), c2 = zy / (nz * ny * ny * ny);
                each(h->stream, nk, [=] __device__(uint64_t i) { BY[i] = -(Z[i] * c1 - Y[i] * c2); });
                train_adjoint(h->stream, T, P, BY, G);
            }
        } else {  // W = M Z; |(1/normA) A W - Z|^2
            CK(cudaMemcpyAsync(T.X, Z, nk * 8, cudaMemcpyDeviceToDevice, h->stream));
            train_forward(h->stream, T, P);
            double* Q = T.W;  // scratch until the adjoint (which rewrites W)
            train_spmm(h, T.Y, Q, kz);
            each(h->stream, nk, [=] __device__(uint64_t i) { Q[i] = Q[i] / norm_a - Z[i]; });
            double s1[1];
            train_sums<1>(h, nk, [=] __device__(uint64_t i, double (&e)[1]) { e[0] = Q[i] * Q[i]; }, s1);
            *loss = s1[0];
            train_spmm(h, Q, BY, kz);
            const double scale = 2.0 / norm_a;
            each(h->stream, nk, [=] __device__(uint64_t i) { BY[i] *= scale; });
            train_adjoint(h->stream, T, P, BY, G);
        }
        CK(cudaGetLastError());
        if (where == HFPG_HOST) CK(cudaMemcpyAsync(grad, R.G, L.total * 8, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        R.have_fwd = true;
    });
}

// train.cpp:136-160: global clip of g to clip_norm, then AdamW with decoupled weight decay
// (device pointers, count elements, step >= 1).
int hfpg_adamw_step(hfpg_handle* h, double* params, double* grad, double* m1, double* m2, uint64_t count,
                    uint64_t step, double lr, double beta1, double beta2, double eps, double weight_decay,
                    double clip_norm, double* gnorm_out) {
    return guarded([&] {
        set_device(h);
        if (step == 0) throw InvalidArgument("adamw: step counts from 1");
        if (!h->tr.part) dalloc(h->tr.part, 4096 * 3);
        const double* g = grad;
        double s1[1];
        train_sums<1>(h, count, [=] __device__(uint64_t i, double (&e)[1]) { e[0] = g[i] * g[i]; }, s1);
        const double gnorm = std::sqrt(s1[0]);
        if (gnorm_out) *gnorm_out = gnorm;
        const double s = (gnorm > clip_norm && gnorm > 0.0) ? clip_norm / gnorm : 1.0;
        const double bc1 = 1.0 - std::pow(beta1, double(step)), bc2 = 1.0 - std::pow(beta2, double(step));
        each(h->stream, count, [=] __device__(uint64_t i) {
            const double gi = s == 1.0 ? grad[i] : grad[i] * s;
            grad[i] = gi;
            m1[i] = beta1 * m1[i] + (1.0 - beta1) * gi;
            m2[i] = beta2 * m2[i] + (1.0 - beta2) * gi * gi;
            const double mhat = m1[i] / bc1, vhat = m2[i] / bc2;
            params[i] -= lr * (mhat / (sqrt(vhat) + eps) + weight_decay * params[i]);
        });
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
    });
}

}  // extern "C"
