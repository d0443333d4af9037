// Toy-network inference + factor assembly on the GPU (toy_net.cpp:170-586): encoder MLP, D^-1 A
// graph convolutions, leaf-window and strip-pooled tile attention with edge biases, highway
// buffers, 4d FFNs and the decoder heads writing the packed factor tensor. Dense contractions
// run on tcgen05 (kind::tf32, TMEM accumulators, TMA-fed); the rest are fp32 SIMT kernels.
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdlib>
#include <initializer_list>
#include <type_traits>
#include <vector>

#include "attention_tcgen05.cuh"
#include "gemm_persistent.cuh"
#include "gemm_tcgen05.cuh"
#include "internal.hpp"
#include "toynet_kernels.cuh"

namespace hfpg {

namespace {

#define TCK(call)                                                                         \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

// ---- weights: toy_net.cpp:170-223, drawn in the reference's exact order ---------------------
struct Mat {
    uint64_t rows = 0, cols = 0;
    std::vector<double> v;  // row-major rows x cols (in x out)
};
struct HostWeights {
    Mat enc1, enc2;
    std::vector<Mat> gcn;
    struct Layer {
        Mat wq, wk, wv, wo, ffn1, ffn2;
    };
    std::vector<Layer> leaf, tile;
    Mat le_w1, le_w2, te_w1, te_w2;
    Mat lh1, lh2, thu, thv, bhu, bhv;
    std::vector<double> gate;
};

HostWeights init_weights(const hfpg_toynet_config& c, uint64_t L, uint64_t Ls, uint64_t seed) {
    if (c.d % c.heads != 0) throw InvalidArgument("toynet: heads must divide embedding width");
    Rng rng(seed, 0, 5);  // RngPurpose::net_weights
    auto random_mat = [&](uint64_t rows, uint64_t cols) {  // toy_net.cpp:43-48
        Mat m;
        m.rows = rows;
        m.cols = cols;
        m.v.resize(rows * cols);
        const double scale = 1.0 / std::sqrt(static_cast<double>(rows));
        for (double& x : m.v) x = scale * rng.normal();
        return m;
    };
    const uint64_t d = c.d, feat = 7 + c.d_global;
    HostWeights w;
    w.enc1 = random_mat(feat, d);
    w.enc2 = random_mat(d, d);
    for (uint64_t g = 0; g < c.gcn_layers; ++g) w.gcn.push_back(random_mat(d, d));
    for (auto* s : {&w.leaf, &w.tile})
        for (uint64_t l = 0; l < c.layers; ++l) {
            HostWeights::Layer x;
            x.wq = random_mat(d, d);
            x.wk = random_mat(d, d);
            x.wv = random_mat(d, d);
            x.wo = random_mat(d, d);
            x.ffn1 = random_mat(4 * d, 4 * d);
            x.ffn2 = random_mat(4 * d, d);
            s->push_back(std::move(x));
        }
    w.le_w1 = random_mat(4, c.edge_hidden);
    w.le_w2 = random_mat(c.edge_hidden, c.heads);
    w.te_w1 = random_mat(4, c.edge_hidden);
    w.te_w2 = random_mat(c.edge_hidden, c.heads);
    w.lh1 = random_mat(d, d);
    w.lh2 = random_mat(d, L);
    w.thu = random_mat(d, Ls / 2);
    w.thv = random_mat(d, Ls / 2);
    w.bhu = random_mat(d, Ls);
    w.bhv = random_mat(d, Ls);
    w.gate.resize(d);
    for (double& x : w.gate) x = rng.normal() / std::sqrt(static_cast<double>(d));
    return w;  // every bias of init_weights is zero
}

// ---- TMA tensor maps (driver entry point fetched through the runtime) -----------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        TCK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}
// fp32 row-major [rows x cols] with row pitch ld (elements); box = box_rows x 32, SWIZZLE_128B.
CUtensorMap tmap(const float* p, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 4};
    cuuint32_t box[2] = {32, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

// ---- GEMM epilogues (k_pgemm_tf32): apply8(row0, col, v[8], ncols, M) — columns col .. col+3
// (ncols valid) of rows row0 + 4 i, i < 8 (rows >= M skipped); coalesced across the warp ---------
__device__ __forceinline__ float4 f4_act(float4 v, float4 b, bool gelu) {
    v = make_float4(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
    if (gelu) v = make_float4(gelu_fast(v.x), gelu_fast(v.y), gelu_fast(v.z), gelu_fast(v.w));
    return v;
}
__device__ __forceinline__ float4 f4_bias(const float* bias, int col, int ncols) {
    if (!bias) return make_float4(0.f, 0.f, 0.f, 0.f);
    if (ncols == 4) return *reinterpret_cast<const float4*>(bias + col);
    float b[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < ncols; ++j) b[j] = bias[col + j];
    return make_float4(b[0], b[1], b[2], b[3]);
}
__device__ __forceinline__ void f4_store(float* o, float4 v, int ncols) {
    if (ncols == 4) {
        *reinterpret_cast<float4*>(o) = v;
    } else {
        const float e[4] = {v.x, v.y, v.z, v.w};
        for (int j = 0; j < ncols; ++j) o[j] = e[j];
    }
}
template <bool GELU>
struct EpiStore {  // out[row, col] = act(v + bias); ld a multiple of 4
    static constexpr bool kWholeRow = false;
    float* out;
    uint32_t ld;
    const float* bias;
    __device__ __forceinline__ void apply8(int row0, int col, float4 (&v)[8], int ncols, int M) const {
        const float4 b = f4_bias(bias, col, ncols);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = row0 + 4 * i;
            if (row < M) f4_store(out + uint64_t(row) * ld + col, f4_act(v[i], b, GELU), ncols);
        }
    }
};
template <bool GELU>
struct EpiResidual {  // out[row, col] += act(v + bias)
    static constexpr bool kWholeRow = false;
    float* out;
    uint32_t ld;
    const float* bias;
    __device__ __forceinline__ void apply8(int row0, int col, float4 (&v)[8], int ncols, int M) const {
        const float4 b = f4_bias(bias, col, ncols);
        float4 a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // all residual loads first
            const int row = row0 + 4 * i;
            a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < M) {
                const float* o = out + uint64_t(row) * ld + col;
                if (ncols == 4) {
                    a[i] = *reinterpret_cast<const float4*>(o);
                } else {
                    float e[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int j = 0; j < ncols; ++j) e[j] = o[j];
                    a[i] = make_float4(e[0], e[1], e[2], e[3]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = row0 + 4 * i;
            const float4 x = f4_act(v[i], b, GELU);
            if (row < M)
                f4_store(out + uint64_t(row) * ld + col, make_float4(a[i].x + x.x, a[i].y + x.y, a[i].z + x.z, a[i].w + x.w),
                         ncols);
        }
    }
};
// Residual + LayerNorm of the updated row (toy_net.cpp:28-41, no affine, eps 1e-5, two-pass):
// x[row] += act(v) (the sublayer output, toy_net.cpp:123 / :435; act = GELU for the GCN update,
// :316), ln[row] = LN(x[row]) — the next sublayer's normalised input, so there is no separate
// LayerNorm pass over the tokens. Rows of d = 128 = BN (k_pgemm_tf32's whole-row epilogue).
struct EpiResidualLN {
    static constexpr bool kWholeRow = true;
    float* x;
    float* ln;
    int gelu;
    __device__ __forceinline__ float act(float v) const { return gelu_fast(v); }
};
// Decoder heads of leaf node `row` (toy_net.cpp:549-567): columns [0, L_s) -> Ũ_k row,
// [L_s, 2 L_s) -> Ṽ_k row, 2 L_s -> gate. Cast to float as the reference does.
struct EpiLeafHeads {
    static constexpr bool kWholeRow = false;
    float* out;
    uint32_t lL, lLs;  // log2 L, log2 L_s (powers of two, as the GPU forward requires)
    uint64_t bridge_base, gate_base;
    __device__ __forceinline__ void apply8(int row0, int col, float4 (&v)[8], int ncols, int M) const {
        const uint32_t Ls = 1u << lLs, L = 1u << lL;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t row = uint64_t(row0 + 4 * i), k = row >> lL, r = row & (L - 1);
            if (row >= uint64_t(M)) continue;
            const float e[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
            float* bu = out + bridge_base + k * (2ull * L * Ls) + r * Ls;
            for (int j = 0; j < ncols; ++j) {
                const uint32_t c = uint32_t(col + j);
                if (c < Ls) bu[c] = e[j];
                else if (c < 2 * Ls) bu[uint64_t(L) * Ls + (c - Ls)] = e[j];
                else if (c == 2 * Ls) out[gate_base + row] = e[j];
            }
        }
    }
};
// Tile heads of tile token `row` = m L_s + tok (toy_net.cpp:570-584): [0, rk) -> U_m[tok],
// [rk, 2 rk) -> V_m[tok].
struct EpiTileHeads {
    static constexpr bool kWholeRow = false;
    float* out;
    uint32_t lLs;  // log2 L_s
    uint64_t tile_base;
    __device__ __forceinline__ void apply8(int row0, int col, float4 (&v)[8], int ncols, int M) const {
        const uint32_t Ls = 1u << lLs, rk = Ls >> 1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t row = uint64_t(row0 + 4 * i), m = row >> lLs, tok = row & (Ls - 1);
            if (row >= uint64_t(M)) continue;
            const float e[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
            for (int j = 0; j < ncols; ++j) {
                const uint32_t c = uint32_t(col + j);
                if (c < 2 * rk) out[tile_base + m * Ls * Ls + (c < rk ? 0 : Ls * rk) + tok * rk + (c % rk)] = e[j];
            }
        }
    }
};

// A operand sources side by side along K (gemm_persistent.cuh): {pointer, row pitch, columns}.
struct ASrc {
    const float* p;
    uint64_t ld, kcols;
};
PgA make_pga(std::initializer_list<ASrc> srcs, uint64_t M) {
    PgA a{};
    int s = 0, kb = 0;
    for (const ASrc& d : srcs) {
        if (s == 3) throw InvalidArgument("gemm: at most three A sources");
        a.map[s] = tmap(d.p, M, d.kcols, d.ld, kGemmBM);
        kb += int((d.kcols + kGemmBK - 1) / kGemmBK);
        a.kb_end[s] = kb;
        if (s + 1 < int(srcs.size()) && d.kcols % kGemmBK) throw InvalidArgument("gemm: inner A sources need K % 32 == 0");
        ++s;
    }
    a.nsrc = s;
    return a;
}
int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        TCK(cudaGetDevice(&dev));
        TCK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}
// C = epi(A * W): A from `pa` (M x K), W^T = Bt (N x K, row pitch ldb).
template <int BN, class Epi>
void pgemm(cudaStream_t st, const PgA& pa, uint64_t M, uint64_t K, const float* Bt, uint64_t N, uint64_t ldb,
           const Epi& epi) {
    static bool configured = false;
    if (!configured) {
        TCK(cudaFuncSetAttribute(k_pgemm_tf32<BN, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(pgemm_smem_bytes<BN, Epi::kWholeRow>())));
        configured = true;
    }
    if (M == 0 || N == 0) return;
    const CUtensorMap tb = tmap(Bt, N, K, ldb, BN);
    const uint64_t tiles = ((M + kGemmBM - 1) / kGemmBM) * ((N + BN - 1) / BN);
    const unsigned grid = unsigned(std::min<uint64_t>(tiles, uint64_t(sm_count())));
    k_pgemm_tf32<BN, Epi><<<grid, kPgThreads, pgemm_smem_bytes<BN, Epi::kWholeRow>(), st>>>(pa, tb, int(M), int(N), int(K), epi);
    TCK(cudaGetLastError());
}
template <int BN, class Epi>
void pgemm1(cudaStream_t st, const float* A, uint64_t M, uint64_t K, uint64_t lda, const float* Bt, uint64_t N,
            uint64_t ldb, const Epi& epi) {
    pgemm<BN>(st, make_pga({ASrc{A, lda, K}}, M), M, K, Bt, N, ldb, epi);
}

// Device copy of W^T (out x in, fp32), optionally padding the input dimension to kpad.
float* upload_t(const Mat& m, std::vector<float*>& owned, uint64_t kpad = 0) {
    const uint64_t kp = std::max(kpad, m.rows);
    std::vector<float> t(m.cols * kp, 0.f);
    for (uint64_t i = 0; i < m.rows; ++i)
        for (uint64_t o = 0; o < m.cols; ++o) t[o * kp + i] = float(m.v[i * m.cols + o]);
    float* p = nullptr;
    TCK(cudaMalloc(&p, t.size() * 4));
    TCK(cudaMemcpy(p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    owned.push_back(p);
    return p;
}
// [W_a | W_b | ...]^T stacked along the output dimension (same input dimension).
float* upload_stack_t(std::vector<const Mat*> ms, std::vector<float*>& owned, uint64_t extra_rows = 0,
                      const std::vector<double>* gate = nullptr) {
    const uint64_t kin = ms[0]->rows;
    uint64_t nout = extra_rows;
    for (auto* m : ms) nout += m->cols;
    std::vector<float> t(nout * kin, 0.f);
    uint64_t o0 = 0;
    for (auto* m : ms) {
        for (uint64_t i = 0; i < m->rows; ++i)
            for (uint64_t o = 0; o < m->cols; ++o) t[(o0 + o) * kin + i] = float(m->v[i * m->cols + o]);
        o0 += m->cols;
    }
    if (gate)
        for (uint64_t i = 0; i < kin; ++i) t[o0 * kin + i] = float((*gate)[i]);
    float* p = nullptr;
    TCK(cudaMalloc(&p, t.size() * 4));
    TCK(cudaMemcpy(p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    owned.push_back(p);
    return p;
}

template <class T>
T* dnew(uint64_t count, std::vector<void*>& owned) {
    T* p = nullptr;
    TCK(cudaMalloc(&p, std::max<uint64_t>(count, 1) * sizeof(T)));
    owned.push_back(p);
    return p;
}

EdgeMlp edge_params(const Mat& w1, const Mat& w2) {
    EdgeMlp e{};
    for (uint64_t i = 0; i < w1.v.size(); ++i) e.w1[i] = float(w1.v[i]);
    for (uint64_t i = 0; i < w2.v.size(); ++i) e.w2[i] = float(w2.v[i]);
    return e;
}

}  // namespace

// A toy-network instance on the device: weights drawn once per (cfg, L, L_s, seed) and kept as
// W^T fp32; activation scratch grown on demand and reused across frames.
struct ToynetModel {
    hfpg_toynet_config cfg{};
    uint64_t L = 0, Ls = 0, seed = 0;
    EdgeMlp le{}, te{};
    std::vector<float*> wbuf;
    float *w_enc1 = nullptr, *w_enc2 = nullptr, *w_lh1 = nullptr, *w_lh2 = nullptr,
          *w_heads = nullptr, *w_theads = nullptr;
    std::vector<float*> w_gcn;
    struct LW {
        float *qkv, *wo, *f1, *f2;
    };
    std::vector<LW> wl, wt;
    std::vector<std::pair<void*, size_t>> scratch;  // (ptr, bytes), index = buffer id
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // the tile stream's chain runs beside the leaf stream's on a second stream (fork / join)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_lbias = nullptr;
    ~ToynetModel() {
        for (float* p : wbuf) cudaFree(p);
        for (auto& b : scratch) cudaFree(b.first);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (ev_lbias) cudaEventDestroy(ev_lbias);
        if (side) cudaStreamDestroy(side);
    }
    template <class T>
    T* buf(size_t id, uint64_t count) {
        if (scratch.size() <= id) scratch.resize(id + 1, {nullptr, 0});
        const size_t bytes = std::max<uint64_t>(count, 1) * sizeof(T);
        if (scratch[id].second < bytes) {
            if (scratch[id].first) cudaFree(scratch[id].first);
            scratch[id].first = nullptr;
            TCK(cudaMalloc(&scratch[id].first, bytes));
            scratch[id].second = bytes;
        }
        return static_cast<T*>(scratch[id].first);
    }
};

ToynetModel* toynet_model_create(const hfpg_toynet_config& cfg, uint64_t L, uint64_t Ls, uint64_t seed) {
    const uint64_t d = cfg.d;
    if (d != 128) throw InvalidArgument("toynet (gpu): embedding width must be 128");
    if (cfg.heads * 16 != d) throw InvalidArgument("toynet (gpu): head dimension must be 16");
    if (cfg.edge_hidden > 8 || cfg.heads > 8 || cfg.d_global > 12)
        throw InvalidArgument("toynet (gpu): edge_hidden, heads <= 8 and d_global <= 12");
    if (!(L == 128 || L == 64 || L == 32 || L == 16 || L == 8 || L == 4) ||
        !(Ls == 32 || Ls == 16 || Ls == 8 || Ls == 4))
        throw InvalidArgument("toynet (gpu): unsupported leaf / coarse size");
    auto* m = new ToynetModel;
    try {
        m->cfg = cfg;
        m->L = L;
        m->Ls = Ls;
        m->seed = seed;
        const HostWeights w = init_weights(cfg, L, Ls, seed);
        m->le = edge_params(w.le_w1, w.le_w2);
        m->te = edge_params(w.te_w1, w.te_w2);
        m->w_enc1 = upload_t(w.enc1, m->wbuf, 32);
        m->w_enc2 = upload_t(w.enc2, m->wbuf);
        for (auto& g : w.gcn) m->w_gcn.push_back(upload_t(g, m->wbuf));
        for (auto* src : {&w.leaf, &w.tile})
            for (auto& x : *src) {
                ToynetModel::LW l{upload_stack_t({&x.wq, &x.wk, &x.wv}, m->wbuf), upload_t(x.wo, m->wbuf),
                                  upload_t(x.ffn1, m->wbuf), upload_t(x.ffn2, m->wbuf)};
                (src == &w.leaf ? m->wl : m->wt).push_back(l);
            }
        m->w_lh1 = upload_t(w.lh1, m->wbuf);
        m->w_lh2 = upload_t(w.lh2, m->wbuf);
        m->w_heads = upload_stack_t({&w.bhu, &w.bhv}, m->wbuf, 1, &w.gate);
        m->w_theads = upload_stack_t({&w.thu, &w.thv}, m->wbuf);
        TCK(cudaEventCreate(&m->ev0));
        TCK(cudaEventCreate(&m->ev1));
        TCK(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
        TCK(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
        TCK(cudaEventCreateWithFlags(&m->ev_lbias, cudaEventDisableTiming));
        TCK(cudaStreamCreateWithFlags(&m->side, cudaStreamNonBlocking));
    } catch (...) {
        delete m;
        throw;
    }
    return m;
}
void toynet_model_destroy(ToynetModel* m) { delete m; }
bool toynet_model_matches(const ToynetModel* m, const hfpg_toynet_config& c, uint64_t L, uint64_t Ls,
                          uint64_t seed) {
    return m && m->L == L && m->Ls == Ls && m->seed == seed && m->cfg.d == c.d &&
           m->cfg.layers == c.layers && m->cfg.heads == c.heads && m->cfg.gcn_layers == c.gcn_layers &&
           m->cfg.d_global == c.d_global && m->cfg.edge_hidden == c.edge_hidden;
}

// The forward proper, from device-resident inputs (the frame's order / rho / CSR / diagonal
// and the global feature vector).
static void toynet_run(ToynetModel* mdl, cudaStream_t st, uint64_t n, uint64_t width, uint64_t height,
                       uint64_t nnz, const uint32_t* d_order, const double* d_rho,
                       const unsigned long long* d_ro, const uint32_t* d_ci, const double* d_v,
                       const double* d_diag, const float* d_glob, float* out, hfpg_toynet_trace* trace) {
    const hfpg_toynet_config& cfg = mdl->cfg;
    const uint64_t L = mdl->L, Ls = mdl->Ls;
    const Layout lay = make_layout(n, L, Ls);
    const uint64_t d = cfg.d;
    TnDims g{};
    g.n = n;
    g.L = L;
    g.Ls = Ls;
    g.rk = Ls / 2;
    g.K = lay.k;
    g.M = lay.m;
    g.D = lay.depth;
    g.width = uint32_t(width);
    g.height = uint32_t(height);
    g.d = uint32_t(d);
    g.heads = uint32_t(cfg.heads);
    g.dglob = uint32_t(cfg.d_global);
    g.eh = uint32_t(cfg.edge_hidden);
    g.feat_pad = 32;
    const uint64_t MT = lay.m * Ls;  // tile tokens
    (void)nnz;

    const auto& wl = mdl->wl;
    const auto& wt = mdl->wt;
    using LW = ToynetModel::LW;
    // chunk-sum pyramids need nested power-of-two chunks: c0 = L / L_s >= 1 (the production
    // L = 128, L_s = 32 gives c0 = 4); other shapes walk each chunk
    const bool pyr = L >= Ls && lay.m > 0;
    uint32_t lev_shift = 0;
    while ((uint64_t(1) << lev_shift) < L / std::max<uint64_t>(Ls, 1)) ++lev_shift;
    const uint32_t c0 = uint32_t(1) << lev_shift, nlev = uint32_t(lay.depth);
    uint64_t pyr_rows = 0;  // entries over all levels
    for (uint32_t l = 0; l < nlev; ++l) pyr_rows += n / (uint64_t(c0) << l);
    // ---- activations -------------------------------------------------------------------------
    auto* feat = mdl->buf<float>(5, n * g.feat_pad);
    auto* x = mdl->buf<float>(6, n * d);       // embedding -> leaf tokens
    auto* h1 = mdl->buf<float>(7, n * d);      // encoder hidden / gcn message / decoder hidden
    auto* tile_tok = mdl->buf<float>(8, std::max<uint64_t>(MT, 1) * d);
    auto* ln = mdl->buf<float>(9, n * d);      // LN(leaf tokens): the next sublayer's input
    auto* qkv = mdl->buf<float>(10, n * 3 * d);
    auto* hout = mdl->buf<float>(11, n * d);
    auto* row_hw = mdl->buf<float>(12, n * d);
    auto* col_hw = mdl->buf<float>(13, n * d);
    auto* ln_t = mdl->buf<float>(14, std::max<uint64_t>(MT, 1) * d);  // LN(tile tokens)
    auto* Hf = mdl->buf<float>(15, n * 4 * d);
    auto* Hf_t = mdl->buf<float>(35, std::max<uint64_t>(MT, 1) * 4 * d);
    auto* qkv_t = mdl->buf<float>(36, std::max<uint64_t>(MT, 1) * 3 * d);
    auto* hout_t = mdl->buf<float>(37, std::max<uint64_t>(MT, 1) * d);
    auto* glob_hw = mdl->buf<float>(16, d);
    const uint32_t nparts = 296;
    const unsigned hw_blocks = pyr ? unsigned((n / c0 * 32 + 255) / 256) : 0u;  // k_tn_highway_chunks CTAs
    auto* partial = mdl->buf<float>(17, (uint64_t(nparts) * 2 + hw_blocks) * d);
    auto* leaf_bias = mdl->buf<__half>(18, lay.k * cfg.heads * L * L);
    auto* tile_bias = mdl->buf<__half>(19, std::max<uint64_t>(lay.m, 1) * cfg.heads * Ls * Ls);
    auto* tile_pos = mdl->buf<double>(26, std::max<uint64_t>(lay.m, 1) * 2 * Ls * 2);
    auto* rmean = mdl->buf<float>(28, std::max<uint64_t>(MT, 1) * d);
    auto* cmean = mdl->buf<float>(29, std::max<uint64_t>(MT, 1) * d);
    auto* pyr_r = mdl->buf<float>(30, std::max<uint64_t>(pyr_rows, 1) * d);  // also the embedding pyramid
    auto* pyr_c = mdl->buf<float>(31, std::max<uint64_t>(pyr_rows, 1) * d);
    auto* b1 = mdl->buf<float>(32, 8 * d);  // glob-slice FFN biases: leaf [0, 4d), tile [4d, 8d)
    const bool audit = trace && !trace->timing_only;
    unsigned int* rowsum_bits = audit ? mdl->buf<unsigned int>(20, 1) : nullptr;
    float* audit_part = audit ? mdl->buf<float>(23, uint64_t(nparts) * d) : nullptr;
    float* audit_sums = audit ? mdl->buf<float>(24, 6 * d) : nullptr;
    float* audit_dev = audit ? mdl->buf<float>(25, cfg.layers) : nullptr;
    if (rowsum_bits) TCK(cudaMemsetAsync(rowsum_bits, 0, 4, st));
    auto levels = [&](float* base) {
        PyrLevels<float> P{};
        uint64_t off = 0;
        for (uint32_t l = 0; l < nlev && l < 24; ++l) {
            P.lev[l] = base + off * d;
            off += n / (uint64_t(c0) << l);
        }
        return P;
    };
    // levels 0 .. nlev-1 of the row-chunk sums of src (n x C), c0 rows per level-0 entry
    auto build_pyramid = [&](cudaStream_t st, auto* src, uint32_t C, const auto& P) {
        using T = std::remove_const_t<std::remove_pointer_t<decltype(src)>>;
        using V = std::conditional_t<std::is_same_v<T, float>, float4, double2>;
        constexpr uint32_t VW = sizeof(V) / sizeof(T);
        uint32_t done = 0, group = c0;
        uint64_t rows = n;
        const T* s0 = src;
        while (done < nlev) {
            uint32_t q = std::min<uint32_t>(nlev - done - 1, 4u);
            while ((group << q) > 32) --q;
            const uint64_t nblocks = rows / (uint64_t(group) << q);
            const uint64_t threads = nblocks * (C / VW);
            const unsigned gr = unsigned((threads + 127) / 128);
            switch (group) {
                case 1: k_tn_pyramid<T, V, 1><<<gr, 128, 0, st>>>(s0, nblocks, C, q, P, done); break;
                case 2: k_tn_pyramid<T, V, 2><<<gr, 128, 0, st>>>(s0, nblocks, C, q, P, done); break;
                case 4: k_tn_pyramid<T, V, 4><<<gr, 128, 0, st>>>(s0, nblocks, C, q, P, done); break;
                case 8: k_tn_pyramid<T, V, 8><<<gr, 128, 0, st>>>(s0, nblocks, C, q, P, done); break;
                case 16: k_tn_pyramid<T, V, 16><<<gr, 128, 0, st>>>(s0, nblocks, C, q, P, done); break;
                default: k_tn_pyramid<T, V, 32><<<gr, 128, 0, st>>>(s0, nblocks, C, q, P, done); break;
            }
            done += q + 1;
            s0 = P.lev[done - 1];
            rows = n / (uint64_t(c0) << (done - 1));
            group = 2;
        }
        TCK(cudaGetLastError());
    };
    const PyrLevels<float> Pr = levels(pyr_r), Pc = levels(pyr_c);

    const unsigned nb = unsigned((n + 255) / 256), nw = unsigned((n * 32 + 255) / 256);
    cudaStream_t st2 = mdl->side;
    auto fork = [&] {  // st2 continues from st's current point
        TCK(cudaEventRecord(mdl->ev_fork, st));
        TCK(cudaStreamWaitEvent(st2, mdl->ev_fork, 0));
    };
    auto join = [&] {  // st waits for st2's work so far
        TCK(cudaEventRecord(mdl->ev_join, st2));
        TCK(cudaStreamWaitEvent(st, mdl->ev_join, 0));
    };
    uint32_t lL = 0, lLs = 0;
    while ((1ull << lL) < L) ++lL;
    while ((1ull << lLs) < Ls) ++lLs;
    TCK(cudaEventRecord(mdl->ev0, st));
    // ---- edge biases (toy_net.cpp:367-415) depend on the frame only: on st2, beside the encoder
    fork();
    k_tn_leaf_bias<<<unsigned(lay.k), 256, 0, st2>>>(
        g, lL, d_order, d_ro, d_ci, d_v, mdl->le, leaf_bias);
    TCK(cudaEventRecord(mdl->ev_lbias, st2));  // the leaf attention waits for this one only
    if (lay.m) {
        if (pyr) {
            auto* pos = mdl->buf<double>(33, n * 2);
            auto* ppos = mdl->buf<double>(34, std::max<uint64_t>(pyr_rows, 1) * 2);
            PyrLevels<double> Pp{};
            uint64_t off = 0;
            for (uint32_t l = 0; l < nlev && l < 24; ++l) {
                Pp.lev[l] = ppos + off * 2;
                off += n / (uint64_t(c0) << l);
            }
            k_tn_positions<<<nb, 256, 0, st2>>>(g, d_order, pos);
            build_pyramid(st2, pos, 2u, Pp);
            k_tn_tile_pos_pyr<<<unsigned(lay.m), 64, 0, st2>>>(g, Pp, lev_shift, tile_pos);
        } else {
            k_tn_tile_pos<<<dim3(unsigned(lay.m), 2), 256, 0, st2>>>(g, d_order, tile_pos);
        }
        k_tn_tile_bias<<<dim3(unsigned(lay.m), unsigned(Ls)), 64, 0, st2>>>(
            g, tile_pos, d_ro, d_ci, d_v, mdl->te, tile_bias);
    }
    TCK(cudaGetLastError());
    // ---- encoder (toy_net.cpp:295-318); the last residual update also writes LN(x) -------------
    k_tn_features<<<nb, 256, 0, st>>>(g, d_order, d_rho, d_ro, d_ci, d_glob, feat);
    pgemm1<128>(st, feat, n, g.feat_pad, g.feat_pad, mdl->w_enc1, d, g.feat_pad, EpiStore<true>{h1, uint32_t(d), nullptr});
    pgemm1<128>(st, h1, n, d, d, mdl->w_enc2, d, d, EpiStore<false>{x, uint32_t(d), nullptr});
    for (size_t gi = 0; gi < mdl->w_gcn.size(); ++gi) {
        k_tn_gcn_msg<<<nw, 256, 0, st>>>(g, d_ro, d_ci, d_v, d_diag, x, h1);
        if (gi + 1 < mdl->w_gcn.size())
            pgemm1<128>(st, h1, n, d, d, mdl->w_gcn[gi], d, d, EpiResidual<true>{x, uint32_t(d), nullptr});
        else
            pgemm1<128>(st, h1, n, d, d, mdl->w_gcn[gi], d, d, EpiResidualLN{x, ln, 1});
    }
    if (mdl->w_gcn.empty()) k_tn_layernorm<<<nw, 256, 0, st>>>(n, uint32_t(d), x, ln, uint32_t(d));
    TCK(cudaGetLastError());
    // ---- tile tokens, edge biases ------------------------------------------------------------
    if (lay.m) {
        if (pyr) {
            build_pyramid(st, x, uint32_t(d), Pr);  // embedding pyramid (pyr_r is reused per layer below)
            k_tn_tile_pool_pyr<<<unsigned((MT * 32 + 255) / 256), 256, 0, st>>>(g, Pr, lev_shift, tile_tok);
        } else {
            k_tn_tile_pool<<<dim3(unsigned(lay.m), unsigned(Ls)), 128, 0, st>>>(g, x, tile_tok);
        }
        k_tn_layernorm<<<unsigned((MT * 32 + 255) / 256), 256, 0, st>>>(MT, uint32_t(d), tile_tok, ln_t, uint32_t(d));
    }
    // the leaf stream's first attention needs the leaf biases; the tile biases stay queued on
    // st2 ahead of the tile stream's attention
    TCK(cudaStreamWaitEvent(st, mdl->ev_lbias, 0));

    // attention sublayer (toy_net.cpp:78-125) on `rows` tokens in windows of T; lnbuf holds
    // LN(tok) on entry and LN(tok + attention) on exit (fused into the O-projection epilogue)
    auto attention = [&](cudaStream_t st, float* tok, float* lnbuf, uint64_t rows, uint64_t T, const LW& lw,
                         const __half* bias, float* qkv, float* hout) {
        pgemm1<128>(st, lnbuf, rows, d, d, lw.qkv, 3 * d, d, EpiStore<false>{qkv, uint32_t(3 * d), nullptr});
        const uint64_t nwin = rows / T;
        if (T == 128 || T == 32) {  // tensor cores (attention_tcgen05.cuh)
            static bool configured = false;
            if (!configured) {
                TCK(cudaFuncSetAttribute(k_tn_attn_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(att_smem_bytes())));
                TCK(cudaFuncSetAttribute(k_tn_attn_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(att_smem_bytes())));
                configured = true;
            }
            const unsigned groups = unsigned((rows + kAttRows - 1) / kAttRows);
            if (T == 128)
                k_tn_attn_tc<128><<<groups, att_threads<128>(), att_smem_bytes(), st>>>(nwin, qkv, bias, hout, rowsum_bits);
            else
                k_tn_attn_tc<32><<<groups, att_threads<32>(), att_smem_bytes(), st>>>(nwin, qkv, bias, hout, rowsum_bits);
        } else {
            const dim3 grid(unsigned(nwin), unsigned(cfg.heads));
            switch (T) {
                case 64: k_tn_attention<64><<<grid, 64, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
                case 16: k_tn_attention<16><<<grid, 16, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
                case 8: k_tn_attention<8><<<grid, 8, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
                case 4: k_tn_attention<4><<<grid, 4, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
                default: throw InvalidArgument("toynet (gpu): unsupported attention window");
            }
        }
        TCK(cudaGetLastError());
        pgemm1<128>(st, hout, rows, d, d, lw.wo, d, d, EpiResidualLN{tok, lnbuf, 0});
    };
    // FFN sublayer (toy_net.cpp:421-436) on [LN(t) | r | c | glob]: K-sliced over the three
    // buffers (no concatenated input), the glob slice folded into the bias (k_tn_glob_bias);
    // the second GEMM's epilogue adds the residual and writes LN of the result
    auto ffn = [&](cudaStream_t st, float* tok, float* lnbuf, const float* r, const float* c, uint64_t rows,
                   const LW& lw, const float* bias, float* Hf) {
        pgemm<256>(st, make_pga({ASrc{lnbuf, d, d}, ASrc{r, d, d}, ASrc{c, d, d}}, rows), rows, 3 * d, lw.f1, 4 * d,
                   4 * d, EpiStore<true>{Hf, uint32_t(4 * d), bias});
        pgemm1<128>(st, Hf, rows, 4 * d, 4 * d, lw.f2, d, 4 * d, EpiResidualLN{tok, lnbuf, 0});
    };

    for (uint64_t layer = 0; layer < cfg.layers; ++layer) {
        // the two attention sublayers touch disjoint tokens: leaf on st, tile on st2
        fork();
        attention(st, x, ln, n, L, wl[layer], leaf_bias, qkv, hout);
        if (lay.m) attention(st2, tile_tok, ln_t, MT, Ls, wt[layer], tile_bias, qkv_t, hout_t);
        join();
        if (pyr) {  // scatter + the leaf tokens' glob partials in one pass
            k_tn_highway_chunks<<<hw_blocks, 256, 0, st>>>(g, c0, x, tile_tok, row_hw, col_hw, partial);
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(MT, uint32_t(d), tile_tok, partial + uint64_t(hw_blocks) * d);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(hw_blocks + nparts, uint32_t(d), partial, glob_hw);
        } else {
            k_tn_highway<<<nw, 256, 0, st>>>(g, x, tile_tok, row_hw, col_hw);
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(n, uint32_t(d), x, partial);
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(MT, uint32_t(d), tile_tok, partial + nparts * d);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(2 * nparts, uint32_t(d), partial, glob_hw);
        }
        k_tn_glob_bias<<<dim3(unsigned((4 * d * 32 + 255) / 256), 2), 256, 0, st>>>(uint32_t(d), glob_hw, wl[layer].f1,
                                                                                  wt[layer].f1, b1, b1 + 4 * d);
        TCK(cudaGetLastError());
        if (audit) {  // highway conservation audit (toy_net.cpp:478-512), on device
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(n, uint32_t(d), row_hw, audit_part);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(nparts, uint32_t(d), audit_part, audit_sums);
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(n, uint32_t(d), col_hw, audit_part);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(nparts, uint32_t(d), audit_part, audit_sums + d);
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(n, uint32_t(d), x, audit_part);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(nparts, uint32_t(d), audit_part, audit_sums + 2 * d);
            k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(MT, uint32_t(d), tile_tok, audit_part);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(nparts, uint32_t(d), audit_part, audit_sums + 3 * d);
            k_tn_colsum_tiles_weighted<<<nparts, unsigned(d), 0, st>>>(g, tile_tok, audit_part);
            k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(nparts, uint32_t(d), audit_part, audit_sums + 4 * d);
            TCK(cudaMemcpyAsync(audit_sums + 5 * d, glob_hw, d * 4, cudaMemcpyDeviceToDevice, st));
            k_tn_highway_audit<<<1, unsigned(d), 0, st>>>(uint32_t(d), audit_sums, audit_dev + layer);
            TCK(cudaGetLastError());
        }
        // FFN sublayers: leaf on st; the tile FFN's strip means + FFN on st2 (both only read
        // row_hw / col_hw; the next layer's scatter joins them first)
        fork();
        ffn(st, x, ln, row_hw, col_hw, n, wl[layer], b1, Hf);
        if (lay.m) {
            if (pyr) {
                build_pyramid(st2, row_hw, uint32_t(d), Pr);
                build_pyramid(st2, col_hw, uint32_t(d), Pc);
                k_tn_tile_means_pyr<<<unsigned((MT * 32 + 255) / 256), 256, 0, st2>>>(g, Pr, Pc, lev_shift, rmean, cmean);
            } else {
                k_tn_tile_means_walk<<<dim3(unsigned(lay.m), unsigned(Ls)), 128, 0, st2>>>(g, row_hw, col_hw, rmean, cmean);
            }
            TCK(cudaGetLastError());
            ffn(st2, tile_tok, ln_t, rmean, cmean, MT, wt[layer], b1 + 4 * d, Hf_t);
        }
        join();
    }

    // ---- decoder heads into the packed layout (toy_net.cpp:540-585) ------------------------
    pgemm1<128>(st, x, n, d, d, mdl->w_lh1, d, d, EpiStore<true>{h1, uint32_t(d), nullptr});
    // F_k rows: leaf_factor(k) + r L = (k L + r) L = i L -> a row-major [n x L] section
    pgemm1<128>(st, h1, n, d, d, mdl->w_lh2, L, d, EpiStore<false>{out, uint32_t(L), nullptr});
    pgemm1<80>(st, x, n, d, d, mdl->w_heads, 2 * Ls + 1, d, EpiLeafHeads{out, lL, lLs, lay.bridge_base, lay.gate_base});
    if (lay.m) pgemm1<32>(st, tile_tok, MT, d, d, mdl->w_theads, Ls, d, EpiTileHeads{out, lLs, lay.tile_base});
    join();  // nothing of this forward is left on st2
    TCK(cudaEventRecord(mdl->ev1, st));
    TCK(cudaStreamSynchronize(st));

    if (trace) {
        if (audit) {
            unsigned int bits = 0;
            TCK(cudaMemcpy(&bits, rowsum_bits, 4, cudaMemcpyDeviceToHost));
            float e;
            std::memcpy(&e, &bits, 4);
            trace->max_attention_row_sum_error = e;
            std::vector<float> hw(cfg.layers, 0.f);
            TCK(cudaMemcpy(hw.data(), audit_dev, cfg.layers * 4, cudaMemcpyDeviceToHost));
            trace->highway_max_deviation = hw.empty() ? 0.0 : *std::max_element(hw.begin(), hw.end());
        }
        trace->leaf_attention_dispatches = cfg.layers;
        trace->tile_attention_dispatches = lay.m ? cfg.layers : 0;
        float dev_ms = 0.f;
        TCK(cudaEventElapsedTime(&dev_ms, mdl->ev0, mdl->ev1));
        trace->ms = dev_ms;  // device time of the forward (all kernels, excl. host setup)
    }
}

// Full forward for one frame: writes the packed factor tensor (device pointer out).
void toynet_forward_device(ToynetModel* mdl, cudaStream_t st, const hfpg_frame_view& fr, float* out,
                           hfpg_toynet_trace* trace) {
    const hfpg_toynet_config& cfg = mdl->cfg;
    const uint64_t L = mdl->L, Ls = mdl->Ls;
    const Layout lay = make_layout(fr.n, L, Ls);
    const uint64_t n = fr.n, d = cfg.d;

    // ---- glob stats on the host, f64 in the reference's order (toy_net.cpp:232-268) --------
    std::vector<double> diag(n, 0.0);
    double rho_mean = 0.0, rho_var = 0.0, dmean = 0.0, offmean = 0.0;
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t p = fr.row_offsets[i]; p < fr.row_offsets[i + 1]; ++p)
            if (fr.col_indices[p] == i) diag[i] = fr.values[p];
    for (uint64_t i = 0; i < n; ++i) rho_mean += fr.rho[i];
    rho_mean /= double(n);
    for (uint64_t i = 0; i < n; ++i) rho_var += (fr.rho[i] - rho_mean) * (fr.rho[i] - rho_mean);
    rho_var /= double(n);
    double dmin = diag[0], dmax = diag[0];
    for (uint64_t i = 0; i < n; ++i) {
        dmean += diag[i];
        dmin = std::min(dmin, diag[i]);
        dmax = std::max(dmax, diag[i]);
        for (uint64_t p = fr.row_offsets[i]; p < fr.row_offsets[i + 1]; ++p)
            if (fr.col_indices[p] != i) {
                offmean += std::fabs(fr.values[p]);
                ++off;
            }
    }
    dmean /= double(n);
    if (off) offmean /= double(off);
    const double stats[12] = {std::log(double(n)), rho_mean, std::sqrt(rho_var),
                              std::log(std::max(fr.rho_heavy, 1.0)), dmean, dmax, dmin, offmean,
                              double(fr.row_offsets[n]) / double(n),
                              double(fr.width) / double(fr.height), dmax / std::max(dmin, 1e-30), 1.0};
    std::vector<float> glob(std::max<uint64_t>(cfg.d_global, 1), 0.f);
    for (uint64_t i = 0; i < cfg.d_global && i < 12; ++i) glob[i] = float(stats[i]);

    // ---- inputs ------------------------------------------------------------------------------
    const uint64_t nnz = fr.row_offsets[n];
    auto* d_order = mdl->buf<uint32_t>(21, n);
    auto* d_rho = mdl->buf<double>(0, n);
    auto* d_ro = mdl->buf<unsigned long long>(1, n + 1);
    auto* d_ci = mdl->buf<uint32_t>(22, nnz);
    auto* d_v = mdl->buf<double>(2, nnz);
    auto* d_diag = mdl->buf<double>(3, n);
    auto* d_glob = mdl->buf<float>(4, glob.size());
    TCK(cudaMemcpyAsync(d_order, fr.cell_order, n * 4, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(d_rho, fr.rho, n * 8, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(d_ro, fr.row_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(d_ci, fr.col_indices, nnz * 4, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(d_v, fr.values, nnz * 8, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(d_diag, diag.data(), n * 8, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(d_glob, glob.data(), glob.size() * 4, cudaMemcpyHostToDevice, st));

    toynet_run(mdl, st, n, fr.width, fr.height, nnz, d_order, d_rho, d_ro, d_ci, d_v, d_diag, d_glob, out, trace);
}

// The same forward from a frame already on the device (the GPU frame generator): the global
// statistics (toy_net.cpp:232-268) are reduced on the device (k_tn_frame_stats, fixed-order
// partial sums — float features, so the order does not matter at the 1e-5 parity bar).
void toynet_forward_device_frame(ToynetModel* mdl, cudaStream_t st, const ToynetDeviceFrame& f, float* out,
                                 hfpg_toynet_trace* trace) {
    const hfpg_toynet_config& cfg = mdl->cfg;
    const uint64_t nglob = std::max<uint64_t>(cfg.d_global, 1);
    auto* d_glob = mdl->buf<float>(4, nglob);
    auto* part = mdl->buf<double>(27, uint64_t(kStatParts) * kStatFields);
    k_tn_frame_stats<<<kStatParts, 256, 0, st>>>(f.n, f.rho, f.ro, f.ci, f.v, f.diag, part);
    k_tn_frame_var<<<kStatParts, 256, 0, st>>>(f.n, f.rho, part);
    k_tn_frame_finish<<<1, 32, 0, st>>>(f.n, f.nnz, f.width, f.height, f.rho_heavy, part,
                                        uint32_t(cfg.d_global), d_glob);
    TCK(cudaGetLastError());
    toynet_run(mdl, st, f.n, f.width, f.height, f.nnz, f.order, f.rho, f.ro, f.ci, f.v, f.diag, d_glob, out, trace);
}

}  // namespace hfpg

extern "C" int hfpg_gemm_tf32(uint64_t M, uint64_t N, uint64_t K, const float* A, const float* Bt,
                              float* C) {
    using namespace hfpg;
    return guarded([&] {
        if (K % 4 || N % 4) throw InvalidArgument("gemm: K and N must be multiples of 4 (16-byte rows)");
        float *dA = nullptr, *dB = nullptr, *dC = nullptr;
        TCK(cudaMalloc(&dA, std::max<uint64_t>(M * K, 1) * 4));
        TCK(cudaMalloc(&dB, std::max<uint64_t>(N * K, 1) * 4));
        TCK(cudaMalloc(&dC, std::max<uint64_t>(M * N, 1) * 4));
        TCK(cudaMemcpy(dA, A, M * K * 4, cudaMemcpyHostToDevice));
        TCK(cudaMemcpy(dB, Bt, N * K * 4, cudaMemcpyHostToDevice));
        pgemm1<128>(0, dA, M, K, K, dB, N, K, EpiStore<false>{dC, uint32_t(N), nullptr});
        TCK(cudaDeviceSynchronize());
        TCK(cudaMemcpy(C, dC, M * N * 4, cudaMemcpyDeviceToHost));
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dC);
    });
}
