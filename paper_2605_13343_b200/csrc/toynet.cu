// Toy-network inference + factor assembly on the GPU (toy_net.cpp:170-586): encoder MLP, D^-1 A
// graph convolutions, leaf-window and strip-pooled tile attention with edge biases, highway
// buffers, 4d FFNs and the decoder heads writing the packed factor tensor. Dense contractions
// run on tcgen05 (kind::tf32, TMEM accumulators, TMA-fed); the rest are fp32 SIMT kernels.
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "attention_tcgen05.cuh"
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

// ---- GEMM epilogues ---------------------------------------------------------------------------
struct EpiStore {  // out[row, col] = act(v + bias)
    float* out;
    uint32_t ld, n;
    const float* bias;
    int gelu;
    // 8 consecutive rows (row0 .. row0+7) of columns col..col+3; values at v[i * ld]
    __device__ void apply4x8(int row0, int col, const float* v, int ld, int nv) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) apply4(row0 + i, col, *reinterpret_cast<const float4*>(v + i * ld), nv);
    }
    __device__ void apply4(int row, int col, float4 v, int nv) const {
        float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] += (bias && j < nv) ? bias[col + j] : 0.f;
            if (gelu) x[j] = gelu_f(x[j]);
        }
        float* o = out + uint64_t(row) * ld + col;
        if (nv == 4 && (ld & 3) == 0) {
            *reinterpret_cast<float4*>(o) = make_float4(x[0], x[1], x[2], x[3]);
        } else {
            for (int j = 0; j < nv; ++j) o[j] = x[j];
        }
    }
};
struct EpiResidual {  // out[row, col] += act(v + bias)
    float* out;
    uint32_t ld, n;
    const float* bias;
    int gelu;
    // 8 rows at once: all residual reads issued before the writes
    __device__ void apply4x8(int row0, int col, const float* v, int ldv, int nv) const {
        if (nv != 4 || (ld & 3) != 0) {
            for (int i = 0; i < 8; ++i) apply4(row0 + i, col, *reinterpret_cast<const float4*>(v + i * ldv), nv);
            return;
        }
        float4 a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4*>(out + uint64_t(row0 + i) * ld + col);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float4 t = *reinterpret_cast<const float4*>(v + i * ldv);
            float x[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                x[j] += bias ? bias[col + j] : 0.f;
                if (gelu) x[j] = gelu_f(x[j]);
            }
            a[i].x += x[0]; a[i].y += x[1]; a[i].z += x[2]; a[i].w += x[3];
            *reinterpret_cast<float4*>(out + uint64_t(row0 + i) * ld + col) = a[i];
        }
    }
    __device__ void apply4(int row, int col, float4 v, int nv) const {
        float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] += (bias && j < nv) ? bias[col + j] : 0.f;
            if (gelu) x[j] = gelu_f(x[j]);
        }
        float* o = out + uint64_t(row) * ld + col;
        if (nv == 4 && (ld & 3) == 0) {
            float4 a = *reinterpret_cast<float4*>(o);
            a.x += x[0]; a.y += x[1]; a.z += x[2]; a.w += x[3];
            *reinterpret_cast<float4*>(o) = a;
        } else {
            for (int j = 0; j < nv; ++j) o[j] += x[j];
        }
    }
};
// Decoder heads of leaf node `row` (toy_net.cpp:549-567): columns [0, L_s) -> Ũ_k row,
// [L_s, 2 L_s) -> Ṽ_k row, 2 L_s -> gate. Cast to float as the reference does.
struct EpiLeafHeads {
    float* out;
    uint64_t L, Ls, bridge_base, gate_base;
    const float* bias;  // 2 Ls + 1
    // 8 consecutive rows (row0 .. row0+7) of columns col..col+3; values at v[i * ld]
    __device__ void apply4x8(int row0, int col, const float* v, int ld, int nv) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) apply4(row0 + i, col, *reinterpret_cast<const float4*>(v + i * ld), nv);
    }
    __device__ void apply4(int row, int col, float4 v, int nv) const {
        const uint64_t k = uint64_t(row) / L, r = uint64_t(row) % L;
        const float vv[4] = {v.x, v.y, v.z, v.w};
        for (int j = 0; j < nv; ++j) {
            const uint64_t c = uint64_t(col + j);
            const float x = vv[j] + (bias && c <= 2 * Ls ? bias[c] : 0.f);
            if (c < Ls) out[bridge_base + k * 2 * L * Ls + r * Ls + c] = x;
            else if (c < 2 * Ls) out[bridge_base + k * 2 * L * Ls + L * Ls + r * Ls + (c - Ls)] = x;
            else if (c == 2 * Ls) out[gate_base + uint64_t(row)] = x;
        }
    }
};
// Tile heads of tile token `row` = m L_s + tok (toy_net.cpp:570-584): [0, rk) -> U_m[tok],
// [rk, 2 rk) -> V_m[tok].
struct EpiTileHeads {
    float* out;
    uint64_t Ls, rk, tile_base;
    const float* bias;
    // 8 consecutive rows (row0 .. row0+7) of columns col..col+3; values at v[i * ld]
    __device__ void apply4x8(int row0, int col, const float* v, int ld, int nv) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) apply4(row0 + i, col, *reinterpret_cast<const float4*>(v + i * ld), nv);
    }
    __device__ void apply4(int row, int col, float4 v, int nv) const {
        const uint64_t m = uint64_t(row) / Ls, tok = uint64_t(row) % Ls;
        const float vv[4] = {v.x, v.y, v.z, v.w};
        for (int j = 0; j < nv; ++j) {
            const uint64_t c = uint64_t(col + j);
            if (c >= 2 * rk) continue;
            const float x = vv[j] + (bias ? bias[c] : 0.f);
            out[tile_base + m * Ls * Ls + (c < rk ? 0 : Ls * rk) + tok * rk + (c % rk)] = x;
        }
    }
};

template <int BN, class Epi>
void gemm(cudaStream_t st, const float* A, uint64_t M, uint64_t K, uint64_t lda, const float* Bt,
          uint64_t N, uint64_t ldb, const Epi& epi) {
    static bool configured = false;
    if (!configured) {
        TCK(cudaFuncSetAttribute(k_gemm_tf32<BN, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(gemm_smem_bytes<BN>())));
        configured = true;
    }
    if (M == 0 || N == 0) return;
    const CUtensorMap ta = tmap(A, M, K, lda, kGemmBM), tb = tmap(Bt, N, K, ldb, BN);
    dim3 grid(unsigned((M + kGemmBM - 1) / kGemmBM), unsigned((N + BN - 1) / BN));
    k_gemm_tf32<BN, Epi><<<grid, kGemmThreads, gemm_smem_bytes<BN>(), st>>>(ta, tb, int(M), int(N), int(K), epi);
    TCK(cudaGetLastError());
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
    ~ToynetModel() {
        for (float* p : wbuf) cudaFree(p);
        for (auto& b : scratch) cudaFree(b.first);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
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
    // ---- activations -------------------------------------------------------------------------
    auto* feat = mdl->buf<float>(5, n * g.feat_pad);
    auto* x = mdl->buf<float>(6, n * d);       // embedding -> leaf tokens
    auto* h1 = mdl->buf<float>(7, n * d);      // encoder hidden / gcn message / decoder hidden
    auto* tile_tok = mdl->buf<float>(8, MT * d);
    auto* ln = mdl->buf<float>(9, std::max(n, MT) * d);
    auto* qkv = mdl->buf<float>(10, std::max(n, MT) * 3 * d);
    auto* hout = mdl->buf<float>(11, std::max(n, MT) * d);
    auto* row_hw = mdl->buf<float>(12, n * d);
    auto* col_hw = mdl->buf<float>(13, n * d);
    auto* Af = mdl->buf<float>(14, std::max(n, MT) * 4 * d);
    auto* Hf = mdl->buf<float>(15, std::max(n, MT) * 4 * d);
    auto* glob_hw = mdl->buf<float>(16, d);
    const uint32_t nparts = 296;
    auto* partial = mdl->buf<float>(17, uint64_t(nparts) * 2 * d);
    auto* leaf_bias = mdl->buf<float>(18, lay.k * cfg.heads * L * L);
    auto* tile_bias = mdl->buf<float>(19, lay.m * cfg.heads * Ls * Ls);
    auto* tile_pos = mdl->buf<double>(26, std::max<uint64_t>(lay.m, 1) * 2 * Ls * 2);
    unsigned int* rowsum_bits = trace ? mdl->buf<unsigned int>(20, 1) : nullptr;
    float* audit_part = trace ? mdl->buf<float>(23, uint64_t(nparts) * d) : nullptr;
    float* audit_sums = trace ? mdl->buf<float>(24, 6 * d) : nullptr;
    float* audit_dev = trace ? mdl->buf<float>(25, cfg.layers) : nullptr;
    if (rowsum_bits) TCK(cudaMemsetAsync(rowsum_bits, 0, 4, st));

    const unsigned nb = unsigned((n + 255) / 256), nw = unsigned((n * 32 + 255) / 256);
    TCK(cudaEventRecord(mdl->ev0, st));
    // ---- encoder (toy_net.cpp:295-318) -----------------------------------------------------
    k_tn_features<<<nb, 256, 0, st>>>(g, d_order, d_rho, d_ro, d_ci, d_glob, feat);
    gemm<128>(st, feat, n, g.feat_pad, g.feat_pad, mdl->w_enc1, d, g.feat_pad, EpiStore{h1, uint32_t(d), uint32_t(d), nullptr, 1});
    gemm<128>(st, h1, n, d, d, mdl->w_enc2, d, d, EpiStore{x, uint32_t(d), uint32_t(d), nullptr, 0});
    for (float* wg : mdl->w_gcn) {
        k_tn_gcn_msg<<<nw, 256, 0, st>>>(g, d_ro, d_ci, d_v, d_diag, x, h1);
        gemm<128>(st, h1, n, d, d, wg, d, d, EpiResidual{x, uint32_t(d), uint32_t(d), nullptr, 1});
    }
    TCK(cudaGetLastError());
    // ---- tile tokens, edge biases ------------------------------------------------------------
    if (lay.m) k_tn_tile_pool<<<dim3(unsigned(lay.m), unsigned(Ls)), 128, 0, st>>>(g, x, tile_tok);
    k_tn_leaf_bias<<<dim3(unsigned((L * L + 255) / 256), unsigned(lay.k)), 256, 0, st>>>(
        g, d_order, d_ro, d_ci, d_v, mdl->le, leaf_bias);
    if (lay.m) {
        k_tn_tile_pos<<<dim3(unsigned(lay.m), 2), 256, 0, st>>>(g, d_order, tile_pos);
        k_tn_tile_bias<<<dim3(unsigned(lay.m), unsigned(Ls)), 64, 0, st>>>(
            g, tile_pos, d_ro, d_ci, d_v, mdl->te, tile_bias);
    }
    TCK(cudaGetLastError());

    auto attention = [&](float* tok, uint64_t rows, uint64_t T, const LW& lw, const float* bias) {
        k_tn_layernorm<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(rows, uint32_t(d), tok, ln, uint32_t(d));
        gemm<128>(st, ln, rows, d, d, lw.qkv, 3 * d, d, EpiStore{qkv, uint32_t(3 * d), uint32_t(3 * d), nullptr, 0});
        const dim3 grid(unsigned(rows / T), unsigned(cfg.heads));
        static const bool simt128 = std::getenv("HFPG_ATTENTION_SIMT") != nullptr;  // A/B checks only
        if (T == 128 && !simt128) {  // tensor-core path (attention_tcgen05.cuh)
            static bool configured = false;
            if (!configured) {
                TCK(cudaFuncSetAttribute(k_tn_attention_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(att_smem_bytes())));
                configured = true;
            }
            k_tn_attention_tc<<<unsigned(rows / T), kAttThreads, att_smem_bytes(), st>>>(
                uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits);
            TCK(cudaGetLastError());
            gemm<128>(st, hout, rows, d, d, lw.wo, d, d, EpiResidual{tok, uint32_t(d), uint32_t(d), nullptr, 0});
            return;
        }
        switch (T) {
            case 128: k_tn_attention<128><<<grid, 128, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
            case 64: k_tn_attention<64><<<grid, 64, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
            case 32: k_tn_attention<32><<<grid, 32, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
            case 16: k_tn_attention<16><<<grid, 16, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
            case 8: k_tn_attention<8><<<grid, 8, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
            case 4: k_tn_attention<4><<<grid, 4, 0, st>>>(uint32_t(d), uint32_t(cfg.heads), qkv, bias, hout, rowsum_bits); break;
            default: throw InvalidArgument("toynet (gpu): unsupported attention window");
        }
        TCK(cudaGetLastError());
        gemm<128>(st, hout, rows, d, d, lw.wo, d, d, EpiResidual{tok, uint32_t(d), uint32_t(d), nullptr, 0});
    };
    auto ffn = [&](float* tok, uint64_t rows, const LW& lw, bool leaf) {
        k_tn_layernorm<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(rows, uint32_t(d), tok, Af, uint32_t(4 * d));
        if (leaf)
            k_tn_ffn_input_leaf<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(g, row_hw, col_hw, glob_hw, Af);
        else
            k_tn_ffn_input_tile<<<dim3(unsigned(lay.m), unsigned(Ls)), 128, 0, st>>>(g, row_hw, col_hw, glob_hw, Af);
        TCK(cudaGetLastError());
        gemm<128>(st, Af, rows, 4 * d, 4 * d, lw.f1, 4 * d, 4 * d, EpiStore{Hf, uint32_t(4 * d), uint32_t(4 * d), nullptr, 1});
        gemm<128>(st, Hf, rows, 4 * d, 4 * d, lw.f2, d, 4 * d, EpiResidual{tok, uint32_t(d), uint32_t(d), nullptr, 0});
    };

    for (uint64_t layer = 0; layer < cfg.layers; ++layer) {
        attention(x, n, L, wl[layer], leaf_bias);
        if (lay.m) attention(tile_tok, MT, Ls, wt[layer], tile_bias);
        k_tn_highway<<<nw, 256, 0, st>>>(g, x, tile_tok, row_hw, col_hw);
        k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(n, uint32_t(d), x, partial);
        k_tn_colsum_partial<<<nparts, unsigned(d), 0, st>>>(MT, uint32_t(d), tile_tok, partial + nparts * d);
        k_tn_colsum_finish<<<unsigned(d), 32, 0, st>>>(2 * nparts, uint32_t(d), partial, glob_hw);
        TCK(cudaGetLastError());
        if (trace) {  // highway conservation audit (toy_net.cpp:478-512), on device
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
        ffn(x, n, wl[layer], true);
        if (lay.m) ffn(tile_tok, MT, wt[layer], false);
    }

    // ---- decoder heads into the packed layout (toy_net.cpp:540-585) ------------------------
    gemm<128>(st, x, n, d, d, mdl->w_lh1, d, d, EpiStore{h1, uint32_t(d), uint32_t(d), nullptr, 1});
    // F_k rows: leaf_factor(k) + r L = (k L + r) L = i L -> a row-major [n x L] section
    gemm<128>(st, h1, n, d, d, mdl->w_lh2, L, d, EpiStore{out, uint32_t(L), uint32_t(L), nullptr, 0});
    gemm<80>(st, x, n, d, d, mdl->w_heads, 2 * Ls + 1, d,
             EpiLeafHeads{out, L, Ls, lay.bridge_base, lay.gate_base, nullptr});
    if (lay.m) gemm<32>(st, tile_tok, MT, d, d, mdl->w_theads, Ls, d, EpiTileHeads{out, Ls, Ls / 2, lay.tile_base, nullptr});
    TCK(cudaEventRecord(mdl->ev1, st));
    TCK(cudaStreamSynchronize(st));

    if (trace) {
        unsigned int bits = 0;
        TCK(cudaMemcpy(&bits, rowsum_bits, 4, cudaMemcpyDeviceToHost));
        float e;
        std::memcpy(&e, &bits, 4);
        trace->max_attention_row_sum_error = e;
        std::vector<float> hw(cfg.layers, 0.f);
        TCK(cudaMemcpy(hw.data(), audit_dev, cfg.layers * 4, cudaMemcpyDeviceToHost));
        trace->highway_max_deviation = hw.empty() ? 0.0 : *std::max_element(hw.begin(), hw.end());
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
        if (K % 4) throw InvalidArgument("gemm: K must be a multiple of 4 (16-byte rows)");
        float *dA = nullptr, *dB = nullptr, *dC = nullptr;
        TCK(cudaMalloc(&dA, std::max<uint64_t>(M * K, 1) * 4));
        TCK(cudaMalloc(&dB, std::max<uint64_t>(N * K, 1) * 4));
        TCK(cudaMalloc(&dC, std::max<uint64_t>(M * N, 1) * 4));
        TCK(cudaMemcpy(dA, A, M * K * 4, cudaMemcpyHostToDevice));
        TCK(cudaMemcpy(dB, Bt, N * K * 4, cudaMemcpyHostToDevice));
        gemm<128>(0, dA, M, K, K, dB, N, K, EpiStore{dC, uint32_t(N), uint32_t(N), nullptr, 0});
        TCK(cudaDeviceSynchronize());
        TCK(cudaMemcpy(C, dC, M * N * 4, cudaMemcpyDeviceToHost));
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dC);
    });
}
