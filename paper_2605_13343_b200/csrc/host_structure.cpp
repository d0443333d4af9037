// Host-side structure of the path: partition + packed layout (partition.cpp, factor_tensor.cpp),
// seeded factor initialisation (factor_tensor.cpp:30-39), HFTC model files (checkpoint.cpp)
// and the synthetic pressure-Poisson frames that feed the solve (frame.cpp, plus a 3D variant).
// Native C++, multi-threaded where the reference is a sequential loop over a counter-based
// stream, and bit-identical to it (tests/test_host.py pins this against oracle/_ref).
#include "internal.hpp"
#include "crmath.cuh"

#include <zlib.h>

#include <algorithm>
#include <memory>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <thread>

namespace hfpg {

// ---- partition.cpp:9-15 preconditions ----------------------------------------------------
void check_partition(uint64_t n, uint64_t leaf) {
    if (leaf == 0 || n % leaf != 0)
        throw InvalidArgument("build_partition: leaf size must divide N");
    const uint64_t k = n / leaf;
    if (k < 2 || (k & (k - 1)) != 0)
        throw InvalidArgument("build_partition: leaf count must be a power of two >= 2");
}

// factor_tensor.cpp:7-28: sections [F_k | (U_m|V_m) | (Ũ_k|Ṽ_k) | gate]
Layout make_layout(uint64_t n, uint64_t leaf, uint64_t ls) {
    check_partition(n, leaf);
    if (ls == 0 || leaf % ls != 0)
        throw InvalidArgument("factor layout: coarse size must divide leaf size");
    if (ls % 2 != 0) throw InvalidArgument("factor layout: coarse size must be even");
    Layout L;
    L.n = n;
    L.l = leaf;
    L.ls = ls;
    L.rk = ls / 2;
    L.k = n / leaf;
    L.m = L.k - 1;
    while ((1ULL << L.depth) < L.k) ++L.depth;
    L.tile_base = L.k * leaf * leaf;
    L.bridge_base = L.tile_base + L.m * ls * ls;
    L.gate_base = L.bridge_base + 2 * n * ls;
    L.total = L.gate_base + n;
    return L;
}

hfpg_layout to_c(const Layout& L) {
    hfpg_layout o;
    o.n = L.n;
    o.leaf_size = L.l;
    o.coarse_size = L.ls;
    o.coupling_rank = L.rk;
    o.leaf_count = L.k;
    o.tile_count = L.m;
    o.leaf_base = 0;
    o.tile_base = L.tile_base;
    o.bridge_base = L.bridge_base;
    o.gate_base = L.gate_base;
    o.total = L.total;
    return o;
}

// Split [0, n) over the host's threads; fn(begin, end).
template <class Fn>
static void parallel_for(uint64_t n, Fn fn, uint64_t min_chunk = 1 << 16) {
    uint64_t nt = std::max(1u, std::thread::hardware_concurrency());
    nt = std::min<uint64_t>(nt, std::max<uint64_t>(1, n / min_chunk));
    if (nt <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < nt; ++t)
        th.emplace_back([=] { fn(n * t / nt, n * (t + 1) / nt); });
    for (auto& x : th) x.join();
}

// factor_tensor.cpp:30-39: draw i of RngStream(seed, frame, factor_init) -> element i below
// the gate, as float(sigma * normal); gate = 1.
void init_factors_host(const Layout& L, double sigma, uint64_t seed, uint64_t frame,
                       float* out) {
    const Rng s(seed, frame, kFactorInit);
    parallel_for(L.gate_base, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i)
            out[i] = static_cast<float>(sigma == 0.0 ? 0.0 : sigma * Rng::normal_of(s.bits_at(i)));
    });
    for (uint64_t i = L.gate_base; i < L.total; ++i) out[i] = 1.0f;
}

// ---- frame.cpp ------------------------------------------------------------------------------
static uint32_t spread2(uint32_t v) {  // morton.hpp:13-20
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
static uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
    v &= 0x1FFFFFULL;
    v = (v | (v << 32)) & 0x1F00000000FFFFULL;
    v = (v | (v << 16)) & 0x1F0000FF0000FFULL;
    v = (v | (v << 8)) & 0x100F00F00F00F00FULL;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ULL;
    v = (v | (v << 2)) & 0x1249249249249249ULL;
    return v;
}

// frame.cpp:60-79 in_heavy_region, generalised to an axis triple (2D: cross/along = x|y).
static bool heavy_at(double cross, double along, const FrameBarrier& b) {
    if (std::fabs(cross - b.center) > 0.5 * b.thickness) return false;
    switch (b.gap) {
        case 0: return along < 0.8;
        case 1: return along > 0.2;
        case 2: return along < 0.4 || along > 0.6;
        default: return true;
    }
}

// frame.cpp:81-98 sample_density: rho_heavy ~ loguniform[5,100], 1-3 barriers.
static std::vector<FrameBarrier> sample_barriers(Rng& s, uint64_t n_axes, double& rho_heavy) {
    rho_heavy = std::exp(s.uniform(std::log(5.0), std::log(100.0)));
    const uint64_t nb = 1 + s.below(3);
    std::vector<FrameBarrier> bars;
    for (uint64_t i = 0; i < nb; ++i) {
        FrameBarrier b;
        b.axis = s.below(n_axes);
        b.center = s.uniform(0.2, 0.8);
        b.thickness = s.uniform(0.05, 0.20);
        b.gap = s.below(4);
        bars.push_back(b);
    }
    return bars;
}

bool frame_crmath() {
    const char* e = std::getenv("HFPG_FRAME_CRMATH");
    return e && e[0] == '1';
}
static double frame_normal(bool cr, uint64_t bits) {
    return cr ? crm::normal_of_cr(bits) : Rng::normal_of(bits);
}

// frame.cpp:161-166 grid_dims and the density/rhs streams of make_frame.
FrameParams frame_params_2d(uint64_t n, uint64_t seed, uint64_t fidx) {
    if (n < 4) throw InvalidArgument("grid_dims: need at least 4 cells");
    uint64_t w = static_cast<uint64_t>(std::ceil(std::sqrt(static_cast<double>(n))));
    while (w * w < n) ++w;
    const uint64_t h = (n + w - 1) / w;
    if (w >= (1u << 16) || h >= (1u << 16))
        throw InvalidArgument("morton_cell_order: grid dimension >= 2^16");
    FrameParams P;
    P.dims = 2;
    P.n = n;
    P.W = w;
    P.H = h;
    Rng s(seed, fidx, kDensity);
    P.bars = sample_barriers(s, 2, P.rho_heavy);
    P.density_key = s.key;
    P.c0 = s.counter;  // one normal per retained cell follows, in Morton order
    P.rhs_key = Rng(seed, fidx, kRhs).key;
    return P;
}

FrameParams frame_params_3d(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed, uint64_t fidx) {
    if (nx < 2 || ny < 2 || nz < 2) throw InvalidArgument("frame_3d: each dimension must be >= 2");
    if (nx > (1u << 21) || ny > (1u << 21) || nz > (1u << 21) || nx * ny * nz > (1ULL << 32))
        throw InvalidArgument("frame_3d: grid too large");
    FrameParams P;
    P.dims = 3;
    P.n = nx * ny * nz;
    P.W = nx;
    P.H = ny;
    P.D = nz;
    Rng s(seed, fidx, kDensity);
    P.bars = sample_barriers(s, 3, P.rho_heavy);
    P.density_key = s.key;
    P.c0 = s.counter;
    P.rhs_key = Rng(seed, fidx, kRhs).key;
    return P;
}

// frame.cpp:154-159 sample_rhs: normals, then b -= mean (sequential mean, :147-152).
static std::vector<double> sample_rhs(uint64_t n, uint64_t seed, uint64_t frame) {
    const Rng s(seed, frame, kRhs);
    const bool cr = frame_crmath();
    std::vector<double> b(n);
    parallel_for(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) b[i] = frame_normal(cr, s.bits_at(i));
    });
    double mean = 0.0;
    for (double v : b) mean += v;
    mean /= static_cast<double>(n);
    for (double& v : b) v -= mean;
    return b;
}

// frame.cpp:100-145 assemble_operator, generalised to 2*dims neighbours in the order
// (x-1, x+1, y-1, y+1[, z-1, z+1]); w = 2 rho_i rho_j / (rho_i + rho_j); columns sorted.
static Csr assemble(const std::vector<double>& rho, const std::vector<uint32_t>& order,
                    uint64_t W, uint64_t H, uint64_t D) {
    const uint64_t n = order.size();
    for (double r : rho)
        if (!(r > 0.0)) throw InvalidArgument("assemble_operator: density must be positive");
    std::vector<int64_t> rank_of(W * H * D, -1);
    for (uint64_t i = 0; i < n; ++i) rank_of[order[i]] = static_cast<int64_t>(i);
    const int nn = D > 1 ? 6 : 4;
    // Row lengths first (prefix sum), then fill rows in parallel.
    std::vector<uint32_t> len(n);
    auto neighbours = [&](uint64_t i, int64_t out[6]) {
        const uint64_t id = order[i];
        const int64_t x = id % W, y = (id / W) % H, z = id / (W * H);
        const int64_t c[6][3] = {{x - 1, y, z}, {x + 1, y, z}, {x, y - 1, z},
                                 {x, y + 1, z}, {x, y, z - 1}, {x, y, z + 1}};
        for (int q = 0; q < nn; ++q) {
            out[q] = -1;
            if (c[q][0] < 0 || c[q][0] >= int64_t(W) || c[q][1] < 0 || c[q][1] >= int64_t(H) ||
                c[q][2] < 0 || c[q][2] >= int64_t(D))
                continue;
            out[q] = rank_of[uint64_t(c[q][2]) * W * H + uint64_t(c[q][1]) * W + uint64_t(c[q][0])];
        }
    };
    parallel_for(n, [&](uint64_t lo, uint64_t hi) {
        int64_t nb[6];
        for (uint64_t i = lo; i < hi; ++i) {
            neighbours(i, nb);
            uint32_t c = 1;
            for (int q = 0; q < nn; ++q) c += nb[q] >= 0;
            len[i] = c;
        }
    });
    Csr A;
    A.n = n;
    A.row_offsets.resize(n + 1);
    A.row_offsets[0] = 0;
    for (uint64_t i = 0; i < n; ++i) A.row_offsets[i + 1] = A.row_offsets[i] + len[i];
    A.cols.resize(A.row_offsets[n]);
    A.vals.resize(A.row_offsets[n]);
    parallel_for(n, [&](uint64_t lo, uint64_t hi) {
        int64_t nb[6];
        std::pair<uint32_t, double> row[7];
        for (uint64_t i = lo; i < hi; ++i) {
            neighbours(i, nb);
            int cnt = 0;
            double diag = 0.0;
            for (int q = 0; q < nn; ++q) {
                if (nb[q] < 0) continue;
                const uint64_t j = uint64_t(nb[q]);
                const double w = 2.0 * rho[i] * rho[j] / (rho[i] + rho[j]);
                diag += w;
                row[cnt++] = {static_cast<uint32_t>(j), -w};
            }
            row[cnt++] = {static_cast<uint32_t>(i), diag};
            std::sort(row, row + cnt);
            for (int q = 0; q < cnt; ++q) {
                A.cols[A.row_offsets[i] + q] = row[q].first;
                A.vals[A.row_offsets[i] + q] = row[q].second;
            }
        }
    });
    return A;
}

// frame.cpp:161-181 make_frame (2D): W = ceil(sqrt N), H = ceil(N/W); Morton-sorted cells
// truncated to N; barrier density with multiplicative noise; Neumann Laplacian; projected rhs.
static hfpg_frame* frame_2d(uint64_t n, uint64_t seed, uint64_t fidx) {
    const FrameParams P = frame_params_2d(n, seed, fidx);
    const uint64_t w = P.W, h = P.H;
    auto* f = new hfpg_frame;
    f->n = n;
    f->width = w;
    f->height = h;
    f->rho_heavy = P.rho_heavy;
    f->master_seed = seed;
    f->frame_index = fidx;
    f->bars = P.bars;
    // frame.cpp:24-41: Morton codes are unique per cell, so a key sort equals the reference's
    // comparator sort.
    std::vector<std::pair<uint32_t, uint32_t>> keyed(w * h);
    for (uint64_t y = 0; y < h; ++y)
        for (uint64_t x = 0; x < w; ++x)
            keyed[y * w + x] = {spread2(uint32_t(x)) | (spread2(uint32_t(y)) << 1),
                                uint32_t(y * w + x)};
    std::sort(keyed.begin(), keyed.end());
    f->cell_order.resize(n);
    for (uint64_t i = 0; i < n; ++i) f->cell_order[i] = keyed[i].second;

    const Rng s(seed, fidx, kDensity);
    const bool cr = frame_crmath();
    f->rho.resize(n);
    parallel_for(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) {
            const uint32_t id = f->cell_order[i];
            const double xn = (static_cast<double>(id % w) + 0.5) / static_cast<double>(w);
            const double yn = (static_cast<double>(id / w) + 0.5) / static_cast<double>(h);
            bool heavy = false;
            for (const FrameBarrier& b : P.bars) {
                const double cross = b.axis == 0 ? xn : yn, along = b.axis == 0 ? yn : xn;
                if (heavy_at(cross, along, b)) {
                    heavy = true;
                    break;
                }
            }
            const double noise = std::max(0.5, 1.0 + 0.05 * frame_normal(cr, s.bits_at(P.c0 + i)));
            f->rho[i] = (heavy ? f->rho_heavy : 1.0) * noise;
        }
    });
    f->A = assemble(f->rho, f->cell_order, w, h, 1);
    f->b = sample_rhs(n, seed, fidx);
    return f;
}

// New 3D analogue: all nx*ny*nz cells in 3D Morton order; slab
// barriers with axis in {x,y,z} (the slab normal), the same center/thickness/gap laws, the gap
// running along the next axis; 7-point harmonic-mean Neumann Laplacian; projected rhs.
static hfpg_frame* frame_3d(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed,
                            uint64_t fidx) {
    const FrameParams P = frame_params_3d(nx, ny, nz, seed, fidx);
    auto* f = new hfpg_frame;
    const uint64_t n = P.n;
    f->n = n;
    f->width = nx;
    f->height = ny;
    f->depth = nz;
    f->rho_heavy = P.rho_heavy;
    f->master_seed = seed;
    f->frame_index = fidx;
    f->bars = P.bars;
    std::vector<std::pair<uint64_t, uint32_t>> keyed(n);
    parallel_for(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t id = lo; id < hi; ++id) {
            const uint64_t x = id % nx, y = (id / nx) % ny, z = id / (nx * ny);
            keyed[id] = {spread3(x) | (spread3(y) << 1) | (spread3(z) << 2), uint32_t(id)};
        }
    });
    std::sort(keyed.begin(), keyed.end());
    f->cell_order.resize(n);
    for (uint64_t i = 0; i < n; ++i) f->cell_order[i] = keyed[i].second;

    const Rng s(seed, fidx, kDensity);
    const bool cr = frame_crmath();
    f->rho.resize(n);
    parallel_for(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) {
            const uint32_t id = f->cell_order[i];
            const double c[3] = {(double(id % nx) + 0.5) / double(nx),
                                 (double((id / nx) % ny) + 0.5) / double(ny),
                                 (double(id / (nx * ny)) + 0.5) / double(nz)};
            bool heavy = false;
            for (const FrameBarrier& b : P.bars)
                if (heavy_at(c[b.axis], c[(b.axis + 1) % 3], b)) {
                    heavy = true;
                    break;
                }
            const double noise = std::max(0.5, 1.0 + 0.05 * frame_normal(cr, s.bits_at(P.c0 + i)));
            f->rho[i] = (heavy ? f->rho_heavy : 1.0) * noise;
        }
    });
    f->A = assemble(f->rho, f->cell_order, nx, ny, nz);
    f->b = sample_rhs(n, seed, fidx);
    return f;
}

// ---- checkpoint.cpp: HFTC v1 ------------------------------------------------------------------
// "HFTC0001" | u64 LE header length | JSON header | f32 LE payload of packed width.
namespace {
const char kMagic[8] = {'H', 'F', 'T', 'C', '0', '0', '0', '1'};

// Minimal JSON reader for the flat HFTC header: top-level scalars by key, plus the raw text of
// the "metadata" value (any JSON).
struct JsonHeader {
    std::vector<std::pair<std::string, std::string>> kv;  // raw value text
    const std::string* get(const char* k) const {
        for (auto& p : kv)
            if (p.first == k) return &p.second;
        return nullptr;
    }
};
void skip_ws(const std::string& s, size_t& i) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
}
std::string parse_string(const std::string& s, size_t& i) {
    if (s[i] != '"') throw IoError("read_checkpoint: malformed header");
    std::string out;
    for (++i; i < s.size() && s[i] != '"'; ++i) {
        if (s[i] == '\\') ++i;
        out += s[i];
    }
    ++i;
    return out;
}
size_t skip_value(const std::string& s, size_t i) {
    if (s[i] == '"') {
        parse_string(s, i);
        return i;
    }
    if (s[i] == '{' || s[i] == '[') {
        int depth = 0;
        for (; i < s.size(); ++i) {
            if (s[i] == '"') {
                parse_string(s, i);
                --i;
                continue;
            }
            if (s[i] == '{' || s[i] == '[') ++depth;
            if (s[i] == '}' || s[i] == ']') {
                if (--depth == 0) return i + 1;
            }
        }
        throw IoError("read_checkpoint: malformed header");
    }
    while (i < s.size() && s[i] != ',' && s[i] != '}') ++i;
    return i;
}
JsonHeader parse_header(const std::string& s) {
    JsonHeader h;
    size_t i = 0;
    skip_ws(s, i);
    if (i >= s.size() || s[i] != '{') throw IoError("read_checkpoint: malformed header");
    ++i;
    for (;;) {
        skip_ws(s, i);
        if (i < s.size() && s[i] == '}') break;
        std::string key = parse_string(s, i);
        skip_ws(s, i);
        if (i >= s.size() || s[i] != ':') throw IoError("read_checkpoint: malformed header");
        ++i;
        skip_ws(s, i);
        const size_t b = i;
        i = skip_value(s, i);
        std::string raw = s.substr(b, i - b);
        while (!raw.empty() && (raw.back() == ' ' || raw.back() == '\n')) raw.pop_back();
        h.kv.emplace_back(key, raw);
        skip_ws(s, i);
        if (i < s.size() && s[i] == ',') {
            ++i;
            continue;
        }
        if (i < s.size() && s[i] == '}') break;
        throw IoError("read_checkpoint: malformed header");
    }
    return h;
}
uint64_t need_u64(const JsonHeader& h, const char* k) {
    const std::string* v = h.get(k);
    if (!v) throw IoError(std::string("read_checkpoint: missing key ") + k);
    return std::stoull(*v);
}
uint32_t crc_of(const float* p, uint64_t n) {
    // The reference passes the whole payload to zlib in one call with the length cast to uInt
    // (checkpoint.cpp:28-30, 79-81): it checksums the first (bytes mod 2^32) bytes only, which
    // matters from 4 GiB payloads on (N >= ~5.6M). Same prefix here, chained in 1 GiB pieces.
    uLong c = ::crc32(0L, Z_NULL, 0);
    const Bytef* b = reinterpret_cast<const Bytef*>(p);
    uint64_t left = ref_crc_len(n * sizeof(float));
    while (left) {
        const uInt chunk = static_cast<uInt>(std::min<uint64_t>(left, 1u << 30));
        c = ::crc32(c, b, chunk);
        b += chunk;
        left -= chunk;
    }
    return static_cast<uint32_t>(c);
}
// Elements of a JSON array's raw text ("[a, b, ...]").
std::vector<std::string> split_array(const std::string& s) {
    std::vector<std::string> out;
    size_t i = 0;
    skip_ws(s, i);
    if (i >= s.size() || s[i] != '[') throw IoError("read_mppf: malformed header");
    ++i;
    for (;;) {
        skip_ws(s, i);
        if (i < s.size() && s[i] == ']') break;
        const size_t b = i;
        i = skip_value(s, i);
        out.push_back(s.substr(b, i - b));
        skip_ws(s, i);
        if (i < s.size() && s[i] == ',') {
            ++i;
            continue;
        }
        if (i < s.size() && s[i] == ']') break;
        throw IoError("read_mppf: malformed header");
    }
    return out;
}
const std::string& need(const JsonHeader& h, const char* k) {
    const std::string* v = h.get(k);
    if (!v) throw IoError(std::string("read_mppf: missing key ") + k);
    return *v;
}
const char kMppfMagic[8] = {'M', 'P', 'P', 'F', '0', '0', '0', '1'};
uint32_t crc_bytes(const void* p, uint64_t bytes) {
    // mppf.cpp:21-24 casts the section length to uInt as well: first (bytes mod 2^32) bytes
    bytes = ref_crc_len(bytes);
    uLong c = ::crc32(0L, Z_NULL, 0);
    const Bytef* b = static_cast<const Bytef*>(p);
    while (bytes) {
        const uInt chunk = static_cast<uInt>(std::min<uint64_t>(bytes, 1u << 30));
        c = ::crc32(c, b, chunk);
        b += chunk;
        bytes -= chunk;
    }
    return static_cast<uint32_t>(c);
}
std::string fmt_double(double v) {
    char num[64];
    std::snprintf(num, sizeof(num), "%.17g", v);
    return num;
}
}  // namespace

// checkpoint.cpp:45-66: magic, header length, JSON header, layout checks (no payload).
HftcHeader hftc_read_header(const char* path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError(std::string("read_checkpoint: cannot open ") + path);
    char magic[8];
    in.read(magic, 8);
    if (!in || std::memcmp(magic, kMagic, 8) != 0) throw IoError("read_checkpoint: bad magic");
    uint64_t len = 0;
    in.read(reinterpret_cast<char*>(&len), 8);
    if (!in || len == 0 || len > (1ULL << 30)) throw IoError("read_checkpoint: bad header length");
    std::string hs(len, '\0');
    in.read(hs.data(), std::streamsize(len));
    if (!in) throw IoError("read_checkpoint: truncated header");
    JsonHeader h = parse_header(hs);
    if (need_u64(h, "layout_version") != 1) throw IoError("read_checkpoint: unsupported layout version");
    HftcHeader out;
    out.L = make_layout(need_u64(h, "n"), need_u64(h, "leaf_size"), need_u64(h, "coarse_size"));
    if (out.L.total != need_u64(h, "packed_width")) throw IoError("read_checkpoint: packed width mismatch");
    const std::string* e = h.get("spd_shift_enabled");
    out.spd_enabled = (e && *e == "true") ? 1 : 0;
    const std::string* r = h.get("spd_shift_raw");
    out.spd_raw = r ? std::stod(*r) : 0.0;
    out.crc = uint32_t(need_u64(h, "payload_crc32"));
    out.payload_offset = 16 + len;
    return out;
}

// mppf.cpp:104-141: magic, header length, JSON header (version, dims, seeds, barriers, sections).
MppfHeader mppf_read_header(const char* path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError(std::string("read_mppf: cannot open ") + path);
    char magic[8];
    in.read(magic, 8);
    if (!in || std::memcmp(magic, kMppfMagic, 8) != 0) throw IoError(std::string("read_mppf: bad magic in ") + path);
    uint64_t len = 0;
    in.read(reinterpret_cast<char*>(&len), 8);
    if (!in || len == 0 || len > (1ULL << 30)) throw IoError(std::string("read_mppf: bad header length in ") + path);
    std::string hs(len, '\0');
    in.read(hs.data(), std::streamsize(len));
    if (!in) throw IoError(std::string("read_mppf: truncated header in ") + path);
    const JsonHeader h = parse_header(hs);
    if (std::stoll(need(h, "version")) != 1) throw IoError("read_mppf: unsupported version");
    MppfHeader m;
    m.n = std::stoull(need(h, "n"));
    m.width = std::stoull(need(h, "width"));
    m.height = std::stoull(need(h, "height"));
    const JsonHeader seeds = parse_header(need(h, "seeds"));
    m.seed = std::stoull(need(seeds, "master"));
    m.frame = std::stoull(need(seeds, "frame"));
    m.rho_heavy = std::stod(need(h, "rho_heavy"));
    for (const std::string& e : split_array(need(h, "barriers"))) {
        const JsonHeader b = parse_header(e);
        FrameBarrier fb;
        fb.axis = std::stoull(need(b, "orientation"));
        fb.center = std::stod(need(b, "center"));
        fb.thickness = std::stod(need(b, "thickness"));
        fb.gap = std::stoull(need(b, "gap"));
        m.bars.push_back(fb);
    }
    for (const std::string& e : split_array(need(h, "sections"))) {
        const JsonHeader sh = parse_header(e);
        MppfSection sec;
        std::string nm = need(sh, "name");
        if (nm.size() >= 2 && nm.front() == '"') nm = nm.substr(1, nm.size() - 2);
        sec.name = nm;
        sec.offset = std::stoull(need(sh, "offset"));
        sec.bytes = std::stoull(need(sh, "bytes"));
        sec.crc = uint32_t(std::stoull(need(sh, "crc32")));
        if (nm != "rho" && nm != "row_offsets" && nm != "col_indices" && nm != "values" && nm != "b")
            throw IoError("read_mppf: unknown section " + nm);
        m.sections.push_back(sec);
    }
    m.payload_offset = 16 + len;
    return m;
}

// csr.cpp:9-53 CsrMatrix::validate(check_symmetric = true), the reference's messages.
void validate_csr_symmetric(const Csr& A, uint64_t n) {
    if (A.row_offsets.size() != n + 1) throw InvalidArgument("csr: row_offsets length != n_rows+1");
    if (A.row_offsets.front() != 0) throw InvalidArgument("csr: row_offsets[0] != 0");
    if (A.row_offsets.back() != A.cols.size() || A.cols.size() != A.vals.size())
        throw InvalidArgument("csr: nnz mismatch");
    for (uint64_t i = 0; i < n; ++i) {
        if (A.row_offsets[i] > A.row_offsets[i + 1]) throw InvalidArgument("csr: row_offsets not nondecreasing");
        for (uint64_t p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p) {
            if (A.cols[p] >= n) throw InvalidArgument("csr: column index out of range");
            if (p > A.row_offsets[i] && A.cols[p] <= A.cols[p - 1])
                throw InvalidArgument("csr: column indices not strictly increasing in row " + std::to_string(i));
        }
    }
    auto entry = [&](uint64_t r, uint32_t c) -> double {
        uint64_t lo = A.row_offsets[r], hi = A.row_offsets[r + 1];
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (A.cols[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        return (lo < A.row_offsets[r + 1] && A.cols[lo] == c) ? A.vals[lo] : 0.0;
    };
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p)
            if (A.vals[p] != entry(A.cols[p], uint32_t(i))) throw InvalidArgument("csr: values not symmetric");
}

// frame.cpp:24-41 morton_cell_order (2D).
std::vector<uint32_t> morton_order_2d(uint64_t w, uint64_t h, uint64_t n) {
    if (w >= (1u << 16) || h >= (1u << 16)) throw InvalidArgument("morton_cell_order: grid dimension >= 2^16");
    std::vector<std::pair<uint32_t, uint32_t>> keyed(w * h);
    for (uint64_t y = 0; y < h; ++y)
        for (uint64_t x = 0; x < w; ++x)
            keyed[y * w + x] = {spread2(uint32_t(x)) | (spread2(uint32_t(y)) << 1), uint32_t(y * w + x)};
    std::sort(keyed.begin(), keyed.end());
    if (n > keyed.size()) throw InvalidArgument("morton_cell_order: n exceeds the grid");
    std::vector<uint32_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = keyed[i].second;
    return order;
}

}  // namespace hfpg

using namespace hfpg;

extern "C" {

// The checksum HFTC payloads and MPPF sections carry (checkpoint.cpp:28-30, mppf.cpp:21-24):
// zlib crc32 of the first (bytes mod 2^32) bytes.
int hfpg_payload_crc32(const void* data, uint64_t bytes, uint32_t* out) {
    return guarded([&] { *out = crc_bytes(data, bytes); });
}

int hfpg_packed_width(uint64_t n, uint64_t leaf, uint64_t ls, uint64_t* out) {
    return guarded([&] {
        check_partition(n, leaf);
        if (ls == 0 || leaf % ls != 0)
            throw InvalidArgument("packed_width: coarse size must divide leaf size");
        const uint64_t k = n / leaf;
        *out = k * leaf * leaf + (k - 1) * ls * ls + 2 * n * ls + n;
    });
}

int hfpg_build_partition(uint64_t n, uint64_t leaf, hfpg_tile* tiles, uint64_t cap,
                         uint64_t* count) {
    return guarded([&] {
        check_partition(n, leaf);
        const uint64_t k = n / leaf;
        if (count) *count = k - 1;
        // Heap order: node m at depth d = floor(log2(m+1)), index i = m + 1 - 2^d, width
        // K / 2^d; identical to the breadth-first enumeration of partition.cpp:22-34.
        for (uint64_t m = 0; m < k - 1 && m < cap; ++m) {
            uint64_t d = 0;
            while ((2ULL << d) <= m + 1) ++d;
            const uint64_t i = m + 1 - (1ULL << d), width = k >> d;
            tiles[m] = {m, width / 2, i * width, i * width + width / 2, d};
        }
    });
}

int hfpg_factor_layout(uint64_t n, uint64_t leaf, uint64_t ls, hfpg_layout* out) {
    return guarded([&] { *out = to_c(make_layout(n, leaf, ls)); });
}

int hfpg_init_factors(uint64_t n, uint64_t leaf, uint64_t ls, double sigma, uint64_t seed,
                      uint64_t frame, float* out) {
    return guarded([&] {
        const Layout L = make_layout(n, leaf, ls);
        if (!out) throw InvalidArgument("init_factors: null output");
        init_factors_host(L, sigma, seed, frame, out);
    });
}

int hfpg_write_checkpoint(const char* path, uint64_t n, uint64_t leaf, uint64_t ls,
                          const float* packed, int32_t spd_enabled, double spd_raw,
                          const char* metadata_json) {
    return guarded([&] {
        const Layout L = make_layout(n, leaf, ls);
        std::string meta = metadata_json && *metadata_json ? metadata_json : "{}";
        char num[64];
        std::snprintf(num, sizeof(num), "%.17g", spd_raw);
        // Keys in nlohmann's (sorted) order, so headers match the reference byte-for-byte
        // apart from number formatting.
        std::string hdr = "{\"coarse_size\":" + std::to_string(ls) +
                          ",\"format\":\"HFTC\",\"layout_version\":1,\"leaf_size\":" +
                          std::to_string(leaf) + ",\"metadata\":" + meta +
                          ",\"n\":" + std::to_string(n) +
                          ",\"packed_width\":" + std::to_string(L.total) +
                          ",\"payload_crc32\":" + std::to_string(crc_of(packed, L.total)) +
                          ",\"spd_shift_enabled\":" + (spd_enabled ? "true" : "false") +
                          ",\"spd_shift_raw\":" + num + "}";
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) throw IoError(std::string("write_checkpoint: cannot open ") + path);
        const uint64_t len = hdr.size();
        out.write(kMagic, 8);
        out.write(reinterpret_cast<const char*>(&len), 8);
        out.write(hdr.data(), std::streamsize(len));
        out.write(reinterpret_cast<const char*>(packed), std::streamsize(L.total * 4));
        if (!out) throw IoError("write_checkpoint: write failed");
    });
}

int hfpg_read_checkpoint(const char* path, hfpg_layout* layout, float* packed,
                         int32_t* spd_enabled, double* spd_raw, char* metadata,
                         uint64_t meta_cap) {
    return guarded([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw IoError(std::string("read_checkpoint: cannot open ") + path);
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, kMagic, 8) != 0) throw IoError("read_checkpoint: bad magic");
        uint64_t len = 0;
        in.read(reinterpret_cast<char*>(&len), 8);
        if (!in || len == 0 || len > (1ULL << 30))
            throw IoError("read_checkpoint: bad header length");
        std::string hs(len, '\0');
        in.read(hs.data(), std::streamsize(len));
        if (!in) throw IoError("read_checkpoint: truncated header");
        JsonHeader h = parse_header(hs);
        if (need_u64(h, "layout_version") != 1)
            throw IoError("read_checkpoint: unsupported layout version");
        const uint64_t n = need_u64(h, "n"), leaf = need_u64(h, "leaf_size"),
                       ls = need_u64(h, "coarse_size");
        const Layout L = make_layout(n, leaf, ls);  // throws invalid_argument like the reference
        if (L.total != need_u64(h, "packed_width"))
            throw IoError("read_checkpoint: packed width mismatch");
        if (layout) *layout = to_c(L);
        if (spd_enabled) {
            const std::string* e = h.get("spd_shift_enabled");
            *spd_enabled = (e && *e == "true") ? 1 : 0;
        }
        if (spd_raw) {
            const std::string* r = h.get("spd_shift_raw");
            *spd_raw = r ? std::stod(*r) : 0.0;
        }
        if (metadata && meta_cap) {
            const std::string* m = h.get("metadata");
            std::string mm = m ? *m : "{}";
            std::strncpy(metadata, mm.c_str(), meta_cap - 1);
            metadata[meta_cap - 1] = '\0';
        }
        if (!packed) return;
        in.read(reinterpret_cast<char*>(packed), std::streamsize(L.total * 4));
        if (!in) throw IoError("read_checkpoint: truncated payload");
        if (crc_of(packed, L.total) != need_u64(h, "payload_crc32"))
            throw IoError("read_checkpoint: payload checksum mismatch");
    });
}

int hfpg_frame_2d(uint64_t n, uint64_t seed, uint64_t frame_index, hfpg_frame** out) {
    return guarded([&] { *out = frame_2d(n, seed, frame_index); });
}

int hfpg_frame_3d(uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed, uint64_t frame_index,
                  hfpg_frame** out) {
    return guarded([&] { *out = frame_3d(nx, ny, nz, seed, frame_index); });
}

int hfpg_frame_info(const hfpg_frame* f, uint64_t* n, uint64_t* nnz, uint64_t* width,
                    uint64_t* height, uint64_t* depth, double* rho_heavy) {
    return guarded([&] {
        if (!f) throw InvalidArgument("frame_info: null frame");
        if (n) *n = f->n;
        if (nnz) *nnz = f->A.row_offsets.back();
        if (width) *width = f->width;
        if (height) *height = f->height;
        if (depth) *depth = f->depth;
        if (rho_heavy) *rho_heavy = f->rho_heavy;
    });
}

int hfpg_frame_copy(const hfpg_frame* f, uint32_t* cell_order, double* rho,
                    uint64_t* row_offsets, uint32_t* col_indices, double* values, double* b) {
    return guarded([&] {
        if (!f) throw InvalidArgument("frame_copy: null frame");
        const uint64_t n = f->n, nnz = f->A.row_offsets.back();
        if (cell_order) std::memcpy(cell_order, f->cell_order.data(), n * 4);
        if (rho) std::memcpy(rho, f->rho.data(), n * 8);
        if (row_offsets) std::memcpy(row_offsets, f->A.row_offsets.data(), (n + 1) * 8);
        if (col_indices) std::memcpy(col_indices, f->A.cols.data(), nnz * 4);
        if (values) std::memcpy(values, f->A.vals.data(), nnz * 8);
        if (b) std::memcpy(b, f->b.data(), n * 8);
    });
}

void hfpg_frame_free(hfpg_frame* f) { delete f; }


int hfpg_frame_meta(const hfpg_frame* f, uint64_t* master_seed, uint64_t* frame_index, uint32_t* nbarriers,
                    double* barriers, uint32_t cap) {
    return guarded([&] {
        if (!f) throw InvalidArgument("frame_meta: null frame");
        if (master_seed) *master_seed = f->master_seed;
        if (frame_index) *frame_index = f->frame_index;
        if (nbarriers) *nbarriers = uint32_t(f->bars.size());
        for (uint32_t i = 0; barriers && i < f->bars.size() && i < cap; ++i) {
            barriers[4 * i + 0] = double(f->bars[i].axis);
            barriers[4 * i + 1] = f->bars[i].center;
            barriers[4 * i + 2] = f->bars[i].thickness;
            barriers[4 * i + 3] = double(f->bars[i].gap);
        }
    });
}

// mppf.cpp:48-100 write_mppf: MPPF v1 ("MPPF0001" | u64 header length | JSON | sections
// rho f64 | row_offsets u64 | col_indices u32 | values f64 | b f64), per-section zlib crc32.
// Keys in nlohmann's sorted order. MPPF frames are 2D (width x height), as the reference's.
int hfpg_write_mppf(const hfpg_frame* f, const char* path) {
    return guarded([&] {
        if (!f) throw InvalidArgument("write_mppf: null frame");
        if (f->depth != 1) throw InvalidArgument("write_mppf: MPPF frames are 2D");
        const uint64_t n = f->n, nnz = f->A.row_offsets.back();
        struct Sec { const char* name; const char* dtype; const void* p; uint64_t bytes; };
        const Sec secs[5] = {{"rho", "f64", f->rho.data(), n * 8},
                             {"row_offsets", "u64", f->A.row_offsets.data(), (n + 1) * 8},
                             {"col_indices", "u32", f->A.cols.data(), nnz * 4},
                             {"values", "f64", f->A.vals.data(), nnz * 8},
                             {"b", "f64", f->b.data(), n * 8}};
        std::string bars = "[";
        for (size_t i = 0; i < f->bars.size(); ++i) {
            const FrameBarrier& b = f->bars[i];
            bars += std::string(i ? "," : "") + "{\"center\":" + fmt_double(b.center) + ",\"gap\":" +
                    std::to_string(b.gap) + ",\"orientation\":" + std::to_string(b.axis) + ",\"thickness\":" +
                    fmt_double(b.thickness) + "}";
        }
        bars += "]";
        std::string sj = "[";
        uint64_t cursor = 0;
        for (int i = 0; i < 5; ++i) {
            sj += std::string(i ? "," : "") + "{\"bytes\":" + std::to_string(secs[i].bytes) + ",\"crc32\":" +
                  std::to_string(crc_bytes(secs[i].p, secs[i].bytes)) + ",\"dtype\":\"" + secs[i].dtype +
                  "\",\"name\":\"" + secs[i].name + "\",\"offset\":" + std::to_string(cursor) + "}";
            cursor += secs[i].bytes;
        }
        sj += "]";
        const std::string hdr = "{\"barriers\":" + bars + ",\"format\":\"MPPF\",\"height\":" +
                                std::to_string(f->height) + ",\"n\":" + std::to_string(n) +
                                ",\"rho_heavy\":" + fmt_double(f->rho_heavy) + ",\"sections\":" + sj +
                                ",\"seeds\":{\"frame\":" + std::to_string(f->frame_index) + ",\"master\":" +
                                std::to_string(f->master_seed) + "},\"version\":1,\"width\":" +
                                std::to_string(f->width) + "}";
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) throw IoError(std::string("write_mppf: cannot open ") + path);
        const uint64_t len = hdr.size();
        out.write(kMppfMagic, 8);
        out.write(reinterpret_cast<const char*>(&len), 8);
        out.write(hdr.data(), std::streamsize(len));
        for (const Sec& sc : secs) out.write(static_cast<const char*>(sc.p), std::streamsize(sc.bytes));
        if (!out) throw IoError(std::string("write_mppf: write failed for ") + path);
    });
}

// mppf.cpp:102-177 read_mppf: every checksum, the CSR invariants (symmetric), section sizes,
// then the Morton cell order of the grid.
int hfpg_read_mppf(const char* path, hfpg_frame** out) {
    return guarded([&] {
        const MppfHeader m = mppf_read_header(path);
        std::ifstream in(path, std::ios::binary);
        if (!in) throw IoError(std::string("read_mppf: cannot open ") + path);
        auto* f = new hfpg_frame;
        std::unique_ptr<hfpg_frame> guard_f(f);
        f->n = m.n;
        f->width = m.width;
        f->height = m.height;
        f->master_seed = m.seed;
        f->frame_index = m.frame;
        f->rho_heavy = m.rho_heavy;
        f->bars = m.bars;
        for (const MppfSection& sc : m.sections) {
            void* dst = nullptr;
            if (sc.name == "rho") { f->rho.resize(sc.bytes / 8); dst = f->rho.data(); }
            else if (sc.name == "row_offsets") { f->A.row_offsets.resize(sc.bytes / 8); dst = f->A.row_offsets.data(); }
            else if (sc.name == "col_indices") { f->A.cols.resize(sc.bytes / 4); dst = f->A.cols.data(); }
            else if (sc.name == "values") { f->A.vals.resize(sc.bytes / 8); dst = f->A.vals.data(); }
            else { f->b.resize(sc.bytes / 8); dst = f->b.data(); }
            in.seekg(std::streamoff(m.payload_offset + sc.offset));
            in.read(static_cast<char*>(dst), std::streamsize(sc.bytes));
            if (!in) throw IoError(std::string("read_mppf: truncated section in ") + path);
            if (crc_bytes(dst, sc.bytes) != sc.crc)
                throw IoError("read_mppf: checksum mismatch in section " + sc.name);
        }
        f->A.n = m.n;
        if (f->A.row_offsets.empty()) throw InvalidArgument("csr: row_offsets length != n_rows+1");
        validate_csr_symmetric(f->A, m.n);
        if (f->rho.size() != m.n || f->b.size() != m.n)
            throw IoError("read_mppf: section sizes inconsistent with n");
        f->cell_order = morton_order_2d(m.width, m.height, m.n);
        *out = guard_f.release();
    });
}


int hfpg_frame_create(uint64_t n, uint64_t width, uint64_t height, uint64_t depth, uint64_t master_seed,
                      uint64_t frame_index, double rho_heavy, uint32_t nbarriers, const double* barriers,
                      const uint32_t* cell_order, const double* rho, const uint64_t* row_offsets,
                      const uint32_t* col_indices, const double* values, const double* b, hfpg_frame** out) {
    return guarded([&] {
        if (n == 0 || !row_offsets) throw InvalidArgument("frame_create: empty frame");
        auto f = std::make_unique<hfpg_frame>();
        f->n = n;
        f->width = width;
        f->height = height;
        f->depth = depth ? depth : 1;
        f->master_seed = master_seed;
        f->frame_index = frame_index;
        f->rho_heavy = rho_heavy;
        for (uint32_t i = 0; i < nbarriers; ++i) {
            FrameBarrier fb;
            fb.axis = uint64_t(barriers[4 * i + 0]);
            fb.center = barriers[4 * i + 1];
            fb.thickness = barriers[4 * i + 2];
            fb.gap = uint64_t(barriers[4 * i + 3]);
            f->bars.push_back(fb);
        }
        const uint64_t nnz = row_offsets[n];
        if (cell_order) f->cell_order.assign(cell_order, cell_order + n);
        f->rho.assign(rho, rho + n);
        f->b.assign(b, b + n);
        f->A.n = n;
        f->A.row_offsets.assign(row_offsets, row_offsets + n + 1);
        f->A.cols.assign(col_indices, col_indices + nnz);
        f->A.vals.assign(values, values + nnz);
        *out = f.release();
    });
}
}  // extern "C"
