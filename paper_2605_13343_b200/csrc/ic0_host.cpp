// IC(0) factorization on the host (ic0.cpp:10-69, Ic0Factor / ic0_factorize), restated
// operation for operation so the lower factor is bit-identical to the reference's: the same
// left-looking merge of row prefixes, the same contraction of `s -= a * b` (this file is built
// with the reference's -O3 -march=x86-64-v3 -ffp-contract=fast), the same shift and pivot test.
// The factor is set-up work done once per system; the per-iteration apply (the two triangular
// sweeps) runs on the GPU (ic0.cuh). Also builds the transposed strictly-lower part the backward
// sweep reads row-wise.
#include "internal.hpp"

#include <cmath>
#include <string>

namespace hfpg {

void ic0_factorize_host(uint64_t n, const uint64_t* ro, const uint32_t* ci, const double* v, int policy,
                        std::vector<uint64_t>& lro, std::vector<uint32_t>& lci, std::vector<double>& lv,
                        double& shift) {
    if (n == 0) throw InvalidArgument("ic0_factorize: empty matrix");
    shift = 0.0;
    if (policy == 1) {  // Ic0Shift::scaled: 1e-8 max(diag) (ic0.cpp:14-18; diagonal() as csr.cpp:52-58)
        double dmax = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            double d = 0.0;
            for (uint64_t p = ro[i]; p < ro[i + 1]; ++p)
                if (ci[p] == i) {
                    d = v[p];
                    break;
                }
            dmax = std::max(dmax, d);
        }
        shift = 1e-8 * dmax;
    } else if (policy != 0) {
        throw InvalidArgument("ic0_factorize: unknown shift policy");
    }
    // pattern: lower triangle of A, diagonal last (a missing diagonal is a zero entry)
    lro.assign(1, 0);
    lci.clear();
    lv.clear();
    lro.reserve(n + 1);
    for (uint64_t i = 0; i < n; ++i) {
        for (uint64_t p = ro[i]; p < ro[i + 1]; ++p)
            if (ci[p] <= i) {
                lci.push_back(ci[p]);
                lv.push_back(v[p]);
            }
        if (lci.empty() || lci.back() != uint32_t(i)) {
            lci.push_back(uint32_t(i));
            lv.push_back(0.0);
        }
        lro.push_back(lci.size());
    }
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t ibeg = lro[i], iend = lro[i + 1];
        for (uint64_t p = ibeg; p < iend; ++p) {
            const uint32_t j = lci[p];
            double s = lv[p];
            const uint64_t jbeg = lro[j], jend = lro[j + 1];
            uint64_t pi = ibeg, pj = jbeg;
            while (pi < p && pj < jend && lci[pj] < j) {
                if (lci[pi] < lci[pj]) {
                    ++pi;
                } else if (lci[pi] > lci[pj]) {
                    ++pj;
                } else {
                    s -= lv[pi] * lv[pj];
                    ++pi;
                    ++pj;
                }
            }
            if (j < i) {
                const double ljj = lv[jend - 1];
                lv[p] = s / ljj;
            } else {
                s += shift;
                if (!(s > 0.0))
                    throw IoError("ic0_factorize: nonpositive pivot at row " + std::to_string(i));
                lv[p] = std::sqrt(s);
            }
        }
    }
}

// Strictly-lower part of L transposed, row j = column j of L, entries in DECREASING row order:
// the order in which the reference's backward sweep (ic0.cpp:88-95) subtracts them from z_j.
void ic0_transpose_host(uint64_t n, const std::vector<uint64_t>& lro, const std::vector<uint32_t>& lci,
                        const std::vector<double>& lv, std::vector<uint64_t>& tro, std::vector<uint32_t>& tci,
                        std::vector<double>& tv) {
    tro.assign(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t p = lro[i]; p + 1 < lro[i + 1]; ++p) ++tro[lci[p] + 1];
    for (uint64_t j = 0; j < n; ++j) tro[j + 1] += tro[j];
    tci.assign(tro[n], 0);
    tv.assign(tro[n], 0.0);
    std::vector<uint64_t> fill(tro.begin(), tro.end() - 1);
    for (uint64_t i = n; i-- > 0;)  // descending rows -> each column list in decreasing row order
        for (uint64_t p = lro[i]; p + 1 < lro[i + 1]; ++p) {
            const uint32_t j = lci[p];
            tci[fill[j]] = uint32_t(i);
            tv[fill[j]] = lv[p];
            ++fill[j];
        }
}

// Level schedules of the two sweeps: perm lists the rows by dependency level (stable in row
// order). Forward: level(i) = 1 + max level(j) over the strictly-lower entries j of row i.
// Backward: level(j) = 1 + max level(i) over the rows i > j with L_ij != 0. A sync-free sweep
// that hands out rows in this order has every dependency earlier in the list, so a row's
// producers are dispatched before it and the wait per row is one hand-off, not a CTA turnover.
void ic0_levels_host(uint64_t n, const std::vector<uint64_t>& lro, const std::vector<uint32_t>& lci,
                     const std::vector<uint64_t>& tro, const std::vector<uint32_t>& tci,
                     std::vector<uint32_t>& fperm, std::vector<uint32_t>& bperm, uint32_t& flevels,
                     uint32_t& blevels) {
    std::vector<uint32_t> lev(n, 0);
    flevels = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t l = 0;
        for (uint64_t p = lro[i]; p + 1 < lro[i + 1]; ++p) l = std::max(l, lev[lci[p]] + 1);
        lev[i] = l;
        flevels = std::max(flevels, l + 1);
    }
    auto order = [&](std::vector<uint32_t>& perm, uint32_t nlev) {
        std::vector<uint64_t> cnt(uint64_t(nlev) + 1, 0);
        for (uint64_t i = 0; i < n; ++i) ++cnt[lev[i] + 1];
        for (uint32_t l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
        perm.assign(n, 0);
        for (uint64_t i = 0; i < n; ++i) perm[cnt[lev[i]]++] = uint32_t(i);
    };
    order(fperm, flevels);
    blevels = 0;
    for (uint64_t j = n; j-- > 0;) {
        uint32_t l = 0;
        for (uint64_t q = tro[j]; q < tro[j + 1]; ++q) l = std::max(l, lev[tci[q]] + 1);
        lev[j] = l;  // rows i > j already hold their backward levels
        blevels = std::max(blevels, l + 1);
    }
    order(bperm, blevels);
}

// Levels of the rows inside their chunk of `chunk` consecutive rows (the chunked sweeps):
// forward, a row's level counts only the dependencies in its own chunk; backward likewise over
// the transposed lists. Per-chunk maxima bound the kernels' level loops.
void ic0_chunk_levels_host(uint64_t n, uint64_t chunk, const std::vector<uint64_t>& lro,
                           const std::vector<uint32_t>& lci, const std::vector<uint64_t>& tro,
                           const std::vector<uint32_t>& tci, std::vector<uint16_t>& flev,
                           std::vector<uint16_t>& blev, std::vector<uint16_t>& fmax, std::vector<uint16_t>& bmax) {
    const uint64_t nch = (n + chunk - 1) / chunk;
    flev.assign(n, 0);
    blev.assign(n, 0);
    fmax.assign(nch, 0);
    bmax.assign(nch, 0);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t c0 = (i / chunk) * chunk;
        uint32_t l = 0;
        for (uint64_t p = lro[i]; p + 1 < lro[i + 1]; ++p)
            if (lci[p] >= c0) l = std::max<uint32_t>(l, uint32_t(flev[lci[p]]) + 1);
        if (l > 65535) throw InvalidArgument("ic0: chunk level overflow");
        flev[i] = uint16_t(l);
        fmax[i / chunk] = std::max<uint16_t>(fmax[i / chunk], uint16_t(l));
    }
    for (uint64_t j = n; j-- > 0;) {
        const uint64_t c1 = (j / chunk + 1) * chunk;
        uint32_t l = 0;
        for (uint64_t q = tro[j]; q < tro[j + 1]; ++q)
            if (tci[q] < c1) l = std::max<uint32_t>(l, uint32_t(blev[tci[q]]) + 1);
        if (l > 65535) throw InvalidArgument("ic0: chunk level overflow");
        blev[j] = uint16_t(l);
        bmax[j / chunk] = std::max<uint16_t>(bmax[j / chunk], uint16_t(l));
    }
}

}  // namespace hfpg
