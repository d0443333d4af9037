// Device side of the on-disk formats: an MPPF frame's CSR checked on the
// GPU exactly as CsrMatrix::validate(check_symmetric = true) does on the host (csr.cpp:9-53), with
// its row lengths and diagonal (csr.cpp:52-58) for the SELL-32 / Jacobi state.
#pragma once

#include <cstdint>

namespace hfpg {

enum : unsigned { kCsrNondecreasing = 1u, kCsrColRange = 2u, kCsrColOrder = 4u, kCsrSymmetric = 8u, kCsrFirst = 16u,
                  kCsrLast = 32u };

__global__ void k_mppf_rows(const unsigned long long* __restrict__ ro, const uint32_t* __restrict__ ci,
                            const double* __restrict__ v, unsigned long long n, unsigned long long nnz,
                            uint32_t* __restrict__ len, double* __restrict__ diag, unsigned* __restrict__ err) {
    const unsigned long long i = blockIdx.x * 256ULL + threadIdx.x;
    if (i == 0 && ro[0] != 0ULL) atomicOr(err, kCsrFirst);
    if (i == 0 && ro[n] != nnz) atomicOr(err, kCsrLast);
    if (i >= n) return;
    const unsigned long long p0 = ro[i], p1 = ro[i + 1];
    unsigned e = 0;
    if (p0 > p1 || p1 > nnz) {
        atomicOr(err, kCsrNondecreasing);
        len[i] = 0;
        diag[i] = 0.0;
        return;
    }
    double d = 0.0;
    for (unsigned long long p = p0; p < p1; ++p) {
        const uint32_t c = ci[p];
        if (c >= n) {
            e |= kCsrColRange;
            continue;
        }
        if (p > p0 && c <= ci[p - 1]) e |= kCsrColOrder;
        if (c == i) d = v[p];
    }
    len[i] = uint32_t(p1 - p0);
    diag[i] = d;
    if (!e) {  // symmetric: A_ij == A_ji (0.0 when absent), by binary search in row j
        for (unsigned long long p = p0; p < p1; ++p) {
            const uint32_t c = ci[p];
            unsigned long long lo = ro[c], hi = ro[c + 1];
            if (lo > hi || hi > nnz) break;  // reported by row c's own thread
            while (lo < hi) {
                const unsigned long long mid = (lo + hi) / 2;
                if (ci[mid] < uint32_t(i)) lo = mid + 1;
                else hi = mid;
            }
            const double t = (lo < ro[c + 1] && ci[lo] == uint32_t(i)) ? v[lo] : 0.0;
            if (v[p] != t) {
                e |= kCsrSymmetric;
                break;
            }
        }
    }
    if (e) atomicOr(err, e);
}

}  // namespace hfpg
