// CRC-32 (zlib's crc32: reflected polynomial 0xEDB88320, init and final xor 0xFFFFFFFF) of a
// device buffer, in parallel — the checksum MPPF / HFTC headers carry per section
// (mppf.cpp:21-24, checkpoint.cpp). Bit-identical to zlib by linearity:
//   raw(M) = CRC register after M from 0 (no conditioning) is linear over GF(2), and
//   raw(A || B) = raw(A) * x^(8|B|) mod P  xor  raw(B);   leading zero bytes leave it unchanged;
//   crc32(M) = raw(M) xor 0xFFFFFFFF * x^(8|M|) mod P  xor  0xFFFFFFFF.
// k_crc32_chunks: every thread takes one 256-byte chunk (slicing-by-4 tables in shared memory,
// 16-byte loads), then warp and CTA shuffle trees merge neighbouring chunks with the uniform
// multipliers x^(8 * 256 * 2^l); the chunk grid is padded with leading zero chunks so the last
// real chunk ends the last CTA. k_crc32_finish merges the CTA results the same way, folds in the
// unaligned head (< 16 bytes, first) and the < 256-byte tail, and applies the conditioning.
#pragma once

#include <cstdint>

namespace hfpg {

constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr int kCrcChunk = 256, kCrcThreads = 256;

// a * b mod P, reflected bit order (zlib multmodp)
__host__ __device__ inline uint32_t crc_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = b & 1 ? (b >> 1) ^ kCrcPoly : b >> 1;
    }
    return p;
}
// x^(n * 2^k) mod P (zlib x2nmodp); x2n[i] = x^(2^i) mod P
__host__ __device__ inline uint32_t crc_x2nmodp(uint64_t n, unsigned k) {
    uint32_t x2n = 1u << 30;  // x^1
    for (unsigned i = 0; i < k; ++i) x2n = crc_multmodp(x2n, x2n);
    uint32_t p = 1u << 31;    // x^0
    while (n) {
        if (n & 1) p = crc_multmodp(x2n, p);
        n >>= 1;
        x2n = crc_multmodp(x2n, x2n);
    }
    return p;
}

__device__ __forceinline__ void crc_tables(uint32_t (*T)[256]) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = uint32_t(i);
        for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ kCrcPoly : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[0][i];
        for (int t = 1; t < 4; ++t) {
            c = (c >> 8) ^ T[0][c & 0xff];
            T[t][i] = c;
        }
    }
    __syncthreads();
}
__device__ __forceinline__ uint32_t crc_word(const uint32_t (*T)[256], uint32_t c, uint32_t w) {
    c ^= w;
    return T[3][c & 0xff] ^ T[2][(c >> 8) & 0xff] ^ T[1][(c >> 16) & 0xff] ^ T[0][c >> 24];
}
__device__ __forceinline__ uint32_t crc_byte(const uint32_t (*T)[256], uint32_t c, uint8_t b) {
    return T[0][(c ^ b) & 0xff] ^ (c >> 8);
}

// Per CTA: raw CRC of kCrcThreads consecutive (virtual) chunks. Virtual chunk v = real chunk
// v - zpad (leading zero chunks for v < zpad). nfull = number of whole 256-byte chunks.
__global__ void __launch_bounds__(kCrcThreads) k_crc32_chunks(const uint8_t* __restrict__ data, uint64_t nfull,
                                                              uint64_t zpad, uint32_t* __restrict__ out) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t mult[8 + 5];
    __shared__ uint32_t part[kCrcThreads / 32];
    crc_tables(T);
    if (threadIdx.x < 13) mult[threadIdx.x] = crc_x2nmodp(uint64_t(kCrcChunk) << threadIdx.x, 3);
    __syncthreads();
    const uint64_t v = uint64_t(blockIdx.x) * kCrcThreads + threadIdx.x;
    uint32_t c = 0;
    if (v >= zpad && v - zpad < nfull) {
        const uint4* p = reinterpret_cast<const uint4*>(data + (v - zpad) * kCrcChunk);
#pragma unroll 4
        for (int q = 0; q < kCrcChunk / 16; ++q) {
            const uint4 w = __ldg(p + q);
            c = crc_word(T, c, w.x);
            c = crc_word(T, c, w.y);
            c = crc_word(T, c, w.z);
            c = crc_word(T, c, w.w);
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int l = 0; l < 5; ++l) {  // merge pairs of runs of 2^l chunks (left * x^(8 |right|) ^ right)
        const uint32_t right = __shfl_down_sync(0xffffffffu, c, 1 << l);
        if ((lane & ((2 << l) - 1)) == 0) c = crc_multmodp(mult[l], c) ^ right;
    }
    if (lane == 0) part[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = part[0];
        for (int w = 1; w < kCrcThreads / 32; ++w) acc = crc_multmodp(mult[5], acc) ^ part[w];  // x^(8*256*32)
        out[blockIdx.x] = acc;
    }
}

// One CTA: merge the nblk CTA results (leading zero blocks pad them to a power of two in the
// tree), fold the tail bytes, condition.
__global__ void __launch_bounds__(1024) k_crc32_finish(const uint32_t* __restrict__ blk, uint64_t nblk, uint64_t zpad,
                                                       const uint8_t* __restrict__ head, uint32_t nhead,
                                                       const uint8_t* __restrict__ tail, uint32_t ntail,
                                                       uint64_t len, uint32_t* __restrict__ result) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t buf[1024];
    crc_tables(T);
    // sequential over groups of 1024 blocks, tree inside each group
    const uint32_t mblk = crc_x2nmodp(uint64_t(kCrcChunk) * kCrcThreads, 3);  // one block's bytes
    __shared__ uint32_t head_raw;
    if (threadIdx.x == 0) {  // the unaligned head bytes come first
        uint32_t h = 0;
        for (uint32_t i = 0; i < nhead; ++i) h = crc_byte(T, h, head[i]);
        head_raw = h;
    }
    __syncthreads();
    uint32_t total = head_raw;
    const uint64_t groups = (nblk + 1023) / 1024;
    for (uint64_t g = 0; g < groups; ++g) {
        const uint64_t b0 = g * 1024, cnt = nblk - b0 < 1024 ? nblk - b0 : 1024;
        // right-align the group's blocks in the 1024 slots (leading zero blocks)
        const uint64_t z = 1024 - cnt;
        buf[threadIdx.x] = threadIdx.x >= z ? blk[b0 + threadIdx.x - z] : 0u;
        __syncthreads();
        uint32_t m = mblk;
        for (int w = 1; w < 1024; w <<= 1) {
            uint32_t val = 0;
            const bool act = (threadIdx.x % (2 * w)) == 0;
            if (act) val = crc_multmodp(m, buf[threadIdx.x]) ^ buf[threadIdx.x + w];
            __syncthreads();
            if (act) buf[threadIdx.x] = val;
            __syncthreads();
            m = crc_multmodp(m, m);
        }
        // shift what precedes the group by the group's REAL length (block 0 opens with zpad zero chunks)
        const uint64_t real = cnt * kCrcChunk * kCrcThreads - (b0 == 0 ? zpad * kCrcChunk : 0);
        if (threadIdx.x == 0) total = crc_multmodp(crc_x2nmodp(real, 3), total) ^ buf[0];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t i = 0; i < ntail; ++i) t = crc_byte(T, t, tail[i]);
        total = crc_multmodp(crc_x2nmodp(ntail, 3), total) ^ t;
        *result = total ^ crc_multmodp(crc_x2nmodp(len, 3), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
    }
}

// zlib crc32 of len bytes at d (device memory), on stream st; scratch holds >= crc_scratch(len)
// words. Returns the device word with the result (scratch[0]).
inline uint64_t crc_scratch_words(uint64_t len) { return (len / kCrcChunk) / kCrcThreads + 2; }
inline void crc32_device(const void* d, uint64_t len, uint32_t* scratch, cudaStream_t st) {
    const uint8_t* p = static_cast<const uint8_t*>(d);
    uint32_t nhead = uint32_t((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15);
    if (nhead > len) nhead = uint32_t(len);
    const uint8_t* body = p + nhead;
    const uint64_t blen = len - nhead, nfull = blen / kCrcChunk;
    const uint64_t nblk = (nfull + kCrcThreads - 1) / kCrcThreads, zpad = nblk * kCrcThreads - nfull;
    if (nblk) k_crc32_chunks<<<unsigned(nblk), kCrcThreads, 0, st>>>(body, nfull, zpad, scratch + 1);
    k_crc32_finish<<<1, 1024, 0, st>>>(scratch + 1, nblk, zpad, p, nhead, body + nfull * kCrcChunk,
                                       uint32_t(blen - nfull * kCrcChunk), len, scratch);
}

}  // namespace hfpg
