// Rank-to-rank exchange of the row-partitioned solve: device mailboxes written over peer
// memory (NVLink P2P / CUDA IPC mappings, or plain device memory for ranks sharing a GPU).
//
// Per PCG iteration a rank sends three messages to every rank (itself included), each a tiny
// f64 payload followed by a release-ordered flag:
//   M1 (after SpMV)      p.Ap, p.p partials                       -> alpha, breakdown
//   M2 (after strip sums) |r|^2 partial + the rank's subtree-root strip sums (2 x 32)
//                                                                  -> rel, the G-1 top tiles
//   M3 (after prolong)   r.z partial, after the z halo rows were stored into the peers'
//                        ghost slots                                -> beta, next SpMV
// Receivers wait with acquire loads on their own mailbox and sum the payloads in rank order,
// so every rank computes bitwise-identical scalars and takes identical branches.
// Slots are double-buffered by message sequence parity; a rank can never be two messages of
// one type ahead of a peer's read, because every send is preceded (stream order) by the wait
// on that peer's previous message of another type.
#pragma once

#include <stdint.h>

namespace hfpg {

constexpr int kMaxRanksDev = 16;
constexpr int kM2Len = 66;  // rr, pad, root_u[32], root_v[32]

struct Mailbox {
    double m1[2][kMaxRanksDev][2];
    double m2[2][kMaxRanksDev][kM2Len];
    double m3[2][kMaxRanksDev][2];
    unsigned long long flag[3][2][kMaxRanksDev];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long msg_tag(int type, unsigned long long seq) {
    return (unsigned long long)(type + 1) << 56 | seq;
}
template <int T>
__device__ __forceinline__ double* msg_slot(Mailbox* mb, int par, unsigned rank) {
    if (T == 0) return mb->m1[par][rank];
    if (T == 1) return mb->m2[par][rank];
    return mb->m3[par][rank];
}

// Send `cnt` doubles to every rank (one warp calls it; all lanes). Payload stores, a system
// fence in every lane, then lane 0 publishes the flags.
template <int T>
__device__ __forceinline__ void mb_send(Mailbox* const* peers, unsigned G, unsigned rank,
                                        unsigned long long seq, const double* payload, int cnt) {
    const int lane = threadIdx.x & 31, par = int(seq & 1);
    for (unsigned q = 0; q < G; ++q) {
        double* dst = msg_slot<T>(peers[q], par, rank);
        for (int i = lane; i < cnt; i += 32) dst[i] = payload[i];
    }
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
        const unsigned long long tag = msg_tag(T, seq);
        for (unsigned q = 0; q < G; ++q) st_release_sys_u64(&peers[q]->flag[T][par][rank], tag);
    }
    __syncwarp();
}

// Wait until every rank's message `seq` of type T is in this rank's mailbox (one thread). A
// stuck peer traps after ~30 s instead of hanging the device.
template <int T>
__device__ __forceinline__ void mb_wait(const Mailbox* mb, unsigned G, unsigned long long seq) {
    const int par = int(seq & 1);
    const unsigned long long tag = msg_tag(T, seq);
    const long long t0 = clock64();
    for (unsigned q = 0; q < G; ++q)
        while (ld_acquire_sys_u64(&mb->flag[T][par][q]) != tag)
            if (clock64() - t0 > (1LL << 36)) __trap();
}

// Rank-ordered sum of element i of every rank's message (after mb_wait).
template <int T>
__device__ __forceinline__ double mb_sum(Mailbox* mb, unsigned G, unsigned long long seq, int i) {
    const int par = int(seq & 1);
    double t = 0.0;
    for (unsigned q = 0; q < G; ++q) t += __ldcg(&msg_slot<T>(mb, par, q)[i]);
    return t;
}

}  // namespace hfpg
