// Shared device helpers: PTX wrappers for TMA bulk copies + mbarriers, deterministic
// warp/block/grid reductions, and the device-resident PCG state.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hfpg {

// Device-resident PCG state (pcg.cpp:53-126 locals). All scalars are f64, as the reference
// requires (pcg.hpp:14-16). Written by the last CTA of each reduction, read by the next kernel.
struct Scalars {
    double rz;            // r.z of the current iterate
    double pap, pp;       // p.Ap, p.p (pcg.cpp:88-89)
    double alpha, beta;   // step sizes
    double r0;            // |r_0|
    double rel;           // last |r_k|/|r_0|
    double rtol;          // SolveConfig::rtol
    double breakdown_tol; // 1e-12 |A|_F (pcg.cpp:80)
    double shift;         // softplus SPD shift (factor_tensor.hpp:64-66)
    unsigned long long k;          // current iteration (1-based inside the loop)
    unsigned long long max_iters;
    unsigned long long iterations;
    unsigned long long breakdown_iter;
    unsigned long long hist_len;
    int status;    // 0 converged, 1 max_iters, 2 breakdown
    int converged;
    int done;      // loop finished: every later kernel of the iteration early-exits
    int pad;
    double rr_loc; // row partition: this rank's |r|^2 partial (leaf -> strip-sum kernel)
    double rzs[2]; // deferred reductions: r.z of iteration k-1, by parity of k (SpMV writes)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) -------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Arrival counters with release / acquire semantics at GPU scope (no SC fence: MEMBAR.SC.GPU
// waits for the issuing warp's in-flight memory operations, TMA bulk copies included).
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Global -> shared bulk copy completing on `bar`; `policy` is an L2 cache-policy descriptor.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Streaming 128-bit load that does not allocate in L1.
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// 128-bit read-only load with an L2 cache-policy hint (e.g. evict_last for data every
// iteration re-reads).
__device__ __forceinline__ float4 ldg_hint(const float4* p, uint64_t policy) {
    float4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(policy));
    return r;
}

__device__ __forceinline__ float ldg_f32_hint(const float* p, uint64_t policy) {
    float r;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(policy));
    return r;
}

__device__ __forceinline__ uint32_t ldg_stream_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ldg_stream_f64(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

// ---- programmatic dependent launch (PDL) -------------------------------------------------------
// The solve's kernels are launched with programmatic stream serialisation (hfpg_device.cu
// launch_k): each lets its dependent grid launch at once (launch_dependents), so the next kernel's
// CTAs are placed and set up as this one's CTAs drain, and then waits for its own predecessor to
// complete and flush (griddepcontrol.wait) before reading anything — a no-op without PDL.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---- deterministic reductions ----------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deferred grid reductions: the producing kernel only publishes one partial per CTA (block
// reduce, no arrival counter, no fence, no last-CTA tail); every CTA of the consuming kernel sums
// all partials itself in one fixed order (one warp: lane-strided sums, then an xor butterfly,
// whose result is bit-identical in every lane — a + b = b + a — and so in every CTA).
template <int NV>
__device__ __forceinline__ void publish_partials(const double (&v)[NV], double* dst) {
    __shared__ double red[NV][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const double s = warp_sum(v[i]);
        if (lane == 0) red[i][warp] = s;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double s = lane < nwarps ? red[i][lane] : 0.0;
            s = warp_sum(s);
            if (lane == 0) dst[blockIdx.x * NV + i] = s;
        }
    }
}
// Called by one whole warp.
template <int NV>
__device__ __forceinline__ void sum_partials(const double* src, uint32_t n, double (&out)[NV]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double acc = 0.0;
        for (uint32_t j = lane; j < n; j += 32) acc += __ldcg(&src[j * NV + i]);
        out[i] = warp_sum(acc);
    }
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Block-reduce NV values, publish the CTA partial, and let the last-arriving CTA reduce all
// partials in CTA order (fixed tree => run-to-run identical results). Returns true in every
// thread of the last CTA, with `total` filled; the arrival counter is reset for the next
// launch. Must be called by all threads of every CTA.
template <int NV>
__device__ bool grid_reduce_last(double (&v)[NV], double* partials, unsigned* counter,
                                 double (&total)[NV]) {
    __shared__ double red[NV][32];
    __shared__ int is_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const double s = warp_sum(v[i]);
        if (lane == 0) red[i][warp] = s;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double s = lane < nwarps ? red[i][lane] : 0.0;
            s = warp_sum(s);
            if (lane == 0) partials[blockIdx.x * NV + i] = s;
        }
        if (lane == 0) {  // release this CTA's partial, acquire the others' (acq_rel, no SC fence)
            const unsigned t = atom_add_acq_rel_gpu(counter, 1u);
            is_last = (t == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (!is_last) return false;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
        for (unsigned j = threadIdx.x; j < gridDim.x; j += blockDim.x)
            s += __ldcg(&partials[j * NV + i]);
        s = warp_sum(s);
        __syncthreads();
        if (lane == 0) red[i][warp] = s;
        __syncthreads();
        double t = lane < nwarps ? red[i][lane] : 0.0;
        total[i] = warp_sum(t);
    }
    if (threadIdx.x == 0) *counter = 0u;
    return true;
}

}  // namespace hfpg
