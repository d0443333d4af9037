// Microbenchmarks of the primitives the persistent solver leans on (B200, sm_100a):
// grid-barrier variants, f32->f64 conversion rate, DFMA rate, f64 shuffle rate, TMA bulk-copy
// issue cost, and the 128-step fp32 FMA chain from shared memory (the leaf kernel's F^T r).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

// variant 0: red.release + ld.acquire polling of the counter
// variant 1: atom.acq_rel arrive; last arriver st.release a flag; others poll flag relaxed + fence
// variant 2: red.release arrive + relaxed polling of the counter + fence.acq_rel
__global__ void k_barrier(unsigned* cnt, unsigned* flag, int reps, int variant, unsigned long long* out) {
    unsigned epoch = 0;
    unsigned long long t0 = 0;
    for (int r = 0; r < reps; ++r) {
        if (r == 1) t0 = gtime();
        __syncthreads();
        ++epoch;
        if (threadIdx.x == 0) {
            const unsigned target = epoch * gridDim.x;
            if (variant == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while (ld_acquire(cnt) < target) {}
            } else if (variant == 1) {
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
                if (old == target - 1) {
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
                } else {
                    while (ld_relaxed(flag) < epoch) {}
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
            } else {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while (ld_relaxed(cnt) < target) {}
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gtime() - t0;
}

__global__ void k_f2f(const float* in, double* out, int reps) {
    float a = in[threadIdx.x & 31], b = a * 1.5f, c = a * 0.5f, d = a + 1.f;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < reps; ++i) {
        s0 += double(a); s1 += double(b); s2 += double(c); s3 += double(d);
        a += 1.f; b += 1.f; c += 1.f; d += 1.f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_dfma(const double* in, double* out, int reps) {
    double a = in[threadIdx.x & 31], s0 = 0, s1 = 1, s2 = 2, s3 = 3, s4 = 4, s5 = 5, s6 = 6, s7 = 7;
    for (int i = 0; i < reps; ++i) {
        s0 = fma(a, s0, a); s1 = fma(a, s1, a); s2 = fma(a, s2, a); s3 = fma(a, s3, a);
        s4 = fma(a, s4, a); s5 = fma(a, s5, a); s6 = fma(a, s6, a); s7 = fma(a, s7, a);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3 + s4 + s5 + s6 + s7;
}
__global__ void k_shfl(const double* in, double* out, int reps) {
    double a = in[threadIdx.x & 31], b = a + 1, c = a + 2, d = a + 3;
    for (int i = 0; i < reps; ++i) {
        a += __shfl_xor_sync(0xffffffffu, a, 1); b += __shfl_xor_sync(0xffffffffu, b, 2);
        c += __shfl_xor_sync(0xffffffffu, c, 4); d += __shfl_xor_sync(0xffffffffu, d, 8);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
// 128-long fp32 chain from smem per thread (tid < nthr), like c = F^T r
__global__ void k_chain(const float* g, float* out, int nthr, int reps, unsigned long long* t) {
    __shared__ float F[60 * 192];
    __shared__ float rin[128];
    for (int i = threadIdx.x; i < 60 * 192; i += blockDim.x) F[i] = g[i & 1023];
    if (threadIdx.x < 128) rin[threadIdx.x] = g[threadIdx.x];
    __syncthreads();
    unsigned long long t0 = clock64();
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x < nthr) {
#pragma unroll 16
            for (int i = 0; i < 128; ++i) acc = fmaf(F[(i % 60) * 192 + threadIdx.x], rin[i], acc);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) t[blockIdx.x] = clock64() - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
// TMA bulk-copy issue cost: one thread issues `nc` copies of `bytes` each
__global__ void k_tma(const float* g, int nc, int bytes, unsigned long long* t) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        unsigned long long t0 = clock64();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(nc * bytes) : "memory");
        for (int q = 0; q < nc; ++q)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sm + q * bytes)), "l"(g + q * bytes / 4), "r"(bytes), "r"(smem_u32(&bar)) : "memory");
        unsigned long long t1 = clock64();
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        unsigned long long t2 = clock64();
        t[blockIdx.x * 2] = t1 - t0;
        t[blockIdx.x * 2 + 1] = t2 - t0;
    }
}

// The leaf phase's F^T r: warps 0-1, lane owns 2 columns (float2), rin float4 broadcast;
// optionally warp 3 lane 0 bulk-copies 96 KB into another smem region concurrently.
__global__ void k_chain2(const float* g, float* out, int with_tma, unsigned long long* t) {
    extern __shared__ __align__(128) float sF[];   // [0, 16384): F; [16384, 16512): rin; then 96 KB TMA target
    __shared__ uint64_t bar;
    float* rin = sF + 16384;
    for (int i = threadIdx.x; i < 16384 + 128; i += blockDim.x) sF[i] = g[i & 4095] + 1e-3f * (i & 7);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (with_tma && warp == 3 && lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(98304) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sF + 16512)), "l"(g), "r"(98304), "r"(smem_u32(&bar)) : "memory");
    }
    if (warp < 2) {
        long long t0 = clock64();
        const int j0 = 64 * warp + 2 * lane;
        float a0 = 0.f, a1 = 0.f;
        const float4* r4 = reinterpret_cast<const float4*>(rin);
#pragma unroll 8
        for (int i4 = 0; i4 < 32; ++i4) {
            const float4 rv = r4[i4];
            const float rr4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
                const float2 f = *reinterpret_cast<const float2*>(&sF[(4 * i4 + tt) * 128 + j0]);
                a0 = fmaf(f.x, rr4[tt], a0);
                a1 = fmaf(f.y, rr4[tt], a1);
            }
        }
        out[blockIdx.x * 64 + j0] = a0 + a1;
        __syncwarp();
        if (lane == 0) t[blockIdx.x * 2 + warp] = clock64() - t0;
    }
    if (with_tma && threadIdx.x == 0)
        asm volatile("{\n\t.reg .pred p;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
}

int main() {
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned *cnt, *flag; unsigned long long* out; float* g; double* d;
    CK(cudaMalloc(&cnt, 256)); CK(cudaMalloc(&flag, 256)); CK(cudaMalloc(&out, 1 << 20));
    CK(cudaMalloc(&g, 64 << 20)); CK(cudaMalloc(&d, 64 << 20));
    CK(cudaMemset(g, 0, 64 << 20)); CK(cudaMemset(d, 0, 64 << 20));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int v = 0; v < 3; ++v) for (int thr : {512, 128}) {
        const int reps = 2001;
        CK(cudaMemset(cnt, 0, 256)); CK(cudaMemset(flag, 0, 256));
        k_barrier<<<sms, thr>>>(cnt, flag + 32, reps, v, out);
        CK(cudaDeviceSynchronize());
        unsigned long long ns; CK(cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost));
        printf("barrier variant %d grid %d x %d: %.3f us/barrier\n", v, sms, thr, ns / 1e3 / (reps - 1));
    }
    const int reps = 4096;
    float ms;
    cudaEventRecord(e0); k_f2f<<<sms * 4, 512>>>(g, d, reps); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("F2F f32->f64: %.1f conv/clk/SM (at 1.9 GHz)\n", 4.0 * reps * sms * 4 * 512 / (ms * 1e-3) / sms / 1.9e9);
    cudaEventRecord(e0); k_dfma<<<sms * 4, 512>>>(d, d + (1 << 20), reps); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA: %.1f fma/clk/SM\n", 8.0 * reps * sms * 4 * 512 / (ms * 1e-3) / sms / 1.9e9);
    cudaEventRecord(e0); k_shfl<<<sms * 4, 512>>>(d, d + (1 << 20), reps); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("SHFL f64: %.2f warp-shfl(f64)/clk/SM\n", 4.0 * reps * sms * 4 * 16 / (ms * 1e-3) / sms / 1.9e9);
    for (int nthr : {128, 192, 512}) {
        k_chain<<<sms, 512>>>(g, (float*)d, nthr < 512 ? nthr : 192, 64, out);
        CK(cudaDeviceSynchronize());
        unsigned long long c; CK(cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost));
        printf("fp32 smem chain (128 steps, %d threads): %.0f cycles/chain\n", nthr, c / 64.0);
    }
    CK(cudaFuncSetAttribute(k_chain2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int wt = 0; wt < 2; ++wt) for (int rep = 0; rep < 2; ++rep) {
        k_chain2<<<sms, 512, 200 * 1024>>>(g, (float*)d, wt, out);
        CK(cudaDeviceSynchronize());
        unsigned long long c[2]; CK(cudaMemcpy(c, out, 16, cudaMemcpyDeviceToHost));
        printf("leaf chain (float2 cols, 128 steps) tma=%d: %llu / %llu cycles\n", wt, c[0], c[1]);
    }
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int cfg = 0; cfg < 4; ++cfg) {
        int nc = cfg == 0 ? 6 : cfg == 1 ? 1 : cfg == 2 ? 10 : 2, bytes = cfg == 0 ? 16384 : cfg == 1 ? 98304 : cfg == 2 ? 8192 : 49152;
        k_tma<<<1, 32, 200 * 1024>>>(g, nc, bytes, out);
        CK(cudaDeviceSynchronize());
        k_tma<<<1, 32, 200 * 1024>>>(g, nc, bytes, out);
        CK(cudaDeviceSynchronize());
        unsigned long long c[2]; CK(cudaMemcpy(c, out, 16, cudaMemcpyDeviceToHost));
        printf("TMA %d x %d B: issue %llu cycles, landed %llu cycles (1 CTA, L2-warm)\n", nc, bytes, c[0], c[1]);
    }
    return 0;
}
