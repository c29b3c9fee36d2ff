// mma_bench.cu -- issue-rate microbenchmark of tcgen05.mma (kind::i8 / kind::f16)
// from shared-memory descriptors: cycles per MMA for M = 128 and several N, for
// the no-swizzle (16-byte core matrix) and 128-byte-swizzle K-major layouts.
// Measurement tool for DESIGN.md's tensor-core correlation (not part of libtm).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = (uint64_t)((a >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ __forceinline__ void mma_ts(uint32_t dt, uint32_t at, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
                 "r"(at), "l"(bd), "r"(id), "r"(acc));
}

__device__ __forceinline__ void mma_elect(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                 "@p tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, q;\n\t}" ::"r"(dt),
                 "l"(ad), "l"(bd), "r"(id), "r"(acc));
}

template <int KIND>  // 0: i8, 1: f16
__device__ __forceinline__ void mma(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
    if constexpr (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
                     "l"(ad), "l"(bd), "r"(id), "r"(acc));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
                     "l"(ad), "l"(bd), "r"(id), "r"(acc));
}

// SW: 0 = no swizzle (core matrices 8 x 16 B, LBO = 128 between K chunks, SBO = 256);
//     2 = 128-byte swizzle (rows of 128 B, SBO = 1024).
template <int KIND, int SW, int MM = 128, bool TS = false>
__global__ void __launch_bounds__(128, 1) bench(int N, int iters, long long *out, int ncopies) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(i, i * 3, i * 7, i * 11);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;
    const uint32_t idesc = ((KIND == 0 ? 2u : 1u) << 4) | ((KIND == 0 ? 1u : 0u) << 7) | ((KIND == 0 ? 1u : 0u) << 10) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        const uint32_t A = su32(sm), B = su32(sm + 64 * 1024);
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint64_t ad, bd;
                // rotate over `ncopies` distinct A tiles (16 KB each) so reuse is not free
                const uint32_t aoff = (uint32_t)((it % ncopies) * 16384);
                if (SW == 0) {
                    ad = sdesc(A + aoff + ks * 256, 128, 256, 0);
                    bd = sdesc(B + ks * 256, 128, 256, 0);
                } else {
                    ad = sdesc(A + aoff + ks * 32, 16, 1024, 2);
                    bd = sdesc(B + ks * 32, 16, 1024, 2);
                }
                if constexpr (TS)
                    mma_ts(tb + (ks & 1) * 128, tb + 256 + ks * 8, bd, idesc, (it | ks) ? 1u : 0u);
                else
                    mma<KIND>(tb + (ks & 1) * 256, ad, bd, idesc, (it | ks) ? 1u : 0u);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        uint32_t done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done)
                         : "r"(su32(&bar)));
        } while (!done);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

__device__ __forceinline__ void mma_ts_elect(uint32_t dt, uint32_t at, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                 "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, q;\n\t}" ::"r"(dt),
                 "r"(at), "l"(bd), "r"(id), "r"(acc));
}

template <int ISS, bool TS = false>
__global__ void __launch_bounds__(128, 1) bench_warp(int N, int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(i, i * 3, i * 7, i * 11);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(ISS));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    if (warp < ISS) {
        const uint32_t A = su32(sm), B = su32(sm + 64 * 1024);
        const uint64_t ad0 = sdesc(A, 128, 256, 0), bd0 = sdesc(B, 128, 256, 0);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                if constexpr (TS)
                    mma_ts_elect(tb + warp * 64 + (ks & 1) * 32, tb + 256 + 8 * ks, bd0 + ks * 16, idesc, (it | ks) ? 1u : 0u);
                else
                    mma_elect(tb + warp * 128 + (ks & 1) * 64, ad0 + ks * 16, bd0 + ks * 16, idesc, (it | ks) ? 1u : 0u);
        }
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                     "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar)));
    }
    if (tid == 0) {
        uint32_t done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done)
                         : "r"(su32(&bar)));
        } while (!done);
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int ISS, bool TS = false>
void run_warp(int N) {
    long long *d, h[1024];
    cudaMalloc(&d, sizeof(long long) * 1024);
    const int iters = 2000, grid = 148;
    auto k = bench_warp<ISS, TS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k<<<grid, 128, 96 * 1024>>>(N, 10, d);
    k<<<grid, 128, 96 * 1024>>>(N, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < grid; ++i) s += h[i];
    const double cyc = s / grid / (iters * 4.0 * ISS);
    printf("%s elect issuers=%d N=%3d: %7.2f cyc/MMA per SM  %7.0f MAC/cyc/SM (%s)\n", TS ? "TS" : "SS", ISS, N, cyc, 128.0 * N * 32 / cyc,
           cudaGetErrorString(e));
    cudaFree(d);
}

template <int KIND, int SW, int MM = 128, bool TS = false>
void run(const char *name, int N, int grid, int ncopies) {
    long long *d, h[1024];
    cudaMalloc(&d, sizeof(long long) * 1024);
    const int iters = 2000;
    auto k = bench<KIND, SW, MM, TS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k<<<grid, 128, 96 * 1024>>>(N, 10, d, ncopies);
    k<<<grid, 128, 96 * 1024>>>(N, iters, d, ncopies);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < grid; ++i) s += h[i];
    const double cyc = s / grid / (iters * 4.0);
    const double macs = (double)MM * N * (KIND == 0 ? 32 : 16);
    printf("%-10s N=%3d grid=%3d copies=%d: %7.2f cyc/MMA  %7.0f MAC/cyc/SM  (%s)\n", name, N, grid, ncopies, cyc,
           macs / cyc, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int N : {16, 32, 64}) { run_warp<1>(N); run_warp<2>(N); run_warp<1, true>(N); run_warp<2, true>(N); }
    return 0;
    for (int N : {32, 256}) {
        run<0, 0>("i8 none", N, 148, 1);
        run<0, 2>("i8 sw128", N, 148, 1);
        run<1, 0>("f16 none", N, 148, 1);
        run<1, 2>("f16 sw128", N, 148, 1);
    }
    for (int N : {32, 64, 128}) {
        run<0, 0, 64>("i8 M64", N, 148, 1);
        run<0, 0, 128, true>("i8 A-tmem", N, 148, 1);
    }
    run<0, 0>("i8 2cta/SM", 32, 296, 1);
    return 0;
}
