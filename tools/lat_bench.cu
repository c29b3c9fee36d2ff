// lat_bench.cu -- latency of tcgen05.commit -> mbarrier completion (with 0/1/8
// preceding TS MMAs) and of tcgen05.st + tcgen05.wait::st, single CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void commit(uint64_t *b) {
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                 "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
    } while (!done);
}
__device__ __forceinline__ void mma_ts(uint32_t dt, uint32_t at, uint64_t bd, uint32_t id) {
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                 "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(dt), "r"(at), "l"(bd), "r"(id));
}
__global__ void lat(int nmma, long long *out) {
    __shared__ __align__(1024) uint8_t B[8192];
    __shared__ uint64_t bar;
    __shared__ uint32_t ts;
    const int tid = threadIdx.x;
    for (int i = tid; i < 8192; i += 32) B[i] = i;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&ts)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = ts;
    uint64_t bd = (uint64_t)((su32(B) >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | (4u << 17) | (8u << 24);
    const int iters = 200;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        for (int m = 0; m < nmma; ++m) mma_ts(tb, tb + 64 + 8 * (m & 3), bd, id);
        commit(&bar);
        wait(&bar, i & 1);
    }
    long long t1 = clock64();
    // tcgen05.st x16 + wait::st
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = i * tid;
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(tb + 64 + (i & 1) * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                     "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    long long t3 = clock64();
    if (tid == 0) { out[blockIdx.x * 2] = (t1 - t0) / iters; out[blockIdx.x * 2 + 1] = (t3 - t2) / iters; }
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}
int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16 * 148);
    for (int nm : {0, 1, 8, 32}) {
        lat<<<1, 32>>>(nm, d);
        lat<<<1, 32>>>(nm, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("nmma=%2d: commit->wait round trip %lld cyc; tcgen05.st x16 + wait::st %lld cyc (%s)\n", nm, h[0], h[1], cudaGetErrorString(e));
    }
    return 0;
}
