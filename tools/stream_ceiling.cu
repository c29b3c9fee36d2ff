// stream_ceiling.cu -- calibration only (not part of libtm): read-only HBM
// streaming ceilings on this B200, to put the fold's fraction in context.
//   (1) grid-stride LDG.128 read + xor reduce, (2) cp.async.bulk (TMA) ring read.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void ldg_sum(const uint4 *__restrict__ p, size_t n, unsigned *out) {
  unsigned acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (; i < n; i += stride) { uint4 v = __ldg(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NST, int STAGE>
__global__ void __launch_bounds__(64, 1) tma_read(const uint8_t *p, size_t chunk_per_cta, unsigned *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *full = (uint64_t *)(sm + NST * STAGE), *empty = full + NST;
  if (threadIdx.x == 0) { for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s]))); }
    asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint8_t *base = p + blockIdx.x * chunk_per_cta;
  size_t nst = chunk_per_cta / STAGE;
  if (threadIdx.x == 32) {
    int s = 0; unsigned ph = 0;
    for (size_t k = 0; k < nst; ++k) {
      unsigned done; do { asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(done) : "r"(su(&empty[s])), "r"(ph ^ 1) : "memory"); } while (!done);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + s * STAGE)), "l"(base + k * STAGE), "r"(STAGE), "r"(su(&full[s])) : "memory");
      if (++s == NST) { s = 0; ph ^= 1; }
    }
  } else if (threadIdx.x < 32) {
    int s = 0; unsigned ph = 0; unsigned acc = 0;
    for (size_t k = 0; k < nst; ++k) {
      unsigned done; do { asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(done) : "r"(su(&full[s])), "r"(ph) : "memory"); } while (!done);
      acc ^= *(const unsigned *)(sm + s * STAGE + threadIdx.x * 4);
      __syncwarp();
      if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
      if (++s == NST) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

int main() {
  const size_t bytes = size_t(4) << 30;
  uint8_t *d; unsigned *o;
  cudaMalloc(&d, bytes); cudaMalloc(&o, 4); cudaMemset(d, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9, ms;
  for (int blocks_per_sm : {2, 4, 8}) {
    best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a); ldg_sum<<<sms * blocks_per_sm, 512>>>((const uint4 *)d, bytes / 16, o); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("ldg_sum  grid=%d x 512: %.1f GB/s\n", sms * blocks_per_sm, bytes / best / 1e6);
  }
  {
    constexpr int NST = 4, STAGE = 32768;
    auto k = tma_read<NST, STAGE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE + 64);
    size_t chunk = bytes / sms / STAGE * STAGE;
    best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a); k<<<sms, 64, NST * STAGE + 64>>>(d, chunk, o); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("tma_read 4x32KB/SM: %.1f GB/s\n", chunk * sms / best / 1e6);
  }
  {
    constexpr int NST = 6, STAGE = 32768;
    auto k = tma_read<NST, STAGE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE + 128);
    size_t chunk = bytes / sms / STAGE * STAGE;
    best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a); k<<<sms, 64, NST * STAGE + 128>>>(d, chunk, o); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("tma_read 6x32KB/SM: %.1f GB/s\n", chunk * sms / best / 1e6);
  }
  // per-SM ceiling: fewer CTAs (1 per SM), deeper rings
  for (int ncta : {32, 48, 64, 96, 128}) {
    constexpr int NST = 6, STAGE = 32768;
    auto k = tma_read<NST, STAGE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE + 128);
    size_t chunk = bytes / ncta / STAGE * STAGE;
    if (chunk > (size_t(256) << 20)) chunk = size_t(256) << 20;
    best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a); k<<<ncta, 64, NST * STAGE + 128>>>(d, chunk, o); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("tma_read 6x32KB, %3d CTAs: %.1f GB/s total, %.1f GB/s per SM\n", ncta, chunk * ncta / best / 1e6, chunk / best / 1e6);
  }
  for (int ncta : {32, 64}) {
    constexpr int NST = 3, STAGE = 65536;
    auto k = tma_read<NST, STAGE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE + 128);
    size_t chunk = bytes / ncta / STAGE * STAGE;
    if (chunk > (size_t(128) << 20)) chunk = size_t(128) << 20;
    best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a); k<<<ncta, 64, NST * STAGE + 128>>>(d, chunk, o); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("tma_read 3x64KB, %3d CTAs: %.1f GB/s total, %.1f GB/s per SM\n", ncta, chunk * ncta / best / 1e6, chunk / best / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
