// Streaming-pattern microbenchmark for the fold: one persistent CTA per SM reads
// whole 1 MiB pairs (pair b = cta, cta + grid, ...) through an NST-stage TMA ring;
// the consumer holds each stage for `delay` cycles before releasing it (a stand-in
// for the fold's work per stage).  Prints GB/s for the cfg2 volume (1024 x 1 MiB).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fold_pattern tools/fold_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int NST, int STAGE, int NCOPY>
__global__ void __launch_bounds__(64, 1) tma_pairs(const uint8_t *p, size_t pair_bytes, int npairs, int delay,
                                                   unsigned *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *full = (uint64_t *)(sm + NST * STAGE), *empty = full + NST;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nst = pair_bytes / STAGE;
  if (threadIdx.x == 32) {
    int s = 0; unsigned ph = 0;
    for (int b = blockIdx.x; b < npairs; b += gridDim.x) {
      const uint8_t *base = p + (size_t)b * pair_bytes;
      for (size_t k = 0; k < nst; ++k) {
        unsigned done;
        do { asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(done) : "r"(su(&empty[s])), "r"(ph ^ 1) : "memory"); } while (!done);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
        for (int c = 0; c < NCOPY; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + s * STAGE + c * (STAGE / NCOPY))), "l"(base + k * STAGE + c * (STAGE / NCOPY)), "r"(STAGE / NCOPY), "r"(su(&full[s])) : "memory");
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
  } else if (threadIdx.x < 32) {
    int s = 0; unsigned ph = 0; unsigned acc = 0;
    for (int b = blockIdx.x; b < npairs; b += gridDim.x) {
      for (size_t k = 0; k < nst; ++k) {
        unsigned done;
        do { asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(done) : "r"(su(&full[s])), "r"(ph) : "memory"); } while (!done);
        acc ^= *(const unsigned *)(sm + s * STAGE + threadIdx.x * 4);
        if (delay) { long long t0 = clock64(); while (clock64() - t0 < delay) {} }
        __syncwarp();
        if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

template <int NST, int STAGE, int NCOPY>
void run(const uint8_t *d, unsigned *o, int sms, int delay) {
  auto k = tma_pairs<NST, STAGE, NCOPY>;
  const int smem = NST * STAGE + 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t pair = size_t(1) << 20; const int np = 1024;
  float best = 1e9, ms;
  for (int it = 0; it < 10; ++it) {
    cudaEventRecord(a); k<<<sms, 64, smem>>>(d, pair, np, delay, o); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("NST=%d STAGE=%5d copies=%d delay=%5d cyc: %7.1f GB/s  (%.1f us)\n", NST, STAGE, NCOPY, delay,
         pair * np / best / 1e6, best * 1e3);
}

int main() {
  const size_t bytes = size_t(1) << 30;
  uint8_t *d; unsigned *o;
  cudaMalloc(&d, bytes); cudaMalloc(&o, 4); cudaMemset(d, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int delay : {0, 400, 800, 1200, 1600}) run<4, 32768, 1>(d, o, sms, delay);
  for (int delay : {0, 800}) run<4, 32768, 8>(d, o, sms, delay);
  for (int delay : {0, 800}) run<3, 32768, 1>(d, o, sms, delay);
  for (int delay : {0, 800, 1600}) run<6, 32768, 1>(d, o, sms, delay);
  for (int delay : {0, 400, 800}) run<8, 16384, 1>(d, o, sms, delay);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
