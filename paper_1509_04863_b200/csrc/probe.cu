// probe.cu -- instrumentation, not part of the method: a read-only HBM streaming
// kernel (cp.async.bulk ring, one persistent CTA per SM) that bench.py times on the
// same box, to report the fold's bandwidth against a live read-only ceiling next to
// the nominal 8 TB/s and the MEASURED_PEAKS.json copy figure.
#include "tm_internal.cuh"

namespace {
constexpr int PST = 4;            // ring stages
constexpr int PSTAGE = 32 * 1024; // bytes per stage

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}"
                     : "=r"(done) : "r"(bar), "r"(ph) : "memory");
}

// CTA c reads stages c, c + grid, c + 2 grid, ... of [p, p + nstage * PSTAGE); warp 1
// issues the bulk copies, warp 0 touches one word per stage and releases it.
__global__ void __launch_bounds__(64, 1) probe_read(const uint8_t *__restrict__ p, int64_t nstage,
                                                    uint32_t *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = (uint64_t *)(sm + PST * PSTAGE), *empty = full + PST;
    if (threadIdx.x == 0) {
        for (int s = 0; s < PST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int64_t mine = nstage > blockIdx.x ? (nstage - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t i = 0; i < mine; ++i) {
            wait_parity(sa(&empty[s]), ph ^ 1);
            const uint8_t *src = p + (blockIdx.x + i * gridDim.x) * (int64_t)PSTAGE;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(PSTAGE)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(sm + s * PSTAGE)), "l"(src), "r"(PSTAGE), "r"(sa(&full[s]))
                         : "memory");
            if (++s == PST) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x < 32) {
        int s = 0;
        uint32_t ph = 0, acc = 0;
        for (int64_t i = 0; i < mine; ++i) {
            wait_parity(sa(&full[s]), ph);
            acc ^= *(const uint32_t *)(sm + s * PSTAGE + threadIdx.x * 4);
            __syncwarp();
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
            if (++s == PST) { s = 0; ph ^= 1; }
        }
        if (acc == 0x9E3779B9u && out) out[0] = acc;  // keeps the reads live
    }
}

// The fold's read pattern (fold_tma.cu): items (column group of `width` bytes,
// chunk of R rows) of a row-major [rows][ldx] byte matrix, column groups fastest
// (order = 0) or row chunks fastest (order = 1); CTA c takes items c, c + grid,
// ...; each stage is 32 KB / width rows, one bulk copy per row piece.
__global__ void __launch_bounds__(64, 1) probe_pattern(const uint8_t *__restrict__ p, int64_t ldx, int width,
                                                       int64_t rows, int64_t R, int order, uint32_t *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = (uint64_t *)(sm + PST * PSTAGE), *empty = full + PST;
    if (threadIdx.x == 0) {
        for (int s = 0; s < PST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int64_t n_groups = ldx / width, n_rc = (rows + R - 1) / R, n_items = n_groups * n_rc;
    const int sr = PSTAGE / width;
    if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const int64_t gi = order ? item / n_rc : item % n_groups;
            const int64_t rc = order ? item % n_rc : item / n_groups;
            const int64_t r0 = rc * R, r1 = min(rows, r0 + R);
            for (int64_t r = r0; r < r1; r += sr) {
                const int nr = (int)min((int64_t)sr, r1 - r);
                wait_parity(sa(&empty[s]), ph ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])),
                             "r"(nr * width) : "memory");
                for (int i = 0; i < nr; ++i)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                        ::"r"(sa(sm + s * PSTAGE + i * width)), "l"(p + (r + i) * ldx + gi * width), "r"(width),
                        "r"(sa(&full[s]))
                        : "memory");
                if (++s == PST) { s = 0; ph ^= 1; }
            }
        }
        // end marker: one more (empty) phase so the consumer loop below terminates
        wait_parity(sa(&empty[s]), ph ^ 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[s])) : "memory");
    } else if (threadIdx.x < 32) {
        int s = 0;
        uint32_t ph = 0, acc = 0;
        int64_t nst = 0;
        for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const int64_t rc = order ? item % n_rc : item / n_groups;
            const int64_t r0 = rc * R, r1 = min(rows, r0 + R);
            nst += (r1 - r0 + sr - 1) / sr;
        }
        for (int64_t i = 0; i <= nst; ++i) {
            wait_parity(sa(&full[s]), ph);
            if (i < nst) acc ^= *(const uint32_t *)(sm + s * PSTAGE + threadIdx.x * 4);
            __syncwarp();
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
            if (++s == PST) { s = 0; ph ^= 1; }
        }
        if (acc == 0x9E3779B9u && out) out[0] = acc;
    }
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int tm_probe_read_pattern(const void *buf, int64_t ldx, int width,
                                                                            int64_t rows, int64_t R, int order,
                                                                            int grid, void *stream) {
    if (!buf || width < 16 || width > PSTAGE || width % 16 || ldx % width || rows < 1 || R < 1) {
        tm_set_error("tm_probe_read_pattern: bad arguments");
        return TM_EINVAL;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)PST * PSTAGE + 2 * PST * 8;
    cudaError_t e = cudaFuncSetAttribute(probe_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return tm_cuda_status(e, "tm_probe_read_pattern: attribute");
    probe_pattern<<<(unsigned)(grid > 0 ? grid : sms), 64, smem, (cudaStream_t)stream>>>(
        (const uint8_t *)buf, ldx, width, rows, R, order, nullptr);
    TM_CHECK_LAUNCH("tm_probe_read_pattern");
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) int tm_probe_read_bw(const void *buf, int64_t bytes, void *stream) {
    if (!buf || bytes < PSTAGE || ((uintptr_t)buf % 16)) {
        tm_set_error("tm_probe_read_bw: NULL or misaligned buffer, or fewer than 32 KiB");
        return TM_EINVAL;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)PST * PSTAGE + 2 * PST * 8;
    cudaError_t e = cudaFuncSetAttribute(probe_read, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return tm_cuda_status(e, "tm_probe_read_bw: attribute");
    const int64_t nstage = bytes / PSTAGE;
    probe_read<<<(unsigned)sms, 64, smem, (cudaStream_t)stream>>>((const uint8_t *)buf, nstage, nullptr);
    TM_CHECK_LAUNCH("tm_probe_read_bw");
    return TM_OK;
}
