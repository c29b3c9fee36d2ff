// generate.cu -- tm_generate: the paper's synthetic workload on the device
// (section 3.5).  Counter-based, keyed by
// (seed, global pair index), so any rank can generate any chunk of any pair
// without communication.  The integer outputs are bit-identical to the host
// generator tmgen/tmgen.c (an independent implementation of the same
// definition); no code is shared.
#include "tm_internal.cuh"

namespace {

constexpr uint64_t TAG_K0 = 0x4000000000000000ULL;
constexpr uint64_t TAG_FLIP = 0x5000000000000000ULL;
constexpr uint64_t TAG_TNOISE = 0x6000000000000000ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}
__device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t pair) {
    return mix64(mix64(seed) + (pair + 1ULL) * 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ uint64_t hk(uint64_t key, uint64_t ctr) {
    return mix64(key ^ (ctr * 0xD1B54A32D192ED03ULL));
}
__device__ __forceinline__ double gauss(uint64_t h) {
    double u1 = (double)((h >> 40) + 1ULL) * (1.0 / 16777216.0);
    double u2 = (double)(h & 0xFFFFFFULL) * (1.0 / 16777216.0);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}
__device__ __forceinline__ int8_t xbit(uint64_t key, int64_t i) {
    uint64_t h = hk(key, (uint64_t)i >> 6);
    return (int8_t)(1 - 2 * (int)((h >> (i & 63)) & 1ULL));
}

// int8 signal chunk: each thread writes 16 consecutive positions.
__global__ void gen_x_i8(uint64_t seed, int64_t pair0, int64_t offset, int64_t len,
                         int8_t *__restrict__ x, int64_t ldx) {
    int64_t b = blockIdx.y;
    uint64_t key = stream_key(seed, (uint64_t)(pair0 + b));
    int8_t *row = x + b * ldx;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j * 16 < len;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t p0 = offset + j * 16;  // global position of the first output
        int64_t n = len - j * 16 < 16 ? len - j * 16 : 16;
        int8_t *dst = row + j * 16;
        if (n == 16 && (p0 & 15) == 0 && (((uintptr_t)dst) & 15) == 0) {
            uint64_t h = hk(key, (uint64_t)p0 >> 6);
            uint32_t bits = (uint32_t)(h >> (p0 & 63)) & 0xFFFFu;
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t v = 0;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    uint32_t bit = (bits >> (4 * q + r)) & 1u;
                    v |= (bit ? 0xFFu : 0x01u) << (8 * r);
                }
                w[q] = v;
            }
            *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
            for (int64_t r = 0; r < n; ++r) dst[r] = xbit(key, p0 + r);
        }
    }
}

__global__ void gen_x_f32(uint64_t seed, int64_t pair0, int64_t offset, int64_t len,
                          float *__restrict__ x, int64_t ldx) {
    int64_t b = blockIdx.y;
    uint64_t key = stream_key(seed, (uint64_t)(pair0 + b));
    float *row = x + b * ldx;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len;
         j += (int64_t)gridDim.x * blockDim.x)
        row[j] = (float)gauss(hk(key, (uint64_t)(offset + j)));
}

__device__ __forceinline__ int64_t k0_of(uint64_t key, int64_t N) {
    return (int64_t)__umul64hi(hk(key, TAG_K0), (uint64_t)N);
}

__global__ void gen_t_i8(uint64_t seed, int64_t pair0, int64_t N, int64_t K, uint64_t thr,
                         int8_t *__restrict__ t, int64_t *__restrict__ k0) {
    int64_t b = blockIdx.y;
    uint64_t key = stream_key(seed, (uint64_t)(pair0 + b));
    int64_t kk = k0_of(key, N);
    if (k0 && blockIdx.x == 0 && threadIdx.x == 0) k0[b] = kk;
    if (!t) return;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t pos = (kk + j) % N;
        int8_t v = xbit(key, pos);
        uint64_t f = hk(key, TAG_FLIP + (uint64_t)j) & 0xFFFFFFFFULL;
        t[b * K + j] = (f < thr) ? (int8_t)(-v) : v;
    }
}

__global__ void gen_t_f32(uint64_t seed, int64_t pair0, int64_t N, int64_t K, double sigma,
                          float *__restrict__ t, int64_t *__restrict__ k0) {
    int64_t b = blockIdx.y;
    uint64_t key = stream_key(seed, (uint64_t)(pair0 + b));
    int64_t kk = k0_of(key, N);
    if (k0 && blockIdx.x == 0 && threadIdx.x == 0) k0[b] = kk;
    if (!t) return;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t pos = (kk + j) % N;
        double xv = (double)(float)gauss(hk(key, (uint64_t)pos));
        t[b * K + j] = (float)(xv + sigma * gauss(hk(key, TAG_TNOISE + (uint64_t)j)));
    }
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int tm_generate(tm_plan p, int64_t pair0, int64_t batch, double noise, int64_t offset,
                           int64_t len, void *x, int64_t ldx, void *t, int64_t *k0, void *stream) {
    if (!p) { tm_set_error("tm_generate: NULL plan"); return TM_EINVAL; }
    if (batch < 0 || pair0 < 0) { tm_set_error("tm_generate: negative batch/pair0"); return TM_EINVAL; }
    if (x && (offset < 0 || len < 0 || offset + len > p->N || ldx < len)) {
        tm_set_error("tm_generate: bad range offset=%lld len=%lld ldx=%lld (N=%lld)", (long long)offset,
                     (long long)len, (long long)ldx, (long long)p->N);
        return TM_EINVAL;
    }
    if (p->dtype == TM_I8 && (noise < 0.0 || noise > 1.0)) { tm_set_error("tm_generate: flip probability %g outside [0,1]", noise); return TM_EINVAL; }
    if (p->dtype == TM_F32 && noise < 0.0) { tm_set_error("tm_generate: sigma %g < 0", noise); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (batch > 65535) { tm_set_error("tm_generate: batch > 65535 per call"); return TM_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    if (x && len > 0) {
        if (p->dtype == TM_I8) {
            int64_t units = (len + 15) / 16;
            int gx = (int)((units + 255) / 256 < 4096 ? (units + 255) / 256 : 4096);
            gen_x_i8<<<dim3(gx, (unsigned)batch), 256, 0, s>>>(p->seed, pair0, offset, len, (int8_t *)x, ldx);
        } else {
            int gx = (int)((len + 255) / 256 < 8192 ? (len + 255) / 256 : 8192);
            gen_x_f32<<<dim3(gx, (unsigned)batch), 256, 0, s>>>(p->seed, pair0, offset, len, (float *)x, ldx);
        }
        TM_CHECK_LAUNCH("tm_generate: x kernel");
    }
    if (t || k0) {
        int gx = (int)((p->K + 255) / 256 < 1024 ? (p->K + 255) / 256 : 1024);
        if (p->dtype == TM_I8) {
            uint64_t thr = noise <= 0.0 ? 0ULL : (noise >= 1.0 ? (1ULL << 32) : (uint64_t)llround(noise * 4294967296.0));
            gen_t_i8<<<dim3(gx, (unsigned)batch), 256, 0, s>>>(p->seed, pair0, p->N, p->K, thr, (int8_t *)t, k0);
        } else {
            gen_t_f32<<<dim3(gx, (unsigned)batch), 256, 0, s>>>(p->seed, pair0, p->N, p->K, noise, (float *)t, k0);
        }
        TM_CHECK_LAUNCH("tm_generate: t kernel");
    }
    return TM_OK;
}
