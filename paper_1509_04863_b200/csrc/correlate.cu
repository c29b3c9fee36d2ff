// correlate.cu -- Algorithm 1 steps 4-9:
//   tm_fold_template  step 4 (t_M = [t 0]) + the template half of step 5,
//   tm_correlate      steps 5-6 read as the correlation of P:61 (reading C3):
//                       r_j[k] = sum_{i<K} t_i y_j[k+i],  k < M_j,
//   tm_match          step 7 (argmax, lowest index on ties) and steps 8-9
//                     (Theorem 4 CRT, k = -1 when z >= N).
//
// Integer data (TM_I8) is correlated EXACTLY with a number-theoretic
// transform: cyclic correlation of length L_j >= M_j + K - 1 (so no needed
// term wraps) modulo p1 = 479*2^21+1 and, when the bound |r| <= K*max|t|*
// max|y| reaches p1/2, also p2 = 119*2^23+1 with an exact CRT combine.
// Forward transforms are decimation-in-frequency (natural in, bit-reversed
// out), the inverse is decimation-in-time (bit-reversed in, natural out), so
// no permutation pass is needed.  The folded template stores
// NTT(t reversed) * L^{-1} with Shoup companions, so the pointwise product
// and the 1/L scaling are one Shoup multiply.
//
// Real data (TM_F32) is correlated directly in fp32 (tiled through shared
// memory, four interleaved partial sums per output).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "tm_internal.cuh"

const uint32_t TM_PRIMES[2] = {TM_P1, TM_P2};
static const uint32_t TM_GENERATORS[2] = {3u, 3u};

namespace {

// ---------------------------------------------------------------------------
// host: root-of-unity tables.  For each length n = 2^l (1 <= l <= TM_MAX_LOGL)
// the table holds w_n^j, j < n/2, at offset n/2 - 1; one table per prime and
// direction (forward w_n, inverse w_n^{-1}), plus Shoup companions.
// ---------------------------------------------------------------------------
uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1;
    b %= m;
    while (e) {
        if (e & 1) r = (unsigned __int128)r * b % m;
        b = (unsigned __int128)b * b % m;
        e >>= 1;
    }
    return r;
}

std::mutex g_tab_mu;
struct DevTables {
    bool ready = false;
    uint32_t *buf = nullptr;
    tm_ntt_tables t{};
};
DevTables g_tabs[64];

}  // namespace

int tm_ntt_tables_get(int device, tm_ntt_tables *out) {
    if (device < 0 || device >= 64) { tm_set_error("tm: device index %d unsupported", device); return TM_EUNSUPPORTED; }
    std::lock_guard<std::mutex> lk(g_tab_mu);
    DevTables &D = g_tabs[device];
    if (!D.ready) {
        TmDeviceGuard guard(device);  // the allocation and upload belong to `device`
        const size_t n = size_t(1) << TM_MAX_LOGL;  // entries per table (sum of n/2 over lengths)
        std::vector<uint32_t> h(16 * n, 0u);  // 8n separate (value | companion) + 8n interleaved
        for (int pi = 0; pi < 2; ++pi) {
            const uint64_t p = TM_PRIMES[pi];
            for (int dir = 0; dir < 2; ++dir) {
                uint32_t *val = h.data() + (size_t)(pi * 2 + dir) * 2 * n;
                uint32_t *sh = val + n;
                for (int l = 1; l <= TM_MAX_LOGL; ++l) {
                    uint64_t len = uint64_t(1) << l;
                    uint64_t w = powmod(TM_GENERATORS[pi], (p - 1) / len, p);
                    if (dir) w = powmod(w, p - 2, p);
                    uint64_t cur = 1;
                    uint32_t *il = h.data() + 8 * n + (size_t)(pi * 2 + dir) * 2 * n;
                    for (uint64_t j = 0; j < len / 2; ++j) {
                        val[len / 2 - 1 + j] = (uint32_t)cur;
                        sh[len / 2 - 1 + j] = (uint32_t)(((unsigned __int128)cur << 32) / p);
                        il[2 * (len / 2 - 1 + j)] = val[len / 2 - 1 + j];
                        il[2 * (len / 2 - 1 + j) + 1] = sh[len / 2 - 1 + j];
                        cur = (unsigned __int128)cur * w % p;
                    }
                }
            }
        }
        uint32_t *d = nullptr;
        cudaError_t e = cudaMalloc(&d, h.size() * sizeof(uint32_t));
        if (e != cudaSuccess) return tm_cuda_status(e, "tm: NTT table allocation");
        e = cudaMemcpy(d, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm: NTT table upload");
        D.buf = d;
        for (int pi = 0; pi < 2; ++pi)
            for (int dir = 0; dir < 2; ++dir) {
                D.t.tw[pi][dir] = d + (size_t)(pi * 2 + dir) * 2 * n;
                D.t.tws[pi][dir] = d + (size_t)(pi * 2 + dir) * 2 * n + n;
                D.t.tw2[pi][dir] = reinterpret_cast<const uint2 *>(d + 8 * n + (size_t)(pi * 2 + dir) * 2 * n);
            }
        D.ready = true;
    }
    *out = D.t;
    return TM_OK;
}

namespace {

// ---------------------------------------------------------------------------
// device modular arithmetic (p < 2^31)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t add_p(uint32_t a, uint32_t b, uint32_t p) {
    uint32_t s = a + b;
    return s >= p ? s - p : s;
}
__device__ __forceinline__ uint32_t sub_p(uint32_t a, uint32_t b, uint32_t p) {
    return a >= b ? a - b : a + p - b;
}
// Shoup: a * w mod p for any a < 2^32, w < p, ws = floor(w 2^32 / p)
__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint32_t w, uint32_t ws, uint32_t p) {
    uint32_t qq = __umulhi(a, ws);
    uint32_t r = a * w - qq * p;
    return r >= p ? r - p : r;
}

// forward DIF, natural -> bit-reversed.  Stage with half-span h uses the
// length-2h table: twiddle w_{2h}^j at offset h - 1 + j.
template <typename Sync>
__device__ void ntt_dif(uint32_t *a, int logL, const uint32_t *__restrict__ tw,
                        const uint32_t *__restrict__ tws, uint32_t p, int tid, int nthr, Sync sync) {
    const int half = 1 << (logL - 1);
    for (int lh = logL - 1; lh >= 0; --lh) {
        const int h = 1 << lh;
        const uint32_t *t = tw + (h - 1), *ts = tws + (h - 1);
        for (int idx = tid; idx < half; idx += nthr) {
            const int j = idx & (h - 1);
            const int i0 = ((idx >> lh) << (lh + 1)) | j;
            const uint32_t X = a[i0], Y = a[i0 + h];
            a[i0] = add_p(X, Y, p);
            a[i0 + h] = mul_shoup(X + p - Y, __ldg(t + j), __ldg(ts + j), p);
        }
        sync();
    }
}

// inverse DIT, bit-reversed -> natural (unscaled; 1/L is folded into the template)
template <typename Sync>
__device__ void ntt_dit_inv(uint32_t *a, int logL, const uint32_t *__restrict__ tw,
                            const uint32_t *__restrict__ tws, uint32_t p, int tid, int nthr, Sync sync) {
    const int half = 1 << (logL - 1);
    for (int lh = 0; lh < logL; ++lh) {
        const int h = 1 << lh;
        const uint32_t *t = tw + (h - 1), *ts = tws + (h - 1);
        for (int idx = tid; idx < half; idx += nthr) {
            const int j = idx & (h - 1);
            const int i0 = ((idx >> lh) << (lh + 1)) | j;
            const uint32_t X = a[i0];
            const uint32_t Y = mul_shoup(a[i0 + h], __ldg(t + j), __ldg(ts + j), p);
            a[i0] = add_p(X, Y, p);
            a[i0 + h] = sub_p(X, Y, p);
        }
        sync();
    }
}

struct BlockSync {
    __device__ void operator()() const { __syncthreads(); }
};

// ---------------------------------------------------------------------------
// template fold: tf[b][prime][slot] = (v, Shoup(v)) with v = NTT_L(t_rev) * L^{-1},
// t_rev[0] = t[0], t_rev[L - i] = t[i]  (the reversal turns step 6's product
// into a correlation, reading C3).  Slot 0: length L1; slot 1: length L2 if != L1.
// ---------------------------------------------------------------------------
struct TfArgs {
    const int8_t *t;
    int64_t K;
    int logL[2];
    int n_len;           // 1 or 2 distinct lengths
    int64_t per_prime;   // uint2 elements per prime per pair
    int n_primes;
    uint2 *tf;
    uint32_t *scratch;   // global scratch for transforms too long for shared memory
    int use_smem;
    tm_ntt_tables tabs;
};

__global__ void __launch_bounds__(1024) template_ntt_kernel(TfArgs A) {
    extern __shared__ uint32_t sm[];
    const int64_t b = blockIdx.x;
    const int pi = blockIdx.y;       // prime
    const int li = blockIdx.z;       // length slot
    if (li >= A.n_len) return;
    const int logL = A.logL[li];
    const int64_t L = int64_t(1) << logL;
    const uint32_t p = pi ? TM_P2 : TM_P1;
    uint32_t *a = A.use_smem ? sm
                             : A.scratch + ((b * A.n_primes + pi) * 2 + li) * (int64_t(1) << A.logL[A.n_len - 1]);
    const int8_t *t = A.t + b * A.K;
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
        int64_t src = (i == 0) ? 0 : L - i;  // t_rev[i] = t[(L - i) mod L]
        int32_t v = (src < A.K) ? (int32_t)t[src] : 0;
        a[i] = v >= 0 ? (uint32_t)v : (uint32_t)((int64_t)p + v);
    }
    __syncthreads();
    ntt_dif(a, logL, A.tabs.tw[pi][0] + 0, A.tabs.tws[pi][0] + 0, p, threadIdx.x, blockDim.x, BlockSync());
    // scale by L^{-1} mod p
    uint64_t Linv = 1, base = (uint64_t)L % p, e = p - 2;
    while (e) { if (e & 1) Linv = Linv * base % p; base = base * base % p; e >>= 1; }
    const uint32_t Li = (uint32_t)Linv, Lis = (uint32_t)(((uint64_t)Li << 32) / p);
    uint2 *dst = A.tf + b * (A.per_prime * A.n_primes) + pi * A.per_prime + (li ? (int64_t(1) << A.logL[0]) : 0);
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
        uint32_t v = mul_shoup(a[i], Li, Lis, p);
        dst[i] = make_uint2(v, (uint32_t)(((uint64_t)v << 32) / p));
    }
}

// ---------------------------------------------------------------------------
// correlation (+ optional argmax) for one (pair, modulus): all primes, CRT.
// ---------------------------------------------------------------------------
struct CorrArgs {
    const int32_t *y[2];
    int64_t len_y[2];
    int64_t nload[2];
    int64_t M[2];
    int64_t K;
    int logL[2];
    int tf_slot[2];          // offset (elements) of this modulus's transform inside a prime block
    int64_t per_prime;
    int n_primes;
    const uint2 *tf;
    int64_t *r[2];           // may be NULL
    int32_t *resid;          // [batch][2] or NULL
    uint32_t *scratch;       // global scratch when !use_smem
    int use_smem;
    int64_t scratch_stride;  // u32 per (pair, modulus) in scratch
    tm_ntt_tables tabs;
};

__device__ __forceinline__ void argmax_merge(int64_t &bv, int64_t &bi, int64_t v, int64_t i) {
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

__global__ void __launch_bounds__(1024) corr_ntt_kernel(CorrArgs A) {
    extern __shared__ uint32_t sm[];
    const int64_t b = blockIdx.x;
    const int j = blockIdx.y;  // modulus
    const int logL = A.logL[j];
    const int64_t L = int64_t(1) << logL;
    const int64_t M = A.M[j];
    uint32_t *a = A.use_smem ? sm : A.scratch + (b * 2 + j) * A.scratch_stride;
    uint32_t *keep = a + L;  // residues of prime 0 (two-prime case)
    const int32_t *y = A.y[j] + b * A.len_y[j];
    const int64_t nload = A.nload[j];  // y[0 .. M+K-2] (y[M+K-1] is never needed), or M (cyclic y1)
    for (int pi = 0; pi < A.n_primes; ++pi) {
        const uint32_t p = pi ? TM_P2 : TM_P1;
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
            int32_t v = (i < nload) ? y[i] : 0;
            int64_t m = (int64_t)v % (int64_t)p;
            if (m < 0) m += p;
            a[i] = (uint32_t)m;
        }
        __syncthreads();
        ntt_dif(a, logL, A.tabs.tw[pi][0], A.tabs.tws[pi][0], p, threadIdx.x, blockDim.x, BlockSync());
        const uint2 *tf = A.tf + b * (A.per_prime * A.n_primes) + pi * A.per_prime + A.tf_slot[j];
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
            uint2 w = tf[i];
            a[i] = mul_shoup(a[i], w.x, w.y, p);
        }
        __syncthreads();
        ntt_dit_inv(a, logL, A.tabs.tw[pi][1], A.tabs.tws[pi][1], p, threadIdx.x, blockDim.x, BlockSync());
        if (pi == 0 && A.n_primes == 2) {
            for (int64_t i = threadIdx.x; i < M; i += blockDim.x) keep[i] = a[i];
            __syncthreads();
        }
    }
    // signed reconstruction, output, argmax
    int64_t bv = INT64_MIN, bi = INT64_MAX;
    int64_t *rout = A.r[j] ? A.r[j] + b * M : nullptr;
    const uint64_t p1 = TM_P1, p2 = TM_P2;
    const uint64_t inv_p1_mod_p2 = TM_P1_INV_MOD_P2;
    for (int64_t k = threadIdx.x; k < M; k += blockDim.x) {
        int64_t v;
        if (A.n_primes == 1) {
            uint32_t u = a[k];
            v = (u > (uint32_t)(p1 / 2)) ? (int64_t)u - (int64_t)p1 : (int64_t)u;
        } else {
            uint64_t a1 = keep[k], a2 = a[k];
            uint64_t d = (a2 + p2 - a1 % p2) % p2;
            uint64_t u = (d * inv_p1_mod_p2) % p2;
            unsigned __int128 z = (unsigned __int128)a1 + (unsigned __int128)p1 * u;  // < p1*p2
            const unsigned __int128 P = (unsigned __int128)p1 * p2;
            v = (z > P / 2) ? (int64_t)((__int128)z - (__int128)P) : (int64_t)z;
        }
        if (rout) rout[k] = v;
        argmax_merge(bv, bi, v, k);
    }
    if (A.resid) {
        __shared__ int64_t s_v[32], s_i[32];
        for (int o = 16; o > 0; o >>= 1) {
            int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
            argmax_merge(bv, bi, ov, oi);
        }
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) { s_v[w] = bv; s_i[w] = bi; }
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            bv = l < nw ? s_v[l] : INT64_MIN;
            bi = l < nw ? s_i[l] : INT64_MAX;
            for (int o = 16; o > 0; o >>= 1) {
                int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
                argmax_merge(bv, bi, ov, oi);
            }
            if (l == 0) A.resid[b * 2 + j] = (int32_t)bi;
        }
    }
}

// ---------------------------------------------------------------------------
// fp32 direct correlation, tiled: block = (pair, modulus, tile of TK outputs)
// ---------------------------------------------------------------------------
constexpr int F_TK = 1024, F_TI = 2048, F_THREADS = 256;

__global__ void __launch_bounds__(F_THREADS) corr_f32_kernel(const float *__restrict__ y1, const float *__restrict__ y2,
                                                             int64_t M1, int64_t M2, int64_t K,
                                                             const float *__restrict__ t, float *r1, float *r2,
                                                             float *tile_best_v, int32_t *tile_best_i, int n_tiles) {
    __shared__ float s_t[F_TI];
    __shared__ float s_y[F_TK + F_TI];
    const int64_t b = blockIdx.y;
    const int j = blockIdx.z;
    const int64_t M = j ? M2 : M1;
    const int64_t k0 = (int64_t)blockIdx.x * F_TK;
    if (k0 >= M) return;
    const float *y = (j ? y2 : y1) + b * (M + K);
    const float *tb = t + b * K;
    constexpr int PER = F_TK / F_THREADS;  // outputs per thread (strided by F_THREADS)
    float acc[PER][4];
#pragma unroll
    for (int u = 0; u < PER; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
    for (int64_t i0 = 0; i0 < K; i0 += F_TI) {
        const int ni = (int)((K - i0) < F_TI ? (K - i0) : F_TI);
        __syncthreads();
        for (int i = threadIdx.x; i < F_TI; i += F_THREADS) s_t[i] = i < ni ? tb[i0 + i] : 0.f;
        for (int i = threadIdx.x; i < F_TK + F_TI; i += F_THREADS) {
            int64_t src = k0 + i0 + i;
            s_y[i] = (src < M + K - 1) ? y[src] : 0.f;
        }
        __syncthreads();
        for (int i = 0; i < ni; i += 4) {
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int kk = threadIdx.x + u * F_THREADS;
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(s_t[i + v], s_y[kk + i + v], acc[u][v]);
            }
        }
    }
    float bv = -INFINITY;
    int32_t bi = 0x7FFFFFFF;
    float *r = j ? r2 : r1;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int64_t k = k0 + threadIdx.x + u * F_THREADS;
        if (k < M) {
            float v = (acc[u][0] + acc[u][1]) + (acc[u][2] + acc[u][3]);
            if (r) r[b * M + k] = v;
            if (v > bv || (v == bv && k < bi)) { bv = v; bi = (int32_t)k; }
        }
    }
    if (tile_best_v) {
        for (int o = 16; o > 0; o >>= 1) {
            float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        __shared__ float s_v[F_THREADS / 32];
        __shared__ int32_t s_i[F_THREADS / 32];
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) { s_v[w] = bv; s_i[w] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < F_THREADS / 32; ++q)
                if (s_v[q] > bv || (s_v[q] == bv && s_i[q] < bi)) { bv = s_v[q]; bi = s_i[q]; }
            int64_t slot = (b * 2 + j) * n_tiles + blockIdx.x;
            tile_best_v[slot] = bv;
            tile_best_i[slot] = bi;
        }
    }
}

// reduce per-tile argmax (fp32) -> residues
__global__ void f32_tiles_to_resid(const float *v, const int32_t *ix, int64_t batch, int n_tiles1, int n_tiles2,
                                   int n_tiles, int32_t *resid) {
    int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= batch * 2) return;
    int j = (int)(id & 1);
    int nt = j ? n_tiles2 : n_tiles1;
    float bv = -INFINITY;
    int32_t bi = 0x7FFFFFFF;
    for (int q = 0; q < nt; ++q) {
        float vv = v[id * n_tiles + q];
        int32_t ii = ix[id * n_tiles + q];
        if (vv > bv || (vv == bv && ii < bi)) { bv = vv; bi = ii; }
    }
    resid[id] = bi;
}

// ---------------------------------------------------------------------------
// staged argmax over materialised r (tm_match)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void argmax_kernel(const T *__restrict__ r1, const T *__restrict__ r2, int64_t M1, int64_t M2,
                              int32_t *resid) {
    const int64_t b = blockIdx.x;
    const int j = blockIdx.y;
    const int64_t M = j ? M2 : M1;
    const T *r = (j ? r2 : r1) + b * M;
    T bv = r[0];
    int64_t bi = 0;
    for (int64_t k = threadIdx.x; k < M; k += blockDim.x) {
        T v = r[k];
        if (v > bv || (v == bv && k < bi)) { bv = v; bi = k; }
    }
    __shared__ T s_v[32];
    __shared__ int64_t s_i[32];
    for (int o = 16; o > 0; o >>= 1) {
        T ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { s_v[w] = bv; s_i[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
            if (s_v[q] > bv || (s_v[q] == bv && s_i[q] < bi)) { bv = s_v[q]; bi = s_i[q]; }
        resid[b * 2 + j] = (int32_t)bi;
    }
}

// steps 8-9 (tm_resolve)
__global__ void crt_kernel(const int32_t *__restrict__ resid, int64_t batch, int64_t M1, int64_t M2,
                           uint32_t inv, int64_t N, int64_t wrap, int32_t *residues_out, int64_t *k) {
    pdl_trigger();
    pdl_wait();
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    int64_t m1 = resid[2 * b], m2 = resid[2 * b + 1];
    k[b] = tm_resolve(m1, m2, M1, M2, inv, N, wrap);
    if (residues_out) { residues_out[2 * b] = (int32_t)m1; residues_out[2 * b + 1] = (int32_t)m2; }
}

int ntt_block_threads(int logL) { return logL >= 11 ? 1024 : (logL >= 8 ? 256 : 64); }

size_t smem_limit() { return 160 * 1024; }

}  // namespace

// ---------------------------------------------------------------------------
// scratch needed outside shared memory (global workspace), u32 elements
// ---------------------------------------------------------------------------
static bool corr_in_smem(const tm_plan_s *p) {
    int64_t L = p->L1 > p->L2 ? p->L1 : p->L2;
    return (size_t)L * 4 * (size_t)p->n_primes <= smem_limit();
}

extern "C" __attribute__((visibility("default"))) int tm_fold_template(tm_plan p, const void *t, int64_t batch, void *tf, void *stream) {
    if (!p) { tm_set_error("tm_fold_template: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_fold_template: batch < 0"); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (!t || !tf) { tm_set_error("tm_fold_template: NULL pointer"); return TM_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    if (p->dtype == TM_F32) {
        if (tm_fft_f32_ok(p)) return tm_fft_f32_template(p, t, p->K, batch, tf, s);
        cudaError_t e = cudaMemcpyAsync(tf, t, (size_t)batch * p->K * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_fold_template: copy");
        return TM_OK;
    }
    if (batch > 0x7FFFFFFF) { tm_set_error("tm_fold_template: batch too large"); return TM_EUNSUPPORTED; }
    if (p->use_tc) return tm_tc_template(p, t, batch, tf, s);
    if (p->fast_corr) return tm_fast_template(p, t, batch, tf, s);
    if (p->big_corr) return tm_gntt_template(p, t, batch, tf, s);
    TfArgs A;
    A.t = (const int8_t *)t; A.K = p->K;
    A.logL[0] = p->logL1; A.logL[1] = p->logL2;
    A.n_len = (p->L1 == p->L2) ? 1 : 2;
    A.per_prime = p->tf_elems; A.n_primes = p->n_primes;
    A.tf = (uint2 *)tf;
    tm_ntt_tables_get(p->device, &A.tabs);
    int64_t Lmax = p->L1 > p->L2 ? p->L1 : p->L2;
    A.use_smem = (size_t)Lmax * 4 <= smem_limit();
    A.scratch = nullptr;
    if (!A.use_smem) {
        // the template's own transform runs in place inside tf's slot (as u32 scratch
        // inside the uint2 output region: element i is read/written only by its slot)
        tm_set_error("tm_fold_template: L=%lld exceeds shared memory; large transforms not built", (long long)Lmax);
        return TM_EUNSUPPORTED;
    }
    size_t smem = (size_t)Lmax * 4;
    cudaFuncSetAttribute(template_ntt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_limit());
    int thr = ntt_block_threads(p->logL2);
    template_ntt_kernel<<<dim3((unsigned)batch, (unsigned)p->n_primes, (unsigned)A.n_len), thr, smem, s>>>(A);
    TM_CHECK_LAUNCH("tm_fold_template");
    return TM_OK;
}

int tm_correlate_impl(const tm_plan_s *p, const void *y1, const void *y2, const void *tf, int64_t batch,
                      void *r1, void *r2, int32_t *resid, void *tile_scratch, void *gntt_scratch, cudaStream_t s,
                      void *tc_ws) {
    if (batch == 0) return TM_OK;
    if (p->dtype == TM_F32 && tm_fft_f32_ok(p))
        return tm_fft_f32_correlate(p, y1, y2, tf, batch, r1, r2, resid, gntt_scratch, s);
    if (p->dtype == TM_F32) {
        const int nt1 = (int)((p->M1 + F_TK - 1) / F_TK), nt2 = (int)((p->M2 + F_TK - 1) / F_TK);
        const int nt = nt2;
        float *tv = nullptr;
        int32_t *ti = nullptr;
        if (resid) {  // per-tile argmax partials (workspace region f32_tiles)
            tv = (float *)tile_scratch;
            ti = (int32_t *)(tv + batch * 2 * nt);
        }
        dim3 grid((unsigned)nt, (unsigned)batch, 2);
        corr_f32_kernel<<<grid, F_THREADS, 0, s>>>((const float *)y1, (const float *)y2, p->M1, p->M2, p->K,
                                                    (const float *)tf, (float *)r1, (float *)r2, tv, ti, nt);
        TM_CHECK_LAUNCH("tm_correlate: corr_f32_kernel");
        if (resid) {
            f32_tiles_to_resid<<<(unsigned)((batch * 2 + 255) / 256), 256, 0, s>>>(tv, ti, batch, nt1, nt2, nt, resid);
            TM_CHECK_LAUNCH("tm_correlate: f32_tiles_to_resid");
        }
        return TM_OK;
    }
    if (p->use_tc) return tm_tc_any(p, y1, y2, tf, p->tf_bytes, batch, r1, r2, resid, nullptr, nullptr, tc_ws, s);
    if (p->fast_corr) return tm_fast_correlate(p, y1, y2, nullptr, tf, batch, r1, r2, resid, s);
    if (p->big_corr) return tm_gntt_correlate(p, y1, y2, nullptr, tf, batch, r1, r2, resid, gntt_scratch, s);
    if (!corr_in_smem(p)) {
        tm_set_error("tm_correlate: transform length %lld x %d primes exceeds shared memory (large path not built)",
                     (long long)(p->L1 > p->L2 ? p->L1 : p->L2), p->n_primes);
        return TM_EUNSUPPORTED;
    }
    CorrArgs A;
    A.y[0] = (const int32_t *)y1; A.y[1] = (const int32_t *)y2;
    A.len_y[0] = p->len_y1; A.len_y[1] = p->len_y2;
    A.nload[0] = p->nload1; A.nload[1] = p->nload2;
    A.M[0] = p->M1; A.M[1] = p->M2; A.K = p->K;
    A.logL[0] = p->logL1; A.logL[1] = p->logL2;
    A.tf_slot[0] = 0; A.tf_slot[1] = (p->L1 == p->L2) ? 0 : (int)p->L1;
    A.per_prime = p->tf_elems; A.n_primes = p->n_primes;
    A.tf = (const uint2 *)tf;
    A.r[0] = (int64_t *)r1; A.r[1] = (int64_t *)r2;
    A.resid = resid;
    A.scratch = nullptr; A.use_smem = 1; A.scratch_stride = 0;
    tm_ntt_tables_get(p->device, &A.tabs);
    int64_t Lmax = p->L1 > p->L2 ? p->L1 : p->L2;
    size_t smem = (size_t)Lmax * 4 * (p->n_primes == 2 ? 2 : 1);
    cudaFuncSetAttribute(corr_ntt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_limit());
    int thr = ntt_block_threads(p->logL2);
    corr_ntt_kernel<<<dim3((unsigned)batch, 2), thr, smem, s>>>(A);
    TM_CHECK_LAUNCH("tm_correlate: corr_ntt_kernel");
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) int tm_correlate(tm_plan p, const void *y1, const void *y2, const void *tf, int64_t batch, void *r1,
                            void *r2, void *ws, void *stream) {
    if (!p) { tm_set_error("tm_correlate: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_correlate: batch < 0"); return TM_EINVAL; }
    if (batch > 0 && (!y1 || !y2 || !tf || !r1 || !r2)) { tm_set_error("tm_correlate: NULL pointer"); return TM_EINVAL; }
    if ((p->big_corr || tm_fft_f32_long(p)) && !ws) {
        tm_set_error("tm_correlate: workspace required for this plan");
        return TM_EINVAL;
    }
    void *g = ws ? (char *)ws + tm_ws(p, batch).gntt : nullptr;
    return tm_correlate_impl(p, y1, y2, tf, batch, r1, r2, nullptr, nullptr, g, (cudaStream_t)stream, ws);
}

int tm_crt_impl(const tm_plan_s *p, const int32_t *resid, int64_t batch, int32_t *residues_out, int64_t *k,
                cudaStream_t s) {
    if (batch == 0) return TM_OK;
    const cudaError_t e = launch_pdl(crt_kernel, dim3((unsigned)((batch + 255) / 256)), dim3(256), 0, s, resid, batch,
                                     p->M1, p->M2, p->crt_inv, p->N, p->crt_wrap, residues_out, k);
    if (e != cudaSuccess) return tm_cuda_status(e, "tm_match: crt_kernel");
    TM_CHECK_LAUNCH("tm_match: crt_kernel");
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) int tm_match(tm_plan p, const void *r1, const void *r2, int64_t batch, int32_t *residues, int64_t *k,
                        void *stream) {
    if (!p) { tm_set_error("tm_match: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_match: batch < 0"); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (!r1 || !r2 || !k || !residues) { tm_set_error("tm_match: NULL pointer"); return TM_EINVAL; }
    if (batch > 0x7FFFFFFF) { tm_set_error("tm_match: batch too large"); return TM_EUNSUPPORTED; }
    cudaStream_t s = (cudaStream_t)stream;
    int32_t *resid = residues;
    if (p->dtype == TM_I8)
        argmax_kernel<int64_t><<<dim3((unsigned)batch, 2), 256, 0, s>>>((const int64_t *)r1, (const int64_t *)r2,
                                                                          p->M1, p->M2, resid);
    else
        argmax_kernel<float><<<dim3((unsigned)batch, 2), 256, 0, s>>>((const float *)r1, (const float *)r2, p->M1,
                                                                        p->M2, resid);
    TM_CHECK_LAUNCH("tm_match: argmax_kernel");
    return tm_crt_impl(p, resid, batch, nullptr, k, s);
}
