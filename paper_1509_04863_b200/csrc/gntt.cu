// gntt.cu -- exact NTT correlation for transforms too long for one CTA
// (L > 2^14: cfg4 with K = 16384, cfg5 with K = 65536).  Algorithm 1 steps
// 4-7 read as the correlation of P:61 (reading C3), the
// same arithmetic as corr_fast.cu, organised as a sequence of grid-wide passes
// over an L2-resident scratch buffer:
//   load   a = y mod p (and t_rev mod p for the template instance)
//   DIF    radix-16 passes from the top bit down (natural -> bit-reversed)
//   mul    a = a * T * L^-1 (pointwise, same bit-reversed order)
//   DIT    radix-16 passes from the bottom bit up (bit-reversed -> natural)
//   final  CRT over the primes, r output, per-block argmax partials
//   argmax reduce the partials (lowest index on ties)
// Every instance (pair, prime) of one modulus goes through the same launches.
// The template spectrum is transformed once at the y2 length L2; the y1
// transform (cyclic, L1 = M1 = L2 / 2) uses its first bit-reversed half, which
// is exactly the length-L1 spectrum of t reversed mod L1.
#include "tm_internal.cuh"

namespace {

constexpr int GT = 256;  // threads per block for passes

__device__ __forceinline__ uint32_t prime_of(int pi) { return pi ? TM_P2 : TM_P1; }
__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint32_t w, uint32_t ws, uint32_t p) {
    const uint32_t r = a * w - __umulhi(a, ws) * p;
    return r >= p ? r - p : r;
}
__device__ __forceinline__ uint32_t add_p(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t s = a + b;
    return s >= p ? s - p : s;
}
__device__ __forceinline__ uint32_t sub_p(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

struct PassArgs {
    uint32_t *data;       // [n_inst][L]
    int64_t n_inst;
    int n_primes;         // instance i uses prime i % n_primes
    int logL, b_lo, nst;  // stages b_lo .. b_lo + nst - 1
    const uint2 *tw[2];   // per prime, direction chosen by the caller
};

// one group of 2^nst elements per thread: index bits outside [b_lo, b_lo+nst) fixed
template <bool INV>
__global__ void __launch_bounds__(GT) gntt_pass(PassArgs A) {
    const int64_t L = int64_t(1) << A.logL;
    const int64_t G = L >> A.nst;
    const int64_t gid = (int64_t)blockIdx.x * GT + threadIdx.x;
    if (gid >= A.n_inst * G) return;
    const int64_t inst = gid / G, g = gid % G;
    const int pi = (int)(inst % A.n_primes);
    const uint32_t p = prime_of(pi);
    const uint2 *tw = A.tw[pi];
    const int64_t lo = g & ((int64_t(1) << A.b_lo) - 1), hi = g >> A.b_lo;
    const int64_t base = (hi << (A.b_lo + A.nst)) | lo;
    uint32_t *d = A.data + inst * L;
    uint32_t v[16];
    const int E = 1 << A.nst;
#pragma unroll
    for (int m = 0; m < 16; ++m)
        if (m < E) v[m] = d[base + ((int64_t)m << A.b_lo)];
    if (!INV) {
#pragma unroll
        for (int u = 3; u >= 0; --u) {
            if (u >= A.nst) continue;
            const int h = 1 << u;
            const uint2 *tab = tw + ((int64_t(1) << (A.b_lo + u)) - 1);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                if (m >= E || (m & h)) continue;
                const uint2 w = tab[((int64_t)(m & (h - 1)) << A.b_lo) | lo];
                const uint32_t X = v[m], Y = v[m | h];
                v[m] = add_p(X, Y, p);
                v[m | h] = mul_shoup(X + p - Y, w.x, w.y, p);
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (u >= A.nst) continue;
            const int h = 1 << u;
            const uint2 *tab = tw + ((int64_t(1) << (A.b_lo + u)) - 1);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                if (m >= E || (m & h)) continue;
                const uint2 w = tab[((int64_t)(m & (h - 1)) << A.b_lo) | lo];
                const uint32_t X = v[m];
                const uint32_t Yw = mul_shoup(v[m | h], w.x, w.y, p);
                v[m] = add_p(X, Yw, p);
                v[m | h] = sub_p(X, Yw, p);
            }
        }
    }
#pragma unroll
    for (int m = 0; m < 16; ++m)
        if (m < E) d[base + ((int64_t)m << A.b_lo)] = v[m];
}

// a[inst][i] = y[b][i] mod p (i < nload), instance = b * n_primes + pi
__global__ void gntt_load_y(const int32_t *__restrict__ y, int64_t ldy, int64_t nload, int64_t n_inst, int n_primes,
                            int logL, uint32_t *a) {
    const int64_t L = int64_t(1) << logL;
    for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n_inst * L;
         id += (int64_t)gridDim.x * blockDim.x) {
        const int64_t inst = id >> logL, i = id & (L - 1);
        const int64_t b = inst / n_primes;
        const uint32_t p = prime_of((int)(inst % n_primes));
        const int32_t v = i < nload ? y[b * ldy + i] : 0;
        a[id] = v >= 0 ? (uint32_t)v % p : (uint32_t)((int64_t)p + v % (int64_t)p) % p;
    }
}

// T[inst][i] = t_rev[i] = t[(L - i) mod L] mod p (zero beyond K)
__global__ void gntt_load_t(const int8_t *__restrict__ t, int64_t K, int64_t n_inst, int n_primes, int logL,
                            uint32_t *T) {
    const int64_t L = int64_t(1) << logL;
    for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n_inst * L;
         id += (int64_t)gridDim.x * blockDim.x) {
        const int64_t inst = id >> logL, i = id & (L - 1);
        const int64_t b = inst / n_primes;
        const uint32_t p = prime_of((int)(inst % n_primes));
        const int64_t src = i == 0 ? 0 : L - i;
        const int32_t v = src < K ? (int32_t)t[b * K + src] : 0;
        T[id] = v >= 0 ? (uint32_t)v : (uint32_t)((int64_t)p + v);
    }
}

// a[inst][i] = a[inst][i] * T[inst][i] * L^{-1} mod p; T has length LT >= L (uses its first L)
__global__ void gntt_pointwise(uint32_t *a, const uint32_t *__restrict__ T, int64_t n_inst, int n_primes, int logL,
                               int logLT, uint32_t linv0, uint32_t linv1) {
    const int64_t L = int64_t(1) << logL;
    for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n_inst * L;
         id += (int64_t)gridDim.x * blockDim.x) {
        const int64_t inst = id >> logL, i = id & (L - 1);
        const int pi = (int)(inst % n_primes);
        const uint32_t p = prime_of(pi);
        const uint64_t tv = T[(inst << logLT) + i];
        const uint64_t v = ((uint64_t)a[id] * tv) % p;
        a[id] = (uint32_t)((v * (pi ? linv1 : linv0)) % p);
    }
}

__device__ __forceinline__ void amax(int64_t &bv, int64_t &bi, int64_t v, int64_t i) {
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

// r[b][k] = CRT over primes of a[b*n_primes + pi][k], k < M; block argmax partials
__global__ void __launch_bounds__(GT) gntt_final(const uint32_t *__restrict__ a, int64_t batch, int n_primes, int logL,
                                                 int64_t M, int64_t *r, int64_t *part_v, int64_t *part_i,
                                                 int blocks_per_pair) {
    const int64_t L = int64_t(1) << logL;
    const int64_t b = blockIdx.y;
    int64_t bv = INT64_MIN, bi = INT64_MAX;
    for (int64_t k = (int64_t)blockIdx.x * GT + threadIdx.x; k < M; k += (int64_t)blocks_per_pair * GT) {
        int64_t val;
        const uint64_t a1 = a[(b * n_primes) * L + k];
        if (n_primes == 1) {
            val = a1 > TM_P1 / 2 ? (int64_t)a1 - (int64_t)TM_P1 : (int64_t)a1;
        } else {
            const uint64_t a2 = a[(b * n_primes + 1) * L + k];
            const uint64_t d = (a2 + TM_P2 - (a1 % TM_P2)) % TM_P2;
            const uint64_t u = (d * TM_P1_INV_MOD_P2) % TM_P2;
            const uint64_t z = a1 + (uint64_t)TM_P1 * u;
            const uint64_t PP = (uint64_t)TM_P1 * TM_P2;
            val = z > PP / 2 ? (int64_t)(z - PP) : (int64_t)z;
        }
        if (r) r[b * M + k] = val;
        amax(bv, bi, val, k);
    }
    __shared__ int64_t sv[GT / 32], si[GT / 32];
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
        amax(bv, bi, ov, oi);
    }
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < GT / 32; ++w) amax(bv, bi, sv[w], si[w]);
        part_v[b * blocks_per_pair + blockIdx.x] = bv;
        part_i[b * blocks_per_pair + blockIdx.x] = bi;
    }
}

__global__ void gntt_argmax_reduce(const int64_t *part_v, const int64_t *part_i, int64_t batch, int blocks_per_pair,
                                   int jmod, int32_t *resid) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    int64_t bv = INT64_MIN, bi = INT64_MAX;
    for (int q = 0; q < blocks_per_pair; ++q) amax(bv, bi, part_v[b * blocks_per_pair + q], part_i[b * blocks_per_pair + q]);
    resid[b * 2 + jmod] = (int32_t)bi;
}

uint32_t linv_host(int logL, uint64_t p) {
    uint64_t r = 1, base = (uint64_t(1) << logL) % p, e = p - 2;
    while (e) { if (e & 1) r = (unsigned __int128)r * base % p; base = (unsigned __int128)base * base % p; e >>= 1; }
    return (uint32_t)r;
}

int run_passes(uint32_t *data, int64_t n_inst, int n_primes, int logL, bool inv, const tm_ntt_tables &tabs,
               cudaStream_t s) {
    PassArgs A;
    A.data = data; A.n_inst = n_inst; A.n_primes = n_primes; A.logL = logL;
    A.tw[0] = tabs.tw2[0][inv ? 1 : 0];
    A.tw[1] = tabs.tw2[1][inv ? 1 : 0];
    // DIF: top bits first; DIT: bottom bits first.  Passes of <= 4 stages.
    int done = 0;
    while (done < logL) {
        const int nst = (logL - done) < 4 ? (logL - done) : 4;
        A.nst = nst;
        A.b_lo = inv ? done : logL - done - nst;
        const int64_t groups = n_inst * ((int64_t(1) << logL) >> nst);
        const unsigned grid = (unsigned)((groups + GT - 1) / GT);
        if (inv) gntt_pass<true><<<grid, GT, 0, s>>>(A);
        else gntt_pass<false><<<grid, GT, 0, s>>>(A);
        TM_CHECK_LAUNCH("tm_correlate: gntt_pass");
        done += nst;
    }
    return TM_OK;
}

}  // namespace

size_t tm_gntt_scratch_bytes(const tm_plan_s *p, int64_t batch) {
    if (p->dtype != TM_I8) return 0;
    const int64_t L = p->L1 > p->L2 ? p->L1 : p->L2;
    // a (largest modulus) + template spectrum at L2 + argmax partials
    return (size_t)batch * p->n_primes * (size_t)(2 * L) * 4 + (size_t)batch * 64 * 16 + 1024;
}

// Whole correlation (+ argmax) via grid passes.  t != NULL: template transformed
// here (tm_run); else tf holds the template spectrum at L2 in natural
// bit-reversed order, u32 [batch][n_primes][L2] (tm_fold_template's output).
int tm_gntt_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *t, const void *tf,
                      int64_t batch, void *r1, void *r2, int32_t *resid, void *scratch, cudaStream_t s) {
    tm_ntt_tables tabs;
    tm_ntt_tables_get(p->device, &tabs);
    const int np = p->n_primes;
    const int64_t n_inst = batch * np;
    const int logLT = p->logL2;
    const int64_t LT = int64_t(1) << logLT;
    uint32_t *a = (uint32_t *)scratch;
    uint32_t *T = a + (size_t)n_inst * LT;
    int64_t *part_v = (int64_t *)(T + (size_t)n_inst * LT);
    const int bpp = 64;  // argmax partial blocks per pair
    int64_t *part_i = part_v + batch * bpp;
    const unsigned ew_grid = (unsigned)((n_inst * LT + 255) / 256 < 65535 * 8 ? (n_inst * LT + 255) / 256 : 65535 * 8);
    if (t) {
        gntt_load_t<<<ew_grid, 256, 0, s>>>((const int8_t *)t, p->K, n_inst, np, logLT, T);
        TM_CHECK_LAUNCH("tm_correlate: gntt_load_t");
        int rc = run_passes(T, n_inst, np, logLT, false, tabs, s);
        if (rc) return rc;
    } else {
        cudaError_t e = cudaMemcpyAsync(T, tf, (size_t)n_inst * LT * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_correlate: tf copy");
    }
    const uint32_t li[2][2] = {{linv_host(p->logL1, TM_P1), linv_host(p->logL1, TM_P2)},
                               {linv_host(p->logL2, TM_P1), linv_host(p->logL2, TM_P2)}};
    for (int j = 0; j < 2; ++j) {
        const int logL = j ? p->logL2 : p->logL1;
        if (logL > logLT) { tm_set_error("gntt: L1 > L2"); return TM_EUNSUPPORTED; }
        const int64_t L = int64_t(1) << logL;
        const unsigned g = (unsigned)((n_inst * L + 255) / 256 < 65535 * 8 ? (n_inst * L + 255) / 256 : 65535 * 8);
        gntt_load_y<<<g, 256, 0, s>>>((const int32_t *)(j ? y2 : y1), j ? p->len_y2 : p->len_y1,
                                      j ? p->nload2 : p->nload1, n_inst, np, logL, a);
        TM_CHECK_LAUNCH("tm_correlate: gntt_load_y");
        int rc = run_passes(a, n_inst, np, logL, false, tabs, s);
        if (rc) return rc;
        gntt_pointwise<<<g, 256, 0, s>>>(a, T, n_inst, np, logL, logLT, li[j][0], li[j][1]);
        TM_CHECK_LAUNCH("tm_correlate: gntt_pointwise");
        rc = run_passes(a, n_inst, np, logL, true, tabs, s);
        if (rc) return rc;
        const int64_t M = j ? p->M2 : p->M1;
        gntt_final<<<dim3(bpp, (unsigned)batch), GT, 0, s>>>(a, batch, np, logL, M, (int64_t *)(j ? r2 : r1),
                                                            part_v, part_i, bpp);
        TM_CHECK_LAUNCH("tm_correlate: gntt_final");
        if (resid) {
            gntt_argmax_reduce<<<(unsigned)((batch + 255) / 256), 256, 0, s>>>(part_v, part_i, batch, bpp, j, resid);
            TM_CHECK_LAUNCH("tm_correlate: gntt_argmax_reduce");
        }
    }
    return TM_OK;
}

// tm_fold_template for plans on the grid-pass path: T = NTT_{L2}(t_rev) (bit-reversed)
int tm_gntt_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s) {
    tm_ntt_tables tabs;
    tm_ntt_tables_get(p->device, &tabs);
    const int np = p->n_primes;
    const int64_t n_inst = batch * np;
    const int64_t LT = int64_t(1) << p->logL2;
    const unsigned g = (unsigned)((n_inst * LT + 255) / 256 < 65535 * 8 ? (n_inst * LT + 255) / 256 : 65535 * 8);
    gntt_load_t<<<g, 256, 0, s>>>((const int8_t *)t, p->K, n_inst, np, p->logL2, (uint32_t *)tf);
    TM_CHECK_LAUNCH("tm_fold_template: gntt_load_t");
    return run_passes((uint32_t *)tf, n_inst, np, p->logL2, false, tabs, s);
}
