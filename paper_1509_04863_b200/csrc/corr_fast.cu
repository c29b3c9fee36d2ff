// corr_fast.cu -- register-resident NTT correlation + argmax (Algorithm 1
// steps 4-7, read as the correlation of P:61, reading C3).
//
// One CTA = one (pair, modulus).  L = 2^LOGL, each of NT = L/E threads holds
// E = 2^LOGE residues in registers.  The index bits are processed top-down
// in "phases" of LOGE bits done entirely in registers; between phases the
// residues are transposed through shared memory (XOR swizzle
// addr = i ^ ((i >> LOGE) & 31), conflict-free for every distribution used);
// the S = (LOGL - LOGE) mod LOGE leftover bits are lane bits and are done with
// warp shuffles.  Forward = decimation in frequency (natural -> bit-reversed
// order, distribution Df), pointwise product with the template spectrum in the
// same distribution (so each thread only needs its own E template values, kept
// in registers), inverse = decimation in time (bit-reversed -> natural, D0).
// The template spectrum is NTT(t reversed) * L^{-1} in Montgomery form, so the
// product is one Montgomery multiply and no 1/L pass is needed.
//
// Twiddles: stage with span h uses the length-2h table w_{2h}^j (uint2 value +
// Shoup companion, per-length compact tables in global memory, L1-resident).
#include <cstdlib>

#include "ntt_core.cuh"

namespace {

template <int LOGL, int LOGE>
constexpr int min_blocks() {  // >= 1024 resident threads per SM -> at most 64 registers
    return (1 << (LOGL - LOGE)) >= 1024 ? 1 : 1024 / (1 << (LOGL - LOGE));
}

// shared memory: buf [L] (transposes) | Ts [L] (FROM_T) | keep [L] (two primes)
template <int LOGL, int LOGE, int NPRIMES, bool FROM_T>
__global__ void __launch_bounds__(1 << (LOGL - LOGE), min_blocks<LOGL, LOGE>()) corr_fast_kernel(FastArgs A) {
    using G = Geo<LOGL, LOGE>;
    extern __shared__ uint32_t buf[];
    uint32_t *Ts = buf + G::L;
    uint32_t *keep = buf + (FROM_T ? 2 : 1) * G::L;
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x;
    uint32_t v[G::E];
    correlate_one_prime<LOGL, LOGE, 0, FROM_T>(v, buf, Ts, t, A, b);
    if constexpr (NPRIMES == 2) {
#pragma unroll
        for (int m = 0; m < G::E; ++m) keep[m * G::NT + t] = v[m];
        correlate_one_prime<LOGL, LOGE, 1, FROM_T>(v, buf, Ts, t, A, b);
    }
    int64_t bv = INT64_MIN;
    int32_t bi = 0x7FFFFFFF;
    int64_t *rout = A.r ? A.r + b * A.M : nullptr;
#pragma unroll
    for (int m = 0; m < G::E; ++m) {
        const int i = G::idx(0, t, m);
        int64_t val;
        if constexpr (NPRIMES == 1) {
            val = v[m] > P1 / 2 ? (int64_t)v[m] - (int64_t)P1 : (int64_t)v[m];
        } else {
            // r = a1 + p1 * ((a2 - a1) p1^{-1} mod p2), centred in (-p1 p2 / 2, p1 p2 / 2]
            const uint64_t a1 = keep[m * G::NT + t], a2 = v[m];
            const uint64_t d = (a2 + P2 - (a1 % P2)) % P2;
            const uint64_t u = (d * TM_P1_INV_MOD_P2) % P2;
            const uint64_t z = a1 + (uint64_t)P1 * u;
            const uint64_t PP = (uint64_t)P1 * P2;
            val = z > PP / 2 ? (int64_t)(z - PP) : (int64_t)z;
        }
        if (i < A.M) {
            if (rout) rout[i] = val;
            amax(bv, bi, val, i);
        }
    }
    if (A.resid) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            amax(bv, bi, ov, oi);
        }
        __syncthreads();  // buf reuse
        int64_t *sv = reinterpret_cast<int64_t *>(buf);
        int32_t *si = reinterpret_cast<int32_t *>(sv + 32);
        const int w = t >> 5, l = t & 31;
        if (l == 0) { sv[w] = bv; si[w] = bi; }
        __syncthreads();
        if (w == 0) {
            constexpr int NW = (G::NT + 31) / 32;
            bv = l < NW ? sv[l] : INT64_MIN;
            bi = l < NW ? si[l] : 0x7FFFFFFF;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                amax(bv, bi, ov, oi);
            }
            if (l == 0) A.resid[b * 2 + A.jmod] = bi;
        }
    }
}

// tm_fold_template for the fast layout: Montgomery-scaled spectra in Df order
template <int LOGL, int LOGE, int NPRIMES>
__global__ void __launch_bounds__(1 << (LOGL - LOGE), min_blocks<LOGL, LOGE>()) template_fast_kernel(FastArgs A) {
    using G = Geo<LOGL, LOGE>;
    extern __shared__ uint32_t buf[];
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x;
    uint32_t T[G::E];
    template_spectrum<LOGL, LOGE, 0>(T, buf, t, A, b);
    uint32_t *dst = A.tf_out + (b * A.np + 0) * A.tf_prime + A.tf_off;
#pragma unroll
    for (int m = 0; m < G::E; ++m) dst[m * G::NT + t] = T[m];
    if constexpr (NPRIMES == 2) {
        template_spectrum<LOGL, LOGE, 1>(T, buf, t, A, b);
        dst = A.tf_out + (b * A.np + 1) * A.tf_prime + A.tf_off;
#pragma unroll
        for (int m = 0; m < G::E; ++m) dst[m * G::NT + t] = T[m];
    }
}

// ---------------------------------------------------------------------------
// One CTA per PAIR (both moduli) for the paper's shape: y1 cyclic with L1 = M1 and
// L2 = 2 L1 (M = K, K | N, K a power of two).  The template is transformed once,
// at L2: the first L1 entries of its bit-reversed spectrum are exactly the
// length-L1 spectrum of t reversed mod L1 (even frequencies, support of t_rev
// does not collide when folded since K <= L1).  NT = L2/16 = L1/8 threads:
// y2 uses 16 residues per thread (Geo<L2,4>), y1 uses 8 (Geo<L1,3>).
// Template spectra live in shared memory in the order each transform reads
// them: Ts2[m * NT + t] (register order of Geo<L2,4>), Ts1[i] natural
// bit-reversed index (read as Ts1[(t << 3) | m], two LDS.128 per thread).
// FROM_T = false reads the same two arrays from tf ([batch][L2 + L1] u32).
// ---------------------------------------------------------------------------
template <int LOGL2, bool FROM_T>
__global__ void __launch_bounds__(1 << (LOGL2 - 4), min_blocks<LOGL2, 4>()) corr_pair_kernel(FastArgs A) {
    constexpr int LOGL1 = LOGL2 - 1;
    using G2 = Geo<LOGL2, 4>;
    static_assert(G2::NT == Geo<LOGL1, 3>::NT, "thread counts must match");
    extern __shared__ uint32_t buf[];
    uint32_t *Ts2 = buf + G2::L;
    uint32_t *Ts1 = Ts2 + G2::L;
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x;
    const uint32_t *ts2, *ts1;
    if constexpr (FROM_T) {
        pair_template_to_smem<LOGL2>(buf, Ts2, Ts1, t, A, b);
        __syncthreads();
        ts2 = Ts2;
        ts1 = Ts1;
    } else {
        ts2 = A.tf + b * A.tf_prime;
        ts1 = ts2 + G2::L;
    }
    pair_modulus2<LOGL2>(buf, ts2, t, A, b);
    pair_modulus1<LOGL2>(buf, ts1, t, A, b);
}

// tm_fold_template for pair-kernel plans: [batch][L2 (register order, * L2^-1 R) + L1 (br order, * L1^-1 R)]
template <int LOGL2>
__global__ void __launch_bounds__(1 << (LOGL2 - 4), min_blocks<LOGL2, 4>()) template_pair_kernel(FastArgs A) {
    constexpr int LOGL1 = LOGL2 - 1;
    using G2 = Geo<LOGL2, 4>;
    constexpr int NT = G2::NT;
    extern __shared__ uint32_t buf[];
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x;
    uint32_t T[16];
    template_spectrum_raw<LOGL2, 4, 0>(T, buf, t, A, b);
    uint32_t *dst = A.tf_out + b * A.tf_prime;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        dst[m * NT + t] = shoup_lz(T[m], A.cL[0], A.cLs[0], P1);
        const int i = (t << 4) | m;  // y1's register order (see pair_template_to_smem)
        if (i < (1 << LOGL1)) dst[G2::L + (i & 7) * NT + (i >> 3)] = shoup_lz(T[m], A.cL1, A.cL1s, P1);
    }
}

template <int LOGL2>
int launch_pair(const FastArgs &A, int64_t batch, bool from_t, bool template_only, cudaStream_t s) {
    using G2 = Geo<LOGL2, 4>;
    if (template_only) {
        const size_t smem = (size_t)G2::L * 4;
        auto k = template_pair_kernel<LOGL2>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<(unsigned)batch, G2::NT, smem, s>>>(A);
        TM_CHECK_LAUNCH("tm_fold_template: template_pair_kernel");
        return TM_OK;
    }
    const size_t smem = (size_t)G2::L * 4 * (from_t ? 2 : 1) + (from_t ? (size_t)G2::L * 2 : 0);
    if (from_t) {
        auto k = corr_pair_kernel<LOGL2, true>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<(unsigned)batch, G2::NT, smem, s>>>(A);
    } else {
        auto k = corr_pair_kernel<LOGL2, false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<(unsigned)batch, G2::NT, smem, s>>>(A);
    }
    TM_CHECK_LAUNCH("tm_correlate: corr_pair_kernel");
    return TM_OK;
}

int dispatch_pair(int logL2, const FastArgs &A, int64_t batch, bool from_t, bool template_only, cudaStream_t s) {
    switch (logL2) {
        case 10: return launch_pair<10>(A, batch, from_t, template_only, s);
        case 11: return launch_pair<11>(A, batch, from_t, template_only, s);
        case 12: return launch_pair<12>(A, batch, from_t, template_only, s);
        case 13: return launch_pair<13>(A, batch, from_t, template_only, s);
        case 14: return launch_pair<14>(A, batch, from_t, template_only, s);
        default: tm_set_error("pair NTT: unsupported length 2^%d", logL2); return TM_EUNSUPPORTED;
    }
}

template <int LOGL, int LOGE, int NP>
int launch_corr(const FastArgs &A, int64_t batch, bool from_t, cudaStream_t s) {
    using G = Geo<LOGL, LOGE>;
    const size_t smem = (size_t)G::L * 4 * (1 + (from_t ? 1 : 0) + (NP == 2 ? 1 : 0));
    if (from_t) {
        auto k = corr_fast_kernel<LOGL, LOGE, NP, true>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<(unsigned)batch, G::NT, smem, s>>>(A);
    } else {
        auto k = corr_fast_kernel<LOGL, LOGE, NP, false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<(unsigned)batch, G::NT, smem, s>>>(A);
    }
    TM_CHECK_LAUNCH("tm_correlate: corr_fast_kernel");
    return TM_OK;
}

template <int LOGL, int LOGE, int NP>
int launch_template(const FastArgs &A, int64_t batch, cudaStream_t s) {
    using G = Geo<LOGL, LOGE>;
    const size_t smem = (size_t)G::L * 4;
    auto k = template_fast_kernel<LOGL, LOGE, NP>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)batch, G::NT, smem, s>>>(A);
    TM_CHECK_LAUNCH("tm_fold_template: template_fast_kernel");
    return TM_OK;
}

template <int NP>
int dispatch_corr(int logL, const FastArgs &A, int64_t batch, bool from_t, cudaStream_t s) {
    switch (logL) {
        case 9: return launch_corr<9, 4, NP>(A, batch, from_t, s);
        case 10: return launch_corr<10, 4, NP>(A, batch, from_t, s);
        case 11: return launch_corr<11, 4, NP>(A, batch, from_t, s);
        case 12: return launch_corr<12, 4, NP>(A, batch, from_t, s);
        case 13: return launch_corr<13, 4, NP>(A, batch, from_t, s);
        case 14: return launch_corr<14, 4, NP>(A, batch, from_t, s);
        default: tm_set_error("fast NTT: unsupported length 2^%d", logL); return TM_EUNSUPPORTED;
    }
}

template <int NP>
int dispatch_template(int logL, const FastArgs &A, int64_t batch, cudaStream_t s) {
    switch (logL) {
        case 9: return launch_template<9, 4, NP>(A, batch, s);
        case 10: return launch_template<10, 4, NP>(A, batch, s);
        case 11: return launch_template<11, 4, NP>(A, batch, s);
        case 12: return launch_template<12, 4, NP>(A, batch, s);
        case 13: return launch_template<13, 4, NP>(A, batch, s);
        case 14: return launch_template<14, 4, NP>(A, batch, s);
        default: tm_set_error("fast NTT: unsupported length 2^%d", logL); return TM_EUNSUPPORTED;
    }
}

void fill_common(const tm_plan_s *p, int logL, FastArgs &A) {
    tm_ntt_tables tabs;
    tm_ntt_tables_get(p->device, &tabs);
    for (int pi = 0; pi < 2; ++pi) {
        A.twf[pi] = tabs.tw2[pi][0];
        A.twi[pi] = tabs.tw2[pi][1];
        const uint64_t P = TM_PRIMES[pi];
        // c = L^{-1} * 2^32 mod p
        uint64_t Linv = 1, base = ((uint64_t)1 << logL) % P, e = P - 2;
        while (e) { if (e & 1) Linv = (unsigned __int128)Linv * base % P; base = (unsigned __int128)base * base % P; e >>= 1; }
        const uint64_t c = (unsigned __int128)Linv * (((unsigned __int128)1 << 32) % P) % P;
        A.cL[pi] = (uint32_t)c;
        A.cLs[pi] = (uint32_t)(((unsigned __int128)c << 32) / P);
    }
    A.tf_prime = p->tf_elems;
    A.np = p->n_primes;
}

}  // namespace

// c = L^{-1} * 2^32 mod p (Montgomery-scaled inverse length) and its Shoup companion
void tm_mont_linv(int logL, uint32_t p, uint32_t *c, uint32_t *cs) {
    const uint64_t P = p;
    uint64_t Linv = 1, base = ((uint64_t)1 << logL) % P, e = P - 2;
    while (e) { if (e & 1) Linv = (unsigned __int128)Linv * base % P; base = (unsigned __int128)base * base % P; e >>= 1; }
    const uint64_t v = (unsigned __int128)Linv * (((unsigned __int128)1 << 32) % P) % P;
    *c = (uint32_t)v;
    *cs = (uint32_t)(((unsigned __int128)v << 32) / P);
}

// the paper's shape (M = K | N, K a power of two): one CTA per pair, shared template
static bool pair_ok(const tm_plan_s *p) {
    return p->n_primes == 1 && p->logL2 == p->logL1 + 1 && p->nload1 == p->M1 && p->L1 == p->M1 &&
           p->logL2 >= 10 && p->logL2 <= 14;
}

static void fill_pair(const tm_plan_s *p, FastArgs &A) {
    fill_common(p, p->logL2, A);
    const uint64_t P = TM_P1;
    uint64_t Linv = 1, base = ((uint64_t)1 << p->logL1) % P, e = P - 2;
    while (e) { if (e & 1) Linv = (unsigned __int128)Linv * base % P; base = (unsigned __int128)base * base % P; e >>= 1; }
    const uint64_t c = (unsigned __int128)Linv * (((unsigned __int128)1 << 32) % P) % P;
    A.cL1 = (uint32_t)c;
    A.cL1s = (uint32_t)(((unsigned __int128)c << 32) / P);
}

bool tm_fast_corr_ok(const tm_plan_s *p) {
    return p->dtype == TM_I8 && p->logL1 >= 9 && p->logL1 <= 14 && p->logL2 >= 9 && p->logL2 <= 14 &&
           p->n_primes >= 1 && p->n_primes <= 2;
}

// tf layout (fast plans): u32 [batch][n_primes][L1 + L2]; slot 0 = y1's length, slot 1 = y2's
int tm_fast_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s) {
    if (pair_ok(p)) {
        FastArgs A{};
        fill_pair(p, A);
        A.t = (const int8_t *)t; A.K = p->K;
        A.tf_out = (uint32_t *)tf;
        return dispatch_pair(p->logL2, A, batch, false, true, s);
    }
    for (int j = 0; j < 2; ++j) {
        const int logL = j ? p->logL2 : p->logL1;
        FastArgs A{};
        fill_common(p, logL, A);
        A.t = (const int8_t *)t; A.K = p->K;
        A.tf_out = (uint32_t *)tf;
        A.tf_off = j ? p->L1 : 0;
        int rc = p->n_primes == 2 ? dispatch_template<2>(logL, A, batch, s) : dispatch_template<1>(logL, A, batch, s);
        if (rc) return rc;
    }
    return TM_OK;
}

int tm_fast_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *t, const void *tf,
                      int64_t batch, void *r1, void *r2, int32_t *resid, cudaStream_t s) {
    if (pair_ok(p)) {
        FastArgs A{};
        fill_pair(p, A);
        A.y1 = (const int32_t *)y1; A.y2 = (const int32_t *)y2;
        A.ldy1 = p->len_y1; A.ldy2 = p->len_y2;
        A.nload1 = p->nload1; A.nload2 = p->nload2;
        A.M1 = p->M1; A.M2 = p->M2;
        A.r1 = (int64_t *)r1; A.r2 = (int64_t *)r2;
        A.resid = resid;
        A.t = (const int8_t *)t; A.K = p->K;
        A.tf = (const uint32_t *)tf;
        return dispatch_pair(p->logL2, A, batch, t != nullptr, false, s);
    }
    for (int j = 0; j < 2; ++j) {
        const int logL = j ? p->logL2 : p->logL1;
        FastArgs A{};
        fill_common(p, logL, A);
        A.y = (const int32_t *)(j ? y2 : y1);
        A.ldy = j ? p->len_y2 : p->len_y1;
        A.M = j ? p->M2 : p->M1;
        A.nload = j ? p->nload2 : p->nload1;
        A.t = (const int8_t *)t; A.K = p->K;
        A.tf = (const uint32_t *)tf;
        A.tf_off = j ? p->L1 : 0;
        A.r = (int64_t *)(j ? r2 : r1);
        A.resid = resid;
        A.jmod = j;
        const bool from_t = (t != nullptr);
        int rc = p->n_primes == 2 ? dispatch_corr<2>(logL, A, batch, from_t, s)
                                  : dispatch_corr<1>(logL, A, batch, from_t, s);
        if (rc) return rc;
    }
    return TM_OK;
}
