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

#include "tm_internal.cuh"

namespace {

constexpr uint32_t P1 = TM_P1, P2 = TM_P2;

struct FastArgs {
    const int32_t *y;      // [batch][ldy]
    int64_t ldy;
    int64_t nload;         // entries of y used (M + K - 1, or M for the cyclic y1 case)
    int64_t M;             // outputs k < M
    const int8_t *t;       // [batch][K]  (FROM_T)
    int64_t K;
    const uint32_t *tf;    // template spectra (FROM_TF): [batch][n_primes][tf_prime] u32
    int64_t tf_prime;      // u32 per prime per pair
    int np;                // primes in use (1 or 2)
    int64_t tf_off;        // offset of this modulus's slot inside a prime block
    uint32_t *tf_out;      // template kernel output (same layout)
    const uint2 *twf[2], *twi[2];  // forward / inverse tables per prime
    uint32_t cL[2], cLs[2];        // L^{-1} * 2^32 mod p and its Shoup companion
    int64_t *r;            // [batch][M] or NULL
    int32_t *resid;        // [batch][2] or NULL
    int jmod;              // 0 or 1 (column in resid)
    // pair kernel (both moduli in one CTA)
    const int32_t *y1, *y2;
    int64_t ldy1, ldy2, nload1, nload2, M1, M2;
    int64_t *r1, *r2;
    uint32_t cL1, cL1s;    // L1^{-1} * 2^32 mod p1 and companion
};

// Lazy (Harvey) arithmetic, valid because 4p < 2^32:
//   red2(s)  : [0, 4p) -> [0, 2p)        (one unsigned min)
//   shoup_lz : a * w mod p into [0, 2p), any a < 2^32, w < p
//   montmul  : a * b * 2^-32 mod p into [0, 2p) for a, b < 2p
__device__ __forceinline__ uint32_t red2(uint32_t s, uint32_t p2) { return min(s, s - p2); }
__device__ __forceinline__ uint32_t shoup_lz(uint32_t a, uint32_t w, uint32_t ws, uint32_t p) {
    return a * w - __umulhi(a, ws) * p;
}
template <int PI>
__device__ __forceinline__ uint32_t montmul(uint32_t a, uint32_t b) {
    constexpr uint32_t p = PI ? P2 : P1;
    constexpr uint32_t pinv = PI ? TM_P2_PINV : TM_P1_PINV;
    uint64_t t = (uint64_t)a * b;
    uint32_t m = (uint32_t)t * pinv;
    return (uint32_t)((t + (uint64_t)m * p) >> 32);
}

// twiddle load; volatile so the compiler neither merges it with the identical load
// of another transform (which would keep it live across the whole kernel) nor
// hoists it far ahead of its use
__device__ __forceinline__ uint2 ldtw(const uint2 *p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

template <int LOGL, int LOGE>
struct Geo {
    static constexpr int L = 1 << LOGL, E = 1 << LOGE, NT = L >> LOGE;
    static constexpr int H = (LOGL - LOGE) / LOGE, S = (LOGL - LOGE) % LOGE;
    // element index of (thread t, register m) in the distribution of phase k (k == H: final)
    static __device__ __forceinline__ int idx(int k, int t, int m) {
        if (k == H) return (t << LOGE) | m;
        const int blo = LOGL - (k + 1) * LOGE;
        return ((t >> blo) << (blo + LOGE)) | (m << blo) | (t & ((1 << blo) - 1));
    }
    static __device__ __forceinline__ int swz(int i) { return i ^ ((i >> LOGE) & 31); }
};

template <int LOGL, int LOGE>
__device__ __forceinline__ void transpose(uint32_t (&v)[1 << LOGE], uint32_t *buf, int t, int kfrom, int kto) {
    using G = Geo<LOGL, LOGE>;
    __syncthreads();
#pragma unroll
    for (int m = 0; m < G::E; ++m) buf[G::swz(G::idx(kfrom, t, m))] = v[m];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < G::E; ++m) v[m] = buf[G::swz(G::idx(kto, t, m))];
}

// forward DIF: input in D0 (natural), output in Df (bit-reversed index (t<<LOGE)|m)
template <int LOGL, int LOGE>
__device__ __forceinline__ void dif(uint32_t (&v)[1 << LOGE], uint32_t *buf, int t, const uint2 *__restrict__ tw,
                                    uint32_t p) {
    using G = Geo<LOGL, LOGE>;
    constexpr int E = G::E;
#pragma unroll
    for (int k = 0; k < G::H; ++k) {
        const int blo = LOGL - (k + 1) * LOGE;
        const int tlow = t & ((1 << blo) - 1);
#pragma unroll
        for (int u = LOGE - 1; u >= 0; --u) {
            const int h = 1 << u;
            const uint2 *tab = tw + ((1 << (blo + u)) - 1);
            uint2 wv[E / 2];
#pragma unroll
            for (int q = 0; q < h; ++q) wv[q] = ldtw(tab + ((q << blo) | tlow));
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if (m & h) continue;
                const uint2 w = wv[m & (h - 1)];
                const uint32_t X = v[m], Y = v[m | h];  // both in [0, 2p)
                v[m] = red2(X + Y, 2 * p);
                v[m | h] = shoup_lz(X + 2 * p - Y, w.x, w.y, p);
            }
        }
        transpose<LOGL, LOGE>(v, buf, t, k, k + 1);
    }
#pragma unroll
    for (int sb = G::S - 1; sb >= 0; --sb) {
        const int b = LOGE + sb;
        const uint2 *tab = tw + ((1 << b) - 1);
        const bool upper = (t >> sb) & 1;
        const int tl = t & ((1 << sb) - 1);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v[m], 1 << sb);
            const uint2 w = ldtw(tab + ((tl << LOGE) | m));
            const uint32_t a = upper ? o + 2 * p - v[m] : v[m] + o;
            v[m] = upper ? shoup_lz(a, w.x, w.y, p) : red2(a, 2 * p);
        }
    }
#pragma unroll
    for (int u = LOGE - 1; u >= 0; --u) {
        const int h = 1 << u;
        const uint2 *tab = tw + (h - 1);
        uint2 wv[E / 2];
#pragma unroll
        for (int q = 0; q < h; ++q) wv[q] = ldtw(tab + q);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            if (m & h) continue;
            const uint2 w = wv[m & (h - 1)];
            const uint32_t X = v[m], Y = v[m | h];
            v[m] = red2(X + Y, 2 * p);
            v[m | h] = shoup_lz(X + 2 * p - Y, w.x, w.y, p);
        }
    }
}

// inverse DIT: input in Df (bit-reversed), output in D0 (natural), unscaled
template <int LOGL, int LOGE>
__device__ __forceinline__ void dit(uint32_t (&v)[1 << LOGE], uint32_t *buf, int t, const uint2 *__restrict__ tw,
                                    uint32_t p) {
    using G = Geo<LOGL, LOGE>;
    constexpr int E = G::E;
#pragma unroll
    for (int u = 0; u < LOGE; ++u) {
        const int h = 1 << u;
        const uint2 *tab = tw + (h - 1);
        uint2 wv[E / 2];
#pragma unroll
        for (int q = 0; q < h; ++q) wv[q] = ldtw(tab + q);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            if (m & h) continue;
            const uint2 w = wv[m & (h - 1)];
            const uint32_t X = red2(v[m], 2 * p);               // inputs in [0, 4p)
            const uint32_t Yw = shoup_lz(v[m | h], w.x, w.y, p);
            v[m] = X + Yw;                                       // outputs in [0, 4p)
            v[m | h] = X + 2 * p - Yw;
        }
    }
#pragma unroll
    for (int sb = 0; sb < G::S; ++sb) {
        const int b = LOGE + sb;
        const uint2 *tab = tw + ((1 << b) - 1);
        const bool upper = (t >> sb) & 1;
        const int tl = t & ((1 << sb) - 1);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const uint2 w = ldtw(tab + ((tl << LOGE) | m));
            const uint32_t send = upper ? shoup_lz(v[m], w.x, w.y, p) : red2(v[m], 2 * p);
            const uint32_t o = __shfl_xor_sync(0xffffffffu, send, 1 << sb);
            v[m] = upper ? o + 2 * p - send : send + o;
        }
    }
#pragma unroll
    for (int k = G::H - 1; k >= 0; --k) {
        transpose<LOGL, LOGE>(v, buf, t, k + 1, k);
        const int blo = LOGL - (k + 1) * LOGE;
        const int tlow = t & ((1 << blo) - 1);
#pragma unroll
        for (int u = 0; u < LOGE; ++u) {
            const int h = 1 << u;
            const uint2 *tab = tw + ((1 << (blo + u)) - 1);
            uint2 wv[E / 2];
#pragma unroll
            for (int q = 0; q < h; ++q) wv[q] = ldtw(tab + ((q << blo) | tlow));
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if (m & h) continue;
                const uint2 w = wv[m & (h - 1)];
                const uint32_t X = red2(v[m], 2 * p);
                const uint32_t Yw = shoup_lz(v[m | h], w.x, w.y, p);
                v[m] = X + Yw;
                v[m | h] = X + 2 * p - Yw;
            }
        }
    }
}

__device__ __forceinline__ uint32_t to_residue(int32_t v, uint32_t p) {
    return v >= 0 ? (uint32_t)v : (uint32_t)((int64_t)p + v);
}

// template spectrum (unscaled, distribution Df, lazily in [0, 2p)) of t_rev[i] = t[(L - i) mod L]
template <int LOGL, int LOGE, int PI>
__device__ __forceinline__ void template_spectrum_raw(uint32_t (&T)[1 << LOGE], uint32_t *buf, int t,
                                                      const FastArgs &A, int64_t b) {
    using G = Geo<LOGL, LOGE>;
    constexpr uint32_t p = PI ? P2 : P1;
    const int8_t *tb = A.t + b * A.K;
#pragma unroll
    for (int m = 0; m < G::E; ++m) {
        const int i = G::idx(0, t, m);
        const int src = i == 0 ? 0 : G::L - i;
        T[m] = to_residue(src < A.K ? (int32_t)tb[src] : 0, p);
    }
    dif<LOGL, LOGE>(T, buf, t, A.twf[PI], p);
}

// template spectrum (Montgomery-scaled, distribution Df) of t_rev[i] = t[(L - i) mod L]
template <int LOGL, int LOGE, int PI>
__device__ __forceinline__ void template_spectrum(uint32_t (&T)[1 << LOGE], uint32_t *buf, int t, const FastArgs &A,
                                                  int64_t b) {
    using G = Geo<LOGL, LOGE>;
    constexpr uint32_t p = PI ? P2 : P1;
    const int8_t *tb = A.t + b * A.K;
#pragma unroll
    for (int m = 0; m < G::E; ++m) {
        const int i = G::idx(0, t, m);
        const int src = i == 0 ? 0 : G::L - i;
        T[m] = to_residue(src < A.K ? (int32_t)tb[src] : 0, p);
    }
    dif<LOGL, LOGE>(T, buf, t, A.twf[PI], p);
#pragma unroll
    for (int m = 0; m < G::E; ++m) T[m] = shoup_lz(T[m], A.cL[PI], A.cLs[PI], p);  // [0, 2p)
}

// separate register allocation for the template transform (noinline)
template <int LOGL, int LOGE, int PI>
__device__ __noinline__ void template_to_smem(uint32_t *buf, uint32_t *Ts, int t, const FastArgs &A, int64_t b) {
    using G = Geo<LOGL, LOGE>;
    uint32_t T[G::E];
    template_spectrum<LOGL, LOGE, PI>(T, buf, t, A, b);
#pragma unroll
    for (int m = 0; m < G::E; ++m) Ts[m * G::NT + t] = T[m];
}

// T spectrum source: FROM_T -> computed here into shared memory (register order
// m * NT + t, conflict-free); otherwise read from tf (same order) at multiply time.
template <int LOGL, int LOGE, int PI, bool FROM_T>
__device__ __forceinline__ void correlate_one_prime(uint32_t (&v)[1 << LOGE], uint32_t *buf, uint32_t *Ts, int t,
                                                    const FastArgs &A, int64_t b) {
    using G = Geo<LOGL, LOGE>;
    constexpr uint32_t p = PI ? P2 : P1;
    if constexpr (FROM_T) {
        template_to_smem<LOGL, LOGE, PI>(buf, Ts, t, A, b);
        __syncthreads();  // also keeps the y loads below from being hoisted into the template NTT
    }
    const int32_t *yb = A.y + b * A.ldy;
#pragma unroll
    for (int m = 0; m < G::E; ++m) {
        const int i = G::idx(0, t, m);
        v[m] = to_residue(i < A.nload ? yb[i] : 0, p);
    }
    dif<LOGL, LOGE>(v, buf, t, A.twf[PI], p);
    const uint32_t *src = FROM_T ? Ts : A.tf + (b * A.np + PI) * A.tf_prime + A.tf_off;
#pragma unroll
    for (int m = 0; m < G::E; ++m) v[m] = montmul<PI>(v[m], src[m * G::NT + t]);  // [0, 2p)
    dit<LOGL, LOGE>(v, buf, t, A.twi[PI], p);
#pragma unroll
    for (int m = 0; m < G::E; ++m) {  // [0, 4p) -> [0, p)
        const uint32_t r = red2(v[m], 2 * p);
        v[m] = min(r, r - p);
    }
}

__device__ __forceinline__ void amax(int64_t &bv, int32_t &bi, int64_t v, int32_t i) {
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

// block-wide (value, lowest index) max; thread 0 stores the index to *out (if non-NULL).
// Uses buf as scratch (synchronises before and after).
template <int NT>
__device__ __forceinline__ void block_argmax_store(int64_t bv, int32_t bi, uint32_t *buf, int32_t *out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        amax(bv, bi, ov, oi);
    }
    __syncthreads();
    int64_t *sv = reinterpret_cast<int64_t *>(buf);
    int32_t *si = reinterpret_cast<int32_t *>(sv + 32);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sv[w] = bv; si[w] = bi; }
    __syncthreads();
    if (w == 0) {
        constexpr int NW = (NT + 31) / 32;
        bv = l < NW ? sv[l] : INT64_MIN;
        bi = l < NW ? si[l] : 0x7FFFFFFF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            amax(bv, bi, ov, oi);
        }
        if (l == 0 && out) *out = bi;
    }
    __syncthreads();
}

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
template <int LOGL2>
__device__ __noinline__ void pair_template_to_smem(uint32_t *buf, uint32_t *Ts2, uint32_t *Ts1, int t,
                                                   const FastArgs &A, int64_t b) {
    constexpr int LOGL1 = LOGL2 - 1;
    constexpr int NT = Geo<LOGL2, 4>::NT;
    uint32_t T[16];
    template_spectrum_raw<LOGL2, 4, 0>(T, buf, t, A, b);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        Ts2[m * NT + t] = shoup_lz(T[m], A.cL[0], A.cLs[0], P1);      // * L2^{-1} R
        const int i = (t << 4) | m;                                    // bit-reversed index
        if (i < (1 << LOGL1)) Ts1[i] = shoup_lz(T[m], A.cL1, A.cL1s, P1);  // * L1^{-1} R
    }
}

template <int LOGL2>
__device__ __noinline__ void pair_modulus2(uint32_t *buf, const uint32_t *ts2, int t, const FastArgs &A, int64_t b) {
    using G2 = Geo<LOGL2, 4>;
    constexpr int NT = G2::NT;
    constexpr uint32_t p = P1;
    int64_t bv = INT64_MIN;
    int32_t bi = 0x7FFFFFFF;
    uint32_t v[16];
    const int32_t *yb = A.y2 + b * A.ldy2;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int i = G2::idx(0, t, m);
        v[m] = to_residue(i < A.nload2 ? yb[i] : 0, p);
    }
    dif<LOGL2, 4>(v, buf, t, A.twf[0], p);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = montmul<0>(v[m], ts2[m * NT + t]);
    dit<LOGL2, 4>(v, buf, t, A.twi[0], p);
    int64_t *rout = A.r2 ? A.r2 + b * A.M2 : nullptr;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const uint32_t r0 = red2(v[m], 2 * p), u = min(r0, r0 - p);
        const int i = G2::idx(0, t, m);
        const int64_t val = u > p / 2 ? (int64_t)u - (int64_t)p : (int64_t)u;
        if (i < A.M2) {
            if (rout) rout[i] = val;
            amax(bv, bi, val, i);
        }
    }
    block_argmax_store<NT>(bv, bi, buf, A.resid ? A.resid + b * 2 + 1 : nullptr);
}

template <int LOGL2>
__device__ __noinline__ void pair_modulus1(uint32_t *buf, const uint32_t *ts1, int t, const FastArgs &A, int64_t b) {
    constexpr int LOGL1 = LOGL2 - 1;
    using G1 = Geo<LOGL1, 3>;
    constexpr int NT = G1::NT;
    constexpr uint32_t p = P1;
    int64_t bv = INT64_MIN;
    int32_t bi = 0x7FFFFFFF;
    uint32_t v[8];
    const int32_t *yb = A.y1 + b * A.ldy1;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int i = G1::idx(0, t, m);
        v[m] = to_residue(i < A.nload1 ? yb[i] : 0, p);
    }
    dif<LOGL1, 3>(v, buf, t, A.twf[0], p);
    const uint4 *tv = reinterpret_cast<const uint4 *>(ts1 + (t << 3));
    const uint4 ta = tv[0], tb = tv[1];
    const uint32_t tt[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = montmul<0>(v[m], tt[m]);
    dit<LOGL1, 3>(v, buf, t, A.twi[0], p);
    int64_t *rout = A.r1 ? A.r1 + b * A.M1 : nullptr;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const uint32_t r0 = red2(v[m], 2 * p), u = min(r0, r0 - p);
        const int i = G1::idx(0, t, m);
        const int64_t val = u > p / 2 ? (int64_t)u - (int64_t)p : (int64_t)u;
        if (i < A.M1) {
            if (rout) rout[i] = val;
            amax(bv, bi, val, i);
        }
    }
    block_argmax_store<NT>(bv, bi, buf, A.resid ? A.resid + b * 2 + 0 : nullptr);
}

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
        const int i = (t << 4) | m;
        if (i < (1 << LOGL1)) dst[G2::L + i] = shoup_lz(T[m], A.cL1, A.cL1s, P1);
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
    static const bool no_pair = getenv("TM_NO_PAIR_KERNEL") != nullptr;
    if (pair_ok(p) && !no_pair) {
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
