// ntt_core.cuh -- device primitives of the register-resident NTT correlation
// (Algorithm 1 steps 4-7, read as the correlation of P:61,
// reading C3).  Shared by corr_fast.cu (stand-alone kernels) and fold_tma.cu
// (NTT warps inside the fused fold kernel).  See corr_fast.cu for the design.
#pragma once
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

// Barrier policies: the whole CTA, or a named barrier over the NT threads of an
// NTT warp group inside a larger (warp-specialised) CTA.
struct CtaBar {
    static __device__ __forceinline__ void sync() { __syncthreads(); }
};
template <int ID, int N>
struct NamedBar {
    static __device__ __forceinline__ void sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory"); }
};

template <int LOGL, int LOGE, class Bar>
__device__ __forceinline__ void transpose(uint32_t (&v)[1 << LOGE], uint32_t *buf, int t, int kfrom, int kto) {
    using G = Geo<LOGL, LOGE>;
    Bar::sync();
#pragma unroll
    for (int m = 0; m < G::E; ++m) buf[G::swz(G::idx(kfrom, t, m))] = v[m];
    Bar::sync();
#pragma unroll
    for (int m = 0; m < G::E; ++m) v[m] = buf[G::swz(G::idx(kto, t, m))];
}

// forward DIF: input in D0 (natural), output in Df (bit-reversed index (t<<LOGE)|m)
template <int LOGL, int LOGE, class Bar = CtaBar>
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
        transpose<LOGL, LOGE, Bar>(v, buf, t, k, k + 1);
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
template <int LOGL, int LOGE, class Bar = CtaBar>
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
        transpose<LOGL, LOGE, Bar>(v, buf, t, k + 1, k);
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
template <int LOGL, int LOGE, int PI, class Bar = CtaBar>
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
    dif<LOGL, LOGE, Bar>(T, buf, t, A.twf[PI], p);
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
template <int NT, class Bar = CtaBar>
__device__ __forceinline__ void block_argmax_store(int64_t bv, int32_t bi, uint32_t *buf, int32_t *out, int t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        amax(bv, bi, ov, oi);
    }
    Bar::sync();
    int64_t *sv = reinterpret_cast<int64_t *>(buf);
    int32_t *si = reinterpret_cast<int32_t *>(sv + 32);
    const int w = t >> 5, l = t & 31;
    if (l == 0) { sv[w] = bv; si[w] = bi; }
    Bar::sync();
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
    Bar::sync();
}

template <int LOGL2, class Bar = CtaBar>
__device__ __noinline__ void pair_template_to_smem(uint32_t *buf, uint32_t *Ts2, uint32_t *Ts1, int t,
                                                   const FastArgs &A, int64_t b) {
    constexpr int LOGL1 = LOGL2 - 1;
    constexpr int NT = Geo<LOGL2, 4>::NT;
    uint32_t T[16];
    template_spectrum_raw<LOGL2, 4, 0, Bar>(T, buf, t, A, b);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        Ts2[m * NT + t] = shoup_lz(T[m], A.cL[0], A.cLs[0], P1);  // * L2^{-1} R
        // bit-reversed index i = (t << 4) | m < L1 is element (i >> 3, i & 7) of y1's
        // final distribution (Geo<L1,3>): store in that register order (2-way conflicts)
        const int i = (t << 4) | m;
        if (i < (1 << LOGL1)) Ts1[(i & 7) * NT + (i >> 3)] = shoup_lz(T[m], A.cL1, A.cL1s, P1);  // * L1^{-1} R
    }
}

template <int LOGL2, class Bar = CtaBar>
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
    dif<LOGL2, 4, Bar>(v, buf, t, A.twf[0], p);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = montmul<0>(v[m], ts2[m * NT + t]);
    dit<LOGL2, 4, Bar>(v, buf, t, A.twi[0], p);
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
    block_argmax_store<NT, Bar>(bv, bi, buf, A.resid ? A.resid + b * 2 + 1 : nullptr, t);
}

template <int LOGL2, class Bar = CtaBar>
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
    dif<LOGL1, 3, Bar>(v, buf, t, A.twf[0], p);
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = montmul<0>(v[m], ts1[m * NT + t]);
    dit<LOGL1, 3, Bar>(v, buf, t, A.twi[0], p);
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
    block_argmax_store<NT, Bar>(bv, bi, buf, A.resid ? A.resid + b * 2 + 0 : nullptr, t);
}


}  // namespace
