// fft_f32.cu -- correlation + argmax for real-valued (float32) pairs
// (Algorithm 1 steps 4-7, read as the correlation of P:61,
// reading C3) with register-resident complex fp32 FFTs.
//
// Both folded signals share one complex transform: with z = y1 + i y2 (each
// zero beyond its Mj + K - 1 entries read, reading C4) and T the spectrum of
// the reversed, zero-padded template t_rev[i] = t[(L - i) mod L],
//     IFFT(FFT(z) . T) = r1 + i r2,
// because the correlation is linear in the signal and r1, r2 are real (the
// real part is y1's correlation, the imaginary part y2's); L = 2^ceil(log2(
// M2 + K - 1)) >= Mj + K - 1, so no needed term wraps.  Per pair: one forward
// transform of the template (tm_fold_template, kept in HBM in the transform's
// register order) and one forward + one inverse transform of z.
//
// Transform layout (the NTT kernels' scheme, corr_fast.cu): L = 2^LOGL, each of
// NT = L / 16 threads holds 16 complex values in registers; index bits are
// processed 4 at a time in registers with XOR-swizzled shared-memory
// transposes (one interleaved float2 plane) between phases, leftover bits by warp
// shuffles.  Forward = decimation in frequency (natural -> bit-reversed),
// inverse = decimation in time (bit-reversed -> natural).  Twiddles: float2
// tables built in double precision on the host, w_n^j at offset n/2 - 1.
// Error: O(log2 L) fp32 roundings per output, ~1e-6 of max |r| at cfg3 sizes,
// inside reading C15's 1e-5 normwise tolerance (test_f32_*, test_cfg3_*).
//
// Transforms longer than one CTA's registers (L = 2^15 .. 2^18, i.e. K up to
// 2^17; Table 2's N = 2^26, K = 2^16 needs L = 2^17): the four-step
// split L = R S, S = 2^14 segment, R = 2 .. 16, index n = s + S r,
// frequency k = k2 + R k1 (decimation in frequency):
//   pass A   b_s[k2] = w_L^(s k2) sum_r x[s + S r] w_R^(r k2)    (R-point DFT per s,
//            one thread per s, written transposed: segment k2 holds b_.[k2])
//   pass B   per segment k2: the register-resident length-S DIF (above) gives
//            X[k2 + R k1] in the kernel's bit-reversed register order;
// the correlation multiplies by the template spectrum in the same order, then
// inverts: pass B^-1 (per segment, DIT back to natural s) and pass A^-1
//   out[s + S r] = sum_k2 c_s[k2] w_L^(-s k2) w_R^(-r k2)
// with the argmax as order-preserving packed keys (float key, ~index) per pair
// and modulus.  Twiddles w_L^j come from sincospif of the exact fraction 2j/L.
#include <cmath>
#include <mutex>
#include <vector>

#include "tm_internal.cuh"

namespace {

constexpr int LOGE = 4, E = 1 << LOGE;
constexpr int FFT_MAX_LOGL = 14;

template <int LOGL>
struct FGeo {
    static constexpr int L = 1 << LOGL, NT = L >> LOGE;
    static constexpr int H = (LOGL - LOGE) / LOGE, S = (LOGL - LOGE) % LOGE;
    static __device__ __forceinline__ int idx(int k, int t, int m) {
        if (k == H) return (t << LOGE) | m;
        const int blo = LOGL - (k + 1) * LOGE;
        return ((t >> blo) << (blo + LOGE)) | (m << blo) | (t & ((1 << blo) - 1));
    }
    static __device__ __forceinline__ int swz(int i) { return i ^ ((i >> LOGE) & 31); }
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

// c_root[dir][j] = exp(-+2 pi i j / 128) (dir 0: forward, 1: inverse), uploaded by
// ftables.  A twiddle w_n^(a 2^b + c) of an in-register layer is w_n^c (one table
// load per layer) times w_n^(a 2^b), a root of order <= 128 whose index is a
// compile-time constant after unrolling (a constant-bank operand, no load).
__constant__ float2 c_root[2][128];
template <int DIR>
__device__ __forceinline__ float2 tw_mul(float2 base, int j128) {
    if (j128 == 0) return base;
    if (j128 == 32) return DIR ? make_float2(-base.y, base.x) : make_float2(base.y, -base.x);  // * (+-i)
    return cmul(base, c_root[DIR][j128]);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

template <int LOGL>
__device__ __forceinline__ void ftranspose(float2 (&v)[E], float *br, float *bi, int t, int kf, int kt) {
    using G = FGeo<LOGL>;
    // one interleaved float2 plane over br .. br + 2L (bi = br + L): one 8-byte
    // access per element; the swizzle keeps each half-warp's 16 indices distinct
    // mod 16 (the 8-byte access's bank-conflict condition)
    (void)bi;
    float2 *buf = reinterpret_cast<float2 *>(br);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m) buf[G::swz(G::idx(kf, t, m))] = v[m];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = buf[G::swz(G::idx(kt, t, m))];
}

// forward DIF: natural (D0) -> bit-reversed (Df: index (t << LOGE) | m)
template <int LOGL>
__device__ __forceinline__ void fdif(float2 (&v)[E], float *br, float *bi, int t, const float2 *__restrict__ tw) {
    using G = FGeo<LOGL>;
#pragma unroll
    for (int k = 0; k < G::H; ++k) {
        const int blo = LOGL - (k + 1) * LOGE;
        const int tlow = t & ((1 << blo) - 1);
#pragma unroll
        for (int u = LOGE - 1; u >= 0; --u) {
            const int h = 1 << u;
            const float2 *tab = tw + ((1 << (blo + u)) - 1);
            const float2 base = __ldg(tab + tlow);  // w_n^tlow, n = 2^(blo + u + 1)
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if (m & h) continue;
                const float2 w = tw_mul<0>(base, (m & (h - 1)) * 64 / h);  // w_n^((m & (h-1)) 2^blo + tlow)
                const float2 X = v[m], Y = v[m | h];
                v[m] = cadd(X, Y);
                v[m | h] = cmul(csub(X, Y), w);
            }
        }
        ftranspose<LOGL>(v, br, bi, t, k, k + 1);
    }
#pragma unroll
    for (int sb = G::S - 1; sb >= 0; --sb) {
        const float2 *tab = tw + ((1 << (LOGE + sb)) - 1);
        const bool upper = (t >> sb) & 1;
        const int tl = t & ((1 << sb) - 1);
        const float2 base = __ldg(tab + (tl << LOGE));  // w_n^(16 tl), n = 2^(LOGE + sb + 1)
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const float ox = __shfl_xor_sync(0xffffffffu, v[m].x, 1 << sb);
            const float oy = __shfl_xor_sync(0xffffffffu, v[m].y, 1 << sb);
            const float2 o = make_float2(ox, oy);
            if (upper) v[m] = cmul(csub(o, v[m]), tw_mul<0>(base, m * (128 >> (LOGE + sb + 1))));
            else v[m] = cadd(v[m], o);
        }
    }
#pragma unroll
    for (int u = LOGE - 1; u >= 0; --u) {
        const int h = 1 << u;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            if (m & h) continue;
            const float2 X = v[m], Y = v[m | h];
            v[m] = cadd(X, Y);
            v[m | h] = tw_mul<0>(csub(X, Y), (m & (h - 1)) * 64 / h);  // w_2h^(m & (h-1))
        }
    }
}

// inverse DIT: bit-reversed (Df) -> natural (D0), unscaled
template <int LOGL>
__device__ __forceinline__ void fdit(float2 (&v)[E], float *br, float *bi, int t, const float2 *__restrict__ tw) {
    using G = FGeo<LOGL>;
#pragma unroll
    for (int u = 0; u < LOGE; ++u) {
        const int h = 1 << u;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            if (m & h) continue;
            const float2 Yw = tw_mul<1>(v[m | h], (m & (h - 1)) * 64 / h);
            const float2 X = v[m];
            v[m] = cadd(X, Yw);
            v[m | h] = csub(X, Yw);
        }
    }
#pragma unroll
    for (int sb = 0; sb < G::S; ++sb) {
        const float2 *tab = tw + ((1 << (LOGE + sb)) - 1);
        const bool upper = (t >> sb) & 1;
        const int tl = t & ((1 << sb) - 1);
        const float2 base = __ldg(tab + (tl << LOGE));
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const float2 send = upper ? cmul(v[m], tw_mul<1>(base, m * (128 >> (LOGE + sb + 1)))) : v[m];
            const float ox = __shfl_xor_sync(0xffffffffu, send.x, 1 << sb);
            const float oy = __shfl_xor_sync(0xffffffffu, send.y, 1 << sb);
            const float2 o = make_float2(ox, oy);
            v[m] = upper ? csub(o, send) : cadd(send, o);
        }
    }
#pragma unroll
    for (int k = G::H - 1; k >= 0; --k) {
        ftranspose<LOGL>(v, br, bi, t, k + 1, k);
        const int blo = LOGL - (k + 1) * LOGE;
        const int tlow = t & ((1 << blo) - 1);
#pragma unroll
        for (int u = 0; u < LOGE; ++u) {
            const int h = 1 << u;
            const float2 *tab = tw + ((1 << (blo + u)) - 1);
            const float2 base = __ldg(tab + tlow);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if (m & h) continue;
                const float2 Yw = cmul(v[m | h], tw_mul<1>(base, (m & (h - 1)) * 64 / h));
                const float2 X = v[m];
                v[m] = cadd(X, Yw);
                v[m | h] = csub(X, Yw);
            }
        }
    }
}

struct FftArgs {
    const float *t;          // [batch][ldt] templates (tf_template) or NULL
    int64_t ldt, K;
    const float2 *twf, *twi;
    float2 *tf;              // [batch][L] spectra in register order (m * NT + t), scaled by 1/L
    const float *y1, *y2;
    int64_t ldy1, ldy2, nload1, nload2, M1, M2;
    float *r1, *r2;          // [batch][Mj] or NULL
    int32_t *resid;          // [batch][2] or NULL
    int64_t nb;              // templates (fft_template_f32: two per CTA)
    int32_t *residues_out;   // [batch][2] or NULL: steps 8-9 fused into the epilogue
    int64_t *k_out;          // [batch] or NULL
    int64_t N, crt_wrap;
    uint32_t crt_inv;
};

// Two templates per transform (they are real): v = t_rev[b0] + i t_rev[b0 + 1],
// V = FFT(v), and with V* the conjugate of V at frequency -f (mod L):
//   T[b0](f) = (V(f) + V*(-f)) / 2,   T[b0 + 1](f) = (V(f) - V*(-f)) / (2i).
// The DIF output holds frequency bitrev((t << LOGE) | m) in thread t, register m;
// V(-f) comes from another thread, through shared memory in natural order.
template <int LOGL>
__global__ void __launch_bounds__(FGeo<LOGL>::NT, 1) fft_template_f32(FftArgs a) {
    pdl_trigger();
    pdl_wait();
    using G = FGeo<LOGL>;
    extern __shared__ float fsm[];
    float *br = fsm, *bi = fsm + G::L;
    const int t = threadIdx.x;
    const int64_t b0 = 2 * (int64_t)blockIdx.x;
    const bool two = b0 + 1 < a.nb;
    const float *tb0 = a.t + b0 * a.ldt, *tb1 = tb0 + a.ldt;
    float2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int i = G::idx(0, t, m);
        const int src = i == 0 ? 0 : G::L - i;  // t_rev[i] = t[(L - i) mod L] (reading C3)
        v[m] = make_float2(src < a.K ? tb0[src] : 0.f, (two && src < a.K) ? tb1[src] : 0.f);
    }
    fdif<LOGL>(v, br, bi, t, a.twf);
    // position p = (t << LOGE) | m holds frequency f = bitrev(p); -f (mod L) keeps f's
    // lowest set bit and flips the bits above it, i.e. p' = p ^ (hb(p) - 1) (hb: the
    // highest set bit): t' = t ^ (hb(t) - 1), m' = 15 - m for t > 0.  Stored as
    // [m][t], both the writes and the partner reads are bank-conflict free.
    __syncthreads();  // br / bi reuse
#pragma unroll
    for (int m = 0; m < E; ++m) {
        br[m * G::NT + t] = v[m].x;
        bi[m * G::NT + t] = v[m].y;
    }
    __syncthreads();
    const float s = 0.5f / (float)G::L;
    float2 *o0 = a.tf + b0 * G::L, *o1 = o0 + G::L;
    const int tp = t ? t ^ ((1 << (31 - __clz(t))) - 1) : 0;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int mp = t ? (E - 1 - m) : (m ? m ^ ((1 << (31 - __clz(m))) - 1) : 0);
        const float wx = br[mp * G::NT + tp], wy = -bi[mp * G::NT + tp];  // V*(-f)
        o0[m * G::NT + t] = make_float2((v[m].x + wx) * s, (v[m].y + wy) * s);
        if (two) o1[m * G::NT + t] = make_float2((v[m].y - wy) * s, (wx - v[m].x) * s);  // (V - V*) / 2i
    }
}

__device__ __forceinline__ void fmax_idx(float &bv, int &bi, float v, int i) {
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

template <int LOGL>
__global__ void __launch_bounds__(FGeo<LOGL>::NT, 1) fft_corr_f32(FftArgs a) {
    pdl_trigger();
    pdl_wait();
    using G = FGeo<LOGL>;
    extern __shared__ float fsm[];
    float *br = fsm, *bi = fsm + G::L;
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x;
    const float *y1 = a.y1 + b * a.ldy1, *y2 = a.y2 + b * a.ldy2;
    float2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int i = G::idx(0, t, m);
        v[m] = make_float2(i < a.nload1 ? y1[i] : 0.f, i < a.nload2 ? y2[i] : 0.f);
    }
    fdif<LOGL>(v, br, bi, t, a.twf);
    const float2 *T = a.tf + b * G::L;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = cmul(v[m], T[m * G::NT + t]);
    fdit<LOGL>(v, br, bi, t, a.twi);
    // natural order: element idx(0, t, m) = r1 (real part) + i r2 (imaginary part)
    float b1 = -INFINITY, b2 = -INFINITY;
    int i1 = 0x7FFFFFFF, i2 = 0x7FFFFFFF;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int i = G::idx(0, t, m);
        if (i < a.M1) {
            if (a.r1) a.r1[b * a.M1 + i] = v[m].x;
            fmax_idx(b1, i1, v[m].x, i);
        }
        if (i < a.M2) {
            if (a.r2) a.r2[b * a.M2 + i] = v[m].y;
            fmax_idx(b2, i2, v[m].y, i);
        }
    }
    if (!a.resid && !a.k_out && !a.residues_out) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        fmax_idx(b1, i1, __shfl_xor_sync(0xffffffffu, b1, o), __shfl_xor_sync(0xffffffffu, i1, o));
        fmax_idx(b2, i2, __shfl_xor_sync(0xffffffffu, b2, o), __shfl_xor_sync(0xffffffffu, i2, o));
    }
    __syncthreads();  // br/bi reuse
    const int w = t >> 5, l = t & 31;
    if (l == 0) { br[w] = b1; bi[w] = b2; reinterpret_cast<int *>(br + 32)[w] = i1; reinterpret_cast<int *>(bi + 32)[w] = i2; }
    __syncthreads();
    if (w == 0) {
        constexpr int NW = (G::NT + 31) / 32;
        b1 = l < NW ? br[l] : -INFINITY;
        b2 = l < NW ? bi[l] : -INFINITY;
        i1 = l < NW ? reinterpret_cast<int *>(br + 32)[l] : 0x7FFFFFFF;
        i2 = l < NW ? reinterpret_cast<int *>(bi + 32)[l] : 0x7FFFFFFF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            fmax_idx(b1, i1, __shfl_xor_sync(0xffffffffu, b1, o), __shfl_xor_sync(0xffffffffu, i1, o));
            fmax_idx(b2, i2, __shfl_xor_sync(0xffffffffu, b2, o), __shfl_xor_sync(0xffffffffu, i2, o));
        }
        if (l == 0) {
            if (a.resid) { a.resid[2 * b] = i1; a.resid[2 * b + 1] = i2; }
            if (a.residues_out) { a.residues_out[2 * b] = i1; a.residues_out[2 * b + 1] = i2; }
            if (a.k_out) a.k_out[b] = tm_resolve(i1, i2, a.M1, a.M2, a.crt_inv, a.N, a.crt_wrap);  // steps 8-9
        }
    }
}

// ---------------------------------------------------------------------------
// long transforms: four-step (pass A in global memory, pass B per segment)
// ---------------------------------------------------------------------------
constexpr int SEG_LOG = 14, SEG = 1 << SEG_LOG;
constexpr int LONG_MAX_LOGL = 18;

struct FtlArgs {
    const float *t;           // templates [batch][ldt] (template mode) or NULL
    int64_t ldt, K;
    const float *y1, *y2;     // folded signals (correlation mode)
    int64_t ldy1, ldy2, nload1, nload2, M1, M2;
    float2 *seg;              // [batch][R][S] segments (template mode: tf itself)
    const float2 *tf;         // [batch][R][S] template spectra, register order, scaled 1/L
    const float2 *twf, *twi;  // length-S tables (ftables)
    float *r1, *r2;           // [batch][Mj] or NULL
    unsigned long long *keys; // [batch][2] packed argmax keys (correlation mode)
    int logL;
};

// w_L^(+-j) (DIR 0: exp(-2 pi i j / L), 1: exp(+2 pi i j / L)), j reduced mod L
template <int DIR>
__device__ __forceinline__ float2 wL(int64_t j, int logL) {
    const int64_t L = (int64_t)1 << logL;
    j &= (L - 1);
    float sn, cs;
    sincospif((float)(2 * j) / (float)L, &sn, &cs);  // 2j/L exact in fp32 (L <= 2^18)
    return make_float2(cs, DIR ? sn : -sn);
}

__device__ __forceinline__ unsigned long long fkey(float v, int64_t i) {
    uint32_t u = __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving
    return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)i);
}

// pass A, forward: thread = s; TEMPL: x = t_rev (real), else x = y1 + i y2
template <int LOGR, bool TEMPL>
__global__ void __launch_bounds__(256) fftl_passA(FtlArgs a) {
    pdl_trigger();
    pdl_wait();
    constexpr int R = 1 << LOGR;
    const int64_t b = blockIdx.y;
    const int64_t s = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t L = (int64_t)SEG << LOGR;
    if (!TEMPL && s == 0 && a.keys) { a.keys[2 * b] = 0; a.keys[2 * b + 1] = 0; }
    float2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t n = s + (int64_t)SEG * r;
        if (TEMPL) {
            const int64_t src = n == 0 ? 0 : L - n;  // t_rev[n] = t[(L - n) mod L] (reading C3)
            x[r] = make_float2(src < a.K ? a.t[b * a.ldt + src] : 0.f, 0.f);
        } else {
            x[r] = make_float2(n < a.nload1 ? a.y1[b * a.ldy1 + n] : 0.f, n < a.nload2 ? a.y2[b * a.ldy2 + n] : 0.f);
        }
    }
    float2 *o = a.seg + b * L + s;
#pragma unroll
    for (int k2 = 0; k2 < R; ++k2) {
        float2 acc = x[0];
#pragma unroll
        for (int r = 1; r < R; ++r) acc = cadd(acc, tw_mul<0>(x[r], ((r * k2) & (R - 1)) * (128 / R)));
        o[(int64_t)SEG * k2] = k2 ? cmul(acc, wL<0>(s * k2, a.logL)) : acc;
    }
}

// pass B: per (pair, segment).  TEMPL: forward DIF, store scaled by 1/L in the
// register order; else forward DIF, times the template spectrum, inverse DIT,
// store back in natural order.
template <bool TEMPL>
__global__ void __launch_bounds__(SEG / E, 1) fftl_passB(FtlArgs a) {
    pdl_trigger();
    pdl_wait();
    using G = FGeo<SEG_LOG>;
    extern __shared__ float fsm[];
    float *br = fsm, *bi = fsm + G::L;
    const int t = threadIdx.x;
    const int64_t R = (int64_t)1 << (a.logL - SEG_LOG);
    const int64_t b = blockIdx.y, k2 = blockIdx.x;
    float2 *sg = a.seg + (b * R + k2) * SEG;
    float2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = sg[G::idx(0, t, m)];
    fdif<SEG_LOG>(v, br, bi, t, a.twf);
    if (TEMPL) {
        const float sc = 1.0f / (float)((int64_t)1 << a.logL);
        __syncthreads();  // every thread has read its natural-order inputs
#pragma unroll
        for (int m = 0; m < E; ++m) sg[m * G::NT + t] = make_float2(v[m].x * sc, v[m].y * sc);
        return;
    }
    const float2 *T = a.tf + (b * R + k2) * SEG;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = cmul(v[m], T[m * G::NT + t]);
    fdit<SEG_LOG>(v, br, bi, t, a.twi);
#pragma unroll
    for (int m = 0; m < E; ++m) sg[G::idx(0, t, m)] = v[m];
}

// pass A, inverse + outputs + argmax: thread = s
template <int LOGR>
__global__ void __launch_bounds__(256) fftl_passAinv(FtlArgs a) {
    pdl_trigger();
    pdl_wait();
    constexpr int R = 1 << LOGR;
    const int64_t b = blockIdx.y;
    const int64_t s = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t L = (int64_t)SEG << LOGR;
    const float2 *in = a.seg + b * L + s;
    float2 c[R];
#pragma unroll
    for (int k2 = 0; k2 < R; ++k2) {
        const float2 v = in[(int64_t)SEG * k2];
        c[k2] = k2 ? cmul(v, wL<1>(s * k2, a.logL)) : v;
    }
    unsigned long long best[2] = {0ull, 0ull};
#pragma unroll
    for (int r = 0; r < R; ++r) {
        float2 acc = c[0];
#pragma unroll
        for (int k2 = 1; k2 < R; ++k2) acc = cadd(acc, tw_mul<1>(c[k2], ((r * k2) & (R - 1)) * (128 / R)));
        const int64_t n = s + (int64_t)SEG * r;  // acc = r1[n] + i r2[n]
        if (n < a.M1) {
            if (a.r1) a.r1[b * a.M1 + n] = acc.x;
            const unsigned long long kk = fkey(acc.x, n);
            if (kk > best[0]) best[0] = kk;
        }
        if (n < a.M2) {
            if (a.r2) a.r2[b * a.M2 + n] = acc.y;
            const unsigned long long kk = fkey(acc.y, n);
            if (kk > best[1]) best[1] = kk;
        }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ov = __shfl_xor_sync(0xffffffffu, best[j], o);
            if (ov > best[j]) best[j] = ov;
        }
        if ((threadIdx.x & 31) == 0 && best[j]) atomicMax(a.keys + 2 * b + j, best[j]);
    }
}

struct FtlOut {
    int32_t *resid, *residues_out;
    int64_t *k_out;
    int64_t N, M1, M2, crt_wrap;
    uint32_t crt_inv;
};
__global__ void fftl_keys_to_resid(const unsigned long long *keys, int64_t batch, FtlOut o) {
    pdl_trigger();
    pdl_wait();
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const int32_t m1 = (int32_t)(0xFFFFFFFFu - (uint32_t)(keys[2 * b] & 0xFFFFFFFFull));
    const int32_t m2 = (int32_t)(0xFFFFFFFFu - (uint32_t)(keys[2 * b + 1] & 0xFFFFFFFFull));
    if (o.resid) { o.resid[2 * b] = m1; o.resid[2 * b + 1] = m2; }
    if (o.residues_out) { o.residues_out[2 * b] = m1; o.residues_out[2 * b + 1] = m2; }
    if (o.k_out) o.k_out[b] = tm_resolve(m1, m2, o.M1, o.M2, o.crt_inv, o.N, o.crt_wrap);  // steps 8-9
}

template <int LOGR>
int launch_long(bool templ, const FtlArgs &A, int64_t batch, const FtlOut &out, cudaStream_t s) {
    const dim3 ga((unsigned)(SEG / 256), (unsigned)batch), gb((unsigned)(1 << LOGR), (unsigned)batch);
    const size_t smem = (size_t)2 * SEG * 4;
    cudaError_t e;
    if (templ) {
        e = launch_pdl(fftl_passA<LOGR, true>, ga, dim3(256), 0, s, A);
        if (e == cudaSuccess) e = tm_smem_attr((const void *)fftl_passB<true>, (int)smem);
        if (e == cudaSuccess) e = launch_pdl(fftl_passB<true>, gb, dim3(SEG / E), smem, s, A);
    } else {
        e = launch_pdl(fftl_passA<LOGR, false>, ga, dim3(256), 0, s, A);
        if (e == cudaSuccess) e = tm_smem_attr((const void *)fftl_passB<false>, (int)smem);
        if (e == cudaSuccess) e = launch_pdl(fftl_passB<false>, gb, dim3(SEG / E), smem, s, A);
        if (e == cudaSuccess) e = launch_pdl(fftl_passAinv<LOGR>, ga, dim3(256), 0, s, A);
        if (e == cudaSuccess && (out.resid || out.residues_out || out.k_out))
            e = launch_pdl(fftl_keys_to_resid, dim3((unsigned)((batch + 255) / 256)), dim3(256), 0, s,
                           (const unsigned long long *)A.keys, batch, out);
    }
    if (e != cudaSuccess) return tm_cuda_status(e, "fft_f32 (long transform)");
    TM_CHECK_LAUNCH("fft_f32 (long transform)");
    return TM_OK;
}

int dispatch_long(int logL, bool templ, const FtlArgs &A, int64_t batch, const FtlOut &out, cudaStream_t s) {
    switch (logL - SEG_LOG) {
        case 1: return launch_long<1>(templ, A, batch, out, s);
        case 2: return launch_long<2>(templ, A, batch, out, s);
        case 3: return launch_long<3>(templ, A, batch, out, s);
        case 4: return launch_long<4>(templ, A, batch, out, s);
        default: return TM_EUNSUPPORTED;
    }
}

std::mutex g_fmu;
struct FTabs {
    bool ready = false;
    float2 *d = nullptr;
};
FTabs g_ftabs[64];

// w_n^j = exp(-+2 pi i j / n), j < n/2, at offset n/2 - 1, for n = 2 .. 2^FFT_MAX_LOGL
int ftables(int device, const float2 **twf, const float2 **twi) {
    if (device < 0 || device >= 64) return TM_EUNSUPPORTED;
    std::lock_guard<std::mutex> lk(g_fmu);
    FTabs &F = g_ftabs[device];
    if (!F.ready) {
        TmDeviceGuard guard(device);  // tables and __constant__ roots of `device`
        const size_t n = size_t(1) << FFT_MAX_LOGL;
        std::vector<float2> h(2 * n);
        for (int dir = 0; dir < 2; ++dir)
            for (int l = 1; l <= FFT_MAX_LOGL; ++l) {
                const size_t len = size_t(1) << l;
                for (size_t j = 0; j < len / 2; ++j) {
                    const double ang = (dir ? 2.0 : -2.0) * M_PI * (double)j / (double)len;
                    h[dir * n + len / 2 - 1 + j] = make_float2((float)std::cos(ang), (float)std::sin(ang));
                }
            }
        cudaError_t e = cudaMalloc(&F.d, h.size() * sizeof(float2));
        if (e != cudaSuccess) return tm_cuda_status(e, "tm: FFT table allocation");
        e = cudaMemcpy(F.d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm: FFT table upload");
        float2 roots[2][128];
        for (int dir = 0; dir < 2; ++dir)
            for (int j = 0; j < 128; ++j) {
                const double ang = (dir ? 2.0 : -2.0) * M_PI * (double)j / 128.0;
                roots[dir][j] = make_float2((float)std::cos(ang), (float)std::sin(ang));
            }
        e = cudaMemcpyToSymbol(c_root, roots, sizeof(roots));
        if (e != cudaSuccess) return tm_cuda_status(e, "tm: FFT root upload");
        F.ready = true;
    }
    *twf = F.d;
    *twi = F.d + (size_t(1) << FFT_MAX_LOGL);
    return TM_OK;
}

template <int LOGL>
int launch_pair(bool templ, const FftArgs &A, int64_t batch, cudaStream_t s) {
    using G = FGeo<LOGL>;
    const size_t smem = (size_t)2 * G::L * 4;
    if (templ) {
        auto k = fft_template_f32<LOGL>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const cudaError_t e = launch_pdl(k, dim3((unsigned)((batch + 1) / 2)), dim3(G::NT), smem, s, A);
        if (e != cudaSuccess) return tm_cuda_status(e, "fft_template_f32");
        TM_CHECK_LAUNCH("fft_template_f32");
    } else {
        auto k = fft_corr_f32<LOGL>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const cudaError_t e = launch_pdl(k, dim3((unsigned)batch), dim3(G::NT), smem, s, A);
        if (e != cudaSuccess) return tm_cuda_status(e, "fft_corr_f32");
        TM_CHECK_LAUNCH("fft_corr_f32");
    }
    return TM_OK;
}

int dispatch(int logL, bool templ, const FftArgs &A, int64_t batch, cudaStream_t s) {
    switch (logL) {
        case 9: return launch_pair<9>(templ, A, batch, s);
        case 10: return launch_pair<10>(templ, A, batch, s);
        case 11: return launch_pair<11>(templ, A, batch, s);
        case 12: return launch_pair<12>(templ, A, batch, s);
        case 13: return launch_pair<13>(templ, A, batch, s);
        case 14: return launch_pair<14>(templ, A, batch, s);
        default: return TM_EUNSUPPORTED;
    }
}

}  // namespace

// float32 plans whose transform length fits the register kernel (L2 <= 2^14) or
// the four-step split (2^15 <= L2 <= 2^18)
bool tm_fft_f32_ok(const tm_plan_s *p) { return p->dtype == TM_F32 && p->logL2 >= 9 && p->logL2 <= LONG_MAX_LOGL; }
bool tm_fft_f32_long(const tm_plan_s *p) { return tm_fft_f32_ok(p) && p->logL2 > FFT_MAX_LOGL; }
size_t tm_fft_f32_scratch_bytes(const tm_plan_s *p, int64_t batch) {
    if (!tm_fft_f32_long(p)) return 0;
    return (size_t)batch * (size_t)p->L2 * 8 + (size_t)batch * 16 + 256;
}

// tf [batch][L2] float2: the template spectrum (tm_fold_template for these plans)
int tm_fft_f32_template(const tm_plan_s *p, const void *t, int64_t ldt, int64_t batch, void *tf, cudaStream_t s) {
    if (!tm_fft_f32_ok(p)) return TM_EUNSUPPORTED;
    if (batch > 0x7FFFFFFF) return TM_EUNSUPPORTED;
    FftArgs A{};
    int rc = ftables(p->device, &A.twf, &A.twi);
    if (rc) return rc;
    if (p->logL2 > FFT_MAX_LOGL) {  // four-step: pass A into tf, pass B in place
        FtlArgs B{};
        B.t = (const float *)t; B.ldt = ldt; B.K = p->K;
        B.seg = (float2 *)tf;
        B.twf = A.twf; B.twi = A.twi;
        B.logL = p->logL2;
        return dispatch_long(p->logL2, true, B, batch, FtlOut{}, s);
    }
    A.t = (const float *)t; A.ldt = ldt; A.K = p->K;
    A.tf = (float2 *)tf;
    A.nb = batch;
    return dispatch(p->logL2, true, A, batch, s);
}

int tm_fft_f32_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *tf, int64_t batch,
                         void *r1, void *r2, int32_t *resid, void *scratch, cudaStream_t s, int32_t *residues_out,
                         int64_t *k_out) {
    if (!tm_fft_f32_ok(p)) return TM_EUNSUPPORTED;
    if (batch > 0x7FFFFFFF) return TM_EUNSUPPORTED;
    FftArgs A{};
    int rc = ftables(p->device, &A.twf, &A.twi);
    if (rc) return rc;
    if (p->logL2 > FFT_MAX_LOGL) {
        if (!scratch) { tm_set_error("tm_correlate: workspace required for this plan"); return TM_EINVAL; }
        if (batch > 65535) return TM_EUNSUPPORTED;
        FtlArgs B{};
        B.y1 = (const float *)y1; B.y2 = (const float *)y2;
        B.ldy1 = p->len_y1; B.ldy2 = p->len_y2;
        B.nload1 = p->M1 + p->K - 1; B.nload2 = p->M2 + p->K - 1;  // reading C4
        B.M1 = p->M1; B.M2 = p->M2;
        B.seg = (float2 *)scratch;
        B.keys = (unsigned long long *)((char *)scratch + (size_t)batch * p->L2 * 8);
        B.tf = (const float2 *)tf;
        B.twf = A.twf; B.twi = A.twi;
        B.r1 = (float *)r1; B.r2 = (float *)r2;
        B.logL = p->logL2;
        FtlOut out{resid, residues_out, k_out, p->N, p->M1, p->M2, p->crt_wrap, p->crt_inv};
        return dispatch_long(p->logL2, false, B, batch, out, s);
    }
    A.tf = (float2 *)const_cast<void *>(tf);
    A.y1 = (const float *)y1; A.y2 = (const float *)y2;
    A.ldy1 = p->len_y1; A.ldy2 = p->len_y2;
    A.nload1 = p->M1 + p->K - 1; A.nload2 = p->M2 + p->K - 1;  // reading C4
    A.M1 = p->M1; A.M2 = p->M2;
    A.r1 = (float *)r1; A.r2 = (float *)r2;
    A.resid = resid;
    A.residues_out = residues_out; A.k_out = k_out;
    A.N = p->N; A.crt_wrap = p->crt_wrap; A.crt_inv = p->crt_inv;
    return dispatch(p->logL2, false, A, batch, s);
}
