// corr_tc.cu -- exact correlation + argmax + CRT (Algorithm 1 steps 4-9,
// PAPER.md P:98-106, correlation read as P:61, reading C3) on the 5th-generation
// tensor cores: tcgen05.mma kind::i8 (int8 x int8 -> int32 in TMEM).
//
// The correlation r_j[k] = sum_{i<K} t[i] y_j[k+i] (k < M_j) of one pair is a
// Toeplitz matrix-vector product; it is recast as a sum of small GEMMs by
// blocking both indices by P = 128:
//
//   k = P a + (P-1-b'),   i = P c + u - (P-1-b')      (b', u in [0,P))
//   r_j[P a + P-1-b'] = sum_c sum_u  A_c[b'][u] * B_c[u][a]
//   A_c[b'][u] = tp(P c + u - P + 1 + b')       (tp = t zero-extended)
//   B_c[u][a]  = y_j[P (a + c) + u]
//
// so D[b'][a] accumulates NC = floor((K+P-2)/P)+1 MMAs of shape M=128 (b'),
// K = 128 (u) over the output blocks a -- no epilogue reduction: D IS r.
// Both operands live in shared memory in the canonical no-swizzle K-major
// layout (8-row x 16-byte core matrices), and every A_c / B_c is a descriptor
// start-address offset:
//   A: S[J][s][e] = tp(16 J + s + e - 127)  (16 byte-shifted copies of the
//      template, s = b' mod 16), J = 8c + h + b'/16  ->  LBO = 256, SBO = 128,
//      +2048 B per c.  The Toeplitz row shift costs 16x the template (64 KB at
//      K = 4096), not 128x.
//   B: one MMA serves both moduli: B row rho = 2 s + j holds block s of y_j
//      (or of one 4-bit limb of it), as 8 chunks [h][rho][16 B] =
//      y_j[P s + 16 h + e].  Shifting all rows by c blocks (= 2c rows, +32c
//      bytes) shifts both streams at once, so MMA column n = 2 a + j
//      accumulates block a of r_j.  SBO = 128, LBO = 16 * rows.  A (4 KB per
//      MMA) is read once for both moduli, which keeps the shared-memory-bound
//      MMA at (4096 + 32 N) / 128 cycles (tools/mma_bench.cu).  Limbs run as
//      successive passes over a one-limb B buffer (small shared memory, so a
//      CTA of this kernel fits next to a fold CTA on the same SM).
// int8 operands are exact; y is split into 4-bit limbs when |y| > 127
// (y = sum_l 16^l v_l, top limb signed), chosen per pair from the data; the
// plan guarantees |y| <= 32767 (<= 3 limbs) and K*128*128 < 2^31 per limb.
#include <cstdlib>

#include "tm_internal.cuh"

namespace {

constexpr int P = 128;
constexpr int NTHR = 256;
constexpr int MAXLEFT = 8;  // outputs k in [P*NA, M) done by warp dot products

struct TcArgs {
    const int8_t *t;
    int64_t ldt, K;
    const int32_t *y[2];
    int64_t ldy[2], len[2], M[2];
    int NA[2];   // output blocks of each modulus done on the tensor cores
    int NMC;     // blocks per modulus in the MMA (multiple of 16, >= NA)
    int R;       // B blocks staged (NMC + NC - 1)
    int NC, JA, LMAX;
    uint32_t ncols;
    uint32_t offB, offTp, offMisc;
    int64_t *r[2];
    int32_t *resid;         // [batch][2] residues (may be NULL)
    int32_t *residues_out;  // [batch][2] (may be NULL)
    int64_t *k_out;         // [batch] (NULL: no CRT)
    int64_t N, M1, M2;
    uint32_t crt_inv;
    long long *dbg;  // optional per-CTA phase timestamps (tm_debug_tc_timestamps)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, no swizzle
}

// kind::i8 instruction descriptor: D s32, A s8, B s8, both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(P >> 4) << 24);
}

// issued by a whole (converged) warp: one elected lane executes the MMA
__device__ __forceinline__ void mma_i8(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "setp.ne.b32 q, %4, 0;\n\t"
        "@p tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, q;\n\t}" ::"r"(dt),
        "l"(ad), "l"(bd), "r"(id), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void amax(int64_t &bv, int64_t &bk, int64_t v, int64_t k) {
    if (v > bv || (v == bv && k < bk)) { bv = v; bk = k; }
}

// pack the low bytes of four int32 into one word (little-endian order)
__device__ __forceinline__ uint32_t pack4(int32_t a, int32_t b, int32_t c, int32_t d) {
    const uint32_t lo = __byte_perm((uint32_t)a, (uint32_t)b, 0x0040);
    const uint32_t hi = __byte_perm((uint32_t)c, (uint32_t)d, 0x0040);
    return __byte_perm(lo, hi, 0x5410);
}

__device__ __forceinline__ int32_t limb(int32_t v, int l, int nl) {
    return (l == nl - 1) ? (v >> (4 * l)) : ((v >> (4 * l)) & 15);
}

// Stage limb l (of nl) of y_1, y_2 (blocks s < R of P entries, zero beyond
// len_j) into the interleaved B layout: row 2 s + j.  One warp per block row:
// lane i holds entries 4i .. 4i+3 (chunk h = i / 4).  Returns this thread's
// range flags (bit 0: some |y| needs 2 limbs, bit 1: 3 limbs).
__device__ __forceinline__ int stage_y(const TcArgs &a, uint8_t *B, int64_t b, int l, int nl, int warp, int lane) {
    int flags = 0;
    const uint32_t lbo = 32u * a.R;  // bytes per chunk column h: 2 R rows of 16 B
    const int h = lane >> 2, wq = lane & 3;
    constexpr int RB = 4;                 // block rows in flight per warp
    constexpr int NW = NTHR / 32;
#pragma unroll 1
    for (int j = 0; j < 2; ++j) {
        const int32_t *yr = a.y[j] + b * a.ldy[j];
        const int64_t len = a.len[j];
        const bool al = ((((uintptr_t)yr) & 15) == 0);
        for (int s0 = warp; s0 < a.R; s0 += RB * NW) {
            int32_t v[RB][4];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const int64_t i0 = (int64_t)P * (s0 + u * NW) + 4 * lane;
                v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0;
                if (s0 + u * NW < a.R) {
                    if (al && i0 + 4 <= len) {
                        const int4 q = __ldg(reinterpret_cast<const int4 *>(yr + i0));
                        v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (i0 + e < len) v[u][e] = __ldg(yr + i0 + e);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const int s = s0 + u * NW;
                if (s >= a.R) break;
                const int32_t v0 = v[u][0], v1 = v[u][1], v2 = v[u][2], v3 = v[u][3];
                const uint32_t o1 = (uint32_t)(v0 + 128) | (uint32_t)(v1 + 128) | (uint32_t)(v2 + 128) | (uint32_t)(v3 + 128);
                const uint32_t o2 = (uint32_t)(v0 + 2048) | (uint32_t)(v1 + 2048) | (uint32_t)(v2 + 2048) | (uint32_t)(v3 + 2048);
                flags |= (o1 > 255u ? 1 : 0) | (o2 > 4095u ? 2 : 0);
                *reinterpret_cast<uint32_t *>(B + lbo * h + 16 * (2 * s + j) + 4 * wq) =
                    nl == 1 ? pack4(v0, v1, v2, v3)
                            : pack4(limb(v0, l, nl), limb(v1, l, nl), limb(v2, l, nl), limb(v3, l, nl));
            }
        }
    }
    return flags;
}

// TMEM -> registers for 8 output blocks [a0, a0 + 8) of both moduli (limb l
// of block a, modulus j is column 2 NMC l + 2 a + j), r = sum_l 16^l D_l;
// argmax with lowest k.
template <int NL>
__device__ __forceinline__ void epi_chunk(const TcArgs &a, uint32_t taddr, int a0, int brow, int64_t b,
                                          int64_t (&bv)[2], int64_t (&bk)[2]) {
    int32_t v[16 * NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) tmem_ld16(taddr + 2 * a.NMC * l + 2 * a0, v + 16 * l);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            int64_t r = 0;
#pragma unroll
            for (int l = 0; l < NL; ++l) r += (int64_t)v[16 * l + 2 * i + j] * ((int64_t)1 << (4 * l));
            const int64_t k = (int64_t)P * (a0 + i) + brow;
            if (a0 + i < a.NA[j] && k < a.M[j]) {
                if (a.r[j]) a.r[j][b * a.M[j] + k] = r;
                amax(bv[j], bk[j], r, k);
            }
        }
    }
}

__global__ void __launch_bounds__(NTHR, 2) corr_tc_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t b = blockIdx.x;
    long long tstamp[6];
    tstamp[0] = clock64();
    uint64_t *mdone = reinterpret_cast<uint64_t *>(sm + a.offMisc);   // all MMAs of the pair done
    uint32_t *tslot = reinterpret_cast<uint32_t *>(sm + a.offMisc + 8);
    int64_t *sv = reinterpret_cast<int64_t *>(sm + a.offMisc + 16);   // [8 warps][2]
    int64_t *sk = sv + 16;                                             // [8][2]
    int64_t *lv = sk + 16;                                             // [2][MAXLEFT]
    uint8_t *B = sm + a.offB;
    uint8_t *tp = sm + a.offTp;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(a.ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mdone)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- template -> tp (tp[j] = t[j - 128], zero outside [0, K)) ----
    const int tpn = 16 * a.JA + 48;
    const int8_t *tr = a.t + b * a.ldt;
    if ((a.K & 15) == 0 && ((((uintptr_t)tr) & 15) == 0)) {
        for (int i = tid; i < tpn / 16; i += NTHR) {
            const int64_t j = 16 * (int64_t)i - 128;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (j >= 0 && j < a.K) v = __ldg(reinterpret_cast<const uint4 *>(tr + j));
            reinterpret_cast<uint4 *>(tp)[i] = v;
        }
    } else {
        for (int i = tid; i < tpn; i += NTHR) {
            const int64_t j = (int64_t)i - 128;
            tp[i] = (j >= 0 && j < a.K) ? (uint8_t)tr[j] : 0;
        }
    }

    // ---- y -> B: limb 0 (= y itself when |y| <= 127, the common case) ----
    tstamp[1] = clock64();
    const int fl = stage_y(a, B, b, 0, 1, warp, lane);
    const int need2 = __syncthreads_or(fl & 1);
    const int need3 = __syncthreads_or(fl & 2);
    int nl = need3 ? 3 : (need2 ? 2 : 1);
    if (nl > a.LMAX) nl = a.LMAX;  // only reachable when the caller breaks TM_BINARY
    if (nl > 1) {                  // re-stage limb 0 as the low 4 bits
        __syncthreads();
        stage_y(a, B, b, 0, nl, warp, lane);
    }

    tstamp[2] = clock64();
    // ---- A: 16 byte-shifted copies of tp, chunk (J, s) = tp[16 J + s + 1 + e] ----
    for (int c = tid; c < a.JA * 16; c += NTHR) {
        const int J = c >> 4, sg = c & 15;
        const int sh = sg + 1, m = sh >> 2, r = 8 * (sh & 3);
        const uint32_t *w = reinterpret_cast<const uint32_t *>(tp + 16 * J) + m;
        const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
        uint4 o;
        o.x = __funnelshift_r(w0, w1, r);
        o.y = __funnelshift_r(w1, w2, r);
        o.z = __funnelshift_r(w2, w3, r);
        o.w = __funnelshift_r(w3, w4, r);
        reinterpret_cast<uint4 *>(sm)[c] = o;
    }
    const uint32_t *tslot_c = tslot;
    uint32_t tbase = 0;
    tstamp[3] = clock64();

    // ---- MMAs, one pass per limb (the B buffer holds one limb): warp 0 issues,
    // descriptors precomputed, only start addresses move.  D columns of limb l:
    // [2 NMC l, 2 NMC (l + 1)), n = 2 a + j.
    const int nsp = 2 * a.NMC > 256 ? a.NMC : 2 * a.NMC;  // N <= 256 per MMA
    const int nsplit = 2 * a.NMC / nsp;
    for (int l = 0; l < nl; ++l) {
        if (l > 0) {  // the previous pass must have finished reading B
            mbar_wait(mdone, (uint32_t)((l - 1) & 1));
            __syncthreads();
            stage_y(a, B, b, l, nl, warp, lane);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tbase = *tslot_c;
        if (warp == 0) {
            const uint32_t lbo = 32u * a.R;
            const uint64_t ad0 = sdesc(smem_u32(sm), 256, 128);
            const uint64_t bd0 = sdesc(smem_u32(B), lbo, 128);
            const uint32_t id = idesc_i8(nsp);
            for (int sp = 0; sp < nsplit; ++sp) {
                const uint32_t dcol = tbase + 2 * a.NMC * l + sp * nsp;
                for (int c = 0; c < a.NC; ++c) {
#pragma unroll
                    for (int ks = 0; ks < P / 32; ++ks) {
                        // A: +2048 B per c, +512 B per k-step.  B: +32 B per c (2 rows),
                        // +2 LBO per k-step, + nsp rows per split
                        const uint64_t ad = ad0 + (uint64_t)(128u * c + 32u * ks);
                        const uint64_t bd = bd0 + (uint64_t)(2u * c + (lbo >> 3) * ks + (uint32_t)(sp * nsp));
                        mma_i8(dcol, ad, bd, id, (c | ks) ? 1u : 0u);
                    }
                }
            }
            umma_commit(mdone);
        }
    }

    // ---- leftover outputs k in [P NA_j, M_j): one warp per output, overlapping the MMAs ----
    {
        const int nleft0 = (int)max((int64_t)0, a.M[0] - (int64_t)P * a.NA[0]);
        const int nleft1 = (int)max((int64_t)0, a.M[1] - (int64_t)P * a.NA[1]);
        for (int w = warp; w < nleft0 + nleft1; w += NTHR / 32) {
            const int j = w < nleft0 ? 0 : 1;
            const int q = j ? w - nleft0 : w;
            const int64_t k = (int64_t)P * a.NA[j] + q;
            const int32_t *yr = a.y[j] + b * a.ldy[j] + k;
            int64_t s = 0;
            for (int64_t i = lane; i < a.K; i += 32) s += (int64_t)(int8_t)tp[128 + i] * __ldg(yr + i);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) {
                lv[j * MAXLEFT + q] = s;
                if (a.r[j]) a.r[j][b * a.M[j] + k] = s;
            }
        }
    }

    // ---- epilogue: warp w reads TMEM lanes 32 (w & 3) + [0, 32) (rows b'),
    // output blocks [hw NMC/2, (hw + 1) NMC/2) of both moduli (hw = w >> 2) ----
    mbar_wait(mdone, (uint32_t)((nl - 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tstamp[4] = clock64();
    {
        const int qw = warp & 3, hw = warp >> 2;
        const int brow = P - 1 - (32 * qw + lane);  // output offset inside a block
        const uint32_t taddr = tbase + ((uint32_t)(32 * qw) << 16);
        int64_t bv[2] = {INT64_MIN, INT64_MIN}, bk[2] = {INT64_MAX, INT64_MAX};
        const int half = a.NMC / 2;
        for (int a0 = hw * half; a0 < (hw + 1) * half; a0 += 8) {
            if (nl == 1) epi_chunk<1>(a, taddr, a0, brow, b, bv, bk);
            else if (nl == 2) epi_chunk<2>(a, taddr, a0, brow, b, bv, bk);
            else epi_chunk<3>(a, taddr, a0, brow, b, bv, bk);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const int64_t ov = __shfl_xor_sync(0xffffffffu, bv[j], o);
                const int64_t ok = __shfl_xor_sync(0xffffffffu, bk[j], o);
                amax(bv[j], bk[j], ov, ok);
            }
            if (lane == 0) { sv[2 * warp + j] = bv[j]; sk[2 * warp + j] = bk[j]; }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        int64_t m[2];
        for (int j = 0; j < 2; ++j) {
            int64_t v = INT64_MIN, kk = INT64_MAX;
            for (int w = 0; w < NTHR / 32; ++w) amax(v, kk, sv[2 * w + j], sk[2 * w + j]);
            const int nleft = (int)max((int64_t)0, a.M[j] - (int64_t)P * a.NA[j]);
            for (int q = 0; q < nleft; ++q) amax(v, kk, lv[j * MAXLEFT + q], (int64_t)P * a.NA[j] + q);
            m[j] = kk;
        }
        if (a.resid) { a.resid[2 * b] = (int32_t)m[0]; a.resid[2 * b + 1] = (int32_t)m[1]; }
        if (a.residues_out) { a.residues_out[2 * b] = (int32_t)m[0]; a.residues_out[2 * b + 1] = (int32_t)m[1]; }
        if (a.k_out) {  // Theorem 4: z = m1 + M1 ((m2 - m1) M1^{-1} mod M2); k = z < N ? z : -1 (C9)
            int64_t d = m[1] - m[0];  // |m2 - m1| < M2
            if (d < 0) d += a.M2;
            const int64_t u = (int64_t)(((uint64_t)d * a.crt_inv) % (uint64_t)a.M2);  // d, inv < M2 <= 2^32
            const int64_t z = m[0] + a.M1 * u;
            a.k_out[b] = z < a.N ? z : -1;
        }
        if (a.dbg) {
            tstamp[5] = clock64();
            int smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            for (int i = 0; i < 6; ++i) a.dbg[b * 8 + i] = tstamp[i];
            a.dbg[b * 8 + 6] = smid;
        }
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(a.ncols));
}

uint32_t align_up(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }

}  // namespace

static long long *g_tc_dbg = nullptr;
// instrumentation: per-CTA clock64 stamps of the tensor-core kernel's phases into
// buf ([batch][8]: start, template staged, y staged, A built, MMAs done, end, smid);
// NULL = off.  Not part of the method.
extern "C" __attribute__((visibility("default"))) void tm_debug_tc_timestamps(void *buf) {
    g_tc_dbg = (long long *)buf;
}

// Plan-time eligibility and geometry (stored in the plan; see tm_internal.cuh).
void tm_tc_plan(tm_plan_s *p) {
    p->tc_ok = 0;
    if (p->dtype != TM_I8) return;
    const double xmax = (p->flags & TM_BINARY) ? 1.0 : 128.0;
    const double ybound = xmax * (double)(p->q1 > p->q2 ? p->q1 : p->q2);
    const int lmax = ybound <= 127 ? 1 : (ybound <= 2047 ? 2 : (ybound <= 32767 ? 3 : 0));
    if (!lmax) return;
    if (p->K > 65536) return;  // per-limb |r| <= K * 128 * 128 < 2^31
    const int NC = (int)((p->K + P - 2) / P) + 1;
    int NA[2];
    for (int j = 0; j < 2; ++j) {
        const int64_t M = j ? p->M2 : p->M1;
        int64_t na = M / P;
        if (M - na * P > MAXLEFT) ++na;
        if (na < 1) na = 1;
        if (na > 256) return;
        NA[j] = (int)na;
    }
    const int NMC = ((NA[0] > NA[1] ? NA[0] : NA[1]) + 15) & ~15;
    const uint32_t cols = 2u * lmax * NMC;  // D columns
    if (cols > 512) return;
    uint32_t ncols = 32;
    while (ncols < cols) ncols *= 2;
    const int R = NMC + NC - 1;
    const int JA = 8 * (NC - 1) + 15;
    uint32_t off = 256u * JA;   // A
    p->tc_offB = off;
    off += 256u * R;            // B (one limb): 8 chunk columns x 2 R rows x 16 B
    p->tc_offTp = off;
    off += align_up(16 * JA + 48, 16);
    p->tc_offMisc = off;
    off += 16 + 2 * 16 * 8 + 2 * MAXLEFT * 8;
    p->tc_smem = align_up(off, 128);
    if (p->tc_smem > 227 * 1024) return;
    p->tc_NA[0] = NA[0]; p->tc_NA[1] = NA[1];
    p->tc_NMC = NMC; p->tc_R = R;
    p->tc_NC = NC;
    p->tc_JA = JA;
    p->tc_lmax = lmax;
    p->tc_ncols = ncols;
    p->tc_ok = 1;
}

// r1/r2 (may be NULL), resid (may be NULL), k (NULL: no CRT).  t is int8 [batch][ldt].
int tm_tc_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *t, int64_t ldt, int64_t batch,
                    void *r1, void *r2, int32_t *resid, int32_t *residues_out, int64_t *k, cudaStream_t s) {
    if (!p->tc_ok) return TM_EUNSUPPORTED;
    if (batch == 0) return TM_OK;
    if (batch > 0x7FFFFFFF) { tm_set_error("tm_correlate: batch too large"); return TM_EUNSUPPORTED; }
    TcArgs a{};
    a.t = (const int8_t *)t; a.ldt = ldt; a.K = p->K;
    a.y[0] = (const int32_t *)y1; a.y[1] = (const int32_t *)y2;
    a.ldy[0] = p->len_y1; a.ldy[1] = p->len_y2;
    a.len[0] = p->len_y1; a.len[1] = p->len_y2;
    a.M[0] = p->M1; a.M[1] = p->M2;
    a.NA[0] = p->tc_NA[0]; a.NA[1] = p->tc_NA[1];
    a.NMC = p->tc_NMC; a.R = p->tc_R;
    a.NC = p->tc_NC; a.JA = p->tc_JA; a.LMAX = p->tc_lmax; a.ncols = p->tc_ncols;
    a.offB = p->tc_offB; a.offTp = p->tc_offTp; a.offMisc = p->tc_offMisc;
    a.r[0] = (int64_t *)r1; a.r[1] = (int64_t *)r2;
    a.resid = resid; a.residues_out = residues_out; a.k_out = k;
    a.N = p->N; a.M1 = p->M1; a.M2 = p->M2; a.crt_inv = p->crt_inv;
    a.dbg = g_tc_dbg;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(corr_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    corr_tc_kernel<<<(unsigned)batch, NTHR, p->tc_smem, s>>>(a);
    TM_CHECK_LAUNCH("corr_tc_kernel");
    return TM_OK;
}

// Staged path of the tensor-core engine: the "folded template" is the template
// itself (the Toeplitz operand is built in shared memory by tm_tc_correlate),
// stored [batch][tf_bytes] with 16-byte rows.
__global__ void tc_template_copy(const int8_t *__restrict__ t, int64_t K, int64_t ld, int8_t *__restrict__ tf) {
    const int64_t b = blockIdx.x;
    for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) tf[b * ld + i] = i < K ? t[b * K + i] : 0;
}

int tm_tc_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s) {
    if (batch > 0x7FFFFFFF) { tm_set_error("tm_fold_template: batch too large"); return TM_EUNSUPPORTED; }
    tc_template_copy<<<(unsigned)batch, 256, 0, s>>>((const int8_t *)t, p->K, p->tf_bytes, (int8_t *)tf);
    TM_CHECK_LAUNCH("tc_template_copy");
    return TM_OK;
}
