// tc_core.cuh -- the tensor-core correlation of one (signal, template) pair
// (Algorithm 1 steps 4-9) as a device routine run by a group of NTHR threads,
// shared by the standalone kernel (corr_tc.cu) and the fused fold +
// correlation kernel (fold_tma.cu).  The method and the operand layouts are
// described at the top of corr_tc.cu.  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>

#include "tm_internal.cuh"

namespace tc {


constexpr int P = 128;
constexpr int NTHR = 256;
constexpr int MAXLEFT = 8;  // outputs k in [P*NA, M) done by warp dot products
#ifndef TC_RB
#define TC_RB 8
#endif
// misc area (offMisc): mbarrier | TMEM slot | sv[16] | sk[16] | pbegin[2] (fused kernel) |
// leftover partial sums [8 warps][2 MAXLEFT]
constexpr int MISC_PBEGIN = 16 + 2 * 16 * 8;
constexpr int MISC_LEFT = MISC_PBEGIN + 16;
constexpr int MISC_BYTES = MISC_LEFT + (NTHR / 32) * 2 * MAXLEFT * 8;

struct TcArgs {
    const int8_t *t;
    int64_t ldt, K;
    const int32_t *y[2];
    int64_t ldy[2], len[2], M[2];
    int NA[2];   // output blocks of each modulus done on the tensor cores
    int NMC;     // blocks per modulus in the MMA (multiple of 16, >= NA)
    int R;       // B blocks staged (NMC + NC - 1)
    int NC, JA, LMAX;
    int CCH;     // template blocks per A-operand chunk (the A buffer holds one chunk)
    uint32_t ncols;
    uint32_t offB, offTp, offMisc;
    int64_t *r[2];
    int32_t *resid;         // [batch][2] residues (may be NULL)
    int32_t *residues_out;  // [batch][2] (may be NULL)
    int64_t *k_out;         // [batch] (NULL: no CRT)
    int64_t N, M1, M2;
    uint32_t crt_inv;
    int64_t crt_wrap;
    long long *dbg;  // optional per-CTA phase timestamps (tm_debug_tc_timestamps)
    int64_t nbatch;  // templates (one shared y, corr_tc_kernel's persistent loop)
    uint32_t bstride;  // != 0: one B buffer per limb, this many bytes apart (staged once)
    int discard_y;   // 1: y rows (128-byte aligned, ldy multiple of 32) are scratch; drop
                     // their L2 lines without write-back once read (fused tm_run)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ long long gtime() {  // %globaltimer (ns), comparable across SMs
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

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
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(MBAR_SUSPEND_NS)
            : "memory");
    } while (!done);
}

// the whole group waits for an mbarrier phase: warp 0 polls, the other warps block
// in the group barrier (no issue slots taken from co-resident warps)
template <class Sync>
__device__ __forceinline__ void group_wait(uint64_t *bar, uint32_t parity, int warp) {
    if (warp == 0) mbar_wait(bar, parity);
    Sync::sync();
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

// Stage limb l (of nl) of y_1, y_2 blocks s_begin + [0, nrows) (P entries each,
// zero outside [0, len_j)) into the interleaved B layout: row 2 s + j.  One warp
// per block row: lane i holds entries 4i .. 4i+3 (chunk h = i / 4).  Returns
// this thread's range flags (bit 0: some |y| needs 2 limbs, bit 1: 3, bit 2: 4).
__device__ __forceinline__ int stage_yw(const TcArgs &a, uint8_t *B, int64_t b, int l, int nl, int64_t s_begin,
                                        int nrows, int warp, int lane, int jlo = 0, int jhi = 2) {
    uint32_t mag = 0;
    const uint32_t lbo = 32u * nrows;  // bytes per chunk column h: 2 nrows rows of 16 B
    const int h = lane >> 2, wq = lane & 3;
    constexpr int RB = TC_RB;             // block rows in flight per warp
    constexpr int NW = NTHR / 32;
#pragma unroll 1
    for (int j = jlo; j < jhi; ++j) {
        const int32_t *yr = a.y[j] + b * a.ldy[j];
        const int64_t len = a.len[j];
        const bool al = ((((uintptr_t)yr) & 15) == 0);
        for (int s0 = warp; s0 < nrows; s0 += RB * NW) {
            int32_t v[RB][4];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const int64_t i0 = (int64_t)P * (s_begin + s0 + u * NW) + 4 * lane;
                v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0;
                if (s0 + u * NW < nrows && i0 >= 0) {
                    if (al && i0 + 4 <= len) {
                        const int4 q = *reinterpret_cast<const int4 *>(yr + i0);
                        v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (i0 + e < len) v[u][e] = yr[i0 + e];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const int s = s0 + u * NW;
                if (s >= nrows) break;
                const int32_t v0 = v[u][0], v1 = v[u][1], v2 = v[u][2], v3 = v[u][3];
                // v ^ (v >> 31) is v (v >= 0) or -v - 1: below 2^b iff v fits b+1 signed
                // bits, and an OR of values below 2^b stays below 2^b (thresholds 2^7,
                // 2^11, 2^15 are the 1-, 2-, 3-limb limits)
                mag |= (uint32_t)(v0 ^ (v0 >> 31)) | (uint32_t)(v1 ^ (v1 >> 31)) | (uint32_t)(v2 ^ (v2 >> 31)) |
                       (uint32_t)(v3 ^ (v3 >> 31));
                *reinterpret_cast<uint32_t *>(B + lbo * h + 16 * (2 * s + j) + 4 * wq) =
                    nl == 1 ? pack4(v0, v1, v2, v3)
                            : pack4(limb(v0, l, nl), limb(v1, l, nl), limb(v2, l, nl), limb(v3, l, nl));
            }
        }
    }
    return (mag > 127u ? 1 : 0) | (mag > 2047u ? 2 : 0) | (mag > 32767u ? 4 : 0);
}

__device__ __forceinline__ int stage_y(const TcArgs &a, uint8_t *B, int64_t b, int l, int nl, int warp, int lane,
                                       int jlo = 0, int jhi = 2) {
    return stage_yw(a, B, b, l, nl, 0, a.R, warp, lane, jlo, jhi);
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
    if constexpr (NL == 1) {
        // common case (one limb, no r output, whole chunk inside both moduli): the
        // thread's outputs of a modulus rise in k with i, so a strict int32 > keeps
        // the lowest index; one merge per chunk
        if (!a.r[0] && !a.r[1] && a0 + 8 <= a.NA[0] && a0 + 8 <= a.NA[1] &&
            (int64_t)P * (a0 + 8) <= a.M[0] && (int64_t)P * (a0 + 8) <= a.M[1]) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                int32_t best = v[j];
                int bi = 0;
#pragma unroll
                for (int i = 1; i < 8; ++i)
                    if (v[2 * i + j] > best) { best = v[2 * i + j]; bi = i; }
                amax(bv[j], bk[j], (int64_t)best, (int64_t)P * (a0 + bi) + brow);
            }
            return;
        }
    }
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


// barriers of the NTHR-thread group: the whole CTA, or a named barrier
struct CtaSync {
    static __device__ __forceinline__ void sync() { __syncthreads(); }
    static __device__ __forceinline__ int sync_or(int p) { return __syncthreads_or(p); }
};
template <int ID>
struct GroupSync {
    static __device__ __forceinline__ void sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NTHR) : "memory"); }
    static __device__ __forceinline__ int sync_or(int p) {
        int r;
        asm volatile(
            "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\t"
            "bar.red.or.pred q, %2, %3, q;\n\tselp.s32 %0, 1, 0, q;\n\t}"
            : "=r"(r)
            : "r"(p), "n"(ID), "n"(NTHR)
            : "memory");
        return r;
    }
};

// A operand for the template blocks c in [c0, c1): chunk (J, s) of the buffer =
// tp[16 (J + 8 c0) + s + 1 + e], J < 8 (c1 - c0 - 1) + 15.
__device__ __forceinline__ void build_a(const TcArgs &a, uint8_t *sm, int c0, int c1, int tid,
                                        uint8_t *dst = nullptr) {
    const uint8_t *tp = sm + a.offTp + 128 * c0;
    const int n = (8 * (c1 - c0 - 1) + 15) * 16;
    for (int c = tid; c < n; c += NTHR) {
        const int J = c >> 4, sg = c & 15;
        const int sh = sg + 1, m = sh >> 2, r = 8 * (sh & 3);
        const uint32_t *w = reinterpret_cast<const uint32_t *>(tp + 16 * J) + m;
        const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
        uint4 o;
        o.x = __funnelshift_r(w0, w1, r);
        o.y = __funnelshift_r(w1, w2, r);
        o.z = __funnelshift_r(w2, w3, r);
        o.w = __funnelshift_r(w3, w4, r);
        reinterpret_cast<uint4 *>(dst ? dst : sm)[c] = o;
    }
}

// Step 4 (template side) for pair b: the zero-padded template and the A operand
// of its first CCH blocks in shared memory.  Needs only t, so the fused kernel
// runs it while the pair is still being folded.
template <class Sync>
__device__ __forceinline__ void tc_pre(const TcArgs &a, uint8_t *sm, int64_t b, int tid) {
    uint8_t *tp = sm + a.offTp;
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
    Sync::sync();
    build_a(a, sm, 0, min(a.NC, a.CCH), tid);
}

// Steps 5-9 for pair b (after tc_pre): y_1, y_2 -> B, MMAs, argmax, CRT.
// tid in [0, NTHR) is the thread's index in the group, qw = (hardware warp
// index) mod 4 = the TMEM lane quarter its warp may access, sm = the group's
// shared-memory region (plan offsets tc_off*), tbase = the group's TMEM columns
// (a.ncols allocated by the caller), mph = commits already completed on the
// group's mbarrier (sm + offMisc, count 1), updated.
template <class Sync>
// fl1 >= 0: y_1 was already staged as limb 0 of a one-limb pass (stage_y with
// jlo = 0, jhi = 1, while y_2 was being finished) and fl1 is this thread's
// range flags of it; only y_2 is staged here.
__device__ __forceinline__ void tc_main(const TcArgs &a, uint8_t *sm, int64_t b, int tid, int qw, uint32_t tbase,
                                        uint32_t &mph, int fl1 = -1, uint8_t *a_alt = nullptr,
                                        int *y_pre = nullptr) {
    const int warp = tid >> 5, lane = tid & 31;
    long long tstamp[6];
    tstamp[0] = gtime();
    tstamp[1] = tstamp[0];
    uint64_t *mdone = reinterpret_cast<uint64_t *>(sm + a.offMisc);   // MMAs of a pass done
    int64_t *sv = reinterpret_cast<int64_t *>(sm + a.offMisc + 16);   // [8 warps][2]
    int64_t *sk = sv + 16;                                             // [8][2]
    int64_t *lp = reinterpret_cast<int64_t *>(sm + a.offMisc + MISC_LEFT);  // [8 warps][2 MAXLEFT]
    uint8_t *B = sm + a.offB;
    uint8_t *tp = sm + a.offTp;

    // ---- y -> B: limb 0 (= y itself when |y| <= 127, the common case) ----
    // y_pre (one folded signal, many templates): *y_pre = 1 once B holds that y as
    // one limb, which every later template of the CTA reuses without restaging
    int nl;
    if (y_pre && *y_pre > 0) {
        nl = *y_pre;  // B (and, with bstride, the other limbs' buffers) already hold y
    } else {
        const int fl = fl1 >= 0 ? (fl1 | stage_y(a, B, b, 0, 1, warp, lane, 1, 2)) : stage_y(a, B, b, 0, 1, warp, lane);
        const int need2 = Sync::sync_or(fl & 1);
        const int need3 = Sync::sync_or(fl & 2);
        nl = need3 ? 3 : (need2 ? 2 : 1);
        if (nl > a.LMAX) nl = a.LMAX;  // only reachable when the caller breaks TM_BINARY
        if (nl > 1) {                  // re-stage limb 0 as the low 4 bits
            Sync::sync();
            stage_y(a, B, b, 0, nl, warp, lane);
            if (a.bstride)             // and every other limb into its own buffer, once
                for (int l = 1; l < nl; ++l) stage_y(a, B + l * a.bstride, b, l, nl, warp, lane);
        }
        if (y_pre) *y_pre = (a.bstride || nl == 1) ? nl : 0;
    }
    tstamp[2] = gtime();
    tstamp[3] = tstamp[2];

    // ---- MMA passes over (A chunk of CCH template blocks) x (limb): the B buffer
    // holds one limb, the A buffer one chunk; before a pass rewrites either, the
    // previous pass's MMAs must have completed.  Warp 0 issues; descriptors are
    // precomputed, only start addresses move.  D columns of limb l:
    // [2 NMC l, 2 NMC (l + 1)), n = 2 a + j.
    const int nsp = 2 * a.NMC > 256 ? a.NMC : 2 * a.NMC;  // N <= 256 per MMA
    const int nsplit = 2 * a.NMC / nsp;
    uint32_t pass = 0;
    int staged = 0;  // limb in B
    int ch = 0;
    for (int c0 = 0; c0 < a.NC; c0 += a.CCH, ++ch) {
        const int c1 = min(a.NC, c0 + a.CCH);
        // a_alt: the A operand of chunk 1 was built elsewhere in advance (the fused
        // kernel's free TMA ring, for a CTA's last pair): no wait, no rebuild
        const bool alt = a_alt != nullptr && ch == 1;
        uint8_t *abuf = alt ? a_alt : sm;
        for (int l = 0; l < nl; ++l) {
            uint8_t *Bl = a.bstride ? B + l * a.bstride : B;
            if (a.bstride) {
                // resident limb buffers: only a new A chunk waits for the MMAs
                if (pass > 0 && l == 0 && !alt) {
                    group_wait<Sync>(mdone, (mph + pass - 1) & 1u, warp);
                    build_a(a, sm, c0, c1, tid);
                }
            } else if (pass > 0 && !(alt && nl == 1)) {
                group_wait<Sync>(mdone, (mph + pass - 1) & 1u, warp);
                if (l == 0 && !alt) build_a(a, sm, c0, c1, tid);
                if (l != staged) { stage_y(a, B, b, l, nl, warp, lane); staged = l; }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            Sync::sync();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (warp == 0) {
                const uint32_t lbo = 32u * a.R;
                const uint64_t ad0 = sdesc(smem_u32(abuf), 256, 128);
                const uint64_t bd0 = sdesc(smem_u32(Bl), lbo, 128);
                const uint32_t id = idesc_i8(nsp);
                for (int sp = 0; sp < nsplit; ++sp) {
                    const uint32_t dcol = tbase + 2 * a.NMC * l + sp * nsp;
                    for (int c = c0; c < c1; ++c) {
#pragma unroll
                        for (int ks = 0; ks < P / 32; ++ks) {
                            // A: +2048 B per c (chunk-relative), +512 B per k-step.  B: +32 B
                            // per c (2 rows), +2 LBO per k-step, + nsp rows per split
                            const uint64_t ad = ad0 + (uint64_t)(128u * (c - c0) + 32u * ks);
                            const uint64_t bd = bd0 + (uint64_t)(2u * c + (lbo >> 3) * ks + (uint32_t)(sp * nsp));
                            mma_i8(dcol, ad, bd, id, (c | ks) ? 1u : 0u);
                        }
                    }
                }
                umma_commit(mdone);
            }
            ++pass;
        }
    }

    // ---- leftover outputs k in [P NA_j, M_j) (at most MAXLEFT per modulus): every
    // thread takes K / NTHR terms (independent loads), partial sums per warp ----
    const int nleft0 = (int)max((int64_t)0, a.M[0] - (int64_t)P * a.NA[0]);
    const int nleft1 = (int)max((int64_t)0, a.M[1] - (int64_t)P * a.NA[1]);
    for (int q = 0; q < nleft0 + nleft1; ++q) {
        const int j = q < nleft0 ? 0 : 1;
        const int64_t k = (int64_t)P * a.NA[j] + (j ? q - nleft0 : q);
        int64_t s = 0;
        if (nl == 1 && (k & 15) == 0 && k + a.K <= (int64_t)P * a.R) {
            // y_j is in B as int8 (one limb): 16-byte chunks of y_j[k + 16c ..] and of
            // the template, 4 dp4a per chunk, no global loads
            const uint32_t lbo = 32u * a.R;
            int32_t s32 = 0;
            for (int c = tid; c < (a.K + 15) / 16; c += NTHR) {
                const int64_t m0 = k + 16 * c;
                const uint4 yv = *reinterpret_cast<const uint4 *>(B + lbo * ((m0 >> 4) & 7) + 16 * (2 * (m0 >> 7) + j));
                const uint4 tv = *reinterpret_cast<const uint4 *>(tp + 128 + 16 * c);
                s32 = __dp4a((int)yv.x, (int)tv.x, s32);
                s32 = __dp4a((int)yv.y, (int)tv.y, s32);
                s32 = __dp4a((int)yv.z, (int)tv.z, s32);
                s32 = __dp4a((int)yv.w, (int)tv.w, s32);
            }
            s = s32;
        } else {
            const int32_t *yr = a.y[j] + b * a.ldy[j] + k;
#pragma unroll 8
            for (int i = tid; i < a.K; i += NTHR) s += (int64_t)(int8_t)tp[128 + i] * yr[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) lp[warp * 2 * MAXLEFT + q] = s;
    }

    // ---- epilogue: warp w reads TMEM lanes 32 (w & 3) + [0, 32) (rows b'),
    // output blocks [hw NMC/2, (hw + 1) NMC/2) of both moduli (hw = w >> 2) ----
    group_wait<Sync>(mdone, (mph + pass - 1) & 1u, warp);
    mph += pass;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tstamp[4] = gtime();
    {
        const int hw = warp >> 2;
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
    Sync::sync();
    if (a.discard_y) {  // every read of y_1, y_2 of this pair is done
        for (int j = 0; j < 2; ++j) {
            const char *row = reinterpret_cast<const char *>(a.y[j] + b * a.ldy[j]);
            for (int64_t o = 128 * (int64_t)tid; o < 4 * a.ldy[j]; o += 128 * NTHR)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + o) : "memory");
        }
    }
    if (tid == 0) {
        int64_t m[2];
        for (int j = 0; j < 2; ++j) {
            int64_t v = INT64_MIN, kk = INT64_MAX;
            for (int w = 0; w < NTHR / 32; ++w) amax(v, kk, sv[2 * w + j], sk[2 * w + j]);
            const int nleft = j ? nleft1 : nleft0;
            for (int q = 0; q < nleft; ++q) {
                int64_t r = 0;
                for (int w = 0; w < NTHR / 32; ++w) r += lp[w * 2 * MAXLEFT + (j ? nleft0 : 0) + q];
                const int64_t k = (int64_t)P * a.NA[j] + q;
                if (a.r[j]) a.r[j][b * a.M[j] + k] = r;
                amax(v, kk, r, k);
            }
            m[j] = kk;
        }
        if (a.resid) { a.resid[2 * b] = (int32_t)m[0]; a.resid[2 * b + 1] = (int32_t)m[1]; }
        if (a.residues_out) { a.residues_out[2 * b] = (int32_t)m[0]; a.residues_out[2 * b + 1] = (int32_t)m[1]; }
        if (a.k_out) a.k_out[b] = tm_resolve(m[0], m[1], a.M1, a.M2, a.crt_inv, a.N, a.crt_wrap);  // steps 8-9
        if (a.dbg) {
            tstamp[5] = gtime();
            int smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            for (int i = 0; i < 6; ++i) a.dbg[b * 8 + i] = tstamp[i];
            a.dbg[b * 8 + 6] = smid;
        }
    }
}

// Steps 4-9 for pair b (tc_pre then tc_main).
template <class Sync>
__device__ __forceinline__ void tc_pair(const TcArgs &a, uint8_t *sm, int64_t b, int tid, int qw, uint32_t tbase,
                                        uint32_t &mph, int *y_pre = nullptr) {
    tc_pre<Sync>(a, sm, b, tid);
    tc_main<Sync>(a, sm, b, tid, qw, tbase, mph, -1, nullptr, y_pre);
}

}  // namespace tc

long long *tm_tc_dbg_buffer();  // instrumentation (tm_debug_tc_timestamps), NULL = off
// host: TcArgs of a plan (corr_tc.cu); r1/r2/resid/residues/k may be NULL
void tm_tc_fill_args(const tm_plan_s *p, const void *y1, const void *y2, const void *t, int64_t ldt, void *r1,
                     void *r2, int32_t *resid, int32_t *residues_out, int64_t *k, tc::TcArgs &a);
