// corr_tc_tiled.cu -- the tensor-core correlation (Algorithm 1 steps 4-9,
// PAPER.md P:98-106 read as P:61, reading C3; the P = 128 Toeplitz blocking of
// corr_tc.cu) split over many CTAs per pair, for long templates and small
// batches (cfg4: 64 pairs at K = 16384; cfg5: one pair at K = 65536; K up to
// 2^20) where one CTA per pair would leave most SMs idle or not fit.
//
// Three kernels, chained with programmatic dependent launch:
//
//  tiled_prep  (one pass over y and t, whole GPU)
//    * B operand planes: every 16-entry piece of y_j is written once per
//      "plane" in exactly the shared-memory image the MMA reads (chunk column
//      h, row 2 s + j, 16 bytes), so a CTA's B window is 8 bulk copies:
//        plane 0          y itself as int8       (pairs whose |y| <= 127)
//        plane 1 + l      (y >> 4l) & 15         (l = 0 .. lmax-2: low limbs)
//        plane lmax-1+l   y >> 4l  (signed)      (l = 1 .. lmax-1: top limb of
//                                                  an (l+1)-limb split)
//      so y = sum_l 16^l v_l with any limb count nl <= lmax reads planes
//      {0} (nl = 1) or {1 .. nl-1, lmax + nl - 2}, exact and int8-valued;
//    * the limbs each 128-entry block needs (max over both moduli), so a CTA
//      uses the fewest limbs its own window allows;
//    * the template's A image S[J][s][e] = t(16 J + s + e - 127) (its 16
//      byte-shifted copies; corr_tc.cu), so an A chunk is ONE bulk copy;
//    * the partial dot products of the <= 8 leftover outputs k in
//      [128 NA_j, M_j) per modulus, per prep CTA (no atomics);
//    * zeroes the keys, tile counters and (several template ranges) the
//      int64 partial sums the main kernel accumulates into.
//  corr_tc_tiled  CTA (pair b, output tile [a0, a0 + NT) blocks, template
//    range [cb, ce)): warp 9 streams (chunk of <= TCCH template blocks, limb)
//    passes into two A and two B buffers with cp.async.bulk (mbarrier
//    transaction counts); warp 8 issues the MMAs of a pass as soon as its
//    bytes have landed and commits them to the buffer's "done" mbarrier,
//    which frees it for the pass after next; warps 0-7 only run the
//    epilogue (TMEM -> registers, limbs combined, lowest-index max).  With one
//    template range per pair the tile's max goes to an atomicMax on a packed
//    key (r + 2^42) << 21 | (2^21 - 1 - k); with several, each CTA stores its
//    partial r (int64, plain coalesced stores) and
//  tiled_reduce  sums the ranges' partials per output in a fixed order (exact),
//    takes the lowest-index max per pair and modulus (packed-key atomicMax).
//  tc_tiled_final  per pair: keys + leftovers -> residues -> steps 8-9.
// NT (output blocks per tile) is 32 or 64: the shared-memory-operand MMA costs
// ~(4096 + 32 N) / 128 cycles (A read once per MMA, corr_tc.cu), so N = 2 NT =
// 128 does twice the work of N = 64 in ~1.3x the time.
#include <algorithm>

#include "tc_core.cuh"

namespace {
using namespace tc;

constexpr int TCCH = 16;    // template blocks per A chunk
constexpr int KEY_SHIFT = 21;
constexpr int64_t KEY_BIAS = (int64_t)1 << 42;
constexpr int TNTHR = NTHR + 64;   // 8 epilogue warps, MMA issuer (warp 8), TMA producer (warp 9)
constexpr int PREP_T = 256;
constexpr int PREP_MINB = 4;  // resident prep CTAs per SM (<= 64 registers); the grid is one wave
constexpr int PREP_MAXCTA = 1024;  // prep CTAs per pair (bound for the leftover partials)
constexpr int SPE = 24;            // sparse single-limb mode: at most this many entries of a pair's y
                                   // outside [-128, 127] (cfg4, K = 16384: ~5 expected per pair)
constexpr int SPREC = 1 + 3 * SPE; // ints per sparse record

struct TiledArgs {
    TcArgs a;              // y, t, K, M, NA, NC, crt constants
    int n_at, n_cr, CR;    // tiles over output blocks, template ranges, blocks per range
    int at0, n_atp;        // this launch's tiles [at0, at0 + n_atp) (a part of a split correlation)
    int lmax, np;          // limb bound of the plan, planes per pair (2 lmax - 1)
    int64_t S;             // blocks per plane (rows 2 S)
    int JT;                // A-image rows (J) per pair
    int n_pcta;            // prep CTAs per pair
    uint8_t *planes;       // [batch][np][8][2 S][16]
    uint8_t *aimg;         // [batch][JT][256]
    uint8_t *bmag;         // [batch][S] limbs block s needs
    int sparse;            // 1: pairs with <= SPE entries of y outside int8 use ONE limb (y clamped
                           // to int8) plus an exact sparse correction (see SparseList)
    int32_t *spcnt;        // [batch][n_pcta] per prep CTA: its entries outside int8
    int32_t *sprec;        // [batch][n_pcta][3 SPE] per prep CTA: its first <= SPE (idx, e, j)
    int32_t *spair;        // [batch][SPREC] the pair's entries, for tiled_reduce (main kernel CTA 0)
    int tsm;               // > 0: the main kernel stages the template (tsm >= K bytes) in shared memory
                           // for the sparse correction of a one-range pair
    int csm;               // > 0: the epilogue warps also compute those corrections while the MMAs
                           // run, into csm bytes of shared memory after the template (NTHR NT int32)
    int NT;                    // output blocks per tile
    unsigned long long *ckeys; // [batch][nkey_cta][2] packed (max r, lowest k) per CTA and modulus
    int nkey_cta;              // CTAs per pair that write ckeys (the pair's last kernel)
    void *part;                // [batch][n_cr][M1 + M2] partial r of each template range (n_cr > 1):
    int part32;                // int32 when every partial provably fits (plan bound), else int64
    int accum;                 // 1: the ranges add their partials into ONE int64 row (red.add) instead
                               // of storing them (part = [batch][M1 + M2] int64, zeroed by prep)
    int64_t *r_out[2];         // [batch][Mj] r outputs (staged tm_correlate) or NULL
    int64_t *lpart;            // [batch][2][MAXLEFT][n_pcta] leftover partial dot products (per prep CTA)
    unsigned *done;            // [batch] CTAs of the pair's last kernel finished (zeroed by prep)
    int n_last;                // CTAs per pair of the last kernel (it runs finish_pair)
    int32_t *resid, *residues_out;   // finish_pair outputs (may be NULL)
    int64_t *k_out, *keys_out;
    int with_left;
};

__device__ __forceinline__ unsigned long long pack_key(int64_t r, int64_t k) {
    return ((unsigned long long)(r + KEY_BIAS) << KEY_SHIFT) | (unsigned long long)(((int64_t)1 << KEY_SHIFT) - 1 - k);
}

__host__ __device__ __forceinline__ int nleft_of(int64_t M, int NA) {
    const int64_t n = M - (int64_t)P * NA;
    return n > 0 ? (int)n : 0;
}

__device__ __forceinline__ int limbs_needed(int32_t v) {
    const uint32_t m = (uint32_t)(v ^ (v >> 31));  // |v| or |v| - 1: fits b + 1 signed bits iff m < 2^b
    return m <= 127u ? 1 : m <= 2047u ? 2 : m <= 32767u ? 3 : m <= 524287u ? 4 : 5;
}

// byte j of t (zero outside [0, K))
__device__ __forceinline__ uint32_t tbyte(const int8_t *tr, int64_t K, int64_t j) {
    return (j >= 0 && j < K) ? (uint32_t)(uint8_t)tr[j] : 0u;
}

// blocks this launch's windows read: [at0 NT, (at0 + n_atp) NT + NC] (every block
// when the leftovers are computed here: the last part holds them)
__device__ __forceinline__ void plane_range(const TiledArgs &T, int64_t &s_lo, int64_t &s_hi) {
    s_lo = (int64_t)T.at0 * T.NT;
    s_hi = min(T.S, (int64_t)(T.at0 + T.n_atp) * T.NT + T.a.NC + 1);
}

__device__ __forceinline__ int32_t clamp8(int32_t v) { return max(-128, min(127, v)); }

// ---------------------------------------------------------------------------
// prep: planes, block limb counts, A image, leftover partials, zeroing
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PREP_T, PREP_MINB) tiled_prep(const TiledArgs T) {
    pdl_trigger();
    pdl_wait();  // y and t come from the preceding launches
    const TcArgs &a = T.a;
    const int64_t b = blockIdx.y;
    const int tid = threadIdx.x;
    __shared__ int sp_n;            // this CTA's entries of y outside int8 (sparse mode)
    __shared__ int32_t sp_ent[3 * SPE];
    if (tid == 0) sp_n = 0;
    __syncthreads();
    const int64_t gtid = (int64_t)blockIdx.x * PREP_T + tid, gstride = (int64_t)gridDim.x * PREP_T;
    const int8_t *tr = a.t + b * a.ldt;
    const int nl0 = nleft_of(a.M[0], a.NA[0]), nl1 = nleft_of(a.M[1], a.NA[1]);
    int64_t lacc = 0;  // leftover q = 0 of this thread's modulus (its pieces keep one modulus j)

    // ---- zeroing (done counts the last kernel's CTAs; the accumulated partial row)
    if (T.accum) {
        int64_t *acc = reinterpret_cast<int64_t *>(T.part) + b * (a.M1 + a.M2);
        for (int64_t i = gtid; i < a.M1 + a.M2; i += gstride) acc[i] = 0;
    }
    if (blockIdx.x == 0 && tid == 0) T.done[b] = 0;

    // ---- planes + block limb counts: thread = 16 entries (block s,
    // modulus j, chunk column h); 16 consecutive threads cover one block of both moduli
    int64_t s_lo, s_hi;
    plane_range(T, s_lo, s_hi);
    const int64_t n16 = (s_hi - s_lo) * 16;
    const int64_t pstride = (int64_t)8 * 32 * T.S;  // bytes per plane (8 columns x 2 S rows x 16)
    uint8_t *pl = T.planes + b * T.np * pstride;
    // (the loop is warp-uniform: the shuffles below combine 16-lane groups)
    for (int64_t w0 = gtid - (tid & 31); w0 < n16; w0 += gstride) {
        const int64_t w = w0 + (tid & 31);
        const bool valid = w < n16;
        const int64_t s = s_lo + (w >> 4);
        const int j = (int)((w >> 3) & 1), h = (int)(w & 7);
        const int32_t *yr = a.y[j] + b * a.ldy[j];
        const int64_t i0 = (int64_t)P * s + 16 * h, len = valid ? a.len[j] : 0;
        int32_t v[16];
        if (i0 + 16 <= len && ((((uintptr_t)(yr + i0)) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int4 u = __ldg(reinterpret_cast<const int4 *>(yr + i0 + 4 * q));
                v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = (i0 + e < len) ? yr[i0 + e] : 0;
        }
        uint32_t mm = 0;  // max of |v| or |v| - 1 (limbs_needed)
#pragma unroll
        for (int e = 0; e < 16; ++e) mm = max(mm, (uint32_t)(v[e] ^ (v[e] >> 31)));
        int need = limbs_needed((int32_t)mm);
        // leftover output P NA_j (q = 0; q >= 1: the pass below): this piece's t(idx - k) y_j(idx)
        if (j ? nl1 : nl0) {
            const int64_t k = (int64_t)P * a.NA[j];
            const int64_t ilo = i0 - k;  // template index of the piece's first entry
            if (ilo >= 0 && ilo + 16 <= a.K) {
                // the whole piece inside the template: 16 taps t[ilo, ilo + 16), summed in
                // int32 (|t v| < 2^26: 4-limb plan bound) -- the partial-overlap loop below
                // cost a quarter of this kernel's instructions (ncu, cfg4)
                uint32_t tw[4];
                const int8_t *tp = tr + ilo;
                if ((((uintptr_t)tp) & 15) == 0) {
                    const uint4 u = __ldg(reinterpret_cast<const uint4 *>(tp));
                    tw[0] = u.x; tw[1] = u.y; tw[2] = u.z; tw[3] = u.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        tw[q] = (uint32_t)(uint8_t)tp[4 * q] | ((uint32_t)(uint8_t)tp[4 * q + 1] << 8) |
                                ((uint32_t)(uint8_t)tp[4 * q + 2] << 16) | ((uint32_t)(uint8_t)tp[4 * q + 3] << 24);
                }
                int32_t s32 = 0;
#pragma unroll
                for (int e = 0; e < 16; ++e) s32 += (int32_t)(int8_t)(tw[e >> 2] >> (8 * (e & 3))) * v[e];
                lacc += s32;
            } else if (ilo + 16 > 0 && ilo < a.K) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int64_t i = ilo + e;
                    if (i >= 0 && i < a.K) lacc += (int64_t)tr[i] * v[e];
                }
            }
        }
        if (T.sparse) {  // record the entries outside int8 (invalid lanes hold 0); one atomic per
                         // warp, none once the CTA has more than SPE (a dense pair)
            int nexc = 0;
            if (mm > 127u) {
#pragma unroll
                for (int e = 0; e < 16; ++e) nexc += v[e] != clamp8(v[e]);
            }
            const int wtot = (int)__reduce_add_sync(0xffffffffu, (unsigned)nexc);
            if (wtot) {
                const int lane = tid & 31;
                int base = 0;
                if (lane == 0) base = *(volatile int *)&sp_n > SPE ? SPE + 1 : atomicAdd(&sp_n, wtot);
                base = __shfl_sync(0xffffffffu, base, 0);
                int pre = nexc;  // inclusive prefix over the lanes
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, pre, o);
                    if (lane >= o) pre += u;
                }
                if (base <= SPE && nexc) {
                    int q = base + pre - nexc;
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        if (v[e] != clamp8(v[e])) {
                            if (q < SPE) {
                                sp_ent[3 * q] = (int32_t)(i0 + e);
                                sp_ent[3 * q + 1] = v[e] - clamp8(v[e]);
                                sp_ent[3 * q + 2] = j;
                            }
                            ++q;
                        }
                    }
                }
            }
        }
        // max over the 16 lanes of the block (both moduli, 8 columns)
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) need = max(need, __shfl_xor_sync(0xffffffffu, need, o));
        if (!valid) continue;
        if ((tid & 15) == 0) T.bmag[b * T.S + s] = (uint8_t)min(need, 255);
        const int64_t roff = (int64_t)h * 32 * T.S + 16 * (2 * s + j);
        // plane p: 0 -> v clamped to int8; 1 + l (l <= lmax-2) -> (v >> 4l) & 15;
        // lmax - 1 + l (l >= 1) -> v >> 4l (pack4 keeps the low byte); one loop per kind
        {
            uint32_t wd[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wd[q] = pack4(clamp8(v[4 * q]), clamp8(v[4 * q + 1]), clamp8(v[4 * q + 2]), clamp8(v[4 * q + 3]));
            *reinterpret_cast<uint4 *>(pl + roff) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
        for (int l = 0; l < T.lmax - 1; ++l) {
            const int sh = 4 * l;
            uint32_t wd[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wd[q] = pack4(v[4 * q] >> sh, v[4 * q + 1] >> sh, v[4 * q + 2] >> sh, v[4 * q + 3] >> sh) & 0x0F0F0F0Fu;
            *reinterpret_cast<uint4 *>(pl + (1 + l) * pstride + roff) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
        for (int l = 1; l < T.lmax; ++l) {
            const int sh = 4 * l;
            uint32_t wd[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wd[q] = pack4(v[4 * q] >> sh, v[4 * q + 1] >> sh, v[4 * q + 2] >> sh, v[4 * q + 3] >> sh);
            *reinterpret_cast<uint4 *>(pl + (T.lmax - 1 + l) * pstride + roff) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
    }

    // ---- A image: row (J, sg) = t(16 J + sg + e - 127), e < 16
    uint8_t *ai = T.aimg + b * (int64_t)T.JT * 256;
    for (int64_t w = gtid; w < (int64_t)T.JT * 16; w += gstride) {
        const int64_t J = w >> 4;
        const int sg = (int)(w & 15);
        const int64_t base = 16 * J + sg - 127;
        uint32_t wd[4];
        const int64_t w0 = base >> 2;  // floor(base / 4)
        if (w0 >= 0 && 4 * (w0 + 5) <= a.K && ((((uintptr_t)tr) & 3) == 0)) {  // interior: 5 aligned words
            const uint32_t *tw = reinterpret_cast<const uint32_t *>(tr) + w0;
            const uint32_t u0 = __ldg(tw), u1 = __ldg(tw + 1), u2 = __ldg(tw + 2), u3 = __ldg(tw + 3),
                           u4 = __ldg(tw + 4);
            const int sh = 8 * (int)(base & 3);
            wd[0] = __funnelshift_r(u0, u1, sh); wd[1] = __funnelshift_r(u1, u2, sh);
            wd[2] = __funnelshift_r(u2, u3, sh); wd[3] = __funnelshift_r(u3, u4, sh);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wd[q] = tbyte(tr, a.K, base + 4 * q) | (tbyte(tr, a.K, base + 4 * q + 1) << 8) |
                        (tbyte(tr, a.K, base + 4 * q + 2) << 16) | (tbyte(tr, a.K, base + 4 * q + 3) << 24);
        }
        *reinterpret_cast<uint4 *>(ai + 256 * J + 16 * sg) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }

    // ---- this CTA's sparse record (count, then its first <= SPE entries)
    if (T.sparse) {
        __syncthreads();
        const int n = sp_n;
        if (tid == 0) T.spcnt[b * T.n_pcta + blockIdx.x] = n;
        if (tid < 3 * min(n, SPE)) T.sprec[(b * T.n_pcta + blockIdx.x) * 3 * SPE + tid] = sp_ent[tid];
    }

    // ---- leftover outputs k = P NA_j + q (q < nleft_j): this CTA's share of
    // sum_idx t(idx - k) y_j(idx) over the blocks this launch reads, one output at a
    // time (the plane loop above keeps no accumulators); fixed order: warp shuffle,
    // then warps in order
    if (nl0 + nl1 == 0) return;
    __shared__ int64_t red[PREP_T / 32][2 * MAXLEFT];
    const int nlm = max(nl0, nl1);
    for (int jq = 0; jq < 2 * MAXLEFT; ++jq) {
        const int j = jq / MAXLEFT, q = jq % MAXLEFT;
        if (q >= nlm) continue;  // uniform; red[][jq] unused (finish_pair reads q < nleft_j)
        int64_t acc = 0;
        if (q == 0) {
            // pieces of modulus j only: the thread's lacc belongs to its own modulus
            acc = ((gtid >> 3) & 1) == j ? lacc : 0;
        } else if (q < (j ? nl1 : nl0)) {
            const int64_t k = (int64_t)P * a.NA[j] + q;
            const int32_t *yr = a.y[j] + b * a.ldy[j];
            const int64_t lo = max(k, s_lo * P), hi = min(min(k + a.K, s_hi * P), a.len[j]);
            for (int64_t pc = (lo >> 4) + gtid; 16 * pc < hi; pc += gstride) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int64_t idx = 16 * pc + e;
                    if (idx >= lo && idx < hi) acc += (int64_t)tr[idx - k] * __ldg(yr + idx);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((tid & 31) == 0) red[tid >> 5][jq] = acc;
    }
    __syncthreads();
    if (tid < 2 * MAXLEFT) {
        int64_t v = 0;
        for (int w = 0; w < PREP_T / 32; ++w) v += red[w][tid];
        T.lpart[(b * 2 * MAXLEFT + tid) * T.n_pcta + blockIdx.x] = v;
    }
}

// the CTA's best (max r, lowest k) per modulus -> ckeys[b][slot] (all threads call;
// bv/bk of threads without outputs are INT64_MIN / INT64_MAX)
__device__ __forceinline__ void cta_keys(const TiledArgs &T, int64_t b, int slot, int64_t (&bv)[2], int64_t (&bk)[2]) {
    __shared__ unsigned long long wk[16][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t ov = __shfl_xor_sync(0xffffffffu, bv[j], o);
            const int64_t ok = __shfl_xor_sync(0xffffffffu, bk[j], o);
            amax(bv[j], bk[j], ov, ok);
        }
        if (lane == 0) wk[warp][j] = bk[j] == INT64_MAX ? 0ull : pack_key(bv[j], bk[j]);
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        unsigned long long m = 0;
        for (int w = 0; w < nw; ++w) m = wk[w][threadIdx.x] > m ? wk[w][threadIdx.x] : m;
        T.ckeys[(b * T.nkey_cta + slot) * 2 + threadIdx.x] = m;
    }
}

// Sparse single-limb mode.  y = c + e with c = clamp(y, -128, 127) (plane 0) and e
// nonzero only where y leaves int8.  r_j(k) = sum_idx t(idx - k) y_j(idx) (the
// staged correlation, reading C3) = [one-limb MMA over c] + sum over the few
// (idx, e) of e t(idx - k): exact in int64.  When a pair has 1..SPE such entries
// in the blocks this launch reads (prep records them per prep CTA), every CTA of
// the pair runs one limb and the kernel that produces the final r (the main
// kernel's epilogue with one template range, else tiled_reduce) adds the
// correction.  Entry order in the list is immaterial (exact integer sums).
struct SparseList {
    int n;
    int32_t ent[3 * SPE];  // (idx, e, j)
};
// the correction of output k of modulus j
__device__ __forceinline__ int64_t sparse_corr(const TiledArgs &T, int64_t b, const SparseList &L, int n, int j,
                                               int64_t k) {
    const int8_t *tr = T.a.t + b * T.a.ldt;
    int64_t c = 0;
    for (int q = 0; q < n; ++q) {
        const int64_t i = (int64_t)L.ent[3 * q] - k;
        if (L.ent[3 * q + 2] == j && i >= 0 && i < T.a.K) c += (int64_t)L.ent[3 * q + 1] * tr[i];
    }
    return c;
}

// Steps 7-9 of pair b, run by the CTA that finishes the pair's last kernel (all its
// threads): the prep CTAs' leftover partials summed in a fixed order, the
// leftovers merged into the tile keys, residues, k (or the split part's keys).
__device__ void finish_pair(const TiledArgs &T, int64_t b) {
    const TcArgs &a = T.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int nleft0 = nleft_of(a.M[0], a.NA[0]), nleft1 = nleft_of(a.M[1], a.NA[1]);
    __shared__ int64_t fred[16][2 * MAXLEFT];
    __shared__ int64_t lsum[2 * MAXLEFT];
    if (T.with_left && nleft0 + nleft1) {
        // per leftover output: the prep CTAs' partials are contiguous (coalesced,
        // several loads in flight per thread)
        for (int q = 0; q < 2 * MAXLEFT; ++q) {
            if (!(q < MAXLEFT ? q < nleft0 : q - MAXLEFT < nleft1)) continue;  // uniform
            const int64_t *src = T.lpart + (b * 2 * MAXLEFT + q) * T.n_pcta;
            int64_t r = 0;
#pragma unroll 4
            for (int c = tid; c < T.n_pcta; c += blockDim.x) r += __ldcg(src + c);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
            if (lane == 0) fred[warp][q] = r;
        }
        __syncthreads();
        if (tid < 2 * MAXLEFT) {
            int64_t r = 0;
            if (tid < MAXLEFT ? tid < nleft0 : tid - MAXLEFT < nleft1)
                for (int w = 0; w < nw; ++w) r += fred[w][tid];
            lsum[tid] = r;
        }
        __syncthreads();
    }
    // the pair's key per modulus: max over the CTAs' keys (packed keys order like (r, -k))
    __shared__ unsigned long long fk[16][2];
    unsigned long long kmax[2] = {0ull, 0ull};
#pragma unroll 4
    for (int c = tid; c < T.nkey_cta; c += blockDim.x) {
        const ulonglong2 u = __ldcg(reinterpret_cast<const ulonglong2 *>(T.ckeys) + b * T.nkey_cta + c);
        kmax[0] = u.x > kmax[0] ? u.x : kmax[0];
        kmax[1] = u.y > kmax[1] ? u.y : kmax[1];
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ov = __shfl_xor_sync(0xffffffffu, kmax[j], o);
            kmax[j] = ov > kmax[j] ? ov : kmax[j];
        }
        if (lane == 0) fk[warp][j] = kmax[j];
    }
    __syncthreads();
    if (tid) return;
    for (int w = 1; w < nw; ++w)
        for (int j = 0; j < 2; ++j) kmax[j] = fk[w][j] > kmax[j] ? fk[w][j] : kmax[j];
    kmax[0] = fk[0][0] > kmax[0] ? fk[0][0] : kmax[0];
    kmax[1] = fk[0][1] > kmax[1] ? fk[0][1] : kmax[1];
    int64_t m[2];
    for (int j = 0; j < 2; ++j) {
        int64_t bv = INT64_MIN, bk = INT64_MAX;
        const unsigned long long key = kmax[j];
        if (key) {
            bk = ((int64_t)1 << KEY_SHIFT) - 1 - (int64_t)(key & (((unsigned long long)1 << KEY_SHIFT) - 1));
            bv = (int64_t)(key >> KEY_SHIFT) - KEY_BIAS;
        }
        const int nleft = T.with_left ? (j ? nleft1 : nleft0) : 0;
        for (int q = 0; q < nleft; ++q) {
            const int64_t r = lsum[j * MAXLEFT + q];
            const int64_t k = (int64_t)P * a.NA[j] + q;
            if (T.r_out[j]) T.r_out[j][b * a.M[j] + k] = r;
            amax(bv, bk, r, k);
        }
        m[j] = bk;
        if (T.keys_out)  // split correlation: this part's (max r, lowest k) as an order-preserving int64
            T.keys_out[2 * b + j] = bk == INT64_MAX ? INT64_MIN : (int64_t)(pack_key(bv, bk) ^ (1ull << 63));
    }
    if (T.keys_out) return;
    if (T.resid) { T.resid[2 * b] = (int32_t)m[0]; T.resid[2 * b + 1] = (int32_t)m[1]; }
    if (T.residues_out) { T.residues_out[2 * b] = (int32_t)m[0]; T.residues_out[2 * b + 1] = (int32_t)m[1]; }
    if (T.k_out) T.k_out[b] = tm_resolve(m[0], m[1], a.M1, a.M2, a.crt_inv, a.N, a.crt_wrap);  // steps 8-9
}

// every CTA of the pair's last kernel calls this after its atomics; the last to
// arrive runs finish_pair (all threads of the CTA must call it)
__device__ __forceinline__ void arrive_and_finish(const TiledArgs &T, int64_t b) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(T.done + b, 1u) == (unsigned)(T.n_last - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    finish_pair(T, b);
}

// ---------------------------------------------------------------------------
// main kernel
// ---------------------------------------------------------------------------
// smem: A [2][A_BYTES] | B [2][B_BYTES] | full[2] | mdone[2] | TMEM slot | flag
constexpr int A_BYTES = (256 * (8 * (TCCH - 1) + 15) + 127) / 128 * 128;
// B chunk-column stride: 32 nrows + 16 bytes (a multiple of 16, as the
// descriptor needs); rows of a column are contiguous (16 B each)
__host__ __device__ __forceinline__ uint32_t b_lbo(int nrows) { return 32u * nrows + 16u; }
template <int NT>
constexpr int b_bytes() { return (8 * (2 * (NT + TCCH - 1) * 16 + 16) + 127) / 128 * 128; }
template <int NT>
constexpr int smem_bytes() { return 2 * A_BYTES + 2 * b_bytes<NT>() + 64; }

__device__ __forceinline__ void mbar_init1(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int NT>
#ifndef TM_TILED_MINB
#define TM_TILED_MINB 2
#endif
__global__ void __launch_bounds__(TNTHR, TM_TILED_MINB) corr_tc_tiled(const TiledArgs T) {
    pdl_trigger();
    pdl_wait();  // the prep kernel's planes, A image and zeroed keys
    constexpr int B_BYTES = b_bytes<NT>();
    extern __shared__ __align__(1024) uint8_t sm[];
    const TcArgs &a = T.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t b = blockIdx.y;
    const int at = T.at0 + blockIdx.x % T.n_atp, cr = blockIdx.x / T.n_atp;
    const int a0 = at * NT;
    const int cb = cr * T.CR, ce = min(a.NC, cb + T.CR);
    uint8_t *Abuf = sm, *Bbuf = sm + 2 * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(Bbuf + 2 * B_BYTES);  // [2]
    uint64_t *mdone = full + 2;                                          // [2]
    uint64_t *fin = mdone + 2;                                           // every MMA of the CTA done
    uint32_t *tslot = reinterpret_cast<uint32_t *>(fin + 1);
    long long ts[4] = {gtime(), 0, 0, 0};  // instrumentation (a.dbg): phase stamps
    long long te[2] = {0, 0};                // epilogue sub-phases (thread 0)
    __shared__ SparseList spl;
    __shared__ int wneed[TNTHR / 32], wcnt[TNTHR / 32];
    if (tid == 0) {
        mbar_init1(full); mbar_init1(full + 1); mbar_init1(mdone); mbar_init1(mdone + 1); mbar_init1(fin);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        spl.n = 0;
    }
    // ---- limb count: the most any block of this CTA's window [a0 + cb, a0 + NT + ce - 1)
    // needs, and (sparse mode) the pair's entries outside int8, in one round trip
    int need = 1, cnt = 0;
    {
        const int64_t s0 = (int64_t)a0 + cb, n = NT + (ce - cb) - 1;
        for (int64_t i = tid; i < n; i += TNTHR)
            if (s0 + i < T.S) need = max(need, (int)T.bmag[b * T.S + s0 + i]);
        if (T.sparse)
            for (int c = tid; c < T.n_pcta; c += TNTHR) cnt += T.spcnt[b * T.n_pcta + c];
    }
    need = __reduce_max_sync(0xffffffffu, need);
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) { wneed[warp] = need; wcnt[warp] = cnt; }
    __syncthreads();
    int nmax = 1, total = 0;
#pragma unroll
    for (int w = 0; w < TNTHR / 32; ++w) { nmax = max(nmax, wneed[w]); total += wcnt[w]; }
    const int nsp = (total >= 1 && total <= SPE) ? total : 0;  // sparse pair: one limb + correction
    if (nsp) {
        for (int c = tid; c < T.n_pcta; c += TNTHR) {
            const int m = T.spcnt[b * T.n_pcta + c];
            if (m) {
                const int32_t *rec = T.sprec + (b * T.n_pcta + c) * 3 * SPE;
                const int o = atomicAdd(&spl.n, m);
                for (int q = 0; q < 3 * m; ++q) spl.ent[3 * o + q] = rec[q];
            }
        }
        __syncthreads();
        if (T.n_cr > 1 && blockIdx.x == 0) {  // for tiled_reduce
            int32_t *dst = T.spair + b * SPREC;
            if (tid < 3 * nsp) dst[1 + tid] = spl.ent[tid];
            if (tid == 0) dst[0] = nsp;
        }
    } else if (T.sparse && T.n_cr > 1 && blockIdx.x == 0 && tid == 0) {
        T.spair[b * SPREC] = 0;
    }
    const int nl = nsp ? 1 : min(T.lmax, nmax);
    // TMEM: 2 NT columns per limb (two CTAs fit per SM while 2 NT nl <= 256)
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(2 * NT * nl)) ncols *= 2;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tslot;
    ts[1] = gtime();
    const int npass = ((ce - cb + TCCH - 1) / TCCH) * nl;

    if (warp == 9) {
        // ---- TMA producer: pass q = (chunk, limb) into A[chunk & 1], B[q & 1]
        if (lane == 0) {
            const int64_t pstride = (int64_t)8 * 32 * T.S;
            const uint8_t *pl = T.planes + b * T.np * pstride;
            const uint8_t *ai = T.aimg + b * (int64_t)T.JT * 256;
            int q = 0, ch = 0;
            for (int c0 = cb; c0 < ce; c0 += TCCH, ++ch) {
                const int c1 = min(ce, c0 + TCCH);
                const int nrows = NT + (c1 - c0) - 1;  // B window: blocks [a0 + c0, a0 + c0 + nrows)
                const uint32_t lbo = b_lbo(nrows);
                const uint32_t abytes = 256u * (8 * (c1 - c0 - 1) + 15);
                for (int l = 0; l < nl; ++l, ++q) {
                    if (q >= 2) mbar_wait(mdone + (q & 1), ((q - 2) >> 1) & 1u);  // buffers of pass q - 2 free
                    const int plane = nl == 1 ? 0 : (l < nl - 1 ? 1 + l : T.lmax + nl - 2);
                    expect_tx(full + (q & 1), (l == 0 ? abytes : 0u) + 8u * 32u * nrows);
                    if (l == 0) bulk_copy(Abuf + (ch & 1) * A_BYTES, ai + 256 * 8 * (int64_t)c0, abytes, full + (q & 1));
                    const uint8_t *src = pl + plane * pstride + 32 * ((int64_t)a0 + c0);
                    uint8_t *B = Bbuf + (q & 1) * B_BYTES;
                    for (int h = 0; h < 8; ++h)
                        bulk_copy(B + h * lbo, src + h * 32 * T.S, 32u * nrows, full + (q & 1));
                }
            }
        }
    } else if (warp == 8) {
        // ---- MMA issuer
        int q = 0, ch = 0;
        for (int c0 = cb; c0 < ce; c0 += TCCH, ++ch) {
            const int c1 = min(ce, c0 + TCCH);
            const int nrows = NT + (c1 - c0) - 1;
            const uint32_t lbo = b_lbo(nrows);
            const uint8_t *A = Abuf + (ch & 1) * A_BYTES;
            for (int l = 0; l < nl; ++l, ++q) {
                mbar_wait(full + (q & 1), (q >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint8_t *B = Bbuf + (q & 1) * B_BYTES;
                const uint64_t ad0 = sdesc(smem_u32(A), 256, 128);
                const uint64_t bd0 = sdesc(smem_u32(B), lbo, 128);
                const uint32_t id = idesc_i8(2 * NT);
                const uint32_t dcol = tbase + 2 * NT * l;
                for (int c = c0; c < c1; ++c) {
#pragma unroll
                    for (int ks = 0; ks < P / 32; ++ks) {
                        const uint64_t ad = ad0 + (uint64_t)(128u * (c - c0) + 32u * ks);
                        const uint64_t bd = bd0 + (uint64_t)(2u * (c - c0) + (lbo >> 3) * ks);
                        mma_i8(dcol, ad, bd, id, (c != cb || ks) ? 1u : 0u);
                    }
                }
                umma_commit(mdone + (q & 1));
            }
        }
        umma_commit(fin);  // tracks every MMA this thread issued
    }
    // sparse pair, one template range: while the MMAs run, the epilogue warps copy the
    // template into shared memory for the corrections (random byte reads of t from
    // L2 in the epilogue measured ~4 us per CTA at cfg4)
    const int8_t *tcor = a.t + b * a.ldt;
    if (nsp && T.n_cr == 1 && T.tsm && warp < NTHR / 32) {
        int8_t *tsh = reinterpret_cast<int8_t *>(sm + smem_bytes<NT>());
        if (((uintptr_t)tcor & 15) == 0) {
            for (int64_t i = tid; 16 * i < a.K; i += NTHR)
                reinterpret_cast<int4 *>(tsh)[i] = __ldg(reinterpret_cast<const int4 *>(tcor) + i);
        } else {
            for (int64_t i = tid; i < a.K; i += NTHR) tsh[i] = tcor[i];
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NTHR) : "memory");  // the epilogue warps only
        tcor = tsh;
        if (T.csm) {
            // the corrections of this thread's NT outputs (the epilogue's (ar0, i, j) order),
            // exact in int32 (see the epilogue), while the tensor pipe runs the loop; the
            // epilogue then only adds them
            int32_t *cb = reinterpret_cast<int32_t *>(sm + smem_bytes<NT>() + T.tsm);
            const int qw = warp & 3, hw = warp >> 2;
            const int kb = P * a0 + P - 1 - (32 * qw + lane);
            const int Kt = (int)a.K;
            for (int it = 0; it < NT / 16; ++it) {
                const int k0 = kb + P * ((NT / 2) * hw + 8 * it);
                int32_t c0[8], c1[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) c0[i] = c1[i] = 0;
                for (int q = 0; q < nsp; ++q) {
                    const int ti0 = spl.ent[3 * q] - k0;
                    const int32_t ev = spl.ent[3 * q + 1];
                    const bool jj = spl.ent[3 * q + 2] != 0;
                    const int32_t e0 = jj ? 0 : ev, e1 = jj ? ev : 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int ti = ti0 - P * i;
                        const int32_t tv = (unsigned)ti < (unsigned)Kt ? (int32_t)tsh[ti] : 0;
                        c0[i] += e0 * tv;
                        c1[i] += e1 * tv;
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cb[((it * 8 + i) * 2) * NTHR + tid] = c0[i];
                    cb[((it * 8 + i) * 2 + 1) * NTHR + tid] = c1[i];
                }
            }
        }
    }
    // every warp: all MMAs complete (fin completes exactly once: parity 0; a wait on
    // mdone's parity would return at once for a phase not yet begun).  Warps 0-7
    // (idle through the loop): warp 0 polls, the others sleep in a named barrier,
    // so they take no issue slots from the MMA issuer, the producer or the
    // co-resident CTA's epilogue
#ifndef TM_TILED_GROUPWAIT
#define TM_TILED_GROUPWAIT 1
#endif
    if (TM_TILED_GROUPWAIT && warp < NTHR / 32) {
        if (warp == 0) mbar_wait(fin, 0);
        asm volatile("bar.sync 2, %0;" ::"n"(NTHR) : "memory");
    } else {
        mbar_wait(fin, 0);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    ts[2] = gtime();

    // ---- epilogue (warps 0-7): warp w: TMEM lanes 32 (w & 3) (rows b'), blocks a0 + (NT / 2) (w >> 2) + [0, NT / 2)
    int64_t mbv[2] = {INT64_MIN, INT64_MIN}, mbk[2] = {INT64_MAX, INT64_MAX};
    if (warp < NTHR / 32) {
        const int qw = warp & 3, hw = warp >> 2;
        const int brow = P - 1 - (32 * qw + lane);
        const uint32_t taddr = tbase + ((uint32_t)(32 * qw) << 16);
        int64_t bv[2] = {INT64_MIN, INT64_MIN}, bk[2] = {INT64_MAX, INT64_MAX};
        // per-thread constants (outputs k < 2^21 fit int): output k = kb + P (ar0 + i) is
        // an MMA output of modulus j iff k < klim_j (block < NA_j and k < M_j)
        const int kb = P * a0 + brow;
        const int klim0 = (int)min((int64_t)P * a.NA[0], a.M[0]), klim1 = (int)min((int64_t)P * a.NA[1], a.M[1]);
        const bool keys_only = T.n_cr == 1 && !T.r_out[0] && !T.r_out[1];
        unsigned long long *accb = reinterpret_cast<unsigned long long *>(T.part) + b * (a.M1 + a.M2);
        for (int ar0 = (NT / 2) * hw; ar0 < (NT / 2) * hw + NT / 2; ar0 += 8) {
            int64_t r[8][2];
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i][0] = r[i][1] = 0;
            for (int l = 0; l < nl; ++l) {
                int32_t v[16];
                tmem_ld16(taddr + 2 * NT * l + 2 * ar0, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (tid == 0 && ar0 == 0 && l == 0) te[0] = gtime();  // (a.dbg) first TMEM load back
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    r[i][0] += (int64_t)v[2 * i] * ((int64_t)1 << (4 * l));
                    r[i][1] += (int64_t)v[2 * i + 1] * ((int64_t)1 << (4 * l));
                }
            }
            const int k0 = kb + P * ar0;  // output of (ar0 + i): k0 + P i
            if (nsp && T.n_cr == 1 && T.csm) {  // corrections computed during the loop
                const int32_t *cb = reinterpret_cast<const int32_t *>(sm + smem_bytes<NT>() + T.tsm);
                const int it = (ar0 - (NT / 2) * hw) / 8;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    r[i][0] += cb[((it * 8 + i) * 2) * NTHR + tid];
                    r[i][1] += cb[((it * 8 + i) * 2 + 1) * NTHR + tid];
                }
            } else if (nsp && T.n_cr == 1) {  // sparse pair: + sum_q e_q t(idx_q - k)
                // |y| <= 524287 (tm_tc_tiled_plan: <= 4 limbs), so |e t| < 2^26 and the
                // <= SPE = 24 terms of an output sum exactly in int32: one IMAD per term
                // and modulus, no branches
                const int8_t *tr = tcor;
                const int Kt = (int)a.K;
                int32_t c0[8], c1[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) c0[i] = c1[i] = 0;
                for (int q = 0; q < nsp; ++q) {
                    const int ti0 = spl.ent[3 * q] - k0;
                    const int32_t ev = spl.ent[3 * q + 1];
                    const bool jj = spl.ent[3 * q + 2] != 0;
                    const int32_t e0 = jj ? 0 : ev, e1 = jj ? ev : 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int ti = ti0 - P * i;
                        const int32_t tv = (unsigned)ti < (unsigned)Kt ? (int32_t)tr[ti] : 0;
                        c0[i] += e0 * tv;
                        c1[i] += e1 * tv;
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) { r[i][0] += c0[i]; r[i][1] += c1[i]; }
            }
            if (keys_only) {  // one template range: the lowest-index max (k increases along the loop)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int k = k0 + P * i;
                    if (k < klim0 && r[i][0] > bv[0]) { bv[0] = r[i][0]; bk[0] = k; }
                    if (k < klim1 && r[i][1] > bv[1]) { bv[1] = r[i][1]; bk[1] = k; }
                }
                continue;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int k = k0 + P * i;
                    if (k < (j ? klim1 : klim0)) {
                        if (T.n_cr > 1) {  // this range's partial r (summed by tiled_reduce)
                            if (T.accum) {  // exact: int64 adds commute
                                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(accb + (j ? a.M1 : 0) + k),
                                             "l"((unsigned long long)r[i][j]) : "memory");
                            } else {
                                const int64_t o = (b * T.n_cr + cr) * (a.M1 + a.M2) + (j ? a.M1 : 0) + k;
                                if (T.part32) reinterpret_cast<int32_t *>(T.part)[o] = (int32_t)r[i][j];
                                else reinterpret_cast<int64_t *>(T.part)[o] = r[i][j];
                            }
                        } else {
                            if (T.r_out[j]) T.r_out[j][b * a.M[j] + k] = r[i][j];
                            amax(bv[j], bk[j], r[i][j], k);
                        }
                    }
                }
            }
        }
        if (T.n_cr == 1) {
            mbv[0] = bv[0]; mbv[1] = bv[1]; mbk[0] = bk[0]; mbk[1] = bk[1];
        }
        if (tid == 0) te[1] = gtime();  // (a.dbg) thread 0's epilogue outputs done
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (T.n_cr == 1) cta_keys(T, b, blockIdx.x, mbv, mbk);
    if (a.dbg && tid == 0) {
        ts[3] = gtime();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long *d = a.dbg + 8 * ((int64_t)blockIdx.y * gridDim.x + blockIdx.x);
        d[0] = ts[0]; d[1] = ts[1]; d[2] = ts[2]; d[3] = ts[3];
        d[4] = 0; d[5] = te[0]; d[6] = te[1];
        d[7] = ((long long)smid << 32) | ((long long)min(nsp, 255) << 24) | ((long long)(npass & 0xFFFF) << 8) | nl;
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols));
    if (T.n_cr == 1) {
        arrive_and_finish(T, b);  // this kernel is the pair's last
        if (a.dbg && tid == 0) {  // [4]: after the arrival (and, for the last CTA, finish_pair)
            long long *d = a.dbg + 8 * ((int64_t)blockIdx.y * gridDim.x + blockIdx.x);
            d[4] = gtime();
        }
    }
}

// several template ranges: r = sum of the ranges' partials (fixed order, exact
// int64), the lowest-index max per pair and modulus -> packed-key atomicMax.
// Thread = RED_E consecutive outputs; the thread's and then the CTA's best output
// as one packed key (pack_key orders like (r, -k), so a u64 max is the
// lowest-index max: half the shuffles of an (r, k) pair reduction).  The kernel is
// a chain of latencies (cfg5: a 1 MB read); RED_E = 4 (fewer arrivals, fewer keys
// for finish_pair) measured 2.5 us slower per cfg5 step than RED_E = 1.
constexpr int RED_T = 256;
#ifndef TM_RED_E
#define TM_RED_E 1
#endif
constexpr int RED_E = TM_RED_E;
template <typename PT>
__global__ void __launch_bounds__(RED_T) tiled_reduce(const TiledArgs T) {
    pdl_trigger();
    pdl_wait();
    const TcArgs &a = T.a;
    const int64_t b = blockIdx.y;
    const int64_t ML = a.M1 + a.M2;
    // over this launch's MMA outputs only (the tiles [at0, at0 + n_atp) of a split
    // correlation; leftovers: finish_pair): k in [klo, khi_j) per modulus
    const int64_t klo = (int64_t)P * T.at0 * T.NT, kt = (int64_t)P * (T.at0 + T.n_atp) * T.NT;
    // (NA_j counts a last partial block with more than MAXLEFT outputs: its outputs end at M_j)
    const int64_t kh0 = min(kt, min((int64_t)P * a.NA[0], a.M[0])), kh1 = min(kt, min((int64_t)P * a.NA[1], a.M[1]));
    const int64_t n0 = max((int64_t)0, kh0 - klo), n1 = max((int64_t)0, kh1 - klo);
    const int64_t e0 = ((int64_t)blockIdx.x * RED_T + threadIdx.x) * RED_E;
    const PT *pp = reinterpret_cast<const PT *>(T.part) + b * T.n_cr * ML;
    __shared__ SparseList spl;
    const int nsp = T.sparse ? __ldcg(T.spair + b * SPREC) : 0;  // written by the main kernel's CTA 0
    int64_t r[RED_E];
    int64_t idx[RED_E];
#pragma unroll
    for (int u = 0; u < RED_E; ++u) {
        const int64_t e = e0 + u;
        const int j = e >= n0 ? 1 : 0;
        const int64_t k = klo + (j ? e - n0 : e);
        idx[u] = e < n0 + n1 ? (j ? a.M1 : 0) + k : -1;
        r[u] = 0;
    }
    if (T.accum) {
#pragma unroll
        for (int u = 0; u < RED_E; ++u)
            if (idx[u] >= 0) r[u] = __ldcg(reinterpret_cast<const int64_t *>(T.part) + b * ML + idx[u]);
    } else {
#pragma unroll
        for (int u = 0; u < RED_E; ++u) {
            if (idx[u] < 0) continue;
            int c = 0;
            for (; c + 8 <= T.n_cr; c += 8) {  // eight loads in flight, summed in range order
                PT v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = __ldcg(pp + (c + q) * ML + idx[u]);
#pragma unroll
                for (int q = 0; q < 8; ++q) r[u] += (int64_t)v[q];
            }
            for (; c < T.n_cr; ++c) r[u] += (int64_t)__ldcg(pp + c * ML + idx[u]);
        }
    }
    if (nsp) {  // sparse pair: + sum_q e_q t(idx_q - k)
        for (int q = threadIdx.x; q < 3 * nsp; q += RED_T) spl.ent[q] = __ldcg(T.spair + b * SPREC + 1 + q);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < RED_E; ++u)
            if (idx[u] >= 0) {
                const int j = idx[u] >= a.M1 ? 1 : 0;
                r[u] += sparse_corr(T, b, spl, nsp, j, idx[u] - (j ? a.M1 : 0));
            }
    }
    unsigned long long key[2] = {0ull, 0ull};  // 0: no output (every real key is > 0)
#pragma unroll
    for (int u = 0; u < RED_E; ++u) {
        if (idx[u] < 0) continue;
        const int j = idx[u] >= a.M1 ? 1 : 0;
        const int64_t k = idx[u] - (j ? a.M1 : 0);
        if (T.r_out[j]) T.r_out[j][b * a.M[j] + k] = r[u];
        const unsigned long long kk = pack_key(r[u], k);
        if (j) key[1] = kk > key[1] ? kk : key[1];  // (no dynamic register-array index)
        else key[0] = kk > key[0] ? kk : key[0];
    }
    __shared__ unsigned long long wk[RED_T / 32][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        unsigned long long m = key[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ov = __shfl_xor_sync(0xffffffffu, m, o);
            m = ov > m ? ov : m;
        }
        if (lane == 0) wk[warp][j] = m;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        unsigned long long m = 0;
#pragma unroll
        for (int w = 0; w < RED_T / 32; ++w) m = wk[w][threadIdx.x] > m ? wk[w][threadIdx.x] : m;
        T.ckeys[(b * T.nkey_cta + blockIdx.x) * 2 + threadIdx.x] = m;
    }
    arrive_and_finish(T, b);
}

// per pair (one CTA of FIN_T threads): tile keys + leftovers -> residues; steps 8-9 (tm_resolve)
constexpr int FIN_T = 256;
// (only when this launch has no tiles -- a part of a split correlation past the
// last tile: then no main kernel runs to finish the pair)
__global__ void __launch_bounds__(FIN_T) tc_tiled_final(const TiledArgs T) {
    pdl_trigger();
    pdl_wait();
    finish_pair(T, blockIdx.x);
}

// split correlation: all-reduced (MAX) keys -> residues -> steps 8-9
__global__ void match_keys_kernel(const int64_t *keys, int64_t batch, int64_t M1, int64_t M2, uint32_t inv,
                                  int64_t N, int64_t wrap, int32_t *residues, int64_t *k) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    int64_t m[2];
    for (int j = 0; j < 2; ++j) {
        const unsigned long long key = (unsigned long long)keys[2 * b + j] ^ (1ull << 63);
        m[j] = ((int64_t)1 << KEY_SHIFT) - 1 - (int64_t)(key & (((unsigned long long)1 << KEY_SHIFT) - 1));
    }
    if (residues) { residues[2 * b] = (int32_t)m[0]; residues[2 * b + 1] = (int32_t)m[1]; }
    if (k) k[b] = tm_resolve(m[0], m[1], M1, M2, inv, N, wrap);
}

// geometry shared by the workspace size and the launch
constexpr size_t PART_BUDGET = (size_t)64 << 20;  // bytes of partial sums (several template ranges)
// NT = 64 (MMA N = 128: fewer A-operand reads per MAC) when the pairs' tiles fill
// the SMs without splitting the template range much; NT = 32 otherwise, where the
// partial sums of more template ranges cost more than the MMAs save (measured,
// same box: cfg5 one pair K = 65536 42 vs 47 us, 64 pairs K = 16384 94 vs 112 us;
// 64 pairs K = 32768 / 65536: 172 / 545 vs 135 / 406 us)
int tiled_nt(const tm_plan_s *p, int64_t batch) {
    static const char *env = getenv("TM_TILED_NT");  // A/B: "32" or "64"
    if (env && (atoi(env) == 32 || atoi(env) == 64)) return atoi(env);
    int64_t na = 1;
    for (int64_t M : {p->M1, p->M2}) na = std::max(na, M / P + (M % P > MAXLEFT ? 1 : 0));
    // (>= 0.85 of the SMs: one CTA per SM at MMA N = 128 beats two per SM at N = 64; cfg4 K =
    // 16384, 128 tiles: correlation 67 -> 63 us)
    return batch * ((na + 63) / 64) * 20 >= (int64_t)p->num_sms * 17 ? 64 : 32;
}
struct Geo {
    int NT, NC, NA[2], n_at, lmax, np, JT, n_pcta, max_cr, max_keys;
    int64_t S;
};
Geo geometry(const tm_plan_s *p, int64_t batch) {
    Geo g{};
    g.NT = tiled_nt(p, batch);
    g.NC = (int)((p->K + P - 2) / P) + 1;
    for (int j = 0; j < 2; ++j) {
        const int64_t M = j ? p->M2 : p->M1;
        int64_t na = M / P;
        if (M - na * P > MAXLEFT) ++na;
        if (na < 1) na = 1;
        g.NA[j] = (int)na;
    }
    const int namax = std::max(g.NA[0], g.NA[1]);
    g.n_at = (namax + g.NT - 1) / g.NT;
    g.S = (int64_t)g.n_at * g.NT + g.NC + 1;  // every window row [a0 + c0, a0 + c0 + nrows)
    g.lmax = std::max(1, p->tct_lmax);
    g.np = 2 * g.lmax - 1;
    g.JT = 8 * (g.NC - 1) + 16;
    const int64_t want = (int64_t)PREP_MINB * p->num_sms / std::max<int64_t>(batch, 1);
    g.n_pcta = (int)std::min<int64_t>(PREP_MAXCTA, std::max<int64_t>(1, want));
    // template ranges of >= one A chunk each, and their partial sums within the budget
    const size_t per = (size_t)std::max<int64_t>(batch, 1) * (size_t)(p->M1 + p->M2) * 8;
    g.max_cr = std::max(1, std::min((g.NC + TCCH - 1) / TCCH, (int)std::min<size_t>(PART_BUDGET / per, 1 << 20)));
    // CTAs per pair writing keys: the reduce kernel's, or the main kernel's (<= n_at max_cr)
    g.max_keys = std::max((int)((p->M1 + p->M2 + RED_T - 1) / RED_T), g.n_at * g.max_cr);
    return g;
}

size_t align_up256(size_t v) { return (v + 255) & ~size_t(255); }
}  // namespace

int tm_tc_match_keys(const tm_plan_s *p, const int64_t *keys, int64_t batch, int32_t *residues, int64_t *k,
                     cudaStream_t s) {
    if (batch == 0) return TM_OK;
    match_keys_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, s>>>(keys, batch, p->M1, p->M2, p->crt_inv, p->N,
                                                                       p->crt_wrap, residues, k);
    TM_CHECK_LAUNCH("tm_match_keys");
    return TM_OK;
}

// Plan-time eligibility (int8 data whose |y| fits 4 four-bit limbs and whose
// |r| fits the packed key).
void tm_tc_tiled_plan(tm_plan_s *p) {
    p->tct_ok = 0;
    if (p->dtype != TM_I8) return;
    const double xmax = (p->flags & TM_BINARY) ? 1.0 : 128.0;
    const double ybound = xmax * (double)(p->q1 > p->q2 ? p->q1 : p->q2);
    const int lmax = ybound <= 127 ? 1 : ybound <= 2047 ? 2 : ybound <= 32767 ? 3 : ybound <= 524287 ? 4 : 0;
    if (!lmax) return;
    if ((double)p->K * xmax * ybound >= (double)((int64_t)1 << 41)) return;  // packed key range
    // per-limb partial sums accumulate in int32 TMEM: |t| * |limb| <= tmax * 128 (the
    // signed top limb, or y itself when one limb holds it) over K terms
    if ((double)p->K * xmax * 128.0 >= (double)((int64_t)1 << 31)) return;
    if (p->M2 >= ((int64_t)1 << KEY_SHIFT)) return;
    p->tct_lmax = lmax;
    p->tct_ok = 1;
}

size_t tm_tc_tiled_ws_bytes(const tm_plan_s *p, int64_t batch) {
    if (!p->tct_ok || batch < 1) return 0;
    const Geo g = geometry(p, batch);
    size_t n = 0;
    n += align_up256((size_t)batch * g.max_keys * 16);                      // per-CTA keys
    n += align_up256(g.max_cr > 1 ? (size_t)batch * g.max_cr * (p->M1 + p->M2) * 8 : 0);  // partial sums
    n += align_up256((size_t)batch * g.S);                                  // block limb counts
    n += align_up256((size_t)batch * g.n_pcta * 4);                         // sparse counts per prep CTA
    n += align_up256((size_t)batch * g.n_pcta * 3 * SPE * 4);               // sparse entries per prep CTA
    n += align_up256((size_t)batch * SPREC * 4);                            // sparse list per pair
    n += align_up256((size_t)batch * g.np * 8 * 32 * g.S);                  // B planes
    n += align_up256((size_t)batch * g.JT * 256);                           // A image
    n += align_up256((size_t)batch * g.n_pcta * 2 * MAXLEFT * 8);           // leftover partials
    n += align_up256((size_t)batch * 4);                                    // done counters
    return n + 256;
}

// r1/r2 (int64, may be NULL), residues_out/resid (may be NULL), k (may be NULL).
int tm_tc_tiled_correlate(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2,
                          const void *t, int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid,
                          int32_t *residues_out, int64_t *k, void *ws, cudaStream_t s, int part, int nparts,
                          int64_t *keys_out) {
    if (!p->tct_ok) return TM_EUNSUPPORTED;
    if (batch == 0) return TM_OK;
    if (batch > 65535) return TM_EUNSUPPORTED;
    const Geo g = geometry(p, batch);
    TiledArgs T{};
    tm_tc_fill_args(p, y1, y2, t, ldt, nullptr, nullptr, nullptr, nullptr, nullptr, T.a);
    T.a.ldy[0] = ldy1; T.a.ldy[1] = ldy2;
    T.a.dbg = tm_tc_dbg_buffer();
    T.a.NC = g.NC;
    T.a.NA[0] = g.NA[0]; T.a.NA[1] = g.NA[1];
    T.NT = g.NT;
    T.lmax = g.lmax; T.np = g.np; T.S = g.S; T.JT = g.JT; T.n_pcta = g.n_pcta;
    T.n_at = g.n_at;
    // split correlation: part `part` of `nparts` takes a contiguous
    // range of output tiles
    T.at0 = (int)((int64_t)T.n_at * part / nparts);
    T.n_atp = (int)((int64_t)T.n_at * (part + 1) / nparts) - T.at0;
    // template ranges: minimise waves x blocks per CTA over 2 resident CTAs per SM
    // (a grid just over one wave doubles the time), fewer ranges on near-ties
    // (each extra range adds one partial sum per output)
    // cost model (us): MMA time of the busiest CTA slot, 4 k-steps x ~2 limbs x the
    // shared-memory-operand MMA ((4096 + 64 NT) / 128 cycles), plus the partial sums'
    // write + read (several ranges) at ~6 TB/s of L2
    const int NC = g.NC;
    const int64_t slots = 2 * (int64_t)p->num_sms;
    const double xmax = (p->flags & TM_BINARY) ? 1.0 : 128.0;
    const double ybound = xmax * (double)(p->q1 > p->q2 ? p->q1 : p->q2);
    const double t_block = 4.0 * 2.0 * (4096.0 + 64.0 * g.NT) / 128.0 / 1900.0 * 2.0;  // 2 CTAs share an SM
    int n_cr = 1;
    double best = 1e300;
    // tiles alone (nearly) filling the SMs: one range, no partial sums (the cost model's
    // two-CTAs-per-SM time overstates one CTA per SM: cfg4 K = 16384 NT = 64, 1 vs 2 ranges
    // 63 vs 110 us)
    const bool one_range = batch * std::max(T.n_atp, 1) * 20 >= (int64_t)p->num_sms * 17;
    for (int c = 1; c <= (one_range ? 1 : g.max_cr); ++c) {
        const int64_t ctas = batch * std::max(T.n_atp, 1) * c;
        const int cr_blocks = (NC + c - 1) / c;
        const bool p32 = (double)cr_blocks * P * xmax * ybound < 2147483647.0;
        const double part = c > 1 ? (double)c * batch * (p->M1 + p->M2) * (p32 ? 4.0 : 8.0) * 3.0 / 6.0e6 : 0.0;
        const double cost = (double)((ctas + slots - 1) / slots) * (double)cr_blocks * t_block + part;
        if (cost < best * 0.97) { best = cost; n_cr = c; }
    }
    {
        static const char *env_ncr = getenv("TM_TILED_NCR");  // A/B: force the template-range count
        if (env_ncr && atoi(env_ncr) >= 1) n_cr = std::min(atoi(env_ncr), g.max_cr);
    }
    T.CR = (NC + n_cr - 1) / n_cr;
    T.n_cr = (NC + T.CR - 1) / T.CR;
    T.part32 = (double)T.CR * P * xmax * ybound < 2147483647.0;  // |partial| <= CR P max|t| max|y|
    {
        // several ranges: accumulate the partials with int64 red.add into one row
        // (exact; cfg5 correlation ~2 us less than storing 17 partial rows and summing
        // them); TM_TILED_ACC=0 stores and sums instead (A/B)
        const char *env_acc = getenv("TM_TILED_ACC");  // read per launch (tests flip it)
        T.accum = (T.n_cr > 1 && !(env_acc && env_acc[0] == '0')) ? 1 : 0;
    }
    char *w = (char *)ws;
    auto carve = [&](size_t bytes) { char *q = w; w += align_up256(bytes); return q; };
    int64_t nred_out = 0;  // the reduce kernel's outputs: this launch's tiles' MMA outputs
    {
        const int64_t klo = (int64_t)P * T.at0 * g.NT, kt = (int64_t)P * (T.at0 + T.n_atp) * g.NT;
        for (int j = 0; j < 2; ++j)
            nred_out += std::max<int64_t>(0, std::min<int64_t>(kt, std::min<int64_t>((int64_t)P * g.NA[j], j ? p->M2 : p->M1)) - klo);
    }
    const int nred_cta = (int)std::max<int64_t>(1, (nred_out + RED_T * RED_E - 1) / (RED_T * RED_E));
    T.nkey_cta = T.n_cr > 1 ? nred_cta : std::max(1, T.n_atp * T.n_cr);
    // a part of a split correlation without tiles launches neither the main kernel nor
    // tiled_reduce: nobody writes CTA keys, so finish_pair must read none (it took one
    // uninitialised key of the workspace for a real one)
    if (T.n_atp == 0) T.nkey_cta = 0;
    T.ckeys = (unsigned long long *)carve((size_t)batch * g.max_keys * 16);
    T.part = (int64_t *)carve(g.max_cr > 1 ? (size_t)batch * g.max_cr * (p->M1 + p->M2) * 8 : 0);
    T.bmag = (uint8_t *)carve((size_t)batch * g.S);
    T.spcnt = (int32_t *)carve((size_t)batch * g.n_pcta * 4);
    T.sprec = (int32_t *)carve((size_t)batch * g.n_pcta * 3 * SPE * 4);
    T.spair = (int32_t *)carve((size_t)batch * SPREC * 4);
    {
        // sparse single-limb mode: plans that may need >= 2 limbs, except +-1 plans whose
        // bins (sums of q signs, sd sqrt(q)) leave int8 often (sqrt(q) > 127 / 3: cfg4b,
        // cfg5 -- there the records and the decision only cost time); TM_TILED_SPARSE=0 /
        // 1: never / always (A/B)
        const char *env_sp = getenv("TM_TILED_SPARSE");  // read per launch (tests flip it)
        const int64_t qmax = p->q1 > p->q2 ? p->q1 : p->q2;
        T.sparse = g.lmax >= 2 && (!(p->flags & TM_BINARY) || 9 * qmax <= 127 * 127) ? 1 : 0;
        if (env_sp) T.sparse = (g.lmax >= 2 && env_sp[0] == '1') ? 1 : 0;
        // the template staged in shared memory for one-range sparse corrections: <= 16 KB
        // (NT = 32 keeps two CTAs per SM)
        T.tsm = (T.sparse && p->K <= 16384) ? (int)((p->K + 15) / 16 * 16) : 0;
    }
    T.planes = (uint8_t *)carve((size_t)batch * g.np * 8 * 32 * g.S);
    T.aimg = (uint8_t *)carve((size_t)batch * g.JT * 256);
    T.lpart = (int64_t *)carve((size_t)batch * g.n_pcta * 2 * MAXLEFT * 8);
    T.done = (unsigned *)carve((size_t)batch * 4);
    T.resid = resid; T.residues_out = residues_out; T.k_out = k; T.keys_out = keys_out;
    T.with_left = part == nparts - 1;  // the leftover outputs: the last part (its windows hold their y)
    T.r_out[0] = (int64_t *)r1;
    T.r_out[1] = (int64_t *)r2;
    {
        const cudaError_t e = launch_pdl(tiled_prep, dim3((unsigned)g.n_pcta, (unsigned)batch), dim3(PREP_T), 0, s, T);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_correlate: tiled_prep");
        TM_CHECK_LAUNCH("tm_correlate: tiled_prep");
    }
    const dim3 grid((unsigned)(T.n_atp * T.n_cr), (unsigned)batch);
    const dim3 gr((unsigned)nred_cta, (unsigned)batch);
    // corrections during the loop: one-range sparse plans whose grid has at most one CTA
    // per SM anyway (the buffer would otherwise cost the second resident CTA)
    T.csm = 0;
#ifndef TM_NO_CSM
    if (T.tsm && T.n_cr == 1 && (int64_t)grid.x * batch <= p->num_sms) {
        const int csm = NTHR * g.NT * 4;
        const int base = (g.NT == 64 ? smem_bytes<64>() : smem_bytes<32>()) + T.tsm;
        if (base + csm + 4096 <= 227 * 1024) T.csm = csm;  // (+ the static shared memory)
    }
#endif
    T.n_last = T.n_cr > 1 ? (int)gr.x : T.n_atp * T.n_cr;
    cudaError_t e = cudaSuccess;
    if (T.n_atp > 0) {
        if (g.NT == 64) {
            const int sb = smem_bytes<64>() + T.tsm + T.csm;
            e = tm_smem_attr((const void *)corr_tc_tiled<64>, sb);
            if (e == cudaSuccess) e = launch_pdl(corr_tc_tiled<64>, grid, dim3(TNTHR), sb, s, T);
        } else {
            const int sb = smem_bytes<32>() + T.tsm + T.csm;
            e = tm_smem_attr((const void *)corr_tc_tiled<32>, sb);
            if (e == cudaSuccess) e = launch_pdl(corr_tc_tiled<32>, grid, dim3(TNTHR), sb, s, T);
        }
        if (e != cudaSuccess) return tm_cuda_status(e, "corr_tc_tiled");
        TM_CHECK_LAUNCH("corr_tc_tiled");
        if (T.n_cr > 1) {
            e = T.part32 ? launch_pdl(tiled_reduce<int32_t>, gr, dim3(RED_T), 0, s, T)
                         : launch_pdl(tiled_reduce<int64_t>, gr, dim3(RED_T), 0, s, T);
            if (e != cudaSuccess) return tm_cuda_status(e, "tiled_reduce");
            TM_CHECK_LAUNCH("tiled_reduce");
        }
        return TM_OK;
    }
    e = launch_pdl(tc_tiled_final, dim3((unsigned)batch), dim3(FIN_T), 0, s, T);
    if (e != cudaSuccess) return tm_cuda_status(e, "tc_tiled_final");
    TM_CHECK_LAUNCH("tc_tiled_final");
    return TM_OK;
}
