// corr_tc_tiled.cu -- the tensor-core correlation (corr_tc.cu, tc_core.cuh)
// split over many CTAs per pair, for long templates and small batches (cfg4:
// 64 pairs at K = 16384; cfg5: one pair at K = 65536) where one CTA per pair
// would leave most SMs idle or not fit in shared memory.
//
// CTA (pair b, output tile [a0, a0 + NT) blocks, template range [cb, ce)):
//   D[b'][2 (a - a0) + j] = sum_{c in [cb, ce)} A_c B_c   (P = 128 blocking of
//   corr_tc.cu), accumulated in TMEM over chunks of <= CCH template blocks;
//   per chunk the CTA stages the template slice, builds A (16 byte-shifted
//   copies), and stages the B window = y_j blocks [a0 + c0, a0 + NT + c1 - 1)
//   once per 4-bit limb (the limb count comes from a scan of the CTA's whole
//   y window, so every chunk uses the same decomposition).
// Epilogue: with one template range per pair, the tile's lowest-index maximum
// per modulus goes to an atomicMax on a packed key (r + 2^42) << 21 | (2^21 -
// 1 - k) (max r, ties to the lowest k); with several ranges the tile's partial
// r are added (int64 atomics, exact) into r, and the CTA that completes a
// tile's last range reduces the tile's final r to the same packed key.
// tc_tiled_leftover computes the <= 8 outputs k in [128 NA_j, M_j) per
// modulus (dot products split over K-slices), and tc_tiled_final combines keys
// and leftovers per pair and does steps 8-9 (tm_resolve).
#include <algorithm>

#include "tc_core.cuh"

namespace {
using namespace tc;

constexpr int NT_MIN = 32;  // output blocks per tile: NT in {32, 64} (MMA N = 2 NT)
constexpr int TCCH = 16;  // template blocks per A chunk
constexpr int KEY_SHIFT = 21;
constexpr int64_t KEY_BIAS = (int64_t)1 << 42;

struct TiledArgs {
    TcArgs a;              // y, t, K, M, NA, crt constants (NMC, R, NC unused except NC)
    int n_at, n_cr, CR;    // tiles over output blocks, template ranges, blocks per range
    int at0, n_atp;        // this launch's tiles [at0, at0 + n_atp) (a part of a split correlation)
    int lmax;
    unsigned long long *keys;  // [batch][2] (n_cr == 1), zeroed
    int64_t *racc[2];          // [batch][Mj] partial sums (n_cr > 1), zeroed; or r outputs
    int write_r;               // n_cr == 1: store r values (staged tm_correlate)
    unsigned *tile_cnt;        // [batch][n_at] template ranges finished per tile (n_cr > 1), zeroed
    int64_t *lsum;             // [batch][2 MAXLEFT] leftover dot products, zeroed
};

__device__ __forceinline__ unsigned long long pack_key(int64_t r, int64_t k) {
    return ((unsigned long long)(r + KEY_BIAS) << KEY_SHIFT) | (unsigned long long)(((int64_t)1 << KEY_SHIFT) - 1 - k);
}

// smem: A [2][256 * (8 (TCCH-1) + 15)] | B [2][8 * 2 (NT + TCCH - 1) * 16] | tp slice | misc.
// Passes (chunk, limb) alternate between the two A and B buffers, so the
// staging of pass p + 1 overlaps the MMAs of pass p (mbarrier mdone[p & 1]).
// An SS MMA costs ~(4096 + 32 N) / 128 cycles (shared-memory operand reads), so
// N = 128 (NT = 64) does twice the work of N = 64 in 1.33x the time.
constexpr int A_BYTES = (256 * (8 * (TCCH - 1) + 15) + 127) / 128 * 128;
template <int NT>
constexpr int b_bytes() { return (8 * (2 * (NT + TCCH - 1) * 16 + 16) + 127) / 128 * 128; }
// B chunk-column stride: 32 nrows + 16 bytes, an odd multiple of 16 modulo 128, so
// the 8 chunk columns a warp's store touches fall in distinct bank quads
__device__ __forceinline__ uint32_t b_lbo(int nrows) { return 32u * nrows + 16u; }
constexpr int TP_BYTES = 128 * TCCH + 256;
template <int NT>
constexpr int smem_bytes() { return 2 * A_BYTES + 2 * b_bytes<NT>() + TP_BYTES + 64; }

// Warp roles: warps 0-7 stage (limb scan, template slices, A copies, B windows,
// epilogue); warp 8 only issues the MMAs, so that staging pass p + 1 overlaps
// the tensor core working on pass p (with one warp doing both, the issue loop
// blocks on the tensor core's queue and staging and MMAs serialise).
// Named barriers: 1 + (p & 1) "pass p staged" (256 arrive, issuer syncs), 3 the
// 256 staging threads.
constexpr int TNTHR = NTHR + 32;
__device__ __forceinline__ void stagers_sync() { asm volatile("bar.sync 3, %0;" ::"n"(NTHR) : "memory"); }

// Stage limb l of the B window (y_1 and y_2 blocks s_begin + [0, nrows)) with
// both moduli's rows in one batch of loads: row r = 2 s + j, warp w takes rows
// w + 8 u, RB rows in flight per warp (one L2 round trip per pass at NT = 32;
// the one-CTA kernel's stage_yw walks the moduli one after the other).
template <int RB>
__device__ __forceinline__ void stage_window(const TcArgs &a, uint8_t *B, int64_t b, int l, int nl, int64_t s_begin,
                                             int nrows, int warp, int lane) {
    const uint32_t lbo = b_lbo(nrows);
    const int h = lane >> 2, wq = lane & 3;
    const int32_t *yr0 = a.y[0] + b * a.ldy[0], *yr1 = a.y[1] + b * a.ldy[1];
    const bool al0 = ((((uintptr_t)yr0) & 15) == 0), al1 = ((((uintptr_t)yr1) & 15) == 0);
    for (int r0 = warp; r0 < 2 * nrows; r0 += RB * (NTHR / 32)) {
        int32_t v[RB][4];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int r = r0 + u * (NTHR / 32), j = r & 1;
            const int64_t i0 = (int64_t)P * (s_begin + (r >> 1)) + 4 * lane;
            const int32_t *yr = j ? yr1 : yr0;
            const int64_t len = a.len[j];
            v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0;
            if (r < 2 * nrows && i0 >= 0) {
                if ((j ? al1 : al0) && i0 + 4 <= len) {
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
            const int r = r0 + u * (NTHR / 32);
            if (r >= 2 * nrows) break;
            *reinterpret_cast<uint32_t *>(B + lbo * h + 16 * r + 4 * wq) =
                nl == 1 ? pack4(v[u][0], v[u][1], v[u][2], v[u][3])
                        : pack4(limb(v[u][0], l, nl), limb(v[u][1], l, nl), limb(v[u][2], l, nl), limb(v[u][3], l, nl));
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(TNTHR, 2) corr_tc_tiled(const TiledArgs T) {
    pdl_trigger();
    pdl_wait();
    constexpr int B_BYTES = b_bytes<NT>();
    extern __shared__ __align__(1024) uint8_t sm[];
    const TcArgs &a = T.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t b = blockIdx.y;
    const int at = T.at0 + blockIdx.x % T.n_atp, cr = blockIdx.x / T.n_atp;
    const int a0 = at * NT;
    const int cb = cr * T.CR, ce = min(a.NC, cb + T.CR);
    uint8_t *Abuf = sm, *Bbuf = sm + 2 * A_BYTES, *tp = Bbuf + 2 * B_BYTES;
    uint64_t *mdone = reinterpret_cast<uint64_t *>(tp + TP_BYTES);  // [2]
    uint32_t *tslot = reinterpret_cast<uint32_t *>(mdone + 2);
    int *nlflag = reinterpret_cast<int *>(mdone + 3);
    long long ts[8] = {gtime(), 0, 0, 0, 0, 0, 0, 0};  // instrumentation (a.dbg): phase stamps
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mdone)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mdone + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // ---- limb count: scan this CTA's whole y window (blocks [a0 + cb, a0 + NT + ce - 1)),
    // 16-byte loads with several in flight (a latency-bound scalar scan cost ~30% of the kernel)
    int fl = 0;
    {
        const int64_t s0 = a0 + cb, n = NT + (ce - cb) - 1;
        uint32_t mag = 0;  // OR of v ^ (v >> 31): below 2^b iff every v fits b + 1 signed bits
        for (int j = 0; j < 2 && tid < NTHR; ++j) {
            const int32_t *yr = a.y[j] + b * a.ldy[j];
            const int64_t lo = P * s0, hi = min(P * (s0 + n), a.len[j]);
            if (hi <= lo) continue;
            if ((((uintptr_t)(yr + lo)) & 15) == 0) {
                const int64_t n4 = (hi - lo) >> 2;
                const int4 *q = reinterpret_cast<const int4 *>(yr + lo);
#pragma unroll 4
                for (int64_t i = tid; i < n4; i += NTHR) {
                    const int4 v = q[i];
                    mag |= (uint32_t)(v.x ^ (v.x >> 31)) | (uint32_t)(v.y ^ (v.y >> 31)) |
                           (uint32_t)(v.z ^ (v.z >> 31)) | (uint32_t)(v.w ^ (v.w >> 31));
                }
                for (int64_t i = lo + 4 * n4 + tid; i < hi; i += NTHR) mag |= (uint32_t)(yr[i] ^ (yr[i] >> 31));
            } else {
#pragma unroll 4
                for (int64_t i = lo + tid; i < hi; i += NTHR) mag |= (uint32_t)(yr[i] ^ (yr[i] >> 31));
            }
        }
        fl = (mag > 127u ? 1 : 0) | (mag > 2047u ? 2 : 0) | (mag > 32767u ? 4 : 0);
    }
    fl = __syncthreads_or(fl & 1) | (__syncthreads_or(fl & 2) << 1) | (__syncthreads_or(fl & 4) << 2);
    int nl = (fl & 4) ? 4 : (fl & 2) ? 3 : (fl & 1) ? 2 : 1;
    if (nl > T.lmax) nl = T.lmax;
    // TMEM: 2 NT columns per limb, allocated after the scan so that two CTAs fit
    // per SM whenever 2 NT nl <= 256
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(2 * NT * nl)) ncols *= 2;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    (void)nlflag;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tslot;
    ts[1] = gtime();

    // pass q = (chunk, limb) uses A[chunk & 1], B[q & 1] and commits to mdone[q & 1]
    // (its (q >> 1)-th phase).  Before staging pass q the stagers wait for pass q - 2,
    // which (commits being cumulative) also frees the A buffer of chunk - 2.
    uint32_t pass = 0;
    if (warp == NTHR / 32) {
        // ---- MMA issuer
        int ch = 0;
        for (int c0 = cb; c0 < ce; c0 += TCCH, ++ch) {
            const int c1 = min(ce, c0 + TCCH);
            const int nrows = NT + (c1 - c0) - 1;
            const uint8_t *A = Abuf + (ch & 1) * A_BYTES;
            for (int l = 0; l < nl; ++l) {
                const uint8_t *B = Bbuf + (pass & 1) * B_BYTES;
                if (pass & 1) asm volatile("bar.sync 2, %0;" ::"n"(TNTHR) : "memory");
                else asm volatile("bar.sync 1, %0;" ::"n"(TNTHR) : "memory");
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t lbo = b_lbo(nrows);
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
                umma_commit(mdone + (pass & 1));
                ++pass;
            }
        }
    } else {
        // ---- stagers.  The template slice of the next chunk is prefetched into
        // registers (tw_) while the current chunk is staged.
        constexpr int TPW = TP_BYTES / 4;
        uint32_t tw_[(TPW + NTHR - 1) / NTHR];
        auto load_slice = [&](int c0v) {  // tp'[j] = t[128 c0v + j - 128] (zero outside [0, K))
            const int8_t *tr = a.t + b * a.ldt;
            const int64_t base = 128 * (int64_t)c0v - 128;
            const bool fast = base >= 0 && base + TP_BYTES <= a.K && ((((uintptr_t)(tr + base)) & 3) == 0);
#pragma unroll
            for (int u = 0; u < (TPW + NTHR - 1) / NTHR; ++u) {
                const int i = tid + u * NTHR;
                if (i >= TPW) break;
                if (fast) {
                    tw_[u] = __ldg(reinterpret_cast<const uint32_t *>(tr + base) + i);
                } else {
                    uint32_t w = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t j = base + 4 * i + e;
                        if (j >= 0 && j < a.K) w |= (uint32_t)(uint8_t)tr[j] << (8 * e);
                    }
                    tw_[u] = w;
                }
            }
        };
        load_slice(cb);
        int ch = 0;
        for (int c0 = cb; c0 < ce; c0 += TCCH, ++ch) {
            const int c1 = min(ce, c0 + TCCH);
            const int nrows = NT + (c1 - c0) - 1;  // B window: blocks [a0 + c0, a0 + c0 + nrows)
            uint8_t *A = Abuf + (ch & 1) * A_BYTES;
            for (int l = 0; l < nl; ++l) {
                uint8_t *B = Bbuf + (pass & 1) * B_BYTES;
                long long tw = gtime();
                if (pass >= 2) mbar_wait(mdone + (pass & 1), ((pass - 2) >> 1) & 1u);
                long long tw2 = gtime();
                ts[4] += tw2 - tw;
                if (l == 0) {
                    stagers_sync();  // every stager is done reading the previous slice
#pragma unroll
                    for (int u = 0; u < (TPW + NTHR - 1) / NTHR; ++u)
                        if (tid + u * NTHR < TPW) reinterpret_cast<uint32_t *>(tp)[tid + u * NTHR] = tw_[u];
                    stagers_sync();
                    if (c1 < ce) load_slice(c1);
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
                        reinterpret_cast<uint4 *>(A)[c] = o;
                    }
                }
                ts[5] += gtime() - tw2;  // template slice + A build
                tw2 = gtime();
                stage_window<12>(a, B, b, l, nl, (int64_t)a0 + c0, nrows, warp, lane);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                if (pass & 1) asm volatile("bar.arrive 2, %0;" ::"n"(TNTHR) : "memory");
                else asm volatile("bar.arrive 1, %0;" ::"n"(TNTHR) : "memory");
                ts[6] += gtime() - tw2;  // B staging
                ++pass;
            }
        }
    }
    mbar_wait(mdone + ((pass - 1) & 1), ((pass - 1) >> 1) & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    ts[2] = gtime();

    // ---- epilogue (warps 0-7): warp w: TMEM lanes 32 (w & 3) (rows b'), blocks a0 + (NT / 2) (w >> 2) + [0, NT / 2)
    if (warp < NTHR / 32) {
        const int qw = warp & 3, hw = warp >> 2;
        const int brow = P - 1 - (32 * qw + lane);
        const uint32_t taddr = tbase + ((uint32_t)(32 * qw) << 16);
        int64_t bv[2] = {INT64_MIN, INT64_MIN}, bk[2] = {INT64_MAX, INT64_MAX};
        for (int ar0 = (NT / 2) * hw; ar0 < (NT / 2) * hw + NT / 2; ar0 += 8) {
            int64_t r[8][2];
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i][0] = r[i][1] = 0;
            for (int l = 0; l < nl; ++l) {
                int32_t v[16];
                tmem_ld16(taddr + 2 * NT * l + 2 * ar0, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    r[i][0] += (int64_t)v[2 * i] * ((int64_t)1 << (4 * l));
                    r[i][1] += (int64_t)v[2 * i + 1] * ((int64_t)1 << (4 * l));
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t ab = a0 + ar0 + i;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int64_t k = P * ab + brow;
                    if (ab < a.NA[j] && k < a.M[j]) {
                        if (T.n_cr > 1) {
                            atomicAdd(reinterpret_cast<unsigned long long *>(T.racc[j] + b * a.M[j] + k),
                                      (unsigned long long)r[i][j]);
                        } else {
                            if (T.write_r) T.racc[j][b * a.M[j] + k] = r[i][j];
                            amax(bv[j], bk[j], r[i][j], k);
                        }
                    }
                }
            }
        }
        if (T.n_cr > 1) {
            // the CTA that completes a tile's last template range reduces its final r
            __threadfence();
            stagers_sync();
            if (tid == 0) *nlflag = (atomicAdd(T.tile_cnt + b * T.n_at + at, 1u) == (unsigned)(T.n_cr - 1));
            stagers_sync();
            if (*nlflag) {
                __threadfence();
                for (int ar0 = (NT / 2) * hw; ar0 < (NT / 2) * hw + NT / 2; ++ar0) {
                    const int64_t ab = a0 + ar0;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int64_t k = P * ab + brow;
                        if (ab < a.NA[j] && k < a.M[j]) amax(bv[j], bk[j], __ldcg(T.racc[j] + b * a.M[j] + k), k);
                    }
                }
            }
        }
        if (T.n_cr == 1 || *nlflag) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int64_t ov = __shfl_xor_sync(0xffffffffu, bv[j], o);
                    const int64_t ok = __shfl_xor_sync(0xffffffffu, bk[j], o);
                    amax(bv[j], bk[j], ov, ok);
                }
                if (lane == 0 && bk[j] != INT64_MAX) atomicMax(T.keys + 2 * b + j, pack_key(bv[j], bk[j]));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (a.dbg && tid == 0) {
        ts[3] = gtime();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        ts[7] = ((long long)smid << 32) | ((long long)pass << 8) | nl;
        long long *d = a.dbg + 8 * ((int64_t)blockIdx.y * gridDim.x + blockIdx.x);
        for (int i = 0; i < 8; ++i) d[i] = ts[i];
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols));
}

// leftover outputs k in [128 NA_j, M_j) (at most MAXLEFT per modulus): CTA
// (K-slice, pair) adds its partial dot products into lsum (exact int64)
constexpr int LSLICE = 1024;  // K-slice per CTA (4 terms per thread: latency-bound loop)
__global__ void __launch_bounds__(256) tc_tiled_leftover(const TiledArgs T) {
    pdl_trigger();
    pdl_wait();
    const TcArgs &a = T.a;
    const int64_t b = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t i0 = (int64_t)blockIdx.x * LSLICE, i1 = min(a.K, i0 + LSLICE);
    __shared__ int64_t part[8];
    const int nleft0 = (int)max((int64_t)0, a.M[0] - (int64_t)P * a.NA[0]);
    const int nleft1 = (int)max((int64_t)0, a.M[1] - (int64_t)P * a.NA[1]);
    const int8_t *tr = a.t + b * a.ldt;
    for (int q = 0; q < nleft0 + nleft1; ++q) {
        const int j = q < nleft0 ? 0 : 1;
        const int64_t k = (int64_t)P * a.NA[j] + (j ? q - nleft0 : q);
        const int32_t *yr = a.y[j] + b * a.ldy[j] + k;
        int64_t sum = 0;
#pragma unroll 4
        for (int64_t i = i0 + tid; i < i1; i += 256) sum += (int64_t)tr[i] * yr[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) part[warp] = sum;
        __syncthreads();
        if (tid == 0) {
            int64_t tot = 0;
            for (int w = 0; w < 8; ++w) tot += part[w];
            atomicAdd(reinterpret_cast<unsigned long long *>(T.lsum + b * 2 * MAXLEFT + q), (unsigned long long)tot);
        }
        __syncthreads();
    }
}

// workspace reset as a PDL kernel (a memset would end the overlap of launches)
__global__ void tiled_zero(int32_t *p0, int64_t n0, int32_t *p1, int64_t n1, int32_t *p2, int64_t n2) {
    pdl_trigger();
    pdl_wait();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1 + n2; i += stride) {
        if (i < n0) p0[i] = 0;
        else if (i < n0 + n1) p1[i - n0] = 0;
        else p2[i - n0 - n1] = 0;
    }
}

// per pair: tile keys + leftovers -> residues; steps 8-9 (tm_resolve)
__global__ void tc_tiled_final(const TiledArgs T, int64_t batch, int32_t *resid, int32_t *residues_out,
                               int64_t *k_out, int64_t *r_out0, int64_t *r_out1, int64_t *keys_out, int with_left) {
    pdl_trigger();
    pdl_wait();
    const TcArgs &a = T.a;
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const int nleft0 = (int)max((int64_t)0, a.M[0] - (int64_t)P * a.NA[0]);
    const int nleft1 = (int)max((int64_t)0, a.M[1] - (int64_t)P * a.NA[1]);
    int64_t m[2];
    for (int j = 0; j < 2; ++j) {
        int64_t bv = INT64_MIN, bk = INT64_MAX;
        const unsigned long long key = T.keys[2 * b + j];
        if (key) {
            bk = ((int64_t)1 << KEY_SHIFT) - 1 - (int64_t)(key & (((unsigned long long)1 << KEY_SHIFT) - 1));
            bv = (int64_t)(key >> KEY_SHIFT) - KEY_BIAS;
        }
        const int nleft = with_left ? (j ? nleft1 : nleft0) : 0;
        for (int q = 0; q < nleft; ++q) {
            const int64_t r = T.lsum[b * 2 * MAXLEFT + (j ? nleft0 : 0) + q];
            const int64_t k = (int64_t)P * a.NA[j] + q;
            int64_t *ro = j ? r_out1 : r_out0;
            if (ro) ro[b * a.M[j] + k] = r;
            amax(bv, bk, r, k);
        }
        m[j] = bk;
        if (keys_out)  // split correlation: this part's (max r, lowest k) as an order-preserving int64
            keys_out[2 * b + j] = bk == INT64_MAX ? INT64_MIN : (int64_t)(pack_key(bv, bk) ^ (1ull << 63));
    }
    if (keys_out) return;
    if (resid) { resid[2 * b] = (int32_t)m[0]; resid[2 * b + 1] = (int32_t)m[1]; }
    if (residues_out) { residues_out[2 * b] = (int32_t)m[0]; residues_out[2 * b + 1] = (int32_t)m[1]; }
    if (k_out) k_out[b] = tm_resolve(m[0], m[1], a.M1, a.M2, a.crt_inv, a.N, a.crt_wrap);  // steps 8-9
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
// |r| fits the packed key) and geometry.
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
    if (!p->tct_ok) return 0;
    // keys [batch][2] | lsum [batch][2 MAXLEFT] | tile counters [batch][<= 2^KEY_SHIFT / (128 NT)] | racc
    return 256 + (size_t)batch * (16 + 16 * MAXLEFT + 4 * (((int64_t)1 << KEY_SHIFT) / (P * NT_MIN) + 1)) +
           (size_t)batch * (p->M1 + p->M2) * 8 + 1024;
}

// r1/r2 (int64, may be NULL), residues_out/resid (may be NULL), k (may be NULL).
int tm_tc_tiled_correlate(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2,
                          const void *t, int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid,
                          int32_t *residues_out, int64_t *k, void *ws, cudaStream_t s, int part, int nparts,
                          int64_t *keys_out) {
    if (!p->tct_ok) return TM_EUNSUPPORTED;
    if (batch == 0) return TM_OK;
    if (batch > 65535) return TM_EUNSUPPORTED;
    TiledArgs T{};
    tm_tc_fill_args(p, y1, y2, t, ldt, nullptr, nullptr, nullptr, nullptr, nullptr, T.a);
    T.a.ldy[0] = ldy1; T.a.ldy[1] = ldy2;
    T.a.dbg = tm_tc_dbg_buffer();
    // the tiles cover NA_j = the plan's block counts (computed here: tc_ok may be false)
    const int NC = (int)((p->K + P - 2) / P) + 1;
    T.a.NC = NC;
    for (int j = 0; j < 2; ++j) {
        const int64_t M = j ? p->M2 : p->M1;
        int64_t na = M / P;
        if (M - na * P > MAXLEFT) ++na;
        if (na < 1) na = 1;
        T.a.NA[j] = (int)na;
    }
    T.lmax = p->tct_lmax;
    const char *env_nt = getenv("TM_TILED_NT");  // A/B: "32" (default, measured faster) or "64"
    const int NT = (env_nt && atoi(env_nt) == 64) ? 64 : 32;
    const int namax = T.a.NA[0] > T.a.NA[1] ? T.a.NA[0] : T.a.NA[1];
    T.n_at = (namax + NT - 1) / NT;
    // split correlation: part `part` of `nparts` takes a contiguous
    // range of output tiles
    T.at0 = (int)((int64_t)T.n_at * part / nparts);
    T.n_atp = (int)((int64_t)T.n_at * (part + 1) / nparts) - T.at0;
    // template ranges: minimise waves x blocks per CTA over 2 resident CTAs per SM
    // (a grid just over one wave doubles the time), fewer ranges on near-ties
    // (each extra range adds one int64 atomic per output)
    const int max_cr = std::max(1, (NC + 2 * TCCH - 1) / (2 * TCCH));
    const int64_t slots = 2 * (int64_t)p->num_sms;
    int n_cr = 1;
    double best = 1e300;
    for (int c = 1; c <= max_cr; ++c) {
        const int64_t ctas = batch * std::max(T.n_atp, 1) * c;
        const double cost = (double)((ctas + slots - 1) / slots) * (double)((NC + c - 1) / c);
        if (cost < best * 0.95) { best = cost; n_cr = c; }
    }
    T.CR = (NC + n_cr - 1) / n_cr;
    T.n_cr = (NC + T.CR - 1) / T.CR;
    char *w = (char *)ws;
    auto carve = [&](size_t bytes) { char *q = w; w += (bytes + 255) / 256 * 256; return q; };
    T.keys = (unsigned long long *)carve((size_t)batch * 16);
    T.lsum = (int64_t *)carve((size_t)batch * 16 * MAXLEFT);
    T.tile_cnt = (unsigned *)carve((size_t)batch * T.n_at * 4);
    const size_t zero_bytes = (size_t)(w - (char *)ws);  // keys, lsum, counters: one memset
    int64_t *racc = (int64_t *)carve((size_t)batch * (p->M1 + p->M2) * 8);
    T.racc[0] = r1 ? (int64_t *)r1 : racc;
    T.racc[1] = r2 ? (int64_t *)r2 : racc + batch * p->M1;
    T.write_r = (r1 != nullptr);
    {
        const int64_t n0 = (int64_t)(zero_bytes / 4);
        const int64_t n1 = T.n_cr > 1 ? batch * p->M1 * 2 : 0, n2 = T.n_cr > 1 ? batch * p->M2 * 2 : 0;
        const int64_t blocks = std::min<int64_t>((n0 + n1 + n2 + 255) / 256, 4 * (int64_t)p->num_sms);
        const cudaError_t e = launch_pdl(tiled_zero, dim3((unsigned)blocks), dim3(256), 0, s, (int32_t *)ws, n0,
                                         (int32_t *)T.racc[0], n1, (int32_t *)T.racc[1], n2);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_correlate: tiled reset");
        TM_CHECK_LAUNCH("tm_correlate: tiled reset");
    }
    {
        cudaError_t e = tm_smem_attr((const void *)corr_tc_tiled<32>, (int)smem_bytes<32>());
        if (e == cudaSuccess) e = tm_smem_attr((const void *)corr_tc_tiled<64>, (int)smem_bytes<64>());
        if (e != cudaSuccess) return tm_cuda_status(e, "corr_tc_tiled: shared-memory attribute");
    }
    const dim3 grid((unsigned)(T.n_atp * T.n_cr), (unsigned)batch);
    if (T.n_atp > 0) {
        const cudaError_t e = NT == 32 ? launch_pdl(corr_tc_tiled<32>, grid, dim3(TNTHR), smem_bytes<32>(), s, T)
                                       : launch_pdl(corr_tc_tiled<64>, grid, dim3(TNTHR), smem_bytes<64>(), s, T);
        if (e != cudaSuccess) return tm_cuda_status(e, "corr_tc_tiled");
        TM_CHECK_LAUNCH("corr_tc_tiled");
    }
    const int nleft = (int)(std::max<int64_t>(0, p->M1 - (int64_t)P * T.a.NA[0]) +
                            std::max<int64_t>(0, p->M2 - (int64_t)P * T.a.NA[1]));
    const int with_left = part == 0;  // the leftover outputs belong to part 0
    if (nleft > 0 && with_left) {
        const cudaError_t e = launch_pdl(tc_tiled_leftover, dim3((unsigned)((p->K + LSLICE - 1) / LSLICE), (unsigned)batch),
                                         dim3(256), 0, s, T);
        if (e != cudaSuccess) return tm_cuda_status(e, "tc_tiled_leftover");
        TM_CHECK_LAUNCH("tc_tiled_leftover");
    }
    {
        const cudaError_t e = launch_pdl(tc_tiled_final, dim3((unsigned)((batch + 127) / 128)), dim3(128), 0, s, T,
                                         batch, resid, residues_out, k, (int64_t *)r1, (int64_t *)r2, keys_out,
                                         with_left);
        if (e != cudaSuccess) return tm_cuda_status(e, "tc_tiled_final");
    }
    TM_CHECK_LAUNCH("tc_tiled_final");
    return TM_OK;
}
