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

constexpr int NT = 32;    // output blocks per tile (MMA N = 2 NT = 64)
constexpr int TCCH = 16;  // template blocks per A chunk
constexpr int KEY_SHIFT = 21;
constexpr int64_t KEY_BIAS = (int64_t)1 << 42;

struct TiledArgs {
    TcArgs a;              // y, t, K, M, NA, crt constants (NMC, R, NC unused except NC)
    int n_at, n_cr, CR;    // tiles over output blocks, template ranges, blocks per range
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

// smem: A [256 * (8 (TCCH-1) + 15)] | B [8 * 2 (NT + TCCH - 1) * 16] | tp slice | misc
constexpr int A_BYTES = 256 * (8 * (TCCH - 1) + 15);
constexpr int B_BYTES = 8 * 2 * (NT + TCCH - 1) * 16;
constexpr int TP_BYTES = 128 * TCCH + 256;
constexpr int SMEM_BYTES = A_BYTES + B_BYTES + TP_BYTES + 64;

__global__ void __launch_bounds__(NTHR, 2) corr_tc_tiled(const TiledArgs T) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const TcArgs &a = T.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t b = blockIdx.y;
    const int at = blockIdx.x % T.n_at, cr = blockIdx.x / T.n_at;
    const int a0 = at * NT;
    const int cb = cr * T.CR, ce = min(a.NC, cb + T.CR);
    uint8_t *A = sm, *B = sm + A_BYTES, *tp = B + B_BYTES;
    uint64_t *mdone = reinterpret_cast<uint64_t *>(tp + TP_BYTES);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(mdone + 1);
    int *nlflag = reinterpret_cast<int *>(mdone + 2);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(a.ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mdone)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // ---- limb count: scan this CTA's whole y window (blocks [a0 + cb, a0 + NT + ce - 1)) ----
    int fl = 0;
    {
        const int64_t s0 = a0 + cb, n = NT + (ce - cb) - 1;
        for (int j = 0; j < 2; ++j) {
            const int32_t *yr = a.y[j] + b * a.ldy[j];
            for (int64_t i = P * s0 + tid; i < P * (s0 + n) && i < a.len[j]; i += NTHR) {
                const int32_t v = yr[i];
                fl |= ((uint32_t)(v + 128) > 255u ? 1 : 0) | ((uint32_t)(v + 2048) > 4095u ? 2 : 0) |
                      ((uint32_t)(v + 32768) > 65535u ? 4 : 0);
            }
        }
    }
    fl = __syncthreads_or(fl & 1) | (__syncthreads_or(fl & 2) << 1) | (__syncthreads_or(fl & 4) << 2);
    int nl = (fl & 4) ? 4 : (fl & 2) ? 3 : (fl & 1) ? 2 : 1;
    if (nl > T.lmax) nl = T.lmax;
    (void)nlflag;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tslot;

    uint32_t pass = 0;
    for (int c0 = cb; c0 < ce; c0 += TCCH) {
        const int c1 = min(ce, c0 + TCCH);
        const int nrows = NT + (c1 - c0) - 1;  // B window: blocks [a0 + c0, a0 + c0 + nrows)
        for (int l = 0; l < nl; ++l) {
            if (pass > 0) group_wait<CtaSync>(mdone, (pass - 1) & 1u, warp);  // previous pass done with A, B
            if (l == 0) {
                // template slice: tp'[j] = t[128 c0 + j - 128] (zero outside [0, K))
                const int8_t *tr = a.t + b * a.ldt;
                for (int i = tid; i < TP_BYTES; i += NTHR) {
                    const int64_t j = 128 * (int64_t)c0 + i - 128;
                    tp[i] = (j >= 0 && j < a.K) ? (uint8_t)tr[j] : 0;
                }
                __syncthreads();
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
            stage_yw(a, B, b, l, nl, (int64_t)a0 + c0, nrows, warp, lane);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (warp == 0) {
                const uint32_t lbo = 32u * nrows;
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
                umma_commit(mdone);
            }
            ++pass;
        }
    }
    group_wait<CtaSync>(mdone, (pass - 1) & 1u, warp);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- epilogue: warp w: TMEM lanes 32 (w & 3) (rows b'), blocks a0 + 16 (w >> 2) + [0, 16)
    {
        const int qw = warp & 3, hw = warp >> 2;
        const int brow = P - 1 - (32 * qw + lane);
        const uint32_t taddr = tbase + ((uint32_t)(32 * qw) << 16);
        int64_t bv[2] = {INT64_MIN, INT64_MIN}, bk[2] = {INT64_MAX, INT64_MAX};
        for (int ar0 = 16 * hw; ar0 < 16 * hw + 16; ar0 += 8) {
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
            __syncthreads();
            if (tid == 0) *nlflag = (atomicAdd(T.tile_cnt + b * T.n_at + at, 1u) == (unsigned)(T.n_cr - 1));
            __syncthreads();
            if (*nlflag) {
                __threadfence();
                for (int ar0 = 16 * hw; ar0 < 16 * hw + 16; ++ar0) {
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
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(a.ncols));
}

// leftover outputs k in [128 NA_j, M_j) (at most MAXLEFT per modulus): CTA
// (K-slice, pair) adds its partial dot products into lsum (exact int64)
constexpr int LSLICE = 4096;
__global__ void __launch_bounds__(256) tc_tiled_leftover(const TiledArgs T) {
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

// per pair: tile keys + leftovers -> residues; steps 8-9 (tm_resolve)
__global__ void tc_tiled_final(const TiledArgs T, int64_t batch, int32_t *resid, int32_t *residues_out,
                               int64_t *k_out, int64_t *r_out0, int64_t *r_out1) {
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
        const int nleft = j ? nleft1 : nleft0;
        for (int q = 0; q < nleft; ++q) {
            const int64_t r = T.lsum[b * 2 * MAXLEFT + (j ? nleft0 : 0) + q];
            const int64_t k = (int64_t)P * a.NA[j] + q;
            int64_t *ro = j ? r_out1 : r_out0;
            if (ro) ro[b * a.M[j] + k] = r;
            amax(bv, bk, r, k);
        }
        m[j] = bk;
    }
    if (resid) { resid[2 * b] = (int32_t)m[0]; resid[2 * b + 1] = (int32_t)m[1]; }
    if (residues_out) { residues_out[2 * b] = (int32_t)m[0]; residues_out[2 * b + 1] = (int32_t)m[1]; }
    if (k_out) k_out[b] = tm_resolve(m[0], m[1], a.M1, a.M2, a.crt_inv, a.N, a.crt_wrap);  // steps 8-9
}

}  // namespace

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
    if (p->K > ((int64_t)1 << 17)) return;                                  // per-limb |r| < 2^31
    if (p->M2 >= ((int64_t)1 << KEY_SHIFT)) return;
    p->tct_lmax = lmax;
    p->tct_ok = 1;
}

size_t tm_tc_tiled_ws_bytes(const tm_plan_s *p, int64_t batch) {
    if (!p->tct_ok) return 0;
    // keys [batch][2] | lsum [batch][2 MAXLEFT] | tile counters [batch][<= 2^KEY_SHIFT / (128 NT)] | racc
    return 256 + (size_t)batch * (16 + 16 * MAXLEFT + 4 * (((int64_t)1 << KEY_SHIFT) / (P * NT) + 1)) +
           (size_t)batch * (p->M1 + p->M2) * 8 + 1024;
}

// r1/r2 (int64, may be NULL), residues_out/resid (may be NULL), k (may be NULL).
int tm_tc_tiled_correlate(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2,
                          const void *t, int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid,
                          int32_t *residues_out, int64_t *k, void *ws, cudaStream_t s) {
    if (!p->tct_ok) return TM_EUNSUPPORTED;
    if (batch == 0) return TM_OK;
    if (batch > 65535) return TM_EUNSUPPORTED;
    TiledArgs T{};
    tm_tc_fill_args(p, y1, y2, t, ldt, nullptr, nullptr, nullptr, nullptr, nullptr, T.a);
    T.a.ldy[0] = ldy1; T.a.ldy[1] = ldy2;
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
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(2 * NT * T.lmax)) ncols *= 2;
    T.a.ncols = ncols;
    const int namax = T.a.NA[0] > T.a.NA[1] ? T.a.NA[0] : T.a.NA[1];
    T.n_at = (namax + NT - 1) / NT;
    // template ranges: enough CTAs for two per SM, ranges of >= 2 chunks
    int n_cr = 1;
    const int max_cr = (NC + 2 * TCCH - 1) / (2 * TCCH);
    while (n_cr < max_cr && batch * T.n_at * n_cr < 2 * p->num_sms) ++n_cr;
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
    cudaError_t e = cudaMemsetAsync(ws, 0, zero_bytes, s);
    if (e == cudaSuccess && T.n_cr > 1) {
        e = cudaMemsetAsync(T.racc[0], 0, (size_t)batch * p->M1 * 8, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(T.racc[1], 0, (size_t)batch * p->M2 * 8, s);
    }
    if (e != cudaSuccess) return tm_cuda_status(e, "tm_correlate: tiled reset");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(corr_tc_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        attr = true;
    }
    corr_tc_tiled<<<dim3((unsigned)(T.n_at * T.n_cr), (unsigned)batch), NTHR, SMEM_BYTES, s>>>(T);
    TM_CHECK_LAUNCH("corr_tc_tiled");
    const int nleft = (int)(std::max<int64_t>(0, p->M1 - (int64_t)P * T.a.NA[0]) +
                            std::max<int64_t>(0, p->M2 - (int64_t)P * T.a.NA[1]));
    if (nleft > 0) {
        tc_tiled_leftover<<<dim3((unsigned)((p->K + LSLICE - 1) / LSLICE), (unsigned)batch), 256, 0, s>>>(T);
        TM_CHECK_LAUNCH("tc_tiled_leftover");
    }
    tc_tiled_final<<<(unsigned)((batch + 127) / 128), 128, 0, s>>>(T, batch, resid, residues_out, k, (int64_t *)r1,
                                                                     (int64_t *)r2);
    TM_CHECK_LAUNCH("tc_tiled_final");
    return TM_OK;
}
