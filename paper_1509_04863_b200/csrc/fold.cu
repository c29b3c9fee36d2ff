// fold.cu -- tm_fold: the O(N)-addition downsampling of Algorithm 1 step 3
// (Eq. 2) for both co-prime moduli, restricted
// to a chunk [offset, offset+len) of global positions (partial fold).
//
// Kernels:
//  * fold_general  -- any N, M, dtype, chunk: one thread per output entry k,
//                     y[k] = sum_i x[(k + i M) mod N] over chunk positions.
//  * the packed +-1 kernel fold_pm1_tma (fold_tma.cu; TM_BINARY, M1 | N,
//    M1 % 512 == 0, row-aligned chunks): ONE pass over x feeds both moduli.
//    With x viewed as rows of M1 columns, x[g][c] = x[g*M1 + c]:
//      - M1 bin of (g, c) is c           (column sums),
//      - M2 bin of (g, c) is (c - g) mod M2, because M1 = -1 (mod M1+1): an
//        anti-diagonal.
//    Each lane owns 16 columns (one 16-byte load per row).  A +-1 byte b is
//    0x01 or 0xFF, so (b & 0x02) is 2*[b == -1]: the kernel counts negatives
//    two at a time in byte lanes (SWAR) and converts  y = n - 2*neg  at the end.
//    For the anti-diagonals a lane's 16 x 16 tile spans 31 bins; rows are
//    grouped by (row mod 4) so every add is word-aligned, and the byte shift
//    is applied once per tile with funnel shifts.  A finished 16-bin block
//    moves lane l -> l+1 (warp shuffle) one tile later, because lane l+1 at
//    tile a+1 covers the same anti-diagonals as lane l at tile a (systolic).
//  * fold_finalize -- converts counts to values and adds the terms Eq. 2 has
//    beyond the single count of every position: the mod-N wrap (reading C5;
//    the first s2 = q positions are counted a second time) and the
//    extension entries k in [M, M+K) (strategy 1, D_{M+K}):
//      y[M + c] = y[c] - x[c] + x[(c + s) mod N]  (exact identity of Eq. 2).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tm_internal.cuh"

namespace {

// ---------------------------------------------------------------------------
// general kernel
// ---------------------------------------------------------------------------
template <typename T, typename Acc>
__global__ void fold_general(const T *__restrict__ x, int64_t ldx, int64_t N, int64_t offset,
                             int64_t len, int64_t M1, int64_t M2, int64_t K, int64_t q1, int64_t q2,
                             Acc *__restrict__ y1, int64_t ldy1, Acc *__restrict__ y2, int64_t ldy2, int accumulate,
                             int block) {
    const int j = blockIdx.z;  // 0: modulus M1, 1: modulus M2
    const int64_t M = j ? M2 : M1, q = j ? q2 : q1;
    Acc *y = (j ? y2 : y1) + (int64_t)blockIdx.y * (j ? ldy2 : ldy1);
    const T *xb = x + (int64_t)blockIdx.y * ldx;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M + K;
         k += (int64_t)gridDim.x * blockDim.x) {
        Acc acc = 0;
        if (block) {  // strategy 2: x zero-padded, no wrap; y[M + c] = y[c] (K <= M)
            for (int64_t p = k < M ? k : k - M; p < N; p += M) {
                const int64_t rel = p - offset;
                if (rel >= 0 && rel < len) acc += (Acc)xb[rel];
            }
            if (accumulate) y[k] += acc; else y[k] = acc;
            continue;
        }
        int64_t p = k % N;
        for (int64_t i = 0; i < q; ++i) {
            int64_t rel = p - offset;
            if (rel >= 0 && rel < len) acc += (Acc)xb[rel];
            p += M;
            while (p >= N) p -= N;
        }
        if (accumulate) y[k] += acc; else y[k] = acc;
    }
}

constexpr int PM_COLS = 8 * 512;  // columns per CTA group of the packed kernel (fold_tma.cu TCOLS)

// ---------------------------------------------------------------------------
// finalize: counts -> values, + wrap + extension (partial-fold semantics)
// ---------------------------------------------------------------------------
// Cross-GPU combine fused into this epilogue (tm_fold_reduce):
// instead of storing its values the kernel ADDS them into n destination folds --
// peer-mapped buffers of the other ranks (red.global.add) or one NVLS multicast
// address (multimem.red.add: the switch adds into every bound GPU's copy).
constexpr int RED_MAX = 8;
struct RedDst {
    int n, multicast;
    int32_t *y1[RED_MAX], *y2[RED_MAX];
};
__device__ __forceinline__ void red_out(const RedDst &rd, int which, int64_t off, int32_t v) {
    for (int d = 0; d < rd.n; ++d) {
        int32_t *p = (which ? rd.y2[d] : rd.y1[d]) + off;
        if (rd.multicast)
            asm volatile("multimem.red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
        else
            asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    }
}

__global__ void fold_finalize(const int8_t *__restrict__ x, int64_t ldx, int64_t N, int64_t offset,
                              int64_t len, int64_t M1, int64_t M2, int64_t K, int64_t q2,
                              int64_t row0, int64_t rows, const int32_t *__restrict__ counts,
                              int32_t *__restrict__ y1, int64_t ldy1, int32_t *__restrict__ y2, int64_t ldy2,
                              int accumulate, int block, const RedDst rd) {
    pdl_trigger();
    pdl_wait();  // the counts of this fold
    const int64_t b = blockIdx.y;
    const int8_t *xb = x + b * ldx;
    const int32_t *c1 = counts + b * (M1 + M2), *c2 = c1 + M1;
    int32_t *o1 = y1 + b * ldy1, *o2 = y2 + b * ldy2;
    auto xat = [&](int64_t pos) -> int32_t {  // x at a global position, 0 outside the chunk
        int64_t rel = pos - offset;
        return (rel >= 0 && rel < len) ? (int32_t)xb[rel] : 0;
    };
    // base bin of M2 k < M2: elements = rows - [the row g* = (M1 - k) mod M2 is in the chunk]
    // (M1 - k lies in [-1, M1], so the reduction is one conditional add: no division)
    const int64_t s2 = q2 * M2 - N;
    auto base2 = [&](int64_t k) -> int32_t {
        int64_t gs = M1 - k;
        if (gs < 0) gs += M2;
        int32_t n = (int32_t)rows - ((gs >= row0 && gs < row0 + rows) ? 1 : 0);
        int32_t v = n - c2[k];
        int64_t j = k - (M2 - q2);               // the mod-N wrap: bin M2 - q + j gets x[j]
        if (!block && j >= 0 && j < q2) v += xat(j);
        return v;
    };
    // bin k < M2 also writes its extension bin M2 + k (k < K) from its own base value:
    // y2[M2 + c] = y2[c] - x[c] + x[c + s2] (strategy 2: y2[M2 + c] = y2[c]).
    // (launched with ~4 bins per thread: the unrolled iterations' loads are independent)
    const int kend = (int)(M1 + K), m1 = (int)M1, m2 = (int)M2, kk = (int)K;  // M1 + K >= M2
#pragma unroll 4
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kend; k += gridDim.x * blockDim.x) {
        const int c = k < m1 ? k : k - m1;       // M1 | N: y1[M1 + c] = y1[c]
        const int32_t v1 = (int32_t)rows - c1[c];
        int32_t v = 0, ve = 0;
        if (k < m2) {
            v = base2(k);
            if (k < kk) {
                int64_t e = k + s2;
                if (e >= N) e -= N;
                ve = block ? v : v - xat(k) + xat(e);
            }
        }
        if (rd.n) {  // fused cross-GPU combine: add into every destination fold
            red_out(rd, 0, b * ldy1 + k, v1);
            if (k < m2) {
                red_out(rd, 1, b * ldy2 + k, v);
                if (k < kk) red_out(rd, 1, b * ldy2 + m2 + k, ve);
            }
            continue;
        }
        if (accumulate) o1[k] += v1; else o1[k] = v1;
        if (k < m2) {
            if (accumulate) o2[k] += v; else o2[k] = v;
            if (k < kk) {
                if (accumulate) o2[m2 + k] += ve; else o2[m2 + k] = ve;
            }
        }
    }
}

// Work split for the persistent TMA kernel (one CTA per SM): the fewest row
// chunks per (pair, column group) whose item count spreads over the SMs with
// < 5% imbalance (items are equal-sized), rows per item in [128, TM_FOLD_RMAX]
// (the per-warp anti-diagonal arrays grow with the rows per item: a smaller
// bound leaves shared memory for more ring stages, TM_FOLD_NST).
#ifndef TM_FOLD_RMAX
#define TM_FOLD_RMAX 1024
#endif
void pick_rows_tma(const tm_plan_s *p, int64_t batch, int64_t rows, int64_t n_groups, int64_t *R_out,
                   int64_t *nrc_out) {
    const int64_t slots = p->num_sms;
    int64_t bestR = 0, bestN = 0;
    double best_eff = -1.0;
    for (int64_t n = (rows + TM_FOLD_RMAX - 1) / TM_FOLD_RMAX; n <= rows; ++n) {
        const int64_t R = ((rows + n - 1) / n + 15) / 16 * 16;
        const int64_t nrc = (rows + R - 1) / R;
        if (nrc != n && n > 1) continue;
        const int64_t items = batch * n_groups * nrc;
        const int64_t g = items < slots ? items : slots;
        const double eff = ((double)items / (double)g) / (double)((items + g - 1) / g) * ((double)g / slots);
        if (eff > best_eff + 1e-9) { best_eff = eff; bestR = R; bestN = nrc; }
        if (eff >= 0.95 || (R < 128 && bestN)) break;
    }
    *R_out = bestR;
    *nrc_out = bestN;
}

}  // namespace

int tm_fold_tma(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *ws, int64_t R, int64_t n_rc,
                cudaStream_t s, bool *used_counts, bool force_counts);

static int fold_impl(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                     void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *ws, cudaStream_t s,
                     const RedDst *rd);

int tm_fold_impl_ld(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                    void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *ws, cudaStream_t s) {
    return fold_impl(p, x, ldx, batch, offset, len, y1, ldy1, y2, ldy2, accumulate, ws, s, nullptr);
}

static int fold_impl(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                     void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *ws, cudaStream_t s,
                     const RedDst *rd) {
    if (batch == 0) return TM_OK;
    RedDst none{};
    const RedDst &R_ = rd ? *rd : none;
    const bool aligned = ((uintptr_t)x % 16 == 0) && (ldx % 16 == 0);
    const bool fast = p->fast_fold && aligned && (offset % p->M1 == 0) && (len % p->M1 == 0) &&
                      batch <= (int64_t(1) << 31) / 64;
    if (fast && len > 0) {
        int64_t R = 0, nrc = 0;
        const int64_t rows = len / p->M1, n_groups = (p->M1 + PM_COLS - 1) / PM_COLS;
        pick_rows_tma(p, batch, rows, n_groups, &R, &nrc);
        bool used_counts = false;
        int rc = tm_fold_tma(p, x, ldx, batch, offset, len, y1, ldy1, y2, ldy2, accumulate, ws, R, nrc, s,
                             &used_counts, rd != nullptr);
        if (rc != TM_EUNSUPPORTED) {
            if (rc != TM_OK || !used_counts) return rc;
            tm_ws_layout L = tm_ws(p, batch);
            // ~4 bins per thread when the grid stays several waves deep (many pairs),
            // one per thread otherwise (one pair: cfg5, 129 -> 513 CTAs)
            int64_t gx = (p->M2 + p->K + 1023) / 1024;
            if (gx * batch < 4 * (int64_t)p->num_sms) gx = (p->M2 + p->K + 255) / 256;
            { const cudaError_t e_ = launch_pdl(fold_finalize, dim3((unsigned)gx, (unsigned)batch), dim3(256), 0, s,
                (const int8_t *)x, ldx, p->N, offset, len, p->M1, p->M2, p->K, p->q2, offset / p->M1, rows,
                (const int32_t *)((char *)ws + L.fold_counts), (int32_t *)y1, ldy1, (int32_t *)y2, ldy2, accumulate,
                p->block, R_);
              if (e_ != cudaSuccess) return tm_cuda_status(e_, "tm_fold: fold_finalize"); }
            TM_CHECK_LAUNCH("tm_fold: fold_finalize");
            return TM_OK;
        }
    }
    if (rd) {
        tm_set_error("tm_fold_reduce: needs the packed +-1 fold (TM_BINARY, M1 | N, M1 %% 512 == 0, row-aligned "
                     "16-byte aligned chunks)");
        return TM_EUNSUPPORTED;
    }
    if (p->dtype == TM_F32 && ws && len > 0) {  // strip kernel + fixed-order finalize
        tm_ws_layout L = tm_ws(p, batch);
        int rc = tm_fold_f32(p, x, ldx, batch, offset, len, y1, ldy1, y2, ldy2, accumulate,
                             (char *)ws + L.fold_counts, s);
        if (rc != TM_EUNSUPPORTED) return rc;
    }
    if (batch > 65535) { tm_set_error("tm_fold: general kernel supports batch <= 65535"); return TM_EUNSUPPORTED; }
    int64_t gx = (p->M2 + p->K + 255) / 256;
    if (gx > 65535) gx = 65535;
    dim3 grid((unsigned)gx, (unsigned)batch, 2);
    if (p->dtype == TM_I8) {
        fold_general<int8_t, int32_t><<<grid, 256, 0, s>>>((const int8_t *)x, ldx, p->N, offset, len,
                                                           p->M1, p->M2, p->K, p->q1, p->q2,
                                                           (int32_t *)y1, ldy1, (int32_t *)y2, ldy2, accumulate,
                                                           p->block);
    } else {
        fold_general<float, float><<<grid, 256, 0, s>>>((const float *)x, ldx, p->N, offset, len,
                                                        p->M1, p->M2, p->K, p->q1, p->q2,
                                                        (float *)y1, ldy1, (float *)y2, ldy2, accumulate,
                                                        p->block);
    }
    TM_CHECK_LAUNCH("tm_fold: fold_general");
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) int tm_fold(tm_plan p, const void *x, int64_t ldx, int64_t batch, int64_t offset,
                       int64_t len, void *y1, void *y2, int accumulate, void *ws, void *stream) {
    if (!p) { tm_set_error("tm_fold: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_fold: batch < 0"); return TM_EINVAL; }
    if (offset < 0 || len < 0 || offset + len > p->N) {
        tm_set_error("tm_fold: chunk [%lld, %lld) outside [0, N=%lld)", (long long)offset,
                     (long long)(offset + len), (long long)p->N);
        return TM_EINVAL;
    }
    if (batch > 0 && (!x || !y1 || !y2 || ldx < len)) {
        tm_set_error("tm_fold: NULL pointer or ldx < len");
        return TM_EINVAL;
    }
    if (batch > 0 && (p->fast_fold || tm_fold_f32_ok(p)) && !ws) {
        tm_set_error("tm_fold: workspace required");
        return TM_EINVAL;
    }
    return tm_fold_impl(p, x, ldx, batch, offset, len, y1, y2, accumulate, ws, (cudaStream_t)stream);
}

extern "C" __attribute__((visibility("default"))) int tm_fold_reduce(tm_plan p, const void *x, int64_t ldx,
                                                                     int64_t batch, int64_t offset, int64_t len,
                                                                     int ndst, void *const *dst_y1,
                                                                     void *const *dst_y2, int multicast, void *ws,
                                                                     void *stream) {
    if (!p) { tm_set_error("tm_fold_reduce: NULL plan"); return TM_EINVAL; }
    if (batch < 0 || offset < 0 || len < 0 || offset + len > p->N) {
        tm_set_error("tm_fold_reduce: bad batch / chunk");
        return TM_EINVAL;
    }
    if (ndst < 1 || ndst > RED_MAX || (multicast && ndst != 1) || !dst_y1 || !dst_y2 || !ws || (batch > 0 && !x)) {
        tm_set_error("tm_fold_reduce: need 1 <= ndst <= %d destinations (1 with multicast), ws and x", RED_MAX);
        return TM_EINVAL;
    }
    if (p->dtype != TM_I8) { tm_set_error("tm_fold_reduce: TM_I8 plans only"); return TM_EUNSUPPORTED; }
    if (batch == 0 || len == 0) return TM_OK;
    RedDst rd{};
    rd.n = ndst;
    rd.multicast = multicast ? 1 : 0;
    for (int d = 0; d < ndst; ++d) {
        if (!dst_y1[d] || !dst_y2[d]) { tm_set_error("tm_fold_reduce: NULL destination"); return TM_EINVAL; }
        rd.y1[d] = (int32_t *)dst_y1[d];
        rd.y2[d] = (int32_t *)dst_y2[d];
    }
    return fold_impl(p, x, ldx, batch, offset, len, nullptr, p->len_y1, nullptr, p->len_y2, 0, ws,
                     (cudaStream_t)stream, &rd);
}
