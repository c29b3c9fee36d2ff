// fold_f32.cu -- the fold of real-valued signals (Algorithm 1 step 3, PAPER.md
// Eq. 2) at HBM speed, deterministic fp32 accumulation.
//
// Same factorisation as the packed +-1 kernel: with K | N
// and the row view x[g][c] = x[g M1 + c], the M1 bin of (g, c) is c (a column
// sum) and the M2 = M1 + 1 bin is (c - g) mod M2 (an anti-diagonal).  A warp
// owns a strip of 128 columns (lane l: columns 4l .. 4l+3, one 16-byte load per
// row) and streams a chunk of R rows:
//   * column sums: 4 registers per lane, rows added in order;
//   * anti-diagonals: 4 registers per lane hold the diagonals d = 4l + e - g of
//     the current row; after each row the window moves one column to the right
//     (registers e -> e+1, lane l's register 3 -> lane l+1's register 0 by one
//     warp shuffle), lane 31's register 3 leaves the strip and is written to a
//     per-warp shared-memory list, and after the last row the 128 registers are.
// Every (strip, row chunk) thus produces R + 127 diagonal partial sums and 128
// column partial sums, written once to the workspace; fold_f32_finalize adds
// them per bin in a fixed order (chunks, then strips ascending), applies the
// mod-N wrap and the strategy-1 extension (as fold_finalize does for counts),
// and writes y1, y2.  Summation order never depends on scheduling, so results
// are bit-reproducible run to run.
#include "tm_internal.cuh"

namespace {

constexpr int FW = 8;          // warps per CTA (strips of 128 columns)
constexpr int FCOLS = FW * 128;
constexpr int RMAX = 1024;     // rows per chunk
constexpr int UR = 16;         // rows in flight per warp (cfg3 A/B: 4 / 8 / 16 / 24 / 32 -> 0.870 /
                               // 0.752 / 0.736 / 0.740 / 0.911 ms per step)

struct F32Args {
    const float *x;
    int64_t ldx;
    int64_t M1, M2, K, N, q2;
    int64_t rows, row0;        // rows of the chunk [offset, offset + len) and its first global row
    int64_t R, nrc;            // rows per item, row chunks
    int64_t g0m, Rm;           // row0 mod M2, R mod M2 (the finalize's diagonal index of a chunk)
    int block;                 // TM_BLOCK: no wrap, cyclic extension
    int x_early;               // TM_INPUTS_STABLE: x may be read before the previous launch completes
    int64_t n_strips, n_groups;
    float *parts;              // [batch][nrc][M1 + n_strips (R + 127)]
};

// floats per (pair, row chunk) of partial sums, a multiple of 4 (the column sums
// are stored as float4)
__host__ __device__ __forceinline__ int64_t part_stride_of(int64_t M1, int64_t n_strips, int64_t R) {
    return (M1 + n_strips * (R + 127) + 3) & ~int64_t(3);
}
__device__ __forceinline__ int64_t part_stride(const F32Args &a) { return part_stride_of(a.M1, a.n_strips, a.R); }

__global__ void __launch_bounds__(FW * 32) fold_f32_strips(F32Args a) {
    extern __shared__ float emit[];  // [FW][RMAX + 127]
    pdl_trigger();
    if (!a.x_early) pdl_wait();  // x may come from the launch right before this one
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = blockIdx.x;
    const int64_t rc = item % a.nrc;
    const int64_t grp = (item / a.nrc) % a.n_groups;
    const int64_t b = item / a.nrc / a.n_groups;
    const int64_t strip = grp * FW + warp;
    if (strip >= a.n_strips) return;
    const int64_t r0 = rc * a.R;
    const int nrow = (int)((a.rows - r0) < a.R ? (a.rows - r0) : a.R);
    const int64_t c0 = strip * 128 + 4 * lane;
    const float *xp = a.x + b * a.ldx + r0 * a.M1 + c0;
    float *em = emit + warp * (RMAX + 127);
    const int R = (int)a.R;
    float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
    for (int g0 = 0; g0 < nrow; g0 += UR) {
        float4 v[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u)
            v[u] = (g0 + u < nrow) ? __ldcs(reinterpret_cast<const float4 *>(xp + (int64_t)(g0 + u) * a.M1))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < UR; ++u) {
            const int g = g0 + u;
            if (g >= nrow) break;
            s1[0] += v[u].x; s1[1] += v[u].y; s1[2] += v[u].z; s1[3] += v[u].w;
            s2[0] += v[u].x; s2[1] += v[u].y; s2[2] += v[u].z; s2[3] += v[u].w;
            if (g == nrow - 1) break;  // the final window is written below
            // diagonal 127 - g (relative to the strip) leaves it: index (127 - g) + R - 1
            if (lane == 31) em[127 - g + R - 1] = s2[3];
            const float in = __shfl_up_sync(0xffffffffu, s2[3], 1);
            s2[3] = s2[2]; s2[2] = s2[1]; s2[1] = s2[0];
            s2[0] = lane ? in : 0.f;
        }
    }
    // after row nrow-1: register e of lane l holds diagonal 4l + e - (nrow - 1)
#pragma unroll
    for (int e = 0; e < 4; ++e) em[4 * lane + e - (nrow - 1) + R - 1] = s2[e];
    __syncwarp();
    float *pp = a.parts + (b * a.nrc + rc) * part_stride(a);
    pdl_wait();  // the previous launch on the stream may still read the partial sums
    // column partial sums
    *reinterpret_cast<float4 *>(pp + c0) = make_float4(s1[0], s1[1], s1[2], s1[3]);
    // diagonal partials: indices [R - nrow, R + 127) were written (shorter chunks leave a zero head)
    float *dp = pp + a.M1 + strip * (a.R + 127);
    for (int i = lane; i < R + 127; i += 32) dp[i] = (i >= R - nrow) ? em[i] : 0.f;
}

// bin sums, wrap and extension; x read only for the wrap/extension terms
// FS: strip slots per diagonal, >= (R - 1) / 128 + 2 (the most strips one diagonal spans)
template <int FS>
__global__ void fold_f32_finalize(F32Args a, int64_t offset, int64_t len, float *__restrict__ y1, int64_t ldy1,
                                  float *__restrict__ y2, int64_t ldy2, int accumulate) {
    pdl_trigger();
    pdl_wait();  // the strips of this fold
    const int64_t b = blockIdx.y;
    const float *__restrict__ xb = a.x + b * a.ldx;
    const float *__restrict__ pb = a.parts + b * a.nrc * part_stride(a);
    float *o1 = y1 + b * ldy1, *o2 = y2 + b * ldy2;
    auto xat = [&](int64_t pos) -> float {  // x at a global position, 0 outside the chunk
        const int64_t rel = pos - offset;
        return (rel >= 0 && rel < len) ? __ldg(xb + rel) : 0.f;
    };
    const int R = (int)a.R, M1 = (int)a.M1, M2 = (int)a.M2;
    const int smax = (int)a.n_strips - 1;
    const int64_t pst = part_stride(a);
    // the strip partials of diagonal u (strips ascending) into t[0 .. n): strips s
    // with 128 s - (R - 1) <= u <= 128 s + 127, partial index u - 128 s + R - 1, i.e.
    // address pp + u + R - 1 + s (R - 1).  FS covers the most strips one diagonal
    // spans (R <= RMAX), so all of them are loaded together and the thread waits one
    // memory latency per diagonal.
    auto dload = [&](const float *__restrict__ pp, int u, float (&t)[FS]) -> int {
        const int slo = u < 0 ? 0 : (u >> 7);
        const int shi = min((u + R - 1) >> 7, smax);
        const int n = (u >= -(R - 1) && u <= M1 - 1) ? shi - slo + 1 : 0;
        const float *__restrict__ q = pp + (u + R - 1 + slo * (R - 1));
#pragma unroll
        for (int i = 0; i < FS; ++i) t[i] = i < n ? __ldg(q + i * (R - 1)) : 0.f;
        return n;
    };
    // sum of the anti-diagonal partials of bin k < M2: chunks in order, within a
    // chunk the diagonals u = (k + G0) mod M2, u - M2, ... (u in [-(R - 1), M1 - 1],
    // G0 = the chunk's first global row), strips ascending -- a fixed order
    auto base2 = [&](int k) -> float {
        float acc = 0.f;
        int g = (int)a.g0m;  // G0 mod M2
        for (int64_t rc = 0; rc < a.nrc; ++rc) {
            const float *__restrict__ pp = pb + rc * pst + M1;
            int u = k + g;
            if (u >= M2) u -= M2;
            // R <= rows < M2 (M1 M2 > N, Alg. 1 step 2): at most two diagonals, u and
            // (only for u >= M2 - R + 1) u - M2, loaded together
            float t1[FS], t0[FS];
            const int n1 = dload(pp, u, t1);
            const bool two = u - M2 >= -(R - 1);
            const int n0 = two ? dload(pp, u - M2, t0) : 0;
#pragma unroll
            for (int i = 0; i < FS; ++i)
                if (i < n1) acc += t1[i];
            if (two) {
#pragma unroll
                for (int i = 0; i < FS; ++i)
                    if (i < n0) acc += t0[i];
            }
            g += (int)a.Rm;
            if (g >= M2) g -= M2;
        }
        const int64_t j = k - (a.M2 - a.q2);  // the mod-N wrap: bin M2 - q + j gets x[j]
        if (!a.block && j >= 0 && j < a.q2) acc += xat(j);
        return acc;
    };
    // bin k < M2 also writes its strategy-1 extension bin M2 + k (k < K):
    // y2[M2 + c] = y2[c] - x[c] + x[c + s2] (strategy 2: y2[M2 + c] = y2[c])
    const int64_t s2 = a.q2 * a.M2 - a.N;
    const int64_t kend = a.M2 > a.M1 + a.K ? a.M2 : a.M1 + a.K;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < kend; k += (int64_t)gridDim.x * blockDim.x) {
        const bool has1 = k < a.M1 + a.K, has2 = k < a.M2;
        float v1 = 0.f;
        if (has1) {
            const int64_t c = k < a.M1 ? k : k - a.M1;   // M1 | N: y1[M1 + c] = y1[c]
            for (int64_t rc = 0; rc < a.nrc; ++rc) v1 += __ldg(pb + rc * pst + c);
        }
        float v = 0.f, ve = 0.f;
        if (has2) {
            v = base2((int)k);
            if (k < a.K) {
                int64_t e = k + s2;
                if (e >= a.N) e -= a.N;
                ve = a.block ? v : v - xat(k) + xat(e);
            }
        }
        if (has1) {
            if (accumulate) o1[k] += v1; else o1[k] = v1;
        }
        if (has2) {
            if (accumulate) o2[k] += v; else o2[k] = v;
            if (k < a.K) {
                if (accumulate) o2[a.M2 + k] += ve; else o2[a.M2 + k] = ve;
            }
        }
    }
}

void geometry(const tm_plan_s *p, int64_t rows, int64_t *R, int64_t *nrc) {
    *nrc = (rows + RMAX - 1) / RMAX;
    if (*nrc < 1) *nrc = 1;
    *R = (rows + *nrc - 1) / *nrc;
    if (*R < 1) *R = 1;
}

}  // namespace

bool tm_fold_f32_ok(const tm_plan_s *p) {
    return p->dtype == TM_F32 && p->N % p->M1 == 0 && p->M1 % 128 == 0 && p->M1 + 1 == p->M2 &&
           p->M2 + p->K < ((int64_t)1 << 30);  // int32 bin and partial indices in the finalize
}

size_t tm_fold_f32_ws_bytes(const tm_plan_s *p, int64_t batch) {
    if (!tm_fold_f32_ok(p)) return 0;
    int64_t R, nrc;
    geometry(p, p->N / p->M1, &R, &nrc);
    return (size_t)batch * nrc * part_stride_of(p->M1, p->M1 / 128, R) * 4;
}

// TM_EUNSUPPORTED (nothing enqueued) when the chunk or alignment does not qualify.
int tm_fold_f32(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *parts, cudaStream_t s) {
    if (!tm_fold_f32_ok(p) || !parts) return TM_EUNSUPPORTED;
    if (((uintptr_t)x % 16) || (ldx % 4) || (offset % p->M1) || (len % p->M1) || len == 0) return TM_EUNSUPPORTED;
    F32Args a{};
    a.x = (const float *)x; a.ldx = ldx;
    a.M1 = p->M1; a.M2 = p->M2; a.K = p->K; a.N = p->N; a.q2 = p->q2;
    a.rows = len / p->M1; a.row0 = offset / p->M1;
    a.block = p->block;
    a.x_early = (p->flags & TM_INPUTS_STABLE) ? 1 : 0;
    geometry(p, a.rows, &a.R, &a.nrc);
    if (a.R >= a.M2) return TM_EUNSUPPORTED;  // the finalize's two-diagonal bound (M1 M2 > N implies R < M2)
    a.g0m = a.row0 % a.M2;
    a.Rm = a.R % a.M2;
    a.n_strips = p->M1 / 128;
    a.n_groups = (a.n_strips + FW - 1) / FW;
    a.parts = (float *)parts;
    const int64_t items = batch * a.n_groups * a.nrc;
    if (items > 0x7FFFFFFF || batch > 65535) return TM_EUNSUPPORTED;
    const size_t smem = (size_t)FW * (RMAX + 127) * 4;
    {
        const cudaError_t e = tm_smem_attr((const void *)fold_f32_strips, (int)smem);
        if (e != cudaSuccess) return tm_cuda_status(e, "fold_f32_strips: shared-memory attribute");
    }
    {
        const cudaError_t e = launch_pdl(fold_f32_strips, dim3((unsigned)items), dim3(FW * 32), smem, s, a);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_fold: fold_f32_strips");
    }
    TM_CHECK_LAUNCH("tm_fold: fold_f32_strips");
    // 4 bins per thread when that still fills the GPU several times over (the
    // per-thread setup is about as long as one bin's work)
    const int64_t kend = p->M2 > p->M1 + p->K ? p->M2 : p->M1 + p->K;
    int64_t gx = (kend + 255) / 256;
    if (gx * batch >= 4 * 8 * (int64_t)p->num_sms) gx = (kend + 1023) / 1024;
    if (gx > 65535) gx = 65535;
    {
        const int need = (int)((a.R - 1) / 128 + 2);
        static_assert((RMAX - 1) / 128 + 2 <= 9, "strip slots");
        auto fin = need <= 3 ? fold_f32_finalize<3> : need <= 5 ? fold_f32_finalize<5> : fold_f32_finalize<9>;
        const cudaError_t e = launch_pdl(fin, dim3((unsigned)gx, (unsigned)batch), dim3(256), 0, s, a, offset, len,
                                         (float *)y1, ldy1, (float *)y2, ldy2, accumulate);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_fold: fold_f32_finalize");
    }
    TM_CHECK_LAUNCH("tm_fold: fold_f32_finalize");
    return TM_OK;
}
