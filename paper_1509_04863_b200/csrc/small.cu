// small.cu -- the whole of Algorithm 1 for SMALL pairs in one
// kernel, one CTA per pair: the latency path (cfg1, N = 4096,
// K = 256, is launch-latency bound; the staged kernels cost two launches and
// a TMEM allocation for ~10^5 multiply-adds).
//
// CTA b: x (N int8) and t (K int8) into shared memory; step 3 (Eq. 2)
// for both moduli, one thread per folded entry, literally
//     y_j[k] = sum_{i < q_j} x[(k + i M_j) mod N]   (strategy 1; reading C5's wrap)
// or the Block fold of Theorem 2 (TM_BLOCK: y_j[k] = sum_{p = k mod M_j} x[p],
// y_j[M_j + c] = y_j[c]); steps 4-6 as the direct correlation of P:61 (reading
// C3) r_j[k] = sum_{i<K} t_i y_j[k+i], exact in int32 (the plan admits the path
// only when K max|t| max|y| < 2^31); step 7 the lowest-index argmax (C6, C7);
// steps 8-9 tm_resolve (Theorem 4, C9, C10).
#include "tm_internal.cuh"

namespace {
constexpr int SM_T = 512;
constexpr int64_t SMALL_MAX_N = 16384;      // x staged in shared memory
constexpr int64_t SMALL_MAX_Y = 4096;       // M_j + K entries of each fold in shared memory
constexpr int64_t SMALL_MAX_WORK = 1 << 21; // K (M1 + M2) multiply-adds per pair

__global__ void __launch_bounds__(SM_T) small_pair_kernel(const int8_t *__restrict__ x, int64_t ldx,
                                                          const int8_t *__restrict__ t, int N, int K, int M1, int M2,
                                                          int q1, int q2, int block, uint32_t crt_inv,
                                                          int64_t crt_wrap, int32_t *residues, int64_t *k_out) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ int32_t sm[];
    int32_t *y1 = sm, *y2 = y1 + (M1 + K), *ts = y2 + (M2 + K);
    int8_t *xs = reinterpret_cast<int8_t *>(ts + K);
    __shared__ int64_t bv[2][SM_T / 32];
    __shared__ int bk[2][SM_T / 32];
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x;
    const int8_t *xb = x + b * ldx, *tb = t + b * (int64_t)K;
    for (int i = tid; i < N; i += SM_T) xs[i] = xb[i];
    for (int i = tid; i < K; i += SM_T) ts[i] = tb[i];
    __syncthreads();
    // step 3: both folds
    for (int j = 0; j < 2; ++j) {
        const int M = j ? M2 : M1, q = j ? q2 : q1;
        int32_t *y = j ? y2 : y1;
        for (int k = tid; k < M + K; k += SM_T) {
            int32_t acc = 0;
            if (block) {  // Theorem 2's Block Phi with Phi_M = I on x zero-padded (reading C21)
                for (int p = k < M ? k : k - M; p < N; p += M) acc += xs[p];
            } else {      // Eq. 2 with the mod-N convention
                int p = k % N;
                for (int i = 0; i < q; ++i) {
                    acc += xs[p];
                    p += M;
                    while (p >= N) p -= N;
                }
            }
            y[k] = acc;
        }
    }
    __syncthreads();
    // steps 4-7: direct correlation, one thread per output of either modulus (outputs
    // o < M1 are r1[o], the rest r2[o - M1]); four partial sums break the dependency
    // chain; then the lowest-index argmax per modulus
    int64_t best[2] = {INT64_MIN, INT64_MIN};
    int bi[2] = {0x7FFFFFFF, 0x7FFFFFFF};
    for (int o = tid; o < M1 + M2; o += SM_T) {  // o rises with the loop: > keeps the lowest index
        const int j = o < M1 ? 0 : 1;
        const int k = j ? o - M1 : o;
        const int32_t *yk = (j ? y2 : y1) + k;
        int32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int i = 0;
        for (; i + 4 <= K; i += 4) {
            a0 += ts[i] * yk[i];
            a1 += ts[i + 1] * yk[i + 1];
            a2 += ts[i + 2] * yk[i + 2];
            a3 += ts[i + 3] * yk[i + 3];
        }
        for (; i < K; ++i) a0 += ts[i] * yk[i];
        const int64_t r = (int64_t)((a0 + a1) + (a2 + a3));  // int32-exact (plan bound), any order
        if (r > best[j]) { best[j] = r; bi[j] = k; }
    }
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t ov = __shfl_xor_sync(0xffffffffu, best[j], o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi[j], o);
            if (ov > best[j] || (ov == best[j] && oi < bi[j])) { best[j] = ov; bi[j] = oi; }
        }
        if ((tid & 31) == 0) { bv[j][tid >> 5] = best[j]; bk[j][tid >> 5] = bi[j]; }
    }
    __syncthreads();
    if (tid == 0) {
        int64_t m[2];
        for (int j = 0; j < 2; ++j) {
            int64_t best = INT64_MIN;
            int bi = 0x7FFFFFFF;
            for (int w = 0; w < SM_T / 32; ++w)
                if (bv[j][w] > best || (bv[j][w] == best && bk[j][w] < bi)) { best = bv[j][w]; bi = bk[j][w]; }
            m[j] = bi;
        }
        if (residues) { residues[2 * b] = (int32_t)m[0]; residues[2 * b + 1] = (int32_t)m[1]; }
        k_out[b] = tm_resolve(m[0], m[1], M1, M2, crt_inv, N, crt_wrap);  // steps 8-9
    }
}
}  // namespace

// Plan-time eligibility: int8 data, everything of a pair fits one CTA's shared
// memory, the correlation is exact in int32, and the work is small enough that one
// CTA per pair beats the staged kernels' launches.
bool tm_small_ok(const tm_plan_s *p) {
    if (p->dtype != TM_I8) return false;
    if (p->N > SMALL_MAX_N || p->M2 + p->K > SMALL_MAX_Y) return false;
    if ((double)p->K * (double)(p->M1 + p->M2) > (double)SMALL_MAX_WORK) return false;
    const double xmax = (p->flags & TM_BINARY) ? 1.0 : 128.0;
    const double ybound = xmax * (double)(p->q1 > p->q2 ? p->q1 : p->q2);
    return (double)p->K * xmax * ybound < 2147483647.0;
}

int tm_small_run(const tm_plan_s *p, const void *x, int64_t ldx, const void *t, int64_t batch, int32_t *residues,
                 int64_t *k, cudaStream_t s) {
    if (batch > 0x7FFFFFFF) return TM_EUNSUPPORTED;
    const size_t smem = (size_t)(p->M1 + p->K + p->M2 + p->K + p->K) * 4 + (size_t)((p->N + 15) / 16 * 16);
    const cudaError_t e0 = tm_smem_attr((const void *)small_pair_kernel, 200 * 1024);
    if (e0 != cudaSuccess) return tm_cuda_status(e0, "small_pair_kernel: shared-memory attribute");
    const cudaError_t e = launch_pdl(small_pair_kernel, dim3((unsigned)batch), dim3(SM_T), smem, s,
                                     (const int8_t *)x, ldx, (const int8_t *)t, (int)p->N, (int)p->K, (int)p->M1,
                                     (int)p->M2, (int)p->q1, (int)p->q2, p->block, p->crt_inv, p->crt_wrap, residues,
                                     k);
    if (e != cudaSuccess) return tm_cuda_status(e, "small_pair_kernel");
    TM_CHECK_LAUNCH("small_pair_kernel");
    return TM_OK;
}
