// tm_internal.cuh -- private declarations of libtm (the B200 hot path of
// arXiv 1509.04863, Algorithm 1).  Nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/tm.h"

#define TM_MAX_LOGL 18           // longest correlation transform: 2^18 (K <= 2^17)
#define TM_NTT_SMEM_MAX_LOGL 14  // transforms up to 2^14 run fully in shared memory

struct tm_plan_s {
    int64_t N, K, M1, M2, q1, q2, s1, s2, len_y1, len_y2;
    int64_t ldy1_run, ldy2_run;  // y row strides inside tm_run's workspace (multiples of 32 entries)
    int64_t L1, L2;
    int logL1, logL2;
    int64_t nload1, nload2;  // entries of y_j the correlation reads (cyclic y1: M1)
    int fast_corr;       // register-resident NTT kernels (corr_fast.cu) usable
    int big_corr;        // grid-pass NTT (gntt.cu) for transforms longer than 2^14
    int n_primes;
    int dtype;
    uint32_t flags;
    int fast_fold;       // packed +-1 kernel eligible for full-row chunks
    uint64_t seed;
    int device;
    int num_sms;
    int64_t tf_elems;    // uint2 (value, shoup) elements per prime per pair (I8) / floats (F32)
    std::mutex host_mu;         // tm_run_host: guards the copy stream / events below
    cudaStream_t host_stream;   // tm_run_host's host->device copy stream (created on first use)
    cudaEvent_t host_ev[4];     // copied[2], freed[2]
    int64_t tf_bytes;
    uint32_t crt_inv;    // M1^{-1} mod M2
    int block;           // TM_BLOCK: strategy 2 (Theorem 2), no wrap, cyclic extension
    int64_t crt_wrap;    // TM_ALIAS_REPAIR with M1 | N: s2 (reading C10), else 0
    // tensor-core correlation engine (corr_tc.cu)
    int use_tc;          // tm_run / tm_correlate use corr_tc_kernel
    int tc_ok;           // plan shape eligible for it
    int tc_NA[2], tc_NMC, tc_R, tc_NC, tc_JA, tc_CCH, tc_lmax;
    int tct_ok, tct_lmax;  // tiled tensor-core correlation (corr_tc_tiled.cu) eligible
    int small_ok;          // tm_run uses the one-kernel small-pair path (small.cu)
    uint32_t tc_ncols, tc_offB, tc_offTp, tc_offMisc, tc_smem;
};

// Alg. 1 steps 8-9 by Theorem 4:
//   z = m1 + M1 ((m2 - m1) M1^{-1} mod M2),  k = z if z < N;
// with the alias repair (reading C10: the candidate sets taken mod N),
// k = z - N if N <= z < N + wrap (wrap = s2 then, 0 otherwise); else NO_MATCH
// (k = -1, reading C9).  Residues are in range, so |m2 - m1| < M2 and
// d * inv < M2^2 <= 2^64.
__host__ __device__ __forceinline__ int64_t tm_resolve(int64_t m1, int64_t m2, int64_t M1, int64_t M2, uint32_t inv,
                                                      int64_t N, int64_t wrap) {
    int64_t d = m2 - m1;
    if (d < 0) d += M2;
    const int64_t u = (int64_t)(((uint64_t)d * inv) % (uint64_t)M2);
    const int64_t z = m1 + M1 * u;
    if (z < N) return z;
    if (z < N + wrap) return z - N;
    return -1;
}

// mbarrier.try_wait suspend-time hint (ns): a waiting thread sleeps until the
// phase completes (or this bound elapses) instead of re-issuing the test
#ifndef MBAR_SUSPEND_NS
#define MBAR_SUSPEND_NS 0
#endif

// ---- error plumbing (plan.cu) ----
void tm_set_error(const char *fmt, ...);
int tm_cuda_status(cudaError_t e, const char *what);
void tm_count_launch();
#define TM_CHECK_LAUNCH(what)                                                  \
    do {                                                                       \
        cudaError_t _e = cudaGetLastError();                                   \
        if (_e != cudaSuccess) return tm_cuda_status(_e, what);                \
        tm_count_launch();                                                     \
    } while (0)
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may be
// scheduled while its predecessor on the stream runs, once that predecessor has
// executed pdl_trigger(); pdl_wait() blocks until the predecessor has completed
// and its memory is visible (a no-op without a PDL predecessor).  Kernels call
// pdl_trigger() at entry and pdl_wait() before their first dependent global
// access.  TM_NO_PDL in the environment launches them normally (A/B).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool tm_pdl_enabled();
// makes `dev` current for a scope (per-device one-time setup: tables, constants)
struct TmDeviceGuard {
    int prev = -1;
    explicit TmDeviceGuard(int dev) {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~TmDeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize = bytes [, max shared carveout]) once
// per (function, device, bytes), thread-safe (plan.cu)
cudaError_t tm_smem_attr(const void *func, int bytes, bool max_carveout = false);
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args) {
    if (!tm_pdl_enabled()) {
        k<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// stage-boundary events of tm_run (tm_profile_events); NULL when disabled
void tm_prof_mark(int stage, cudaStream_t s);

// ---- NTT constants ----
// Two NTT-friendly primes below 2^30 (so that 4p < 2^32 and butterflies can keep
// residues lazily in [0, 2p) / [0, 4p)): p1 = 479*2^21+1 (transforms up to 2^21),
// p2 = 119*2^23+1; both have primitive root 3.  tests/test_abi.py re-derives them.
#define TM_P1 1004535809u
#define TM_P2 998244353u
#define TM_P1_PINV 1004535807u   // -p1^{-1} mod 2^32 (Montgomery)
#define TM_P2_PINV 998244351u    // -p2^{-1} mod 2^32
#define TM_P1_INV_MOD_P2 332747959ull
struct tm_ntt_tables {
    const uint32_t *tw[2][2];   // [prime][dir] values,  per-length compact tables
    const uint32_t *tws[2][2];  // Shoup companions floor(w * 2^32 / p)
    const uint2 *tw2[2][2];     // the same, interleaved (value, companion)
};
int tm_ntt_tables_get(int device, tm_ntt_tables *out);
extern const uint32_t TM_PRIMES[2];

// ---- workspace layout (plan.cu) ----
struct tm_ws_layout {
    size_t fold_counts;   // int32 [batch][M1 + M2] base-bin accumulators
    size_t fold_bytes;
    size_t resid;         // int32 [batch][2] residues (tm_run)
    size_t f32_tiles;     // fp32 per-tile argmax partials (tm_run, TM_F32)
    size_t gntt;          // grid-pass NTT scratch (big_corr plans)
    size_t counters;      // int32 work counters (tm_run overlap mode, one per chunk)
    size_t tiled;         // tiled tensor-core correlation: packed keys + partial sums
    size_t total;
};
tm_ws_layout tm_ws(const tm_plan_s *p, int64_t batch);
size_t tm_run_ws_bytes(const tm_plan_s *p, int64_t batch);  // run.cu

// ---- internal launchers ----
bool tm_fast_corr_ok(const tm_plan_s *p);
void tm_mont_linv(int logL, uint32_t p, uint32_t *c, uint32_t *cs);
bool tm_fused_tc_ok(const tm_plan_s *p, int64_t batch);
bool tm_small_ok(const tm_plan_s *p);   // small.cu: one CTA per pair, the latency path
int tm_small_run(const tm_plan_s *p, const void *x, int64_t ldx, const void *t, int64_t batch, int32_t *residues,
                 int64_t *k, cudaStream_t s);
int tm_fold_tc_fused(const tm_plan_s *p, const void *x, int64_t ldx, const void *t, int64_t batch, void *y1,
                     void *y2, int32_t *residues, int64_t *k, void *ws, cudaStream_t s);
size_t tm_gntt_scratch_bytes(const tm_plan_s *p, int64_t batch);
int tm_gntt_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *t, const void *tf,
                      int64_t batch, void *r1, void *r2, int32_t *resid, void *scratch, cudaStream_t s);
int tm_gntt_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s);
int tm_fast_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s);
int tm_fast_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *t, const void *tf,
                      int64_t batch, void *r1, void *r2, int32_t *resid, cudaStream_t s);
bool tm_fft_f32_ok(const tm_plan_s *p);
int tm_fft_f32_template(const tm_plan_s *p, const void *t, int64_t ldt, int64_t batch, void *tf, cudaStream_t s);
bool tm_fft_f32_long(const tm_plan_s *p);
size_t tm_fft_f32_scratch_bytes(const tm_plan_s *p, int64_t batch);
int tm_fft_f32_correlate(const tm_plan_s *p, const void *y1, const void *y2, const void *tf, int64_t batch,
                         void *r1, void *r2, int32_t *resid, void *scratch, cudaStream_t s,
                         int32_t *residues_out = nullptr, int64_t *k_out = nullptr);
bool tm_fold_f32_ok(const tm_plan_s *p);
size_t tm_fold_f32_ws_bytes(const tm_plan_s *p, int64_t batch);
int tm_fold_f32(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *parts, cudaStream_t s);
// tm_fold with explicit row strides of y1, y2 (>= len_y1, len_y2; the public
// tm_fold uses len_y*, tm_run's staged paths the 16-byte aligned ldy*_run)
int tm_plan_create_impl(tm_plan *out, int64_t N, int64_t K, int64_t M, uint64_t seed, int dtype, uint32_t flags,
                        int need_product);
int tm_fold_impl_ld(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                    void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *ws, cudaStream_t s);
inline int tm_fold_impl(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset,
                        int64_t len, void *y1, void *y2, int accumulate, void *ws, cudaStream_t s) {
    return tm_fold_impl_ld(p, x, ldx, batch, offset, len, y1, p->len_y1, y2, p->len_y2, accumulate, ws, s);
}
int tm_correlate_impl(const tm_plan_s *p, const void *y1, const void *y2, const void *tf,
                      int64_t batch, void *r1, void *r2, int32_t *resid, void *tile_scratch,
                      void *gntt_scratch, cudaStream_t s, void *tc_ws = nullptr);
void tm_tc_plan(tm_plan_s *p);
int tm_tc_correlate(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2, const void *t,
                    int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid, int32_t *residues_out,
                    int64_t *k, cudaStream_t s);
int tm_tc_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s);
void tm_tc_tiled_plan(tm_plan_s *p);
size_t tm_tc_tiled_ws_bytes(const tm_plan_s *p, int64_t batch);
int tm_tc_tiled_correlate(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2,
                          const void *t, int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid,
                          int32_t *residues_out, int64_t *k, void *ws, cudaStream_t s, int part = 0,
                          int nparts = 1, int64_t *keys_out = nullptr);
int tm_tc_match_keys(const tm_plan_s *p, const int64_t *keys, int64_t batch, int32_t *residues, int64_t *k,
                     cudaStream_t s);
// the tensor-core engine for a batch: one CTA per pair (corr_tc.cu) or tiled
// over CTAs (few pairs / long templates); ws = the whole tm_workspace_bytes area
int tm_tc_any(const tm_plan_s *p, const void *y1, const void *y2, const void *t, int64_t ldt, int64_t batch,
              void *r1, void *r2, int32_t *resid, int32_t *residues_out, int64_t *k, void *ws, cudaStream_t s);
int tm_tc_any_ld(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2, const void *t,
                 int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid, int32_t *residues_out, int64_t *k,
                 void *ws, cudaStream_t s);
int tm_crt_impl(const tm_plan_s *p, const int32_t *resid, int64_t batch, int32_t *residues_out,
                int64_t *k, cudaStream_t s);
