/*
 * tm.h -- C ABI of the B200 hot path of arXiv 1509.04863 ("fast template
 * matching"), Algorithm 1 FTM().
 *
 * Problem: given a signal x in R^N and a template t in R^K,
 * find m = argmax_k (Tx)_k,  (Tx)_k = sum_{i<K} t_i x_{(k+i) mod N}.
 * The method folds x through the subsampled circulant Phi for two co-prime
 * moduli (Eq. 2, Alg. 1 step 3), correlates each fold with the template in
 * the low-dimensional space (steps 4-6), takes the two argmaxes (step 7) and
 * recovers the shift by the CRT (steps 8-9, Theorem 4).
 *
 * Conventions for every entry point
 *   - All array arguments are DEVICE pointers on the current CUDA device,
 *     owned by the caller (in practice torch tensors), unless the name ends
 *     in _host.  The library never frees or retains them.
 *   - `stream` is a cudaStream_t (0 = legacy default stream).  Every call only
 *     enqueues work on `stream` and returns; nothing synchronises the host.
 *   - Batches are row-major: pair b's signal starts at x + b*ldx elements.
 *   - Return value: TM_OK, or an error code.  Argument errors are detected
 *     synchronously before any launch and nothing is enqueued.  Asynchronous
 *     kernel faults surface as TM_ECUDA on a later call.  tm_last_error()
 *     returns a thread-local human-readable detail of the last failure.
 *   - A failed match is data, not an error: k = -1 (NO_MATCH, reading C9 of
 *     DESIGN.md) with the residues still reported.
 *   - Plans are immutable after creation; one plan may be used concurrently
 *     on several streams, each call with its own workspace and output
 *     buffers (the Python Pipeline / SingleSignal(depth=) rely on this: the
 *     tm_fold of step i+1 on one stream beside the tm_correlate_match of
 *     step i on another).
 *
 * Element types
 *   TM_I8 : x, t int8;  y1, y2 int32 (exact);  r1, r2 int64 (exact).
 *   TM_F32: x, t, y1, y2, r1, r2 float32.
 *   residues int32 [batch][2];  k int64 [batch].
 */
#ifndef TM_H
#define TM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tm_plan_s *tm_plan;

enum { TM_I8 = 0, TM_F32 = 1 };

enum {
    TM_OK = 0,
    TM_EINVAL = 1,        /* bad argument (see each call) */
    TM_EUNSUPPORTED = 2,  /* valid for the paper, not supported by this build */
    TM_ECUDA = 3,         /* CUDA error (launch or asynchronous fault) */
};

/* flags */
#define TM_BINARY 1u  /* caller asserts every x and t entry is -1 or +1 (int8
                         only): enables the packed +-1 fold kernel.  Passing
                         other values with this flag gives unspecified y. */
#define TM_CORR_NTT 2u  /* TM_I8 correlation engine: number-theoretic transform
                           (CUDA cores).  Default: the tensor-core engine when
                           the plan is eligible for it, else the NTT. */
#define TM_ALIAS_REPAIR 8u  /* steps 8-9 with the candidate sets reduced mod N
                               (reading C10 of DESIGN.md): when M1 | N and
                               N <= z < N + s2, k = z - N instead of NO_MATCH
                               (a true peak m < s2 that the mod-N wrap of Eq. 2
                               moved into bin m + M2 - s2).  Default: off, the
                               literal unreduced sets of P:104-105 (C9).
                               TM_EUNSUPPORTED unless M1 | N (the closed form;
                               the oracle's literal mod-N sets also cover
                               M1 not dividing N). */
#define TM_BLOCK 16u    /* strategy 2 of P:150-151: the Block sampling matrix
                           Phi = [Phi_M ... Phi_M] of Theorem 2 with
                           Eq. 3's Phi_M = I, on x zero-padded to a multiple of
                           M_j: y_j[k] = sum_{p < N, p = k mod M_j} x[p]
                           (no sample counted twice), and the correlation is
                           cyclic, (T^ y)_k = sum_i t_i y[(k+i) mod M_j].  The
                           y buffers keep their M_j + K entries; the tail is the
                           cyclic copy y[M_j + c] = y[c].  Exclusive with
                           TM_ALIAS_REPAIR (no wrap alias exists).  Default:
                           strategy 1 (D_{M+K}). */
#define TM_CORR_TC 4u   /* TM_I8 correlation engine: int8 tensor cores
                           (tcgen05.mma kind::i8, exact int32 accumulation of
                           4-bit limbs of y); TM_EUNSUPPORTED if the plan is not
                           eligible (|y| bound > 32767, K > 65536, shared
                           memory).  The two engines give identical results. */

#define TM_INPUTS_STABLE 32u  /* caller asserts that x and t are not being written
                                 when tm_run / tm_fold is enqueued: they were
                                 written by work that has completed (e.g. before a
                                 host synchronisation) and nothing writes them while
                                 the call runs.  Lets back-to-back tm_run calls on a
                                 stream overlap (programmatic dependent launch,
                                 PDL): the next launch streams x while the previous
                                 one finishes its tail, waiting for it
                                 (griddepcontrol.wait) only before its first global
                                 write.  Default (flag off): every thread of a
                                 PDL-launched fold kernel waits for the previous
                                 launch to complete before reading anything, so a
                                 kernel that produces x right before tm_run is safe. */
#define TM_KEEP_Y 64u   /* test hook: the fused tm_run kernel (TM_PATH_FUSED_TC)
                           keeps the folded rows y1, y2 it writes into the
                           workspace instead of dropping them from L2 without
                           write-back once correlated; tm_run_fold_rows locates
                           them.  Costs HBM write traffic; not for production. */

typedef struct {
    int64_t N;          /* signal length */
    int64_t K;          /* template length */
    int64_t M1, M2;     /* co-prime moduli, M2 = M1 + 1 (Alg. 1 step 2) */
    int64_t q1, q2;     /* ceil(N / Mj): terms per folded entry (Eq. 2) */
    int64_t s1, s2;     /* qj*Mj - N: samples counted twice by the mod-N wrap (reading C5) */
    int64_t len_y1;     /* M1 + K entries of y1 (strategy 1, D_{M+K}) */
    int64_t len_y2;     /* M2 + K entries of y2 */
    int64_t L1, L2;     /* transform lengths used for the correlation of y1 / y2 */
    int32_t n_primes;   /* TM_I8: NTT primes used (1 or 2) for exact correlation */
    int32_t dtype;      /* TM_I8 or TM_F32 */
    uint32_t flags;
    int32_t fast_fold;  /* 1 if the full-signal fold uses the packed +-1 kernel */
    int64_t tf_bytes;   /* bytes of one folded template (tm_fold_template output) */
    uint64_t seed;      /* seed of tm_generate */
    int32_t corr_engine; /* TM_I8: 1 = tensor-core correlation (TM_CORR_TC), 0 = NTT */
} tm_plan_info;

/*
 * tm_plan_create -- Alg. 1 step 2.
 *   N      signal length, 1 <= N < 2^62.
 *   K      template length, 1 <= K <= M1.
 *   M      first modulus; 0 selects the paper's rule M1 = K.  M2 = M1 + 1.
 *   seed   base seed of the synthetic generator tm_generate (Phi itself is
 *          deterministic, r_k = 1 iff k mod M = 0).
 *   dtype  TM_I8 or TM_F32.   flags  0 or TM_BINARY.
 * Errors: TM_EINVAL if N < 1, K < 1, M1 < K, M1*M2 <= N (the minimal valid
 * K is reported in tm_last_error), bad dtype/flags, out == NULL.
 * TM_ECUDA if the CUDA device cannot be initialised.
 * The plan holds only host scalars (plus one-time NTT root tables in static
 * device memory of the library).
 */
int tm_plan_create(tm_plan *out, int64_t N, int64_t K, int64_t M, uint64_t seed,
                   int dtype, uint32_t flags);

/* tm_plan_query -- fills *info.  TM_EINVAL on NULL arguments. */
int tm_plan_query(tm_plan plan, tm_plan_info *info);

/* Bytes of device workspace `ws` needed by tm_fold / tm_correlate / tm_run
 * for `batch` pairs (256-byte aligned).  0 on invalid arguments. */
size_t tm_workspace_bytes(tm_plan plan, int64_t batch);

void tm_plan_destroy(tm_plan plan);

/*
 * tm_generate -- the paper's synthetic workload (section 3.5
 * P:234-244): counter-based generator keyed by (seed, global pair index).
 *   pair0, batch   global pair indices [pair0, pair0+batch).
 *   noise          TM_I8: template bit-flip probability in [0,1];
 *                  TM_F32: template Gaussian noise sigma >= 0.
 *   offset, len    positions [offset, offset+len) of each signal to write to
 *                  x (so a rank can generate only its chunk).  x may be NULL.
 *   x [batch][ldx] signal chunk (ldx >= len).
 *   t [batch][K]   template (may be NULL); k0 [batch] planted shift (may be NULL).
 * int8 outputs are bit-identical to tmgen/ (host); fp32 outputs agree to
 * float rounding of the same formula.
 * Errors: TM_EINVAL on offset/len outside [0, N], ldx < len, batch < 0.
 */
int tm_generate(tm_plan plan, int64_t pair0, int64_t batch, double noise,
                int64_t offset, int64_t len, void *x, int64_t ldx,
                void *t, int64_t *k0, void *stream);

/*
 * tm_fold -- Eq. (2), Alg. 1 step 3 with D_{M+K}
 * (strategy 1) and the mod-N index convention:
 *     y_j[k] = sum_{i < ceil(N/Mj)} x[(k + i*Mj) mod N],  k < Mj + K, j = 1, 2,
 * restricted to the global positions p in [offset, offset+len) (partial fold;
 * offset = 0, len = N is the paper's fold).  x points at position `offset`
 * of pair 0.  The sum of partial folds over any partition of [0, N) is the
 * full fold (exactly for TM_I8) -- this is how a signal split over GPUs is
 * folded (sum the partials with an all-reduce).
 *   y1 [batch][M1+K], y2 [batch][M2+K]   int32 (TM_I8) or float32 (TM_F32).
 *   accumulate     0: overwrite y; 1: add into y.
 *   ws             workspace of tm_workspace_bytes(plan, batch) bytes.
 * Errors: TM_EINVAL on NULL pointers, batch < 0, ldx < len, range outside
 * [0, N].  x must be 16-byte aligned with ldx*elem a multiple of 16 for the
 * fast kernels; otherwise a slower general kernel is used.
 */
int tm_fold(tm_plan plan, const void *x, int64_t ldx, int64_t batch,
            int64_t offset, int64_t len, void *y1, void *y2, int accumulate,
            void *ws, void *stream);

/*
 * tm_fold_template -- Alg. 1 step 4: t_M = [t 0] zero-padded, and the
 * template half of step 5: the forward transform of the reversed padded
 * template (reading C3: correlation, not convolution), in the layout
 * tm_correlate consumes (TM_I8: NTT residues mod the plan's primes, bit-
 * reversed order; TM_F32: the zero-padded template).
 *   t  [batch][K];   tf  [batch] x tf_bytes (see tm_plan_query).
 */
int tm_fold_template(tm_plan plan, const void *t, int64_t batch, void *tf, void *stream);

/*
 * tm_correlate -- Alg. 1 steps 5-6 read as the correlation of
 * P:61 (reading C3):  r_j[k] = sum_{i<K} t_i y_j[k+i],  k < Mj.
 * Exact for TM_I8 (number-theoretic transform, exact CRT over n_primes);
 * float32 for TM_F32.
 *   y1, y2 from tm_fold; tf from tm_fold_template;
 *   r1 [batch][M1], r2 [batch][M2]   int64 (TM_I8) or float32 (TM_F32).
 */
int tm_correlate(tm_plan plan, const void *y1, const void *y2, const void *tf,
                 int64_t batch, void *r1, void *r2, void *ws, void *stream);

/*
 * tm_match -- Alg. 1 step 7: m~_j = the lowest index of max r_j over
 * [0, Mj) (readings C6, C7); steps 8-9 by Theorem 4:
 * z = the unique value in [0, M1*M2) with z = m~1 (mod M1), z = m~2 (mod M2);
 * k = z if z < N else -1 (NO_MATCH, reading C9).
 *   residues [batch][2] int32 (may be NULL);  k [batch] int64.
 */
int tm_match(tm_plan plan, const void *r1, const void *r2, int64_t batch,
             int32_t *residues, int64_t *k, void *stream);

/*
 * tm_run -- the whole hot path, == tm_fold(offset 0, len N) o tm_fold_template
 * o tm_correlate o tm_match, without materialising r (argmax fused into the
 * correlation epilogue).  x [batch][ldx], t [batch][K].
 * Its kernels use programmatic dependent launch: consecutive tm_run calls on
 * one stream may overlap on the device (the next call streams its inputs
 * while the previous one finishes), but every write of a call happens after
 * the previous call on the stream has completed, so results and the ordering
 * against other stream operations are as for plain stream order.  (The
 * inputs x, t of a call must not be written by the immediately preceding
 * tm_run / tm_fold kernel on the stream -- they never are by this library.)
 */
int tm_run(tm_plan plan, const void *x, int64_t ldx, const void *t, int64_t batch,
           int32_t *residues, int64_t *k, void *ws, void *stream);

/*
 * tm_correlate_match -- Alg. 1 steps 4-9 on already-folded vectors (the part
 * of tm_run after the fold): used after partial folds of one signal split over
 * several GPUs have been summed (all-reduce).  y1, y2 as produced by tm_fold
 * over the whole of [0, N); t [batch][K]; outputs as tm_match; ws as tm_run.
 */
int tm_correlate_match(tm_plan plan, const void *y1, const void *y2, const void *t, int64_t batch,
                       int32_t *residues, int64_t *k, void *ws, void *stream);

/*
 * tm_correlate_many -- steps 4-9 for ONE folded signal against many templates
 * (the GPS / CDMA acquisition shape of section 3.5: one received
 * code, one template per satellite / user): template i's
 * k[i] is what tm_correlate_match would return for the pair (x, t_i).  Fold
 * once (tm_fold), then call this.  y1 [len_y1], y2 [len_y2] of the one
 * signal; t [n_templates][K]; residues [n][2] (may be NULL), k [n].  ws of
 * tm_workspace_bytes(plan, n_templates).  The tensor-core engine reads y with
 * stride 0 (no copies); the other engines broadcast y into the workspace.
 */
int tm_correlate_many(tm_plan plan, const void *y1, const void *y2, const void *t, int64_t n_templates,
                      int32_t *residues, int64_t *k, void *ws, void *stream);

/*
 * tm_run_host -- tm_run on HOST buffers: copies x_host/t_host (pinned memory
 * recommended) to the caller's device staging buffers in chunks of
 * `chunk` pairs, overlapping the copy of chunk i+1 with the compute of chunk
 * i, and copies residues/k back to residues_host/k_host.  Enqueues on
 * `stream`; the results are valid after the stream synchronises.
 *   dev_x   device buffer of 2*chunk*ldx elements (double buffer)
 *   dev_t   device buffer of 2*chunk*K elements
 *   dev_out device buffer of batch*(8 + 2*4) bytes for k and residues
 *   ws      tm_workspace_bytes(plan, chunk) bytes
 */
int tm_run_host(tm_plan plan, const void *x_host, int64_t ldx, const void *t_host,
                int64_t batch, int64_t chunk, int32_t *residues_host, int64_t *k_host,
                void *dev_x, void *dev_t, void *dev_out, void *ws, void *stream);

/*
 * Instrumentation (not part of the method).
 * tm_launch_count: number of CUDA kernels this library has launched in the
 *   process (all threads), for launch accounting in benchmarks.
 * tm_profile_events: make subsequent tm_run calls on the calling thread record
 *   events[0..n-1] (cudaEvent_t, n <= 5) on their stream before the fold, after
 *   the fold (after the fused kernel on TM_PATH_FUSED_TC), after the template
 *   fold, after the correlation+argmax, after the CRT.  Each record costs ~2.7
 *   us of GPU time between kernels: measure on a subset of steps.
 *   events = NULL disables.  TM_EINVAL if n < 2.
 */
uint64_t tm_launch_count(void);
int tm_profile_events(void **events, int n);
/* tm_run_path: the kernel sequence tm_run(plan, batch) launches, -1 on bad
 * arguments.  TM_PATH_FUSED_TC: one persistent kernel (packed fold warps +
 * tensor-core correlation warps, argmax and CRT in its epilogue);
 * TM_PATH_STAGED_TC: fold kernel, then the tensor-core correlation kernel;
 * TM_PATH_STAGED: fold, then the NTT (or fp32) correlation and the CRT kernel;
 * TM_PATH_SMALL: small int8 pairs (N <= 16384, M2 + K <= 4096, K (M1 + M2) <=
 * 2^21, no engine flag): the whole path in one kernel, one CTA per pair. */
enum { TM_PATH_STAGED = 0, TM_PATH_STAGED_TC = 1, TM_PATH_FUSED_TC = 2, TM_PATH_SMALL = 3 };
int tm_run_path(tm_plan plan, int64_t batch);
/* tm_run_fold_rows: where tm_run(plan, batch, ws) writes the folded rows y1, y2
 * inside ws: out[0] = byte offset of y1 [batch][out[1]] (int32/fp32 entries,
 * row stride out[1] >= len_y1), out[2] = byte offset of y2 [batch][out[3]].
 * With TM_KEEP_Y these rows hold Eq. 2's y_j after the call on every path; without
 * it the fused path drops them (test instrumentation).  TM_EINVAL on bad args. */
int tm_run_fold_rows(tm_plan plan, int64_t batch, int64_t *out);
/* tm_probe_read_bw: enqueue one read-only HBM streaming pass over buf[0, bytes)
 * (cp.async.bulk ring, one CTA per SM; bytes rounded down to 32 KiB; buf 16-byte
 * aligned device memory) on stream, for timing a live read-only bandwidth
 * ceiling with events (bench.py).  Not part of the method. */
int tm_probe_read_bw(const void *buf, int64_t bytes, void *stream);
/* tm_probe_read_pattern: the same streaming pass with the fold's access pattern
 * over a row-major [rows][ldx] byte matrix: items of (column group of `width`
 * bytes, R rows), column groups fastest (order 0) or row chunks fastest (1),
 * 32 KB / width rows per stage, `grid` CTAs (0: one per SM).  Instrumentation. */
int tm_probe_read_pattern(const void *buf, int64_t ldx, int width, int64_t rows, int64_t R, int order, int grid,
                          void *stream);

/*
 * ---- One huge signal over several GPUs: the correlation split by outputs ----
 * SURVEY 8(e)(ii).  After the all-reduce of the partial folds every rank holds
 * the whole y1, y2; tm_correlate_match_part computes steps 5-7 (Eq. 4 and the
 * argmax) for part `part` of `nparts` contiguous ranges of output blocks only,
 * on the tiled tensor-core engine, and writes per pair and modulus the best
 * (r, k) of its range (max r, lowest k on ties, reading C7) as an
 * order-preserving int64 key: keys int64 [batch][2] (device), key =
 * (((r + 2^42) << 21) | (2^21 - 1 - k)) XOR 2^63 read as int64 (|r| < 2^41,
 * k < 2^21), INT64_MIN for an empty range.  The element-wise MAX of the keys over all parts (one
 * all-reduce MAX of 16 bytes per pair) is the key of the whole correlation;
 * tm_match_keys turns it into residues int32 [batch][2] (may be NULL) and k
 * int64 [batch] (steps 8-9, as tm_match).  ws: tm_workspace_bytes.
 * TM_EUNSUPPORTED if the plan is not eligible for the tiled engine (int8 data,
 * K <= 2^17, M2 < 2^21, |r| < 2^41).
 */
int tm_correlate_match_part(tm_plan plan, const void *y1, const void *y2, const void *t, int64_t batch, int part,
                            int nparts, int64_t *keys, void *ws, void *stream);
int tm_match_keys(tm_plan plan, const int64_t *keys, int64_t batch, int32_t *residues, int64_t *k, void *stream);

/*
 * tm_fold_reduce -- the cross-GPU combine of SURVEY.md 8(f) f4(iii), fused into
 * the fold's epilogue.  Eq. 2 is a sum over positions, so the fold of
 * one signal is the sum of the folds of its chunks; this call folds the chunk
 * [offset, offset + len) of each pair exactly as tm_fold does, but instead of
 * storing y1, y2 it ADDS them (int32, exact, order-free) into ndst destination
 * folds at once: dst_y1[d] int32 [batch][len_y1], dst_y2[d] int32 [batch][len_y2]
 * (host arrays of device pointers; peer-mapped memory of other GPUs, e.g. torch
 * symmetric-memory buffers, with red.global.add), or, with multicast != 0, ONE
 * NVLS multicast address each (ndst == 1; multimem.red.add: the switch adds into
 * the copy on every GPU bound to the multicast object).  The destinations must
 * hold zero (or other chunks' contributions) beforehand; the caller orders the
 * ranks around the call (barrier before: destinations zeroed; after: every
 * chunk added).  TM_I8 plans on the packed fold only (TM_BINARY, M1 | N, M1 a
 * multiple of 512, row-aligned 16-byte aligned chunks), 1 <= ndst <= 8;
 * otherwise TM_EINVAL / TM_EUNSUPPORTED before any launch.  ws: tm_workspace_bytes.
 */
int tm_fold_reduce(tm_plan plan, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len, int ndst,
                   void *const *dst_y1, void *const *dst_y2, int multicast, void *ws, void *stream);

/*
 * ---- More than two moduli: Theorem 4 with alpha moduli ----
 * "Any integer m is uniquely specified mod N by its remainders modulo alpha
 * relatively prime integers M_1 .. M_alpha as long as prod M_i >= N" (read as
 * > N, reading C8); Algorithm 1 is the case alpha = 2, M_2 = M_1 + 1.
 * More moduli allow M_j far below sqrt(N) (each M_j >= K still), at the
 * price of one fold + correlation per pair of moduli.
 *
 * tm_mplan_create -- moduli: host array of alpha (2 <= alpha <= 8) pairwise
 *   co-prime integers, K <= M_j < 2^31, prod M_j > N.  Each M_j is folded,
 *   correlated and argmax-ed exactly as in Algorithm 1 (strategy 1, Eq. 2,
 *   reading C5's mod-N wrap), by sub-plans of moduli (M, M + 1): when both M
 *   and M + 1 are in the set one sub-plan serves both, otherwise the M + 1
 *   residue is computed and discarded.  dtype / flags as tm_plan_create
 *   (TM_ALIAS_REPAIR is rejected).  Errors: TM_EINVAL for bad arguments (the
 *   reason in tm_last_error), TM_EUNSUPPORTED / TM_ECUDA from a sub-plan.
 * tm_mplan_workspace_bytes -- device workspace tm_mplan_run needs for batch.
 * tm_mplan_run -- x int8 [batch][ldx] (ldx >= N), t int8 [batch][K], device;
 *   residues int32 [batch][alpha] (may be NULL): m~_j of modulus moduli[j];
 *   k int64 [batch]: the CRT value z in [0, prod M_j) if z < N, else -1
 *   (reading C9).  Enqueued on stream; ws as sized above.
 * tm_crt_multi -- steps 8-9 alone (Garner's mixed-radix CRT, one thread per
 *   pair): residues int32 [batch][alpha] (device), moduli host [alpha] as
 *   above, k int64 [batch] (device).
 */
typedef struct tm_mplan_s *tm_mplan;
int tm_mplan_create(tm_mplan *out, int64_t N, int64_t K, const int64_t *moduli, int alpha, uint64_t seed,
                    int dtype, uint32_t flags);
size_t tm_mplan_workspace_bytes(tm_mplan plan, int64_t batch);
int tm_mplan_run(tm_mplan plan, const void *x, int64_t ldx, const void *t, int64_t batch, int32_t *residues,
                 int64_t *k, void *ws, void *stream);
int tm_crt_multi(const int32_t *residues, int64_t batch, int alpha, const int64_t *moduli, int64_t N, int64_t *k,
                 void *stream);
void tm_mplan_destroy(tm_mplan plan);

const char *tm_status_string(int status);
const char *tm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TM_H */
