// plan.cu -- plan creation (Alg. 1 step 2),
// status strings, thread-local error detail and the workspace layout.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tm_internal.cuh"

#include <atomic>
#include <mutex>
#include <new>
#include <map>
#include <set>
#include <tuple>

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};
static thread_local void **g_prof_ev = nullptr;
static thread_local int g_prof_n = 0;

void tm_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" __attribute__((visibility("default"))) uint64_t tm_launch_count(void) {
    return (uint64_t)g_launches.load(std::memory_order_relaxed);
}

extern "C" __attribute__((visibility("default"))) int tm_profile_events(void **events, int n) {
    if (events && n < 2) { tm_set_error("tm_profile_events: need >= 2 events"); return TM_EINVAL; }
    g_prof_ev = events;
    g_prof_n = events ? n : 0;
    return TM_OK;
}

void tm_prof_mark(int stage, cudaStream_t s) {
    if (g_prof_ev && stage < g_prof_n && g_prof_ev[stage]) cudaEventRecord((cudaEvent_t)g_prof_ev[stage], s);
}

void tm_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int tm_cuda_status(cudaError_t e, const char *what) {
    tm_set_error("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    return TM_ECUDA;
}

extern "C" __attribute__((visibility("default"))) const char *tm_last_error(void) { return g_err; }

extern "C" __attribute__((visibility("default"))) const char *tm_status_string(int s) {
    switch (s) {
        case TM_OK: return "TM_OK";
        case TM_EINVAL: return "TM_EINVAL";
        case TM_EUNSUPPORTED: return "TM_EUNSUPPORTED";
        case TM_ECUDA: return "TM_ECUDA";
        default: return "TM_UNKNOWN";
    }
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int ilog2_ceil(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}

// M1^{-1} mod M2 by the extended Euclidean algorithm (Theorem 4's CRT needs
// gcd(M1, M2) = 1, which holds for M2 = M1 + 1).
static uint32_t inv_mod(int64_t a, int64_t m) {
    int64_t r0 = m, r1 = a % m, s0 = 0, s1 = 1;
    while (r1 != 0) {
        int64_t qq = r0 / r1, t;
        t = r0 - qq * r1; r0 = r1; r1 = t;
        t = s0 - qq * s1; s0 = s1; s1 = t;
    }
    int64_t v = s0 % m;
    if (v < 0) v += m;
    return (uint32_t)v;
}

// need_product = 0: a sub-plan of a multi-modulus plan (tm_mplan_create), whose
// own pair of moduli need not cover N (Theorem 4 is applied to all alpha moduli)
int tm_plan_create_impl(tm_plan *out, int64_t N, int64_t K, int64_t M, uint64_t seed, int dtype, uint32_t flags,
                        int need_product) {
    if (!out) { tm_set_error("tm_plan_create: out is NULL"); return TM_EINVAL; }
    *out = nullptr;
    if (N < 1 || N >= (int64_t(1) << 62)) { tm_set_error("tm_plan_create: N=%lld out of range", (long long)N); return TM_EINVAL; }
    if (K < 1) { tm_set_error("tm_plan_create: K=%lld < 1", (long long)K); return TM_EINVAL; }
    if (dtype != TM_I8 && dtype != TM_F32) { tm_set_error("tm_plan_create: bad dtype %d", dtype); return TM_EINVAL; }
    if ((flags & TM_BLOCK) && (flags & TM_ALIAS_REPAIR)) { tm_set_error("tm_plan_create: TM_BLOCK and TM_ALIAS_REPAIR are exclusive"); return TM_EINVAL; }
    if (flags & ~(TM_BINARY | TM_CORR_NTT | TM_CORR_TC | TM_ALIAS_REPAIR | TM_BLOCK | TM_INPUTS_STABLE | TM_KEEP_Y)) { tm_set_error("tm_plan_create: unknown flags 0x%x", flags); return TM_EINVAL; }
    if ((flags & TM_CORR_NTT) && (flags & TM_CORR_TC)) { tm_set_error("tm_plan_create: TM_CORR_NTT and TM_CORR_TC are exclusive"); return TM_EINVAL; }
    if ((flags & (TM_CORR_NTT | TM_CORR_TC)) && dtype != TM_I8) { tm_set_error("tm_plan_create: TM_CORR_* needs TM_I8"); return TM_EINVAL; }
    if ((flags & TM_BINARY) && dtype != TM_I8) { tm_set_error("tm_plan_create: TM_BINARY needs TM_I8"); return TM_EINVAL; }
    int64_t M1 = M ? M : K, M2 = M1 + 1;
    if ((flags & TM_ALIAS_REPAIR) && N % (M1 ? M1 : 1) != 0) {
        tm_set_error("tm_plan_create: TM_ALIAS_REPAIR is implemented for M1 | N only (reading C10's closed form)");
        return TM_EUNSUPPORTED;
    }
    if (M1 < K) { tm_set_error("tm_plan_create: M1=%lld < K=%lld (Alg. 1 step 2 needs M1 >= K)", (long long)M1, (long long)K); return TM_EINVAL; }
    if (need_product && (__int128)M1 * (__int128)M2 <= (__int128)N) {
        int64_t kmin = 1;
        while ((__int128)kmin * (kmin + 1) <= (__int128)N) kmin *= 2;
        int64_t lo = kmin / 2;
        while (lo + 1 < kmin) { int64_t mid = (lo + kmin) / 2; if ((__int128)mid * (mid + 1) > N) kmin = mid; else lo = mid; }
        tm_set_error("tm_plan_create: M1*M2 = %lld*%lld <= N = %lld (Alg. 1 step 2); the smallest valid M1 is %lld",
                     (long long)M1, (long long)M2, (long long)N, (long long)kmin);
        return TM_EINVAL;
    }
    // y1 is M1-periodic when M1 | N (y1[M1 + c] = y1[c]): then a cyclic transform of
    // length exactly M1 suffices if M1 is a power of two; otherwise zero-pad to
    // L >= M + K - 1 so that no needed term wraps.
    const bool cyc1 = (N % M1 == 0) && ((M1 & (M1 - 1)) == 0);
    int64_t L1 = cyc1 ? M1 : int64_t(1) << ilog2_ceil(M1 + K - 1);
    int64_t L2 = int64_t(1) << ilog2_ceil(M2 + K - 1);
    // the NTT engine's root tables stop at 2^TM_MAX_LOGL; longer correlations
    // (K > 2^17) run on the tiled tensor-core engine (int8) or the direct fp32 kernel
    const bool ntt_len_ok = ilog2_ceil(M2 + K - 1) <= TM_MAX_LOGL;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return tm_cuda_status(e, "tm_plan_create: cudaGetDevice");
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return tm_cuda_status(e, "tm_plan_create: cudaDeviceGetAttribute");

    tm_plan_s *p = new (std::nothrow) tm_plan_s();  // value-initialised: every scalar 0
    if (!p) { tm_set_error("tm_plan_create: out of host memory"); return TM_EINVAL; }
    p->N = N; p->K = K; p->M1 = M1; p->M2 = M2;
    p->q1 = ceil_div(N, M1); p->q2 = ceil_div(N, M2);
    p->s1 = p->q1 * M1 - N; p->s2 = p->q2 * M2 - N;
    p->len_y1 = M1 + K; p->len_y2 = M2 + K;
    p->ldy1_run = (p->len_y1 + 31) / 32 * 32; p->ldy2_run = (p->len_y2 + 31) / 32 * 32;
    p->L1 = L1; p->L2 = L2;
    p->logL1 = ilog2_ceil(L1); p->logL2 = ilog2_ceil(L2);
    p->nload1 = cyc1 ? M1 : M1 + K - 1;
    p->nload2 = M2 + K - 1;
    p->dtype = dtype; p->flags = flags; p->seed = seed;
    p->device = dev; p->num_sms = sms;
    p->crt_inv = inv_mod(M1, M2);
    // reading C10's repair applies when M1 | N (then S_M1 needs no reduction mod N)
    p->block = (flags & TM_BLOCK) ? 1 : 0;
    p->crt_wrap = ((flags & TM_ALIAS_REPAIR) && N % M1 == 0) ? p->s2 : 0;
    // fast packed +-1 fold: rows of M1 int8 columns, 512-column warp strips
    p->fast_fold = (dtype == TM_I8) && (flags & TM_BINARY) && (N % M1 == 0) && (M1 % 512 == 0) &&
                   (M1 <= (int64_t(1) << 30));
    if (dtype == TM_I8) {
        // exactness bound on |r| (reading C16): |r| <= sum|t| * max|y|
        double tmax = (flags & TM_BINARY) ? 1.0 : 128.0;
        double bound = (double)K * tmax * (double)(p->q1 > p->q2 ? p->q1 : p->q2) * tmax;
        p->n_primes = (bound < (double)(TM_PRIMES[0] / 2) - 1.0) ? 1 : 2;
        p->fast_corr = ntt_len_ok && tm_fast_corr_ok(p);
        p->big_corr = ntt_len_ok && !p->fast_corr && p->logL2 > 14;
        if (p->big_corr) {   // u32 natural bit-reversed spectra at L2 (first L1 serve y1)
            p->tf_elems = L2;
            p->tf_bytes = L2 * p->n_primes * 4;
        } else if (p->fast_corr) {  // u32 Montgomery spectra in the fast kernel's register order
            p->tf_elems = L1 + L2;
            p->tf_bytes = (L1 + L2) * p->n_primes * 4;
        } else {             // uint2 (value, Shoup companion), natural bit-reversed order
            int64_t per_prime = L1 + (L2 != L1 ? L2 : 0);
            p->tf_elems = per_prime;
            p->tf_bytes = per_prime * p->n_primes * 8;
        }
        tm_ntt_tables t;
        int rc = tm_ntt_tables_get(dev, &t);
        if (rc != TM_OK) { delete p; return rc; }
        // correlation engine: tensor cores when eligible (TM_CORR=ntt in the
        // environment forces the NTT for A/B measurements of the default)
        tm_tc_plan(p);
        tm_tc_tiled_plan(p);
        static const char *env = getenv("TM_CORR");
        const bool env_ntt = env && strcmp(env, "ntt") == 0;
        if (flags & TM_CORR_TC) {
            if (!p->tc_ok && !p->tct_ok) {
                delete p;
                tm_set_error("tm_plan_create: TM_CORR_TC: plan not eligible for the tensor-core engine");
                return TM_EUNSUPPORTED;
            }
            p->use_tc = 1;
        } else {
            p->use_tc = (p->tc_ok || p->tct_ok) && !(flags & TM_CORR_NTT) && !env_ntt;
        }
        if (!ntt_len_ok && !p->use_tc) {
            delete p;
            tm_set_error("tm_plan_create: correlation length 2^%d exceeds the NTT engine's 2^%d and the plan is not "
                         "eligible for the tiled tensor-core engine (int8 data, |y| <= 524287, M2 < 2^21)",
                         ilog2_ceil(M2 + K - 1), TM_MAX_LOGL);
            return TM_EUNSUPPORTED;
        }
        {   // the latency path for small pairs (not when an engine was requested explicitly)
            static const char *env_small = getenv("TM_SMALL");  // A/B: "0" disables
            p->small_ok = tm_small_ok(p) && !(flags & (TM_CORR_NTT | TM_CORR_TC)) &&
                          !(env_small && env_small[0] == '0');
        }
        if (p->use_tc) {  // the folded template is the int8 template itself, 16-byte rows
            p->tf_bytes = (K + 15) / 16 * 16;
            p->tf_elems = p->tf_bytes;
        }
    } else {
        p->n_primes = 0;
        if (tm_fft_f32_ok(p)) {  // complex spectrum of the reversed template (fft_f32.cu)
            p->tf_elems = p->L2;
            p->tf_bytes = p->L2 * 8;
        } else {                 // the template itself (direct correlation)
            p->tf_elems = K;
            p->tf_bytes = K * 4;
        }
    }
    *out = p;
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) int tm_plan_create(tm_plan *out, int64_t N, int64_t K, int64_t M, uint64_t seed,
                              int dtype, uint32_t flags) {
    return tm_plan_create_impl(out, N, K, M, seed, dtype, flags, 1);
}

extern "C" __attribute__((visibility("default"))) int tm_plan_query(tm_plan plan, tm_plan_info *info) {
    if (!plan || !info) { tm_set_error("tm_plan_query: NULL argument"); return TM_EINVAL; }
    info->N = plan->N; info->K = plan->K; info->M1 = plan->M1; info->M2 = plan->M2;
    info->q1 = plan->q1; info->q2 = plan->q2; info->s1 = plan->s1; info->s2 = plan->s2;
    info->len_y1 = plan->len_y1; info->len_y2 = plan->len_y2;
    info->L1 = plan->L1; info->L2 = plan->L2;
    info->n_primes = plan->n_primes; info->dtype = plan->dtype; info->flags = plan->flags;
    info->fast_fold = plan->fast_fold; info->tf_bytes = plan->tf_bytes; info->seed = plan->seed;
    info->corr_engine = plan->use_tc;
    return TM_OK;
}

extern "C" __attribute__((visibility("default"))) void tm_plan_destroy(tm_plan plan) {
    if (!plan) return;
    if (plan->host_stream) {
        cudaStreamDestroy(plan->host_stream);
        for (int i = 0; i < 4; ++i) cudaEventDestroy(plan->host_ev[i]);
    }
    delete plan;
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// cudaFuncSetAttribute acts on the current device: remember (function, device)
// pairs already set, under a mutex (plans may be used from several threads and
// on several devices of one process)
cudaError_t tm_smem_attr(const void *func, int bytes, bool max_carveout) {
    // the attribute is a per-(function, device) maximum: only ever raised (setting a
    // smaller value for one launch would break a later, larger launch)
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> set_to;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(func, dev);
    const auto it = set_to.find(key);
    if (it != set_to.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && max_carveout)
        e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess) set_to[key] = bytes;
    return e;
}

bool tm_pdl_enabled() {
    static const bool on = getenv("TM_NO_PDL") == nullptr;
    return on;
}

tm_ws_layout tm_ws(const tm_plan_s *p, int64_t batch) {
    tm_ws_layout w{};
    size_t off = 0;
    w.fold_counts = off;
    w.fold_bytes = align256((size_t)batch * (size_t)(p->M1 + p->M2) * 4);
    const size_t f32 = align256(tm_fold_f32_ws_bytes(p, batch));  // fp32 fold partial sums
    if (f32 > w.fold_bytes) w.fold_bytes = f32;
    off += w.fold_bytes;
    w.resid = off;
    off += align256((size_t)batch * 2 * 4);
    w.f32_tiles = off;
    if (p->dtype == TM_F32) off += align256((size_t)batch * 2 * ((p->M2 + 1023) / 1024) * 8);
    w.gntt = off;
    if (p->big_corr) off += align256(tm_gntt_scratch_bytes(p, batch));
    off += align256(tm_fft_f32_scratch_bytes(p, batch));  // fp32 four-step FFT segments + keys
    w.counters = off;
    off += 256;
    w.tiled = off;
    off += align256(tm_tc_tiled_ws_bytes(p, batch));
    w.total = off;
    return w;
}

extern "C" __attribute__((visibility("default"))) size_t tm_workspace_bytes(tm_plan plan, int64_t batch) {
    if (!plan || batch < 0) return 0;
    return tm_run_ws_bytes(plan, batch);  // superset of tm_fold's and tm_correlate's needs
}
