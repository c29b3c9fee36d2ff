// run.cu -- tm_run (the whole of Algorithm 1 FTM(), on
// device buffers) and tm_run_host (the same on host buffers, with the
// host->device copies of chunk i+1 overlapped with the compute of chunk i).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "tm_internal.cuh"

namespace {
size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

struct RunWs {
    char *fold_ws;   // tm_fold workspace (its own layout at offset 0)
    void *y1, *y2;   // folded signal
    void *tf;        // folded template
    int32_t *resid;  // [batch][2]
    void *tiles;     // fp32 argmax partials
    void *gntt;      // grid-pass NTT scratch
    size_t total;
};

RunWs run_ws(const tm_plan_s *p, int64_t batch, void *ws) {
    tm_ws_layout F = tm_ws(p, batch);
    RunWs r{};
    char *base = (char *)ws;
    size_t off = F.total;
    r.fold_ws = base;
    r.resid = (int32_t *)(base + F.resid);
    r.tiles = base + F.f32_tiles;
    r.gntt = base + F.gntt;
    const size_t ey = p->dtype == TM_I8 ? 4 : 4;
    r.y1 = base + off; off += align256((size_t)batch * p->ldy1_run * ey);  // >= every path's stride
    r.y2 = base + off; off += align256((size_t)batch * p->ldy2_run * ey);
    r.tf = base + off; off += align256((size_t)batch * p->tf_bytes);
    r.total = off;
    return r;
}
}  // namespace

size_t tm_run_ws_bytes(const tm_plan_s *p, int64_t batch) { return run_ws(p, batch, nullptr).total; }

extern "C" __attribute__((visibility("default"))) int tm_run(tm_plan p, const void *x, int64_t ldx, const void *t, int64_t batch, int32_t *residues,
                      int64_t *k, void *ws, void *stream) {
    if (!p) { tm_set_error("tm_run: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_run: batch < 0"); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (!x || !t || !k || !ws || ldx < p->N) { tm_set_error("tm_run: NULL pointer or ldx < N"); return TM_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    RunWs W = run_ws(p, batch, ws);
    tm_prof_mark(0, s);
    if (p->small_ok) {  // small pairs: the whole path in one kernel, one CTA per pair
        const int rc = tm_small_run(p, x, ldx, t, batch, residues, k, s);
        for (int i = 1; i <= 4; ++i) tm_prof_mark(i, s);
        return rc;
    }
    if (p->use_tc) {
        if (tm_fused_tc_ok(p, batch)) {  // the whole path in one persistent kernel
            int rc = tm_fold_tc_fused(p, x, ldx, t, batch, W.y1, W.y2, residues, k, W.fold_ws, s);
            if (rc != TM_EUNSUPPORTED) {
                tm_prof_mark(1, s);  // one kernel: the later stage marks would only add gaps
                return rc;
            }
        }
        // step 3, then steps 4-9 in one tensor-core kernel (argmax + CRT in its epilogue)
        // (y rows at the 16-byte aligned strides ldy*_run: vector loads in the correlation)
        int rc = tm_fold_impl_ld(p, x, ldx, batch, 0, p->N, W.y1, p->ldy1_run, W.y2, p->ldy2_run, 0, W.fold_ws, s);
        if (rc) return rc;
        tm_prof_mark(1, s);
        tm_prof_mark(2, s);
        rc = tm_tc_any_ld(p, W.y1, W.y2, p->ldy1_run, p->ldy2_run, t, p->K, batch, nullptr, nullptr, nullptr,
                          residues, k, ws, s);
        tm_prof_mark(3, s);
        tm_prof_mark(4, s);
        return rc;
    }
    int rc = tm_fold_impl(p, x, ldx, batch, 0, p->N, W.y1, W.y2, 0, W.fold_ws, s);     // step 3
    if (rc) return rc;
    tm_prof_mark(1, s);
    if (p->fast_corr) {
        // steps 4-7 in one kernel per modulus: the template spectrum is computed in
        // registers next to the signal's (no tf round trip through HBM)
        tm_prof_mark(2, s);
        rc = tm_fast_correlate(p, W.y1, W.y2, t, nullptr, batch, nullptr, nullptr, W.resid, s);
        if (rc) return rc;
    } else if (p->big_corr) {
        tm_prof_mark(2, s);
        rc = tm_gntt_correlate(p, W.y1, W.y2, t, nullptr, batch, nullptr, nullptr, W.resid, W.gntt, s);
        if (rc) return rc;
    } else {
        rc = tm_fold_template(p, t, batch, W.tf, stream);                            // step 4 (+5 for t)
        if (rc) return rc;
        tm_prof_mark(2, s);
        if (p->dtype == TM_F32 && tm_fft_f32_ok(p)) {  // steps 5-9: the CRT in the FFT kernel's epilogue
            rc = tm_fft_f32_correlate(p, W.y1, W.y2, W.tf, batch, nullptr, nullptr, nullptr, W.gntt, s, residues, k);
            tm_prof_mark(3, s);
            tm_prof_mark(4, s);
            return rc;
        }
        rc = tm_correlate_impl(p, W.y1, W.y2, W.tf, batch, nullptr, nullptr, W.resid, W.tiles, W.gntt, s);  // 5-7
        if (rc) return rc;
    }
    tm_prof_mark(3, s);
    rc = tm_crt_impl(p, W.resid, batch, residues, k, s);                              // steps 8-9
    tm_prof_mark(4, s);
    return rc;
}

// Instrumentation: which kernel sequence tm_run(plan, batch) launches.
extern "C" __attribute__((visibility("default"))) int tm_run_path(tm_plan p, int64_t batch) {
    if (!p || batch <= 0) return -1;
    if (p->small_ok) return TM_PATH_SMALL;
    if (p->use_tc) {
        if (tm_fused_tc_ok(p, batch)) return TM_PATH_FUSED_TC;
        return TM_PATH_STAGED_TC;
    }
    return TM_PATH_STAGED;
}

extern "C" __attribute__((visibility("default"))) int tm_run_fold_rows(tm_plan p, int64_t batch, int64_t *out) {
    if (!p || batch < 1 || !out) { tm_set_error("tm_run_fold_rows: bad arguments"); return TM_EINVAL; }
    RunWs W = run_ws(p, batch, nullptr);
    out[0] = (int64_t)(uintptr_t)W.y1;
    out[2] = (int64_t)(uintptr_t)W.y2;
    // the fused kernel and the staged tensor-core path use the 32-entry aligned strides
    const bool aligned = p->use_tc;
    out[1] = aligned ? p->ldy1_run : p->len_y1;
    out[3] = aligned ? p->ldy2_run : p->len_y2;
    return TM_OK;
}

// the correlation of one huge signal split over ranks by output
// tiles; each rank's best (r, k) per modulus as order-preserving int64 keys
extern "C" __attribute__((visibility("default"))) int tm_correlate_match_part(tm_plan p, const void *y1,
                                                                              const void *y2, const void *t,
                                                                              int64_t batch, int part, int nparts,
                                                                              int64_t *keys, void *ws, void *stream) {
    if (!p) { tm_set_error("tm_correlate_match_part: NULL plan"); return TM_EINVAL; }
    if (batch < 0 || nparts < 1 || part < 0 || part >= nparts) {
        tm_set_error("tm_correlate_match_part: bad batch / part / nparts");
        return TM_EINVAL;
    }
    if (batch == 0) return TM_OK;
    if (!y1 || !y2 || !t || !keys || !ws) { tm_set_error("tm_correlate_match_part: NULL pointer"); return TM_EINVAL; }
    if (!p->tct_ok) {
        tm_set_error("tm_correlate_match_part: plan not eligible for the tiled tensor-core engine");
        return TM_EUNSUPPORTED;
    }
    return tm_tc_tiled_correlate(p, y1, y2, p->len_y1, p->len_y2, t, p->K, batch, nullptr, nullptr, nullptr, nullptr,
                                 nullptr, (char *)ws + tm_ws(p, batch).tiled, (cudaStream_t)stream, part, nparts,
                                 keys);
}

extern "C" __attribute__((visibility("default"))) int tm_match_keys(tm_plan p, const int64_t *keys, int64_t batch,
                                                                    int32_t *residues, int64_t *k, void *stream) {
    if (!p || batch < 0) { tm_set_error("tm_match_keys: bad arguments"); return TM_EINVAL; }
    if (batch > 0 && (!keys || !k)) { tm_set_error("tm_match_keys: NULL pointer"); return TM_EINVAL; }
    return tm_tc_match_keys(p, keys, batch, residues, k, (cudaStream_t)stream);
}

// steps 4-9 on already-folded vectors (e.g. after an all-reduce of partial folds)
extern "C" __attribute__((visibility("default"))) int tm_correlate_match(tm_plan p, const void *y1, const void *y2,
                                                                         const void *t, int64_t batch,
                                                                         int32_t *residues, int64_t *k, void *ws,
                                                                         void *stream) {
    if (!p) { tm_set_error("tm_correlate_match: NULL plan"); return TM_EINVAL; }
    if (batch < 0) { tm_set_error("tm_correlate_match: batch < 0"); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (!y1 || !y2 || !t || !k || !ws) { tm_set_error("tm_correlate_match: NULL pointer"); return TM_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    RunWs W = run_ws(p, batch, ws);
    int rc;
    if (p->use_tc) return tm_tc_any(p, y1, y2, t, p->K, batch, nullptr, nullptr, nullptr, residues, k, ws, s);
    if (p->fast_corr) {
        rc = tm_fast_correlate(p, y1, y2, t, nullptr, batch, nullptr, nullptr, W.resid, s);
    } else if (p->big_corr) {
        rc = tm_gntt_correlate(p, y1, y2, t, nullptr, batch, nullptr, nullptr, W.resid, W.gntt, s);
    } else {
        rc = tm_fold_template(p, t, batch, W.tf, stream);
        if (rc == TM_OK)
            rc = tm_correlate_impl(p, y1, y2, W.tf, batch, nullptr, nullptr, W.resid, W.tiles, W.gntt, s);
    }
    if (rc) return rc;
    return tm_crt_impl(p, W.resid, batch, residues, k, s);
}

extern "C" __attribute__((visibility("default"))) int tm_run_host(tm_plan p, const void *x_host, int64_t ldx, const void *t_host, int64_t batch,
                           int64_t chunk, int32_t *residues_host, int64_t *k_host, void *dev_x, void *dev_t,
                           void *dev_out, void *ws, void *stream) {
    if (!p) { tm_set_error("tm_run_host: NULL plan"); return TM_EINVAL; }
    if (batch < 0 || chunk < 1) { tm_set_error("tm_run_host: batch < 0 or chunk < 1"); return TM_EINVAL; }
    if (batch == 0) return TM_OK;
    if (!x_host || !t_host || !k_host || !dev_x || !dev_t || !dev_out || !ws || ldx < p->N) {
        tm_set_error("tm_run_host: NULL pointer or ldx < N");
        return TM_EINVAL;
    }
    const size_t ex = p->dtype == TM_I8 ? 1 : 4;
    cudaStream_t s = (cudaStream_t)stream;
    // the plan's copy stream and events, created on first use and kept until
    // tm_plan_destroy; the mutex serialises concurrent tm_run_host calls on one plan
    // while they enqueue (the records and waits of one call must not interleave)
    tm_plan_s *pm = const_cast<tm_plan_s *>(p);
    std::lock_guard<std::mutex> lk(pm->host_mu);
    cudaError_t e = cudaSuccess;
    if (!pm->host_stream) {
        e = cudaStreamCreateWithFlags(&pm->host_stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { pm->host_stream = nullptr; return tm_cuda_status(e, "tm_run_host: stream"); }
        for (int i = 0; i < 4; ++i) cudaEventCreateWithFlags(&pm->host_ev[i], cudaEventDisableTiming);
    }
    cudaStream_t sc = pm->host_stream;
    cudaEvent_t *copied = pm->host_ev, *freed = pm->host_ev + 2;
    // the copy stream must not overwrite a slot the caller's stream still reads from a
    // previous call: start after everything already queued on s
    cudaEventRecord(freed[0], s);
    cudaEventRecord(freed[1], s);
    int64_t *dk = (int64_t *)dev_out;
    int32_t *dres = (int32_t *)((char *)dev_out + ((size_t)batch * 8 + 255) / 256 * 256);
    int rc = TM_OK;
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks && rc == TM_OK; ++c) {
        const int slot = (int)(c & 1);
        const int64_t b0 = c * chunk, nb = (batch - b0) < chunk ? (batch - b0) : chunk;
        char *sx = (char *)dev_x + (size_t)slot * chunk * ldx * ex;
        char *st = (char *)dev_t + (size_t)slot * chunk * p->K * ex;
        cudaStreamWaitEvent(sc, freed[slot], 0);
        e = cudaMemcpyAsync(sx, (const char *)x_host + (size_t)b0 * ldx * ex, (size_t)nb * ldx * ex,
                            cudaMemcpyHostToDevice, sc);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(st, (const char *)t_host + (size_t)b0 * p->K * ex, (size_t)nb * p->K * ex,
                                cudaMemcpyHostToDevice, sc);
        if (e != cudaSuccess) { rc = tm_cuda_status(e, "tm_run_host: H2D"); break; }
        cudaEventRecord(copied[slot], sc);
        cudaStreamWaitEvent(s, copied[slot], 0);
        rc = tm_run(p, sx, ldx, st, nb, dres + 2 * b0, dk + b0, ws, stream);
        cudaEventRecord(freed[slot], s);
    }
    if (rc == TM_OK) {
        e = cudaMemcpyAsync(k_host, dk, (size_t)batch * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && residues_host)
            e = cudaMemcpyAsync(residues_host, dres, (size_t)batch * 8, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) rc = tm_cuda_status(e, "tm_run_host: D2H");
    }
    return rc;
}

// copy one folded signal into every row of a batch (the non-tensor-core engines
// of tm_correlate_many read y with a per-pair stride)
__global__ void broadcast_rows(const uint32_t *__restrict__ src, int64_t n, int64_t ld, int64_t rows,
                               uint32_t *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * rows; i += (int64_t)gridDim.x * blockDim.x)
        dst[(i / n) * ld + i % n] = src[i % n];
}

extern "C" __attribute__((visibility("default"))) int tm_correlate_many(tm_plan p, const void *y1, const void *y2,
                                                                        const void *t, int64_t n_templates,
                                                                        int32_t *residues, int64_t *k, void *ws,
                                                                        void *stream) {
    if (!p) { tm_set_error("tm_correlate_many: NULL plan"); return TM_EINVAL; }
    if (n_templates < 0) { tm_set_error("tm_correlate_many: n_templates < 0"); return TM_EINVAL; }
    if (n_templates == 0) return TM_OK;
    if (!y1 || !y2 || !t || !k || !ws) { tm_set_error("tm_correlate_many: NULL pointer"); return TM_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    if (p->use_tc)  // y read with stride 0: every template's CTAs stage the same folded signal
        return tm_tc_any_ld(p, y1, y2, 0, 0, t, p->K, n_templates, nullptr, nullptr, nullptr, residues, k, ws, s);
    RunWs W = run_ws(p, n_templates, ws);
    const unsigned g = (unsigned)std::min<int64_t>((n_templates * (p->len_y1 + p->len_y2) + 255) / 256, 65535 * 4);
    broadcast_rows<<<g, 256, 0, s>>>((const uint32_t *)y1, p->len_y1, p->len_y1, n_templates, (uint32_t *)W.y1);
    TM_CHECK_LAUNCH("tm_correlate_many: broadcast");
    broadcast_rows<<<g, 256, 0, s>>>((const uint32_t *)y2, p->len_y2, p->len_y2, n_templates, (uint32_t *)W.y2);
    TM_CHECK_LAUNCH("tm_correlate_many: broadcast");
    return tm_correlate_match(p, W.y1, W.y2, t, n_templates, residues, k, ws, stream);
}
