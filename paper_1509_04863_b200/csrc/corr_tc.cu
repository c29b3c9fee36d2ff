// corr_tc.cu -- exact correlation + argmax + CRT (Algorithm 1 steps 4-9,
// PAPER.md P:98-106, correlation read as P:61, reading C3) on the 5th-generation
// tensor cores: tcgen05.mma kind::i8 (int8 x int8 -> int32 in TMEM).
//
// The correlation r_j[k] = sum_{i<K} t[i] y_j[k+i] (k < M_j) of one pair is a
// Toeplitz matrix-vector product; it is recast as a sum of small GEMMs by
// blocking both indices by P = 128:
//
//   k = P a + (P-1-b'),   i = P c + u - (P-1-b')      (b', u in [0,P))
//   r_j[P a + P-1-b'] = sum_c sum_u  A_c[b'][u] * B_c[u][a]
//   A_c[b'][u] = tp(P c + u - P + 1 + b')       (tp = t zero-extended)
//   B_c[u][a]  = y_j[P (a + c) + u]
//
// so D[b'][a] accumulates NC = floor((K+P-2)/P)+1 MMAs of shape M=128 (b'),
// K = 128 (u) over the output blocks a -- no epilogue reduction: D IS r.
// Both operands live in shared memory in the canonical no-swizzle K-major
// layout (8-row x 16-byte core matrices), and every A_c / B_c is a descriptor
// start-address offset:
//   A: S[J][s][e] = tp(16 J + s + e - 127)  (16 byte-shifted copies of the
//      template, s = b' mod 16), J = 8c + h + b'/16  ->  LBO = 256, SBO = 128,
//      +2048 B per c.  The Toeplitz row shift costs 16x the template (64 KB at
//      K = 4096), not 128x.
//   B: one MMA serves both moduli: B row rho = 2 s + j holds block s of y_j
//      (or of one 4-bit limb of it), as 8 chunks [h][rho][16 B] =
//      y_j[P s + 16 h + e].  Shifting all rows by c blocks (= 2c rows, +32c
//      bytes) shifts both streams at once, so MMA column n = 2 a + j
//      accumulates block a of r_j.  SBO = 128, LBO = 16 * rows.  A (4 KB per
//      MMA) is read once for both moduli, which keeps the shared-memory-bound
//      MMA at (4096 + 32 N) / 128 cycles (tools/mma_bench.cu).  Limbs run as
//      successive passes over a one-limb B buffer (small shared memory, so a
//      CTA of this kernel fits next to a fold CTA on the same SM).
// int8 operands are exact; y is split into 4-bit limbs when |y| > 127
// (y = sum_l 16^l v_l, top limb signed), chosen per pair from the data; the
// plan guarantees |y| <= 32767 (<= 3 limbs) and K*128*128 < 2^31 per limb.
#include <cstdlib>

#include <algorithm>

#include "tc_core.cuh"

namespace {
using namespace tc;

__global__ void __launch_bounds__(NTHR, 2) corr_tc_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    pdl_trigger();
    pdl_wait();  // y (and t) come from the preceding launches
    const int tid = threadIdx.x, warp = tid >> 5;
    uint64_t *mdone = reinterpret_cast<uint64_t *>(sm + a.offMisc);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(sm + a.offMisc + 8);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(a.ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mdone)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tslot;
    uint32_t mph = 0;
    if (a.ldy[0] == 0 && a.ldy[1] == 0) {
        // one folded signal against many templates (tm_correlate_many): persistent
        // over templates, y staged into B once per CTA (when it needs one limb)
        int y_pre = 0;
        for (int64_t b = blockIdx.x; b < a.nbatch; b += gridDim.x)
            tc_pair<CtaSync>(a, sm, b, tid, warp & 3, tbase, mph, &y_pre);
    } else {
        tc_pair<CtaSync>(a, sm, blockIdx.x, tid, warp & 3, tbase, mph);
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(a.ncols));
}

uint32_t align_up(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }

}  // namespace

static long long *g_tc_dbg = nullptr;
// instrumentation: per-CTA clock64 stamps of the tensor-core kernel's phases into
// buf ([batch][8]: start, template staged, y staged, A built, MMAs done, end, smid);
// NULL = off.  Not part of the method.
extern "C" __attribute__((visibility("default"))) void tm_debug_tc_timestamps(void *buf) {
    g_tc_dbg = (long long *)buf;
}
long long *tm_tc_dbg_buffer() { return g_tc_dbg; }

// Plan-time eligibility and geometry (stored in the plan; see tm_internal.cuh).
void tm_tc_plan(tm_plan_s *p) {
    p->tc_ok = 0;
    if (p->dtype != TM_I8) return;
    const double xmax = (p->flags & TM_BINARY) ? 1.0 : 128.0;
    const double ybound = xmax * (double)(p->q1 > p->q2 ? p->q1 : p->q2);
    const int lmax = ybound <= 127 ? 1 : (ybound <= 2047 ? 2 : (ybound <= 32767 ? 3 : 0));
    if (!lmax) return;
    if (p->K > 65536) return;  // per-limb |r| <= K * 128 * 128 < 2^31
    const int NC = (int)((p->K + P - 2) / P) + 1;
    int NA[2];
    for (int j = 0; j < 2; ++j) {
        const int64_t M = j ? p->M2 : p->M1;
        int64_t na = M / P;
        if (M - na * P > MAXLEFT) ++na;
        if (na < 1) na = 1;
        if (na > 256) return;
        NA[j] = (int)na;
    }
    const int NMC = ((NA[0] > NA[1] ? NA[0] : NA[1]) + 15) & ~15;
    const uint32_t cols = 2u * lmax * NMC;  // D columns
    if (cols > 512) return;
    uint32_t ncols = 32;
    while (ncols < cols) ncols *= 2;
    const int R = NMC + NC - 1;
    const int JA = 8 * (NC - 1) + 15;            // 16-byte chunks of the whole padded template
    const int CCH = NC > 17 ? (NC + 1) / 2 : NC;  // A operand built in chunks of CCH template blocks
    uint32_t off = 256u * (8 * (CCH - 1) + 15);  // A (one chunk)
    p->tc_offB = off;
    off += 256u * R;            // B (one limb): 8 chunk columns x 2 R rows x 16 B
    p->tc_offTp = off;
    off += align_up(16 * JA + 48, 16);
    p->tc_offMisc = off;
    off += MISC_BYTES;
    p->tc_smem = align_up(off, 128);
    if (p->tc_smem > 227 * 1024) return;
    p->tc_NA[0] = NA[0]; p->tc_NA[1] = NA[1];
    p->tc_NMC = NMC; p->tc_R = R;
    p->tc_NC = NC;
    p->tc_JA = JA;
    p->tc_CCH = CCH;
    p->tc_lmax = lmax;
    p->tc_ncols = ncols;
    p->tc_ok = 1;
}

void tm_tc_fill_args(const tm_plan_s *p, const void *y1, const void *y2, const void *t, int64_t ldt, void *r1,
                     void *r2, int32_t *resid, int32_t *residues_out, int64_t *k, tc::TcArgs &a) {
    a = tc::TcArgs{};
    a.t = (const int8_t *)t; a.ldt = ldt; a.K = p->K;
    a.y[0] = (const int32_t *)y1; a.y[1] = (const int32_t *)y2;
    a.ldy[0] = p->len_y1; a.ldy[1] = p->len_y2;
    a.len[0] = p->len_y1; a.len[1] = p->len_y2;
    a.M[0] = p->M1; a.M[1] = p->M2;
    a.NA[0] = p->tc_NA[0]; a.NA[1] = p->tc_NA[1];
    a.NMC = p->tc_NMC; a.R = p->tc_R;
    a.NC = p->tc_NC; a.JA = p->tc_JA; a.CCH = p->tc_CCH; a.LMAX = p->tc_lmax; a.ncols = p->tc_ncols;
    a.offB = p->tc_offB; a.offTp = p->tc_offTp; a.offMisc = p->tc_offMisc;
    a.r[0] = (int64_t *)r1; a.r[1] = (int64_t *)r2;
    a.resid = resid; a.residues_out = residues_out; a.k_out = k;
    a.N = p->N; a.M1 = p->M1; a.M2 = p->M2; a.crt_inv = p->crt_inv; a.crt_wrap = p->crt_wrap;
}

// r1/r2 (may be NULL), resid (may be NULL), k (NULL: no CRT).  t is int8 [batch][ldt].
int tm_tc_correlate(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2, const void *t,
                    int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid, int32_t *residues_out,
                    int64_t *k, cudaStream_t s) {
    if (!p->tc_ok) return TM_EUNSUPPORTED;
    if (batch == 0) return TM_OK;
    if (batch > 0x7FFFFFFF) { tm_set_error("tm_correlate: batch too large"); return TM_EUNSUPPORTED; }
    TcArgs a{};
    tm_tc_fill_args(p, y1, y2, t, ldt, r1, r2, resid, residues_out, k, a);
    a.ldy[0] = ldy1; a.ldy[1] = ldy2;  // 0: one folded signal shared by every template
    a.dbg = g_tc_dbg;
    {  // per device, once (same maximal carveout as the fold kernel: no reconfiguration between them)
        const cudaError_t e = tm_smem_attr((const void *)corr_tc_kernel, 227 * 1024, true);
        if (e != cudaSuccess) return tm_cuda_status(e, "corr_tc_kernel: shared-memory attribute");
    }
    a.nbatch = batch;
    const bool shared_y = ldy1 == 0 && ldy2 == 0;
    const int64_t grid = shared_y ? std::min<int64_t>(batch, 2 * (int64_t)p->num_sms) : batch;
    size_t smem = p->tc_smem;
    if (shared_y && p->tc_lmax > 1) {
        // one folded signal, many templates: a B buffer per limb, staged once per CTA
        // (tp and the misc area move up behind them), while two CTAs still fit per SM
        const uint32_t bs = (uint32_t)(256 * p->tc_R + 127) / 128 * 128;
        const size_t extra = (size_t)(p->tc_lmax - 1) * bs;
        if (smem + extra <= 113 * 1024) {
            a.bstride = bs;
            a.offTp += (uint32_t)extra;
            a.offMisc += (uint32_t)extra;
            smem += extra;
        }
    }
    {
        const cudaError_t e = launch_pdl(corr_tc_kernel, dim3((unsigned)grid), dim3(NTHR), smem, s, a);
        if (e != cudaSuccess) return tm_cuda_status(e, "corr_tc_kernel");
    }
    TM_CHECK_LAUNCH("corr_tc_kernel");
    return TM_OK;
}

// Staged path of the tensor-core engine: the "folded template" is the template
// itself (the Toeplitz operand is built in shared memory by tm_tc_correlate),
// stored [batch][tf_bytes] with 16-byte rows.
__global__ void tc_template_copy(const int8_t *__restrict__ t, int64_t K, int64_t ld, int8_t *__restrict__ tf) {
    const int64_t b = blockIdx.x;
    for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) tf[b * ld + i] = i < K ? t[b * K + i] : 0;
}

int tm_tc_template(const tm_plan_s *p, const void *t, int64_t batch, void *tf, cudaStream_t s) {
    if (batch > 0x7FFFFFFF) { tm_set_error("tm_fold_template: batch too large"); return TM_EUNSUPPORTED; }
    tc_template_copy<<<(unsigned)batch, 256, 0, s>>>((const int8_t *)t, p->K, p->tf_bytes, (int8_t *)tf);
    TM_CHECK_LAUNCH("tc_template_copy");
    return TM_OK;
}

int tm_tc_any(const tm_plan_s *p, const void *y1, const void *y2, const void *t, int64_t ldt, int64_t batch,
              void *r1, void *r2, int32_t *resid, int32_t *residues_out, int64_t *k, void *ws, cudaStream_t s) {
    return tm_tc_any_ld(p, y1, y2, p->len_y1, p->len_y2, t, ldt, batch, r1, r2, resid, residues_out, k, ws, s);
}

int tm_tc_any_ld(const tm_plan_s *p, const void *y1, const void *y2, int64_t ldy1, int64_t ldy2, const void *t,
                 int64_t ldt, int64_t batch, void *r1, void *r2, int32_t *resid, int32_t *residues_out, int64_t *k,
                 void *ws, cudaStream_t s) {
    const char *env = getenv("TM_TC_TILED");  // tests / A-B: "0" never, "1" whenever eligible
    const bool force = env && env[0] == '1', never = env && env[0] == '0';
    // one CTA per pair when it fits, except for long templates on fewer pairs than
    // SMs (measured, 64 pairs, late round 2: K = 8192 tiled 45 us vs one-CTA 59 us
    // (0.2197 vs 0.2240 ms per step); K = 4096 44 vs 37 us); the tiled kernel also
    // takes the plans the one-CTA kernel cannot (cfg5: K = 65536)
    const bool tiled_wins = batch < p->num_sms && p->K >= 8192;
    if (p->tct_ok && ws && !never && (force || !p->tc_ok || tiled_wins))
        return tm_tc_tiled_correlate(p, y1, y2, ldy1, ldy2, t, ldt, batch, r1, r2, resid, residues_out, k,
                                     (char *)ws + tm_ws(p, batch).tiled, s);
    return tm_tc_correlate(p, y1, y2, ldy1, ldy2, t, ldt, batch, r1, r2, resid, residues_out, k, s);
}
