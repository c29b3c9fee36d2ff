// fold_tma.cu -- the packed +-1 fold (Algorithm 1 step 3, Eq. 2,
// P:117-120) as a persistent, warp-specialised kernel fed by bulk-async (TMA)
// copies through a shared-memory ring.
//
// Arithmetic is the one documented in fold.cu (fold_pm1): rows of M1 columns,
// M1 bin = column, M2 bin = (column - row) mod M2 (anti-diagonal), counts of
// negatives two at a time in byte lanes (b & 0x02), class accumulators by row
// mod 4 with one funnel-shift combine per 16-row tile, systolic lane -> lane+1
// hand-off of finished 16-bin blocks.
//
// What changes here is the memory side:
//  * one CTA per SM loops over work items (pair, 4096-column group, row range);
//  * warp 8 (one elected lane) streams 8-row stages of the item into a 4-stage
//    ring with cp.async.bulk + mbarrier transaction counts, running ahead across
//    item boundaries, so HBM reads never wait for the consumers' arithmetic or
//    for the per-item flush;
//  * warps 0-7 read their 16x16-byte tiles with LDS.128 and release each stage
//    as soon as it is in registers;
//  * when an item is a whole pair (M1 <= 4096, full fold) the consumers write
//    the finished y1/y2 directly (counts -> values, the mod-N wrap and the
//    strategy-1 extension), so no workspace, memset or second kernel is needed.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ntt_core.cuh"
#include "tc_core.cuh"

namespace {

constexpr int TW = 8;                 // consumer warps, one 512-column strip each
constexpr int TCOLS = TW * 512;       // columns per CTA group
#ifndef TM_SROWS
#define TM_SROWS 8
#endif
constexpr int SROWS = TM_SROWS;       // rows per ring stage (8, or 4 with twice the stages)
constexpr int GPS = SROWS / 4;        // 4-row groups per stage
static_assert(SROWS == 8 || SROWS == 4 || SROWS == 16, "SROWS");
constexpr int STAGE_BYTES = SROWS * TCOLS;

struct TmaArgs {
    const int8_t *x;
    int64_t ldx;
    int64_t N, M1, M2, K, q2;
    int64_t rows;        // rows in the chunk
    int64_t row0;        // global row of the chunk's first row
    int64_t R;           // rows per item
    int64_t n_rc, n_groups, n_items;
    int contig;          // split items as one contiguous range of (pair, group, row) per CTA
    int64_t n_segs;      // contig: segments (pair, column group) of `rows` rows each
    int owner;           // items are whole pairs of a full fold: write y directly
    int accumulate;
    int acc_words;       // y2 accumulator words reserved in shared memory
    int priv_stride;     // words per warp-private anti-diagonal array (512 + 16 ceil(R/16))
    int32_t *counts;     // non-owner: [batch][M1 + M2]
    int32_t *y1, *y2;    // owner outputs
    int block;            // TM_BLOCK: no wrap term, cyclic extension
    int xs_bytes;        // bytes reserved for the epilogue's x[0 .. K + q) stage
    int x_early;         // PDL launch may read x (and t) before the previous grid completes
                         // (plan flag TM_INPUTS_STABLE); 0: every thread waits at entry
    // tensor-core fused mode: 8 warps correlate pair i (tc_core.cuh) while the fold streams pair i+1
    tc::TcArgs tca;
    uint32_t tc_off;     // shared-memory offset of the tensor-core group's region
    int64_t ldy1, ldy2;  // owner outputs: row strides of y1, y2 (>= M + K)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(MBAR_SUSPEND_NS)
            : "memory");
    } while (!done);
}
// Programmatic dependent launch (fused kernel, consecutive tm_run calls on a
// stream): every CTA lets the next launch be scheduled at once (it can only take
// an SM this grid has left), and each warp role waits for the previous grid
// (griddepcontrol.wait: completed, memory visible) only before its first global
// write -- so the next launch streams x while this one finishes its tail.

// x is streamed exactly once: its L2 lines are marked evict-first so that the
// folded vectors (written, then read back by the correlation) stay in L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_ef(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                            uint64_t pol) {
#ifdef TM_NO_EVICT_FIRST  // A/B only
    (void)pol;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
    return;
#endif
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, int sh) { return __funnelshift_r(lo, hi, sh); }

struct Item {
    int64_t b, gi, ra, nrow, cs_cta, width;
};
// contig items: (segment s << 36) | (first row << 12) | rows (<= 4095); CONTIG =
// false compiles the round-robin decode only (the fused kernel: whole pairs)
template <bool CONTIG = true>
__device__ __forceinline__ Item decode(const TmaArgs &a, int64_t item) {
    Item it;
    if (CONTIG && a.contig) {
        const int64_t sgm = item >> 36;
        it.gi = sgm % a.n_groups;
        it.b = sgm / a.n_groups;
        it.ra = (item >> 12) & 0xFFFFFF;
        it.nrow = item & 0xFFF;
        it.cs_cta = it.gi * TCOLS;
        it.width = (a.M1 - it.cs_cta < TCOLS) ? a.M1 - it.cs_cta : TCOLS;
        return it;
    }
    // column groups fastest: CTAs running at the same time read adjacent 4 KB pieces
    // of the same rows (cfg5, 16 groups: 0.412 -> 0.407 ms; row chunks fastest before)
    it.gi = item % a.n_groups;
    item /= a.n_groups;
    const int64_t rc = item % a.n_rc;
    it.b = item / a.n_rc;
    it.ra = rc * a.R;
    const int64_t rb = (it.ra + a.R < a.rows) ? it.ra + a.R : a.rows;
    it.nrow = rb - it.ra;
    it.cs_cta = it.gi * TCOLS;
    it.width = (a.M1 - it.cs_cta < TCOLS) ? a.M1 - it.cs_cta : TCOLS;
    return it;
}

#ifndef TM_NE
#define TM_NE 8
#endif
constexpr int NE = TM_NE;  // epilogue warps

// comb(d): total count of unwrapped diagonal d (relative to the CTA's first column)
// from the warp-private arrays of one buffer: only the <= 3 warps whose strip
// [512 w - 16 ntile, 512 w + 511] contains d contribute.
__device__ __forceinline__ int32_t comb_at(const uint16_t *pv, int stride, int d, int ntile, int width) {
    const int pad = 16 * ntile;
    int wlo = (d - 511 + 511 + 512 * 64) / 512 - 64;  // ceil((d - 511) / 512)
    if (wlo < 0) wlo = 0;
    int whi = (d + pad) >> 9;                          // floor((d + pad) / 512)
    const int wmax = (width >> 9) - 1;
    if (whi > wmax) whi = wmax;
    int32_t v = 0;
    for (int w = wlo; w <= whi; ++w) {
        const int j = d - 512 * w + pad;
        if (j >= 0 && j < 512 + pad) v += (int32_t)pv[w * stride + j];
    }
    return v;
}

// comb_at for pad = 16 ntile <= 1024 (at most three strips hold a diagonal): the
// strips are w1 = max(d, 0) >> 9 and the next two, with no loop
__device__ __forceinline__ int32_t comb3(const uint16_t *pv, int stride, int d, int pad, int nw) {
    const int w1 = d < 0 ? 0 : (d >> 9);
    int32_t v = 0;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const int w = w1 + e, j = d - 512 * w + pad;
        if (w < nw && j >= 0 && j < 512 + pad) v += (int32_t)pv[w * stride + j];
    }
    return v;
}

// NST: ring stages.  TCM selects the fused kernel: 8 extra warps correlate each
// finished pair on the tensor cores (tc_core.cuh) while the fold streams the next.
constexpr int TC_GROUP = 5;  // named barrier of the tensor-core warps

template <int NST, int MINB = 1, bool TCM = false, int NEP = NE>
__global__ void __launch_bounds__((TW + 1 + NEP) * 32 + (TCM ? tc::NTHR : 0), MINB)
    fold_pm1_tma(TmaArgs a) {
    constexpr bool FUSED = TCM;
    extern __shared__ __align__(1024) uint8_t smem[];
    pdl_trigger();
    // without TM_INPUTS_STABLE the previous launch on the stream may still be writing
    // x or t: nothing is read before it has completed (griddepcontrol.wait)
    if (!a.x_early) pdl_wait();
    uint8_t *ring = smem;
    uint16_t *privb = reinterpret_cast<uint16_t *>(smem + NST * STAGE_BYTES);  // [2][TW][priv_stride]
    uint64_t *full = reinterpret_cast<uint64_t *>(privb + 2 * TW * a.priv_stride);
    uint64_t *empty = full + NST;
    uint64_t *pfull = empty + NST;   // [2]: consumers -> epilogue (count TW)
    uint64_t *pempty = pfull + 2;    // [2]: epilogue -> consumers (count NEP)
    uint64_t *yready = pempty + 2;   // [2]: y1 + y2 of a pair in global memory (count TW + NEP)
    uint64_t *ydone = yready + 2;    // [2]: tensor-core warps finished with a pair (count NTHR / 32)
    int64_t *item_q = reinterpret_cast<int64_t *>(ydone + 2);  // [8] producer -> consumers: item of seq
    int64_t *pitem = item_q + 8;     // [2] consumers -> epilogue / NTT warps: item of a buffer (-1 = end)
    uint4 *xs = reinterpret_cast<uint4 *>(pitem + 2);  // owner epilogue: x[0 .. K + q)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NTW = TCM ? tc::NTHR / 32 : 0;
    long long t_entry = 0;
    if constexpr (TCM) t_entry = tc::gtime();
    if (threadIdx.x == 0) {
        if constexpr (TCM) {
            mbar_init(reinterpret_cast<uint64_t *>(smem + a.tc_off + a.tca.offMisc), 1);  // MMA passes
            for (int b = 0; b < 2; ++b)  // pbegin: consumers -> tensor-core warps, pair of a buffer known
                mbar_init(reinterpret_cast<uint64_t *>(smem + a.tc_off + a.tca.offMisc + tc::MISC_PBEGIN) + b, 1);
        }
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TW);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&pfull[b], TW);
            mbar_init(&pempty[b], NEP);
            mbar_init(&yready[b], TW + NEP);
            mbar_init(&ydone[b], NTW > 0 ? NTW : 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if constexpr (TCM) {
        if (warp >= TW + 1 + NEP) {
            // ------------------------------------------------- tensor-core warps
            // steps 4-9 of each finished pair (tc_core.cuh), one pair behind the fold
            using GS = tc::GroupSync<TC_GROUP>;
            const int gt = threadIdx.x - (TW + 1 + NEP) * 32;
            uint8_t *tsm = smem + a.tc_off;
            uint32_t *tslot = reinterpret_cast<uint32_t *>(tsm + a.tca.offMisc + 8);
            if (gt < 32) {
                asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                                 smem_u32(tslot)),
                             "r"(a.tca.ncols));
                asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            GS::sync();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tbase = *tslot;
            uint32_t mph = 0;
            int pb = 0;
            uint32_t pph = 0;
            uint64_t *pbegin = reinterpret_cast<uint64_t *>(tsm + a.tca.offMisc + tc::MISC_PBEGIN);
            bool pdl_done = false;
            if (a.tca.dbg && gt == 0) a.tca.dbg[8 * a.n_items + 2 * blockIdx.x] = t_entry;
            for (;;) {
                tc::group_wait<GS>(&pbegin[pb], pph, gt >> 5);
                const int64_t b = pitem[pb];  // fused mode: items are whole pairs
                if (b < 0) break;
                tc::tc_pre<GS>(a.tca, tsm, b, gt);  // template side while the pair is being folded
                // y_1 is complete when the consumers finish the pair (pfull): stage it
                // while the epilogue warps finish y_2
                tc::group_wait<GS>(&pfull[pb], pph, gt >> 5);
                const int fl1 = tc::stage_y(a.tca, tsm + a.tca.offB, b, 0, 1, gt >> 5, lane, 0, 1);
                // the CTA's last pair (static schedule): the TMA ring is idle from here on,
                // so the A operand of the second template chunk is built into it now and
                // the MMAs of both chunks run back to back on the kernel's tail
                uint8_t *a_alt = nullptr;
#ifndef TM_NO_RING_A
                if (b + (int64_t)gridDim.x >= a.n_items && a.tca.NC > a.tca.CCH &&
                    2 * a.tca.CCH >= a.tca.NC &&
                    (uint32_t)(256 * (8 * (a.tca.NC - a.tca.CCH - 1) + 15)) <= (uint32_t)(NST * STAGE_BYTES)) {
                    tc::build_a(a.tca, tsm, a.tca.CCH, a.tca.NC, gt, smem);
                    a_alt = smem;
                }
#endif
                tc::group_wait<GS>(&yready[pb], pph, gt >> 5);
                if (!pdl_done) { pdl_wait(); pdl_done = true; }  // before the first residues / k stores
                tc::tc_main<GS>(a.tca, tsm, b, gt, warp & 3, tbase, mph, fl1, a_alt);
                __syncwarp();
                if (lane == 0) mbar_arrive(&ydone[pb]);
                if (++pb == 2) { pb = 0; pph ^= 1; }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            GS::sync();
            if (a.tca.dbg && gt == 0) a.tca.dbg[8 * a.n_items + 2 * blockIdx.x + 1] = tc::gtime();
            if (gt < 32)
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(a.tca.ncols));
            return;
        }
    }
    if (warp == TW) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const uint64_t pol = l2_evict_first_policy();
            // contig: this CTA's range [lin, lend) of the (segment, row) space, cut at
            // segment ends and every R rows (range ends on multiples of 16 rows)
            const int64_t Tr = a.n_segs * a.rows;
            auto rb = [&](int64_t c) -> int64_t {
                return c >= (int64_t)gridDim.x ? Tr : (c * Tr / (int64_t)gridDim.x) / 16 * 16;
            };
            int64_t lin = rb(blockIdx.x), lend = rb(blockIdx.x + 1);
            for (int64_t seq = 0;; ++seq) {
                int64_t item;
                if (!TCM && a.contig) {
                    if (lin >= lend) {
                        item = -1;
                    } else {
                        const int64_t sg = lin / a.rows, r0 = lin - sg * a.rows;
                        int64_t nr = a.rows - r0;
                        if (nr > a.R) nr = a.R;
                        if (nr > lend - lin) nr = lend - lin;
                        item = (sg << 36) | (r0 << 12) | nr;
                        lin += nr;
                    }
                } else {
                    item = blockIdx.x + seq * gridDim.x;
                    if (item >= a.n_items) item = -1;
                }
                item_q[seq & 7] = item;  // published by the arrive on the item's first stage
                if (item < 0) {          // end: complete one more stage phase with no data
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive(&full[s]);
                    break;
                }
                const Item it = decode<!TCM>(a, item);
                const int8_t *base = a.x + it.b * a.ldx + it.ra * a.M1 + it.cs_cta;
                for (int64_t r0 = 0; r0 < it.nrow; r0 += SROWS) {
                    const int nr = (int)((it.nrow - r0) < SROWS ? (it.nrow - r0) : SROWS);
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], (uint32_t)(nr * it.width));
                    uint8_t *dst = ring + s * STAGE_BYTES;
                    if (it.width == a.M1) {  // rows are contiguous in global memory
                        bulk_g2s_ef(dst, base + r0 * a.M1, (uint32_t)(nr * it.width), &full[s], pol);
                    } else {
                        for (int r = 0; r < nr; ++r)
                            bulk_g2s_ef(dst + r * it.width, base + (r0 + r) * a.M1, (uint32_t)it.width, &full[s], pol);
                    }
                    if (++s == NST) { s = 0; ph ^= 1; }
                }
            }
        }
        return;
    }

    if (warp > TW) {
        // ------------------------------------------------------------ epilogue
        const int et = threadIdx.x - (TW + 1) * 32;  // 0 .. NEP*32-1
        int pb = 0;
        uint32_t pph = 0;
        bool pdl_done = false;
        for (;;) {
            if constexpr (TCM) {
                // the pair of this buffer is known as soon as its fold starts: stage
                // x[0 .. K + q) (the wrap / extension terms) while it is being folded
                mbar_wait(reinterpret_cast<uint64_t *>(smem + a.tc_off + a.tca.offMisc + tc::MISC_PBEGIN) + pb, pph);
                const int64_t item0 = pitem[pb];
                if (item0 >= 0 && a.owner && !a.block) {
                    const int nx = (int)((a.K + decode<!TCM>(a, item0).nrow + 15) / 16);
                    const uint4 *src = reinterpret_cast<const uint4 *>(a.x + decode<!TCM>(a, item0).b * a.ldx);
                    uint4 *dst = reinterpret_cast<uint4 *>(xs);
                    for (int i = et; i < nx; i += NEP * 32) dst[i] = src[i];
                }
            }
            mbar_wait(&pfull[pb], pph);
            if (!pdl_done) { pdl_wait(); pdl_done = true; }  // before this warp's first y2 store / counts atomic
            long long te0 = 0;
            if constexpr (TCM) te0 = tc::gtime();
            const int64_t item = pitem[pb];
            if (item < 0) {
                if constexpr (FUSED) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&yready[pb]);
                }
                break;
            }
            const Item it = decode<!TCM>(a, item);
            const int ntile = (int)((it.nrow + 15) / 16);
            const int width = (int)it.width;
            const uint16_t *pv = privb + pb * TW * a.priv_stride;
            if (a.owner) {
                // whole pair, full fold: counts -> values, + wrap + extension, store y2
                const int q = (int)it.nrow;  // = q1 = q2 (M1 | N)
                // stage x[0 .. K + q) (all the wrap/extension terms read) with coalesced
                // 16-byte loads: one memory latency per pair instead of one per bin
                // (TM_BLOCK reads neither term)
                if (!a.block) {
                    if constexpr (!TCM) {  // (TCM: staged above, before the fold finished)
                        const int nx = (int)((a.K + q + 15) / 16);
                        const uint4 *src = reinterpret_cast<const uint4 *>(a.x + it.b * a.ldx);
                        uint4 *dst = reinterpret_cast<uint4 *>(xs);
                        for (int i = et; i < nx; i += NEP * 32) dst[i] = src[i];
                    }
                    asm volatile("bar.sync 2, %0;" ::"n"(NEP * 32) : "memory");
                }
                const int8_t *xb = reinterpret_cast<const int8_t *>(xs);
                int32_t *o2 = a.y2 + it.b * a.ldy2;
                const int M2 = (int)a.M2, M1 = (int)a.M1, K = (int)a.K;
                const int dlo = -16 * ntile;
                // (a straight-line / unrolled variant of this loop measured slower in the
                // fused kernel: it competes harder with the fold warps for issue slots)
                const int pad = 16 * ntile, nw = width >> 9;
                const bool c3 = pad <= 1024;
                // the CTA's last pair (its epilogue is on the kernel's tail; mid-run the
                // gentler per-bin loop below costs the concurrent fold less): runs of 16
                // consecutive bins per thread with 16-byte loads and stores (pad <= 512:
                // a diagonal then lies in at most two strips, or strip 0 when d < 0)
                const bool runs = TCM && item + (int64_t)gridDim.x >= a.n_items &&
                                  pad <= 512 && (q & 15) == 0 && (M1 & 15) == 0 && !a.accumulate &&
                                  ((reinterpret_cast<uintptr_t>(o2) & 15) == 0);
                if (runs) {
                    const int stride = a.priv_stride;
                    if (et == NEP * 32 - 1) {
                        // bin M1 = M2 - 1 in closed form: only the diagonal d = -1 (strip 0,
                        // index pad - 1) reaches it; its row g* = 0 < q is one element short,
                        // and the mod-N wrap adds x[q - 1]
                        int32_t v = q - 1 - (int32_t)pv[pad - 1];
                        if (!a.block) v += xb[q - 1];
                        o2[M1] = v;
                    }
                    for (int r = et; r < (M1 >> 4); r += NEP * 32) {
                        const int k0 = r << 4;
                        const int w1 = k0 >> 9, rel = (k0 & 511) + pad;
                        int32_t C[16];
                        {
                            const uint4 *sp = reinterpret_cast<const uint4 *>(pv + w1 * stride + rel);
                            const uint4 u0 = sp[0], u1 = sp[1];
                            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
                            for (int i = 0; i < 8; ++i) { C[2 * i] = (int32_t)(w[i] & 0xFFFFu); C[2 * i + 1] = (int32_t)(w[i] >> 16); }
                        }
                        if (rel >= 512 && w1 + 1 < nw) {
                            const uint4 *sp = reinterpret_cast<const uint4 *>(pv + (w1 + 1) * stride + rel - 512);
                            const uint4 u0 = sp[0], u1 = sp[1];
                            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
                            for (int i = 0; i < 8; ++i) { C[2 * i] += (int32_t)(w[i] & 0xFFFFu); C[2 * i + 1] += (int32_t)(w[i] >> 16); }
                        }
                        if (k0 + 15 >= M2 - pad) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (k0 + i >= M2 - pad) C[i] += (int32_t)pv[k0 + i - M2 + pad];
                        }
                        int32_t v[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = q - (M1 - (k0 + i) < q ? 1 : 0) - C[i];
                        if (!a.block && k0 + 15 >= M2 - q) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (k0 + i >= M2 - q) v[i] += xb[k0 + i - (M2 - q)];
                        }
                        int4 *dst = reinterpret_cast<int4 *>(o2 + k0);
#pragma unroll
                        for (int i = 0; i < 4; ++i) dst[i] = make_int4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                        if (k0 < K) {
                            int32_t e[16];
                            if (a.block) {
#pragma unroll
                                for (int i = 0; i < 16; ++i) e[i] = v[i];
                            } else {
                                const uint4 xk = *reinterpret_cast<const uint4 *>(xb + k0);
                                const uint4 xq = *reinterpret_cast<const uint4 *>(xb + k0 + q);
                                const uint32_t wk[4] = {xk.x, xk.y, xk.z, xk.w}, wq[4] = {xq.x, xq.y, xq.z, xq.w};
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    e[i] = v[i] - (int32_t)(int8_t)(wk[i >> 2] >> (8 * (i & 3))) +
                                           (int32_t)(int8_t)(wq[i >> 2] >> (8 * (i & 3)));
                            }
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (k0 + i < K) o2[M2 + k0 + i] = e[i];
                        }
                    }
                }
#pragma unroll 2
                for (int k = runs ? M2 : et; k < M2; k += NEP * 32) {  // (runs: every bin is done)
                    // bin k collects the unwrapped diagonals d = k and d = k - M2 (d >= dlo)
                    int32_t C = c3 ? comb3(pv, a.priv_stride, k, pad, nw) : comb_at(pv, a.priv_stride, k, ntile, width);
                    if (k - M2 >= dlo)
                        C += c3 ? comb3(pv, a.priv_stride, k - M2, pad, nw)
                                : comb_at(pv, a.priv_stride, k - M2, ntile, width);
                    int gs = M1 - k;
                    if (gs < 0) gs += M2;
                    int32_t v = q - (gs < q ? 1 : 0) - C;
                    const int j = k - (M2 - q);  // mod-N wrap: bin M2 - q + j gets x[j]
                    if (j >= 0 && !a.block) v += xb[j];
                    if (a.accumulate) o2[k] += v; else o2[k] = v;
                    if (k < K) {                 // y2[M2 + k] = y2[k] - x[k] + x[k + q]  (s2 = q)
                        const int32_t e = a.block ? v : v - xb[k] + xb[k + q];
                        if (a.accumulate) o2[M2 + k] += e; else o2[M2 + k] = e;
                    }
                }
                asm volatile("bar.sync 2, %0;" ::"n"(NEP * 32) : "memory");  // xs reuse
            } else {
                int32_t *c2 = a.counts + it.b * (a.M1 + a.M2) + a.M1;
                const int64_t g0 = a.row0 + it.ra;
                const int dlo = -16 * ntile;
                int64_t bin0 = ((int64_t)dlo + it.cs_cta - g0) % a.M2;
                if (bin0 < 0) bin0 += a.M2;
                const int pad = 16 * ntile, nw = width >> 9;
                const bool c3 = pad <= 1024;
                for (int i = et; i < width - dlo; i += NEP * 32) {
                    const int v = c3 ? comb3(pv, a.priv_stride, dlo + i, pad, nw)
                                     : comb_at(pv, a.priv_stride, dlo + i, ntile, width);
                    if (v) {
                        int64_t bin = bin0 + i;
                        while (bin >= a.M2) bin -= a.M2;
                        atomicAdd(&c2[bin], v);
                    }
                }
            }
            if constexpr (FUSED) __threadfence_block();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pempty[pb]);
                if constexpr (FUSED) mbar_arrive(&yready[pb]);
            }
            if constexpr (TCM) {  // instrumentation: duration of this CTA's latest epilogue
                if (a.tca.dbg && et == 0) a.tca.dbg[8 * a.n_items + 3 * gridDim.x + blockIdx.x] = tc::gtime() - te0;
            }
            if (++pb == 2) { pb = 0; pph ^= 1; }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // Per-warp private anti-diagonal arrays priv[w][0 .. 512 + 16*ntile): warp w's
    // unwrapped diagonal d (relative to its strip start cs_w) lives at index
    // d + 16*ntile.  Every index is written exactly once: lane 31's finished block
    // of tile t (the chain output) and, after the last tile, each lane's low block
    // plus its left neighbour's pending carry.  No atomics, no zero-fill.  The two
    // buffers alternate between items; the epilogue warps turn one into y2 while
    // the consumers fill the other.
    int s = 0;
    uint32_t ph = 0;
    int pb = 0;
    uint32_t pph = 0;
    const uint32_t ring_u32 = smem_u32(ring);
#ifdef TM_CONS_PROF
    long long cp_wait = 0, cp_busy = 0, cp_t = clock64();
#endif
    for (int64_t seq = 0;; ++seq) {
        mbar_wait(&full[s], ph);  // first stage of the next item (or the end marker)
        const int64_t item = item_q[seq & 7];
        mbar_wait(&pempty[pb], pph ^ 1);
        if constexpr (FUSED) mbar_wait(&ydone[pb], pph ^ 1);  // bounds the fold's lead over the correlation
        if (item < 0) {  // tell the epilogue (and the NTT / tensor-core warps) to stop
#ifdef TM_CONS_PROF
            if constexpr (TCM) {
                if (a.tca.dbg && lane == 0 && warp < 8) {
                    long long *d = a.tca.dbg + 8 * a.n_items + 4 * gridDim.x + 16 * blockIdx.x + 2 * warp;
                    d[0] = cp_wait; d[1] = cp_busy;
                }
            }
#endif
            if (lane == 0 && warp == 0) {
                pitem[pb] = -1;
                if constexpr (TCM) mbar_arrive(reinterpret_cast<uint64_t *>(smem + a.tc_off + a.tca.offMisc + tc::MISC_PBEGIN) + pb);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pfull[pb]);
                if constexpr (FUSED) mbar_arrive(&yready[pb]);
            }
            break;
        }
        const Item it = decode<!TCM>(a, item);
        const int nrow = (int)it.nrow;
        const int ntile = (nrow + 15) / 16;
        const int width = (int)it.width;
        const bool active = warp * 512 < width;
        const int colb = warp * 512 + 16 * lane;  // byte column inside a stage row
        uint16_t *priv = privb + (pb * TW + warp) * a.priv_stride;
        if (lane == 0 && warp == 0) {
            pitem[pb] = item;
            if constexpr (TCM) mbar_arrive(reinterpret_cast<uint64_t *>(smem + a.tc_off + a.tca.offMisc + tc::MISC_PBEGIN) + pb);
        }
        uint32_t y1w[8], carry[8], W[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { y1w[i] = 0; carry[i] = 0; W[i] = 0; }
        uint32_t a1[4] = {0, 0, 0, 0};
        for (int t = 0; t < ntile; ++t) {
            // the finished low block of the previous tile becomes this tile's high block
#pragma unroll
            for (int i = 0; i < 4; ++i) { W[4 + i] = W[i]; W[i] = 0; }
            const bool full_tile = (t * 16 + 16 <= nrow) && width == TCOLS;
#pragma unroll
            for (int half = 0; half < 16 / SROWS; ++half) {
                const int rbase = t * 16 + half * SROWS;
                if (rbase >= nrow) break;
#ifdef TM_CONS_PROF
                { long long t1 = clock64(); cp_busy += t1 - cp_t; cp_t = t1; }
#endif
                mbar_wait(&full[s], ph);
#ifdef TM_CONS_PROF
                { long long t1 = clock64(); cp_wait += t1 - cp_t; cp_t = t1; }
#endif
                const uint32_t st = ring_u32 + s * STAGE_BYTES + colb;
                const uint32_t rstride = full_tile ? TCOLS : width;
#pragma unroll
                for (int g = 0; g < GPS; ++g) {
                    // 4 rows r = SROWS half + 4 g + rho, rho = 0..3 (alpha = r >> 2 = GPS half + g).
                    // FULL (the tile is 16 whole rows of TCOLS columns): no row masks.
                    auto group = [&](auto fullc) {
                        constexpr bool FULL = decltype(fullc)::value;
                        uint32_t m[4][4];
#pragma unroll
                        for (int rho = 0; rho < 4; ++rho) {
                            const int rr = g * 4 + rho;
                            uint4 v;
                            // branch-free: every lane loads inside the stage (rows past the
                            // item's end hold stale bytes) and a row mask zeroes what is not data
                            const uint32_t msk = (FULL || (active && rbase + rr < nrow)) ? 0x02020202u : 0u;
                            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                         : "r"(st + rr * (FULL ? (uint32_t)TCOLS : rstride)));
                            m[rho][0] = v.x & msk; m[rho][1] = v.y & msk;
                            m[rho][2] = v.z & msk; m[rho][3] = v.w & msk;
                        }
                        if (!FULL && !active) return;
                        // M1: column sums in byte lanes
#pragma unroll
                        for (int w = 0; w < 4; ++w) a1[w] = a1[w] + (m[0][w] + m[1][w]) + (m[2][w] + m[3][w]);
                        // M2: row r, byte j -> window byte 16 - r + j.  With alpha = r >> 2 and
                        // rho = r & 3, window word 4 - alpha + k' (k' = -1..3) receives
                        // funnelshift_r(m[k'], m[k'+1], 8 rho) (m[-1] = m[4] = 0).
                        const int alpha = half * GPS + g;
#pragma unroll
                        for (int kk = -1; kk < 4; ++kk) {
                            uint32_t add = (kk >= 0) ? m[0][kk] : 0u;
#pragma unroll
                            for (int rho = 1; rho < 4; ++rho) {
                                const uint32_t lo = (kk >= 0) ? m[rho][kk] : 0u;
                                const uint32_t hi = (kk + 1 < 4) ? m[rho][kk + 1] : 0u;
                                add += fsr(lo, hi, 8 * rho);
                            }
                            W[4 - alpha + kk] += add;
                        }
                    };
#ifndef TM_FOLD_NOCOMPUTE
                    if (full_tile) group(std::true_type{});
                    else group(std::false_type{});
#else  // A/B only: the fold's streaming without its arithmetic (results are wrong)
                    (void)full_tile;
#endif
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (++s == NST) { s = 0; ph ^= 1; }
            }
            if (!active) continue;
            if ((t & 3) == 3 || t == ntile - 1) {  // widen byte counters before they can overflow
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    y1w[2 * w] += __byte_perm(a1[w], 0, 0x4140);
                    y1w[2 * w + 1] += __byte_perm(a1[w], 0, 0x4342);
                    a1[w] = 0;
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, carry[i], 1);
                const uint32_t add = __byte_perm(W[4 + (i >> 1)], 0, (i & 1) ? 0x4342 : 0x4140);
                carry[i] = (lane ? v : 0u) + add;
            }
            if (lane == 31) {  // finished block of the whole warp: bins cs_w + 496 - 16 t + [0, 16)
                // carry[i] holds bins 2i (low half) and 2i + 1 (high half): already packed u16 pairs
                uint4 *dst = reinterpret_cast<uint4 *>(priv + 496 - 16 * t + 16 * ntile);
                dst[0] = make_uint4(carry[0], carry[1], carry[2], carry[3]);
                dst[1] = make_uint4(carry[4], carry[5], carry[6], carry[7]);
            }
        }
        const int64_t c0 = it.cs_cta + warp * 512 + 16 * lane;
        if (seq == 0) pdl_wait();  // first global write of this warp (y1 / counts) follows
        if (active) {
            // drain: lane l's low block (bins 16 l - 16 ntile + [0,16)) + lane l-1's pending carry
            uint32_t lo[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t c = __shfl_up_sync(0xffffffffu, carry[i], 1);
                lo[i] = __byte_perm(W[i >> 1], 0, (i & 1) ? 0x4342 : 0x4140) + ((lane && ntile) ? c : 0u);
            }
            uint4 *dst = reinterpret_cast<uint4 *>(priv + 16 * lane);
            dst[0] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            dst[1] = make_uint4(lo[4], lo[5], lo[6], lo[7]);
            // M1 bins are owned by this lane: write them now
            if (a.owner) {
                const int32_t q = nrow;
                int32_t v[16];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    v[2 * i] = q - (int32_t)(y1w[i] & 0xFFFFu);
                    v[2 * i + 1] = q - (int32_t)(y1w[i] >> 16);
                }
                int32_t *o1 = a.y1 + it.b * a.ldy1;
#pragma unroll
                for (int rep = 0; rep < 2; ++rep) {  // y1[c] and y1[M1 + c] = y1[c] (M1 | N), c < K
                    const int64_t base = rep ? a.M1 + c0 : c0;
                    if (rep && c0 >= a.K) break;
                    if (!rep || c0 + 16 <= a.K) {
                        if ((((uintptr_t)(o1 + base)) & 15) == 0) {
                            int4 *d0 = reinterpret_cast<int4 *>(o1 + base);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                int4 w = make_int4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                                if (a.accumulate) {
                                    const int4 o = d0[i];
                                    w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
                                }
                                d0[i] = w;
                            }
                            continue;
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        if (rep && c0 + i >= a.K) break;
                        if (a.accumulate) o1[base + i] += v[i]; else o1[base + i] = v[i];
                    }
                }
            } else {
                int32_t *cnt = a.counts + it.b * (a.M1 + a.M2);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    atomicAdd(&cnt[c0 + 2 * i], (int)(y1w[i] & 0xFFFFu));
                    atomicAdd(&cnt[c0 + 2 * i + 1], (int)(y1w[i] >> 16));
                }
            }
        }
        if constexpr (FUSED) __threadfence_block();
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&pfull[pb]);
            if constexpr (FUSED) mbar_arrive(&yready[pb]);
        }
        if constexpr (TCM) {  // instrumentation: end of this CTA's latest fold item
            if (a.tca.dbg && warp == 0 && lane == 0) a.tca.dbg[8 * a.n_items + 2 * gridDim.x + blockIdx.x] = tc::gtime();
        }
        if (++pb == 2) { pb = 0; pph ^= 1; }
    }
}

}  // namespace

// Returns TM_OK after enqueueing, or TM_EUNSUPPORTED when the shape is not covered
// (the caller then uses the register-streaming fold_pm1).
namespace {

int setup_args(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len, void *y1,
               void *y2, int accumulate, void *ws, int64_t R, int64_t n_rc, TmaArgs &a) {
    a.x = (const int8_t *)x; a.ldx = ldx;
    a.N = p->N; a.M1 = p->M1; a.M2 = p->M2; a.K = p->K; a.q2 = p->q2;
    a.block = p->block;
    a.rows = len / p->M1; a.row0 = offset / p->M1;
    a.n_groups = (p->M1 + TCOLS - 1) / TCOLS;
    a.R = R; a.n_rc = n_rc;
    a.n_items = batch * a.n_groups * a.n_rc;
    a.owner = (a.n_groups == 1 && a.n_rc == 1 && offset == 0 && len == p->N) ? 1 : 0;
    a.accumulate = accumulate;
    a.x_early = (p->flags & TM_INPUTS_STABLE) ? 1 : 0;
    if (R > 2048) return TM_EUNSUPPORTED;
    a.priv_stride = (int)(512 + (R + 15) / 16 * 16);
    a.acc_words = TW * a.priv_stride;
    tm_ws_layout L = tm_ws(p, batch);
    a.counts = (int32_t *)((char *)ws + L.fold_counts);
    a.y1 = (int32_t *)y1; a.y2 = (int32_t *)y2;
    a.ldy1 = p->M1 + p->K; a.ldy2 = p->M2 + p->K;
    a.xs_bytes = a.owner ? (int)((p->K + R + 15) / 16 * 16) : 0;
    return TM_OK;
}

#ifndef TM_FOLD_NST
#define TM_FOLD_NST 4
#endif
constexpr int TM_FOLD_NST_DEF = TM_FOLD_NST;

size_t smem_bytes(const TmaArgs &a, int nst) {
    return (size_t)nst * STAGE_BYTES + (size_t)2 * a.acc_words * 2 + (2 * nst + 8) * 8 + 10 * 8 + a.xs_bytes;
}

template <int NST, int MINB = 1, bool TCM = false, int NEP = NE>
int launch(const TmaArgs &a, int64_t grid, size_t smem, cudaStream_t s) {
    auto k = fold_pm1_tma<NST, MINB, TCM, NEP>;
    cudaError_t e = tm_smem_attr((const void *)k, 227 * 1024, true);
    if (e != cudaSuccess) return tm_cuda_status(e, "fold_pm1_tma: shared-memory attribute");
    const unsigned nthr = (TW + 1 + NEP) * 32 + (TCM ? tc::NTHR : 0);
    if (tm_pdl_enabled()) {  // programmatic dependent launch: see pdl_trigger / pdl_wait
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(nthr);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, k, a);
        if (e != cudaSuccess) return tm_cuda_status(e, "fold_pm1_tma (PDL launch)");
        TM_CHECK_LAUNCH("fold_pm1_tma");
        return TM_OK;
    }
    k<<<(unsigned)grid, nthr, smem, s>>>(a);
    TM_CHECK_LAUNCH("fold_pm1_tma");
    return TM_OK;
}

}  // namespace

// counts workspace reset as a PDL kernel (a memset between kernels would end the
// overlap of consecutive steps): waits for the previous launch, then zeroes
__global__ void zero_i32(int32_t *p, int64_t n) {
    pdl_trigger();
    pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0;
}

int tm_fold_tma(const tm_plan_s *p, const void *x, int64_t ldx, int64_t batch, int64_t offset, int64_t len,
                void *y1, int64_t ldy1, void *y2, int64_t ldy2, int accumulate, void *ws, int64_t R, int64_t n_rc,
                cudaStream_t s, bool *used_counts, bool force_counts) {
    TmaArgs a{};
    int rc = setup_args(p, x, ldx, batch, offset, len, y1, y2, accumulate, ws, R, n_rc, a);
    if (rc) return rc;
    if (force_counts && a.owner) {  // tm_fold_reduce: the finalize kernel writes the outputs
        a.owner = 0;
        a.xs_bytes = 0;
    }
    a.ldy1 = ldy1; a.ldy2 = ldy2;
    *used_counts = !a.owner;
    static const char *env_contig = getenv("TM_FOLD_CONTIG");  // A/B: "0" = round-robin row chunks
    // ring stages: 5 for rows read as >= 8 separate 4 KB pieces (wide M1: cfg5's 16
    // column groups, 0.3389 -> 0.3355 ms), 4 otherwise (contiguous 32 KB stages
    // measured 4-5% slower with 5: cfg4a 0.177 -> 0.185 ms)
    int nst = (a.n_groups >= 8 && TM_FOLD_NST_DEF == 4) ? 5 : TM_FOLD_NST_DEF;
    // dual: two smaller fold CTAs per SM (2-stage rings, 4 epilogue warps, items <= 1024
    // rows): 16 consumer warps per SM instead of 8
    // (same box, per step: cfg5 (16 groups) 0.383 -> 0.375 ms, K = 8192 (2 groups)
    // 0.233 -> 0.223, K = 4096 (1 group) 0.200 -> 0.197, but K = 16384 (4 groups)
    // 0.277 -> 0.285 and K = 32768 / 65536 (8 / 16 groups of 64 pairs) unchanged:
    // dual except for 3..7 column groups; TM_FOLD_DUAL=0/1 forces)
    static const char *env_dual = getenv("TM_FOLD_DUAL");
    bool dual = !a.owner && (a.n_groups <= 2 || a.n_groups >= 8);
    if (env_dual) dual = !a.owner && env_dual[0] == '1';
    if (dual) nst = 2;
    if (!a.owner && !(env_contig && env_contig[0] == '0')) {
        // split items: each CTA folds one contiguous range of (pair, group, row) --
        // balanced to 16 rows, with R up to the shared-memory budget -- instead of
        // round-robin row chunks: fewer, longer items (fewer count atomics and
        // item hand-offs) without a last-wave imbalance
        a.contig = 1;
        a.n_segs = batch * a.n_groups;
#ifndef TM_FOLD_RCAP
#define TM_FOLD_RCAP 2048
#endif
        int64_t Rc = dual ? 1024 : TM_FOLD_RCAP;
        const size_t budget = dual ? (size_t)112 * 1024 : (size_t)227 * 1024;
        while (Rc > 16) {
            a.R = Rc;
            a.priv_stride = (int)(512 + Rc);
            a.acc_words = TW * a.priv_stride;
            if (smem_bytes(a, nst) <= budget) break;
            Rc -= 256;
        }
    }
    if (!a.owner) {
        const int64_t n = batch * (p->M1 + p->M2);
        const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4 * (int64_t)p->num_sms);
        const cudaError_t e = launch_pdl(zero_i32, dim3((unsigned)blocks), dim3(256), 0, s, a.counts, n);
        if (e != cudaSuccess) return tm_cuda_status(e, "tm_fold: counts reset");
        TM_CHECK_LAUNCH("tm_fold: zero_i32");
    }
    const size_t smem = smem_bytes(a, nst);
    if (smem > 227 * 1024) return TM_EUNSUPPORTED;
#ifndef TM_FOLD_MINB
#define TM_FOLD_MINB 1  // A/B: 2 = two (smaller) fold CTAs per SM
#endif
    int64_t slots = (int64_t)p->num_sms * (dual ? 2 : TM_FOLD_MINB);
    {   // A/B: cap on the fold's CTAs (SMs left half free for a concurrently resident correlation)
        const char *env_cap = getenv("TM_FOLD_SLOTS");
        if (env_cap && atoll(env_cap) > 0 && atoll(env_cap) < slots) slots = atoll(env_cap);
    }
    int64_t grid = a.n_items < slots ? a.n_items : slots;
    if (a.contig) {
        const int64_t units = (a.n_segs * a.rows + 15) / 16;
        grid = units < slots ? units : slots;
    }
    if (dual) return launch<2, 2, false, 4>(a, grid, smem, s);
    if (nst == 5) return launch<5, TM_FOLD_MINB>(a, grid, smem, s);
    return launch<TM_FOLD_NST, TM_FOLD_MINB>(a, grid, smem, s);
}

// The whole of Algorithm 1 in ONE persistent kernel with the tensor-core
// correlation: per SM, the fold warps stream pair i+1 while 8 tensor-core
// warps correlate pair i (tc_core.cuh).  Whole pairs per item (M1 <= 4096,
// q <= 1024).  Returns TM_EUNSUPPORTED (nothing enqueued) when the plan/batch
// does not qualify.
bool tm_fused_tc_ok(const tm_plan_s *p, int64_t batch) {
    static const char *env = getenv("TM_FUSED_TC");  // A/B: "0" forces the staged kernels
    static const bool off = env && env[0] == '0';
    if (off) return false;
    return p->use_tc && p->tc_ok && p->fast_fold && p->M1 <= TCOLS && p->q1 <= 1024 && p->N == p->M1 * p->q1 &&
           batch >= 1;
}

int tm_fold_tc_fused(const tm_plan_s *p, const void *x, int64_t ldx, const void *t, int64_t batch, void *y1,
                     void *y2, int32_t *residues, int64_t *k, void *ws, cudaStream_t s) {
    if (!tm_fused_tc_ok(p, batch)) return TM_EUNSUPPORTED;
    if (((uintptr_t)x % 16) || (ldx % 16)) return TM_EUNSUPPORTED;
    TmaArgs a{};
    const int64_t R = (p->q1 + 15) / 16 * 16;
    int rc = setup_args(p, x, ldx, batch, 0, p->N, y1, y2, 0, ws, R, 1, a);
    if (rc) return rc;
    if (!a.owner) return TM_EUNSUPPORTED;
    tm_tc_fill_args(p, y1, y2, t, p->K, nullptr, nullptr, nullptr, residues, k, a.tca);
    a.tca.dbg = tm_tc_dbg_buffer();
    // y is scratch here: 128-byte rows, dropped from L2 without write-back once
    // correlated (TM_KEEP_Y, a test hook, keeps them for inspection)
    a.ldy1 = a.tca.ldy[0] = p->ldy1_run;
    a.ldy2 = a.tca.ldy[1] = p->ldy2_run;
    a.tca.discard_y = (p->flags & TM_KEEP_Y) ? 0 : 1;
    // 4-stage ring when the tensor-core region fits next to it, else 3 stages
    constexpr int K4 = 32 / SROWS;   // "4 stages" of 8 rows: the same 128 KB ring in SROWS-row stages
    constexpr int K3 = 24 / SROWS;
    const size_t base4 = (smem_bytes(a, K4) + 1023) / 1024 * 1024;
    const size_t base3 = (smem_bytes(a, K3) + 1023) / 1024 * 1024;
    const int nst = (base4 + p->tc_smem <= 227 * 1024) ? K4 : K3;
    const size_t base = nst == K4 ? base4 : base3;
    a.tc_off = (uint32_t)base;
    const size_t sm = base + p->tc_smem;
    if (sm > 227 * 1024) return TM_EUNSUPPORTED;
    // whole pairs are equal-sized items: the static round-robin schedule balances
    // them as well as a dynamic counter and needs no per-launch reset
    const int64_t grid = batch < p->num_sms ? batch : p->num_sms;
    if (nst == K4) return launch<K4, 1, true>(a, grid, sm, s);
    return launch<K3, 1, true>(a, grid, sm, s);
}
