// dip_order.cu -- sm_100a kernel for schedules given as per-rank stage orders (SURVEY §8(f) rows
// f1 / f2 / f3 with the dual-queue interleaving of PAPER.md §5.2, reading R-29):
//
//   BUILD  (dip_interleave): from a record's split and forward / backward PRIORITY
//          orders, run DIP's dual-queue greedy -- every rank keeps its ready forward / backward
//          stages as bitmaps over priority positions; the greedy places on the rank with the
//          smallest t_min (REDUX over the lanes), which picks the direction (1F1B alternation
//          when both queues are ready before t_last, else the smaller minimum start, ties to the
//          backward) and its highest-priority stage among those starting as early as possible,
//          places it and publishes its end to the consumers' ready sets. Emits every rank's order.
//          A step also places on every other rank that no earlier placement of the serial greedy
//          can reach (a conservative lookahead over the ring of ranks, below): the same orders in
//          about a third of the steps on 94B.
//   TIME   (dip_eval_orders): the longest path of explicit per-rank orders, lock-step
//          rounds as the record scorer, optionally with each stage pair's f3 selection (M4) and
//          per-stage timelines (f4).
//
// One group of G lanes per schedule, lane = pipeline rank. Dependencies live in per-SEGMENT state
// in shared memory (the segment DAG is a set of chains over ranks): slot[s] holds the end of the
// stage last done for segment s -- the input of the next rank -- and, before the segment's first
// stage on its entry rank (rank 0 for F, rank P-1 for B), the wrap/join accumulator of the
// cross-chunk / cross-module edges (pending count in bits 56..63, max value below, as in the
// record scorer). No channel rings and no spill: a chain has one live value at a time.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dip_internal.h"

namespace dipk {

namespace {

__device__ __forceinline__ uint32_t o_smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void o_mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(o_smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void o_mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(o_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void o_tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            o_smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(o_smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void o_mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(o_smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

template <int G>
__device__ __forceinline__ uint64_t o_group_max(uint64_t v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o, G);
        v = w > v ? w : v;
    }
    return v;
}
template <int G>
__device__ __forceinline__ uint64_t o_group_min(uint64_t v) {
    if constexpr (G == 32) {
        const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
        const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
        const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
        return ((uint64_t)mh << 32) | ml;
    } else {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o, G);
            v = w < v ? w : v;
        }
        return v;
    }
}
template <int G>
__device__ __forceinline__ uint64_t o_group_sum(uint64_t v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

constexpr uint64_t O_HIGH = ~VAL_MASK;
constexpr uint64_t O_INF = ~0ull;
// BUILD's lookahead: times relative to the step's smallest key, saturated (a smaller bound or key
// only makes a rank wait); rounds of the neighbour-bound relaxation per step
constexpr uint32_t O_CAP = 0x7FFFFFFFu;
#ifndef DIP_ORDER_NIT
#define DIP_ORDER_NIT 3
#endif
constexpr int O_NIT = DIP_ORDER_NIT;

// fold `value` into a wrap / join accumulator; true when it became ready (last producer)
__device__ __forceinline__ bool wrap_publish(uint64_t *slot, uint64_t value) {
    const uint64_t old = *slot, c = (old & O_HIGH) | (value & VAL_MASK);
    const uint64_t nv = (c > old ? c : old) + (1ull << PEND_SHIFT);
    *slot = nv;
    return (nv >> PEND_SHIFT) == 0;
}

}  // namespace

// OM: 0 = TIME of explicit per-rank orders, 1 = BUILD (f1), 2 = TIME of a record's own orders (its
// shared sequences + F/B bit rows: the record scorer on per-segment state)
template <int G, int OM>
__global__ void __launch_bounds__(768) dip_order_kernel(const KParams kp) {
    constexpr bool BUILD = OM == 1;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t blob_bar;
    constexpr int CPG = 32 / G;
    const unsigned FULL = 0xffffffffu;

    if (threadIdx.x == 0) {   // static tables -> smem, one TMA bulk copy per CTA
        o_mbar_init(&blob_bar, 1);
        o_mbar_expect_tx(&blob_bar, kp.blob_bytes);
        o_tma_bulk_g2s(smem, kp.blob, kp.blob_bytes, &blob_bar);
    }
    __syncthreads();
    o_mbar_wait(&blob_bar, 0);

    const ModInfo *mi = reinterpret_cast<const ModInfo *>(smem + kp.b_modinfo);
    const uint32_t *segdec = reinterpret_cast<const uint32_t *>(smem + kp.b_segdec);
    const uint16_t *layers = reinterpret_cast<const uint16_t *>(smem + kp.b_layers);
    const uint4 *tab = reinterpret_cast<const uint4 *>(smem + kp.b_tab);
    const uint32_t *woff = reinterpret_cast<const uint32_t *>(smem + kp.b_woff);
    const uint16_t *wtab = reinterpret_cast<const uint16_t *>(smem + kp.b_wtab);
    const uint16_t *nbi = reinterpret_cast<const uint16_t *>(smem + kp.b_nbi);
    const uint16_t *sbase = reinterpret_cast<const uint16_t *>(smem + kp.b_sbase);
    const uint32_t *budget = reinterpret_cast<const uint32_t *>(smem + kp.b_budget);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / G, r = lane % G;
    const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (g * G));
    const uint32_t P = kp.P, nmod = kp.nmod, nq = kp.m * kp.nmod, n_max = kp.n_max;
    const uint32_t nw = (n_max + 31) / 32;
    uint8_t *ga = smem + kp.blob_bytes + (size_t)(warp * CPG + g) * kp.o_bytes;
    uint32_t *rowx = reinterpret_cast<uint32_t *>(ga + kp.o_row);     // [n_max] per segment: tab | layer row << 12
    uint16_t *seqF = reinterpret_cast<uint16_t *>(ga + kp.o_seq);     // [n_pad] priority position -> segment
    uint16_t *seqB = seqF + kp.n_pad;
    uint16_t *pofF = reinterpret_cast<uint16_t *>(ga + kp.o_posof);   // [n_max] segment -> priority position
    uint16_t *pofB = pofF + n_max;
    uint64_t *slF = reinterpret_cast<uint64_t *>(ga + kp.o_sl);       // [n_max] per-segment F / B slots
    uint64_t *slB = slF + n_max;
    uint8_t *hF = ga + kp.o_h;                                        // [n_max] ranks done (F: from 0 up,
    uint8_t *hB = hF + n_max;                                         //   B: from P-1 down)
    uint32_t *bmF = reinterpret_cast<uint32_t *>(ga + kp.o_bm);       // [P][nw] ready F positions (BUILD)
    uint32_t *bmB = bmF + P * nw;                                     // [P][nw] ready B positions
    uint32_t *smF = reinterpret_cast<uint32_t *>(ga + kp.o_sum);      // [P] non-empty words of bmF rows
    uint32_t *smB = smF + P;                                          // [P] ... of bmB rows
    uint8_t *Mb = ga + kp.o_mb;
    uint8_t *Pc = Mb + nq;
    uint8_t *Cc = Pc + nq;
    const bool isFirst = r == 0, isLast = r == (int)P - 1, laneOn = r < (int)P;
    const uint32_t bud = budget[laneOn ? r : 0];

    unsigned long long best = ~0ull;

    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(kp.counter, (unsigned long long)CPG);
        base = __shfl_sync(FULL, base, 0);
        if (base >= kp.count) break;
        const uint64_t cand = base + g;
        const bool gvalid = cand < kp.count;
        const uint8_t *rec = kp.records + (gvalid ? cand : 0) * (uint64_t)kp.stride;

        // ---------------- decode + validate (split, counts; BUILD: priority orders; TIME: orders)
        const uint32_t hdr = __ldg(reinterpret_cast<const uint32_t *>(rec));
        const uint32_t n = hdr & 0xFFFFu;
        bool bad = !gvalid || (hdr >> 16) != 0 || n > n_max;
        uint32_t nsum = 0;
        for (uint32_t q = r; q < nq; q += G) {
            const uint32_t b = q / nmod, i = q - b * nmod;
            const uint32_t N = nbi[q], Mx = mi[i].max_split;
            uint32_t M;
            if (Mx > 1) {
                const uint32_t nib = b * kp.nsplit + mi[i].nib_slot;
                M = (__ldg(rec + kp.off_nib + (nib >> 1)) >> ((nib & 1) * 4)) & 15u;
            } else {
                M = N > 0 ? 1u : 0u;
            }
            const uint32_t hi = N < Mx ? N : Mx;
            if ((N == 0) != (M == 0) || M > hi) bad = true;
            Mb[q] = (uint8_t)M;
            nsum += M * mi[i].K;
        }
        nsum = (uint32_t)o_group_sum<G>(nsum);
        if (nsum != n) bad = true;
        for (uint32_t w = r; w < 2 * P * nw; w += G) bmF[w] = 0u;
        __syncwarp();
        for (uint32_t q = r; q < nq; q += G) {   // join fan-in / fan-out counts (R-5, R-6)
            const uint32_t b = q / nmod, i = q - b * nmod;
            uint32_t pc = 0, cc = 0;
            for (uint32_t x = 0; x < nmod; x++) {
                if ((mi[i].prod_mask >> x) & 1u) pc += Mb[b * nmod + x];
                if ((mi[i].cons_mask >> x) & 1u) cc += Mb[b * nmod + x];
            }
            Pc[q] = (uint8_t)pc;
            Cc[q] = (uint8_t)cc;
        }
        __syncwarp();
        uint32_t wcur = 0, wnext = 0;
        if (OM == 2 && laneOn) {   // the record's F/B bit row: exactly n ones in [0, 2n), zeros beyond
            const uint32_t lim = 2 * n;
            uint32_t ones = 0;
            for (uint32_t w = 0; w < kp.fbw; w++) {
                const uint32_t word = __ldg(reinterpret_cast<const uint32_t *>(rec + kp.off_fb) + w * P + r);
                if (w == 0) wcur = word;
                if (w == 1) wnext = word;
                if (32 * w + 32 <= lim) {
                    ones += __popc(word);
                } else if (32 * w >= lim) {
                    if (word) bad = true;
                } else {
                    const uint32_t msk = (1u << (lim - 32 * w)) - 1u;
                    ones += __popc(word & msk);
                    if (word & ~msk) bad = true;
                }
            }
            if (ones != n) bad = true;
        }
        if (OM >= 1) {
            // priority orders: 16-byte loads; permutations of the present segment ids, 0xFFFF padding
            // (validation bitmaps: rank 0's and rank 1's rows of bmF, cleared again below)
            uint32_t *vF = bmF, *vB = bmB;
            const uint32_t nv = kp.n_pad / 8;
            for (uint32_t v = r; v < nv; v += G) {
                const uint4 f4 = __ldg(reinterpret_cast<const uint4 *>(rec + kp.off_fwd) + v);
                const uint4 b4 = __ldg(reinterpret_cast<const uint4 *>(rec + kp.off_bwd) + v);
                reinterpret_cast<uint4 *>(seqF)[v] = f4;
                reinterpret_cast<uint4 *>(seqB)[v] = b4;
                const uint32_t fw[4] = {f4.x, f4.y, f4.z, f4.w}, bw[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const uint32_t pos = 8 * v + e;
                    const uint32_t idf = (fw[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
                    const uint32_t idb = (bw[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
                    if (pos < n) {
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const uint32_t id = h ? idb : idf;
                            if (id >= n_max) { bad = true; continue; }
                            const uint32_t dc = segdec[id];
                            const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15;
                            if (j >= Mb[b * nmod + i]) { bad = true; continue; }
                            const uint32_t old = atomicOr(&(h ? vB : vF)[id >> 5], 1u << (id & 31));
                            if (old & (1u << (id & 31))) bad = true;
                            else (h ? pofB : pofF)[id] = (uint16_t)pos;
                        }
                    } else if (pos < n_max && (idf != 0xFFFFu || idb != 0xFFFFu)) {
                        bad = true;
                    }
                }
            }
        } else if (laneOn) {
            // explicit orders: every present segment exactly once as F and once as B on this rank
            uint32_t *vF = bmF + r * nw, *vB = bmB + r * nw;
            const uint16_t *row = kp.orders_in + (cand * P + r) * (uint64_t)(2 * n_max);
            for (uint32_t t = 0; t < 2 * n_max && !bad; t++) {
                const uint32_t e = gvalid ? __ldg(&row[t]) : 0xFFFFu;
                if (t >= 2 * n) { if (e != 0xFFFFu) bad = true; continue; }
                const uint32_t id = e & 0x7FFFu, d = e >> 15;
                if (id >= n_max) { bad = true; continue; }
                const uint32_t dc = segdec[id];
                const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15;
                if (j >= Mb[b * nmod + i]) { bad = true; continue; }
                uint32_t *vv = d ? vB : vF;
                if (vv[id >> 5] & (1u << (id & 31))) bad = true;
                vv[id >> 5] |= 1u << (id & 31);
            }
        }
        bad = (__ballot_sync(FULL, bad) & gmask) != 0;
        __syncwarp();
        for (uint32_t w = r; w < 2 * P * nw; w += G) bmF[w] = 0u;   // validation scratch -> ready sets
        for (uint32_t w = r; w < 2 * P; w += G) smF[w] = 0u;
        __syncwarp();

        // ---------------- per-segment cost rows and state
        if (!bad) {
            for (uint32_t s = r; s < n_max; s += G) {
                const uint32_t dc = segdec[s];
                const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15, k = (dc >> 15) & 0xFF;
                const uint32_t Km1 = dc >> 23, q = b * nmod + i, M = Mb[q];
                if (!BUILD) { hF[s] = 0; hB[s] = 0; }          // (BUILD's area has no counters)
                if (j >= M) { slF[s] = 0; slB[s] = 0; rowx[s] = 0; continue; }
                const uint32_t W = wtab[woff[q] + M * (M - 1) / 2 + j];
                rowx[s] = (mi[i].tab_off + W) | ((mi[i].lay_off + k * P) << 12);
                const uint32_t pf = k > 0 ? 1u : Pc[q];
                const uint32_t pbk = (k < Km1 || Cc[q] == 0) ? 1u : Cc[q];
                slF[s] = (uint64_t)((256u - pf) & 0xFFu) << PEND_SHIFT;
                slB[s] = (uint64_t)((256u - pbk) & 0xFFu) << PEND_SHIFT;
                if (BUILD && pf == 0) {      // no predecessor: ready on rank 0 from the start
                    const uint32_t p = pofF[s];
                    atomicOr(&bmF[p >> 5], 1u << (p & 31));
                    atomicOr(&smF[0], 1u << (p >> 5));
                }
            }
        }
        __syncwarp();

        bool dl = false;
        uint64_t tlast = 0, busy = 0;
        uint32_t cur = 0, peak = 0, cnt = 0, fi = 0, bi = 0;
        const uint32_t S2 = 2 * n;
        uint16_t *ordOut = (BUILD && kp.orders_out && laneOn && gvalid)
                               ? kp.orders_out + (cand * P + r) * (uint64_t)(2 * n_max) : nullptr;

        // publication of stage (d, s) on rank r ending at `end`: on an interior rank the next rank's
        // ready time end + p2p goes into the segment's slot (BUILD: and the position into its ready
        // set); on the exit rank the wrap / join accumulators of the successor segments on the entry
        // rank (which add their own p2p). BUILD bookkeeping: when exactly one stage became ready on
        // the ring neighbour in d's direction (forward: r + 1, rank P-1 wraps to rank 0; backward:
        // r - 1, rank 0 wraps to P-1), `aseg` = its segment + 1 and `addv` its ready time -- an ADD
        // event the neighbour folds into its minima in O(1); the loss turnaround readies a backward
        // stage on this rank itself (`selfB` = segment + 1); when several became ready the returned
        // mask asks the entry rank to re-derive (bit 0: rank 0's forwards, bit 1: rank P-1's
        // backwards).
        auto setbit = [&](uint32_t *bm, uint32_t *sm, uint32_t rr, uint32_t p) {
            bm[rr * nw + (p >> 5)] |= 1u << (p & 31);
            sm[rr] |= 1u << (p >> 5);
        };
        auto publish = [&](uint32_t d, uint32_t s, uint64_t end, uint64_t &addv, uint32_t &aseg,
                           uint32_t &selfB) -> uint32_t {
            uint32_t full = 0;
            if (d == 0) {
                if (!BUILD) hF[s] = (uint8_t)(r + 1);
                if (!isLast) {
                    addv = end + tab[rowx[s] & 0xFFFu].w;
                    slF[s] = addv;
                    if (BUILD) { setbit(bmF, smF, r + 1, pofF[s]); aseg = s + 1u; }
                } else {
                    slF[s] = end;
                    const uint32_t dc = segdec[s];
                    const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, k = (dc >> 15) & 0xFF, K = (dc >> 23) + 1;
                    const uint32_t w = tab[rowx[s] & 0xFFFu].w;
                    if (k + 1 < K) {
                        if (wrap_publish(&slF[s + 1], end + w) && BUILD) {
                            setbit(bmF, smF, 0, pofF[s + 1]);
                            aseg = s + 2u;
                            addv = slF[s + 1];
                        }
                    } else if (Cc[b * nmod + i]) {
                        uint32_t nr = 0, last = 0;
                        for (uint32_t c = 0; c < nmod; c++) {
                            if (!((mi[i].cons_mask >> c) & 1u)) continue;
                            const uint32_t Mc = Mb[b * nmod + c];
                            for (uint32_t jc = 0; jc < Mc; jc++) {
                                const uint32_t t2 = sbase[b * nmod + c] + jc * mi[c].K;
                                if (wrap_publish(&slF[t2], end + w) && BUILD) { setbit(bmF, smF, 0, pofF[t2]); nr++; last = t2; }
                            }
                        }
                        if (nr == 1) { aseg = last + 1u; addv = slF[last]; }
                        else if (nr > 1) full |= 1u;
                    } else {                                   // loss turnaround (R-6)
                        if (wrap_publish(&slB[s], end) && BUILD) { setbit(bmB, smB, P - 1, pofB[s]); selfB = s + 1u; }
                    }
                }
            } else {
                if (!BUILD) hB[s] = (uint8_t)(P - r);
                if (!isFirst) {
                    addv = end + tab[rowx[s] & 0xFFFu].w;
                    slB[s] = addv;
                    if (BUILD) { setbit(bmB, smB, r - 1, pofB[s]); aseg = s + 1u; }
                } else {
                    slB[s] = end;
                    const uint32_t dc = segdec[s];
                    const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, k = (dc >> 15) & 0xFF;
                    if (k > 0) {                               // previous chunk, rank P-1 (+ its p2p)
                        if (wrap_publish(&slB[s - 1], end + tab[rowx[s - 1] & 0xFFFu].w) && BUILD) {
                            setbit(bmB, smB, P - 1, pofB[s - 1]);
                            aseg = s;
                            addv = slB[s - 1];
                        }
                    } else {                                   // producers' last chunks (+ their p2p)
                        uint32_t nr = 0, last = 0;
                        for (uint32_t pm = 0; pm < nmod; pm++) {
                            if (!((mi[i].prod_mask >> pm) & 1u)) continue;
                            const uint32_t Mp = Mb[b * nmod + pm];
                            for (uint32_t jp = 0; jp < Mp; jp++) {
                                const uint32_t t2 = sbase[b * nmod + pm] + jp * mi[pm].K + mi[pm].K - 1;
                                if (wrap_publish(&slB[t2], end + tab[rowx[t2] & 0xFFFu].w) && BUILD) {
                                    setbit(bmB, smB, P - 1, pofB[t2]);
                                    nr++;
                                    last = t2;
                                }
                            }
                        }
                        if (nr == 1) { aseg = last + 1u; addv = slB[last]; }
                        else if (nr > 1) full |= 2u;
                    }
                }
            }
            return full;
        };

        if (BUILD) {
            // ---------------- f1: the dual-queue greedy, one stage per step
            bool done = bad || !laneOn || n == 0;
            uint64_t tF = O_INF, tG = O_INF, tB = O_INF;   // min t_start: ungated F, any F, B
            // the second smallest t_start of either queue (duplicates counted), valid while v2 has
            // the direction's bit: removing a queue's minimum then needs no re-derivation
            uint64_t tG2 = O_INF, tB2 = O_INF;
            uint32_t v2 = 0;
            uint32_t need = 3;                             // bit 0: re-derive t_fw / t_gated, bit 1: t_bw
            int last = -1;
            uint32_t fstep = 0;
            auto actOf = [&](uint32_t s) -> uint32_t {
                const uint32_t e = rowx[s];
                return (uint32_t)layers[(e >> 12) + r] * tab[e & 0xFFFu].z;
            };
            // the largest activation of any of this rank's stages: below budget - it, no forward is gated;
            // dlt: a lower bound on (start of any placement here) -> (the ready time it publishes to a
            // neighbour): the shortest stage of this rank plus the smallest p2p of any segment
            uint32_t maxact = 0, dlt = 0;
            if (laneOn && !bad) {
                uint64_t latmin = O_INF;
                uint32_t wmin = 0xFFFFFFFFu;
                for (uint32_t p = 0; p < n; p++) {
                    const uint32_t e = rowx[seqF[p]];
                    const uint4 T = tab[e & 0xFFFu];
                    const uint32_t lay = layers[(e >> 12) + r];
                    const uint32_t a = lay * T.z;
                    maxact = a > maxact ? a : maxact;
                    const uint64_t lt = (uint64_t)lay * (T.x < T.y ? T.x : T.y);
                    latmin = lt < latmin ? lt : latmin;
                    wmin = T.w < wmin ? T.w : wmin;
                }
                const uint64_t d = n ? latmin + wmin : 0;
                dlt = d < O_CAP ? (uint32_t)d : O_CAP;
            }
            // ring neighbours (a forward stage feeds the next rank, the last rank wraps to rank 0, and
            // backward the other way round)
            const int nbl = r == 0 ? (int)P - 1 : r - 1, nbr = r + 1 >= (int)P ? 0 : r + 1;
            const uint32_t *mF = bmF + (laneOn ? r : 0) * nw, *mB = bmB + (laneOn ? r : 0) * nw;
            for (;;) {
                // re-derive the queue minima from the ready bitmaps (a ready stage's slot holds its
                // t_start with a zero pending byte: no masking)
                if ((need & 1u) && !done) {
                    tF = tG = tG2 = O_INF;
                    uint32_t ws = smF[r];
                    if (cur + maxact <= bud) {     // no forward can be gated: t_fw = t_gated
                        while (ws) {
                            const uint32_t w = __ffs(ws) - 1;
                            ws &= ws - 1;
                            uint32_t bits = mF[w];
                            while (bits) {            // two stages per pass: independent load chains
                                const uint32_t p = 32 * w + __ffs(bits) - 1;
                                bits &= bits - 1;
                                const uint32_t q = bits ? 32 * w + __ffs(bits) - 1 : p;
                                bits &= bits - 1;
                                const uint64_t t = slF[seqF[p]], u = slF[seqF[q]];
                                tG2 = t < tG2 ? (t < tG ? tG : t) : tG2;
                                tG = t < tG ? t : tG;
                                if (q != p) {
                                    tG2 = u < tG2 ? (u < tG ? tG : u) : tG2;
                                    tG = u < tG ? u : tG;
                                }
                            }
                        }
                        tF = tG;
                    } else {
                        while (ws) {
                            const uint32_t w = __ffs(ws) - 1;
                            ws &= ws - 1;
                            uint32_t bits = mF[w];
                            while (bits) {
                                const uint32_t p = 32 * w + __ffs(bits) - 1;
                                bits &= bits - 1;
                                const uint32_t s = seqF[p];
                                const uint64_t t = slF[s];
                                tG2 = t < tG2 ? (t < tG ? tG : t) : tG2;
                                tG = t < tG ? t : tG;
                                if (cur + actOf(s) <= bud) tF = t < tF ? t : tF;
                            }
                        }
                    }
                    v2 |= 1u;
                }
                if ((need & 2u) && !done) {
                    tB = tB2 = O_INF;
                    uint32_t ws = smB[r];
                    while (ws) {
                        const uint32_t w = __ffs(ws) - 1;
                        ws &= ws - 1;
                        uint32_t bits = mB[w];
                        while (bits) {                // two stages per pass, as above
                            const uint32_t p = 32 * w + __ffs(bits) - 1;
                            bits &= bits - 1;
                            const uint32_t q = bits ? 32 * w + __ffs(bits) - 1 : p;
                            bits &= bits - 1;
                            const uint64_t t = slB[seqB[p]], u = slB[seqB[q]];
                            tB2 = t < tB2 ? (t < tB ? tB : t) : tB2;
                            tB = t < tB ? t : tB;
                            if (q != p) {
                                tB2 = u < tB2 ? (u < tB ? tB : u) : tB2;
                                tB = u < tB ? u : tB;
                            }
                        }
                    }
                    v2 |= 2u;
                }
                const uint64_t tmin = done ? O_INF : (tF < tB ? tF : tB);
                uint64_t gk = o_group_min<G>(tmin == O_INF ? O_INF : ((tmin << 5) | (uint64_t)r));
                bool relax = false;
                if (G == 32 ? gk == O_INF : __any_sync(FULL, gk == O_INF)) {   // gates only? (R-31)
                    const uint64_t g2 = o_group_min<G>((done || tG == O_INF) ? O_INF : ((tG << 5) | (uint64_t)r));
                    if (gk == O_INF) { gk = g2; relax = true; }
                }
                if (G < 32 || (++fstep & 7) == 0) {
                    const uint32_t alive = __ballot_sync(FULL, !done);
                    if (alive == 0) break;
                    if (gk == O_INF && (alive & gmask)) { dl = true; done = true; }   // unreachable (acyclic)
                }
                // Which ranks place in this step. The serial greedy places on the rank holding the
                // smallest key; a rank may place now as well when no placement that precedes its
                // own in that serial order can reach it. Its inputs come only from its two ring
                // neighbours j, and a neighbour's next placement has a key >= K_j, a lower bound on
                // every key j can still reach: K_j = min(key_j, A_{j-1}, A_{j+1}) with
                // A_i = max(t_last_i, K_i) + dlt_i the earliest ready time rank i can publish (it
                // starts no earlier than its clock or its key). Relaxed O_NIT times from the
                // smallest key (every iterate is a valid bound), rank r places when its key is below
                // both neighbours' bounds. Such ranks are never adjacent, so their placements touch
                // disjoint state; the result is the serial greedy's (the parity tests).
                // (every lane of the warp runs the shuffles: the groups of a warp may differ in relax)
                bool mine = !done && gk != O_INF && (uint32_t)(gk & 31u) == (uint32_t)r;
                {
                    const bool par = !relax && P > 1 && gk != O_INF;
                    const uint64_t g0 = par ? gk >> 5 : 0;
                    const bool live = par && !done && tmin != O_INF;
                    const uint64_t kd = live ? tmin - g0 : 0, td = tlast > g0 ? tlast - g0 : 0;
                    const uint32_t kr = live ? (kd < O_CAP ? (uint32_t)kd : O_CAP) : O_CAP;
                    const uint32_t tr = td < O_CAP ? (uint32_t)td : O_CAP;
                    uint32_t K = 0;
#pragma unroll
                    for (int it = 0; it < O_NIT; it++) {
                        const uint32_t a0 = (tr > K ? tr : K) + dlt;
                        const uint32_t A = done ? O_CAP : (a0 < O_CAP ? a0 : O_CAP);
                        const uint32_t AL = __shfl_sync(FULL, A, nbl, G), AR = __shfl_sync(FULL, A, nbr, G);
                        K = min(kr, min(AL, AR));
                    }
                    const uint32_t KL = __shfl_sync(FULL, K, nbl, G), KR = __shfl_sync(FULL, K, nbr, G);
                    mine = mine || (live && kr < KL && kr < KR);
                }
                __syncwarp();
                uint32_t pl = 0, aF = 0, aB = 0, selfneed = 0;
                uint64_t addv = 0;
                if (mine) {
                    const uint64_t fmin = relax ? tG : tF, bmin = tB;
                    uint32_t dir;
                    if (fmin != O_INF && bmin != O_INF && fmin < tlast && bmin < tlast) dir = last == 0 ? 1u : 0u;
                    else if (fmin == O_INF) dir = 1u;
                    else if (bmin == O_INF) dir = 0u;
                    else dir = bmin <= fmin ? 1u : 0u;
                    const uint64_t td = dir ? bmin : fmin, lim = td > tlast ? td : tlast;
                    const bool nogate = relax || cur + maxact <= bud;
                    // the highest-priority (lowest position) stage starting as early as possible
                    uint32_t *mrow = (dir ? bmB : bmF) + r * nw;
                    uint32_t *msum = (dir ? smB : smF) + r;
                    const uint16_t *seq = dir ? seqB : seqF;
                    const uint64_t *sl = dir ? slB : slF;
                    uint32_t s = 0, pos = 0;
                    uint64_t ts = 0;
                    uint32_t ws = *msum;
                    bool found = false;
                    while (ws && !found) {
                        const uint32_t w = __ffs(ws) - 1;
                        ws &= ws - 1;
                        uint32_t bits = mrow[w];
                        while (bits) {
                            const uint32_t p = 32 * w + __ffs(bits) - 1;
                            bits &= bits - 1;
                            const uint32_t sg = seq[p];
                            const uint64_t t = sl[sg];
                            if (t > lim) continue;
                            if (!dir && !nogate && cur + actOf(sg) > bud) continue;
                            s = sg; pos = p; ts = t; found = true;
                            break;
                        }
                    }
                    const uint32_t wrd = mrow[pos >> 5] & ~(1u << (pos & 31));
                    mrow[pos >> 5] = wrd;
                    if (!wrd) *msum &= ~(1u << (pos >> 5));
                    const uint32_t e = rowx[s];
                    const uint4 T = tab[e & 0xFFFu];
                    const uint32_t lay = layers[(e >> 12) + r];
                    const uint64_t st = ts > tlast ? ts : tlast;
                    const uint64_t end = st + (uint64_t)lay * (dir ? T.y : T.x);
                    busy += end - st;
                    tlast = end;
                    const uint32_t act = lay * T.z;
                    cur = dir ? cur - act : cur + act;
                    peak = cur > peak ? cur : peak;
                    if (ordOut) ordOut[cnt] = (uint16_t)(s | (dir ? 0x8000u : 0u));
                    cnt++;
                    last = (int)dir;
                    done = cnt == S2;
                    uint32_t aseg = 0, selfB = 0;
                    pl = publish(dir, s, end, addv, aseg, selfB);
                    // the placer's own minima: its placed direction lost the stage starting at ts --
                    // the queue's minimum moves to the cached second smallest (then unknown), a stage
                    // at the second smallest makes it unknown, a later one changes nothing; without a
                    // known second the queue is re-derived. t_fw = t_gated while no forward can be
                    // gated (a backward placement only lowers the memory), else the forwards are
                    // re-derived.
                    {
                        uint64_t &m1 = dir ? tB : tG, &m2 = dir ? tB2 : tG2;
                        const uint32_t bit = dir ? 2u : 1u;
                        if (ts == m1) {
                            if (v2 & bit) m1 = m2;
                            else selfneed |= bit;
                            v2 &= ~bit;
                        } else if (ts == m2) {
                            v2 &= ~bit;
                        }
                    }
                    if (cur + maxact <= bud) tF = tG;
                    else selfneed |= 1u;
                    // ONE ready stage for the ring neighbour (segment + 1), and the turnaround's
                    // backward stage on this rank itself
                    if (dir == 0) aF = aseg; else aB = aseg;
                    if (selfB) {
                        const uint64_t v = slB[selfB - 1u];
                        if (v < tB) { tB2 = tB; tB = v; v2 |= 2u; }
                        else if (v < tB2) tB2 = v;
                    }
                }
                __syncwarp();
                {
                    // the placers' news (within the group): lanes to re-derive (wraps reach rank 0 or
                    // P-1 only) and the ADD events from the left (forward) and right (backward)
                    // neighbours, which the target folds into its minima in O(1)
                    const uint32_t w0 = __ballot_sync(FULL, (pl & 1u) != 0) & gmask;
                    const uint32_t wl = __ballot_sync(FULL, (pl & 2u) != 0) & gmask;
                    const uint32_t sF = __shfl_sync(FULL, aF, nbl, G);
                    const uint64_t vF = __shfl_sync(FULL, addv, nbl, G);
                    const uint32_t sB = __shfl_sync(FULL, aB, nbr, G);
                    const uint64_t vB = __shfl_sync(FULL, addv, nbr, G);
                    need = ((isFirst && w0) ? 1u : 0u) | ((isLast && wl) ? 2u : 0u) | selfneed;
                    if (!done) {
                        if (sF && !(need & 1u)) {
                            if (vF < tG) { tG2 = tG; tG = vF; v2 |= 1u; }   // the old minimum is second
                            else if (vF < tG2) tG2 = vF;
                            if (cur + maxact <= bud || cur + actOf(sF - 1u) <= bud) tF = vF < tF ? vF : tF;
                        }
                        if (sB && !(need & 2u)) {
                            if (vB < tB) { tB2 = tB; tB = vB; v2 |= 2u; }
                            else if (vB < tB2) tB2 = vB;
                        }
                    }
                }
            }
        } else {
            // ---------------- TIME: lock-step longest path of explicit per-rank orders (OM 0) or of the
            // record's shared sequences + F/B bits (OM 2)
            const uint16_t *row = OM == 0 ? kp.orders_in + ((gvalid ? cand : 0) * P + (laneOn ? r : 0)) * (uint64_t)(2 * n_max)
                                          : nullptr;
            const uint32_t *wptr = reinterpret_cast<const uint32_t *>(rec + kp.off_fb) + 2 * P + r;   // word 2
            bool done = bad || !laneOn || n == 0;
            uint32_t rnd = 0;
            for (;;) {
                uint32_t d, s;
                if constexpr (OM == 0) {
                    const uint32_t e16 = done ? 0u : __ldg(&row[cnt]);
                    d = e16 >> 15;
                    s = e16 & 0x7FFFu;
                } else {
                    d = (wcur >> (cnt & 31)) & 1u;
                    s = done ? 0u : (d ? seqB[bi] : seqF[fi]);
                }
                bool ready = false;
                uint64_t dep = 0;
                if (!done) {   // the slot holds the ready time (end + p2p, or the wrap / join value)
                    if (d == 0) {
                        const uint64_t v = slF[s];
                        ready = isFirst ? (hF[s] == 0 && (v >> PEND_SHIFT) == 0) : hF[s] == (uint32_t)r;
                        dep = v;
                    } else {
                        const uint64_t v = slB[s];
                        ready = isLast ? (hB[s] == 0 && (v >> PEND_SHIFT) == 0) : hB[s] == P - 1 - (uint32_t)r;
                        dep = v;
                    }
                }
                if ((++rnd & 7) == 0) {
                    const uint32_t prog = __ballot_sync(FULL, ready);
                    const uint32_t alive = __ballot_sync(FULL, !done);
                    if (alive == 0) break;
                    if ((alive & gmask) && !(prog & gmask)) { dl = true; done = true; }   // a cycle
                }
                __syncwarp();
                if (ready && !done) {
                    const uint32_t e = rowx[s];
                    uint64_t lat = (uint64_t)layers[(e >> 12) + r] * (d ? tab[e & 0xFFFu].y : tab[e & 0xFFFu].x);
                    uint32_t act = (uint32_t)layers[(e >> 12) + r] * tab[e & 0xFFFu].z;
                    if (kp.sel) {   // f3 (M4): the stage pair's selected memory-strategy candidate
                        const uint32_t idx = d ? bi : fi;
                        const uint32_t c = kp.sel[((cand * P + r) * 2 + d) * (uint64_t)n_max + idx];
                        const uint4 E = __ldg(&kp.ctab[__ldg(&kp.crow[(e >> 12) + r]) + (int32_t)((e & 0xFFFu) * kp.S + c)]);
                        lat = d ? E.y : E.x;
                        act = E.z;
                    }
                    const uint64_t st = dep > tlast ? dep : tlast;
                    const uint64_t end = st + lat;
                    if (kp.tl_start) {
                        const uint64_t o = (cand * P + r) * (uint64_t)(2 * n_max) + cnt;
                        kp.tl_start[o] = st;
                        kp.tl_end[o] = end;
                    }
                    tlast = end;
                    busy += lat;
                    cur = d ? cur - act : cur + act;
                    peak = cur > peak ? cur : peak;
                    uint64_t addv;
                    uint32_t aseg, selfB;
                    publish(d, s, end, addv, aseg, selfB);
                    if (d) bi++; else fi++;
                    cnt++;
                    if (OM == 2 && (cnt & 31) == 0) {      // next 32 F/B bits (the word after next prefetched)
                        wcur = wnext;
                        if (cnt + 32 < S2) wnext = __ldg(wptr);
                        wptr += P;
                    }
                    done = cnt == S2;
                }
                __syncwarp();
            }
            if (dl && laneOn) {   // deadlocked: finish the order-only memory scan (R-9)
                while (cnt < S2) {
                    uint32_t d, s;
                    if constexpr (OM == 0) {
                        const uint32_t e16 = __ldg(&row[cnt]);
                        d = e16 >> 15;
                        s = e16 & 0x7FFFu;
                    } else {
                        const uint32_t word = __ldg(reinterpret_cast<const uint32_t *>(rec + kp.off_fb) + (cnt >> 5) * P + r);
                        d = (word >> (cnt & 31)) & 1u;
                        s = d ? seqB[bi] : seqF[fi];
                    }
                    const uint32_t e = rowx[s];
                    uint32_t a = (uint32_t)layers[(e >> 12) + r] * tab[e & 0xFFFu].z;
                    if (kp.sel) {
                        const uint32_t idx = d ? bi : fi;
                        const uint32_t c = kp.sel[((cand * P + r) * 2 + d) * (uint64_t)n_max + idx];
                        a = __ldg(&kp.ctab[__ldg(&kp.crow[(e >> 12) + r]) + (int32_t)((e & 0xFFFu) * kp.S + c)]).z;
                    }
                    if (!d) { cur += a; peak = cur > peak ? cur : peak; fi++; }
                    else { cur -= a; bi++; }
                    cnt++;
                }
            }
        }
        // padding of the emitted orders
        if (ordOut) {
            const uint32_t from = bad ? 0u : cnt;
            for (uint32_t t = from; t < 2 * n_max; t++) ordOut[t] = 0xFFFFu;
        }

        // ---------------- results + fused argmin
        const uint64_t mk = o_group_max<G>(tlast);
        const uint64_t bsum = o_group_sum<G>(busy);
        const bool over = laneOn && !bad && peak > bud;
        const uint32_t oom = (__ballot_sync(FULL, over) & gmask) >> (g * G);
        if (gvalid) {
            uint32_t status;
            uint64_t mko;
            double bub;
            if (bad) { status = DIP_CAND_BAD_ENCODING; mko = ~0ull; bub = -1.0; }
            else if (dl) { status = DIP_CAND_DEADLOCK; mko = ~0ull; bub = -1.0; }
            else {
                status = oom ? DIP_CAND_OOM : DIP_CAND_OK;
                mko = mk;
                const uint64_t den = (uint64_t)P * mk;
                bub = den ? (double)(den - bsum) / (double)den : 0.0;
            }
            if (r == 0) {
                dip_result res;
                res.makespan_ns = mko;
                res.status = status;
                res.oom_mask = bad ? 0u : oom;
                res.bubble = bub;
                kp.results[cand] = res;
                if (status == DIP_CAND_OK && kp.fused_key) {
                    const unsigned long long key = ((unsigned long long)mk << kp.idx_bits) | (kp.index_base + cand);
                    best = key < best ? key : best;
                }
            }
            if (kp.peaks && laneOn) kp.peaks[cand * P + r] = bad ? 0u : peak;
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(FULL, best, o);
        best = w < best ? w : best;
    }
    if (lane == 0 && best != ~0ull) atomicMin(kp.best_key, best);
}

template <int G>
static const void *okfun(int om) {
    return om == 1 ? reinterpret_cast<const void *>(&dip_order_kernel<G, 1>)
         : om == 2 ? reinterpret_cast<const void *>(&dip_order_kernel<G, 2>)
                   : reinterpret_cast<const void *>(&dip_order_kernel<G, 0>);
}
static const void *order_kernel_for(int G, int om) {
    switch (G) {
    case 4: return okfun<4>(om);
    case 8: return okfun<8>(om);
    case 16: return okfun<16>(om);
    case 32: return okfun<32>(om);
    default: return nullptr;
    }
}

cudaError_t prepare_order(int G, size_t smem) {
    for (int b = 0; b < 3; b++) {
        const void *f = order_kernel_for(G, b);
        if (!f) return cudaErrorInvalidValue;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t occupancy_order(int G, int block, size_t smem, int *blocks_per_sm) {
    int best = 1 << 30;
    for (int b = 0; b < 3; b++) {
        const void *f = order_kernel_for(G, b);
        if (!f) return cudaErrorInvalidValue;
        int x = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, f, block, smem);
        if (e != cudaSuccess) return e;
        best = x < best ? x : best;
    }
    *blocks_per_sm = best;
    return cudaSuccess;
}

template <int G>
static void launch_og(const KParams &kp, int om, int grid, int block, size_t smem, cudaStream_t s) {
    if (om == 1) dip_order_kernel<G, 1><<<grid, block, smem, s>>>(kp);
    else if (om == 2) dip_order_kernel<G, 2><<<grid, block, smem, s>>>(kp);
    else dip_order_kernel<G, 0><<<grid, block, smem, s>>>(kp);
}

cudaError_t launch_order(const KParams &kp, int G, int om, int grid, int block, size_t smem, cudaStream_t s) {
    switch (G) {
    case 4: launch_og<4>(kp, om, grid, block, smem, s); break;
    case 8: launch_og<8>(kp, om, grid, block, smem, s); break;
    case 16: launch_og<16>(kp, om, grid, block, smem, s); break;
    case 32: launch_og<32>(kp, om, grid, block, smem, s); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace dipk
