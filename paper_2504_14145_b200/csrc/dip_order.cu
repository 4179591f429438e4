// dip_order.cu -- sm_100a kernel for schedules given as per-rank stage orders (SURVEY §8(f) rows
// f1 / f2 / f3 with the dual-queue interleaving of PAPER.md §5.2, reading R-29):
//
//   BUILD  (dip_interleave): from a record's split and forward / backward PRIORITY
//          orders, run DIP's dual-queue greedy -- every rank keeps its ready forward / backward
//          stages as bitmaps over priority positions; per step the group takes the rank with the
//          smallest t_min (REDUX over the lanes), that rank picks the direction (1F1B alternation
//          when both queues are ready before t_last, else the smaller minimum start, ties to the
//          backward) and its highest-priority stage among those starting as early as possible,
//          places it and publishes its end to the consumers' ready sets. Emits every rank's order.
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

// fold `value` into a wrap / join accumulator; true when it became ready (last producer)
__device__ __forceinline__ bool wrap_publish(uint64_t *slot, uint64_t value) {
    const uint64_t old = *slot, c = (old & O_HIGH) | (value & VAL_MASK);
    const uint64_t nv = (c > old ? c : old) + (1ull << PEND_SHIFT);
    *slot = nv;
    return (nv >> PEND_SHIFT) == 0;
}

}  // namespace

template <int G, bool BUILD>
__global__ void __launch_bounds__(256) dip_order_kernel(const KParams kp) {
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
        if (BUILD) {
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
        __syncwarp();

        // ---------------- per-segment cost rows and state
        if (!bad) {
            for (uint32_t s = r; s < n_max; s += G) {
                const uint32_t dc = segdec[s];
                const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15, k = (dc >> 15) & 0xFF;
                const uint32_t Km1 = dc >> 23, q = b * nmod + i, M = Mb[q];
                hF[s] = 0;
                hB[s] = 0;
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

        // publication of stage (d, s) on rank r ending at `end`: the next rank's input, or the
        // wrap / join accumulators of the successor segments on the entry rank. Returns a bitmask
        // of the lanes whose ready sets changed (BUILD sets the bits itself).
        auto publish = [&](uint32_t d, uint32_t s, uint64_t end) -> uint32_t {
            uint32_t touched = 0;
            if (d == 0) {
                hF[s] = (uint8_t)(r + 1);
                slF[s] = end;
                if (!isLast) {
                    if (BUILD) { const uint32_t p = pofF[s]; bmF[(r + 1) * nw + (p >> 5)] |= 1u << (p & 31); }
                    touched |= 1u << (r + 1);
                } else {
                    const uint32_t dc = segdec[s];
                    const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, k = (dc >> 15) & 0xFF, K = (dc >> 23) + 1;
                    const uint32_t w = tab[rowx[s] & 0xFFFu].w;
                    if (k + 1 < K) {
                        if (wrap_publish(&slF[s + 1], end + w) && BUILD) {
                            const uint32_t p = pofF[s + 1];
                            bmF[p >> 5] |= 1u << (p & 31);
                        }
                        touched |= 1u;
                    } else if (Cc[b * nmod + i]) {
                        for (uint32_t c = 0; c < nmod; c++) {
                            if (!((mi[i].cons_mask >> c) & 1u)) continue;
                            const uint32_t Mc = Mb[b * nmod + c];
                            for (uint32_t jc = 0; jc < Mc; jc++) {
                                const uint32_t t2 = sbase[b * nmod + c] + jc * mi[c].K;
                                if (wrap_publish(&slF[t2], end + w) && BUILD) {
                                    const uint32_t p = pofF[t2];
                                    bmF[p >> 5] |= 1u << (p & 31);
                                }
                            }
                        }
                        touched |= 1u;
                    } else {                                   // loss turnaround (R-6)
                        if (wrap_publish(&slB[s], end) && BUILD) {
                            const uint32_t p = pofB[s];
                            bmB[(P - 1) * nw + (p >> 5)] |= 1u << (p & 31);
                        }
                        touched |= 1u << (P - 1);
                    }
                }
            } else {
                hB[s] = (uint8_t)(P - r);
                slB[s] = end;
                if (!isFirst) {
                    if (BUILD) { const uint32_t p = pofB[s]; bmB[(r - 1) * nw + (p >> 5)] |= 1u << (p & 31); }
                    touched |= 1u << (r - 1);
                } else {
                    const uint32_t dc = segdec[s];
                    const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, k = (dc >> 15) & 0xFF;
                    if (k > 0) {                               // previous chunk, rank P-1 (+ its p2p)
                        if (wrap_publish(&slB[s - 1], end + tab[rowx[s - 1] & 0xFFFu].w) && BUILD) {
                            const uint32_t p = pofB[s - 1];
                            bmB[(P - 1) * nw + (p >> 5)] |= 1u << (p & 31);
                        }
                    } else {                                   // producers' last chunks (+ their p2p)
                        for (uint32_t pm = 0; pm < nmod; pm++) {
                            if (!((mi[i].prod_mask >> pm) & 1u)) continue;
                            const uint32_t Mp = Mb[b * nmod + pm];
                            for (uint32_t jp = 0; jp < Mp; jp++) {
                                const uint32_t t2 = sbase[b * nmod + pm] + jp * mi[pm].K + mi[pm].K - 1;
                                if (wrap_publish(&slB[t2], end + tab[rowx[t2] & 0xFFFu].w) && BUILD) {
                                    const uint32_t p = pofB[t2];
                                    bmB[(P - 1) * nw + (p >> 5)] |= 1u << (p & 31);
                                }
                            }
                        }
                    }
                    touched |= 1u << (P - 1);
                }
            }
            return touched;
        };

        if (BUILD) {
            // ---------------- f1: the dual-queue greedy, one stage per step
            bool done = bad || !laneOn || n == 0;
            uint64_t tF = O_INF, tG = O_INF, tB = O_INF;   // min t_start: ungated F, any F, B
            bool need = true;
            int last = -1;
            uint32_t fstep = 0;
            // t_start of ready stage s on this rank
            auto tsF = [&](uint32_t s) -> uint64_t {
                return isFirst ? (slF[s] & VAL_MASK) : slF[s] + tab[rowx[s] & 0xFFFu].w;
            };
            auto tsB = [&](uint32_t s) -> uint64_t {
                return isLast ? (slB[s] & VAL_MASK) : slB[s] + tab[rowx[s] & 0xFFFu].w;
            };
            auto actOf = [&](uint32_t s) -> uint32_t {
                const uint32_t e = rowx[s];
                return (uint32_t)layers[(e >> 12) + r] * tab[e & 0xFFFu].z;
            };
            for (;;) {
                if (need && !done) {        // re-derive the queue minima from the ready bitmaps
                    tF = tG = tB = O_INF;
                    const uint32_t *mF = bmF + r * nw, *mB = bmB + r * nw;
                    for (uint32_t w = 0; w < nw; w++) {
                        uint32_t bits = mF[w];
                        while (bits) {
                            const uint32_t p = 32 * w + __ffs(bits) - 1;
                            bits &= bits - 1;
                            const uint32_t s = seqF[p];
                            const uint64_t t = tsF(s);
                            tG = t < tG ? t : tG;
                            if (cur + actOf(s) <= bud) tF = t < tF ? t : tF;
                        }
                        bits = mB[w];
                        while (bits) {
                            const uint32_t p = 32 * w + __ffs(bits) - 1;
                            bits &= bits - 1;
                            const uint64_t t = tsB(seqB[p]);
                            tB = t < tB ? t : tB;
                        }
                    }
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
                __syncwarp();
                uint32_t pl = 0xFFFFFFFFu, pdir = 0, psg = 0;
                if (!done && gk != O_INF && (uint32_t)(gk & 31u) == (uint32_t)r) {
                    const uint64_t fmin = relax ? tG : tF, bmin = tB;
                    uint32_t dir;
                    if (fmin != O_INF && bmin != O_INF && fmin < tlast && bmin < tlast) dir = last == 0 ? 1u : 0u;
                    else if (fmin == O_INF) dir = 1u;
                    else if (bmin == O_INF) dir = 0u;
                    else dir = bmin <= fmin ? 1u : 0u;
                    const uint64_t td = dir ? bmin : fmin, lim = td > tlast ? td : tlast;
                    // the highest-priority (lowest position) stage starting as early as possible
                    uint32_t *mrow = (dir ? bmB : bmF) + r * nw;
                    const uint16_t *seq = dir ? seqB : seqF;
                    uint32_t s = 0, pos = 0;
                    uint64_t ts = 0;
                    bool found = false;
                    for (uint32_t w = 0; w < nw && !found; w++) {
                        uint32_t bits = mrow[w];
                        while (bits) {
                            const uint32_t p = 32 * w + __ffs(bits) - 1;
                            bits &= bits - 1;
                            const uint32_t sg = seq[p];
                            const uint64_t t = dir ? tsB(sg) : tsF(sg);
                            if (t > lim) continue;
                            if (!dir && !relax && cur + actOf(sg) > bud) continue;
                            s = sg; pos = p; ts = t; found = true;
                            break;
                        }
                    }
                    mrow[pos >> 5] &= ~(1u << (pos & 31));
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
                    pl = publish(dir, s, end) | (1u << r);
                    pdir = dir;
                    psg = s;
                }
                // which lanes must re-derive their minima: the placer and the lanes whose ready sets
                // it changed (a whole-warp group shares the mask through one shuffle)
                __syncwarp();
                if constexpr (G == 32) {
                    const uint32_t who = (uint32_t)(gk & 31u);
                    const uint32_t msk = gk != O_INF ? __shfl_sync(FULL, pl, (int)who) : 0u;
                    need = (msk >> r) & 1u;
                } else {
                    need = true;
                }
                (void)pdir; (void)psg;
            }
        } else {
            // ---------------- TIME: lock-step longest path of explicit per-rank orders
            const uint16_t *row = kp.orders_in + ((gvalid ? cand : 0) * P + (laneOn ? r : 0)) * (uint64_t)(2 * n_max);
            bool done = bad || !laneOn || n == 0;
            uint32_t rnd = 0;
            for (;;) {
                const uint32_t e16 = done ? 0u : __ldg(&row[cnt]);
                const uint32_t d = e16 >> 15, s = e16 & 0x7FFFu;
                bool ready = false;
                uint64_t dep = 0;
                if (!done) {
                    const uint32_t w = tab[rowx[s] & 0xFFFu].w;
                    if (d == 0) {
                        const uint64_t v = slF[s];
                        ready = isFirst ? (hF[s] == 0 && (v >> PEND_SHIFT) == 0) : hF[s] == (uint32_t)r;
                        dep = isFirst ? v : v + w;
                    } else {
                        const uint64_t v = slB[s];
                        ready = isLast ? (hB[s] == 0 && (v >> PEND_SHIFT) == 0) : hB[s] == P - 1 - (uint32_t)r;
                        dep = isLast ? v : v + w;
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
                    publish(d, s, end);
                    if (d) bi++; else fi++;
                    cnt++;
                    done = cnt == S2;
                }
                __syncwarp();
            }
            if (dl && laneOn) {   // deadlocked: finish the order-only memory scan (R-9)
                while (cnt < S2) {
                    const uint32_t e16 = __ldg(&row[cnt]);
                    const uint32_t d = e16 >> 15, s = e16 & 0x7FFFu, e = rowx[s];
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
static const void *okfun(bool build) {
    return build ? reinterpret_cast<const void *>(&dip_order_kernel<G, true>)
                 : reinterpret_cast<const void *>(&dip_order_kernel<G, false>);
}
static const void *order_kernel_for(int G, bool build) {
    switch (G) {
    case 4: return okfun<4>(build);
    case 8: return okfun<8>(build);
    case 16: return okfun<16>(build);
    case 32: return okfun<32>(build);
    default: return nullptr;
    }
}

cudaError_t prepare_order(int G, size_t smem) {
    for (int b = 0; b < 2; b++) {
        const void *f = order_kernel_for(G, b != 0);
        if (!f) return cudaErrorInvalidValue;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t occupancy_order(int G, int block, size_t smem, int *blocks_per_sm) {
    int best = 1 << 30;
    for (int b = 0; b < 2; b++) {
        const void *f = order_kernel_for(G, b != 0);
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
static void launch_og(const KParams &kp, bool build, int grid, int block, size_t smem, cudaStream_t s) {
    if (build) dip_order_kernel<G, true><<<grid, block, smem, s>>>(kp);
    else dip_order_kernel<G, false><<<grid, block, smem, s>>>(kp);
}

cudaError_t launch_order(const KParams &kp, int G, bool build, int grid, int block, size_t smem, cudaStream_t s) {
    switch (G) {
    case 4: launch_og<4>(kp, build, grid, block, smem, s); break;
    case 8: launch_og<8>(kp, build, grid, block, smem, s); break;
    case 16: launch_og<16>(kp, build, grid, block, smem, s); break;
    case 32: launch_og<32>(kp, build, grid, block, smem, s); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace dipk
