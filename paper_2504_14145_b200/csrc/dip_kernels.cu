// dip_kernels.cu -- sm_100a kernels of the DIP candidate-schedule scorer.
//
// One persistent kernel does the whole per-candidate hot path:
//   K1 decode      packed record -> split M_{b,i}, balanced parts (R-2), segment
//                  orders; 128-bit coalesced loads; validation (R-11)
//   K2 cost lookup per stage: layers(i, k*P+r) x T_i[W_j]; the tables
//                  live in shared memory, staged once per CTA by a TMA bulk copy
//   K3 wavefront   longest path over the stage x slot DAG (R-4..R-6), one group of
//                  G lanes per candidate, lane = pipeline rank, lock-step rounds; per-rank
//                  memory running sum / peak and OOM mask (R-9, R-10)
//   K4 argmin      packed (makespan, index) key: register min -> warp shuffle -> atomicMin
//                  (R-15)
// Integer nanoseconds in u64; the bubble (R-16) is one IEEE double division.
//
// Inter-rank dependencies travel through per-rank FIFO channels in shared memory (depth
// RING_D) with an exact spill to global memory when a producer runs more than RING_D
// stages ahead of its consumer, so the lock-step wavefront never blocks on a full channel
// (no false deadlocks: "no lane can progress" <=> the candidate's DAG has a cycle).
//
// The same kernel template serves the §8(f) rows on records: MODE 2 also records every stage's
// start / end (f4's timelines), MODE 3 takes each stage pair's latency and activation from the f3
// candidate table through a per-(candidate, rank, position) selection. Schedules given
// as per-rank orders (f1's dual-queue output) run in dip_order.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "dip_internal.h"

namespace dipk {

// ------------------------------------------------------------------ PTX helpers ----------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ uint4 ldg128(const uint8_t *p) { return __ldg(reinterpret_cast<const uint4 *>(p)); }
__device__ __forceinline__ uint32_t ldg32(const uint8_t *p) { return __ldg(reinterpret_cast<const uint32_t *>(p)); }

template <int G>
__device__ __forceinline__ uint64_t group_max(uint64_t v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        uint64_t w = __shfl_xor_sync(0xffffffffu, v, o, G);
        v = w > v ? w : v;
    }
    return v;
}
template <int G>
__device__ __forceinline__ uint64_t group_min(uint64_t v) {
    if constexpr (G == 32) {   // whole warp: two 32-bit REDUX (high word, then low word among its minima)
        const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
        const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
        const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
        return ((uint64_t)mh << 32) | ml;
    } else {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            uint64_t w = __shfl_xor_sync(0xffffffffu, v, o, G);
            v = w < v ? w : v;
        }
        return v;
    }
}
template <int G>
__device__ __forceinline__ uint64_t group_sum(uint64_t v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

// ------------------------------------------------------------------ the scorer -----------
// Per-position entry (uint2), built at decode:
//   x = tab_index (12 bits) | layer_row << 12 (12 bits) | flags << 24
//   y = consume slot | publish slot << 16, both absolute indices into the wrap table
//       (E_MULTI rows: publish field = SINK + 1 + segment id; the plain store is clamped to SINK)
//       depAll = [F slots (nslotF) | B slots (nslotB) | ZERO | SINK] (compact, host-assigned)
// F rows: rank 0 consumes its wrap slot, rank P-1 publishes end + p2p (chain / join) or, for the
// loss turnaround, end - p2p into the B slot so that the B consumer's uniform "+ p2p" cancels.
// B rows: rank P-1 consumes (+ own p2p), rank 0 publishes end. Rows without a wrap dependency
// consume ZERO (always ready, value 0); rows with nothing to publish write to SINK.
// bits 24-25: signed publish factor s in {-1, 0, +1}: a wrap publication writes end + s * p2p
//   (F chain / join: +1; F loss turnaround: -1, its B consumer adds p2p back; B rows: 0)
constexpr uint32_t E_SPLUS = 1u << 24;
constexpr uint32_t E_SMINUS = 3u << 24;
constexpr uint32_t E_MULTI = 4u << 24;    // several join targets: slower loop (publish slot = SINK + 1 + segment id)
// Wrap slots: value in bits 0..55; bits 56..63 = (256 - producers still to come) mod 256, so a slot is
// ready when its top byte is 0, and a producer publishes with one 64-bit max and one add:
//   slot = max(slot, (slot & HIGH) | value) + (1 << 56)
constexpr uint64_t HIGH_MASK = ~VAL_MASK;





// rare paths kept out of line (a call is never if-converted into the round's common path)
__device__ __noinline__ uint64_t spill_load(const unsigned long long *spill, uint32_t d, uint32_t r, uint32_t P,
                                            uint32_t n_max, uint32_t idx) {
    return spill[(d ? (P + r + 1) : (r - 1)) * n_max + idx];
}
__device__ __noinline__ void spill_keep(unsigned long long *spill, uint32_t d, uint32_t r, uint32_t P,
                                        uint32_t n_max, uint32_t idx, uint64_t v) {
    spill[(d ? (P + r) : r) * n_max + idx - RING_D] = v;
}

// MODE 0: score the given schedules; MODE 2: score and record every stage's start / end (f4);
// MODE 3: score with each stage pair's selected memory strategy (f3)
template <int G, int MODE>
__global__ void __launch_bounds__(768) dip_eval_kernel(const KParams kp) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t blob_bar;
    constexpr int CPG = 32 / G;
    constexpr uint32_t D = RING_D;
    const unsigned FULL = 0xffffffffu;

    // (a1) static tables -> smem, one TMA bulk copy per CTA
    if (threadIdx.x == 0) {
        mbar_init(&blob_bar, 1);
        mbar_expect_tx(&blob_bar, kp.blob_bytes);
        tma_bulk_g2s(smem, kp.blob, kp.blob_bytes, &blob_bar);
    }
    __syncthreads();
    mbar_wait(&blob_bar, 0);

    const ModInfo *mi = reinterpret_cast<const ModInfo *>(smem + kp.b_modinfo);
    const uint32_t *segdec = reinterpret_cast<const uint32_t *>(smem + kp.b_segdec);
    const uint16_t *layers = reinterpret_cast<const uint16_t *>(smem + kp.b_layers);
    const uint4 *tab = reinterpret_cast<const uint4 *>(smem + kp.b_tab);
    const uint32_t *woff = reinterpret_cast<const uint32_t *>(smem + kp.b_woff);
    const uint16_t *wtab = reinterpret_cast<const uint16_t *>(smem + kp.b_wtab);
    const uint16_t *nbi = reinterpret_cast<const uint16_t *>(smem + kp.b_nbi);
    const uint16_t *sbase = reinterpret_cast<const uint16_t *>(smem + kp.b_sbase);
    const uint32_t *budget = reinterpret_cast<const uint32_t *>(smem + kp.b_budget);
    const uint16_t *slotF = reinterpret_cast<const uint16_t *>(smem + kp.b_slotF);   // compact wrap slots
    const uint16_t *slotB = reinterpret_cast<const uint16_t *>(smem + kp.b_slotB);
    const uint32_t nF = kp.nslotF;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / G, r = lane % G;
    const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (g * G));
    const uint32_t P = kp.P, nmod = kp.nmod, nq = kp.m * kp.nmod, n_max = kp.n_max;
    uint8_t *ga = smem + kp.blob_bytes + (size_t)(warp * CPG + g) * kp.g_bytes;
    uint2 *posAll = reinterpret_cast<uint2 *>(ga + kp.g_posF);       // [2][n_max]: F then B
    uint64_t *depAll = reinterpret_cast<uint64_t *>(ga + kp.g_depF0);  // [2][n_max]: depF0 then depBP
    uint64_t *ringAll = reinterpret_cast<uint64_t *>(ga + kp.g_ring);  // [2][P][D]: F rings then B rings
    uint16_t *seqF = reinterpret_cast<uint16_t *>(ga + kp.g_depF0);    // decode scratch (dep region)
    uint16_t *seqB = seqF + kp.n_pad;
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(ga + kp.g_posF);   // validation scratch (pos region)
    uint8_t *Mb = ga + kp.g_bmf;          // M_{b,i}
    uint8_t *Pc = Mb + nq;                // present producer sub-microbatches of (b,i)
    uint8_t *Cc = Pc + nq;                // present consumer sub-microbatches of (b,i)
    const uint64_t slot_id = ((uint64_t)blockIdx.x * kp.warps_per_block + warp) * CPG + g;
    unsigned long long *spill = kp.spill + slot_id * 2ull * P * n_max;   // [2][P][n_max]
    const uint32_t nwords = (n_max + 31) / 32;
    const bool isFirst = r == 0, isLast = r == (int)P - 1, laneOn = r < (int)P;

    unsigned long long best = ~0ull;

    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(kp.counter, (unsigned long long)CPG);
        base = __shfl_sync(FULL, base, 0);
        if (base >= kp.count) break;
        const uint64_t cand = base + g;
        const bool gvalid = cand < kp.count;
        const uint8_t *rec = kp.records + (gvalid ? cand : 0) * (uint64_t)kp.stride;

        // ---------------- K1: decode + validate ----------------
        const uint32_t hdr = ldg32(rec);
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
        nsum = (uint32_t)group_sum<G>(nsum);
        if (nsum != n) bad = true;
        for (uint32_t w = r; w < 2 * nwords; w += G) bitmap[w] = 0;
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
        // sequences: 16-byte loads, copy to smem scratch, check they are permutations of the present ids
        const uint32_t nv = kp.n_pad / 8;
        for (uint32_t v = r; v < nv; v += G) {
            const uint4 f4 = ldg128(rec + kp.off_fwd + 16 * v);
            const uint4 b4 = ldg128(rec + kp.off_bwd + 16 * v);
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
                        const uint32_t old = atomicOr(&bitmap[h * nwords + (id >> 5)], 1u << (id & 31));
                        if (old & (1u << (id & 31))) bad = true;
                    }
                } else if (idf != 0xFFFFu || idb != 0xFFFFu) {
                    bad = true;
                }
            }
        }
        // F/B bit rows: exactly n ones in [0, 2n), zeros beyond
        uint32_t wcur = 0, wnext = 0;
        if (laneOn) {
            const uint32_t lim = 2 * n;
            uint32_t ones = 0;
            for (uint32_t w = 0; w < kp.fbw; w++) {
                const uint32_t word = ldg32(rec + kp.off_fb + 4 * (w * P + r));
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
        bad = (__ballot_sync(FULL, bad) & gmask) != 0;
        __syncwarp();

        // ---------------- K2: per-position cost rows and wrap-edge slots ----------------
        const uint32_t ZS = kp.nslotF + kp.nslotB, SINK = ZS + 1;
        if (!bad) {
            for (uint32_t x = r; x < 2 * n; x += G) {
                const bool hb = x >= n;
                const uint32_t p = hb ? x - n : x;
                const uint32_t s = hb ? seqB[p] : seqF[p];
                const uint32_t dc = segdec[s];
                const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15, k = (dc >> 15) & 0xFF;
                const uint32_t K = (dc >> 23) + 1, q = b * nmod + i, M = Mb[q];
                const uint32_t W = wtab[woff[q] + M * (M - 1) / 2 + j];
                uint32_t ex = (mi[i].tab_off + W) | ((mi[i].lay_off + k * P) << 12);
                uint32_t cs, ps;
                if (!hb) {
                    ex |= E_SPLUS;
                    if (k > 0) cs = slotF[s];                       // previous segment, rank P-1 (R-4)
                    else if (Pc[q]) cs = slotF[s - j * K];          // producer join slot (R-5)
                    else cs = ZS;
                    if (k + 1 < K) ps = slotF[s + 1];
                    else if (Cc[q] == 0) { ps = nF + slotB[s]; ex = (ex & ~(3u << 24)) | E_SMINUS; }   // loss turnaround (R-6)
                    else {
                        uint32_t cmods = 0, c1 = 0;
                        for (uint32_t c = 0; c < nmod; c++)
                            if (((mi[i].cons_mask >> c) & 1u) && Mb[b * nmod + c]) { cmods++; c1 = c; }
                        if (cmods == 1) ps = slotF[sbase[b * nmod + c1]];
                        else { ps = SINK + 1 + s; ex |= E_MULTI; }
                    }
                } else {
                    if (k + 1 < K) cs = nF + slotB[s];              // next segment, rank 0
                    else if (Cc[q]) cs = nF + slotB[s - j * K];     // consumer join slot id(b,i,0,K-1)
                    else cs = nF + slotB[s];                        // turnaround (same rank)
                    if (k > 0) ps = nF + slotB[s - 1];
                    else {
                        uint32_t pmods = 0, p1 = 0;
                        for (uint32_t pp = 0; pp < nmod; pp++)
                            if (((mi[i].prod_mask >> pp) & 1u) && Mb[b * nmod + pp]) { pmods++; p1 = pp; }
                        if (pmods == 0) ps = SINK;
                        else if (pmods == 1) ps = nF + slotB[sbase[b * nmod + p1] + mi[p1].K - 1];
                        else { ps = SINK + 1 + s; ex |= E_MULTI; }
                    }
                }
                posAll[(hb ? n_max : 0) + p] = make_uint2(ex, cs | (ps << 16));
            }
        }
        __syncwarp();
        if (!bad) {   // wrap slots: pending counts in bits 56..63 (seq scratch is dead now)
            for (uint32_t s = r; s < n_max; s += G) {
                const uint32_t dc = segdec[s];
                const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15, k = (dc >> 15) & 0xFF;
                const uint32_t Km1 = dc >> 23, q = b * nmod + i;
                const bool pres = j < Mb[q];
                if (slotF[s] != 0xFFFFu) {
                    uint64_t f0 = 0;
                    if (pres) f0 = (uint64_t)((256u - (k > 0 ? 1u : Pc[q])) & 0xFFu) << PEND_SHIFT;
                    depAll[slotF[s]] = f0;
                }
                if (slotB[s] != 0xFFFFu) {
                    uint64_t bp = 0;
                    if (pres) bp = (uint64_t)((256u - ((k < Km1 || Cc[q] == 0) ? 1u : Cc[q])) & 0xFFu) << PEND_SHIFT;
                    depAll[nF + slotB[s]] = bp;
                }
            }
            if (r == 0) { depAll[ZS] = 0; depAll[SINK] = 0; }
        }
        __syncwarp();

        bool dl = false;
        uint64_t tlast = 0, busy = 0;
        uint32_t cur = 0, peak = 0;
        const uint32_t S2 = 2 * n;
        {   // MODE 0 / 3: score; MODE 2: score and record every stage's start/end
        // ---------------- K3: lock-step wavefront longest path ----------------
        // Per round every lane of the group tries its next slot (F if bit t is 0, else B):
        // dependency value from its producer neighbour's channel ring (or, at rank 0 for F / rank
        // P-1 for B, from a wrap slot), end = max(t_last, dep + p2p) + layers * lat, then publish
        // end into its own channel ring (or read-modify-write a wrap slot). The neighbours' F and B
        // counts travel packed in two shuffles. Exit and cycle checks run every 8th round.
        // Channel rings are [2][D][P] u64 (F rings, then B rings; lane x owns column x).
        bool done = bad || !laneOn || n == 0;
        uint32_t t = 0, cF = 0, cB = 0;          // forward / backward stages placed so far
        uint32_t rnd = 0;
        const uint32_t *wptr = reinterpret_cast<const uint32_t *>(rec + kp.off_fb) + 2 * P + r;   // word 2 of this row
        const uint32_t colIn0 = (uint32_t)r - 1, colIn1 = P * D + r + 1;   // producer columns (F, B)
        const uint32_t colOut0 = (uint32_t)r, colOut1 = P * D + r;         // own columns (F, B)
        const uint32_t wrapBits = (isFirst ? 1u : 0u) | (isLast ? 2u : 0u);   // bit d: consumes dir d via wrap
        const uint32_t wrapPub = (isLast ? 1u : 0u) | (isFirst ? 2u : 0u);    // bit d: publishes dir d via wrap
        for (;;) {
            const uint32_t d = (wcur >> (t & 31)) & 1u;            // 0 = F, 1 = B
            const bool wrapC = (wrapBits >> d) & 1u;
            const bool wrapP = (wrapPub >> d) & 1u;
            // the neighbours' F / B counts, packed in one word: two shuffles (A/B on B200: +1 % 94B,
            // +4 % 12B over four separate shuffles)
            const uint32_t cFB = cF | (cB << 16);
            const uint32_t up = __shfl_up_sync(FULL, cFB, 1, G), dn = __shfl_down_sync(FULL, cFB, 1, G);
            const uint32_t fu = up & 0xFFFFu, bu = up >> 16, fd = dn & 0xFFFFu, bd = dn >> 16;
            const uint32_t idx = d ? cB : cF;
            const uint32_t nb = wrapC ? 0xFFFFu : (d ? bd : fu);                        // producer's count
            // done lanes read the zero row: its wrap-slot fields are in range (a clamped real row's
            // would not be -- rows past n are never written; measured: illegal address)
            const uint2 e = done ? make_uint2(0u, 0u) : posAll[d * n_max + idx];
            const uint32_t ring = (idx & (D - 1)) * P;
            const uint64_t *ca = wrapC ? &depAll[e.y & 0xFFFFu] : &ringAll[ring + (d ? colIn1 : colIn0)];
            uint64_t *pa = wrapP ? &depAll[min(e.y >> 16, SINK)] : &ringAll[ring + (d ? colOut1 : colOut0)];
            const uint4 T = tab[e.x & 0xFFFu];
            const uint32_t lay = layers[((e.x >> 12) & 0xFFFu) + r];
            const uint64_t v = *ca;
            const uint64_t pold = *pa;
            // a ready value has a zero pending byte, so it needs no mask (v < 2^56 <=> high word < 2^24)
            const bool ready = !done && nb > idx && (uint32_t)(v >> 32) < (1u << 24);
            const uint32_t w = (wrapC && !d) ? 0u : T.w;   // rank 0's F wrap slot already holds + p2p
            uint64_t dep = v + w;
            if (ready && !wrapC && idx + D < nb)   // evicted from the channel ring: exact spill copy
                dep = spill_load(spill, d, r, P, n_max, idx) + w;

            // exit / cycle checks every 8th round: a round without progress repeats forever, so the
            // verdict is exact; finished lanes just idle for at most 7 rounds
            if ((++rnd & 7) == 0) {
                const uint32_t prog = __ballot_sync(FULL, ready);
                const uint32_t alive = __ballot_sync(FULL, !done);
                if (alive == 0) break;
                if ((alive & gmask) && !(prog & gmask)) {   // no lane of this group can move: a cycle
                    dl = true;
                    done = true;
                }
            }
            __syncwarp();
            if (ready) {
                uint64_t lat = (uint64_t)lay * (d ? T.y : T.x);
                uint32_t act = lay * T.z;
                if (MODE == 3) {   // f3: the stage pair's selected memory-strategy candidate
                    const uint32_t c = kp.sel[((cand * P + r) * 2 + d) * (uint64_t)n_max + idx];
                    const uint4 E = __ldg(&kp.ctab[__ldg(&kp.crow[((e.x >> 12) & 0xFFFu) + r]) + (int32_t)((e.x & 0xFFFu) * kp.S + c)]);
                    lat = d ? E.y : E.x;
                    act = E.z;
                }
                const uint64_t st = dep > tlast ? dep : tlast;
                const uint64_t end = st + lat;
                tlast = end;
                if (MODE == 2) {
                    const uint64_t o = (cand * P + r) * (uint64_t)(2 * n_max) + t;
                    kp.tl_start[o] = st;
                    kp.tl_end[o] = end;
                }
                busy += lat;
                cur = d ? cur - act : cur + act;
                peak = cur > peak ? cur : peak;
                if (!wrapP) {
                    *pa = end;
                    const uint32_t cc = d ? bu : fd;                       // consumer neighbour's count
                    if (idx >= cc + D)                    // consumer is >= D behind: keep the old entry
                        spill_keep(spill, d, r, P, n_max, idx, pold);
                } else {                                  // rank 0 / P-1: the wrap slot's read-modify-write
                    const int32_t sgn = (int32_t)(e.x << 6) >> 30;             // publish factor -1 / 0 / +1
                    const uint64_t pv = (end + (uint64_t)((int64_t)sgn * (int64_t)T.w)) & VAL_MASK;
                    const uint64_t cand = (pold & HIGH_MASK) | pv;
                    *pa = (cand > pold ? cand : pold) + (1ull << PEND_SHIFT);
                    if (e.x & E_MULTI) {           // several join targets (rare); the plain store hit SINK
                        const uint32_t s = (e.y >> 16) - SINK - 1, dc = segdec[s];
                        const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7;
                        const uint32_t msk = d ? mi[i].prod_mask : mi[i].cons_mask;
                        for (uint32_t c = 0; c < nmod; c++) {
                            if (!((msk >> c) & 1u) || Mb[b * nmod + c] == 0) continue;
                            uint64_t *sl = &depAll[d ? nF + slotB[sbase[b * nmod + c] + mi[c].K - 1] : slotF[sbase[b * nmod + c]]];
                            const uint64_t old = *sl, c2 = (old & HIGH_MASK) | pv;
                            *sl = (c2 > old ? c2 : old) + (1ull << PEND_SHIFT);
                        }
                    }
                }
                if (d) cB++; else cF++;
                t++;
                if ((t & 31) == 0) {                      // next 32 F/B bits: the word after next is prefetched
                    wcur = wnext;
                    if (t + 32 < S2) wnext = __ldg(wptr);
                    wptr += P;
                }
                done = t == S2;
            }
            __syncwarp();
        }
        uint32_t fi = cF, bi = cB;
        // deadlocked candidates: finish the order-only memory scan (R-9)
        if (dl && laneOn) {
            while (t < S2) {
                if ((t & 31) == 0 && t > 0) wcur = ldg32(rec + kp.off_fb + 4 * ((t >> 5) * P + r));
                const bool b1 = (wcur >> (t & 31)) & 1u;
                const uint32_t pi = b1 ? bi++ : fi++;
                const uint2 ee = posAll[(b1 ? n_max : 0) + pi];
                uint32_t a = (uint32_t)layers[((ee.x >> 12) & 0xFFFu) + r] * tab[ee.x & 0xFFFu].z;
                if (MODE == 3) {
                    const uint32_t c = kp.sel[((cand * P + r) * 2 + (b1 ? 1 : 0)) * (uint64_t)n_max + pi];
                    a = __ldg(&kp.ctab[__ldg(&kp.crow[((ee.x >> 12) & 0xFFFu) + r]) + (int32_t)((ee.x & 0xFFFu) * kp.S + c)]).z;
                }
                if (!b1) { cur += a; peak = cur > peak ? cur : peak; }
                else cur -= a;
                t++;
            }
        }

        }

        // ---------------- results + K4 argmin ----------------
        const uint64_t mk = group_max<G>(tlast);
        const uint64_t bsum = group_sum<G>(busy);
        const bool over = r < (int)P && !bad && peak > budget[r < (int)P ? r : 0];
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
            if (kp.peaks && r < (int)P) kp.peaks[cand * P + r] = bad ? 0u : peak;
        }
        __syncwarp();
    }
    // fused argmin epilogue: warp shuffle min, one atomicMin per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(FULL, best, o);
        best = w < best ? w : best;
    }
    if (lane == 0 && best != ~0ull) atomicMin(kp.best_key, best);
}

// exact fallback argmin when the packed key could overflow: pass 1 min makespan
__global__ void scan_min_makespan(const dip_result *res, uint64_t count, unsigned long long *mk_out) {
    unsigned long long best = ~0ull;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < count; x += (uint64_t)gridDim.x * blockDim.x)
        if (res[x].status == DIP_CAND_OK && res[x].makespan_ns < best) best = res[x].makespan_ns;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, best, o);
        best = w < best ? w : best;
    }
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(mk_out, best);
}
// pass 2: min index among candidates with that makespan
__global__ void scan_min_index(const dip_result *res, uint64_t count, uint64_t index_base,
                               const unsigned long long *mk_in, unsigned long long *idx_out) {
    const unsigned long long target = *mk_in;
    unsigned long long best = ~0ull;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < count; x += (uint64_t)gridDim.x * blockDim.x)
        if (res[x].status == DIP_CAND_OK && res[x].makespan_ns == target && index_base + x < best) best = index_base + x;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, best, o);
        best = w < best ? w : best;
    }
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(idx_out, best);
}
// per-GPU key (makespan << idx_bits | local) -> cross-rank key (makespan, rank, local)
__global__ void make_gkey(const unsigned long long *key, unsigned long long *gkey, uint32_t idx_bits, uint32_t ibits,
                          uint32_t rbits, uint32_t rank) {
    const unsigned long long k = *key;
    if (k == ~0ull) { *gkey = ~0ull; return; }
    const unsigned long long mk = k >> idx_bits, local = k & ((1ull << idx_bits) - 1);
    *gkey = (mk << (rbits + ibits)) | ((unsigned long long)rank << ibits) | local;
}

template <int G>
static cudaError_t launch_g(const KParams &kp, int grid, int block, size_t smem, cudaStream_t s) {
    if (kp.tl_start) dip_eval_kernel<G, 2><<<grid, block, smem, s>>>(kp);
    else if (kp.sel) dip_eval_kernel<G, 3><<<grid, block, smem, s>>>(kp);
    else dip_eval_kernel<G, 0><<<grid, block, smem, s>>>(kp);
    return cudaGetLastError();
}

cudaError_t launch_eval(const KParams &kp, int G, int grid, int block, size_t smem, cudaStream_t s) {
    switch (G) {
    case 4: return launch_g<4>(kp, grid, block, smem, s);
    case 8: return launch_g<8>(kp, grid, block, smem, s);
    case 16: return launch_g<16>(kp, grid, block, smem, s);
    case 32: return launch_g<32>(kp, grid, block, smem, s);
    default: return cudaErrorInvalidValue;
    }
}

template <int G, int MODE>
static const void *kfun() { return reinterpret_cast<const void *>(&dip_eval_kernel<G, MODE>); }
static const void *kernel_for(int G, int mode) {
    switch (G * 4 + mode) {
    case 16: return kfun<4, 0>();
    case 18: return kfun<4, 2>();
    case 19: return kfun<4, 3>();
    case 32: return kfun<8, 0>();
    case 34: return kfun<8, 2>();
    case 35: return kfun<8, 3>();
    case 64: return kfun<16, 0>();
    case 66: return kfun<16, 2>();
    case 67: return kfun<16, 3>();
    case 128: return kfun<32, 0>();
    case 130: return kfun<32, 2>();
    case 131: return kfun<32, 3>();
    default: return nullptr;
    }
}

cudaError_t prepare_eval(int G, size_t smem) {
    for (int mode = 0; mode < 4; mode++) {
        if (mode == 1) continue;   // (mode 1, the old in-order f1, lives in dip_order.cu now)
        const void *f = kernel_for(G, mode);
        if (!f) return cudaErrorInvalidValue;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t occupancy_eval(int G, int block, size_t smem, int *blocks_per_sm) {
    int best = 1 << 30;
    for (int mode = 0; mode < 1; mode++) {   // the scorer sets the shape; modes 2, 3 reuse it
        const void *f = kernel_for(G, mode);
        if (!f) return cudaErrorInvalidValue;
        int b = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, f, block, smem);
        if (e != cudaSuccess) return e;
        best = b < best ? b : best;
    }
    *blocks_per_sm = best;
    return cudaSuccess;
}

cudaError_t launch_scan_argmin(const dip_result *res, uint64_t count, uint64_t /*index_base*/,
                               unsigned long long *mk_out, unsigned long long * /*idx_out*/, cudaStream_t s) {
    scan_min_makespan<<<592, 256, 0, s>>>(res, count, mk_out);
    return cudaGetLastError();
}
cudaError_t launch_scan_argmin_idx(const dip_result *res, uint64_t count, uint64_t index_base,
                                   const unsigned long long *mk_in, unsigned long long *idx_out, cudaStream_t s) {
    scan_min_index<<<592, 256, 0, s>>>(res, count, index_base, mk_in, idx_out);
    return cudaGetLastError();
}
cudaError_t launch_make_gkey(const unsigned long long *key, unsigned long long *gkey, uint32_t idx_bits,
                             uint32_t ibits, uint32_t rbits, uint32_t rank, cudaStream_t s) {
    make_gkey<<<1, 1, 0, s>>>(key, gkey, idx_bits, ibits, rbits, rank);
    return cudaGetLastError();
}

}  // namespace dipk
