// dip_memopt.cu -- SURVEY §8(f) row f3: DIP's per-layer memory optimisation (§5.3,
// P:550-590) on sm_100a. Two kernels:
//
//  * dip_mcand_kernel (readings R-37/R-38): the <= S strategy candidates of every stage
//    pair type (module i, layers per chunk l, width W) -- one thread per (type, W) enumerates the
//    strategy-count vectors of the l identical layers (the exact multiple-choice knapsack), keeps
//    the fastest, the most memory-efficient and the fastest of each of the S-2 memory buckets,
//    drops duplicates / dominated entries and sorts by memory. Runs once per menu.
//  * dip_memopt_kernel (R-39): the per-rank selection for a batch of schedules -- one
//    warp per (schedule, rank). The warp rebuilds the rank's order from the record (forward
//    position p -> its point range [p, e_p) over the rank's forward slots, e_p = slot of the
//    pair's backward - its backward position), builds the slack profile of candidate 0 with a
//    difference array + warp scan, then runs the greedy: every lane proposes its best pair
//    (largest latency saving per KiB, ties to the lower p, as a 32-bit key built from the host's
//    exact ranking of all steps of the candidate table), one REDUX picks the winner, and only
//    then is the winner's step checked against the range minimum of the slack (lanes over its
//    points): if it fits the lanes subtract it, else the pair is blocked for good (the slack never
//    grows), which makes this lazy order pick exactly the oracle's "best feasible pair".
//    17 B of shared memory per segment (32 warps/SM for 94B). Output: sel[x][r][0][p] / [1][q].
//  The re-timing with the selected candidates (M4) is the scorer's MODE 3 (dip_kernels.cu).
#include <cstdint>

#include "dip_internal.h"

namespace dipk {

namespace {

__device__ __forceinline__ uint32_t ldg32u(const uint8_t *p) { return __ldg(reinterpret_cast<const uint32_t *>(p)); }

struct MC { unsigned long long f, b, mem; };

__device__ __forceinline__ bool mc_before(const MC &a, const MC &b, bool by_mem) {
    const unsigned long long la = a.f + a.b, lb = b.f + b.b;
    if (by_mem) {
        if (a.mem != b.mem) return a.mem < b.mem;
        if (la != lb) return la < lb;
    } else {
        if (la != lb) return la < lb;
        if (a.mem != b.mem) return a.mem < b.mem;
    }
    return a.f < b.f;
}

// ---- M3b / M3c helpers (one warp per (schedule, rank); all control is warp-uniform)
__device__ __forceinline__ unsigned __int128 warp_sum_u128(unsigned __int128 v) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o), hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
        const unsigned long long s = lo + lo2;
        hi = hi + hi2 + (s < lo ? 1ull : 0ull);
        lo = s;
    }
    return ((unsigned __int128)hi << 64) | lo;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int ILP_SHIFT = 16;   // mu = mu_int / 2^16 (the oracle's fixed point)

// D(mu) = sum over free pairs p >= nfix of c_p * memory of argmin_c (lat_c * 2^16 + mu * c_p * mem_c)
// (ties: the earlier = smaller-memory candidate), V(mu) = sum of the minima; warp-summed, exact
__device__ __forceinline__ void ilp_eval(const uint4 *__restrict__ ctab, const uint16_t *cbr, const uint8_t *cn,
                                         const uint32_t *cpa, uint32_t S, uint32_t n, uint32_t nfix,
                                         unsigned long long mu, bool wantV, unsigned long long *D,
                                         unsigned __int128 *V) {
    unsigned long long d = 0;
    unsigned __int128 v = 0;
    for (uint32_t p = nfix + (threadIdx.x & 31); p < n; p += 32) {
        const uint32_t cb = (uint32_t)cbr[p] * S, cnt = (cn[p] >> 4) + 1u;
        const unsigned long long cp = cpa[p];
        unsigned __int128 best = 0;
        unsigned long long bm = 0;
        for (uint32_t c = 0; c < cnt; c++) {
            const uint4 E = __ldg(&ctab[cb + c]);
            const unsigned __int128 x = ((unsigned __int128)((unsigned long long)E.x + E.y) << ILP_SHIFT) +
                                        (unsigned __int128)mu * (cp * E.z);
            if (c == 0 || x < best) { best = x; bm = E.z; }
        }
        d += cp * bm;
        v += best;
    }
    *D = warp_sum_u64(d);
    if (wantV) *V = warp_sum_u128(v);
}

__device__ __forceinline__ unsigned long long ilp_L(const uint4 *__restrict__ ctab, const uint16_t *cbr, const uint8_t *cn,
                                                    const uint32_t *cpa, uint32_t S, uint32_t n, uint32_t nfix,
                                                    unsigned long long mu, long long R, unsigned long long fixed) {
    unsigned long long D;
    unsigned __int128 V;
    ilp_eval(ctab, cbr, cn, cpa, S, n, nfix, mu, true, &D, &V);
    const unsigned __int128 take = (unsigned __int128)mu * (unsigned long long)R;
    if (V <= take) return fixed;
    const unsigned __int128 num = V - take;
    return fixed + (unsigned long long)(num >> ILP_SHIFT) + ((num & ((1u << ILP_SHIFT) - 1)) ? 1ull : 0ull);
}

// M3b: the Lagrangian bound with pairs < nfix fixed (their latency summed in `fixed`, their memory
// taken out of R = sum over K* of (budget - fixed memory live there)); mu bracketed by x16 steps and
// bisected to 1/64 relative width exactly as the oracle (same integer sequence, so the same bound)
__device__ unsigned long long ilp_bound(const uint4 *__restrict__ ctab, const uint16_t *cbr, const uint8_t *cn,
                                        const uint32_t *cpa, uint32_t S, uint32_t n, uint32_t nfix, long long R,
                                        unsigned long long fixed) {
    unsigned long long D;
    unsigned __int128 V;
    ilp_eval(ctab, cbr, cn, cpa, S, n, nfix, 0ull, false, &D, &V);
    if ((long long)D <= R) return ilp_L(ctab, cbr, cn, cpa, S, n, nfix, 0ull, R, fixed);
    unsigned long long lo = 0, hi = 1;
    for (int it = 0; it < 16; it++) {
        ilp_eval(ctab, cbr, cn, cpa, S, n, nfix, hi, false, &D, &V);
        if ((long long)D <= R) break;
        lo = hi;
        hi *= 16;
    }
    while (hi - lo > 1 && hi - lo > (hi >> 6)) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        ilp_eval(ctab, cbr, cn, cpa, S, n, nfix, mid, false, &D, &V);
        if ((long long)D <= R) hi = mid; else lo = mid;
    }
    const unsigned long long a = ilp_L(ctab, cbr, cn, cpa, S, n, nfix, lo, R, fixed);
    const unsigned long long b = ilp_L(ctab, cbr, cn, cpa, S, n, nfix, hi, R, fixed);
    return a > b ? a : b;
}

__device__ __forceinline__ bool ilp_within(unsigned long long bound, unsigned long long inc, uint32_t gap_pm) {
    return (unsigned __int128)bound * 1000u >= (unsigned __int128)inc * (1000u - gap_pm);
}

}  // namespace

constexpr int MAX_S = 16;
constexpr int MAX_STRAT = 8;

__global__ void __launch_bounds__(128) dip_mcand_kernel(const MCandParams p) {
    const uint32_t item = blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= p.n_items) return;
    uint32_t t = 0;
    while (t + 1 < p.n_types && p.t_item[t + 1] <= item) t++;
    const uint32_t W = item - p.t_item[t], L = p.t_lay[t], C = p.n_strat, S = p.S;
    const uint32_t col = p.t_toff[t] + W;
    uint4 *out = p.ctab + p.t_base[t] + (size_t)W * S;
    if (L == 0) {   // a chunk without layers: one empty candidate
        out[0] = make_uint4(0u, 0u, 0u, 1u);
        for (uint32_t c = 1; c < S; c++) out[c] = make_uint4(0u, 0u, 0u, 1u);
        return;
    }
    uint32_t fv[MAX_STRAT], bv[MAX_STRAT], av[MAX_STRAT];
    for (uint32_t c = 0; c < C; c++) {
        fv[c] = __ldg(&p.mf[(size_t)c * p.T + col]);
        bv[c] = __ldg(&p.mb[(size_t)c * p.T + col]);
        av[c] = __ldg(&p.ma[(size_t)c * p.T + col]);
    }
    // every count vector (n_0 .. n_{C-1}), sum L, in odometer order over the first C-1 counts
    MC fast{0, 0, 0}, small{0, 0, 0}, bb[MAX_S];
    bool have[MAX_S];
    for (int u = 0; u < MAX_S; u++) have[u] = false;
    for (int pass = 0; pass < 2; pass++) {
        unsigned long long span = 0;
        if (pass == 1) {
            if (!(S > 2 && fast.mem > small.mem)) break;
            span = fast.mem - small.mem;
        }
        uint32_t cnt[MAX_STRAT];
        for (uint32_t c = 0; c < C; c++) cnt[c] = 0;
        bool first = true;
        for (;;) {
            uint32_t used = 0;
            for (uint32_t c = 0; c + 1 < C; c++) used += cnt[c];
            if (used <= L) {
                cnt[C - 1] = L - used;
                MC x{0, 0, 0};
                for (uint32_t c = 0; c < C; c++) {
                    x.f += (unsigned long long)cnt[c] * fv[c];
                    x.b += (unsigned long long)cnt[c] * bv[c];
                    x.mem += (unsigned long long)cnt[c] * av[c];
                }
                if (pass == 0) {
                    if (first) { fast = x; small = x; first = false; }
                    else {
                        if (mc_before(x, fast, false)) fast = x;
                        if (mc_before(x, small, true)) small = x;
                    }
                } else if (x.mem < fast.mem) {
                    // bucket u: [small + floor(span u / (S-2)), small + floor(span (u+1) / (S-2)))
                    const unsigned long long d = x.mem - small.mem;
                    const uint32_t u = (uint32_t)(((d + 1) * (S - 2) - 1) / span);
                    if (!have[u] || mc_before(x, bb[u], false)) { bb[u] = x; have[u] = true; }
                }
            }
            uint32_t c = 0;
            while (c + 1 < C) {
                if (++cnt[c] <= L) break;
                cnt[c] = 0;
                c++;
            }
            if (c + 1 >= C) break;
        }
    }
    MC pick[MAX_S + 2];
    uint32_t np = 0;
    pick[np++] = fast;
    pick[np++] = small;
    if (S > 2 && fast.mem > small.mem)
        for (uint32_t u = 0; u < S - 2; u++)
            if (have[u]) pick[np++] = bb[u];
    uint32_t k = 0;
    for (uint32_t x = 0; x < np; x++) {
        bool drop = false;
        for (uint32_t y = 0; y < np && !drop; y++) {
            if (y == x) continue;
            const unsigned long long lx = pick[x].f + pick[x].b, ly = pick[y].f + pick[y].b;
            const bool same = pick[y].f == pick[x].f && pick[y].b == pick[x].b && pick[y].mem == pick[x].mem;
            if (same && y < x) drop = true;
            if (!same && pick[y].mem <= pick[x].mem && ly <= lx && (pick[y].mem < pick[x].mem || ly < lx)) drop = true;
        }
        if (!drop) pick[k++] = pick[x];
    }
    for (uint32_t x = 1; x < k; x++)
        for (uint32_t y = x; y > 0 && pick[y].mem < pick[y - 1].mem; y--) {
            const MC tmp = pick[y];
            pick[y] = pick[y - 1];
            pick[y - 1] = tmp;
        }
    for (uint32_t c = 0; c < S; c++) {
        const MC &v = pick[c < k ? c : 0];
        out[c] = c < k ? make_uint4((uint32_t)v.f, (uint32_t)v.b, (uint32_t)v.mem, k) : make_uint4(0u, 0u, 0u, k);
    }
}

// ------------------------------------------------------------------------------------------------
// per (schedule, rank) selection: one warp each, persistent over an atomic work counter
__global__ void __launch_bounds__(128) dip_memopt_kernel(const KParams kp, uint8_t *sel_out, uint32_t warp_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const unsigned FULL = 0xffffffffu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t P = kp.P, nmod = kp.nmod, nq = kp.m * kp.nmod, n_max = kp.n_max, S = kp.S;
    const ModInfo *mi = reinterpret_cast<const ModInfo *>(kp.blob + kp.b_modinfo);
    const uint32_t *segdec = reinterpret_cast<const uint32_t *>(kp.blob + kp.b_segdec);
    const uint32_t *woff = reinterpret_cast<const uint32_t *>(kp.blob + kp.b_woff);
    const uint16_t *wtab = reinterpret_cast<const uint16_t *>(kp.blob + kp.b_wtab);
    const uint16_t *nbi = reinterpret_cast<const uint16_t *>(kp.blob + kp.b_nbi);
    const uint32_t *budget = reinterpret_cast<const uint32_t *>(kp.blob + kp.b_budget);

    uint8_t *wa = smem + (size_t)warp * warp_bytes;
    int32_t *slack = reinterpret_cast<int32_t *>(wa);                      // [n_max] (|values| < 2^31: host guard)
    uint32_t *key = reinterpret_cast<uint32_t *>(wa + 4 * ((n_max + 1) & ~1u));  // [n_max] next step's key
    uint32_t *dms = key + n_max;                                            // [n_max] next step's KiB
    uint16_t *fw = reinterpret_cast<uint16_t *>(key);                       // decode scratch, dead before key is
    uint16_t *invB = fw + n_max;                                            //   written: forward sequence,
    uint16_t *bsl = invB + n_max;                                           //   segment -> backward position,
                                                                            //   slot of the q-th backward
    uint16_t *cbr = reinterpret_cast<uint16_t *>(dms + n_max);              // [n_max] ctab row / S of pair p
    uint16_t *eP = cbr + n_max;                                             // end of pair p's point range
    uint8_t *cn = reinterpret_cast<uint8_t *>(eP + n_max);                  // selected candidate | (count-1) << 4
    uint8_t *Mb = cn + n_max;                                               // [nq]
    uint32_t *bmx = reinterpret_cast<uint32_t *>(                           // [n_max / 32] max of each
        (reinterpret_cast<uintptr_t>(Mb + nq) + 3) & ~(uintptr_t)3);        //   32 keys (warm start)

    const int32_t INF = 0x7FFFFFFF;
    for (;;) {
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(kp.counter, 1ull);
        item = __shfl_sync(FULL, item, 0);
        if (item >= kp.count * P) break;
        const uint64_t x = item / P;
        const uint32_t r = (uint32_t)(item - x * P);
        const uint8_t *rec = kp.records + x * (uint64_t)kp.stride;
        uint8_t *selF = sel_out + (x * P + r) * 2ull * n_max, *selB = selF + n_max;

        // ---- decode (necessary conditions of a valid record; the scorer makes the verdict)
        const uint32_t hdr = ldg32u(rec);
        const uint32_t n = hdr & 0xFFFFu;
        bool bad = (hdr >> 16) != 0 || n > n_max;
        uint32_t nsum = 0;
        for (uint32_t q = lane; q < nq && !bad; q += 32) {
            const uint32_t b = q / nmod, i = q - b * nmod;
            const uint32_t N = __ldg(&nbi[q]), Mx = __ldg(&mi[i].max_split);
            uint32_t M;
            if (Mx > 1) {
                const uint32_t nib = b * kp.nsplit + __ldg(&mi[i].nib_slot);
                M = (__ldg(rec + kp.off_nib + (nib >> 1)) >> ((nib & 1) * 4)) & 15u;
            } else {
                M = N > 0 ? 1u : 0u;
            }
            if ((N == 0) != (M == 0) || M > (N < Mx ? N : Mx)) bad = true;
            Mb[q] = (uint8_t)M;
            nsum += M * __ldg(&mi[i].K);
        }
        for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(FULL, nsum, o);
        if (nsum != n) bad = true;
        bad = __any_sync(FULL, bad);
        const uint16_t *orow = kp.orders_in ? kp.orders_in + (x * P + r) * (uint64_t)(2 * n_max) : nullptr;
        if (!bad && orow) {
            // explicit per-rank orders (f1's output): the p-th forward's segment, each segment's
            // backward position q and the slot of the q-th backward, by warp ballots over the row
            for (uint32_t p = lane; p < n_max; p += 32) invB[p] = 0xFFFFu;
            __syncwarp();
            uint32_t nF = 0, nB = 0;
            const uint32_t below = (1u << lane) - 1u;
            for (uint32_t t0 = 0; t0 < 2 * n; t0 += 32) {
                const uint32_t t = t0 + lane;
                const uint32_t e = t < 2 * n ? __ldg(&orow[t]) : 0xFFFFu;
                const bool isB = t < 2 * n && (e & 0x8000u), isF = t < 2 * n && !(e & 0x8000u);
                const uint32_t bF = __ballot_sync(FULL, isF), bB = __ballot_sync(FULL, isB), sg = e & 0x7FFFu;
                if (isF) {
                    const uint32_t p = nF + __popc(bF & below);
                    if (p < n_max && sg < n_max) fw[p] = (uint16_t)sg;
                    else bad = true;
                }
                if (isB) {
                    const uint32_t q = nB + __popc(bB & below);
                    if (q < n_max && sg < n_max) { invB[sg] = (uint16_t)q; bsl[q] = (uint16_t)t; }
                    else bad = true;
                }
                nF += __popc(bF);
                nB += __popc(bB);
            }
            if (nF != n || nB != n) bad = true;
            bad = __any_sync(FULL, bad);
            __syncwarp();
        } else if (!bad) {
            for (uint32_t p = lane; p < n_max; p += 32) {
                fw[p] = __ldg(reinterpret_cast<const uint16_t *>(rec + kp.off_fwd) + p);
                invB[p] = 0xFFFFu;
            }
            __syncwarp();
            for (uint32_t q = lane; q < n; q += 32) {
                const uint32_t s = __ldg(reinterpret_cast<const uint16_t *>(rec + kp.off_bwd) + q);
                if (s >= n_max) bad = true;
                else invB[s] = (uint16_t)q;
            }
            // the rank's bit row: slot of every backward stage (prefix popcounts across lanes)
            uint32_t carry = 0;
            for (uint32_t w0 = 0; w0 < kp.fbw; w0 += 32) {
                const uint32_t w = w0 + lane;
                uint32_t word = 0;
                if (w < kp.fbw) {
                    word = ldg32u(rec + kp.off_fb + 4 * (w * P + r));
                    const uint32_t lim = 2 * n;
                    if (32 * w >= lim) word = 0;
                    else if (32 * w + 32 > lim) word &= (1u << (lim - 32 * w)) - 1u;
                }
                const uint32_t pc = __popc(word);
                uint32_t incl = pc;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += v;
                }
                uint32_t q = carry + incl - pc;
                while (word) {
                    const uint32_t bit = __ffs(word) - 1;
                    word &= word - 1;
                    if (q < n_max) bsl[q] = (uint16_t)(32 * w + bit);
                    q++;
                }
                carry += __shfl_sync(FULL, incl, 31);
            }
            if (carry != n) bad = true;
            bad = __any_sync(FULL, bad);
            __syncwarp();
        }
        if (!bad) {   // pairs: range, candidate row, candidate 0's memory in the difference array
            for (uint32_t k = lane; k < n; k += 32) slack[k] = 0;
            __syncwarp();
            for (uint32_t p = lane; p < n; p += 32) {
                const uint32_t s = fw[p];
                const uint32_t q = s < n_max ? invB[s] : 0xFFFFu;
                if (q == 0xFFFFu) { bad = true; continue; }
                const uint32_t e = (uint32_t)bsl[q] - q;
                eP[p] = (uint16_t)e;
                const uint32_t dc = __ldg(&segdec[s]);
                const uint32_t b = dc & 0xFF, i = (dc >> 8) & 7, j = (dc >> 11) & 15, k = (dc >> 15) & 0xFF;
                const uint32_t qq = b * nmod + i, M = Mb[qq];
                const uint32_t W = __ldg(&wtab[__ldg(&woff[qq]) + M * (M - 1) / 2 + j]);
                const int32_t row = __ldg(&kp.crow[__ldg(&mi[i].lay_off) + k * P + r]) + (int32_t)((__ldg(&mi[i].tab_off) + W) * S);
                cbr[p] = (uint16_t)((uint32_t)row / S);   // rows are S-aligned; < 65536 rows (host guard)
                const uint4 E = __ldg(&kp.ctab[row]);
                cn[p] = (uint8_t)((E.w - 1u) << 4);      // candidate 0, E.w candidates (1..16)
                if (e > p) {
                    atomicAdd(&slack[p], (int32_t)E.z);
                    if (e < n) atomicSub(&slack[e], (int32_t)E.z);
                }
            }
            bad = __any_sync(FULL, bad);
            __syncwarp();
        }
        if (bad) {
            for (uint32_t p = lane; p < 2 * n_max; p += 32) selF[p] = 0;
            continue;
        }
        // prefix sum -> slack = budget - used at every forward slot
        const int32_t bud = (int32_t)__ldg(&budget[r]);
        bool feasible = true;
        {
            int32_t run = 0;
            for (uint32_t k0 = 0; k0 < n; k0 += 32) {
                const uint32_t k = k0 + lane;
                int32_t v = k < n ? slack[k] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t u = __shfl_up_sync(FULL, v, o);
                    if (lane >= o) v += u;
                }
                if (k < n) {
                    slack[k] = bud - (run + v);
                    if (slack[k] < 0) feasible = false;
                }
                run += __shfl_sync(FULL, v, 31);
            }
            feasible = __all_sync(FULL, feasible);
            __syncwarp();
        }
        if (feasible) {
            // key[p] = (0xFFFF - rank of pair p's next step) << 16 | (0xFFFF - p), 0 = none left:
            // the host ranks every step of the candidate table by its exact latency saving per KiB
            // (equal ratios share a rank), so the warp max of the keys is the oracle's choice --
            // largest ratio, ties to the lower p -- in one REDUX instead of a cross-multiplied
            // shuffle tournament
            for (uint32_t p = lane; p < n; p += 32) {
                uint32_t k = 0, dm = 0;
                if ((cn[p] >> 4) > 0) {
                    const uint32_t cb = (uint32_t)cbr[p] * S;
                    k = ((0xFFFFu - (uint32_t)__ldg(&kp.srank[cb])) << 16) | (0xFFFFu - p);
                    dm = __ldg(&kp.ctab[cb + 1]).z - __ldg(&kp.ctab[cb]).z;
                }
                key[p] = k;
                dms[p] = dm;
            }
            __syncwarp();
            // the max of every 32 keys, so that the argmax reads n / 32 words instead of n
            const uint32_t nb = (n + 31) >> 5;
            for (uint32_t b = 0; b < nb; b++) {
                const uint32_t v = __reduce_max_sync(FULL, 32 * b + lane < n ? key[32 * b + lane] : 0u);
                if (lane == 0) bmx[b] = v;
            }
            __syncwarp();
            for (;;) {
                // the best pair not yet known to be blocked; its feasibility is checked only now
                // (lazily): a pair whose step does not fit is blocked for good (the slack never grows)
                uint32_t bm = 0;
                for (uint32_t b = lane; b < nb; b += 32) bm = max(bm, bmx[b]);
                const uint32_t best = __reduce_max_sync(FULL, bm);
                if (best == 0) break;
                const uint32_t a0 = 0xFFFFu - (best & 0xFFFFu), a1 = eP[a0], bdm = dms[a0];
                int32_t mn = INF;
                for (uint32_t k = a0 + lane; k < a1; k += 32) mn = min(mn, slack[k]);
                mn = __reduce_min_sync(FULL, mn);
                __syncwarp();
                const uint32_t ab = a0 >> 5, ai = 32 * ab + lane;
                if ((int64_t)bdm > (int64_t)mn) {          // blocked for good
                    if (lane == 0) key[a0] = 0;
                    __syncwarp();
                    const uint32_t v = __reduce_max_sync(FULL, ai < n ? key[ai] : 0u);
                    if (lane == 0) bmx[ab] = v;
                    __syncwarp();
                    continue;
                }
                for (uint32_t k = a0 + lane; k < a1; k += 32) slack[k] -= (int32_t)bdm;
                if (lane == 0) {
                    const uint32_t v = cn[a0], c = (v & 15u) + 1u, cb = (uint32_t)cbr[a0] * S;
                    cn[a0] = (uint8_t)((v & 0xF0u) | c);
                    uint32_t k = 0, dm = 0;
                    if (c < (v >> 4)) {                      // c + 1 < count
                        k = ((0xFFFFu - (uint32_t)__ldg(&kp.srank[cb + c])) << 16) | (0xFFFFu - a0);
                        dm = __ldg(&kp.ctab[cb + c + 1]).z - __ldg(&kp.ctab[cb + c]).z;
                    }
                    key[a0] = k;
                    dms[a0] = dm;
                }
                __syncwarp();
                const uint32_t v = __reduce_max_sync(FULL, ai < n ? key[ai] : 0u);
                if (lane == 0) bmx[ab] = v;
                __syncwarp();
            }
        }
        if (feasible) {
            // ---- M3b / M3c: is the warm start provably within the gap? else branch and bound
            const uint4 *__restrict__ ctab = kp.ctab;
            // K*: the points where the warm start blocks a pair (dms[p] = its next step's KiB, 0 = none)
            for (uint32_t k = lane; k < n; k += 32) key[k] = 0;
            __syncwarp();
            for (uint32_t p = lane; p < n; p += 32) {
                const uint32_t dm = dms[p], e = eP[p];
                if (!dm) continue;
                for (uint32_t k = p; k < e; k++)
                    if ((int64_t)slack[k] < (int64_t)dm) key[k] = 1u;
            }
            __syncwarp();
            uint32_t nK = 0;
            for (uint32_t k0 = 0; k0 < n; k0 += 32) {       // inclusive prefix count of K* in key[]
                const uint32_t k = k0 + lane;
                uint32_t v = k < n ? key[k] : 0u;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t u = __shfl_up_sync(FULL, v, o);
                    if (lane >= o) v += u;
                }
                if (k < n) key[k] = nK + v;
                nK += __shfl_sync(FULL, v, 31);
            }
            __syncwarp();
            // c_p = K* points in pair p's range (into dms[], dead now); the warm start's objective
            unsigned long long inc = 0;
            for (uint32_t p = lane; p < n; p += 32) {
                const uint32_t e = eP[p];
                dms[p] = e > p ? key[e - 1] - (p ? key[p - 1] : 0u) : 0u;
                const uint4 E = __ldg(&ctab[(uint32_t)cbr[p] * S + (cn[p] & 15u)]);
                inc += (unsigned long long)E.x + E.y;
            }
            inc = warp_sum_u64(inc);
            __syncwarp();
            const uint32_t *cpa = dms;
            const long long Mk = (long long)nK * (long long)bud;
            const unsigned long long lb0 = ilp_bound(ctab, cbr, cn, cpa, S, n, 0, Mk, 0ull);
            const bool certified = ilp_within(lb0, inc, kp.gap_pm);
            unsigned long long nodes = 0;
            bool capped = false;
            if (!certified) {
                // branch and bound (the oracle's depth-first order): candidate-0 slack profile again
                for (uint32_t k = lane; k < n; k += 32) slack[k] = 0;
                __syncwarp();
                for (uint32_t p = lane; p < n; p += 32) {
                    const uint32_t e = eP[p];
                    if (e > p) {
                        const int32_t z = (int32_t)__ldg(&ctab[(uint32_t)cbr[p] * S]).z;
                        atomicAdd(&slack[p], z);
                        if (e < n) atomicSub(&slack[e], z);
                    }
                }
                __syncwarp();
                {
                    int32_t run = 0;
                    for (uint32_t k0 = 0; k0 < n; k0 += 32) {
                        const uint32_t k = k0 + lane;
                        int32_t v = k < n ? slack[k] : 0;
                        for (int o = 1; o < 32; o <<= 1) {
                            const int32_t u = __shfl_up_sync(FULL, v, o);
                            if (lane >= o) v += u;
                        }
                        if (k < n) slack[k] = bud - (run + v);
                        run += __shfl_sync(FULL, v, 31);
                    }
                }
                uint8_t *dpick = reinterpret_cast<uint8_t *>(key);   // key[] is dead: picks and
                uint8_t *tryc = dpick + n_max;                          // next-candidate-to-try + 1
                if (lane == 0) tryc[0] = (uint8_t)((cn[0] >> 4) + 1u);
                __syncwarp();
                uint32_t d = 0;
                unsigned long long fixed = 0;
                long long rfix = 0;
                for (;;) {
                    const uint32_t t = tryc[d];
                    if (t == 0) {                                    // exhausted: back to d - 1
                        if (d == 0) break;
                        d--;
                        const uint32_t c = dpick[d], cb = (uint32_t)cbr[d] * S;
                        const uint4 E = __ldg(&ctab[cb + c]);
                        const int32_t dm = (int32_t)(E.z - __ldg(&ctab[cb]).z);
                        for (uint32_t k = d + lane; k < (uint32_t)eP[d]; k += 32) slack[k] += dm;
                        fixed -= (unsigned long long)E.x + E.y;
                        rfix -= (long long)cpa[d] * E.z;
                        __syncwarp();
                        continue;
                    }
                    if (nodes >= kp.node_cap) { capped = true; break; }
                    nodes++;
                    const uint32_t c = t - 1u, cb = (uint32_t)cbr[d] * S, e = eP[d];
                    __syncwarp();
                    if (lane == 0) tryc[d] = (uint8_t)c;
                    const uint4 E = __ldg(&ctab[cb + c]);
                    const int32_t dm = (int32_t)(E.z - __ldg(&ctab[cb]).z);
                    int32_t mn = INF;
                    for (uint32_t k = d + lane; k < e; k += 32) mn = min(mn, slack[k]);
                    mn = __reduce_min_sync(FULL, mn);
                    if ((int64_t)mn < (int64_t)dm) { __syncwarp(); continue; }      // does not fit
                    __syncwarp();
                    for (uint32_t k = d + lane; k < e; k += 32) slack[k] -= dm;
                    if (lane == 0) dpick[d] = (uint8_t)c;
                    fixed += (unsigned long long)E.x + E.y;
                    rfix += (long long)cpa[d] * E.z;
                    __syncwarp();
                    bool descend = false;
                    if (d + 1 == n) {                                 // a complete selection
                        if (fixed < inc) {
                            inc = fixed;
                            for (uint32_t p = lane; p < n; p += 32) cn[p] = (uint8_t)((cn[p] & 0xF0u) | dpick[p]);
                        }
                    } else {
                        const unsigned long long lb = ilp_bound(ctab, cbr, cn, cpa, S, n, d + 1, Mk - rfix, fixed);
                        descend = !ilp_within(lb, inc, kp.gap_pm);
                    }
                    __syncwarp();
                    if (descend) {
                        d++;
                        if (lane == 0) tryc[d] = (uint8_t)((cn[d] >> 4) + 1u);
                        __syncwarp();
                        continue;
                    }
                    for (uint32_t k = d + lane; k < e; k += 32) slack[k] += dm;   // undo the pick
                    fixed -= (unsigned long long)E.x + E.y;
                    rfix -= (long long)cpa[d] * E.z;
                    __syncwarp();
                }
            }
            if (lane == 0 && kp.mo_stats && n > 0) {
                atomicAdd(kp.mo_stats + 0, 1ull);
                atomicAdd(kp.mo_stats + (certified ? 1 : 2), 1ull);
                if (capped) atomicAdd(kp.mo_stats + 3, 1ull);
                if (nodes) atomicAdd(kp.mo_stats + 4, nodes);
            }
        }
        // the backward row needs each pair's backward position again: rebuild the segment -> position
        // map into the (now dead) step arrays -- from the record's sequences, or from the orders
        if (orow) {
            uint16_t *invF = invB;                   // segment -> forward position
            uint32_t nF = 0, nB = 0;
            const uint32_t below = (1u << lane) - 1u;
            for (uint32_t t0 = 0; t0 < 2 * n; t0 += 32) {
                const uint32_t t = t0 + lane;
                const uint32_t e = t < 2 * n ? __ldg(&orow[t]) : 0xFFFFu;
                const bool isF = t < 2 * n && !(e & 0x8000u);
                const uint32_t bF = __ballot_sync(FULL, isF);
                if (isF) invF[e & 0x7FFFu] = (uint16_t)(nF + __popc(bF & below));
                nF += __popc(bF);
            }
            __syncwarp();
            for (uint32_t p = lane; p < n_max; p += 32) selF[p] = p < n ? (cn[p] & 15u) : 0;
            for (uint32_t t0 = 0; t0 < 2 * n; t0 += 32) {
                const uint32_t t = t0 + lane;
                const uint32_t e = t < 2 * n ? __ldg(&orow[t]) : 0xFFFFu;
                const bool isB = t < 2 * n && (e & 0x8000u);
                const uint32_t bB = __ballot_sync(FULL, isB);
                if (isB) selB[nB + __popc(bB & below)] = cn[invF[e & 0x7FFFu]] & 15u;
                nB += __popc(bB);
            }
        } else {
            for (uint32_t q = lane; q < n; q += 32)
                invB[__ldg(reinterpret_cast<const uint16_t *>(rec + kp.off_bwd) + q)] = (uint16_t)q;
            __syncwarp();
            for (uint32_t p = lane; p < n_max; p += 32) {
                const uint8_t c = p < n ? (cn[p] & 15u) : 0;
                selF[p] = c;
                if (p < n) selB[invB[__ldg(reinterpret_cast<const uint16_t *>(rec + kp.off_fwd) + p)]] = c;
            }
        }
        if (n < n_max)
            for (uint32_t q = n + lane; q < n_max; q += 32) selB[q] = 0;
        __syncwarp();
    }
}

cudaError_t launch_mcand(const MCandParams &p, cudaStream_t s) {
    const uint32_t blocks = (p.n_items + 127) / 128;
    dip_mcand_kernel<<<blocks ? blocks : 1, 128, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t prepare_memopt(size_t smem) {
    return cudaFuncSetAttribute(dip_memopt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t occupancy_memopt(size_t smem, int *blocks_per_sm) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, dip_memopt_kernel, 128, smem);
}

cudaError_t launch_memopt(const KParams &kp, uint8_t *sel, uint32_t warp_bytes, int grid, cudaStream_t s) {
    dip_memopt_kernel<<<grid, 128, 4 * (size_t)warp_bytes, s>>>(kp, sel, warp_bytes);
    return cudaGetLastError();
}

}  // namespace dipk
