// dip_plan.cpp -- SURVEY §8(f) row f4: compile a scored schedule into per-rank action lists
// (§6.3, following DynaPipe): fw_stage / bw_stage actions, asynchronous
// isend / irecv for every cross-rank dependency, wait_isend / wait_irecv synchronisation placed from
// the simulated timeline, consecutive P2P actions grouped into one batch; and a
// discrete-event validator that executes a plan (P2P priced like the simulator) to check matching,
// termination and that every stage starts at its simulated time.
//
// Placement (reading R-36): each message m (producer stage -> consumer stage on another
// rank) gets tag = its index in the compiled order; isend(m) right after the producing stage;
// wait_isend(m) right before the producer rank's next stage (or at the end); irecv(m) right after
// the last stage of the consumer rank that ends no later than the producing stage starts (at the
// start of the list if none), so every receive is posted before its send in simulated time;
// wait_irecv(m) right before the consuming stage.
#include <algorithm>
#include <cstring>
#include <vector>

#include "dip_host_internal.h"

using namespace diph;

namespace {

struct Msg {
    uint32_t src_r, src_t, dst_r, dst_t;   // producer (rank, slot) -> consumer (rank, slot)
    uint64_t p2p;                          // transfer time on the edge (R-7)
};

struct Sched {
    uint32_t P, n;
    std::vector<uint32_t> seg;             // [P][2n] segment of (rank, slot)
    std::vector<uint8_t> dir;              // [P][2n]
    std::vector<uint64_t> lat;             // [P][2n]
    std::vector<uint32_t> slotF, slotB;    // [P][n_max] slot of F(s) / B(s) on rank r
};

// decode one record (host) into per-rank slot lists -- each rank's order from the record's shared
// sequences + F/B bits, or from explicit per-rank orders ([P][2 n_max], dip_interleave's format);
// returns false if malformed (a segment missing, duplicated or absent from the split on any rank)
bool decode(const dip_model *M, const uint8_t *rec, const uint16_t *orders, Sched &S, std::vector<uint8_t> &Mv,
            std::vector<uint32_t> &W) {
    const uint32_t P = M->P, nm = M->nmod, m = M->m;
    uint16_t n16, flags;
    std::memcpy(&n16, rec, 2);
    std::memcpy(&flags, rec + 2, 2);
    if (flags) return false;
    S.P = P;
    S.n = n16;
    const uint32_t n = S.n;
    Mv.assign(m * nm, 0);
    uint32_t nsum = 0;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            const uint32_t q = b * nm + i, N = M->nbi[q];
            uint32_t v = N > 0 ? 1u : 0u;
            if (M->max_split[i] > 1) {
                const uint32_t nib = b * M->nsplit + M->nib_slot[i];
                v = (rec[M->off_nib + nib / 2] >> ((nib & 1) * 4)) & 15u;
            }
            if ((N == 0) != (v == 0) || v > std::min(N, M->max_split[i])) return false;
            Mv[q] = (uint8_t)v;
            nsum += v * M->Kv[i];
        }
    if (nsum != n || n > M->n_max) return false;
    W.assign(M->n_max, 0);
    std::vector<uint8_t> present(M->n_max, 0);
    for (uint32_t q = 0; q < m * nm; q++) {
        const uint32_t i = q % nm, K = M->Kv[i];
        for (uint32_t j = 0; j < Mv[q]; j++)
            for (uint32_t k = 0; k < K; k++) {
                const uint32_t s = M->sbase[q] + j * K + k;
                present[s] = 1;
                W[s] = M->wtab[M->woff[q] + Mv[q] * (Mv[q] - 1) / 2 + j];
            }
    }
    const uint16_t *fwd = reinterpret_cast<const uint16_t *>(rec + M->off_fwd);
    const uint16_t *bwd = reinterpret_cast<const uint16_t *>(rec + M->off_bwd);
    const uint32_t *fb = reinterpret_cast<const uint32_t *>(rec + M->off_fb);
    S.seg.assign(P * 2 * n, 0);
    S.dir.assign(P * 2 * n, 0);
    S.lat.assign(P * 2 * n, 0);
    S.slotF.assign(P * M->n_max, ~0u);
    S.slotB.assign(P * M->n_max, ~0u);
    for (uint32_t r = 0; r < P; r++) {
        uint32_t fi = 0, bi = 0;
        if (orders)
            for (uint32_t t = 2 * n; t < 2 * M->n_max; t++)
                if (orders[(size_t)r * 2 * M->n_max + t] != 0xFFFFu) return false;
        for (uint32_t t = 0; t < 2 * n; t++) {
            uint32_t isb, s;
            if (orders) {
                const uint32_t e = orders[(size_t)r * 2 * M->n_max + t];
                isb = e >> 15;
                s = e & 0x7FFFu;
                if ((isb ? bi : fi) >= n) return false;
                (isb ? bi : fi)++;
            } else {
                isb = (fb[(t / 32) * P + r] >> (t % 32)) & 1u;
                if ((isb ? bi : fi) >= n) return false;
                s = isb ? bwd[bi++] : fwd[fi++];
            }
            if (s >= M->n_max || !present[s]) return false;
            uint32_t &slot = (isb ? S.slotB : S.slotF)[r * M->n_max + s];
            if (slot != ~0u) return false;                       // the same segment twice on this rank
            slot = t;
            S.seg[r * 2 * n + t] = s;
            S.dir[r * 2 * n + t] = (uint8_t)isb;
            uint32_t q = 0;
            while (q + 1 < m * nm && M->sbase[q + 1] <= s) q++;
            const uint32_t i = q % nm, k = (s - M->sbase[q]) % M->Kv[i];
            const uint32_t t4 = 4 * (M->tab_off[i] + W[s]);
            S.lat[r * 2 * n + t] = (uint64_t)M->layers[M->lay_off[i] + k * P + r] * M->tab[t4 + isb];
        }
    }
    return true;
}

uint64_t p2p_of(const dip_model *M, const std::vector<uint32_t> &W, uint32_t s) {
    uint32_t q = 0;
    while (q + 1 < M->m * M->nmod && M->sbase[q + 1] <= s) q++;
    return M->P > 1 ? M->tab[4 * (M->tab_off[q % M->nmod] + W[s]) + 3] : 0;
}

// every cross-rank dependency edge of the schedule (the edges of SURVEY §8(a4) between ranks)
void messages(const dip_model *M, const Sched &S, const std::vector<uint8_t> &Mv, const std::vector<uint32_t> &W,
              std::vector<Msg> &out) {
    const uint32_t P = S.P, n = S.n, nm = M->nmod;
    auto slotF = [&](uint32_t r, uint32_t s) { return S.slotF[r * M->n_max + s]; };
    auto slotB = [&](uint32_t r, uint32_t s) { return S.slotB[r * M->n_max + s]; };
    for (uint32_t r = 0; r < P; r++)
        for (uint32_t t = 0; t < 2 * n; t++) {
            const uint32_t s = S.seg[r * 2 * n + t];
            const bool isb = S.dir[r * 2 * n + t];
            uint32_t q = 0;
            while (q + 1 < M->m * nm && M->sbase[q + 1] <= s) q++;
            const uint32_t b = q / nm, i = q % nm, K = M->Kv[i], k = (s - M->sbase[q]) % K;
            if (!isb) {
                if (r > 0) out.push_back({r - 1, slotF(r - 1, s), r, t, p2p_of(M, W, s)});
                else if (P > 1) {
                    if (k > 0) out.push_back({P - 1, slotF(P - 1, s - 1), 0, t, p2p_of(M, W, s - 1)});
                    else for (uint32_t p = 0; p < nm; p++)
                        if ((M->prod_mask[i] >> p) & 1u)
                            for (uint32_t jj = 0; jj < Mv[b * nm + p]; jj++) {
                                const uint32_t pr = M->sbase[b * nm + p] + jj * M->Kv[p] + M->Kv[p] - 1;
                                out.push_back({P - 1, slotF(P - 1, pr), 0, t, p2p_of(M, W, pr)});
                            }
                }
            } else {
                if (r + 1 < P) out.push_back({r + 1, slotB(r + 1, s), r, t, p2p_of(M, W, s)});
                else if (P > 1) {
                    if (k + 1 < K) out.push_back({0, slotB(0, s + 1), P - 1, t, p2p_of(M, W, s)});
                    else for (uint32_t c = 0; c < nm; c++)
                        if ((M->cons_mask[i] >> c) & 1u)
                            for (uint32_t jj = 0; jj < Mv[b * nm + c]; jj++)
                                out.push_back({0, slotB(0, M->sbase[b * nm + c] + jj * M->Kv[c]), P - 1, t, p2p_of(M, W, s)});
                }
            }
        }
}

}  // namespace

extern "C" dip_status dip_compile_plan(const dip_model *M, const void *record, const uint16_t *orders,
                                       const uint64_t *start, const uint64_t *end, dip_action *actions,
                                       size_t capacity, uint32_t *rank_off, uint32_t *n_messages) {
    if (!M || !record || !start || !end || !rank_off) return fail(DIP_EINVAL, "null argument");
    Sched S;
    std::vector<uint8_t> Mv;
    std::vector<uint32_t> W;
    if (!decode(M, static_cast<const uint8_t *>(record), orders, S, Mv, W)) return fail(DIP_EINVAL, "malformed record");
    const uint32_t P = S.P, n = S.n, n2 = 2 * M->n_max;   // timeline rows are 2*n_max long
    std::vector<Msg> msgs;
    messages(M, S, Mv, W, msgs);
    // per rank: actions before / after each slot
    std::vector<std::vector<std::vector<dip_action>>> pre(P), post(P);
    for (uint32_t r = 0; r < P; r++) { pre[r].assign(2 * n + 1, {}); post[r].assign(2 * n + 1, {}); }
    for (uint32_t x = 0; x < msgs.size(); x++) {
        const Msg &g = msgs[x];
        const uint64_t send_start = start[g.src_r * n2 + g.src_t];
        // isend right after the producing stage; wait_isend before the producer's next stage
        post[g.src_r][g.src_t].push_back({DIP_ACT_ISEND, g.dst_r, x, 0, g.src_t});
        pre[g.src_r][g.src_t + 1].push_back({DIP_ACT_WAIT_ISEND, g.dst_r, x, 0, g.src_t});
        // irecv after the consumer's last stage ending no later than send_start
        uint32_t at = 0;   // position = "before slot at"
        for (uint32_t t = 0; t < g.dst_t; t++)
            if (end[g.dst_r * n2 + t] <= send_start) at = t + 1;
        pre[g.dst_r][at].insert(pre[g.dst_r][at].begin(), {DIP_ACT_IRECV, g.src_r, x, 0, g.dst_t});
        pre[g.dst_r][g.dst_t].push_back({DIP_ACT_WAIT_IRECV, g.src_r, x, 0, g.dst_t});
    }
    size_t cnt = 0;
    uint32_t batch = 0;
    for (uint32_t r = 0; r < P; r++) {
        rank_off[r] = (uint32_t)cnt;
        bool in_p2p = false;
        auto emit = [&](dip_action a) {
            const bool p2p = a.kind == DIP_ACT_ISEND || a.kind == DIP_ACT_IRECV;
            if (p2p && !in_p2p) batch++;
            in_p2p = p2p;
            a.batch = p2p ? batch : 0;
            if (cnt < capacity && actions) actions[cnt] = a;
            cnt++;
        };
        for (uint32_t t = 0; t <= 2 * n; t++) {
            // receives are posted first, then the previous stage's sends complete, then this
            // stage's receives are waited for, then the stage runs
            for (const dip_action &a : pre[r][t]) if (a.kind == DIP_ACT_IRECV) emit(a);
            for (const dip_action &a : pre[r][t]) if (a.kind == DIP_ACT_WAIT_ISEND) emit(a);
            for (const dip_action &a : pre[r][t]) if (a.kind == DIP_ACT_WAIT_IRECV) emit(a);
            if (t == 2 * n) break;
            emit({S.dir[r * 2 * n + t] ? (uint32_t)DIP_ACT_BW_STAGE : (uint32_t)DIP_ACT_FW_STAGE, r,
                  S.seg[r * 2 * n + t], 0, t});
            for (const dip_action &a : post[r][t]) emit(a);
        }
    }
    rank_off[P] = (uint32_t)cnt;
    if (n_messages) *n_messages = (uint32_t)msgs.size();
    if (cnt > capacity) return fail(DIP_ERANGE, "action buffer too small (rank_off[P] holds the size)");
    return DIP_OK;
}

extern "C" dip_status dip_validate_plan(const dip_model *M, const void *record, const uint16_t *orders,
                                        const dip_action *actions, const uint32_t *rank_off, uint64_t *stage_start,
                                        int32_t *ok) {
    // discrete-event execution: a rank runs its list in order; isend / irecv post instantly; a
    // wait_irecv completes when the message has arrived (send time + p2p); a wait_isend when the
    // receive has been posted; a stage starts at the rank's clock and runs for its latency.
    if (!M || !record || !actions || !rank_off || !ok) return fail(DIP_EINVAL, "null argument");
    *ok = 0;
    Sched S;
    std::vector<uint8_t> Mv;
    std::vector<uint32_t> W;
    if (!decode(M, static_cast<const uint8_t *>(record), orders, S, Mv, W)) return fail(DIP_EINVAL, "malformed record");
    const uint32_t P = S.P, n = S.n, n2 = 2 * M->n_max;
    std::vector<Msg> msgs;
    messages(M, S, Mv, W, msgs);
    const size_t nmsg = msgs.size();
    for (uint32_t r = 1; r <= P; r++)
        if (rank_off[r] < rank_off[r - 1]) return fail(DIP_EINVAL, "rank_off not monotone");
    for (uint32_t r = 0; r < P; r++)          // caller-supplied actions: reject out-of-range fields
        for (uint32_t a = rank_off[r]; a < rank_off[r + 1]; a++) {
            const dip_action &x = actions[a];
            if (x.kind > DIP_ACT_WAIT_IRECV) return DIP_OK;
            if ((x.kind == DIP_ACT_FW_STAGE || x.kind == DIP_ACT_BW_STAGE) &&
                (x.slot >= 2 * n || S.dir[r * 2 * n + x.slot] != (x.kind == DIP_ACT_BW_STAGE ? 1u : 0u)))
                return DIP_OK;
            if (x.kind >= DIP_ACT_ISEND && x.tag >= nmsg) return DIP_OK;
        }

    std::vector<int64_t> sent(nmsg, -1), posted(nmsg, -1);
    std::vector<uint32_t> nsend(nmsg, 0), nrecv(nmsg, 0);
    std::vector<uint32_t> pc(P);
    std::vector<uint64_t> clk(P, 0);
    for (uint32_t r = 0; r < P; r++) {
        pc[r] = rank_off[r];
        for (uint32_t a = rank_off[r]; a < rank_off[r + 1]; a++) {
            const dip_action &x = actions[a];
            if (x.kind == DIP_ACT_ISEND || x.kind == DIP_ACT_IRECV) {
                if (x.tag >= nmsg) return DIP_OK;                     // unmatched tag
                const Msg &g = msgs[x.tag];
                if (x.kind == DIP_ACT_ISEND && (g.src_r != r || g.dst_r != x.peer)) return DIP_OK;
                if (x.kind == DIP_ACT_IRECV && (g.dst_r != r || g.src_r != x.peer)) return DIP_OK;
                (x.kind == DIP_ACT_ISEND ? nsend : nrecv)[x.tag]++;
            }
        }
    }
    for (size_t x = 0; x < nmsg; x++) if (nsend[x] != 1 || nrecv[x] != 1) return DIP_OK;   // perfect pairing
    if (stage_start) std::memset(stage_start, 0, sizeof(uint64_t) * P * n2);
    for (;;) {
        bool progress = false, all = true;
        for (uint32_t r = 0; r < P; r++) {
            while (pc[r] < rank_off[r + 1]) {
                const dip_action &x = actions[pc[r]];
                if (x.kind == DIP_ACT_ISEND) sent[x.tag] = (int64_t)clk[r];
                else if (x.kind == DIP_ACT_IRECV) posted[x.tag] = (int64_t)clk[r];
                else if (x.kind == DIP_ACT_WAIT_IRECV) {
                    if (sent[x.tag] < 0) break;
                    clk[r] = std::max(clk[r], (uint64_t)sent[x.tag] + msgs[x.tag].p2p);
                } else if (x.kind == DIP_ACT_WAIT_ISEND) {
                    if (posted[x.tag] < 0) break;
                } else {
                    const uint32_t t = x.slot;
                    if (stage_start) stage_start[r * n2 + t] = clk[r];
                    clk[r] += S.lat[r * 2 * n + t];
                }
                pc[r]++;
                progress = true;
            }
            all &= pc[r] == rank_off[r + 1];
        }
        if (all) { *ok = 1; return DIP_OK; }
        if (!progress) return DIP_OK;                                   // deadlock: *ok = 0
    }
}
