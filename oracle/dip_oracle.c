/* dip_oracle.c -- the CPU ORACLE for DIP candidate-schedule scoring.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this file's
 * library.  It shares no code, header, table or helper with the CUDA path
 * (paper_2504_14145_b200/), and never imports it.
 *
 * A plain, slow, obviously-correct simulator of one candidate schedule, written
 * step by step in the order of SURVEY.md §8(c) (O1-O11) and of the paper:
 *
 *   O1  chunking           P:457-459 "distributes layers across P*K_i model chunks" (R-3)
 *   O2  split              P:461-467 "M_i ... uniformly partitioned sub-microbatches" (R-2, R-21)
 *   O3  segments           P:466-467 "2 M_i K_i pipeline segments"
 *   O4  encoding checks    (R-11)
 *   O5  per-rank orders    (R-1)
 *   O6  stage costs        P:522-523 (simulator latencies), P:685-700 (R-7, R-20)
 *   O7  explicit edge list P:368 (segments span all P ranks), R-4..R-6
 *   O8  Kahn longest path  P:702 "populates operator timestamps in topological order" (R-12)
 *   O9  memory timeline    P:703-705 "tensor lifetimes ... peak memory usage" (R-9, R-10)
 *   O10 outputs            P:499 score = "end-to-end iteration time"; bubble P:248 (R-16)
 *   O11 argmin             P:499-501 best score; ties -> lowest index (R-14, R-15)
 *   I1-I6 interleaving     P:511-548 the dual-queue greedy, see below
 *   S1-S6 search           P:472-509 MCTS segment reordering, see below
 *   M1-M4 memory opt.      P:550-590 per-layer memory optimisation, see below
 *
 * Integers everywhere (ns, KiB); u64 accumulators.  The only floating-point
 * value, the bubble ratio, is one IEEE double division of two exact integers.
 * Multi-threaded only across candidates (pthreads).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint32_t P, nmod, m;
    const uint32_t *L, *K, *max_split, *w_max, *producer_mask;   /* [nmod] */
    const uint32_t *tab_off;                                      /* [nmod+1] */
    const uint32_t *tab_f, *tab_b, *tab_act, *tab_p2p;            /* per-layer T_i[W] */
    const uint32_t *chunk_off;      /* [nmod+1]; empty range -> default O1 rule */
    const uint32_t *chunk_layers;   /* explicit layers per chunk (P*K_i entries) */
    const uint32_t *inst_off;       /* [m*nmod+1] */
    const uint16_t *inst_units;
    const uint32_t *budget_kib;     /* [P] */
} oproblem;

typedef struct {
    uint32_t n_max, fbw;
    const uint8_t *split;           /* [N][m*nmod] */
    const uint32_t *n;              /* [N] */
    const uint16_t *fwd, *bwd;      /* [N][n_max] */
    const uint32_t *fb;             /* [N][P][fbw] */
    const uint16_t *ord;            /* NULL, or [N][P][2 n_max] explicit per-rank orders (segment id |
                                       0x8000 for a backward stage; 0xFFFF beyond 2n) replacing the
                                       shared sequences + F/B bits in O4/O5 (f1's output, R-29) */
} ocands;

enum { ST_OK = 0, ST_OOM = 1, ST_DEADLOCK = 2, ST_BAD = 3 };

/* ---------------- O1: layers per chunk (R-3) ----------------
 * C = P*K chunks of consecutive layers; the first L mod C chunks get one extra
 * layer.  Segment k on rank r uses chunk k*P + r.  C > L is an error. */
int oracle_chunk_layers(uint32_t L, uint32_t P, uint32_t K, uint32_t *out) {
    uint32_t C = P * K;
    if (C == 0 || C > L) return -1;
    for (uint32_t c = 0; c < C; c++) out[c] = L / C + (c < L % C ? 1u : 0u);
    return 0;
}

/* ---------------- O2: balanced contiguous split (R-2) ----------------
 * Part j of N instances split M ways covers [j*q + min(j, rho), (j+1)*q + min(j+1, rho))
 * with q = floor(N/M), rho = N mod M.  start has M+1 entries. */
int oracle_split(uint32_t N, uint32_t M, uint32_t *start) {
    if (M == 0) return -1;
    uint32_t q = N / M, rho = N % M;
    for (uint32_t j = 0; j <= M; j++) start[j] = j * q + (j < rho ? j : rho);
    return 0;
}

typedef struct {
    uint64_t makespan, busy;
    uint32_t status, oom_mask;
    double bubble;
} ores;

static uint32_t seg_count_max(const oproblem *pb) {
    uint32_t t = 0;
    for (uint32_t i = 0; i < pb->nmod; i++) t += pb->max_split[i] * pb->K[i];
    return t * pb->m;
}

/* layers of module i, chunk c (O1, or the explicit override) */
static uint32_t layers_of(const oproblem *pb, uint32_t i, uint32_t c) {
    uint32_t lo = pb->chunk_off[i], hi = pb->chunk_off[i + 1];
    if (hi > lo) return pb->chunk_layers[lo + c];
    uint32_t C = pb->P * pb->K[i], L = pb->L[i];
    return L / C + (c < L % C ? 1u : 0u);
}

/* Evaluate candidate x.  peaks: [P] (u64), may be NULL.  If tl_start/tl_end are
 * given they receive per (rank, slot) start/end times ([P][2n]).  If ovr is given
 * ([P][idmax+1][3]: F latency, B latency, activation of each (rank, segment) stage pair), it
 * replaces O6's table costs (M4 of the per-layer memory optimisation below). */
static void eval_one(const oproblem *pb, const ocands *cs, uint64_t x, ores *res, uint64_t *peaks,
                     uint64_t *tl_start, uint64_t *tl_end, const uint64_t *ovr) {
    const uint32_t P = pb->P, nm = pb->nmod, m = pb->m;
    const uint32_t n_max = cs->n_max, fbw = cs->fbw;
    const uint8_t *split = cs->split + x * (uint64_t)m * nm;
    const uint16_t *fwd = cs->fwd + x * (uint64_t)n_max;
    const uint16_t *bwd = cs->bwd + x * (uint64_t)n_max;
    const uint32_t *fb = cs->fb + x * (uint64_t)P * fbw;
    uint32_t ncand = cs->n[x];

    res->makespan = UINT64_MAX;
    res->busy = 0;
    res->status = ST_BAD;
    res->oom_mask = 0;
    res->bubble = -1.0;
    if (peaks) for (uint32_t r = 0; r < P; r++) peaks[r] = 0;

    /* segment-id space: id(b,i,j,k) = base(b,i) + j*K_i + k, b-major */
    uint32_t idmax = seg_count_max(pb);
    uint32_t *base = malloc(sizeof(uint32_t) * (m * nm + 1));
    uint32_t *W = calloc(idmax + 1, sizeof(uint32_t));       /* work units of the segment's part */
    uint8_t *present = calloc(idmax + 1, 1);
    uint32_t *sb = malloc(sizeof(uint32_t) * (idmax + 1)), *si = malloc(sizeof(uint32_t) * (idmax + 1));
    uint32_t *sj = malloc(sizeof(uint32_t) * (idmax + 1)), *sk = malloc(sizeof(uint32_t) * (idmax + 1));
    int bad = 0;
    uint32_t acc = 0, n = 0;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            base[b * nm + i] = acc;
            for (uint32_t j = 0; j < pb->max_split[i]; j++)
                for (uint32_t k = 0; k < pb->K[i]; k++) {
                    uint32_t id = acc + j * pb->K[i] + k;
                    sb[id] = b; si[id] = i; sj[id] = j; sk[id] = k;
                }
            acc += pb->max_split[i] * pb->K[i];
        }
    /* O2: split and work per part */
    for (uint32_t b = 0; b < m && !bad; b++)
        for (uint32_t i = 0; i < nm; i++) {
            uint32_t q = b * nm + i;
            uint32_t lo = pb->inst_off[q], N = pb->inst_off[q + 1] - lo, M = split[q];
            uint32_t cap = N < pb->max_split[i] ? N : pb->max_split[i];
            if ((N == 0) != (M == 0) || M > cap) { bad = 1; break; }
            if (M == 0) continue;
            uint32_t st[16];
            oracle_split(N, M, st);
            for (uint32_t j = 0; j < M; j++) {
                uint32_t w = 0;
                for (uint32_t u = st[j]; u < st[j + 1]; u++) w += pb->inst_units[lo + u];
                for (uint32_t k = 0; k < pb->K[i]; k++) {
                    uint32_t id = base[q] + j * pb->K[i] + k;
                    present[id] = 1;
                    W[id] = w;
                    n++;   /* O3 */
                }
            }
        }
    /* O4: encoding checks */
    if (!bad && (ncand != n || n > n_max)) bad = 1;
    const uint16_t *ord = cs->ord ? cs->ord + x * (uint64_t)P * 2 * n_max : NULL;
    if (!bad && ord) {          /* explicit per-rank orders: every stage of the rank exactly once */
        uint8_t *seen = malloc(2 * (size_t)(idmax + 1));
        for (uint32_t r = 0; r < P && !bad; r++) {
            memset(seen, 0, 2 * (size_t)(idmax + 1));
            for (uint32_t t = 0; t < 2 * n_max && !bad; t++) {
                uint32_t e = ord[(size_t)r * 2 * n_max + t], sg = e & 0x7FFFu, dr = e >> 15;
                if (t >= 2 * n) { if (e != 0xFFFF) bad = 1; continue; }
                if (sg >= idmax || !present[sg] || seen[dr * (idmax + 1) + sg]) bad = 1;
                else seen[dr * (idmax + 1) + sg] = 1;
            }
        }
        free(seen);
    }
    if (!bad && !ord) {
        uint8_t *seenF = calloc(idmax + 1, 1), *seenB = calloc(idmax + 1, 1);
        for (uint32_t p = 0; p < n_max && !bad; p++) {
            if (p < n) {
                uint32_t a = fwd[p], c = bwd[p];
                if (a >= idmax || c >= idmax || !present[a] || !present[c] || seenF[a] || seenB[c]) bad = 1;
                else { seenF[a] = 1; seenB[c] = 1; }
            } else if (fwd[p] != 0xFFFF || bwd[p] != 0xFFFF) bad = 1;
        }
        free(seenF); free(seenB);
        for (uint32_t r = 0; r < P && !bad; r++) {
            uint32_t ones = 0;
            for (uint32_t t = 0; t < 32 * fbw; t++) {
                uint32_t bit = (fb[r * fbw + t / 32] >> (t % 32)) & 1u;
                if (t < 2 * n) ones += bit;
                else if (bit) bad = 1;
            }
            if (ones != n) bad = 1;
        }
    }
    if (bad) goto done;
    if (n == 0) {
        res->makespan = 0;
        res->status = ST_OK;
        res->bubble = 0.0;
        goto done;
    }
    {
        const uint32_t S = 2 * n, NN = P * S;
        /* O5: per-rank orders; O6: costs */
        uint8_t *dir = malloc(NN);
        uint32_t *seg = malloc(sizeof(uint32_t) * NN);
        uint64_t *lat = malloc(sizeof(uint64_t) * NN), *act = malloc(sizeof(uint64_t) * NN);
        uint32_t *slotF = malloc(sizeof(uint32_t) * P * (idmax + 1)), *slotB = malloc(sizeof(uint32_t) * P * (idmax + 1));
        for (uint32_t r = 0; r < P; r++) {
            uint32_t fi = 0, bi = 0;
            for (uint32_t t = 0; t < S; t++) {
                uint32_t node = r * S + t, isb, s;
                if (ord) {
                    uint32_t e = ord[(size_t)r * 2 * n_max + t];
                    isb = e >> 15;
                    s = e & 0x7FFFu;
                } else {
                    isb = (fb[r * fbw + t / 32] >> (t % 32)) & 1u;
                    s = isb ? bwd[bi++] : fwd[fi++];
                }
                if (isb) slotB[r * (idmax + 1) + s] = t;
                else slotF[r * (idmax + 1) + s] = t;
                dir[node] = (uint8_t)isb;
                seg[node] = s;
                uint32_t i = si[s], k = sk[s];
                uint32_t toff = pb->tab_off[i] + W[s];
                uint64_t lay = layers_of(pb, i, k * P + r);
                lat[node] = lay * (uint64_t)(isb ? pb->tab_b[toff] : pb->tab_f[toff]);
                act[node] = lay * (uint64_t)pb->tab_act[toff];
                if (ovr) {
                    const uint64_t *o = ovr + ((uint64_t)r * (idmax + 1) + s) * 3;
                    lat[node] = o[isb];
                    act[node] = o[2];
                }
            }
        }
        /* O7: explicit predecessor lists (dst node, src node, weight) */
        uint32_t cap = NN * 4 + 16, ne = 0;
        uint32_t *esrc = malloc(sizeof(uint32_t) * cap), *edst = malloc(sizeof(uint32_t) * cap);
        uint64_t *ew = malloc(sizeof(uint64_t) * cap);
#define ADD_EDGE(SRC, DST, WT) do { \
        if (ne == cap) { cap *= 2; esrc = realloc(esrc, sizeof(uint32_t) * cap); \
            edst = realloc(edst, sizeof(uint32_t) * cap); ew = realloc(ew, sizeof(uint64_t) * cap); } \
        esrc[ne] = (SRC); edst[ne] = (DST); ew[ne] = (WT); ne++; } while (0)
        for (uint32_t r = 0; r < P; r++)
            for (uint32_t t = 0; t < S; t++) {
                uint32_t node = r * S + t, s = seg[node];
                uint32_t b = sb[s], i = si[s], k = sk[s], K = pb->K[i];
                uint64_t p2p_s = pb->tab_p2p[pb->tab_off[i] + W[s]];
                if (t > 0) ADD_EDGE(node - 1, node, 0);                 /* same rank, previous slot */
                if (dir[node] == 0) {                                    /* forward stage */
                    if (r > 0) ADD_EDGE((r - 1) * S + slotF[(r - 1) * (idmax + 1) + s], node, p2p_s); /* R-4 */
                    else if (k > 0) {                                    /* previous segment, rank P-1 */
                        uint32_t pr = s - 1;
                        uint64_t wgt = P > 1 ? pb->tab_p2p[pb->tab_off[i] + W[pr]] : 0;
                        ADD_EDGE((P - 1) * S + slotF[(P - 1) * (idmax + 1) + pr], node, wgt);
                    } else {                                             /* producer join (R-5) */
                        for (uint32_t ip = 0; ip < nm; ip++) {
                            if (!((pb->producer_mask[i] >> ip) & 1u)) continue;
                            for (uint32_t jp = 0; jp < split[b * nm + ip]; jp++) {
                                uint32_t pr = base[b * nm + ip] + jp * pb->K[ip] + pb->K[ip] - 1;
                                uint64_t wgt = P > 1 ? pb->tab_p2p[pb->tab_off[ip] + W[pr]] : 0;
                                ADD_EDGE((P - 1) * S + slotF[(P - 1) * (idmax + 1) + pr], node, wgt);
                            }
                        }
                    }
                } else {                                                 /* backward stage */
                    if (r + 1 < P) ADD_EDGE((r + 1) * S + slotB[(r + 1) * (idmax + 1) + s], node, p2p_s);
                    else if (k + 1 < K) {                                /* next segment, rank 0 */
                        ADD_EDGE(0 * S + slotB[0 * (idmax + 1) + s + 1], node, P > 1 ? p2p_s : 0);
                    } else {
                        int any = 0;                                     /* consumer join (R-5) */
                        for (uint32_t ic = 0; ic < nm; ic++) {
                            if (!((pb->producer_mask[ic] >> i) & 1u)) continue;
                            for (uint32_t jc = 0; jc < split[b * nm + ic]; jc++) {
                                uint32_t cn = base[b * nm + ic] + jc * pb->K[ic];
                                ADD_EDGE(0 * S + slotB[0 * (idmax + 1) + cn], node, P > 1 ? p2p_s : 0);
                                any = 1;
                            }
                        }
                        if (!any)                                        /* loss turnaround (R-6) */
                            ADD_EDGE((P - 1) * S + slotF[(P - 1) * (idmax + 1) + s], node, 0);
                    }
                }
            }
#undef ADD_EDGE
        /* O8: Kahn with a FIFO queue */
        uint32_t *indeg = calloc(NN, sizeof(uint32_t)), *soff = calloc(NN + 1, sizeof(uint32_t));
        for (uint32_t e = 0; e < ne; e++) { indeg[edst[e]]++; soff[esrc[e] + 1]++; }
        for (uint32_t v = 0; v < NN; v++) soff[v + 1] += soff[v];
        uint32_t *sorder = malloc(sizeof(uint32_t) * (ne + 1)), *fill = calloc(NN, sizeof(uint32_t));
        for (uint32_t e = 0; e < ne; e++) sorder[soff[esrc[e]] + fill[esrc[e]]++] = e;
        uint64_t *start = calloc(NN, sizeof(uint64_t)), *end = calloc(NN, sizeof(uint64_t));
        uint32_t *queue = malloc(sizeof(uint32_t) * NN), qh = 0, qt = 0;
        for (uint32_t v = 0; v < NN; v++) if (indeg[v] == 0) queue[qt++] = v;
        while (qh < qt) {
            uint32_t v = queue[qh++];
            end[v] = start[v] + lat[v];
            for (uint32_t q = soff[v]; q < soff[v + 1]; q++) {
                uint32_t e = sorder[q], d = edst[e];
                uint64_t cand = end[v] + ew[e];
                if (cand > start[d]) start[d] = cand;
                if (--indeg[d] == 0) queue[qt++] = d;
            }
        }
        /* O9: memory per rank in slot order (order only; also for DEADLOCK), in u32 KiB (R-9: the
         * load-time guard keeps a rank's activation sum below 2^32 KiB, so a valid order never wraps;
         * an order that releases a backward before its forward -- a DEADLOCK -- wraps modulo 2^32) */
        uint32_t oom = 0;
        for (uint32_t r = 0; r < P; r++) {
            uint32_t cur = 0, peak = 0;
            for (uint32_t t = 0; t < S; t++) {
                uint32_t node = r * S + t;
                if (dir[node] == 0) { cur += (uint32_t)act[node]; if (cur > peak) peak = cur; }
                else cur -= (uint32_t)act[node];
            }
            if (peaks) peaks[r] = peak;
            if (peak > pb->budget_kib[r]) oom |= 1u << r;
        }
        res->oom_mask = oom;
        if (qt < NN) {
            res->status = ST_DEADLOCK;            /* fewer than P*2n nodes popped: a cycle */
        } else {
            /* O10 */
            uint64_t mk = 0, busy = 0;
            for (uint32_t v = 0; v < NN; v++) { if (end[v] > mk) mk = end[v]; busy += lat[v]; }
            res->makespan = mk;
            res->busy = busy;
            uint64_t den = (uint64_t)P * mk;
            res->bubble = den ? (double)(den - busy) / (double)den : 0.0;
            res->status = oom ? ST_OOM : ST_OK;
            if (tl_start)
                for (uint32_t v = 0; v < NN; v++) { tl_start[v] = start[v]; tl_end[v] = end[v]; }
        }
        free(dir); free(seg); free(lat); free(act); free(slotF); free(slotB);
        free(esrc); free(edst); free(ew); free(indeg); free(soff); free(sorder); free(fill);
        free(start); free(end); free(queue);
    }
done:
    free(base); free(W); free(present); free(sb); free(si); free(sj); free(sk);
}

typedef struct {
    const oproblem *pb;
    const ocands *cs;
    uint64_t lo, hi, first;
    uint64_t *makespan, *busy, *peaks;
    uint32_t *status, *oom;
    double *bubble;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    for (uint64_t x = j->lo; x < j->hi; x++) {
        ores r;
        uint64_t o = x - j->first;
        eval_one(j->pb, j->cs, x, &r, j->peaks ? j->peaks + o * j->pb->P : NULL, NULL, NULL, NULL);
        j->makespan[o] = r.makespan;
        j->busy[o] = r.busy;
        j->status[o] = r.status;
        j->oom[o] = r.oom_mask;
        j->bubble[o] = r.bubble;
    }
    return NULL;
}

/* Evaluate candidates [first, first+count) of cs (indices into cs arrays). */
int oracle_eval(const oproblem *pb, const ocands *cs, uint64_t first, uint64_t count,
                uint64_t *makespan, uint32_t *status, uint32_t *oom_mask, double *bubble,
                uint64_t *peaks /* [count][P] or NULL */, uint64_t *busy, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    if ((uint64_t)threads > count) threads = count ? (int)count : 1;
    pthread_t th[512];
    job_t jobs[512];
    uint64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        uint64_t lo = first + per * t, hi = lo + per;
        if (hi > first + count) hi = first + count;
        if (lo > hi) lo = hi;
        jobs[t] = (job_t){pb, cs, lo, hi, first, makespan, busy, peaks, status, oom_mask, bubble};
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* Per-(rank, slot) start/end times of candidate x ([P][2n] each); returns the status. */
int oracle_timeline(const oproblem *pb, const ocands *cs, uint64_t x, uint64_t *tl_start, uint64_t *tl_end) {
    ores r;
    eval_one(pb, cs, x, &r, NULL, tl_start, tl_end, NULL);
    return (int)r.status;
}

/* ======================================================================================
 * I1-I6: DIP's greedy dual-queue stage interleaving (§5.2), the row f1 of
 * given a split and segment priorities (the forward and backward priority orders
 * = fwd_seq / bwd_seq of a candidate: position p = priority rank, 0 highest; its F/B bits are
 * ignored), build every rank's stage order and its timing. Readings:
 *   I1 the split and the priority orders are validated as O2-O4 (else BAD_ENCODING).
 *   I2 stage costs as O6.
 *   I3 every rank keeps two priority queues of its unscheduled forward / backward stages
 *      (P:527-528); a stage's t_start is finite once all its predecessors (the cross-rank edges of
 *      O7) are scheduled: the max over them of end + transfer; the queue's minimum
 *      start time t_fw / t_bw is the min over its stages ("among stages in Q_fw and Q_bw",
 *      reading R-29: every queued stage counts, the queue's priority orders its ready stages).
 *   I4 memory gating (R-30): a forward stage whose activation would take the rank
 *      above its budget is disabled (not counted in t_fw and not schedulable).
 *   I5 the rank with the smallest t_min = min(t_fw, t_bw), ties to the lowest rank; if
 *      every rank is blocked by its gates only, the gates are lifted for one step (R-31: the rank
 *      of the smallest gated forward t_start) and the overflow shows as OOM.
 *   I6 steps 2-4: the direction -- if t_fw < t_last and t_bw < t_last, alternate on
 *      the last scheduled type (1F1B emulation; forward first), otherwise the queue of the smaller
 *      minimum start time (step 4 "the stage with the smallest t_start", ties to the backward,
 *      R-29) -- then that queue's highest-priority stage among those that start as early as its
 *      earliest one (t_start <= max(t_dir, t_last)). The stage starts at max(t_start, t_last).
 * The stage DAG is acyclic, so every step schedules a stage: no DEADLOCK. The output is each
 * rank's order: ord[r][t] = segment id | direction << 15 (1 = backward).
 * ====================================================================================== */
#define ORD_B 0x8000u
static void interleave_one(const oproblem *pb, const ocands *cs, uint64_t x, uint16_t *ord_out /* [P][2 n_max] */,
                           ores *res, uint64_t *peaks) {
    const uint32_t P = pb->P, nm = pb->nmod, m = pb->m;
    const uint32_t n_max = cs->n_max;
    const uint8_t *split = cs->split + x * (uint64_t)m * nm;
    const uint16_t *fwd = cs->fwd + x * (uint64_t)n_max;
    const uint16_t *bwd = cs->bwd + x * (uint64_t)n_max;
    const uint32_t ncand = cs->n[x];
    res->makespan = UINT64_MAX; res->busy = 0; res->status = ST_BAD; res->oom_mask = 0; res->bubble = -1.0;
    for (uint32_t r = 0; r < P; r++) { if (peaks) peaks[r] = 0; }
    for (size_t t = 0; t < (size_t)P * 2 * n_max; t++) ord_out[t] = 0xFFFF;

    /* I1 (= O1-O4 without the bit strings): segment ids, split, work units, sequences */
    uint32_t idmax = seg_count_max(pb);
    uint32_t *base = malloc(sizeof(uint32_t) * (m * nm + 1));
    uint32_t *W = calloc(idmax + 1, sizeof(uint32_t));
    uint8_t *present = calloc(idmax + 1, 1);
    uint32_t *sb = malloc(sizeof(uint32_t) * (idmax + 1)), *si = malloc(sizeof(uint32_t) * (idmax + 1));
    uint32_t *sj = malloc(sizeof(uint32_t) * (idmax + 1)), *sk = malloc(sizeof(uint32_t) * (idmax + 1));
    uint32_t *prio = malloc(sizeof(uint32_t) * 2 * (idmax + 1));     /* [dir][s]: position in its order */
    int bad = 0;
    uint32_t acc = 0, n = 0;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            base[b * nm + i] = acc;
            for (uint32_t j = 0; j < pb->max_split[i]; j++)
                for (uint32_t k = 0; k < pb->K[i]; k++) {
                    uint32_t id = acc + j * pb->K[i] + k;
                    sb[id] = b; si[id] = i; sj[id] = j; sk[id] = k;
                }
            acc += pb->max_split[i] * pb->K[i];
        }
    for (uint32_t b = 0; b < m && !bad; b++)
        for (uint32_t i = 0; i < nm; i++) {
            uint32_t q = b * nm + i;
            uint32_t lo = pb->inst_off[q], N = pb->inst_off[q + 1] - lo, M = split[q];
            uint32_t cap = N < pb->max_split[i] ? N : pb->max_split[i];
            if ((N == 0) != (M == 0) || M > cap) { bad = 1; break; }
            if (M == 0) continue;
            uint32_t st[16];
            oracle_split(N, M, st);
            for (uint32_t j = 0; j < M; j++) {
                uint32_t w = 0;
                for (uint32_t u = st[j]; u < st[j + 1]; u++) w += pb->inst_units[lo + u];
                for (uint32_t k = 0; k < pb->K[i]; k++) {
                    uint32_t id = base[q] + j * pb->K[i] + k;
                    present[id] = 1; W[id] = w; n++;
                }
            }
        }
    if (!bad && (ncand != n || n > n_max)) bad = 1;
    if (!bad) {
        uint8_t *seenF = calloc(idmax + 1, 1), *seenB = calloc(idmax + 1, 1);
        for (uint32_t p = 0; p < n_max && !bad; p++) {
            if (p < n) {
                uint32_t a = fwd[p], c = bwd[p];
                if (a >= idmax || c >= idmax || !present[a] || !present[c] || seenF[a] || seenB[c]) bad = 1;
                else { seenF[a] = 1; seenB[c] = 1; prio[a] = p; prio[idmax + 1 + c] = p; }
            } else if (fwd[p] != 0xFFFF || bwd[p] != 0xFFFF) bad = 1;
        }
        free(seenF); free(seenB);
    }
    if (bad) goto done;
    if (n == 0) { res->makespan = 0; res->status = ST_OK; res->bubble = 0.0; goto done; }
    {
        /* node (dir, s, r) -> index (r * 2 + dir) * (idmax + 1) + s */
        const uint32_t IS = idmax + 1, NN = P * 2 * IS;
#define NODE(dir, s, r) (((r) * 2u + (dir)) * IS + (s))
#define LAYERS(i, k, r) ((uint64_t)layers_of(pb, (i), (k) * P + (r)))
#define LAT(dir, s, r) (LAYERS(si[s], sk[s], r) * (uint64_t)((dir) ? pb->tab_b[pb->tab_off[si[s]] + W[s]] : pb->tab_f[pb->tab_off[si[s]] + W[s]]))
#define ACT(s, r) (LAYERS(si[s], sk[s], r) * (uint64_t)pb->tab_act[pb->tab_off[si[s]] + W[s]])
#define P2P(s) ((uint64_t)pb->tab_p2p[pb->tab_off[si[s]] + W[s]])
        uint32_t *indeg = calloc(NN, sizeof(uint32_t));   /* predecessors not yet scheduled */
        uint64_t *tst = calloc(NN, sizeof(uint64_t));     /* running max of pred end + transfer */
        uint64_t *endt = calloc(NN, sizeof(uint64_t));
        /* per rank and direction: the ready list (segment ids) */
        uint32_t *rl = malloc(sizeof(uint32_t) * (size_t)P * 2 * IS), *rc = calloc(P * 2, sizeof(uint32_t));
        uint64_t *tlast = calloc(P, sizeof(uint64_t)), *cur = calloc(P, sizeof(uint64_t)), *pk = calloc(P, sizeof(uint64_t));
        uint32_t *cnt = calloc(P, sizeof(uint32_t));
        int *last = malloc(sizeof(int) * P);
        for (uint32_t r = 0; r < P; r++) last[r] = -1;
        /* I3: predecessor counts (the cross-rank edges of O7; succ() below enumerates the same edges) */
        for (uint32_t s = 0; s < idmax; s++) {
            if (!present[s]) continue;
            uint32_t b = sb[s], i = si[s], k = sk[s], K = pb->K[i];
            for (uint32_t r = 0; r < P; r++) {
                uint32_t dF = 0, dB = 0;
                if (r > 0) dF = 1;
                else if (k > 0) dF = 1;
                else for (uint32_t ip = 0; ip < nm; ip++) if ((pb->producer_mask[i] >> ip) & 1u) dF += split[b * nm + ip];
                if (r + 1 < P) dB = 1;
                else if (k + 1 < K) dB = 1;
                else {
                    for (uint32_t ic = 0; ic < nm; ic++) if ((pb->producer_mask[ic] >> i) & 1u) dB += split[b * nm + ic];
                    if (dB == 0) dB = 1;                                 /* loss turnaround (R-6) */
                }
                indeg[NODE(0, s, r)] = dF;
                indeg[NODE(1, s, r)] = dB;
                if (dF == 0) rl[(r * 2 + 0) * IS + rc[r * 2 + 0]++] = s;
            }
        }
        uint64_t mk = 0, busy = 0;
        int dead = 0;
        for (uint32_t step = 0; step < P * 2 * n; step++) {
            /* I3 / I4: per rank, t_fw over its ungated ready forwards, t_bw over its ready backwards,
               and the smallest forward t_start regardless of the gate (for R-31) */
            uint64_t tf[32], tb[32], tg[32];
            for (uint32_t r = 0; r < P; r++) {
                tf[r] = tb[r] = tg[r] = UINT64_MAX;
                for (uint32_t a = 0; a < rc[r * 2 + 0]; a++) {
                    uint32_t s = rl[(r * 2 + 0) * IS + a];
                    uint64_t t = tst[NODE(0, s, r)];
                    if (t < tg[r]) tg[r] = t;
                    if (cur[r] + ACT(s, r) <= pb->budget_kib[r] && t < tf[r]) tf[r] = t;
                }
                for (uint32_t a = 0; a < rc[r * 2 + 1]; a++) {
                    uint64_t t = tst[NODE(1, rl[(r * 2 + 1) * IS + a], r)];
                    if (t < tb[r]) tb[r] = t;
                }
            }
            /* I5 */
            int rr = -1, relax = 0;
            uint64_t best = UINT64_MAX;
            for (uint32_t r = 0; r < P; r++) {
                uint64_t tm = tf[r] < tb[r] ? tf[r] : tb[r];
                if (tm < best) { best = tm; rr = (int)r; }
            }
            if (rr < 0) {                       /* every rank blocked by its gates only (R-31) */
                for (uint32_t r = 0; r < P; r++)
                    if (tg[r] < best) { best = tg[r]; rr = (int)r; }
                relax = 1;
            }
            if (rr < 0) { dead = 1; break; }    /* unreachable: the stage DAG is acyclic */
            const uint32_t r = (uint32_t)rr;
            const uint64_t fmin = relax ? tg[r] : tf[r], bmin = tb[r];
            /* I6: the direction (step 3: alternate; step 4: the smaller of t_fw / t_bw, ties to the
               backward), then that queue's highest-priority stage among those that start as early as
               its earliest one, i.e. with t_start <= max(t_dir, t_last) */
            int dir;
            if (fmin != UINT64_MAX && bmin != UINT64_MAX && fmin < tlast[r] && bmin < tlast[r])
                dir = last[r] == 0 ? 1 : 0;                         /* emulate 1F1B: alternate */
            else if (fmin == UINT64_MAX) dir = 1;
            else if (bmin == UINT64_MAX) dir = 0;
            else dir = bmin <= fmin ? 1 : 0;                        /* smallest t_start; ties -> B */
            const uint64_t tdir = dir ? bmin : fmin, lim = tdir > tlast[r] ? tdir : tlast[r];
            uint32_t pick = 0, bp = UINT32_MAX;
            for (uint32_t a = 0; a < rc[r * 2 + dir]; a++) {
                uint32_t s = rl[(r * 2 + dir) * IS + a];
                if (tst[NODE(dir, s, r)] > lim) continue;
                if (dir == 0 && !relax && cur[r] + ACT(s, r) > pb->budget_kib[r]) continue;
                if (prio[dir * IS + s] < bp) { bp = prio[dir * IS + s]; pick = s; }
            }
            /* place (dir, pick) on rank r */
            const uint32_t s = pick, nd = NODE(dir, s, r);
            for (uint32_t a = 0; a < rc[r * 2 + dir]; a++)          /* dequeue */
                if (rl[(r * 2 + dir) * IS + a] == s) { rl[(r * 2 + dir) * IS + a] = rl[(r * 2 + dir) * IS + --rc[r * 2 + dir]]; break; }
            uint64_t st = tst[nd] > tlast[r] ? tst[nd] : tlast[r];
            uint64_t lat = LAT(dir, s, r), en = st + lat;
            endt[nd] = en;
            tlast[r] = en;
            last[r] = dir;
            busy += lat;
            if (en > mk) mk = en;
            ord_out[(size_t)r * 2 * n_max + cnt[r]++] = (uint16_t)(s | (dir ? ORD_B : 0u));
            if (dir) cur[r] -= ACT(s, r);
            else { cur[r] += ACT(s, r); if (cur[r] > pk[r]) pk[r] = cur[r]; }
            /* successors (the edges of O7): their t_start and readiness */
            uint32_t b = sb[s], i = si[s], k = sk[s], K = pb->K[i];
#define RELEASE(D2, S2, R2, WT) do { uint32_t v_ = NODE((D2), (S2), (R2)); \
            if (en + (WT) > tst[v_]) tst[v_] = en + (WT); \
            if (--indeg[v_] == 0) rl[((R2) * 2 + (D2)) * IS + rc[(R2) * 2 + (D2)]++] = (S2); } while (0)
            if (dir == 0) {
                if (r + 1 < P) RELEASE(0, s, r + 1, P2P(s));
                else if (k + 1 < K) RELEASE(0, s + 1, 0, P > 1 ? P2P(s) : 0);
                else {
                    int any = 0;
                    for (uint32_t ic = 0; ic < nm; ic++) {
                        if (!((pb->producer_mask[ic] >> i) & 1u)) continue;
                        for (uint32_t jc = 0; jc < split[b * nm + ic]; jc++) {
                            RELEASE(0, base[b * nm + ic] + jc * pb->K[ic], 0, P > 1 ? P2P(s) : 0);
                            any = 1;
                        }
                    }
                    if (!any) RELEASE(1, s, P - 1, 0);                   /* loss turnaround (R-6) */
                }
            } else {
                if (r > 0) RELEASE(1, s, r - 1, P2P(s));
                else if (k > 0) RELEASE(1, s - 1, P - 1, P > 1 ? P2P(s - 1) : 0);
                else
                    for (uint32_t ip = 0; ip < nm; ip++) {
                        if (!((pb->producer_mask[i] >> ip) & 1u)) continue;
                        for (uint32_t jp = 0; jp < split[b * nm + ip]; jp++) {
                            uint32_t pr = base[b * nm + ip] + jp * pb->K[ip] + pb->K[ip] - 1;
                            RELEASE(1, pr, P - 1, P > 1 ? P2P(pr) : 0);
                        }
                    }
            }
#undef RELEASE
        }
        uint32_t oom = 0;
        for (uint32_t r = 0; r < P; r++) {
            if (peaks) peaks[r] = pk[r];
            if (pk[r] > pb->budget_kib[r]) oom |= 1u << r;
        }
        res->oom_mask = oom;
        if (dead) {
            res->status = ST_DEADLOCK;
        } else {
            res->makespan = mk;
            res->busy = busy;
            uint64_t den = (uint64_t)P * mk;
            res->bubble = den ? (double)(den - busy) / (double)den : 0.0;
            res->status = oom ? ST_OOM : ST_OK;
        }
#undef LAYERS
#undef LAT
#undef ACT
#undef P2P
#undef NODE
        free(indeg); free(tst); free(endt); free(rl); free(rc); free(tlast); free(cur); free(pk); free(cnt); free(last);
    }
done:
    free(base); free(W); free(present); free(sb); free(si); free(sj); free(sk); free(prio);
}

typedef struct {
    const oproblem *pb;
    const ocands *cs;
    uint64_t lo, hi, first;
    uint16_t *ord;
    uint64_t *makespan, *busy, *peaks;
    uint32_t *status, *oom;
    double *bubble;
} ijob_t;

static void *iworker(void *arg) {
    ijob_t *j = (ijob_t *)arg;
    const uint32_t P = j->pb->P, n_max = j->cs->n_max;
    for (uint64_t x = j->lo; x < j->hi; x++) {
        ores r;
        uint64_t o = x - j->first;
        interleave_one(j->pb, j->cs, x, j->ord + o * P * 2 * n_max, &r, j->peaks ? j->peaks + o * P : NULL);
        j->makespan[o] = r.makespan; j->busy[o] = r.busy; j->status[o] = r.status;
        j->oom[o] = r.oom_mask; j->bubble[o] = r.bubble;
    }
    return NULL;
}

/* Interleave candidates [first, first+count): writes each one's per-rank orders
 * ([count][P][2 n_max], id | 0x8000 for backward) and the resulting schedule's score (as oracle_eval). */
int oracle_interleave(const oproblem *pb, const ocands *cs, uint64_t first, uint64_t count, uint16_t *ord,
                      uint64_t *makespan, uint32_t *status, uint32_t *oom_mask, double *bubble, uint64_t *peaks,
                      uint64_t *busy, int threads) {
    if (pb->P > 32) return -1;
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    if ((uint64_t)threads > count) threads = count ? (int)count : 1;
    pthread_t th[512];
    ijob_t jobs[512];
    uint64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        uint64_t lo = first + per * t, hi = lo + per;
        if (hi > first + count) hi = first + count;
        if (lo > hi) lo = hi;
        jobs[t] = (ijob_t){pb, cs, lo, hi, first, ord, makespan, busy, peaks, status, oom_mask, bubble};
        pthread_create(&th[t], NULL, iworker, &jobs[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* ======================================================================================
 * S1-S6: DIP's MCTS segment reordering (§5.1), the row f2 of SURVEY §8(f),
 * written step by step from the paper with the readings of DESIGN.md §3 (R-32..R-35):
 *   S1 classes: (direction, microbatch b, module i, chunk k) with M_{b,i} > 0 -- the M_{b,i}
 *      sub-microbatch segments of one modality, microbatch and chunk share a priority and keep a
 *      fixed order, j ascending (reading R-32); forward classes in (b, i, k) order, then
 *      the backward classes in the same order.
 *   S2 a sequence (permutation of the Cn classes) gives priority Cn-1-p to the class at position p
 *      (P:481); the forward / backward queue order of a rank = repeatedly the ready segment of the
 *      highest priority (within a class: j ascending).
 *   S3 rollout score: interleave (I1-I6) -- and, if a strategy menu is given, the per-layer
 *      memory optimisation (M1-M4, "undergoes pipeline stage interleaving ... and per-layer
 *      memory optimization") -- and score LB / makespan if OK, else 0, with LB the busiest rank's
 *      summed latency of the split (base tables).
 *   S4 selection: from the root, while the node has all its children, move to the child of
 *      largest s^alpha + beta * sqrt(ln N_x / N_v) (ties: first child, i.e. lowest class); counts
 *      include the virtual visits of the current round.
 *   S5 expansion: add the child of the next unused class in class order; rollouts:
 *      `rollouts` uniformly random completions (one if the sequence is complete), the u-th rollout
 *      drawing from a splitmix64 stream seeded with splitmix64(seed ^ splitmix64(u + 0x51A9)).
 *   S6 backpropagation: along the path, s = max(s, best trial), N += 1.
 *   A round selects `leaves` leaves (virtual visit on every node of each path), then scores all
 *   their rollouts, then backpropagates leaf by leaf.
 * ====================================================================================== */
static uint64_t smix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct { int parent, cls, depth, nch, cap; int *ch; double s; uint32_t N, vl; } snode;

/* M1-M4 (below): per-layer memory optimisation of one schedule, used by S3 when a menu is given */
typedef struct {
    uint32_t n_strat, S;
    const uint32_t *f, *b, *act;    /* [n_strat][tab_off[nmod]] per-layer menu (M1) */
    uint32_t gap_pm, node_cap;      /* M3: optimality gap in per mille, B&B child budget */
} omenu;
static void memopt_one(const oproblem *pb, const omenu *mn, const ocands *cs, uint64_t x, uint8_t *sel,
                       ores *res, uint64_t *peaks, uint64_t *rstats);

/* S2: queue order of one direction from class priorities (plain selection, O(n^2)) */
static void s_order(const oproblem *pb, const uint8_t *split, const uint32_t *base, const int *clsof, uint32_t C,
                    uint32_t Cn, const uint32_t *prio, int dir, uint32_t n_max, uint16_t *out) {
    const uint32_t nm = pb->nmod, m = pb->m;
    uint32_t idmax = seg_count_max(pb);
    int32_t *indeg = malloc(sizeof(int32_t) * (idmax + 1));
    uint64_t *key = malloc(sizeof(uint64_t) * (idmax + 1));
    uint8_t *ready = calloc(idmax + 1, 1);
    uint32_t n = 0;
    for (uint32_t x = 0; x <= idmax; x++) indeg[x] = -1;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            uint32_t q = b * nm + i, K = pb->K[i];
            for (uint32_t j = 0; j < split[q]; j++)
                for (uint32_t k = 0; k < K; k++) {
                    uint32_t s = base[q] + j * K + k;
                    int32_t d = 0;
                    if (dir == 0) {
                        if (k > 0) d = 1;
                        else for (uint32_t p = 0; p < nm; p++) if ((pb->producer_mask[i] >> p) & 1u) d += split[b * nm + p];
                    } else {
                        if (k + 1 < K) d = 1;
                        else for (uint32_t c = 0; c < nm; c++) if ((pb->producer_mask[c] >> i) & 1u) d += split[b * nm + c];
                    }
                    indeg[s] = d;
                    uint32_t c = (uint32_t)clsof[q] + k + (dir ? C : 0);
                    key[s] = ((uint64_t)(Cn - 1 - prio[c]) << 40) | ((uint64_t)j << 24);
                    if (d == 0) ready[s] = 1;
                    n++;
                }
        }
    for (uint32_t cnt = 0; cnt < n; cnt++) {
        uint32_t pick = 0xFFFFFFFFu;
        for (uint32_t s = 0; s < idmax; s++)
            if (ready[s] && (pick == 0xFFFFFFFFu || key[s] < key[pick])) pick = s;
        out[cnt] = (uint16_t)pick;
        ready[pick] = 0;
        /* successors of pick in this direction */
        uint32_t q = 0;
        while (q + 1 < m * nm && base[q + 1] <= pick) q++;
        uint32_t b = q / nm, i = q % nm, K = pb->K[i], k = (pick - base[q]) % K;
        if (dir == 0) {
            if (k + 1 < K) { if (--indeg[pick + 1] == 0) ready[pick + 1] = 1; }
            else for (uint32_t c = 0; c < nm; c++)
                if ((pb->producer_mask[c] >> i) & 1u)
                    for (uint32_t jj = 0; jj < split[b * nm + c]; jj++) {
                        uint32_t t = base[b * nm + c] + jj * pb->K[c];
                        if (--indeg[t] == 0) ready[t] = 1;
                    }
        } else {
            if (k > 0) { if (--indeg[pick - 1] == 0) ready[pick - 1] = 1; }
            else for (uint32_t p = 0; p < nm; p++)
                if ((pb->producer_mask[i] >> p) & 1u)
                    for (uint32_t jj = 0; jj < split[b * nm + p]; jj++) {
                        uint32_t t = base[b * nm + p] + jj * pb->K[p] + pb->K[p] - 1;
                        if (--indeg[t] == 0) ready[t] = 1;
                    }
        }
    }
    for (uint32_t p = n; p < n_max; p++) out[p] = 0xFFFF;
    free(indeg); free(key); free(ready);
}

/* S4-S6 + the rollout draws: the MCTS loop over sequences of Cn classes, with the rollout scoring
 * (S3) left to `score` (count sequences [count][Cn] -> scores). Returns the number of tree nodes;
 * optional outputs: trace [rounds] best score after each round, leaves_out [rounds][leaves] the
 * selected / expanded leaf of every slot, the tree (parent, class, N, s) of every node. */
typedef void (*mcts_score_fn)(void *ctx, uint32_t count, const uint32_t *seqs, const int *owner, double *scores);
/* policy (the paper's search-efficiency comparison): 0 = MCTS (UCB selection, S4-S5);
 * 1 = random exploration (every leaf is the root: all rollouts are uniformly random sequences);
 * 2 = depth-first search (the leaf is the next node of a pre-order traversal of the sequence tree,
 * children in class order: expand the previous leaf if it is incomplete, else its nearest ancestor
 * with an unexpanded child). Rollouts, scoring and backpropagation are the same for all three. */
static uint32_t mcts_run(uint32_t Cn, uint64_t seed, uint32_t rounds, uint32_t leaves, uint32_t rollouts,
                         double alpha, double beta, mcts_score_fn score, void *ctx, double *trace,
                         int32_t *leaves_out, int32_t *t_parent, int32_t *t_cls, uint32_t *t_N, double *t_s,
                         uint64_t *scored_out, uint32_t policy) {
    uint32_t ncap = 1 + rounds * leaves, nn = 1;
    snode *T = calloc(ncap, sizeof(snode));
    T[0].parent = -1; T[0].cls = -1; T[0].depth = 0;
    uint32_t maxr = leaves * rollouts;
    uint32_t *seqs = malloc(sizeof(uint32_t) * (size_t)(maxr ? maxr : 1) * Cn);
    double *sc = malloc(sizeof(double) * (maxr ? maxr : 1));
    int *owner = malloc(sizeof(int) * (maxr ? maxr : 1)), *leaf = malloc(sizeof(int) * leaves);
    uint32_t *seq = malloc(sizeof(uint32_t) * Cn), *rest = malloc(sizeof(uint32_t) * Cn);
    uint8_t *used = malloc(Cn);
    double best = -1.0;
    uint64_t u = 0;
    int dfs_cur = 0;
    *scored_out = 0;
    for (uint32_t rd = 0; rd < rounds; rd++) {
        uint32_t cnt = 0;
        for (uint32_t l = 0; l < leaves; l++) {
            int v = 0;
            memset(used, 0, Cn);
            if (policy == 2) {                                   /* DFS: climb from the previous leaf */
                v = dfs_cur;
                while (v > 0 && (uint32_t)T[v].nch >= Cn - (uint32_t)T[v].depth) v = T[v].parent;
                if (v == 0 && (uint32_t)T[0].nch >= Cn) v = dfs_cur;   /* the whole tree is explored */
                for (int x = v; x > 0; x = T[x].parent) used[T[x].cls] = 1;
            }
            for (; policy != 1;) {                               /* S4 / S5 (random: the root) */
                snode *nd = &T[v];
                if ((uint32_t)nd->depth == Cn) break;
                if ((uint32_t)nd->nch < Cn - nd->depth) {        /* S5: the next unused class */
                    uint32_t c, seen = 0;
                    for (c = 0; c < Cn; c++) { if (used[c]) continue; if (seen++ == (uint32_t)nd->nch) break; }
                    int id = (int)nn++;
                    T[id].parent = v; T[id].cls = (int)c; T[id].depth = nd->depth + 1;
                    if (nd->nch == nd->cap) { nd->cap = nd->cap ? 2 * nd->cap : 4; nd->ch = realloc(nd->ch, sizeof(int) * nd->cap); }
                    nd->ch[nd->nch++] = id;
                    used[c] = 1;
                    v = id;
                    break;
                }
                if (policy == 2) break;                          /* DFS: a complete leaf again */
                double Nx = (double)(nd->N + nd->vl), bu = -1.0;   /* S4: UCB */
                int bc = -1;
                for (int x = 0; x < nd->nch; x++) {
                    snode *cn = &T[nd->ch[x]];
                    double Nv = (double)(cn->N + cn->vl);
                    double ucb = pow(cn->s, alpha) + beta * sqrt(log(Nx) / Nv);
                    if (ucb > bu) { bu = ucb; bc = nd->ch[x]; }
                }
                used[T[bc].cls] = 1;
                v = bc;
            }
            for (int x = v; x >= 0; x = T[x].parent) T[x].vl++;
            leaf[l] = v;
            dfs_cur = v;
            if (leaves_out) leaves_out[rd * leaves + l] = v;
            uint32_t d = (uint32_t)T[v].depth;
            for (int x = v; x > 0; x = T[x].parent) seq[T[x].depth - 1] = (uint32_t)T[x].cls;
            uint32_t trials = d == Cn ? 1 : rollouts;
            for (uint32_t tr = 0; tr < trials; tr++) {           /* rollouts: random completions */
                uint32_t nr = 0;
                for (uint32_t c = 0; c < Cn; c++) {
                    int on = 0;
                    for (uint32_t p = 0; p < d; p++) if (seq[p] == c) on = 1;
                    if (!on) rest[nr++] = c;
                }
                uint64_t rs = smix(seed ^ smix(u + 0x51A9u));
                for (uint32_t x = nr; x > 1; x--) {
                    rs += 0x9E3779B97F4A7C15ull;
                    uint32_t y = (uint32_t)(smix(rs) % x), t2 = rest[x - 1];
                    rest[x - 1] = rest[y]; rest[y] = t2;
                }
                for (uint32_t x = 0; x < nr; x++) seq[d + x] = rest[x];
                memcpy(seqs + (size_t)cnt * Cn, seq, sizeof(uint32_t) * Cn);
                owner[cnt] = (int)l;
                cnt++;
                u++;
            }
        }
        score(ctx, cnt, seqs, owner, sc);                        /* S3 */
        double *lb = calloc(leaves, sizeof(double));
        for (uint32_t x = 0; x < cnt; x++) {
            if (sc[x] > lb[owner[x]]) lb[owner[x]] = sc[x];
            if (sc[x] > best) best = sc[x];
        }
        *scored_out += cnt;
        for (uint32_t l = 0; l < leaves; l++)                       /* S6 */
            for (int x = leaf[l]; x >= 0; x = T[x].parent) {
                if (lb[l] > T[x].s) T[x].s = lb[l];
                T[x].N++;
                T[x].vl--;
            }
        free(lb);
        if (trace) trace[rd] = best;
    }
    for (uint32_t x = 0; x < nn; x++) {
        if (t_parent) t_parent[x] = T[x].parent;
        if (t_cls) t_cls[x] = T[x].cls;
        if (t_N) t_N[x] = T[x].N;
        if (t_s) t_s[x] = T[x].s;
        free(T[x].ch);
    }
    free(T); free(seqs); free(sc); free(owner); free(leaf); free(seq); free(rest); free(used);
    return nn;
}

/* The MCTS loop alone, scored by a table over the first two classes of a sequence:
 * score(seq) = table[seq[0] * Cn + seq[1]] (a test fixture for S4-S6, independent of f1). */
typedef struct { uint32_t Cn; const double *table; } tab_ctx;
static void tab_score(void *ctx, uint32_t count, const uint32_t *seqs, const int *owner, double *scores) {
    (void)owner;
    tab_ctx *t = (tab_ctx *)ctx;
    for (uint32_t x = 0; x < count; x++) {
        const uint32_t *q = seqs + (size_t)x * t->Cn;
        scores[x] = t->table[q[0] * t->Cn + (t->Cn > 1 ? q[1] : 0)];
    }
}
uint32_t oracle_mcts_table(uint32_t Cn, uint64_t seed, uint32_t rounds, uint32_t leaves, uint32_t rollouts,
                           double alpha, double beta, const double *table, double *trace, int32_t *leaves_out,
                           int32_t *t_parent, int32_t *t_cls, uint32_t *t_N, double *t_s, uint32_t policy) {
    tab_ctx c = {Cn, table};
    uint64_t scored;
    return mcts_run(Cn, seed, rounds, leaves, rollouts, alpha, beta, tab_score, &c, trace, leaves_out, t_parent,
                    t_cls, t_N, t_s, &scored, policy);
}

/* S1-S3 for oracle_search: a class sequence -> priority orders (S2) -> interleaving (I1-I6, orders)
 * -> optionally M1-M4 -> LB / makespan */
typedef struct {
    const oproblem *pb;
    const omenu *mn;
    uint32_t n_max, fbw, n, C, Cn;
    const uint8_t *split;
    const uint32_t *base;
    const int *clsof;
    double LB, best;
    uint64_t *best_makespan;
    uint16_t *best_fwd, *best_bwd, *best_ord;
} srch_ctx;

static void search_score(void *ctxp, uint32_t cnt, const uint32_t *seqs, const int *owner, double *scores) {
    (void)owner;
    srch_ctx *c = (srch_ctx *)ctxp;
    const oproblem *pb = c->pb;
    const uint32_t P = pb->P, nm = pb->nmod, m = pb->m, n_max = c->n_max, Cn = c->Cn;
    uint8_t *spl = malloc((size_t)(cnt ? cnt : 1) * m * nm);
    uint32_t *nn_ = malloc(sizeof(uint32_t) * (cnt ? cnt : 1)), *prio = malloc(sizeof(uint32_t) * Cn);
    uint16_t *fw = malloc(sizeof(uint16_t) * (size_t)(cnt ? cnt : 1) * n_max), *bw = malloc(sizeof(uint16_t) * (size_t)(cnt ? cnt : 1) * n_max);
    uint32_t *fb = calloc((size_t)(cnt ? cnt : 1) * P * c->fbw, sizeof(uint32_t));
    uint16_t *ord = malloc(sizeof(uint16_t) * (size_t)(cnt ? cnt : 1) * P * 2 * n_max);
    for (uint32_t x = 0; x < cnt; x++) {
        for (uint32_t p = 0; p < Cn; p++) prio[seqs[(size_t)x * Cn + p]] = Cn - 1 - p;   /* S2 */
        memcpy(spl + (size_t)x * m * nm, c->split, m * nm);
        nn_[x] = c->n;
        s_order(pb, c->split, c->base, c->clsof, c->C, Cn, prio, 0, n_max, fw + (size_t)x * n_max);
        s_order(pb, c->split, c->base, c->clsof, c->C, Cn, prio, 1, n_max, bw + (size_t)x * n_max);
    }
    ocands cs = {n_max, c->fbw, spl, nn_, fw, bw, fb, NULL};
    for (uint32_t x = 0; x < cnt; x++) {
        ores r;
        uint16_t *ox = ord + (size_t)x * P * 2 * n_max;
        interleave_one(pb, &cs, x, ox, &r, NULL);
        if (c->mn->n_strat && r.status != ST_BAD) {           /* then per-layer memory opt. */
            ocands c1 = {n_max, c->fbw, spl + (size_t)x * m * nm, nn_ + x, fw + (size_t)x * n_max,
                         bw + (size_t)x * n_max, fb + (size_t)x * P * c->fbw, ox};
            uint8_t *sel = malloc((size_t)P * 2 * n_max);
            memopt_one(pb, c->mn, &c1, 0, sel, &r, NULL, NULL);
            free(sel);
        }
        double sc = r.status == ST_OK ? c->LB / (double)r.makespan : 0.0;
        scores[x] = sc;
        if (sc > c->best) {
            c->best = sc;
            *c->best_makespan = r.makespan;
            if (c->best_fwd) memcpy(c->best_fwd, fw + (size_t)x * n_max, sizeof(uint16_t) * n_max);
            if (c->best_bwd) memcpy(c->best_bwd, bw + (size_t)x * n_max, sizeof(uint16_t) * n_max);
            if (c->best_ord) memcpy(c->best_ord, ox, sizeof(uint16_t) * P * 2 * n_max);
        }
    }
    free(spl); free(nn_); free(prio); free(fw); free(bw); free(fb); free(ord);
}

int oracle_search(const oproblem *pb, uint32_t n_max, uint32_t fbw, const uint8_t *split, uint64_t seed,
                  uint32_t rounds, uint32_t leaves, uint32_t rollouts, double alpha, double beta,
                  double *trace, double *best_score, uint64_t *best_makespan, uint16_t *best_fwd,
                  uint16_t *best_bwd, uint16_t *best_ord /* [P][2 n_max] */, uint64_t *scored_out,
                  uint32_t n_strat, const uint32_t *mf, const uint32_t *mb, const uint32_t *ma, uint32_t S,
                  uint32_t policy) {
    omenu mn = {n_strat, S, mf, mb, ma, 50, 4096};   /* n_strat = 0: rollouts are interleaved only */
    const uint32_t P = pb->P, nm = pb->nmod, m = pb->m;
    uint32_t *base = malloc(sizeof(uint32_t) * (m * nm + 1));
    int *clsof = malloc(sizeof(int) * m * nm);
    uint32_t acc = 0, C = 0, n = 0;
    for (uint32_t q = 0; q < m * nm; q++) {
        base[q] = acc;
        acc += pb->max_split[q % nm] * pb->K[q % nm];
        clsof[q] = split[q] ? (int)C : -1;                   /* S1: classes (b, i, 0..K_i-1) */
        if (split[q]) C += pb->K[q % nm];
        n += split[q] * pb->K[q % nm];
    }
    const uint32_t Cn = 2 * C;
    *best_score = 0.0;
    *best_makespan = UINT64_MAX;
    *scored_out = 0;
    if (C == 0) { free(base); free(clsof); return 0; }
    /* S3: LB = the busiest rank's summed latency of this split (O1, O2 of the fixed-order oracle) */
    double LB = 0.0;
    for (uint32_t r = 0; r < P; r++) {
        uint64_t tot = 0;
        for (uint32_t q = 0; q < m * nm; q++) {
            uint32_t i = q % nm, Mv = split[q];
            if (!Mv) continue;
            uint32_t lo = pb->inst_off[q], N = pb->inst_off[q + 1] - lo, st[16];
            oracle_split(N, Mv, st);
            for (uint32_t j = 0; j < Mv; j++) {
                uint32_t w = 0;
                for (uint32_t x = st[j]; x < st[j + 1]; x++) w += pb->inst_units[lo + x];
                for (uint32_t k = 0; k < pb->K[i]; k++)
                    tot += (uint64_t)layers_of(pb, i, k * P + r) *
                           ((uint64_t)pb->tab_f[pb->tab_off[i] + w] + pb->tab_b[pb->tab_off[i] + w]);
            }
        }
        if ((double)tot > LB) LB = (double)tot;
    }
    srch_ctx c = {pb, &mn, n_max, fbw, n, C, Cn, split, base, clsof, LB, -1.0, best_makespan, best_fwd, best_bwd, best_ord};
    mcts_run(Cn, seed, rounds, leaves, rollouts, alpha, beta, search_score, &c, trace, NULL, NULL, NULL, NULL, NULL,
             scored_out, policy);
    *best_score = c.best > 0.0 ? c.best : 0.0;
    if (!(c.best > 0.0)) *best_makespan = UINT64_MAX;     /* no feasible (status OK) rollout */
    free(base); free(clsof);
    return 0;
}

/* O11: lowest index among status OK with minimal makespan; returns -1 if none. */
int64_t oracle_argmin(const uint64_t *makespan, const uint32_t *status, uint64_t count) {
    int64_t best = -1;
    for (uint64_t x = 0; x < count; x++)
        if (status[x] == ST_OK && (best < 0 || makespan[x] < makespan[best])) best = (int64_t)x;
    return best;
}

/* ======================================================================================
 * M1-M4: DIP's per-layer memory optimisation (§5.3), the row f3 of
 * SURVEY §8(f), step by step with the readings of DESIGN.md §3 (R-37..R-40):
 *   M1 menu: every layer of module i has n_strat strategies c with per-layer
 *      (F ns, B ns, activation KiB) at width W -- an input, like the O6 tables; strategy 0 is
 *      the scheme of the O6 tables (the "most memory-efficient scheme" the interleaving uses,
 *      P:522-524).
 *   M2 candidates of a stage pair: the pair = the forward stage and its backward
 *      stage on one rank (chunk of `layers` identical layers at width W); a combination gives one
 *      strategy to each layer (lat = sum F + B, mem = sum act). (1) the fastest combination,
 *      (2) the most memory-efficient one, (3) the range [mem_min, mem_fast] cut evenly into S-2
 *      buckets [lo_u, hi_u) and, in each, the fastest combination whose memory falls in it
 *      (the multiple-choice knapsack optimum, written out as enumeration: the layers are
 *      identical, so a combination is fixed by how many layers take each strategy). Ties: less
 *      memory, then the smaller forward latency. Duplicates and dominated entries dropped;
 *      sorted by memory ascending (so latency strictly decreases).
 *   M3 selection on each rank, the ILP of P:572-582: pairs i with interval
 *      [slot of F, slot of B) in the rank's order; minimise sum_i lat_i (lat = F + B of the
 *      selected candidate) subject to: at every forward slot s_k the selected memory of the pairs
 *      live there stays <= the rank's budget M. Solved as P:584-590 describes, to a relative
 *      optimality gap <= gap (default 5 %), warm-started by a greedy:
 *      M3a warm start: candidate 0 everywhere (the min-memory one, feasible iff the schedule is
 *          not OOM; if it is, nothing changes and M3b/M3c are skipped), then repeatedly move the
 *          pair with the largest latency saving per KiB of extra memory (next candidate; ties:
 *          earliest forward slot) to its next candidate as long as every point it covers keeps
 *          slack.
 *      M3b lower bound (the solver's relaxation bound, reading R-39): a Lagrangian relaxation of
 *          the memory constraints at the points K* where the warm start blocks a pair, with one
 *          multiplier mu (fixed point 2^-16) bracketed by x16 steps and bisected to 1/64 relative
 *          width; every pair then picks its candidate independently and the bound is ceil(L(mu))
 *          at the better end of the bracket, valid for any mu >= 0.
 *      M3c branch and bound: if bound >= (1 - gap) * incumbent the incumbent is within the gap and
 *          is the answer; else depth-first over the pairs in forward order, each pair's candidates
 *          fastest first, a child skipped if it does not fit its points, a subtree entered only
 *          if its bound < (1 - gap) * incumbent, a complete selection taken if strictly better.
 *          At most `node_cap` children are visited (then the incumbent stands; reported).
 *   M4 score: the schedule re-timed (O7-O10) with every pair's selected latencies and
 *      activations.
 * ====================================================================================== */
typedef struct { uint64_t f, b, mem; } mcand;

static int mc_better(const mcand *a, const mcand *b, int by_mem) {   /* strict "a before b" */
    uint64_t la = a->f + a->b, lb = b->f + b->b;
    if (by_mem) {
        if (a->mem != b->mem) return a->mem < b->mem;
        if (la != lb) return la < lb;
    } else {
        if (la != lb) return la < lb;
        if (a->mem != b->mem) return a->mem < b->mem;
    }
    return a->f < b->f;
}

/* M2: out [S][3] = (F ns, B ns, mem KiB) of the pair's candidates; returns their count. */
int oracle_mem_candidates(uint32_t n_strat, const uint32_t *f, const uint32_t *b, const uint32_t *act,
                          uint32_t layers, uint32_t S, uint64_t *out) {
    if (n_strat == 0 || n_strat > 8 || S < 2 || layers == 0) return 0;
    /* every count vector (n_0 .. n_{C-1}) with sum = layers */
    uint32_t cnt[8] = {0}, ncomb = 0, cap = 64;
    mcand *all = malloc(sizeof(mcand) * cap);
    cnt[n_strat - 1] = 0;
    for (;;) {
        uint32_t used = 0;
        for (uint32_t c = 0; c + 1 < n_strat; c++) used += cnt[c];
        if (used <= layers) {
            cnt[n_strat - 1] = layers - used;
            mcand x = {0, 0, 0};
            for (uint32_t c = 0; c < n_strat; c++) {
                x.f += (uint64_t)cnt[c] * f[c];
                x.b += (uint64_t)cnt[c] * b[c];
                x.mem += (uint64_t)cnt[c] * act[c];
            }
            if (ncomb == cap) { cap *= 2; all = realloc(all, sizeof(mcand) * cap); }
            all[ncomb++] = x;
        }
        /* next vector of the first n_strat-1 counts (odometer, each in [0, layers]) */
        uint32_t c = 0;
        while (c + 1 < n_strat) {
            if (++cnt[c] <= layers) break;
            cnt[c] = 0;
            c++;
        }
        if (c + 1 >= n_strat) break;
    }
    mcand *pick = malloc(sizeof(mcand) * S);
    uint32_t np = 0;
    mcand fast = all[0], small = all[0];
    for (uint32_t x = 1; x < ncomb; x++) {
        if (mc_better(&all[x], &fast, 0)) fast = all[x];
        if (mc_better(&all[x], &small, 1)) small = all[x];
    }
    pick[np++] = fast;
    pick[np++] = small;
    if (S > 2 && fast.mem > small.mem) {
        uint64_t span = fast.mem - small.mem;
        for (uint32_t u = 0; u < S - 2; u++) {
            uint64_t lo = small.mem + span * u / (S - 2), hi = small.mem + span * (u + 1) / (S - 2);
            int have = 0;
            mcand best = {0, 0, 0};
            for (uint32_t x = 0; x < ncomb; x++)
                if (all[x].mem >= lo && all[x].mem < hi && (!have || mc_better(&all[x], &best, 0))) { best = all[x]; have = 1; }
            if (have) pick[np++] = best;
        }
    }
    /* drop duplicates and dominated entries, then sort by memory ascending */
    uint32_t k = 0;
    for (uint32_t x = 0; x < np; x++) {
        int drop = 0;
        for (uint32_t y = 0; y < np && !drop; y++) {
            if (y == x) continue;
            uint64_t lx = pick[x].f + pick[x].b, ly = pick[y].f + pick[y].b;
            int same = pick[y].f == pick[x].f && pick[y].b == pick[x].b && pick[y].mem == pick[x].mem;
            if (same && y < x) drop = 1;
            if (!same && pick[y].mem <= pick[x].mem && ly <= lx && (pick[y].mem < pick[x].mem || ly < lx)) drop = 1;
        }
        if (!drop) pick[k++] = pick[x];
    }
    for (uint32_t x = 1; x < k; x++)
        for (uint32_t y = x; y > 0 && pick[y].mem < pick[y - 1].mem; y--) { mcand t = pick[y]; pick[y] = pick[y - 1]; pick[y - 1] = t; }
    for (uint32_t x = 0; x < k; x++) { out[3 * x] = pick[x].f; out[3 * x + 1] = pick[x].b; out[3 * x + 2] = pick[x].mem; }
    free(all); free(pick);
    return (int)k;
}

/* ---------------- M3: the per-rank ILP ----------------
 * n pairs in forward order; pair p is live at point k (the k-th forward slot, sF[k]) iff
 * sF[p] <= sF[k] < sB[p]; cand[(p*Sst + c)*3 + {0,1,2}] = (F, B, mem) of candidate c < nc[p],
 * sorted by memory ascending. cur[p] (out) = the selected candidate. stats (may be NULL):
 * [0] warm-start objective, [1] root bound, [2] final objective, [3] B&B children visited,
 * [4] flags: 1 = candidate 0 infeasible (nothing selected), 2 = the warm start was within the gap
 * at the root, 4 = node_cap reached (oracle_memopt adds 8 = malformed record / n = 0, not solved).
 * Returns 0. */
typedef struct {
    uint32_t n, Sst, gap_pm, node_cap;
    const uint32_t *sF, *sB, *nc;
    const uint64_t *cand;
    int64_t M;
    uint32_t *pick;      /* current partial selection (depth-first) */
    uint32_t *best;      /* incumbent */
    uint8_t *kstar;      /* M3b: the points whose constraint the bound keeps */
    uint64_t inc, nodes;
    int capped;
} ilp_t;

static uint64_t c_lat(const ilp_t *I, uint32_t p, uint32_t c) {
    const uint64_t *a = I->cand + ((size_t)p * I->Sst + c) * 3;
    return a[0] + a[1];
}
static uint64_t c_mem(const ilp_t *I, uint32_t p, uint32_t c) { return I->cand[((size_t)p * I->Sst + c) * 3 + 2]; }
static int live_at(const ilp_t *I, uint32_t p, uint32_t k) { return I->sF[p] <= I->sF[k] && I->sF[k] < I->sB[p]; }

/* memory at point k: pairs < nfix at their pick, the others at candidate 0 */
static int64_t used_at(const ilp_t *I, uint32_t k, uint32_t nfix) {
    int64_t u = 0;
    for (uint32_t p = 0; p < I->n; p++)
        if (live_at(I, p, k)) u += (int64_t)c_mem(I, p, p < nfix ? I->pick[p] : 0);
    return u;
}

/* M3b: lower bound on sum lat with pairs < nfix fixed at their pick; UINT64_MAX if infeasible.
 * Lagrangian relaxation of the memory constraints at the points K* (kstar[k] = 1) with one
 * multiplier mu >= 0 (fixed point, mu = mu_int / 2^16): for ANY mu
 *   L(mu) = sum_fixed lat + sum_free min_c (lat_c + mu * c_p * mem_c) - mu * R,
 *   c_p = #{k in K*: p live at k},  R = sum_{k in K*} (M - memory of the fixed pairs live at k),
 * is <= the ILP optimum (weak duality: every feasible selection has sum_free c_p mem_p <= R).
 * mu is found by bisection on the sign of R - D(mu), D(mu) = sum_free c_p * mem of the pair's
 * minimiser (ties: less memory); the bound is the ILP-integral ceil(L) at the better end. */
#define ILP_SHIFT 16
static void ilp_eval(const ilp_t *I, uint32_t nfix, const uint32_t *cp, uint64_t mu, uint64_t *D, unsigned __int128 *V) {
    *D = 0; *V = 0;
    for (uint32_t p = nfix; p < I->n; p++) {
        unsigned __int128 best = 0;
        uint64_t bm = 0;
        for (uint32_t c = 0; c < I->nc[p]; c++) {
            unsigned __int128 v = ((unsigned __int128)c_lat(I, p, c) << ILP_SHIFT) + (unsigned __int128)mu * cp[p] * c_mem(I, p, c);
            if (c == 0 || v < best || (v == best && c_mem(I, p, c) < bm)) { best = v; bm = c_mem(I, p, c); }
        }
        *V += best;
        *D += (uint64_t)cp[p] * bm;
    }
}

static uint64_t ilp_L(const ilp_t *I, uint32_t nfix, const uint32_t *cp, uint64_t mu, int64_t R, uint64_t fixed) {
    uint64_t D;
    unsigned __int128 V;
    ilp_eval(I, nfix, cp, mu, &D, &V);
    unsigned __int128 take = (unsigned __int128)mu * (uint64_t)R;      /* R >= 0 when feasible */
    if (V <= take) return fixed;
    unsigned __int128 num = V - take;
    uint64_t q = (uint64_t)(num >> ILP_SHIFT) + ((num & ((1u << ILP_SHIFT) - 1)) ? 1 : 0);   /* ceil */
    return fixed + q;
}

static uint64_t ilp_bound(const ilp_t *I, uint32_t nfix) {
    const uint32_t n = I->n;
    for (uint32_t k = 0; k < n; k++)
        if (used_at(I, k, nfix) > I->M) return UINT64_MAX;
    uint64_t fixed = 0;
    for (uint32_t p = 0; p < nfix; p++) fixed += c_lat(I, p, I->pick[p]);
    uint32_t *cp = calloc(n + 1, sizeof(uint32_t));
    int64_t R = 0;
    for (uint32_t k = 0; k < n; k++) {
        if (!I->kstar[k]) continue;
        int64_t fx = 0;
        for (uint32_t p = 0; p < n; p++)
            if (live_at(I, p, k)) {
                if (p < nfix) fx += (int64_t)c_mem(I, p, I->pick[p]);
                else cp[p]++;
            }
        R += I->M - fx;
    }
    uint64_t D;
    unsigned __int128 V;
    uint64_t lo = 0, hi = 1, out;
    ilp_eval(I, nfix, cp, 0, &D, &V);
    if ((int64_t)D <= R) {
        out = ilp_L(I, nfix, cp, 0, R, fixed);
    } else {
        for (int it = 0; it < 16; it++) {          /* D(hi) <= R: every pair at its least memory fits */
            ilp_eval(I, nfix, cp, hi, &D, &V);
            if ((int64_t)D <= R) break;
            lo = hi;
            hi *= 16;
        }
        while (hi - lo > 1 && hi - lo > (hi >> 6)) {    /* to 1/64 relative: any mu gives a valid bound */
            uint64_t mid = lo + (hi - lo) / 2;
            ilp_eval(I, nfix, cp, mid, &D, &V);
            if ((int64_t)D <= R) hi = mid; else lo = mid;
        }
        uint64_t a = ilp_L(I, nfix, cp, lo, R, fixed), b = ilp_L(I, nfix, cp, hi, R, fixed);
        out = a > b ? a : b;
    }
    free(cp);
    return out;
}

/* within the gap: 1000 * bound >= (1000 - gap) * incumbent */
static int ilp_within(const ilp_t *I, uint64_t bound) {
    return (unsigned __int128)bound * 1000u >= (unsigned __int128)I->inc * (1000u - I->gap_pm);
}

/* M3c: depth-first over pair d's candidates, fastest first */
static void ilp_dfs(ilp_t *I, uint32_t d) {
    for (int c = (int)I->nc[d] - 1; c >= 0; c--) {
        if (I->nodes >= I->node_cap) { I->capped = 1; return; }
        I->nodes++;
        I->pick[d] = (uint32_t)c;
        int fits = 1;
        for (uint32_t k = 0; k < I->n && fits; k++)
            if (live_at(I, d, k) && used_at(I, k, d + 1) > I->M) fits = 0;
        if (!fits) continue;
        if (d + 1 == I->n) {
            uint64_t obj = 0;
            for (uint32_t p = 0; p < I->n; p++) obj += c_lat(I, p, I->pick[p]);
            if (obj < I->inc) { I->inc = obj; memcpy(I->best, I->pick, sizeof(uint32_t) * I->n); }
            continue;
        }
        uint64_t lb = ilp_bound(I, d + 1);
        if (lb != UINT64_MAX && !ilp_within(I, lb)) ilp_dfs(I, d + 1);
        if (I->capped) return;
    }
}

int oracle_select_rank(uint32_t n, const uint32_t *sF, const uint32_t *sB, const uint32_t *nc, const uint64_t *cand,
                       uint32_t Sst, int64_t M, uint32_t gap_pm, uint32_t node_cap, uint32_t *cur, uint64_t *stats) {
    uint64_t sv[5] = {0, 0, 0, 0, 0};
    ilp_t I = {n, Sst, gap_pm > 1000 ? 1000 : gap_pm, node_cap, sF, sB, nc, cand, M, NULL, NULL, NULL, 0, 0, 0};
    I.pick = calloc(n + 1, sizeof(uint32_t));
    I.best = calloc(n + 1, sizeof(uint32_t));
    I.kstar = calloc(n + 1, 1);
    for (uint32_t p = 0; p < n; p++) cur[p] = 0;
    /* M3a: the greedy warm start */
    int64_t *slack = malloc(sizeof(int64_t) * (n + 1));
    int feasible = 1;
    for (uint32_t k = 0; k < n; k++) {
        slack[k] = M - used_at(&I, k, 0);
        if (slack[k] < 0) feasible = 0;
    }
    while (feasible) {
        int best = -1;
        uint64_t bl = 0, bm = 1;
        for (uint32_t p = 0; p < n; p++) {
            if (cur[p] + 1 >= nc[p]) continue;
            uint64_t dl = c_lat(&I, p, cur[p]) - c_lat(&I, p, cur[p] + 1), dm = c_mem(&I, p, cur[p] + 1) - c_mem(&I, p, cur[p]);
            int ok = 1;
            for (uint32_t k = 0; k < n && ok; k++)
                if (live_at(&I, p, k) && slack[k] < (int64_t)dm) ok = 0;
            if (!ok) continue;
            /* dl/dm > bl/bm, exactly; ties keep the earlier forward slot (lower p) */
            if (best < 0 || (unsigned __int128)dl * bm > (unsigned __int128)bl * dm) { best = (int)p; bl = dl; bm = dm; }
        }
        if (best < 0) break;
        for (uint32_t k = 0; k < n; k++)
            if (live_at(&I, (uint32_t)best, k)) slack[k] -= (int64_t)bm;
        cur[best]++;
    }
    /* K*: the points where the warm start blocks a pair (its next step does not fit there) */
    for (uint32_t k = 0; k < n && feasible; k++)
        for (uint32_t p = 0; p < n; p++)
            if (live_at(&I, p, k) && cur[p] + 1 < nc[p] && slack[k] < (int64_t)(c_mem(&I, p, cur[p] + 1) - c_mem(&I, p, cur[p])))
                I.kstar[k] = 1;
    free(slack);
    if (!feasible) {
        sv[4] = 1;
    } else {
        for (uint32_t p = 0; p < n; p++) { I.inc += c_lat(&I, p, cur[p]); I.best[p] = cur[p]; }
        sv[0] = I.inc;
        /* M3b at the root, M3c if the warm start is not provably within the gap */
        uint64_t lb = ilp_bound(&I, 0);
        sv[1] = lb;
        if (ilp_within(&I, lb)) sv[4] |= 2;
        else if (n > 0) ilp_dfs(&I, 0);
        if (I.capped) sv[4] |= 4;
        for (uint32_t p = 0; p < n; p++) cur[p] = I.best[p];
        sv[2] = I.inc;
        sv[3] = I.nodes;
    }
    if (stats) memcpy(stats, sv, sizeof(sv));
    free(I.pick); free(I.best); free(I.kstar);
    return 0;
}

/* M2-M4 for candidate x: sel [P][2][n_max] (candidate index of the pair at forward position p /
 * backward position q), then the re-timed result. */
static void memopt_one(const oproblem *pb, const omenu *mn, const ocands *cs, uint64_t x, uint8_t *sel,
                       ores *res, uint64_t *peaks, uint64_t *rstats /* [P][5] or NULL */) {
    const uint32_t P = pb->P, nm = pb->nmod, m = pb->m, n_max = cs->n_max, fbw = cs->fbw;
    const uint8_t *split = cs->split + x * (uint64_t)m * nm;
    const uint16_t *fwd = cs->fwd + x * (uint64_t)n_max, *bwd = cs->bwd + x * (uint64_t)n_max;
    const uint32_t *fb = cs->fb + x * (uint64_t)P * fbw;
    const uint32_t n = cs->n[x], T = pb->tab_off[nm];
    memset(sel, 0, (size_t)P * 2 * n_max);
    ores r0;
    eval_one(pb, cs, x, &r0, NULL, NULL, NULL, NULL);             /* encoding checks (O4) */
    if (r0.status == ST_BAD || n == 0) {
        if (rstats) for (uint32_t r = 0; r < P; r++) { memset(rstats + 5 * (size_t)r, 0, 5 * sizeof(uint64_t)); rstats[5 * (size_t)r + 4] = 8; }
        eval_one(pb, cs, x, res, peaks, NULL, NULL, NULL);
        return;
    }
    uint32_t idmax = seg_count_max(pb);
    uint32_t *base = malloc(sizeof(uint32_t) * (m * nm + 1));
    uint32_t *W = calloc(idmax + 1, sizeof(uint32_t)), *si = calloc(idmax + 1, sizeof(uint32_t)), *sk = calloc(idmax + 1, sizeof(uint32_t));
    uint32_t acc = 0;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            uint32_t q = b * nm + i;
            base[q] = acc;
            uint32_t lo = pb->inst_off[q], N = pb->inst_off[q + 1] - lo, M = split[q], st[16];
            if (M) oracle_split(N, M, st);
            for (uint32_t j = 0; j < pb->max_split[i]; j++)
                for (uint32_t k = 0; k < pb->K[i]; k++) {
                    uint32_t id = acc + j * pb->K[i] + k, w = 0;
                    if (j < M) for (uint32_t u = st[j]; u < st[j + 1]; u++) w += pb->inst_units[lo + u];
                    W[id] = w; si[id] = i; sk[id] = k;
                }
            acc += pb->max_split[i] * pb->K[i];
        }
    uint64_t *ovr = calloc((size_t)P * (idmax + 1) * 3, sizeof(uint64_t));
    uint64_t *cl = malloc(sizeof(uint64_t) * 3 * mn->S * n);     /* candidates of each pair */
    uint32_t *nc = malloc(sizeof(uint32_t) * n), *cur = malloc(sizeof(uint32_t) * n);
    uint32_t *sF = malloc(sizeof(uint32_t) * n), *sB = malloc(sizeof(uint32_t) * n), *qpos = malloc(sizeof(uint32_t) * n);
    uint32_t *fseg = malloc(sizeof(uint32_t) * n);
    for (uint32_t r = 0; r < P; r++) {
        /* the rank's order: slot of the p-th forward and of the q-th backward stage (O5) */
        uint32_t fi = 0, bi = 0;
        uint32_t *slotB_of_seg = malloc(sizeof(uint32_t) * (idmax + 1)), *qpos_of_seg = malloc(sizeof(uint32_t) * (idmax + 1));
        const uint16_t *ordr = cs->ord ? cs->ord + (x * (uint64_t)P + r) * 2 * n_max : NULL;
        for (uint32_t t = 0; t < 2 * n; t++) {
            uint32_t isb = ordr ? (uint32_t)(ordr[t] >> 15) : ((fb[r * fbw + t / 32] >> (t % 32)) & 1u);
            if (isb) { uint32_t sg = ordr ? (ordr[t] & 0x7FFFu) : bwd[bi]; slotB_of_seg[sg] = t; qpos_of_seg[sg] = bi; bi++; }
            else { fseg[fi] = ordr ? (ordr[t] & 0x7FFFu) : fwd[fi]; sF[fi] = t; fi++; }
        }
        for (uint32_t p = 0; p < n; p++) {                          /* pair p = the p-th forward stage */
            uint32_t s = fseg[p], i = si[s], lay = layers_of(pb, i, sk[s] * P + r), toff = pb->tab_off[i] + W[s];
            uint32_t ff[8], bb[8], aa[8];
            for (uint32_t c = 0; c < mn->n_strat; c++) {
                ff[c] = mn->f[c * T + toff]; bb[c] = mn->b[c * T + toff]; aa[c] = mn->act[c * T + toff];
            }
            nc[p] = lay ? (uint32_t)oracle_mem_candidates(mn->n_strat, ff, bb, aa, lay, mn->S, cl + (size_t)3 * mn->S * p) : 0;
            if (nc[p] == 0) { nc[p] = 1; cl[(size_t)3 * mn->S * p] = 0; cl[(size_t)3 * mn->S * p + 1] = 0; cl[(size_t)3 * mn->S * p + 2] = 0; }
            cur[p] = 0;
            sB[p] = slotB_of_seg[s];
            qpos[p] = qpos_of_seg[s];
        }
        /* M3: the rank's ILP */
        oracle_select_rank(n, sF, sB, nc, cl, mn->S, (int64_t)pb->budget_kib[r], mn->gap_pm, mn->node_cap, cur,
                           rstats ? rstats + 5 * (size_t)r : NULL);
        for (uint32_t p = 0; p < n; p++) {
            const uint64_t *a = cl + (size_t)3 * mn->S * p + 3 * cur[p];
            uint64_t *o = ovr + ((uint64_t)r * (idmax + 1) + fseg[p]) * 3;
            o[0] = a[0]; o[1] = a[1]; o[2] = a[2];
            sel[((size_t)r * 2 + 0) * n_max + p] = (uint8_t)cur[p];
            sel[((size_t)r * 2 + 1) * n_max + qpos[p]] = (uint8_t)cur[p];
        }
        free(slotB_of_seg); free(qpos_of_seg);
    }
    eval_one(pb, cs, x, res, peaks, NULL, NULL, ovr);          /* M4 */
    free(base); free(W); free(si); free(sk); free(ovr); free(cl); free(nc); free(cur);
    free(sF); free(sB); free(qpos); free(fseg);
}

typedef struct {
    const oproblem *pb;
    const omenu *mn;
    const ocands *cs;
    uint64_t lo, hi, first;
    uint8_t *sel;
    uint64_t *makespan, *busy, *peaks, *rstats;
    uint32_t *status, *oom;
    double *bubble;
} mjob_t;

static void *mworker(void *arg) {
    mjob_t *j = (mjob_t *)arg;
    const uint32_t P = j->pb->P;
    for (uint64_t x = j->lo; x < j->hi; x++) {
        ores r;
        uint64_t o = x - j->first;
        memopt_one(j->pb, j->mn, j->cs, x, j->sel + o * (uint64_t)P * 2 * j->cs->n_max, &r, j->peaks ? j->peaks + o * P : NULL,
                   j->rstats ? j->rstats + o * 5 * P : NULL);
        j->makespan[o] = r.makespan; j->busy[o] = r.busy; j->status[o] = r.status;
        j->oom[o] = r.oom_mask; j->bubble[o] = r.bubble;
    }
    return NULL;
}

int oracle_memopt(const oproblem *pb, uint32_t n_strat, const uint32_t *mf, const uint32_t *mb, const uint32_t *ma,
                  uint32_t S, const ocands *cs, uint64_t first, uint64_t count, uint8_t *sel /* [count][P][2][n_max] */,
                  uint64_t *makespan, uint32_t *status, uint32_t *oom_mask, double *bubble, uint64_t *peaks,
                  uint64_t *busy, int threads, uint32_t gap_pm, uint32_t node_cap,
                  uint64_t *rank_stats /* [count][P][5] (oracle_select_rank's stats) or NULL */) {
    if (n_strat == 0 || n_strat > 8 || S < 2 || S > 16) return -1;
    omenu mn = {n_strat, S, mf, mb, ma, gap_pm, node_cap};
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    if ((uint64_t)threads > count) threads = count ? (int)count : 1;
    pthread_t th[512];
    mjob_t jobs[512];
    uint64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        uint64_t lo = first + per * t, hi = lo + per;
        if (hi > first + count) hi = first + count;
        if (lo > hi) lo = hi;
        jobs[t] = (mjob_t){pb, &mn, cs, lo, hi, first, sel, makespan, busy, peaks, rank_stats, status, oom_mask, bubble};
        pthread_create(&th[t], NULL, mworker, &jobs[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    return 0;
}
