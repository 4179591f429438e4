/* dip_gen.c -- seeded synthetic CANDIDATE generator (input generation only).
 *
 * Shared by the oracle tests and the CUDA path, so it contains none of the hot
 * path's arithmetic: it never reads a latency, an activation size or a work
 * unit, never computes a time, a memory peak or a sub-microbatch split of the
 * instances.  It only decides *orders*:
 *
 *   split  M_{b,i}   in [1, min(N, M_max)]  (paper's ceil(N/B_i) rule or uniform; R-2)
 *   fwd_seq / bwd_seq  priority-driven linear extensions of the segment DAG
 *                      (equal-priority classes per (microbatch, module), P:506-509;
 *                       Megatron / encoder-first / random-priority / VPP families)
 *   fb bits          per-rank F/B interleaving built by a *dependency-readiness*
 *                    replay (no time): in lock-step rounds each rank takes its next
 *                    backward if its producer is done, else its next forward if its
 *                    producer is done and fewer than cap_r forwards are in flight
 *                    (the paper's memory gating, in segment counts).
 *
 * Deliberate perturbations (adjacent F/B swaps -> some deadlocks; corrupted
 * encodings) exercise the DEADLOCK / BAD_ENCODING statuses.
 *
 * Candidate c is a pure function of (seed, c), so any shard can be generated
 * independently of the world size.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint32_t P, nmod, m, n_max, fbw;
    const uint32_t *K;             /* [nmod] */
    const uint32_t *max_split;     /* [nmod] */
    const uint32_t *producer_mask; /* [nmod] */
    const uint32_t *nbi;           /* [m*nmod] instance counts N_{b,i} */
    uint64_t seed;
    uint32_t mode;                 /* 0 random families, 1 toy exhaustive */
    uint32_t split_rule_b;         /* B_i of the ceil(N/B) rule */
    double p_mutate, p_bad;
} gen_cfg;

static inline uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
typedef struct { uint64_t s; } rng_t;
static inline uint64_t rnext(rng_t *r) { r->s += 0x9E3779B97F4A7C15ull; return mix64(r->s); }
static inline uint32_t rbelow(rng_t *r, uint32_t n) { return n ? (uint32_t)(rnext(r) % n) : 0; }
static inline double runit(rng_t *r) { return (double)(rnext(r) >> 11) * (1.0 / 9007199254740992.0); }

typedef struct {
    /* per-thread scratch sized by n_max / P */
    uint32_t *segb, *segi, *segj, *segk;  /* decode of present segments by id */
    uint8_t *present;
    int32_t *indeg;
    uint64_t *heap_key;
    uint32_t *heap_id;
    uint32_t *prio;      /* [m*nmod] */
    uint32_t *fpos;      /* forward position of each id */
    int32_t *cntF0, *cntBP;
    uint32_t *fi, *bi, *cap;
    uint8_t *dec;
    uint32_t *base;      /* [m*nmod] */
    uint8_t *M;          /* [m*nmod] */
    uint16_t *fmb, *bmb; /* [P][m] per-rank F/B segments done per microbatch */
    uint32_t *segs_mb, *infl, *cons;
    uint64_t *fk;
    uint32_t *posf, *posb, *perm;
    uint8_t *newmb, *endmb;
} scratch_t;

static void heap_push(scratch_t *w, uint32_t *hn, uint64_t key, uint32_t id) {
    uint32_t i = (*hn)++;
    while (i > 0) {
        uint32_t p = (i - 1) / 2;
        if (w->heap_key[p] < key || (w->heap_key[p] == key && w->heap_id[p] < id)) break;
        w->heap_key[i] = w->heap_key[p];
        w->heap_id[i] = w->heap_id[p];
        i = p;
    }
    w->heap_key[i] = key;
    w->heap_id[i] = id;
}
static uint32_t heap_pop(scratch_t *w, uint32_t *hn) {
    uint32_t top = w->heap_id[0];
    uint32_t n = --(*hn);
    uint64_t k = w->heap_key[n];
    uint32_t id = w->heap_id[n];
    uint32_t i = 0;
    for (;;) {
        uint32_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && (w->heap_key[c + 1] < w->heap_key[c] ||
                          (w->heap_key[c + 1] == w->heap_key[c] && w->heap_id[c + 1] < w->heap_id[c])))
            c++;
        if (k < w->heap_key[c] || (k == w->heap_key[c] && id < w->heap_id[c])) break;
        w->heap_key[i] = w->heap_key[c];
        w->heap_id[i] = w->heap_id[c];
        i = c;
    }
    w->heap_key[i] = k;
    w->heap_id[i] = id;
    return top;
}

enum { FWD_MB = 0, FWD_ENCFIRST = 1, FWD_RANDPRIO = 2, FWD_VPP = 3 };
enum { BWD_MIRROR = 0, BWD_RANDPRIO = 1 };
enum { BITS_1F1B = 0, BITS_SCALED = 1, BITS_GPIPE = 2, BITS_UNIFORM = 3 };

static uint32_t consumers_of(const gen_cfg *c, uint32_t i) {
    uint32_t mask = 0;
    for (uint32_t x = 0; x < c->nmod; x++)
        if ((c->producer_mask[x] >> i) & 1u) mask |= 1u << x;
    return mask;
}

/* Build a priority-driven linear extension of the forward (dir=0) or backward
 * (dir=1) segment DAG.  Forward preds of (b,i,j,k): (b,i,j,k-1), or for k = 0 the
 * last segment of every present producer sub-microbatch of the same microbatch
 * (R-4, R-5).  The backward DAG is the reverse. */
static void linear_extension(const gen_cfg *c, scratch_t *w, int dir, const uint64_t *key,
                             uint16_t *out) {
    const uint32_t nm = c->nmod;
    uint32_t hn = 0, cnt = 0;
    for (uint32_t id = 0; id < c->n_max; id++) {
        w->indeg[id] = -1;
        if (!w->present[id]) continue;
        uint32_t b = w->segb[id], i = w->segi[id], k = w->segk[id];
        int32_t d = 0;
        if (dir == 0) {
            if (k > 0) d = 1;
            else for (uint32_t p = 0; p < nm; p++)
                if ((c->producer_mask[i] >> p) & 1u) d += w->M[b * nm + p];
        } else {
            if (k + 1 < c->K[i]) d = 1;
            else {
                uint32_t cm = consumers_of(c, i);
                for (uint32_t q = 0; q < nm; q++)
                    if ((cm >> q) & 1u) d += w->M[b * nm + q];
            }
        }
        w->indeg[id] = d;
        if (d == 0) heap_push(w, &hn, key[id], id);
    }
    while (hn) {
        uint32_t id = heap_pop(w, &hn);
        out[cnt++] = (uint16_t)id;
        uint32_t b = w->segb[id], i = w->segi[id], k = w->segk[id];
        /* successors in this direction */
        uint32_t succ[256];
        uint32_t ns = 0;
        if (dir == 0) {
            if (k + 1 < c->K[i]) succ[ns++] = id + 1;
            else {
                uint32_t cm = consumers_of(c, i);
                for (uint32_t q = 0; q < nm; q++)
                    if ((cm >> q) & 1u)
                        for (uint32_t jj = 0; jj < w->M[b * nm + q] && ns < 256; jj++)
                            succ[ns++] = w->base[b * nm + q] + jj * c->K[q];
            }
        } else {
            if (k > 0) succ[ns++] = id - 1;
            else for (uint32_t p = 0; p < nm; p++)
                if ((c->producer_mask[i] >> p) & 1u)
                    for (uint32_t jj = 0; jj < w->M[b * nm + p] && ns < 256; jj++)
                        succ[ns++] = w->base[b * nm + p] + jj * c->K[p] + (c->K[p] - 1);
        }
        for (uint32_t x = 0; x < ns; x++) {
            uint32_t s = succ[x];
            if (--w->indeg[s] == 0) heap_push(w, &hn, key[s], s);
        }
    }
}

/* Dependency-readiness replay: decides each rank's F/B bit string.  A rank may
 * start the forward of a *new* microbatch (its first backbone segment) only while
 * fewer than cap_r microbatches are in flight on it (memory gating in microbatch
 * units; 1F1B = P - r).  If no rank can act, the caps are relaxed for one round.
 * Returns 0 on success (always, for linear-extension sequences). */
static int readiness_bits(const gen_cfg *c, scratch_t *w, uint32_t n, const uint16_t *fwd,
                          const uint16_t *bwd, int ffirst, uint32_t *fb /* [P][fbw] */) {
    const uint32_t P = c->P, nm = c->nmod;
    for (uint32_t b = 0; b < c->m; b++) {
        uint32_t t = 0;
        for (uint32_t i = 0; i < nm; i++) if (!w->cons[i]) t += w->M[b * nm + i] * c->K[i];
        w->segs_mb[b] = t;
    }
    for (uint32_t id = 0; id < c->n_max; id++) {
        if (!w->present[id]) continue;
        uint32_t b = w->segb[id], i = w->segi[id], k = w->segk[id];
        int32_t f0 = 0, bp = 0;
        if (k > 0) f0 = 1;
        else for (uint32_t p = 0; p < nm; p++)
            if ((c->producer_mask[i] >> p) & 1u) f0 += w->M[b * nm + p];
        if (k + 1 < c->K[i]) bp = 1;
        else {
            uint32_t cm = w->cons[i];
            for (uint32_t q = 0; q < nm; q++)
                if ((cm >> q) & 1u) bp += w->M[b * nm + q];
            if (bp == 0) bp = 1; /* terminal: turnaround from its own F at rank P-1 (R-6) */
        }
        w->cntF0[id] = f0;
        w->cntBP[id] = bp;
    }
    /* per-position flags: newmb[p] = fwd[p] is the first backbone segment of its microbatch in
     * forward order; endmb[p] = bwd[p] is the last backbone segment of its microbatch in
     * backward order (a rank's in-flight microbatch count changes exactly there) */
    for (uint32_t b = 0; b < c->m; b++) { w->fmb[b] = 0; w->bmb[b] = 0; }
    for (uint32_t p = 0; p < n; p++) {
        uint32_t s = fwd[p], bb = w->segb[s];
        w->newmb[p] = (!w->cons[w->segi[s]] && w->fmb[bb]++ == 0);
    }
    for (uint32_t p = 0; p < n; p++) {
        uint32_t s = bwd[p], bb = w->segb[s];
        w->endmb[p] = (!w->cons[w->segi[s]] && ++w->bmb[bb] == w->segs_mb[bb]);
    }
    w->newmb[n] = 0;
    w->endmb[n] = 0;
    for (uint32_t r = 0; r < P; r++) { w->fi[r] = 0; w->bi[r] = 0; w->infl[r] = 0; }
    memset(fb, 0, sizeof(uint32_t) * P * c->fbw);
    uint32_t remaining = P * 2 * n;
    uint32_t relax = 0;
    uint32_t *fi = w->fi, *bi = w->bi, *infl = w->infl, *cap = w->cap;
    /* one fused sweep per lock-step round: rank r decides on the start-of-round state (fi[r-1] is
     * carried in `fprev` before rank r-1's update; bi[r+1] and cntF0 are not yet updated when read;
     * rank 0's backward publications to cntBP are deferred until after rank P-1 decided) */
    while (remaining) {
        uint32_t acted = 0, fprev = 0, defer_s = 0xFFFFFFFFu;
        for (uint32_t r = 0; r < P; r++) {
            const uint32_t fr = fi[r], br = bi[r];
            uint32_t frdy, brdy;
            if (r == 0) frdy = fr < n && w->cntF0[fwd[fr]] == 0;
            else frdy = (fr < n) & (fprev > fr);
            if (r + 1 == P) brdy = br < n && w->cntBP[bwd[br]] == 0;
            else brdy = (br < n) & (bi[r + 1] > br);
            const uint32_t under = relax | (uint32_t)(w->newmb[fr] == 0) | (uint32_t)(infl[r] < cap[r]);
            const uint32_t fok = frdy & under;
            const uint32_t d = ffirst ? (fok ? 1u : 2u * brdy) : (brdy ? 2u : fok);
            fprev = fr;
            if (!d) continue;
            acted = 1;
            const uint32_t t = fr + br;
            if (d == 1) {
                fi[r] = fr + 1;
                const uint32_t s = fwd[fr];
                infl[r] += w->newmb[fr];
                if (r == P - 1) {
                    uint32_t b = w->segb[s], i = w->segi[s], k = w->segk[s];
                    if (k + 1 < c->K[i]) w->cntF0[s + 1]--;
                    else {
                        uint32_t cm = w->cons[i], any = 0;
                        for (uint32_t q = 0; q < nm; q++)
                            if ((cm >> q) & 1u)
                                for (uint32_t jj = 0; jj < w->M[b * nm + q]; jj++) {
                                    w->cntF0[w->base[b * nm + q] + jj * c->K[q]]--;
                                    any = 1;
                                }
                        if (!any) w->cntBP[s]--;
                    }
                }
            } else {
                fb[r * c->fbw + (t >> 5)] |= 1u << (t & 31);
                bi[r] = br + 1;
                const uint32_t s = bwd[br];
                infl[r] -= w->endmb[br];
                if (r == 0) defer_s = s;
            }
            remaining--;
        }
        if (defer_s != 0xFFFFFFFFu) {   /* rank 0's backward publication (after rank P-1 decided) */
            const uint32_t s = defer_s;
            uint32_t b = w->segb[s], i = w->segi[s], k = w->segk[s];
            if (k > 0) w->cntBP[s - 1]--;
            else for (uint32_t pp = 0; pp < nm; pp++)
                if ((c->producer_mask[i] >> pp) & 1u)
                    for (uint32_t jj = 0; jj < w->M[b * nm + pp]; jj++)
                        w->cntBP[w->base[b * nm + pp] + jj * c->K[pp] + c->K[pp] - 1]--;
        }
        if (!acted) {
            if (relax) return -1;
            relax = 1;
            continue;
        }
        relax = 0;
    }
    return 0;
}

static int gen_one(const gen_cfg *c, scratch_t *w, uint64_t idx, uint8_t *split, uint32_t *nout,
                   uint16_t *fwd, uint16_t *bwd, uint32_t *fb, uint8_t *family) {
    const uint32_t P = c->P, nm = c->nmod, m = c->m;
    rng_t rg = { mix64(c->seed ^ mix64(idx * 0xD1B54A32D192ED03ull + 1)) };
    int fam_split, fam_f, fam_b, fam_bits;
    uint32_t tmpl = 0;
    rng_t trg = rg; /* order-template rng (toy mode: depends on the template only) */
    if (c->mode == 1) {
        tmpl = (uint32_t)(idx % 16);
        trg.s = mix64(c->seed ^ (0xABCDull + tmpl));
        fam_split = 2;
        if (tmpl == 0) { fam_f = FWD_MB; fam_b = BWD_MIRROR; fam_bits = BITS_1F1B; }
        else if (tmpl == 1) { fam_f = FWD_MB; fam_b = BWD_MIRROR; fam_bits = BITS_GPIPE; }
        else if (tmpl == 2) { fam_f = FWD_ENCFIRST; fam_b = BWD_MIRROR; fam_bits = BITS_1F1B; }
        else { fam_f = FWD_RANDPRIO; fam_b = BWD_RANDPRIO; fam_bits = (tmpl & 1) ? BITS_SCALED : BITS_UNIFORM; }
    } else {
        fam_split = (int)rbelow(&rg, 2);
        uint32_t u = rbelow(&rg, 100);
        fam_f = u < 5 ? FWD_MB : u < 25 ? FWD_ENCFIRST : u < 70 ? FWD_RANDPRIO : FWD_VPP;
        fam_b = rbelow(&rg, 100) < 60 ? BWD_MIRROR : BWD_RANDPRIO;
        u = rbelow(&rg, 100);
        fam_bits = u < 25 ? BITS_1F1B : u < 75 ? BITS_SCALED : u < 85 ? BITS_GPIPE : BITS_UNIFORM;
        trg = rg;
    }
    /* 1. split M_{b,i} */
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            uint32_t N = c->nbi[b * nm + i], Mx = c->max_split[i], M;
            uint32_t hi = N < Mx ? N : Mx;
            if (N == 0) M = 0;
            else if (Mx == 1) M = 1;
            else if (fam_split == 2) M = 1 + (uint32_t)((idx / 16 >> (b % 32)) & 1u);
            else if (fam_split == 0) { M = (N + c->split_rule_b - 1) / c->split_rule_b; }
            else M = 1 + rbelow(&rg, hi);
            if (M < 1 && N > 0) M = 1;
            if (M > hi) M = hi;
            w->M[b * nm + i] = (uint8_t)M;
            split[b * nm + i] = (uint8_t)M;
        }
    /* 2. segments */
    uint32_t n = 0, acc = 0;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            w->base[b * nm + i] = acc;
            for (uint32_t j = 0; j < c->max_split[i]; j++)
                for (uint32_t k = 0; k < c->K[i]; k++) {
                    uint32_t id = acc + j * c->K[i] + k;
                    w->segb[id] = b; w->segi[id] = i; w->segj[id] = j; w->segk[id] = k;
                    w->present[id] = j < w->M[b * nm + i];
                    n += w->present[id];
                }
            acc += c->max_split[i] * c->K[i];
        }
    /* 3. sequences: microbatches are taken in groups of g (g = P: Megatron VPP grouping,
     * chunk-major inside a group); classes (b, i) keep a fixed internal order. */
    uint32_t g = 1;
    if (c->mode == 0) {
        uint32_t u = rbelow(&rg, 100);
        g = u < 4 ? 1 : u < 30 ? (P / 2 ? P / 2 : 1) : u < 80 ? P : 2 * P;
    } else if (tmpl >= 3) {
        g = 1 + rbelow(&trg, m);
    }
    if (fam_f == FWD_MB) g = 1;
    if (g > m) g = m ? m : 1;
    for (uint32_t q = 0; q < m * nm; q++) w->prio[q] = (uint32_t)(rnext(&trg) & 0xFFFFF);
    for (uint32_t p = 0; p < c->n_max; p++) { fwd[p] = 0xFFFF; bwd[p] = 0xFFFF; }
    uint64_t *fk = w->fk, *bkey = w->heap_key + c->n_max; /* heap uses the lower half */
    /* encoder lookahead: encoder segments of microbatch b run beside the backbone of
     * microbatch b - delta (forward) / b + delta (backward), so the encoder->backbone
     * join (R-5) is not on the critical path of every microbatch. */
    uint32_t kbb = 1;
    for (uint32_t i = 0; i < nm; i++) if (!w->cons[i] && c->K[i] > kbb) kbb = c->K[i];
    double segs_mb = m ? (double)n / (double)m : 1.0;
    uint32_t delta = (uint32_t)((double)P / (segs_mb > 1.0 ? segs_mb : 1.0) + 0.999);
    if (c->mode == 0) delta = (uint32_t)(delta * (0.5 + 1.5 * runit(&trg)) + 0.5);
    else if (tmpl < 3) delta = 0;
    /* microbatch order: position pf[b] in the forward order, pb[b] in the backward order
     * (identity, or shuffled inside each group of g for the random-priority families) */
    uint32_t *pf = w->posf, *pbk = w->posb, *tmp = w->perm;
    for (uint32_t q = 0; q < m; q++) tmp[q] = q;
    if (fam_f == FWD_RANDPRIO)
        for (uint32_t g0 = 0; g0 < m; g0 += g) {
            uint32_t len = g0 + g <= m ? g : m - g0;
            for (uint32_t x = len; x > 1; x--) {
                uint32_t y = rbelow(&trg, x);
                uint32_t t2 = tmp[g0 + x - 1]; tmp[g0 + x - 1] = tmp[g0 + y]; tmp[g0 + y] = t2;
            }
        }
    for (uint32_t q = 0; q < m; q++) pf[tmp[q]] = q;
    if (fam_b == BWD_RANDPRIO)
        for (uint32_t g0 = 0; g0 < m; g0 += g) {
            uint32_t len = g0 + g <= m ? g : m - g0;
            for (uint32_t x = len; x > 1; x--) {
                uint32_t y = rbelow(&trg, x);
                uint32_t t2 = tmp[g0 + x - 1]; tmp[g0 + x - 1] = tmp[g0 + y]; tmp[g0 + y] = t2;
            }
        }
    for (uint32_t q = 0; q < m; q++) pbk[tmp[q]] = q;
    for (uint32_t id = 0; id < c->n_max; id++) {
        if (!w->present[id]) continue;
        uint64_t b = w->segb[id], i = w->segi[id], j = w->segj[id], k = w->segk[id];
        uint64_t K = c->K[i];
        uint64_t qf = pf[b], qb = pbk[b];
        uint64_t tail = (b << 15) | (i << 12) | (j << 8);
        if (w->cons[i]) { /* encoder module: runs beside backbone position qf - delta / qb + delta */
            if (fam_f == FWD_ENCFIRST) fk[id] = (qf << 24) | tail;
            else {
                uint64_t at = qf >= delta ? qf - delta : 0;
                fk[id] = (1ull << 62) | ((at / g) << 52) | (at << 24) | tail;
            }
            uint64_t at = qb + delta;
            if (at < m) bkey[id] = ((at / g) << 52) | ((uint64_t)(kbb - 1) << 44) | (at << 24) | (1ull << 23) | tail;
            else bkey[id] = (0x3FFull << 52) | (qb << 24) | tail;
        } else {          /* backbone (terminal) module */
            fk[id] = (1ull << 62) | ((qf / g) << 52) | (k << 44) | (qf << 24) | (1ull << 23) | tail;
            bkey[id] = ((qb / g) << 52) | ((K - 1 - k) << 44) | (qb << 24) | tail;
        }
    }
    linear_extension(c, w, 0, fk, fwd);
    linear_extension(c, w, 1, bkey, bwd);
    /* 4. bits: caps in microbatches in flight per rank (1F1B: P - r) */
    int ffirst = 0;
    uint32_t sa = 0, sb = 0, su = 0;
    if (fam_bits == BITS_SCALED) { sa = rbelow(&trg, 8); sb = rbelow(&trg, 4); }
    if (fam_bits == BITS_UNIFORM) { su = 1 + rbelow(&trg, 2 * P); ffirst = (int)rbelow(&trg, 2); }
    uint32_t kmax = 1;
    for (uint32_t i = 0; i < nm; i++) if (c->K[i] > kmax) kmax = c->K[i];
    /* interleaved (K > 1) pipelines need (K-1)P/K more microbatches in flight (Megatron VPP warm-up) */
    const double vpp_extra = (double)((kmax - 1) * P + kmax - 1) / (double)kmax;
    for (uint32_t r = 0; r < P; r++) {
        static const double alphas[8] = {0.5, 0.75, 1.0, 1.25, 1.5, 2.0, 2.5, 3.0};
        double cap;
        switch (fam_bits) {
        case BITS_1F1B: cap = (double)(P - r) + (double)(uint32_t)vpp_extra; break;
        case BITS_GPIPE: cap = 1e18; ffirst = 1; break;
        case BITS_SCALED: cap = alphas[sa] * ((double)(P - r) + vpp_extra) + (double)sb; break;
        default: cap = (double)su;
        }
        if (cap < 1.0) cap = 1.0;
        w->cap[r] = cap > 4e9 ? 0xFFFFFFFFu : (uint32_t)(cap + 0.999999);
    }
    if (readiness_bits(c, w, n, fwd, bwd, ffirst, fb) != 0) return -1;
    uint8_t fam = (uint8_t)(fam_f | (fam_b << 2) | (fam_bits << 3));
    /* 5. perturbations */
    if (c->mode == 0 && n > 0 && runit(&rg) < c->p_mutate) {
        uint32_t nsw = 1 + rbelow(&rg, 4);
        for (uint32_t s = 0; s < nsw; s++) {
            uint32_t r = rbelow(&rg, P);
            uint32_t *row = fb + r * c->fbw;
            uint32_t t0 = rbelow(&rg, 2 * n - 1);
            for (uint32_t d = 0; d + 1 < 2 * n; d++) {
                uint32_t t = (t0 + d) % (2 * n - 1);
                uint32_t a = (row[t >> 5] >> (t & 31)) & 1u, bb = (row[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u;
                if (a != bb) {
                    row[t >> 5] ^= 1u << (t & 31);
                    row[(t + 1) >> 5] ^= 1u << ((t + 1) & 31);
                    break;
                }
            }
        }
        fam |= 1u << 5;
    }
    if (c->mode == 0 && runit(&rg) < c->p_bad) {
        uint32_t kind = rbelow(&rg, 4);
        if (kind == 0) {
            uint32_t q = rbelow(&rg, m * nm);
            split[q] = (uint8_t)(split[q] + 1 + rbelow(&rg, 3));
        } else if (kind == 1 && n >= 2) {
            uint32_t a = rbelow(&rg, n), bq = rbelow(&rg, n);
            if (a == bq) bq = (a + 1) % n;
            fwd[a] = fwd[bq];
        } else if (kind == 2) {
            uint32_t r = rbelow(&rg, P), t = rbelow(&rg, 2 * c->n_max);
            fb[r * c->fbw + (t >> 5)] ^= 1u << (t & 31);
        } else {
            n += 1;
        }
        fam |= 1u << 6;
    }
    *nout = n;
    if (family) *family = fam;
    return 0;
}

typedef struct {
    const gen_cfg *c;
    uint64_t first, lo, hi;
    uint8_t *split; uint32_t *n; uint16_t *fwd, *bwd; uint32_t *fb; uint8_t *family;
    int err;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    const gen_cfg *c = j->c;
    const uint32_t nmx = c->n_max ? c->n_max : 1, mn = c->m * c->nmod;
    scratch_t w;
    w.segb = malloc(sizeof(uint32_t) * nmx); w.segi = malloc(sizeof(uint32_t) * nmx);
    w.segj = malloc(sizeof(uint32_t) * nmx); w.segk = malloc(sizeof(uint32_t) * nmx);
    w.present = malloc(nmx); w.indeg = malloc(sizeof(int32_t) * nmx);
    w.heap_key = malloc(sizeof(uint64_t) * 2 * nmx); w.heap_id = malloc(sizeof(uint32_t) * nmx);
    w.prio = malloc(sizeof(uint32_t) * (mn + 1)); w.fpos = malloc(sizeof(uint32_t) * nmx);
    w.cntF0 = malloc(sizeof(int32_t) * nmx); w.cntBP = malloc(sizeof(int32_t) * nmx);
    w.fi = malloc(sizeof(uint32_t) * c->P); w.bi = malloc(sizeof(uint32_t) * c->P);
    w.cap = malloc(sizeof(uint32_t) * (c->P + 2)); w.dec = malloc(c->P);
    w.base = malloc(sizeof(uint32_t) * (mn + 1)); w.M = malloc(mn + 1);
    w.fmb = malloc(sizeof(uint16_t) * c->P * c->m + 2); w.bmb = malloc(sizeof(uint16_t) * c->P * c->m + 2);
    w.segs_mb = malloc(sizeof(uint32_t) * (c->m + 1)); w.infl = malloc(sizeof(uint32_t) * c->P);
    w.cons = malloc(sizeof(uint32_t) * (c->nmod + 1)); w.fk = malloc(sizeof(uint64_t) * nmx);
    w.posf = malloc(sizeof(uint32_t) * (c->m + 1)); w.posb = malloc(sizeof(uint32_t) * (c->m + 1)); w.perm = malloc(sizeof(uint32_t) * (c->m + 1));
    w.newmb = malloc(nmx + 1); w.endmb = malloc(nmx + 1);
    for (uint32_t i = 0; i < c->nmod; i++) w.cons[i] = consumers_of(c, i);
    for (uint64_t x = j->lo; x < j->hi; x++) {
        uint64_t o = x - j->first;
        if (gen_one(c, &w, x, j->split + o * mn, j->n + o, j->fwd + o * c->n_max, j->bwd + o * c->n_max,
                    j->fb + o * (uint64_t)c->P * c->fbw, j->family ? j->family + o : NULL) != 0)
            j->err = -1;
    }
    free(w.segb); free(w.segi); free(w.segj); free(w.segk); free(w.present); free(w.indeg);
    free(w.heap_key); free(w.heap_id); free(w.prio); free(w.fpos); free(w.cntF0); free(w.cntBP);
    free(w.fi); free(w.bi); free(w.cap); free(w.dec); free(w.base); free(w.M); free(w.fmb); free(w.bmb); free(w.segs_mb); free(w.infl); free(w.cons); free(w.fk); free(w.posf); free(w.posb); free(w.perm); free(w.newmb); free(w.endmb);
    return NULL;
}

/* Generate candidates [first, first+count) into caller-owned host-view arrays:
 *   split  u8  [count][m*nmod]
 *   n      u32 [count]
 *   fwd    u16 [count][n_max]   (pad 0xFFFF)
 *   bwd    u16 [count][n_max]
 *   fb     u32 [count][P][fbw]  rank r, slot t: bit t%32 of word t/32; 1 = backward
 *   family u8  [count] or NULL  (fwd | bwd<<2 | bits<<3 | mutated<<5 | bad<<6)
 * Returns 0, or -1 if a generated order could not be completed. */
int dip_gen_candidates(const gen_cfg *c, uint64_t first, uint64_t count, uint8_t *split, uint32_t *n,
                       uint16_t *fwd, uint16_t *bwd, uint32_t *fb, uint8_t *family, int threads) {
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > count) threads = count ? (int)count : 1;
    pthread_t th[256];
    job_t jobs[256];
    if (threads > 256) threads = 256;
    uint64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        uint64_t lo = first + per * t, hi = lo + per;
        if (hi > first + count) hi = first + count;
        if (lo > hi) lo = hi;
        jobs[t] = (job_t){c, first, lo, hi, split, n, fwd, bwd, fb, family, 0};
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    int err = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        err |= jobs[t].err;
    }
    return err;
}
