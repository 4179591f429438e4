// dip_search.cpp -- SURVEY §8(f) row f2: DIP's MCTS segment reordering (§5.1)
// driving batched GPU rollouts (each rollout = priorities -> dual-queue interleaving (f1) -> score).
//
// Search space (reading R-32): for a fixed split, the classes are (direction,
// microbatch b, module i, chunk k) with M_{b,i} > 0 -- the sub-microbatch segments of one modality,
// microbatch and chunk share a priority and keep a fixed internal order (j ascending) -- and a
// sequence is a permutation of all classes; the class at position p gets priority Cn - 1 - p. A
// forward (backward) priority order is the highest-priority ready segment first over the forward
// (backward) segment DAG, so it is always a linear extension.
// Tree: node at depth d fixes the class of position d; s_v = best score below v,
// N_v = visits. Selection: UCB s_v^alpha + beta * sqrt(ln N_x / N_v), ties to the lowest
// class; expansion: the next child in class order; rollouts: uniformly random
// completions of the remaining positions (counter-based splitmix64 stream per rollout); score
// (P:499): LB / makespan for a feasible (OK) schedule, 0 otherwise, LB = the busiest rank's total
// latency (base tables); with memopt the rollout is interleaved and then memory-optimised (f3,
// P:498 "undergoes pipeline stage interleaving ... and per-layer memory optimization"); backpropagation: s_v = max(s_v, best trial), N_v += 1 along the path.
// Batching (the GPU analogue of the paper's parallel workers sharing one tree): each
// round selects `leaves` leaves with a virtual visit on every node of each selected path, expands
// them, scores all their rollouts in one dip_interleave launch, then backpropagates leaf by leaf.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <thread>
#include <vector>

#include "dip_host_internal.h"

using namespace diph;

namespace {

inline uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
struct PinnedBuf {   // page-locked host array (falls back to pageable memory if pinning fails)
    T *p = nullptr;
    bool pinned = false;
    explicit PinnedBuf(size_t n) {
        if (cudaMallocHost(reinterpret_cast<void **>(&p), n * sizeof(T)) == cudaSuccess) pinned = true;
        else p = static_cast<T *>(std::malloc(n * sizeof(T)));
    }
    ~PinnedBuf() { if (pinned) cudaFreeHost(p); else std::free(p); }
    T &operator[](size_t i) { return p[i]; }
    T *data() { return p; }
};

struct Node {
    int parent = -1;
    int cls = -1;                 // class fixed at this node's depth (-1 for the root)
    int depth = 0;
    std::vector<int> children;    // in creation order = increasing class index
    double s = 0.0;
    uint32_t N = 0, vloss = 0;
};

struct Setup {
    uint32_t P, nm, m, n, C, Cn;
    std::vector<uint8_t> M;            // [m*nm]
    std::vector<int> cls_of;           // [m*nm] -> class index of (b,i,k=0) (forward), -1 if absent
    std::vector<uint32_t> cls_q;       // present (b*nm + i), in class order
    std::vector<uint32_t> q_of_seg;    // segment id -> (b*nm + i)
    double LB;
};

// priority-driven linear extension over the forward (dir 0) or backward (dir 1) segment DAG
void order(const dip_model *Md, const Setup &S, const std::vector<uint32_t> &prio /* [Cn] */, int dir,
           uint16_t *out) {
    const uint32_t nm = S.nm;
    std::vector<int32_t> indeg(Md->n_max, -1);
    typedef std::pair<uint64_t, uint32_t> E;
    std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
    auto key = [&](uint32_t b, uint32_t i, uint32_t j, uint32_t k, uint32_t K) -> uint64_t {
        (void)K;
        const uint32_t c = (uint32_t)S.cls_of[b * nm + i] + k + (dir ? S.C : 0);
        const uint64_t rank = (uint64_t)(S.Cn - 1 - prio[c]);                 // higher priority first
        return (rank << 40) | ((uint64_t)j << 24);
    };
    for (uint32_t b = 0; b < S.m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            const uint32_t q = b * nm + i, K = Md->Kv[i];
            for (uint32_t j = 0; j < S.M[q]; j++)
                for (uint32_t k = 0; k < K; k++) {
                    const uint32_t s = Md->sbase[q] + j * K + k;
                    int32_t d = 0;
                    if (dir == 0) {
                        if (k > 0) d = 1;
                        else for (uint32_t p = 0; p < nm; p++)
                            if ((Md->prod_mask[i] >> p) & 1u) d += S.M[b * nm + p];
                    } else {
                        if (k + 1 < K) d = 1;
                        else for (uint32_t c = 0; c < nm; c++)
                            if ((Md->cons_mask[i] >> c) & 1u) d += S.M[b * nm + c];
                    }
                    indeg[s] = d;
                    if (d == 0) pq.push(E(key(b, i, j, k, K), s));
                }
        }
    uint32_t cnt = 0;
    while (!pq.empty()) {
        const uint32_t s = pq.top().second;
        pq.pop();
        out[cnt++] = (uint16_t)s;
        const uint32_t q = S.q_of_seg[s];                                    // s -> (b, i, j, k)
        const uint32_t b = q / nm, i = q % nm, K = Md->Kv[i], j = (s - Md->sbase[q]) / K, k = (s - Md->sbase[q]) % K;
        auto relax = [&](uint32_t t, uint32_t tb, uint32_t ti, uint32_t tj, uint32_t tk) {
            if (--indeg[t] == 0) pq.push(E(key(tb, ti, tj, tk, Md->Kv[ti]), t));
        };
        if (dir == 0) {
            if (k + 1 < K) relax(s + 1, b, i, j, k + 1);
            else for (uint32_t c = 0; c < nm; c++)
                if ((Md->cons_mask[i] >> c) & 1u)
                    for (uint32_t jj = 0; jj < S.M[b * nm + c]; jj++)
                        relax(Md->sbase[b * nm + c] + jj * Md->Kv[c], b, c, jj, 0);
        } else {
            if (k > 0) relax(s - 1, b, i, j, k - 1);
            else for (uint32_t p = 0; p < nm; p++)
                if ((Md->prod_mask[i] >> p) & 1u)
                    for (uint32_t jj = 0; jj < S.M[b * nm + p]; jj++)
                        relax(Md->sbase[b * nm + p] + jj * Md->Kv[p] + Md->Kv[p] - 1, b, p, jj, Md->Kv[p] - 1);
        }
    }
    for (uint32_t p = cnt; p < Md->n_pad; p++) out[p] = 0xFFFF;
}

// one record (split nibbles + priority orders; the F/B bits are filled by the GPU interleaving)
void build_record(const dip_model *Md, const Setup &S, const std::vector<uint32_t> &seq, uint8_t *rec) {
    std::memset(rec, 0, Md->stride);
    const uint16_t n16 = (uint16_t)S.n;
    std::memcpy(rec, &n16, 2);
    for (uint32_t b = 0; b < S.m; b++)
        for (uint32_t i = 0; i < S.nm; i++)
            if (Md->max_split[i] > 1) {
                const uint32_t nib = b * Md->nsplit + Md->nib_slot[i];
                rec[Md->off_nib + nib / 2] |= (uint8_t)((S.M[b * S.nm + i] & 15u) << ((nib & 1) * 4));
            }
    std::vector<uint32_t> prio(S.Cn);
    for (uint32_t p = 0; p < S.Cn; p++) prio[seq[p]] = S.Cn - 1 - p;   // position p -> priority Cn-1-p
    order(Md, S, prio, 0, reinterpret_cast<uint16_t *>(rec + Md->off_fwd));
    order(Md, S, prio, 1, reinterpret_cast<uint16_t *>(rec + Md->off_bwd));
}

}  // namespace

extern "C" dip_status dip_search(const dip_model *Md, dip_workspace *w, const uint8_t *split,
                                 const dip_search_params *prm, void *best_record_out, uint16_t *best_orders_out,
                                 double *trace, dip_search_result *out, void *stream) {
    if (!Md || !w || w->model != Md || !split || !prm || !out) return fail(DIP_EINVAL, "null argument");
    if (prm->rounds == 0 || prm->leaves == 0 || prm->rollouts == 0) return fail(DIP_EINVAL, "empty budget");
    if (prm->memopt && !Md->S) return fail(DIP_EINVAL, "memopt rollouts need a strategy menu (dip_set_strategies)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Setup S;
    S.P = Md->P; S.nm = Md->nmod; S.m = Md->m;
    S.M.assign(split, split + S.m * S.nm);
    S.cls_of.assign(S.m * S.nm, -1);
    S.n = 0;
    S.C = 0;
    for (uint32_t b = 0; b < S.m; b++)
        for (uint32_t i = 0; i < S.nm; i++) {
            const uint32_t q = b * S.nm + i, N = Md->nbi[q], Mv = S.M[q];
            if ((N == 0) != (Mv == 0) || Mv > std::min(N, Md->max_split[i])) return fail(DIP_EINVAL, "invalid split");
            if (Mv) { S.cls_of[q] = (int)S.C; S.C += Md->Kv[i]; S.cls_q.push_back(q); }
            S.n += Mv * Md->Kv[i];
        }
    S.q_of_seg.assign(Md->n_max, 0);
    for (uint32_t q = 0; q < S.m * S.nm; q++)
        for (uint32_t x = 0; x < Md->max_split[q % S.nm] * Md->Kv[q % S.nm]; x++) S.q_of_seg[Md->sbase[q] + x] = q;
    S.Cn = 2 * S.C;
    std::memset(out, 0, sizeof(*out));
    if (S.C == 0) { out->found = 1; return DIP_OK; }
    // LB = the busiest rank's total latency of this split (score = LB / makespan <= 1)
    {
        double lb = 0.0;
        for (uint32_t r = 0; r < S.P; r++) {
            uint64_t tot = 0;
            for (uint32_t q : S.cls_q) {
                const uint32_t i = q % S.nm, K = Md->Kv[i], Mv = S.M[q];
                for (uint32_t j = 0; j < Mv; j++) {
                    const uint32_t W = Md->wtab[Md->woff[q] + Mv * (Mv - 1) / 2 + j];
                    const uint32_t t = Md->tab_off[i] + W;
                    for (uint32_t k = 0; k < K; k++)
                        tot += (uint64_t)Md->layers[Md->lay_off[i] + k * S.P + r] * ((uint64_t)Md->tab[4 * t] + Md->tab[4 * t + 1]);
                }
            }
            lb = std::max(lb, (double)tot);
        }
        S.LB = lb;
    }
    const uint32_t R = prm->rollouts, B = prm->leaves;
    const size_t cap = (size_t)B * R;
    PinnedBuf<uint8_t> h_rec(cap * Md->stride);      // pinned: the per-round H2D runs at full PCIe rate
    PinnedBuf<dip_result> h_res(cap);
    if (!h_rec.data() || !h_res.data()) return fail(DIP_ENOMEM, "search host buffers");
    uint8_t *d_rec = nullptr;
    dip_result *d_res = nullptr;
    uint8_t *d_sel = nullptr;
    uint16_t *d_ord = nullptr;
    const size_t ord_elems = (size_t)Md->P * 2 * Md->n_max;     // per-rank orders of one rollout
    CUDA_TRY(cudaMalloc(&d_rec, cap * Md->stride));
    if (cudaMalloc(&d_res, cap * sizeof(dip_result)) != cudaSuccess) { cudaFree(d_rec); return fail(DIP_ENOMEM, "search buffers"); }
    if (cudaMalloc(&d_ord, cap * ord_elems * 2) != cudaSuccess ||
        (prm->memopt && cudaMalloc(&d_sel, cap * Md->P * 2ull * Md->n_max) != cudaSuccess)) {
        cudaFree(d_rec); cudaFree(d_res);
        if (d_ord) cudaFree(d_ord);
        return fail(DIP_ENOMEM, "search buffers");
    }
    std::vector<Node> tree(1);
    tree.reserve(1 + (size_t)prm->rounds * B);
    double best = -1.0;
    uint64_t best_mk = ~0ull, u = 0, scored = 0;
    // record-building threads: all cores by default, but not more than one per 32 rollouts of a round
    int nth = prm->threads > 0 ? prm->threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nth = std::max(1, std::min<int>(nth, (int)((cap + 31) / 32)));
    dip_status status = DIP_OK;
    uint32_t rd = 0;
    const bool prof = std::getenv("DIP_SEARCH_PROFILE") != nullptr;   // per-phase wall times to stderr
    double t_sel = 0, t_build = 0, t_gpu = 0, t_back = 0;
    auto now = []() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    if (prm->policy < 0 || prm->policy > 2) { cudaFree(d_rec); cudaFree(d_res); cudaFree(d_ord); if (d_sel) cudaFree(d_sel);
        return fail(DIP_EINVAL, "policy must be 0 (MCTS), 1 (random) or 2 (DFS)"); }
    int dfs_cur = 0;
    const double t_start = now();
    for (; rd < prm->rounds; rd++) {
        double t0 = now();
        // ---- selection + expansion of B leaves (virtual visits keep the batch diverse)
        std::vector<int> leaf(B);
        std::vector<std::vector<uint32_t>> prefixes(B);
        std::vector<int> owner;
        std::vector<uint64_t> ctr;
        for (uint32_t l = 0; l < B; l++) {
            int v = 0;
            std::vector<char> used(S.Cn, 0);
            if (prm->policy == 2) {   // DFS: from the previous leaf, up to the nearest node with an unexpanded child
                v = dfs_cur;
                while (v > 0 && tree[v].children.size() >= S.Cn - (uint32_t)tree[v].depth) v = tree[v].parent;
                if (v == 0 && tree[0].children.size() >= S.Cn) v = dfs_cur;   // the whole tree is explored
                for (int x = v; x > 0; x = tree[x].parent) used[tree[x].cls] = 1;
            }
            for (; prm->policy != 1;) {   // (random exploration: the root)
                Node &nd = tree[v];
                if ((uint32_t)nd.depth == S.Cn) break;
                const uint32_t remaining = S.Cn - nd.depth;
                if (nd.children.size() < remaining) {            // expansion: next class in order
                    uint32_t c = 0, seen = 0;
                    for (c = 0; c < S.Cn; c++) {
                        if (used[c]) continue;
                        if (seen++ == nd.children.size()) break;
                    }
                    Node ch;
                    ch.parent = v; ch.cls = (int)c; ch.depth = nd.depth + 1;
                    tree.push_back(ch);
                    const int id = (int)tree.size() - 1;
                    tree[v].children.push_back(id);
                    used[c] = 1;
                    v = id;
                    break;
                }
                if (prm->policy == 2) break;                    // DFS: a complete leaf again
                const double Nx = (double)(nd.N + nd.vloss), lnNx = std::log(Nx);
                const bool a1 = prm->alpha == 1.0;       // pow(s, 1) is s exactly: skip the call
                int bestc = -1;
                double bu = -1.0;
                for (int c : nd.children) {
                    const Node &cn = tree[c];
                    const double Nv = (double)(cn.N + cn.vloss);
                    const double ucb = (a1 ? cn.s : std::pow(cn.s, prm->alpha)) + prm->beta * std::sqrt(lnNx / Nv);
                    if (ucb > bu) { bu = ucb; bestc = c; }
                }
                used[tree[bestc].cls] = 1;
                v = bestc;
            }
            for (int x = v; x >= 0; x = tree[x].parent) tree[x].vloss++;
            leaf[l] = v;
            dfs_cur = v;
            // the fixed prefix; its R uniformly random completions (one for a complete sequence) are
            // drawn by the record-building threads below, each from its own counter-based stream
            std::vector<uint32_t> prefix;
            for (int x = v; x > 0; x = tree[x].parent) prefix.push_back((uint32_t)tree[x].cls);
            std::reverse(prefix.begin(), prefix.end());
            prefixes[l] = prefix;
            const uint32_t trials = (uint32_t)tree[v].depth == S.Cn ? 1 : R;
            for (uint32_t tr = 0; tr < trials; tr++) {
                owner.push_back((int)l);
                ctr.push_back(u);
                u++;
            }
        }
        // ---- rollouts: sequences + records on the host (threads), interleave + score on the GPU
        const size_t cnt = owner.size();
        double t1 = now();
        t_sel += t1 - t0;
        {
            std::vector<std::thread> th;
            const size_t per = (cnt + nth - 1) / nth;
            for (int t = 0; t < nth; t++) {
                const size_t lo = per * t, hi = std::min(cnt, lo + per);
                if (lo >= hi) break;
                th.emplace_back([&, lo, hi]() {
                    std::vector<char> inpre(S.Cn);
                    std::vector<uint32_t> seq, rest;
                    for (size_t x = lo; x < hi; x++) {
                        const std::vector<uint32_t> &prefix = prefixes[owner[x]];
                        std::fill(inpre.begin(), inpre.end(), 0);
                        for (uint32_t c : prefix) inpre[c] = 1;
                        rest.clear();
                        for (uint32_t c = 0; c < S.Cn; c++) if (!inpre[c]) rest.push_back(c);
                        uint64_t rs = mix64(prm->seed ^ mix64(ctr[x] + 0x51A9u));
                        for (uint32_t y = (uint32_t)rest.size(); y > 1; y--) {
                            rs += 0x9E3779B97F4A7C15ull;
                            const uint32_t z = (uint32_t)(mix64(rs) % y);
                            std::swap(rest[y - 1], rest[z]);
                        }
                        seq.assign(prefix.begin(), prefix.end());
                        seq.insert(seq.end(), rest.begin(), rest.end());
                        build_record(Md, S, seq, &h_rec[x * Md->stride]);
                    }
                });
            }
            for (auto &t : th) t.join();
        }
        double t2 = now();
        t_build += t2 - t1;
        if (cudaMemcpyAsync(d_rec, h_rec.data(), cnt * Md->stride, cudaMemcpyHostToDevice, st) != cudaSuccess) {
            status = fail(DIP_ECUDA, "search H2D");
            break;
        }
        status = dip_interleave(Md, w, d_rec, cnt, d_res, nullptr, d_ord, stream);
        if (status != DIP_OK) break;
        if (prm->memopt) {   // interleaving, then per-layer memory optimisation (f3)
            status = dip_memopt(Md, w, d_rec, d_ord, cnt, d_sel, d_res, nullptr, stream);
            if (status != DIP_OK) break;
        }
        if (cudaMemcpyAsync(h_res.data(), d_res, cnt * sizeof(dip_result), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            status = fail(DIP_ECUDA, "search D2H");
            break;
        }
        scored += cnt;
        double t3 = now();
        t_gpu += t3 - t2;
        // ---- backpropagation, leaf by leaf
        std::vector<double> lbest(B, 0.0);
        size_t arg = cnt;
        for (size_t x = 0; x < cnt; x++) {
            const double sc = h_res[x].status == DIP_CAND_OK ? S.LB / (double)h_res[x].makespan_ns : 0.0;
            lbest[owner[x]] = std::max(lbest[owner[x]], sc);
            if (sc > best) { best = sc; best_mk = h_res[x].makespan_ns; arg = x; }
        }
        for (uint32_t l = 0; l < B; l++)
            for (int x = leaf[l]; x >= 0; x = tree[x].parent) {
                tree[x].s = std::max(tree[x].s, lbest[l]);
                tree[x].N++;
                tree[x].vloss--;
            }
        if (arg < cnt && best_record_out) {
            if (cudaMemcpy(best_record_out, d_rec + arg * Md->stride, Md->stride, cudaMemcpyDeviceToHost) != cudaSuccess) {
                status = fail(DIP_ECUDA, "search best record");
                break;
            }
        }
        if (arg < cnt && best_orders_out) {
            if (cudaMemcpy(best_orders_out, d_ord + arg * ord_elems, ord_elems * 2, cudaMemcpyDeviceToHost) != cudaSuccess) {
                status = fail(DIP_ECUDA, "search best orders");
                break;
            }
        }
        if (trace) trace[rd] = best;
        t_back += now() - t3;
        if (prm->time_budget_ms > 0 && (now() - t_start) * 1e3 >= prm->time_budget_ms) { rd++; break; }
    }
    if (prof)
        std::fprintf(stderr, "dip_search: select %.1f ms, build %.1f ms, gpu %.1f ms, backprop %.1f ms over %u rounds\n",
                     t_sel * 1e3, t_build * 1e3, t_gpu * 1e3, t_back * 1e3, rd);
    cudaFree(d_rec);
    cudaFree(d_res);
    cudaFree(d_ord);
    if (d_sel) cudaFree(d_sel);
    if (status != DIP_OK) return status;
    out->found = best > 0.0;
    out->makespan_ns = out->found ? best_mk : ~0ull;
    out->score = std::max(best, 0.0);
    out->rollouts_scored = scored;
    out->rounds_done = rd;
    out->tree_nodes = tree.size();
    return DIP_OK;
}
