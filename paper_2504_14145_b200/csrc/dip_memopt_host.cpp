// dip_memopt_host.cpp -- C-ABI of SURVEY §8(f) row f3 (§5.3): strategy menu ->
// GPU candidate table (dip_mcand_kernel), per-rank greedy selection (dip_memopt_kernel) and the
// re-timing with the selected candidates (scorer MODE 3). See include/dip.h for the contract.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "dip_host_internal.h"

using namespace diph;

extern "C" dip_status dip_set_strategies(dip_model *M, uint32_t n_strat, const uint32_t *f_ns, const uint32_t *b_ns,
                                         const uint32_t *act_kib, uint32_t S) {
    if (!M || !f_ns || !b_ns || !act_kib) return fail(DIP_EINVAL, "null argument");
    if (M->device < 0 || !M->d_blob) return fail(DIP_EINVAL, "host-only model (cuda_device < 0)");
    if (n_strat < 1 || n_strat > 8) return fail(DIP_EINVAL, "n_strat must be in 1..8");
    if (S < 2 || S > 16) return fail(DIP_EINVAL, "S must be in 2..16");
    CUDA_TRY(cudaSetDevice(M->device));
    const uint32_t nm = M->nmod, P = M->P, T = (uint32_t)(M->tab.size() / 4);
    // candidate types = distinct (module, layers per chunk); crow[row] = type base - tab_off * S
    std::map<std::pair<uint32_t, uint32_t>, uint32_t> type_of;
    std::vector<uint32_t> t_mod, t_lay, t_base, t_item, t_toff;
    std::vector<int32_t> crow(M->layers.size(), 0);
    uint32_t base = 0, items = 0;
    for (uint32_t i = 0; i < nm; i++) {
        const uint32_t wn = (i + 1 < nm ? M->tab_off[i + 1] : T) - M->tab_off[i];
        for (uint32_t c = 0; c < P * M->Kv[i]; c++) {
            const uint32_t row = M->lay_off[i] + c, l = M->layers[row];
            auto key = std::make_pair(i, l);
            auto it = type_of.find(key);
            uint32_t t;
            if (it == type_of.end()) {
                t = (uint32_t)t_mod.size();
                type_of[key] = t;
                t_mod.push_back(i); t_lay.push_back(l); t_base.push_back(base); t_item.push_back(items);
                t_toff.push_back(M->tab_off[i]);
                // guards: u32 pair totals, bounded enumeration
                uint64_t mx = 0;
                for (uint32_t s = 0; s < n_strat; s++)
                    for (uint32_t w = 0; w < wn; w++) {
                        const size_t o = (size_t)s * T + M->tab_off[i] + w;
                        mx = std::max<uint64_t>(mx, std::max(f_ns[o], std::max(b_ns[o], act_kib[o])));
                    }
                if ((unsigned __int128)mx * l * 2 >= ((unsigned __int128)1 << 32))
                    return fail(DIP_ERANGE, "a stage-pair total may exceed u32");
                double combos = 1.0;
                for (uint32_t s = 1; s < n_strat; s++) combos *= (double)(l + 1);
                if (combos > (double)(1u << 20)) return fail(DIP_ERANGE, "too many strategy combinations per pair");
                base += wn * S;
                items += wn;
            } else {
                t = it->second;
            }
            crow[row] = (int32_t)t_base[t] - (int32_t)(M->tab_off[i] * S);
        }
    }
    if ((uint64_t)base >= (1ull << 31) || base / S >= 65536u)   // the selection keeps u16 row indices
        return fail(DIP_ERANGE, "candidate table too large");
    // device buffers
    std::vector<void *> tmp;
    auto cleanup = [&]() { for (void *p : tmp) cudaFree(p); };
    auto upload = [&](const void *src, size_t bytes, void **dst) -> bool {
        if (cudaMalloc(dst, bytes ? bytes : 4) != cudaSuccess) return false;
        tmp.push_back(*dst);
        return !bytes || cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    dipk::MCandParams p{};
    void *d_mf, *d_mb, *d_ma, *d_ti, *d_tl, *d_tt, *d_tb;
    const size_t mb = (size_t)n_strat * T * 4, tb = t_mod.size() * 4;
    if (!upload(f_ns, mb, &d_mf) || !upload(b_ns, mb, &d_mb) || !upload(act_kib, mb, &d_ma) ||
        !upload(t_item.data(), tb, &d_ti) || !upload(t_lay.data(), tb, &d_tl) || !upload(t_toff.data(), tb, &d_tt) ||
        !upload(t_base.data(), tb, &d_tb)) {
        cleanup();
        return fail(DIP_ECUDA, "strategy menu upload");
    }
    uint4 *d_ctab = nullptr;
    int32_t *d_crow = nullptr;
    if (cudaMalloc(&d_ctab, (size_t)base * sizeof(uint4)) != cudaSuccess ||
        cudaMalloc(&d_crow, crow.size() * 4) != cudaSuccess) {
        cleanup();
        if (d_ctab) cudaFree(d_ctab);
        return fail(DIP_ENOMEM, "candidate table");
    }
    p.n_items = items; p.n_types = (uint32_t)t_mod.size(); p.n_strat = n_strat; p.S = S; p.T = T;
    p.t_item = (const uint32_t *)d_ti; p.t_lay = (const uint32_t *)d_tl; p.t_toff = (const uint32_t *)d_tt;
    p.t_base = (const uint32_t *)d_tb;
    p.mf = (const uint32_t *)d_mf; p.mb = (const uint32_t *)d_mb; p.ma = (const uint32_t *)d_ma;
    p.ctab = d_ctab;
    cudaError_t e = dipk::launch_mcand(p, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    g_launches++;
    std::vector<uint4> h(base);
    if (e == cudaSuccess) e = cudaMemcpy(h.data(), d_ctab, (size_t)base * sizeof(uint4), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(d_crow, crow.data(), crow.size() * 4, cudaMemcpyHostToDevice);
    cleanup();
    if (e != cudaSuccess) {
        cudaFree(d_ctab); cudaFree(d_crow);
        return fail(DIP_ECUDA, std::string("candidate generation: ") + cudaGetErrorString(e));
    }
    // the selection needs strictly increasing memory and strictly decreasing latency
    for (size_t row = 0; row < base; row += S) {
        const uint32_t k = h[row].w;
        if (k < 1 || k > S) { cudaFree(d_ctab); cudaFree(d_crow); return fail(DIP_ECUDA, "candidate table corrupt"); }
        for (uint32_t c = 1; c < k; c++) {
            const uint4 &a = h[row + c - 1], &b = h[row + c];
            if (!(b.z > a.z && (uint64_t)b.x + b.y < (uint64_t)a.x + a.y)) {
                cudaFree(d_ctab); cudaFree(d_crow);
                return fail(DIP_ERANGE, "menu yields candidates of equal memory or latency");
            }
        }
    }
    {   // the makespan bound of f3's re-timing: a selected candidate's stage latency may exceed the
        // base tables' (a menu whose strategy 0 is not the base scheme), so the fused argmin key's
        // packing and the 2^53 bubble guard are re-checked with the candidate table's largest stage
        uint64_t maxc = 0, maxp2p = 0;
        for (size_t x = 0; x < h.size(); x++) maxc = std::max<uint64_t>(maxc, std::max(h[x].x, h[x].y));
        for (size_t t = 0; t + 3 < M->tab.size(); t += 4) maxp2p = std::max<uint64_t>(maxp2p, M->tab[t + 3]);
        const unsigned __int128 b3 = (unsigned __int128)P * 2ull * M->n_max * (maxc + maxp2p);
        if (b3 * P >= ((unsigned __int128)1 << 53)) {
            cudaFree(d_ctab); cudaFree(d_crow);
            return fail(DIP_ERANGE, "makespan bound with the strategy candidates exceeds 2^53 / P");
        }
        if ((uint64_t)b3 > M->mk_bound) M->mk_bound = (uint64_t)b3;
    }
    {   // the selection keeps slack in int32: budget and the live memory must stay below 2^31 KiB
        uint64_t maxmem = 0, maxbud = 0;
        for (size_t x = 0; x < h.size(); x++) maxmem = std::max<uint64_t>(maxmem, h[x].z);
        const uint32_t *bud = reinterpret_cast<const uint32_t *>(M->blob.data() + M->kp.b_budget);
        for (uint32_t r = 0; r < P; r++) maxbud = std::max<uint64_t>(maxbud, bud[r]);
        if (maxbud >= (1ull << 31) || (unsigned __int128)maxmem * M->n_max + maxbud >= ((unsigned __int128)1 << 31)) {
            cudaFree(d_ctab); cudaFree(d_crow);
            return fail(DIP_ERANGE, "budget / live memory of a rank may exceed 2^31 KiB");
        }
    }
    // exact ranking of every step c -> c+1 by latency saving per KiB (equal ratios share a rank):
    // the selection kernel then compares 32-bit keys (rank, pair) instead of cross-multiplying
    std::vector<uint16_t> srank(base, 0xFFFFu);
    {
        struct Step { uint64_t dl, dm; uint32_t at; };
        std::vector<Step> steps;
        for (size_t row = 0; row < base; row += S)
            for (uint32_t c = 0; c + 1 < h[row].w; c++) {
                const uint4 &a = h[row + c], &b = h[row + c + 1];
                steps.push_back({(uint64_t)a.x + a.y - ((uint64_t)b.x + b.y), (uint64_t)b.z - a.z, (uint32_t)(row + c)});
            }
        auto better = [](const Step &x, const Step &y) {
            return (unsigned __int128)x.dl * y.dm > (unsigned __int128)y.dl * x.dm;
        };
        std::stable_sort(steps.begin(), steps.end(), better);
        uint32_t rank = 0;
        for (size_t x = 0; x < steps.size(); x++) {
            if (x > 0 && better(steps[x - 1], steps[x])) rank++;
            if (rank >= 0xFFFFu) { cudaFree(d_ctab); cudaFree(d_crow); return fail(DIP_ERANGE, "more than 65534 distinct step ratios"); }
            srank[steps[x].at] = (uint16_t)rank;
        }
    }
    uint16_t *d_srank = nullptr;
    if (cudaMalloc(&d_srank, srank.size() * 2 + 2) != cudaSuccess ||
        cudaMemcpy(d_srank, srank.data(), srank.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d_ctab); cudaFree(d_crow);
        if (d_srank) cudaFree(d_srank);
        return fail(DIP_ECUDA, "step ranks");
    }
    if (M->d_ctab) cudaFree(M->d_ctab);
    if (M->d_crow) cudaFree(M->d_crow);
    if (M->d_srank) cudaFree(M->d_srank);
    M->d_srank = d_srank;
    M->kp.srank = d_srank;
    M->d_ctab = d_ctab;
    M->d_crow = d_crow;
    M->h_ctab.swap(h);
    M->t_mod = t_mod; M->t_lay = t_lay; M->t_base = t_base;
    M->n_strat = n_strat;
    M->S = S;
    M->kp.ctab = d_ctab;
    M->kp.crow = d_crow;
    M->kp.S = S;
    // selection kernel shape: 4 warps per block, per-warp working set in shared memory
    const uint32_t nmx = M->n_max, nq = M->m * nm;
    M->mo_warp_bytes = up16(((4 * ((nmx + 1) & ~1u) + nmx * (8 + 2 + 2 + 1) + nq + 3) & ~3u) + 4 * ((nmx + 31) / 32));
    const size_t smem = 4 * (size_t)M->mo_warp_bytes;
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, M->device));
    if (smem > prop.sharedMemPerBlockOptin) return fail(DIP_ERANGE, "memopt working set exceeds shared memory");
    CUDA_TRY(dipk::prepare_memopt(smem));
    int bps = 0;
    CUDA_TRY(dipk::occupancy_memopt(smem, &bps));
    M->mo_grid = M->num_sms * std::max(1, bps);
    return DIP_OK;
}

extern "C" dip_status dip_strategy_candidates(const dip_model *M, uint32_t module, uint32_t layers, uint32_t W,
                                              uint64_t *out, uint32_t *count) {
    if (!M || !out || !count) return fail(DIP_EINVAL, "null argument");
    if (!M->S) return fail(DIP_EINVAL, "no strategy menu (dip_set_strategies)");
    for (size_t t = 0; t < M->t_mod.size(); t++) {
        if (M->t_mod[t] != module || M->t_lay[t] != layers) continue;
        const uint32_t T = (uint32_t)(M->tab.size() / 4);
        const uint32_t wn = (module + 1 < M->nmod ? M->tab_off[module + 1] : T) - M->tab_off[module];
        if (W >= wn) return fail(DIP_EINVAL, "W > w_max");
        const uint4 *row = M->h_ctab.data() + M->t_base[t] + (size_t)W * M->S;
        *count = row[0].w;
        for (uint32_t c = 0; c < row[0].w; c++) {
            out[3 * c] = row[c].x;
            out[3 * c + 1] = row[c].y;
            out[3 * c + 2] = row[c].z;
        }
        return DIP_OK;
    }
    return fail(DIP_EINVAL, "no stage pair of this (module, layers)");
}

extern "C" dip_status dip_memopt(const dip_model *M, dip_workspace *w, const void *d_records, const uint16_t *d_orders,
                                 size_t count, uint8_t *d_sel, dip_result *d_results, uint32_t *d_peaks, void *stream) {
    if (!M || !w || w->model != M) return fail(DIP_EINVAL, "model / workspace mismatch");
    if (!M->S) return fail(DIP_EINVAL, "no strategy menu (dip_set_strategies)");
    if (count && (!d_records || !d_results || !d_sel)) return fail(DIP_EINVAL, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t idx_bits = bits_for(std::max<uint64_t>(count, 2));
    const bool fused = fused_ok(M, idx_bits);
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 1, 0xFF, sizeof(unsigned long long), s));
    w->last_results = d_results;
    w->last_count = count;
    w->last_idx_bits = idx_bits;
    w->last_fused = fused;
    if (!count) return DIP_OK;
    dipk::KParams kp = M->kp;
    kp.records = static_cast<const uint8_t *>(d_records);
    kp.count = count;
    kp.counter = w->d_misc + 5;
    kp.mo_stats = w->d_misc + 10;
    kp.orders_in = d_orders;
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 5, 0, sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 10, 0, 5 * sizeof(unsigned long long), s));
    const uint64_t warps = std::min<uint64_t>((uint64_t)M->mo_grid * 4, count * M->P);
    CUDA_TRY(dipk::launch_memopt(kp, d_sel, M->mo_warp_bytes, (int)((warps + 3) / 4), s));
    g_launches++;
    if (d_orders)   // M4 on explicit orders: the per-rank-order kernel's timing with the selection
        return dip_eval_orders(M, w, d_records, d_orders, count, d_sel, d_results, d_peaks, nullptr, nullptr, s);
    return launch_chunk(M, w, d_records, count, 0, idx_bits, fused, d_results, d_peaks, s, nullptr, d_sel);
}

extern "C" dip_status dip_set_memopt_solver(dip_model *M, uint32_t gap_permille, uint32_t node_cap) {
    if (!M) return fail(DIP_EINVAL, "null model");
    if (gap_permille > 1000 || node_cap == 0) return fail(DIP_EINVAL, "gap_permille must be <= 1000, node_cap > 0");
    M->kp.gap_pm = gap_permille;
    M->kp.node_cap = node_cap;
    return DIP_OK;
}

extern "C" dip_status dip_memopt_stats(const dip_workspace *w, uint64_t *out, void *stream) {
    if (!w || !out) return fail(DIP_EINVAL, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaMemcpyAsync(out, w->d_misc + 10, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return DIP_OK;
}
