// dip_host.cpp -- the C-ABI (include/dip.h): batch setup, candidate packing, launches,
// argmin with the NCCL allreduce, and the end-to-end host path.
//
// (a1) batch setup: derive layers per chunk (R-3),
//      the segment-id decode table, per (microbatch, module) the balanced-split work
//      table W_j for every M in [1, M_max] (R-2), the per-layer cost rows, and
//      pack them into one 16-B aligned blob that the kernel stages into shared memory
//      with a TMA bulk copy.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "dip.h"
#include "dip_host_internal.h"
#include "dip_internal.h"

using dipk::KParams;
using dipk::ModInfo;

thread_local std::string diph::g_err;
std::atomic<uint64_t> diph::g_launches{0};

using namespace diph;

static void fill_shape(dip_model *M) {
    KParams &kp = M->kp;
    kp.P = M->P; kp.nmod = M->nmod; kp.m = M->m; kp.n_max = M->n_max; kp.n_pad = M->n_pad; kp.fbw = M->fbw;
    kp.stride = M->stride;
    kp.off_nib = M->off_nib; kp.off_fwd = M->off_fwd; kp.off_bwd = M->off_bwd; kp.off_fb = M->off_fb;
    kp.nsplit = M->nsplit;
    kp.warps_per_block = M->wpb;
    kp.cpg = M->cpg;
    if (!kp.node_cap) {            // f3 solver defaults (dip_set_memopt_solver): 5 % gap
        kp.gap_pm = 50;
        kp.node_cap = 4096;
    }
}

extern "C" {

const char *dip_status_str(dip_status s) {
    switch (s) {
    case DIP_OK: return "DIP_OK";
    case DIP_EINVAL: return "DIP_EINVAL";
    case DIP_ECUDA: return "DIP_ECUDA";
    case DIP_ENOMEM: return "DIP_ENOMEM";
    case DIP_ERANGE: return "DIP_ERANGE";
    case DIP_ENCCL: return "DIP_ENCCL";
    case DIP_ENOFEASIBLE: return "DIP_ENOFEASIBLE";
    }
    return "DIP_?";
}
const char *dip_last_error(void) { return g_err.c_str(); }
uint64_t dip_launch_count(void) { return g_launches.load(); }

dip_status dip_load_cost_model(const dip_problem_desc *d, int cuda_device, dip_model **out) {
    if (!d || !out || !d->modules || !d->inst_off || !d->budget_kib) return fail(DIP_EINVAL, "null argument");
    const uint32_t P = d->P, nm = d->n_modules, m = d->m;
    if (P < 1 || P > 32) return fail(DIP_EINVAL, "P must be in 1..32");
    if (nm < 1 || nm > 8) return fail(DIP_EINVAL, "n_modules must be in 1..8");
    if (m < 1 || m > 255) return fail(DIP_EINVAL, "m must be in 1..255");
    dip_model *M = new (std::nothrow) dip_model();
    if (!M) return fail(DIP_ENOMEM, "host allocation");
    struct Guard {   // on any failure below, release what was allocated so far
        dip_model *m;
        ~Guard() { if (m) dip_model_free(m); }
        dip_model *release() { dip_model *x = m; m = nullptr; return x; }
    } guard{M};
    M->device = cuda_device;
    M->P = P; M->nmod = nm; M->m = m;

    // ---- per module: chunks (R-3), consumers, table offsets
    std::vector<ModInfo> mi(nm);
    std::vector<uint16_t> layers;
    std::vector<uint32_t> tab;   // 4 x u32 per entry
    uint32_t maxlat_layers = 0;
    uint64_t maxlat = 0, maxp2p = 0, maxact = 0;
    uint32_t nsplit = 0;
    for (uint32_t i = 0; i < nm; i++) {
        const dip_module_desc &md = d->modules[i];
        if (md.K < 1 || md.K > 255) return fail(DIP_EINVAL, "K must be in 1..255");
        if (md.max_split < 1 || md.max_split > 15) return fail(DIP_EINVAL, "max_split must be in 1..15");
        if (!md.f_ns || !md.b_ns || !md.act_kib) return fail(DIP_EINVAL, "null cost table");
        if (md.producer_mask >> i) return fail(DIP_EINVAL, "producer_mask must name earlier modules only");
        const uint32_t C = P * md.K;
        if (!md.chunk_layers && C > md.L) return fail(DIP_EINVAL, "P*K > L (TooManyChunks)");
        ModInfo &x = mi[i];
        x.K = md.K;
        x.max_split = md.max_split;
        x.prod_mask = md.producer_mask;
        x.cons_mask = 0;
        for (uint32_t c = 0; c < nm; c++)
            if ((d->modules[c].producer_mask >> i) & 1u) x.cons_mask |= 1u << c;
        x.lay_off = (uint32_t)layers.size();
        for (uint32_t c = 0; c < C; c++) {
            const uint32_t l = md.chunk_layers ? md.chunk_layers[c] : md.L / C + (c < md.L % C ? 1u : 0u);
            if (l > 65535) return fail(DIP_ERANGE, "layers per chunk > 65535");
            layers.push_back((uint16_t)l);
            maxlat_layers = std::max(maxlat_layers, l);
        }
        x.tab_off = (uint32_t)(tab.size() / 4);
        x.w_max = md.w_max;
        for (uint32_t w = 0; w <= md.w_max; w++) {
            const uint32_t p2p = (md.p2p_ns && P > 1) ? md.p2p_ns[w] : 0u;   // P = 1: no cross-rank edge
            tab.push_back(md.f_ns[w]);
            tab.push_back(md.b_ns[w]);
            tab.push_back(md.act_kib[w]);
            tab.push_back(p2p);
            maxlat = std::max<uint64_t>(maxlat, std::max(md.f_ns[w], md.b_ns[w]));
            maxact = std::max<uint64_t>(maxact, md.act_kib[w]);
            maxp2p = std::max<uint64_t>(maxp2p, p2p);
        }
        x.nib_slot = md.max_split > 1 ? nsplit++ : 0xFFu;
        M->max_split.push_back(md.max_split);
        M->nib_slot.push_back(x.nib_slot);
    }
    if (tab.size() / 4 > 4096 || layers.size() > 4096) return fail(DIP_ERANGE, "tables exceed the 12-bit row indices");

    // ---- segment ids, decode table, per-(b,i) base, balanced-split work table (R-2)
    uint32_t n_max = 0;
    std::vector<uint16_t> sbase(m * nm);
    std::vector<uint32_t> segdec;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            sbase[b * nm + i] = (uint16_t)n_max;
            for (uint32_t j = 0; j < mi[i].max_split; j++)
                for (uint32_t k = 0; k < mi[i].K; k++) segdec.push_back(dipk::segdec_pack(b, i, j, k, mi[i].K));
            n_max += mi[i].max_split * mi[i].K;
            if (n_max > 32766) return fail(DIP_ERANGE, "segment-id space exceeds 32766");
        }
    std::vector<uint32_t> woff(m * nm);
    std::vector<uint16_t> wtab, nbi(m * nm);
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            const uint32_t q = b * nm + i, lo = d->inst_off[q], hi = d->inst_off[q + 1];
            if (hi < lo) return fail(DIP_EINVAL, "inst_off must be non-decreasing");
            const uint32_t N = hi - lo;
            if (N > 65535) return fail(DIP_ERANGE, "too many instances");
            nbi[q] = (uint16_t)N;
            M->nbi.push_back(N);
            woff[q] = (uint32_t)wtab.size();
            uint64_t total = 0;
            for (uint32_t u = lo; u < hi; u++) total += d->inst_units[u];
            if (total > mi[i].w_max) return fail(DIP_ERANGE, "a (microbatch, module) work exceeds w_max");
            for (uint32_t Ms = 1; Ms <= mi[i].max_split; Ms++) {
                // part j covers instances [j*q + min(j,rho), (j+1)*q + min(j+1,rho)) (balanced, contiguous)
                const uint32_t qq = Ms ? N / Ms : 0, rho = Ms ? N % Ms : 0;
                for (uint32_t j = 0; j < Ms; j++) {
                    const uint32_t a = j * qq + std::min(j, rho), e = (j + 1) * qq + std::min(j + 1, rho);
                    uint32_t w = 0;
                    for (uint32_t u = a; u < e; u++) w += d->inst_units[lo + u];
                    wtab.push_back((uint16_t)w);
                }
            }
        }

    // ---- compact wrap slots (only segments that can ever own a wrap dependency get one):
    // F slot: rank 0's forward waits on rank P-1 -- segments with k > 0, and the join base
    //         (j = 0, k = 0) of modules with a producer that has instances in this microbatch;
    // B slot: rank P-1's backward waits on rank 0 or on its own forward -- segments with k < K-1,
    //         the join base (j = 0, k = K-1) and, when no consumer has instances here, every
    //         last segment (loss turnaround, R-6).
    std::vector<uint16_t> slotF(n_max, 0xFFFF), slotB(n_max, 0xFFFF);
    uint32_t nslotF = 0, nslotB = 0;
    for (uint32_t b = 0; b < m; b++)
        for (uint32_t i = 0; i < nm; i++) {
            bool prod_any = false, cons_any = false;
            for (uint32_t x = 0; x < nm; x++) {
                if (((mi[i].prod_mask >> x) & 1u) && nbi[b * nm + x]) prod_any = true;
                if (((mi[i].cons_mask >> x) & 1u) && nbi[b * nm + x]) cons_any = true;
            }
            for (uint32_t j = 0; j < mi[i].max_split; j++)
                for (uint32_t k = 0; k < mi[i].K; k++) {
                    const uint32_t id = sbase[b * nm + i] + j * mi[i].K + k;
                    if (k > 0 || (j == 0 && prod_any)) slotF[id] = (uint16_t)nslotF++;
                    if (k + 1 < mi[i].K || j == 0 || !cons_any) slotB[id] = (uint16_t)nslotB++;
                }
        }

    // ---- overflow guards (DIP_ERANGE)
    const uint64_t nodes = (uint64_t)P * 2ull * n_max;
    const unsigned __int128 bound = (unsigned __int128)nodes * ((unsigned __int128)maxlat_layers * maxlat + maxp2p);
    if (bound * P >= ((unsigned __int128)1 << 53)) return fail(DIP_ERANGE, "makespan bound exceeds 2^53 / P");
    if ((unsigned __int128)n_max * maxlat_layers * maxact >= ((unsigned __int128)1 << 32))
        return fail(DIP_ERANGE, "per-rank activation sum may exceed u32 KiB");
    M->mk_bound = (uint64_t)bound;

    // ---- blob (16-B aligned sections)
    std::vector<uint8_t> &blob = M->blob;
    auto put = [&](const void *src, size_t bytes) {
        const uint32_t off = up16((uint32_t)blob.size());
        blob.resize(off + bytes);
        if (bytes) std::memcpy(blob.data() + off, src, bytes);
        return off;
    };
    KParams &kp = M->kp;
    kp.b_modinfo = put(mi.data(), mi.size() * sizeof(ModInfo));
    kp.b_tab = put(tab.data(), tab.size() * 4);
    kp.b_segdec = put(segdec.data(), segdec.size() * 4);
    kp.b_woff = put(woff.data(), woff.size() * 4);
    kp.b_layers = put(layers.data(), layers.size() * 2);
    kp.b_wtab = put(wtab.data(), wtab.size() * 2);
    kp.b_nbi = put(nbi.data(), nbi.size() * 2);
    kp.b_sbase = put(sbase.data(), sbase.size() * 2);
    kp.b_budget = put(d->budget_kib, P * 4);
    kp.b_slotF = put(slotF.data(), slotF.size() * 2);
    kp.b_slotB = put(slotB.data(), slotB.size() * 2);
    kp.nslotF = nslotF;
    kp.nslotB = nslotB;
    blob.resize(up16((uint32_t)blob.size()));
    kp.blob_bytes = (uint32_t)blob.size();

    // host copies of the structure and tables (used by the search, f2)
    for (uint32_t i = 0; i < nm; i++) {
        M->Kv.push_back(mi[i].K);
        M->prod_mask.push_back(mi[i].prod_mask);
        M->cons_mask.push_back(mi[i].cons_mask);
        M->tab_off.push_back(mi[i].tab_off);
        M->lay_off.push_back(mi[i].lay_off);
    }
    M->tab = tab;
    M->layers = layers;
    M->woff = woff;
    M->wtab = wtab;
    M->sbase = sbase;

    // ---- record layout
    M->n_max = n_max;
    M->n_pad = (n_max + 7) & ~7u;
    M->fbw = std::max<uint32_t>(1, (2 * n_max + 31) / 32);
    M->nsplit = nsplit;
    M->off_nib = 4;
    M->off_fwd = up16(4 + (m * nsplit + 1) / 2);
    M->off_bwd = M->off_fwd + 2 * M->n_pad;
    M->off_fb = up16(M->off_bwd + 2 * M->n_pad);
    M->stride = up16(M->off_fb + 4 * M->fbw * P);

    // ---- kernel shape: group of G lanes per candidate, per-group smem working set
    int G = 4;
    while (G < (int)P) G *= 2;
    M->G = G;
    M->cpg = 32 / G;
    uint32_t go = 0;
    auto gput = [&](uint32_t bytes) { const uint32_t o = go; go = up16(go + bytes); return o; };
    // per-candidate working set: per-position rows [2][n_max] uint2 (validation bitmaps alias it),
    // wrap slots [2][n_max] u64 (the decode copy of the sequences aliases it), channel rings
    // [2][P][RING_D] u64, and M / producer / consumer counts per (b, i)
    kp.g_seqF = kp.g_seqB = kp.g_posB = kp.g_depBP = 0;
    kp.g_posF = gput(std::max<uint32_t>(16 * n_max, 8 * ((n_max + 31) / 32)));
    kp.g_depF0 = gput(std::max<uint32_t>(8 * (nslotF + nslotB + 2), 4 * M->n_pad));
    kp.g_ring = gput(2 * P * dipk::RING_D * 8);
    kp.g_bmf = gput(3 * m * nm);
    kp.g_bytes = go;
    // per-rank-order kernel (f1 build / explicit-order timing): per-segment cost rows, priority
    // orders and their inverses, per-segment F / B slots, ranks-done counters, per-rank ready bitmaps
    {
        uint32_t oo = 0;
        auto oput = [&](uint32_t bytes) { const uint32_t o = oo; oo = up16(oo + bytes); return o; };
        const uint32_t nwd = (n_max + 31) / 32;
        kp.o_row = oput(4 * n_max);
        kp.o_seq = oput(2 * 2 * M->n_pad);
        kp.o_posof = oput(2 * 2 * n_max);
        kp.o_sl = oput(2 * 8 * n_max);
        kp.o_bm = oput(2 * 4 * P * nwd);
        kp.o_sum = oput(2 * 4 * P);
        kp.o_mb = oput(3 * m * nm);
        M->o_bytes_build = oo;          // the f1 build needs no ranks-done counters: they come last
        kp.o_h = oput(2 * n_max);
        kp.o_bytes = oo;
    }

    if (cuda_device < 0) {   // host-only model: encoding and validation, no device resources
        *out = guard.release();
        fill_shape(*out);
        return DIP_OK;
    }
    CUDA_TRY(cudaSetDevice(cuda_device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, cuda_device));
    M->num_sms = prop.multiProcessorCount;
    const size_t smem_cap = prop.sharedMemPerBlockOptin;
    const size_t per_warp = (size_t)M->cpg * kp.g_bytes;
    int best_w = 0, best_wpb = 0, best_bps = 0;
    size_t best_smem = 0;
    // up to 24 warps per block: one large block per SM stages the table blob once instead of once per
    // small block, which leaves room for more candidates (A/B on B200, 94B: 18 -> 19 warps/SM,
    // 6.75 -> 7.13 M candidates/s; T2V +6 %; DIP_MAXWPB overrides for A/B runs)
    const int max_wpb = std::getenv("DIP_MAXWPB") ? std::max(1, std::min(24, std::atoi(std::getenv("DIP_MAXWPB")))) : 24;
    for (int wpb = 1; wpb <= max_wpb; wpb++) {
        const size_t sm = kp.blob_bytes + wpb * per_warp;
        if (sm > smem_cap) break;
        CUDA_TRY(dipk::prepare_eval(G, sm));
        int bps = 0;
        CUDA_TRY(dipk::occupancy_eval(G, wpb * 32, sm, &bps));
        if (bps < 1) continue;
        if (wpb * bps >= best_w) { best_w = wpb * bps; best_wpb = wpb; best_bps = bps; best_smem = sm; }
    }
    if (!best_w) return fail(DIP_ERANGE, "per-candidate working set does not fit in shared memory");
    M->wpb = best_wpb;
    M->bps = best_bps;
    M->smem = best_smem;
    M->grid = M->num_sms * best_bps;
    CUDA_TRY(dipk::prepare_eval(G, best_smem));
    if (n_max <= 1024) {   // the per-rank-order kernel's shapes (its ready-set summaries hold 32 words)
        // (up to 24 warps per block, as the scorer; BUILD and TIME have their own per-schedule bytes)
        size_t smax = 0;
        for (int mode = 0; mode < 2; mode++) {
            const size_t per_warp_o = (size_t)M->cpg * (mode ? M->o_bytes_build : kp.o_bytes);
            int bw = 0, bwpb = 0, bbps = 0;
            size_t bsm = 0;
            for (int wpb = 1; wpb <= 24; wpb++) {
                const size_t sm = kp.blob_bytes + wpb * per_warp_o;
                if (sm > smem_cap) break;
                CUDA_TRY(dipk::prepare_order(G, sm));
                int bps = 0;
                CUDA_TRY(dipk::occupancy_order(G, wpb * 32, sm, &bps));
                if (bps < 1) continue;
                if (wpb * bps >= bw) { bw = wpb * bps; bwpb = wpb; bbps = bps; bsm = sm; }
            }
            if (!bw) return fail(DIP_ERANGE, "per-schedule order working set does not fit in shared memory");
            (mode ? M->ob_wpb : M->o_wpb) = bwpb;
            (mode ? M->ob_smem : M->o_smem) = bsm;
            (mode ? M->ob_grid : M->o_grid) = M->num_sms * bbps;
            smax = std::max(smax, bsm);
        }
        CUDA_TRY(dipk::prepare_order(G, smax));
    }

    CUDA_TRY(cudaMalloc(&M->d_blob, kp.blob_bytes));
    CUDA_TRY(cudaMemcpy(M->d_blob, blob.data(), kp.blob_bytes, cudaMemcpyHostToDevice));
    kp.blob = M->d_blob;
    fill_shape(M);
    *out = guard.release();
    return DIP_OK;
}

dip_status dip_model_free(dip_model *m) {
    if (!m) return DIP_OK;
    if (m->d_blob) cudaFree(m->d_blob);
    if (m->d_ctab) cudaFree(m->d_ctab);
    if (m->d_crow) cudaFree(m->d_crow);
    if (m->d_srank) cudaFree(m->d_srank);
    delete m;
    return DIP_OK;
}

dip_status dip_model_get_info(const dip_model *m, dip_model_info *o) {
    if (!m || !o) return fail(DIP_EINVAL, "null argument");
    o->P = m->P; o->n_modules = m->nmod; o->m = m->m; o->n_max = m->n_max; o->fbw = m->fbw;
    o->record_stride = m->stride; o->group_lanes = (uint32_t)m->G; o->smem_per_block = (uint32_t)m->smem;
    o->warps_per_block = (uint32_t)m->wpb; o->blocks_per_sm = (uint32_t)m->bps; o->grid = (uint32_t)m->grid;
    o->makespan_bound = m->mk_bound;
    return DIP_OK;
}

// ---------------------------------------------------------------- encode (host) --------
static void encode_range(const dip_model *M, const dip_candidate_batch *c, size_t lo, size_t hi, uint8_t *out) {
    const uint32_t P = M->P, nm = M->nmod, m = M->m, n_max = M->n_max, fbw = M->fbw;
    for (size_t x = lo; x < hi; x++) {
        uint8_t *rec = out + x * M->stride;
        std::memset(rec, 0, M->stride);
        const uint32_t n = c->n[x];
        uint16_t flags = 0;
        if (n > n_max || n > 65535) flags |= 1;
        const uint16_t nh = (uint16_t)std::min<uint32_t>(n, 65535);
        std::memcpy(rec, &nh, 2);
        const uint8_t *sp = c->split + x * (size_t)m * nm;
        for (uint32_t b = 0; b < m; b++)
            for (uint32_t i = 0; i < nm; i++) {
                const uint32_t v = sp[b * nm + i];
                if (M->max_split[i] > 1) {
                    if (v > 15) flags |= 1;
                    const uint32_t nib = b * M->nsplit + M->nib_slot[i];
                    rec[M->off_nib + nib / 2] |= (uint8_t)((v & 15u) << ((nib & 1) * 4));
                } else if (v != (M->nbi[b * nm + i] > 0 ? 1u : 0u)) {
                    flags |= 1;   // unrepresentable: the implied value is the only valid one
                }
            }
        std::memcpy(rec + 2, &flags, 2);
        uint16_t *fw = reinterpret_cast<uint16_t *>(rec + M->off_fwd);
        uint16_t *bw = reinterpret_cast<uint16_t *>(rec + M->off_bwd);
        std::memcpy(fw, c->fwd_seq + x * (size_t)n_max, 2 * n_max);
        std::memcpy(bw, c->bwd_seq + x * (size_t)n_max, 2 * n_max);
        for (uint32_t p = n_max; p < M->n_pad; p++) { fw[p] = 0xFFFF; bw[p] = 0xFFFF; }
        uint32_t *fb = reinterpret_cast<uint32_t *>(rec + M->off_fb);
        const uint32_t *src = c->fb_bits + x * (size_t)P * fbw;
        for (uint32_t r = 0; r < P; r++)
            for (uint32_t w = 0; w < fbw; w++) fb[w * P + r] = src[r * fbw + w];
    }
}

dip_status dip_encode_candidates(const dip_model *M, const dip_candidate_batch *c, size_t count, void *out,
                                 int threads) {
    if (!M || !c || (!out && count)) return fail(DIP_EINVAL, "null argument");
    if (!count) return DIP_OK;
    if (!c->split || !c->n || !c->fwd_seq || !c->bwd_seq || !c->fb_bits) return fail(DIP_EINVAL, "null array");
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<size_t>(threads, std::max<size_t>(1, count / 256));
    std::vector<std::thread> th;
    const size_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        const size_t lo = per * t, hi = std::min(count, lo + per);
        if (lo >= hi) break;
        th.emplace_back(encode_range, M, c, lo, hi, static_cast<uint8_t *>(out));
    }
    for (auto &t : th) t.join();
    return DIP_OK;
}

// ---------------------------------------------------------------- workspace ------------
dip_status dip_workspace_create(const dip_model *M, size_t host_chunk, dip_workspace **out) {
    if (!M || !out) return fail(DIP_EINVAL, "null argument");
    if (M->device < 0 || !M->d_blob) return fail(DIP_EINVAL, "host-only model (cuda_device < 0)");
    CUDA_TRY(cudaSetDevice(M->device));
    dip_workspace *w = new (std::nothrow) dip_workspace();
    if (!w) return fail(DIP_ENOMEM, "host allocation");
    struct Guard {   // on any failure below, release what was allocated so far
        dip_workspace *w;
        ~Guard() { if (w) dip_workspace_free(w); }
        dip_workspace *release() { dip_workspace *x = w; w = nullptr; return x; }
    } guard{w};
    w->model = M;
    CUDA_TRY(cudaMalloc(&w->d_misc, 16 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemset(w->d_misc, 0, 16 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMallocHost(&w->h_misc, 16 * sizeof(unsigned long long)));
    const size_t slots = (size_t)M->grid * M->wpb * M->cpg;
    w->spill_bytes = slots * 2ull * M->P * M->n_max * sizeof(unsigned long long);
    CUDA_TRY(cudaMalloc(&w->d_spill, w->spill_bytes));
    w->host_chunk = host_chunk;
    if (host_chunk) {
        for (int b = 0; b < dip_workspace::NBUF; b++) {
            CUDA_TRY(cudaMalloc(&w->d_rec[b], host_chunk * M->stride));
            CUDA_TRY(cudaEventCreateWithFlags(&w->ev_copied[b], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&w->ev_free[b], cudaEventDisableTiming));
        }
        CUDA_TRY(cudaMalloc(&w->d_res, dip_workspace::NBUF * host_chunk * sizeof(dip_result)));
        CUDA_TRY(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&w->comp2, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&w->ev_start, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming));
        CUDA_TRY(cudaMalloc(&w->d_spill2, w->spill_bytes));
    }
    *out = guard.release();
    return DIP_OK;
}

dip_status dip_workspace_free(dip_workspace *w) {
    if (!w) return DIP_OK;
    if (w->d_misc) cudaFree(w->d_misc);
    if (w->h_misc) cudaFreeHost(w->h_misc);
    if (w->d_spill) cudaFree(w->d_spill);
    for (int b = 0; b < dip_workspace::NBUF; b++) {
        if (w->d_rec[b]) cudaFree(w->d_rec[b]);
        if (w->ev_copied[b]) cudaEventDestroy(w->ev_copied[b]);
        if (w->ev_free[b]) cudaEventDestroy(w->ev_free[b]);
    }
    if (w->d_res) cudaFree(w->d_res);
    if (w->copy_stream) cudaStreamDestroy(w->copy_stream);
    if (w->comp2) cudaStreamDestroy(w->comp2);
    if (w->ev_start) cudaEventDestroy(w->ev_start);
    if (w->ev_join) cudaEventDestroy(w->ev_join);
    if (w->d_spill2) cudaFree(w->d_spill2);
    for (int b = 0; b < dip_workspace::NBUF; b++)
        if (w->d_view[b]) cudaFree(w->d_view[b]);
    delete w;
    return DIP_OK;
}

// ---------------------------------------------------------------- eval -----------------
static const bool g_scorer_segment = std::getenv("DIP_SCORER") && std::string(std::getenv("DIP_SCORER")) == "segment";
static dip_status launch_orders(const dip_model *M, dip_workspace *w, const void *d_records, size_t count, int om,
                                const uint16_t *orders_in, uint16_t *orders_out, const uint8_t *sel,
                                dip_result *d_results, uint32_t *d_peaks, uint64_t *d_start, uint64_t *d_end,
                                cudaStream_t s);
extern "C++" {
dip_status diph::launch_chunk(const dip_model *M, dip_workspace *w, const void *d_records, size_t count,
                               uint64_t index_base, uint32_t idx_bits, bool fused, dip_result *d_results,
                               uint32_t *d_peaks, cudaStream_t s, uint8_t *records_out, const uint8_t *sel,
                               unsigned long long *spill, unsigned long long *counter) {
    KParams kp = M->kp;
    kp.records = static_cast<const uint8_t *>(d_records);
    kp.records_out = records_out;
    kp.sel = sel;
    kp.tl_start = nullptr;
    kp.tl_end = nullptr;
    kp.count = count;
    kp.index_base = index_base;
    kp.results = d_results;
    kp.peaks = d_peaks;
    kp.counter = counter ? counter : w->d_misc + 0;
    kp.best_key = w->d_misc + 1;
    kp.spill = spill ? spill : w->d_spill;
    kp.fused_key = fused ? 1u : 0u;
    kp.idx_bits = idx_bits;
    CUDA_TRY(cudaMemsetAsync(kp.counter, 0, sizeof(unsigned long long), s));
    const int grid = (int)std::min<uint64_t>((uint64_t)M->grid,
                                             std::max<uint64_t>(1, (count + M->cpg * M->wpb - 1) / (M->cpg * M->wpb)));
    CUDA_TRY(dipk::launch_eval(kp, M->G, grid, M->wpb * 32, M->smem, s));
    g_launches++;
    return DIP_OK;
}

bool diph::fused_ok(const dip_model *M, uint32_t idx_bits) {
    return idx_bits < 63 && (M->mk_bound >> (64 - idx_bits)) == 0;
}
}  // extern "C++"

dip_status dip_eval_schedules(const dip_model *M, dip_workspace *w, const void *d_records, size_t count,
                              dip_result *d_results, uint32_t *d_peaks, void *stream) {
    if (!M || !w || w->model != M) return fail(DIP_EINVAL, "model / workspace mismatch");
    if (count && (!d_records || !d_results)) return fail(DIP_EINVAL, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t idx_bits = bits_for(std::max<uint64_t>(count, 2));
    const bool fused = fused_ok(M, idx_bits);
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 1, 0xFF, sizeof(unsigned long long), s));
    w->last_results = d_results;
    w->last_count = count;
    w->last_idx_bits = idx_bits;
    w->last_fused = fused;
    if (!count) return DIP_OK;
    if (g_scorer_segment)   // A/B: the per-segment-state kernel on the record's own orders
        return launch_orders(M, w, d_records, count, 2, nullptr, nullptr, nullptr, d_results, d_peaks, nullptr,
                             nullptr, s);
    return launch_chunk(M, w, d_records, count, 0, idx_bits, fused, d_results, d_peaks, s);
}

// the per-rank-order kernel: BUILD (f1) or TIME (explicit orders, optional f3 selection / timelines)
static dip_status launch_orders(const dip_model *M, dip_workspace *w, const void *d_records, size_t count,
                                int om, const uint16_t *orders_in, uint16_t *orders_out, const uint8_t *sel,
                                dip_result *d_results, uint32_t *d_peaks, uint64_t *d_start, uint64_t *d_end,
                                cudaStream_t s) {
    const uint32_t idx_bits = bits_for(std::max<uint64_t>(count, 2));
    const bool fused = fused_ok(M, idx_bits);
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 1, 0xFF, sizeof(unsigned long long), s));
    w->last_results = d_results;
    w->last_count = count;
    w->last_idx_bits = idx_bits;
    w->last_fused = fused;
    if (!count) return DIP_OK;
    KParams kp = M->kp;
    kp.records = static_cast<const uint8_t *>(d_records);
    kp.records_out = nullptr;
    kp.orders_out = orders_out;
    kp.orders_in = orders_in;
    kp.sel = sel;
    kp.tl_start = d_start;
    kp.tl_end = d_end;
    kp.count = count;
    kp.index_base = 0;
    kp.results = d_results;
    kp.peaks = d_peaks;
    kp.counter = w->d_misc + 0;
    kp.best_key = w->d_misc + 1;
    kp.spill = nullptr;
    kp.fused_key = fused ? 1u : 0u;
    kp.idx_bits = idx_bits;
    CUDA_TRY(cudaMemsetAsync(kp.counter, 0, sizeof(unsigned long long), s));
    if (d_start) {
        CUDA_TRY(cudaMemsetAsync(d_start, 0, count * M->P * 2ull * M->n_max * 8, s));
        CUDA_TRY(cudaMemsetAsync(d_end, 0, count * M->P * 2ull * M->n_max * 8, s));
    }
    if (M->n_max > 1024) return fail(DIP_ERANGE, "per-rank-order kernel: n_max > 1024 (32 ready-set words)");
    const bool build = om == 1;
    if (build) kp.o_bytes = M->o_bytes_build;
    const int owpb = build ? M->ob_wpb : M->o_wpb, ogrid = build ? M->ob_grid : M->o_grid;
    const int grid = (int)std::min<uint64_t>((uint64_t)ogrid,
                                             std::max<uint64_t>(1, (count + M->cpg * owpb - 1) / (M->cpg * owpb)));
    CUDA_TRY(dipk::launch_order(kp, M->G, om, grid, owpb * 32, build ? M->ob_smem : M->o_smem, s));
    g_launches++;
    return DIP_OK;
}

dip_status dip_interleave(const dip_model *M, dip_workspace *w, const void *d_records, size_t count,
                          dip_result *d_results, uint32_t *d_peaks, uint16_t *d_orders, void *stream) {
    if (!M || !w || w->model != M) return fail(DIP_EINVAL, "model / workspace mismatch");
    if (count && (!d_records || !d_results)) return fail(DIP_EINVAL, "null buffer");
    if (M->device < 0 || !M->d_blob) return fail(DIP_EINVAL, "host-only model (cuda_device < 0)");
    return launch_orders(M, w, d_records, count, 1, nullptr, d_orders, nullptr, d_results, d_peaks, nullptr,
                         nullptr, static_cast<cudaStream_t>(stream));
}

dip_status dip_eval_orders(const dip_model *M, dip_workspace *w, const void *d_records, const uint16_t *d_orders,
                           size_t count, const uint8_t *d_sel, dip_result *d_results, uint32_t *d_peaks,
                           uint64_t *d_start, uint64_t *d_end, void *stream) {
    if (!M || !w || w->model != M) return fail(DIP_EINVAL, "model / workspace mismatch");
    if (count && (!d_records || !d_orders || !d_results)) return fail(DIP_EINVAL, "null buffer");
    if (!d_start != !d_end) return fail(DIP_EINVAL, "d_start and d_end go together");
    if (d_sel && !M->S) return fail(DIP_EINVAL, "a selection needs a strategy menu (dip_set_strategies)");
    if (M->device < 0 || !M->d_blob) return fail(DIP_EINVAL, "host-only model (cuda_device < 0)");
    return launch_orders(M, w, d_records, count, 0, d_orders, nullptr, d_sel, d_results, d_peaks, d_start, d_end,
                         static_cast<cudaStream_t>(stream));
}

dip_status dip_timeline(const dip_model *M, dip_workspace *w, const void *d_records, size_t count, dip_result *d_results,
                        uint64_t *d_start, uint64_t *d_end, void *stream) {
    if (!M || !w || w->model != M) return fail(DIP_EINVAL, "model / workspace mismatch");
    if (count && (!d_records || !d_results || !d_start || !d_end)) return fail(DIP_EINVAL, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 1, 0xFF, sizeof(unsigned long long), s));
    w->last_results = d_results;
    w->last_count = count;
    w->last_idx_bits = bits_for(std::max<uint64_t>(count, 2));
    w->last_fused = fused_ok(M, w->last_idx_bits);
    if (!count) return DIP_OK;
    KParams kp = M->kp;
    kp.records = static_cast<const uint8_t *>(d_records);
    kp.records_out = nullptr;
    kp.sel = nullptr;
    kp.tl_start = d_start;
    kp.tl_end = d_end;
    kp.count = count;
    kp.index_base = 0;
    kp.results = d_results;
    kp.peaks = nullptr;
    kp.counter = w->d_misc + 0;
    kp.best_key = w->d_misc + 1;
    kp.spill = w->d_spill;
    kp.fused_key = w->last_fused ? 1u : 0u;
    kp.idx_bits = w->last_idx_bits;
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 0, 0, sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(d_start, 0, count * M->P * 2ull * M->n_max * 8, s));
    CUDA_TRY(cudaMemsetAsync(d_end, 0, count * M->P * 2ull * M->n_max * 8, s));
    const int grid = (int)std::min<uint64_t>((uint64_t)M->grid,
                                             std::max<uint64_t>(1, (count + M->cpg * M->wpb - 1) / (M->cpg * M->wpb)));
    CUDA_TRY(dipk::launch_eval(kp, M->G, grid, M->wpb * 32, M->smem, s));
    g_launches++;
    return DIP_OK;
}

// local winner -> (makespan, local index) on the host; exact two-pass scan when not fused
static dip_status local_best(const dip_model *M, dip_workspace *w, cudaStream_t s, uint64_t *mk, uint64_t *idx,
                             bool *found) {
    if (w->last_fused) {
        CUDA_TRY(cudaMemcpyAsync(w->h_misc, w->d_misc + 1, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        const unsigned long long k = w->h_misc[0];
        *found = k != ~0ull;
        *mk = *found ? k >> w->last_idx_bits : ~0ull;
        *idx = *found ? k & ((1ull << w->last_idx_bits) - 1) : ~0ull;
        return DIP_OK;
    }
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 3, 0xFF, 16, s));
    if (w->last_count) {
        CUDA_TRY(dipk::launch_scan_argmin(w->last_results, w->last_count, 0, w->d_misc + 3, nullptr, s));
        CUDA_TRY(dipk::launch_scan_argmin_idx(w->last_results, w->last_count, 0, w->d_misc + 3, w->d_misc + 4, s));
        g_launches += 2;
    }
    CUDA_TRY(cudaMemcpyAsync(w->h_misc, w->d_misc + 3, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *found = w->h_misc[0] != ~0ull;
    *mk = w->h_misc[0];
    *idx = w->h_misc[1];
    return DIP_OK;
}

dip_status dip_argmin(const dip_model *M, dip_workspace *w, size_t count, uint64_t shard_stride, uint32_t rank,
                      uint32_t world, dip_comm *comm, dip_winner *out, void *stream) {
    if (!M || !w || !out) return fail(DIP_EINVAL, "null argument");
    if (world < 1 || rank >= world || (world > 1 && !comm)) return fail(DIP_EINVAL, "bad rank/world/comm");
    if (count != w->last_count) return fail(DIP_EINVAL, "count differs from the last eval on this workspace");
    if (shard_stride < count) return fail(DIP_EINVAL, "shard_stride < count");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::memset(out, 0, sizeof(*out));
    if (world == 1) {
        uint64_t mk, idx;
        bool found;
        dip_status st = local_best(M, w, s, &mk, &idx, &found);
        if (st != DIP_OK) return st;
        out->found = found;
        out->rank = 0;
        out->global_index = found ? idx : ~0ull;
        out->makespan_ns = mk;
        return DIP_OK;
    }
    const uint32_t ibits = bits_for(std::max<uint64_t>(shard_stride, 2)), rbits = bits_for(std::max<uint32_t>(world, 2));
    const bool packed = w->last_fused && ibits + rbits < 63 && (M->mk_bound >> (64 - ibits - rbits)) == 0;
    if (packed) {
        // one allreduce of the packed (makespan, rank, local index) key
        CUDA_TRY(dipk::launch_make_gkey(w->d_misc + 1, w->d_misc + 2, w->last_idx_bits, ibits, rbits, rank, s));
        g_launches++;
        NCCL_TRY(ncclAllReduce(w->d_misc + 2, w->d_misc + 2, 1, ncclUint64, ncclMin, comm->comm, s));
        CUDA_TRY(cudaMemcpyAsync(w->h_misc, w->d_misc + 2, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return dip_unpack_key(w->h_misc[0], shard_stride, world, out);
    }
    // exact fallback: min makespan, then min global index among ties (two allreduces)
    uint64_t mk, idx;
    bool found;
    dip_status st = local_best(M, w, s, &mk, &idx, &found);
    if (st != DIP_OK) return st;
    w->h_misc[2] = found ? mk : ~0ull;
    CUDA_TRY(cudaMemcpyAsync(w->d_misc + 5, w->h_misc + 2, 8, cudaMemcpyHostToDevice, s));
    NCCL_TRY(ncclAllReduce(w->d_misc + 5, w->d_misc + 5, 1, ncclUint64, ncclMin, comm->comm, s));
    CUDA_TRY(cudaMemcpyAsync(w->h_misc + 3, w->d_misc + 5, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const uint64_t gmk = w->h_misc[3];
    w->h_misc[4] = (found && mk == gmk) ? (uint64_t)rank * shard_stride + idx : ~0ull;
    CUDA_TRY(cudaMemcpyAsync(w->d_misc + 6, w->h_misc + 4, 8, cudaMemcpyHostToDevice, s));
    NCCL_TRY(ncclAllReduce(w->d_misc + 6, w->d_misc + 6, 1, ncclUint64, ncclMin, comm->comm, s));
    CUDA_TRY(cudaMemcpyAsync(w->h_misc + 5, w->d_misc + 6, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    out->found = gmk != ~0ull;
    out->makespan_ns = gmk;
    out->global_index = w->h_misc[5];
    out->rank = out->found ? (int32_t)(w->h_misc[5] / shard_stride) : -1;
    return DIP_OK;
}

// Cross-rank key layout: makespan << (rbits + ibits) | rank << ibits | local index,
// ibits = bits(shard_stride), rbits = bits(world). Under contiguous shards the u64 order of keys is
// the (makespan, global index) order (R-15). The device kernel make_gkey builds the same layout.
dip_status dip_pack_key(uint64_t makespan_ns, uint32_t rank, uint64_t local, uint64_t shard_stride, uint32_t world,
                        uint64_t *key_out) {
    if (!key_out || world < 1 || rank >= world || local >= shard_stride) return fail(DIP_EINVAL, "bad argument");
    const uint32_t ibits = bits_for(std::max<uint64_t>(shard_stride, 2)), rbits = bits_for(std::max<uint32_t>(world, 2));
    if (ibits + rbits >= 63 || (makespan_ns >> (64 - ibits - rbits)) != 0)
        return fail(DIP_ERANGE, "makespan does not fit the packed key");
    *key_out = (makespan_ns << (rbits + ibits)) | ((uint64_t)rank << ibits) | local;
    return DIP_OK;
}

dip_status dip_unpack_key(uint64_t key, uint64_t shard_stride, uint32_t world, dip_winner *out) {
    if (!out || world < 1) return fail(DIP_EINVAL, "bad argument");
    const uint32_t ibits = bits_for(std::max<uint64_t>(shard_stride, 2)), rbits = bits_for(std::max<uint32_t>(world, 2));
    out->found = key != ~0ull;
    if (out->found) {
        const uint64_t local = key & ((1ull << ibits) - 1);
        out->rank = (int32_t)((key >> ibits) & ((1ull << rbits) - 1));
        out->makespan_ns = key >> (ibits + rbits);
        out->global_index = (uint64_t)out->rank * shard_stride + local;
    } else {
        out->rank = -1;
        out->makespan_ns = ~0ull;
        out->global_index = ~0ull;
    }
    return DIP_OK;
}

dip_status dip_eval_host(const dip_model *M, dip_workspace *w, const void *h_records, size_t count,
                         dip_result *h_results, uint64_t shard_stride, uint32_t rank, uint32_t world, dip_comm *comm,
                         dip_winner *out, void *stream) {
    if (!M || !w || w->model != M || !out) return fail(DIP_EINVAL, "null argument");
    if (!w->host_chunk) return fail(DIP_EINVAL, "workspace has no host staging (host_chunk = 0)");
    if (count && !h_records) return fail(DIP_EINVAL, "null records");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t idx_bits = bits_for(std::max<uint64_t>(count, 2));
    const bool fused = fused_ok(M, idx_bits);
    if (!fused) return fail(DIP_ERANGE, "host path needs the fused argmin key (makespan bound too large)");
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 1, 0xFF, sizeof(unsigned long long), s));
    // at least ~8 chunks when the batch allows it, so that the first copy (not overlapped) is short
    const size_t C = std::min<size_t>(w->host_chunk, std::max<size_t>(8192, (count + 7) / 8));
    const size_t nch = (count + C - 1) / C;
    CUDA_TRY(cudaEventRecord(w->ev_start, s));              // comp2 starts after the key reset
    CUDA_TRY(cudaStreamWaitEvent(w->comp2, w->ev_start, 0));
    // the copies too: work the caller queued on `s` before this call (e.g. an asynchronous fill of
    // the pinned h_records) must complete before the first chunk is read
    CUDA_TRY(cudaStreamWaitEvent(w->copy_stream, w->ev_start, 0));
    for (size_t c = 0; c < nch; c++) {
        const int b = (int)(c % dip_workspace::NBUF);
        const bool odd = (c & 1) != 0;
        cudaStream_t sc = odd ? w->comp2 : s;
        const size_t lo = c * C, cnt = std::min(C, count - lo);
        if (c >= (size_t)dip_workspace::NBUF) CUDA_TRY(cudaStreamWaitEvent(w->copy_stream, w->ev_free[b], 0));
        CUDA_TRY(cudaMemcpyAsync(w->d_rec[b], static_cast<const uint8_t *>(h_records) + lo * M->stride,
                                 cnt * M->stride, cudaMemcpyHostToDevice, w->copy_stream));
        CUDA_TRY(cudaEventRecord(w->ev_copied[b], w->copy_stream));
        CUDA_TRY(cudaStreamWaitEvent(sc, w->ev_copied[b], 0));
        dip_result *dres = w->d_res + b * C;
        dip_status st = launch_chunk(M, w, w->d_rec[b], cnt, lo, idx_bits, true, dres, nullptr, sc, nullptr, nullptr,
                                     odd ? w->d_spill2 : w->d_spill, w->d_misc + (odd ? 8 : 0));
        if (st != DIP_OK) return st;
        if (h_results) CUDA_TRY(cudaMemcpyAsync(h_results + lo, dres, cnt * sizeof(dip_result), cudaMemcpyDeviceToHost, sc));
        CUDA_TRY(cudaEventRecord(w->ev_free[b], sc));
    }
    CUDA_TRY(cudaEventRecord(w->ev_join, w->comp2));        // the argmin sees both streams' chunks
    CUDA_TRY(cudaStreamWaitEvent(s, w->ev_join, 0));
    w->last_results = nullptr;
    w->last_count = count;
    w->last_idx_bits = idx_bits;
    w->last_fused = true;
    return dip_argmin(M, w, count, shard_stride, rank, world, comm, out, stream);
}

// ---------------------------------------------------------------- device-mode encoding --
static dipk::EncParams enc_params(const dip_model *M) {
    dipk::EncParams p{};
    p.P = M->P; p.nm = M->nmod; p.m = M->m; p.n_max = M->n_max; p.n_pad = M->n_pad; p.fbw = M->fbw;
    p.stride = M->stride; p.off_nib = M->off_nib; p.off_fwd = M->off_fwd; p.off_bwd = M->off_bwd;
    p.off_fb = M->off_fb; p.nsplit = M->nsplit;
    for (uint32_t i = 0; i < M->nmod && i < 8; i++) {
        if (M->max_split[i] > 1) p.maxsplit_gt1 |= 1u << i;
        p.nib_slot[i] = M->nib_slot[i];
    }
    p.nbi = reinterpret_cast<const uint16_t *>(M->d_blob + M->kp.b_nbi);
    return p;
}

dip_status dip_encode_candidates_device(const dip_model *M, const dip_candidate_batch *d, size_t count, void *d_out,
                                        void *stream) {
    if (!M || !d || (!d_out && count)) return fail(DIP_EINVAL, "null argument");
    if (M->device < 0 || !M->d_blob) return fail(DIP_EINVAL, "host-only model (cuda_device < 0)");
    if (!count) return DIP_OK;
    if (!d->split || !d->n || !d->fwd_seq || !d->bwd_seq || !d->fb_bits) return fail(DIP_EINVAL, "null array");
    dipk::EncParams p = enc_params(M);
    p.split = d->split; p.n = d->n; p.fwd = d->fwd_seq; p.bwd = d->bwd_seq; p.fb = d->fb_bits;
    p.out = static_cast<uint8_t *>(d_out);
    p.count = count;
    CUDA_TRY(dipk::launch_encode(p, M->num_sms, static_cast<cudaStream_t>(stream)));
    g_launches++;
    return DIP_OK;
}

// end to end from the HOST VIEW: per chunk, H2D of the candidates' arrays, the device encoder, the
// scorer, the results D2H; copies of chunk c+1 overlap the encode + score of chunk c
dip_status dip_eval_host_view(const dip_model *M, dip_workspace *w, const dip_candidate_batch *h, size_t count,
                              dip_result *h_results, uint64_t shard_stride, uint32_t rank, uint32_t world,
                              dip_comm *comm, dip_winner *out, void *stream) {
    if (!M || !w || w->model != M || !out || (count && !h)) return fail(DIP_EINVAL, "null argument");
    if (!w->host_chunk) return fail(DIP_EINVAL, "workspace has no host staging (host_chunk = 0)");
    if (count && (!h->split || !h->n || !h->fwd_seq || !h->bwd_seq || !h->fb_bits)) return fail(DIP_EINVAL, "null array");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t idx_bits = bits_for(std::max<uint64_t>(count, 2));
    if (!fused_ok(M, idx_bits)) return fail(DIP_ERANGE, "host path needs the fused argmin key (makespan bound too large)");
    const size_t nq = (size_t)M->m * M->nmod, C = w->host_chunk;
    // staging layout of one chunk: split [C][nq] | n [C] | fwd [C][n_max] | bwd [C][n_max] | fb [C][P][fbw]
    auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const size_t o_n = up(C * nq), o_f = o_n + up(C * 4), o_b = o_f + up(C * 2 * M->n_max),
                 o_fb = o_b + up(C * 2 * M->n_max), bytes = o_fb + up(C * 4ull * M->P * M->fbw);
    for (int b = 0; b < dip_workspace::NBUF; b++)
        if (!w->d_view[b]) CUDA_TRY(cudaMalloc(&w->d_view[b], bytes));
    CUDA_TRY(cudaMemsetAsync(w->d_misc + 1, 0xFF, sizeof(unsigned long long), s));
    const size_t Cc = std::min<size_t>(C, std::max<size_t>(8192, (count + 7) / 8));
    const size_t nch = (count + Cc - 1) / Cc;
    CUDA_TRY(cudaEventRecord(w->ev_start, s));
    CUDA_TRY(cudaStreamWaitEvent(w->comp2, w->ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(w->copy_stream, w->ev_start, 0));
    dipk::EncParams ep = enc_params(M);
    for (size_t c = 0; c < nch; c++) {
        const int b = (int)(c % dip_workspace::NBUF);
        const bool odd = (c & 1) != 0;
        cudaStream_t sc = odd ? w->comp2 : s;
        const size_t lo = c * Cc, cnt = std::min(Cc, count - lo);
        uint8_t *v = w->d_view[b];
        if (c >= (size_t)dip_workspace::NBUF) CUDA_TRY(cudaStreamWaitEvent(w->copy_stream, w->ev_free[b], 0));
        cudaStream_t cs = w->copy_stream;
        CUDA_TRY(cudaMemcpyAsync(v, h->split + lo * nq, cnt * nq, cudaMemcpyHostToDevice, cs));
        CUDA_TRY(cudaMemcpyAsync(v + o_n, h->n + lo, cnt * 4, cudaMemcpyHostToDevice, cs));
        CUDA_TRY(cudaMemcpyAsync(v + o_f, h->fwd_seq + lo * M->n_max, cnt * 2 * M->n_max, cudaMemcpyHostToDevice, cs));
        CUDA_TRY(cudaMemcpyAsync(v + o_b, h->bwd_seq + lo * M->n_max, cnt * 2 * M->n_max, cudaMemcpyHostToDevice, cs));
        CUDA_TRY(cudaMemcpyAsync(v + o_fb, h->fb_bits + lo * (size_t)M->P * M->fbw, cnt * 4ull * M->P * M->fbw,
                                 cudaMemcpyHostToDevice, cs));
        CUDA_TRY(cudaEventRecord(w->ev_copied[b], cs));
        CUDA_TRY(cudaStreamWaitEvent(sc, w->ev_copied[b], 0));
        ep.split = v;
        ep.n = reinterpret_cast<const uint32_t *>(v + o_n);
        ep.fwd = reinterpret_cast<const uint16_t *>(v + o_f);
        ep.bwd = reinterpret_cast<const uint16_t *>(v + o_b);
        ep.fb = reinterpret_cast<const uint32_t *>(v + o_fb);
        ep.out = w->d_rec[b];
        ep.count = cnt;
        CUDA_TRY(dipk::launch_encode(ep, M->num_sms, sc));
        g_launches++;
        dip_result *dres = w->d_res + b * C;
        dip_status st = launch_chunk(M, w, w->d_rec[b], cnt, lo, idx_bits, true, dres, nullptr, sc, nullptr, nullptr,
                                     odd ? w->d_spill2 : w->d_spill, w->d_misc + (odd ? 8 : 0));
        if (st != DIP_OK) return st;
        if (h_results) CUDA_TRY(cudaMemcpyAsync(h_results + lo, dres, cnt * sizeof(dip_result), cudaMemcpyDeviceToHost, sc));
        CUDA_TRY(cudaEventRecord(w->ev_free[b], sc));
    }
    CUDA_TRY(cudaEventRecord(w->ev_join, w->comp2));
    CUDA_TRY(cudaStreamWaitEvent(s, w->ev_join, 0));
    w->last_results = nullptr;
    w->last_count = count;
    w->last_idx_bits = idx_bits;
    w->last_fused = true;
    return dip_argmin(M, w, count, shard_stride, rank, world, comm, out, stream);
}

// ---------------------------------------------------------------- NCCL -----------------
dip_status dip_comm_unique_id(uint8_t id_out[128]) {
    if (!id_out) return fail(DIP_EINVAL, "null argument");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id_out, &id, 128);
    return DIP_OK;
}

dip_status dip_comm_init(const uint8_t id[128], int rank, int world, int cuda_device, dip_comm **out) {
    if (!id || !out || world < 1 || rank < 0 || rank >= world) return fail(DIP_EINVAL, "bad argument");
    CUDA_TRY(cudaSetDevice(cuda_device));
    dip_comm *c = new (std::nothrow) dip_comm();
    if (!c) return fail(DIP_ENOMEM, "host allocation");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(DIP_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->rank = rank;
    c->world = world;
    *out = c;
    return DIP_OK;
}

dip_status dip_comm_free(dip_comm *c) {
    if (!c) return DIP_OK;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
    return DIP_OK;
}

}  // extern "C"
