// dip_host_internal.h -- host-side internals shared by the C-ABI translation units
// (dip_host.cpp, dip_search.cpp). Not part of the public ABI (include/dip.h).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "dip.h"
#include "dip_internal.h"

namespace diph {

extern thread_local std::string g_err;
extern std::atomic<uint64_t> g_launches;

inline dip_status fail(dip_status s, const std::string &msg) {
    g_err = msg;
    return s;
}
#define CUDA_TRY(x)                                                                            \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess) return diph::fail(DIP_ECUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
    } while (0)
#define NCCL_TRY(x)                                                                            \
    do {                                                                                       \
        ncclResult_t _r = (x);                                                                 \
        if (_r != ncclSuccess) return diph::fail(DIP_ENCCL, std::string(#x) + ": " + ncclGetErrorString(_r)); \
    } while (0)

inline uint32_t up16(uint32_t x) { return (x + 15u) & ~15u; }
inline uint32_t bits_for(uint64_t n) {   // smallest b >= 1 with n <= 2^b
    uint32_t b = 1;
    while (b < 63 && (1ull << b) < n) b++;
    return b;
}

}  // namespace diph

struct dip_model {
    int device = 0;
    uint32_t P = 0, nmod = 0, m = 0, n_max = 0, n_pad = 0, fbw = 0, stride = 0;
    uint32_t off_nib = 0, off_fwd = 0, off_bwd = 0, off_fb = 0, nsplit = 0;
    std::vector<uint32_t> max_split, nib_slot, nbi;   // host copies for encode
    // host copies of the structure and tables (for the search, f2)
    std::vector<uint32_t> Kv, prod_mask, cons_mask, tab_off, lay_off, woff;
    std::vector<uint32_t> tab;        // 4 x u32 per (module, W): F, B, act, p2p
    std::vector<uint16_t> layers, wtab, sbase;
    std::vector<uint8_t> blob;
    uint8_t *d_blob = nullptr;
    dipk::KParams kp{};            // shape + blob + layout; per-launch fields filled per call
    int G = 32, cpg = 1, wpb = 1, bps = 1, grid = 1, num_sms = 148;
    size_t smem = 0;
    int o_wpb = 1, o_grid = 1;         // per-rank-order kernel (dip_order.cu) shape: TIME modes
    size_t o_smem = 0;
    int ob_wpb = 1, ob_grid = 1;       // ... and the f1 BUILD mode (no ranks-done counters)
    size_t ob_smem = 0;
    uint32_t o_bytes_build = 0;
    uint64_t mk_bound = 0;
    // f3 (per-layer memory optimisation): strategy menu -> candidate table
    uint32_t n_strat = 0, S = 0;
    std::vector<uint32_t> t_mod, t_lay, t_base;   // candidate types (module, layers per chunk)
    std::vector<uint4> h_ctab;                    // host copy of the candidate table
    uint4 *d_ctab = nullptr;
    int32_t *d_crow = nullptr;
    uint16_t *d_srank = nullptr;
    uint32_t mo_warp_bytes = 0;
    int mo_grid = 0;
};

struct dip_workspace {
    const dip_model *model = nullptr;
    unsigned long long *d_misc = nullptr;   // [0] counter [1] key [2] gkey [3] mk [4] idx [5] f3 counter / fallback [6] fallback [8] comp2 counter
    unsigned long long *h_misc = nullptr;   // pinned
    unsigned long long *d_spill = nullptr;
    size_t spill_bytes = 0;
    // last eval
    const dip_result *last_results = nullptr;
    uint64_t last_count = 0;
    uint32_t last_idx_bits = 1;
    bool last_fused = true;
    // host path
    size_t host_chunk = 0;
    // host path: 3 staging buffers, copies on copy_stream, chunks alternating between the caller's
    // stream and comp2 (each with its own spill area and work counter) so that one chunk's tail
    // overlaps the next chunk's start
    static constexpr int NBUF = 3;
    uint8_t *d_rec[NBUF] = {nullptr, nullptr, nullptr};
    dip_result *d_res = nullptr;           // NBUF * host_chunk results
    cudaStream_t copy_stream = nullptr, comp2 = nullptr;
    cudaEvent_t ev_copied[NBUF] = {nullptr, nullptr, nullptr}, ev_free[NBUF] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev_start = nullptr, ev_join = nullptr;
    unsigned long long *d_spill2 = nullptr;
    // host-view path (dip_eval_host_view): NBUF device staging areas for the candidates' host-view
    // arrays of one chunk (split | n | fwd | bwd | fb), allocated on first use
    uint8_t *d_view[NBUF] = {nullptr, nullptr, nullptr};
};

struct dip_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};

namespace diph {
dip_status launch_chunk(const dip_model *M, dip_workspace *w, const void *d_records, size_t count,
                        uint64_t index_base, uint32_t idx_bits, bool fused, dip_result *d_results,
                        uint32_t *d_peaks, cudaStream_t s, uint8_t *records_out = nullptr,
                        const uint8_t *sel = nullptr, unsigned long long *spill = nullptr,
                        unsigned long long *counter = nullptr);
bool fused_ok(const dip_model *M, uint32_t idx_bits);
}  // namespace diph
