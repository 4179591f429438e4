// dip_internal.h -- layout contract between the host side (dip_host.cpp) and the
// sm_100a kernels (dip_kernels.cu). Not part of the public ABI (include/dip.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dip.h"

namespace dipk {

#ifndef DIP_RING_D
#define DIP_RING_D 2
#endif
constexpr int RING_D = DIP_RING_D;     // depth of the smem inter-rank channels (exact spill beyond; power of 2)
constexpr uint64_t PEND_SHIFT = 56;    // wrap-dependency slot: pending count in bits 56..63
constexpr uint64_t VAL_MASK = (1ull << PEND_SHIFT) - 1;

// per-module constants staged in shared memory (32 B)
struct ModInfo {
    uint32_t K, max_split, prod_mask, cons_mask;
    uint32_t tab_off, lay_off, nib_slot, w_max;
};

// segdec[id] bit fields: b [0,8) i [8,11) j [11,15) k [15,23) K-1 [23,31)
__host__ __device__ inline uint32_t segdec_pack(uint32_t b, uint32_t i, uint32_t j, uint32_t k, uint32_t K) {
    return b | (i << 8) | (j << 11) | (k << 15) | ((K - 1) << 23);
}

struct KParams {
    // problem shape
    uint32_t P, nmod, m, n_max, n_pad, fbw, stride;
    uint32_t off_nib, off_fwd, off_bwd, off_fb, nsplit;   // record layout
    // static tables, one contiguous 16-B aligned blob staged to smem by a TMA bulk copy
    const uint8_t *blob;
    uint32_t blob_bytes;   // multiple of 16
    uint32_t b_modinfo, b_segdec, b_layers, b_tab, b_woff, b_wtab, b_nbi, b_sbase, b_budget, b_slotF, b_slotB;
    uint32_t nslotF, nslotB;   // compact wrap-slot counts: depAll = [F slots | B slots | ZERO | SINK]
    // per-candidate shared-memory working set (byte offsets inside a group area)
    uint32_t g_seqF, g_seqB, g_posF, g_posB, g_depF0, g_depBP, g_ring, g_bmf, g_bytes;
    uint32_t warps_per_block, cpg;
    // per-schedule working set of the per-rank-order kernel (dip_order.cu), byte offsets in a group area
    uint32_t o_row, o_seq, o_posof, o_sl, o_h, o_bm, o_sum, o_mb, o_bytes;
    // per launch
    const uint8_t *records;
    uint8_t *records_out;       // non-null: interleave mode (f1) writes the F/B bit rows here
    uint64_t *tl_start, *tl_end;  // non-null: timeline mode, [count][P][2*n_max] per-slot start / end
    const uint8_t *sel;         // non-null: f3 mode, [count][P][2][n_max] selected candidate per stage pair
    uint16_t *orders_out;       // order kernel, BUILD: [count][P][2 n_max] per-rank orders out (or null)
    const uint16_t *orders_in;  // order kernel, TIME: [count][P][2 n_max] per-rank orders in
    const uint4 *ctab;          // f3 candidates {F ns, B ns, act KiB, count} per (type, W, c)
    const int32_t *crow;        // f3: per chunk row, ctab base of its (module, layers) type - tab_off * S
    const uint16_t *srank;      // f3: per ctab entry c, the rank of the step c -> c+1 by saving per KiB
    uint32_t S;                 // f3: candidates per (type, W)
    uint32_t gap_pm, node_cap;  // f3: the per-rank ILP's optimality gap (per mille) and B&B child budget
    unsigned long long *mo_stats;   // f3: [5] solved, certified at the root, searched, capped, B&B children
    uint64_t count, index_base;
    dip_result *results;
    uint32_t *peaks;
    unsigned long long *best_key;
    unsigned long long *counter;
    unsigned long long *spill;   // per group slot: 2 * P * n_max u64
    uint32_t fused_key, idx_bits;
};

// f3 candidate generation: one thread per (type, W); a type = (module i, layers per chunk l)
struct MCandParams {
    uint32_t n_items, n_types, n_strat, S, T;
    const uint32_t *t_item, *t_lay, *t_toff, *t_base;   // [n_types]: first item, l, tab_off[i], ctab base
    const uint32_t *mf, *mb, *ma;                       // menu [n_strat][T]
    uint4 *ctab;                                        // out: [sum (w_max_i + 1)] x S
};

// device-mode encoding (dip_encode.cu): host-view arrays already on the device -> records
struct EncParams {
    const uint8_t *split;
    const uint32_t *n;
    const uint16_t *fwd, *bwd;
    const uint32_t *fb;
    const uint16_t *nbi;       // [m*nm] instances per (b, i) (the blob's copy)
    uint8_t *out;
    uint64_t count;
    uint32_t P, nm, m, n_max, n_pad, fbw, stride, off_nib, off_fwd, off_bwd, off_fb, nsplit, maxsplit_gt1;
    uint32_t nib_slot[8];
};
cudaError_t launch_encode(const EncParams &p, int num_sms, cudaStream_t s);

cudaError_t launch_eval(const KParams &kp, int G, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t launch_mcand(const MCandParams &p, cudaStream_t s);
cudaError_t prepare_memopt(size_t smem);
cudaError_t occupancy_memopt(size_t smem, int *blocks_per_sm);
cudaError_t launch_memopt(const KParams &kp, uint8_t *sel, uint32_t warp_bytes, int grid, cudaStream_t s);
cudaError_t prepare_eval(int G, size_t smem);
cudaError_t prepare_order(int G, size_t smem);
cudaError_t occupancy_order(int G, int block, size_t smem, int *blocks_per_sm);
cudaError_t launch_order(const KParams &kp, int G, int om, int grid, int block, size_t smem, cudaStream_t s);
cudaError_t occupancy_eval(int G, int block, size_t smem, int *blocks_per_sm);
cudaError_t launch_scan_argmin(const dip_result *res, uint64_t count, uint64_t index_base,
                               unsigned long long *mk_out, unsigned long long *idx_out, cudaStream_t s);
cudaError_t launch_scan_argmin_idx(const dip_result *res, uint64_t count, uint64_t index_base,
                                   const unsigned long long *mk_in, unsigned long long *idx_out, cudaStream_t s);
cudaError_t launch_make_gkey(const unsigned long long *key, unsigned long long *gkey, uint32_t idx_bits,
                             uint32_t ibits, uint32_t rbits, uint32_t rank, cudaStream_t s);

}  // namespace dipk
