/* dip.h -- C-ABI of the B200-native DIP candidate-schedule scorer.
 *
 * The hot path of DIP (arXiv 2504.14145): for ONE input batch, score a large
 * batch of candidate pipeline schedules and return the best feasible one.
 *   - PAPER.md §3.2: per iteration the planner fetches batch
 *     metadata, builds modality-specific sub-microbatches and searches for the
 *     schedule with the best score;
 *   - P:498-499: every rollout "undergoes pipeline stage interleaving ... to
 *     compute performance scores (i.e., end-to-end iteration time)";
 *   - P:546-548: memory capacity M per rank must not be exceeded;
 *   - P:702-705: the simulator "populates operator timestamps in topological
 *     order, then determines tensor lifetimes ... peak memory usage".
 * A candidate = a sub-microbatch split M_{b,i} per (microbatch b, module i)
 * + a shared forward and a shared backward segment sequence + a
 * per-rank forward/backward interleaving (reading R-1 of DESIGN.md).
 *
 * Beyond the scorer, the planner's other steps: dip_interleave (§5.2 dual-queue
 * interleaving; emits per-rank orders) and dip_eval_orders (schedules given as per-rank orders),
 * dip_search (§5.1 MCTS with batched GPU rollouts, and the random / depth-first variants of the
 * paper's comparison), dip_set_strategies / dip_strategy_candidates / dip_memopt /
 * dip_set_memopt_solver / dip_memopt_stats (§5.3 per-layer memory optimisation, the per-rank ILP
 * to a 5 % gap), dip_timeline / dip_compile_plan / dip_validate_plan (§6.3 execution plans).
 * End to end: dip_encode_candidates_device and dip_eval_host_view (from the host view),
 * dip_eval_host (from host records). dip_ubench_int measures the integer-pipe roofline peak.
 *
 * Units: time in integer nanoseconds (u64 accumulators), memory in KiB (u32).
 * All calls return dip_status (0 = DIP_OK); no C++ exception crosses the ABI.
 * Per-candidate problems are DATA (dip_result.status), never call errors.
 * Streams are passed as `void *` holding a cudaStream_t (NULL = legacy default).
 */
#ifndef DIP_H
#define DIP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DIP_OK = 0,
    DIP_EINVAL = 1,       /* bad argument or malformed problem description */
    DIP_ECUDA = 2,        /* CUDA runtime error (detail: dip_last_error()) */
    DIP_ENOMEM = 3,       /* device or host allocation failed */
    DIP_ERANGE = 4,       /* a load-time overflow guard failed (u32 activations, 2^53 bubble bound) */
    DIP_ENCCL = 5,        /* NCCL error */
    DIP_ENOFEASIBLE = 6   /* reserved */
} dip_status;

/* Per-candidate status, precedence BAD_ENCODING > DEADLOCK > OOM > OK (R-13). */
typedef enum {
    DIP_CAND_OK = 0,
    DIP_CAND_OOM = 1,           /* timed; some rank's peak > its budget (strict >, R-10) */
    DIP_CAND_DEADLOCK = 2,      /* the stage x slot dependency graph has a cycle (R-12) */
    DIP_CAND_BAD_ENCODING = 3   /* malformed candidate (R-11) */
} dip_cand_status;

/* One modality module. Tables are per LAYER, indexed by the work W of a
 * sub-microbatch (W = sum of its instances' work units, R-21), W in [0, w_max]. */
typedef struct {
    uint32_t L;               /* layers */
    uint32_t K;               /* pipeline segments; the module has P*K chunks */
    uint32_t max_split;       /* M_max in [1, 15]: candidates choose M in [1, min(N, M_max)] (R-2) */
    uint32_t w_max;           /* tables have w_max + 1 entries */
    uint32_t producer_mask;   /* bit p: module p (p < this module's index) feeds this one (R-5) */
    const uint32_t *chunk_layers; /* NULL (default: P*K chunks of consecutive layers, remainder to
                                     the earliest, R-3) or [P*K] explicit layers per chunk */
    const uint32_t *f_ns;     /* [w_max+1] forward ns per layer */
    const uint32_t *b_ns;     /* [w_max+1] backward ns per layer */
    const uint32_t *act_kib;  /* [w_max+1] activation KiB per layer, held from F start to B end (R-9) */
    const uint32_t *p2p_ns;   /* [w_max+1] boundary transfer ns on cross-rank edges (R-7); NULL = 0 */
} dip_module_desc;

/* Problem = model partition + per-layer cost tables + batch metadata. */
typedef struct {
    uint32_t P;               /* pipeline ranks, 1..32 */
    uint32_t n_modules;       /* 1..8, in topological order (producers first) */
    uint32_t m;               /* microbatches, 1..255 */
    const dip_module_desc *modules;
    const uint32_t *inst_off; /* [m*n_modules+1] b-major offsets into inst_units: (b,i) owns
                                 instances [inst_off[b*n+i], inst_off[b*n+i+1]) in packing order */
    const uint16_t *inst_units; /* per-instance work units */
    const uint32_t *budget_kib; /* [P] activation budget per rank (capacity - static), KiB */
} dip_problem_desc;

typedef struct dip_model dip_model;           /* opaque, library-owned, immutable after load */
typedef struct dip_workspace dip_workspace;   /* opaque per-stream scratch (work queue, argmin key, spill) */
typedef struct dip_comm dip_comm;             /* opaque NCCL communicator */

typedef struct {
    uint32_t P, n_modules, m;
    uint32_t n_max;           /* segment-id space: id(b,i,j,k) = base(b,i) + j*K_i + k (b-major) */
    uint32_t fbw;             /* 32-bit words per rank of F/B bits: ceil(2*n_max/32) */
    uint32_t record_stride;   /* bytes per packed candidate record (multiple of 16) */
    uint32_t group_lanes;     /* lanes per candidate in the kernel (power of two >= P) */
    uint32_t smem_per_block;  /* dynamic shared memory of the scoring kernel */
    uint32_t warps_per_block, blocks_per_sm, grid;
    uint64_t makespan_bound;  /* load-time upper bound on any makespan (overflow guards) */
} dip_model_info;

/* cuda_device < 0 gives a host-only model (encoding, validation, dip_model_get_info).
 * Validate the problem, derive the segment-decode table, layers per chunk, the
 * balanced-split work table (R-2) and copy them to `cuda_device`.
 * The descriptor is read only during the call. Errors: DIP_EINVAL (P not in
 * 1..32, P*K > L without chunk_layers, producer_mask not topological, M_max > 15,
 * ...), DIP_ERANGE (a (b,i) total work exceeds w_max, or an overflow guard),
 * DIP_ECUDA, DIP_ENOMEM. */
dip_status dip_load_cost_model(const dip_problem_desc *d, int cuda_device, dip_model **out);
dip_status dip_model_free(dip_model *m);
dip_status dip_model_get_info(const dip_model *m, dip_model_info *out);

/* Host view of `count` candidates (struct of arrays, row-major):
 *   split   u8  [count][m*n_modules]  M_{b,i}
 *   n       u32 [count]               number of forward segments
 *   fwd_seq u16 [count][n_max]        segment ids in forward order, pad 0xFFFF
 *   bwd_seq u16 [count][n_max]        segment ids in backward order, pad 0xFFFF
 *   fb_bits u32 [count][P][fbw]       rank r, slot t: bit t%32 of word t/32; 1 = next backward
 * Rank r's slot t runs the next unread fwd_seq entry (bit 0) or bwd_seq entry (bit 1). */
typedef struct {
    const uint8_t *split;
    const uint32_t *n;
    const uint16_t *fwd_seq, *bwd_seq;
    const uint32_t *fb_bits;
} dip_candidate_batch;

/* Pack candidates into records of info.record_stride bytes (HOST memory, e.g. pinned),
 * the layout dip_eval_schedules reads:
 *   off 0   u16 n, u16 flags (bit 0: encoding unrepresentable -> BAD_ENCODING)
 *   off 4   u8  nibbles: M_{b,i} for the modules with M_max > 1, b-major
 *   off A   u16 fwd[n_pad], then u16 bwd[n_pad]   (n_pad = n_max rounded up to 8; pad 0xFFFF)
 *   off C   u32 fb[fbw][P]   (word-major: the P lanes of a candidate read one 4P-byte row)
 * Unrepresentable inputs (n > n_max, split > 15, ...) set flag bit 0 so that the
 * kernel reports BAD_ENCODING exactly like the oracle. threads <= 0: all cores. */
dip_status dip_encode_candidates(const dip_model *m, const dip_candidate_batch *c, size_t count,
                                 void *out_records, int threads);

/* SURVEY §8(b)'s device mode of dip_encode_candidates: the batch's five arrays are DEVICE pointers
 * (same layouts as above); the records are written to device memory d_out (count * record_stride
 * bytes) by a GPU kernel (the F/B rows' rank-major -> word-major transpose runs on the GPU),
 * byte-identical to the host encoder. Asynchronous on `stream`. */
dip_status dip_encode_candidates_device(const dip_model *m, const dip_candidate_batch *d_batch, size_t count,
                                        void *d_out, void *stream);

/* 24-byte result per candidate. BAD_ENCODING/DEADLOCK: makespan = UINT64_MAX,
 * bubble = -1.0. bubble = (P*makespan - sum of busy ns) / (P*makespan) as one IEEE
 * double division of exact integers (R-16); 0.0 when P*makespan = 0. */
typedef struct {
    uint64_t makespan_ns;
    uint32_t status;          /* dip_cand_status */
    uint32_t oom_mask;        /* bit r: peak_r > budget_r */
    double bubble;
} dip_result;

/* Per-stream scratch: work-queue counter, fused argmin key, spill area for the
 * DP's inter-rank channels, and (if host_chunk > 0) the dip_eval_host pipeline:
 * three device staging buffers of host_chunk records, a copy stream, a second
 * compute stream with its own spill area (chunks alternate between the caller's
 * stream and it, so one chunk's tail overlaps the next chunk's start). */
dip_status dip_workspace_create(const dip_model *m, size_t host_chunk, dip_workspace **out);
dip_status dip_workspace_free(dip_workspace *w);

/* Score `count` device-resident records (d_records, count*stride bytes) on `stream`:
 * decode + cost lookup + longest-path DP + memory peaks + bubble, and the fused
 * argmin epilogue into the workspace key. Asynchronous. d_results: [count] device;
 * d_peaks_kib: [count][P] device or NULL. Candidate i's index is i (local). */
dip_status dip_eval_schedules(const dip_model *m, dip_workspace *w, const void *d_records, size_t count,
                              dip_result *d_results, uint32_t *d_peaks_kib, void *stream);

/* dip_eval_schedules plus every stage's simulated start / end time: d_start / d_end are device
 * [count][P][2*n_max] u64, entry (c, r, t) = rank r's slot t of candidate c (zero beyond 2n and for
 * candidates that are not timed). For Gantt charts and the plan compiler (f4). Asynchronous. */
dip_status dip_timeline(const dip_model *m, dip_workspace *w, const void *d_records, size_t count,
                        dip_result *d_results, uint64_t *d_start, uint64_t *d_end, void *stream);

/* DIP's greedy dual-queue stage interleaving (§5.2):
 * for every record, take its split and its forward / backward segment orders as the PRIORITY
 * orders of the per-rank queues (position 0 = highest; its F/B bit rows are ignored) and build each
 * rank's stage order with the paper's iterative scheduling (R-29..R-31): a stage is
 * ready once its predecessors are placed, t_fw / t_bw = the minimum t_start over a queue's ready
 * stages, the rank with the smallest t_min places one stage -- 1F1B alternation when both are
 * below t_last, else the queue of the smaller t_start (ties to the backward) -- namely that queue's
 * highest-priority stage among those starting as early as possible; a forward stage whose
 * activation would exceed the rank's budget is disabled, and if every rank is blocked
 * by that alone the gate is lifted for one step (OOM). Scores the built schedule (d_results,
 * d_peaks_kib as dip_eval_schedules; never DEADLOCK) and updates the fused argmin key
 * (dip_argmin works after it). d_orders: device [count][P][2*n_max] u16 out, or NULL: rank r's
 * t-th stage = segment id | 0x8000 for a backward stage, 0xFFFF beyond 2n (all 0xFFFF for
 * BAD_ENCODING records). The records are not modified. Asynchronous on `stream`. */
dip_status dip_interleave(const dip_model *m, dip_workspace *w, const void *d_records, size_t count,
                          dip_result *d_results, uint32_t *d_peaks_kib, uint16_t *d_orders, void *stream);

/* Score schedules given as explicit per-rank orders (the format dip_interleave emits) instead of
 * the records' shared sequences + F/B bits: the longest path over the stage DAG with
 * the records' splits, O1-O10 semantics (BAD_ENCODING unless every rank's order holds each present
 * segment once as F and once as B, 0xFFFF padding; DEADLOCK iff the orders close a cycle).
 * d_sel (or NULL): a dip_memopt selection [count][P][2][n_max] whose candidates replace the tables'
 * latencies and activations (f3's re-timing). d_start / d_end (both or neither): device
 * [count][P][2*n_max] u64 per-slot start / end times (f4). Asynchronous on `stream`. */
dip_status dip_eval_orders(const dip_model *m, dip_workspace *w, const void *d_records, const uint16_t *d_orders,
                           size_t count, const uint8_t *d_sel, dip_result *d_results, uint32_t *d_peaks_kib,
                           uint64_t *d_start, uint64_t *d_end, void *stream);

/* DIP's per-layer memory optimisation (§5.3).
 *
 * dip_set_strategies: the per-layer strategy menu (R-37). f_ns / b_ns /
 * act_kib are host arrays [n_strat][T], T = sum over modules of (w_max_i + 1), entry (c, tab_off_i + W)
 * = strategy c's per-layer F ns, B ns and activation KiB of module i at width W (the same column
 * order as the cost tables of dip_load_cost_model). Strategy 0 must be the tables' own scheme (the
 * most memory-efficient one); this is the caller's contract. For every stage-pair type
 * (module, layers per chunk) and width the GPU builds <= S candidates (R-38: fastest,
 * smallest, fastest of each of S-2 memory buckets; Pareto, memory ascending). 1 <= n_strat <= 8,
 * 2 <= S <= 16. DIP_ERANGE if a pair total exceeds u32, the enumeration exceeds 2^20 count
 * vectors per pair, the menu yields two candidates of equal memory or latency, or a rank's budget
 * plus n_max x the largest candidate memory reaches 2^31 KiB (the selection works in int32), or the
 * candidate table exceeds 65535 rows of S entries. Replaces a
 * previous menu. Synchronous. Device model only. */
dip_status dip_set_strategies(dip_model *m, uint32_t n_strat, const uint32_t *f_ns, const uint32_t *b_ns,
                              const uint32_t *act_kib, uint32_t S);

/* The candidates of the stage pair (module, layers per chunk, width W) after dip_set_strategies:
 * out [S][3] host (F ns, B ns, memory KiB), memory ascending; *count receives their number.
 * DIP_EINVAL if no such pair type exists. */
dip_status dip_strategy_candidates(const dip_model *m, uint32_t module, uint32_t layers, uint32_t W,
                                   uint64_t *out, uint32_t *count);

/* Per-rank strategy selection and re-timing of `count` device records (R-39, R-40):
 * for every (record, rank) the per-rank ILP of P:572-582 (minimise the summed pair latency subject
 * to the rank's budget at every forward slot) is solved to the relative optimality gap set by
 * dip_set_memopt_solver (default 5 %): the pairs start at candidate 0, the greedy warm
 * start moves the pair with the largest latency saving per KiB up while every forward slot
 * it covers stays within the budget; a Lagrangian bound (R-39) certifies it, else a
 * depth-first branch and bound improves it (at most node_cap children per rank). Then the schedules
 * are scored with the selected latencies and activations (results / peaks / fused argmin key as
 * dip_eval_schedules). d_orders: NULL (the records' shared sequences + F/B bits define each rank's
 * order) or device [count][P][2*n_max] explicit per-rank orders as dip_interleave emits them (then
 * the re-timing is dip_eval_orders with the selection). d_sel: device
 * [count][P][2][n_max] u8 out -- sel[c][r][0][p] = candidate of the pair whose forward is the
 * p-th forward stage, sel[c][r][1][q] = the same for the q-th backward stage (zero beyond n;
 * unspecified for BAD_ENCODING records). Two launches on `stream`, asynchronous. */
dip_status dip_memopt(const dip_model *m, dip_workspace *w, const void *d_records, const uint16_t *d_orders,
                      size_t count, uint8_t *d_sel, dip_result *d_results, uint32_t *d_peaks_kib, void *stream);

/* The per-rank ILP solver's settings for dip_memopt: relative optimality gap in per mille
 * (default 50 = the paper's 5 %, 0 = exact) and the branch-and-bound child budget per (record, rank)
 * (default 4096; when it is reached the incumbent stands and dip_memopt_stats counts it).
 * DIP_EINVAL if gap_permille > 1000 or node_cap == 0. */
dip_status dip_set_memopt_solver(dip_model *m, uint32_t gap_permille, uint32_t node_cap);

/* Counters of the last dip_memopt on `w`, out[5] host: (record, rank) instances solved, certified
 * at the root (the warm start within the gap), searched by branch and bound, stopped by node_cap,
 * and the branch-and-bound children visited in total. Synchronous on `stream`. */
dip_status dip_memopt_stats(const dip_workspace *w, uint64_t *out, void *stream);

/* DIP's MCTS segment reordering (§5.1) with batched
 * GPU rollouts. For the given split, classes = (direction, microbatch, module, chunk k) with M > 0
 * (one priority per modality, microbatch and chunk; its M sub-microbatch segments keep a fixed
 * order, R-32); a sequence of classes
 * gives priorities (position p -> Cn-1-p) -> forward / backward priority orders -> f1
 * interleaving -> score LB / makespan (0 if not OK; LB = busiest rank's total latency). Each
 * round selects `leaves` leaves by UCB s^alpha + beta*sqrt(ln N_parent / N_child) with
 * virtual visits, expands one child each (next class in order), scores `rollouts` random
 * completions per leaf in one dip_interleave launch (then dip_memopt on the built orders if
 * memopt is set) and backpropagates the best trial
 * (s = max, N + 1). Deterministic for a seed (rollout u draws from splitmix64(seed, u)).
 * Allocates its rollout buffers for the duration of the call. Synchronous. */
typedef struct {
    uint64_t seed;
    uint32_t rounds;          /* search rounds */
    uint32_t leaves;          /* leaves expanded per round (one batched GPU launch) */
    uint32_t rollouts;        /* random completions per leaf ("e.g., 10 trials") */
    int32_t threads;          /* host threads building rollout records (<= 0: all cores) */
    double alpha, beta;       /* UCB hyper-parameters */
    int32_t memopt;           /* nonzero: score each rollout after dip_memopt (f3); needs
                                 dip_set_strategies; the score's LB stays the base-table bound */
    int32_t policy;           /* 0 = MCTS; the paper's comparison variants: 1 = random
                                 exploration (every rollout a uniformly random sequence from the root),
                                 2 = depth-first search (pre-order over the sequence tree, children
                                 in class order); rollouts / scoring / backpropagation unchanged */
    double time_budget_ms;    /* > 0: stop after the first round that ends past this wall time
                                 ("until a predefined time budget is exhausted"); the rounds
                                 done are reported; 0 = run all `rounds` */
} dip_search_params;

typedef struct {
    int32_t found;            /* a feasible (status OK) schedule was found */
    uint32_t rounds_done;
    uint64_t makespan_ns;     /* of the best schedule */
    double score;             /* LB / makespan of the best schedule */
    uint64_t rollouts_scored;
    uint64_t tree_nodes;
} dip_search_result;

/* best_record_out: host buffer of record_stride bytes receiving the best rollout's record (split and
 * priority orders; its F/B bit rows are not meaningful), or NULL; best_orders_out: host
 * [P][2*n_max] u16 receiving the best rollout's per-rank orders as dip_interleave emits them, or
 * NULL; trace: [rounds] best score after each round, or NULL. */
dip_status dip_search(const dip_model *m, dip_workspace *w, const uint8_t *split /* [m*n_modules] */,
                      const dip_search_params *p, void *best_record_out, uint16_t *best_orders_out,
                      double *trace, dip_search_result *out, void *stream);

typedef struct {
    int32_t found;            /* 0 if no candidate has status OK on any rank */
    int32_t rank;             /* owning rank */
    uint64_t global_index;    /* rank * shard_stride + local index (contiguous shards) */
    uint64_t makespan_ns;
} dip_winner;

/* Lowest (makespan, global index) among status-OK candidates of the last
 * dip_eval_schedules/dip_eval_host on `w` (R-15), reduced over `world` ranks with
 * one ncclAllReduce(MIN) of a packed (makespan, rank, index) u64 key on `stream`
 * (comm may be NULL when world == 1). Synchronous: returns after the host has the
 * winner. shard_stride = candidates per rank shard (>= count). */
dip_status dip_argmin(const dip_model *m, dip_workspace *w, size_t count, uint64_t shard_stride,
                      uint32_t rank, uint32_t world, dip_comm *comm, dip_winner *out, void *stream);

/* Host helpers of the cross-rank key (also what dip_argmin uses): key = makespan << (rbits+ibits)
 * | rank << ibits | local, ibits = ceil(log2(shard_stride)), rbits = ceil(log2(world)) (both >= 1).
 * The unsigned order of keys is the (makespan, global index) order under contiguous shards (R-15).
 * dip_pack_key returns DIP_ERANGE if the makespan does not fit; UINT64_MAX unpacks to found = 0. */
dip_status dip_pack_key(uint64_t makespan_ns, uint32_t rank, uint64_t local, uint64_t shard_stride, uint32_t world,
                        uint64_t *key_out);
dip_status dip_unpack_key(uint64_t key, uint64_t shard_stride, uint32_t world, dip_winner *out);

/* End to end from HOST records (pinned for overlap): chunked H2D copies overlapped
 * with scoring (chunks of min(host_chunk, max(8192, count/8)) records), then dip_argmin. h_results ([count], host) may be NULL. Requires a
 * workspace created with host_chunk > 0. Synchronous. */
/* End to end from the candidates' HOST VIEW (the dip_candidate_batch arrays in host memory; pinned
 * for full copy speed): per chunk of the workspace's host_chunk, H2D of the chunk's arrays, the
 * device encoder (dip_encode_candidates_device), dip_eval_schedules, the D2H of its results (if
 * h_results != NULL), copies overlapped with encode + scoring; then dip_argmin as dip_eval_host.
 * Synchronous. The device staging for the host view is allocated on first use. */
dip_status dip_eval_host_view(const dip_model *m, dip_workspace *w, const dip_candidate_batch *h_batch, size_t count,
                              dip_result *h_results, uint64_t shard_stride, uint32_t rank, uint32_t world,
                              dip_comm *comm, dip_winner *out, void *stream);

dip_status dip_eval_host(const dip_model *m, dip_workspace *w, const void *h_records, size_t count,
                         dip_result *h_results, uint64_t shard_stride, uint32_t rank, uint32_t world,
                         dip_comm *comm, dip_winner *out, void *stream);

/* compile one scored schedule into per-rank action lists (§6.3,
 * P:717-734): fw_stage / bw_stage per stage; for every cross-rank dependency edge an asynchronous
 * isend right after the producing stage, wait_isend before the producer's next stage, irecv right
 * after the consumer's last stage that ends no later than the producer starts (so every receive is
 * posted before its send in simulated time) and wait_irecv right before the consuming stage;
 * consecutive isend / irecv actions share a batch id ("grouped into a batched operation").
 * record: one host record (as encoded); orders: NULL (the record's shared sequences + F/B bits give
 * each rank's order) or the schedule's host per-rank orders [P][2*n_max] as dip_interleave emits
 * them; start / end: its host timeline rows ([P][2*n_max], from dip_timeline or dip_eval_orders).
 * DIP_EINVAL for a malformed record / orders (a segment missing or repeated on a rank). actions: capacity entries, rank r's list is
 * actions[rank_off[r] .. rank_off[r+1]). DIP_ERANGE if capacity is too small (rank_off[P] = size). */
enum { DIP_ACT_FW_STAGE = 0, DIP_ACT_BW_STAGE = 1, DIP_ACT_ISEND = 2, DIP_ACT_IRECV = 3,
       DIP_ACT_WAIT_ISEND = 4, DIP_ACT_WAIT_IRECV = 5 };
typedef struct {
    uint32_t kind;            /* DIP_ACT_* */
    uint32_t peer;            /* P2P: the other rank; stages: own rank */
    uint32_t tag;             /* P2P: message tag (dense, in compile order); stages: segment id */
    uint32_t batch;           /* P2P: batch id (consecutive P2P actions share one); stages: 0 */
    uint32_t slot;            /* the stage slot the action belongs to */
} dip_action;
dip_status dip_compile_plan(const dip_model *m, const void *record, const uint16_t *orders,
                            const uint64_t *start, const uint64_t *end, dip_action *actions, size_t capacity,
                            uint32_t *rank_off /* [P+1] */, uint32_t *n_messages);
/* Discrete-event execution of a plan (P2P priced as on the schedule's edges): *ok = 1 iff every
 * isend / irecv tag is perfectly paired and the plan terminates; stage_start ([P][2*n_max], or
 * NULL) receives each stage's start time, which equals the source timeline for compiled plans. */
dip_status dip_validate_plan(const dip_model *m, const void *record, const uint16_t *orders, const dip_action *actions,
                             const uint32_t *rank_off, uint64_t *stage_start, int32_t *ok);

/* Integer-pipe microbenchmark (the scorer's ALU roofline denominator, measured on this device):
 * kind 0 IADD3, 1 VIMNMX (min / max), 2 ISETP + SEL, 3 SHFL.BFLY + add, 4 64-bit add (IADD3 +
 * IADD3.X), 5 IMAD; *ops_per_s = thread-level SASS instructions per second over the whole GPU
 * (8 independent chains per thread, every SM full), *ms = the best of 5 launches (or NULL).
 * Synchronous. */
dip_status dip_ubench_int(uint32_t kind, int cuda_device, double *ops_per_s, double *ms);

/* NCCL communicator for the argmin: rank 0 calls dip_comm_unique_id, broadcasts
 * the 128 bytes (e.g. over torch.distributed), every rank calls dip_comm_init. */
dip_status dip_comm_unique_id(uint8_t id_out[128]);
dip_status dip_comm_init(const uint8_t id[128], int rank, int world, int cuda_device, dip_comm **out);
dip_status dip_comm_free(dip_comm *c);

/* Number of kernel launches issued by this process so far (the scorer's own kernels). */
uint64_t dip_launch_count(void);
const char *dip_status_str(dip_status s);
const char *dip_last_error(void);   /* thread-local detail of the last failing call */

#ifdef __cplusplus
}
#endif
#endif /* DIP_H */
