/*
 * dfsim_b200.h -- C-ABI of the B200-native batched strategy simulator.
 *
 * The reference (arXiv 2002.06790's `dfsim`, pure Python) has no FFI; its
 * drop-in surface is the Python API re-exported from pkg/src/dfsim/__init__.py:6-43.
 * Each entry point below replaces one reference function, batched over many
 * candidate strategies (see INTEGRATION.md for the ctypes binding a dfsim
 * maintainer would add):
 *
 *   dfsim_expand_dp          strategy.py:170-282  expand_data_parallel (+ graph.py:122-135 CSR);
 *                                                also the parameter-server expansion (ps.py, new)
 *   dfsim_topo_order         graph.py:424-443     topological order (any valid order, device)
 *   dfsim_topological_order  graph.py:424-443     topological_order (the reference's order, host)
 *   dfsim_predict_batch      costmodel.py:158-165 predict
 *   dfsim_comm_batch         costmodel.py:168-223 comm_time_us / transfer_time / allreduce_time
 *   dfsim_estimate_batch     costmodel.py:282-376 estimate_all (predict 158-165, comm 168-223)
 *   dfsim_simulate_batch     engine.py:96-146     simulate (+ _finalize 69-93)
 *   dfsim_critical_path_batch graph.py:446-485    critical_path on finish-start (reporting.py:128)
 *   dfsim_argmin             (no reference function: cmd_simulate's per-config makespans,
 *                            cli.py:133-148, reduced to the first minimum)
 *   dfsim_summarize          reporting.py:117-162 summarize (op shares, busy folds, overlap)
 *   dfsim_trace_write        reporting.py:43-74   to_trace (host-side writer, byte-identical)
 *
 * Conventions
 *  - Every pointer in a *view* struct or argument is a DEVICE pointer owned by
 *    the caller, unless the name ends in _host.  The library never frees caller
 *    memory.  Node index == rank of the node-id string in code-point order;
 *    device index == rank of the device-id string.
 *  - Calls are asynchronous on the context's stream unless documented otherwise.
 *    Per-simulation outcomes (cycle, unknown op) are written to caller arrays;
 *    the return value reports argument/launch problems.
 *  - Threads: a context is not re-entrant.  Calls on one context must be
 *    serialised by the caller (the Python binding holds a per-context lock
 *    across dfsim_ctx_set_stream + the call); distinct contexts are independent.
 *    Device scratch inside a context is kept per stream (internally locked), so
 *    serialised callers on different streams never share a scratch buffer.
 *  - Status codes map 1:1 onto the reference exceptions (errors.py:6-92):
 */
#ifndef DFSIM_B200_H
#define DFSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFSIM_OK 0
#define DFSIM_CYCLE 1            /* CycleError: some node never placed */
#define DFSIM_MISSING_DURATION 2 /* MissingDurationError */
#define DFSIM_UNKNOWN_OP 3       /* UnknownOpError: estimation chain exhausted */
#define DFSIM_CONFIG 4           /* ConfigError */
#define DFSIM_CUDA 5             /* device / launch failure */
#define DFSIM_BAD_ARGUMENT 6     /* ValueError-class argument problems */
#define DFSIM_NEGATIVE_DURATION 7 /* DurationEntry(<0 or NaN) -> ValueError */
#define DFSIM_CHECK_FAILED 8      /* checked build only (libdfsim_b200_checked.so): a device-side bounds
                                     check of a launch failed; last_error names the kernel and check bits */

/* per-(sim,node) duration source tags written by dfsim_estimate_batch */
#define DFSIM_SRC_OVERRIDE 0
#define DFSIM_SRC_EXACT 1
#define DFSIM_SRC_FITTED 2
#define DFSIM_SRC_COMM 3
#define DFSIM_SRC_BAD_BYTES 253  /* Transfer with bytes <= 0: transfer_time raises ValueError */
#define DFSIM_SRC_NEGATIVE 254   /* value not >= 0 */
#define DFSIM_SRC_UNKNOWN 255

typedef struct dfsim_ctx dfsim_ctx;

/* One execution context per (device, stream).  stream may be NULL (legacy default). */
int dfsim_ctx_create(int32_t device, void *stream, dfsim_ctx **out);
int dfsim_ctx_destroy(dfsim_ctx *ctx);
int dfsim_ctx_set_stream(dfsim_ctx *ctx, void *stream);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t dfsim_ctx_launch_count(const dfsim_ctx *ctx);
/* Human-readable text of the last failure on this context (host memory, owned by ctx). */
const char *dfsim_ctx_last_error(const dfsim_ctx *ctx);
int32_t dfsim_abi_version(void);

/* ---------------------------------------------------------------- graph (one topology class) */
typedef struct {
    int32_t n_nodes;          /* N */
    int32_t n_devices;        /* D, devices that nodes are placed on (<= 32 for the warp engine) */
    int64_t n_edges;          /* E, non-dangling successor references */
    const int32_t *succ_off;  /* [N+1] */
    const int32_t *succ_idx;  /* [E] consumer ranks, ascending per producer, multiplicity kept */
    const int32_t *indeg;     /* [N] input references incl. dangling ones (graph.py:133-135) */
    const int32_t *device;    /* [N] device rank */
    const int32_t *sources;   /* [n_sources] ranks with indeg == 0, ascending */
    int32_t n_sources;
    const int32_t *queue_off; /* [D+1] prefix of per-device node counts (FIFO capacity) */
    const int32_t *topo;      /* [N] a topological order, or NULL when only simulating */
    int32_t max_indeg;        /* max over indeg[] (selects 8/16/32-bit packed counters) */
} dfsim_graph;

/* Kahn order of g into topo[N] (device); *n_ordered_host receives how many were ordered
 * (< N means a cycle).  Synchronous. */
int dfsim_topo_order(dfsim_ctx *ctx, const dfsim_graph *g, int32_t *topo, int32_t *n_ordered_host);

/* ---------------------------------------------------------------- expansion (K1) */
typedef struct {
    int32_t n_base;            /* N0 nodes in base insertion order */
    const int32_t *in_off;     /* [N0+1] input refs per base node */
    const int32_t *in_src;     /* [refs] producer base index, -1 if dangling */
    const int32_t *base_dev;   /* [N0] expanded-device rank for non-remapped clones */
    const uint8_t *remap;      /* [N0] 1 if the clone moves to device_map[k] (Compute + device_map) */
    const int32_t *marked;     /* [N0] collective index g (0..G-1) if the node is a marked gradient, else -1 */
    int32_t n_refs;            /* in_off[N0] if known on the host, else -1 (read back, synchronising) */
} dfsim_base_graph;

typedef struct {
    int32_t replicas;          /* R */
    int32_t n_collectives;     /* G (0 when R == 1) */
    const int32_t *clone_rank; /* [R*N0] rank of "<id>@r<k>" at index k*N0+v */
    const int32_t *coll_rank;  /* [G] rank of "allreduce_<gid>" */
    const int32_t *map_dev;    /* [R] device rank of device_map[k] (ignored where remap==0) */
    int32_t fabric_dev;        /* device rank of the collective fabric */
    /* parameter-server mode (ps != 0; new code, no reference: ps.py): each marked gradient g gets
     * push_<g>@r<k> (input g@r<k>, device up_dev[k]), aggregate_<g> (inputs push_<g>@r*, rank
     * coll_rank[g], device ps_dev) and pull_<g>@r<k> (input aggregate_<g>, device down_dev[k]);
     * consumers of g@r<k> read pull_<g>@r<k> instead (slot kept). */
    int32_t ps;
    const int32_t *push_rank;  /* [G*R] rank of push_<g>@r<k> at g*R+k */
    const int32_t *pull_rank;  /* [G*R] rank of pull_<g>@r<k> */
    const int32_t *up_dev;     /* [R] device rank of the worker k -> PS link */
    const int32_t *down_dev;   /* [R] device rank of the PS -> worker k link */
    int32_t ps_dev;            /* device rank of the parameter server */
} dfsim_expand_plan;

/* Emits the expanded graph's CSR (succ_off/succ_idx), indeg, device, sources, queue_off
 * and topo into the caller-allocated arrays of *out (sizes: N = R*N0 + G, or R*N0 +
 * G*(2R+1) in PS mode; succ_capacity >= R*refs + G*R, or R*refs + 3*G*R in PS mode; E given
 * by *n_edges_host after the call).  Synchronous when the three *_host count pointers are
 * given; with all three NULL (and base->n_refs >= 0) it is fully asynchronous. */
int dfsim_expand_dp(dfsim_ctx *ctx, const dfsim_base_graph *base, const dfsim_expand_plan *plan,
                    int32_t *succ_off, int32_t *succ_idx, int64_t succ_capacity, int32_t *indeg,
                    int32_t *device, int32_t *sources, int32_t *queue_off, int32_t *topo,
                    int32_t n_devices, int64_t *n_edges_host, int32_t *n_sources_host,
                    int32_t *n_ordered_host);

/* ---------------------------------------------------------------- profile tables (K2) */
typedef struct {
    /* per node; the rows marked [GV][N] hold one row per graph variant (graphs of identical
     * structure whose attributes / shapes differ, e.g. one per batch size) */
    const int32_t *op;          /* [N] op-type id */
    const uint8_t *kind;        /* [N] 0 Compute, 1 Transfer, 2 Collective */
    const int32_t *sig;         /* [GV][N] feature-vector id */
    const int64_t *comm_bytes;  /* [GV][N] attrs["bytes"] when it is a Python int, else ignored */
    const uint8_t *comm_ok;     /* [GV][N] Transfer: Link device and int bytes; Collective: list group and int bytes */
    const int32_t *group_size;  /* [GV][N] len(attrs["group"]) for collectives */
    const double *link_thr;     /* [GV][N] Transfer: link throughput MB/s */
    const double *link_lat;     /* [GV][N] Transfer: link latency us */
    /* feature vectors, names sorted by string rank */
    int32_t n_sigs;
    const int32_t *sig_off;     /* [n_sigs+1] */
    const int32_t *sig_name;    /* feature-name ids */
    const double *sig_val;
    /* exact records: keys sorted ascending, key = hw<<42 | op<<21 | sig */
    int32_t n_exact;
    const uint64_t *exact_key;
    const double *exact_mean;
    /* fitted models: keys sorted ascending, key = hw<<21 | op; model m uses
     * names/coefs[model_off[m] .. model_off[m+1]) and intercept[m] */
    int32_t n_models;
    const uint64_t *model_key;
    const int32_t *model_off;
    const int32_t *model_name;
    const double *model_coef;
    const double *model_icpt;
    /* links: nccl-allreduce records keyed path<<32 | participants (sorted) and
     * gpu-gpu-uni/path/2 per path id (uni_ok==0 when absent) */
    int32_t n_nccl;
    const uint64_t *nccl_key;
    const double *nccl_thr;
    int32_t n_paths;
    const uint8_t *uni_ok;
    const double *uni_thr;
    const double *uni_lat;
    /* overrides: per override set, sorted node ranks and values */
    int32_t n_override_sets;
    const int32_t *ov_off;
    const int32_t *ov_node;
    const double *ov_val;
} dfsim_profile_tables;

typedef struct {
    int64_t n_sims;
    const int32_t *hw;         /* [S] hardware-tag id */
    const double *op_gap;      /* [S] op_gap_us */
    const uint8_t *algo;       /* [S] 0 MeasuredThroughput, 1 RingAnalytic */
    const int32_t *path;       /* [S] collective path id */
    const int32_t *override_set; /* [S] -1 for none */
    const int32_t *gvariant;   /* [S] graph variant, or NULL for variant 0 */
} dfsim_strategies;

/* dur[s*N+v], src[s*N+v]; bad[s] = number of nodes whose source is >= 253 */
int dfsim_estimate_batch(dfsim_ctx *ctx, int32_t n_nodes, const dfsim_profile_tables *t,
                         const dfsim_strategies *st, double *dur, uint8_t *src, int32_t *bad);

/* ---------------------------------------------------------------- simulation (K3) */
/* dur is [n_sims][dur_stride] (dur_stride >= N, or 0 to broadcast one row).
 * start/finish are [n_sims][N] (both NULL: makespan-only mode).  busy is
 * [n_sims][n_devices] or NULL.  n_placed[s] < N marks a CycleError for sim s. */
int dfsim_simulate_batch(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                         int64_t dur_stride, double *start, double *finish, double *makespan,
                         double *busy, int32_t *n_placed);

/* Exact engine with remapped outputs (the fused engine's overflow fallback):
 * row s of dur is simulated and written to output row out_rows[s] (or s when
 * NULL), node v at column pos[v] (or v when NULL).  interleaved 1: start points at
 * [rows][N] (start, finish) pairs and finish is ignored; 2: the same pairs in the fused
 * engine's tiled layout (see dfsim_simulate_fused). */
int dfsim_simulate_batch_ex(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *dur,
                            int64_t dur_stride, double *start, double *finish, double *makespan, double *busy,
                            int32_t *n_placed, const int32_t *pos, const int64_t *out_rows, int32_t interleaved);

/* ---------------------------------------------------------------- fused hot path (K2a + K3 v2 + K4 v2) */
/* Class tables built once per topology class (paper_2002_06790_b200/prepare.py).
 * Nodes are numbered by level position p (the output column); rank[p] is the node's
 * rank (id order), used for the FIFO tie-break, overrides and the source order. */
typedef struct {
    int32_t n_nodes;           /* N <= 65535 */
    int32_t n_devices;         /* D <= 32 */
    int64_t n_edges;
    const uint32_t *meta;      /* [N] by position: successor begin (24 bits) | out-degree (8 bits, < 255) */
    const int32_t *succ_off;   /* [N+1] (rank CSR; sizes only) */
    const uint32_t *succ;      /* [E] by reading position: consumer position | device << 16 | single-input << 21 */
    const uint16_t *cidx;      /* [N] by position: counter code of nodes with >= 2 input references:
                                  word << 7 | bit shift << 2 | log2(width) - 1, width 2/4/8/16 bits */
    const uint32_t *cnt_init;  /* [n_counter_words] packed initial counters (<= 512 words) */
    int32_t n_counter_words;
    int32_t counter_bits;      /* widest counter field (2, 4, 8 or 16) */
    const uint16_t *rank;      /* [N] rank of the node at position p */
    const int32_t *sources;    /* positions of the in-degree-0 nodes, in ascending rank */
    int32_t n_sources;
    int32_t qcap;              /* per-device FIFO ring capacity (power of two); overflow flags the candidate */
    const int32_t *device;     /* [N] device index by rank */
    int32_t succ_packed;       /* 1: succ[j] = consumer position (13 bits) | device << 13 (4 bits) | single << 17 |
                                  wide << 18 | shift << 19 | word << 24 (N <= 8192, D <= 16, counters of
                                  2/4 bits in <= 256 words; cidx unused); 0: the layout above */
} dfsim_sim_tables;

typedef struct {
    int64_t n_sims;
    int32_t n_variants;
    const double *base;        /* [V][N] from dfsim_resolve_variants */
    int32_t n_chunks;          /* work items of <= 32 candidates sharing one variant */
    const int64_t *order;      /* [S] candidate indices grouped by variant */
    const int32_t *chunk_first;
    const int32_t *chunk_count;
    const int32_t *chunk_variant;
    const double *op_gap;      /* [S] */
    const int32_t *override_set; /* [S] or NULL */
    const int32_t *ov_off;
    const int32_t *ov_node;
    const double *ov_val;
    int32_t max_chunk;         /* largest chunk_count (0: the capacity); CTAs are sized to it, so a
                                  small class spread over many small chunks fills the SMs */
    const uint32_t *ov_any;    /* [(N + 31) / 32] bit per node rank: in some override set (NULL: search
                                  every popped node of a candidate with overrides) */
    int32_t sched_tiled;       /* 1: the tiled schedule layout (for K4 v3); 0: rows sched[S][N][2] (K4 v2) */
} dfsim_fused_strategies;

/* K2a: base[var*N+v] = estimate of node v under variant var = (graph variant, hw, algo, path) with
 * op_gap 0; sign bit set when the candidate's op_gap must be added.  status is the
 * DFSIM_SRC_* tag per (var, v). */
int dfsim_resolve_variants(dfsim_ctx *ctx, int32_t n_nodes, const dfsim_profile_tables *t, int32_t n_variants,
                           const int32_t *var_hw, const uint8_t *var_algo, const int32_t *var_path,
                           const int32_t *var_gv, double *base, uint8_t *status);

/* Rows of (variant, override set) combinations for the fused engine: out[c][r] = base[combo_variant[c]][r],
 * with the override values of set combo_set[c] (-1: none) stamped in at their ranks (sign clear:
 * an override replaces the estimate, costmodel.py:302-304).  Candidates then need no override
 * lookup in the engine (dfsim_fused_strategies.override_set = NULL). */
int dfsim_override_rows(dfsim_ctx *ctx, int32_t n_nodes, int32_t n_combos, const double *base,
                        const int32_t *combo_variant, const int32_t *combo_set, const int32_t *ov_off,
                        const int32_t *ov_node, const double *ov_val, double *out);

/* Candidates one CTA of the fused engine holds; chunks of dfsim_fused_strategies
 * must not exceed it (0: the class does not fit the fused engine). */
int32_t dfsim_fused_capacity(const dfsim_sim_tables *g);

/* Chunk size for a class of n_sims candidates on a GPU of num_sms SMs: small classes are
 * cut finer so their CTAs cover the SMs, never below the size at which a CTA's copy of
 * the class tables outweighs its candidates' state; <= dfsim_fused_capacity. */
int32_t dfsim_fused_chunk(const dfsim_sim_tables *g, int64_t n_sims, int32_t num_sms);

/* K3 v2: outputs (start, finish) pairs by level position.  st->sched_tiled = 1 (classes on K4 v3):
 * in 32-candidate tiles -- the candidate at position k of st->order (its "slot"), node position p
 * at pair ((k / 32) * N + p) * 32 + k % 32 of sched (room for ceil(S / 32) * 32 slots); the
 * candidates of one chunk are neighbours, so a tile's writes meet in L2.  0 (K4 v2): rows,
 * candidate s at pairs [s * N, s * N + N).  16-byte aligned.  A warp of K4 v3 (lane = candidate) thus reads one
 * contiguous 512-byte run per position; a schedule row is a stride-32 gather;
 * flags[s] = 1 when the FIFO ring overflowed (re-run s with dfsim_simulate_batch_ex);
 * n_placed[s] = -1 then. */
int dfsim_simulate_fused(dfsim_ctx *ctx, const dfsim_sim_tables *g, const dfsim_fused_strategies *st,
                         double *sched, double *makespan, double *busy, int32_t *n_placed, int32_t *flags);

typedef struct {
    int32_t n_nodes;
    int32_t n_slots;           /* suffix slots per candidate (interval colouring) */
    int32_t n_edges;
    const int32_t *rank_of_pos;
    const uint32_t *cp_meta;   /* [N] by position: successor begin | count << 16 | source << 24 */
    const uint16_t *cp_slot;   /* [N] by position (0xFFFF: none) */
    const uint16_t *cp_succ_slot; /* [E] index (doubles) of the successor's value in the candidate's shared
                                     region: a slot, or a prefetched spill value of the reader's chunk stage */
    int32_t n_groups;
    const int32_t *group_off;  /* <= 16 positions of one level each (a half-warp per candidate) */
    int32_t n_chunks;
    const int32_t *chunk_off;  /* groups per prefetch chunk */
    int32_t chunk_positions;   /* max positions per chunk */
    int32_t n_long;            /* spilled suffix values per candidate (read >= 2 chunks later) */
    const uint16_t *cp_spill;  /* [N] by position: spill index written (0xFFFF none) */
    const int32_t *spill_off;  /* [n_chunks+1] spill values each chunk reads */
    const uint16_t *spill_list;/* spill indices, per chunk */
    int32_t max_spill_reads;   /* max spill values one chunk reads */
    const uint32_t *pinfo;     /* [N] by position: slot | has-slot << 15 | spill index << 16 | spill << 31 */
    int32_t slot_region;       /* doubles of suffix slots at the start of a candidate's shared region */
    int32_t stage_doubles;     /* doubles per prefetch stage: (start, finish) x K | spill values R */
} dfsim_cp_tables;

/* K4 v2: critical-path length and its start node per candidate over the fused engine's
 * (start, finish) pairs in the rows layout (dfsim_simulate_fused, sched_tiled = 0); row k holds
 * candidate cand_of_slot[k] (NULL: k), whose cp_len / cp_src are written. */
int dfsim_critical_path_levels(dfsim_ctx *ctx, const dfsim_cp_tables *t, int64_t n_sims,
                               const int64_t *cand_of_slot, const double *sched, double *cp_len, int32_t *cp_src);

/* Candidates one CTA of dfsim_critical_path_levels holds (0: the class tables do not fit
 * in shared memory; such a class uses the rank-layout kernels instead). */
int32_t dfsim_critical_path_levels_capacity(const dfsim_cp_tables *t);

/* K4 v3 (lane per candidate): graph.py:446-474 on finish - start over the fused engine's
 * tiled (start, finish) pairs (dfsim_simulate_fused).  Every lane of a warp is one candidate and the warp
 * walks the class's positions in reverse (one node at a time, all lanes in step), so the
 * class tables are read once per 32 candidates.  A node's suffix value lives in a shared-
 * memory slot while it is read within its own or the next prefetch chunk, otherwise in a
 * per-warp spill row [n_long][32] in global memory, prefetched with the reading chunk.
 * Node records stream from global memory with the schedule data, one block per chunk.
 * Tables come from dfsim_cp_lanes_plan (host). */
typedef struct {
    int32_t n_nodes;
    int32_t n_chunks;          /* prefetch chunks, in processing order (highest positions first) */
    int32_t chunk_positions;   /* K: a chunk covers at most K positions (8: the register window) */
    int32_t n_slots;           /* shared-memory suffix rows per warp (slots) */
    int32_t rmax;              /* spill values prefetched per chunk, at most */
    int32_t n_long;            /* values kept in spill rows */
    int32_t n_spill_list;      /* length of spill_list (= spill_off[n_chunks]) */
    int32_t block_max;         /* largest chunk block, in 16-byte units */
    const uint32_t *blocks;    /* [4 per 16-byte unit] per chunk, in processing order: one 16-byte record per position
                                  {x: slot | has_slot << 12 | source << 13 | has_spill << 14 | spill << 15,
                                   y: successors | extra << 8 (u16 offset of successors 5.. in the block),
                                   z, w: rows of successors 1-4 (16 bits each)}, then the extra rows */
    const int32_t *block_off;  /* [n_chunks + 1] in 16-byte units */
    const int32_t *bounds;     /* [n_chunks + 1]: chunk q covers positions [bounds[q+1], bounds[q]) */
    const int32_t *spill_off;  /* [n_chunks + 1] */
    const uint16_t *spill_list; /* spill indices prefetched with each chunk, in stage-row order */
    const int32_t *rank_of_pos; /* [N] node rank of each position (source tie-break) */
} dfsim_cp_lane_tables;

/* Host planner of dfsim_cp_lane_tables (C++, no device work): positions 0..N-1 in a level
 * order (every edge from a lower to a higher position), succ_off[N+1] / succ_pos[E] the
 * successors of each position, is_source[N].  Chunks of <= K positions are cut in reverse
 * order so that no chunk prefetches more than max(rmax_min, widest node) spill values.
 * A value read within near_chunks chunks of its writer's (at least `stages`) keeps a slot.
 * Value rows of a warp's shared region: [slots | spill stage 0 .. stages-1].  Output arrays
 * are caller-allocated at their bounds: blocks[4 * (2N + E/8 + 2)] u32, block_off[N+1],
 * bounds[N+1], spill_off[N+1], spill_list[E]; info[6] = {n_chunks, n_slots, rmax, n_long,
 * spill_list length, block_max}.  Returns DFSIM_BAD_ARGUMENT when a field overflows. */
int dfsim_cp_lanes_plan(int32_t n, const int32_t *succ_off, const int32_t *succ_pos, const uint8_t *is_source,
                        int32_t K, int32_t rmax_min, int32_t stages, int32_t near_chunks, uint32_t *blocks,
                        int32_t *block_off, int32_t *bounds, int32_t *spill_off, uint16_t *spill_list,
                        int32_t *info);

/* stages: must be 0 (the register-window kernel; the tables are planned with 2 smem stages). */
int dfsim_critical_path_lanes(dfsim_ctx *ctx, const dfsim_cp_lane_tables *t, int32_t stages, int64_t n_sims,
                              const int64_t *cand_of_slot, const double *sched, double *cp_len, int32_t *cp_src);

/* Schedules are read at their slots in the fused engine's tiled layout; the candidate of slot
 * k is cand_of_slot[k] (the engine's candidate order; NULL: k), and cp_len / cp_src are written
 * at the candidate.  _ex: only the slots slots[0..n_sims) (device int64; NULL: 0..n_sims-1),
 * with at most max_warps warps a CTA (0: as many as fit) so that the kernel can share SMs with
 * a concurrently running engine launch. */
int dfsim_critical_path_lanes_ex(dfsim_ctx *ctx, const dfsim_cp_lane_tables *t, int32_t stages, int64_t n_sims,
                                 const int64_t *slots, const int64_t *cand_of_slot, int32_t max_warps,
                                 const double *sched, double *cp_len, int32_t *cp_src);

/* Warps (32 candidates each) one CTA of dfsim_critical_path_lanes holds (0: does not fit). */
int32_t dfsim_critical_path_lanes_capacity(const dfsim_cp_lane_tables *t, int32_t stages);

/* ---------------------------------------------------------------- critical path (K4) */
/* Over d = finish - start (reporting.py:128), or over d = finish when start is NULL
 * (the plain critical_path(g, durations) call).  cp_len[s]; cp_path [n_sims][N] and
 * cp_path_len[s] are optional (NULL skips the path walk).  Needs g->topo. */
int dfsim_critical_path_batch(dfsim_ctx *ctx, const dfsim_graph *g, int64_t n_sims, const double *start,
                              const double *finish, double *cp_len, int32_t *cp_path, int32_t *cp_path_len);

/* K4 wide, for graphs beyond dfsim_critical_path_levels (N > 65535): one CTA per candidate
 * walks the levels in reverse (order[N]: ranks grouped by level, level_off[n_levels+1]; every
 * edge goes to a higher level), one thread per node of a level.  cp_len[s]; cp_src[s] = rank
 * of the path's start node (optional).  start NULL: finish holds durations.  [n_sims][N] by rank. */
int dfsim_critical_path_wide(dfsim_ctx *ctx, const dfsim_graph *g, const int32_t *order, const int32_t *level_off,
                             int32_t n_levels, int64_t n_sims, const double *start, const double *finish,
                             double *cp_len, int32_t *cp_src);

/* ---------------------------------------------------------------- scalar formulas (drop-in) */
/* predict (costmodel.py:158-165) for n feature vectors feats[n][k] of one linear model:
 * out[i] = max(0.0, intercept + sum(coef[j] * feats[i][j])) with CPython 3.12's float sum. */
int dfsim_predict_batch(dfsim_ctx *ctx, int32_t k, const double *coef, double intercept, int64_t n,
                        const double *feats, double *out);
/* Communication formulas (costmodel.py:168-223) for n rows: kind 0 = comm_time_us
 * (transfer_time, measured allreduce with lat 0), kind 1 = ring allreduce over a link. */
int dfsim_comm_batch(dfsim_ctx *ctx, int64_t n, const uint8_t *kind, const int64_t *bytes,
                     const int32_t *participants, const double *thr, const double *lat, double *out);
/* topological_order (graph.py:424-443) on the host: Kahn with a min-heap of ranks into
 * order[n]; returns how many nodes were ordered (< n: a cycle), -1 on bad arguments. */
int32_t dfsim_topological_order(int32_t n, const int32_t *succ_off, const int32_t *succ_idx, const int32_t *indeg,
                                int32_t *order);
/* Host planning of a topology class (csrc/levels.cpp; no reference counterpart: table layout).
 * dfsim_level_order: Kahn waves (each sorted by rank) into order[n], level[n] and
 * level_off[n + 1]; returns the number of levels, -1 for a cycle, -2 on bad arguments. */
int32_t dfsim_level_order(int32_t n, const int32_t *succ_off, const int32_t *succ_idx, const int32_t *indeg,
                          int32_t *order, int32_t *level, int32_t *level_off);
/* dfsim_cp_levels_plan: the K4 v2 tables (CpTables) from the rank CSR and the level order.
 * Capacities: group_off / chunk_off / spill_off n + 1, slot_of_pos / spill_of_pos / cp_meta /
 * pinfo n, spill_list / cp_succ / cp_succ_abs n_edges.  info[8] = n_groups, n_chunks, n_slots,
 * n_long, max_spill_reads, n_spill_list, slot_region, stage_doubles.  0 on success. */
int32_t dfsim_cp_levels_plan(int32_t n, const int32_t *succ_off, const int32_t *succ_idx, const int32_t *indeg,
                             const int32_t *order, const int32_t *level_off, int32_t n_levels, int32_t group,
                             int32_t chunk, int32_t *group_off, int32_t *chunk_off, int32_t *slot_of_pos,
                             int32_t *spill_of_pos, int32_t *spill_off, int32_t *spill_list, int32_t *cp_succ,
                             int32_t *cp_succ_abs, uint32_t *cp_meta, uint32_t *pinfo, int32_t *info);

/* ---------------------------------------------------------------- best strategy (K5) */
/* First minimum of (value, index) over n values; index = index_base + i.
 * Writes one 16-byte record {double value; int64_t index} to out_record (device). */
int dfsim_argmin(dfsim_ctx *ctx, int64_t n, const double *values, int64_t index_base, void *out_record);
/* Lexicographic min over n gathered records (e.g. after an NCCL all-gather). */
int dfsim_argmin_records(dfsim_ctx *ctx, int64_t n, const void *records, void *out_record);

/* ---------------------------------------------------------------- schedule summary (K6) */
/* reporting.summarize (reporting.py:117-162) for a batch of schedules resident on the
 * device.  Class-wide tables, indexed by node rank: */
typedef struct {
    int32_t n_nodes;
    int32_t n_keys;              /* distinct op keys (`op_type or node_id`, reporting.py:132) */
    const int32_t *base_order;   /* [N] node ranks sorted by (device string rank, node rank) */
    const int32_t *key;          /* [N] op key index of each node (0..n_keys-1) */
    const uint8_t *comm;         /* [N] 1 when the node's device is not Compute (reporting.py:140) */
} dfsim_summary_tables;

/* start/finish: [n_rows][ld] by node rank.  entry_order [n_rows][N]: the schedule's entry
 * order (engine.py:88), written unless order_given (then read, e.g. a drop-in Schedule).
 * Outputs: key_total/key_first [n_rows][n_keys] (per-key total folded in entry order;
 * entry index of the key's first appearance or -1), sums [n_rows][3] = compute_us,
 * comm_us, overlap_us.  Asynchronous on the ctx stream. */
int dfsim_summarize(dfsim_ctx *ctx, const dfsim_summary_tables *t, int64_t n_rows, const double *start,
                    const double *finish, int64_t ld, int32_t *entry_order, int32_t order_given,
                    double *key_total, int32_t *key_first, double *sums);

/* ---------------------------------------------------------------- Chrome trace (host) */
/* reporting.to_trace (reporting.py:43-74), byte-identical: json.dumps(events, indent=1)
 * with ensure_ascii escaping and round-half-even integer ts/dur.  Host memory only. */
typedef struct {
    int32_t n_nodes;
    int32_t n_tracks;             /* devices of the schedule's busy dict, sorted (tid order) */
    const char *id_blob;          /* node ids, UTF-8: node v = id_blob[id_off[v] .. id_off[v+1]) */
    const int64_t *id_off;        /* [N+1] */
    const char *name_blob;        /* event names (`op_type or node_id`) */
    const int64_t *name_off;      /* [N+1] */
    const uint8_t *tag;           /* [N] duration source tag index */
    const char *const *tag_name;  /* tag strings (NUL-terminated) */
    const int32_t *track;         /* [N] tid of the node's device (n_tracks when absent) */
    const char *const *track_name;/* [n_tracks] NUL-terminated UTF-8 */
} dfsim_trace_tables;

/* Writes the document for entries entry_node[0..n_entries) (node indices in entry order)
 * with start/finish indexed by node.  Returns the document length in bytes; the text is
 * copied to buf only when it fits in cap (call with cap = 0 to size it).  < 0 on bad args. */
int64_t dfsim_trace_write(const dfsim_trace_tables *t, int64_t n_entries, const int32_t *entry_node,
                          const double *start, const double *finish, char *buf, int64_t cap);

/* ---------------------------------------------------------------- graph documents (host) */
/* parse_graph (graph.py:192-293) + the lowering's CSR / node rows for large documents, in C++.
 * Only well-formed documents load; anything the reference warns about or rejects returns
 * DFSIM_CONFIG with a reason, and the caller re-parses with the reference semantics. */
typedef struct {
    int32_t n_nodes, n_devices, n_ops, n_sigs, n_fnames, n_declared, max_indeg, n_sources;
    int64_t n_edges;
    const char *id_blob; const int64_t *id_off;       /* node ids in rank (code-point) order */
    const char *op_blob; const int64_t *op_off;       /* op types, first appearance in rank order */
    const char *dev_blob; const int64_t *dev_off;     /* node devices, sorted (the device ranks) */
    const char *fname_blob; const int64_t *fname_off; /* feature names */
    const int32_t *op_of; const uint8_t *kind_of;     /* per node: op index, kind 0/1/2 */
    const int32_t *dev_of, *indeg, *succ_off, *succ_idx, *sources, *queue_off;  /* host_csr arrays */
    const int32_t *sig_of; const int64_t *sig_off;    /* feature signature per node (first appearance) */
    const int32_t *sig_fname; const double *sig_fval; /* signature k: names/values [sig_off[k], sig_off[k+1]) */
    const uint8_t *comm_ok; const int64_t *comm_bytes; const int32_t *group_size;
    const double *link_thr, *link_lat;                /* node_rows communication attributes */
    const int64_t *node_lo, *node_hi;                 /* byte range of each node's JSON object */
    int64_t meta_lo, meta_hi;                         /* metadata object (-1: absent) */
    int64_t decl_lo, decl_hi;                         /* devices list (-1: absent) */
} dfsim_document;

int dfsim_document_parse(const char *text, int64_t len, void **doc_out, char *why, int64_t why_cap);
const dfsim_document *dfsim_document_view(const void *doc);
void dfsim_document_free(void *doc);

#ifdef __cplusplus
}
#endif
#endif /* DFSIM_B200_H */
