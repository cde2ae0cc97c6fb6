/*
 * pgmoe.h — C ABI of the B200-native pre-gated MoE block (libpgmoe.so).
 *
 * Drop-in boundary for the reference package `moesim`
 * (/root/reference/pkg/src/moesim).  Each entry point names the reference
 * interface it replaces (file:line).  Plain pointers and sizes only: no
 * torch types cross this boundary.  Activations are fp32, weights fp32 or
 * bf16 (bf16 = RNE of the fp32 value the reference is fed).
 *
 * Conventions
 *  - Every call returns a pgmoe_status.  Status codes map 1:1 onto the
 *    reference exception tree (errors.py:4-33); see pgmoe_status below.
 *  - Calls taking a `stream` are stream-ordered and asynchronous.  Errors
 *    the device detects (non-finite logits, zero routing weight) are written
 *    to the routing buffer's `status[0]` and surfaced by pgmoe_check_routing()
 *    (or by the synchronous *_host entry points), i.e. at the next sync
 *    point, not eagerly as Python raises them.
 *  - Device pointers are caller-owned unless produced by a *_create call.
 *  - No CPU fallback: every compute entry point launches sm_100a kernels.
 */
#ifndef PGMOE_H
#define PGMOE_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PGMOE_API __attribute__((visibility("default")))
#else
#define PGMOE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *pgmoe_stream_t; /* == cudaStream_t */

/* errors.py:4-33 — the Python shim raises the same-named exception. */
typedef enum {
    PGMOE_OK = 0,
    PGMOE_E_CONFIG = 1,          /* ConfigError          (core.py:54-70, :291) */
    PGMOE_E_SHAPE = 2,           /* ShapeError           (core.py:293, :310)   */
    PGMOE_E_GATE_OVERFLOW = 3,   /* GateOverflowError "numerical overflow in gate" (core.py:297) */
    PGMOE_E_GATE_UNDERFLOW = 4,  /* GateOverflowError "gate routing weight underflowed to zero" (core.py:303) */
    PGMOE_E_ROUTING = 5,         /* RoutingError         (core.py:110-140, :332, :369-382) */
    PGMOE_E_OOM = 6,             /* OomError             (tiers.py:134-157; HBM exhausted) */
    PGMOE_E_CUDA = 7,            /* MoESimError (device/runtime failure) */
    PGMOE_E_NCCL = 8,            /* MoESimError (collective failure) */
    PGMOE_E_WEIGHT_FILE = 9,     /* WeightFileError      (model_io.py:63-105) */
    PGMOE_E_INVARIANT = 10       /* InvariantError       (scheduler.py:127-145) */
} pgmoe_status;

typedef enum { PGMOE_F32 = 0, PGMOE_BF16 = 1, PGMOE_F64 = 2 /* gate weights of pgmoe_gate_forward_f64 only */ } pgmoe_dtype;
typedef enum { PGMOE_RESIDENT = 0, PGMOE_OFFLOADED = 1 } pgmoe_placement;
typedef enum { PGMOE_KERNEL_AUTO = 0, PGMOE_KERNEL_SIMT = 1, PGMOE_KERNEL_TCGEN05 = 2 } pgmoe_kernel;
/* Expert migration policy of an offloaded model (scheduler.py:36-49).  The
 * resident strategy is PGMOE_RESIDENT placement. */
typedef enum { PGMOE_PRE_GATED = 0, PGMOE_ON_DEMAND = 1, PGMOE_PREFETCH_ALL = 2 } pgmoe_strategy;

/* core.py:34-70 ModelConfig (dtype_bytes is implied by the weight dtype). */
typedef struct {
    int32_t d_model, d_ff, num_blocks, num_experts, top_k, activation_level;
    uint64_t seed;
} pgmoe_config;

/* Device routing buffers for T tokens (the batched RoutingDecision,
 * core.py:110-140, plus the SURVEY §8 a8 permutation). */
typedef struct {
    int32_t *ids;    /* [T][k] expert ids, descending logit, ties -> lower id */
    float *w;        /* [T][k] softmax probabilities of the selected experts */
    int32_t *hist;   /* [E]    tokens routed to each expert */
    int32_t *off;    /* [E+1]  exclusive scan of hist */
    int32_t *perm;   /* [T*k]  entry index t*k+s grouped by expert, stable */
    float *w_perm;   /* [T*k]  w of perm[r] */
    int32_t *act;    /* [E]    active experts ascending (first *n_act valid) */
    int32_t *n_act;  /* [1] */
    int32_t *status; /* [4] [0] device error code, [1] tokens that needed the
                        serial-fp64 recompute, [2], [3] reserved */
    int32_t *inv;    /* [T*k] optional (may be NULL): position of entry t*k+s in perm */
} pgmoe_routing;

/* ---------------------------------------------------------------- kernels */

/* Bytes of device scratch pgmoe_gate_forward needs for T tokens. */
PGMOE_API size_t pgmoe_route_workspace_bytes(int32_t T, int32_t E);

/* K1 pre-gate / route.  Replaces gate_forward (core.py:284-305) for T
 * tokens at once, fused with the per-expert histogram, exclusive scan and
 * stable permutation.  x: fp32 [T][d]; gate_w: [d][E] (in x out, as the
 * reference stores it).  Ids are bit-exact with the reference's serial fp64
 * logits (certified fast logits + serial fallback).  `workspace` must hold
 * pgmoe_route_workspace_bytes(T, E) bytes, zeroed once before first use. */
PGMOE_API int pgmoe_gate_forward(const float *x, int32_t T, int32_t d, const void *gate_w,
                       int32_t wdtype, int32_t E, int32_t k, const pgmoe_routing *out,
                       void *workspace, pgmoe_stream_t stream);

/* K1 at the reference's own precision: x fp64 [T][d] and gate_w fp64 [d][E]
 * (moesim's init_model matrices and inputs are fp64 Python floats,
 * core.py:200-211, :274-277).  Products are no longer exact in fp64, so
 * the certification bound takes one more rounding (gamma_{d+1}); the serial
 * fallback is the same __dadd_rn(__dmul_rn) loop.  Ids equal moesim's
 * gate_forward bit-for-bit on unrounded inputs.  Same workspace as above. */
PGMOE_API int pgmoe_gate_forward_f64(const double *x, int32_t T, int32_t d, const double *gate_w, int32_t E,
                                     int32_t k, const pgmoe_routing *out, void *workspace, pgmoe_stream_t stream);

/* K2 grouped expert FFN with fused combine.  Replaces expert_forward
 * (core.py:308-316) x k plus weighted_sum (linalg.py:45-51): for every
 * routed entry r, yw[perm[r]] = w_perm[r] * W2 relu(W1 x[perm[r]/k]).
 * Expert e's weights live at experts + slot(e) * expert_stride bytes with
 * W1 [f][d] first and W2 [d][f] after it; slot(e) = e when
 * `indexed_by_act` == 0 (resident), else its position i in act (slot cache).
 * h: fp32 scratch [T*k][f]; yw: fp32 [T*k][d]. */
PGMOE_API int pgmoe_expert_forward(const float *x, int32_t T, int32_t d, int32_t f, int32_t k,
                         const void *experts, size_t expert_stride, int32_t wdtype,
                         int32_t indexed_by_act, const pgmoe_routing *r, float *h, float *yw,
                         int32_t kernel, pgmoe_stream_t stream);

/* K3 dense non-MoE layer (core.py:338): y[t] = D . sum_s yw[t*k+s]
 * (slot order = routing order, linalg.py:45-51).  D: [d][d] out x in. */
PGMOE_API int pgmoe_dense_forward(const float *yw, int32_t T, int32_t d, int32_t k, const void *dense_w,
                        int32_t wdtype, float *y, int32_t kernel, pgmoe_stream_t stream);

/* ---------------------------------------------- expert parallelism (EP) */

/* Dispatch packing: out[r] = src[perm[r] / k] for r < n (rows of d floats). */
PGMOE_API int pgmoe_gather_rows(const float *src, const int32_t *perm, int32_t n, int32_t d, int32_t k,
                                float *out, pgmoe_stream_t stream);

/* Combine un-permute: yw[perm[r]] = w_perm[r] * back[r] (linalg.py:45-51 weights). */
PGMOE_API int pgmoe_unpermute_combine(const float *back, const int32_t *perm, const float *w_perm, int32_t n,
                                      int32_t d, float *yw, pgmoe_stream_t stream);

/* Receiver routing over rows received from P ranks: recv_cnt [P][El] holds
 * how many rows each source sent for each local expert (rows arrive grouped
 * by source, then by expert).  Fills hist/off/perm/act/n_act (w_perm = 1). */
PGMOE_API int pgmoe_ep_local_routing(const int32_t *recv_cnt, int32_t P, int32_t El, const pgmoe_routing *out,
                                     pgmoe_stream_t stream);

/* Fixed-size (padded) expert-parallel exchange: no host round trip for the
 * all-to-all split sizes, and ONE all-to-all for rows and counts.  Rank p
 * owns experts [p*El, (p+1)*El); every rank sends every peer a slot of
 * slot_rows(cap, El, d) rows: cap (>= T*k) routed rows, then header rows
 * carrying the sender's per-expert counts for that peer (int32 [El]).
 *   slot_rows: cap + ceil(4 El / 2 d);
 *   pack_send: send[p][i] = bf16(x[perm[r] / k]), r = off[p*El] + i — the
 *     rows the tcgen05 FFN consumes in bf16, so exact at half the bytes —
 *     and send[p][cap..] = hist[p*El .. (p+1)*El);
 *   local_routing_padded: receiver routing over the padded rows, counts read
 *     from the received headers (source p's rows start at p * slot_rows);
 *   pack_recv: the received rows in local-expert order (the FFN operand),
 *     count read on the device (off[El]);
 *   expert_forward_packed: expert FFN on that operand, y rows scattered back
 *     to their padded receive positions;
 *   unpermute_padded: yw[perm[r]] = w_perm[r] * back[p][r - off[p*El]]
 *     (back in the same slot layout). */
PGMOE_API int pgmoe_ep_pack_send(const float *x, const pgmoe_routing *r, int32_t T, int32_t d, int32_t k, int32_t P,
                                 int32_t El, int32_t cap, uint16_t *send, pgmoe_stream_t stream);
PGMOE_API int32_t pgmoe_ep_slot_rows(int32_t cap, int32_t El, int32_t d);
PGMOE_API int pgmoe_ep_local_routing_padded(const uint16_t *recv, int32_t P, int32_t El, int32_t cap, int32_t d,
                                            const pgmoe_routing *out, pgmoe_stream_t stream);
PGMOE_API int pgmoe_ep_pack_recv(const uint16_t *recv, const pgmoe_routing *local, int32_t El, int32_t n_max,
                                 int32_t d, uint16_t *xb, pgmoe_stream_t stream);
/* pgmoe_ep_local_routing_padded + pgmoe_ep_pack_recv in one launch: the local
 * routing (out) and the received rows packed in local-expert order (xb,
 * P*cap rows max).  Same outputs as the two calls. */
PGMOE_API int pgmoe_ep_recv_route_pack(const uint16_t *recv, int32_t P, int32_t El, int32_t cap, int32_t d,
                                       const pgmoe_routing *out, uint16_t *xb, pgmoe_stream_t stream);
PGMOE_API int pgmoe_expert_forward_packed(const uint16_t *xb, int32_t n_max, int32_t d, int32_t f,
                                          const void *experts, size_t expert_stride, const pgmoe_routing *r,
                                          uint16_t *hb, float *y, pgmoe_stream_t stream);
PGMOE_API int pgmoe_ep_unpermute_padded(const float *back, const pgmoe_routing *r, int32_t T, int32_t d, int32_t k,
                                        int32_t P, int32_t El, int32_t cap, float *yw, pgmoe_stream_t stream);
/* Top-1: the combine weight applied and the result written as the dense
 * layer's bf16 operand mixb [T][d] (linalg.py:45-51 for k = 1), consumed by
 * pgmoe_dense_forward_packed (core.py:338) — one launch fewer per EP block. */
PGMOE_API int pgmoe_ep_unpermute_padded_bf16(const float *back, const pgmoe_routing *r, int32_t T, int32_t d,
                                             int32_t P, int32_t El, int32_t cap, uint16_t *mixb,
                                             pgmoe_stream_t stream);
PGMOE_API int pgmoe_dense_forward_packed(const uint16_t *mixb, int32_t T, int32_t d, const void *dense_w, float *y,
                                         pgmoe_stream_t stream);

/* Reads routing status after a sync: returns the device-detected error (or
 * PGMOE_OK) and optionally the serial-fallback counter.  (Flips against the
 * reference are not a device quantity: tests/ and bench.py measure them by
 * running the oracle on the same inputs.) */
PGMOE_API int pgmoe_check_routing(const pgmoe_routing *r, int32_t *fallbacks);

/* Supplied decisions: the `supplied_decisions` path of decoder_iteration
 * (core.py:342-364) and synthetic routing traces (gen_routing_trace,
 * core.py:436-479).  ids [T][k] / w [T][k] (device) are copied into `out`
 * with RoutingDecision's checks (core.py:110-140: ids distinct and in
 * [0, E), weights in (0, 1]; a violation sets status[0] = PGMOE_E_ROUTING),
 * and the same histogram / scan / stable permutation K1 builds. */
PGMOE_API int pgmoe_route_from_decisions(const int32_t *ids, const float *w, int32_t T, int32_t E, int32_t k,
                                         const pgmoe_routing *out, pgmoe_stream_t stream);

/* Deterministic weights: fills `out` ([rows][cols], wdtype) on the device
 * with Xoshiro256StarStar(derive_seed(seed, tag, block, expert)).fill_matrix
 * rounded to fp32 (then bf16), rng.py:15-93 + core.py:200-211. */
PGMOE_API int pgmoe_fill_weights(void *out, int32_t wdtype, uint64_t seed, int32_t tag, int32_t block,
                       int32_t expert, int64_t rows, int64_t cols, pgmoe_stream_t stream);

/* ------------------------------------------------------------ the model */

typedef struct pgmoe_model pgmoe_model;

typedef struct {
    int64_t pinned_hbm_bytes;     /* gates + dense (tiers.py:89-115 pinned_bytes) */
    int64_t slot_capacity_bytes;  /* bytes reserved per expert slot (offloaded) */
    int64_t eq1_peak_bytes;       /* pinned + max_N(act_N + act_N+1), tiers.py:68-86 */
    int64_t ledger_peak_bytes;    /* measured: max over event-ordered intervals */
    int64_t h2d_bytes;            /* expert bytes migrated since reset */
    int64_t h2d_copies;
    int64_t route_fallbacks;      /* tokens needing the serial fp64 recompute */
    int64_t reserved0;
    double h2d_seconds;           /* copy-stream busy time (CUDA events) */
    double last_step_seconds;
    int64_t cache_bytes;          /* HBM expert-cache region (0 = no cache) */
    int64_t cache_hits, cache_misses;
    int64_t d2d_bytes;            /* cache <-> working-slot copies */
    int64_t fused_blocks;         /* blocks whose dense layer ran inside the expert-FFN launch */
    int64_t fused_routes;         /* pre-gates computed inside the block launch (resident) */
} pgmoe_stats;

/* init_model (core.py:266) + placement (tiers.py:134-157).  max_tokens
 * bounds T for every later call.  Weights are not filled yet. */
PGMOE_API int pgmoe_model_create(const pgmoe_config *cfg, int32_t wdtype, int32_t placement,
                       int32_t max_tokens, pgmoe_model **out);
PGMOE_API int pgmoe_model_destroy(pgmoe_model *m);

/* Expert-parallel shard: same model, but only experts [expert_begin,
 * expert_end) are stored (gates and dense layers are replicated).  Weight
 * seeds use the global expert id, so shards reproduce the single-GPU model. */
PGMOE_API int pgmoe_model_create_ex(const pgmoe_config *cfg, int32_t wdtype, int32_t placement,
                                    int32_t max_tokens, int32_t expert_begin, int32_t expert_end,
                                    pgmoe_model **out);

/* Device base of block `block`'s expert records (W1 then W2 per record). */
PGMOE_API int pgmoe_model_expert_records(pgmoe_model *m, int32_t block, const void **base, size_t *stride,
                                         int32_t *expert_begin, int32_t *n_local);

/* Fill every matrix from the reference generator (device RNG; offloaded
 * experts are generated on the device then copied to pinned host memory). */
PGMOE_API int pgmoe_model_init_weights(pgmoe_model *m);

/* Copy one matrix in from host memory (the BlockParams `loaded` hook,
 * core.py:185-211; model_io.load_model).  name: "gate", "pre_gate", "w1",
 * "w2", "non_moe"; expert = -1 for non-expert matrices.  Host data is in
 * the model's weight dtype, row-major. */
PGMOE_API int pgmoe_model_set_matrix(pgmoe_model *m, const char *name, int32_t block, int32_t expert,
                           const void *host_data, size_t nbytes);
PGMOE_API int pgmoe_model_get_matrix(pgmoe_model *m, const char *name, int32_t block, int32_t expert,
                           void *host_data, size_t nbytes);

/* The model's configuration and weight dtype. */
PGMOE_API int pgmoe_model_config(pgmoe_model *m, pgmoe_config *cfg, int32_t *wdtype);

/* PGMOE1 weight files (model_io.py:1-105): header-only read (no GPU needed),
 * load into a model of matching dimensions (fp32 file -> model dtype, RNE for
 * bf16; expert-parallel shards keep their own experts), and save (fp32).
 * Malformed files return PGMOE_E_WEIGHT_FILE with the reference's messages. */
PGMOE_API int pgmoe_weight_file_config(const char *path, pgmoe_config *out);
PGMOE_API int pgmoe_model_load_pgmoe1(pgmoe_model *m, const char *path);
PGMOE_API int pgmoe_model_save_pgmoe1(pgmoe_model *m, const char *path);

/* Migration strategy of an offloaded model (default pre_gated).  Numerical
 * outputs are identical under every strategy; only the copy schedule and
 * the HBM footprint change (prefetch_all reserves two whole-block slots). */
PGMOE_API int pgmoe_model_set_strategy(pgmoe_model *m, int32_t strategy);

/* HBM expert cache of an offloaded model (cache.py:49-103): policy 0 none,
 * 1 LIFO, 2 LFU, 3 LRU; capacity = fraction of all expert bytes.  Keys are
 * (block, expert); accesses follow each fetch list in order (active experts
 * ascending, or all experts for prefetch_all).  Hits cost an HBM copy
 * instead of a PCIe transfer; outputs are unchanged. */
PGMOE_API int pgmoe_model_set_cache(pgmoe_model *m, int32_t policy, double capacity_fraction);
/* Replays an access sequence through the cache index (no GPU needed):
 * hit[i] and the number of entries access i evicted. */
PGMOE_API int pgmoe_cache_replay(int32_t policy, int32_t capacity_records, const int32_t *blocks,
                                 const int32_t *experts, int32_t n, int32_t *hit, int32_t *n_evicted);

/* Kernel family for K2/K3 (AUTO: tcgen05 for bf16, SIMT for fp32). */
PGMOE_API int pgmoe_model_set_kernel(pgmoe_model *m, int32_t kernel);
/* Resident top-1 decoding computes each block's pre-gate (gate_forward of
 * the next block's decision, core.py:327-329) inside that block's tcgen05
 * launch, overlapped with its expert GEMMs (default on).  0 restores the
 * separate K1 launch; routing and outputs are identical either way. */
PGMOE_API int pgmoe_model_set_fused_route(pgmoe_model *m, int32_t enabled);
/* Resident top-1 decoding at small batches (T <= max_tokens, at most 64):
 * ONE persistent launch per decoder iteration runs every block — expert
 * up/down, combine, dense and the next block's pre-gate — with K split over
 * 8-CTA thread-block clusters and the partials summed in distributed shared
 * memory (decode_tc.cu).  Replaces the per-block launches of
 * decoder_iteration's block loop (core.py:361-380); routing is identical, block
 * outputs equal the per-block path within the bf16 tolerance (different
 * split-K grouping).  enabled = 0 restores the per-block launches; max_tokens
 * = 0 keeps the current threshold (default 1, PGMOE_DECODE_MAX_T). */
PGMOE_API int pgmoe_model_set_decode(pgmoe_model *m, int32_t enabled, int32_t max_tokens);
/* Decoder iterations served by the persistent small-batch launch so far. */
PGMOE_API int64_t pgmoe_model_decode_iterations(pgmoe_model *m);
/* Low-latency small-batch decoder (decode_ll.cu, T <= 8): one persistent
 * launch per decoder iteration whose phases exchange flag-in-word (LL)
 * stores; takes precedence over pgmoe_model_set_decode's kernel for
 * T <= max_tokens.  Same contract as decoder_iteration (core.py:342-383). */
PGMOE_API int pgmoe_model_set_ll_decode(pgmoe_model *m, int32_t enabled, int32_t max_tokens);
PGMOE_API int64_t pgmoe_model_ll_decode_iterations(pgmoe_model *m);
/* Device %globaltimer stamps (ns) of the last resident decoder iteration that
 * ran chained block launches: out[b+1] = when block b's dense layer completed
 * (out[0] unused).  Consecutive differences are the reference's block
 * latencies (scheduler.py:374-397), measured on graph-replayed iterations. */
PGMOE_API int pgmoe_model_block_stamps(pgmoe_model *m, int64_t *out, int32_t n);

/* decoder_iteration (core.py:342-383) for T tokens, device buffers.
 * x_in / y_out: fp32 [T][d] device.  ids_trace / w_trace (optional, device):
 * [num_blocks][T][k] consumed decisions.  Pre-gated migration
 * (scheduler.py:344-373) runs on the model's copy stream when offloaded. */
PGMOE_API int pgmoe_decoder_iteration(pgmoe_model *m, const float *x_in, int32_t T, float *y_out,
                            int32_t *ids_trace, float *w_trace, pgmoe_stream_t stream);

/* Optional inputs / outputs of one decoder iteration (all device, may be NULL):
 *   ids_trace / w_trace  [num_blocks][T][k]  decisions each block consumed
 *   x_trace              [num_blocks][T][d]  each block's input (fp32), for
 *                        teacher-forced parity at the exact launch sequence
 *   ids_supplied / w_supplied [num_blocks][T][k]  supplied decisions
 *                        (core.py:342-364): every block consumes them, no
 *                        gate runs; migration follows the same issue points */
typedef struct {
    int32_t *ids_trace;
    float *w_trace;
    float *x_trace;
    const int32_t *ids_supplied;
    const float *w_supplied;
} pgmoe_iteration_io;

PGMOE_API int pgmoe_decoder_iteration_ex(pgmoe_model *m, const float *x_in, int32_t T, float *y_out,
                                         const pgmoe_iteration_io *io, pgmoe_stream_t stream);

/* Synchronises and surfaces a device-detected routing error of the model's
 * last iterations (GateOverflowError / RoutingError), then clears it. */
PGMOE_API int pgmoe_model_check_routing(pgmoe_model *m);

/* Same call on HOST buffers: copies x in, runs, copies y (and the trace)
 * back, synchronises, and raises device-detected routing errors. */
PGMOE_API int pgmoe_decoder_iteration_host(pgmoe_model *m, const float *x_in, int32_t T, float *y_out,
                                 int32_t *ids_trace, float *w_trace);

/* moe_block_forward (core.py:319-339) for block b on T tokens with the
 * consumed routing `r_in` already on the device; emits routing_out into
 * `r_out` when the block carries a lookahead gate (may be NULL). */
PGMOE_API int pgmoe_moe_block_forward(pgmoe_model *m, int32_t block, const float *x, int32_t T,
                            const pgmoe_routing *r_in, float *y, const pgmoe_routing *r_out,
                            pgmoe_stream_t stream);

/* Device pointers of the model's resident matrices (for the drop-in shim). */
PGMOE_API const void *pgmoe_model_matrix_ptr(pgmoe_model *m, const char *name, int32_t block, int32_t expert);

PGMOE_API int pgmoe_model_stats(pgmoe_model *m, pgmoe_stats *out);
PGMOE_API int pgmoe_model_reset_stats(pgmoe_model *m);

/* Timeline (events since the last set_timeline call) in the reference JSONL schema
 * (scheduler.py:147-156): one line per event, lanes "compute"/"transfer".
 * Writes at most `cap` bytes; returns bytes needed (excluding NUL). */
PGMOE_API int64_t pgmoe_model_timeline_jsonl(pgmoe_model *m, char *buf, int64_t cap);
PGMOE_API int pgmoe_model_set_timeline(pgmoe_model *m, int32_t enabled);

PGMOE_API const char *pgmoe_last_error(void);
PGMOE_API const char *pgmoe_version(void);
/* Kernels this library has launched since load (benchmark evidence). */
PGMOE_API int64_t pgmoe_launch_count(void);
/* Debug only (no reference counterpart): install a device buffer of
 * [rows][16] uint64 that kernels of `kind` (0 route, 1 tcgen05 block kernel)
 * stamp with %globaltimer at fixed points, one row per CTA, consecutive
 * launches taking consecutive rows (wrapping); nullptr disables.  Launches
 * enqueued (or graphs captured) while installed keep writing to it. */
PGMOE_API int pgmoe_debug_set_probe(int32_t kind, void *device_buffer, int64_t rows);
/* Debug only: create a green context of at least `min_sms` SMs on the current
 * device and make it current on the calling thread (persistent kernels size
 * their grid from the current context's SMs); *sms_out = SMs granted. */
PGMOE_API int pgmoe_debug_green_context(int32_t min_sms, int32_t *sms_out);

#ifdef __cplusplus
}
#endif
#endif /* PGMOE_H */
