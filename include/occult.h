/*
 * occult.h — C-ABI of the B200-native Occult expert-parallel MoE layer.
 *
 * Drop-in boundary for the reference's C++ library API (moesim, namespace
 * `moesim`; /root/reference/proj/include/moesim/ headers).  Every entry point
 * below names the reference interface it replaces.  The reference is a
 * header-level C++ library with value semantics and exceptions; this ABI is
 * plain C: device buffers are caller-owned raw pointers, every call is
 * ordered on the caller's CUDA stream, and errors are returned as
 * `occ_status` values that map 1:1 onto the reference's exception taxonomy
 * (common.hpp:11-34).  Nothing throws across the ABI.
 *
 * Layout conventions (row-major everywhere, like moesim::Matrix):
 *   tokens   x       [n, D]       bf16
 *   routing  ids     [n, k]       int32, weights [n, k] f32 (f64 for *_f64)
 *   experts  w1, w3  [E_l, D, F]  bf16  (reference ExpertWeights::w1, D x H)
 *            w2      [E_l, F, D]  bf16  (reference ExpertWeights::w2, H x D)
 *   placement        [N_d, P]     int32, P = E / N_d, list order significant
 *                                 (reference Placement::devices)
 *
 * One handle per GPU.  A handle with world_size == 1 hosts all N_d logical
 * EP devices on one GPU exactly as the reference simulates them in one
 * process (pipeline.cpp:393-466); with world_size == N_d each rank is one
 * EP device and the two exchanges run over NCCL.  Handles are not
 * thread-safe, and one handle's work must be ordered on one stream at a time
 * (its workspaces -- including the grouped GEMMs' tile counters -- are
 * reused by every call; use one handle per concurrent stream).
 */
#ifndef OCCULT_H
#define OCCULT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* occ_stream_t; /* == cudaStream_t */

/* Status codes; 1..6 mirror moesim::{Shape,Config,Placement,Routing,
 * Capacity,State}Error (common.hpp:11-28). */
typedef enum {
    OCC_OK = 0,
    OCC_ERR_SHAPE = 1,
    OCC_ERR_CONFIG = 2,
    OCC_ERR_PLACEMENT = 3,
    OCC_ERR_ROUTING = 4,
    OCC_ERR_CAPACITY = 5,
    OCC_ERR_STATE = 6,
    OCC_ERR_CUDA = 10,
    OCC_ERR_NCCL = 11,
    OCC_ERR_ARG = 12,
    OCC_ERR_UNSUPPORTED = 13
} occ_status;

/* moesim::Activation (config.hpp:10) + the gated SwiGLU extension
 * (silu(x w1) * (x w3); not in the reference). */
typedef enum { OCC_ACT_IDENTITY = 0, OCC_ACT_SILU = 1, OCC_ACT_RELU = 2, OCC_ACT_SWIGLU = 3 } occ_activation;

/* moesim::PruneMode / ReplacementWeightPolicy (pruning.hpp:14-18). */
typedef enum { OCC_PRUNE_NONE = 0, OCC_PRUNE_ROUTER = 1, OCC_PRUNE_SIMILARITY = 2 } occ_prune_mode;

/* Router / layer config — replaces moesim::MoEConfig (config.hpp:12-28). */
typedef struct {
    int num_experts;  /* E */
    int top_k;        /* k */
    int num_devices;  /* N_d: EP degree (logical devices) */
    int embed_dim;    /* D */
    int hidden_dim;   /* F (reference: H) */
    int renormalize;  /* renormalise top-k weights (MoEConfig::renormalize) */
    int activation;   /* occ_activation */
    int dedup;        /* 1: Occult dispatch, one copy per (token, device);
                         0: naive replicate-k baseline, one copy per (token, expert) */
} occ_config;

/* Pruning knob — replaces moesim::PruneSpec (pruning.hpp:32-39).  The
 * similarity table is attached separately (occ_set_similarity). */
typedef struct {
    int mode;          /* occ_prune_mode */
    int device_budget; /* max devices a token's experts may span */
    int own_score;     /* 1: ReplacementWeightPolicy::OwnScore, 0: Inherit */
} occ_prune;

/* Communication accounting — replaces moesim::CommReport (collab.hpp:36-43)
 * for the last occ_forward call, plus the naive top-k comparison. */
typedef struct {
    double mean_replicas;             /* E(C_T): mean per-token device span */
    double cap_replicas;              /* min(k, N_d) or the prune budget */
    double intra_share, inter_share;  /* co-activated pair shares */
    long long cross_device_bytes;     /* dispatch rows crossing devices x D x bytes_per_scalar */
    long long crossing_rows;          /* Occult (dedup) rows leaving their source device */
    long long naive_crossing_rows;    /* replicate-k rows that would leave their source */
    long long n_sfd;                  /* total Sfd rows (sum over sources) */
    long long n_epd;                  /* total Epd rows */
    long long per_device_rows[64];    /* Sfd rows received per device (CommReport::per_device_token_counts) */
} occ_comm_report;

typedef struct occ_handle occ_handle;

/* ------------------------------------------------------------ lifecycle */
/* Validates like MoEConfig::validate (core.cpp:10-23) + Placement::validate
 * (placement.cpp:32-45).  placement is a HOST pointer [N_d * P]. */
occ_status occ_create(const occ_config* cfg, const int32_t* placement, int world_size, int rank, occ_handle** out);
occ_status occ_destroy(occ_handle* h);
/* Replace the expert-placement table (e.g. after occ_reschedule_placement).
 * Must be followed by occ_load_experts. HOST pointer. */
occ_status occ_set_placement(occ_handle* h, const int32_t* placement);
/* Resident expert weights, reference layout (token.hpp:30-44), DEVICE
 * pointers.  world_size == 1: all E experts in expert-id order.
 * world_size > 1: this rank's P local experts in placement-list order.
 * w3 is required iff activation == OCC_ACT_SWIGLU, else NULL. */
occ_status occ_load_experts(occ_handle* h, const void* w1, const void* w3, const void* w2, occ_stream_t stream);
/* Shared (always-active) experts of DeepSeek-MoE / Qwen-MoE layers
 * (BASELINE configs 3 and 5).  Not in the reference
 * (SPEC.md:9): the layer output becomes
 *     out[t] = bf16( sum_d return_d[t] + bf16(g_t * sum_s FFN_s(x[t])) )
 * with FFN_s the same expert type as the routed experts (SwiGLU or the
 * 2-matrix act expert) and g_t = sigmoid(x[t] . gate) when `gate` is given
 * (Qwen's shared_expert_gate) or 1.  Shared experts run on every token's
 * SOURCE device — no all-to-all — as one dense FFN of width
 * num_shared * d_ff_shared (the S experts stacked along the hidden dim,
 * which sums their outputs).  Restated in oracle/occ_oracle.c
 * (orc_shared_experts).  DEVICE pointers, reference layout:
 *   w1, w3 [S, D, F_s] bf16 (w3 iff SwiGLU), w2 [S, F_s, D] bf16,
 *   gate [D] bf16 or NULL.  num_shared = 0 detaches them. */
occ_status occ_load_shared_experts(occ_handle* h, int num_shared, int d_ff_shared, const void* w1, const void* w3,
                                   const void* w2, const void* gate, occ_stream_t stream);
/* Similarity profiling (SimilarityAccumulator, pruning.cpp:165-219):
 * occ_similarity_accumulate adds one batch of router logits [n, e] (DEVICE,
 * fp64 when logits_fp64, else f32) into the [e, e] DEVICE double Gram
 * `inner` (zero it first); bit-exact with the reference for fp64 logits.
 * occ_similarity_finalize turns a HOST copy of `inner` and the token count
 * into the squared-cosine values (HOST) for occ_set_similarity.
 * occ_router_logits writes the production router's f32 logits x g^T. */
occ_status occ_similarity_accumulate(const void* logits, int logits_fp64, int n, int e, double* inner,
                                     occ_stream_t stream);
occ_status occ_similarity_finalize(const double* inner, long long tokens, int e, double* values);
occ_status occ_router_logits(occ_handle* h, const void* x, const void* gate, int n, float* logits,
                             occ_stream_t stream);
/* Squared-cosine similarity table (SimilarityTable::values, pruning.hpp:25-30),
 * HOST pointer [E * E]; the per-expert ranking is built as the reference does. */
occ_status occ_set_similarity(occ_handle* h, const double* values);

/* Validation (default on): synchronise at the end of occ_route/occ_forward
 * and report RoutingError/CapacityError/ShapeError found on the device.
 * Off: fully asynchronous and CUDA-graph capturable. */
occ_status occ_set_validate(occ_handle* h, int on);

/* NCCL plumbing for world_size > 1 (one process per GPU). */
occ_status occ_comm_unique_id(void* id128);
occ_status occ_comm_init(occ_handle* h, const void* id128);
/* Transport over a caller-supplied host all-gather (ranks in separate
 * processes, no NCCL): fn(ctx, send, bytes, recv) must gather `bytes` from
 * every rank into recv [world_size * bytes] in rank order and return 0; it is
 * called collectively, in the same order on every rank (e.g. over
 * torch.distributed / gloo, MPI).  It bootstraps the CUDA IPC mapping of
 * occ_comm_enable_peer (which then carries the whole forward with no host
 * involvement; this also works for several processes sharing one GPU, which
 * NCCL refuses) and runs the remaining exchanges (backward, non-peer
 * forward, histogram all-reduce) through host staging. */
typedef int (*occ_host_allgather_fn)(void* ctx, const void* send, size_t bytes, void* recv);
occ_status occ_comm_init_host(occ_handle* h, occ_host_allgather_fn fn, void* ctx);
/* Validation transport: the world_size ranks are host threads of ONE process
 * sharing one GPU (each with its own handle and stream); the exchanges become
 * device-to-device copies between the ranks' buffers.  Same layer code path
 * as NCCL, for checking world_size > 1 on a single GPU. */
occ_status occ_comm_init_loopback(occ_handle* h, long group_key);

/* Fused exchange over peer memory (collective; call on every rank after
 * occ_comm_init / occ_comm_init_loopback): each rank's inbox and
 * returned-row buffers are mapped into every rank (CUDA IPC over NVLink /
 * NVSwitch; plain pointers for loopback ranks), and the dispatch pack and the
 * return partial combine store straight into the peers' buffers, with
 * arrival flags instead of all-to-all calls.  Buffers are sized for
 * max_tokens_per_rank tokens per forward (larger batches: OCC_ERR_SHAPE). */
occ_status occ_comm_enable_peer(occ_handle* h, int max_tokens_per_rank);
/* Compute/communication overlap: every forward runs as two
 * micro-batches, tokens [0, ceil(n/2)) on this handle and the rest on an
 * internal sibling handle (its own workspace and communicator — ncclCommSplit
 * — the same resident weights) on a second stream, so one half's dispatch /
 * return exchange overlaps the other half's expert GEMMs; outputs are
 * identical to the unsplit forward (rows are independent given routing) and
 * the CommReport covers both halves. The GEMMs leave comm_sms SMs to the other
 * half's exchange kernels (-1: 16 when world_size > 1, else 0).
 * micro_batches 1 or 2. Collective when world_size > 1 (every rank, after
 * occ_comm_init / occ_comm_enable_peer). Inference only; occ_saved_index
 * refuses a micro-batched forward. */
occ_status occ_set_micro_batches(occ_handle* h, int micro_batches, int comm_sms);

/* -------------------------------------------------------------- routing */
/* gate_scores (routing.cpp:33-52), exact fp64 mode: logits accumulated
 * sequentially in ascending k without FMA, softmax with max subtraction. */
occ_status occ_gate_scores_f64(const double* x, int n, int d, const double* gate, int e, double* scores,
                               occ_stream_t stream);
/* The router logits x @ gate^T of gate_scores before the softmax
 * (tiled_matmul in Precision::Double, matrix.cpp:9-38, k ascending): the
 * similarity-table profiling input of the simulate driver (cli.cpp:296-299). */
occ_status occ_gate_logits_f64(const double* x, int n, int d, const double* gate, int e, double* logits,
                               occ_stream_t stream);
/* topk_route (routing.cpp:60-84): (score desc, index asc), optional
 * renormalisation; bit-exact with the reference. */
occ_status occ_topk_route_f64(const double* scores, int n, int e, int k, int renormalize, int32_t* ids,
                              double* weights, occ_stream_t stream);
/* prune_routing (pruning.cpp:141-163) on fp64 scores; bit-exact.
 * Per-token CapacityError is reported through the return status. */
occ_status occ_prune_routing_f64(occ_handle* h, const double* scores, const int32_t* ids_in, const double* w_in,
                                 int n, const occ_prune* prune, int32_t* ids, double* weights, occ_stream_t stream);
/* Router arithmetic of occ_route / occ_forward_expert_parallel / occ_forward_host:
 *   OCC_ROUTER_TC (default): x g^T on tcgen05 tensor cores (bf16 operands, f32
 *     accumulation) with softmax / top-k / router-score pruning fused in the
 *     epilogue: the fast path, equal to the reference except where two
 *     reference scores are within f32 rounding of each other (declared
 *     tolerance: < 1% of tokens, only at near-ties);
 *   OCC_ROUTER_EXACT: the reference's arithmetic (occ_route_exact), bit-exact
 *     ids and weights; the layer then uses the weights rounded to f32. */
typedef enum { OCC_ROUTER_TC = 0, OCC_ROUTER_EXACT = 1 } occ_router_mode;
occ_status occ_set_router_mode(occ_handle* h, int mode);
/* gate_scores -> topk_route -> prune_routing exactly as forward_expert_parallel
 * (pipeline.cpp:509-512; routing.cpp:33-84; pruning.cpp:141-163) on the bf16
 * tokens x [n, D] and gate [E, D] widened to double: logits summed in
 * ascending k without FMA, softmax with glibc's exp (bit for bit), fp64
 * top-k / renormalisation / pruning.  ids [n, k] int32, weights [n, k] f64,
 * scores (nullable) [n, E] f64 softmax rows; all bit-exact with the
 * reference.  prune may be NULL. */
occ_status occ_route_exact(occ_handle* h, const void* x, const void* gate, int n, const occ_prune* prune, int32_t* ids,
                           double* weights, double* scores, occ_stream_t stream);
/* Production router (forward_expert_parallel's routing stage,
 * pipeline.cpp:509-512): logits = x g^T (bf16 in, f32 accumulate),
 * softmax, top-k, renormalise, optional pruning (prune may be NULL).
 * scores (nullable, [n, E] f32) receives the softmax rows. */
occ_status occ_route(occ_handle* h, const void* x, const void* gate, int n, const occ_prune* prune, int32_t* ids,
                     float* weights, float* scores, occ_stream_t stream);

/* ------------------------------------------------------------- EP path */
/* build_dispatch_index (pipeline.cpp:24-50).
 * world_size == 1: every source at once; sources: [n] device of each token
 * (NULL = round_robin_sources, pipeline.cpp:12-16); brim0 (nullable):
 * concatenation over sources s of the N_d x n_s BRIM0 matrices; counts
 * (nullable): [N_d * N_d] Sfd rows per (source, destination).
 * world_size > 1: the n tokens are this rank's (source = rank, sources
 * ignored); brim0 [N_d x n], counts [N_d] (this source's row). */
occ_status occ_build_dispatch(occ_handle* h, const int32_t* ids, const int32_t* sources, int n, int32_t* brim0,
                              int32_t* counts, occ_stream_t stream);

/* ------------------------------------------- stage-level entry points ---
 * The reference's data path one stage at a time (pipeline.hpp:89-123), for a
 * caller that runs its own exchange between the stages (e.g. its NCCL
 * all-to-all with the layout of occ_exchange_layout).  Stream-ordered, no
 * host synchronisation unless validation is on; chaining
 *   occ_build_dispatch -> occ_dispatch -> (exchange) -> occ_expert_compute
 *   -> (return exchange) -> occ_combine
 * gives occ_forward's output bit for bit.  `device` is the EP device whose
 * experts run: [0, N_d) on a world_size 1 handle, this rank otherwise. */
/* dispatch (pipeline.cpp:91-123) of one source's n tokens by its BRIM0
 * [N_d x n]: Sfd row c = BRIM0[d, i] >= 0 receives x row i [D] bf16, the
 * routing row (ids [k] int32, weights [k] f32) and sfd_token[c] = i.  Rows for
 * destination d are contiguous (device-major counters). */
occ_status occ_dispatch(occ_handle* h, const void* x, const int32_t* ids, const float* weights, int n,
                        const int32_t* brim0, void* sfd_x, int32_t* sfd_ids, float* sfd_weights, int32_t* sfd_token,
                        occ_stream_t stream);
/* build_compute_index (pipeline.cpp:52-89) over the `rows` inbox rows of EP
 * device `device` (their routing rows in_ids [rows, k], in_weights [rows, k]):
 * cindex [P x rows] int32 (nullable), n_epd (nullable, DEVICE int32).  A row
 * with no local expert or an invalid id: RoutingError (validation on). */
occ_status occ_build_compute(occ_handle* h, int device, const int32_t* in_ids, const float* in_weights, int rows,
                             int32_t* cindex, int32_t* n_epd, occ_stream_t stream);
/* scatter_matmul -> apply_activation -> weight_modulate -> merge_matmul
 * (pipeline.cpp:178-283) of EP device `device` over its inbox rows
 * (in_x [rows, D] bf16 + routing rows): y_out [rows, D] bf16, row r = the
 * intra-device partial combine sum over the row's local experts in
 * placement-list order (fp32 accumulation, one bf16 rounding: the return
 * payload).  Grouped GEMMs on tcgen05 as in occ_forward. */
occ_status occ_expert_compute(occ_handle* h, int device, const void* in_x, const int32_t* in_ids,
                              const float* in_weights, int rows, void* y_out, occ_stream_t stream);
/* combine (pipeline.cpp:285-300) of one source: out[i] = bf16( sum over
 * devices d ascending of y_returned[BRIM0[d, i]] ), fp32 accumulation;
 * y_returned [n_sfd, D] bf16 in Sfd order, brim0 [N_d x n]. */
occ_status occ_combine(occ_handle* h, const void* y_returned, const int32_t* brim0, int n, void* out,
                       occ_stream_t stream);
/* forward_given_routing (pipeline.cpp:360-501): dispatch -> exchange ->
 * grouped expert FFN -> intra-device partial combine -> return exchange ->
 * combine.  world_size == 1: x/out hold all n tokens, sources as above.
 * world_size > 1: x/out hold this rank's n tokens (sources ignored). */
occ_status occ_forward(occ_handle* h, const void* x, const int32_t* ids, const float* weights,
                       const int32_t* sources, int n, void* out, occ_stream_t stream);
/* forward_expert_parallel (pipeline.cpp:503-517): occ_route + occ_forward. */
occ_status occ_forward_expert_parallel(occ_handle* h, const void* x, const void* gate, const occ_prune* prune,
                                       const int32_t* sources, int n, void* out, occ_stream_t stream);
/* forward_expert_parallel end to end from pinned HOST memory: x_host and
 * out_host are [n, D] bf16 host buffers (pinned for overlap), gate is a
 * DEVICE pointer.  Asynchronous and double-buffered: the host->device copy
 * of this call and the device->host copy of the previous one overlap the
 * layer, on two copy streams owned by the handle; the batch may further be
 * cut into `chunks` token chunks (rows are independent given routing,
 * pipeline.cpp:548-560).  x_host must stay unchanged, and out_host may only
 * be read, after occ_host_wait has been ordered on a stream and that stream
 * has completed. */
occ_status occ_forward_host(occ_handle* h, const void* x_host, const void* gate, const occ_prune* prune, int n,
                            void* out_host, int chunks, occ_stream_t stream);
/* Make `stream` wait until every enqueued occ_forward_host result is in host memory. */
occ_status occ_host_wait(occ_handle* h, occ_stream_t stream);
/* Training: keep the pre-activations and the reference-orientation weights
 * so occ_backward can follow the next forward (call before occ_load_experts).
 * world_size 1 in this build. */
occ_status occ_set_training(occ_handle* h, int on);
/* backward_vjps (backward.cpp:24-161) for the last occ_forward: routing ids
 * held fixed, gradients for tokens, expert weights and routing weights.
 *   upstream  [n, D] bf16 (d loss / d out)
 *   g_x       [n, D] f32;  g_w1, g_w3 [E_l, D, F] f32 (g_w3 only for SwiGLU);
 *   g_w2      [E_l, F, D] f32;  g_weights [n, k] f32, aligned with the routing.
 * StateError if the forward was not run with occ_set_training(h, 1). */
occ_status occ_backward(occ_handle* h, const void* upstream, float* g_x, float* g_w1, float* g_w3, float* g_w2,
                        float* g_weights, occ_stream_t stream);
/* Token gradient dtype of occ_backward: 0 (default) f32, 1 bf16 (g_x then
 * points to [n, D] bf16; mixed-precision training halves its size). */
occ_status occ_set_grad_x_bf16(occ_handle* h, int on);
/* CommReport of the last forward (synchronises the stream).
 * bytes_per_scalar as in forward_given_routing's argument. */
occ_status occ_comm_report_get(occ_handle* h, int bytes_per_scalar, occ_comm_report* rep, occ_stream_t stream);
/* Saved index state of the last forward (ForwardState, pipeline.hpp:155-165),
 * DEVICE pointers, each nullable:
 *   inbox_token/source/slot [sum_d R_d]  (DeviceInbox::token/source/source_slot)
 *   cindex [sum_d P x R_d]                (ShardRecord::cindex, BRIM1, unpadded counters) */
occ_status occ_saved_index(occ_handle* h, int32_t* inbox_token, int32_t* inbox_source, int32_t* inbox_slot,
                           int32_t* cindex, occ_stream_t stream);

/* ----------------------------------------------- collaboration profiling */
/* accumulate_collab (collab.cpp:10-23): counts [E, E] int64 DEVICE buffer,
 * accumulated in place. */
occ_status occ_coactivation_histogram(const int32_t* ids, int n, int k, int e, int64_t* counts, occ_stream_t stream);
/* normalize_graph (collab.cpp:31-39), HOST buffers. */
occ_status occ_normalize_graph(const int64_t* counts, int e, double* p);
/* reschedule_placement (placement.cpp:88-148, Alg. 1), HOST buffers; bit-exact. */
occ_status occ_reschedule_placement(const double* p, int e, int num_devices, int32_t* placement);
/* Sum the histogram across ranks (world_size > 1; ncclAllReduce). */
occ_status occ_allreduce_histogram(occ_handle* h, int64_t* counts, occ_stream_t stream);
/* Index-chain implementation of the one-GPU forward (world_size 1, dedup,
 * E <= 64, k <= 8): 1 (default) = one cooperative kernel for BRIM0, the
 * inbox records, BRIM1, the Epd A operand and the CommReport counters
 * (occ_plan.cu); 0 = the multi-kernel chain.  Identical results. */
occ_status occ_set_plan_kernels(occ_handle* h, int fused);

/* Stage profiling with CUDA events on the launching stream (default off).
 * occ_stage_ms fills ms[0..10) for the last occ_forward_expert_parallel /
 * occ_forward: route, plan, pack, compute_index, gather, gemm1, gemm2,
 * shared, partial_combine, combine (ms < 0: stage not recorded); returns
 * the count. */
occ_status occ_set_profiling(occ_handle* h, int on);
int occ_stage_ms(occ_handle* h, float* ms, int max_stages);

/* Host-side layout of the dispatch/return all-to-alls for EP rank `rank`
 * from the all-gathered (source, destination) Sfd row counts C [nd * nd]
 * (row s = source s): per peer p, where this rank's rows for p start in its
 * device-major Sfd batch and how many there are, and where the rows from
 * p land in this device's (source asc, counter asc) inbox
 * (all_to_all_exchange, pipeline.cpp:125-176).  HOST buffers. */
occ_status occ_exchange_layout(const int32_t* C, int nd, int rank, int64_t* send_off, int64_t* send_cnt,
                               int64_t* recv_off, int64_t* recv_cnt);

/* Human-readable message of the last error on this thread. */
const char* occ_last_error(void);
/* Kernel launches issued by this process so far (for launch accounting). */
long long occ_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* OCCULT_H */
