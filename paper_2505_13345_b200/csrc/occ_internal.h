// occ_internal.h — kernel launchers shared by the C-ABI layer (occ_capi.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace occ {

constexpr int kMaxDev = 64;    // N_d <= 64 (uint64 device masks)
constexpr int kMaxLocal = 64;  // P <= 64 experts per device
constexpr int kRankChunk = 256;
constexpr int kMaxTopK = 64;  // k <= 64 on the device path
constexpr int kBM = 256;       // GEMM pair-tile rows (Epd segments are padded to it)

extern long long g_launches;
inline void count_launch(int n = 1) { g_launches += n; }

// Programmatic dependent launch (PDL) for the layer's chain of kernels: the
// next kernel is launched while its predecessor drains, runs its prologue
// (barrier init, TMEM allocation, descriptor prefetch) and blocks in
// griddepcontrol.wait (pdl_wait in occ_common.cuh) until the predecessor's
// memory is visible.  Only kernels that call pdl_wait() before touching
// dependent data may be launched this way.  OCC_PDL=0 turns it off.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (pdl_enabled()) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- generic stable bucketed rank ("warp-ballot / scan compaction") ----
// Items i < n carry group g_i in [0,G) and a bucket mask m_i (bits < B).
// rank(i, b) = #{i' < i : g_i' = g_i, b in m_i'}; grank(i) = #{i' < i : g_i' = g_i}.
// Phase 1 counts per (chunk, key), phase 2 scans chunks per key, phase 3
// re-derives the in-chunk ranks and hands them to an emitter.
struct RankWs {
    int* chunk_cnt;  // [nchunks][G*(B+1)] -> exclusive bases after phase 2
    int* totals;     // [G*(B+1)]
};

// Dispatch plan (BRIM0 + inbox placement), all sources resident on one GPU
// or (world>1) this rank's tokens only.
struct PlanArgs {
    int n, k, nd, dedup;
    const int32_t* ids;       // [n,k]
    const float* w;           // [n,k]
    const int32_t* sources;   // [n] or null (round robin)
    int src_fixed;            // >=0: all tokens have this source (world>1)
    const int32_t* dev_of;    // [E]
    const int32_t* slot_of;   // [E]
    int E;
    // outputs / workspace
    uint64_t* mask;           // [items]
    int32_t* group;           // [items]
    int32_t* err;             // device error flag
};

void launch_plan_mask(const PlanArgs& a, cudaStream_t st);
void launch_rank_count(int n_items, const int32_t* group, const uint64_t* mask, int G, int B, RankWs ws,
                       cudaStream_t st);
void launch_rank_count_dev(int n_max, const int* n_dev, const int32_t* group, const uint64_t* mask, int G, int B,
                           RankWs ws, cudaStream_t st);
void launch_rank_scan(int n_items, int G, int B, RankWs ws, cudaStream_t st);

// Offsets derived from the dispatch counts (device-side, no host sync).
struct DispatchOffsets {
    int* C;          // [nd*nd] counts (s,d)
    int* off_sd;     // [nd*nd] BRIM0 counter base per (s,d)
    int* inoff;      // [nd*nd] inbox offset of source s within device d (index d*nd+s)
    int* in_base;    // [nd+1]  concatenated inbox base per device (world=1)
    int* nsfd;       // [nd]    Sfd rows per source
    int* src_base;   // [nd+1]  concatenated Sfd base per source
    int* ntok;       // [nd]    tokens per source
    long long* stats;  // [8]: 0 crossing rows, 1 naive crossing, 2 span sum, 3 intra pairs, 4 inter pairs, 5 n_sfd total
};
void launch_dispatch_finalize(int nd, const int* totals, DispatchOffsets o, cudaStream_t st);

struct EmitDispatch {
    int n, k, nd, dedup;
    const int32_t* ids;
    const float* w;
    const int32_t* sources;
    int src_fixed;
    const int32_t* dev_of;
    DispatchOffsets o;
    int world1;              // inbox rows are global (all devices resident)
    int32_t* tok_row;        // [items*nd or items] inbox row per (token,device) / item (world=1)
    int32_t* tok_sfd;        // same shape: BRIM0 counter (Sfd slot within the source)
    int32_t* lam;            // [n] local index of the token within its source (dedup only)
    int32_t* in_tok;         // [R] (world=1)
    int32_t* in_src;
    int32_t* in_slot;
    int32_t* in_dev;
};
void launch_rank_emit_dispatch(int n_items, const int32_t* group, const uint64_t* mask, int G, int B, RankWs ws,
                               const EmitDispatch& e, cudaStream_t st);

// BRIM0 extraction (per source N_d x n_s, concatenated) from tok_sfd.
void launch_extract_brim0(int n, int nd, const int32_t* sources, int src_fixed, const uint64_t* mask,
                          const int32_t* lam, const int32_t* tok_sfd, const int* src_tok_base, int32_t* brim0,
                          cudaStream_t st);

// Pack x rows (and the routing rows) into the inbox / send buffer.
struct PackArgs {
    int n, k, nd, D, dedup;
    const __nv_bfloat16* x;
    const int32_t* ids;
    const float* w;
    const uint64_t* mask;      // dedup: device mask per token
    const int32_t* tok_row;    // dedup [n*nd]; naive [n*k]
    __nv_bfloat16* dst_x;      // rows
    int32_t* dst_ids;          // [rows*k]
    float* dst_w;              // [rows*k]
};
void launch_pack(const PackArgs& a, cudaStream_t st);

// BRIM1 (compute index) over inbox rows.
struct ComputeArgs {
    int R_max;                 // upper bound on inbox rows (grid sizing)
    const int* R_total;        // device: actual rows (world=1: in_base[nd]; world>1: recv total)
    int k, P, G;               // G local devices (world=1: nd; else 1)
    const int32_t* row_ids;    // [R*k] routing ids carried with each row
    const float* row_w;        // [R*k]
    const int32_t* row_dev;    // [R] local device of row (null -> 0)
    const int32_t* dev_of;     // [E]
    const int32_t* slot_of;    // [E]
    int dev_base;              // world>1: global device id of local device 0
    uint64_t* mask;            // [R] out: local slot mask
    int32_t* group;            // [R] out
    int32_t* err;
};
void launch_compute_mask(const ComputeArgs& a, cudaStream_t st);

struct ComputeOffsets {
    int* cnt;          // [G*P] Epd rows per group (local device, slot)
    int* seg_base;     // [G*P] padded Epd base per group
    int* unp_base;     // [G*P] unpadded BRIM1 base per group (within device)
    int* n_mblk;       // [1] total m-blocks
    int* grp_mb;       // [G*P+1] prefix of m-blocks per group (GEMM tile decode)
    int* q_total;      // [1] padded Epd rows
    const int32_t* widx;  // [G*P] weight index of each group
    long long* stats;  // stats[6] += n_epd
};
void launch_compute_finalize(int G, int P, const int* totals, ComputeOffsets o, cudaStream_t st);

struct EmitCompute {
    int k, P, dev_base;
    const int32_t* row_ids;
    const float* row_w;
    const int32_t* slot_of;
    const int32_t* dev_of;
    ComputeOffsets o;
    int32_t* row_epd;     // [R*P] padded Epd row per (row, slot)
    int32_t* epd_src;     // [Q] inbox row feeding each padded Epd row
    float* epd_w;         // [Q] routing weight of each Epd row
    int32_t* epd_j;       // [Q] routing slot (0..k-1) of each Epd row within its row's routing (nullable)
};
void launch_rank_emit_compute(int R_max, const int* R_total, const int32_t* group, const uint64_t* mask, int G,
                              int B, RankWs ws, const EmitCompute& e, cudaStream_t st);
void launch_init_epd(int Q_max, int32_t* epd_src, float* epd_w, cudaStream_t st);


// Epd A operand by scatter: every inbox row read once, written to each of its
// Epd rows (row_epd); padding rows of the NG segments zeroed.  src row of
// inbox row r = src_rows ? src_rows[r] : r.
void launch_scatter_rows(int R_max, const int* R_total, int P, int D, const __nv_bfloat16* src,
                         const int32_t* src_rows, const int32_t* row_epd, int NG, const ComputeOffsets& o,
                         __nv_bfloat16* dst, cudaStream_t st);

// Intra-device partial combine: ret[r] = bf16( sum_{p asc} Y[row_epd[r,p]] ).
void launch_partial_combine(int R_max, const int* R_total, int P, int D, const int32_t* row_epd,
                            const __nv_bfloat16* Y, __nv_bfloat16* ret, cudaStream_t st);
// Final combine: out[t] = bf16( sum_{d asc} ret[row_of(t,d)] ).
// ys (nullable): shared-expert output rows [n, D], added last.
void launch_combine(int n, int nd, int k, int dedup, int D, const uint64_t* mask, const int32_t* tok_row,
                    const __nv_bfloat16* ret, const __nv_bfloat16* ys, __nv_bfloat16* out, cudaStream_t st);

// Stage-level entry points: dispatch of one source from its BRIM0 (N_d x n)
// into Sfd rows, and the combine of returned Sfd rows through BRIM0.
void launch_dispatch_sfd(int n, int nd, int k, int D, const __nv_bfloat16* x, const int32_t* ids, const float* w,
                         const int32_t* brim0, __nv_bfloat16* sfd_x, int32_t* sfd_ids, float* sfd_w, int32_t* sfd_tok,
                         cudaStream_t st);
void launch_combine_brim0(int n, int nd, int D, const int32_t* brim0, const __nv_bfloat16* y, __nv_bfloat16* out,
                          cudaStream_t st);
void launch_set_int(int* p, int v, cudaStream_t st);
// world_size > 1 backward: token gradient (f32 or bf16) and routing-weight
// gradients summed over a token's returned rows (devices ascending).
void launch_combine_back(int n, int nd, int k, int dedup, int D, const uint64_t* mask, const int32_t* tok_row,
                         const __nv_bfloat16* y, const float* ygw, void* gx, int gx_bf16, float* gw, cudaStream_t st);
void launch_brim0_one_source(int n, int nd, const uint64_t* mask, const int32_t* tok_sfd, int32_t* brim0,
                             cudaStream_t st);
void launch_one_source_totals(int nd, int r, int* totals, cudaStream_t st);
// world_size == 1: partial combine + return + combine fused (reads Y once).
void launch_combine_fused(int n, int nd, int k, int P, int dedup, int D, const uint64_t* mask,
                          const int32_t* tok_row, const int32_t* row_epd, const __nv_bfloat16* Y,
                          const __nv_bfloat16* ys, __nv_bfloat16* out, cudaStream_t st);
// Shared experts: per-token weight g[0..n_pad) (sigmoid(x . gate), or 1 when
// gate is null; 0 on the padded rows) and the one-group GEMM tile table
// grp = {0, n_pad / kBM, 0}.
void launch_shared_gate(int n, int n_pad, int D, const __nv_bfloat16* x, const __nv_bfloat16* gate, float* g,
                        int* grp, cudaStream_t st);

// Saved-index extraction (parity): unpadded BRIM1 per device, P x R_d.
void launch_extract_cindex(int R_max, const int* R_total, int P, const int32_t* row_dev, const int* in_base,
                           const int32_t* row_epd, const ComputeOffsets& o, int32_t* cindex, cudaStream_t st);

// Backward (world_size == 1; the upstream rows reach the Epd layout through launch_scatter_rows):
// the scatter-adjoint rows summed back onto tokens, routing-weight gradients.
void launch_combine_grad(int n, int nd, int k, int P, int dedup, int D, const uint64_t* mask, const int32_t* tok_row,
                         const int32_t* row_epd, const __nv_bfloat16* Y, void* out, int out_bf16, cudaStream_t st);
void launch_gw_scatter(int Q_max, const int* q_total, int NB, const float* gw_part, const int32_t* epd_src,
                       const int32_t* in_tok, const int32_t* epd_j, int k, float* g_weights, cudaStream_t st);

// Peer-memory exchange (world_size > 1): every rank's inbox (x, ids, w),
// returned-row buffer, arrival flags and count matrix mapped for every rank;
// peer_tab[p * kPeerSlots + {0 in_x, 1 in_ids, 2 in_w, 3 y_src, 4 flags, 5 counts}].
constexpr int kPeerSlots = 6;
// count all-gather: this source's row of counts into every peer's matrix
void launch_peer_counts(void* const* peer_tab, int nd, int me, const int* totals, cudaStream_t st);
// dispatch: each token row stored straight into every destination's inbox
void launch_peer_pack(const PackArgs& a, int me, const int32_t* dev_of, const int* off_sd, const int* inoff,
                      void* const* peer_tab, cudaStream_t st);
// publish `seq` into flag slot (base + me) of every peer / wait for all peers' `seq` at base..base+nd
// seq: DEVICE pointer to the forward counter (bumped by launch_seq_bump)
void launch_seq_bump(unsigned long long* seq, cudaStream_t st);
void launch_peer_signal(void* const* peer_tab, int nd, int me, int base, const unsigned long long* seq,
                        cudaStream_t st);
void launch_peer_wait(const unsigned long long* flags, int nd, int base, const unsigned long long* seq,
                      long long timeout_ns,
                      int32_t* err, cudaStream_t st);
// intra-device partial combine fused with the return: rows go straight into the sources' buffers
void launch_peer_return(int R_max, const int* R_total, int nd, int me, int P, int D, const int32_t* row_epd,
                        const __nv_bfloat16* Y, const int* C, const int* off_sd, const int* inoff,
                        void* const* peer_tab, cudaStream_t st);

// SimilarityAccumulator::add (pruning.cpp:169-183) on the device: inner [E, E]
// double accumulated in place from one batch of logits (fp64 or fp32 rows).
void launch_similarity_add(const void* logits, int fp64, int n, int e, double* inner, cudaStream_t st);

// Collaboration histogram (K8).
// Bins in shared memory up to kHistSmemMax bytes (E <= 236), global atomics above.
constexpr size_t kHistSmemMax = 220 * 1024;
void launch_histogram(const int32_t* ids, int n, int k, int e, int64_t* counts, cudaStream_t st);

// Comm statistics (spans, pair shares, naive crossings) per token.
void launch_token_stats(int n, int k, int nd, const int32_t* ids, const int32_t* sources, int src_fixed,
                        const int32_t* dev_of, int E, long long* stats, cudaStream_t st);

// Routers.
void launch_gate_scores_f64(const double* x, int n, int d, const double* g, int e, double* s, cudaStream_t st,
                            bool softmax = true);
// Exact router from bf16 operands: fp64 logits (ascending k, no FMA) + the
// glibc-exact softmax (gate_scores, routing.cpp:33-52), scores [n, e] f64.
void launch_gate_scores_bf16_f64(const __nv_bfloat16* x, int n, int d, const __nv_bfloat16* g, int e, double* s,
                                 cudaStream_t st);
void launch_f64_to_f32(const double* a, long n, float* b, cudaStream_t st);
void launch_topk_f64(const double* s, int n, int e, int k, int renorm, int32_t* ids, double* w, int32_t* err,
                     cudaStream_t st);
struct PruneDev {
    int mode, budget, own_score, renorm, nd;
    const int32_t* dev_of;   // [E]
    const int32_t* ranking;  // [E*(E-1)] or null
};
void launch_prune_f64(const double* s, int n, int e, int k, const int32_t* ids_in, const double* w_in, PruneDev p,
                      int32_t* ids, double* w, int32_t* err, cudaStream_t st);
// Tensor-core router (occ_router.cu): returns false when the shape needs the
// logits path (E > 128 without logits_out, or k > 64).
// prune (nullable): router-score pruning (mode 1) runs in the epilogue;
// err receives CapacityError (5).
struct PruneDev;
bool launch_router_tc(const void* tmap_x, const void* tmap_g, int n, int d, int e, int k, int renorm, int32_t* ids,
                      float* w, float* logits_out, int num_sms, cudaStream_t st, const PruneDev* prune = nullptr,
                      int32_t* err = nullptr);
void launch_router_select(float* logits, int n, int e, int k, int renorm, PruneDev p, int32_t* ids, float* w,
                          float* scores, int32_t* err, cudaStream_t st);

// Weight layout conversion: reference [E, K, N] row-major -> K-major [E, N, K]
// (optionally interleaving w1/w3 in 128-column blocks for SwiGLU).
void launch_transpose_weights(const __nv_bfloat16* w, int E, int K, int N, __nv_bfloat16* out, int out_rows_per_e,
                              int interleave_half, cudaStream_t st, int pitch = 0);

// The whole one-GPU index chain in one cooperative kernel (occ_plan.cu):
// BRIM0 + inbox records + routing rows + BRIM1 + Epd A operand + CommReport
// counters.  world_size == 1, dedup, k <= 32, tables within 96 KB of shared memory.
struct FusedPlanArgs {
    int n, k, nd, E, P, D;
    const int32_t* ids;
    const float* w;
    const int32_t* sources;  // null: round robin
    const int32_t* dev_of;
    const int32_t* slot_of;
    const __nv_bfloat16* x;
    int* chunk_cnt;          // [K * nchunks], K = nd(nd+1) + nd E
    int* totals;             // [K]
    DispatchOffsets dofs;
    int* tok_base;           // [nd] prefix of tokens per source
    ComputeOffsets cofs;
    uint64_t* mask;          // [n] destination-device mask per token
    int32_t *tok_row, *tok_sfd, *lam, *in_tok, *in_src, *in_slot, *in_dev, *in_ids;
    float* in_w;
    int32_t *row_epd, *epd_src, *epd_j;
    float* epd_w;
    __nv_bfloat16* x_epd;    // null: no A-operand copy (TMA gather path)
    long long* stats;
    int32_t* err;
    int scatter = 1;         // copy the Epd A rows in the kernel (else the caller runs launch_scatter_rows)
    int zero_stats = 0;      // stats[0..7] zeroed in the kernel (no memset node before it)
    unsigned long long* dbg = nullptr;  // OCC_PLAN_DEBUG phase timeline
};
bool fused_plan_supported(int nd, int E, int k);
size_t fused_plan_chunks(int n, int k);            // rank chunks of n tokens
size_t fused_plan_ws(int n, int nd, int E, int k);  // chunk_cnt + totals ints
bool launch_fused_plan(const FusedPlanArgs& a, int num_sms, cudaStream_t st);

// Grouped GEMM on tcgen05 (occ_gemm.cu).
enum EpiMode {
    EPI_ACT_BF16 = 0,    // forward GEMM-1: act(acc) * w -> bf16 (+ pre-activation when training)
    EPI_SWIGLU_BF16 = 1, // forward GEMM-1: silu(a) * b * w -> bf16 (+ a, b when training)
    EPI_F32 = 2,         // plain fp32 output (GEMM-2, data gradient of the scatter)
    EPI_BWD_ACT = 3,     // data gradient of the merge + modulation/activation adjoints
    EPI_BWD_SWIGLU = 4,  // same for SwiGLU: g_a | g_b
    EPI_WGRAD = 5        // per-expert weight gradient (MN-major operands, K = the expert's rows)
};
struct GemmArgs {
    const void* tmap_a = nullptr;  // CUtensorMap* (host object, passed by value to the kernel)
    const void* tmap_b = nullptr;
    const void* tmap_c = nullptr;
    const int* a_rows = nullptr;   // gathered A: row of tmap_a (box 64 x 1) for each padded Epd row, -1 = zero  // bf16 forward output [rows, ldo] (box 32 x 32, 64 B swizzle): TMA-store epilogue
    int K = 0;                     // reduction dim (forward / data gradient)
    int N = 0;                     // output columns per expert (GEMM-1 SwiGLU: F; B rows per expert = 2F)
    int b_rows_per_e = 0;          // rows of B per expert in the stacked K-major weight matrix
    const int* grp_mb = nullptr;   // device [ngroups+1]: pair-tile prefix per expert group
    const int* grp_w = nullptr;    // device [ngroups]: weight index of each group
    int ngroups = 0;
    int band = 1 << 20;            // pair tiles per raster band inside a group
    const int* grp_cnt = nullptr;  // wgrad: rows per group
    const int* seg_base = nullptr; // wgrad: first padded row per group
    int M = 0;                     // wgrad: output rows
    const float* row_w = nullptr;  // per padded Epd row routing weight, null = 1
    void* out = nullptr;           // [Q, N] bf16 / f32, or wgrad [E, M, ldo] f32
    int ldo = 0;                   // output row stride (elements)
    long out_estride = 0;          // wgrad: elements per expert
    void* out2 = nullptr;          // wgrad: columns >= split go here (SwiGLU w3 gradient)
    int split = 1 << 30;
    int act = 0;                   // occ_activation
    __nv_bfloat16* save_a = nullptr;  // forward training outputs
    __nv_bfloat16* save_b = nullptr;
    const __nv_bfloat16* pre_a = nullptr;  // backward epilogue inputs
    const __nv_bfloat16* pre_b = nullptr;
    float* gw_part = nullptr;      // backward: routing-weight gradient partial per (row, n-tile)
    int max_tiles = 0;             // static upper bound (grid sizing)
    int* sched = nullptr;          // dynamic tile scheduler slot (2 zeroed ints; null = static schedule)
};
// Scheduler slots per handle (launch sites that can run concurrently get their own).
enum SchedSlot { SCHED_GEMM1 = 0, SCHED_GEMM2, SCHED_SHARED1, SCHED_SHARED2, SCHED_BWD0, kSchedSlots = 16 };
void launch_grouped_gemm(EpiMode mode, const GemmArgs& a, int num_sms, cudaStream_t st);
bool make_tmap_2d(void* tmap, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                  uint32_t box_outer, int swizzle_bytes = 128, uint64_t pitch_elems = 0);
// Output map of the TMA-store epilogue: bf16 [outer, inner] row-major, 32 x 32 boxes.
inline bool make_tmap_out(void* tmap, const void* base, uint64_t inner, uint64_t outer) {
    return make_tmap_2d(tmap, base, inner, outer, 32, 32, 64);
}

}  // namespace occ
