// occ_capi.cu — the C-ABI (include/occult.h): handle, workspace, stage
// entry points and the fused end-to-end forward.
//
// Per forward (world_size == 1, all N_d logical devices on this GPU, the
// reference's single-process simulation made real):
//   plan_mask -> rank(count, scan) -> dispatch_finalize -> rank(emit)    BRIM0, inbox slots
//   pack                                                                  dispatch + exchange placement
//   compute_mask -> rank(count, scan) -> compute_finalize -> rank(emit)   BRIM1, Epd segments
//   gather -> grouped GEMM-1 (tcgen05, act/SwiGLU x routing weight)       scatter_matmul+act+modulate
//   grouped GEMM-2 (tcgen05, fp32)                                        merge_matmul products
//   partial_combine (intra-device, placement order)                       merge_matmul sum
//   combine (devices ascending)                                           return exchange + combine
// Everything is stream-ordered with device-side counts: no host sync
// unless validation is on (the default; occ_set_validate(h, 0) for
// capture/benchmarks).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/occult.h"
#include "occ_internal.h"

using namespace occ;

namespace {

thread_local std::string g_err;

occ_status fail(occ_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define NCCL_TRY(x)                                                                        \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess) return fail(OCC_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

#define CUDA_TRY(x)                                                                        \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) return fail(OCC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Bumped whenever any device buffer is (re)allocated or freed: captured
// CUDA graphs hold raw pointers and are re-captured when it moves.
long long g_buf_gen = 0;

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t count) {
        if (count <= n && p) return cudaSuccess;
        ++g_buf_gen;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) n = count;
        return e;
    }
    void release() {
        if (p) ++g_buf_gen;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace

// Stage boundaries recorded by occ_forward_expert_parallel / occ_forward.
enum Stage { ST_ROUTE = 0, ST_PLAN, ST_PACK, ST_CINDEX, ST_GATHER, ST_GEMM1, ST_GEMM2, ST_SHARED, ST_PCOMBINE, ST_COMBINE,
             kStages };

// ------------------------------------------------------------ transport --
// The two exchanges of the EP layer are an all-gather of the per-source
// count rows and variable-size all-to-alls.  NcclTransport is the product
// multi-GPU path (NVLink/NVSwitch); LoopbackTransport runs N ranks as host
// threads on ONE GPU (device-to-device copies between the ranks' buffers) so
// the world_size > 1 code path can be validated on a single B200.
struct Transport {
    virtual ~Transport() {}
    virtual const char* name() const = 0;
    // send: this rank's nd ints (device); recv: nd x nd ints (device), row s = rank s
    virtual occ_status allgather_counts(const int* send, int* recv, int nd, cudaStream_t st) = 0;
    // variable all-to-all in elements of `es` bytes; offsets/counts in elements per peer
    virtual occ_status alltoallv(const void* send, const std::vector<size_t>& soff, const std::vector<size_t>& scnt,
                                 void* recv, const std::vector<size_t>& roff, const std::vector<size_t>& rcnt, int es,
                                 cudaStream_t st) = 0;
    virtual occ_status allreduce_i64(int64_t* buf, size_t count, cudaStream_t st) = 0;
    // host-level barrier of all ranks (collective set-up calls end with one so
    // no rank starts a forward -- whose peer arrival waits spin on the device --
    // while another is still allocating)
    virtual occ_status barrier() = 0;
    // peer-memory mapping: every rank's `mine` device pointers, usable by this
    // rank (world x mine.size(), row p = rank p); opened mappings are returned
    // in `opened` for release
    virtual occ_status exchange_pointers(const std::vector<void*>& mine, std::vector<void*>& all,
                                         std::vector<void*>& opened) = 0;
    // a second, independent channel between the same ranks (collective: every
    // rank calls it once, in the same order)
    virtual occ_status split(Transport** out) = 0;
    // several all-to-alls with the same row layout (element sizes es[i]) as one exchange
    struct Part {
        const void* send;
        void* recv;
        int es;
    };
    virtual occ_status alltoallv_parts(const std::vector<Part>& parts, const std::vector<size_t>& soff,
                                       const std::vector<size_t>& scnt, const std::vector<size_t>& roff,
                                       const std::vector<size_t>& rcnt, cudaStream_t st) {
        for (const Part& pt : parts) {
            occ_status s = alltoallv(pt.send, soff, scnt, pt.recv, roff, rcnt, pt.es, st);
            if (s != OCC_OK) return s;
        }
        return OCC_OK;
    }
};

struct alignas(64) TmapBox {
    alignas(64) unsigned char bytes[128];
};

struct occ_handle {
    occ_config cfg{};
    int E = 0, k = 0, nd = 0, D = 0, F = 0, P = 0, world = 1, rank = 0;
    int gated = 0;
    int validate = 1;
    int num_sms = 148;
    std::vector<int32_t> plist;  // nd * P
    std::vector<int32_t> dev_of, slot_of;
    DevBuf<int32_t> d_dev_of, d_slot_of, d_widx, d_ranking;
    bool have_ranking = false;
    // resident weights, K-major
    DevBuf<__nv_bfloat16> w13t, w2t;
    int n1rows = 0;  // B rows per expert of GEMM-1
    bool weights_loaded = false;
    // workspace
    int n_cap = -1;
    DevBuf<uint64_t> mask, rmask;
    DevBuf<int32_t> group, rgroup, chunk_cnt, chunk_cnt2, totals, totals2, c_all;
    DevBuf<__nv_bfloat16> snd_x, y_src;  // world_size > 1: Sfd send batch, returned rows
    DevBuf<int32_t> snd_ids;
    DevBuf<float> snd_w;
    int* d_R = nullptr;                   // device copy of the received row count
    int last_R = 0;
    std::vector<int> h_C;                 // host copy of the (source, destination) counts
    DevBuf<int> offs;  // dispatch + compute offset arrays
    DevBuf<long long> stats;
    DevBuf<int32_t> err;
    DevBuf<int32_t> tok_row, tok_sfd, lam;
    DevBuf<__nv_bfloat16> in_x, x_epd, hbuf, ret, y16;
    DevBuf<int32_t> in_ids, in_tok, in_src, in_slot, in_dev, row_epd, epd_src, epd_j;
    DevBuf<float> in_w, epd_w, logits, rt_w;
    DevBuf<int32_t> rt_ids;  // routing of occ_forward_expert_parallel
    // exact router (occ_set_router_mode(h, OCC_ROUTER_EXACT)): fp64 scores,
    // unpruned top-k, fp64 weights
    int router_mode = 0;
    DevBuf<double> x_s64, x_w64, x_w64b;
    DevBuf<int32_t> x_ids;
    size_t R_max = 0, Q_max = 0, max_mblk = 0;
    int last_n = 0;
    bool have_forward = false;
    TmapBox tmA1, tmA2, tmB1, tmB2, tmRX, tmRG, tmC1, tmC2, tmAX;
    // OCC_GEMM_GATHER=1: GEMM-1 reads its A rows straight from the inbox with
    // TMA tile::gather4 instead of the Epd copy.  Measured 3x slower (32
    // gather4 per K block saturate the TMA unit: profiles/r01_gemm_micro.md),
    // so the copy is the default.
    int gather_a = 0;
    // one-GPU index chain as ONE cooperative kernel (occ_plan.cu; default) or
    // the multi-kernel chain (occ_set_plan_kernels(h, 0) / OCC_FUSED_PLAN=0)
    int fused_plan = 1;
    DevBuf<int> fp_ws;
    // dynamic tile schedulers of the grouped GEMMs: 2 ints (next tile, pairs
    // done) per launch site, zeroed once, left zeroed by every launch
    DevBuf<int> gsched;
    DispatchOffsets dofs{};
    ComputeOffsets cofs{};
    int* d_tok_base = nullptr;
    int* d_n_mblk = nullptr;
    int* d_q_total = nullptr;
    // world_size > 1
    Transport* tp = nullptr;
    // stage profiling (CUDA events on the launching stream)
    int profiling = 0;
    cudaEvent_t ev[kStages + 1] = {};
    int ev_recorded = 0;
    int in_ep = 0;
    // training: saved pre-activations + backward workspace
    int training = 0;
    bool have_train_state = false;
    bool bwd_weights_ready = false;  // w13o / w2o + their tensor maps built (training on at occ_load_experts)
    DevBuf<__nv_bfloat16> save_a, save_b, w13o, w2o, g_epd, gpre;
    DevBuf<float> gw_part, gw_row;
    // world_size > 1 backward: received upstream rows, returned gradient rows,
    // per-row routing-weight gradients (sent / received)
    DevBuf<__nv_bfloat16> g_in, g_ysrc;
    DevBuf<float> ret_gw, y_gw;
    TmapBox tmG_k, tmW2o, tmP_k, tmW1o, tmH_mn, tmG_mn, tmX_mn, tmP_mn, tmP_out;
    int bwd_tmaps_q = -1;
    // host-buffer pipeline (occ_forward_host)
    cudaStream_t s_in = nullptr, s_out = nullptr, s_cap = nullptr;
    // per staging slot: the layer on that slot captured as a CUDA graph
    // (validation off, world_size 1), re-captured when the call changes
    struct HostGraph {
        cudaGraphExec_t exec = nullptr;
        int n = -1;
        const void* gate = nullptr;
        occ_prune prune{};
        bool has_prune = false;
        int chunks = 0;
        long long gen = -1;  // g_buf_gen at capture
        int training = 0;
    } hgraph[2];
    std::vector<cudaEvent_t> pev;
    DevBuf<__nv_bfloat16> x_stage, o_stage;
    long long host_calls = 0;
    bool host_slot_used[2] = {false, false};
    // shared experts (occ_load_shared_experts): one dense FFN of width Fsh on
    // every token at its source
    int n_shared = 0, Fsh = 0, sh_rows = 0;
    bool sh_gate = false;
    DevBuf<__nv_bfloat16> w13s, w2s, sgate, hs, ys;
    DevBuf<float> sw;
    DevBuf<int> sh_grp;
    size_t sh_cap = 0;
    TmapBox tmBS1, tmBS2, tmAS1, tmAS2, tmCS1, tmCS2;
    cudaStream_t s_aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // peer-memory exchange (occ_comm_enable_peer)
    int gx_bf16 = 0;  // occ_set_grad_x_bf16: token gradient written as bf16
    bool peer = false;
    int peer_cap = 0;                  // max tokens per rank per forward
    // forwards issued = the arrival flag value, kept ON THE DEVICE (bumped by a
    // kernel at the start of every peer forward) so a captured CUDA graph
    // advances it on every replay
    DevBuf<unsigned long long> peer_seq;
    DevBuf<unsigned long long> flags;  // [3 * world]: dispatch arrivals, return arrivals, count rows
    DevBuf<int> c_peer;                // [world * world] (source, destination) counts, rows written by the sources
    DevBuf<void*> peer_tab;            // [world * kPeerSlots]
    std::vector<void*> ipc_opened;
    // micro-batching (occ_set_micro_batches): the second half of every
    // forward runs on a sibling handle (own workspace, own communicator,
    // the parent's resident weights) on its own stream, so one half's
    // exchange overlaps the other half's expert GEMMs
    int mb = 1;
    int comm_sms = 0;               // SMs the GEMMs leave to the other half's exchange
    int full_sms = 148;
    occ_handle* sib = nullptr;
    bool borrowed = false;          // weights / shared weights / ranking belong to the parent
    bool last_split = false;        // the last forward ran as two micro-batches
    cudaStream_t s_mb = nullptr;
    cudaEvent_t ev_mb[2] = {nullptr, nullptr};
};

namespace {


// ---------------------------------------------------------- transports ---
struct NcclTransport : Transport {
    ncclComm_t comm;
    int world;
    explicit NcclTransport(ncclComm_t c, int w) : comm(c), world(w) {}
    ~NcclTransport() override {
        ncclCommDestroy(comm);
        if (bar_buf) cudaFree(bar_buf);
    }
    const char* name() const override { return "nccl"; }
    occ_status allgather_counts(const int* send, int* recv, int nd, cudaStream_t st) override {
        NCCL_TRY(ncclAllGather(send, recv, nd, ncclInt32, comm, st));
        return OCC_OK;
    }
    occ_status alltoallv(const void* send, const std::vector<size_t>& soff, const std::vector<size_t>& scnt, void* recv,
                         const std::vector<size_t>& roff, const std::vector<size_t>& rcnt, int es,
                         cudaStream_t st) override {
        const char* sp = reinterpret_cast<const char*>(send);
        char* rp = reinterpret_cast<char*>(recv);
        NCCL_TRY(ncclGroupStart());
        for (int p = 0; p < world; ++p) {
            if (scnt[p]) NCCL_TRY(ncclSend(sp + soff[p] * es, scnt[p] * es, ncclUint8, p, comm, st));
            if (rcnt[p]) NCCL_TRY(ncclRecv(rp + roff[p] * es, rcnt[p] * es, ncclUint8, p, comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        return OCC_OK;
    }
    occ_status allreduce_i64(int64_t* buf, size_t count, cudaStream_t st) override {
        NCCL_TRY(ncclAllReduce(buf, buf, count, ncclInt64, ncclSum, comm, st));
        return OCC_OK;
    }
    int* bar_buf = nullptr;
    occ_status barrier() override {
        if (!bar_buf) CUDA_TRY(cudaMalloc(&bar_buf, sizeof(int)));
        NCCL_TRY(ncclAllReduce(bar_buf, bar_buf, 1, ncclInt32, ncclSum, comm, 0));
        CUDA_TRY(cudaStreamSynchronize(0));
        return OCC_OK;
    }
    occ_status exchange_pointers(const std::vector<void*>& mine, std::vector<void*>& all,
                                 std::vector<void*>& opened) override {
        const size_t m = mine.size(), hb = sizeof(cudaIpcMemHandle_t);
        std::vector<cudaIpcMemHandle_t> hs(m);
        for (size_t i = 0; i < m; ++i) CUDA_TRY(cudaIpcGetMemHandle(&hs[i], mine[i]));
        void* dsend = nullptr;
        void* drecv = nullptr;
        CUDA_TRY(cudaMalloc(&dsend, m * hb));
        CUDA_TRY(cudaMalloc(&drecv, m * hb * world));
        CUDA_TRY(cudaMemcpy(dsend, hs.data(), m * hb, cudaMemcpyHostToDevice));
        int rank = 0;
        NCCL_TRY(ncclCommUserRank(comm, &rank));
        NCCL_TRY(ncclAllGather(dsend, drecv, m * hb, ncclUint8, comm, 0));
        std::vector<cudaIpcMemHandle_t> allh(m * world);
        CUDA_TRY(cudaMemcpy(allh.data(), drecv, m * hb * world, cudaMemcpyDeviceToHost));
        cudaFree(dsend);
        cudaFree(drecv);
        all.assign(m * world, nullptr);
        for (int p = 0; p < world; ++p)
            for (size_t i = 0; i < m; ++i) {
                if (p == rank) {
                    all[p * m + i] = mine[i];
                    continue;
                }
                void* ptr = nullptr;
                CUDA_TRY(cudaIpcOpenMemHandle(&ptr, allh[p * m + i], cudaIpcMemLazyEnablePeerAccess));
                all[p * m + i] = ptr;
                opened.push_back(ptr);
            }
        return OCC_OK;
    }
    occ_status split(Transport** out) override {
        ncclComm_t c2;
        int rank = 0;
        NCCL_TRY(ncclCommUserRank(comm, &rank));
        NCCL_TRY(ncclCommSplit(comm, 0, rank, &c2, nullptr));
        *out = new NcclTransport(c2, world);
        return OCC_OK;
    }
    // one NCCL group (one launch) for the token rows and their routing metadata
    occ_status alltoallv_parts(const std::vector<Part>& parts, const std::vector<size_t>& soff,
                               const std::vector<size_t>& scnt, const std::vector<size_t>& roff,
                               const std::vector<size_t>& rcnt, cudaStream_t st) override {
        NCCL_TRY(ncclGroupStart());
        for (const Part& pt : parts) {
            const char* sp = reinterpret_cast<const char*>(pt.send);
            char* rp = reinterpret_cast<char*>(pt.recv);
            for (int p = 0; p < world; ++p) {
                if (scnt[p]) NCCL_TRY(ncclSend(sp + soff[p] * pt.es, scnt[p] * pt.es, ncclUint8, p, comm, st));
                if (rcnt[p]) NCCL_TRY(ncclRecv(rp + roff[p] * pt.es, rcnt[p] * pt.es, ncclUint8, p, comm, st));
            }
        }
        NCCL_TRY(ncclGroupEnd());
        return OCC_OK;
    }
};

// N ranks as host threads of one process on one GPU.
struct LoopGroup {
    int world;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<const void*> send;
    std::vector<std::vector<size_t>> soff, scnt;
    std::vector<std::vector<int>> counts;
    std::vector<std::vector<int64_t>> vals;
    std::vector<std::vector<void*>> ptrs;
    std::shared_ptr<LoopGroup> child;  // Transport::split: one more group of the same ranks
    explicit LoopGroup(int w) : world(w), send(w), soff(w), scnt(w), counts(w), vals(w), ptrs(w) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
std::mutex g_loop_m;
std::map<long, std::shared_ptr<LoopGroup>> g_loop;

struct LoopbackTransport : Transport {
    std::shared_ptr<LoopGroup> grp;
    int rank;
    LoopbackTransport(std::shared_ptr<LoopGroup> g, int r) : grp(std::move(g)), rank(r) {}
    const char* name() const override { return "loopback"; }
    occ_status allgather_counts(const int* send, int* recv, int nd, cudaStream_t st) override {
        std::vector<int> mine(nd);
        CUDA_TRY(cudaMemcpyAsync(mine.data(), send, sizeof(int) * nd, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        grp->counts[rank] = mine;
        grp->barrier();
        std::vector<int> all((size_t)nd * nd);
        for (int s = 0; s < nd; ++s) std::copy(grp->counts[s].begin(), grp->counts[s].end(), all.begin() + (size_t)s * nd);
        grp->barrier();
        CUDA_TRY(cudaMemcpyAsync(recv, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        return OCC_OK;
    }
    occ_status alltoallv(const void* send, const std::vector<size_t>& soff, const std::vector<size_t>& scnt, void* recv,
                         const std::vector<size_t>& roff, const std::vector<size_t>& rcnt, int es,
                         cudaStream_t st) override {
        CUDA_TRY(cudaStreamSynchronize(st));  // send data complete
        grp->send[rank] = send;
        grp->soff[rank] = soff;
        grp->scnt[rank] = scnt;
        grp->barrier();
        char* rp = reinterpret_cast<char*>(recv);
        for (int p = 0; p < grp->world; ++p) {
            if (grp->scnt[p][rank] != rcnt[p]) return fail(OCC_ERR_SHAPE, "loopback: send/recv count mismatch");
            if (!rcnt[p]) continue;
            const char* src = reinterpret_cast<const char*>(grp->send[p]) + grp->soff[p][rank] * es;
            CUDA_TRY(cudaMemcpyAsync(rp + roff[p] * es, src, rcnt[p] * es, cudaMemcpyDeviceToDevice, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
        grp->barrier();  // peers may reuse their send buffers only after every copy landed
        return OCC_OK;
    }
    occ_status exchange_pointers(const std::vector<void*>& mine, std::vector<void*>& all,
                                 std::vector<void*>&) override {
        grp->ptrs[rank] = mine;  // same process, same device: the pointers themselves
        grp->barrier();
        all.clear();
        for (int p = 0; p < grp->world; ++p) all.insert(all.end(), grp->ptrs[p].begin(), grp->ptrs[p].end());
        grp->barrier();
        return OCC_OK;
    }
    occ_status barrier() override {
        grp->barrier();
        return OCC_OK;
    }
    occ_status split(Transport** out) override {
        std::shared_ptr<LoopGroup> c;
        {
            std::lock_guard<std::mutex> lk(grp->m);
            if (!grp->child) grp->child = std::make_shared<LoopGroup>(grp->world);
            c = grp->child;
        }
        *out = new LoopbackTransport(c, rank);
        return OCC_OK;
    }
    occ_status allreduce_i64(int64_t* buf, size_t count, cudaStream_t st) override {
        std::vector<int64_t> mine(count);
        CUDA_TRY(cudaMemcpyAsync(mine.data(), buf, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        grp->vals[rank] = mine;
        grp->barrier();
        std::vector<int64_t> sum(count, 0);
        for (int p = 0; p < grp->world; ++p)
            for (size_t i = 0; i < count; ++i) sum[i] += grp->vals[p][i];
        grp->barrier();
        CUDA_TRY(cudaMemcpyAsync(buf, sum.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        return OCC_OK;
    }
};

// Ranks in separate processes, wired by a caller-supplied host all-gather
// (occ_comm_init_host: e.g. torch.distributed over gloo, MPI, a TCP store).
// It bootstraps the CUDA IPC peer mapping without NCCL (so it also works for
// several processes sharing one GPU, which NCCL refuses) and carries the
// (small) collectives; the data all-to-alls go through host staging, so the
// intended data path with this transport is the fused peer-memory exchange.
struct HostTransport : Transport {
    occ_host_allgather_fn fn;
    void* ctx;
    int world, rank;
    HostTransport(occ_host_allgather_fn f, void* c, int w, int r) : fn(f), ctx(c), world(w), rank(r) {}
    const char* name() const override { return "host"; }
    occ_status gather(const void* send, size_t bytes, void* recv) {
        if (fn(ctx, send, bytes, recv) != 0) return fail(OCC_ERR_NCCL, "host all-gather callback failed");
        return OCC_OK;
    }
    occ_status allgather_counts(const int* send, int* recv, int nd, cudaStream_t st) override {
        std::vector<int> mine(nd), all((size_t)nd * world);
        CUDA_TRY(cudaMemcpyAsync(mine.data(), send, sizeof(int) * nd, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        occ_status s = gather(mine.data(), sizeof(int) * nd, all.data());
        if (s != OCC_OK) return s;
        CUDA_TRY(cudaMemcpyAsync(recv, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        return OCC_OK;
    }
    occ_status alltoallv(const void* send, const std::vector<size_t>& soff, const std::vector<size_t>& scnt, void* recv,
                         const std::vector<size_t>& roff, const std::vector<size_t>& rcnt, int es,
                         cudaStream_t st) override {
        // host-staged: every rank publishes [per-peer element counts | rows in
        // peer order]; each keeps the part addressed to it
        size_t tot = 0;
        for (int p = 0; p < world; ++p) tot += scnt[p];
        std::vector<char> pkt(sizeof(uint64_t) * world + tot * es);
        auto* hdr = reinterpret_cast<uint64_t*>(pkt.data());
        size_t pos = sizeof(uint64_t) * world;
        for (int p = 0; p < world; ++p) {
            hdr[p] = scnt[p];
            if (scnt[p])
                CUDA_TRY(cudaMemcpyAsync(pkt.data() + pos, reinterpret_cast<const char*>(send) + soff[p] * es,
                                         scnt[p] * es, cudaMemcpyDeviceToHost, st));
            pos += scnt[p] * es;
        }
        CUDA_TRY(cudaStreamSynchronize(st));
        uint64_t len = pkt.size(), maxlen = 0;
        std::vector<uint64_t> lens(world);
        occ_status s = gather(&len, sizeof(len), lens.data());
        if (s != OCC_OK) return s;
        for (uint64_t l : lens) maxlen = std::max(maxlen, l);
        pkt.resize(maxlen);
        std::vector<char> all(maxlen * world);
        if ((s = gather(pkt.data(), maxlen, all.data())) != OCC_OK) return s;
        for (int p = 0; p < world; ++p) {
            const char* q = all.data() + maxlen * p;
            const auto* ph = reinterpret_cast<const uint64_t*>(q);
            size_t off = sizeof(uint64_t) * world;
            for (int d = 0; d < rank; ++d) off += ph[d] * es;
            if (ph[rank] != rcnt[p]) return fail(OCC_ERR_SHAPE, "host transport: send/recv count mismatch");
            if (rcnt[p])
                CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(recv) + roff[p] * es, q + off, rcnt[p] * es,
                                         cudaMemcpyHostToDevice, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
        return OCC_OK;
    }
    occ_status allreduce_i64(int64_t* buf, size_t count, cudaStream_t st) override {
        std::vector<int64_t> mine(count), all(count * world), sum(count, 0);
        CUDA_TRY(cudaMemcpyAsync(mine.data(), buf, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        occ_status s = gather(mine.data(), sizeof(int64_t) * count, all.data());
        if (s != OCC_OK) return s;
        for (int p = 0; p < world; ++p)
            for (size_t i = 0; i < count; ++i) sum[i] += all[p * count + i];
        CUDA_TRY(cudaMemcpyAsync(buf, sum.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        return OCC_OK;
    }
    occ_status exchange_pointers(const std::vector<void*>& mine, std::vector<void*>& all,
                                 std::vector<void*>& opened) override {
        const size_t m = mine.size(), hb = sizeof(cudaIpcMemHandle_t);
        std::vector<cudaIpcMemHandle_t> hs(m), allh(m * world);
        for (size_t i = 0; i < m; ++i) CUDA_TRY(cudaIpcGetMemHandle(&hs[i], mine[i]));
        occ_status s = gather(hs.data(), m * hb, allh.data());
        if (s != OCC_OK) return s;
        all.assign(m * world, nullptr);
        for (int p = 0; p < world; ++p)
            for (size_t i = 0; i < m; ++i) {
                if (p == rank) {
                    all[p * m + i] = mine[i];
                    continue;
                }
                void* ptr = nullptr;
                CUDA_TRY(cudaIpcOpenMemHandle(&ptr, allh[p * m + i], cudaIpcMemLazyEnablePeerAccess));
                all[p * m + i] = ptr;
                opened.push_back(ptr);
            }
        return OCC_OK;
    }
    occ_status barrier() override {
        const char mine = 1;
        std::vector<char> all(world);
        return gather(&mine, 1, all.data());
    }
    occ_status split(Transport** out) override {  // same callback: calls stay in the same order on every rank
        *out = new HostTransport(fn, ctx, world, rank);
        return OCC_OK;
    }
};

occ_status validate_placement(const occ_config& c, const int32_t* pl, std::vector<int32_t>& dev_of,
                              std::vector<int32_t>& slot_of) {
    const int E = c.num_experts, nd = c.num_devices, P = E / nd;
    dev_of.assign(E, -1);
    slot_of.assign(E, -1);
    for (int d = 0; d < nd; ++d)
        for (int i = 0; i < P; ++i) {
            const int e = pl[d * P + i];
            if (e < 0 || e >= E || dev_of[e] >= 0)
                return fail(OCC_ERR_PLACEMENT, "placement: device lists are not a partition of [0, E)");
            dev_of[e] = d;
            slot_of[e] = i;
        }
    return OCC_OK;
}

occ_status upload_tables(occ_handle* h) {
    CUDA_TRY(h->d_dev_of.ensure(h->E));
    CUDA_TRY(h->d_slot_of.ensure(h->E));
    const int G = h->world == 1 ? h->nd : 1;
    CUDA_TRY(h->d_widx.ensure(G * h->P));
    std::vector<int32_t> widx(G * h->P);
    for (int g = 0; g < G; ++g)
        for (int p = 0; p < h->P; ++p) widx[g * h->P + p] = h->world == 1 ? h->plist[g * h->P + p] : p;
    CUDA_TRY(cudaMemcpy(h->d_dev_of.p, h->dev_of.data(), sizeof(int32_t) * h->E, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(h->d_slot_of.p, h->slot_of.data(), sizeof(int32_t) * h->E, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(h->d_widx.p, widx.data(), sizeof(int32_t) * widx.size(), cudaMemcpyHostToDevice));
    if (!h->gsched.p) {
        CUDA_TRY(h->gsched.ensure(2 * kSchedSlots));
        CUDA_TRY(cudaMemset(h->gsched.p, 0, sizeof(int) * 2 * kSchedSlots));
    }
    return OCC_OK;
}

// Receive-side (expert-compute) workspace for R inbox rows.  world_size
// == 1: R is the static dedup bound n * min(k, N_d) (n * k for the naive
// path) and n_epd = n * k exactly; world_size > 1: R is the exact received
// row count (known after the count exchange) and n_epd <= R * min(k, P).
// Columns of the saved pre-activations: whole 32-column tiles (occ_gemm.cu).
inline size_t pre_cols(int F) { return (size_t)(F + 31) / 32 * 32; }

occ_status ensure_recv(occ_handle* h, size_t R, size_t epd_bound) {
    const int k = h->k, P = h->P, D = h->D, F = h->F;
    const int G = h->world == 1 ? h->nd : 1;
    size_t Q = epd_bound + (size_t)G * P * (kBM - 1);
    Q = (Q + kBM - 1) / kBM * kBM;
    const size_t nchunks = (R + kRankChunk - 1) / kRankChunk + 1;
    const size_t K2 = (size_t)G * (P + 1);
    CUDA_TRY(h->chunk_cnt2.ensure(nchunks * K2));
    if (R > h->R_max || !h->in_x.p) {
        CUDA_TRY(h->in_x.ensure(R * D));
        CUDA_TRY(h->in_ids.ensure(R * k));
        CUDA_TRY(h->in_w.ensure(R * k));
        CUDA_TRY(h->in_tok.ensure(R));
        CUDA_TRY(h->in_src.ensure(R));
        CUDA_TRY(h->in_slot.ensure(R));
        CUDA_TRY(h->in_dev.ensure(R));
        CUDA_TRY(h->rmask.ensure(R));
        CUDA_TRY(h->rgroup.ensure(R));
        CUDA_TRY(h->row_epd.ensure(R * P));
        CUDA_TRY(h->ret.ensure(R * D));
        h->R_max = R;
        if (!make_tmap_2d(h->tmAX.bytes, h->in_x.p, D, std::max<size_t>(R, 1), 64, 1))
            return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (inbox rows)");
    }
    if (h->training) {
        CUDA_TRY(h->save_a.ensure(std::max(Q, h->Q_max) * pre_cols(F)));
        if (h->gated) CUDA_TRY(h->save_b.ensure(std::max(Q, h->Q_max) * pre_cols(F)));
    }
    if (Q > h->Q_max || !h->x_epd.p) {
        CUDA_TRY(h->epd_src.ensure(Q));
        CUDA_TRY(h->epd_j.ensure(Q));
        CUDA_TRY(h->epd_w.ensure(Q));
        CUDA_TRY(h->x_epd.ensure(Q * D));
        CUDA_TRY(h->hbuf.ensure(Q * F));
        CUDA_TRY(h->y16.ensure(Q * D));
        h->Q_max = Q;
        h->max_mblk = Q / kBM;
        h->bwd_tmaps_q = -1;
        if (!make_tmap_2d(h->tmA1.bytes, h->x_epd.p, D, h->Q_max, 64, kBM / 2) ||
            !make_tmap_2d(h->tmA2.bytes, h->hbuf.p, F, h->Q_max, 64, kBM / 2) ||
            !make_tmap_out(h->tmC1.bytes, h->hbuf.p, F, h->Q_max) ||
            !make_tmap_out(h->tmC2.bytes, h->y16.p, D, h->Q_max))
            return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (A operands)");
    }
    return OCC_OK;
}

// Grow-only token-side workspace for n tokens (+ the receive side when all
// devices are local).
occ_status ensure_ws(occ_handle* h, int n) {
    if (n <= h->n_cap) return OCC_OK;
    const int nd = h->nd, k = h->k, P = h->P, D = h->D;
    const int G = h->world == 1 ? nd : 1;
    const int dedup = h->cfg.dedup;
    const size_t items = dedup ? (size_t)n : (size_t)n * k;
    const size_t span_max = dedup ? (size_t)std::min(k, nd) : (size_t)k;
    const size_t nchunks = (items + kRankChunk - 1) / kRankChunk + 1;
    const size_t K1 = (size_t)nd * (nd + 1);
    CUDA_TRY(h->mask.ensure(items));
    CUDA_TRY(h->group.ensure(items));
    CUDA_TRY(h->chunk_cnt.ensure(nchunks * K1));
    CUDA_TRY(h->totals.ensure(K1));
    CUDA_TRY(h->totals2.ensure((size_t)G * (P + 1)));
    CUDA_TRY(h->c_all.ensure((size_t)nd * nd + nd));
    // offsets: C, off_sd, inoff (3 nd^2) + in_base(nd+1) + nsfd(nd) + src_base(nd+1) + tok_base(2nd)
    //          + cnt/seg_base/unp_base (3 G P) + grp_mb (G P + 1) + n_mblk + q_total + R_dev
    const size_t noffs = 3 * (size_t)nd * nd + (nd + 1) + nd + (nd + 1) + 2 * nd + 4 * (size_t)G * P + 4;
    CUDA_TRY(h->offs.ensure(noffs));
    CUDA_TRY(h->stats.ensure(8));
    CUDA_TRY(h->err.ensure(1));
    CUDA_TRY(h->tok_row.ensure(dedup ? (size_t)n * nd : items));
    CUDA_TRY(h->tok_sfd.ensure(dedup ? (size_t)n * nd : items));
    CUDA_TRY(h->lam.ensure(n));
    if (h->world > 1) {  // send batch (Sfd, device-major) and the returned rows
        CUDA_TRY(h->snd_x.ensure((size_t)n * span_max * D));
        CUDA_TRY(h->snd_ids.ensure((size_t)n * span_max * k));
        CUDA_TRY(h->snd_w.ensure((size_t)n * span_max * k));
        CUDA_TRY(h->y_src.ensure((size_t)n * span_max * D));
    }
    int* o = h->offs.p;
    DispatchOffsets& d = h->dofs;
    d.C = o; o += nd * nd;
    d.off_sd = o; o += nd * nd;
    d.inoff = o; o += nd * nd;
    d.in_base = o; o += nd + 1;
    d.nsfd = o; o += nd;
    d.src_base = o; o += nd + 1;
    h->d_tok_base = o; o += 2 * nd;
    d.ntok = h->d_tok_base + nd;
    d.stats = h->stats.p;
    ComputeOffsets& c = h->cofs;
    c.cnt = o; o += G * P;
    c.seg_base = o; o += G * P;
    c.unp_base = o; o += G * P;
    c.grp_mb = o; o += G * P + 1;
    c.n_mblk = o; o += 1;
    c.q_total = o; o += 1;
    h->d_R = o; o += 1;
    c.widx = h->d_widx.p;
    c.stats = h->stats.p;
    h->d_n_mblk = c.n_mblk;
    h->d_q_total = c.q_total;
    if (h->world == 1) {
        occ_status s = ensure_recv(h, (size_t)n * span_max, (size_t)n * k);
        if (s != OCC_OK) return s;
        if (dedup && fused_plan_supported(nd, h->E, k)) CUDA_TRY(h->fp_ws.ensure(fused_plan_ws(n, nd, h->E, k)));
    }
    h->n_cap = n;
    return OCC_OK;
}

// Forward GEMM-1 (scatter + activation + modulation) and GEMM-2 (merge products).
void launch_gemm1(occ_handle* h, int ngroups, cudaStream_t st, bool gathered, const int* widx = nullptr) {
    GemmArgs g;
    g.tmap_a = gathered ? h->tmAX.bytes : h->tmA1.bytes;
    g.a_rows = gathered ? h->epd_src.p : nullptr;
    g.tmap_b = h->tmB1.bytes;
    g.tmap_c = h->tmC1.bytes;
    g.K = h->D;
    g.N = h->F;
    g.b_rows_per_e = h->n1rows;
    g.grp_mb = h->cofs.grp_mb;
    g.grp_w = widx ? widx : h->d_widx.p;
    g.ngroups = ngroups;
    g.row_w = h->epd_w.p;
    g.out = h->hbuf.p;
    g.ldo = h->F;
    g.act = h->cfg.activation;
    if (h->training) {
        g.save_a = h->save_a.p;
        g.save_b = h->gated ? h->save_b.p : nullptr;
    }
    g.band = h->D >= 4096 ? (1 << 20) : 8;  // see launch_gemm2
    g.max_tiles = (int)h->max_mblk * (h->gated ? h->F / 128 : (h->F + 255) / 256);
    g.sched = h->gsched.p + 2 * SCHED_GEMM1;
    launch_grouped_gemm(h->gated ? EPI_SWIGLU_BF16 : EPI_ACT_BF16, g, h->num_sms, st);
}

void launch_gemm2(occ_handle* h, int ngroups, cudaStream_t st, const int* widx = nullptr) {
    GemmArgs g;
    g.tmap_a = h->tmA2.bytes;
    g.tmap_b = h->tmB2.bytes;
    g.tmap_c = h->tmC2.bytes;
    g.K = h->F;
    g.N = h->D;
    g.b_rows_per_e = h->D;
    g.grp_mb = h->cofs.grp_mb;
    g.grp_w = widx ? widx : h->d_widx.p;
    g.ngroups = ngroups;
    // raster band (m-tiles per band): whole experts for long K (Mixtral GEMM-2,
    // K = 14336: +5%), 8 for short K (64-expert layers: +3-4%); profiles/r01_gemm_micro.md
    g.band = h->F >= 4096 ? (1 << 20) : 8;
    g.out = h->y16.p;  // per-expert products in bf16 (halves the store + combine traffic)
    g.ldo = h->D;
    g.act = OCC_ACT_IDENTITY;
    g.max_tiles = (int)h->max_mblk * ((h->D + 255) / 256);
    g.sched = h->gsched.p + 2 * SCHED_GEMM2;
    launch_grouped_gemm(EPI_ACT_BF16, g, h->num_sms, st);
}

// Shared experts on this device's n tokens: g = sigmoid(x . gate) (or 1),
// GEMM-1 x @ [w1s|w3s] with the act/SwiGLU x g epilogue, GEMM-2 h @ w2s
// -> ys [n, D] bf16 (added last by the combine).
// Shared-expert workspace for n tokens (grow-only).
occ_status ensure_shared(occ_handle* h, int n) {
    const int D = h->D, Fs = h->Fsh;
    const size_t n_pad = (size_t)(n + kBM - 1) / kBM * kBM;
    if (n_pad > h->sh_cap || !h->hs.p) {
        CUDA_TRY(h->hs.ensure(n_pad * Fs));
        CUDA_TRY(h->ys.ensure(n_pad * D));
        CUDA_TRY(h->sw.ensure(n_pad));
        h->sh_cap = n_pad;
        if (!make_tmap_2d(h->tmAS2.bytes, h->hs.p, Fs, n_pad, 64, kBM / 2) ||
            !make_tmap_out(h->tmCS1.bytes, h->hs.p, Fs, n_pad) || !make_tmap_out(h->tmCS2.bytes, h->ys.p, D, n_pad))
            return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (shared h)");
    }
    return OCC_OK;
}

occ_status run_shared(occ_handle* h, const __nv_bfloat16* x, int n, cudaStream_t st) {
    const int D = h->D, Fs = h->Fsh;
    const size_t n_pad = (size_t)(n + kBM - 1) / kBM * kBM;
    occ_status s0 = ensure_shared(h, n);
    if (s0 != OCC_OK) return s0;
    if (!make_tmap_2d(h->tmAS1.bytes, x, D, (uint64_t)n, 64, kBM / 2))
        return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (tokens; x must be 16-byte aligned)");
    launch_shared_gate(n, (int)n_pad, D, x, h->sh_gate ? h->sgate.p : nullptr, h->sw.p, h->sh_grp.p, st);
    const int nmb = (int)(n_pad / kBM);
    GemmArgs g;
    g.tmap_a = h->tmAS1.bytes;
    g.tmap_b = h->tmBS1.bytes;
    g.tmap_c = h->tmCS1.bytes;
    g.K = D;
    g.N = Fs;
    g.b_rows_per_e = h->sh_rows;
    g.grp_mb = h->sh_grp.p;
    g.grp_w = h->sh_grp.p + 2;
    g.ngroups = 1;
    g.row_w = h->sw.p;
    g.out = h->hs.p;
    g.ldo = Fs;
    g.act = h->cfg.activation;
    g.max_tiles = nmb * (h->gated ? Fs / 128 : (Fs + 255) / 256);
    g.sched = h->gsched.p + 2 * SCHED_SHARED1;
    launch_grouped_gemm(h->gated ? EPI_SWIGLU_BF16 : EPI_ACT_BF16, g, h->num_sms, st);
    GemmArgs g2;
    g2.tmap_a = h->tmAS2.bytes;
    g2.tmap_b = h->tmBS2.bytes;
    g2.tmap_c = h->tmCS2.bytes;
    g2.K = Fs;
    g2.N = D;
    g2.b_rows_per_e = D;
    g2.grp_mb = h->sh_grp.p;
    g2.grp_w = h->sh_grp.p + 2;
    g2.ngroups = 1;
    g2.band = h->Fsh >= 4096 ? (1 << 20) : 8;
    g2.out = h->ys.p;
    g2.ldo = D;
    g2.act = OCC_ACT_IDENTITY;
    g2.max_tiles = nmb * ((D + 255) / 256);
    g2.sched = h->gsched.p + 2 * SCHED_SHARED2;
    launch_grouped_gemm(EPI_ACT_BF16, g2, h->num_sms, st);
    return OCC_OK;
}

__global__ void tok_base_kernel(int nd, int* tok_base) {
    // tok_base[0..nd) = exclusive prefix of ntok = tok_base[nd..2nd)
    if (threadIdx.x == 0) {
        int run = 0;
        for (int s = 0; s < nd; ++s) {
            tok_base[s] = run;
            run += tok_base[nd + s];
        }
    }
}

// Dispatch plan: BRIM0 + inbox placement (+ stats). world_size == 1.
occ_status run_plan(occ_handle* h, const int32_t* ids, const float* w, const int32_t* sources, int n,
                    cudaStream_t st) {
    const int nd = h->nd, k = h->k, dedup = h->cfg.dedup;
    const int items = dedup ? n : n * k;
    PlanArgs pa{n, k, nd, dedup, ids, w, sources, -1, h->d_dev_of.p, h->d_slot_of.p, h->E, h->mask.p, h->group.p,
                h->err.p};
    launch_plan_mask(pa, st);
    RankWs ws{h->chunk_cnt.p, h->totals.p};
    launch_rank_count(items, h->group.p, h->mask.p, nd, nd, ws, st);
    launch_rank_scan(items, nd, nd, ws, st);
    launch_dispatch_finalize(nd, h->totals.p, h->dofs, st);
    tok_base_kernel<<<1, 32, 0, st>>>(nd, h->d_tok_base);
    count_launch();
    EmitDispatch em{n, k, nd, dedup, ids, w, sources, -1, h->d_dev_of.p, h->dofs, 1, h->tok_row.p, h->tok_sfd.p,
                    h->lam.p, h->in_tok.p, h->in_src.p, h->in_slot.p, h->in_dev.p};
    launch_rank_emit_dispatch(items, h->group.p, h->mask.p, nd, nd, ws, em, st);
    launch_token_stats(n, k, nd, ids, sources, -1, h->d_dev_of.p, h->E, h->stats.p, st);
    return OCC_OK;
}

void mark(occ_handle* h, int i, cudaStream_t st) {
    if (!h->profiling) return;
    if (!h->ev[i]) cudaEventCreate(&h->ev[i]);
    cudaEventRecord(h->ev[i], st);
    h->ev_recorded |= 1 << i;
}

// Bound on a peer arrival wait (default 10 s, then an error instead of a
// hang); OCC_PEER_TIMEOUT_MS shortens it for profiling runs that serialise the
// ranks' kernels (ncu on loopback ranks).
long long peer_timeout_ns() {
    static const long long v = getenv("OCC_PEER_TIMEOUT_MS") ? atoll(getenv("OCC_PEER_TIMEOUT_MS")) * 1000000LL
                                                              : 10000000000LL;
    return v;
}

occ_status check_err(occ_handle* h, cudaStream_t st) {
    CUDA_TRY(cudaStreamSynchronize(st));
    int32_t e = 0;
    CUDA_TRY(cudaMemcpy(&e, h->err.p, sizeof(e), cudaMemcpyDeviceToHost));
    if (e == 1) return fail(OCC_ERR_SHAPE, "forward: source device out of range");
    if (e == 4) return fail(OCC_ERR_ROUTING, "routing: invalid expert id, duplicate id, non-positive weight, or a row with no local expert");
    if (e == 5) return fail(OCC_ERR_CAPACITY, "prune: device budget too small for top-k");
    if (e == 7) return fail(OCC_ERR_CUDA, "peer exchange: a peer did not signal within the timeout");
    if (e) return fail(OCC_ERR_ROUTING, "routing error");
    return OCC_OK;
}

}  // namespace

__global__ void c_to_totals_kernel(int nd, const int* C, int* totals, int r, int* R_out) {
    // full (source, destination) count matrix -> the rank-key layout s*(nd+1)+d
    for (int i = threadIdx.x; i < nd * (nd + 1); i += blockDim.x) {
        const int s = i / (nd + 1), d = i % (nd + 1);
        totals[i] = d < nd ? C[s * nd + d] : 0;
    }
    if (threadIdx.x == 0) {  // rows this device receives
        int R = 0;
        for (int s = 0; s < nd; ++s) R += C[s * nd + r];
        *R_out = R;
    }
}

// Expert-parallel forward across world_size == N_d GPUs (this rank = EP
// device `rank`, owning the tokens in x).  Exchange layout (all_to_all_exchange,
// pipeline.cpp:125-176): the send batch is this source's Sfd batch
// (device-major BRIM0 counters, so the rows for destination d are contiguous
// at off[rank][d]); the inbox of this device is ordered (source asc, counter
// asc), i.e. source s lands at inoff[rank][s] = sum_{s'<s} C[s'][rank].  The
// return exchange is the exact inverse: inbox rows go back into the source's
// Sfd slots, which combine (pipeline.cpp:285-300) reads by BRIM0 counter.
occ_status forward_multi(occ_handle* h, const __nv_bfloat16* x, const int32_t* ids, const float* weights, int n,
                         __nv_bfloat16* out, cudaStream_t st) {
    if (!h->tp) return fail(OCC_ERR_STATE, "forward: world_size > 1 needs occ_comm_init");
    Transport* tp = h->tp;
    const int nd = h->nd, k = h->k, P = h->P, D = h->D, F = h->F, dedup = h->cfg.dedup, r = h->rank;
    const int items = dedup ? n : n * k;
    if (h->peer && n > h->peer_cap) return fail(OCC_ERR_SHAPE, "peer exchange: more tokens than max_tokens_per_rank");
    occ_status s = ensure_ws(h, std::max(n, 1));
    if (s != OCC_OK) return s;
    CUDA_TRY(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * 8, st));
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    if (!h->in_ep) h->ev_recorded = 0;
    mark(h, ST_PLAN, st);
    // 1. local dispatch plan: counts to every destination, all-gathered
    PlanArgs pa{n, k, nd, dedup, ids, weights, nullptr, r, h->d_dev_of.p, h->d_slot_of.p, h->E, h->mask.p,
                h->group.p, h->err.p};
    launch_plan_mask(pa, st);
    RankWs ws{h->chunk_cnt.p, h->totals.p};
    launch_rank_count(items, h->group.p, h->mask.p, 1, nd, ws, st);
    launch_rank_scan(items, 1, nd, ws, st);
    int* C_all = h->c_all.p;
    const unsigned long long* seq = h->peer_seq.p;
    void* const* tab = h->peer_tab.p;
    if (h->peer) {
        launch_seq_bump(h->peer_seq.p, st);
        // count all-gather over peer memory: this source's row stored into
        // every peer's count matrix, then an arrival flag (no collective, no
        // host round trip: the whole forward stays stream-ordered)
        C_all = h->c_peer.p;
        launch_peer_counts(tab, nd, r, h->totals.p, st);
        launch_peer_signal(tab, nd, r, 2 * nd, seq, st);
        launch_peer_wait(h->flags.p, nd, 2 * nd, seq, peer_timeout_ns(), h->err.p, st);
    } else {
        s = tp->allgather_counts(h->totals.p, C_all, nd, st);
        if (s != OCC_OK) return s;
    }
    // (the received row count of this device, R = sum_s C[s][r], on the device)
    c_to_totals_kernel<<<1, 256, 0, st>>>(nd, C_all, h->totals.p, r, h->d_R);
    count_launch();
    launch_dispatch_finalize(nd, h->totals.p, h->dofs, st);
    EmitDispatch em{n, k, nd, dedup, ids, weights, nullptr, r, h->d_dev_of.p, h->dofs, 0, h->tok_row.p,
                    h->tok_sfd.p, h->lam.p, nullptr, nullptr, nullptr, nullptr};
    launch_rank_emit_dispatch(items, h->group.p, h->mask.p, 1, nd, ws, em, st);
    launch_token_stats(n, k, nd, ids, nullptr, r, h->d_dev_of.p, h->E, h->stats.p, st);
    // 2. pack this source's Sfd batch (peer mode: straight into the peers' inboxes, below)
    mark(h, ST_PACK, st);
    PackArgs pk{n, k, nd, D, dedup, x, ids, weights, h->mask.p, h->tok_row.p, h->snd_x.p, h->snd_ids.p, h->snd_w.p};
    if (!h->peer) launch_pack(pk, st);
    // shared experts: source-side dense FFN on a second stream, overlapping
    // the dispatch exchange and the routed expert compute
    const bool shared = h->n_shared > 0 && n > 0;
    if (shared) {
        CUDA_TRY(cudaEventRecord(h->ev_fork, st));
        CUDA_TRY(cudaStreamWaitEvent(h->s_aux, h->ev_fork, 0));
        if ((s = run_shared(h, x, n, h->s_aux)) != OCC_OK) return s;
        CUDA_TRY(cudaEventRecord(h->ev_join, h->s_aux));
    }
    // 3. dispatch exchange.  Peer mode: sized by the static bound (at most one
    // row per (token, device) from each of the N_d sources, fixed when the
    // buffers were mapped), so the received count stays on the device.  NCCL
    // / host transports: the counts are needed on the host.
    long long R = (long long)h->R_max;
    std::vector<size_t> so(nd), sc(nd), ro(nd), rc(nd);
    if (!h->peer) {
        h->h_C.resize((size_t)nd * nd);
        CUDA_TRY(cudaMemcpyAsync(h->h_C.data(), C_all, sizeof(int) * nd * nd, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        std::vector<int64_t> off(nd), scnt64(nd), inoff(nd), rcnt64(nd);
        occ_exchange_layout(h->h_C.data(), nd, r, off.data(), scnt64.data(), inoff.data(), rcnt64.data());
        R = 0;
        for (int p = 0; p < nd; ++p) {
            so[p] = (size_t)off[p];
            sc[p] = (size_t)scnt64[p];
            ro[p] = (size_t)inoff[p];
            rc[p] = (size_t)rcnt64[p];
            R += rcnt64[p];
        }
        s = ensure_recv(h, (size_t)std::max<long long>(R, 1), (size_t)std::max<long long>(R, 1) * std::min(k, P));
        if (s != OCC_OK) return s;
        h->last_R = (int)R;
    }
    if (h->peer) {  // fused dispatch: pack stores into every destination's inbox, then arrival flags
        launch_peer_pack(pk, r, h->d_dev_of.p, h->dofs.off_sd, h->dofs.inoff, tab, st);
        launch_peer_signal(tab, nd, r, 0, seq, st);
        launch_peer_wait(h->flags.p, nd, 0, seq, peer_timeout_ns(), h->err.p, st);
    } else {
        const std::vector<Transport::Part> parts{{h->snd_x.p, h->in_x.p, D * 2},
                                                 {h->snd_ids.p, h->in_ids.p, k * 4},
                                                 {h->snd_w.p, h->in_w.p, k * 4}};
        if ((s = tp->alltoallv_parts(parts, so, sc, ro, rc, st)) != OCC_OK) return s;
    }
    // 4. compute index over the received rows
    mark(h, ST_CINDEX, st);
    const int Rm = (int)std::max<long long>(R, 1);
    ComputeArgs ca{Rm, h->d_R, k, P, 1, h->in_ids.p, h->in_w.p, nullptr, h->d_dev_of.p, h->d_slot_of.p, r,
                   h->rmask.p, h->rgroup.p, h->err.p};
    launch_compute_mask(ca, st);
    RankWs ws2{h->chunk_cnt2.p, h->totals2.p};
    launch_rank_count_dev(Rm, h->d_R, h->rgroup.p, h->rmask.p, 1, P, ws2, st);
    launch_rank_scan(Rm, 1, P, ws2, st);
    launch_compute_finalize(1, P, h->totals2.p, h->cofs, st);
    launch_init_epd((int)h->Q_max, h->epd_src.p, h->epd_w.p, st);
    EmitCompute ec{k, P, r, h->in_ids.p, h->in_w.p, h->d_slot_of.p, h->d_dev_of.p, h->cofs, h->row_epd.p,
                   h->epd_src.p, h->epd_w.p, h->epd_j.p};
    launch_rank_emit_compute(Rm, h->d_R, h->rgroup.p, h->rmask.p, 1, P, ws2, ec, st);
    // 5. grouped expert FFN (A rows gathered from the inbox by TMA, or copied)
    const bool gathered = h->gather_a && !h->training;
    if (!gathered) {  // Epd A operand: each received row read once, written to its Epd rows
        mark(h, ST_GATHER, st);
        launch_scatter_rows(Rm, h->d_R, P, D, h->in_x.p, nullptr, h->row_epd.p, P, h->cofs, h->x_epd.p, st);
    }
    mark(h, ST_GEMM1, st);
    launch_gemm1(h, P, st, gathered);
    mark(h, ST_GEMM2, st);
    launch_gemm2(h, P, st);
    // 6. intra-device partial combine -> bf16 return payload in inbox order
    mark(h, ST_PCOMBINE, st);
    if (h->peer) {  // fused partial combine + return straight into the sources' buffers
        launch_peer_return(Rm, h->d_R, nd, r, P, D, h->row_epd.p, h->y16.p, h->dofs.C, h->dofs.off_sd, h->dofs.inoff,
                           tab, st);
        launch_peer_signal(tab, nd, r, nd, seq, st);
        launch_peer_wait(h->flags.p, nd, nd, seq, peer_timeout_ns(), h->err.p, st);
    } else {
        launch_partial_combine(Rm, h->d_R, P, D, h->row_epd.p, h->y16.p, h->ret.p, st);
        // 7. return all-to-all: inbox rows back to their source's Sfd slots
        if ((s = tp->alltoallv(h->ret.p, ro, rc, h->y_src.p, so, sc, D * 2, st)) != OCC_OK) return s;
    }
    // 8. combine over devices ascending
    mark(h, ST_COMBINE, st);
    if (shared) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
    launch_combine(n, nd, k, dedup, D, h->mask.p, h->tok_row.p, h->y_src.p, shared ? h->ys.p : nullptr, out, st);
    mark(h, kStages, st);
    CUDA_TRY(cudaGetLastError());
    h->last_n = n;
    h->have_forward = true;
    h->have_train_state = h->training != 0;
    if (h->validate) return check_err(h, st);
    return OCC_OK;
}

static occ_status backward_multi(occ_handle* h, const __nv_bfloat16* up, void* g_x, float* g_w1, float* g_w3,
                                 float* g_w2, float* g_weights, cudaStream_t st);
static void bwd_gemms(occ_handle* h, int NG, const int* widx, float* g_w1, float* g_w3, float* g_w2, cudaStream_t st);

// The expert side of EP device `dev` over R inbox rows (stage-level entry
// points and the world_size > 1 forward): BRIM1 (build_compute_index,
// pipeline.cpp:52-89) -> Epd rows of the A operand -> grouped GEMM-1 (scatter
// + activation + modulation, pipeline.cpp:178-248) -> grouped GEMM-2 (merge
// products, pipeline.cpp:250-283) into h->y16 (per Epd row); the caller sums
// the products per row (partial combine) or extracts the index.  d_R: device
// row count (<= R_max, which sizes the grids).
static occ_status expert_side(occ_handle* h, int dev, const __nv_bfloat16* in_x, const int32_t* in_ids,
                              const float* in_w, int R_max, const int* d_R, bool gemms, cudaStream_t st) {
    const int k = h->k, P = h->P, D = h->D;
    const int Rm = std::max(R_max, 1);
    const int* widx = h->d_widx.p + (h->world == 1 ? (size_t)dev * P : 0);
    ComputeArgs ca{Rm, d_R, k, P, 1, in_ids, in_w, nullptr, h->d_dev_of.p, h->d_slot_of.p, dev,
                   h->rmask.p, h->rgroup.p, h->err.p};
    launch_compute_mask(ca, st);
    RankWs ws2{h->chunk_cnt2.p, h->totals2.p};
    launch_rank_count_dev(Rm, d_R, h->rgroup.p, h->rmask.p, 1, P, ws2, st);
    launch_rank_scan(Rm, 1, P, ws2, st);
    launch_compute_finalize(1, P, h->totals2.p, h->cofs, st);
    launch_init_epd((int)h->Q_max, h->epd_src.p, h->epd_w.p, st);
    EmitCompute ec{k, P, dev, in_ids, in_w, h->d_slot_of.p, h->d_dev_of.p, h->cofs, h->row_epd.p, h->epd_src.p,
                   h->epd_w.p, h->epd_j.p};
    launch_rank_emit_compute(Rm, d_R, h->rgroup.p, h->rmask.p, 1, P, ws2, ec, st);
    if (!gemms) return OCC_OK;
    mark(h, ST_GATHER, st);
    launch_scatter_rows(Rm, d_R, P, D, in_x, nullptr, h->row_epd.p, P, h->cofs, h->x_epd.p, st);
    mark(h, ST_GEMM1, st);
    launch_gemm1(h, P, st, false, widx);
    mark(h, ST_GEMM2, st);
    launch_gemm2(h, P, st, widx);
    return OCC_OK;
}

static occ_status stage_device(occ_handle* h, int device) {
    if (h->world == 1 ? (device < 0 || device >= h->nd) : device != h->rank)
        return fail(OCC_ERR_CONFIG, "stage: device must be in [0, num_devices) (world_size 1) or this rank");
    return OCC_OK;
}

extern "C" {

static void sync_sibling(occ_handle* h);

const char* occ_last_error(void) { return g_err.c_str(); }

occ_status occ_dispatch(occ_handle* h, const void* x, const int32_t* ids, const float* weights, int n,
                        const int32_t* brim0, void* sfd_x, int32_t* sfd_ids, float* sfd_weights, int32_t* sfd_token,
                        occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (n < 0) return fail(OCC_ERR_SHAPE, "dispatch: negative token count");
    if (n > 0 && (!x || !ids || !weights || !brim0 || !sfd_x || !sfd_ids || !sfd_weights || !sfd_token))
        return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    launch_dispatch_sfd(n, h->nd, h->k, h->D, reinterpret_cast<const __nv_bfloat16*>(x), ids, weights, brim0,
                        reinterpret_cast<__nv_bfloat16*>(sfd_x), sfd_ids, sfd_weights, sfd_token, st);
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}

occ_status occ_build_compute(occ_handle* h, int device, const int32_t* in_ids, const float* in_weights, int rows,
                             int32_t* cindex, int32_t* n_epd, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    occ_status s = stage_device(h, device);
    if (s != OCC_OK) return s;
    if (rows < 0) return fail(OCC_ERR_SHAPE, "build_compute: negative row count");
    if (rows > 0 && (!in_ids || !in_weights)) return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if ((s = ensure_ws(h, 1)) != OCC_OK) return s;
    const size_t R = (size_t)std::max(rows, 1);
    if ((s = ensure_recv(h, R, R * std::min(h->k, h->P))) != OCC_OK) return s;
    h->have_train_state = false;
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    CUDA_TRY(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * 8, st));
    launch_set_int(h->d_R, rows, st);
    if (rows > 0) {
        if ((s = expert_side(h, device, nullptr, in_ids, in_weights, rows, h->d_R, false, st)) != OCC_OK) return s;
        if (cindex) launch_extract_cindex(rows, h->d_R, h->P, nullptr, nullptr, h->row_epd.p, h->cofs, cindex, st);
    }
    if (n_epd) CUDA_TRY(cudaMemcpyAsync(n_epd, h->stats.p + 6, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaGetLastError());
    if (h->validate) return check_err(h, st);
    return OCC_OK;
}

occ_status occ_expert_compute(occ_handle* h, int device, const void* in_x, const int32_t* in_ids,
                              const float* in_weights, int rows, void* y_out, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    occ_status s = stage_device(h, device);
    if (s != OCC_OK) return s;
    if (!h->weights_loaded) return fail(OCC_ERR_STATE, "expert_compute: experts not loaded");
    if (rows < 0) return fail(OCC_ERR_SHAPE, "expert_compute: negative row count");
    if (rows > 0 && (!in_x || !in_ids || !in_weights || !y_out)) return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if ((s = ensure_ws(h, 1)) != OCC_OK) return s;
    const size_t R = (size_t)std::max(rows, 1);
    if ((s = ensure_recv(h, R, R * std::min(h->k, h->P))) != OCC_OK) return s;
    if (h->training) {
        CUDA_TRY(h->save_a.ensure(h->Q_max * pre_cols(h->F)));
        if (h->gated) CUDA_TRY(h->save_b.ensure(h->Q_max * pre_cols(h->F)));
    }
    h->have_train_state = false;
    if (rows == 0) return OCC_OK;
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    CUDA_TRY(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * 8, st));
    launch_set_int(h->d_R, rows, st);
    if ((s = expert_side(h, device, reinterpret_cast<const __nv_bfloat16*>(in_x), in_ids, in_weights, rows, h->d_R,
                         true, st)) != OCC_OK)
        return s;
    launch_partial_combine(rows, h->d_R, h->P, h->D, h->row_epd.p, h->y16.p, reinterpret_cast<__nv_bfloat16*>(y_out),
                           st);
    CUDA_TRY(cudaGetLastError());
    if (h->validate) return check_err(h, st);
    return OCC_OK;
}

occ_status occ_combine(occ_handle* h, const void* y_returned, const int32_t* brim0, int n, void* out,
                       occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (n < 0) return fail(OCC_ERR_SHAPE, "combine: negative token count");
    if (n > 0 && (!y_returned || !brim0 || !out)) return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    launch_combine_brim0(n, h->nd, h->D, brim0, reinterpret_cast<const __nv_bfloat16*>(y_returned),
                         reinterpret_cast<__nv_bfloat16*>(out), st);
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}
long long occ_launch_count(void) { return g_launches; }

static void unborrow(occ_handle* b);

occ_status occ_create(const occ_config* cfg, const int32_t* placement, int world_size, int rank, occ_handle** out) {
    if (!cfg || !placement || !out) return fail(OCC_ERR_ARG, "null argument");
    const occ_config& c = *cfg;
    // MoEConfig::validate (core.cpp:10-23)
    if (c.num_experts < 1) return fail(OCC_ERR_CONFIG, "config: num_experts must be >= 1");
    if (c.num_devices < 1) return fail(OCC_ERR_CONFIG, "config: num_devices must be >= 1");
    if (c.top_k < 1 || c.top_k > c.num_experts) return fail(OCC_ERR_CONFIG, "config: top_k must satisfy 1 <= k <= num_experts");
    if (c.top_k > 64) return fail(OCC_ERR_UNSUPPORTED, "top_k <= 64 on the device path");
    if (c.num_experts % c.num_devices) return fail(OCC_ERR_CONFIG, "config: num_experts must be divisible by num_devices");
    if (c.embed_dim < 1 || c.hidden_dim < 1) return fail(OCC_ERR_CONFIG, "config: dims must be >= 1");
    // B200 path constraints
    if (c.num_devices > kMaxDev || c.num_experts / c.num_devices > kMaxLocal || c.num_experts > 256)
        return fail(OCC_ERR_UNSUPPORTED, "N_d <= 64, experts per device <= 64, E <= 256");
    if (c.embed_dim % 8 || c.hidden_dim % 8) return fail(OCC_ERR_UNSUPPORTED, "embed_dim and hidden_dim must be multiples of 8");
    if (c.activation == OCC_ACT_SWIGLU && c.hidden_dim % 128)
        return fail(OCC_ERR_UNSUPPORTED, "SwiGLU needs hidden_dim % 128 == 0");
    if (c.activation < 0 || c.activation > 3) return fail(OCC_ERR_CONFIG, "config: bad activation");
    if (world_size != 1 && world_size != c.num_devices)
        return fail(OCC_ERR_CONFIG, "world_size must be 1 (all devices local) or num_devices");
    if (rank < 0 || rank >= world_size) return fail(OCC_ERR_CONFIG, "rank out of range");
    occ_handle* h = new occ_handle();
    h->cfg = c;
    h->E = c.num_experts;
    h->k = c.top_k;
    h->nd = c.num_devices;
    h->D = c.embed_dim;
    h->F = c.hidden_dim;
    h->P = h->E / h->nd;
    h->world = world_size;
    h->rank = rank;
    h->gated = c.activation == OCC_ACT_SWIGLU;
    if (const char* e = getenv("OCC_GEMM_GATHER")) h->gather_a = atoi(e);
    if (const char* e = getenv("OCC_FUSED_PLAN")) h->fused_plan = atoi(e);
    h->plist.assign(placement, placement + h->E);
    occ_status s = validate_placement(c, placement, h->dev_of, h->slot_of);
    if (s != OCC_OK) { delete h; return s; }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
    h->full_sms = h->num_sms;
    s = upload_tables(h);
    if (s != OCC_OK) { delete h; return s; }
    *out = h;
    return OCC_OK;
}

occ_status occ_destroy(occ_handle* h) {
    if (!h) return OCC_OK;
    if (h->sib) {
        unborrow(h->sib);
        occ_destroy(h->sib);
        h->sib = nullptr;
    }
    if (h->s_mb) cudaStreamDestroy(h->s_mb);
    for (auto& e : h->ev_mb)
        if (e) cudaEventDestroy(e);
    for (auto* b : {&h->d_dev_of, &h->d_slot_of, &h->d_widx, &h->d_ranking, &h->group, &h->rgroup, &h->chunk_cnt,
                    &h->chunk_cnt2, &h->totals, &h->totals2, &h->c_all, &h->snd_ids, &h->err, &h->tok_row, &h->tok_sfd, &h->lam, &h->in_ids, &h->in_tok,
                    &h->in_src, &h->in_slot, &h->in_dev, &h->row_epd, &h->epd_src})
        b->release();
    h->offs.release();
    h->fp_ws.release();
    h->stats.release();
    h->mask.release();
    h->rmask.release();
    for (auto* b : {&h->w13t, &h->w2t, &h->in_x, &h->x_epd, &h->hbuf, &h->ret, &h->snd_x, &h->y_src, &h->y16}) b->release();
    h->snd_w.release();
    for (auto* b : {&h->in_w, &h->epd_w, &h->logits, &h->rt_w}) b->release();
    h->rt_ids.release();
    for (auto* b : {&h->x_s64, &h->x_w64, &h->x_w64b}) b->release();
    h->x_ids.release();
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : h->pev) cudaEventDestroy(e);
    delete h->tp;
    for (auto& hg : h->hgraph)
        if (hg.exec) cudaGraphExecDestroy(hg.exec);
    if (h->s_cap) cudaStreamDestroy(h->s_cap);
    if (h->s_in) cudaStreamDestroy(h->s_in);
    if (h->s_out) cudaStreamDestroy(h->s_out);
    h->x_stage.release();
    h->o_stage.release();
    for (auto* b : {&h->save_a, &h->save_b, &h->w13o, &h->w2o, &h->g_epd, &h->gpre}) b->release();
    h->gw_part.release();
    h->gw_row.release();
    h->g_in.release();
    h->g_ysrc.release();
    h->ret_gw.release();
    h->y_gw.release();
    h->epd_j.release();
    for (void* ptr : h->ipc_opened) cudaIpcCloseMemHandle(ptr);
    h->flags.release();
    h->c_peer.release();
    h->peer_seq.release();
    h->peer_tab.release();
    for (auto* b : {&h->w13s, &h->w2s, &h->sgate, &h->hs, &h->ys}) b->release();
    h->sw.release();
    h->sh_grp.release();
    h->gsched.release();
    if (h->s_aux) cudaStreamDestroy(h->s_aux);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    delete h;
    return OCC_OK;
}

occ_status occ_set_placement(occ_handle* h, const int32_t* placement) {
    if (!h || !placement) return fail(OCC_ERR_ARG, "null argument");
    std::vector<int32_t> dev_of, slot_of;
    occ_status s = validate_placement(h->cfg, placement, dev_of, slot_of);
    if (s != OCC_OK) return s;
    h->plist.assign(placement, placement + h->E);
    h->dev_of = dev_of;
    h->slot_of = slot_of;
    h->weights_loaded = h->world == 1 && h->weights_loaded;  // world>1: local experts changed
    h->have_train_state = false;  // the saved Epd grouping belongs to the old table
    if (h->sib) {  // the micro-batch sibling plans with the same table
        occ_status s2 = occ_set_placement(h->sib, placement);
        if (s2 != OCC_OK) return s2;
    }
    return upload_tables(h);
}

occ_status occ_load_experts(occ_handle* h, const void* w1, const void* w3, const void* w2, occ_stream_t stream) {
    if (!h || !w1 || !w2) return fail(OCC_ERR_ARG, "null weight pointer");
    if (h->gated != (w3 != nullptr)) return fail(OCC_ERR_SHAPE, "w3 must be given iff activation is SwiGLU");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int El = h->world == 1 ? h->E : h->P;
    const int D = h->D, F = h->F;
    h->n1rows = h->gated ? 2 * F : F;
    h->have_train_state = false;
    h->bwd_weights_ready = false;
    // resident K-major rows (row pitch = K; padding the pitch to spread L2 sets
    // was measured: no change in DRAM traffic or time, profiles/r01_l2_traffic.md)
    const int p1 = D, p2 = F;
    CUDA_TRY(h->w13t.ensure((size_t)El * h->n1rows * p1));
    CUDA_TRY(h->w2t.ensure((size_t)El * D * p2));
    const auto* b1 = reinterpret_cast<const __nv_bfloat16*>(w1);
    const auto* b2 = reinterpret_cast<const __nv_bfloat16*>(w2);
    if (h->gated) {
        launch_transpose_weights(b1, El, D, F, h->w13t.p, h->n1rows, 1, st, p1);
        launch_transpose_weights(reinterpret_cast<const __nv_bfloat16*>(w3), El, D, F, h->w13t.p, h->n1rows, 2, st,
                                 p1);
    } else {
        launch_transpose_weights(b1, El, D, F, h->w13t.p, h->n1rows, 0, st, p1);
    }
    launch_transpose_weights(b2, El, F, D, h->w2t.p, D, 0, st, p2);
    CUDA_TRY(cudaGetLastError());
    if (h->training) {
        // backward needs the reference orientation: w2 [E, F, D] is K-major for
        // the merge adjoint (K = D); [w1 | w3] [E, D, F or 2F] for the scatter
        // adjoint (K = F or 2F).
        const int kw = h->gated ? 2 * F : F;
        CUDA_TRY(h->w2o.ensure((size_t)El * F * D));
        CUDA_TRY(h->w13o.ensure((size_t)El * D * kw));
        CUDA_TRY(cudaMemcpyAsync(h->w2o.p, b2, sizeof(__nv_bfloat16) * El * F * D, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpy2DAsync(h->w13o.p, kw * 2, b1, F * 2, F * 2, (size_t)El * D, cudaMemcpyDeviceToDevice, st));
        if (h->gated)
            CUDA_TRY(cudaMemcpy2DAsync(h->w13o.p + F, kw * 2, w3, F * 2, F * 2, (size_t)El * D,
                                       cudaMemcpyDeviceToDevice, st));
        if (!make_tmap_2d(h->tmW2o.bytes, h->w2o.p, D, (uint64_t)El * F, 64, 128) ||
            !make_tmap_2d(h->tmW1o.bytes, h->w13o.p, kw, (uint64_t)El * D, 64, 128))
            return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (backward weights)");
        h->bwd_weights_ready = true;
    }
    if (!make_tmap_2d(h->tmB1.bytes, h->w13t.p, D, (uint64_t)El * h->n1rows, 64, 128, 128, p1) ||
        !make_tmap_2d(h->tmB2.bytes, h->w2t.p, F, (uint64_t)El * D, 64, 128, 128, p2))
        return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (weights)");
    h->weights_loaded = true;
    return OCC_OK;
}

occ_status occ_load_shared_experts(occ_handle* h, int num_shared, int d_ff_shared, const void* w1, const void* w3,
                                   const void* w2, const void* gate, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (num_shared < 0) return fail(OCC_ERR_CONFIG, "shared experts: num_shared must be >= 0");
    // captured graphs (occ_forward_host) bake run_shared in or out and hold the
    // old buffers / tensor maps: any change re-captures; the micro-batch
    // sibling re-sizes its own h / ys buffers for the new width
    ++g_buf_gen;
    if (h->sib) h->sib->sh_cap = 0;
    if (num_shared == 0) {
        h->n_shared = 0;
        return OCC_OK;
    }
    if (!w1 || !w2) return fail(OCC_ERR_ARG, "null weight pointer");
    if (h->gated != (w3 != nullptr)) return fail(OCC_ERR_SHAPE, "w3 must be given iff activation is SwiGLU");
    if (d_ff_shared < 1 || d_ff_shared % 8) return fail(OCC_ERR_UNSUPPORTED, "d_ff_shared must be a multiple of 8");
    if (h->gated && d_ff_shared % 128) return fail(OCC_ERR_UNSUPPORTED, "SwiGLU needs d_ff_shared % 128 == 0");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int S = num_shared, F = d_ff_shared, D = h->D, Fs = S * F;
    h->sh_rows = h->gated ? 2 * Fs : Fs;
    CUDA_TRY(h->w13s.ensure((size_t)h->sh_rows * D));
    CUDA_TRY(h->w2s.ensure((size_t)D * Fs));
    const auto* b1 = reinterpret_cast<const __nv_bfloat16*>(w1);
    // stacking the S experts along the hidden dim: expert s's K-major rows
    // land at s*F (s*2F with the 128-row w1/w3 interleave), which is exactly
    // the layout of one FFN of width S*F; w2 [S, F, D] is already [S*F, D].
    if (h->gated) {
        launch_transpose_weights(b1, S, D, F, h->w13s.p, 2 * F, 1, st);
        launch_transpose_weights(reinterpret_cast<const __nv_bfloat16*>(w3), S, D, F, h->w13s.p, 2 * F, 2, st);
    } else {
        launch_transpose_weights(b1, S, D, F, h->w13s.p, F, 0, st);
    }
    launch_transpose_weights(reinterpret_cast<const __nv_bfloat16*>(w2), 1, Fs, D, h->w2s.p, D, 0, st);
    h->sh_gate = gate != nullptr;
    if (gate) {
        CUDA_TRY(h->sgate.ensure(D));
        CUDA_TRY(cudaMemcpyAsync(h->sgate.p, gate, sizeof(__nv_bfloat16) * D, cudaMemcpyDeviceToDevice, st));
    }
    CUDA_TRY(h->sh_grp.ensure(4));
    if (!h->s_aux) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->s_aux, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaGetLastError());
    if (!make_tmap_2d(h->tmBS1.bytes, h->w13s.p, D, (uint64_t)h->sh_rows, 64, 128) ||
        !make_tmap_2d(h->tmBS2.bytes, h->w2s.p, Fs, (uint64_t)D, 64, 128))
        return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (shared weights)");
    h->n_shared = S;
    h->Fsh = Fs;
    h->sh_cap = 0;  // h tensor map follows Fs
    if (h->peer) return ensure_shared(h, h->peer_cap);  // no allocation on the peer forward path
    return OCC_OK;
}

occ_status occ_set_similarity(occ_handle* h, const double* values) {
    if (!h || !values) return fail(OCC_ERR_ARG, "null argument");
    const int E = h->E;
    // ranking exactly as SimilarityAccumulator::finalize (pruning.cpp:203-211)
    std::vector<int32_t> rk((size_t)E * (E - 1 > 0 ? E - 1 : 1));
    for (int i = 0; i < E; ++i) {
        std::vector<int> r;
        for (int j = 0; j < E; ++j)
            if (j != i) r.push_back(j);
        const double* row = values + (size_t)i * E;
        std::stable_sort(r.begin(), r.end(), [&](int a, int b) {
            if (row[a] != row[b]) return row[a] > row[b];
            return a < b;
        });
        std::copy(r.begin(), r.end(), rk.begin() + (size_t)i * (E - 1));
    }
    CUDA_TRY(h->d_ranking.ensure(rk.size()));
    CUDA_TRY(cudaMemcpy(h->d_ranking.p, rk.data(), sizeof(int32_t) * rk.size(), cudaMemcpyHostToDevice));
    h->have_ranking = true;
    return OCC_OK;
}

occ_status occ_similarity_accumulate(const void* logits, int logits_fp64, int n, int e, double* inner,
                                     occ_stream_t stream) {
    if (n < 0 || e < 1) return fail(OCC_ERR_SHAPE, "similarity: bad shape");
    if (n > 0 && (!logits || !inner)) return fail(OCC_ERR_ARG, "null argument");
    launch_similarity_add(logits, logits_fp64, n, e, inner, reinterpret_cast<cudaStream_t>(stream));
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}

occ_status occ_similarity_finalize(const double* inner, long long tokens, int e, double* values) {
    if (!inner || !values || e < 1) return fail(OCC_ERR_ARG, "null argument");
    // SimilarityAccumulator::finalize (pruning.cpp:186-201), same operation order
    const double n = tokens > 0 ? (double)tokens : 1.0;
    for (int i = 0; i < e; ++i)
        for (int j = 0; j < e; ++j) {
            const double si = inner[(size_t)i * e + i], sj = inner[(size_t)j * e + j];
            double v = 0.0;
            if (!(si <= 0.0 || sj <= 0.0)) {
                const double mean_ip = inner[(size_t)i * e + j] / n;
                const double denom = (si / n) * (sj / n);
                v = std::min(1.0, mean_ip * mean_ip / denom);
            }
            values[(size_t)i * e + j] = v;
        }
    return OCC_OK;
}

occ_status occ_router_logits(occ_handle* h, const void* x, const void* gate, int n, float* logits,
                             occ_stream_t stream) {
    if (!h || !x || !gate || !logits) return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n <= 0) return OCC_OK;
    CUDA_TRY(h->rt_ids.ensure((size_t)n * h->k));
    CUDA_TRY(h->rt_w.ensure((size_t)n * h->k));
    CUDA_TRY(h->err.ensure(1));
    const int np = (h->E + 31) / 32 * 32;
    if (!make_tmap_2d(h->tmRX.bytes, x, h->D, n, 64, 128) || !make_tmap_2d(h->tmRG.bytes, gate, h->D, h->E, 64, np))
        return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (router)");
    if (!launch_router_tc(h->tmRX.bytes, h->tmRG.bytes, n, h->D, h->E, h->k, h->cfg.renormalize, h->rt_ids.p,
                          h->rt_w.p, logits, h->num_sms, st))
        return fail(OCC_ERR_UNSUPPORTED, "router: E <= 256");
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}

occ_status occ_set_grad_x_bf16(occ_handle* h, int on) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    h->gx_bf16 = on ? 1 : 0;
    return OCC_OK;
}

occ_status occ_set_plan_kernels(occ_handle* h, int fused) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    h->fused_plan = fused ? 1 : 0;
    if (h->sib) h->sib->fused_plan = h->fused_plan;
    return OCC_OK;
}

occ_status occ_set_validate(occ_handle* h, int on) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    h->validate = on;
    return OCC_OK;
}

// ----------------------------------------------------------------- routing
occ_status occ_gate_scores_f64(const double* x, int n, int d, const double* gate, int e, double* scores,
                               occ_stream_t stream) {
    if (n < 0 || d < 1 || e < 1) return fail(OCC_ERR_SHAPE, "gate_scores: bad shape");
    launch_gate_scores_f64(x, n, d, gate, e, scores, reinterpret_cast<cudaStream_t>(stream));
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}

occ_status occ_gate_logits_f64(const double* x, int n, int d, const double* gate, int e, double* logits,
                               occ_stream_t stream) {
    if (n < 0 || d < 1 || e < 1) return fail(OCC_ERR_SHAPE, "gate_logits: bad shape");
    launch_gate_scores_f64(x, n, d, gate, e, logits, reinterpret_cast<cudaStream_t>(stream), false);
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}

occ_status occ_topk_route_f64(const double* scores, int n, int e, int k, int renormalize, int32_t* ids,
                              double* weights, occ_stream_t stream) {
    if (k < 1 || k > e || e > 256) return fail(OCC_ERR_ROUTING, "topk_route: k out of range");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int32_t* err = nullptr;
    CUDA_TRY(cudaMallocAsync(&err, sizeof(int32_t), st));
    CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    launch_topk_f64(scores, n, e, k, renormalize, ids, weights, err, st);
    int32_t he = 0;
    CUDA_TRY(cudaMemcpyAsync(&he, err, sizeof(he), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaFreeAsync(err, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (he) return fail(OCC_ERR_ROUTING, "renormalize: non-positive weight sum");
    return OCC_OK;
}

static occ_status prune_dev(occ_handle* h, const occ_prune* prune, PruneDev& p) {
    p = PruneDev{0, 1, 0, h->cfg.renormalize, h->nd, h->d_dev_of.p, nullptr};
    if (!prune || prune->mode == OCC_PRUNE_NONE) return OCC_OK;
    if (prune->device_budget < 1 || prune->device_budget > h->nd)
        return fail(OCC_ERR_CONFIG, "prune: device budget must be in [1, num_devices]");
    if (prune->mode == OCC_PRUNE_SIMILARITY && !h->have_ranking)
        return fail(OCC_ERR_CONFIG, "prune: similarity mode requires a similarity table");
    p.mode = prune->mode;
    p.budget = prune->device_budget;
    p.own_score = prune->own_score;
    p.ranking = h->d_ranking.p;
    return OCC_OK;
}

occ_status occ_prune_routing_f64(occ_handle* h, const double* scores, const int32_t* ids_in, const double* w_in,
                                 int n, const occ_prune* prune, int32_t* ids, double* weights, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    PruneDev p;
    occ_status s = prune_dev(h, prune, p);
    if (s != OCC_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CUDA_TRY(h->err.ensure(1));
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    launch_prune_f64(scores, n, h->E, h->k, ids_in, w_in, p, ids, weights, h->err.p, st);
    return check_err(h, st);
}

// gate_scores -> topk_route -> prune_routing (pipeline.cpp:509-512) in the
// reference's arithmetic: fp64 logits of the bf16 operands in ascending k
// without FMA, softmax with glibc's exp, (score desc, index asc) top-k,
// renormalisation and pruning in fp64.  Bit-exact with the reference.
static occ_status route_exact(occ_handle* h, const void* x, const void* gate, int n, const PruneDev& p, int32_t* ids,
                              double* weights, double* scores, cudaStream_t st) {
    const int E = h->E, k = h->k;
    const size_t nn = (size_t)std::max(n, 1);
    double* s64 = scores;
    if (!s64) {
        CUDA_TRY(h->x_s64.ensure(nn * E));
        s64 = h->x_s64.p;
    }
    launch_gate_scores_bf16_f64(reinterpret_cast<const __nv_bfloat16*>(x), n, h->D,
                                reinterpret_cast<const __nv_bfloat16*>(gate), E, s64, st);
    if (p.mode == OCC_PRUNE_NONE) {
        launch_topk_f64(s64, n, E, k, h->cfg.renormalize, ids, weights, h->err.p, st);
    } else {
        CUDA_TRY(h->x_ids.ensure(nn * k));
        CUDA_TRY(h->x_w64b.ensure(nn * k));
        launch_topk_f64(s64, n, E, k, h->cfg.renormalize, h->x_ids.p, h->x_w64b.p, h->err.p, st);
        launch_prune_f64(s64, n, E, k, h->x_ids.p, h->x_w64b.p, p, ids, weights, h->err.p, st);
    }
    return OCC_OK;
}

occ_status occ_set_router_mode(occ_handle* h, int mode) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (mode != OCC_ROUTER_TC && mode != OCC_ROUTER_EXACT) return fail(OCC_ERR_CONFIG, "router mode: 0 (tc) or 1 (exact)");
    h->router_mode = mode;
    if (h->sib) h->sib->router_mode = mode;
    return OCC_OK;
}

occ_status occ_route_exact(occ_handle* h, const void* x, const void* gate, int n, const occ_prune* prune, int32_t* ids,
                           double* weights, double* scores, occ_stream_t stream) {
    if (!h || !gate || (n > 0 && (!x || !ids || !weights))) return fail(OCC_ERR_ARG, "null argument");
    if (n < 0) return fail(OCC_ERR_SHAPE, "route: negative token count");
    PruneDev p;
    occ_status s = prune_dev(h, prune, p);
    if (s != OCC_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CUDA_TRY(h->err.ensure(1));
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    if (n > 0 && (s = route_exact(h, x, gate, n, p, ids, weights, scores, st)) != OCC_OK) return s;
    CUDA_TRY(cudaGetLastError());
    if (h->validate) return check_err(h, st);
    return OCC_OK;
}

occ_status occ_route(occ_handle* h, const void* x, const void* gate, int n, const occ_prune* prune, int32_t* ids,
                     float* weights, float* scores, occ_stream_t stream) {
    if (!h || !gate || (n > 0 && (!x || !ids || !weights))) return fail(OCC_ERR_ARG, "null argument");
    if (n < 0) return fail(OCC_ERR_SHAPE, "route: negative token count");
    PruneDev p;
    occ_status s = prune_dev(h, prune, p);
    if (s != OCC_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CUDA_TRY(h->logits.ensure((size_t)std::max(n, 1) * h->E));
    CUDA_TRY(h->err.ensure(1));
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    if (n > 0 && h->router_mode == OCC_ROUTER_EXACT) {
        const size_t nn = (size_t)n;
        CUDA_TRY(h->x_w64.ensure(nn * h->k));
        double* s64 = nullptr;
        if (scores) {
            CUDA_TRY(h->x_s64.ensure(nn * h->E));
            s64 = h->x_s64.p;
        }
        if ((s = route_exact(h, x, gate, n, p, ids, h->x_w64.p, s64, st)) != OCC_OK) return s;
        launch_f64_to_f32(h->x_w64.p, (long)nn * h->k, weights, st);
        if (scores) launch_f64_to_f32(s64, (long)nn * h->E, scores, st);
    } else if (n > 0) {
        // logits = x g^T on tcgen05; softmax + top-k fused in the epilogue
        // unless pruning / score rows need the full rows (router_select)
        const int np = (h->E + 31) / 32 * 32;
        // router-score pruning runs in the epilogue too; similarity pruning and
        // score rows go through router_select on the written logits
        const bool need_rows = p.mode == OCC_PRUNE_SIMILARITY || scores != nullptr || np > 128;
        if (!make_tmap_2d(h->tmRX.bytes, x, h->D, n, 64, 128) ||
            !make_tmap_2d(h->tmRG.bytes, gate, h->D, h->E, 64, np))
            return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (router)");
        if (!launch_router_tc(h->tmRX.bytes, h->tmRG.bytes, n, h->D, h->E, h->k, h->cfg.renormalize, ids, weights,
                              need_rows ? h->logits.p : nullptr, h->num_sms, st, need_rows ? nullptr : &p, h->err.p))
            return fail(OCC_ERR_UNSUPPORTED, "router: E <= 256 and k <= 64");
        if (need_rows)
            launch_router_select(h->logits.p, n, h->E, h->k, h->cfg.renormalize, p, ids, weights, scores, h->err.p,
                                 st);
    }
    CUDA_TRY(cudaGetLastError());
    if (h->validate) return check_err(h, st);
    return OCC_OK;
}

// ----------------------------------------------------------------- EP path
occ_status occ_build_dispatch(occ_handle* h, const int32_t* ids, const int32_t* sources, int n, int32_t* brim0,
                              int32_t* counts, occ_stream_t stream) {
    if (!h || (!ids && n > 0)) return fail(OCC_ERR_ARG, "null argument");
    if (!h->cfg.dedup) return fail(OCC_ERR_UNSUPPORTED, "BRIM0 is defined for the dedup dispatch");
    if (n < 0) return fail(OCC_ERR_SHAPE, "build_dispatch: negative token count");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    occ_status s = ensure_ws(h, std::max(n, 1));
    if (s != OCC_OK) return s;
    if (h->world > 1) {
        // this rank's tokens are one source (= rank): BRIM0 N_d x n and its
        // count row, from the local plan alone (counters are per source,
        // pipeline.cpp:24-50; no exchange needed)
        const int nd = h->nd, k = h->k, r = h->rank;
        h->have_train_state = false;
        CUDA_TRY(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * 8, st));
        CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
        if (n > 0) {
            PlanArgs pa{n, k, nd, 1, ids, nullptr, nullptr, r, h->d_dev_of.p, h->d_slot_of.p, h->E, h->mask.p,
                        h->group.p, h->err.p};
            launch_plan_mask(pa, st);
            RankWs ws{h->chunk_cnt.p, h->totals.p};
            launch_rank_count(n, h->group.p, h->mask.p, 1, nd, ws, st);
            launch_rank_scan(n, 1, nd, ws, st);
            launch_one_source_totals(nd, r, h->totals.p, st);
            launch_dispatch_finalize(nd, h->totals.p, h->dofs, st);
            EmitDispatch em{n, k, nd, 1, ids, nullptr, nullptr, r, h->d_dev_of.p, h->dofs, 0, h->tok_row.p,
                            h->tok_sfd.p, h->lam.p, nullptr, nullptr, nullptr, nullptr};
            launch_rank_emit_dispatch(n, h->group.p, h->mask.p, 1, nd, ws, em, st);
            if (brim0) launch_brim0_one_source(n, nd, h->mask.p, h->tok_sfd.p, brim0, st);
        }
        if (counts) {
            if (n > 0)
                CUDA_TRY(cudaMemcpyAsync(counts, h->dofs.C + (size_t)r * nd, sizeof(int) * nd, cudaMemcpyDeviceToDevice,
                                         st));
            else
                CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * nd, st));
        }
        CUDA_TRY(cudaGetLastError());
        return check_err(h, st);
    }
    CUDA_TRY(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * 8, st));
    CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    h->have_train_state = false;  // the plan buffers no longer hold the saved forward
    s = run_plan(h, ids, nullptr, sources, n, st);
    if (s != OCC_OK) return s;
    if (brim0) launch_extract_brim0(n, h->nd, sources, -1, h->mask.p, h->lam.p, h->tok_sfd.p, h->d_tok_base, brim0, st);
    if (counts) CUDA_TRY(cudaMemcpyAsync(counts, h->dofs.C, sizeof(int) * h->nd * h->nd, cudaMemcpyDeviceToDevice, st));
    h->last_n = n;
    h->have_forward = true;  // the CommReport of the plan is available
    CUDA_TRY(cudaGetLastError());
    return check_err(h, st);
}

static occ_status forward_one(occ_handle* h, const void* x, const int32_t* ids, const float* weights,
                              const int32_t* sources, int n, void* out, cudaStream_t st);

// Sibling views of the parent's resident weights, shared experts and
// similarity ranking (borrowed: never reallocated or freed by the sibling).
static void sync_sibling(occ_handle* h) {
    occ_handle* b = h->sib;
    b->w13t.p = h->w13t.p, b->w13t.n = h->w13t.n;
    b->w2t.p = h->w2t.p, b->w2t.n = h->w2t.n;
    b->tmB1 = h->tmB1, b->tmB2 = h->tmB2;
    b->n1rows = h->n1rows;
    b->weights_loaded = h->weights_loaded;
    b->n_shared = h->n_shared, b->Fsh = h->Fsh, b->sh_rows = h->sh_rows, b->sh_gate = h->sh_gate;
    b->w13s.p = h->w13s.p, b->w13s.n = h->w13s.n;
    b->w2s.p = h->w2s.p, b->w2s.n = h->w2s.n;
    b->sgate.p = h->sgate.p, b->sgate.n = h->sgate.n;
    b->tmBS1 = h->tmBS1, b->tmBS2 = h->tmBS2;
    b->d_ranking.p = h->d_ranking.p, b->d_ranking.n = h->d_ranking.n;
    b->have_ranking = h->have_ranking;
    b->validate = h->validate;
    b->router_mode = h->router_mode;
    b->num_sms = h->num_sms;
    b->gather_a = h->gather_a;
    b->fused_plan = h->fused_plan;
}

static void unborrow(occ_handle* b) {
    for (auto* d : {&b->w13t, &b->w2t, &b->w13s, &b->w2s, &b->sgate}) d->p = nullptr, d->n = 0;
    b->d_ranking.p = nullptr, b->d_ranking.n = 0;
}

// Two micro-batches: tokens [0, n0) on this handle and `st`, [n0, n) on the
// sibling and its stream, forked from and joined back into `st`.
static occ_status forward_split(occ_handle* h, const void* x, const int32_t* ids, const float* weights,
                                const int32_t* sources, int n, void* out, cudaStream_t st) {
    occ_handle* b = h->sib;
    sync_sibling(h);
    if (b->n_shared > 0) {
        CUDA_TRY(b->sh_grp.ensure(4));
        if (!b->s_aux) {
            CUDA_TRY(cudaStreamCreateWithFlags(&b->s_aux, cudaStreamNonBlocking));
            CUDA_TRY(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&b->ev_join, cudaEventDisableTiming));
        }
    }
    int n0 = (n + 1) / 2;
    // round-robin sources (t mod N_d) stay those of the whole batch
    if (h->world == 1 && !sources) n0 = std::min(n, (n0 + h->nd - 1) / h->nd * h->nd);
    const int n1 = n - n0;
    const size_t D = h->D, k = h->k;
    CUDA_TRY(cudaEventRecord(h->ev_mb[0], st));
    CUDA_TRY(cudaStreamWaitEvent(h->s_mb, h->ev_mb[0], 0));
    occ_status s = forward_one(h, x, ids, weights, sources, n0, out, st);
    if (s != OCC_OK) return s;
    const bool second = n1 > 0 || h->world > 1;  // every rank joins the sibling's collectives
    if (second) {
        s = forward_one(b, reinterpret_cast<const __nv_bfloat16*>(x) + n0 * D, ids + n0 * k, weights + n0 * k,
                        sources ? sources + n0 : nullptr, n1, reinterpret_cast<__nv_bfloat16*>(out) + n0 * D,
                        h->s_mb);
        if (s != OCC_OK) return s;
    } else {
        b->last_n = 0;
    }
    CUDA_TRY(cudaEventRecord(h->ev_mb[1], h->s_mb));
    CUDA_TRY(cudaStreamWaitEvent(st, h->ev_mb[1], 0));
    h->last_split = second;
    return OCC_OK;
}

occ_status occ_forward(occ_handle* h, const void* x, const int32_t* ids, const float* weights,
                       const int32_t* sources, int n, void* out, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (n > 0 && (!x || !ids || !weights || !out)) return fail(OCC_ERR_ARG, "null argument");
    if (!h->weights_loaded) return fail(OCC_ERR_STATE, "forward: experts not loaded");
    if (n < 0) return fail(OCC_ERR_SHAPE, "forward: negative token count");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (h->mb > 1 && h->sib) return forward_split(h, x, ids, weights, sources, n, out, st);
    h->last_split = false;
    return forward_one(h, x, ids, weights, sources, n, out, st);
}

static occ_status forward_one(occ_handle* h, const void* x, const int32_t* ids, const float* weights,
                              const int32_t* sources, int n, void* out, cudaStream_t st) {
    if (h->world > 1)
        return forward_multi(h, reinterpret_cast<const __nv_bfloat16*>(x), ids, weights, n,
                             reinterpret_cast<__nv_bfloat16*>(out), st);
    occ_status s = ensure_ws(h, n);
    if (s != OCC_OK) return s;
    if (h->training) {
        CUDA_TRY(h->save_a.ensure(h->Q_max * pre_cols(h->F)));
        if (h->gated) CUDA_TRY(h->save_b.ensure(h->Q_max * pre_cols(h->F)));
    }
    h->last_n = n;
    h->have_forward = true;
    h->have_train_state = h->training && h->world == 1;
    if (n == 0) return OCC_OK;
    const int nd = h->nd, k = h->k, P = h->P, D = h->D, F = h->F, dedup = h->cfg.dedup;
    const int G = nd;
    // (inside forward_expert_parallel the route has just zeroed the error flag,
    // and a router error must survive to check_err; the fused plan zeroes the
    // CommReport counters itself: no memset nodes between route and plan)
    if (!h->in_ep) CUDA_TRY(cudaMemsetAsync(h->err.p, 0, sizeof(int32_t), st));
    if (!h->in_ep) h->ev_recorded = 0;
    // shared experts (every token, at its source; no exchange) on a second
    // stream from the start: their dense GEMMs fill the SMs the index chain and
    // the scatter leave idle and the routed GEMMs' tail waves (the dynamic tile
    // schedulers of both take tiles as CTAs free up); joined before the combine.
    // Profiling keeps them in line so the stage times stay separable.
    static const int shared_async_env = getenv("OCC_SHARED_ASYNC") ? atoi(getenv("OCC_SHARED_ASYNC")) : 1;
    const bool shared = h->n_shared > 0;
    const bool shared_async = shared && shared_async_env && !h->profiling && h->s_aux && h->ev_fork && h->ev_join;
    if (shared_async) {
        CUDA_TRY(cudaEventRecord(h->ev_fork, st));
        CUDA_TRY(cudaStreamWaitEvent(h->s_aux, h->ev_fork, 0));
        s = run_shared(h, reinterpret_cast<const __nv_bfloat16*>(x), n, h->s_aux);
        if (s != OCC_OK) return s;
        CUDA_TRY(cudaEventRecord(h->ev_join, h->s_aux));
    }
    mark(h, ST_PLAN, st);
    const bool gathered = h->gather_a && !h->training;
    bool fused = h->fused_plan && dedup && !h->gather_a && h->fp_ws.p && fused_plan_supported(nd, h->E, k);
    if (fused) {  // BRIM0 + routing rows + BRIM1 + Epd A operand in one cooperative kernel
        const size_t K = (size_t)nd * (nd + 1) + (size_t)nd * h->E;
        const size_t nchunks = fused_plan_chunks(n, k);
        FusedPlanArgs fa{n, k, nd, h->E, P, D, ids, weights, sources, h->d_dev_of.p, h->d_slot_of.p,
                         reinterpret_cast<const __nv_bfloat16*>(x), h->fp_ws.p, h->fp_ws.p + K * nchunks, h->dofs,
                         h->d_tok_base, h->cofs, h->mask.p, h->tok_row.p, h->tok_sfd.p, h->lam.p, h->in_tok.p, h->in_src.p,
                         h->in_slot.p, h->in_dev.p, h->in_ids.p, h->in_w.p, h->row_epd.p, h->epd_src.p, h->epd_j.p,
                         h->epd_w.p, h->x_epd.p, h->stats.p, h->err.p};
        // the Epd A rows: copied inside the cooperative kernel for small batches
        // (no extra launch), by the full-occupancy scatter kernel for large ones
        static const int scatter_env = getenv("OCC_PLAN_SCATTER") ? atoi(getenv("OCC_PLAN_SCATTER")) : -1;
        // (the Epd rows written: n * k of them; above 64 MB the full-occupancy
        // scatter kernel streams faster than the cooperative grid -- DeepSeek's
        // 403 MB: 0.125 vs 0.129 ms for plan + copy)
        const long copy_bytes = (long)n * k * D * 2;
        fa.scatter = scatter_env >= 0 ? scatter_env : copy_bytes <= (64l << 20);
        fa.zero_stats = 1;
        fused = launch_fused_plan(fa, h->num_sms, st);
        if (fused && !fa.scatter) {
            mark(h, ST_GATHER, st);
            launch_scatter_rows((int)h->R_max, h->dofs.in_base + nd, P, D, reinterpret_cast<const __nv_bfloat16*>(x),
                                h->in_tok.p, h->row_epd.p, nd * P, h->cofs, h->x_epd.p, st);
        }
    }
    if (!fused) {  // the multi-kernel chain
    CUDA_TRY(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * 8, st));
    // 1. dispatch plan (BRIM0) and exchange placement
    s = run_plan(h, ids, weights, sources, n, st);
    if (s != OCC_OK) return s;
    mark(h, ST_PACK, st);
    // 2. pack: x rows -> inbox rows of every destination device
    const int32_t* rowmap = h->tok_row.p;
    // (all devices are local: the Epd scatter below reads x itself, so the
    // inbox carries only the routing rows unless the gather4 GEMM path needs them)
    PackArgs pk{n, k, nd, D, dedup, reinterpret_cast<const __nv_bfloat16*>(x), ids, weights, h->mask.p, rowmap,
                h->gather_a ? h->in_x.p : nullptr, h->in_ids.p, h->in_w.p};
    launch_pack(pk, st);
    mark(h, ST_CINDEX, st);
    // 3. compute index (BRIM1) over the inbox rows
    const int* R_total = h->dofs.in_base + nd;
    const int R_max = (int)h->R_max;
    ComputeArgs ca{R_max, R_total, k, P, G, h->in_ids.p, h->in_w.p, h->in_dev.p, h->d_dev_of.p, h->d_slot_of.p, 0,
                   h->rmask.p, h->rgroup.p, h->err.p};
    launch_compute_mask(ca, st);
    RankWs ws{h->chunk_cnt2.p, h->totals2.p};
    launch_rank_count_dev(R_max, R_total, h->rgroup.p, h->rmask.p, G, P, ws, st);
    launch_rank_scan(R_max, G, P, ws, st);
    launch_compute_finalize(G, P, h->totals2.p, h->cofs, st);
    launch_init_epd((int)h->Q_max, h->epd_src.p, h->epd_w.p, st);
    EmitCompute ec{k, P, 0, h->in_ids.p, h->in_w.p, h->d_slot_of.p, h->d_dev_of.p, h->cofs, h->row_epd.p,
                   h->epd_src.p, h->epd_w.p, h->epd_j.p};
    launch_rank_emit_compute(R_max, R_total, h->rgroup.p, h->rmask.p, G, P, ws, ec, st);
    // 4. grouped GEMM-1 (activation / SwiGLU, routing weight fused); its A rows
    // come straight from the inbox (TMA gather4) unless training needs the
    // Epd copy for the weight gradient
    if (!gathered) {  // Epd A operand: each token row read once, written to its Epd rows
        mark(h, ST_GATHER, st);
        launch_scatter_rows(R_max, R_total, P, D, reinterpret_cast<const __nv_bfloat16*>(x), h->in_tok.p,
                            h->row_epd.p, G * P, h->cofs, h->x_epd.p, st);
    }
    }  // !fused
    mark(h, ST_GEMM1, st);
    launch_gemm1(h, G * P, st, gathered);
    mark(h, ST_GEMM2, st);
    // 5. grouped GEMM-2 (per-expert products, fp32)
    launch_gemm2(h, G * P, st);
    if (shared && !shared_async) {
        mark(h, ST_SHARED, st);
        s = run_shared(h, reinterpret_cast<const __nv_bfloat16*>(x), n, st);
        if (s != OCC_OK) return s;
    }
    // 6+7. intra-device partial combine (placement order) -> bf16 return
    // payload -> combine over devices ascending, fused on one GPU
    mark(h, ST_COMBINE, st);
    if (shared_async) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
    launch_combine_fused(n, nd, k, P, dedup, D, h->mask.p, h->tok_row.p, h->row_epd.p, h->y16.p,
                         shared ? h->ys.p : nullptr, reinterpret_cast<__nv_bfloat16*>(out), st);
    mark(h, kStages, st);
    CUDA_TRY(cudaGetLastError());
    if (h->validate) return check_err(h, st);
    return OCC_OK;
}

occ_status occ_forward_expert_parallel(occ_handle* h, const void* x, const void* gate, const occ_prune* prune,
                                       const int32_t* sources, int n, void* out, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CUDA_TRY(h->rt_ids.ensure((size_t)std::max(n, 1) * h->k));
    CUDA_TRY(h->rt_w.ensure((size_t)std::max(n, 1) * h->k));
    int32_t* ids = h->rt_ids.p;
    float* w = h->rt_w.p;
    h->ev_recorded = 0;
    mark(h, ST_ROUTE, st);
    occ_status s = occ_route(h, x, gate, n, prune, ids, w, nullptr, stream);
    h->in_ep = 1;
    if (s == OCC_OK) s = occ_forward(h, x, ids, w, sources, n, out, stream);
    h->in_ep = 0;
    return s;
}

occ_status occ_set_training(occ_handle* h, int on) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (on && h->mb > 1) return fail(OCC_ERR_UNSUPPORTED, "training: micro-batching is inference-only");
    h->training = on;
    h->have_train_state = false;
    return OCC_OK;
}

static occ_status ensure_bwd(occ_handle* h) {
    const size_t Q = h->Q_max;
    const int D = h->D, F = h->F, kw = h->gated ? 2 * F : F;
    const int NBf = (F + 255) / 256;
    CUDA_TRY(h->g_epd.ensure(Q * D));
    CUDA_TRY(h->gpre.ensure(Q * kw));
    CUDA_TRY(h->gw_part.ensure(Q * NBf * 2));  // per (row, n-tile, epilogue column half)
    if (h->bwd_tmaps_q != (int)Q) {
        if (!make_tmap_2d(h->tmG_k.bytes, h->g_epd.p, D, Q, 64, 128) ||
            !make_tmap_2d(h->tmP_k.bytes, h->gpre.p, kw, Q, 64, 128) ||
            !make_tmap_out(h->tmP_out.bytes, h->gpre.p, kw, Q) ||
            !make_tmap_2d(h->tmH_mn.bytes, h->hbuf.p, F, Q, 64, 64) ||
            !make_tmap_2d(h->tmG_mn.bytes, h->g_epd.p, D, Q, 64, 64) ||
            !make_tmap_2d(h->tmX_mn.bytes, h->x_epd.p, D, Q, 64, 64) ||
            !make_tmap_2d(h->tmP_mn.bytes, h->gpre.p, kw, Q, 64, 64))
            return fail(OCC_ERR_CUDA, "cuTensorMapEncodeTiled failed (backward)");
        h->bwd_tmaps_q = (int)Q;
    }
    return OCC_OK;
}

occ_status occ_backward(occ_handle* h, const void* upstream, float* g_x, float* g_w1, float* g_w3, float* g_w2,
                        float* g_weights, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (!h->have_train_state) return fail(OCC_ERR_STATE, "backward: forward state was not saved (occ_set_training)");
    if (!h->bwd_weights_ready)
        return fail(OCC_ERR_STATE, "backward: occ_set_training(h, 1) must precede occ_load_experts");
    if (h->n_shared) return fail(OCC_ERR_UNSUPPORTED, "backward: shared experts are forward-only in this build");
    const int n = h->last_n, k = h->k, P = h->P, D = h->D, F = h->F, nd = h->nd;
    const int El = h->world == 1 ? h->E : P;  // weight gradients of the resident experts
    if (!g_w1 || !g_w2 || (h->gated && !g_w3) || (n > 0 && (!upstream || !g_x || !g_weights)))
        return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaMemsetAsync(g_w1, 0, sizeof(float) * El * D * F, st));
    CUDA_TRY(cudaMemsetAsync(g_w2, 0, sizeof(float) * El * F * D, st));
    if (h->gated) CUDA_TRY(cudaMemsetAsync(g_w3, 0, sizeof(float) * El * D * F, st));
    if (h->world > 1)  // collective: every rank joins the exchanges, even with no tokens
        return backward_multi(h, reinterpret_cast<const __nv_bfloat16*>(upstream), g_x, g_w1, g_w3, g_w2, g_weights,
                              st);
    if (n == 0) return OCC_OK;
    occ_status s = ensure_bwd(h);
    if (s != OCC_OK) return s;
    // combine + return adjoints: the token's upstream row on every Epd row
    launch_scatter_rows((int)h->R_max, h->dofs.in_base + nd, P, D, reinterpret_cast<const __nv_bfloat16*>(upstream),
                        h->in_tok.p, h->row_epd.p, nd * P, h->cofs, h->g_epd.p, st);
    bwd_gemms(h, nd * P, h->d_widx.p, g_w1, g_w3, g_w2, st);
    // dispatch adjoint: sum each token's rows (device ascending), fp32
    launch_combine_grad(n, nd, k, P, h->cfg.dedup, D, h->mask.p, h->tok_row.p, h->row_epd.p, h->y16.p, g_x,
                        h->gx_bf16, st);
    launch_gw_scatter((int)h->Q_max, h->d_q_total, 2 * ((F + 255) / 256), h->gw_part.p, h->epd_src.p, h->in_tok.p,
                      h->epd_j.p, k, g_weights, st);
    CUDA_TRY(cudaGetLastError());
    if (h->validate) CUDA_TRY(cudaStreamSynchronize(st));
    return OCC_OK;
}

}  // extern "C"

// The four backward GEMMs of the saved Epd grouping (NG groups, weight index
// widx): merge adjoint (data, with the modulation / activation adjoints and
// the routing-weight partials in the epilogue) -> gpre; scatter adjoint (data)
// -> y16 per Epd row; merge / scatter adjoints (weights) -> g_w2, g_w1 | g_w3.
static void bwd_gemms(occ_handle* h, int NG, const int* widx, float* g_w1, float* g_w3, float* g_w2,
                      cudaStream_t st) {
    const int D = h->D, F = h->F, kw = h->gated ? 2 * F : F;
    // merge adjoint (data): g_mod = g_y w2^T, with modulation + activation
    // adjoints and the routing-weight partials fused in the epilogue
    GemmArgs g;
    g.tmap_a = h->tmG_k.bytes;
    g.tmap_c = h->tmP_out.bytes;  // g_a | g_b leave through smem + TMA stores
    g.tmap_b = h->tmW2o.bytes;
    g.K = D;
    g.N = F;
    g.b_rows_per_e = F;
    g.grp_mb = h->cofs.grp_mb;
    g.grp_w = widx;
    g.ngroups = NG;
    g.row_w = h->epd_w.p;
    g.out = h->gpre.p;
    g.ldo = kw;
    g.act = h->cfg.activation;
    g.pre_a = h->save_a.p;
    g.pre_b = h->gated ? h->save_b.p : nullptr;
    g.gw_part = h->gw_part.p;
    g.band = D >= 4096 ? (1 << 20) : 8;  // band from K, as in the forward (-3% at OLMoE)
    g.max_tiles = (int)h->max_mblk * ((F + 255) / 256);
    g.sched = h->gsched.p + 2 * SCHED_BWD0;
    launch_grouped_gemm(h->gated ? EPI_BWD_SWIGLU : EPI_BWD_ACT, g, h->num_sms, st);
    // scatter adjoint (data): g_x per Epd row = g_pre [w1 | w3]^T, fp32
    // accumulate, bf16 rows (the forward's product buffer is free by now)
    GemmArgs d1;
    d1.tmap_a = h->tmP_k.bytes;
    d1.tmap_b = h->tmW1o.bytes;
    d1.tmap_c = h->tmC2.bytes;
    d1.K = kw;
    d1.N = D;
    d1.b_rows_per_e = D;
    d1.grp_mb = h->cofs.grp_mb;
    d1.grp_w = widx;
    d1.ngroups = NG;
    d1.band = kw >= 4096 ? (1 << 20) : 8;
    d1.out = h->y16.p;
    d1.ldo = D;
    d1.act = OCC_ACT_IDENTITY;
    d1.max_tiles = (int)h->max_mblk * ((D + 255) / 256);
    d1.sched = h->gsched.p + 2 * (SCHED_BWD0 + 1);
    launch_grouped_gemm(EPI_ACT_BF16, d1, h->num_sms, st);
    // merge adjoint (weights): g_w2[e] = mod_e^T g_y_e (backward.cpp:84-93)
    GemmArgs w2;
    w2.tmap_a = h->tmH_mn.bytes;
    w2.tmap_b = h->tmG_mn.bytes;
    w2.N = D;
    w2.M = F;
    w2.grp_cnt = h->cofs.cnt;
    w2.seg_base = h->cofs.seg_base;
    w2.grp_w = widx;
    w2.ngroups = NG;
    w2.out = g_w2;
    w2.ldo = D;
    w2.out_estride = (long)F * D;
    w2.max_tiles = NG * ((F + 255) / 256) * ((D + 255) / 256);
    w2.sched = h->gsched.p + 2 * (SCHED_BWD0 + 2);
    launch_grouped_gemm(EPI_WGRAD, w2, h->num_sms, st);
    // scatter adjoint (weights): [g_w1 | g_w3][e] = x_e^T g_pre_e (backward.cpp:123-133)
    GemmArgs w1;
    w1.tmap_a = h->tmX_mn.bytes;
    w1.tmap_b = h->tmP_mn.bytes;
    w1.N = kw;
    w1.M = D;
    w1.grp_cnt = h->cofs.cnt;
    w1.seg_base = h->cofs.seg_base;
    w1.grp_w = widx;
    w1.ngroups = NG;
    w1.out = g_w1;
    w1.out2 = h->gated ? g_w3 : nullptr;
    w1.split = F;
    w1.ldo = F;
    w1.out_estride = (long)D * F;
    w1.max_tiles = NG * ((D + 255) / 256) * ((kw + 255) / 256);
    w1.sched = h->gsched.p + 2 * (SCHED_BWD0 + 3);
    launch_grouped_gemm(EPI_WGRAD, w1, h->num_sms, st);
}

// backward_vjps across ranks (world_size == N_d; backward.cpp:24-161 with
// the two reverse exchanges made real): the upstream rows go out along the
// forward's dispatch layout (the combine adjoint, backward.cpp:43-54: every
// Sfd row gets its token's upstream row; gathered per device, :74-78), the
// expert-side adjoints run on this rank's saved Epd grouping, each inbox
// row's scatter-adjoint partial sum (over its local experts, placement order)
// and its routing-weight gradients go back along the return layout (:136-139),
// and the source sums them per token over devices ascending (dispatch
// adjoint, :143-152).  Exchanges over the handle's transport (NCCL, the
// host-callback transport or loopback ranks).
static occ_status backward_multi(occ_handle* h, const __nv_bfloat16* up, void* g_x, float* g_w1, float* g_w3,
                                 float* g_w2, float* g_weights, cudaStream_t st) {
    if (!h->tp) return fail(OCC_ERR_STATE, "backward: world_size > 1 needs a communicator");
    Transport* tp = h->tp;
    const int n = h->last_n, k = h->k, P = h->P, D = h->D, F = h->F, nd = h->nd, r = h->rank, dedup = h->cfg.dedup;
    occ_status s = ensure_bwd(h);
    if (s != OCC_OK) return s;
    // the forward's exchange layout (its counts are still on the device)
    std::vector<int> hC((size_t)nd * nd);
    CUDA_TRY(cudaMemcpyAsync(hC.data(), h->dofs.C, sizeof(int) * nd * nd, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<int64_t> off(nd), scnt(nd), inoff(nd), rcnt(nd);
    occ_exchange_layout(hC.data(), nd, r, off.data(), scnt.data(), inoff.data(), rcnt.data());
    std::vector<size_t> so(nd), sc(nd), ro(nd), rc(nd);
    size_t R = 0, S = 0;
    for (int p = 0; p < nd; ++p) {
        so[p] = (size_t)off[p], sc[p] = (size_t)scnt[p], ro[p] = (size_t)inoff[p], rc[p] = (size_t)rcnt[p];
        R += rc[p];
        S += sc[p];
    }
    const size_t Rb = std::max<size_t>(h->R_max, 1), Sb = std::max<size_t>(S, 1);
    CUDA_TRY(h->g_in.ensure(Rb * D));
    CUDA_TRY(h->g_ysrc.ensure(Sb * D));
    CUDA_TRY(h->ret_gw.ensure(Rb * k));
    CUDA_TRY(h->y_gw.ensure(Sb * k));
    // 1. combine adjoint: this source's upstream rows into its Sfd send batch
    PackArgs pk{n, k, nd, D, dedup, up, nullptr, nullptr, h->mask.p, h->tok_row.p, h->snd_x.p, nullptr, nullptr};
    launch_pack(pk, st);
    if ((s = tp->alltoallv(h->snd_x.p, so, sc, h->g_in.p, ro, rc, D * 2, st)) != OCC_OK) return s;
    // 2. expert-side adjoints over the received rows (the forward's BRIM1 / Epd grouping)
    const int Rm = (int)std::max<size_t>(R, 1);
    if (R > 0) {
        launch_scatter_rows(Rm, h->d_R, P, D, h->g_in.p, nullptr, h->row_epd.p, P, h->cofs, h->g_epd.p, st);
        bwd_gemms(h, P, h->d_widx.p, g_w1, g_w3, g_w2, st);
        // scatter adjoint summed over the row's local experts -> return payload
        launch_partial_combine(Rm, h->d_R, P, D, h->row_epd.p, h->y16.p, h->ret.p, st);
        CUDA_TRY(cudaMemsetAsync(h->ret_gw.p, 0, sizeof(float) * R * k, st));
        launch_gw_scatter((int)h->Q_max, h->d_q_total, 2 * ((F + 255) / 256), h->gw_part.p, h->epd_src.p, nullptr,
                          h->epd_j.p, k, h->ret_gw.p, st);
    }
    // 3. reverse exchange back into the sources' Sfd slots
    if ((s = tp->alltoallv(h->ret.p, ro, rc, h->g_ysrc.p, so, sc, D * 2, st)) != OCC_OK) return s;
    if ((s = tp->alltoallv(h->ret_gw.p, ro, rc, h->y_gw.p, so, sc, k * 4, st)) != OCC_OK) return s;
    // 4. dispatch adjoint at the source
    launch_combine_back(n, nd, k, dedup, D, h->mask.p, h->tok_row.p, h->g_ysrc.p, h->y_gw.p, g_x, h->gx_bf16,
                        g_weights, st);
    CUDA_TRY(cudaGetLastError());
    if (h->validate) CUDA_TRY(cudaStreamSynchronize(st));
    return OCC_OK;
}

extern "C" {

occ_status occ_set_profiling(occ_handle* h, int on) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    h->profiling = on;
    return OCC_OK;
}

int occ_stage_ms(occ_handle* h, float* ms, int max_stages) {
    // Elapsed time of each recorded stage of the last forward (ms[i] < 0: not recorded).
    if (!h || !ms) return -1;
    int n = 0;
    for (int i = 0; i < kStages && i < max_stages; ++i, ++n) {
        ms[i] = -1.0f;
        if (!(h->ev_recorded >> i & 1)) continue;
        int j = i + 1;
        while (j <= kStages && !(h->ev_recorded >> j & 1)) ++j;
        if (j > kStages) continue;
        cudaEventSynchronize(h->ev[j]);
        cudaEventElapsedTime(&ms[i], h->ev[i], h->ev[j]);
    }
    return n;
}

occ_status occ_forward_host(occ_handle* h, const void* x_host, const void* gate, const occ_prune* prune, int n,
                            void* out_host, int chunks, occ_stream_t stream) {
    // Double-buffered host pipeline.  Call i uses staging slot i % 2:
    //   s_in   : wait slot's x buffer free -> H2D chunks -> ev_in[c]
    //   stream : wait ev_in[c] (+ slot's out buffer free) -> layer -> ev_comp[c]
    //   s_out  : wait ev_comp[c] -> D2H chunks -> slot's out buffer free
    // so the copies of call i+1 / i-1 overlap the layer of call i.  Results
    // are in out_host once occ_host_wait() has been ordered on a stream.
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (n > 0 && (!x_host || !gate || !out_host)) return fail(OCC_ERR_ARG, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    chunks = std::max(1, std::min(chunks, 16));
    if (n < chunks) chunks = std::max(1, n);
    const size_t row = (size_t)h->D * sizeof(__nv_bfloat16);
    const size_t slot_elems = (size_t)std::max(n, 1) * h->D;
    if (h->x_stage.n < 2 * slot_elems) {
        CUDA_TRY(cudaDeviceSynchronize());  // staging regrow: no copy may be in flight
        CUDA_TRY(h->x_stage.ensure(2 * slot_elems));
        CUDA_TRY(h->o_stage.ensure(2 * slot_elems));
        h->host_slot_used[0] = h->host_slot_used[1] = false;
        for (auto& g : h->hgraph) g.n = -1;  // buffers moved: re-capture
    }
    if (!h->s_in) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    }
    // events: [slot][0] x free, [slot][1] out free, [slot][2 + 2c] in, [slot][3 + 2c] comp
    const int per_slot = 2 + 2 * 16;
    while ((int)h->pev.size() < 2 * per_slot + 1) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->pev.push_back(e);
    }
    const int slot = h->host_calls++ & 1;
    cudaEvent_t* ev = h->pev.data() + slot * per_slot;
    // slot stride = half the allocated staging capacity (fixed between
    // regrows), not this call's n * D: with a shrinking batch the two slots
    // must still never overlap the region the other slot's in-flight copies
    // and layer use
    const size_t base_el = slot * (h->x_stage.n / 2);
    if (h->host_slot_used[slot]) {
        CUDA_TRY(cudaStreamWaitEvent(h->s_in, ev[0], 0));  // previous layer on this slot read x
        CUDA_TRY(cudaStreamWaitEvent(st, ev[1], 0));       // previous D2H on this slot read out
    }
    const char* xh = reinterpret_cast<const char*>(x_host);
    char* oh = reinterpret_cast<char*>(out_host);
    // With validation off (no host synchronisation inside the layer) and all
    // devices local, the layer of each (slot, chunk) replays as a CUDA graph:
    // small batches are otherwise bound by the ~20 kernel launches per call.
    auto& hg = h->hgraph[slot];
    const bool use_graph = !h->validate && h->world == 1 && !h->profiling && chunks == 1 && n > 0 && h->mb == 1;
    if (use_graph) {
        const bool same = hg.exec && hg.n == n && hg.gate == gate && hg.chunks == chunks && hg.gen == g_buf_gen &&
                          hg.training == h->training &&
                          hg.has_prune == (prune != nullptr) &&
                          (!prune || memcmp(&hg.prune, prune, sizeof(occ_prune)) == 0);
        if (!same) {
            if (hg.exec) cudaGraphExecDestroy(hg.exec);
            hg.exec = nullptr;
            if (!h->s_cap) CUDA_TRY(cudaStreamCreateWithFlags(&h->s_cap, cudaStreamNonBlocking));
            auto* xs = h->x_stage.p + base_el;
            auto* os = h->o_stage.p + base_el;
            // eager once (grows the workspace), then capture on the handle's stream
            CUDA_TRY(cudaStreamSynchronize(st));
            occ_status s = occ_forward_expert_parallel(h, xs, gate, prune, nullptr, n, os,
                                                       reinterpret_cast<occ_stream_t>(h->s_cap));
            if (s != OCC_OK) return s;
            CUDA_TRY(cudaStreamSynchronize(h->s_cap));
            cudaGraph_t graph;
            CUDA_TRY(cudaStreamBeginCapture(h->s_cap, cudaStreamCaptureModeThreadLocal));
            s = occ_forward_expert_parallel(h, xs, gate, prune, nullptr, n, os, reinterpret_cast<occ_stream_t>(h->s_cap));
            cudaError_t ce = cudaStreamEndCapture(h->s_cap, &graph);
            if (s != OCC_OK) return s;
            CUDA_TRY(ce);
            CUDA_TRY(cudaGraphInstantiate(&hg.exec, graph, 0));
            cudaGraphDestroy(graph);
            hg.gen = g_buf_gen;
            hg.training = h->training;
            hg.n = n;
            hg.gate = gate;
            hg.chunks = chunks;
            hg.has_prune = prune != nullptr;
            if (prune) hg.prune = *prune;
        }
    }
    int base = 0;
    for (int c = 0; c < chunks; ++c) {
        const int nc = n / chunks + (c < n % chunks ? 1 : 0);
        auto* xs = h->x_stage.p + base_el + (size_t)base * h->D;
        auto* os = h->o_stage.p + base_el + (size_t)base * h->D;
        CUDA_TRY(cudaMemcpyAsync(xs, xh + base * row, nc * row, cudaMemcpyHostToDevice, h->s_in));
        CUDA_TRY(cudaEventRecord(ev[2 + 2 * c], h->s_in));
        CUDA_TRY(cudaStreamWaitEvent(st, ev[2 + 2 * c], 0));
        if (use_graph) {
            CUDA_TRY(cudaGraphLaunch(hg.exec, st));
        } else {
            occ_status s = occ_forward_expert_parallel(h, xs, gate, prune, nullptr, nc, os, stream);
            if (s != OCC_OK) return s;
        }
        CUDA_TRY(cudaEventRecord(ev[3 + 2 * c], st));
        CUDA_TRY(cudaStreamWaitEvent(h->s_out, ev[3 + 2 * c], 0));
        CUDA_TRY(cudaMemcpyAsync(oh + base * row, os, nc * row, cudaMemcpyDeviceToHost, h->s_out));
        base += nc;
    }
    CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(cudaEventRecord(ev[1], h->s_out));
    h->host_slot_used[slot] = true;
    return OCC_OK;
}

occ_status occ_host_wait(occ_handle* h, occ_stream_t stream) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (!h->s_out) return OCC_OK;
    cudaEvent_t e = h->pev[2 * (2 + 2 * 16)];
    CUDA_TRY(cudaEventRecord(e, h->s_out));
    CUDA_TRY(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), e, 0));
    return OCC_OK;
}

occ_status occ_comm_report_get(occ_handle* h, int bytes_per_scalar, occ_comm_report* rep, occ_stream_t stream) {
    if (!h || !rep) return fail(OCC_ERR_ARG, "null argument");
    if (!h->have_forward) return fail(OCC_ERR_STATE, "no forward to report");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaStreamSynchronize(st));
    std::memset(rep, 0, sizeof(*rep));
    const int nd = h->nd;
    rep->cap_replicas = (double)std::min(h->k, nd);
    // a micro-batched forward reports both halves together
    occ_handle* parts[2] = {h, h->last_split ? h->sib : nullptr};
    long long stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::vector<long long> C(nd * nd, 0);
    long long n = 0;
    for (occ_handle* x : parts) {
        if (!x || x->last_n == 0) continue;
        if (x != h) CUDA_TRY(cudaStreamSynchronize(h->s_mb));
        long long st8[8];
        std::vector<int> Cx(nd * nd);
        CUDA_TRY(cudaMemcpy(st8, x->stats.p, sizeof(st8), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(Cx.data(), x->dofs.C, sizeof(int) * nd * nd, cudaMemcpyDeviceToHost));
        for (int i = 0; i < 8; ++i) stats[i] += st8[i];
        for (int i = 0; i < nd * nd; ++i) C[i] += Cx[i];
        n += x->last_n;
    }
    if (n == 0) return OCC_OK;
    rep->mean_replicas = (double)stats[2] / n;
    const long long pairs = stats[3] + stats[4];
    rep->intra_share = pairs ? (double)stats[3] / pairs : 0.0;
    rep->inter_share = pairs ? (double)stats[4] / pairs : 0.0;
    rep->crossing_rows = stats[0];
    rep->naive_crossing_rows = stats[1];
    rep->cross_device_bytes = stats[0] * (long long)h->D * bytes_per_scalar;
    rep->n_sfd = stats[5];
    rep->n_epd = stats[6];
    for (int d = 0; d < nd; ++d) {
        long long r = 0;
        for (int s2 = 0; s2 < nd; ++s2) r += C[s2 * nd + d];
        rep->per_device_rows[d] = r;
    }
    return OCC_OK;
}

occ_status occ_saved_index(occ_handle* h, int32_t* inbox_token, int32_t* inbox_source, int32_t* inbox_slot,
                           int32_t* cindex, occ_stream_t stream) {
    if (h && h->last_split) return fail(OCC_ERR_STATE, "saved index: the last forward ran as two micro-batches");
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (!h->have_forward) return fail(OCC_ERR_STATE, "no saved forward state");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (h->last_n == 0) return OCC_OK;
    CUDA_TRY(cudaStreamSynchronize(st));
    int R = 0;
    CUDA_TRY(cudaMemcpy(&R, h->dofs.in_base + h->nd, sizeof(int), cudaMemcpyDeviceToHost));
    if (inbox_token) CUDA_TRY(cudaMemcpyAsync(inbox_token, h->in_tok.p, sizeof(int) * R, cudaMemcpyDeviceToDevice, st));
    if (inbox_source) CUDA_TRY(cudaMemcpyAsync(inbox_source, h->in_src.p, sizeof(int) * R, cudaMemcpyDeviceToDevice, st));
    if (inbox_slot) CUDA_TRY(cudaMemcpyAsync(inbox_slot, h->in_slot.p, sizeof(int) * R, cudaMemcpyDeviceToDevice, st));
    if (cindex)
        launch_extract_cindex((int)h->R_max, h->dofs.in_base + h->nd, h->P, h->in_dev.p, h->dofs.in_base,
                              h->row_epd.p, h->cofs, cindex, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(st));
    return OCC_OK;
}

occ_status occ_coactivation_histogram(const int32_t* ids, int n, int k, int e, int64_t* counts, occ_stream_t stream) {
    if ((!ids && n > 0) || !counts) return fail(OCC_ERR_ARG, "null argument");
    if (e < 1 || k < 1 || n < 0) return fail(OCC_ERR_SHAPE, "histogram: need E >= 1, k >= 1, n >= 0");
    launch_histogram(ids, n, k, e, counts, reinterpret_cast<cudaStream_t>(stream));
    CUDA_TRY(cudaGetLastError());
    return OCC_OK;
}

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

occ_status occ_comm_unique_id(void* id128) {
    if (!id128) return fail(OCC_ERR_ARG, "null id buffer");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
    return OCC_OK;
}

occ_status occ_comm_init(occ_handle* h, const void* id128) {
    if (!h || !id128) return fail(OCC_ERR_ARG, "null argument");
    if (h->world == 1) return OCC_OK;  // all devices local: no communicator needed
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    NCCL_TRY(ncclCommInitRank(&comm, h->world, id, h->rank));
    delete h->tp;
    h->tp = new NcclTransport(comm, h->world);
    return OCC_OK;
}

occ_status occ_comm_init_host(occ_handle* h, occ_host_allgather_fn fn, void* ctx) {
    if (!h || !fn) return fail(OCC_ERR_ARG, "null argument");
    if (h->world == 1) return OCC_OK;
    delete h->tp;
    h->tp = new HostTransport(fn, ctx, h->world, h->rank);
    return OCC_OK;
}

occ_status occ_comm_init_loopback(occ_handle* h, long group_key) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (h->world == 1) return OCC_OK;
    std::shared_ptr<LoopGroup> g;
    {
        std::lock_guard<std::mutex> lk(g_loop_m);
        auto& slot = g_loop[group_key];
        if (!slot || slot->world != h->world) slot = std::make_shared<LoopGroup>(h->world);
        g = slot;
    }
    delete h->tp;
    h->tp = new LoopbackTransport(g, h->rank);
    return OCC_OK;
}

// CUDA 12 loads kernels lazily by default (CUDA_MODULE_LOADING); a first
// launch then synchronises with the kernels running in the context.
static bool lazy_module_loading() {
    typedef CUresult (*GetModeFn)(CUmoduleLoadingMode*);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    CUmoduleLoadingMode mode = CU_MODULE_EAGER_LOADING;
    return reinterpret_cast<GetModeFn>(fn)(&mode) == CUDA_SUCCESS && mode == CU_MODULE_LAZY_LOADING;
}

occ_status occ_comm_enable_peer(occ_handle* h, int max_tokens_per_rank) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (h->world == 1) return OCC_OK;
    if (!h->tp) return fail(OCC_ERR_STATE, "peer exchange: call occ_comm_init / occ_comm_init_loopback first");
    if (max_tokens_per_rank < 1) return fail(OCC_ERR_CONFIG, "peer exchange: max_tokens_per_rank must be >= 1");
    if (std::string(h->tp->name()) == "loopback" && lazy_module_loading())
        return fail(OCC_ERR_STATE,
                    "peer exchange between ranks of one process needs CUDA_MODULE_LOADING=EAGER (set before CUDA "
                    "starts): a lazily loaded kernel's first launch waits for the other ranks' spinning arrival waits");
    const int nd = h->nd, k = h->k, P = h->P;
    const size_t per_dev = h->cfg.dedup ? 1 : (size_t)std::min(k, P);   // rows per (token, device)
    const size_t R_cap = (size_t)max_tokens_per_rank * nd * per_dev;
    occ_status s = ensure_ws(h, max_tokens_per_rank);
    if (s != OCC_OK) return s;
    s = ensure_recv(h, R_cap, R_cap * std::min(k, P));
    if (s != OCC_OK) return s;
    // flags: [0, nd) dispatch arrivals, [nd, 2nd) return arrivals, [2nd, 3nd) count rows
    CUDA_TRY(h->flags.ensure(3 * nd));
    CUDA_TRY(cudaMemset(h->flags.p, 0, sizeof(unsigned long long) * 3 * nd));
    CUDA_TRY(h->c_peer.ensure((size_t)nd * nd));
    CUDA_TRY(cudaMemset(h->c_peer.p, 0, sizeof(int) * nd * nd));
    CUDA_TRY(h->peer_tab.ensure((size_t)h->world * kPeerSlots));
    CUDA_TRY(h->peer_seq.ensure(1));
    CUDA_TRY(cudaMemset(h->peer_seq.p, 0, sizeof(unsigned long long)));
    if (h->n_shared > 0 && (s = ensure_shared(h, max_tokens_per_rank)) != OCC_OK) return s;
    CUDA_TRY(cudaDeviceSynchronize());
    const std::vector<void*> mine{h->in_x.p, h->in_ids.p, h->in_w.p, h->y_src.p, h->flags.p, h->c_peer.p};
    std::vector<void*> all;
    for (void* ptr : h->ipc_opened) cudaIpcCloseMemHandle(ptr);
    h->ipc_opened.clear();
    s = h->tp->exchange_pointers(mine, all, h->ipc_opened);
    if (s != OCC_OK) return s;
    CUDA_TRY(cudaMemcpy(h->peer_tab.p, all.data(), sizeof(void*) * all.size(), cudaMemcpyHostToDevice));
    h->peer = true;
    h->peer_cap = max_tokens_per_rank;
    if (h->sib) {
        sync_sibling(h);  // (the sibling pre-sizes the shared-expert buffers too)
        if ((s = occ_comm_enable_peer(h->sib, max_tokens_per_rank)) != OCC_OK) return s;
    }
    return h->tp->barrier();
}

occ_status occ_set_micro_batches(occ_handle* h, int micro_batches, int comm_sms) {
    if (!h) return fail(OCC_ERR_ARG, "null handle");
    if (h->borrowed) return fail(OCC_ERR_STATE, "micro-batches: not on a sibling handle");
    if (micro_batches < 1 || micro_batches > 2) return fail(OCC_ERR_UNSUPPORTED, "micro_batches must be 1 or 2");
    if (micro_batches > 1 && h->training) return fail(OCC_ERR_UNSUPPORTED, "micro-batching is inference-only");
    if (micro_batches == 1) {
        if (h->sib) {
            unborrow(h->sib);
            occ_destroy(h->sib);
            h->sib = nullptr;
        }
        h->mb = 1;
        h->last_split = false;
        h->num_sms = h->full_sms;
        return OCC_OK;
    }
    if (h->world > 1 && !h->tp) return fail(OCC_ERR_STATE, "micro-batches: call occ_comm_init first");
    if (!h->sib) {
        occ_handle* b = nullptr;
        occ_status s = occ_create(&h->cfg, h->plist.data(), h->world, h->rank, &b);
        if (s != OCC_OK) return s;
        b->borrowed = true;
        if (h->world > 1) {
            Transport* t2 = nullptr;
            if ((s = h->tp->split(&t2)) != OCC_OK) {
                occ_destroy(b);
                return s;
            }
            b->tp = t2;
            if (h->peer && (s = occ_comm_enable_peer(b, h->peer_cap)) != OCC_OK) {
                occ_destroy(b);
                return s;
            }
        }
        if (!h->s_mb) {
            CUDA_TRY(cudaStreamCreateWithFlags(&h->s_mb, cudaStreamNonBlocking));
            for (auto& e : h->ev_mb) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        h->sib = b;
    }
    h->mb = 2;
    h->comm_sms = comm_sms >= 0 ? comm_sms : (h->world > 1 ? 16 : 0);
    h->num_sms = std::max(2, (h->full_sms - h->comm_sms) & ~1);
    if (h->world > 1) {  // the sibling's first forward allocates nothing; every rank is set up
        if (h->n_shared > 0) {
            sync_sibling(h);
            occ_status s = ensure_shared(h->sib, h->peer ? h->peer_cap : 1);
            if (s != OCC_OK) return s;
            CUDA_TRY(h->sib->sh_grp.ensure(4));
        }
        return h->tp->barrier();
    }
    return OCC_OK;
}

occ_status occ_allreduce_histogram(occ_handle* h, int64_t* counts, occ_stream_t stream) {
    if (!h || !counts) return fail(OCC_ERR_ARG, "null argument");
    if (h->world == 1) return OCC_OK;
    if (!h->tp) return fail(OCC_ERR_STATE, "occ_comm_init first");
    return h->tp->allreduce_i64(counts, (size_t)h->E * h->E, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace occ {
// Error reporting for the host-only translation unit (occ_host.cpp).
occ_status host_fail(occ_status s, const char* msg) { return fail(s, msg); }
}  // namespace occ
