// occ_kernels.cu — HBM-bound kernels of the Occult EP path on sm_100a:
// dispatch plan (BRIM0), pack (dispatch + exchange placement), compute
// index (BRIM1), gather, intra-device partial combine, combine, the
// co-activation histogram and the routers.  Citations are to
// /root/reference/proj/<file>:<line>.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cstdlib>

#include "occ_common.cuh"
#include "occ_glibc_exp.h"
#include "occ_internal.h"

namespace occ {

long long g_launches = 0;
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("OCC_PDL");
        return !e || atoi(e) != 0;
    }();
    return on;
}

namespace {

constexpr int kRankThreads = kRankChunk;  // one item per thread, 8 warps
constexpr int kRankWarps = kRankThreads / 32;

__device__ __forceinline__ int item_valid(int i, int n_host, const int* n_dev) {
    return i < (n_dev ? *n_dev : n_host);
}

// ------------------------------------------------------------- plan mask --
// Per token (dedup) or per (token, slot) item (naive): source group and
// destination-device mask.  Validates the routing like
// RoutingOutcome::validate (routing.cpp:11-31).
__global__ void plan_mask_kernel(PlanArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n) return;
    const int s = a.src_fixed >= 0 ? 0 : (a.sources ? a.sources[t] : t % a.nd);
    // an invalid token is flagged and planned with no destinations, so nothing
    // downstream indexes by its ids / source (the forward then reports the error)
    auto drop = [&](int code) {
        atomicExch(a.err, code);
        if (a.dedup) { a.mask[t] = 0; a.group[t] = 0; }
        else
            for (int j = 0; j < a.k; ++j) { a.mask[(long)t * a.k + j] = 0; a.group[(long)t * a.k + j] = 0; }
    };
    if (s < 0 || s >= a.nd) { drop(1); return; }  // ShapeError: source out of range
    uint64_t m = 0;
    for (int j = 0; j < a.k; ++j) {
        const int e = a.ids[(long)t * a.k + j];
        const float wt = a.w ? a.w[(long)t * a.k + j] : 1.0f;
        bool bad = e < 0 || e >= a.E || !(wt > 0.0f);
        for (int l = 0; l < j && !bad; ++l) bad = a.ids[(long)t * a.k + l] == e;
        if (bad) { drop(4); return; }  // RoutingError
        const uint64_t bit = 1ull << a.dev_of[e];
        if (a.dedup) m |= bit;
        else { a.mask[(long)t * a.k + j] = bit; a.group[(long)t * a.k + j] = s; }
    }
    if (a.dedup) { a.mask[t] = m; a.group[t] = s; }
}

// ------------------------------------------------------ generic rank core --
// Computes, for the calling warp, its per-key counts into wcnt[warp][key].
__device__ __forceinline__ void warp_key_counts(int valid, int g, uint64_t m, int B, int K, int* wcnt, int warp,
                                                int lane) {
    const uint32_t same = __match_any_sync(0xffffffffu, valid ? g : -1);
    const bool leader = (__ffs(same) - 1) == lane;
    for (int b = 0; b < B; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, valid && ((m >> b) & 1));
        if (valid && leader) wcnt[warp * K + g * (B + 1) + b] = __popc(bal & same);
    }
    if (valid && leader) wcnt[warp * K + g * (B + 1) + B] = __popc(same);
}

__global__ void __launch_bounds__(kRankThreads) rank_count_kernel(int n, const int* n_dev, const int32_t* group,
                                                                  const uint64_t* mask, int G, int B, int* chunk_cnt,
                                                                  int nchunks) {
    extern __shared__ int wcnt[];
    const int K = G * (B + 1);
    for (int i = threadIdx.x; i < kRankWarps * K; i += kRankThreads) wcnt[i] = 0;
    __syncthreads();
    const int i = blockIdx.x * kRankThreads + threadIdx.x;
    const int valid = item_valid(i, n, n_dev);
    const int g = valid ? group[i] : -1;
    const uint64_t m = valid ? mask[i] : 0;
    warp_key_counts(valid, g, m, B, K, wcnt, threadIdx.x >> 5, threadIdx.x & 31);
    __syncthreads();
    for (int key = threadIdx.x; key < K; key += kRankThreads) {
        int s = 0;
        for (int w = 0; w < kRankWarps; ++w) s += wcnt[w * K + key];
        chunk_cnt[(long)key * nchunks + blockIdx.x] = s;
    }
}

// One block per key: exclusive scan of the per-chunk counts.
__global__ void __launch_bounds__(1024) rank_scan_kernel(int* chunk_cnt, int nchunks, int* totals) {
    __shared__ int warp_sums[32];
    const int key = blockIdx.x;
    int* row = chunk_cnt + (long)key * nchunks;
    const int per = (nchunks + 1023) / 1024;
    const int c0 = threadIdx.x * per;
    int local = 0;
    for (int c = c0; c < c0 + per && c < nchunks; ++c) local += row[c];
    // block exclusive scan of `local`
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int v = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int ws = warp_sums[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += u;
        }
        warp_sums[lane] = ws;  // inclusive
    }
    __syncthreads();
    int run = v - local + (warp ? warp_sums[warp - 1] : 0);
    for (int c = c0; c < c0 + per && c < nchunks; ++c) {
        const int x = row[c];
        row[c] = run;
        run += x;
    }
    if (threadIdx.x == 1023) totals[key] = run;
}

// Phase 3: in-chunk ranks, handed to an emitter.
template <class Emit>
__global__ void __launch_bounds__(kRankThreads) rank_emit_kernel(int n, const int* n_dev, const int32_t* group,
                                                                 const uint64_t* mask, int G, int B,
                                                                 const int* chunk_cnt, int nchunks, Emit em) {
    extern __shared__ int wcnt[];
    const int K = G * (B + 1);
    for (int i = threadIdx.x; i < kRankWarps * K; i += kRankThreads) wcnt[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * kRankThreads + threadIdx.x;
    const int valid = item_valid(i, n, n_dev);
    const int g = valid ? group[i] : -1;
    const uint64_t m = valid ? mask[i] : 0;
    warp_key_counts(valid, g, m, B, K, wcnt, warp, lane);
    __syncthreads();
    for (int key = threadIdx.x; key < K; key += kRankThreads) {
        int run = chunk_cnt[(long)key * nchunks + blockIdx.x];
        for (int w = 0; w < kRankWarps; ++w) {
            const int x = wcnt[w * K + key];
            wcnt[w * K + key] = run;
            run += x;
        }
    }
    __syncthreads();
    const uint32_t same = __match_any_sync(0xffffffffu, valid ? g : -1);
    const uint32_t lt = lanemask_lt();
    if (valid) em.group_rank(i, g, wcnt[warp * K + g * (B + 1) + B] + __popc(same & lt));
    for (int b = 0; b < B; ++b) {
        const bool hit = valid && ((m >> b) & 1);
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (hit) em.emit(i, g, b, wcnt[warp * K + g * (B + 1) + b] + __popc(bal & same & lt));
        else if (valid) em.miss(i, b);
    }
}

size_t rank_smem(int G, int B) { return sizeof(int) * (size_t)kRankWarps * G * (B + 1); }

template <class Emit>
void launch_rank_emit(int n_host, const int* n_dev, const int32_t* group, const uint64_t* mask, int G, int B,
                      RankWs ws, const Emit& em, cudaStream_t st) {
    const int nchunks = (n_host + kRankChunk - 1) / kRankChunk;
    if (nchunks == 0) return;
    const size_t smem = rank_smem(G, B);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rank_emit_kernel<Emit>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rank_emit_kernel<Emit><<<nchunks, kRankThreads, smem, st>>>(n_host, n_dev, group, mask, G, B, ws.chunk_cnt,
                                                                nchunks, em);
    count_launch();
}

// ---------------------------------------------------------- dispatch plan --
// From the per-key totals (key = s*(nd+1)+d) derive every offset of
// build_dispatch_index (pipeline.cpp:24-50: counters device-major per
// source) and all_to_all_exchange (pipeline.cpp:153-174: inbox of d is
// ordered by (source asc, counter asc)).
__global__ void dispatch_finalize_kernel(int nd, const int* totals, DispatchOffsets o) {
    const int tid = threadIdx.x;
    for (int i = tid; i < nd * nd; i += blockDim.x) {
        const int s = i / nd, d = i % nd;
        o.C[i] = totals[s * (nd + 1) + d];
    }
    __syncthreads();
    if (tid < nd) {  // per source: row scan
        const int s = tid;
        int run = 0;
        for (int d = 0; d < nd; ++d) {
            o.off_sd[s * nd + d] = run;
            run += o.C[s * nd + d];
        }
        o.nsfd[s] = run;
        o.ntok[s] = totals[s * (nd + 1) + nd];
    } else if (tid >= 64 && tid < 64 + nd) {  // per destination: column scan
        const int d = tid - 64;
        int run = 0;
        for (int s = 0; s < nd; ++s) {
            o.inoff[d * nd + s] = run;
            run += o.C[s * nd + d];
        }
        o.in_base[d] = run;  // temporarily R_d
    }
    __syncthreads();
    if (tid == 0) {
        int run = 0;
        for (int d = 0; d < nd; ++d) {
            const int r = o.in_base[d];
            o.in_base[d] = run;
            run += r;
        }
        o.in_base[nd] = run;
        run = 0;
        long long cross = 0;
        for (int s = 0; s < nd; ++s) {
            o.src_base[s] = run;
            run += o.nsfd[s];
            for (int d = 0; d < nd; ++d)
                if (d != s) cross += o.C[s * nd + d];
        }
        o.src_base[nd] = run;
        o.stats[0] = cross;
        o.stats[5] = run;
    }
}

__device__ __forceinline__ int token_source(const EmitDispatch& e, int t) {
    return e.src_fixed >= 0 ? e.src_fixed : (e.sources ? e.sources[t] : t % e.nd);
}

struct DispatchEmitter {
    EmitDispatch e;
    __device__ void group_rank(int i, int, int r) {
        if (e.dedup) e.lam[i] = r;
    }
    __device__ void emit(int i, int, int d, int r) {
        const int t = e.dedup ? i : i / e.k;
        const int s = token_source(e, t);
        const int c = e.o.off_sd[s * e.nd + d] + r;  // BRIM0 counter
        const long slot = e.dedup ? (long)t * e.nd + d : (long)i;
        e.tok_sfd[slot] = c;
        if (e.world1) {
            const int row = e.o.in_base[d] + e.o.inoff[d * e.nd + s] + r;
            e.tok_row[slot] = row;
            e.in_tok[row] = t;
            e.in_src[row] = s;
            e.in_slot[row] = c;
            e.in_dev[row] = d;
        } else {
            e.tok_row[slot] = c;  // send buffer is the Sfd batch (device-major)
        }
    }
    __device__ void miss(int i, int d) {
        if (!e.dedup) return;
        e.tok_sfd[(long)i * e.nd + d] = -1;
        e.tok_row[(long)i * e.nd + d] = -1;
    }
};

// BRIM0 per source: nd x n_s, column = local token index.
__global__ void extract_brim0_kernel(int n, int nd, const int32_t* sources, int src_fixed, const uint64_t* mask,
                                     const int32_t* lam, const int32_t* tok_sfd, const int* src_tok_base,
                                     const int* ntok, int32_t* brim0) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)n * nd) return;
    const int t = (int)(i / nd), d = (int)(i % nd);
    const int s = src_fixed >= 0 ? 0 : (sources ? sources[t] : t % nd);
    const long base = (long)src_tok_base[s] * nd;
    brim0[base + (long)d * ntok[s] + lam[t]] = ((mask[t] >> d) & 1) ? tok_sfd[(long)t * nd + d] : -1;
}

// ------------------------------------------------------------------ pack ---
// dispatch (pipeline.cpp:91-123) fused with the exchange placement
// (pipeline.cpp:154-174): each token row is read once from HBM and written
// to every destination row (one per device under dedup), with its routing
// row alongside.  One warp per token, 16-byte vectors, 8 vectors in flight
// per lane.
constexpr int kPackVec = 8;  // 16-byte vectors per lane in flight in the pack kernels

__device__ __forceinline__ void pack_token(const PackArgs& a, int t, int lane) {
    const int nvec = a.D / 8;
    const uint4* src = reinterpret_cast<const uint4*>(a.x + (long)t * a.D);
    // the row's first slice is in flight while the destination rows resolve
    // (mask -> tok_row is a dependent chain of two loads)
    uint4 buf[kPackVec];
    if (a.dst_x) {
#pragma unroll
        for (int u = 0; u < kPackVec; ++u) {
            const int v = u * 32 + lane;
            if (v < nvec) buf[u] = __ldg(src + v);
        }
    }
    int rows[kMaxDev];
    int nrows = 0;
    if (a.dedup) {
        uint64_t m = a.mask[t];
        while (m) {
            const int d = __ffsll(m) - 1;
            m &= m - 1;
            rows[nrows++] = a.tok_row[(long)t * a.nd + d];
        }
    } else {
        for (int j = 0; j < a.k; ++j)
            if (a.mask[(long)t * a.k + j]) rows[nrows++] = a.tok_row[(long)t * a.k + j];
    }
    // the whole row in flight (16 x 16 B per lane covers D = 4096 in one round trip)
    for (int v0 = 0; a.dst_x && v0 < nvec; v0 += kPackVec * 32) {
        if (v0) {
#pragma unroll
            for (int u = 0; u < kPackVec; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < nvec) buf[u] = __ldg(src + v);
            }
        }
        for (int q = 0; q < nrows; ++q) {
            uint4* dst = reinterpret_cast<uint4*>(a.dst_x + (long)rows[q] * a.D);
#pragma unroll
            for (int u = 0; u < kPackVec; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < nvec) dst[v] = buf[u];
            }
        }
    }
    // (a token's naive rows are all kept or all dropped, so row q carries slot q)
    for (int q = 0; a.dst_ids && q < nrows; ++q) {
        for (int j = lane; j < a.k; j += 32) {
            const long di = (long)rows[q] * a.k + j;
            const bool keep = a.dedup || j == q;  // naive rows carry only their own expert
            a.dst_ids[di] = keep ? a.ids[(long)t * a.k + j] : -1;
            a.dst_w[di] = keep ? a.w[(long)t * a.k + j] : 0.0f;
        }
    }
}

// persistent: one warp per token, grid-stride over the tokens (no partial
// last wave of blocks)
__global__ void __launch_bounds__(256) pack_kernel(PackArgs a) {
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < a.n; t += (gridDim.x * blockDim.x) >> 5)
        pack_token(a, t, lane);
}

// -------------------------------------------------------- compute index ---
// Per received Sfd row: local-expert mask in placement-list slots
// (pipeline.cpp:409-421) and validation (build_compute_index rejects rows
// with no local expert, pipeline.cpp:66-69).
__global__ void compute_mask_kernel(ComputeArgs a) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= *a.R_total) return;
    const int dl = a.row_dev ? a.row_dev[r] : 0;
    const int gdev = a.dev_base + dl;
    uint64_t m = 0;
    for (int j = 0; j < a.k; ++j) {
        const int e = a.row_ids[(long)r * a.k + j];
        if (e >= 0 && a.dev_of[e] == gdev) m |= 1ull << a.slot_of[e];
    }
    if (!m) atomicExch(a.err, 4);
    a.mask[r] = m;
    a.group[r] = dl;
}

// Epd segment layout: group g = (local device, slot) in placement-list
// order (pipeline.cpp:79-86, expert-major counters); each segment padded
// to the GEMM M tile so no tile straddles two experts.
__global__ void compute_finalize_kernel(int G, int P, const int* totals, ComputeOffsets o) {
    const int NG = G * P;
    for (int g = threadIdx.x; g < NG; g += blockDim.x) {
        const int d = g / P, p = g % P;
        o.cnt[g] = totals[d * (P + 1) + p];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0, mb = 0;
        long long nepd = 0;
        for (int g = 0; g < NG; ++g) {
            const int m = (o.cnt[g] + kBM - 1) / kBM;
            o.seg_base[g] = run;
            o.grp_mb[g] = mb;
            run += m * kBM;
            mb += m;
            nepd += o.cnt[g];
        }
        o.grp_mb[NG] = mb;
        for (int d = 0; d < G; ++d) {
            int u = 0;
            for (int p = 0; p < P; ++p) {
                o.unp_base[d * P + p] = u;
                u += o.cnt[d * P + p];
            }
        }
        *o.n_mblk = mb;
        *o.q_total = run;
        o.stats[6] += nepd;
    }
}

struct ComputeEmitter {
    EmitCompute e;
    uint32_t slots[2];  // k <= 8: local slot of routing entry j in byte j (0xFF: other device)
    __device__ void group_rank(int r, int g, int) {
        if (e.k > 8) return;
        const int gdev = e.dev_base + g;
        slots[0] = slots[1] = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= e.k) break;
            const int ex = e.row_ids[(long)r * e.k + j];
            if (ex >= 0 && e.dev_of[ex] == gdev) {
                const uint32_t sh = 8 * (j & 3);
                slots[j >> 2] = (slots[j >> 2] & ~(0xFFu << sh)) | ((uint32_t)e.slot_of[ex] << sh);
            }
        }
    }
    __device__ void emit(int r, int g, int p, int rank) {
        const int q = e.o.seg_base[g * e.P + p] + rank;
        e.row_epd[(long)r * e.P + p] = q;
        e.epd_src[q] = r;
        int jj = -1;
        if (e.k <= 8) {  // slot -> routing entry from the packed bytes (no loads)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (jj < 0 && ((slots[j >> 2] >> (8 * (j & 3))) & 0xFFu) == (uint32_t)p) jj = j;
        } else {
            const int gdev = e.dev_base + g;
            for (int j = 0; j < e.k; ++j) {
                const int ex = e.row_ids[(long)r * e.k + j];
                if (ex >= 0 && e.dev_of[ex] == gdev && e.slot_of[ex] == p) {
                    jj = j;
                    break;
                }
            }
        }
        e.epd_w[q] = jj >= 0 ? e.row_w[(long)r * e.k + jj] : 0.0f;
        if (e.epd_j) e.epd_j[q] = jj;
    }
    __device__ void miss(int, int) {}  // row_epd is pre-filled with -1 (launch_rank_emit_compute)
};

__global__ void init_epd_kernel(int Q, int32_t* src, float* w) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < Q) { src[q] = -1; w[q] = 0.0f; }
}

// Scatter (replaces the Epd-order gather): each inbox row is read ONCE and
// written to every Epd row that uses it (its local experts, placement order)
// — n_epd row writes but only R row reads, instead of n_epd scattered reads.
// src row of inbox row r = src_rows ? src_rows[r] : r (world_size == 1 reads
// the tokens themselves: src = x, src_rows = inbox token).
__global__ void __launch_bounds__(256) scatter_rows_kernel(int R_max, const int* R_total, int P, int D,
                                                           const __nv_bfloat16* src, const int32_t* src_rows,
                                                           const int32_t* row_epd, __nv_bfloat16* dst) {
    pdl_trigger();
    pdl_wait();  // launched with PDL: inputs come from the previous kernel
    // one warp per (row, 2 KB slice): 4 uint4 per lane in flight
    constexpr int kSlice = 128;  // uint4 per slice
    const int nvec = D / 8;
    const int nsl = (nvec + kSlice - 1) / kSlice;
    const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int r = (int)(w / nsl), sl = (int)(w % nsl);
    if (r >= *R_total) return;
    const int sr = src_rows ? src_rows[r] : r;
    const uint4* in = reinterpret_cast<const uint4*>(src + (long)sr * D);
    // destinations: lane p holds row_epd[r, p] (P <= 64: two words)
    const int q_lo = lane < P ? row_epd[(long)r * P + lane] : -1;
    const int q_hi = lane + 32 < P ? row_epd[(long)r * P + lane + 32] : -1;
    const unsigned m_lo = __ballot_sync(0xffffffffu, q_lo >= 0), m_hi = __ballot_sync(0xffffffffu, q_hi >= 0);
    const int v0 = sl * kSlice;
    uint4 buf[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < nvec) buf[u] = __ldg(in + v);
    }
    for (int half = 0; half < 2; ++half) {
        unsigned m = half ? m_hi : m_lo;
        while (m) {
            const int p = __ffs(m) - 1;
            m &= m - 1;
            const int q = __shfl_sync(0xffffffffu, half ? q_hi : q_lo, p);
            uint4* out = reinterpret_cast<uint4*>(dst + (long)q * D);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < nvec) out[v] = buf[u];
            }
        }
    }
}

// Zero the padding rows of every Epd segment (rows cnt..roundup(cnt, kBM)).
__global__ void __launch_bounds__(256) zero_pad_rows_kernel(int NG, ComputeOffsets o, int D, __nv_bfloat16* dst) {
    pdl_trigger();
    pdl_wait();  // launched with PDL: inputs come from the previous kernel
    const int g = blockIdx.x;
    if (g >= NG) return;
    const int cnt = o.cnt[g];
    const int pad = (cnt + kBM - 1) / kBM * kBM - cnt;
    if (!pad) return;
    uint4* base = reinterpret_cast<uint4*>(dst + (long)(o.seg_base[g] + cnt) * D);
    const long nvec = (long)pad * D / 8;
    for (long v = (long)blockIdx.y * blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.y * blockDim.x)
        base[v] = make_uint4(0, 0, 0, 0);
}

// ------------------------------------------------------- partial combine --
// merge_matmul's per-row sum over local experts (pipeline.cpp:263-281),
// done after the grouped GEMM: ascending placement-list order, fp32.

#ifndef OCC_CMB_VEC
#define OCC_CMB_VEC 8  // row vectors in flight per lane in the ordered row sums (KU rows x OCC_CMB_VEC / KU)
#endif
// Streaming 16-byte store (evict-first): the combine / return outputs are
// written once and not re-read by this layer (profiles/probes/hbm_pattern_probe.cu:
// 2-rows-in / 1-row-out at 5.6 TB/s with plain stores, 6.0 TB/s with .cs).
__device__ __forceinline__ void st_stream(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void add_bf16x8(float* a, const uint4& u) {
    const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(hh[e]);
        a[2 * e] += f.x;
        a[2 * e + 1] += f.y;
    }
}

// Ordered sum of nq bf16 rows Y[qs[0..nq)] (+ an optional extra row), fp32,
// rounded to bf16.  GROUPS: bit i of `opens` starts a new group at entry i;
// each group's partial sum is rounded to bf16 (the payload the multi-GPU
// return would carry) before it is added, so one-GPU results equal the
// exchanged path bit for bit.  Per element the summation order is the list
// order in every configuration.  A lane keeps V 16-byte vectors of each of KU
// rows in flight (KU x V loads per round trip; V x 512 B per warp and row).
// ROUND_FIRST (one group, then the extra row): the rows' sum is rounded to
// bf16 before the extra row is added -- GROUPS with a single group, without
// the second accumulator.
template <int KU, int V, bool GROUPS, bool ROUND_FIRST = false>
__device__ __forceinline__ void sum_rows_v(const __nv_bfloat16* Y, const int* qs, int nq, uint64_t opens, int D,
                                           int lane, const __nv_bfloat16* extra, __nv_bfloat16* dst) {
    const int nv = D / 8;
    for (int v0 = 0; v0 < nv; v0 += 32 * V) {
        float acc[V][8], grp[GROUPS ? V : 1][8];
#pragma unroll
        for (int w = 0; w < V; ++w)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                acc[w][e] = 0.f;
                if constexpr (GROUPS) grp[w][e] = 0.f;
            }
        for (int i0 = 0; i0 < nq; i0 += KU) {
            uint4 u[KU][V];
#pragma unroll
            for (int j = 0; j < KU; ++j)
                if (i0 + j < nq) {
                    const uint4* r = reinterpret_cast<const uint4*>(Y + (long)qs[i0 + j] * D) + v0 + lane;
#pragma unroll
                    for (int w = 0; w < V; ++w)
                        if (v0 + lane + 32 * w < nv) u[j][w] = __ldg(r + 32 * w);
                }
#pragma unroll
            for (int j = 0; j < KU; ++j) {
                if (i0 + j >= nq) break;
                if constexpr (GROUPS) {
                    if (i0 + j && i0 + j < 64 && ((opens >> (i0 + j)) & 1)) {
#pragma unroll
                        for (int w = 0; w < V; ++w)
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                acc[w][e] += __bfloat162float(__float2bfloat16(grp[w][e]));
                                grp[w][e] = 0.f;
                            }
                    }
#pragma unroll
                    for (int w = 0; w < V; ++w) add_bf16x8(grp[w], u[j][w]);
                } else {
#pragma unroll
                    for (int w = 0; w < V; ++w) add_bf16x8(acc[w], u[j][w]);
                }
            }
        }
#pragma unroll
        for (int w = 0; w < V; ++w) {
            const int vv = v0 + lane + 32 * w;
            if (vv >= nv) break;
            if constexpr (GROUPS) {
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[w][e] += __bfloat162float(__float2bfloat16(grp[w][e]));
            }
            if constexpr (ROUND_FIRST) {
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[w][e] = __bfloat162float(__float2bfloat16(acc[w][e]));
            }
            if (extra) add_bf16x8(acc[w], __ldg(reinterpret_cast<const uint4*>(extra) + vv));
            uint4 o;
            o.x = pack_bf16(acc[w][0], acc[w][1]);
            o.y = pack_bf16(acc[w][2], acc[w][3]);
            o.z = pack_bf16(acc[w][4], acc[w][5]);
            o.w = pack_bf16(acc[w][6], acc[w][7]);
            st_stream(reinterpret_cast<uint4*>(dst) + vv, o);
        }
    }
}

// Sum of nq bf16 rows (indices in shared memory, summed in list order, fp32)
// + an optional extra row, rounded to bf16: KU rows x (8 / KU) vectors in flight.
template <int KU>
__device__ __forceinline__ void sum_rows_ordered(const __nv_bfloat16* Y, const int* qs, int nq, int D, int lane,
                                                 const __nv_bfloat16* extra, __nv_bfloat16* dst) {
    sum_rows_v<KU, (KU >= 8 ? 1 : OCC_CMB_VEC / KU), false>(Y, qs, nq, 0, D, lane, extra, dst);
}

// Append the non-negative entries of idx[0..cnt) (lane-parallel, order kept)
// to the warp's list qs[nq..]; returns the new length.
__device__ __forceinline__ int warp_compact_append(const int32_t* idx, int cnt, int* qs, int nq, int cap, int lane) {
    const uint32_t lt = (1u << lane) - 1u;
    for (int p0 = 0; p0 < cnt; p0 += 32) {
        const int q = p0 + lane < cnt ? idx[p0 + lane] : -1;
        const uint32_t b = __ballot_sync(0xffffffffu, q >= 0);
        const int pos = nq + __popc(b & lt);
        if (q >= 0 && pos < cap) qs[pos] = q;
        nq += __popc(b);
    }
    return nq < cap ? nq : cap;
}

// merge_matmul's per-row sum over local experts (pipeline.cpp:263-281),
// done after the grouped GEMM: ascending placement-list order, fp32.
template <int KU>
__global__ void __launch_bounds__(256) partial_combine_kernel(int R_max, const int* R_total, int P, int D,
                                                              const int32_t* row_epd, const __nv_bfloat16* Y,
                                                              __nv_bfloat16* ret) {
    __shared__ int s_q[8][kMaxLocal];
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= *R_total) return;
    int* qs = s_q[threadIdx.x >> 5];
    const int nq = warp_compact_append(row_epd + (long)r * P, P, qs, 0, kMaxLocal, lane);
    __syncwarp();
    sum_rows_ordered<KU>(Y, qs, nq, D, lane, nullptr, ret + (long)r * D);
}

// ---------------------------------------------------------------- combine --
// combine (pipeline.cpp:285-300): Ori row = sum over devices ascending of
// the returned rows; fp32 accumulation, bf16 out; shared-expert rows added last.
template <int KU>
__global__ void __launch_bounds__(256) combine_kernel(int n, int nd, int k, int dedup, int D, const uint64_t* mask,
                                                      const int32_t* tok_row, const __nv_bfloat16* ret,
                                                      const __nv_bfloat16* ys, __nv_bfloat16* out) {
    __shared__ int s_q[8][kMaxDev];
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n) return;
    int* qs = s_q[threadIdx.x >> 5];
    int nr = 0;
    if (dedup) {  // devices ascending: tok_row of the devices in the token's mask
        const uint64_t m = mask[t];
        for (int d0 = 0; d0 < nd; d0 += 32) {
            const int d = d0 + lane;
            const int rr = d < nd && ((m >> d) & 1) ? tok_row[(long)t * nd + d] : -1;
            const uint32_t b = __ballot_sync(0xffffffffu, rr >= 0);
            const int pos = nr + __popc(b & ((1u << lane) - 1u));
            if (rr >= 0 && pos < kMaxDev) qs[pos] = rr;
            nr += __popc(b);
        }
        nr = nr < kMaxDev ? nr : kMaxDev;
    } else {
        nr = warp_compact_append(tok_row + (long)t * k, k, qs, 0, kMaxDev, lane);
    }
    __syncwarp();
    sum_rows_ordered<KU>(ret, qs, nr, D, lane, ys ? ys + (long)t * D : nullptr, out + (long)t * D);
}

// ------------------------------------------------- stage-level entry points --
// dispatch (pipeline.cpp:91-123) of one source's tokens from its BRIM0
// (N_d x n, device-major counters): Sfd row c = BRIM0[d, i] >= 0 receives x
// row i, the full routing row and the token index.  One warp per token: the
// x row is read once (16-byte vectors) and stored to each of its Sfd rows.
__global__ void __launch_bounds__(256) dispatch_sfd_kernel(int n, int nd, int k, int D, const __nv_bfloat16* x,
                                                           const int32_t* ids, const float* w, const int32_t* brim0,
                                                           __nv_bfloat16* sfd_x, int32_t* sfd_ids, float* sfd_w,
                                                           int32_t* sfd_tok) {
    __shared__ int s_c[8][kMaxDev];
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int* cs = s_c[threadIdx.x >> 5];
    int nc = 0;
    for (int d0 = 0; d0 < nd; d0 += 32) {
        const int d = d0 + lane;
        const int c = d < nd ? brim0[(long)d * n + i] : -1;
        const uint32_t b = __ballot_sync(0xffffffffu, c >= 0);
        if (c >= 0) cs[nc + __popc(b & ((1u << lane) - 1u))] = c;
        nc += __popc(b);
    }
    __syncwarp();
    const int nv = D / 8;
    const uint4* src = reinterpret_cast<const uint4*>(x + (long)i * D);
    for (int v = lane; v < nv; v += 32) {
        const uint4 u = __ldg(src + v);
        for (int j = 0; j < nc; ++j) reinterpret_cast<uint4*>(sfd_x + (long)cs[j] * D)[v] = u;
    }
    for (int j = 0; j < nc; ++j) {
        const long c = cs[j];
        for (int q = lane; q < k; q += 32) {
            sfd_ids[c * k + q] = ids[(long)i * k + q];
            sfd_w[c * k + q] = w[(long)i * k + q];
        }
        if (lane == 0) sfd_tok[c] = i;
    }
}

// combine (pipeline.cpp:285-300) from BRIM0: Ori row i = bf16( sum over
// devices ascending of returned Sfd row BRIM0[d, i] ), fp32 accumulation.
template <int KU>
__global__ void __launch_bounds__(256) combine_brim0_kernel(int n, int nd, int D, const int32_t* brim0,
                                                            const __nv_bfloat16* y, __nv_bfloat16* out) {
    __shared__ int s_q[8][kMaxDev];
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int* qs = s_q[threadIdx.x >> 5];
    int nq = 0;
    for (int d0 = 0; d0 < nd; d0 += 32) {
        const int d = d0 + lane;
        const int c = d < nd ? brim0[(long)d * n + i] : -1;
        const uint32_t b = __ballot_sync(0xffffffffu, c >= 0);
        if (c >= 0) qs[nq + __popc(b & ((1u << lane) - 1u))] = c;
        nq += __popc(b);
    }
    __syncwarp();
    sum_rows_ordered<KU>(y, qs, nq, D, lane, nullptr, out + (long)i * D);
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// world_size > 1 backward, dispatch adjoint at the source (backward.cpp:143-152):
// g_x[t] = sum over the token's returned rows (devices ascending) of the
// scatter-adjoint partial sums, and g_weights[t, j] = sum over the same rows
// of their routing-weight gradients (exactly one row holds slot j), fp32.
template <class OutT>
__global__ void __launch_bounds__(256) combine_back_kernel(int n, int nd, int k, int dedup, int D,
                                                           const uint64_t* mask, const int32_t* tok_row,
                                                           const __nv_bfloat16* y, const float* ygw, OutT* gx,
                                                           float* gw) {
    __shared__ int s_q[8][kMaxTopK > kMaxDev ? kMaxTopK : kMaxDev];
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n) return;
    int* qs = s_q[threadIdx.x >> 5];
    int nr = 0;
    const uint32_t lt = (1u << lane) - 1u;
    if (dedup) {
        const uint64_t m = mask[t];
        for (int d0 = 0; d0 < nd; d0 += 32) {
            const int d = d0 + lane;
            const int rr = d < nd && ((m >> d) & 1) ? tok_row[(long)t * nd + d] : -1;
            const uint32_t b = __ballot_sync(0xffffffffu, rr >= 0);
            if (rr >= 0) qs[nr + __popc(b & lt)] = rr;
            nr += __popc(b);
        }
    } else {
        for (int j0 = 0; j0 < k; j0 += 32) {
            const int j = j0 + lane;
            const int rr = j < k && mask[(long)t * k + j] ? tok_row[(long)t * k + j] : -1;
            const uint32_t b = __ballot_sync(0xffffffffu, rr >= 0);
            if (rr >= 0) qs[nr + __popc(b & lt)] = rr;
            nr += __popc(b);
        }
    }
    __syncwarp();
    for (int v = lane; v < D / 8; v += 32) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < nr; ++i) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(y + (long)qs[i] * D) + v);
            const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(hh[e]);
                acc[2 * e] += f.x;
                acc[2 * e + 1] += f.y;
            }
        }
        if constexpr (sizeof(OutT) == 4) {
            float4* o = reinterpret_cast<float4*>(gx + (long)t * D) + 2 * v;
            o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {
            uint4 o;
            o.x = pack_bf16(acc[0], acc[1]);
            o.y = pack_bf16(acc[2], acc[3]);
            o.z = pack_bf16(acc[4], acc[5]);
            o.w = pack_bf16(acc[6], acc[7]);
            reinterpret_cast<uint4*>(gx + (long)t * D)[v] = o;
        }
    }
    for (int j = lane; j < k; j += 32) {
        float s = 0.f;
        for (int i = 0; i < nr; ++i) s += ygw[(long)qs[i] * k + j];
        gw[(long)t * k + j] = s;
    }
}

// One source's BRIM0 (world_size > 1: this rank's tokens) from the plan:
// brim0[d, t] = counter of token t on device d, or -1.
__global__ void brim0_one_source_kernel(int n, int nd, const uint64_t* mask, const int32_t* tok_sfd, int32_t* brim0) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)n * nd) return;
    const int d = (int)(i / n), t = (int)(i % n);
    brim0[i] = ((mask[t] >> d) & 1) ? tok_sfd[(long)t * nd + d] : -1;
}

// Rank-key totals of one source (row 0, from a G = 1 count) moved to row r,
// every other source's row zero: the local dispatch plan of rank r.
__global__ void one_source_totals_kernel(int nd, int r, int* totals) {
    __shared__ int row[kMaxDev + 1];
    for (int d = threadIdx.x; d <= nd; d += blockDim.x) row[d] = totals[d];
    __syncthreads();
    for (int i = threadIdx.x; i < nd * (nd + 1); i += blockDim.x) totals[i] = i / (nd + 1) == r ? row[i % (nd + 1)] : 0;
}

// world_size == 1: intra-device partial combine + return + combine in one
// pass.  Each token gathers its k Epd product rows (exactly one per selected
// expert) ordered by device ascending, then placement slot; every device's
// partial sum is rounded to the bf16 return payload exactly as the
// multi-GPU exchange would carry it, then summed over devices in fp32.
// The token's row list is built warp-parallel (lane p reads row_epd[r, p],
// ballot-compacted into shared memory); KU product rows are in flight per
// 16-byte vector (KU = 2 / 4 / 8 picked from k at launch).
// GROUPED = 0 (one device): every row of a token is one group, so the plain
// ordered sum gives the same bits with half the accumulators (more warps
// resident, more row loads in flight) -- bf16(bf16(sum)) == bf16(sum), and
// with shared experts the sum is rounded before their row is added
// (ROUND_FIRST), exactly what the one-group grouped sum does.
template <int KU, bool GROUPED>
__global__ void __launch_bounds__(256) combine_fused_kernel(int n, int nd, int k, int P, int dedup, int D,
                                                            const uint64_t* mask, const int32_t* tok_row,
                                                            const int32_t* row_epd, const __nv_bfloat16* Y,
                                                            const __nv_bfloat16* ys, __nv_bfloat16* out) {
    pdl_trigger();
    pdl_wait();  // launched with PDL: inputs come from the previous kernel
    __shared__ int s_q[8][kMaxTopK];
    const int wib = threadIdx.x >> 5;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n) return;
    int* qs = s_q[wib];
    uint64_t newdev = 0;  // bit i: entry i opens a new device group
    int nq = 0;
    const uint32_t lt = (1u << lane) - 1u;
    auto add_row = [&](int r) {  // the row's local experts, placement order
        for (int p0 = 0; p0 < P; p0 += 32) {
            const int q = p0 + lane < P ? row_epd[(long)r * P + p0 + lane] : -1;
            const uint32_t b = __ballot_sync(0xffffffffu, q >= 0);
            if (q >= 0 && nq + __popc(b & lt) < kMaxTopK) qs[nq + __popc(b & lt)] = q;
            nq += __popc(b);
        }
    };
    if (dedup) {
        uint64_t m = mask[t];
        while (m) {
            const int d = __ffsll(m) - 1;
            m &= m - 1;
            if (nq < 64) newdev |= 1ull << nq;
            add_row(tok_row[(long)t * nd + d]);
        }
    } else {
        for (int j = 0; j < k; ++j) {
            if (nq < 64) newdev |= 1ull << nq;
            add_row(tok_row[(long)t * k + j]);
        }
    }
    nq = nq < kMaxTopK ? nq : kMaxTopK;
    __syncwarp();
    // devices in ascending order, each device's rows rounded to the bf16 return
    // payload, the shared-expert row last
    sum_rows_v<KU, (KU >= 8 ? 1 : OCC_CMB_VEC / KU), GROUPED, !GROUPED>(Y, qs, nq, newdev, D, lane,
                                                                       ys ? ys + (long)t * D : nullptr,
                                                                       out + (long)t * D);
}

// ------------------------------------------------- peer-memory exchange ---
// world_size > 1 without a collective library on the data path: every rank's
// inbox / return buffers are mapped into every other rank's address space
// (CUDA IPC over NVLink / NVSwitch, or plain pointers for the single-GPU
// loopback ranks), and the dispatch pack and the return partial combine store
// straight into the peer's buffers — the all-to-all is fused into the
// producing kernel.  Table layout: peer_tab[p * kPeerSlots + i].
constexpr int kPeerInX = 0, kPeerInIds = 1, kPeerInW = 2, kPeerYSrc = 3, kPeerFlags = 4, kPeerCounts = 5;
static_assert(kPeerSlots == 6, "peer table slots");

// Count all-gather over peer memory: this source's Sfd row counts per
// destination (rank-key totals row 0) stored as row `me` of every peer's
// (source, destination) count matrix.
__global__ void peer_counts_kernel(void* const* peer_tab, int nd, int me, const int* totals) {
    for (int i = threadIdx.x; i < nd * nd; i += blockDim.x) {
        const int p = i / nd, d = i % nd;
        int* cp = reinterpret_cast<int*>(peer_tab[p * kPeerSlots + kPeerCounts]);
        cp[me * nd + d] = totals[d];
    }
}

// pack_kernel, but rows go directly to each destination's inbox:
// row = inoff[d][me] + (BRIM0 counter - off_sd[me][d]) (all_to_all_exchange
// order: source ascending, counter ascending, pipeline.cpp:153-174).
__device__ __forceinline__ void peer_pack_token(const PackArgs& a, int me, const int32_t* dev_of, const int* off_sd,
                                                const int* inoff, void* const* peer_tab, int t, int lane) {
    const int nvec = a.D / 8;
    const uint4* src = reinterpret_cast<const uint4*>(a.x + (long)t * a.D);
    uint4 buf[kPackVec];  // the row's first slice in flight while the destination rows resolve
#pragma unroll
    for (int u = 0; u < kPackVec; ++u) {
        const int v = u * 32 + lane;
        if (v < nvec) buf[u] = __ldg(src + v);
    }
    int nrow = 0, dsts[kMaxTopK], rows[kMaxTopK], jsel[kMaxTopK];
    if (a.dedup) {  // one row per destination device
        uint64_t m = a.mask[t];
        while (m) {
            const int d = __ffsll(m) - 1;
            m &= m - 1;
            dsts[nrow] = d;
            jsel[nrow] = -1;
            rows[nrow++] = inoff[d * a.nd + me] + a.tok_row[(long)t * a.nd + d] - off_sd[me * a.nd + d];
        }
    } else {  // replicate-k baseline: one row per (token, expert), carrying only that expert
        for (int j = 0; j < a.k; ++j) {
            if (!a.mask[(long)t * a.k + j]) continue;  // dropped (invalid) token
            const int d = dev_of[a.ids[(long)t * a.k + j]];
            dsts[nrow] = d;
            jsel[nrow] = j;
            rows[nrow++] = inoff[d * a.nd + me] + a.tok_row[(long)t * a.k + j] - off_sd[me * a.nd + d];
        }
    }
    // x row: read once, the whole row in flight (16 16-byte vectors per lane),
    // stored to every destination inbox row (NVLink peer stores)
    for (int v0 = 0; v0 < nvec; v0 += kPackVec * 32) {
        if (v0) {
#pragma unroll
            for (int u = 0; u < kPackVec; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < nvec) buf[u] = __ldg(src + v);
            }
        }
        for (int q = 0; q < nrow; ++q) {
            uint4* dst = reinterpret_cast<uint4*>(
                reinterpret_cast<__nv_bfloat16*>(peer_tab[dsts[q] * kPeerSlots + kPeerInX]) + (long)rows[q] * a.D);
#pragma unroll
            for (int u = 0; u < kPackVec; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < nvec) dst[v] = buf[u];
            }
        }
    }
    for (int q = 0; q < nrow; ++q) {
        const int d = dsts[q];
        int32_t* pid = reinterpret_cast<int32_t*>(peer_tab[d * kPeerSlots + kPeerInIds]);
        float* pw = reinterpret_cast<float*>(peer_tab[d * kPeerSlots + kPeerInW]);
        for (int j = lane; j < a.k; j += 32) {
            const long di = (long)rows[q] * a.k + j;
            const bool keep = jsel[q] < 0 || j == jsel[q];
            pid[di] = keep ? a.ids[(long)t * a.k + j] : -1;
            pw[di] = keep ? a.w[(long)t * a.k + j] : 0.0f;
        }
    }
}

__global__ void __launch_bounds__(256) peer_pack_kernel(PackArgs a, int me, const int32_t* dev_of, const int* off_sd,
                                                        const int* inoff, void* const* peer_tab) {
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < a.n; t += (gridDim.x * blockDim.x) >> 5)
        peer_pack_token(a, me, dev_of, off_sd, inoff, peer_tab, t, lane);
}

// Arrival signal: after this stream's peer stores, publish `seq` into slot
// (base + me) of every peer's flag array (release, system scope).
__global__ void seq_bump_kernel(unsigned long long* seq) { *seq += 1; }

__global__ void peer_signal_kernel(void* const* peer_tab, int nd, int me, int base, const unsigned long long* seq_p) {
    const int d = threadIdx.x;
    if (d >= nd) return;
    const unsigned long long seq = *seq_p;
    __threadfence_system();
    unsigned long long* f = reinterpret_cast<unsigned long long*>(peer_tab[d * kPeerSlots + kPeerFlags]);
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f + base + me), "l"(seq) : "memory");
}

// Wait until every peer has published `seq` in slots base..base+nd of this
// rank's flags; bounded (err = 7 after `timeout_ns`) so a lost peer cannot
// hang the device.
__global__ void peer_wait_kernel(const unsigned long long* flags, int nd, int base, const unsigned long long* seq_p,
                                 long long timeout_ns, int32_t* err) {
    const int s = threadIdx.x;
    if (s >= nd) return;
    const unsigned long long seq = *seq_p;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + base + s) : "memory");
        if (v >= seq) break;
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if ((long long)(t1 - t0) > timeout_ns) {
            atomicExch(err, 7);
            printf("occ peer wait: timeout on flag slot %d (phase base %d): saw %llu, want %llu\n", base + s, base, v,
                   seq);
            break;
        }
        __nanosleep(256);
    }
    __threadfence_system();
}

// Intra-device partial combine fused with the return exchange: inbox row r
// (from source s, slot counter c) is summed over its local experts and
// stored straight into source s's returned-row buffer at row c.
__global__ void __launch_bounds__(256) peer_return_kernel(const int* R_total, int nd, int me, int P, int D,
                                                          const int32_t* row_epd, const __nv_bfloat16* Y, const int* C,
                                                          const int* off_sd, const int* inoff, void* const* peer_tab) {
    __shared__ int s_q[8][kMaxLocal];
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= *R_total) return;
    int s = 0;  // source of inbox row r: rows of source s are [inoff[me][s], inoff[me][s] + C[s][me])
    while (s < nd - 1 && r >= inoff[me * nd + s] + C[s * nd + me]) ++s;
    const int c = off_sd[s * nd + me] + (r - inoff[me * nd + s]);
    int* qs = s_q[threadIdx.x >> 5];
    const int nq = warp_compact_append(row_epd + (long)r * P, P, qs, 0, kMaxLocal, lane);
    __syncwarp();
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(peer_tab[s * kPeerSlots + kPeerYSrc]) + (long)c * D;
    if (P <= 2) sum_rows_ordered<2>(Y, qs, nq, D, lane, nullptr, dst);
    else if (P <= 4) sum_rows_ordered<4>(Y, qs, nq, D, lane, nullptr, dst);
    else sum_rows_ordered<8>(Y, qs, nq, D, lane, nullptr, dst);
}

// SimilarityAccumulator::add (pruning.cpp:169-183): inner[i][j] += sum_t
// l[t][i] * l[t][j] over one batch, accumulated in double in ascending t
// (one thread per upper-triangle pair, the batch sum added once, mirrored),
// bit-exact with the reference for fp64 logits.
template <class T>
__global__ void similarity_add_kernel(const T* logits, int n, int e, double* inner) {
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < i || j >= e) return;
    double dot = 0.0;
    for (int t = 0; t < n; ++t) dot = __dadd_rn(dot, __dmul_rn((double)logits[(long)t * e + i], (double)logits[(long)t * e + j]));
    inner[(long)i * e + j] = __dadd_rn(inner[(long)i * e + j], dot);
    if (i != j) inner[(long)j * e + i] = __dadd_rn(inner[(long)j * e + i], dot);
}

// Shared-expert gate (Qwen's shared_expert_gate): g_t = sigmoid(x[t] . gate),
// one warp per token, fp32 accumulation.  Rows n..n_pad of the padded
// GEMM m-tile get 0 so the padded rows stay finite.
__global__ void __launch_bounds__(256) shared_gate_kernel(int n, int n_pad, int D, const __nv_bfloat16* x,
                                                          const __nv_bfloat16* gate, float* g) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n_pad) return;
    if (t >= n) {
        if (lane == 0) g[t] = 0.f;
        return;
    }
    float acc = 0.f;
    for (int v = lane; v < D / 8; v += 32) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(x + (long)t * D) + v);
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(gate) + v);
        const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
        const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 fa = __bfloat1622float2(ha[q]), fb = __bfloat1622float2(hb[q]);
            acc += fa.x * fb.x + fa.y * fb.y;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) g[t] = 1.0f / (1.0f + __expf(-acc));
}

__global__ void fill_f32_kernel(float* p, int n, int n_pad, float v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_pad) p[i] = i < n ? v : 0.f;
}

__global__ void set_group_kernel(int* g, int nmb) {
    g[0] = 0;
    g[1] = nmb;
    g[2] = 0;
}

__global__ void extract_cindex_kernel(int R_max, const int* R_total, int P, const int32_t* row_dev,
                                      const int* in_base, const int32_t* row_epd, ComputeOffsets o, int32_t* cindex) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int R = *R_total;
    if (i >= (long)R * P) return;
    const int r = (int)(i / P), p = (int)(i % P);
    const int d = row_dev ? row_dev[r] : 0;
    const int base = in_base ? in_base[d] : 0;
    const int Rd = (in_base ? in_base[d + 1] : R) - base;
    const int q = row_epd[(long)r * P + p];
    const int g = d * P + p;
    const int v = q < 0 ? -1 : q - o.seg_base[g] + o.unp_base[g];
    // per device: P x R_d block, blocks concatenated in device order
    cindex[(long)base * P + (long)p * Rd + (r - base)] = v;
}

// -------------------------------------------------------------- backward --

// Scatter adjoint summed per device then over devices (backward.cpp:136-152):
// g_x[t] = sum over the token's k Epd rows, device ascending, placement
// order inside a device; fp32 throughout.
template <class OutT>
__global__ void __launch_bounds__(256) combine_grad_kernel(int n, int nd, int k, int P, int dedup, int D,
                                                           const uint64_t* mask, const int32_t* tok_row,
                                                           const int32_t* row_epd, const __nv_bfloat16* Y,
                                                           OutT* out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n) return;
    int qs[kMaxTopK];
    int nq = 0;
    if (dedup) {
        uint64_t m = mask[t];
        while (m) {
            const int d = __ffsll(m) - 1;
            m &= m - 1;
            const int r = tok_row[(long)t * nd + d];
            for (int p = 0; p < P && nq < kMaxTopK; ++p) {
                const int q = row_epd[(long)r * P + p];
                if (q >= 0) qs[nq++] = q;
            }
        }
    } else {
        for (int j = 0; j < k; ++j) {
            const int r = tok_row[(long)t * k + j];
            for (int p = 0; p < P; ++p) {
                const int q = row_epd[(long)r * P + p];
                if (q >= 0) qs[nq++] = q;
            }
        }
    }
    const int nv = D / 8;
    for (int v = lane; v < nv; v += 32) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i0 = 0; i0 < nq; i0 += 8) {
            uint4 u[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (i0 + j < nq) u[j] = __ldg(reinterpret_cast<const uint4*>(Y + (long)qs[i0 + j] * D) + v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (i0 + j >= nq) break;
                const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u[j]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(hh[e]);
                    acc[2 * e] += f.x;
                    acc[2 * e + 1] += f.y;
                }
            }
        }
        if constexpr (sizeof(OutT) == 4) {
            float4* o = reinterpret_cast<float4*>(out + (long)t * D) + 2 * v;
            o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {  // bf16 token gradient (mixed-precision training output)
            uint4 o;
            o.x = pack_bf16(acc[0], acc[1]);
            o.y = pack_bf16(acc[2], acc[3]);
            o.z = pack_bf16(acc[4], acc[5]);
            o.w = pack_bf16(acc[6], acc[7]);
            reinterpret_cast<uint4*>(out + (long)t * D)[v] = o;
        }
    }
}

// Routing-weight gradients (backward.cpp:97-111): reduce the per-n-tile
// partials of each Epd row in order and write them to (token, slot).
__global__ void gw_scatter_kernel(int Q_max, const int* q_total, int NB, const float* gw_part, const int32_t* epd_src,
                                  const int32_t* in_tok, const int32_t* epd_j, int k, float* g_weights) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *q_total) return;
    const int r = epd_src[q];
    if (r < 0) return;
    float s = 0.f;
    for (int b = 0; b < NB; ++b) s += gw_part[(long)q * NB + b];
    g_weights[(long)(in_tok ? in_tok[r] : r) * k + epd_j[q]] = s;  // in_tok null: per inbox row
}

// ------------------------------------------------------------- histogram --
// accumulate_collab (collab.cpp:10-23): privatised E x E counters in shared
// memory, flushed with one 64-bit atomic per non-zero bin.
__global__ void __launch_bounds__(256) histogram_kernel(const int32_t* ids, int n, int k, int e,
                                                        unsigned long long* counts) {
    extern __shared__ unsigned int h[];
    for (int i = threadIdx.x; i < e * e; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int32_t* row = ids + (long)t * k;
        for (int a = 0; a < k; ++a) {
            const int ea = row[a];
            if ((unsigned)ea >= (unsigned)e) continue;  // invalid ids are not counted
            for (int b = a + 1; b < k; ++b) {
                const int eb = row[b];
                if ((unsigned)eb >= (unsigned)e) continue;
                atomicAdd(&h[ea * e + eb], 1u);
                atomicAdd(&h[eb * e + ea], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < e * e; i += blockDim.x)
        if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

// Experts beyond the shared-memory bins: count straight into the int64 table.
__global__ void __launch_bounds__(256) histogram_global_kernel(const int32_t* ids, int n, int k, int e,
                                                               unsigned long long* counts) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int32_t* row = ids + (long)t * k;
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) {
                if ((unsigned)row[a] >= (unsigned)e || (unsigned)row[b] >= (unsigned)e) continue;
                atomicAdd(&counts[(long)row[a] * e + row[b]], 1ull);
                atomicAdd(&counts[(long)row[b] * e + row[a]], 1ull);
            }
    }
}

// ------------------------------------------------------------ token stats --
// Per-pass accounting (CommReport, pipeline.cpp:479-487): device span
// (mean_token_replicas, collab.cpp:41-61), co-activated pair shares
// (collab.cpp:105-118) and naive replicate-k crossings
// (test_simnet.cpp:167-180 brute force, per expert instead of per device).
__global__ void token_stats_kernel(int n, int k, int nd, const int32_t* ids, const int32_t* sources, int src_fixed,
                                   const int32_t* dev_of, int E, long long* stats) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    long long span = 0, naive = 0, intra = 0, inter = 0;
    bool ok = t < n;
    for (int j = 0; ok && j < k; ++j) ok = (unsigned)ids[(long)t * k + j] < (unsigned)E;  // invalid: flagged by the plan
    if (ok) {
        const int s = src_fixed >= 0 ? src_fixed : (sources ? sources[t] : t % nd);
        uint64_t m = 0;
        for (int j = 0; j < k; ++j) {
            const int d = dev_of[ids[(long)t * k + j]];
            m |= 1ull << d;
            naive += d != s;
            for (int l = j + 1; l < k; ++l) {
                if (dev_of[ids[(long)t * k + l]] == d) ++intra;
                else ++inter;
            }
        }
        span = __popcll(m);
    }
    for (int o = 16; o; o >>= 1) {
        span += __shfl_xor_sync(0xffffffffu, span, o);
        naive += __shfl_xor_sync(0xffffffffu, naive, o);
        intra += __shfl_xor_sync(0xffffffffu, intra, o);
        inter += __shfl_xor_sync(0xffffffffu, inter, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&stats[1]), (unsigned long long)naive);
        atomicAdd(reinterpret_cast<unsigned long long*>(&stats[2]), (unsigned long long)span);
        atomicAdd(reinterpret_cast<unsigned long long*>(&stats[3]), (unsigned long long)intra);
        atomicAdd(reinterpret_cast<unsigned long long*>(&stats[4]), (unsigned long long)inter);
    }
}

// ------------------------------------------------------- routers (fp64) --
// gate_scores (routing.cpp:33-52) in exact mode: one thread per (token,
// expert), sequential ascending-k double accumulation without FMA
// (matrix.cpp:25-31), then per-row max-subtracted softmax.
__global__ void gate_logits_f64_kernel(const double* x, int n, int d, const double* g, int e, double* s) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)n * e) return;
    const int t = (int)(i / e), j = (int)(i % e);
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = __dadd_rn(acc, __dmul_rn(x[(long)t * d + c], g[(long)j * d + c]));
    s[i] = acc;
}
__global__ void softmax_f64_kernel(int n, int e, double* s) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double* row = s + (long)t * e;
    double mx = row[0];
    for (int j = 1; j < e; ++j) mx = row[j] > mx ? row[j] : mx;
    double sum = 0.0;
    for (int j = 0; j < e; ++j) {
        row[j] = occ::glibc_exp::exp(__dsub_rn(row[j], mx));  // std::exp of routing.cpp:44, bit for bit
        sum = __dadd_rn(sum, row[j]);
    }
    for (int j = 0; j < e; ++j) row[j] = __ddiv_rn(row[j], sum);
}

// Exact router from the production bf16 operands: the reference's
// gate_scores logits (tiled_matmul in Precision::Double, matrix.cpp:25-31:
// per output, products added in ascending k, no FMA) of the bf16 tokens and
// gate widened exactly to double.  Tile: 32 tokens x 8 experts per block,
// 64-deep k slices staged in shared memory; each thread keeps the strict
// sequential k order of its own (token, expert) sum.
constexpr int kLgT = 32, kLgE = 8, kLgK = 64;
__global__ void __launch_bounds__(kLgT * kLgE) gate_logits_bf16_f64_kernel(const __nv_bfloat16* __restrict__ x, int n,
                                                                          int d, const __nv_bfloat16* __restrict__ g,
                                                                          int e, double* __restrict__ s) {
    __shared__ double xs[kLgT][kLgK + 1];
    __shared__ double gs[kLgE][kLgK + 1];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kLgT + tx;
    const int t0 = blockIdx.x * kLgT, e0 = blockIdx.y * kLgE;
    double acc = 0.0;
    for (int k0 = 0; k0 < d; k0 += kLgK) {
        for (int i = tid; i < kLgT * kLgK; i += kLgT * kLgE) {
            const int r = i / kLgK, c = i % kLgK;
            const int t = t0 + r, kk = k0 + c;
            xs[r][c] = (t < n && kk < d) ? (double)__bfloat162float(x[(long)t * d + kk]) : 0.0;
        }
        for (int i = tid; i < kLgE * kLgK; i += kLgT * kLgE) {
            const int r = i / kLgK, c = i % kLgK;
            const int j = e0 + r, kk = k0 + c;
            gs[r][c] = (j < e && kk < d) ? (double)__bfloat162float(g[(long)j * d + kk]) : 0.0;
        }
        __syncthreads();
        const int kn = min(kLgK, d - k0);
        for (int c = 0; c < kn; ++c) acc = __dadd_rn(acc, __dmul_rn(xs[tx][c], gs[ty][c]));
        __syncthreads();
    }
    const int t = t0 + tx, j = e0 + ty;
    if (t < n && j < e) s[(long)t * e + j] = acc;
}

__global__ void f64_to_f32_kernel(const double* a, long n, float* b) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}

template <class T>
__device__ __forceinline__ bool score_before(const T* row, int a, int b) {
    if (row[a] != row[b]) return row[a] > row[b];
    return a < b;
}

// Selection of the k best under (score desc, index asc): identical to
// std::partial_sort with the reference comparator (routing.cpp:71-74).
template <class T>
__device__ void select_topk(const T* row, int e, int k, int* out) {
    for (int j = 0; j < k; ++j) {
        int best = -1;
        for (int c = 0; c < e; ++c) {
            bool taken = false;
            for (int l = 0; l < j; ++l) taken |= out[l] == c;
            if (taken) continue;
            if (best < 0 || score_before(row, c, best)) best = c;
        }
        out[j] = best;
    }
}

template <class T>
__device__ bool renorm_row(T* w, int k) {  // renormalize_row, routing.cpp:54-58
    T sum = 0;
    for (int j = 0; j < k; ++j) sum += w[j];
    if (!(sum > 0)) return false;
    for (int j = 0; j < k; ++j) w[j] = w[j] / sum;
    return true;
}

__global__ void topk_f64_kernel(const double* s, int n, int e, int k, int renorm, int32_t* ids, double* w,
                                int32_t* err) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double* row = s + (long)t * e;
    int sel[256];
    select_topk(row, e, k, sel);
    double wt[256];
    for (int j = 0; j < k; ++j) wt[j] = row[sel[j]];
    if (renorm && !renorm_row(wt, k)) atomicExch(err, 4);
    for (int j = 0; j < k; ++j) {
        ids[(long)t * k + j] = sel[j];
        w[(long)t * k + j] = wt[j];
    }
}

// ------------------------------------------------------------- pruning ---
// allowed_devices (pruning.cpp:21-33): first `budget` distinct devices in
// the given order.
__device__ int allowed_devices(const int* ids, int k, const int32_t* dev_of, int budget, int* devs) {
    int na = 0;
    for (int j = 0; j < k; ++j) {
        const int d = dev_of[ids[j]];
        bool found = false;
        for (int i = 0; i < na; ++i) found |= devs[i] == d;
        if (!found) {
            if (na == budget) break;
            devs[na++] = d;
        }
    }
    return na;
}

// prune_router_score (pruning.cpp:35-64) / prune_similarity (:66-122) for
// one token.  Returns 0 or an occ_status.
template <class T>
__device__ int prune_token(const T* row, int e, int k, const int* ids_in, const PruneDev& p, int* ids, T* w) {
    int devs[kMaxDev];
    bool in_range[kMaxDev];
    for (int d = 0; d < p.nd; ++d) in_range[d] = false;
    if (p.mode == 1) {
        int top[256];
        select_topk(row, e, k, top);
        const int na = allowed_devices(top, k, p.dev_of, p.budget, devs);
        for (int i = 0; i < na; ++i) in_range[devs[i]] = true;
        // walk experts in full score order, keep those on allowed devices
        int m = 0;
        int last = -1;
        while (m < k) {
            int best = -1;
            for (int c = 0; c < e; ++c) {
                if (!in_range[p.dev_of[c]]) continue;
                if (last >= 0 && !score_before(row, last, c)) continue;  // strictly after `last`
                if (best < 0 || score_before(row, c, best)) best = c;
            }
            if (best < 0) return 5;  // CapacityError
            ids[m] = best;
            w[m] = row[best];
            last = best;
            ++m;
        }
        if (p.renorm && !renorm_row(w, k)) return 4;
        return 0;
    }
    // similarity
    const int na = allowed_devices(ids_in, k, p.dev_of, p.budget, devs);
    for (int i = 0; i < na; ++i) in_range[devs[i]] = true;
    bool selected[256];
    for (int c = 0; c < e; ++c) selected[c] = false;
    bool replaced[256];
    for (int j = 0; j < k; ++j)
        if (in_range[p.dev_of[ids_in[j]]]) selected[ids_in[j]] = true;
    for (int j = 0; j < k; ++j) {
        const int ex = ids_in[j];
        replaced[j] = false;
        if (in_range[p.dev_of[ex]]) { ids[j] = ex; continue; }
        int pick = -1;
        for (int c = 0; c < e - 1; ++c) {
            const int cand = p.ranking[(long)ex * (e - 1) + c];
            if (!in_range[p.dev_of[cand]] || selected[cand]) continue;
            pick = cand;
            break;
        }
        if (pick < 0) return 5;
        selected[pick] = true;
        ids[j] = pick;
        replaced[j] = true;
    }
    // pruned_weight_policy (pruning.cpp:124-139): originals are raw scores
    for (int j = 0; j < k; ++j) w[j] = (p.own_score && replaced[j]) ? row[ids[j]] : row[ids_in[j]];
    if (p.renorm && !renorm_row(w, k)) return 4;
    if (p.own_score) {  // pruning.cpp:106-119: (weight desc, id asc)
        for (int i = 1; i < k; ++i) {
            const int vi = ids[i];
            const T vw = w[i];
            int q = i - 1;
            while (q >= 0 && (vw > w[q] || (vw == w[q] && vi < ids[q]))) {
                ids[q + 1] = ids[q];
                w[q + 1] = w[q];
                --q;
            }
            ids[q + 1] = vi;
            w[q + 1] = vw;
        }
    }
    return 0;
}

__global__ void prune_f64_kernel(const double* s, int n, int e, int k, const int32_t* ids_in, const double* w_in,
                                 PruneDev p, int32_t* ids, double* w, int32_t* err) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    if (p.mode == 0) {
        for (int j = 0; j < k; ++j) {
            ids[(long)t * k + j] = ids_in[(long)t * k + j];
            w[(long)t * k + j] = w_in[(long)t * k + j];
        }
        return;
    }
    int in[256], oi[256];
    double ow[256];
    for (int j = 0; j < k; ++j) in[j] = ids_in[(long)t * k + j];
    const int rc = prune_token(s + (long)t * e, e, k, in, p, oi, ow);
    if (rc) { atomicExch(err, rc); return; }
    for (int j = 0; j < k; ++j) {
        ids[(long)t * k + j] = oi[j];
        w[(long)t * k + j] = ow[j];
    }
}

// ------------------------------------------------- production router ---
// softmax + top-k + renormalise (+ pruning) for one token, fp32; `row`
// holds the logits and is overwritten with the softmax scores.
__device__ void route_token(float* row, int t, int e, int k, int renorm, const PruneDev& p, int32_t* ids, float* w,
                            float* scores, int32_t* err) {
    float mx = row[0];
    for (int j = 1; j < e; ++j) mx = fmaxf(mx, row[j]);
    float sum = 0.f;
    for (int j = 0; j < e; ++j) {
        row[j] = __expf(row[j] - mx);
        sum += row[j];
    }
    const float inv = 1.0f / sum;
    for (int j = 0; j < e; ++j) row[j] *= inv;
    if (scores)
        for (int j = 0; j < e; ++j) scores[(long)t * e + j] = row[j];
    int sel[kMaxTopK];
    float wt[kMaxTopK];
    select_topk(row, e, k, sel);
    if (p.mode != 0) {
        int oi[kMaxTopK];
        const int rc = prune_token(row, e, k, sel, p, oi, wt);
        if (rc) { atomicExch(err, rc); return; }
        for (int j = 0; j < k; ++j) sel[j] = oi[j];
    } else {
        for (int j = 0; j < k; ++j) wt[j] = row[sel[j]];
        if (renorm && !renorm_row(wt, k)) atomicExch(err, 4);
    }
    for (int j = 0; j < k; ++j) {
        ids[(long)t * k + j] = sel[j];
        w[(long)t * k + j] = wt[j];
    }
}

__global__ void router_select_kernel(float* logits, int n, int e, int k, int renorm, PruneDev p, int32_t* ids,
                                     float* w, float* scores, int32_t* err) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    route_token(logits + (long)t * e, t, e, k, renorm, p, ids, w, scores, err);
}

// -------------------------------------------------- weight re-layout ---
// Reference expert matrices are [K, N] row-major (token.hpp:30-44); the
// tensor-core path wants them K-major ([N, K]).  For SwiGLU the w1/w3 rows
// are interleaved in 128-row blocks so one 256-row B tile holds matching
// gate/up columns.
__global__ void transpose_weights_kernel(const __nv_bfloat16* w, int K, int N, __nv_bfloat16* out, int out_rows_per_e,
                                         int interleave_half, int pitch) {
    __shared__ __nv_bfloat16 tile[32][33];
    const int e = blockIdx.z;
    const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    const __nv_bfloat16* src = w + (long)e * K * N;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int kk = k0 + i, nn = n0 + threadIdx.x;
        if (kk < K && nn < N) tile[i][threadIdx.x] = src[(long)kk * N + nn];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int nn = n0 + i, kk = k0 + threadIdx.x;
        if (kk < K && nn < N) {
            long orow = nn;
            if (interleave_half) orow = (long)(nn / 128) * 256 + (interleave_half - 1) * 128 + nn % 128;
            out[((long)e * out_rows_per_e + orow) * pitch + kk] = tile[threadIdx.x][i];
        }
    }
}

}  // namespace

// ================================================================ launchers
void launch_plan_mask(const PlanArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    plan_mask_kernel<<<(a.n + 255) / 256, 256, 0, st>>>(a);
    count_launch();
}

void launch_rank_count(int n_items, const int32_t* group, const uint64_t* mask, int G, int B, RankWs ws,
                       cudaStream_t st) {
    const int nchunks = (n_items + kRankChunk - 1) / kRankChunk;
    if (nchunks == 0) return;
    const size_t smem = rank_smem(G, B);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rank_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rank_count_kernel<<<nchunks, kRankThreads, smem, st>>>(n_items, nullptr, group, mask, G, B, ws.chunk_cnt, nchunks);
    count_launch();
}

void launch_rank_count_dev(int n_max, const int* n_dev, const int32_t* group, const uint64_t* mask, int G, int B,
                           RankWs ws, cudaStream_t st) {
    const int nchunks = (n_max + kRankChunk - 1) / kRankChunk;
    if (nchunks == 0) return;
    const size_t smem = rank_smem(G, B);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rank_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rank_count_kernel<<<nchunks, kRankThreads, smem, st>>>(n_max, n_dev, group, mask, G, B, ws.chunk_cnt, nchunks);
    count_launch();
}

void launch_rank_scan(int n_items, int G, int B, RankWs ws, cudaStream_t st) {
    const int nchunks = (n_items + kRankChunk - 1) / kRankChunk;
    const int K = G * (B + 1);
    if (nchunks == 0) {
        cudaMemsetAsync(ws.totals, 0, sizeof(int) * K, st);
        return;
    }
    rank_scan_kernel<<<K, 1024, 0, st>>>(ws.chunk_cnt, nchunks, ws.totals);
    count_launch();
}

void launch_dispatch_finalize(int nd, const int* totals, DispatchOffsets o, cudaStream_t st) {
    dispatch_finalize_kernel<<<1, 128, 0, st>>>(nd, totals, o);
    count_launch();
}

void launch_rank_emit_dispatch(int n_items, const int32_t* group, const uint64_t* mask, int G, int B, RankWs ws,
                               const EmitDispatch& e, cudaStream_t st) {
    launch_rank_emit(n_items, nullptr, group, mask, G, B, ws, DispatchEmitter{e}, st);
}

void launch_extract_brim0(int n, int nd, const int32_t* sources, int src_fixed, const uint64_t* mask,
                          const int32_t* lam, const int32_t* tok_sfd, const int* src_tok_base, int32_t* brim0,
                          cudaStream_t st) {
    // src_tok_base holds [nd] prefix of tokens per source followed by ntok[nd]
    const long total = (long)n * nd;
    if (!total) return;
    extract_brim0_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(n, nd, sources, src_fixed, mask, lam,
                                                                            tok_sfd, src_tok_base,
                                                                            src_tok_base + nd, brim0);
    count_launch();
}

void launch_pack(const PackArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    pack_kernel<<<std::min((a.n + 7) / 8, 148 * 8), 256, 0, st>>>(a);
    count_launch();
}

void launch_compute_mask(const ComputeArgs& a, cudaStream_t st) {
    if (a.R_max == 0) return;
    compute_mask_kernel<<<(a.R_max + 255) / 256, 256, 0, st>>>(a);
    count_launch();
}

void launch_compute_finalize(int G, int P, const int* totals, ComputeOffsets o, cudaStream_t st) {
    compute_finalize_kernel<<<1, 256, 0, st>>>(G, P, totals, o);
    count_launch();
}

void launch_rank_emit_compute(int R_max, const int* R_total, const int32_t* group, const uint64_t* mask, int G,
                              int B, RankWs ws, const EmitCompute& e, cudaStream_t st) {
    // misses: one coalesced fill instead of P scattered 4-byte stores per row
    cudaMemsetAsync(e.row_epd, 0xFF, sizeof(int32_t) * (size_t)R_max * e.P, st);
    launch_rank_emit(R_max, R_total, group, mask, G, B, ws, ComputeEmitter{e}, st);
}

void launch_init_epd(int Q_max, int32_t* epd_src, float* epd_w, cudaStream_t st) {
    if (!Q_max) return;
    init_epd_kernel<<<(Q_max + 255) / 256, 256, 0, st>>>(Q_max, epd_src, epd_w);
    count_launch();
}

void launch_similarity_add(const void* logits, int fp64, int n, int e, double* inner, cudaStream_t st) {
    if (n <= 0) return;
    const dim3 grid((e + 63) / 64, e);
    if (fp64) similarity_add_kernel<double><<<grid, 64, 0, st>>>(reinterpret_cast<const double*>(logits), n, e, inner);
    else similarity_add_kernel<float><<<grid, 64, 0, st>>>(reinterpret_cast<const float*>(logits), n, e, inner);
    count_launch();
}

void launch_scatter_rows(int R_max, const int* R_total, int P, int D, const __nv_bfloat16* src,
                         const int32_t* src_rows, const int32_t* row_epd, int NG, const ComputeOffsets& o,
                         __nv_bfloat16* dst, cudaStream_t st) {
    if (!R_max) return;
    const long warps = (long)R_max * ((D / 8 + 127) / 128);
    launch_pdl(scatter_rows_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, st, R_max, R_total, P, D, src,
               src_rows, row_epd, dst);
    // up to kBM - 1 padding rows per segment: spread each over enough blocks
    const int ny = std::max(1, std::min(64, (int)((long)(kBM - 1) * D / 8 / (256 * 16))));
    launch_pdl(zero_pad_rows_kernel, dim3(NG, ny), dim3(256), 0, st, NG, o, D, dst);
    count_launch(2);
}

void launch_partial_combine(int R_max, const int* R_total, int P, int D, const int32_t* row_epd,
                            const __nv_bfloat16* Y, __nv_bfloat16* ret, cudaStream_t st) {
    if (!R_max) return;
    if (P <= 2)
        partial_combine_kernel<2><<<(R_max + 7) / 8, 256, 0, st>>>(R_max, R_total, P, D, row_epd, Y, ret);
    else if (P <= 4)
        partial_combine_kernel<4><<<(R_max + 7) / 8, 256, 0, st>>>(R_max, R_total, P, D, row_epd, Y, ret);
    else
        partial_combine_kernel<8><<<(R_max + 7) / 8, 256, 0, st>>>(R_max, R_total, P, D, row_epd, Y, ret);
    count_launch();
}

void launch_combine(int n, int nd, int k, int dedup, int D, const uint64_t* mask, const int32_t* tok_row,
                    const __nv_bfloat16* ret, const __nv_bfloat16* ys, __nv_bfloat16* out, cudaStream_t st) {
    if (!n) return;
    if (k <= 2)
        combine_kernel<2><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, dedup, D, mask, tok_row, ret, ys, out);
    else if (k <= 4)
        combine_kernel<4><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, dedup, D, mask, tok_row, ret, ys, out);
    else
        combine_kernel<8><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, dedup, D, mask, tok_row, ret, ys, out);
    count_launch();
}

void launch_dispatch_sfd(int n, int nd, int k, int D, const __nv_bfloat16* x, const int32_t* ids, const float* w,
                         const int32_t* brim0, __nv_bfloat16* sfd_x, int32_t* sfd_ids, float* sfd_w, int32_t* sfd_tok,
                         cudaStream_t st) {
    if (!n) return;
    dispatch_sfd_kernel<<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, D, x, ids, w, brim0, sfd_x, sfd_ids, sfd_w, sfd_tok);
    count_launch();
}

void launch_combine_brim0(int n, int nd, int D, const int32_t* brim0, const __nv_bfloat16* y, __nv_bfloat16* out,
                          cudaStream_t st) {
    if (!n) return;
    if (nd <= 2)
        combine_brim0_kernel<2><<<(n + 7) / 8, 256, 0, st>>>(n, nd, D, brim0, y, out);
    else if (nd <= 4)
        combine_brim0_kernel<4><<<(n + 7) / 8, 256, 0, st>>>(n, nd, D, brim0, y, out);
    else
        combine_brim0_kernel<8><<<(n + 7) / 8, 256, 0, st>>>(n, nd, D, brim0, y, out);
    count_launch();
}

void launch_brim0_one_source(int n, int nd, const uint64_t* mask, const int32_t* tok_sfd, int32_t* brim0,
                             cudaStream_t st) {
    const long total = (long)n * nd;
    if (!total) return;
    brim0_one_source_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(n, nd, mask, tok_sfd, brim0);
    count_launch();
}

void launch_one_source_totals(int nd, int r, int* totals, cudaStream_t st) {
    one_source_totals_kernel<<<1, 256, 0, st>>>(nd, r, totals);
    count_launch();
}

void launch_combine_back(int n, int nd, int k, int dedup, int D, const uint64_t* mask, const int32_t* tok_row,
                         const __nv_bfloat16* y, const float* ygw, void* gx, int gx_bf16, float* gw, cudaStream_t st) {
    if (!n) return;
    if (gx_bf16)
        combine_back_kernel<__nv_bfloat16><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, dedup, D, mask, tok_row, y, ygw,
                                                                         reinterpret_cast<__nv_bfloat16*>(gx), gw);
    else
        combine_back_kernel<float><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, dedup, D, mask, tok_row, y, ygw,
                                                                 reinterpret_cast<float*>(gx), gw);
    count_launch();
}

void launch_set_int(int* p, int v, cudaStream_t st) {
    set_int_kernel<<<1, 1, 0, st>>>(p, v);
    count_launch();
}

void launch_combine_fused(int n, int nd, int k, int P, int dedup, int D, const uint64_t* mask,
                          const int32_t* tok_row, const int32_t* row_epd, const __nv_bfloat16* Y,
                          const __nv_bfloat16* ys, __nv_bfloat16* out, cudaStream_t st) {
    if (!n) return;
    const dim3 grid((n + 7) / 8);
    const bool grouped = !(nd == 1 && dedup);
#define OCC_CF(KU, G) \
    launch_pdl(combine_fused_kernel<KU, G>, grid, dim3(256), 0, st, n, nd, k, P, dedup, D, mask, tok_row, row_epd, Y, ys, out)
    if (k <= 2) grouped ? OCC_CF(2, true) : OCC_CF(2, false);
    else if (k <= 4) grouped ? OCC_CF(4, true) : OCC_CF(4, false);
    else grouped ? OCC_CF(8, true) : OCC_CF(8, false);
#undef OCC_CF
    count_launch();
}

void launch_shared_gate(int n, int n_pad, int D, const __nv_bfloat16* x, const __nv_bfloat16* gate, float* g,
                        int* grp, cudaStream_t st) {
    if (!n_pad) return;
    if (gate)
        shared_gate_kernel<<<(n_pad + 7) / 8, 256, 0, st>>>(n, n_pad, D, x, gate, g);
    else
        fill_f32_kernel<<<(n_pad + 255) / 256, 256, 0, st>>>(g, n, n_pad, 1.0f);
    set_group_kernel<<<1, 1, 0, st>>>(grp, n_pad / kBM);
    count_launch(2);
}

void launch_peer_pack(const PackArgs& a, int me, const int32_t* dev_of, const int* off_sd, const int* inoff,
                      void* const* peer_tab, cudaStream_t st) {
    if (!a.n) return;
    peer_pack_kernel<<<std::min((a.n + 7) / 8, 148 * 8), 256, 0, st>>>(a, me, dev_of, off_sd, inoff, peer_tab);
    count_launch();
}
void launch_seq_bump(unsigned long long* seq, cudaStream_t st) {
    seq_bump_kernel<<<1, 1, 0, st>>>(seq);
    count_launch();
}
void launch_peer_signal(void* const* peer_tab, int nd, int me, int base, const unsigned long long* seq,
                        cudaStream_t st) {
    peer_signal_kernel<<<1, 64, 0, st>>>(peer_tab, nd, me, base, seq);
    count_launch();
}
void launch_peer_wait(const unsigned long long* flags, int nd, int base, const unsigned long long* seq,
                      long long timeout_ns,
                      int32_t* err, cudaStream_t st) {
    peer_wait_kernel<<<1, 64, 0, st>>>(flags, nd, base, seq, timeout_ns, err);
    count_launch();
}
void launch_peer_return(int R_max, const int* R_total, int nd, int me, int P, int D, const int32_t* row_epd,
                        const __nv_bfloat16* Y, const int* C, const int* off_sd, const int* inoff,
                        void* const* peer_tab, cudaStream_t st) {
    if (!R_max) return;
    peer_return_kernel<<<(R_max + 7) / 8, 256, 0, st>>>(R_total, nd, me, P, D, row_epd, Y, C, off_sd, inoff,
                                                        peer_tab);
    count_launch();
}
void launch_peer_counts(void* const* peer_tab, int nd, int me, const int* totals, cudaStream_t st) {
    peer_counts_kernel<<<1, 256, 0, st>>>(peer_tab, nd, me, totals);
    count_launch();
}


void launch_combine_grad(int n, int nd, int k, int P, int dedup, int D, const uint64_t* mask, const int32_t* tok_row,
                         const int32_t* row_epd, const __nv_bfloat16* Y, void* out, int out_bf16, cudaStream_t st) {
    if (!n) return;
    if (out_bf16)
        combine_grad_kernel<__nv_bfloat16><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, P, dedup, D, mask, tok_row, row_epd,
                                                                        Y, reinterpret_cast<__nv_bfloat16*>(out));
    else
        combine_grad_kernel<float><<<(n + 7) / 8, 256, 0, st>>>(n, nd, k, P, dedup, D, mask, tok_row, row_epd, Y,
                                                                reinterpret_cast<float*>(out));
    count_launch();
}

void launch_gw_scatter(int Q_max, const int* q_total, int NB, const float* gw_part, const int32_t* epd_src,
                       const int32_t* in_tok, const int32_t* epd_j, int k, float* g_weights, cudaStream_t st) {
    if (!Q_max) return;
    gw_scatter_kernel<<<(Q_max + 255) / 256, 256, 0, st>>>(Q_max, q_total, NB, gw_part, epd_src, in_tok, epd_j, k,
                                                           g_weights);
    count_launch();
}

void launch_extract_cindex(int R_max, const int* R_total, int P, const int32_t* row_dev, const int* in_base,
                           const int32_t* row_epd, const ComputeOffsets& o, int32_t* cindex, cudaStream_t st) {
    const long total = (long)R_max * P;
    if (!total) return;
    extract_cindex_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(R_max, R_total, P, row_dev, in_base,
                                                                             row_epd, o, cindex);
    count_launch();
}

void launch_histogram(const int32_t* ids, int n, int k, int e, int64_t* counts, cudaStream_t st) {
    if (!n) return;
    int blocks = (n + 255) / 256;
    if (blocks > 148 * 4) blocks = 148 * 4;
    const size_t smem = sizeof(unsigned) * (size_t)e * e;
    if (smem > kHistSmemMax) {
        histogram_global_kernel<<<blocks, 256, 0, st>>>(ids, n, k, e, reinterpret_cast<unsigned long long*>(counts));
    } else {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(histogram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        histogram_kernel<<<blocks, 256, smem, st>>>(ids, n, k, e, reinterpret_cast<unsigned long long*>(counts));
    }
    count_launch();
}


void launch_token_stats(int n, int k, int nd, const int32_t* ids, const int32_t* sources, int src_fixed,
                        const int32_t* dev_of, int E, long long* stats, cudaStream_t st) {
    if (!n) return;
    token_stats_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, k, nd, ids, sources, src_fixed, dev_of, E, stats);
    count_launch();
}

void launch_gate_scores_f64(const double* x, int n, int d, const double* g, int e, double* s, cudaStream_t st,
                            bool softmax) {
    const long total = (long)n * e;
    if (!total) return;
    gate_logits_f64_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(x, n, d, g, e, s);
    count_launch();
    if (!softmax) return;
    softmax_f64_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, e, s);
    count_launch();
}

void launch_gate_scores_bf16_f64(const __nv_bfloat16* x, int n, int d, const __nv_bfloat16* g, int e, double* s,
                                 cudaStream_t st) {
    if (!n) return;
    dim3 grid((n + kLgT - 1) / kLgT, (e + kLgE - 1) / kLgE);
    gate_logits_bf16_f64_kernel<<<grid, dim3(kLgT, kLgE), 0, st>>>(x, n, d, g, e, s);
    count_launch();
    softmax_f64_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, e, s);
    count_launch();
}

void launch_f64_to_f32(const double* a, long n, float* b, cudaStream_t st) {
    if (!n) return;
    f64_to_f32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, n, b);
    count_launch();
}

void launch_topk_f64(const double* s, int n, int e, int k, int renorm, int32_t* ids, double* w, int32_t* err,
                     cudaStream_t st) {
    if (!n) return;
    topk_f64_kernel<<<(n + 127) / 128, 128, 0, st>>>(s, n, e, k, renorm, ids, w, err);
    count_launch();
}

void launch_prune_f64(const double* s, int n, int e, int k, const int32_t* ids_in, const double* w_in, PruneDev p,
                      int32_t* ids, double* w, int32_t* err, cudaStream_t st) {
    if (!n) return;
    prune_f64_kernel<<<(n + 127) / 128, 128, 0, st>>>(s, n, e, k, ids_in, w_in, p, ids, w, err);
    count_launch();
}

void launch_router_select(float* logits, int n, int e, int k, int renorm, PruneDev p, int32_t* ids, float* w,
                          float* scores, int32_t* err, cudaStream_t st) {
    if (!n) return;
    router_select_kernel<<<(n + 127) / 128, 128, 0, st>>>(logits, n, e, k, renorm, p, ids, w, scores, err);
    count_launch();
}

void launch_transpose_weights(const __nv_bfloat16* w, int E, int K, int N, __nv_bfloat16* out, int out_rows_per_e,
                              int interleave_half, cudaStream_t st, int pitch) {
    dim3 grid((N + 31) / 32, (K + 31) / 32, E);
    transpose_weights_kernel<<<grid, dim3(32, 8), 0, st>>>(w, K, N, out, out_rows_per_e, interleave_half,
                                                              pitch > 0 ? pitch : K);
    count_launch();
}

}  // namespace occ
