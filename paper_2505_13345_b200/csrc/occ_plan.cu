// occ_plan.cu — the whole one-GPU index chain of the EP layer in ONE
// cooperative (persistent) kernel, for world_size == 1 and the dedup dispatch:
//
//   build_dispatch_index (BRIM0, pipeline.cpp:24-50)  + dispatch / exchange
//   placement of the routing rows (pipeline.cpp:91-176) + build_compute_index
//   (BRIM1, pipeline.cpp:52-89) + the Epd A operand (scatter of each token row
//   to its expert rows, zero-padded 256-row segments) + CommReport counters.
//
// Round 1 ran this as 16 dependent launches (mask, count, scan, finalize,
// emit, stats, pack, compute mask/count/scan/finalize/init/emit, scatter,
// zero-pad), which made the ~20 us-per-launch-chain the largest fixed cost of
// small batches.  Here the same stable bucketed ranks are computed with two
// keys per token in a single pass:
//
//   dispatch key (s, d): rank of token t among the tokens of source s that
//       hit device d      -> BRIM0 counter off_sd[s][d] + rank, inbox row
//       in_base[d] + inoff[d][s] + rank (all_to_all_exchange order: source
//       asc, counter asc);
//   expert key (s, e):   rank of t among the tokens of source s routed to e
//       -> Epd row ebase[s][e] + rank with ebase[s][e] = seg_base[(d,p)] +
//       sum_{s'<s} count(s', e): exactly build_compute_index's expert-major
//       counter over device d's inbox (whose rows are ordered source asc,
//       token asc), because BRIM1 ranks rows of device d by inbox position.
//
// Phases (grid-wide barriers between them, cooperative launch):
//   A  per 256-token chunk: validate routing, device / expert masks, warp
//      ballot counts per key -> chunk_cnt[key][chunk]
//   B  per key: exclusive scan over chunks (one warp per key)
//   C  every block derives the (small) offset tables from the totals into its
//      own shared memory (block 0 also publishes them for the GEMMs / combine)
//   D  per chunk: in-chunk ranks -> BRIM0, inbox records, routing rows, BRIM1
//      (row_epd, epd_src / epd_w / epd_j), CommReport token statistics
//   E  Epd rows: each inbox row's token row copied to its expert rows (one
//      warp per row slice, 16-byte vectors), segment padding zeroed
// Bit-identical to the multi-kernel chain (tests/test_gpu_parity.py runs both).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "occ_common.cuh"
#include "occ_internal.h"

namespace cg = cooperative_groups;

namespace occ {
namespace {

constexpr int kThreads = 256;  // = kRankChunk tokens per chunk, 8 warps
constexpr int kWarps = kThreads / 32;

struct Tables {  // phase C results, in shared memory
    int *C, *off_sd, *inoff, *in_base, *ntok, *tok_base, *cnt, *seg_base, *ebase;
};

__device__ __forceinline__ int token_src(const FusedPlanArgs& a, int t) {
    return a.sources ? a.sources[t] : t % a.nd;
}

// Token t's validated routing: device mask, expert mask, source (dropped
// token: masks 0, source 0 -- the forward reports the error, as plan_mask).
__device__ __forceinline__ void token_masks(const FusedPlanArgs& a, int t, uint64_t& dm, uint64_t& em, int& s) {
    dm = 0, em = 0;
    s = token_src(a, t);
    if (s < 0 || s >= a.nd) {
        atomicExch(a.err, 1);
        s = 0;
        return;
    }
    for (int j = 0; j < a.k; ++j) {
        const int e = a.ids[(long)t * a.k + j];
        const float wt = a.w[(long)t * a.k + j];
        bool bad = e < 0 || e >= a.E || !(wt > 0.0f);
        for (int l = 0; l < j && !bad; ++l) bad = a.ids[(long)t * a.k + l] == e;
        if (bad) {
            atomicExch(a.err, 4);
            dm = em = 0;
            s = 0;
            return;
        }
        dm |= 1ull << a.dev_of[e];
        em |= 1ull << e;
    }
}

// Per-warp counts of every key held by this warp's tokens.
__device__ __forceinline__ void warp_counts(const FusedPlanArgs& a, int valid, int s, uint64_t dm, uint64_t em,
                                            int* wk, int lane) {
    const int KD = a.nd * (a.nd + 1);
    const uint32_t same = __match_any_sync(0xffffffffu, valid ? s : -1);
    const bool leader = valid && (__ffs(same) - 1) == lane;
    for (int d = 0; d < a.nd; ++d) {
        const uint32_t b = __ballot_sync(0xffffffffu, valid && ((dm >> d) & 1));
        if (leader) wk[s * (a.nd + 1) + d] = __popc(b & same);
    }
    if (leader) wk[s * (a.nd + 1) + a.nd] = __popc(same);
    for (int e = 0; e < a.E; ++e) {
        const uint32_t b = __ballot_sync(0xffffffffu, valid && ((em >> e) & 1));
        if (leader) wk[KD + s * a.E + e] = __popc(b & same);
    }
}

__global__ void __launch_bounds__(kThreads) fused_plan_kernel(FusedPlanArgs a) {
    extern __shared__ int smem[];
    cg::grid_group grid = cg::this_grid();
    const int nd = a.nd, E = a.E, P = a.P, k = a.k;
    const int KD = nd * (nd + 1), K = KD + nd * E;
    const int nchunks = (a.n + kThreads - 1) / kThreads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* wcnt = smem;  // [kWarps][K]
    int* tab = wcnt + kWarps * K;

    // ---------------------------------------------------------------- A --
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        for (int i = threadIdx.x; i < kWarps * K; i += kThreads) wcnt[i] = 0;
        __syncthreads();
        const int t = c * kThreads + threadIdx.x;
        const int valid = t < a.n;
        uint64_t dm = 0, em = 0;
        int s = 0;
        if (valid) token_masks(a, t, dm, em, s);
        warp_counts(a, valid, s, dm, em, wcnt + warp * K, lane);
        __syncthreads();
        for (int key = threadIdx.x; key < K; key += kThreads) {
            int sum = 0;
            for (int w = 0; w < kWarps; ++w) sum += wcnt[w * K + key];
            a.chunk_cnt[(long)key * nchunks + c] = sum;
        }
        __syncthreads();
    }
    grid.sync();
    // ---------------------------------------------------------------- B --
    const int gw = (blockIdx.x * kThreads + threadIdx.x) >> 5, nw = gridDim.x * kWarps;
    for (int key = gw; key < K; key += nw) {
        int* row = a.chunk_cnt + (long)key * nchunks;
        int run = 0;
        for (int c0 = 0; c0 < nchunks; c0 += 32) {
            const int c = c0 + lane;
            const int v = c < nchunks ? row[c] : 0;
            int x = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += u;
            }
            if (c < nchunks) row[c] = run + x - v;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) a.totals[key] = run;
    }
    grid.sync();
    // ---------------------------------------------------------------- C --
    Tables T;
    {
        int* p = tab;
        T.C = p, p += nd * nd;
        T.off_sd = p, p += nd * nd;
        T.inoff = p, p += nd * nd;
        T.in_base = p, p += nd + 1;
        T.ntok = p, p += nd;
        T.tok_base = p, p += nd;
        T.cnt = p, p += E;        // per group g = (d, p), E = nd * P groups
        T.seg_base = p, p += E;
        T.ebase = p;               // [nd][E]
    }
    for (int i = threadIdx.x; i < nd * nd; i += kThreads) T.C[i] = a.totals[(i / nd) * (nd + 1) + i % nd];
    for (int g = threadIdx.x; g < E; g += kThreads) T.cnt[g] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += kThreads) {  // group counts from the expert keys
        int c = 0;
        for (int s = 0; s < nd; ++s) c += a.totals[KD + s * E + e];
        T.cnt[a.dev_of[e] * P + a.slot_of[e]] = c;
    }
    __syncthreads();
    if (threadIdx.x < nd) {  // per source: counter offsets (device-major), token counts
        const int s = threadIdx.x;
        int run = 0;
        for (int d = 0; d < nd; ++d) {
            T.off_sd[s * nd + d] = run;
            run += T.C[s * nd + d];
        }
        T.ntok[s] = a.totals[s * (nd + 1) + nd];
    } else if (threadIdx.x >= 64 && threadIdx.x < 64 + nd) {  // per destination: inbox offsets
        const int d = threadIdx.x - 64;
        int run = 0;
        for (int s = 0; s < nd; ++s) {
            T.inoff[d * nd + s] = run;
            run += T.C[s * nd + d];
        }
        T.in_base[d] = run;  // R_d for now
    } else if (threadIdx.x == 128) {  // Epd segments: padded to the 256-row GEMM tile
        int run = 0;
        for (int g = 0; g < E; ++g) {
            T.seg_base[g] = run;
            run += (T.cnt[g] + kBM - 1) / kBM * kBM;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0, tb = 0;
        for (int d = 0; d < nd; ++d) {
            const int r = T.in_base[d];
            T.in_base[d] = run;
            run += r;
        }
        T.in_base[nd] = run;
        for (int s = 0; s < nd; ++s) {
            T.tok_base[s] = tb;
            tb += T.ntok[s];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += kThreads) {  // Epd base of (source, expert)
        int run = T.seg_base[a.dev_of[e] * P + a.slot_of[e]];
        for (int s = 0; s < nd; ++s) {
            T.ebase[s * E + e] = run;
            run += a.totals[KD + s * E + e];
        }
    }
    __syncthreads();
    if (blockIdx.x == 0) {  // publish: the GEMMs, combine and CommReport read these
        const DispatchOffsets& o = a.dofs;
        for (int i = threadIdx.x; i < nd * nd; i += kThreads) {
            o.C[i] = T.C[i];
            o.off_sd[i] = T.off_sd[i];
            o.inoff[i] = T.inoff[i];
        }
        for (int i = threadIdx.x; i <= nd; i += kThreads) o.in_base[i] = T.in_base[i];
        for (int s = threadIdx.x; s < nd; s += kThreads) {
            o.ntok[s] = T.ntok[s];
            a.tok_base[s] = T.tok_base[s];
            int ns = 0;
            for (int d = 0; d < nd; ++d) ns += T.C[s * nd + d];
            o.nsfd[s] = ns;
        }
        const ComputeOffsets& q = a.cofs;
        for (int g = threadIdx.x; g < E; g += kThreads) {
            q.cnt[g] = T.cnt[g];
            q.seg_base[g] = T.seg_base[g];
            const int d = g / P;
            int u = 0;
            for (int p = 0; p < g % P; ++p) u += T.cnt[d * P + p];
            q.unp_base[g] = u;
        }
        if (threadIdx.x == 0) {
            int mb = 0, run = 0;
            long long nepd = 0, cross = 0;
            for (int g = 0; g < E; ++g) {
                q.grp_mb[g] = mb;
                mb += (T.cnt[g] + kBM - 1) / kBM;
                nepd += T.cnt[g];
            }
            q.grp_mb[E] = mb;
            *q.n_mblk = mb;
            *q.q_total = mb * kBM;
            for (int s = 0; s < nd; ++s) {
                o.src_base[s] = run;
                for (int d = 0; d < nd; ++d) {
                    run += T.C[s * nd + d];
                    if (d != s) cross += T.C[s * nd + d];
                }
            }
            o.src_base[nd] = run;
            a.stats[0] = cross;
            a.stats[5] = run;
            a.stats[6] = nepd;
        }
    }
    // ---------------------------------------------------------------- D --
    long long st_naive = 0, st_span = 0, st_intra = 0, st_inter = 0;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        for (int i = threadIdx.x; i < kWarps * K; i += kThreads) wcnt[i] = 0;
        __syncthreads();
        const int t = c * kThreads + threadIdx.x;
        const int valid = t < a.n;
        uint64_t dm = 0, em = 0;
        int s = 0;
        if (valid) token_masks(a, t, dm, em, s);
        warp_counts(a, valid, s, dm, em, wcnt + warp * K, lane);
        __syncthreads();
        for (int key = threadIdx.x; key < K; key += kThreads) {  // exclusive bases per warp
            int run = a.chunk_cnt[(long)key * nchunks + c];
            for (int w = 0; w < kWarps; ++w) {
                const int x = wcnt[w * K + key];
                wcnt[w * K + key] = run;
                run += x;
            }
        }
        __syncthreads();
        const int* wb = wcnt + warp * K;
        const uint32_t same = __match_any_sync(0xffffffffu, valid ? s : -1);
        const uint32_t lt = lanemask_lt();
        int rows[kMaxDev > 64 ? 64 : kMaxDev];  // inbox row per destination device (dedup)
        if (valid) {
            a.lam[t] = wb[s * (nd + 1) + nd] + __popc(same & lt);
            a.mask[t] = dm;  // destination devices (combine, backward)
        }
        for (int d = 0; d < nd; ++d) {
            const bool hit = valid && ((dm >> d) & 1);
            const uint32_t b = __ballot_sync(0xffffffffu, hit);
            if (!valid) continue;
            const long slot = (long)t * nd + d;
            if (!hit) {
                a.tok_sfd[slot] = -1;
                a.tok_row[slot] = -1;
                continue;
            }
            const int r = wb[s * (nd + 1) + d] + __popc(b & same & lt);
            const int cc = T.off_sd[s * nd + d] + r;
            const int row = T.in_base[d] + T.inoff[d * nd + s] + r;
            rows[d] = row;
            a.tok_sfd[slot] = cc;
            a.tok_row[slot] = row;
            a.in_tok[row] = t;
            a.in_src[row] = s;
            a.in_slot[row] = cc;
            a.in_dev[row] = d;
            for (int j = 0; j < k; ++j) {  // the routing row carried with the inbox row
                a.in_ids[(long)row * k + j] = a.ids[(long)t * k + j];
                a.in_w[(long)row * k + j] = a.w[(long)t * k + j];
            }
            for (int p = 0; p < P; ++p) a.row_epd[(long)row * P + p] = -1;
        }
        for (int e = 0; e < E; ++e) {
            const bool hit = valid && ((em >> e) & 1);
            const uint32_t b = __ballot_sync(0xffffffffu, hit);
            if (!hit) continue;
            const int q = T.ebase[s * E + e] + wb[KD + s * E + e] + __popc(b & same & lt);
            const int d = a.dev_of[e], p = a.slot_of[e];
            int j = 0;
            while (a.ids[(long)t * k + j] != e) ++j;
            const int row = rows[d];
            a.row_epd[(long)row * P + p] = q;
            a.epd_src[q] = row;
            a.epd_w[q] = a.w[(long)t * k + j];
            a.epd_j[q] = j;
        }
        if (valid && dm) {  // CommReport (collab.cpp:41-118): span, naive crossings, pair shares
            st_span += __popcll(dm);
            for (int j = 0; j < k; ++j) {
                const int dj = a.dev_of[a.ids[(long)t * k + j]];
                st_naive += dj != s;
                for (int l = j + 1; l < k; ++l) {
                    if (a.dev_of[a.ids[(long)t * k + l]] == dj) ++st_intra;
                    else ++st_inter;
                }
            }
        }
        __syncthreads();
    }
    for (int o = 16; o; o >>= 1) {
        st_span += __shfl_xor_sync(0xffffffffu, st_span, o);
        st_naive += __shfl_xor_sync(0xffffffffu, st_naive, o);
        st_intra += __shfl_xor_sync(0xffffffffu, st_intra, o);
        st_inter += __shfl_xor_sync(0xffffffffu, st_inter, o);
    }
    if (lane == 0 && (st_span | st_naive | st_intra | st_inter)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.stats[1]), (unsigned long long)st_naive);
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.stats[2]), (unsigned long long)st_span);
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.stats[3]), (unsigned long long)st_intra);
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.stats[4]), (unsigned long long)st_inter);
    }
    // padding rows of every segment: no source row, zero weight, zero A row
    for (int g = blockIdx.x; g < E; g += gridDim.x) {
        const int lo = T.seg_base[g] + T.cnt[g], hi = T.seg_base[g] + (T.cnt[g] + kBM - 1) / kBM * kBM;
        for (int q = lo + threadIdx.x; q < hi; q += kThreads) {
            a.epd_src[q] = -1;
            a.epd_w[q] = 0.0f;
        }
        if (a.x_epd) {
            uint4* base = reinterpret_cast<uint4*>(a.x_epd + (long)lo * a.D);
            const long nv = (long)(hi - lo) * a.D / 8;
            for (long v = threadIdx.x; v < nv; v += kThreads) base[v] = make_uint4(0, 0, 0, 0);
        }
    }
    if (!a.x_epd) return;
    grid.sync();
    // ---------------------------------------------------------------- E --
    // Epd A operand: inbox row r's token row (read once) to each of its
    // expert rows; one warp per (row, 4 KB slice).
    const int R = T.in_base[nd];
    const int nvec = a.D / 8;
    constexpr int kSl = 256;  // uint4 per slice: 8 per lane in flight
    const int nsl = (nvec + kSl - 1) / kSl;
    for (long wi = gw; wi < (long)R * nsl; wi += nw) {
        const int r = (int)(wi / nsl), sl = (int)(wi % nsl);
        const uint4* in = reinterpret_cast<const uint4*>(a.x + (long)a.in_tok[r] * a.D);
        const int q_lo = lane < P ? a.row_epd[(long)r * P + lane] : -1;
        const int q_hi = lane + 32 < P ? a.row_epd[(long)r * P + lane + 32] : -1;
        const unsigned m_lo = __ballot_sync(0xffffffffu, q_lo >= 0), m_hi = __ballot_sync(0xffffffffu, q_hi >= 0);
        uint4 buf[8];
        const int v0 = sl * kSl;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nvec) buf[u] = __ldg(in + v);
        }
        for (int half = 0; half < 2; ++half) {
            unsigned m = half ? m_hi : m_lo;
            while (m) {
                const int p = __ffs(m) - 1;
                m &= m - 1;
                const int q = __shfl_sync(0xffffffffu, half ? q_hi : q_lo, p);
                uint4* out = reinterpret_cast<uint4*>(a.x_epd + (long)q * a.D);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int v = v0 + u * 32 + lane;
                    if (v < nvec) out[v] = buf[u];
                }
            }
        }
    }
}

size_t fused_smem(int nd, int E) {
    const int K = nd * (nd + 1) + nd * E;
    const int tabs = 3 * nd * nd + (nd + 1) + 2 * nd + 2 * E + nd * E;
    return sizeof(int) * ((size_t)kWarps * K + tabs);
}

}  // namespace

size_t fused_plan_ws(int n, int nd, int E) {
    const size_t K = (size_t)nd * (nd + 1) + (size_t)nd * E;
    return K * ((size_t)(n + kThreads - 1) / kThreads + 1);
}

bool fused_plan_supported(int nd, int E, int k) {
    return nd <= 64 && E <= 64 && k <= 8 && fused_smem(nd, E) <= 96 * 1024;
}

bool launch_fused_plan(const FusedPlanArgs& a, int num_sms, cudaStream_t st) {
    if (a.n <= 0) return true;
    const size_t smem = fused_smem(a.nd, a.E);
    static int configured = 0;
    if (!configured) {
        cudaFuncSetAttribute(fused_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        configured = 1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_plan_kernel, kThreads, smem) != cudaSuccess ||
        per_sm < 1)
        return false;
    const int blocks = num_sms * std::min(per_sm, 2);
    FusedPlanArgs args = a;
    void* params[] = {&args};
    if (cudaLaunchCooperativeKernel((const void*)fused_plan_kernel, blocks, kThreads, params, smem, st) != cudaSuccess)
        return false;
    count_launch();
    return true;
}

}  // namespace occ
