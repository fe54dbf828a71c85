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
#include <cstdio>
#include <cstdlib>

#include "occ_common.cuh"
#include "occ_internal.h"

namespace cg = cooperative_groups;

namespace occ {
namespace {

constexpr int kThreads = 256;  // 8 warps per block
constexpr int kWarps = kThreads / 32;
constexpr long kSmallCounts = 4096;  // count-matrix size below which the scan phase is skipped

struct Tables {  // phase C results, in shared memory
    int *C, *off_sd, *inoff, *in_base, *ntok, *tok_base, *cnt, *seg_base, *ebase, *padpre, *dev, *slot, *pre;
};

__device__ __forceinline__ int token_src(const FusedPlanArgs& a, int t) {
    return a.sources ? a.sources[t] : t % a.nd;
}

constexpr unsigned kFull = 0xffffffffu;

// One routing entry (token t, slot j) per lane: a warp covers tpw = 32 / k
// tokens (lanes >= tpw * k idle), a block chunk 8 * tpw tokens.  Everything a
// lane needs about its token comes from the token's other lanes by shuffles
// (the token's lanes are adjacent: tok0 .. tok0 + k - 1).
struct Entry {
    int t, j, s, e, d, p;   // e, d, p = -1 unless the entry is valid
    float w;
    bool in;                // a token of the batch
    bool valid;             // its routing is valid (RoutingOutcome::validate)
    bool owner;             // first entry of the token on device d: holds the (t, d) Sfd / inbox row
    int owner_lane;         // lane of that owner
    uint64_t dm;            // the token's destination-device mask (0 for an invalid token)
    uint64_t smask;         // the token's local-slot mask on device d
    int tok0;
};

__device__ __forceinline__ Entry load_entry(const FusedPlanArgs& a, const Tables& T, int c, int tpw, int warp,
                                            int lane) {
    Entry x;
    const int k = a.k;
    const int lt = lane / k;
    x.j = lane - lt * k;
    x.tok0 = lane - x.j;
    x.t = c * kWarps * tpw + warp * tpw + lt;
    x.in = lt < tpw && x.t < a.n;
    int e = -1, s = 0;
    float w = 0.0f;
    if (x.in) {
        e = a.ids[(long)x.t * k + x.j];
        w = a.w[(long)x.t * k + x.j];
        s = token_src(a, x.t);
    }
    const bool badsrc = x.in && (s < 0 || s >= a.nd);
    bool bad = x.in && (e < 0 || e >= a.E || !(w > 0.0f));
    const int de = x.in && !bad ? T.dev[e] : -1;
    const int pe = x.in && !bad ? T.slot[e] : -1;
    int jfirst = x.j;  // first slot of this token on device de
    uint64_t dm = 0, sm = 0;
    for (int jj = 0; jj < k; ++jj) {  // the token's other entries (uniform loop)
        const int src = min(x.tok0 + jj, 31);
        const int oe = __shfl_sync(kFull, e, src);
        const int od = __shfl_sync(kFull, de, src);
        const int op = __shfl_sync(kFull, pe, src);
        if (jj != x.j && oe == e) bad = true;  // duplicate expert id
        if (jj < jfirst && od == de) jfirst = jj;
        if (od >= 0) dm |= 1ull << od;
        if (od >= 0 && od == de) sm |= 1ull << op;
    }
    bool tbad = bad || badsrc, any_bad = false, any_src = false;
    for (int jj = 0; jj < k; ++jj) {
        const int src = min(x.tok0 + jj, 31);
        any_bad |= __shfl_sync(kFull, tbad, src);
        any_src |= __shfl_sync(kFull, badsrc, src);
    }
    if (x.in && x.j == 0 && any_bad) atomicExch(a.err, any_src ? 1 : 4);  // ShapeError / RoutingError
    x.valid = x.in && !any_bad;
    // an invalid token is planned with no destinations and source 0 (as plan_mask)
    x.s = any_bad ? 0 : s;
    x.e = x.valid ? e : -1;
    x.d = x.valid ? de : -1;
    x.p = x.valid ? pe : -1;
    x.w = w;
    x.dm = x.valid ? dm : 0;
    x.smask = sm;
    x.owner = x.valid && jfirst == x.j;
    x.owner_lane = x.tok0 + jfirst;
    return x;
}

// Per-warp key counts into wk[key] (zeroed): the leader of each equal-key
// lane group writes the group size.  Keys: dispatch (s, d) per owner entry,
// source group (s) per token, expert (s, e) per valid entry.
__device__ __forceinline__ void entry_counts(const FusedPlanArgs& a, const Entry& x, int* wk, int lane,
                                             uint32_t& md, uint32_t& mg, uint32_t& me) {
    const int nd = a.nd, KD = nd * (nd + 1);
    const int kd = x.owner ? x.s * (nd + 1) + x.d : -1;
    const int kg = x.in && x.j == 0 ? x.s * (nd + 1) + nd : -1;
    const int ke = x.valid ? KD + x.s * a.E + x.e : -1;
    md = __match_any_sync(kFull, kd);
    mg = __match_any_sync(kFull, kg);
    me = __match_any_sync(kFull, ke);
    if (kd >= 0 && __ffs(md) - 1 == lane) wk[kd] = __popc(md);
    if (kg >= 0 && __ffs(mg) - 1 == lane) wk[kg] = __popc(mg);
    if (ke >= 0 && __ffs(me) - 1 == lane) wk[ke] = __popc(me);
}

// OCC_PLAN_DEBUG: earliest block start / latest phase end over all blocks (ns).
__device__ __forceinline__ void phase_mark(const FusedPlanArgs& a, int i) {
    if (!a.dbg || threadIdx.x) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (i == 0) atomicMin(a.dbg, t);
    else atomicMax(a.dbg + i, t);
}

__global__ void __launch_bounds__(kThreads) fused_plan_kernel(FusedPlanArgs a) {
    pdl_trigger();
    pdl_wait();  // routing comes from the router kernel (PDL launch)
    phase_mark(a, 0);
    extern __shared__ int smem[];
    cg::grid_group grid = cg::this_grid();
    const int nd = a.nd, E = a.E, P = a.P, k = a.k;
    const int KD = nd * (nd + 1), K = KD + nd * E;
    const int tpw = 32 / k;                     // tokens per warp (one lane per routing entry)
    const int tpb = kWarps * tpw;               // tokens per block chunk
    const int nchunks = (a.n + tpb - 1) / tpb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* wcnt = smem;  // [kWarps][K] per-warp key counts / bases (phase C: the totals)
    Tables T;
    {
        int* p = wcnt + kWarps * K;
        T.C = p, p += nd * nd;
        T.off_sd = p, p += nd * nd;
        T.inoff = p, p += nd * nd;
        T.in_base = p, p += nd + 1;
        T.ntok = p, p += nd;
        T.tok_base = p, p += nd;
        T.cnt = p, p += E;        // per group g = (d, p), E = nd * P groups
        T.seg_base = p, p += E;
        T.padpre = p, p += E + 1; // prefix of padding rows per group
        T.dev = p, p += E;
        T.slot = p, p += E;
        T.ebase = p, p += nd * E; // [nd][E]
        T.pre = p, p += K;        // small mode: this block's chunk prefix per key
    }
    // global warp index, spread so consecutive work items land on different SMs
    // (blocks are placed round-robin over the SMs)
    const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * kWarps;
    for (int e = threadIdx.x; e < E; e += kThreads) {
        T.dev[e] = a.dev_of[e];
        T.slot[e] = a.slot_of[e];
    }
    __syncthreads();

    // ---------------------------------------------------------------- A --
    if (a.zero_stats && blockIdx.x == 0 && threadIdx.x < 8) a.stats[threadIdx.x] = 0;  // atomics start after the barrier
    // small count matrices (K x nchunks <= kSmallCounts): no scan phase; every
    // block sums the matrix itself (totals and its own chunk's prefix), which
    // saves a grid-wide barrier and a dependent phase on small batches
    const bool small = (long)K * nchunks <= kSmallCounts && nchunks <= (int)gridDim.x;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        for (int i = threadIdx.x; i < kWarps * K; i += kThreads) wcnt[i] = 0;
        __syncthreads();
        const Entry x = load_entry(a, T, c, tpw, warp, lane);
        uint32_t md, mg, me;
        entry_counts(a, x, wcnt + warp * K, lane, md, mg, me);
        __syncthreads();
        for (int key = threadIdx.x; key < K; key += kThreads) {
            int sum = 0;
            for (int w = 0; w < kWarps; ++w) sum += wcnt[w * K + key];
            a.chunk_cnt[(long)key * nchunks + c] = sum;
        }
        __syncthreads();
    }
    phase_mark(a, 1);
    grid.sync();
    int* tot = wcnt;  // the K totals, staged (phase C)
    if (small) {
        // one chunk per block at most: totals and this block's exclusive prefix in one pass
        // one warp per key: lanes stride over the chunks (coalesced, all loads
        // in flight together), shuffle reductions
        int* pre = T.pre;
        const int mine = blockIdx.x;
        for (int key = warp; key < K; key += kWarps) {
            const int* row = a.chunk_cnt + (long)key * nchunks;
            int t = 0, b = 0;
#pragma unroll 4
            for (int c = lane; c < nchunks; c += 32) {
                const int v = __ldcg(row + c);
                b += c < mine ? v : 0;
                t += v;
            }
            for (int o = 16; o; o >>= 1) {
                t += __shfl_xor_sync(kFull, t, o);
                b += __shfl_xor_sync(kFull, b, o);
            }
            if (lane == 0) {
                tot[key] = t;
                pre[key] = b;
            }
        }
        if (blockIdx.x == 0)
            for (int key = threadIdx.x; key < K; key += kThreads) a.totals[key] = tot[key];
        phase_mark(a, 2);
        __syncthreads();
    } else {
    // ---------------------------------------------------------------- B --
    // one block per key: each thread scans a contiguous run of chunks (loads
    // independent, in flight together), block exclusive scan of the run sums
    {
        __shared__ int s_part[kWarps];
        const int per = (nchunks + kThreads - 1) / kThreads;
        for (int key = blockIdx.x; key < K; key += gridDim.x) {
            int* row = a.chunk_cnt + (long)key * nchunks;
            const int c0 = threadIdx.x * per, c1 = min(c0 + per, nchunks);
            int local = 0;
            for (int c = c0; c < c1; ++c) local += row[c];
            int x = local;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_part[warp] = x;
            __syncthreads();
            int wbase = 0, total = 0;
            for (int w = 0; w < kWarps; ++w) {
                if (w < warp) wbase += s_part[w];
                total += s_part[w];
            }
            int run = wbase + x - local;
            for (int c = c0; c < c1; ++c) {
                const int v = row[c];
                row[c] = run;
                run += v;
            }
            if (threadIdx.x == 0) a.totals[key] = total;
            __syncthreads();
        }
    }
    phase_mark(a, 2);
    grid.sync();
    for (int i = threadIdx.x; i < K; i += kThreads) tot[i] = a.totals[i];
    __syncthreads();
    }
    // ---------------------------------------------------------------- C --
    for (int i = threadIdx.x; i < nd * nd; i += kThreads) T.C[i] = tot[(i / nd) * (nd + 1) + i % nd];
    for (int e = threadIdx.x; e < E; e += kThreads) {  // group counts from the expert keys
        int c = 0;
        for (int s = 0; s < nd; ++s) c += tot[KD + s * E + e];
        T.cnt[T.dev[e] * P + T.slot[e]] = c;
    }
    __syncthreads();
    if (threadIdx.x < nd) {  // per source: counter offsets (device-major), token counts
        const int s = threadIdx.x;
        int run = 0;
        for (int d = 0; d < nd; ++d) {
            T.off_sd[s * nd + d] = run;
            run += T.C[s * nd + d];
        }
        T.ntok[s] = tot[s * (nd + 1) + nd];
    } else if (threadIdx.x >= 64 && threadIdx.x < 64 + nd) {  // per destination: inbox offsets
        const int d = threadIdx.x - 64;
        int run = 0;
        for (int s = 0; s < nd; ++s) {
            T.inoff[d * nd + s] = run;
            run += T.C[s * nd + d];
        }
        T.in_base[d] = run;  // R_d for now
    } else if (threadIdx.x == 128) {  // Epd segments: padded to the 256-row GEMM tile
        int run = 0, pad = 0;
        for (int g = 0; g < E; ++g) {
            T.seg_base[g] = run;
            const int m = (T.cnt[g] + kBM - 1) / kBM * kBM;
            T.padpre[g] = pad;
            pad += m - T.cnt[g];
            run += m;
        }
        T.padpre[E] = pad;
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
        int run = T.seg_base[T.dev[e] * P + T.slot[e]];
        for (int s = 0; s < nd; ++s) {
            T.ebase[s * E + e] = run;
            run += tot[KD + s * E + e];
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
    phase_mark(a, 3);
    __syncthreads();  // (the staged totals in wcnt are dead from here)

    // ---------------------------------------------------------------- D --
    long long st_naive = 0, st_span = 0, st_intra = 0, st_inter = 0;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        for (int i = threadIdx.x; i < kWarps * K; i += kThreads) wcnt[i] = 0;
        __syncthreads();
        const Entry x = load_entry(a, T, c, tpw, warp, lane);
        uint32_t md, mg, me;
        entry_counts(a, x, wcnt + warp * K, lane, md, mg, me);
        __syncthreads();
        for (int key = threadIdx.x; key < K; key += kThreads) {  // exclusive bases per warp
            int run = small ? T.pre[key] : a.chunk_cnt[(long)key * nchunks + c];
            for (int w = 0; w < kWarps; ++w) {
                const int v = wcnt[w * K + key];
                wcnt[w * K + key] = run;
                run += v;
            }
        }
        __syncthreads();
        const int* wb = wcnt + warp * K;
        const uint32_t lt = lanemask_lt();
        const int s = x.s, t = x.t, d = x.d;
        int row = -1, cc = -1;
        if (x.owner) {  // BRIM0 counter and inbox row of (t, d)
            const int r = wb[s * (nd + 1) + d] + __popc(md & lt);
            cc = T.off_sd[s * nd + d] + r;
            row = T.in_base[d] + T.inoff[d * nd + s] + r;
            const long slot = (long)t * nd + d;
            a.tok_sfd[slot] = cc;
            a.tok_row[slot] = row;
            a.in_tok[row] = t;
            a.in_src[row] = s;
            a.in_slot[row] = cc;
            a.in_dev[row] = d;
            for (int p = 0; p < P; ++p)  // slots of this row the token does not use
                if (!((x.smask >> p) & 1)) a.row_epd[(long)row * P + p] = -1;
        }
        const int my_row = __shfl_sync(kFull, row, x.owner_lane);
        for (int jj = 0; jj < k; ++jj) {  // the routing row carried with each of the token's inbox rows
            const int src = min(x.tok0 + jj, 31);
            const int oe = __shfl_sync(kFull, x.e, src);
            const float ow = __shfl_sync(kFull, x.w, src);
            if (x.owner) {
                a.in_ids[(long)row * k + jj] = oe;
                a.in_w[(long)row * k + jj] = ow;
            }
        }
        if (x.in) {
            for (int dd = x.j; dd < nd; dd += k)  // devices the token does not reach
                if (!((x.dm >> dd) & 1)) {
                    a.tok_sfd[(long)t * nd + dd] = -1;
                    a.tok_row[(long)t * nd + dd] = -1;
                }
            if (x.j == 0) {
                a.lam[t] = wb[s * (nd + 1) + nd] + __popc(mg & lt);
                a.mask[t] = x.dm;
            }
        }
        if (x.valid) {  // BRIM1: the Epd row of (t, e), expert-major over device d's inbox
            const int q = T.ebase[s * E + x.e] + wb[KD + s * E + x.e] + __popc(me & lt);
            a.row_epd[(long)my_row * P + x.p] = q;
            a.epd_src[q] = my_row;
            a.epd_w[q] = x.w;
            a.epd_j[q] = x.j;
        }
        // CommReport (collab.cpp:41-118): span, naive crossings, co-activated pair shares
        for (int jj = 0; jj < k; ++jj) {
            const int od = __shfl_sync(kFull, d, min(x.tok0 + jj, 31));
            if (x.valid && jj > x.j) {
                if (od == d) ++st_intra;
                else ++st_inter;
            }
        }
        if (x.valid) {
            st_naive += d != s;
            if (x.j == 0) st_span += __popcll(x.dm);
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
    // padding rows of every segment: no source row, zero weight
    for (int pr = blockIdx.x * kThreads + threadIdx.x; pr < T.padpre[E]; pr += gridDim.x * kThreads) {
        int g = 0;
        while (T.padpre[g + 1] <= pr) ++g;
        const int q = T.seg_base[g] + T.cnt[g] + (pr - T.padpre[g]);
        a.epd_src[q] = -1;
        a.epd_w[q] = 0.0f;
    }
    phase_mark(a, 4);
    if (!a.scatter) return;  // large batches: the Epd rows are copied by a full-occupancy kernel
    grid.sync();
    // ---------------------------------------------------------------- E --
    // Epd A operand: inbox row r's token row (read once) to each of its expert
    // rows, one warp per (row, 4 KB slice); then every segment's padding rows
    // (no source row, zero weight, zero A row), one warp per row.
    const int R = T.in_base[nd];
    const int nvec = a.D / 8;
    constexpr int kSl = 256;  // uint4 per slice: 8 per lane in flight
    const int nsl = (nvec + kSl - 1) / kSl;
    const long n_copy = (long)R * nsl, n_items = n_copy + T.padpre[E];
    for (long wi = gw; wi < n_items; wi += nw) {
        if (wi >= n_copy) {  // a padding row
            const int pr = (int)(wi - n_copy);
            int g = 0;
            while (T.padpre[g + 1] <= pr) ++g;
            const int q = T.seg_base[g] + T.cnt[g] + (pr - T.padpre[g]);
            uint4* out = reinterpret_cast<uint4*>(a.x_epd + (long)q * a.D);
            for (int v = lane; v < nvec; v += 32) out[v] = make_uint4(0, 0, 0, 0);
            continue;
        }
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
    phase_mark(a, 5);
}

size_t fused_smem(int nd, int E, int k) {
    const int K = nd * (nd + 1) + nd * E;
    const int tabs = 3 * nd * nd + (nd + 1) + 2 * nd + 5 * E + 1 + nd * E + K;
    (void)k;
    return sizeof(int) * ((size_t)kWarps * K + tabs);
}

}  // namespace

size_t fused_plan_chunks(int n, int k) {
    const int tpb = kWarps * (32 / k);
    return (size_t)(n + tpb - 1) / tpb;
}

size_t fused_plan_ws(int n, int nd, int E, int k) {
    const size_t K = (size_t)nd * (nd + 1) + (size_t)nd * E;
    return K * (fused_plan_chunks(n, k) + 1);
}

bool fused_plan_supported(int nd, int E, int k) {
    return nd <= 64 && E <= 256 && k <= 32 && fused_smem(nd, E, k) <= 96 * 1024;
}

bool launch_fused_plan(const FusedPlanArgs& a, int num_sms, cudaStream_t st) {
    if (a.n <= 0) return true;
    const size_t smem = fused_smem(a.nd, a.E, a.k);
    static int configured = 0;
    if (!configured) {
        cudaFuncSetAttribute(fused_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        configured = 1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_plan_kernel, kThreads, smem) != cudaSuccess ||
        per_sm < 1)
        return false;
    int blocks = num_sms * std::min(per_sm, 4);
    static const int blocks_env = getenv("OCC_PLAN_BLOCKS") ? atoi(getenv("OCC_PLAN_BLOCKS")) : 0;  // sweeps (profiles/)
    if (blocks_env > 0) blocks = std::min(blocks_env, num_sms * per_sm);
    FusedPlanArgs args = a;
    static const bool dbg_on = getenv("OCC_PLAN_DEBUG") != nullptr;  // phase timeline (diagnostics only)
    static unsigned long long* dbg = nullptr;
    if (dbg_on) {
        if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 8);
        cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 8, st);
        cudaMemsetAsync(dbg, 0xFF, sizeof(unsigned long long), st);
        args.dbg = dbg;
    }
    // cooperative (grid-wide barriers) and, when allowed, programmatic: the
    // kernel's blocks become resident while the router drains
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    if (cudaLaunchKernelEx(&cfg, fused_plan_kernel, args) != cudaSuccess) {
        cudaGetLastError();
        if (cfg.numAttrs == 1) return false;
        cfg.numAttrs = 1;  // this driver refuses cooperative + programmatic: plain cooperative launch
        if (cudaLaunchKernelEx(&cfg, fused_plan_kernel, args) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
    }
    count_launch();
    if (dbg_on) {
        unsigned long long h[8];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[plan dbg] n=%d nd=%d E=%d blocks=%d: A %.1f  B %.1f  C %.1f  D %.1f  E %.1f us (from start)\n",
                a.n, a.nd, a.E, blocks, (h[1] - h[0]) / 1e3, (h[2] - h[0]) / 1e3, (h[3] - h[0]) / 1e3,
                (h[4] - h[0]) / 1e3, (h[5] - h[0]) / 1e3);
    }
    return true;
}

}  // namespace occ
