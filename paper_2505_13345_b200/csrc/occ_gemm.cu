// occ_gemm.cu — grouped per-expert GEMMs on 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM, operands staged by TMA).
//
// Forward: replaces the reference's two indexed matmul loops,
// scatter_matmul (pipeline.cpp:178-211, Alg. 6; fused here with
// apply_activation :213-224 and weight_modulate :226-248, Alg. 7) and
// merge_matmul (pipeline.cpp:250-283, Alg. 8).  Backward (backward.cpp:24-161):
// the two data-gradient GEMMs (merge/scatter adjoints, pipeline.cpp:302-344)
// with the modulation/activation adjoints fused in the epilogue, and the two
// per-expert weight-gradient GEMMs.
//
// Rows of every expert are contiguous and padded to the 256-row pair tile
// (compute-index segments), so each forward/data-gradient tile belongs to
// exactly one expert and B is that expert's resident weight slice; a
// weight-gradient tile reduces over exactly one expert's rows.
//
// Persistent, warp-specialised, CTA pairs (cluster 2x1x1, cta_group::2):
// one 256x256 output tile per pair, each CTA staging its 128 A rows and its
// half (128 rows) of the B tile per 64-deep K block (32 KB per CTA, 6 stages
// in 192 KB of shared memory, 128-byte swizzle).
//   warp 0      TMA producer in both CTAs (completion on the leader's barrier)
//   warp 1      TMEM allocator (both CTAs) + single-thread tcgen05.mma issuer
//               in the leader CTA (M=256, N=256, K=16, fp32 accumulate)
//   warps 2..5  epilogue in both CTAs: tcgen05.ld -> fused epilogue ->
//               global stores; double-buffered TMEM accumulators (2 x 256
//               columns) overlap the epilogue with the next tile's MMAs.
// Operand majorness: forward/data-gradient GEMMs read both operands K-major
// ([rows, K] row-major, 64x128 TMA boxes); weight-gradient GEMMs reduce over
// the token rows, so both operands are read MN-major straight from the same
// row-major activation buffers (2 x 64x64 boxes, tcgen05 MN-major
// descriptors) — no transposes.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>

#include <algorithm>

#include "occ_common.cuh"
#include "occ_internal.h"

namespace occ {
namespace {

constexpr int BM = 128;               // rows per CTA (pair tile: 256)
#ifndef OCC_GEMM_STAGES
#define OCC_GEMM_STAGES 6
#endif
#ifndef OCC_STG_PER_WARP
#define OCC_STG_PER_WARP 1
#endif
constexpr int BN = 256, BK = 64, STAGES = OCC_GEMM_STAGES;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = (BN / 2) * BK * 2;  // 16 KB: this CTA's half of the B tile
// Epilogue staging for TMA stores: per epilogue warp two 32-row x 32-column
// bf16 buffers (2 KB each, 64-byte swizzle) = 16 KB.
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, each on half of the tile's columns
constexpr int STG_BYTES = 2048;
constexpr int STG_PER_WARP = OCC_STG_PER_WARP;  // staging buffers per epilogue warp (TMA stores in flight)
constexpr int EPI_STAGE_BYTES = EPI_WARPS * STG_PER_WARP * STG_BYTES;
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + EPI_STAGE_BYTES + 256;
constexpr int THREADS = 64 + 32 * 8;  // producer + MMA + EPI_WARPS epilogue warps
constexpr int MAX_GROUPS = 256;
static_assert(kBM == 2 * BM, "Epd segments are padded to the pair tile");

// K-major SW128 descriptors advance 32 B per K=16 step inside the swizzle
// atom; MN-major SW128 tiles are two 64-column boxes (LBO = 8 KB apart) of
// 8-row x 128 B atoms (SBO = 1 KB), advancing 16 rows = 2 KB per K step.
OCC_DEV uint64_t sdesc_mn_sw128(uint32_t smem_addr) {
    return (uint64_t)((smem_addr & 0x3FFFF) >> 4) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_mn(int m, int n) {
    return idesc_bf16_f32(m, n) | (1u << 15) | (1u << 16);  // A and B MN-major
}

struct Params {
    int K, N, b_rows_per_e, act;
    const int* grp_mb;  // forward: m-tile prefix per group
    const int* grp_w;
    int ngroups, band;
    const int* grp_cnt;   // wgrad: rows per group
    const int* seg_base;  // wgrad: first padded row per group
    int M;                // wgrad: output rows (the MN extent of A)
    const float* row_w;
    void* out;
    int ldo;
    long out_estride;  // wgrad: elements per expert in out/out2
    void* out2;
    int split;
    __nv_bfloat16* save_a;  // forward training: pre-activations
    __nv_bfloat16* save_b;
    const __nv_bfloat16* pre_a;  // backward epilogue inputs
    const __nv_bfloat16* pre_b;
    float* gw_part;
    int tma_out;         // bf16 forward outputs leave through smem + TMA stores (tmC)
    unsigned long long* dbg;  // OCC_GEMM_DEBUG: per-CTA stall cycles [cta][4]
    unsigned long long* tl;   // OCC_GEMM_TIMELINE: globaltimer per CTA at 8 points [cta][8]
    int tail_split;           // wide kernel: split the tail wave's super-tiles into halves
    int hint;                 // L2 policies: 1 B loads evict_first, 2 C stores evict_first, 4 A loads evict_last
    int* sched;               // dynamic tile scheduler [next tile, pairs done]; null = static cid + i * ncl
    const int* a_rows;   // non-null: A row q of the padded Epd layout is row a_rows[q] of tmA
                         // (tile::gather4, box 64 x 1; -1 = zero padding row)
};

// Tile scheduling.  Static: pair c runs tiles c, c + ncl, c + 2 ncl, ...
// Dynamic (p.sched): the first tile is still c, every further one is taken
// from a global counter in launch order, so the pairs that share an operand
// (the 16 m-tiles of one B block, the n-blocks of one A m-tile) start it
// within a fraction of a tile of each other however the pairs' speeds drift
// over ~100 waves -- with the static walk they drift apart by more than the
// ~80 MB the L2 holds between two reads (profiles/r02_gemm_l2.md).  The
// leader's producer thread is the scheduler: it publishes each tile index
// into a 4-deep ring in both CTAs' shared memory -- locally a store + arrive,
// into the peer with st.async completing the transaction count of the peer's
// barrier (the TMA-load contract: no cluster-scope fence, which cost a GPU
// membar per consumer warp per tile); the consumers (peer producer, MMA
// issuer, 16 epilogue warps) hand slots back on the leader's `empty`
// barrier.  The last pair to finish re-zeroes the counter for the next launch.
constexpr int TQN = 4;
constexpr int TQ_CONSUMERS = 2 + 2 * 8;  // peer producer + MMA issuer + epilogue warps of both CTAs
struct TileQueue {
    int* tile;        // [TQN] this CTA's copy of the published indices
    uint64_t* full;   // [TQN] this CTA: index published
    uint64_t* empty;  // [TQN] leader: slot consumed by every consumer
    int cid, ncl;
    bool dyn;
    // i-th tile of this pair (every lane of a consuming warp calls it)
    __device__ __forceinline__ int get(int i) const {
        if (!dyn) return cid + i * ncl;
        const int s = i % TQN;
        mbar_wait(&full[s], (i / TQN) & 1);
        return ld_shared_s32(&tile[s]);
    }
    // one thread per consuming warp, after every lane's get(i) (the index is
    // in registers: the slot may be rewritten)
    __device__ __forceinline__ void release(int i, uint32_t rank) const {
        if (!dyn) return;
        const int s = i % TQN;
        if (rank == 0) mbar_arrive(&empty[s]);
        else mbar_arrive_cluster(mapa_rank(&empty[s], 0));
    }
    // scheduler (leader producer thread): publish the i-th tile to both CTAs
    __device__ __forceinline__ void publish(int i, int t) const {
        const int s = i % TQN;
        mbar_wait(&empty[s], ((i / TQN) & 1) ^ 1);
        tile[s] = t;
        mbar_arrive(&full[s]);
        const uint32_t rbar = mapa_rank(&full[s], 1);
        mbar_arrive_expect_tx_cluster(rbar, 4);
        st_async_s32(mapa_rank(&tile[s], 1), t, rbar);
    }
};
// end of kernel (after the final cluster sync): the last pair re-zeroes the counter
__device__ __forceinline__ void sched_done(int* sched, int ncl) {
    __threadfence();
    if (atomicAdd(sched + 1, 1) == ncl - 1) {
        atomicExch(sched, 0);
        atomicExch(sched + 1, 0);
        __threadfence();
    }
}

// Forward / data-gradient tiles: expert group by group, bands of `band`
// m-tiles walked n-block-major (resident CTAs share B n-blocks, a band's A
// rows stay in L2; no band straddles two experts).
// Largest g in [0, ng) with pre[g] * scale <= tile (pre non-decreasing): the
// group of a tile.  Binary search: every role decodes every tile, and the
// linear walk over 64 experts' prefixes (dependent shared loads) was ~15% of
// the warp-stall samples of the 64-expert GEMMs (ncu source view).
__device__ __forceinline__ int group_of(int tile, const int* pre, int ng, int scale) {
    int lo = 0, hi = ng - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] * scale <= tile) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void tile_coords(int tile, const int* gmb, const int* gw, int ng, int NB, int band,
                                            int& mb, int& nb, int& w) {
    const int g = group_of(tile, gmb, ng, NB);
    const int lt = tile - gmb[g] * NB;
    const int cnt = gmb[g + 1] - gmb[g];
    const int b = lt / (band * NB);
    const int rem = lt - b * band * NB;
    int bm = cnt - b * band;
    bm = bm < band ? bm : band;
    nb = rem / bm;
    mb = gmb[g] + b * band + rem % bm;
    w = gw[g];
}

// Weight-gradient tiles: (group, m-tile, n-tile) over groups with rows.
__device__ __forceinline__ void wtile_coords(int tile, const int* tb, int ng, int NB, int& g, int& mt, int& nt) {
    g = group_of(tile, tb, ng, 1);
    const int lt = tile - tb[g];
    mt = lt / NB;
    nt = lt - mt * NB;
}

// Activations (0 identity, 1 SiLU, 2 ReLU) as compile-time functors.  The
// runtime activation is dispatched ONCE per 32-value chunk (act_dispatch), not
// per element: a per-element switch puts a branch between the elements, so
// their dependent MUFU chains (ex2 -> rcp) cannot interleave and a chunk took
// ~1.5 us instead of ~0.1 us (OCC_GEMM_TIMELINE on the C1 layer; identity
// chunks 0.6 us) -- the epilogue, not the MMAs, then bounded short-K GEMMs.
template <int A>
__device__ __forceinline__ float act_t(float v) {
    if constexpr (A == 1) return silu(v);
    else if constexpr (A == 2) return v > 0.f ? v : 0.f;
    else return v;
}
template <int A>
__device__ __forceinline__ float act_grad_t(float v) {  // backward.cpp:11-20
    if constexpr (A == 1) {
        const float s = sigmoid_fast(v);
        return s * (1.0f + v * (1.0f - s));
    } else if constexpr (A == 2) {
        return v > 0.f ? 1.f : 0.f;
    } else {
        return 1.f;
    }
}
template <int A>
struct ActTag {
    static constexpr int value = A;
};
template <typename Fn>
__device__ __forceinline__ void act_dispatch(int act, Fn&& fn) {
    if (act == 1) fn(ActTag<1>());
    else if (act == 2) fn(ActTag<2>());
    else fn(ActTag<0>());
}

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* p, const float (&h)[32], int valid_cols) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (u * 8 < valid_cols) {
            uint4 o;
            o.x = pack_bf16(h[8 * u + 0], h[8 * u + 1]);
            o.y = pack_bf16(h[8 * u + 2], h[8 * u + 3]);
            o.z = pack_bf16(h[8 * u + 4], h[8 * u + 5]);
            o.w = pack_bf16(h[8 * u + 6], h[8 * u + 7]);
            *reinterpret_cast<uint4*>(p + 8 * u) = o;
        }
}

__device__ __forceinline__ void unpack_bf16x32(const uint4 (&w)[4], float (&f)[32]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 x = __bfloat1622float2(h[q]);
            f[8 * u + 2 * q] = x.x;
            f[8 * u + 2 * q + 1] = x.y;
        }
    }
}

// Backward epilogue outputs, warp-cooperative and coalesced: a warp's 32 rows
// x 32 columns bf16 block leaves the one-row-per-thread layout of tcgen05.ld
// 32x32b through the warp's 2 KB smem staging buffer (64-byte swizzle,
// conflict-free both ways) as 4 stores of 8 rows x 64 B (instead of 32
// row-scattered 16 B accesses per instruction).  Lane L, step u covers row
// u*8 + L/4, 16-byte chunk L%4.
__device__ __forceinline__ uint32_t stg_off(int r, int c) { return r * 64 + ((c ^ ((r >> 1) & 3)) << 4); }

// this lane's row (32 floats -> bf16) -> coalesced global stores
__device__ __forceinline__ void row_to_global(uint8_t* stg, const float (&h)[32], __nv_bfloat16* base, long ld,
                                              int ncols, int lane) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint4 o;
        o.x = pack_bf16(h[8 * c + 0], h[8 * c + 1]);
        o.y = pack_bf16(h[8 * c + 2], h[8 * c + 3]);
        o.z = pack_bf16(h[8 * c + 4], h[8 * c + 5]);
        o.w = pack_bf16(h[8 * c + 6], h[8 * c + 7]);
        sts128(stg + stg_off(lane, c), o);
    }
    __syncwarp();
    const int c = lane & 3;
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (c * 8 < ncols)
            reinterpret_cast<uint4*>(base + (long)(u * 8 + (lane >> 2)) * ld)[c] =
                lds128(stg + stg_off(u * 8 + (lane >> 2), c));
    __syncwarp();
}
// Saved pre-activations (training forward -> backward epilogue, internal to
// the library) are stored in 32-row x 32-column tiles, lane-major: element
// (r, c) of tile (R, C) at ((R * CT + C) * 4 + c / 8) * 256 + (r % 32) * 8 + c % 8,
// CT = ceil(N / 32) tiles per 32-row band.  The epilogue lane that owns row r
// (tcgen05.ld 32x32b: one row per lane) then writes -- forward -- and reads --
// backward -- its 32 values of a chunk as 4 x 16 bytes with every warp access
// one contiguous 512-byte run: no shared-memory transposes (which were ~1/4 of
// the backward epilogue's instructions).
__device__ __forceinline__ long pre_tile(long rowbase, int col0, int N) {
    return ((rowbase >> 5) * ((N + 31) >> 5) + (col0 >> 5)) * 1024;
}
__device__ __forceinline__ void store_pre_tiled(__nv_bfloat16* base, long rowbase, int col0, int N, int lane,
                                                const float (&h)[32]) {
    uint4* t = reinterpret_cast<uint4*>(base + pre_tile(rowbase, col0, N)) + lane;
#pragma unroll
    for (int u = 0; u < 4; ++u)
        t[u * 32] = make_uint4(pack_bf16(h[8 * u + 0], h[8 * u + 1]), pack_bf16(h[8 * u + 2], h[8 * u + 3]),
                               pack_bf16(h[8 * u + 4], h[8 * u + 5]), pack_bf16(h[8 * u + 6], h[8 * u + 7]));
}
// this lane's row of a chunk's pre-activations (rows rowbase..+31, columns col0..+31)
template <int EPI>
__device__ __forceinline__ void load_pre_chunk(const Params& p, long rowbase, int col0, int lane, uint4 (&A)[4],
                                               uint4 (&B)[4]) {
    if (col0 >= p.N) return;
    const long t = pre_tile(rowbase, col0, p.N);
    const uint4* ta = reinterpret_cast<const uint4*>(p.pre_a + t) + lane;
#pragma unroll
    for (int u = 0; u < 4; ++u) A[u] = __ldg(ta + u * 32);
    if constexpr (EPI == EPI_BWD_SWIGLU) {
        const uint4* tb = reinterpret_cast<const uint4*>(p.pre_b + t) + lane;
#pragma unroll
        for (int u = 0; u < 4; ++u) B[u] = __ldg(tb + u * 32);
    }
}

__device__ __forceinline__ void tl_mark(const Params& p, int i) {
    if (!p.tl) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.tl[blockIdx.x * 16 + i] = t;
}

__device__ __forceinline__ void store_c(const CUtensorMap* tmC, const void* stg, int x, int y, int hint) {
    if (hint & 2) tma_store_2d_hint(tmC, stg, x, y, l2_policy_evict_first());
    else tma_store_2d(tmC, stg, x, y);
}
// This lane's row of a 32 x 32 bf16 block (rows y..y+31, columns x..x+31)
// out through the warp's 2 KB staging buffer (64-byte swizzle) and one TMA
// store; waits for the buffer's previous store to have read it.
__device__ __forceinline__ void row_to_tma(const CUtensorMap* tmC, uint8_t* stg, const float (&h)[32], int x, int y,
                                           int lane) {
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u)
        sts128(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4),
               make_uint4(pack_bf16(h[8 * u + 0], h[8 * u + 1]), pack_bf16(h[8 * u + 2], h[8 * u + 3]),
                          pack_bf16(h[8 * u + 4], h[8 * u + 5]), pack_bf16(h[8 * u + 6], h[8 * u + 7])));
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        tma_store_2d(tmC, stg, x, y);
        bulk_commit();
    }
}

template <int EPI, bool WGRAD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint8_t* sC = sB + STAGES * B_BYTES;  // epilogue staging (1024-aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(sC + EPI_STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* tq_full = tempty + 2;
    uint64_t* tq_empty = tq_full + TQN;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_empty + TQN);
    __shared__ int s_gmb[MAX_GROUPS + 1];  // forward: m-tile prefix; wgrad: tile prefix
    __shared__ int s_gw[MAX_GROUPS];
    __shared__ int s_tq[TQN];
    __shared__ int s_kb0[MAX_GROUPS];      // wgrad: first K block / K block count per group
    __shared__ int s_kbn[MAX_GROUPS];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) tl_mark(p, 0);
    const int NB = WGRAD ? (p.N + BN - 1) / BN : (EPI == EPI_SWIGLU_BF16 ? (p.N + 127) / 128 : (p.N + BN - 1) / BN);
    const int MT = (p.M + 2 * BM - 1) / (2 * BM);  // wgrad m-tiles
    pdl_trigger();
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        if (p.tma_out) tma_prefetch_desc(&tmC);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);   // leader: one expect_tx arrival + both CTAs' bytes
            mbar_init(&empty[s], 1);  // one multicast commit per phase
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * EPI_WARPS);  // leader: epilogue warps of both CTAs
        }
        for (int s = 0; s < TQN; ++s) {
            mbar_init(&tq_full[s], 1);
            mbar_init(&tq_empty[s], TQ_CONSUMERS);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // the group tables come from the index chain (previous kernels): after the
    // prologue above, which overlaps the predecessor's tail under PDL
    pdl_wait();
    if constexpr (WGRAD) {
        if (threadIdx.x == 0) {
            int run = 0;
            for (int g = 0; g < p.ngroups; ++g) {
                s_gmb[g] = run;
                const int rows = p.grp_cnt[g];
                s_kb0[g] = p.seg_base[g] / BK;
                s_kbn[g] = (rows + BK - 1) / BK;
                if (rows > 0) run += MT * NB;
            }
            s_gmb[p.ngroups] = run;
        }
        for (int i = threadIdx.x; i < p.ngroups; i += blockDim.x) s_gw[i] = p.grp_w[i];
    } else {
        for (int i = threadIdx.x; i <= p.ngroups; i += blockDim.x) s_gmb[i] = p.grp_mb[i];
        for (int i = threadIdx.x; i < p.ngroups; i += blockDim.x) s_gw[i] = p.grp_w[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) tl_mark(p, 1);

    const int num_tiles = WGRAD ? s_gmb[p.ngroups] : s_gmb[p.ngroups] * NB;
    const int KB_fwd = (p.K + BK - 1) / BK;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const bool compact = num_tiles <= 2 * ncl;  // <= 2 tiles per CTA: rolled epilogue (see there)
    const TileQueue tq{s_tq, tq_full, tq_empty, cid, ncl, p.sched != nullptr};

    if (warp == 0 && !WGRAD && p.a_rows) {
        // ------------------------------------------------ TMA producer, gathered A rows:
        // each lane gathers 4 of the CTA's 128 A rows per K block (tile::gather4
        // straight from the inbox / token rows: no Epd copy of the activations)
        int stage = 0;
        uint32_t phase = 0;
        int next = cid;
        for (int i = 0;; ++i) {
            int tile = 0;
            if (tq.dyn && rank == 0) {
                if (lane == 0) {
                    tq.publish(i, next);
                    tile = next;
                    if (tile < num_tiles) next = ncl + atomicAdd(p.sched, 1);
                }
                tile = __shfl_sync(0xffffffffu, tile, 0);
            } else {
                tile = tq.get(i);
                __syncwarp();
                if (lane == 0) tq.release(i, rank);
            }
            if (tile >= num_tiles) break;
            int mb, nb, wi;
            tile_coords(tile, s_gmb, s_gw, p.ngroups, NB, p.band, mb, nb, wi);
            const int q0 = mb * 2 * BM + rank * BM;
            const int4 rows = __ldg(reinterpret_cast<const int4*>(p.a_rows + q0) + lane);
            const int by = wi * p.b_rows_per_e + nb * BN + rank * (BN / 2);
            for (int kb = 0; kb < KB_fwd; ++kb) {
                if (lane == 0) mbar_wait(&empty[stage], phase ^ 1);
                __syncwarp();
                const uint32_t lbar = smem_u32(&full[stage]) & kPeerBitMask;
                uint8_t* a_dst = sA + stage * A_BYTES;
                if (lane == 0) {
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
                    tma_load_2d_cg2(sB + stage * B_BYTES, &tmB, lbar, kb * BK, by);
                }
                tma_gather4_cg2(a_dst + lane * 512, &tmA, lbar, kb * BK, rows);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int next = cid;
            for (int i = 0;; ++i) {
                int tile;
                if (tq.dyn && rank == 0) {
                    tile = next;
                    tq.publish(i, tile);
                    if (tile < num_tiles) next = ncl + atomicAdd(p.sched, 1);
                } else {
                    tile = tq.get(i);
                    tq.release(i, rank);
                }
                if (tile >= num_tiles) break;
                int kb0 = 0, KB = KB_fwd, ax = 0, ay = 0, bx = 0, by = 0;
                if constexpr (WGRAD) {
                    int g, mt, nt;
                    wtile_coords(tile, s_gmb, p.ngroups, NB, g, mt, nt);
                    kb0 = s_kb0[g];
                    KB = s_kbn[g];
                    ax = mt * 2 * BM + rank * BM;    // MN columns of A
                    bx = nt * BN + rank * (BN / 2);  // MN columns of B
                } else {
                    int mb, nb, wi;
                    tile_coords(tile, s_gmb, s_gw, p.ngroups, NB, p.band, mb, nb, wi);
                    ay = mb * 2 * BM + rank * BM;
                    by = wi * p.b_rows_per_e + nb * BN + rank * (BN / 2);
                }
                for (int kb = 0; kb < KB; ++kb) {
                    { const long long t0 = p.dbg ? clock64() : 0;
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (p.dbg) p.dbg[blockIdx.x * 4 + 0] += clock64() - t0; }
                    const uint32_t lbar = smem_u32(&full[stage]) & kPeerBitMask;
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
                    uint8_t* a_dst = sA + stage * A_BYTES;
                    uint8_t* b_dst = sB + stage * B_BYTES;
                    if constexpr (WGRAD) {
                        const int k = (kb0 + kb) * BK;  // token rows of this K block
                        tma_load_2d_cg2(a_dst, &tmA, lbar, ax, k);
                        tma_load_2d_cg2(a_dst + A_BYTES / 2, &tmA, lbar, ax + 64, k);
                        tma_load_2d_cg2(b_dst, &tmB, lbar, bx, k);
                        tma_load_2d_cg2(b_dst + B_BYTES / 2, &tmB, lbar, bx + 64, k);
                    } else {
                        if (p.hint & 4) tma_load_2d_cg2_hint(a_dst, &tmA, lbar, kb * BK, ay, l2_policy_evict_last());
                        else tma_load_2d_cg2(a_dst, &tmA, lbar, kb * BK, ay);
                        if (p.hint & 1) tma_load_2d_cg2_hint(b_dst, &tmB, lbar, kb * BK, by, l2_policy_evict_first());
                        else tma_load_2d_cg2(b_dst, &tmB, lbar, kb * BK, by);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (rank == 0) {
            constexpr uint32_t IDESC = WGRAD ? idesc_mn(2 * BM, BN) : idesc_bf16_f32(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int i = 0;; ++i) {
                const int tile = tq.get(i);
                __syncwarp();
                if (lane == 0) tq.release(i, rank);
                if (tile >= num_tiles) break;
                int KB = KB_fwd;
                if constexpr (WGRAD) {
                    int g, mt, nt;
                    wtile_coords(tile, s_gmb, p.ngroups, NB, g, mt, nt);
                    KB = s_kbn[g];
                }
                { const long long t0 = p.dbg ? clock64() : 0;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                if (p.dbg && lane == 0) p.dbg[blockIdx.x * 4 + 1] += clock64() - t0; }
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < KB; ++kb) {
                    { const long long t0 = p.dbg ? clock64() : 0;
                    mbar_wait(&full[stage], phase);
                    if (p.dbg && lane == 0) p.dbg[blockIdx.x * 4 + 2] += clock64() - t0; }
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t ad = WGRAD ? sdesc_mn_sw128(a0 + k * 2048) : sdesc_k_sw128(a0 + k * 32);
                            const uint64_t bd = WGRAD ? sdesc_mn_sw128(b0 + k * 2048) : sdesc_k_sw128(b0 + k * 32);
                            umma_bf16_cg2(d_tmem, ad, bd, IDESC, (kb | k) != 0);
                        }
                        umma_commit_cg2_mc(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (lane == 0) umma_commit_cg2_mc(&tfull[acc]);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ epilogue
        const int q = warp & 3;           // TMEM lane quarter accessible to this warp
        const int hsel = (warp - 2) >> 2;  // which half of the tile's 32-column chunks
        uint32_t stg_n = 0;      // TMA-store staging buffer counter
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int tile = tq.get(i);
            __syncwarp();
            if (lane == 0) tq.release(i, rank);
            if (tile >= num_tiles) break;
            // backward epilogue inputs (pre-activations) of this tile's first
            // chunk are fetched before waiting for the accumulator, so their
            // latency hides under the tile's MMAs
            uint4 pa_cur[4], pb_cur[4];
            if constexpr (!WGRAD && (EPI == EPI_BWD_ACT || EPI == EPI_BWD_SWIGLU)) {
                int mb0, nb0, wi0;
                tile_coords(tile, s_gmb, s_gw, p.ngroups, NB, p.band, mb0, nb0, wi0);
                const long rowbase0 = (long)mb0 * 2 * BM + rank * BM + q * 32;
                const int colh = nb0 * BN + hsel * (BN / 64) * 32;
                load_pre_chunk<EPI>(p, rowbase0, colh, lane, pa_cur, pb_cur);
                // the later chunks' inputs into L2 now (one register-free prefetch per
                // 128-byte line of this lane's row): their loads, one chunk ahead of
                // the math, then hit L2 instead of waiting on DRAM (ncu: the
                // transposes' staging stores stalled on those loads)
#ifndef OCC_NO_BWD_PF
                if (colh < p.N) {  // this warp's chunks: consecutive 2 KB tiles, 128 B per lane each
                    const long t0 = pre_tile(rowbase0, colh, p.N);
                    const int ntiles = min(BN / 64, (p.N - colh + 31) / 32);
                    for (int tt = 0; tt < ntiles; ++tt) {
                        prefetch_l2(p.pre_a + t0 + tt * 1024 + lane * 64);
                        if constexpr (EPI == EPI_BWD_SWIGLU) prefetch_l2(p.pre_b + t0 + tt * 1024 + lane * 64);
                    }
                }
#endif
            }
            { const long long t0 = p.dbg ? clock64() : 0;
            mbar_wait(&tfull[acc], acc_phase);
            if (p.dbg && lane == 0 && warp == 2) p.dbg[blockIdx.x * 4 + 3] += clock64() - t0; }
            if (warp == 2 && lane == 0 && tile == cid) tl_mark(p, 2);  // first accumulator ready
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            bool released = false;  // TMEM buffer handed back to the MMA warp early
            if constexpr (WGRAD) {
                // dW[e][m][n] = sum over the expert's rows; every tile is complete
                int g, mt, nt;
                wtile_coords(tile, s_gmb, p.ngroups, NB, g, mt, nt);
                const int m = mt * 2 * BM + rank * BM + q * 32 + lane;
                const long ebase = (long)s_gw[g] * p.out_estride;
#pragma unroll 1
                for (int c = hsel * (BN / 64); c < (hsel + 1) * (BN / 64); ++c) {
                    uint32_t v[32];
                    tmem_ld32(tbase + c * 32, v);
                    tmem_ld_wait();
                    const int col0 = nt * BN + c * 32;
                    if (m >= p.M) continue;
                    float* o = reinterpret_cast<float*>(p.out) + ebase + (long)m * p.ldo;
                    int c0 = col0;
                    if (p.out2 && col0 >= p.split) {
                        o = reinterpret_cast<float*>(p.out2) + ebase + (long)m * p.ldo;
                        c0 = col0 - p.split;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (col0 + u * 4 < p.N)
                            *reinterpret_cast<float4*>(o + c0 + u * 4) =
                                make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]),
                                            __uint_as_float(v[4 * u + 2]), __uint_as_float(v[4 * u + 3]));
                }
            } else {
                int mb, nb, wi;
                tile_coords(tile, s_gmb, s_gw, p.ngroups, NB, p.band, mb, nb, wi);
                const long row = (long)mb * 2 * BM + rank * BM + q * 32 + lane;
                if constexpr (EPI == EPI_F32) {
                    float* out = reinterpret_cast<float*>(p.out) + row * p.ldo;
#pragma unroll 1
                    for (int c = hsel * (BN / 64); c < (hsel + 1) * (BN / 64); ++c) {
                        uint32_t v[32];
                        tmem_ld32(tbase + c * 32, v);
                        tmem_ld_wait();
                        const int col0 = nb * BN + c * 32;
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (col0 + u * 4 < p.N)
                                *reinterpret_cast<float4*>(out + col0 + u * 4) =
                                    make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]),
                                                __uint_as_float(v[4 * u + 2]), __uint_as_float(v[4 * u + 3]));
                    }
                } else if constexpr (EPI == EPI_BWD_ACT || EPI == EPI_BWD_SWIGLU) {
                    // g_mod = g_y W2^T in TMEM; modulation + activation adjoints
                    // (backward.cpp:95-118): routing-weight partial <act, g_mod>,
                    // g_pre = g_mod * w * act'(pre)  (SwiGLU: g_a, g_b).
                    const float wr = p.row_w[row];
                    const int F = p.N;
                    float gw = 0.f;
                    const long rowbase = row - lane;
                    uint8_t* stg = sC + (warp - 2) * STG_PER_WARP * STG_BYTES;
                    __nv_bfloat16* outb = reinterpret_cast<__nv_bfloat16*>(p.out) + rowbase * p.ldo;
#pragma unroll 1
                    for (int c = hsel * (BN / 64); c < (hsel + 1) * (BN / 64); ++c) {
                        const int col0 = nb * BN + c * 32;
                        uint4 pa_nxt[4], pb_nxt[4];  // prefetch the next chunk's inputs
                        if (c + 1 < (hsel + 1) * (BN / 64)) load_pre_chunk<EPI>(p, rowbase, col0 + 32, lane, pa_nxt, pb_nxt);
                        uint32_t v[32];
                        tmem_ld32(tbase + c * 32, v);
                        tmem_ld_wait();
                        if (col0 < F) {  // warp-uniform
                            const int nv = F - col0 < 32 ? F - col0 : 32;
                            float a[32], r0[32];
                            unpack_bf16x32(pa_cur, a);
                            if constexpr (EPI == EPI_BWD_SWIGLU) {
                                float b[32], r1[32];
                                unpack_bf16x32(pb_cur, b);
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    const float gm = i < nv ? __uint_as_float(v[i]) : 0.f;
                                    const float s = sigmoid_fast(a[i]);
                                    const float sa = a[i] * s;
                                    gw += sa * b[i] * gm;
                                    const float gh = gm * wr;
                                    r0[i] = gh * b[i] * s * (1.0f + a[i] * (1.0f - s));
                                    r1[i] = gh * sa;
                                }
                                if (p.tma_out) {  // (SwiGLU: F % 128 == 0, whole blocks)
                                    row_to_tma(&tmC, stg, r0, col0, (int)rowbase, lane);
                                    row_to_tma(&tmC, stg, r1, F + col0, (int)rowbase, lane);
                                } else {
                                    row_to_global(stg, r0, outb + col0, p.ldo, F - col0, lane);
                                    row_to_global(stg, r1, outb + F + col0, p.ldo, F - col0, lane);
                                }
                            } else {
                                act_dispatch(p.act, [&](auto tag) {
                                    constexpr int A = decltype(tag)::value;
#pragma unroll
                                    for (int i = 0; i < 32; ++i) {
                                        const float gm = i < nv ? __uint_as_float(v[i]) : 0.f;
                                        gw += act_t<A>(a[i]) * gm;
                                        r0[i] = gm * wr * act_grad_t<A>(a[i]);
                                    }
                                });
                                // (the map's width is F: a partial last block is clipped)
                                if (p.tma_out) row_to_tma(&tmC, stg, r0, col0, (int)rowbase, lane);
                                else row_to_global(stg, r0, outb + col0, p.ldo, F - col0, lane);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            pa_cur[u] = pa_nxt[u];
                            pb_cur[u] = pb_nxt[u];
                        }
                    }
                    p.gw_part[(row * NB + nb) * 2 + hsel] = gw;
                } else {
                    const float wr = p.row_w ? p.row_w[row] : 1.0f;
                    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo;
                    constexpr bool SW = EPI == EPI_SWIGLU_BF16;
                    constexpr int NCH = SW ? 4 : BN / 32;  // 32-column chunks per tile
                    constexpr int MY = NCH / 2;            // this warp's half
                    const int ncol = SW ? 128 : BN;
                    if (compact && !p.save_a && p.tma_out) {
                        // At most two tiles per CTA (no tile i+2 waits on this accumulator):
                        // one chunk at a time in a rolled loop, so one chunk's instructions
                        // serve every chunk.  With a single tile per CTA the unrolled drain
                        // below is bound by cold instruction fetch, not by its math (~1.7 us
                        // per 32-column chunk, OCC_GEMM_TIMELINE on the C1 layer).
#pragma unroll 1
                        for (int cc = 0; cc < MY; ++cc) {
                            const int c = hsel * MY + cc;
                            uint32_t av[32], bv[32];
                            tmem_ld32(tbase + c * 32, av);
                            if constexpr (SW) tmem_ld32(tbase + 128 + c * 32, bv);
                            tmem_ld_wait();
                            const bool tlm = warp == 2 && lane == 0 && tile == cid;
                            if (tlm && cc == 1) tl_mark(p, 10);  // c1 in registers
                            if (cc == MY - 1) {  // every column of this warp is in registers
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
                            }
                            const int col0 = nb * ncol + c * 32;
                            if (col0 >= p.N) continue;
                            float h[32];
                            if constexpr (SW) {
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    h[i] = silu(__uint_as_float(av[i])) * __uint_as_float(bv[i]) * wr;
                            } else {
                                act_dispatch(p.act, [&](auto tag) {
#pragma unroll
                                    for (int i = 0; i < 32; ++i)
                                        h[i] = act_t<decltype(tag)::value>(__uint_as_float(av[i])) * wr;
                                });
                            }
                            uint8_t* stg = sC + ((warp - 2) * STG_PER_WARP + stg_n % STG_PER_WARP) * STG_BYTES;
                            if (tlm && cc < 2) tl_mark(p, 8 + 3 * cc);  // c0 / c1 math done (8, 11)
                            if (lane == 0) bulk_wait_read<STG_PER_WARP - 1>();
                            __syncwarp();
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                uint4 o;
                                o.x = pack_bf16(h[8 * u + 0], h[8 * u + 1]);
                                o.y = pack_bf16(h[8 * u + 2], h[8 * u + 3]);
                                o.z = pack_bf16(h[8 * u + 4], h[8 * u + 5]);
                                o.w = pack_bf16(h[8 * u + 6], h[8 * u + 7]);
                                sts128(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4), o);
                            }
                            if (tlm && cc < 2) tl_mark(p, 12 + 2 * cc);  // staged (12, 14)
                            fence_proxy_async();
                            __syncwarp();
                            if (tlm && cc < 2) tl_mark(p, 13 + 2 * cc);  // fenced (13, 15)
                            if (lane == 0) {
                                store_c(&tmC, stg, col0, (int)(row - lane), p.hint);
                                bulk_commit();
                            }
                            if (tlm && cc == 0) tl_mark(p, 9);  // first store issued
                            ++stg_n;
                        }
                        released = true;
                    } else {
                    // all of this warp's accumulator columns to registers first, then
                    // release the TMEM buffer: the MMAs of tile i+2 no longer wait for
                    // this tile's math and stores (short-K GEMMs were epilogue-bound)
                    uint32_t v[MY][32], g[SW ? MY : 1][32];
#pragma unroll
                    for (int cc = 0; cc < MY; ++cc) {
                        const int c = hsel * MY + cc;
                        tmem_ld32(tbase + c * 32, v[cc]);
                        if constexpr (SW) tmem_ld32(tbase + 128 + c * 32, g[cc]);
                    }
                    tmem_ld_wait();
                    if (warp == 2 && lane == 0 && tile == cid) tl_mark(p, 6);  // accumulator in registers
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
                    released = true;
#pragma unroll
                    for (int cc = 0; cc < MY; ++cc) {
                        const int c = hsel * MY + cc;
                        float h[32];
                        const int col0 = nb * ncol + c * 32;
                        if constexpr (SW) {
                            if (p.save_a && col0 < p.N) {  // training: keep a = x w1, b = x w3
                                float fa[32], fb[32];
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    fa[i] = __uint_as_float(v[cc][i]);
                                    fb[i] = __uint_as_float(g[cc][i]);
                                }
                                // coalesced through the warp's staging buffer (free once
                                // the previous TMA store has read it)
                                store_pre_tiled(p.save_a, row - lane, col0, p.N, lane, fa);
                                store_pre_tiled(p.save_b, row - lane, col0, p.N, lane, fb);
                            }
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                h[i] = silu(__uint_as_float(v[cc][i])) * __uint_as_float(g[cc][i]) * wr;
                        } else {
                            if (p.save_a && col0 < p.N) {  // training: keep the pre-activation
                                float fa[32];
#pragma unroll
                                for (int i = 0; i < 32; ++i) fa[i] = __uint_as_float(v[cc][i]);
                                store_pre_tiled(p.save_a, row - lane, col0, p.N, lane, fa);
                            }
                            act_dispatch(p.act, [&](auto tag) {
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    h[i] = act_t<decltype(tag)::value>(__uint_as_float(v[cc][i])) * wr;
                            });
                        }
                        if (col0 < p.N) {
                            if (p.tma_out) {
                                // coalesced: stage the warp's 32 x 32 bf16 block in smem
                                // (64-byte swizzle: 16-byte chunk u of row r at u ^ ((r >> 1) & 3)),
                                // one TMA store per block
                                uint8_t* stg = sC + ((warp - 2) * STG_PER_WARP + stg_n % STG_PER_WARP) * STG_BYTES;
                                if (warp == 2 && lane == 0 && tile == cid) tl_mark(p, 8 + 2 * cc);  // chunk math done
                                if (lane == 0) bulk_wait_read<STG_PER_WARP - 1>();
                                __syncwarp();
                                if (warp == 2 && lane == 0 && tile == cid) tl_mark(p, 9 + 2 * cc);  // staging free
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    uint4 o;
                                    o.x = pack_bf16(h[8 * u + 0], h[8 * u + 1]);
                                    o.y = pack_bf16(h[8 * u + 2], h[8 * u + 3]);
                                    o.z = pack_bf16(h[8 * u + 4], h[8 * u + 5]);
                                    o.w = pack_bf16(h[8 * u + 6], h[8 * u + 7]);
                                    sts128(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4), o);
                                }
                                fence_proxy_async();
                                __syncwarp();
                                if (lane == 0) {
                                    store_c(&tmC, stg, col0, (int)(row - lane), p.hint);
                                    bulk_commit();
                                }
                                if (warp == 2 && lane == 0 && tile == cid && cc == 0) tl_mark(p, 7);  // first store
                                ++stg_n;
                            } else {
                                store_bf16x32(out + col0, h, p.N - col0);
                            }
                        }
                    }
                    }  // !compact
                }
            }
            if (!released) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (warp == 2 && lane == 0) tl_mark(p, 3);  // epilogue issued everything
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (warp == 2 && lane == 0) tl_mark(p, 4);  // stores complete
    }
    tc_fence_before();
    cluster_sync();
    if (threadIdx.x == 0) tl_mark(p, 5);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2<512>(tmem_base);
    }
    if (tq.dyn && rank == 0 && threadIdx.x == 0) sched_done(p.sched, ncl);
}

// ---------------------------------------------------------------------------
// Wide tiles for the long-K forward GEMMs: one CTA pair computes a 256 x 512
// super-tile as two 256 x 256 accumulators sharing each A K-block (both TMEM
// halves, 512 columns).  Per CTA and K block it stages A 16 KB + 2 x B 16 KB =
// 48 KB for two MMAs instead of 2 x 32 KB: 25% less L2 -> SM operand traffic.
// The price is one accumulator buffer (no double buffering): the inference
// epilogue drains it into packed bf16 registers, hands it back, and only then
// stages + TMA-stores (training keeps a two-round drain, with the fp32
// pre-activation stores between the rounds), so the MMAs of the next
// super-tile wait for the TMEM loads alone.  4-stage ring (192 KB).
constexpr int W_STAGES = 4;
// TMEM chunks loaded per tcgen05.wait::ld in the inference drain of the
// non-gated epilogue: 4 (two waits for the 8 chunks) measured best; 1-2 chunks
// per wait expose the TMEM load latency (168-register cap with 10 warps,
// profiles/r01_wide_drain_ab.md)
constexpr int W_LDC = 4;
constexpr int W_B2 = 2 * B_BYTES;  // both B halves of this CTA per stage
constexpr int W_SMEM_BYTES = W_STAGES * (A_BYTES + W_B2) + EPI_STAGE_BYTES + 256;

// Wide tile list: S super-tiles in raster order; when the last wave holds
// r < half the pairs, its r super-tiles are issued as 2r single-block halves
// so the tail wave takes half as long.  Every role decodes the same list.
struct WTile {
    int mb, wi, nb0;  // m-tile, weight index, first 256-row B block
    bool two;         // both accumulators (else only the first, block nb0)
    bool valid;
};
__device__ __forceinline__ WTile wide_decode(int tile, int S, int split, const int* gmb, const int* gw, int ng,
                                             int NBW, int NB, int band) {
    WTile w;
    int nbw, half = 0;
    if (NB & 1) {  // odd block count: every double super-tile first, then the last block of each m-tile
        const int S2 = gmb[ng] * (NB >> 1);
        if (tile < S2) {
            tile_coords(tile, gmb, gw, ng, NB >> 1, band, w.mb, nbw, w.wi);
            w.nb0 = 2 * nbw;
            w.two = true;
        } else {
            tile_coords(tile - S2, gmb, gw, ng, 1, band, w.mb, nbw, w.wi);
            w.nb0 = NB - 1;
            w.two = false;
        }
        w.valid = tile < S;
        return w;
    }
    int st = tile;
    if (tile >= S - split) {
        const int h = tile - (S - split);
        st = S - split + (h >> 1);
        half = h & 1;
    }
    tile_coords(st, gmb, gw, ng, NBW, band, w.mb, nbw, w.wi);
    w.nb0 = 2 * nbw + half;
    w.two = tile < S - split && w.nb0 + 1 < NB;
    w.valid = w.nb0 < NB;
    return w;
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    wide_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, Params p) {
    static_assert(EPI == EPI_ACT_BF16 || EPI == EPI_SWIGLU_BF16, "forward bf16 epilogues only");
    constexpr bool SW = EPI == EPI_SWIGLU_BF16;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + W_STAGES * A_BYTES;
    uint8_t* sC = sB + W_STAGES * W_B2;
    uint64_t* full = reinterpret_cast<uint64_t*>(sC + EPI_STAGE_BYTES);
    uint64_t* empty = full + W_STAGES;
    uint64_t* tfull = empty + W_STAGES;
    uint64_t* tempty = tfull + 1;
    uint64_t* tq_full = tempty + 1;
    uint64_t* tq_empty = tq_full + TQN;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_empty + TQN);
    __shared__ int s_gmb[MAX_GROUPS + 1];
    __shared__ int s_gw[MAX_GROUPS];
    __shared__ int s_tq[TQN];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int NB = SW ? (p.N + 127) / 128 : (p.N + BN - 1) / BN;  // 256-row B blocks
    const int NBW = (NB + 1) / 2;  // super-tiles along N (an odd NB leaves a last single-block super-tile)
    pdl_trigger();
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        if (p.tma_out) tma_prefetch_desc(&tmC);
        for (int s = 0; s < W_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], 2 * EPI_WARPS);
        for (int s = 0; s < TQN; ++s) {
            mbar_init(&tq_full[s], 1);
            mbar_init(&tq_empty[s], TQ_CONSUMERS);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // group tables and operands come from the previous kernels
    for (int i = threadIdx.x; i <= p.ngroups; i += blockDim.x) s_gmb[i] = p.grp_mb[i];
    for (int i = threadIdx.x; i < p.ngroups; i += blockDim.x) s_gw[i] = p.grp_w[i];
    __syncthreads();
    const int KB = (p.K + BK - 1) / BK;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int S = s_gmb[p.ngroups] * NBW;        // super-tiles
    const int tail = S % ncl;
    // tail super-tiles issued as halves (odd block counts end in single-block tiles already)
    const int split = p.tail_split && !(NB & 1) && 2 * tail <= ncl ? tail : 0;
    const int num_tiles = S + split;
    const TileQueue tq{s_tq, tq_full, tq_empty, cid, ncl, p.sched != nullptr};

    if (warp == 0) {
        if (lane == 0) {  // -------------------------------------------- TMA producer
            const uint64_t pol_b = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            int next = cid;  // scheduler: the tile index taken for this pair's next tile
            for (int i = 0;; ++i) {
                int tile;
                if (tq.dyn && rank == 0) {
                    tile = next;
                    tq.publish(i, tile);
                    if (tile < num_tiles) next = ncl + atomicAdd(p.sched, 1);  // used next iteration
                } else {
                    tile = tq.get(i);
                    tq.release(i, rank);
                }
                if (tile >= num_tiles) break;
                const WTile wt = wide_decode(tile, S, split, s_gmb, s_gw, p.ngroups, NBW, NB, p.band);
                if (!wt.valid) continue;
                const int ay = wt.mb * 2 * BM + rank * BM;
                const int by0 = wt.wi * p.b_rows_per_e + wt.nb0 * BN + rank * (BN / 2);
                const bool two = wt.two;  // the second 256-row B block is part of this tile
                for (int kb = 0; kb < KB; ++kb) {
                    { const long long t0 = p.dbg ? clock64() : 0;
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (p.dbg) p.dbg[blockIdx.x * 4 + 0] += clock64() - t0; }
                    const uint32_t lbar = smem_u32(&full[stage]) & kPeerBitMask;
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + (two ? W_B2 : B_BYTES)));
                    uint8_t* b_dst = sB + stage * W_B2;
                    if (p.hint & 4) tma_load_2d_cg2_hint(sA + stage * A_BYTES, &tmA, lbar, kb * BK, ay, pol_a);
                    else tma_load_2d_cg2(sA + stage * A_BYTES, &tmA, lbar, kb * BK, ay);
                    if (p.hint & 1) {
                        tma_load_2d_cg2_hint(b_dst, &tmB, lbar, kb * BK, by0, pol_b);
                        if (two) tma_load_2d_cg2_hint(b_dst + B_BYTES, &tmB, lbar, kb * BK, by0 + BN, pol_b);
                    } else {
                        tma_load_2d_cg2(b_dst, &tmB, lbar, kb * BK, by0);
                        if (two) tma_load_2d_cg2(b_dst + B_BYTES, &tmB, lbar, kb * BK, by0 + BN);
                    }
                    if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // --------------------------------- MMA issuer (leader CTA)
            constexpr uint32_t IDESC = idesc_bf16_f32(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int i = 0;; ++i) {
                const int tile = tq.get(i);
                __syncwarp();
                if (lane == 0) tq.release(i, rank);
                if (tile >= num_tiles) break;
                const WTile wt = wide_decode(tile, S, split, s_gmb, s_gw, p.ngroups, NBW, NB, p.band);
                if (!wt.valid) continue;
                const bool two = wt.two;
                { const long long t0 = p.dbg ? clock64() : 0;
                mbar_wait(&tempty[0], acc_phase ^ 1);
                if (p.dbg && lane == 0) p.dbg[blockIdx.x * 4 + 1] += clock64() - t0; }
                tc_fence_after();
                for (int kb = 0; kb < KB; ++kb) {
                    { const long long t0 = p.dbg ? clock64() : 0;
                    mbar_wait(&full[stage], phase);
                    if (p.dbg && lane == 0) p.dbg[blockIdx.x * 4 + 2] += clock64() - t0; }
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * W_B2);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t ad = sdesc_k_sw128(a0 + k * 32);
                            umma_bf16_cg2(tmem_base, ad, sdesc_k_sw128(b0 + k * 32), IDESC, (kb | k) != 0);
                            if (two)
                                umma_bf16_cg2(tmem_base + BN, ad, sdesc_k_sw128(b0 + B_BYTES + k * 32), IDESC,
                                              (kb | k) != 0);
                        }
                        umma_commit_cg2_mc(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
                }
                if (lane == 0) umma_commit_cg2_mc(&tfull[0]);
                __syncwarp();
                acc_phase ^= 1;
            }
        }
    } else {  // ------------------------------------------------------------ epilogue
        const int q = warp & 3;            // TMEM lane quarter
        const int t = (warp - 2) >> 2;     // which accumulator (256-column half of the super-tile)
        uint8_t* stg = sC + (warp - 2) * STG_PER_WARP * STG_BYTES;
        uint32_t acc_phase = 0;
        constexpr int NCH = SW ? 4 : BN / 32;  // output chunks of 32 columns per accumulator
        constexpr int HALF = NCH / 2;          // chunks per drain round (128 registers)
        for (int i = 0;; ++i) {
            const int tile = tq.get(i);
            __syncwarp();
            if (lane == 0) tq.release(i, rank);
            if (tile >= num_tiles) break;
            const WTile wt = wide_decode(tile, S, split, s_gmb, s_gw, p.ngroups, NBW, NB, p.band);
            if (!wt.valid) continue;
            const int mb = wt.mb;
            { const long long t0 = p.dbg ? clock64() : 0;
            mbar_wait(&tfull[0], acc_phase);
            if (p.dbg && lane == 0 && warp == 2) p.dbg[blockIdx.x * 4 + 3] += clock64() - t0; }
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + t * BN;
            const long row = (long)mb * 2 * BM + rank * BM + q * 32 + lane;
            const float wr = p.row_w ? p.row_w[row] : 1.0f;
            const int nb = wt.nb0 + t;
            const int ncol = SW ? 128 : BN;
            if (t == 1 && !wt.two) {  // single-block tile: the second accumulator holds nothing
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[0]) & kPeerBitMask);
                acc_phase ^= 1;
                continue;
            }
            if (p.tma_out && !p.save_a) {
                // Inference: drain the whole accumulator into packed bf16 registers
                // (two TMEM loads in flight per wait), hand TMEM back, and only then
                // stage + TMA-store, so the stores overlap the next super-tile's MMAs
                // instead of holding its accumulator.
                uint32_t pk[NCH][16];
                if constexpr (SW) {
#pragma unroll
                    for (int c = 0; c < NCH; ++c) {
                        uint32_t v[32], g[32];
                        tmem_ld32(tbase + c * 32, v);
                        tmem_ld32(tbase + 128 + c * 32, g);
                        tmem_ld_wait();
                        if (c == NCH - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[0]) & kPeerBitMask);
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            pk[c][i] = pack_bf16(silu(__uint_as_float(v[2 * i])) * __uint_as_float(g[2 * i]) * wr,
                                                 silu(__uint_as_float(v[2 * i + 1])) * __uint_as_float(g[2 * i + 1]) * wr);
                    }
                } else {
                    act_dispatch(p.act, [&](auto tag) {
                        constexpr int A = decltype(tag)::value;
#pragma unroll
                        for (int c = 0; c < NCH; c += W_LDC) {
                            uint32_t v[W_LDC][32];
#pragma unroll
                            for (int cc = 0; cc < W_LDC; ++cc) tmem_ld32(tbase + (c + cc) * 32, v[cc]);
                            tmem_ld_wait();
                            if (c == NCH - W_LDC) {
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[0]) & kPeerBitMask);
                            }
#pragma unroll
                            for (int cc = 0; cc < W_LDC; ++cc)
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    pk[c + cc][i] = pack_bf16(act_t<A>(__uint_as_float(v[cc][2 * i])) * wr,
                                                              act_t<A>(__uint_as_float(v[cc][2 * i + 1])) * wr);
                        }
                    });
                }
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const int col0 = nb * ncol + c * 32;
                    if (col0 >= p.N) break;
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        sts128(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4),
                               make_uint4(pk[c][4 * u], pk[c][4 * u + 1], pk[c][4 * u + 2], pk[c][4 * u + 3]));
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        store_c(&tmC, stg, col0, (int)(row - lane), p.hint);
                        bulk_commit();
                    }
                }
                acc_phase ^= 1;
                continue;
            }
#pragma unroll 1
            for (int round = 0; round < 2; ++round) {
                uint32_t v[HALF][32], g[SW ? HALF : 1][32];
#pragma unroll
                for (int cc = 0; cc < HALF; ++cc) {
                    const int c = round * HALF + cc;
                    tmem_ld32(tbase + c * 32, v[cc]);
                    if constexpr (SW) tmem_ld32(tbase + 128 + c * 32, g[cc]);
                }
                tmem_ld_wait();
                if (round == 1) {  // every column is in registers: hand the accumulator back
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[0]) & kPeerBitMask);
                }
#pragma unroll
                for (int cc = 0; cc < HALF; ++cc) {
                    const int col0 = nb * ncol + (round * HALF + cc) * 32;
                    if (p.save_a && col0 < p.N) {  // training: keep a = x w1 (and b = x w3), tiled
                        float fa[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) fa[i] = __uint_as_float(v[cc][i]);
                        store_pre_tiled(p.save_a, row - lane, col0, p.N, lane, fa);
                        if constexpr (SW) {
#pragma unroll
                            for (int i = 0; i < 32; ++i) fa[i] = __uint_as_float(g[cc][i]);
                            store_pre_tiled(p.save_b, row - lane, col0, p.N, lane, fa);
                        }
                    }
                    float h[32];
                    if constexpr (SW) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) h[i] = silu(__uint_as_float(v[cc][i])) * __uint_as_float(g[cc][i]) * wr;
                    } else {
                        act_dispatch(p.act, [&](auto tag) {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                h[i] = act_t<decltype(tag)::value>(__uint_as_float(v[cc][i])) * wr;
                        });
                    }
                    if (col0 >= p.N) continue;
                    if (p.tma_out) {
                        if (lane == 0) bulk_wait_read<0>();
                        __syncwarp();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            uint4 o;
                            o.x = pack_bf16(h[8 * u + 0], h[8 * u + 1]);
                            o.y = pack_bf16(h[8 * u + 2], h[8 * u + 3]);
                            o.z = pack_bf16(h[8 * u + 4], h[8 * u + 5]);
                            o.w = pack_bf16(h[8 * u + 6], h[8 * u + 7]);
                            sts128(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4), o);
                        }
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) {
                            store_c(&tmC, stg, col0, (int)(row - lane), p.hint);
                            bulk_commit();
                        }
                    } else {
                        store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo + col0, h, p.N - col0);
                    }
                }
            }
            acc_phase ^= 1;
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2<512>(tmem_base);
    }
    if (tq.dyn && rank == 0 && threadIdx.x == 0) sched_done(p.sched, ncl);
}

// Weight-gradient GEMMs with the same 256 x 512 super-tiles: per expert
// group, dW[e] (M x N) = sum over the group's rows (K) of A^T B, both
// operands read MN-major straight from the row-major activations; two
// 256-column accumulators share every A K-block.  fp32 outputs (split into
// out / out2 at `split` for the SwiGLU w1 | w3 gradient).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    wide_wgrad_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + W_STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + W_STAGES * W_B2);
    uint64_t* empty = full + W_STAGES;
    uint64_t* tfull = empty + W_STAGES;
    uint64_t* tempty = tfull + 1;
    uint64_t* tq_full = tempty + 1;
    uint64_t* tq_empty = tq_full + TQN;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_empty + TQN);
    __shared__ int s_tb[MAX_GROUPS + 1];  // super-tile prefix per group
    __shared__ int s_gw[MAX_GROUPS];
    __shared__ int s_kb0[MAX_GROUPS];
    __shared__ int s_kbn[MAX_GROUPS];
    __shared__ int s_tq[TQN];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int NBW = (p.N + 2 * BN - 1) / (2 * BN);
    const int MT = (p.M + 2 * BM - 1) / (2 * BM);
    pdl_trigger();
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int st = 0; st < W_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 1);
        }
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], 2 * EPI_WARPS);
        for (int s = 0; s < TQN; ++s) {
            mbar_init(&tq_full[s], 1);
            mbar_init(&tq_empty[s], TQ_CONSUMERS);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // group tables and operands come from the previous kernels
    if (threadIdx.x == 0) {
        int run = 0;
        for (int g = 0; g < p.ngroups; ++g) {
            s_tb[g] = run;
            const int rows = p.grp_cnt[g];
            s_kb0[g] = p.seg_base[g] / BK;
            s_kbn[g] = (rows + BK - 1) / BK;
            if (rows > 0) run += MT * NBW;
        }
        s_tb[p.ngroups] = run;
    }
    for (int i = threadIdx.x; i < p.ngroups; i += blockDim.x) s_gw[i] = p.grp_w[i];
    __syncthreads();
    const int num_tiles = s_tb[p.ngroups];
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const TileQueue tq{s_tq, tq_full, tq_empty, cid, ncl, p.sched != nullptr};

    if (warp == 0) {
        if (lane == 0) {  // -------------------------------------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            int next = cid;
            for (int i = 0;; ++i) {
                int tile;
                if (tq.dyn && rank == 0) {
                    tile = next;
                    tq.publish(i, tile);
                    if (tile < num_tiles) next = ncl + atomicAdd(p.sched, 1);
                } else {
                    tile = tq.get(i);
                    tq.release(i, rank);
                }
                if (tile >= num_tiles) break;
                int g, mt, ntw;
                wtile_coords(tile, s_tb, p.ngroups, NBW, g, mt, ntw);
                const int ax = mt * 2 * BM + rank * BM;
                const int bx = 2 * ntw * BN + rank * (BN / 2);
                for (int kb = 0; kb < s_kbn[g]; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t lbar = smem_u32(&full[stage]) & kPeerBitMask;
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + W_B2));
                    const int k = (s_kb0[g] + kb) * BK;  // token rows of this K block
                    uint8_t* a_dst = sA + stage * A_BYTES;
                    uint8_t* b_dst = sB + stage * W_B2;
                    tma_load_2d_cg2(a_dst, &tmA, lbar, ax, k);
                    tma_load_2d_cg2(a_dst + A_BYTES / 2, &tmA, lbar, ax + 64, k);
                    tma_load_2d_cg2(b_dst, &tmB, lbar, bx, k);
                    tma_load_2d_cg2(b_dst + B_BYTES / 2, &tmB, lbar, bx + 64, k);
                    tma_load_2d_cg2(b_dst + B_BYTES, &tmB, lbar, bx + BN, k);
                    tma_load_2d_cg2(b_dst + B_BYTES + B_BYTES / 2, &tmB, lbar, bx + BN + 64, k);
                    if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // --------------------------------- MMA issuer (leader CTA)
            constexpr uint32_t IDESC = idesc_mn(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int i = 0;; ++i) {
                const int tile = tq.get(i);
                __syncwarp();
                if (lane == 0) tq.release(i, rank);
                if (tile >= num_tiles) break;
                int g, mt, ntw;
                wtile_coords(tile, s_tb, p.ngroups, NBW, g, mt, ntw);
                mbar_wait(&tempty[0], acc_phase ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < s_kbn[g]; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * W_B2);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t ad = sdesc_mn_sw128(a0 + k * 2048);
                            umma_bf16_cg2(tmem_base, ad, sdesc_mn_sw128(b0 + k * 2048), IDESC, (kb | k) != 0);
                            umma_bf16_cg2(tmem_base + BN, ad, sdesc_mn_sw128(b0 + B_BYTES + k * 2048), IDESC,
                                          (kb | k) != 0);
                        }
                        umma_commit_cg2_mc(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
                }
                if (lane == 0) umma_commit_cg2_mc(&tfull[0]);
                __syncwarp();
                acc_phase ^= 1;
            }
        }
    } else {  // ------------------------------------------------------------ epilogue
        const int q = warp & 3, t = (warp - 2) >> 2;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int tile = tq.get(i);
            __syncwarp();
            if (lane == 0) tq.release(i, rank);
            if (tile >= num_tiles) break;
            int g, mt, ntw;
            wtile_coords(tile, s_tb, p.ngroups, NBW, g, mt, ntw);
            mbar_wait(&tfull[0], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + t * BN;
            const int m = mt * 2 * BM + rank * BM + q * 32 + lane;
            const long ebase = (long)s_gw[g] * p.out_estride;
#pragma unroll 1
            for (int round = 0; round < 2; ++round) {
                uint32_t v[4][32];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) tmem_ld32(tbase + (round * 4 + cc) * 32, v[cc]);
                tmem_ld_wait();
                if (round == 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[0]) & kPeerBitMask);
                }
                if (m >= p.M) continue;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int col0 = (2 * ntw + t) * BN + (round * 4 + cc) * 32;
                    if (col0 >= p.N) continue;
                    float* o = reinterpret_cast<float*>(p.out) + ebase + (long)m * p.ldo;
                    int c0 = col0;
                    if (p.out2 && col0 >= p.split) {
                        o = reinterpret_cast<float*>(p.out2) + ebase + (long)m * p.ldo;
                        c0 = col0 - p.split;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (col0 + u * 4 < p.N)
                            *reinterpret_cast<float4*>(o + c0 + u * 4) =
                                make_float4(__uint_as_float(v[cc][4 * u]), __uint_as_float(v[cc][4 * u + 1]),
                                            __uint_as_float(v[cc][4 * u + 2]), __uint_as_float(v[cc][4 * u + 3]));
                }
            }
            acc_phase ^= 1;
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2<512>(tmem_base);
    }
    if (tq.dyn && rank == 0 && threadIdx.x == 0) sched_done(p.sched, ncl);
}

template <int EPI>
void launch_wide(int grid, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const Params& p,
                 cudaStream_t st) {
    const int smem = W_SMEM_BYTES + 1024;
    cudaFuncSetAttribute(wide_gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_pdl(wide_gemm_kernel<EPI>, grid, THREADS, smem, st, ta, tb, tc, p);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

template <int EPI, bool WGRAD>
void launch_one(int grid, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const Params& p,
                cudaStream_t st) {
    const int smem = SMEM_BYTES + 1024;
    cudaFuncSetAttribute(grouped_gemm_kernel<EPI, WGRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_pdl(grouped_gemm_kernel<EPI, WGRAD>, grid, THREADS, smem, st, ta, tb, tc, p);
}

}  // namespace

// Row-major bf16 matrix [outer, inner], 128-byte swizzled boxes of
// box_inner (=64) x box_outer elements.  OOB reads are zero-filled.
bool make_tmap_2d(void* tmap, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                  uint32_t box_outer, int swizzle_bytes, uint64_t pitch_elems) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {(pitch_elems ? pitch_elems : inner) * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    static const int promo_env = [] {  // L2 promotion experiments (profiles/), not a product knob
        const char* e = getenv("OCC_TMAP_PROMO");
        return e ? atoi(e) : 3;
    }();
    static const CUtensorMapL2promotion promos[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    return enc(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
               promos[promo_env & 3], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_grouped_gemm(EpiMode mode, const GemmArgs& a, int num_sms, cudaStream_t st) {
    Params p{};
    p.K = a.K;
    p.N = a.N;
    p.b_rows_per_e = a.b_rows_per_e;
    p.act = a.act;
    p.grp_mb = a.grp_mb;
    p.grp_w = a.grp_w;
    p.ngroups = a.ngroups;
    p.band = a.band;
    p.grp_cnt = a.grp_cnt;
    p.seg_base = a.seg_base;
    p.M = a.M;
    p.row_w = a.row_w;
    p.out = a.out;
    p.ldo = a.ldo;
    p.out_estride = a.out_estride;
    p.out2 = a.out2;
    p.split = a.split;
    p.save_a = a.save_a;
    p.save_b = a.save_b;
    p.pre_a = a.pre_a;
    p.pre_b = a.pre_b;
    p.gw_part = a.gw_part;
    p.a_rows = a.a_rows;
    static const bool tl_on = getenv("OCC_GEMM_TIMELINE") != nullptr;
    static unsigned long long* tl_buf = nullptr;
    if (tl_on) {
        if (!tl_buf) cudaMalloc(&tl_buf, sizeof(unsigned long long) * 16 * 1024);
        cudaMemsetAsync(tl_buf, 0, sizeof(unsigned long long) * 16 * 1024, st);
        p.tl = tl_buf;
    }
    static const bool dbg_on = getenv("OCC_GEMM_DEBUG") != nullptr;
    static unsigned long long* dbg_buf = nullptr;
    static cudaEvent_t dbg_ev[2];
    if (dbg_on) {
        if (!dbg_buf) {
            cudaMalloc(&dbg_buf, sizeof(unsigned long long) * 4 * 1024);
            cudaEventCreate(&dbg_ev[0]);
            cudaEventCreate(&dbg_ev[1]);
        }
        cudaMemsetAsync(dbg_buf, 0, sizeof(unsigned long long) * 4 * 1024, st);
        p.dbg = dbg_buf;
        cudaEventRecord(dbg_ev[0], st);
    }
    const CUtensorMap& ta = *reinterpret_cast<const CUtensorMap*>(a.tmap_a);
    const CUtensorMap& tb = *reinterpret_cast<const CUtensorMap*>(a.tmap_b);
    static const int tma_store_env = getenv("OCC_GEMM_TMASTORE") ? atoi(getenv("OCC_GEMM_TMASTORE")) : 1;
    p.tma_out = tma_store_env && a.tmap_c != nullptr &&
                (mode == EPI_ACT_BF16 || mode == EPI_SWIGLU_BF16 || mode == EPI_BWD_ACT || mode == EPI_BWD_SWIGLU);
    const CUtensorMap& tc = p.tma_out ? *reinterpret_cast<const CUtensorMap*>(a.tmap_c) : ta;
    static const int band_override = [] {  // raster experiments (profiles/), not a product knob
        const char* e = getenv("OCC_GEMM_BAND");
        return e ? atoi(e) : 0;
    }();
    static const int band1_override = [] {
        const char* e = getenv("OCC_GEMM_BAND_G1");
        return e ? atoi(e) : 0;
    }();
    if (mode == EPI_SWIGLU_BF16 && band1_override > 0) p.band = band1_override;
    else if (band_override > 0 && !(mode == EPI_WGRAD)) p.band = band_override;
    int grid = 2 * a.max_tiles < num_sms ? 2 * a.max_tiles : num_sms;
    grid &= ~1;  // CTA pairs
    if (grid <= 0) return;
    // wide 256 x 512 super-tiles for long-K forward GEMMs (OCC_GEMM_WIDE: 0 off,
    // 1 auto = K >= 1024 and an even number of 256-row B blocks, 2 force, odd counts >= 5 too)
    static const int wide_env = getenv("OCC_GEMM_WIDE") ? atoi(getenv("OCC_GEMM_WIDE")) : 1;
    static const int tail_env = getenv("OCC_GEMM_TAILSPLIT") ? atoi(getenv("OCC_GEMM_TAILSPLIT")) : 1;
    p.tail_split = tail_env;
    static const int hint_env = getenv("OCC_GEMM_HINT") ? atoi(getenv("OCC_GEMM_HINT")) : 0;
    p.hint = hint_env;
    static const int dyn_env = getenv("OCC_GEMM_DYN") ? atoi(getenv("OCC_GEMM_DYN")) : 1;
    p.sched = dyn_env ? a.sched : nullptr;
    bool wide = false;
    if ((mode == EPI_ACT_BF16 || mode == EPI_SWIGLU_BF16) && !a.a_rows) {
        const int nbk = mode == EPI_SWIGLU_BF16 ? (a.N + 127) / 128 : (a.N + BN - 1) / BN;
        // an odd block count ends in a single-block super-tile; worth it from 5 blocks up
        // an odd block count ends in a single-block super-tile: supported (forced mode) but
        // measured 3% slower than the narrow kernel on DeepSeek's 11 blocks, so auto needs even
        const bool ok = (nbk % 2 == 0 || (nbk >= 5 && wide_env == 2)) && (mode != EPI_SWIGLU_BF16 || a.N % 128 == 0);
        // (auto also needs at least one full wave of narrow tiles: with fewer,
        // halving the tile count only lengthens each pair's serial K loop --
        // small batches, C1 GEMM-2 31 -> 20 us with narrow tiles)
        if (ok && (wide_env == 2 || (wide_env == 1 && a.K >= 1024 && a.max_tiles >= num_sms))) {
            if (mode == EPI_ACT_BF16) launch_wide<EPI_ACT_BF16>(grid, ta, tb, tc, p, st);
            else launch_wide<EPI_SWIGLU_BF16>(grid, ta, tb, tc, p, st);
            wide = true;
        }
    }
    if (!wide) switch (mode) {
        case EPI_ACT_BF16: launch_one<EPI_ACT_BF16, false>(grid, ta, tb, tc, p, st); break;
        case EPI_SWIGLU_BF16: launch_one<EPI_SWIGLU_BF16, false>(grid, ta, tb, tc, p, st); break;
        case EPI_F32: launch_one<EPI_F32, false>(grid, ta, tb, tc, p, st); break;
        case EPI_BWD_ACT: launch_one<EPI_BWD_ACT, false>(grid, ta, tb, tc, p, st); break;
        case EPI_BWD_SWIGLU: launch_one<EPI_BWD_SWIGLU, false>(grid, ta, tb, tc, p, st); break;
        case EPI_WGRAD: {
            // wide super-tiles when the output columns split into pairs of 256-column blocks
            if (wide_env != 0 && ((a.N + BN - 1) / BN) % 2 == 0) {
                const int smem = W_STAGES * (A_BYTES + W_B2) + 256 + 1024;
                cudaFuncSetAttribute(wide_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                launch_pdl(wide_wgrad_kernel, grid, THREADS, smem, st, ta, tb, p);
            } else {
                launch_one<EPI_F32, true>(grid, ta, tb, tc, p, st);
            }
            break;
        }
    }
    if (tl_on) {  // per-CTA timeline (narrow kernel; diagnostics only)
        static unsigned long long h[16 * 1024];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, tl_buf, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < grid; ++c)
            if (h[c * 16] && h[c * 16] < t0) t0 = h[c * 16];
        // (compact epilogue marks: 8 c0 math, 12 c0 staged, 13 c0 fenced, 9 c0 stored, 10 c1 loaded,
        //  11 c1 math, 14 c1 staged, 15 c1 fenced; unrolled epilogue: 6 in-regs, 7 first store)
        static const char* names[16] = {"start", "setup", "acc-ready", "epi-issued", "stores-done", "exit", "in-regs",
                                        "first-store", "c0-math", "c0-stored", "c1-loaded", "c1-math", "c0-staged",
                                        "c0-fenced", "c1-staged", "c1-fenced"};
        fprintf(stderr, "[gemm tl] mode=%d K=%d N=%d grid=%d us from first CTA start (min/median/max over CTAs):", (int)mode,
                a.K, a.N, grid);
        static const int order[16] = {0, 1, 2, 6, 7, 8, 12, 13, 9, 10, 11, 14, 15, 3, 4, 5};
        for (int oi = 0; oi < 16; ++oi) {
            const int i = order[oi];
            double v[1024];
            int nv = 0;
            for (int c = 0; c < grid; ++c)
                if (h[c * 16 + i]) v[nv++] = (h[c * 16 + i] - t0) / 1e3;
            if (!nv) continue;
            std::sort(v, v + nv);
            fprintf(stderr, " %s %.1f/%.1f/%.1f", names[i], v[0], v[nv / 2], v[nv - 1]);
        }
        fprintf(stderr, "\n");
    }
    if (dbg_on) {  // stall-cycle breakdown, averaged over CTAs (diagnostics only)
        unsigned long long h[4 * 1024];
        cudaEventRecord(dbg_ev[1], st);
        cudaStreamSynchronize(st);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, dbg_ev[0], dbg_ev[1]);
        cudaMemcpy(h, dbg_buf, sizeof(unsigned long long) * 4 * grid, cudaMemcpyDeviceToHost);
        double sum[4] = {0, 0, 0, 0};
        int nl = 0;
        for (int c = 0; c < grid; ++c) {
            for (int i = 0; i < 4; ++i) sum[i] += (double)h[c * 4 + i];
            nl += (c % 2 == 0);
        }
        fprintf(stderr, "[gemm dbg] %s mode=%d K=%d N=%d: producer-empty %.0f, mma-tempty %.0f, mma-full %.0f, epi-tfull %.0f (kcycles/CTA), %.3f ms\n",
                wide ? "wide" : "narrow", (int)mode, a.K, a.N, sum[0] / grid / 1e3, sum[1] / nl / 1e3, sum[2] / nl / 1e3, sum[3] / grid / 1e3, ms);
    }
    count_launch();
}

}  // namespace occ
