// occ_gemm.cu — grouped per-expert GEMM on 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM, operands staged by TMA).
//
// Replaces the reference's two indexed matmul loops, scatter_matmul
// (pipeline.cpp:178-211, Alg. 6; fused here with apply_activation
// :213-224 and weight_modulate :226-248, Alg. 7) and merge_matmul
// (pipeline.cpp:250-283, Alg. 8).  Rows of every expert are contiguous and
// padded to the 128-row M tile (compute-index segments, see
// compute_finalize_kernel), so each tile belongs to exactly one expert and
// the B operand is that expert's resident K-major weight slice.
//
// Persistent, warp-specialised, CTA pairs (cluster 2x1x1, cta_group::2):
// one 256x256 output tile per pair and K-step, each CTA staging its 128 A
// rows and its half (128 rows) of the B tile, so per-SM operand traffic is
// 32 KB per 64-deep K block (6 stages in 192 KB of shared memory).
//   warp 0      TMA producer in both CTAs (completion on the leader's barrier)
//   warp 1      TMEM allocator (both CTAs) + single-thread tcgen05.mma issuer
//               in the leader CTA (M=256, N=256, K=16, fp32 accumulate)
//   warps 2..5  epilogue in both CTAs: tcgen05.ld -> activation / SwiGLU /
//               routing weight -> global stores; double-buffered TMEM
//               accumulators (2 x 256 columns) overlap the next tile.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "occ_common.cuh"
#include "occ_internal.h"

namespace occ {
namespace {

constexpr int BM = 128;               // rows per CTA (pair tile: 256)
constexpr int BN = 256, BK = 64, STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = (BN / 2) * BK * 2;  // 16 KB: this CTA's half of the B tile
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 256;
constexpr int THREADS = 192;
constexpr int MAX_GROUPS = 256;
constexpr uint32_t IDESC = idesc_bf16_f32(2 * BM, BN);
static_assert(kBM == 2 * BM, "Epd segments are padded to the pair tile");

struct Params {
    int K, N, b_rows_per_e, act;
    const int* grp_mb;
    const int* grp_w;
    int ngroups, band;
    const float* row_w;
    void* out;
    int ldo;
};

// Tile -> (m-block, n-block, weight slice).  Tiles are enumerated expert
// group by expert group, and inside a group in bands of `band` m-blocks
// walked n-block-major, so concurrently resident CTAs share B (weight)
// n-blocks and a band's A rows stay in L2; no band straddles two experts.
__device__ __forceinline__ void tile_coords(int tile, const int* gmb, const int* gw, int ng, int NB, int band,
                                            int& mb, int& nb, int& w) {
    int g = 0;
    while (g < ng - 1 && gmb[g + 1] * NB <= tile) ++g;
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

__device__ __forceinline__ float act_f(float v, int act) {
    if (act == 1) return silu(v);
    if (act == 2) return v > 0.f ? v : 0.f;
    return v;
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    __shared__ int s_gmb[MAX_GROUPS + 1];
    __shared__ int s_gw[MAX_GROUPS];
    for (int i = threadIdx.x; i <= p.ngroups; i += blockDim.x) s_gmb[i] = p.grp_mb[i];
    for (int i = threadIdx.x; i < p.ngroups; i += blockDim.x) s_gw[i] = p.grp_w[i];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);   // leader: one expect_tx arrival + both CTAs' bytes
            mbar_init(&empty[s], 1);  // one multicast commit per phase
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);  // leader: 4 epilogue warps x 2 CTAs
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int MB = s_gmb[p.ngroups];  // pair tiles of 256 rows
    const int NB = EPI == EPI_SWIGLU_BF16 ? (p.N + 127) / 128 : (p.N + BN - 1) / BN;
    const int num_tiles = MB * NB;
    const int KB = (p.K + BK - 1) / BK;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = cid; tile < num_tiles; tile += ncl) {
                int mb, nb, wi;
                tile_coords(tile, s_gmb, s_gw, p.ngroups, NB, p.band, mb, nb, wi);
                const int arow = mb * 2 * BM + rank * BM;
                const int brow = wi * p.b_rows_per_e + nb * BN + rank * (BN / 2);
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t lbar = smem_u32(&full[stage]) & kPeerBitMask;
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
                    tma_load_2d_cg2(sA + stage * A_BYTES, &tmA, lbar, kb * BK, arow);
                    tma_load_2d_cg2(sB + stage * B_BYTES, &tmB, lbar, kb * BK, brow);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = cid; tile < num_tiles; tile += ncl) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_bf16_cg2(d_tmem, sdesc_k_sw128(a0 + k * 32), sdesc_k_sw128(b0 + k * 32), IDESC,
                                          (kb | k) != 0);
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
        const int q = warp & 3;  // TMEM lane quarter accessible to this warp
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = cid; tile < num_tiles; tile += ncl) {
            int mb, nb, wi;
            tile_coords(tile, s_gmb, s_gw, p.ngroups, NB, p.band, mb, nb, wi);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const long row = (long)mb * 2 * BM + rank * BM + q * 32 + lane;
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            if constexpr (EPI == EPI_F32) {
                float* out = reinterpret_cast<float*>(p.out) + row * p.ldo;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
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
            } else {
                const float wr = p.row_w ? p.row_w[row] : 1.0f;
                __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo;
                constexpr int NCH = EPI == EPI_SWIGLU_BF16 ? 4 : BN / 32;
                const int ncol = EPI == EPI_SWIGLU_BF16 ? 128 : BN;
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) {
                    uint32_t v[32];
                    float h[32];
                    tmem_ld32(tbase + c * 32, v);
                    if constexpr (EPI == EPI_SWIGLU_BF16) {
                        uint32_t g[32];
                        tmem_ld32(tbase + 128 + c * 32, g);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            h[i] = silu(__uint_as_float(v[i])) * __uint_as_float(g[i]) * wr;
                    } else {
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) h[i] = act_f(__uint_as_float(v[i]), p.act) * wr;
                    }
                    const int col0 = nb * ncol + c * 32;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (col0 + u * 8 < p.N) {
                            uint4 o;
                            o.x = pack_bf16(h[8 * u + 0], h[8 * u + 1]);
                            o.y = pack_bf16(h[8 * u + 2], h[8 * u + 3]);
                            o.z = pack_bf16(h[8 * u + 4], h[8 * u + 5]);
                            o.w = pack_bf16(h[8 * u + 6], h[8 * u + 7]);
                            *reinterpret_cast<uint4*>(out + col0 + u * 8) = o;
                        }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2<512>(tmem_base);
    }
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

}  // namespace

// Row-major bf16 matrix [outer, inner], 128-byte swizzled boxes of
// box_inner (=64) x box_outer elements.  OOB reads are zero-filled.
bool make_tmap_2d(void* tmap, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                  uint32_t box_outer) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_grouped_gemm(EpiMode mode, const GemmArgs& a, int num_sms, cudaStream_t st) {
    Params p{a.K, a.N, a.b_rows_per_e, a.act, a.grp_mb, a.grp_w, a.ngroups, a.band, a.row_w, a.out, a.ldo};
    const CUtensorMap& ta = *reinterpret_cast<const CUtensorMap*>(a.tmap_a);
    const CUtensorMap& tb = *reinterpret_cast<const CUtensorMap*>(a.tmap_b);
    int grid = 2 * a.max_tiles < num_sms ? 2 * a.max_tiles : num_sms;
    grid &= ~1;  // CTA pairs
    if (grid <= 0) return;
    const int smem = SMEM_BYTES + 1024;
    switch (mode) {
        case EPI_ACT_BF16:
            cudaFuncSetAttribute(grouped_gemm_kernel<EPI_ACT_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            grouped_gemm_kernel<EPI_ACT_BF16><<<grid, THREADS, smem, st>>>(ta, tb, p);
            break;
        case EPI_SWIGLU_BF16:
            cudaFuncSetAttribute(grouped_gemm_kernel<EPI_SWIGLU_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem);
            grouped_gemm_kernel<EPI_SWIGLU_BF16><<<grid, THREADS, smem, st>>>(ta, tb, p);
            break;
        case EPI_F32:
            cudaFuncSetAttribute(grouped_gemm_kernel<EPI_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            grouped_gemm_kernel<EPI_F32><<<grid, THREADS, smem, st>>>(ta, tb, p);
            break;
    }
    count_launch();
}

}  // namespace occ
