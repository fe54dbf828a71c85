// occ_router.cu — the routing stage on tensor cores.
//
// gate_scores (routing.cpp:33-52) + topk_route (routing.cpp:60-84) +
// renormalize_row (:54-58) in one persistent kernel: logits = x g^T is a
// [128 tokens x E] tcgen05 tile (bf16 in, fp32 accumulate in TMEM, K = D
// streamed by TMA), and the epilogue thread that owns a token row runs the
// softmax (max-subtracted) and the (score desc, index asc) top-k selection
// straight out of TMEM, then renormalises.  HBM-bound on reading x once.
// With pruning, or when the caller wants the score rows, the epilogue
// writes the logits and the per-token selection runs in router_select.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "occ_common.cuh"
#include "occ_internal.h"

namespace occ {
namespace {

constexpr int RM = 128, RK = 64, RTHREADS = 192;
// deeper TMA ring for narrow gates (more bytes of x in flight per SM)
template <int NPMAX>
constexpr int rstages() { return NPMAX <= 64 ? 8 : (NPMAX <= 128 ? 6 : 4); }
constexpr int R_A_BYTES = RM * RK * 2;  // 16 KB

struct RouterParams {
    int n, d, e, np, k, renorm;
    int32_t* ids;
    float* w;
    float* logits_out;  // non-null: write logits [n, e], skip the selection
    // collaboration pruning in the epilogue (router-score mode, pruning.cpp:35-64)
    int prune, budget, prune_renorm;
    const int32_t* dev_of;  // [e]
    int32_t* err;
};

template <int NPMAX>
__global__ void __launch_bounds__(RTHREADS, 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG, RouterParams p) {
    constexpr int RSTAGES = rstages<NPMAX>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int b_bytes = p.np * RK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + RSTAGES * R_A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + RSTAGES * b_bytes);
    uint64_t* empty = full + RSTAGES;
    uint64_t* tfull = empty + RSTAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ uint8_t s_dev[256];  // expert -> device (pruning)
    pdl_trigger();
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmG);
        for (int s = 0; s < RSTAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        fence_barrier_init();
    }
    constexpr int TCOLS = 2 * NPMAX <= 32 ? 32 : (2 * NPMAX <= 64 ? 64 : (2 * NPMAX <= 128 ? 128 : (2 * NPMAX <= 256 ? 256 : 512)));
    if (warp == 1) tmem_alloc<TCOLS>(tmem_slot);
    pdl_wait();  // x (and the tables) may come from the previous kernel in the stream
    if (p.prune)
        for (int i = threadIdx.x; i < p.e; i += blockDim.x) s_dev[i] = (uint8_t)p.dev_of[i];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int tiles = (p.n + RM - 1) / RM;
    const int KB = (p.d + RK - 1) / RK;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x)
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], R_A_BYTES + b_bytes);
                    tma_load_2d(sA + stage * R_A_BYTES, &tmX, &full[stage], kb * RK, tile * RM);
                    tma_load_2d(sB + stage * b_bytes, &tmG, &full[stage], kb * RK, 0);
                    if (++stage == RSTAGES) { stage = 0; phase ^= 1; }
                }
        }
    } else if (warp == 1) {
        const uint32_t idesc = idesc_bf16_f32(RM, p.np);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * NPMAX;
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA + stage * R_A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * b_bytes);
#pragma unroll
                    for (int k = 0; k < RK / 16; ++k)
                        umma_bf16(d_tmem, sdesc_k_sw128(a0 + k * 32), sdesc_k_sw128(b0 + k * 32), idesc,
                                  (kb | k) != 0);
                    umma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == RSTAGES) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) umma_commit(&tfull[acc]);
            __syncwarp();
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    } else {
        const int q = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int t = tile * RM + q * 32 + lane;
            const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * NPMAX;
            constexpr int NCH = NPMAX / 32;
            if (p.logits_out) {  // pruning / score rows: hand the logits to router_select
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) {
                    if (c * 32 >= p.np) break;
                    uint32_t u[32];
                    tmem_ld32(tb + c * 32, u);
                    tmem_ld_wait();
                    if (t < p.n)
                        for (int i = 0; i < 32; ++i)
                            if (c * 32 + i < p.e) p.logits_out[(long)t * p.e + c * 32 + i] = __uint_as_float(u[i]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                continue;
            }
            if constexpr (NPMAX <= 128) {
            uint32_t v[NCH][32];
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                if (c * 32 < p.np) tmem_ld32(tb + c * 32, v[c]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            if (t >= p.n) continue;
            // softmax with max subtraction (routing.cpp:44-49), fp32
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (c * 32 + i < p.e) mx = fmaxf(mx, __uint_as_float(v[c][i]));
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (c * 32 + i < p.e) {
                        const float s = __expf(__uint_as_float(v[c][i]) - mx);
                        v[c][i] = __float_as_uint(s);
                        sum += s;
                    }
            const float inv = 1.0f / sum;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    v[c][i] = __float_as_uint(c * 32 + i < p.e ? __uint_as_float(v[c][i]) * inv : -1.0f);
            if (p.prune) {
                // prune_router_score (pruning.cpp:35-64) on the register row: the
                // first `budget` distinct devices of the top-k in score order, then
                // the k best experts on those devices.  Rounds walk the order
                // (score desc, index asc) strictly after the previous pick.
                uint64_t allowed = 0;
                int na = 0;
                float ls = 2.0f;
                int lj = -1;
                for (int r = 0; r < p.k; ++r) {
                    float best = -2.0f;
                    int bj = -1;
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int j = c * 32 + i;
                            const float sv = __uint_as_float(v[c][i]);
                            const bool after = sv < ls || (sv == ls && j > lj);
                            if (after && sv > best) { best = sv; bj = j; }
                        }
                    ls = best;
                    lj = bj;
                    const uint64_t bit = 1ull << s_dev[bj];
                    if (!(allowed & bit) && na < p.budget) { allowed |= bit; ++na; }
                }
                int32_t* ids = p.ids + (long)t * p.k;
                float* wout = p.w + (long)t * p.k;
                float tot = 0.f;
                ls = 2.0f;
                lj = -1;
                for (int r = 0; r < p.k; ++r) {
                    float best = -2.0f;
                    int bj = -1;
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int j = c * 32 + i;
                            const float sv = __uint_as_float(v[c][i]);
                            const bool after = sv < ls || (sv == ls && j > lj);
                            if (after && sv > best && j < p.e && ((allowed >> s_dev[j < p.e ? j : 0]) & 1)) {
                                best = sv;
                                bj = j;
                            }
                        }
                    if (bj < 0) {  // CapacityError
                        atomicExch(p.err, 5);
                        break;
                    }
                    ids[r] = bj;
                    wout[r] = best;
                    tot += best;
                    ls = best;
                    lj = bj;
                }
                if (p.prune_renorm)
                    for (int r = 0; r < p.k; ++r) wout[r] = wout[r] / tot;
                continue;
            }
            // top-k by (score desc, index asc): k argmax rounds over the
            // register-resident row (strict > in ascending index order keeps
            // the lower index on ties); selected entries become -1
            float tot = 0.f;
            int32_t* ids = p.ids + (long)t * p.k;
            float* wout = p.w + (long)t * p.k;
            for (int r = 0; r < p.k; ++r) {
                float best = -2.0f;
                int bj = 0;
#pragma unroll
                for (int c = 0; c < NCH; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float s = __uint_as_float(v[c][i]);
                        if (s > best) { best = s; bj = c * 32 + i; }
                    }
#pragma unroll
                for (int c = 0; c < NCH; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (c * 32 + i == bj) v[c][i] = __float_as_uint(-1.0f);
                ids[r] = bj;
                wout[r] = best;
                tot += best;
            }
            if (p.renorm)
                for (int r = 0; r < p.k; ++r) wout[r] = wout[r] / tot;
            }  // NPMAX <= 128
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TCOLS>(tmem_base);
    }
}

template <int NPMAX>
void launch_router_np(const CUtensorMap& tx, const CUtensorMap& tg, const RouterParams& p, int num_sms,
                      cudaStream_t st) {
    const int tiles = (p.n + RM - 1) / RM;
    const int grid = tiles < num_sms ? tiles : num_sms;
    const int smem = rstages<NPMAX>() * (R_A_BYTES + p.np * RK * 2) + 256 + 1024;
    cudaFuncSetAttribute(router_tc_kernel<NPMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_pdl(router_tc_kernel<NPMAX>, grid, RTHREADS, smem, st, tx, tg, p);
}

}  // namespace

bool launch_router_tc(const void* tmap_x, const void* tmap_g, int n, int d, int e, int k, int renorm, int32_t* ids,
                      float* w, float* logits_out, int num_sms, cudaStream_t st, const PruneDev* prune,
                      int32_t* err) {
    if (n <= 0) return true;
    const int np = (e + 31) / 32 * 32;
    if (np > 256 || k > kMaxTopK) return false;
    RouterParams p{n, d, e, np, k, renorm, ids, w, logits_out, 0, 0, 0, nullptr, err};
    if (prune && prune->mode == 1) {
        p.prune = 1;
        p.budget = prune->budget;
        p.prune_renorm = prune->renorm;
        p.dev_of = prune->dev_of;
    }
    const CUtensorMap& tx = *reinterpret_cast<const CUtensorMap*>(tmap_x);
    const CUtensorMap& tg = *reinterpret_cast<const CUtensorMap*>(tmap_g);
    if (np > 128 && !logits_out) return false;  // wide gates: select in router_select
    if (np <= 32) launch_router_np<32>(tx, tg, p, num_sms, st);
    else if (np <= 64) launch_router_np<64>(tx, tg, p, num_sms, st);
    else if (np <= 128) launch_router_np<128>(tx, tg, p, num_sms, st);
    else launch_router_np<256>(tx, tg, p, num_sms, st);
    count_launch();
    return true;
}

}  // namespace occ
