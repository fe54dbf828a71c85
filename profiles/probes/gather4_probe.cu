// Probe: TMA tile::gather4 semantics on sm_100a (box shape accepted by the
// tensor map, smem placement with 128-byte swizzle) vs a plain tile load.
// nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "../../paper_2505_13345_b200/csrc/occ_common.cuh"

using namespace occ;

__global__ void probe(const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap g4_map,
                      const int* rows, uint8_t* out_tile, uint8_t* out_g4) {
    __shared__ __align__(1024) uint8_t sA[16384];
    __shared__ __align__(1024) uint8_t sB[16384];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[0], 16384);
        tma_load_2d(sA, &tile_map, &bar[0], 0, 0);  // rows 0..127 (identity order)
        mbar_arrive_expect_tx(&bar[1], 16384);
        for (int i = 0; i < 32; ++i)
            tma_gather4(sB + i * 512, &g4_map, &bar[1], 0, rows[4 * i], rows[4 * i + 1], rows[4 * i + 2],
                        rows[4 * i + 3]);
    }
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1], 0);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) {
        out_tile[i] = sA[i];
        out_g4[i] = sB[i];
    }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int R = 512, C = 256;  // bf16 [R, C]
    __nv_bfloat16* h = (__nv_bfloat16*)malloc(R * C * 2);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) h[r * C + c] = __float2bfloat16((float)((r * 7 + c) % 251));
    void* d;
    cudaMalloc(&d, R * C * 2);
    cudaMemcpy(d, h, R * C * 2, cudaMemcpyHostToDevice);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Enc enc = (Enc)fn;
    CUtensorMap tm, g4;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    CUresult r1 = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int* drows;
    cudaMalloc(&drows, 128 * 4);
    uint8_t *ot, *og;
    cudaMalloc(&ot, 16384);
    cudaMalloc(&og, 16384);
    uint8_t* ht = (uint8_t*)malloc(16384);
    uint8_t* hg = (uint8_t*)malloc(16384);
    for (int boxh = 1; boxh <= 4; boxh *= 4) {
        cuuint32_t gbox[2] = {64, (cuuint32_t)boxh};
        CUresult r2 = enc(&g4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, gbox, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("boxh=%d encode tile=%d gather=%d\n", boxh, (int)r1, (int)r2);
        if (r2) continue;
        for (int pass = 0; pass < 2; ++pass) {
            int hr[128];
            for (int i = 0; i < 128; ++i) hr[i] = pass == 0 ? i : (i == 5 ? -1 : (i == 6 ? R + 3 : (i * 37) % R));
            cudaMemcpy(drows, hr, sizeof(hr), cudaMemcpyHostToDevice);
            cudaMemset(og, 0xAB, 16384);
            probe<<<1, 128>>>(tm, g4, drows, ot, og);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("  kernel error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(ht, ot, 16384, cudaMemcpyDeviceToHost);
            cudaMemcpy(hg, og, 16384, cudaMemcpyDeviceToHost);
            if (pass == 0) {
                printf("  identity rows: gather4 smem == tile smem: %s\n", memcmp(ht, hg, 16384) ? "NO" : "yes");
            } else {
                // check: de-swizzle gather smem: element (row i, col c) at i*128 + ((c/8) ^ (i%8))*16 + (c%8)*2
                int bad = 0, zero_ok = 1;
                for (int i = 0; i < 128; ++i)
                    for (int c = 0; c < 64; ++c) {
                        uint16_t v;
                        memcpy(&v, hg + i * 128 + (((c / 8) ^ (i % 8)) * 16) + (c % 8) * 2, 2);
                        uint16_t want;
                        if (hr[i] < 0 || hr[i] >= R) { want = 0; if (v != 0) zero_ok = 0; continue; }
                        __nv_bfloat16 w = h[hr[i] * C + c];
                        memcpy(&want, &w, 2);
                        if (v != want) ++bad;
                    }
                printf("  permuted rows: mismatches=%d  OOB rows zero=%d\n", bad, zero_ok);
            }
        }
    }
    return 0;
}
