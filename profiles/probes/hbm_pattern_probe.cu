// hbm_pattern_probe.cu — what HBM bandwidth do the layer's row-copy patterns
// reach with plain vector kernels?  Mixtral shapes: 16,384 token rows of
// 8 KB (D = 4096 bf16), 32,768 expert rows.
//   copy   : row i -> row i                        (1 read : 1 write)
//   fanout : row i -> rows dst[2i], dst[2i+1]       (1 : 2, pack / scatter)
//   fanin  : rows src[2i] + src[2i+1] -> row i     (2 : 1, combine), fp32 sum
// Variants: V 16-byte vectors per lane in flight (whole-row unroll), block
// size, grid (persistent 148 x B vs one warp per row), streaming store hint.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a hbm_pattern_probe.cu -o hbm_pattern_probe
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

constexpr int D = 4096, NV = D / 8;  // uint4 per row

__device__ __forceinline__ void st_cs(uint4* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int V, bool CS>
__global__ void fanout_k(const uint4* __restrict__ x, uint4* __restrict__ y, const int* __restrict__ dst, int n, int f) {
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += (gridDim.x * blockDim.x) >> 5) {
        int rows[4];
        for (int q = 0; q < f; ++q) rows[q] = dst[t * f + q];
        for (int v0 = 0; v0 < NV; v0 += V * 32) {
            uint4 b[V];
#pragma unroll
            for (int u = 0; u < V; ++u) b[u] = ld_nc(x + (long)t * NV + v0 + u * 32 + lane);
            for (int q = 0; q < f; ++q) {
                uint4* o = y + (long)rows[q] * NV + v0 + lane;
#pragma unroll
                for (int u = 0; u < V; ++u) {
                    if (CS) st_cs(o + u * 32, b[u]);
                    else o[u * 32] = b[u];
                }
            }
        }
    }
}

__device__ __forceinline__ void addbf(float* a, uint4 u) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(h[e]);
        a[2 * e] += f.x;
        a[2 * e + 1] += f.y;
    }
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

template <int V, bool CS>
__global__ void fanin_k(const uint4* __restrict__ y, uint4* __restrict__ out, const int* __restrict__ src, int n) {
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += (gridDim.x * blockDim.x) >> 5) {
        const int r0 = src[2 * t], r1 = src[2 * t + 1];
        for (int v0 = 0; v0 < NV; v0 += V * 32) {
            uint4 a[V], b[V];
#pragma unroll
            for (int u = 0; u < V; ++u) {
                a[u] = ld_nc(y + (long)r0 * NV + v0 + u * 32 + lane);
                b[u] = ld_nc(y + (long)r1 * NV + v0 + u * 32 + lane);
            }
#pragma unroll
            for (int u = 0; u < V; ++u) {
                float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                addbf(acc, a[u]);
                addbf(acc, b[u]);
                uint4 o = make_uint4(pk(acc[0], acc[1]), pk(acc[2], acc[3]), pk(acc[4], acc[5]), pk(acc[6], acc[7]));
                if (CS) st_cs(out + (long)t * NV + v0 + u * 32 + lane, o);
                else out[(long)t * NV + v0 + u * 32 + lane] = o;
            }
        }
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <typename L>
float timeit(L launch, int iters = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / iters;
}

int main() {
    const int n = 16384, R = 2 * n;
    uint4 *x, *y, *out;
    int *dst, *src, *ident;
    CK(cudaMalloc(&x, (size_t)n * D * 2));
    CK(cudaMalloc(&y, (size_t)R * D * 2));
    CK(cudaMalloc(&out, (size_t)n * D * 2));
    CK(cudaMemset(x, 1, (size_t)n * D * 2));
    CK(cudaMemset(y, 1, (size_t)R * D * 2));
    std::vector<int> perm(R), id(2 * n);
    for (int i = 0; i < R; ++i) perm[i] = i;
    std::mt19937 g(1);
    std::shuffle(perm.begin(), perm.end(), g);
    for (int i = 0; i < n; ++i) id[i] = i;
    CK(cudaMalloc(&dst, R * 4));
    CK(cudaMalloc(&src, R * 4));
    CK(cudaMalloc(&ident, R * 4));
    CK(cudaMemcpy(dst, perm.data(), R * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(src, perm.data(), R * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ident, id.data(), n * 4, cudaMemcpyHostToDevice));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double rowb = D * 2.0;
    auto report = [&](const char* name, float ms, double bytes) {
        printf("%-40s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    {
        float ms = timeit([&] { cudaMemcpyAsync(out, x, (size_t)n * D * 2, cudaMemcpyDeviceToDevice); });
        report("cudaMemcpy d2d 134MB", ms, 2.0 * n * rowb);
    }
    char nm[128];
#define RUN_FO(V, CS, TPB, GRID)                                                                                 \
    {                                                                                                            \
        const int grid = (GRID) ? (GRID) : (n * 32 + TPB - 1) / TPB;                                             \
        float ms = timeit([&] { fanout_k<V, CS><<<grid, TPB>>>(x, out, ident, n, 1); });                         \
        snprintf(nm, sizeof nm, "copy   V=%d cs=%d tpb=%d grid=%d", V, CS, TPB, grid);                             \
        report(nm, ms, 2.0 * n * rowb);                                                                          \
        ms = timeit([&] { fanout_k<V, CS><<<grid, TPB>>>(x, y, dst, n, 2); });                                   \
        snprintf(nm, sizeof nm, "fanout V=%d cs=%d tpb=%d grid=%d", V, CS, TPB, grid);                             \
        report(nm, ms, 3.0 * n * rowb);                                                                          \
        ms = timeit([&] { fanin_k<V, CS><<<grid, TPB>>>(y, out, src, n); });                                     \
        snprintf(nm, sizeof nm, "fanin  V=%d cs=%d tpb=%d grid=%d", V, CS, TPB, grid);                             \
        report(nm, ms, 3.0 * n * rowb);                                                                          \
    }
    RUN_FO(2, false, 256, 0)
    RUN_FO(4, false, 256, 0)
    RUN_FO(8, false, 256, 0)
    RUN_FO(16, false, 256, 0)
    RUN_FO(4, true, 256, 0)
    RUN_FO(8, true, 256, 0)
    RUN_FO(4, false, 512, 0)
    RUN_FO(8, false, 512, 0)
    RUN_FO(4, false, 256, sms * 8)
    RUN_FO(8, false, 256, sms * 8)
    RUN_FO(4, true, 256, sms * 8)
    RUN_FO(8, true, 256, sms * 8)
    RUN_FO(4, false, 1024, sms * 2)
    RUN_FO(8, false, 1024, sms * 2)
    RUN_FO(16, false, 512, sms * 2)
    return 0;
}
