// Probe: how much of a buffer survives in L2 between two passes, and does a
// line brought in by one SM hit for an SM on the other die?
// One CTA per SM; pass 1: CTA i streams chunk i of an X MB buffer; grid
// barrier; pass 2: CTA i streams chunk (i + shift) % ctas.  ncu
// dram__bytes_read.sum ~ X MB means the whole buffer stayed resident (and is
// shared across dies when shift moves chunks to the other die's SMs); ~2X
// means nothing survived.
// nvcc -gencode arch=compute_100a,code=sm_100a -o l2_capacity_probe l2_capacity_probe.cu
// usage: l2_capacity_probe MB [shift] [ctas]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ unsigned int g_bar;

__device__ __forceinline__ uint4 ldcg(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__global__ void two_pass(const uint4* __restrict__ buf, size_t chunk16, int shift, unsigned long long* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint4* c1 = buf + blockIdx.x * chunk16;
    for (size_t i = threadIdx.x; i < chunk16; i += blockDim.x) {
        const uint4 v = ldcg(c1 + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&g_bar, 1u);
        while (atomicAdd(&g_bar, 0u) < gridDim.x) __nanosleep(100);
    }
    __syncthreads();
    const uint4* c2 = buf + ((blockIdx.x + shift) % gridDim.x) * chunk16;
    for (size_t i = threadIdx.x; i < chunk16; i += blockDim.x) {
        const uint4 v = ldcg(c2 + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void fill(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4((unsigned)i, 1, 2, 3);
}

int main(int argc, char** argv) {
    const int mb = argc > 1 ? atoi(argv[1]) : 64;
    const int shift = argc > 2 ? atoi(argv[2]) : 0;
    const int ctas = argc > 3 ? atoi(argv[3]) : 148;
    const size_t chunk16 = (size_t)mb * (1 << 20) / 16 / ctas;
    uint4* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, chunk16 * ctas * 16);
    cudaMalloc(&sink, 8);
    fill<<<1024, 256>>>(buf, chunk16 * ctas);
    const unsigned int zero = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpyToSymbol(g_bar, &zero, sizeof(zero));
        two_pass<<<ctas, 1024>>>(buf, chunk16, shift, sink);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("buffer %d MB, shift %d, %d CTAs: %s\n", mb, shift, ctas, cudaGetErrorString(e));
    return 0;
}
