// Probe: does a buffer read by every SM come from DRAM once or once per die?
// All CTAs (one per SM) stream the same `mb` MB (ld.global.cg, L2 only) after
// an L2 flush; compare ncu dram__bytes_read.sum with the buffer size.
// nvcc -gencode arch=compute_100a,code=sm_100a -o l2_share_probe l2_share_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void stream_all(const uint4* __restrict__ buf, size_t n16, unsigned long long* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (size_t i = threadIdx.x; i < n16; i += blockDim.x) {
        uint4 v;
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(buf + i));
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void fill(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4((unsigned)i, 1, 2, 3);
}

int main(int argc, char** argv) {
    const int mb = argc > 1 ? atoi(argv[1]) : 16;
    const int ctas = argc > 2 ? atoi(argv[2]) : 148;
    size_t n16 = (size_t)mb * (1 << 20) / 16;
    uint4 *buf, *flush;
    unsigned long long* sink;
    cudaMalloc(&buf, n16 * 16);
    cudaMalloc(&flush, (size_t)512 << 20);
    cudaMalloc(&sink, 8);
    fill<<<1024, 256>>>(buf, n16);
    for (int rep = 0; rep < 3; ++rep) {
        fill<<<4096, 256>>>(flush, ((size_t)512 << 20) / 16);  // evict L2
        stream_all<<<ctas, 1024>>>(buf, n16, sink);
    }
    cudaDeviceSynchronize();
    printf("buffer %d MB, %d CTAs each streaming it once: expect %d MB of DRAM reads if L2 is shared\n", mb, ctas, mb);
    return 0;
}
