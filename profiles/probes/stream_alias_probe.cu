// Probe: which streams of one context share a hardware queue with stream 0?
// A bounded spin-wait kernel on stream 0 waits for a flag that a kernel on
// stream j sets; if stream j's kernel is queued behind the spinning one (the
// two streams alias onto one of CUDA_DEVICE_MAX_CONNECTIONS queues) the wait
// times out.   nvcc -gencode arch=compute_100a,code=sm_100a -o stream_alias_probe stream_alias_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void spin(volatile unsigned* flag, unsigned want, unsigned long long budget_ns, int* timed_out) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*flag != want) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > budget_ns) {
            *timed_out = 1;
            return;
        }
        __nanosleep(200);
    }
}
__global__ void set(volatile unsigned* flag, unsigned v) { *flag = v; }

int main(int argc, char** argv) {
    const int S = argc > 1 ? atoi(argv[1]) : 48;
    const char* e = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    cudaStream_t* s = new cudaStream_t[S];
    for (int i = 0; i < S; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
    unsigned* flag;
    int* to;
    cudaMalloc(&flag, 4);
    cudaMalloc(&to, 4);
    printf("CUDA_DEVICE_MAX_CONNECTIONS=%s streams=%d; aliased with stream 0:", e ? e : "(unset)", S);
    int n_alias = 0;
    for (int j = 1; j < S; ++j) {
        cudaMemset(flag, 0, 4);
        cudaMemset(to, 0, 4);
        cudaDeviceSynchronize();
        spin<<<1, 1, 0, s[0]>>>(flag, j, 20000000ull, to);
        set<<<1, 1, 0, s[j]>>>(flag, j);
        cudaDeviceSynchronize();
        int h = 0;
        cudaMemcpy(&h, to, 4, cudaMemcpyDeviceToHost);
        if (h) {
            printf(" %d", j);
            ++n_alias;
        }
    }
    printf("  (%d of %d)\n", n_alias, S - 1);
    return 0;
}
