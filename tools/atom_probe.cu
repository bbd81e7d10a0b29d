// Same-address atomic throughput on B200: each warp leader issues `per` atomics
// to one of `naddr` addresses (1 KiB apart).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/atom_probe.cu -o /tmp/atom_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_rmw(unsigned long long* a, int per, int naddr, unsigned long long* sink) {
    if ((threadIdx.x & 31) == 0) {
        unsigned long long acc = 0;
        const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        unsigned long long* p = a + (w % naddr) * 128;
        for (int i = 0; i < per; ++i) acc += atomicAdd(p, 1ull);
        if (acc == 42) *sink = acc;
    }
}
__global__ void k_red(unsigned long long* a, int per, int naddr) {
    if ((threadIdx.x & 31) == 0) {
        const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        unsigned long long* p = a + (w % naddr) * 128;
        for (int i = 0; i < per; ++i) atomicAdd(p, 1ull);
    }
}
__global__ void k_cas(unsigned long long* a, int per, int naddr) {
    if ((threadIdx.x & 31) == 0) {
        const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        unsigned long long* p = a + (w % naddr) * 128;
        for (int i = 0; i < per; ++i) {
            unsigned long long m = *(volatile unsigned long long*)p;
            for (;;) { unsigned long long prev = atomicCAS(p, m, m + 1); if (prev == m) break; m = prev; }
        }
    }
}
int main() {
    unsigned long long *a, *sink;
    cudaMalloc(&a, 1 << 24); cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int warps = 32768, per = 1;
    for (int naddr : {1, 2, 4, 16, 256}) {
        for (int kind = 0; kind < 3; ++kind) {
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaMemset(a, 0, 1 << 24);
                cudaEventRecord(e0);
                if (kind == 0) k_rmw<<<warps / 8, 256>>>(a, per, naddr, sink);
                else if (kind == 1) k_red<<<warps / 8, 256>>>(a, per, naddr);
                else k_cas<<<warps / 8, 256>>>(a, per, naddr);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
            }
            const char* nm[] = {"atomicAdd(ret)", "red.add", "CAS loop"};
            printf("naddr %3d %-15s %8.2f us  %.2f ns/op/addr\n", naddr, nm[kind], best * 1e3, best * 1e6 / (warps * per / naddr));
        }
    }
    // baseline: empty kernel
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k_red<<<warps / 8, 256>>>(a, 0, 1); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("empty kernel %.2f us\n", best * 1e3);
    return 0;
}
