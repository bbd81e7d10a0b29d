// tools/round_cost.cu -- cycles per retry-round primitive on a fully occupied B200
// (64 warps/SM): fence.sc.cta, fence.acq_rel.cta, fence.sc.gpu, nanosleep(0),
// globaltimer, shared-memory load.  Used to choose FenceRetry's GPU form.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned long long* out, int iters) {
    __shared__ unsigned long long s[8];
    if (threadIdx.x < 8) s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    unsigned long long acc = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) asm volatile("fence.sc.cta;" ::: "memory");
        if (MODE == 1) asm volatile("fence.acq_rel.cta;" ::: "memory");
        if (MODE == 2) asm volatile("fence.sc.gpu;" ::: "memory");
        if (MODE == 3) __nanosleep(0);
        if (MODE == 4) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); acc += t; }
        if (MODE == 5) acc += *reinterpret_cast<volatile unsigned long long*>(&s[i & 7]);
        if (MODE == 6) { asm volatile("fence.sc.cta;" ::: "memory"); __nanosleep(0); }
    }
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
    if (acc == 42) out[1] = acc;
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const char* names[] = {"fence.sc.cta", "fence.acq_rel.cta", "fence.sc.gpu", "nanosleep(0)", "globaltimer", "lds", "sc.cta+nanosleep0"};
    void (*ks[])(unsigned long long*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
    for (int m = 0; m < 7; ++m) {
        cudaMemset(d, 0, 16);
        const int iters = 256, blocks = 148 * 8, threads = 256;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        ks[m]<<<blocks, threads>>>(d, iters);
        cudaMemset(d, 0, 16);
        cudaEventRecord(a);
        ks[m]<<<blocks, threads>>>(d, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        const double warps = blocks * threads / 32.0;
        std::printf("%-20s %8.1f cycles/iter/warp   kernel %.3f ms (%.1f ns per warp-iter wall)\n", names[m],
                    cyc / warps / iters, ms, ms * 1e6 / iters);
    }
    return 0;
}
