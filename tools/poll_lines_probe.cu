// Dependent-load latency of retry polls vs pollers per line: 888 blocks (6 per
// SM), one polling warp each, 64 back-to-back .relaxed.gpu loads of line
// (block % lines).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/poll_lines_probe.cu -o /tmp/poll_lines_probe
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__global__ void __launch_bounds__(256, 6) k_poll(const unsigned long long* a, int lines, int rounds, unsigned long long* cyc) {
    if (threadIdx.x != 0) return;
    const unsigned long long* p = a + (unsigned long long)(blockIdx.x % lines) * 64;  // 512 B apart
    unsigned long long acc = 0;
    const long long t0 = clock64();
#pragma unroll 16
    unsigned long long v = 0;
    for (int i = 0; i < rounds; ++i) { v = ld_rlx(p + (v >> 63)); acc += v; }  // dependent chain
    const long long t1 = clock64();
    atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (acc == 12345) atomicAdd(cyc + 1, 1ull);
}
int main() {
    unsigned long long *a, *cyc;
    cudaMalloc(&a, 1 << 24); cudaMemset(a, 0, 1 << 24); cudaMalloc(&cyc, 16);
    const int blocks = 148 * 6, rounds = 64;
    for (int lines : {1, 2, 4, 8, 16, 32, 64, 888}) {
        unsigned long long h = 0;
        for (int r = 0; r < 3; ++r) {
            cudaMemset(cyc, 0, 16);
            k_poll<<<blocks, 256>>>(a, lines, rounds, cyc);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("lines %4d  pollers/line %6.1f  cycles/load %.0f\n", lines, (double)blocks / lines,
               (double)h / blocks / rounds);
    }
    return 0;
}
