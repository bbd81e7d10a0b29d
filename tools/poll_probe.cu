// poll_probe.cu -- what a failed retry round is made of on B200 (cycles, SM clock):
//   nanosleep(t) actual length, %globaltimer read cost / update step, shared-memory
//   CAS latency, and the latency of a .relaxed.gpu load of ONE hot word while
//   B blocks x 1 leader lane poll it back to back (the OOM-storm pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/poll_probe tools/poll_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 ld_rlx(const u64* p) {
    u64 r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ u64 gtime() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_misc(u64* out) {
    __shared__ u64 s[4];
    if (threadIdx.x) return;
    s[0] = 0;
    const int sleeps[5] = {0, 32, 100, 256, 1000};
    for (int j = 0; j < 5; ++j) {
        u64 c0 = clock64();
        for (int i = 0; i < 64; ++i) __nanosleep(sleeps[j]);
        out[j] = (clock64() - c0) / 64;
    }
    // globaltimer read cost and smallest observed step
    u64 c0 = clock64(), prev = gtime(), step = ~0ull;
    for (int i = 0; i < 4096; ++i) {
        const u64 t = gtime();
        if (t != prev && t - prev < step) step = t - prev;
        prev = t;
    }
    out[5] = (clock64() - c0) / 4096;
    out[6] = step;
    // shared CAS round trip
    c0 = clock64();
    u64 x = 0;
    for (int i = 0; i < 256; ++i) x = atomicCAS(&s[0], x, x + 1);
    out[7] = (clock64() - c0) / 256;
    out[8] = x;
}

// every block: lane 0 of warp 0 loads the hot word `iters` times back to back
__global__ void k_poll(const u64* hot, int iters, u64* cyc) {
    if (threadIdx.x) return;
    u64 acc = 0;
    const u64 c0 = clock64();
    for (int i = 0; i < iters; ++i) acc += ld_rlx(hot + (acc >> 63));  // address depends on the last load
    if (acc == 12345) cyc[2] = acc;  // consume before reading the clock
    const u64 c1 = clock64();
    atomicAdd(&cyc[0], (c1 - c0) / iters);
    atomicAdd(&cyc[1], 1ull + (acc & 0));
}

int main() {
    u64 *out, *hot, *cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&hot, 1 << 20);
    cudaMalloc(&cyc, 32);
    cudaMemset(hot, 0, 1 << 20);
    k_misc<<<1, 32>>>(out);
    u64 h[16];
    cudaMemcpy(h, out, 9 * 8, cudaMemcpyDeviceToHost);
    printf("nanosleep(0/32/100/256/1000) cycles: %llu %llu %llu %llu %llu\n", h[0], h[1], h[2], h[3], h[4]);
    printf("globaltimer read: %llu cycles, min step %llu ns\n", h[5], h[6]);
    printf("shared CAS round trip: %llu cycles\n", h[7]);
    for (int blocks : {1, 148, 592, 888, 1776, 3552}) {
        cudaMemset(cyc, 0, 16);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_poll<<<blocks, 32>>>(hot, 256, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        u64 c[2];
        cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
        printf("hot-word poll, %5d blocks: %6llu cycles per load, %.1f us, %.2f G loads/s\n", blocks,
               c[0] / (c[1] ? c[1] : 1), ms * 1e3, blocks * 256.0 / (ms * 1e6));
    }
    return 0;
}
