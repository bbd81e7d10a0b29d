// tools/combine_probe.cu -- does block-level combining (one outstanding global
// reservation per block, arrivals batch up while it is in flight, no window)
// relieve the same-address chain measured by chain_probe?
// Modes: 0 per-warp pair (baseline), 1 block combining, 2 combining + slot load.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
struct Comb { u64 acc; unsigned done; unsigned pad; u64 res[8]; };
__device__ __forceinline__ u64 ld_vol(const u64* p) { return *(volatile const u64*)p; }
__device__ __forceinline__ unsigned ld_vol32(const unsigned* p) { return *(volatile const unsigned*)p; }

__device__ u64 global_pair(u64* c, unsigned n) {
    const long long old = (long long)atomicAdd(c, (u64)-(long long)n);
    return atomicAdd(c + 128, (u64)(old > -(1ll << 40) ? n : 0));
}

template <int MODE>
__global__ void k(u64* ctr, u64* slots, u64* out) {
    __shared__ Comb cb;
    if (threadIdx.x == 0) { cb.acc = 0; cb.done = 0xffffffffu; }
    __syncthreads();
    const unsigned lane = threadIdx.x & 31;
    u64 t = 0;
    if (MODE == 0) {
        if (lane == 0) t = global_pair(ctr, 32);
    } else if (lane == 0) {
        const u64 o = atomicAdd(&cb.acc, 32ull);          // join the open batch
        const unsigned seq = (unsigned)(o >> 32), off = (unsigned)o;
        if (off == 0) {                                    // first arrival: combiner of batch seq
            while (ld_vol32(&cb.done) != seq - 1) { }      // previous batch issued & published
            const u64 tot = atomicExch(&cb.acc, (u64)(seq + 1) << 32);
            const u64 base = global_pair(ctr, (unsigned)tot);
            *(volatile u64*)&cb.res[seq & 7] = base;
            __threadfence_block();
            *(volatile unsigned*)&cb.done = seq;
            t = base;
        } else {
            while ((int)(ld_vol32(&cb.done) - seq) < 0) { }
            t = ld_vol(&cb.res[seq & 7]) + off;
        }
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    u64 x = t;
    if (MODE == 2) x = *reinterpret_cast<volatile u64*>(slots + ((t + lane) & ((1 << 22) - 1)));
    if (x == 0x1234567) out[0] = x;
}
int main() {
    u64 *ctr, *slots, *out;
    cudaMalloc(&ctr, 4096 * 2 * 128 * 8); cudaMemset(ctr, 0, 4096 * 2 * 128 * 8);
    cudaMalloc(&slots, 8ull << 22); cudaMemset(slots, 0, 8ull << 22);
    cudaMalloc(&out, 8);
    const char* names[] = {"per-warp pair", "block combining", "block combining + slot load"};
    void (*ks[])(u64*, u64*, u64*) = {k<0>, k<1>, k<2>};
    for (int bs : {128, 256, 512, 1024})
    for (int m = 0; m < 3; ++m) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const int grid = (1 << 20) / bs;
        ks[m]<<<grid, bs>>>(ctr, slots, out);
        cudaEventRecord(a); ks[m]<<<grid, bs>>>(ctr, slots, out); cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        u64 h[129]; cudaMemcpy(h, ctr, sizeof h, cudaMemcpyDeviceToHost);
        std::printf("block %4d %-30s %6.1f us  (head %llu)\n", bs, names[m], ms * 1e3, h[128]);
    }
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
