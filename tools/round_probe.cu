// tools/round_probe.cu -- counts spins / CAS wins / L2 polls per observed_empty
// call under the bench's grid (4096 x 256, leader lanes looping 64 rounds).
#include <cstdio>
#include <cuda_runtime.h>
#include "ouro_device.cuh"
using namespace ouro_dev;
__device__ unsigned long long g_calls, g_spins, g_polls, g_fresh, g_reuse, g_wait;
__device__ bool probe_empty(ouro_queue_dev* Q) {
    const u64 tag = (((u64)Q >> 10) ^ ((u64)Q >> 15)) & 31u;
    u64* slot = poll_cache() + (tag & 7);
    atomicAdd(&g_calls, 1ull);
    for (int spins = 0; spins < 256; ++spins) {
        atomicAdd(&g_spins, 1ull);
        const u64 now = gtime256();
        const u64 e = *reinterpret_cast<volatile u64*>(slot);
        const bool match = ((e >> 3) & 31u) == tag;
        const i64 age = (i64)(now - (e >> 8));
        if (match && !(e & 4u)) {
            if (!(e & 2u) && age < (i64)kPollWindow) { atomicAdd(&g_fresh, 1ull); return (e & 1u) != 0; }
            if ((e & 2u) && age < 4 * (i64)kPollWindow) { atomicAdd(&g_reuse, 1ull); return (e & 1u) != 0; }
        }
        if (match && (e & 6u) == 6u && age < 4 * (i64)kPollWindow) { atomicAdd(&g_wait, 1ull); __nanosleep(32); continue; }
        const u64 mine = (match && !(e & 4u)) ? (e | 2u) : ((now << 8) | (tag << 3) | 6u);
        if (atomicCAS(slot, e, mine) != e) continue;
        atomicAdd(&g_polls, 1ull);
        const bool empty = (i64)ld_rlx((const u64*)&Q->count) <= 0;
        atomicExch(slot, (gtime256() << 8) | (tag << 3) | (empty ? 1u : 0u));
        return empty;
    }
    return true;
}
__global__ void k(ouro_heap_view v, ouro_queue_dev* Q, int rounds) {
    const unsigned lane = threadIdx.x & 31;
    unsigned a = 0;
    if (lane == 0) {
        for (;;) {
            if (++a >= (unsigned)rounds) break;
            backoff(v, a);
            if (!probe_empty(Q)) break;
        }
    }
    a = __shfl_sync(0xffffffffu, a, 0);
}
__global__ void clk(unsigned long long* o) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < 1000000; ++i) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); if (t1 != t0) break; }
    o[0] = t1 - t0;
}
int main() {
    ouro_queue_dev* Q;
    cudaMalloc(&Q, sizeof(ouro_queue_dev));
    cudaMemset(Q, 0, sizeof(ouro_queue_dev));
    ouro_heap_view v{};
    v.backoff = OURO_BACKOFF_FENCE;
    unsigned long long z = 0, h[6];
    for (auto* s : {&g_calls, &g_spins, &g_polls, &g_fresh, &g_reuse, &g_wait}) cudaMemcpyToSymbol(*s, &z, 8);
    k<<<4096, 256>>>(v, Q, 64);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&h[0], g_calls, 8); cudaMemcpyFromSymbol(&h[1], g_spins, 8);
    cudaMemcpyFromSymbol(&h[2], g_polls, 8); cudaMemcpyFromSymbol(&h[3], g_fresh, 8);
    cudaMemcpyFromSymbol(&h[4], g_reuse, 8); cudaMemcpyFromSymbol(&h[5], g_wait, 8);
    std::printf("calls %llu spins %llu polls %llu fresh %llu reuse %llu wait %llu\n", h[0], h[1], h[2], h[3], h[4], h[5]);
    unsigned long long* o; cudaMalloc(&o, 8);
    clk<<<1, 1>>>(o);
    unsigned long long tick; cudaMemcpy(&tick, o, 8, cudaMemcpyDeviceToHost);
    std::printf("globaltimer tick = %llu ns\n", tick);
    return 0;
}
