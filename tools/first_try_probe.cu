// tools/first_try_probe.cu -- decompose the fixed cost of an OOM storm's first try
// (2^20 threads, 4096 x 256, queue empty): which part of a failing first try costs
// what.  Modes add one component at a time on top of the previous.
#include <cstdio>
#include <cuda_runtime.h>
#include "ouro_device.cuh"
using namespace ouro_dev;
template <int MODE>
__global__ void k(ouro_heap_view v, ouro_queue_dev* Q, void** out) {
    const u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const u32 lane = threadIdx.x & 31;
    u32 got = 0;
    if (lane == 0) {
        if (MODE == 1) got = (i64)ld_rlx((const u64*)&Q->count) > 0;          // same-address L2 load
        if (MODE == 2) got = reserve_deq(Q, 32, 0, false, false);              // hinted first try
        if (MODE == 3) got = reserve_deq(Q, 32, 0, true, true);                // combined poll
        if (MODE == 4) {                                                       // RMW + undo, no hint
            const i64 old = (i64)atomicAdd((u64*)&Q->count, (u64)-32ll);
            if (old < 32) atomicAdd((u64*)&Q->count, 32ull);
            got = old > 0;
        }
        if (MODE == 5) atomicAdd(ctr_at(v, 3), 32ull);                         // sharded OOM counter
    }
    got = __shfl_sync(0xffffffffu, got, 0);
    out[i] = got ? (void*)out : nullptr;
}
int main() {
    ouro_queue_dev* Q;
    cudaMalloc(&Q, sizeof(ouro_queue_dev));
    cudaMemset(Q, 0, sizeof(ouro_queue_dev));
    void** out;
    cudaMalloc(&out, 8 << 20);
    ouro_heap_view v{};
    cudaMalloc(&v.ctr, 8 * OURO_CTR_SHARDS * 256);
    const char* names[] = {"store nullptr only", "+ L2 load of count", "hinted first try (reserve_deq)",
                           "combined poll (retry form)", "RMW + undo per warp", "sharded ctr add"};
    void (*ks[])(ouro_heap_view, ouro_queue_dev*, void**) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
    for (int m = 0; m < 6; ++m) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            ks[m]<<<4096, 256>>>(v, Q, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        std::printf("%-34s %7.1f us\n", names[m], best * 1e3);
    }
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
