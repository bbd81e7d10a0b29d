// tools/round_loop.cu -- the failed-retry round of ouro_device.cuh in isolation:
// leader lane loops {fence + yield, observed_empty(empty queue)} R times while
// the other 31 lanes wait; full occupancy, 4096 blocks x 256 (the bench grid).
#include <cstdio>
#include <cuda_runtime.h>
#include "ouro_device.cuh"
using namespace ouro_dev;
template <int MODE>
__global__ void k(ouro_heap_view v, ouro_queue_dev* Q, int rounds, unsigned long long* out) {
    const unsigned lane = threadIdx.x & 31;
    unsigned a = 0;
    if (lane == 0) {
        for (;;) {
            if (++a >= (unsigned)rounds) break;
            if (MODE == 0) { backoff(v, a); if (!observed_empty(Q, 0)) break; }
            if (MODE == 1) { backoff(v, a); }
            if (MODE == 2) { if (!observed_empty(Q, 0)) break; }
            if (MODE == 3) { backoff(v, a); if ((long long)ld_rlx((const u64*)&Q->count) > 0) break; }
        }
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    if (a == 12345) out[0] = a;
}
int main() {
    ouro_queue_dev* Q;
    cudaMalloc(&Q, sizeof(ouro_queue_dev));
    cudaMemset(Q, 0, sizeof(ouro_queue_dev));
    unsigned long long* out;
    cudaMalloc(&out, 8);
    ouro_heap_view v{};
    v.backoff = OURO_BACKOFF_FENCE;
    const char* names[] = {"fence+yield+combined poll", "fence+yield only", "combined poll only", "fence+yield+direct L2 poll"};
    void (*ks[])(ouro_heap_view, ouro_queue_dev*, int, unsigned long long*) = {k<0>, k<1>, k<2>, k<3>};
    for (int m = 0; m < 4; ++m)
        for (int r : {1, 64}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            ks[m]<<<4096, 256>>>(v, Q, r, out);
            cudaEventRecord(a);
            ks[m]<<<4096, 256>>>(v, Q, r, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            std::printf("%-28s rounds=%3d  %8.1f us\n", names[m], r, ms * 1e3);
        }
    return 0;
}
