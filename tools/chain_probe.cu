// tools/chain_probe.cu -- is a 2^20-thread warp-aggregated dequeue bound by the
// same-address RMW chain?  Per warp, the leader does count RMW -> head RMW
// (dependent), like reserve + ticket.  A: one counter pair for the whole grid;
// B: one pair per block (no cross-block contention); C: A plus a dependent
// 8-byte slot load per lane at the ticket (the real dequeue's third round trip).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned long long* ctr, unsigned long long* slots, unsigned long long* out) {
    const unsigned lane = threadIdx.x & 31;
    unsigned long long* c = MODE == 1 ? ctr + 2 * 128 * blockIdx.x : ctr;   // 1 KiB apart per block
    unsigned long long t = 0;
    if (lane == 0) {
        const long long old = (long long)atomicAdd(c, (unsigned long long)-32ll);
        t = atomicAdd(c + 128, (unsigned long long)(old > -(1ll << 40) ? 32 : 0));
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    unsigned long long x = t;
    if (MODE == 2) x = *reinterpret_cast<volatile unsigned long long*>(slots + ((t + lane) & ((1 << 22) - 1)));
    if (x == 0x1234567) out[0] = x;
}
int main() {
    unsigned long long *ctr, *slots, *out;
    cudaMalloc(&ctr, 4096 * 2 * 128 * 8); cudaMemset(ctr, 0, 4096 * 2 * 128 * 8);
    cudaMalloc(&slots, 8ull << 22); cudaMemset(slots, 0, 8ull << 22);
    cudaMalloc(&out, 8);
    const char* names[] = {"A shared pair", "B per-block pair", "C shared pair + slot load"};
    void (*ks[])(unsigned long long*, unsigned long long*, unsigned long long*) = {k<0>, k<1>, k<2>};
    for (int m = 0; m < 3; ++m) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        ks[m]<<<4096, 256>>>(ctr, slots, out);
        cudaEventRecord(a); ks[m]<<<4096, 256>>>(ctr, slots, out); cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        std::printf("%-28s %6.1f us\n", names[m], ms * 1e3);
    }
    return 0;
}
