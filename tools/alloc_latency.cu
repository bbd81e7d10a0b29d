// tools/alloc_latency.cu -- per-warp latency of ouro_malloc / ouro_free inside a
// 2^20-thread launch (page kind, 1 GiB heap, malloc(16)): globaltimer at warp
// entry/exit gives each warp's latency and the number of warps in flight.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "ouro_device.cuh"
#include "ouro.h"

__global__ void k(ouro_heap_view v, void** out, unsigned long long* t, int do_free) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned long long a, b;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
    if (!do_free) out[i] = ouro_malloc_t<OURO_KIND_PAGE, OURO_FLAVOR_ARRAY>(v, 16, nullptr, 0xffffffffu);
    else ouro_free_t<OURO_KIND_PAGE, OURO_FLAVOR_ARRAY>(v, out[i], 0xffffffffu);
    __syncwarp();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b));
    if ((threadIdx.x & 31) == 0) { t[2 * (i / 32)] = a; t[2 * (i / 32) + 1] = b; }
}
int main() {
    ouro_config c; ouro_config_default(&c); c.heap_bytes = 1ull << 30;
    ouro_heap* h; if (ouro_heap_create(&c, 0, &h)) return 1;
    ouro_heap_view v; ouro_heap_get_view(h, &v, sizeof v);
    const int n = 1 << 20, W = n / 32;
    void** out; cudaMalloc(&out, n * 8);
    unsigned long long* t; cudaMalloc(&t, W * 16);
    std::vector<unsigned long long> ht(2 * W);
    for (int rep = 0; rep < 3; ++rep)
        for (int f = 0; f < 2; ++f) {
            k<<<n / 256, 256>>>(v, out, t, f);
            cudaDeviceSynchronize();
            if (rep < 2) continue;
            cudaMemcpy(ht.data(), t, W * 16, cudaMemcpyDeviceToHost);
            unsigned long long t0 = ~0ull, t1 = 0;
            std::vector<double> lat(W);
            for (int w = 0; w < W; ++w) { t0 = std::min(t0, ht[2*w]); t1 = std::max(t1, ht[2*w+1]); lat[w] = (ht[2*w+1] - ht[2*w]) / 1e3; }
            std::sort(lat.begin(), lat.end());
            double sum = 0; for (double x : lat) sum += x;
            std::printf("%s: span %.1f us, warp latency mean %.2f p50 %.2f p90 %.2f p99 %.2f max %.2f us, mean warps in flight %.0f\n",
                        f ? "free " : "alloc", (t1 - t0) / 1e3, sum / W, lat[W/2], lat[W*9/10], lat[W*99/100], lat[W-1],
                        sum / ((t1 - t0) / 1e3));
        }
    return 0;
}
