// A second translation unit including the device header: proves the header is
// ODR-safe to include from several files of one program.
#include <cuda_runtime.h>

#include "ouro_device.cuh"

__global__ void one_alloc(ouro_heap_view h, int* ok) {
    void* p;
    if (h.kind == OURO_KIND_PAGE && h.flavor == OURO_FLAVOR_ARRAY) {
        p = ouro_malloc_t<OURO_KIND_PAGE, OURO_FLAVOR_ARRAY>(h, 100);   // compile-time variant
        ok[threadIdx.x] = p != nullptr;
        ouro_free_t<OURO_KIND_PAGE, OURO_FLAVOR_ARRAY>(h, p);
    } else {
        p = ouro_malloc(h, 100);                                        // runtime dispatch
        ok[threadIdx.x] = p != nullptr;
        ouro_free(h, p);
    }
}

int second_tu_check(const ouro_heap_view& v) {
    int* ok;
    cudaMalloc(&ok, 32 * sizeof(int));
    one_alloc<<<1, 32>>>(v, ok);
    int h[32] = {0};
    cudaMemcpy(h, ok, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(ok);
    for (int i = 0; i < 32; ++i)
        if (!h[i]) return 1;
    return 0;
}
