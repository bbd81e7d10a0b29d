// examples/user_kernel.cu -- how a user program drops the allocator in:
// a C++ host that builds an ouro::DeviceHeap from an ouro::HeapConfig (the
// reference's config type) and a kernel that calls ouro_malloc / ouro_free
// per thread.  Built by examples/Makefile against ../paper_2504_18211_b200/libouro_b200.so.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ouro/ouro.hpp"
#include "ouro_device.cuh"

int second_tu_check(const ouro_heap_view& v);  // second translation unit (header-only linkage)

struct Node { unsigned long long key; Node* next; };

// Every thread builds a short linked list out of device-heap nodes, checks it, frees it.
__global__ void lists(ouro_heap_view h, int len, unsigned long long* bad) {
    const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    Node* head = nullptr;
    for (int i = 0; i < len; ++i) {
        Node* n = static_cast<Node*>(ouro_malloc(h, sizeof(Node)));  // runtime-dispatched variant
        if (!n) break;
        n->key = tid * 1000 + i;
        n->next = head;
        head = n;
    }
    int i = len;
    while (head) {
        --i;
        if (head->key != tid * 1000 + i) atomicAdd(bad, 1ull);
        Node* nx = head->next;
        ouro_free(h, head);
        head = nx;
    }
}

int main(int argc, char** argv) {
    // optional: argv[1] = variant name to run alone ("all" = every variant), argv[2] = blocks
    const int blocks = argc > 2 ? std::atoi(argv[2]) : 512;
    for (auto v : ouro::kAllVariants) {
        if (argc > 1 && std::string(argv[1]) != "all" && ouro::variant_name(v) != argv[1]) continue;
        ouro::HeapConfig cfg;                     // reference defaults: 64 MiB, 64 KiB chunks
        cfg.heap_bytes = 256ull << 20;
        cfg.allocator_kind = v.kind;
        cfg.queue_flavor = v.flavor;
        ouro::DeviceHeap heap(cfg);
        auto view = heap.view<ouro_heap_view>();
        unsigned long long* bad;
        cudaMalloc(&bad, 8);
        cudaMemset(bad, 0, 8);
        lists<<<blocks, 256>>>(view, 8, bad);
        if (second_tu_check(view) != 0) { std::printf("second TU failed\n"); return 1; }
        unsigned long long hb = 0;
        cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
        cudaFree(bad);
        heap.check_device_errors();
        const ouro_digest d = heap.digest();
        std::printf("%-8s bad=%llu live_pages=%llu partition_ok=%u\n",
                    std::string(ouro::variant_name(v)).c_str(), hb, (unsigned long long)d.live_pages,
                    d.partition_ok);
        if (hb || d.live_pages || !d.partition_ok) return 1;
    }
    try {
        ouro::HeapConfig bad;
        bad.chunk_bytes = 3 << 10;
        bad.validate();
        return 1;
    } catch (const ouro::ConfigError& e) {
        std::printf("ConfigError: %s\n", e.what());
    }
    std::printf("ok\n");
    return 0;
}
