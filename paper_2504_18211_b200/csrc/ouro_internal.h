// ouro_internal.h -- private host-side types of libouro_b200.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/ouro.h"
#include "../../include/ouro/device_view.h"

namespace ouro_host {

struct Geometry {
    uint64_t heap, chunk, minp, maxp;
    uint32_t N, K, page_bits, chunk_bits, chunk_shift, min_shift, Wmax, gen_bits, gmask, cmask;
    uint32_t ppc(uint32_t k) const { return (uint32_t)(chunk >> (min_shift + k)); }
    uint32_t words(uint32_t k) const { return (ppc(k) + 63) / 64; }
    uint64_t page_bytes(uint32_t k) const { return minp << k; }
};

ouro_status geometry(const ouro_config* c, Geometry* g);

}  // namespace ouro_host

struct ouro_heap {
    ouro_config cfg;
    ouro_host::Geometry g;
    int device = 0;
    // device allocations
    uint8_t* d_heap = nullptr;
    ouro_u64* d_meta = nullptr;
    ouro_u64* d_bitmap = nullptr;
    uint32_t* d_assigned = nullptr;
    ouro_queue_dev* d_q = nullptr;
    ouro_u64* d_ctr = nullptr;
    uint32_t* d_sticky = nullptr;
    ouro_u64* d_sm_hint = nullptr;  // per-SM queue hints (256 x 32)
    uint32_t* d_pq = nullptr;      // page kind partition: start[K], n[K], s[K]
    uint8_t* d_touched = nullptr;  // churn reuse bitmap (lazy)
    std::vector<void*> owned;      // slot rings, dirs, dcnts
    // host mirror of the construction plan
    std::vector<ouro_queue_dev> hq;  // 2K+1 queue descriptors as built
    std::vector<uint32_t> pq_start, pq_n, pq_s;
    int64_t floor_F = 0;
    ouro_heap_view view{};
    uint32_t nq = 0;
    // launch shape of this heap's alloc/free/churn launchers (ouro_heap_set_launch_shape)
    int op_block = 256;
    int op_waves = 0;
};
