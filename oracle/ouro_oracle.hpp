// ouro_oracle.hpp -- CPU restatement of the reference allocator (TEST INFRASTRUCTURE).
//
// This is the oracle of the B200 build: a thread-level, std::atomic restatement
// of the SPEC's hot-path modules, written from
//   /root/reference/SPEC.md:17-99    arena     (geometry, size classes, handles, page_region)
//   /root/reference/SPEC.md:101-177  queues    (IndexQueue: Array / VirtualArray / VirtualList)
//   /root/reference/SPEC.md:179-237  chunk     (ChunkHeader bitmap, assign/acquire/release)
//   /root/reference/SPEC.md:239-309  allocators(Page / Chunk variants, backoff, stats)
//   /root/reference/SPEC.md:311-362  coalesce  (active mask, group allocation)
//   /root/reference/SPEC.md:364-430  bench     (run_trial, pattern)
// and the only reference code on the path:
//   /root/reference/proj/include/ouro/config.hpp:26-73, proj/src/config.cpp:16-59
//
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
// load it (libouro_oracle.so via ctypes).  The product library never links it.
//
// Parity status: the reference tree contains no allocator implementation
// (SURVEY.md §0).  The oracle is pinned against (a) the reference's own
// config.cpp compiled into oracle/_ref (validate() reject set, variant names)
// and (b) every SPEC known-answer example (tests/golden/spec_kats.json).
// Parity with upstream Ouroboros CUDA/SYCL is unpinned: that code is not
// vendored and no commit is named.
#pragma once
#include "../include/ouro.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_heap orc_heap;
typedef struct orc_qt orc_qt;

ouro_status orc_config_validate(const ouro_config* cfg, char* msg, size_t msg_len);
ouro_status orc_config_geometry(const ouro_config* cfg, ouro_geometry* out);
const char* orc_variant_name(uint8_t kind, uint8_t flavor);
int orc_variant_from_name(const char* name, uint8_t* kind, uint8_t* flavor);
ouro_status orc_size_class(const ouro_config* cfg, uint64_t bytes, uint32_t* cls);
ouro_status orc_handle_encode(const ouro_config* cfg, uint32_t c, uint32_t p, uint32_t* h);
ouro_status orc_handle_decode(const ouro_config* cfg, uint32_t h, uint32_t* c, uint32_t* p);
uint64_t orc_backoff_ns(uint8_t policy, uint32_t attempt, uint32_t base_ns, uint32_t cap_ns);
uint64_t orc_pattern_word(uint64_t seed, uint64_t slot, uint32_t iteration, uint64_t word);
uint64_t orc_mix64(uint64_t x);

ouro_status orc_heap_create(const ouro_config* cfg, orc_heap** out);
void orc_heap_destroy(orc_heap* h);
ouro_status orc_alloc_group(orc_heap* h, uint32_t n, const uint64_t* sizes, uint64_t* out_off,
                            int32_t* out_status);
ouro_status orc_free_group(orc_heap* h, uint32_t n, const uint64_t* offs, int32_t* out_status);
ouro_status orc_alloc_coalesced(orc_heap* h, uint32_t n, uint64_t bytes, uint64_t* out_off,
                                int32_t* out_status);
ouro_status orc_run_script(orc_heap* h, const ouro_script_step* steps, uint32_t nsteps,
                           uint64_t* out_offset, int32_t* out_status);
ouro_status orc_page_region(orc_heap* h, uint32_t handle, uint64_t* off, uint64_t* len);
ouro_status orc_stats(orc_heap* h, ouro_stats* out);
ouro_status orc_digest(orc_heap* h, ouro_digest* out);
uint64_t orc_queue_ops(orc_heap* h); /* total queue operations (coalescing criterion) */
uint64_t orc_pool_dequeues(orc_heap* h);

/* chunk module ops on a chunk-kind heap */
ouro_status orc_chunk_assign(orc_heap* h, uint32_t c, uint32_t cls, uint32_t* gen);
ouro_status orc_chunk_acquire(orc_heap* h, uint32_t c, uint32_t* page);
ouro_status orc_chunk_release(orc_heap* h, uint32_t c, uint32_t page, uint32_t* occ_after);
ouro_status orc_chunk_unassign(orc_heap* h, uint32_t c);
ouro_status orc_chunk_state(orc_heap* h, uint32_t c, uint32_t* state, uint32_t* free_count,
                            uint32_t* gen, uint64_t* bitmap_popcount);

/* standalone index queue with its own segment pool */
ouro_status orc_qt_new(uint8_t flavor, uint64_t capacity, uint32_t pool_chunks,
                       uint64_t chunk_bytes, orc_qt** out);
void orc_qt_destroy(orc_qt* q);
ouro_status orc_qt_enqueue(orc_qt* q, uint32_t v);
ouro_status orc_qt_dequeue(orc_qt* q, uint32_t* v);
uint64_t orc_qt_len(orc_qt* q);
uint64_t orc_qt_pool_len(orc_qt* q);
uint64_t orc_qt_seg_live(orc_qt* q);
/* P producers each enqueue `per` distinct values (p*per + i), C consumers
 * dequeue until all are delivered; hist[v] counts deliveries.  Returns OK if it
 * completed within timeout. */
ouro_status orc_qt_mt_churn(orc_qt* q, uint32_t producers, uint32_t consumers, uint32_t per,
                            uint32_t* hist, double timeout_s);

/* coalesce: CPU threads as lanes of one LaneGroup.
 * active[i] = 1 active, 0 inactive, -1 never arrives. */
ouro_status orc_active_mask(uint32_t width, const int32_t* active, uint32_t timeout_ms,
                            uint64_t* mask_out);

/* bench on CPU threads: the reference CPU allocator timing.
 * sizes may be NULL (uniform). Per-iteration phase wall-clock times in ms. */
typedef struct orc_trial_out {
    double alloc_ms[64];
    double free_ms[64];
    uint64_t ok_allocs;
    uint64_t failed_allocs;
    uint32_t verified;
    uint32_t threads;
} orc_trial_out;
ouro_status orc_bench_trial(orc_heap* h, uint64_t n, uint64_t bytes, const uint32_t* sizes,
                            uint32_t iterations, uint32_t threads, uint64_t seed,
                            orc_trial_out* out);
/* churn (BASELINE configs[3]) on CPU threads over n slots for `rounds` rounds. */
ouro_status orc_churn(orc_heap* h, uint64_t n, uint32_t round_begin, uint32_t rounds,
                      uint64_t seed, uint32_t threads, uint64_t* slots, ouro_churn_result* out,
                      double* ms);
/* Free every non-~0 offset in slots (single thread, slot order) and reset them. */
ouro_status orc_free_all(orc_heap* h, uint64_t n, uint64_t* slots);
/* n slots in warp groups of `group` lanes in slot order, one thread (the demand
 * of the GPU driver phases); out[i] = offset or ~0; *ok = successes. */
ouro_status orc_alloc_slots(orc_heap* h, uint64_t n, uint64_t bytes, const uint32_t* sizes, uint32_t group,
                            uint64_t* out, uint64_t* ok);
ouro_status orc_free_slots(orc_heap* h, uint64_t n, const uint64_t* offs, uint32_t group);

#ifdef __cplusplus
}
#endif
