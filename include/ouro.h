/*
 * ouro.h -- C-ABI of the B200-native Ouroboros-style device allocator.
 *
 * This is the drop-in boundary for the reference's allocator API
 * (arXiv 2504.18211 artifact, /root/reference).  Every entry point names the
 * reference interface it replaces.  Paths are relative to /root/reference.
 *
 *   reference (C++20, namespace ouro)                 this ABI
 *   -----------------------------------------------   ---------------------------------
 *   HeapConfig (proj/include/ouro/config.hpp:26-52)   ouro_config (same field order,
 *                                                      same defaults, same 48-byte layout)
 *   HeapConfig::validate (proj/src/config.cpp:16-42)  ouro_config_validate
 *   num_chunks / max_pages_per_chunk (config.hpp:45-51) ouro_config_geometry
 *   variant_name (proj/src/config.cpp:44-52)          ouro_variant_name
 *   variant_from_name (proj/src/config.cpp:54-59)     ouro_variant_from_name
 *   error classes (proj/include/ouro/errors.hpp:11-46) ouro_status codes 1..6
 *   new_arena                         ouro_heap_create
 *   size_class_of                     ouro_size_class (host mirror of the
 *                                                      device routine)
 *   encode/decode_handle, page_region ouro_handle_encode/decode,
 *                                                      ouro_page_region
 *   alloc / dealloc                 ouro_malloc / ouro_free (__device__,
 *                                                      include/ouro_device.cuh) and the
 *                                                      batch launchers below
 *   backoff                         ouro_backoff_ns (mapping) + device
 *   stats                           ouro_heap_stats
 *   alloc_coalesced                 ouro_malloc_coalesced (__device__)
 *   run_trial                       ouro_run_trial
 *   write_and_verify_pattern        ouro_launch_write / ouro_launch_verify
 *
 * Plain C: no CUDA or torch types.  Streams are passed as `void*`
 * (a cudaStream_t; NULL = legacy default stream).  Device pointers are `void*`
 * / `uint64_t*` into device memory and are documented as such.
 */
#ifndef OURO_H
#define OURO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  1..6 are the reference's exception classes
 * (errors.hpp:11-46); 7.. are the SPEC's return values. */
typedef enum ouro_status {
    OURO_OK = 0,
    OURO_ERR_CONFIG = 1,           /* ConfigError         errors.hpp:11 */
    OURO_ERR_INVALID_HANDLE = 2,   /* InvalidHandleError  errors.hpp:17 */
    OURO_ERR_DOUBLE_FREE = 3,      /* DoubleFreeError     errors.hpp:24 */
    OURO_ERR_RANGE = 4,            /* RangeError          errors.hpp:30 */
    OURO_ERR_TIMEOUT = 5,          /* TimeoutError        errors.hpp:36 */
    OURO_ERR_CORRUPTION = 6,       /* CorruptionError     errors.hpp:43 */
    OURO_ERR_OOM = 7,              /* OutOfMemory */
    OURO_ERR_TOO_LARGE = 8,        /* TooLarge            SPEC.md:58 (also size 0, gap G5) */
    OURO_ERR_CUDA = 9,             /* CUDA runtime failure */
    OURO_ERR_FULL = 10,            /* queue Full */
    OURO_ERR_EMPTY = 11,           /* queue Empty */
    OURO_ERR_CHUNK_FULL = 12,      /* ChunkFull */
    OURO_ERR_ALREADY_ASSIGNED = 13,/* AlreadyAssigned */
    OURO_ERR_VERIFICATION = 14,    /* VerificationFailed */
    OURO_ERR_USAGE = 15            /* UsageError */
} ouro_status;

/* QueueFlavor / AllocatorKind / BackoffPolicy, config.hpp:17,21,24. */
enum { OURO_FLAVOR_ARRAY = 0, OURO_FLAVOR_VIRTUAL_ARRAY = 1, OURO_FLAVOR_VIRTUAL_LIST = 2 };
enum { OURO_KIND_PAGE = 0, OURO_KIND_CHUNK = 1 };
enum { OURO_BACKOFF_FENCE = 0, OURO_BACKOFF_SLEEP = 1 };

#define OURO_MAX_CLASSES 32

/* HeapConfig, config.hpp:26-38.  Field order, defaults and layout (48 bytes,
 * align 8) are the reference's, so a HeapConfig can be passed by pointer. */
typedef struct ouro_config {
    uint64_t heap_bytes;      /* default 64 MiB */
    uint64_t chunk_bytes;     /* default 64 KiB */
    uint64_t min_page_bytes;  /* default 16 */
    uint64_t max_page_bytes;  /* default 8192 */
    uint8_t queue_flavor;     /* OURO_FLAVOR_*, default Array */
    uint8_t allocator_kind;   /* OURO_KIND_*, default Page */
    uint8_t backoff;          /* OURO_BACKOFF_*, default FenceRetry */
    uint8_t reserved0;
    uint32_t max_retries;     /* default 64 */
    uint32_t sleep_base_ns;   /* default 100 */
    uint32_t sleep_cap_ns;    /* default 100000 */
} ouro_config;

/* Derived geometry (config.hpp:45-51 plus SPEC.md:48 class table). */
typedef struct ouro_geometry {
    uint32_t num_chunks;         /* heap/chunk                      config.hpp:45-47 */
    uint32_t max_pages_per_chunk;/* chunk/min_page                  config.hpp:49-51 */
    uint32_t num_classes;        /* floor(log2(max/min))+1 */
    uint32_t page_bits;          /* countr_zero(chunk/min)          config.cpp:34 */
    uint32_t chunk_bits;         /* bit_length(num_chunks-1)        config.cpp:35 */
    uint32_t gen_bits;           /* generation bits kept in chunk-queue entries */
    uint32_t bitmap_words;       /* 64-bit bitmap words per chunk header */
    uint32_t reserved0;
} ouro_geometry;

typedef struct ouro_class_stats {
    uint64_t page_bytes;
    uint64_t pages_per_chunk;
    uint64_t chunks;        /* page kind: page chunks of the partition; chunk kind: assigned now */
    uint64_t live_pages;    /* quiescent recount from chunk headers */
    uint64_t queue_len;     /* raw occupancy count of the class queue */
    uint64_t queued_live;   /* entries that are current (stale chunk entries excluded) */
    uint64_t seg_live;      /* virtual flavours: segments currently held */
    uint64_t seg_hwm;       /* segment high-watermark */
    uint64_t retries;       /* lane backoff rounds */
    uint64_t ooms;          /* lanes that got OutOfMemory */
} ouro_class_stats;

typedef struct ouro_stats {
    uint32_t num_classes;
    uint32_t num_chunks;
    uint32_t sticky_first;   /* first device error (ouro_status), 0 if none */
    uint32_t sticky_mask;    /* OR of (1 << status) over every device error */
    uint64_t pool_len;       /* chunk kind: free-chunk pool occupancy */
    uint64_t stale_drops;    /* chunk-queue entries dropped as stale / ChunkFull (gap G4) */
    uint64_t double_frees;
    uint64_t invalid_frees;
    uint64_t bad_sizes;      /* TooLarge / size 0 requests */
    uint64_t timeouts;
    uint64_t corruptions;
    ouro_class_stats cls[OURO_MAX_CLASSES];
} ouro_stats;

/* Canonical quiescent-state digest.  Every field is
 * independent of thread interleaving, so an oracle run and a concurrent GPU run
 * of the same workload must produce identical digests (compare with memcmp). */
typedef struct ouro_digest {
    uint32_t num_chunks;
    uint32_t num_classes;
    uint32_t partition_ok;      /* every chunk in exactly one place, entries unique */
    uint32_t sticky_mask;
    uint64_t live_pages;
    uint64_t unassigned_chunks; /* pool + free segment storage (not page-bearing) */
    uint64_t header_hash;       /* page kind: per-index headers; chunk kind: header multiset w/o gen */
    uint64_t queue_hash;        /* page kind: multiset of queued handles per class; chunk kind: 0 */
    uint64_t class_chunks[OURO_MAX_CLASSES];
    uint64_t class_queued_live[OURO_MAX_CLASSES];
    uint64_t class_live_pages[OURO_MAX_CLASSES];
} ouro_digest;

/* ---------------- configuration (host only, no GPU needed) ---------------- */
ouro_status ouro_config_default(ouro_config* cfg);
/* Same reject set and messages as HeapConfig::validate (config.cpp:16-42). */
ouro_status ouro_config_validate(const ouro_config* cfg, char* msg, size_t msg_len);
/* Geometry of a valid config; OURO_ERR_CONFIG if invalid or unsupported. */
ouro_status ouro_config_geometry(const ouro_config* cfg, ouro_geometry* out);
/* "page","chunk","va-page","va-chunk","vl-page","vl-chunk"; "?" otherwise. */
const char* ouro_variant_name(uint8_t kind, uint8_t flavor);
/* 1 and fills kind/flavor on a match, 0 otherwise. */
int ouro_variant_from_name(const char* name, uint8_t* kind, uint8_t* flavor);
/* size_class_of: class index, or OURO_ERR_TOO_LARGE. */
ouro_status ouro_size_class(const ouro_config* cfg, uint64_t bytes, uint32_t* cls);
ouro_status ouro_handle_encode(const ouro_config* cfg, uint32_t chunk, uint32_t page, uint32_t* h);
ouro_status ouro_handle_decode(const ouro_config* cfg, uint32_t h, uint32_t* chunk, uint32_t* page);
/* backoff: nanoseconds slept for (policy, attempt); 0 = fence only. */
uint64_t ouro_backoff_ns(uint8_t policy, uint32_t attempt, uint32_t base_ns, uint32_t cap_ns);

/* ---------------- heap lifetime (needs a GPU) ---------------- */
typedef struct ouro_heap ouro_heap;
/* new_arena + allocator construction. Host calls are
 * not concurrent per heap; device ops are safe from any thread. */
ouro_status ouro_heap_create(const ouro_config* cfg, int device, ouro_heap** out);
ouro_status ouro_heap_destroy(ouro_heap* heap);
/* Re-initialise the heap to its freshly created state. */
ouro_status ouro_heap_reset(ouro_heap* heap, void* stream);
/* Copy the POD device view (struct ouro_heap_view in ouro_device.cuh). */
ouro_status ouro_heap_get_view(const ouro_heap* heap, void* view_out, size_t view_size);
size_t ouro_heap_view_size(void);
/* Default launch shape of the alloc/free/churn launchers of heaps created later: threads per
 * block (multiple of 32, <= 256); waves: 0 = one thread per request, w >= 1 =
 * persistent grid of w x resident blocks that grid-strides (measured slower,
 * DESIGN.md section 4).  Default 256, 0. */
ouro_status ouro_set_launch_shape(int block_threads, int waves);
/* The same for one heap (launch shape is per heap; new heaps take the process default). */
ouro_status ouro_heap_set_launch_shape(ouro_heap* heap, int block_threads, int waves);
/* Debug mode: verify queue/bitmap invariants on every device op (CorruptionError
 * on mismatch).  Off by default; affects views fetched afterwards. */
ouro_status ouro_heap_set_checks(ouro_heap* heap, int on);
/* Bounded waits (TimeoutError, errors.hpp:35-39): iterations a device wait may
 * spin before raising OURO_ERR_TIMEOUT in the sticky word and failing the
 * operation instead of hanging the GPU.  Default 2^22 (~seconds). */
ouro_status ouro_heap_set_spin_limit(ouro_heap* heap, uint64_t limit);
/* Test-only fault injection: add delta to queue qi's occupancy count (e.g. a
 * count that promises entries no slot holds, so a dequeue must time out). */
ouro_status ouro_heap_debug_add_count(ouro_heap* heap, uint32_t qi, int64_t delta);
ouro_status ouro_heap_config(const ouro_heap* heap, ouro_config* cfg, ouro_geometry* geo);
uint64_t ouro_heap_base(const ouro_heap* heap); /* device address of heap byte 0 */
/* page_region against live device state; InvalidHandle if the
 * chunk is not assigned or the page index is out of range. */
ouro_status ouro_page_region(ouro_heap* heap, uint32_t h, uint64_t* offset, uint64_t* len);
/* stats; exact at quiescence. */
ouro_status ouro_heap_stats(ouro_heap* heap, ouro_stats* out, void* stream);
/* Debug/test: queue qi's {count, head ticket, VirtualList head link, tail link}
 * (links {seq:32|chunk:32}); synchronises the device. */
ouro_status ouro_heap_queue_links(ouro_heap* heap, uint32_t qi, uint64_t out[4]);
/* Debug/test: queue qi's dequeue-side VirtualList ring (256 links). */
ouro_status ouro_heap_vl_ring(ouro_heap* heap, uint32_t qi, uint64_t out[256]);
/* Canonical digest; call at quiescence. */
ouro_status ouro_heap_digest(ouro_heap* heap, ouro_digest* out, void* stream);
/* Sticky device error word; clear != 0 resets it. */
ouro_status ouro_heap_last_error(ouro_heap* heap, uint32_t* first, uint32_t* mask, int clear);

/* ---------------- batch launchers: the paper's driver phases ---------------- */
/* One device thread per slot i < n: d_out[i] = ouro_malloc(size_i)
 * (size_i = d_sizes ? d_sizes[i] : uniform_bytes).  NULL on OOM/TooLarge. */
ouro_status ouro_launch_alloc(ouro_heap* heap, uint64_t n, uint64_t uniform_bytes,
                              const uint32_t* d_sizes, void** d_out, void* stream);
/* Same with 16-bit request sizes (every valid request is <= max_page_bytes <=
 * 65535 B; a request that does not fit 16 bits is TooLarge anyway): half the
 * bytes to move when the request array comes from the host. */
ouro_status ouro_launch_alloc_u16(ouro_heap* heap, uint64_t n, const uint16_t* d_sizes, void** d_out,
                                  void* stream);
/* One device thread per slot: ouro_free(d_ptrs[i]) (NULL slots skipped). */
ouro_status ouro_launch_free(ouro_heap* heap, uint64_t n, void* const* d_ptrs, void* stream);
/* Fill every live page (its full page_region) with the slot/iteration-keyed
 * pattern, one mix per 8-byte word (gap G6). */
ouro_status ouro_launch_write(ouro_heap* heap, uint64_t n, void* const* d_ptrs,
                              uint64_t seed, uint32_t iteration, void* stream);
/* Verify; d_result[0] += mismatching words, d_result[1] = min bad slot (init ~0). */
ouro_status ouro_launch_verify(ouro_heap* heap, uint64_t n, void* const* d_ptrs,
                               uint64_t seed, uint32_t iteration, uint64_t* d_result,
                               void* stream);
/* Count non-NULL pointers into d_count[0] (device u64, accumulated). */
ouro_status ouro_launch_count(ouro_heap* heap, uint64_t n, void* const* d_ptrs,
                              uint64_t* d_count, void* stream);

/* Stop-the-world audit of n live pointers: in-heap, naturally aligned,
 * pairwise disjoint (sort by offset, check neighbours), page bit marked used. */
typedef struct ouro_audit_result {
    uint64_t live;        /* non-NULL pointers audited */
    uint64_t out_of_heap;
    uint64_t misaligned;
    uint64_t overlaps;    /* neighbouring regions that intersect */
    uint64_t not_marked;  /* page whose bitmap bit says free */
    uint64_t bytes;       /* sum of region lengths */
} ouro_audit_result;
ouro_status ouro_audit(ouro_heap* heap, uint64_t n, void* const* d_ptrs,
                       ouro_audit_result* out, void* stream);

/* Mixed churn (BASELINE configs[3]): n threads x rounds; per (t, r):
 * h = splitmix64(seed ^ t<<32 ^ r); if slot holds a page and h&1: free it,
 * else malloc(8 + (h>>1) % 4089) and write its first word.  d_slots (n device
 * pointers, NULL-initialised) persist across calls. */
typedef struct ouro_churn_result {
    uint64_t mallocs_ok;
    uint64_t mallocs_failed;
    uint64_t frees;
    uint64_t reused;     /* mallocs whose page had been handed out before */
    uint64_t check_failures;
} ouro_churn_result;
ouro_status ouro_launch_churn(ouro_heap* heap, uint64_t n, uint32_t round_begin,
                              uint32_t rounds, uint64_t seed, void** d_slots,
                              uint64_t* d_result /* 5 x u64, accumulated */, void* stream);

/* ---------------- single-warp op scripts (parity with the oracle) ----------------
 * A script is nsteps steps; step s has op (0 alloc, 1 free, 2 alloc_coalesced), an active lane
 * mask and one argument per lane.  Alloc: arg = request bytes.  Free: if bit 63
 * is set, arg & ~bit63 is a raw heap offset; otherwise arg = index (s'*32+lane)
 * of an earlier alloc result.  Results: out_offset[s*32+lane] = heap offset or
 * ~0; out_status[s*32+lane] = ouro_status.  Runs on ONE warp, so it is
 * deterministic and must match the oracle bit-exactly. */
typedef struct ouro_script_step {
    uint32_t op;
    uint32_t lane_mask;
    uint64_t arg[32];
} ouro_script_step;
ouro_status ouro_run_script(ouro_heap* heap, const ouro_script_step* steps, uint32_t nsteps,
                            uint64_t* out_offset, int32_t* out_status);

/* ---------------- run_trial, host-facing ---------------- */
typedef struct ouro_trial_config {
    uint64_t num_allocations;
    uint64_t allocation_bytes;   /* uniform size, used when sizes == NULL */
    const uint32_t* sizes;       /* optional HOST array of num_allocations sizes */
    uint32_t iterations;         /* >= 2 */
    uint32_t reserved0;
    uint64_t seed;
} ouro_trial_config;
typedef struct ouro_trial_result {
    double alloc_ms[64];
    double free_ms[64];
    double write_ms[64];
    double verify_ms[64];
    uint32_t iterations;
    uint32_t verified;           /* 1 iff every iteration verified clean */
    uint64_t ok_allocs;          /* successful allocations, summed over iterations */
    uint64_t failed_allocs;
    double mean_all_ms;          /* alloc phase */
    double mean_subsequent_ms;   /* alloc phase, iterations 2..n */
    double mean_subsequent_free_ms;
    uint64_t h2d_bytes;          /* host->device bytes copied per iteration */
    uint64_t d2h_bytes;
} ouro_trial_result;
/* Host buffers in, host results out: copies (sizes H2D, counters D2H) are part
 * of every iteration.  Times are CUDA-event milliseconds per phase. */
ouro_status ouro_run_trial(ouro_heap* heap, const ouro_trial_config* cfg, ouro_trial_result* out);
/* mean_all / mean_subsequent. */
ouro_status ouro_trial_means(const double* ms, uint32_t n, double* mean_all, double* mean_subsequent);

/* ---------------- multi-device driver (BASELINE configs[4]) ----------------
 * One host thread per device, each with its own heap (cfg) in its own HBM, a host
 * barrier before every step; a step runs every size once: alloc kernel of
 * threads_per_device requests, count, free kernel, each timed kernel after an L2
 * flush, CUDA events per device.  No collective: pointers never cross devices.
 * Devices may repeat (several heaps on one device).  Aggregate (weak scaling) =
 * pairs summed over devices / the slowest device's summed alloc + free time.
 * Replaces the paper driver's single-device loop for N GPUs. */
#define OURO_MAX_DEVICES 16
typedef struct ouro_multi_result {
    uint32_t ndev;
    uint32_t verified;            /* 1 iff every device's sticky error word stayed 0 */
    uint64_t pairs_total;         /* successful malloc+free pairs over devices and timed steps */
    double max_ms;                /* max over devices of its summed alloc + free kernel time */
    double pairs_per_s;           /* pairs_total / max_ms */
    double dev_ms[OURO_MAX_DEVICES];
    uint64_t dev_pairs[OURO_MAX_DEVICES];
} ouro_multi_result;
ouro_status ouro_multi_sweep(const ouro_config* cfg, uint32_t ndev, const int* devices,
                             uint64_t threads_per_device, const uint32_t* sizes, uint32_t nsizes,
                             uint32_t warmup, uint32_t steps, ouro_multi_result* out);

/* ---------------- micro-benchmarks for the roofline denominators ---------------- */
/* mode 0: distinct-address 32-bit atomicAdd (one per 32 B sector, coalesced);
 * mode 1: distinct-address 64-bit atomicCAS; mode 2: same-address atomicAdd, one
 * per warp (aggregated); mode 3: same-address atomicAdd from every lane;
 * mode 4: 888 blocks (6 per SM) each issue 256 dependent .relaxed.gpu loads of
 * ONE word -- the retry-round poll of an OOM storm -- and the result is the
 * loads per second of one poller (1 / hot-word latency under that contention).
 * Returns element-ops per second measured with CUDA events. */
ouro_status ouro_atomic_peak(int device, int mode, double* ops_per_s);

const char* ouro_status_name(ouro_status s);
const char* ouro_build_info(void);
/* Retry-machinery event counters of an experiment build compiled with
 * -DOURO_STORM_STATS=1 (all zero in the product build); reset != 0 clears them. */
ouro_status ouro_debug_counters(uint64_t out[32], int reset);

#ifdef __cplusplus
}
#endif
#endif /* OURO_H */
