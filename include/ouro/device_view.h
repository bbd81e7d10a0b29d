/*
 * device_view.h -- POD layout of a heap in HBM, shared by the host library and
 * the header-only device code.  Plain C types only.
 *
 * HBM layout of one heap:
 *   payload      heap_bytes, chunk c at base + c*chunk_bytes
 *   meta[N]      u64 per chunk: {free:32 | state:8 | gen:24}      (ChunkHeader)
 *   bitmap[N*W]  u64 words, 1 = allocated page (SPEC.md:185 with the bit sense
 *                inverted: unassigned / fully free chunks are all-zero)
 *   queues[2K+1] ouro_queue_dev: K class queues, the chunk pool, K private
 *                segment pools (page kind, virtual flavours)
 *   slots        Array-flavour rings, u64 {tag:32 | value:32}
 *   dir / dcnt   VirtualArray directories
 *   assigned[K]  chunk kind: chunks assigned per class (watermark, gap G3)
 *   ctr[]        stats counters; sticky[2] error word
 */
#ifndef OURO_DEVICE_VIEW_H
#define OURO_DEVICE_VIEW_H
#include <stdint.h>

/* CUDA atomics take (unsigned) long long; uint64_t is `unsigned long` on LP64. */
typedef unsigned long long ouro_u64;
typedef long long ouro_i64;

/* Each hot counter sits in its own 1 KiB slot so that count/head/tail of one
 * queue hash to different L2 slices (LTS hash uses address bits 8 and 10+). */
#define OURO_HOT_STRIDE 1024

typedef struct ouro_queue_dev {
    ouro_i64 count;                     /* occupancy reservation counter */
    uint8_t pad0[OURO_HOT_STRIDE - 8];
    ouro_u64 head;                     /* dequeue ticket */
    uint8_t pad1[OURO_HOT_STRIDE - 8];
    ouro_u64 tail;                     /* enqueue ticket */
    uint8_t pad2[OURO_HOT_STRIDE - 8];
    ouro_u64 vl_head;                  /* VirtualList head segment link {seq:32|chunk:32} */
    uint8_t pad3[OURO_HOT_STRIDE - 8];
    ouro_u64 vl_tail;                  /* VirtualList tail segment link */
    uint8_t pad4[OURO_HOT_STRIDE - 8];
    /* cold, read-only after construction */
    ouro_u64 cap;
    ouro_u64 ring_mask;
    uint32_t ring_shift;
    uint32_t flavor;
    uint32_t D;                        /* VirtualArray directory entries */
    int32_t seg_src;                   /* queue index supplying segment chunks */
    ouro_u64* slots;
    ouro_u64* dir;
    uint32_t* dcnt;
    ouro_u64 seg_live;                 /* stats */
    ouro_u64 seg_hwm;
    /* VirtualList lookup accelerator: links {seq:32|chunk:32} of the most
     * recently created segments (creation ring, sized per queue by the host).
     * The list itself stays the source of truth; an entry is used only when its
     * seq matches (a segment cannot retire while a caller still needs it). */
#define OURO_VL_RECENT 256
    ouro_u64* vl_recent;               /* device array of vl_rmask + 1 links at [seq & vl_rmask] */
    ouro_u64 vl_rmask;                 /* ring size - 1: >= 2x the segments in-flight tickets can span */
    ouro_u64 vl_recent_pad[OURO_VL_RECENT - 2];
    /* Dequeue-side accelerator: links of the segments at and ahead of the head at
     * [seq % OURO_VL_RECENT], kept ahead of consumption by the dequeuer that starts
     * each segment (ouro_device.cuh vl_extend_ring); walkers record every hop they
     * validate.  Same rule: used only on a seq match. */
    ouro_u64 vl_deq[OURO_VL_RECENT];
    uint32_t vl_front;                 /* highest seq recorded contiguously in vl_deq */
    uint32_t vl_pad;
    uint8_t pad5[5 * OURO_HOT_STRIDE - 88 - 16 * OURO_VL_RECENT];
} ouro_queue_dev;

/* Counter indices in ctr[] (after 2*K per-class retries/ooms). */
enum {
    OURO_CTR_STALE = 0,
    OURO_CTR_DOUBLE_FREE = 1,
    OURO_CTR_INVALID_FREE = 2,
    OURO_CTR_BAD_SIZE = 3,
    OURO_CTR_TIMEOUT = 4,
    OURO_CTR_CORRUPTION = 5,
    OURO_CTR_POOL_DEQ = 6,
    OURO_CTR_CLAIM_RETRY = 7,   /* chunk-bitmap picks lost to a concurrent holder (retried) */
    OURO_CTR_N = 8
};
/* ctr[] holds OURO_CTR_SHARDS copies of the 2K + OURO_CTR_N counters (by SM). */
#define OURO_CTR_SHARDS 32

typedef struct ouro_heap_view {
    uint8_t* base;
    ouro_u64* meta;
    ouro_u64* bitmap;
    uint32_t* assigned;
    ouro_queue_dev* q;
    ouro_u64* ctr;          /* [0,K) retries, [K,2K) ooms, 2K + OURO_CTR_* */
    uint32_t* sticky;       /* [0] first error, [1] mask */
    ouro_u64 heap_bytes;
    ouro_u64 chunk_bytes;
    ouro_u64 S_va;          /* VirtualArray slots per segment = chunk/8 */
    ouro_u64 S_vl;          /* VirtualList slots per segment = chunk/8 - 2 */
    ouro_i64 floor_F;        /* chunk kind, virtual: pool chunks kept for segments */
    ouro_u64 spin_limit;    /* bounded waits: iterations before TimeoutError */
    uint32_t N, K;
    uint32_t page_bits, chunk_bits, chunk_shift, min_shift;
    uint32_t Wmax, gmask, cmask;
    uint32_t kind, flavor, backoff;
    uint32_t max_retries, sleep_base_ns, sleep_cap_ns;
    uint32_t checks;        /* 1: verify queue/bitmap invariants on every op (debug) */
    /* page kind static partition: class k owns chunks
     * [start_k, start_k + n_k), the first s_k of them segment storage (gap G1);
     * n_0 = pq_n0, n_k = pq_q for k > 0, so decode is arithmetic, not a load. */
    uint32_t pq_n0, pq_q;
    uint32_t pq_s[32];
    /* latest queue observation per (SM, queue tag): 256 x 32 u64 hints (see
     * ouro_device.cuh sm_hint_row); hints only, never a retry round's observation */
    ouro_u64* sm_hint;
} ouro_heap_view;

#endif
