// ouro_device.cuh -- in-kernel malloc/free for B200 (sm_100a), header-only.
//
//   #include "ouro_device.cuh"
//   __global__ void k(ouro_heap_view h) { void* p = ouro_malloc(h, 1000); ... ouro_free(h, p); }
//
// Replaces the reference's alloc / dealloc / alloc_coalesced
// for the six variants
// {page, chunk} x {array, virtual-array, virtual-list} (config.hpp:55-69).
// The protocol is the oracle's (oracle/ouro_oracle.cpp); this
// file is its warp-aggregated CUDA form:
//   * every call groups the converged lanes of a warp by size class
//     (ballot/shfl on the leader's class), one leader does the count/ticket
//     atomics for the whole group and broadcasts the ticket base with __shfl;
//   * queue slots are 8-byte {tag, value} words read/written by each lane at
//     ticket base + rank (coalesced: a warp touches 256 contiguous bytes);
//   * chunk bitmaps are claimed cooperatively: each lane scans two 64-bit words
//     (one 128-byte-coalesced pass over a 512 B bitmap), prefix sums by
//     ballot, one fetch-AND per word;
//   * frees aggregate by bitmap word (__match_any_sync + __reduce_or_sync) and
//     by chunk, so a warp freeing 32 neighbouring pages does one fetch-OR and
//     one free-count add.
// Groups inside one warp are served in order of their lowest lane, ranks in
// lane order, which makes a single-warp run deterministic and bit-identical to
// the oracle's group operations.
#ifndef OURO_DEVICE_CUH
#define OURO_DEVICE_CUH

#include <stdint.h>

#include "ouro.h"
#include "ouro/device_view.h"

namespace ouro_dev {

typedef unsigned long long u64;
typedef unsigned int u32;
typedef long long i64;

constexpr u32 NONE = 0xFFFFFFFFu;
constexpr u64 NONE_LINK = ~0ull;
constexpr u32 ST_UNASSIGNED = 0;
constexpr u32 ST_RESERVED = 0xFF;
constexpr int KIND_PAGE = OURO_KIND_PAGE;
constexpr int KIND_CHUNK = OURO_KIND_CHUNK;
constexpr int FL_ARRAY = OURO_FLAVOR_ARRAY;
constexpr int FL_VA = OURO_FLAVOR_VIRTUAL_ARRAY;
constexpr int FL_VL = OURO_FLAVOR_VIRTUAL_LIST;

// ------------------------------------------------------------ primitives ----
__device__ __forceinline__ u32 lane_id() { u32 r; asm volatile("mov.u32 %0, %%laneid;" : "=r"(r)); return r; }
__device__ __forceinline__ u32 lanemask_lt() { u32 r; asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r)); return r; }
__device__ __forceinline__ u32 sm_id() { u32 r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
// Statistics counters are sharded OURO_CTR_SHARDS ways by SM (the host sums the
// shards): OOM storms update them once per warp, and unsharded they would be
// one more same-address RMW chain beside the queue counters.
__device__ __forceinline__ u64* ctr_at(const ouro_heap_view& v, u32 idx) {
    return v.ctr + (u64)(sm_id() % OURO_CTR_SHARDS) * (2 * v.K + OURO_CTR_N) + idx;
}

__device__ __forceinline__ u64 ld_rlx(const u64* p) {
    u64 r; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory"); return r;
}
__device__ __forceinline__ u64 ld_acq(const u64* p) {
    u64 r; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory"); return r;
}
__device__ __forceinline__ u32 ld_acq32(const u32* p) {
    u32 r; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory"); return r;
}
__device__ __forceinline__ u32 ld_rlx32(const u32* p) {
    u32 r; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory"); return r;
}
// Reads of directory entries / segment links / segment headers use ld_rlx,
// not ld.acquire: every such value is the address of the next access (the
// hardware cannot issue that access before the load returns), and publishers
// fence before their release store, so an acquire would only add its
// CCTL.IVALL (an L1 invalidate per lookup -- measured as the dominant stall of
// the virtual-list free path).
__device__ __forceinline__ void ld_rlx_v2(const u64* p, u64& a, u64& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_rlx(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rel(u64* p, u64 v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_zero_v2(u64* p) {
    asm volatile("st.global.v2.u64 [%0], {%1,%1};" :: "l"(p), "l"(0ull) : "memory");
}
__device__ __forceinline__ u64 shfl64(u32 mask, u64 v, u32 src) { return __shfl_sync(mask, v, src); }

// exclusive prefix / total over the lanes of `mask` for values < 256
__device__ __forceinline__ void ballot_scan8(u32 mask, u32 v, u32 lt, u32* pre, u32* tot) {
    u32 p = 0, t = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const u32 bl = __ballot_sync(mask, (v >> b) & 1u);
        p += (u32)__popc(bl & lt) << b;
        t += (u32)__popc(bl) << b;
    }
    *pre = p;
    *tot = t;
}

// Position of the x-th (0-based) set bit of b; b must have more than x set bits.
// (find-nth-set instead of clearing x bits one by one: a requester's page in a
// fresh chunk is up to 31 bits in.  The pick loops in warp_claim stay bit by bit:
// replacing them too cost configs[3]'s chunk churn 9 %.)
__device__ __forceinline__ u32 nth_set64(u64 b, u32 x) {
    const u32 lo = (u32)b, clo = (u32)__popc(lo);
    return x < clo ? __fns(lo, 0, (int)x + 1) : 32u + __fns((u32)(b >> 32), 0, (int)(x - clo) + 1);
}

__device__ __forceinline__ void raise_err(const ouro_heap_view& v, int code) {
    atomicCAS(&v.sticky[0], 0u, (u32)code);
    atomicOr(&v.sticky[1], 1u << code);
    if (code == OURO_ERR_TIMEOUT) atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_TIMEOUT), 1ull);
    if (code == OURO_ERR_CORRUPTION) atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_CORRUPTION), 1ull);
}

// Bounded spin: TimeoutError instead of a hung GPU.
struct Spin {
    u64 n = 0;
    __device__ __forceinline__ bool step(const ouro_heap_view& v) {
        ++n;
        if (n > 16) __nanosleep(n < 4096 ? 32 : 256);
        return n < v.spin_limit;
    }
};

// backoff: FenceRetry = a fence between retries, no sleep --
// the SYCL port's substitute for nanosleep.  The SPEC's extra
// "yield" is for preemptible CPU threads; warps are hardware-scheduled, and
// nanosleep(0) alone measured ~300 cycles per round (tools/round_cost.cu).
// SleepRetry = nanosleep(min(base * 2^attempt, cap)).
// The retry poll is a .relaxed.gpu load of the queue count, served by L2, so it
// observes every other SM's frees without any fence; a device-scope fence
// (fence.sc/acq_rel.gpu -> MEMBAR.GPU + ERRBAR + CCTL.IVALL, measured ~2.5 us
// per round on B200) would only add delay.  The default therefore fences at CTA
// scope (orders this warp's own accesses); build with -DOURO_FENCE_SCOPE_GPU=1
// for the literal device-wide seq-cst fence.
#ifndef OURO_FENCE_SCOPE_GPU
#define OURO_FENCE_SCOPE_GPU 0
#endif
__device__ __forceinline__ void backoff_policy(u32 policy, u32 base_ns, u32 cap_ns, u32 attempt) {
    if (policy == OURO_BACKOFF_SLEEP) {
        u64 ns = attempt >= 40 ? cap_ns : ((u64)base_ns << attempt);
        if (ns > cap_ns) ns = cap_ns;
        __nanosleep((u32)ns);
    } else {
#if OURO_FENCE_SCOPE_GPU
        asm volatile("fence.sc.gpu;" ::: "memory");
#else
        asm volatile("fence.sc.cta;" ::: "memory");
#endif
    }
}
__device__ __forceinline__ void backoff(const ouro_heap_view& v, u32 attempt) {
    backoff_policy(v.backoff, v.sleep_base_ns, v.sleep_cap_ns, attempt);
}

// size_class_of; size 0 rejected like TooLarge (gap G5).
__device__ __forceinline__ bool size_class(const ouro_heap_view& v, u64 req, u32* k) {
    const u64 maxp = 1ull << (v.min_shift + v.K - 1);
    if (req == 0 || req > maxp) return false;
    const u32 lg = req <= 1 ? 0u : (u32)(64 - __clzll((long long)(req - 1)));
    *k = lg > v.min_shift ? lg - v.min_shift : 0u;
    return true;
}

__device__ __forceinline__ u32 m_free(u64 m) { return (u32)m; }
__device__ __forceinline__ u32 m_state(u64 m) { return (u32)(m >> 32) & 0xFFu; }
__device__ __forceinline__ u32 m_gen(u64 m) { return (u32)(m >> 40); }
__device__ __forceinline__ u64 mk_meta(u32 gen, u32 state, u32 fr) {
    return ((u64)(gen & 0xFFFFFFu) << 40) | ((u64)state << 32) | fr;
}
__device__ __forceinline__ u32 ppc_of(const ouro_heap_view& v, u32 k) { return (u32)(v.chunk_bytes >> (v.min_shift + k)); }
__device__ __forceinline__ u32 words_of(const ouro_heap_view& v, u32 k) { return (ppc_of(v, k) + 63u) / 64u; }
__device__ __forceinline__ u64* bm_row(const ouro_heap_view& v, u32 c) { return v.bitmap + (u64)c * v.Wmax; }
__device__ __forceinline__ u64* chunk_words(const ouro_heap_view& v, u32 c) {
    return reinterpret_cast<u64*>(v.base + ((u64)c << v.chunk_shift));
}
__device__ __forceinline__ u32 q_entry(const ouro_heap_view& v, u32 c, u32 gen) {
    return v.chunk_bits >= 32 ? c : (c | ((gen & v.gmask) << v.chunk_bits));
}

// ------------------------------------------------------- count / tickets ----
// Retry rounds.  An OOM storm is ~10^6 lanes x
// max_retries rounds, every round needing its OWN observation of the queue's
// count word -- and same-address loads serialise in one L2 slice.  Within a
// block the rounds share observations through a "pump": the first warp that
// needs one becomes the pump and polls the count back to back (one dependent
// L2 load per round, no shared-memory handshake, no global store on the way),
// publishing each result with a sequence number in a shared-memory entry; the
// block's other retrying warps spin on that entry and take the next result.
// A round accepts only a poll whose sequence is higher than the one its
// previous round used (for the first round: higher than any poll that may have
// been in flight when its failed try returned), so OutOfMemory is declared only
// after max_retries distinct observations, each issued after the previous one
// completed -- a queue that refills while a warp retries is seen by its next
// round.  The pump keeps the role across its own rounds and releases it when
// they end; a waiter that finds no pump takes the role over.  (Measured in
// isolation, tools/storm_probe.cu mode 5: 2^20 threads x 63 rounds in 98 us;
// the earlier design -- every round re-acquired the entry by shared CAS,
// checked %globaltimer windows and published an SM hint to HBM, whose store the
// next round's fence then waited on -- took 229 us for the same storm.)
// Observation entry: [63:32] sequence, [7:3] queue tag, [2] pool empty (pair
// polls), [1] pump active, [0] empty.  Hint entry (first-try hints and
// pre-checks only, never a round's observation): [63:32] issue time
// (globaltimer / 256 ns), [7:3] tag, [0] empty.  Shared memory is not
// initialised for kernels that do not call ouro_block_init, so hints count only
// if their time lies in [now - window, now + kPollSkew], an entry of another
// tag is simply taken over, and a pump that makes no progress for kPumpSteal
// spins is replaced.
constexpr u32 kPollWindow = 32;  // x 256 ns = 8.2 us
constexpr u32 kPollSkew = 2;     // hints written just after we read the clock
constexpr u32 kPumpSteal = 1u << 12;
__device__ __forceinline__ u32 gtime32() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (u32)(t >> 8);
}
__device__ __forceinline__ bool time_recent(u32 now, u64 e, u32 window) {
    return now - (u32)(e >> 32) + kPollSkew < window + kPollSkew;
}
__device__ __forceinline__ u32 e_seq(u64 e) { return (u32)(e >> 32); }
__device__ __forceinline__ u64 mk_entry(u32 hi, u64 tag, u32 flags) { return ((u64)hi << 32) | (tag << 3) | flags; }
// Observation entries also carry [31:12] the run of consecutive empty polls ending
// with this one (saturating): a warp that fell behind its pump can see that every
// poll it skipped found the queue empty as well.
constexpr u32 kStreakMax = 0xFFFFFu;
__device__ __forceinline__ u32 e_streak(u64 e) { return (u32)e >> 12; }
__device__ __forceinline__ u64 mk_obs(u32 seq, u64 tag, u32 flags, u32 streak) {
    return mk_entry(seq, tag, flags) | ((u64)(streak < kStreakMax ? streak : kStreakMax) << 12);
}
// OURO_STORM_STATS=1: per-SM event counters of the retry machinery (experiment
// builds only; read with ouro_debug_counters).
#ifndef OURO_STORM_STATS
#define OURO_STORM_STATS 0
#endif
#if OURO_STORM_STATS
__device__ unsigned long long g_storm_dbg[256 * 32];
#define OURO_DBG(i, x) atomicAdd(&g_storm_dbg[(sm_id() & 255u) * 32u + (i)], (unsigned long long)(x))
#else
#define OURO_DBG(i, x) ((void)0)
#endif
constexpr u64 kPump = 2u;
constexpr u32 kPoolEmpty = 4u;
constexpr u32 kPollEntries = 16;
// How a warp waiting for its block's pump idles between checks (< 0: spins).
#ifndef OURO_POLL_WAIT_NS
#define OURO_POLL_WAIT_NS -1
#endif
__device__ __forceinline__ void poll_wait() {
#if OURO_POLL_WAIT_NS >= 0
    __nanosleep(OURO_POLL_WAIT_NS);
#endif
}
__device__ __forceinline__ u64* poll_cache() {
    __shared__ u64 cache[3 * kPollEntries];  // [0,16) observations, [16,32) hints, [32,48) pair observations
    return cache;
}
// Queue structs are laid out consecutively, so the struct index is a collision-free
// slot for up to 16 consecutive queues (the K class queues and the pool at K <= 15).
__device__ __forceinline__ u64 poll_tag(const ouro_queue_dev* Q) {
    return ((u64)Q / sizeof(ouro_queue_dev)) & 31u;
}
__device__ __forceinline__ u64* poll_slot(u64 tag) { return poll_cache() + (tag & 15); }
__device__ __forceinline__ u64* hint_slot(u64 tag) { return poll_cache() + kPollEntries + (tag & 15); }
// Chunk-kind retry rounds observe the class queue AND the pool: a pair poll
// issues both count loads back to back (one L2 round trip, not two) and its
// entry, keyed by the class queue's tag, holds empty = both empty.  Pair entries
// live in their own slots, so a round never mistakes a class-queue-only
// observation for one that also covered the pool.
__device__ __forceinline__ u64* pair_slot(u64 tag) { return poll_cache() + 2 * kPollEntries + (tag & 15); }
__device__ __forceinline__ bool tag_is(u64 e, u64 tag) { return ((e >> 3) & 31u) == tag; }
__device__ __forceinline__ u64 ld_sh(const u64* p) { return *reinterpret_cast<const volatile u64*>(p); }

// Per-SM hints in HBM (v.sm_hint: 32 entries per SM, hint format): the latest
// observation any block on this SM published for each queue.  ouro_block_init(v)
// seeds a fresh block's hints from them, so the blocks of an OOM storm that
// start after the queue ran dry make their first try a block-combined
// observation instead of an RMW + undo pair per warp.
__device__ __forceinline__ u64* sm_hint_row(const ouro_heap_view& v) {
    return v.sm_hint ? v.sm_hint + (u64)(sm_id() & 255u) * 32u : nullptr;
}
__device__ __forceinline__ void publish_hint(u64* smh, u64 tag, u64 h) {
    *reinterpret_cast<volatile u64*>(hint_slot(tag)) = h;
    if (smh) st_rlx(smh + tag, h);
}

// One poll: empty = (Q.count - floor <= 0) [and, with P, (P.count - pfloor <= 0)
// -> bit kPoolEmpty], both loads issued back to back.
__device__ __forceinline__ u32 poll_load(ouro_queue_dev* Q, i64 floor, ouro_queue_dev* P, i64 pfloor) {
    if (!P) return (i64)ld_rlx((const u64*)&Q->count) - floor <= 0 ? 1u : 0u;
    const i64 cq = (i64)ld_rlx((const u64*)&Q->count);
    const i64 cp = (i64)ld_rlx((const u64*)&P->count);
    const u32 ep = cp - pfloor <= 0 ? 1u : 0u;
    return ((cq - floor <= 0 ? 1u : 0u) & ep) | (ep ? kPoolEmpty : 0u);
}

// The lowest sequence the first round after a failed try may use: above the
// entry's, and above a pump's poll that may have been issued before the try.
// An entry of another queue (or uninitialised memory) is taken over.
__device__ __forceinline__ u32 obs_need(u64* slot, u64 tag) {
    for (;;) {
        const u64 e = ld_sh(slot);
        if (tag_is(e, tag)) return e_seq(e) + 1u + (u32)((e & kPump) >> 1);
        if (atomicCAS(slot, e, mk_entry(0, tag, 0)) == e) return 1u;
    }
}
// One round's observation: a poll with sequence >= *need, taken from this block's
// pump, or made by this warp when no pump is active (it then becomes the pump:
// *pumpv holds the entry it wrote, and its next round polls straight away and
// publishes with a plain store -- waiters only read the entry; a thief that
// replaced a stalled pump is simply overwritten).  Returns the poll's flag bits
// (bit 0 = empty).
__device__ __forceinline__ u32 obs_round(ouro_queue_dev* Q, i64 floor, ouro_queue_dev* P, i64 pfloor, u64* slot,
                                         u64 tag, u32* need, u64* pumpv) {
    if (*pumpv) {
        const u32 fl = poll_load(Q, floor, P, pfloor);
        const u32 s = e_seq(*pumpv) + 1u;
        const u64 nv = mk_obs(s, tag, (u32)kPump | fl, (fl & 1u) ? e_streak(*pumpv) + 1u : 0u);
        *reinterpret_cast<volatile u64*>(slot) = nv;
        *pumpv = nv;
        *need = s + 1u;
        return fl;
    }
    for (;;) {
        const u64 e = ld_sh(slot);
        const bool mine = tag_is(e, tag);
        if (mine && (int)(e_seq(e) - *need) >= 0) {  // another warp's poll, new enough
            *need = e_seq(e) + 1u;
            return (u32)e & (1u | kPoolEmpty);
        }
        if (mine && (e & kPump)) {  // wait for the pump's next publication
            u32 spins = 0;
            while (ld_sh(slot) == e && ++spins < kPumpSteal) poll_wait();
            if (spins < kPumpSteal) continue;
        }
        // no pump (or it stalled): poll, publish, take the role
        const u32 fl = poll_load(Q, floor, P, pfloor);
        const u32 s = mine ? e_seq(e) + 1u : *need;
        const u64 nv = mk_obs(s, tag, (u32)kPump | fl, (fl & 1u) ? (mine && (e & 1u) ? e_streak(e) + 1u : 1u) : 0u);
        *pumpv = atomicCAS(slot, e, nv) == e ? nv : 0;  // lost: someone published first; ours stays private
        *need = s + 1u;
        return fl;
    }
}
__device__ __forceinline__ void obs_release(u64* slot, u64 pumpv) {
    if (pumpv) atomicCAS(slot, pumpv, pumpv & ~kPump);
}
// A single block-combined observation issued after the call (first-try hints,
// pre-checks): bit 0 = empty.
static __device__ __noinline__ u32 observe_once(ouro_queue_dev* Q, i64 floor, u64* smh) {
    OURO_DBG(5, 1);
    const u64 tag = poll_tag(Q);
    u64* slot = poll_slot(tag);
    u32 need = obs_need(slot, tag);
    u64 pumpv = 0;
    const u32 fl = obs_round(Q, floor, nullptr, 0, slot, tag, &need, &pumpv);
    obs_release(slot, pumpv);
    if (pumpv) publish_hint(smh, tag, mk_entry(gtime32(), tag, fl & 1u));
    return fl & 1u;
}

// Pre-check before a reservation RMW (hint: the RMW decides).  One LDS, one
// clock read when this block has a recent observation.
__device__ __forceinline__ bool observed_empty(ouro_queue_dev* Q, i64 floor, u64* smh) {
    const u64 tag = poll_tag(Q);
    const u64 h = ld_sh(hint_slot(tag));
    if (tag_is(h, tag) && time_recent(gtime32(), h, kPollWindow)) return (h & 1u) != 0;
    return observe_once(Q, floor, smh) != 0;
}

// Failed retry rounds on a group leader: backoff, then an
// observation of the class queue (and, for the chunk kind, of the pool) newer than
// the previous round's; stops when one sees work (returns false) or when the
// budget is spent (returns true: OutOfMemory).  *attempt counts rounds as the
// oracle does.  The round loop is ONE out-of-line call with the polls inlined and
// scalar arguments: a call per round made the caller spill its live state to
// local memory around every round.  PAIR (chunk kind) and SLEEP (backoff policy)
// are template parameters so each loop carries only its own code.
#ifndef OURO_PUMP_UNROLL
#define OURO_PUMP_UNROLL 16
#endif
constexpr int kPumpUnroll = OURO_PUMP_UNROLL;
#ifndef OURO_PUMP_PIPELINE
#define OURO_PUMP_PIPELINE 1
#endif
template <bool PAIR, bool SLEEP>
static __device__ __noinline__ u32 fail_rounds_loop(ouro_queue_dev* Q, ouro_queue_dev* P, i64 pfloor, u32 a,
                                                    u32 maxr, u32 base_ns, u32 cap_ns, u64* smh) {
    if (!PAIR) P = nullptr;
    const u64 tag = poll_tag(Q);
    u64* slot = PAIR ? pair_slot(tag) : poll_slot(tag);
    u32 need = obs_need(slot, tag), fl = 1u, seq = 0, streak = 0, extra = 0;
#if OURO_STORM_STATS
    const u64 c0 = clock64();
    const u32 a0 = a;
    OURO_DBG(0, 1);
#endif
    // Waiting rounds: take the pump's polls, or claim the role when there is no pump.
    for (;;) {
        if (++a >= maxr) {
#if OURO_STORM_STATS
            OURO_DBG(1, a - a0);
            OURO_DBG(11, clock64() - c0);
#endif
            return (a << 1) | 1u;
        }
        backoff_policy(SLEEP ? (u32)OURO_BACKOFF_SLEEP : (u32)OURO_BACKOFF_FENCE, base_ns, cap_ns, a);
        // FenceRetry: a round may take a poll the pump made while this warp was
        // still on an earlier round -- each such poll is newer than the previous
        // round's and found the queue empty (streak), so it is this round's
        // observation.  (SleepRetry keeps one poll per round: its sleeps pace it.)
        if (!SLEEP && extra) { --extra; continue; }
        bool claimed = false;
        for (u32 spins = 0;;) {
            const u64 e = ld_sh(slot);
            const bool mine = tag_is(e, tag);
            if (mine && (int)(e_seq(e) - need) >= 0) {  // the pump's poll, new enough
                fl = (u32)e & (1u | kPoolEmpty);
                const u32 avail = e_seq(e) - need;       // older polls this warp skipped
                if (!SLEEP && (fl & 1u) && e_streak(e) > avail) extra = avail;
                need = e_seq(e) + 1u;
                break;
            }
            if (!(mine && (e & kPump) && ++spins < kPumpSteal)) {
                // no pump (or it stalled): claim the role; this round's poll is ours
                seq = mine ? e_seq(e) : need - 1u;
                streak = mine && (e & 1u) ? e_streak(e) : 0u;
                if (atomicCAS(slot, e, mk_obs(seq, tag, (u32)kPump, streak)) == e) { claimed = true; break; }
                spins = 0;
            }
            poll_wait();
        }
        if (claimed) break;
        if (!(fl & 1u)) {
#if OURO_STORM_STATS
            OURO_DBG(1, a - a0);
            OURO_DBG(11, clock64() - c0);
#endif
            return a << 1;
        }
    }
#if OURO_STORM_STATS
    const u32 ap = a;
#endif
    // Pump rounds: poll back to back (this round's poll first).  Unrolled: ptxas
    // puts a YIELD at the head of a loop whose exit depends on a loaded value, and
    // a yield per round cost the pump ~350 cycles with the SM's other warps ready
    // (tools/rounds_probe.cu: 127 -> 78 us for 2^20 threads x 62 rounds).
    // Each round's poll is issued as soon as the previous one returned and failed
    // (and the backoff ran); the previous one is published while the new load is
    // in flight, so the shared-memory store and the entry arithmetic are off the
    // poll-to-poll critical path.  (A poll is still issued only after the previous
    // one completed, and waiters take them in sequence order as before.)
    u32 r;
#if OURO_PUMP_PIPELINE
    u64 p0, p1 = 0;
    p0 = ld_rlx((const u64*)&Q->count);  // this round's poll
    if (PAIR) p1 = ld_rlx((const u64*)&P->count);
#pragma unroll kPumpUnroll
    for (;;) {
        ++seq;
        // The entry this poll gets if it finds the queue empty -- the only case that
        // publishes inside the loop -- does not depend on the loaded value: built
        // while the load is in flight.
        const u64 ob = mk_obs(seq, tag, (u32)kPump | 1u | (PAIR ? kPoolEmpty : 0u), streak + 1u);
        if (PAIR) {
            const u32 ep = (i64)p1 - pfloor <= 0 ? 1u : 0u;
            fl = (((i64)p0 <= 0 ? 1u : 0u) & ep) | (ep ? kPoolEmpty : 0u);
        } else {
            fl = (i64)p0 <= 0 ? 1u : 0u;
        }
        if (!(fl & 1u)) { streak = 0; r = a << 1; break; }
        ++streak;
        if (SLEEP) {
            if (++a >= maxr) { r = (a << 1) | 1u; break; }
            backoff_policy(OURO_BACKOFF_SLEEP, base_ns, cap_ns, a);
            p0 = ld_rlx((const u64*)&Q->count);  // next round's poll ...
            if (PAIR) p1 = ld_rlx((const u64*)&P->count);
        } else {
            // FenceRetry: the fence, then the next round's poll, issued before the
            // budget check (a poll past the budget is simply dropped)
            backoff_policy(OURO_BACKOFF_FENCE, base_ns, cap_ns, a + 1);
            p0 = ld_rlx((const u64*)&Q->count);
            if (PAIR) p1 = ld_rlx((const u64*)&P->count);
            if (++a >= maxr) { r = (a << 1) | 1u; break; }
        }
        *reinterpret_cast<volatile u64*>(slot) = ob;  // ... then this one's entry
    }
#else
    bool first = true;
#pragma unroll kPumpUnroll
    for (;;) {
        if (!first) {
            if (++a >= maxr) { r = (a << 1) | 1u; break; }
            backoff_policy(SLEEP ? (u32)OURO_BACKOFF_SLEEP : (u32)OURO_BACKOFF_FENCE, base_ns, cap_ns, a);
        }
        first = false;
        fl = poll_load(Q, 0, P, pfloor);
        ++seq;
        streak = (fl & 1u) ? streak + 1u : 0u;
        *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, (u32)kPump | fl, streak);
        if (!(fl & 1u)) { r = a << 1; break; }
    }
#endif
    *reinterpret_cast<volatile u64*>(slot) = mk_obs(seq, tag, fl, streak);  // release: the last poll stays readable
#if OURO_STORM_STATS
    OURO_DBG(1, a - a0);
    OURO_DBG(14, a - ap + 1);
    OURO_DBG(11, clock64() - c0);
#endif
    // seed the hints of blocks that start later on this SM (one store per pump term)
    if (PAIR) publish_hint(smh, poll_tag(P), mk_entry(gtime32(), poll_tag(P), (fl & kPoolEmpty) ? 1u : 0u));
    else publish_hint(smh, tag, mk_entry(gtime32(), tag, fl & 1u));
    return r;
}
__device__ __forceinline__ bool fail_rounds(const ouro_heap_view& v, ouro_queue_dev* Q, ouro_queue_dev* P,
                                            i64 pfloor, u32* attempt) {
    const bool sl = v.backoff == OURO_BACKOFF_SLEEP;
    u64* smh = sm_hint_row(v);
    const u32 r = P ? (sl ? fail_rounds_loop<true, true>(Q, P, pfloor, *attempt, v.max_retries, v.sleep_base_ns,
                                                         v.sleep_cap_ns, smh)
                          : fail_rounds_loop<true, false>(Q, P, pfloor, *attempt, v.max_retries, v.sleep_base_ns,
                                                          v.sleep_cap_ns, smh))
                    : (sl ? fail_rounds_loop<false, true>(Q, nullptr, 0, *attempt, v.max_retries, v.sleep_base_ns,
                                                          v.sleep_cap_ns, smh)
                          : fail_rounds_loop<false, false>(Q, nullptr, 0, *attempt, v.max_retries, v.sleep_base_ns,
                                                           v.sleep_cap_ns, smh));
    *attempt = r >> 1;
    return (r & 1u) != 0;
}

// Did this block see the queue empty lately?  A pump active in this block (its
// latest poll) is the freshest evidence, else a hint at most kPollWindow old --
// this block's failed RMWs and pump terms, or seeded from the SM's (block start).
// Then the call's first try fails on that observation instead of an RMW + undo
// pair per warp (the retry rounds that follow each make a fresh observation, so
// OutOfMemory still takes max_retries of them).  With
// OURO_FIRST_TRY_OBSERVE=1 the try is a block-combined poll issued after the call
// began instead (measured: ~3 us per warp at the start of each OOM-storm wave, the
// block's warps polling one after another).
#ifndef OURO_FIRST_TRY_OBSERVE
#define OURO_FIRST_TRY_OBSERVE 0
#endif
#ifndef OURO_HINT_PUMP
#define OURO_HINT_PUMP 1
#endif
#ifndef OURO_POOL_HINT_SKIP
#define OURO_POOL_HINT_SKIP 1  // chunk-kind pool first tries fail on a recent empty hint (0: observe first)
#endif
#ifndef OURO_CQ_CLASS_HINT
#define OURO_CQ_CLASS_HINT 1   // chunk-kind class queue first tries: 0 ignore hints, 1 observe on a hint
#endif
__device__ __forceinline__ bool hint_empty(const ouro_queue_dev* Q) {
    const u64 tag = poll_tag(Q);
#if OURO_HINT_PUMP
    const u64 o = ld_sh(poll_slot(tag));
    if (tag_is(o, tag) && (o & kPump)) return (o & 1u) != 0;
#endif
    const u64 e = ld_sh(hint_slot(tag));
    return tag_is(e, tag) && (e & 1u) && time_recent(gtime32(), e, kPollWindow);
}
// A reservation RMW issued at tick t0 found the queue empty: record the hint.
__device__ __forceinline__ void note_empty(const ouro_queue_dev* Q, u32 t0, u64* smh) {
    const u64 tag = poll_tag(Q);
    publish_hint(smh, tag, mk_entry(t0, tag, 1u));
}

// Count reservation (broker-queue style).
// `precheck`: read the count first and skip the RMW when it is already empty
// (retries and chunk-queue probes); the reservation result is the same either way.
// `combine`: take the pre-check from the block's poll combiner (retry rounds).
// Without precheck the first try goes straight to the RMW unless this block (or,
// through the seeded hints, its SM) saw the queue empty lately: then the try
// starts with a block-combined observation issued after the call began (an OOM
// storm costs one count load per block, not an RMW + undo pair per warp); a
// non-empty answer still goes through the RMW, which decides.
// `hint_skip`: on a recent "empty" hint the try fails without an RMW (page-kind
// class queues, the pool); false: the hint only triggers a fresh block-combined
// observation first (chunk-kind class queues: empty whenever their few entries are
// in transit, so a hint would send served requests to the pool).
__device__ __forceinline__ u32 reserve_deq(const ouro_heap_view& v, ouro_queue_dev* Q, u32 n, i64 floor,
                                           bool precheck = true, bool combine = false, bool hint_skip = true) {
    if (precheck) {
        if (combine) {
            if (observed_empty(Q, floor, sm_hint_row(v))) return 0;
        } else if ((i64)ld_rlx((const u64*)&Q->count) - floor <= 0) {
            return 0;
        }
    } else if ((hint_skip || OURO_CQ_CLASS_HINT) && hint_empty(Q)) {
        if (!hint_skip || OURO_FIRST_TRY_OBSERVE) {
            if (observe_once(Q, floor, sm_hint_row(v))) return 0;
        } else {
            return 0;
        }
    }
    const u32 t0 = gtime32();
    OURO_DBG(7, 1);
    const i64 old = (i64)atomicAdd((u64*)&Q->count, (u64)(-(i64)n));
    const i64 avail = old - floor;
    const u32 got = avail <= 0 ? 0u : (avail >= (i64)n ? n : (u32)avail);
    if (got < n) {
        atomicAdd((u64*)&Q->count, (u64)(n - got));
        note_empty(Q, t0, sm_hint_row(v));
    }
    return got;
}
// An enqueue by this block makes its "empty" hint for Q wrong: drop it, so a first
// try of this block does not fail on it (a single warp that frees and allocates
// again behaves exactly like the oracle's group operations).
__device__ __forceinline__ void clear_hint(const ouro_queue_dev* Q) {
    const u64 tag = poll_tag(Q);
    u64* h = hint_slot(tag);
    if (tag_is(ld_sh(h), tag)) *reinterpret_cast<volatile u64*>(h) = 0;
}
__device__ __forceinline__ bool reserve_enq(ouro_queue_dev* Q, u32 n) {
    clear_hint(Q);
    const i64 old = (i64)atomicAdd((u64*)&Q->count, (u64)n);
    if (old + (i64)n > (i64)Q->cap) { atomicAdd((u64*)&Q->count, (u64)(-(i64)n)); return false; }
    return true;
}

// Enqueue reservation for queues that cannot overflow by construction (page
// queues hold each page at most once -- the bitmap rejects double frees --
// and pools hold each chunk at most once): fire-and-forget add, no round trip.
__device__ __forceinline__ void reserve_enq_nofull(ouro_queue_dev* Q, u32 n) {
    atomicAdd((u64*)&Q->count, (u64)n);
    clear_hint(Q);
}

// Tag of a filled virtual-queue slot: the segment's sequence number (each slot
// of a segment is written once per segment life), so a recycled segment chunk's
// old tags never match: a collision needs the same chunk to serve segments 2^31
// apart.  (A ticket-based tag would collide after 2^31 tickets.)  Empty = 0.
__device__ __forceinline__ u32 vtag_seg(u64 seg) { return ((u32)seg & 0x7FFFFFFFu) | 0x80000000u; }

// ---------------------------------------------------------- Array slots ----
// slot t&mask in round r = t>>shift: tag 2r empty, 2r+1 full.
__device__ __forceinline__ bool arr_put(const ouro_heap_view& v, ouro_queue_dev* Q, u64 t, u32 val) {
    u64* s = Q->slots + (t & Q->ring_mask);
    const u32 r = (u32)(t >> Q->ring_shift);
    Spin sp;
    while ((u32)(ld_rlx(s) >> 32) != 2u * r)
        if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); return false; }
    st_rlx(s, ((u64)(2u * r + 1u) << 32) | val);
    return true;
}
__device__ __forceinline__ bool arr_take(const ouro_heap_view& v, ouro_queue_dev* Q, u64 t, u32* val) {
    u64* s = Q->slots + (t & Q->ring_mask);
    const u32 r = (u32)(t >> Q->ring_shift);
    Spin sp;
    u64 x;
    while ((u32)((x = ld_rlx(s)) >> 32) != 2u * r + 1u)
        if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); return false; }
    *val = (u32)x;
    st_rlx(s, (u64)(2u * r + 2u) << 32);
    return true;
}

// Warp-collective Array enqueue: lanes in `part` (all of one queue) enqueue
// their value in lane order.  Called by every lane of `mask`.
__device__ __forceinline__ bool arr_enqueue(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask,
                                            u32 lane, u32 part, u32 val, bool nofull = false) {
    if (!part) return true;
    const u32 leader = __ffs(part) - 1, n = __popc(part), rank = __popc(part & lanemask_lt());
    u64 t0 = 0;
    u32 ok = 0;
    if (lane == leader) {
        if (nofull) {
            reserve_enq_nofull(Q, n);
            ok = 1;
        } else {
            Spin sp;
            while (!(ok = reserve_enq(Q, n) ? 1u : 0u))
                if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); break; }
        }
        if (ok) t0 = atomicAdd((u64*)&Q->tail, (u64)n);
    }
    ok = __shfl_sync(mask, ok, leader);
    t0 = shfl64(mask, t0, leader);
    if (!ok) return false;
    if ((part >> lane) & 1u) return arr_put(v, Q, t0 + rank, val);
    return true;
}

// Warp-collective Array dequeue for the lanes of `todo`: returns how many were
// served; the `got` lowest-ranked lanes of todo get *val (NONE on timeout).
__device__ __forceinline__ u32 arr_dequeue(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask,
                                           u32 lane, u32 todo, i64 floor, u32* val, bool precheck = true,
                                           bool combine = false, bool hint_skip = true) {
    const u32 leader = __ffs(todo) - 1, n = __popc(todo), rank = __popc(todo & lanemask_lt());
    u32 got = 0;
    u64 t0 = 0;
    if (lane == leader) {
        got = reserve_deq(v, Q, n, floor, precheck, combine, hint_skip);
        if (got) t0 = atomicAdd((u64*)&Q->head, (u64)got);
    }
    got = __shfl_sync(mask, got, leader);
    t0 = shfl64(mask, t0, leader);
    if (((todo >> lane) & 1u) && rank < got) {
        if (!arr_take(v, Q, t0 + rank, val)) *val = NONE;
    }
    return got;
}

__device__ __forceinline__ void seg_count(ouro_queue_dev* Q, int d) {
    if (d > 0) {
        const u64 now = atomicAdd((u64*)&Q->seg_live, 1ull) + 1ull;
        atomicMax((u64*)&Q->seg_hwm, now);
    } else {
        atomicAdd((u64*)&Q->seg_live, (u64)-1ll);
    }
}

// Acquire one segment chunk from the queue's Array source for lane `who`,
// then have every lane of `mask` zero it (16-byte stores).  Returns the chunk
// (broadcast) or NONE after a timeout.
__device__ __forceinline__ u32 seg_acquire_zero(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask,
                                                u32 lane, u32 who) {
    ouro_queue_dev* P = v.q + Q->seg_src;
    u32 c = NONE;
    Spin sp;
    for (u32 attempt = 1;; ++attempt) {
        const u32 got = arr_dequeue(v, P, mask, lane, 1u << who, 0, &c);
        if (got) break;
        u32 more = (lane == who) ? (sp.step(v) ? 1u : 0u) : 0u;
        more = __shfl_sync(mask, more, who);
        if (!more) { if (lane == who) raise_err(v, OURO_ERR_TIMEOUT); return NONE; }
        backoff(v, attempt < 8 ? attempt : 8);
    }
    c = __shfl_sync(mask, c, who);
    if (c == NONE) return NONE;
    // Chunks from the shared chunk pool (chunk kind) held payload, which could
    // look like a filled slot: zero them.  A page kind's private segment pool
    // only ever holds segment chunks (zeroed at heap creation) whose stale slot
    // tags name older segments, so only the header words need resetting (the
    // creators do that).
    if (v.kind == KIND_CHUNK) {
        const u32 L = __popc(mask), li = __popc(mask & lanemask_lt());
        u64* w = chunk_words(v, c);
        const u64 nw = v.chunk_bytes / 8;
        for (u64 i = 2ull * li; i < nw; i += 2ull * L) st_zero_v2(w + i);
        __threadfence();
    }
    __syncwarp(mask);
    return c;
}

// --------------------------------------------------------- VirtualArray ----
__device__ __forceinline__ bool va_find(const ouro_heap_view& v, ouro_queue_dev* Q, u64 s, u32* c) {
    u64* e = Q->dir + (s % Q->D);
    Spin sp;
    for (;;) {
        const u64 x = ld_rlx(e);
        if ((u32)(x >> 32) == (u32)s && (u32)x != NONE) { *c = (u32)x; return true; }
        if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); return false; }
    }
}
__device__ __forceinline__ bool va_create(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask, u32 lane,
                                          u32 who, u64 s) {
    u64* e = Q->dir + (s % Q->D);
    u32 ok = 1;
    if (lane == who) {
        const u64 want = ((u64)(u32)s << 32) | NONE;
        Spin sp;
        while (ld_rlx(e) != want)
            if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); ok = 0; break; }
    }
    ok = __shfl_sync(mask, ok, who);
    if (!ok) return false;
    const u32 c = seg_acquire_zero(v, Q, mask, lane, who);
    if (c == NONE) return false;
    if (lane == who) {
        *reinterpret_cast<volatile u32*>(Q->dcnt + (s % Q->D)) = 0u;
        __threadfence();  // the dequeue count (and a zeroed chunk) before the publication
        st_rlx(e, ((u64)(u32)s << 32) | c);
        seg_count(Q, +1);  // statistics, after the publication that the enqueuers wait for
    }
    __syncwarp(mask);
    return true;
}

// ---------------------------------------------------------- VirtualList ----
__device__ __forceinline__ u32 lseq(u64 l) { return (u32)(l >> 32); }
__device__ __forceinline__ u32 lchk(u64 l) { return (u32)l; }
__device__ __forceinline__ u64 mklink(u64 s, u32 c) { return ((u64)(u32)s << 32) | c; }
__device__ __forceinline__ u32* vl_counter(const ouro_heap_view& v, u32 c) {
    return reinterpret_cast<u32*>(chunk_words(v, c) + 1);
}
// Upper half of header word 1: set once the predecessor links to this segment
// (segment 0 and the prefilled segments start with it set).
__device__ __forceinline__ u32* vl_inflag(const ouro_heap_view& v, u32 c) { return vl_counter(v, c) + 1; }

// Find the chunk of segment s.  First the ring of recently created segments
// (vl_recent, written by each creator as soon as its chunk is ready).
// from_tail (enqueuers, segment creators): the target is the newest segment or
// one being created now, so a ring slot still holding an older segment means
// "not created yet": wait on that slot (waiters of different segments poll
// different lines, not the one tail word the creators update).  Only a target
// older than the ring, or a dequeuer's target, is walked from the head; a walk
// validates every hop against the head so a retired segment is never followed.
__device__ __forceinline__ bool vl_locate(const ouro_heap_view& v, ouro_queue_dev* Q, u64 s, u32* out,
                                          bool from_tail = false) {
    Spin sp;
    for (;;) {
        const u64 r = ld_rlx(&Q->vl_recent[(s) & Q->vl_rmask]);
        const u64 d = from_tail ? NONE_LINK : ld_rlx(&Q->vl_deq[s % OURO_VL_RECENT]);  // issued together
        if (lchk(r) != NONE && lseq(r) == (u32)s) { *out = lchk(r); return true; }
        if (lchk(d) != NONE && lseq(d) == (u32)s) { *out = lchk(d); return true; }
        if (from_tail && (lchk(r) == NONE || (int)((u32)s - lseq(r)) > 0)) {  // creator of s not done yet
            if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); return false; }
            continue;
        }
        const u64 tl = ld_rlx(&Q->vl_tail);
        if (lchk(tl) != NONE && lseq(tl) == (u32)s) { *out = lchk(tl); return true; }
        const u64 h = ld_rlx(&Q->vl_head);
        if (lchk(h) != NONE) {
            u32 i = lseq(h), cur = lchk(h);
            if ((u32)((u32)s - i) >= 0x80000000u) { raise_err(v, OURO_ERR_CORRUPTION); return false; }
            bool ok = true;
            while (i != (u32)s) {
                const u64 nx = ld_rlx(chunk_words(v, cur));
                // The link read is valid iff it names segment i + 1: a link word only
                // ever holds the link to its own segment's successor, and a recycled
                // chunk serves a newer segment (higher seq) or is being zeroed.  The
                // head re-check just stops walks that fell behind.
                if (nx == NONE_LINK || lseq(nx) != i + 1u || (int)(lseq(ld_rlx(&Q->vl_head)) - i) > 0) {
                    ok = false;
                    break;
                }
                cur = lchk(nx);
                ++i;
                if (!from_tail) st_rlx(&Q->vl_deq[i % OURO_VL_RECENT], nx);  // record the hop
            }
            if (ok) { *out = cur; return true; }
        }
        if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); return false; }
    }
}
__device__ __forceinline__ void vl_tail_max(ouro_queue_dev* Q, u64 l) {
    u64 cur = ld_rlx(&Q->vl_tail);
    for (;;) {
        if (lchk(cur) != NONE && (int)(lseq(l) - lseq(cur)) <= 0) return;
        const u64 prev = atomicCAS((u64*)&Q->vl_tail, cur, l);
        if (prev == cur) return;
        cur = prev;
    }
}

// Keep the dequeue-side ring ahead of the dequeuers.  The dequeuer that takes
// the first slot of segment s makes sure segment T = s + OURO_VL_RECENT - kVlSlack
// is recorded: it walks from the frontier (vl_front, the highest seq recorded
// contiguously, advanced with atomicMax -- no CAS loop, racing extenders write
// the same entries) to T, normally one hop.  If the frontier entry is gone (its
// slot recycled) or the head overtook it, the walk restarts at the head link.
// T's slot belonged to segment s - kVlSlack, which only a straggler still needs.
// Each hop's link is read from a segment ahead of the head and validated against
// the head afterwards, as in vl_locate.
constexpr u32 kVlSlack = 128;  // in-flight tickets span a few dozen segments (measured: 32 evicted live entries)
__device__ __forceinline__ void vl_extend_ring(const ouro_heap_view& v, ouro_queue_dev* Q, u32 s) {
    const u32 T = s + OURO_VL_RECENT - kVlSlack;
    const u32 f = *reinterpret_cast<volatile const u32*>(&Q->vl_front);
    if ((int)(f - T) >= 0) return;  // already recorded
    u64 e[4];
#pragma unroll
    for (u32 d = 0; d < 4; ++d) e[d] = ld_rlx(&Q->vl_deq[(f - d) % OURO_VL_RECENT]);
    const u64 h = ld_rlx(&Q->vl_head);
    if (lchk(h) == NONE) return;
    u32 i = lseq(h), cur = lchk(h);
#pragma unroll
    for (u32 d = 0; d < 4; ++d) {  // the frontier entry, or one just below it
        if (lchk(e[d]) != NONE && lseq(e[d]) == f - d && (int)(f - d - lseq(h)) >= 0) {
            i = f - d;
            cur = lchk(e[d]);
            break;
        }
    }
    while (i != T) {
        const u64 nx = ld_rlx(chunk_words(v, cur));
        if (nx == NONE_LINK || lseq(nx) != i + 1u || (int)(lseq(ld_rlx(&Q->vl_head)) - i) > 0) break;
        cur = lchk(nx);
        ++i;
        st_rlx(&Q->vl_deq[i % OURO_VL_RECENT], nx);
    }
    if ((int)(i - f) > 0) {
        __threadfence();  // the recorded entries before the frontier that names them
        atomicMax(&Q->vl_front, i);
    }
}

// Warp-collective retirement, batched: lane l looks at segment head + l (its
// chunk from the dequeue-side ring, lane 0 from the head link), the run of
// retired segments (counter == S'+1, successor linked) from the head moves the
// head with ONE CAS, and the run's chunks go back to the segment source with
// one warp enqueue (in segment order).  Only the CAS winner continues; a loser
// stops.  A segment c completed while the head was behind it is not lost: its
// completer increments c's counter, fences, then reads the head (vl_add); the
// advancer CASes the head, fences, then reads the new head segment's counter
// again (the next loop iteration) -- with both fences seq-cst, at least one
// sees the other's write (store-buffering litmus).  The winner must re-read:
// counters it read BEFORE its CAS may predate a completer that then saw the old
// head and lost its own CAS to ours (that lost wakeup stalled the head and
// starved segment creation under 2^20-thread VLPQ loads).
__device__ __forceinline__ void vl_try_advance(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask,
                                               u32 lane, u32 who) {
    const u32 full = (u32)v.S_vl + 1u;
    const u32 li = __popc(mask & lanemask_lt());
    for (;;) {
        u64 h = 0;
        if (lane == who) h = ld_rlx(&Q->vl_head);
        h = shfl64(mask, h, who);
        if (lchk(h) == NONE) return;
        const u32 seq = lseq(h) + li;
        u32 c = NONE;
        if (li == 0) {
            c = lchk(h);
        } else {
            const u64 e = ld_rlx(&Q->vl_deq[seq % OURO_VL_RECENT]);
            if (lchk(e) != NONE && lseq(e) == seq) c = lchk(e);
        }
        u64 nx = NONE_LINK;
        bool done = false;
        if (c != NONE && ld_rlx32(vl_counter(v, c)) == full) {
            nx = ld_rlx(chunk_words(v, c));
            done = nx != NONE_LINK && lseq(nx) == seq + 1u;
        }
        const u32 notdone = __ballot_sync(mask, !done);
        // run = lanes (in mask order) before the first not-retired one
        u32 run = 0;
        for (u32 m = mask; m; m &= m - 1) {
            if ((notdone >> (__ffs(m) - 1)) & 1u) break;
            ++run;
        }
        if (run == 0) return;
        u32 last = mask;  // the run's last lane: its link is the new head
        for (u32 r = 1; r < run; ++r) last &= last - 1;
        const u32 ll = __ffs(last) - 1;
        const u64 nh = shfl64(mask, nx, ll);
        u32 won = 0;
        if (lane == who) won = atomicCAS((u64*)&Q->vl_head, h, nh) == h ? 1u : 0u;
        if (!__shfl_sync(mask, won, who)) return;
        asm volatile("fence.sc.gpu;" ::: "memory");  // our CAS before every lane's next counter reads
        const u32 part = __ballot_sync(mask, li < run);
        arr_enqueue(v, v.q + Q->seg_src, mask, lane, part, c, true);
        if (lane == who) atomicAdd((u64*)&Q->seg_live, (u64)-(i64)run);
    }
}
// Warp-collective: lanes in `part` add `cnt` to segment `c`'s retire counter
// (one lane per distinct segment); the lowest lane that completed one drives
// the head advance.
__device__ __forceinline__ void vl_add(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask, u32 lane,
                                       bool part, u32 c, u32 cnt) {
    u32 done = 0;
    if (part) done = (atomicAdd(vl_counter(v, c), cnt) + cnt == (u32)v.S_vl + 1u) ? 1u : 0u;
    const u32 dm = __ballot_sync(mask, done);
    if (dm) {
        // every lane: the completers' counter adds before any lane's head / counter reads
        asm volatile("fence.sc.gpu;" ::: "memory");
        vl_try_advance(v, Q, mask, lane, __ffs(dm) - 1);
    }
}
// A published segment's chunk from the creation ring, without waiting: NONE if
// seq s is not in its slot; *newer: the slot already holds a later segment.
__device__ __forceinline__ u32 vl_ring_peek(ouro_queue_dev* Q, u32 s, bool* newer) {
    const u64 r = ld_rlx(&Q->vl_recent[(s) & Q->vl_rmask]);
    *newer = lchk(r) != NONE && (int)(lseq(r) - s) > 0;
    return (lchk(r) != NONE && lseq(r) == s) ? lchk(r) : NONE;
}
// Link segment s-1 (chunk p) to segment s (chunk c); true for the one caller that did.
__device__ __forceinline__ bool vl_link(const ouro_heap_view& v, u32 p, u32 s, u32 c) {
    if (atomicCAS(chunk_words(v, p), NONE_LINK, mklink(s, c)) != NONE_LINK) return false;
    atomicExch(vl_inflag(v, c), 1u);
    return true;
}
// Segment creation without a chain: the creator of s publishes its chunk in the
// creation ring as soon as it is zeroed (the enqueuers of s need only that), then
// links whichever neighbours are already published -- s-1 -> s and s -> s+1.
// Each creator publishes, fences (seq-cst), then reads its neighbours' ring slots,
// so of two adjacent creators at least one sees the other (store-buffering
// litmus); the link word's CAS from NONE_LINK picks the one that links and counts
// the link event on the predecessor's retire counter.  (Linking s into s-1 before
// publishing s made the creations of a burst a serial chain: ~4 us per segment,
// 497 us to free 2^20 16 B pages into 128 new VLPQ segments.)
// A ring slot is reused only once its occupant is linked both ways (or retired),
// so a neighbour missing from the ring because a later segment took its slot is
// already linked to us; with tiny segments (thousands in flight) creators wait
// here for the linking to catch up instead of losing a link.
__device__ __forceinline__ bool vl_create(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask, u32 lane,
                                          u32 who, u64 s) {
    const u32 c = seg_acquire_zero(v, Q, mask, lane, who);
    if (c == NONE) return false;
    u32 back = NONE, fwd = 0, ok = 1;
    u64* slot = &Q->vl_recent[(s) & Q->vl_rmask];
    if (lane == who) {
        st_rlx(chunk_words(v, c), NONE_LINK);
        // retire counter 0, in-link flag set only for segment 0 (no predecessor); the
        // chunk may not have been zeroed
        st_rlx(reinterpret_cast<u64*>(vl_counter(v, c)), s == 0 ? (1ull << 32) : 0ull);
        __threadfence();  // the zeroed chunk and its header before the publication
        Spin sp;
        for (;;) {  // the slot's occupant must be fully linked (or retired) before we take it
            const u64 r = ld_rlx(slot);
            if (lchk(r) == NONE || (int)(lseq(r) - (u32)s) >= 0) break;
            if ((int)(lseq(ld_rlx(&Q->vl_head)) - lseq(r)) > 0) break;  // retired
            if (ld_rlx(chunk_words(v, lchk(r))) != NONE_LINK && ld_rlx32(vl_inflag(v, lchk(r))) != 0) break;
            if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); ok = 0; break; }
        }
    }
    ok = __shfl_sync(mask, ok, who);
    if (!ok) {
        // timed out waiting for the occupant to be linked: do not overwrite it (its
        // link could be lost and the head stall) -- give the chunk back unpublished
        arr_enqueue(v, v.q + Q->seg_src, mask, lane, 1u << who, c, true);
        return false;
    }
    if (lane == who) {
        const u64 me = mklink(s, c);
        if (s == 0) st_rlx(&Q->vl_head, me);
        st_rlx(slot, me);  // publish: wakes the enqueuers of s
        seg_count(Q, +1);
        vl_tail_max(Q, me);
        asm volatile("fence.sc.gpu;" ::: "memory");  // publication before the neighbour reads
        bool newer;
        if (s != 0) {
            const u32 p = vl_ring_peek(Q, (u32)s - 1u, &newer);  // newer: s-1 fully linked already
            if (p != NONE && vl_link(v, p, (u32)s, c)) back = p;
        }
        const u32 n = vl_ring_peek(Q, (u32)s + 1u, &newer);
        if (n != NONE && vl_link(v, c, (u32)s + 1u, n)) fwd = 1;
    }
    back = __shfl_sync(mask, back, who);
    fwd = __shfl_sync(mask, fwd, who);
    if (back != NONE) vl_add(v, Q, mask, lane, lane == who, back, 1u);  // link event of s-1
    if (fwd) vl_add(v, Q, mask, lane, lane == who, c, 1u);              // link event of s
    return true;
}

// ------------------------------------------------- flavour-generic queue ----
template <int FL>
__device__ __forceinline__ u64 seg_slots(const ouro_heap_view& v) { return FL == FL_VA ? v.S_va : v.S_vl; }

// Chunk holding ticket t's segment, located once per distinct segment of the
// group (VirtualList: one walk per group instead of one per lane; VirtualArray:
// one directory read, broadcast).  All lanes of `mask` call it.
template <int FL>
__device__ __forceinline__ u32 group_segment(const ouro_heap_view& v, ouro_queue_dev* Q, u32 mask, u32 lane,
                                             bool part, u64 t, bool from_tail) {
    const u64 s = t / seg_slots<FL>(v);
    const u32 grp = __match_any_sync(mask, part ? s : (~0ull - lane));
    const u32 gl = __ffs(grp) - 1;
    u32 c = NONE;
    if (part && lane == gl) {
        bool ok = FL == FL_VA ? va_find(v, Q, s, &c) : vl_locate(v, Q, s, &c, from_tail);
        if (!ok) c = NONE;
    }
    return __shfl_sync(mask, c, gl);
}
template <int FL>
__device__ __forceinline__ u64* slot_in(const ouro_heap_view& v, u32 c, u64 t) {
    return chunk_words(v, c) + (FL == FL_VA ? t % v.S_va : 2 + t % v.S_vl);
}
template <int FL>
__device__ __forceinline__ bool q_put(const ouro_heap_view& v, ouro_queue_dev* Q, u64 t, u32 val, u32 c) {
    if (FL == FL_ARRAY) return arr_put(v, Q, t, val);
    if (c == NONE) return false;
    st_rlx(slot_in<FL>(v, c, t), ((u64)vtag_seg(t / seg_slots<FL>(v)) << 32) | val);
    return true;
}
template <int FL>
__device__ __forceinline__ bool q_take(const ouro_heap_view& v, ouro_queue_dev* Q, u64 t, u32* val, u32 c) {
    if (FL == FL_ARRAY) return arr_take(v, Q, t, val);
    if (c == NONE) return false;
    u64* s = slot_in<FL>(v, c, t);
    Spin sp;
    u64 x;
    const u32 want = vtag_seg(t / seg_slots<FL>(v));
    while ((u32)((x = ld_rlx(s)) >> 32) != want)
        if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); return false; }
    *val = (u32)x;
    return true;
}

// Warp-collective enqueue of the lanes in `part` into queue `qi` (lane order).
template <int FL>
__device__ __forceinline__ bool q_enqueue(const ouro_heap_view& v, u32 qi, u32 mask, u32 lane, u32 part, u32 val,
                                          bool nofull = false) {
    ouro_queue_dev* Q = v.q + qi;
    if (FL == FL_ARRAY) return arr_enqueue(v, Q, mask, lane, part, val, nofull);
    if (!part) return true;
    const u32 leader = __ffs(part) - 1, n = __popc(part), rank = __popc(part & lanemask_lt());
    u64 t0 = 0;
    u32 ok = 0;
    if (lane == leader) {
        if (nofull) {
            reserve_enq_nofull(Q, n);
            ok = 1;
        } else {
            Spin sp;
            while (!(ok = reserve_enq(Q, n) ? 1u : 0u))
                if (!sp.step(v)) { raise_err(v, OURO_ERR_TIMEOUT); break; }
        }
        if (ok) t0 = atomicAdd((u64*)&Q->tail, (u64)n);
    }
    ok = __shfl_sync(mask, ok, leader);
    t0 = shfl64(mask, t0, leader);
    if (!ok) return false;
    const bool me = (part >> lane) & 1u;
    const u64 t = t0 + rank;
    const u64 S = seg_slots<FL>(v);
    u32 creators = __ballot_sync(mask, me && (t % S) == 0);
    bool good = true;
    while (creators) {  // segment creations in ticket order, whole warp helps
        const u32 cl = __ffs(creators) - 1;
        const u64 s = shfl64(mask, t / S, cl);
        const bool r = FL == FL_VA ? va_create(v, Q, mask, lane, cl, s) : vl_create(v, Q, mask, lane, cl, s);
        good = good && r;
        creators &= creators - 1;
    }
    const u32 c = group_segment<FL>(v, Q, mask, lane, me, t, true);
    if (me) good = q_put<FL>(v, Q, t, val, c) && good;
    return good;
}

// Warp-collective dequeue for the lanes of `todo` (all on queue `qi`).
template <int FL>
__device__ __forceinline__ u32 q_dequeue(const ouro_heap_view& v, u32 qi, u32 mask, u32 lane, u32 todo,
                                         i64 floor, u32* val, bool precheck = true, bool combine = false,
                                         bool hint_skip = true) {
    ouro_queue_dev* Q = v.q + qi;
    if (FL == FL_ARRAY) return arr_dequeue(v, Q, mask, lane, todo, floor, val, precheck, combine, hint_skip);
    const u32 leader = __ffs(todo) - 1, n = __popc(todo), rank = __popc(todo & lanemask_lt());
    u32 got = 0;
    u64 t0 = 0;
    if (lane == leader) {
        got = reserve_deq(v, Q, n, floor, precheck, combine, hint_skip);
        if (got) t0 = atomicAdd((u64*)&Q->head, (u64)got);
    }
    got = __shfl_sync(mask, got, leader);
    t0 = shfl64(mask, t0, leader);
    if (!got) return 0;
    const bool me = ((todo >> lane) & 1u) && rank < got;
    const u64 t = t0 + rank;
    const u32 segc = group_segment<FL>(v, Q, mask, lane, me, t, false);
    bool okt = false;
    if (me) {
        okt = q_take<FL>(v, Q, t, val, segc);
        if (!okt) *val = NONE;
    }
    // consumption bookkeeping per segment (one add per distinct segment)
    const bool part = me && okt;
    if (FL == FL_VA) {
        const u64 s = t / v.S_va;
        const u64 key = part ? s : (~0ull - lane);
        const u32 grp = __match_any_sync(mask, key);
        const u32 gl = __ffs(grp) - 1;
        const u32 cnt = __popc(grp);
        u32 retire = 0, rc = NONE;
        if (part && lane == gl) {
            if (atomicAdd(Q->dcnt + (s % Q->D), cnt) + cnt == (u32)v.S_va) {
                retire = 1;
                rc = (u32)ld_rlx(Q->dir + (s % Q->D));
            }
        }
        const u32 rm = __ballot_sync(mask, retire);
        if (rm) {
            arr_enqueue(v, v.q + Q->seg_src, mask, lane, rm, rc, true);
            if (retire) {
                __threadfence();
                st_rel(Q->dir + (s % Q->D), ((u64)(u32)(s + Q->D) << 32) | NONE);
                seg_count(Q, -1);
            }
        }
    } else {
        const u64 key = part ? (u64)segc : (~0ull - lane);
        const u32 grp = __match_any_sync(mask, key);
        const u32 gl = __ffs(grp) - 1;
        if (part && t % v.S_vl == 0) vl_extend_ring(v, Q, (u32)(t / v.S_vl));  // first slot of a segment
        vl_add(v, Q, mask, lane, part && lane == gl, segc, __popc(grp));
    }
    return got;
}

// Warp-collective: enqueue each participating lane's value into its own
// queue qi, groups served in order of their lowest lane.
template <int FL>
__device__ __forceinline__ void q_enqueue_by_queue(const ouro_heap_view& v, u32 mask, u32 lane, bool part,
                                                   u32 qi, u32 val, bool nofull = false) {
    u32 pending = __ballot_sync(mask, part);
    while (pending) {
        const u32 leader = __ffs(pending) - 1;
        const u32 gq = __shfl_sync(mask, qi, leader);
        const u32 grp = __ballot_sync(mask, part && ((pending >> lane) & 1u) && qi == gq);
        if (!q_enqueue<FL>(v, gq, mask, lane, grp, val, nofull) && ((grp >> lane) & 1u))
            raise_err(v, OURO_ERR_CORRUPTION);
        pending &= ~grp;
    }
}

// ---------------------------------------------------------- chunk bitmap ----
// Claim the `take` lowest free pages (clear bits below ppc) of chunk c
// (lowest free word first, fetch-OR the chosen bits).
// Each lane of `mask` scans two words per window; the requester of rank
// `req` (< take, NONE for others) receives the req-th lowest claimed page.
__device__ __forceinline__ u32 warp_claim(const ouro_heap_view& v, u32 c, u32 k, u32 take, u32 mask,
                                          u32 lane, u32 req) {
    const u32 L = __popc(mask), lt = lanemask_lt(), li = __popc(mask & lt);
    const u32 W = words_of(v, k);
    const u32 ppc = ppc_of(v, k);
    u64* row = bm_row(v, c);
    u32 claimed = 0, page = NONE;
    Spin sp;
    while (claimed < take) {
        for (u32 wb = 0; wb < W && claimed < take; wb += 2 * L) {
            const u32 wi = wb + 2 * li;
            u64 w0 = 0, w1 = 0;
            if (wi + 1 < W) {
                if ((v.Wmax & 1u) == 0) ld_rlx_v2(row + wi, w0, w1);
                else { w0 = ld_rlx(row + wi); w1 = ld_rlx(row + wi + 1); }
            } else if (wi < W) {
                w0 = ld_rlx(row + wi);
            }
            // free = clear bits below ppc
            w0 = wi < W ? (~w0 & (ppc - wi * 64 >= 64 ? ~0ull : ((1ull << (ppc - wi * 64)) - 1ull))) : 0ull;
            w1 = wi + 1 < W ? (~w1 & (ppc - (wi + 1) * 64 >= 64 ? ~0ull : ((1ull << (ppc - (wi + 1) * 64)) - 1ull)))
                            : 0ull;
            const u32 cnt = (u32)(__popcll((long long)w0) + __popcll((long long)w1));
            u32 pre, tot;
            ballot_scan8(mask, cnt, lt, &pre, &tot);
            const u32 need = take - claimed;
            u32 my = pre >= need ? 0u : min(cnt, need - pre);
            u64 p0 = 0, p1 = 0;
            for (u64 b = w0; my && b; b &= b - 1, --my) p0 |= b & (~b + 1);
            for (u64 b = w1; my && b; b &= b - 1, --my) p1 |= b & (~b + 1);
            u64 g0 = 0, g1 = 0;
            if (p0) g0 = ~atomicOr(row + wi, p0) & p0;
            if (p1) g1 = ~atomicOr(row + wi + 1, p1) & p1;
            // A bit another holder took since our load is contention, not corruption:
            // holders reserve on free_count before claiming (cq_alloc), so the bitmap
            // always has enough clear bits for every reservation and a rescan finds them.
            const u32 lost = __ballot_sync(mask, g0 != p0 || g1 != p1);
            if (lost && lane == __ffs(lost) - 1) atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_CLAIM_RETRY), 1ull);
            const u32 gc = (u32)(__popcll((long long)g0) + __popcll((long long)g1));
            u32 gpre, gtot;
            ballot_scan8(mask, gc, lt, &gpre, &gtot);
            u32 owners = __ballot_sync(mask, gc > 0);
            while (owners) {
                const u32 o = __ffs(owners) - 1;
                const u64 ob0 = shfl64(mask, g0, o), ob1 = shfl64(mask, g1, o);
                const u32 opre = __shfl_sync(mask, gpre, o), ow = __shfl_sync(mask, wi, o);
                const u32 n0 = (u32)__popcll((long long)ob0);
                const u32 ocnt = n0 + (u32)__popcll((long long)ob1);
                if (req != NONE && req >= claimed + opre && req < claimed + opre + ocnt) {
                    const u32 x = req - claimed - opre;
                    page = x < n0 ? ow * 64 + nth_set64(ob0, x) : (ow + 1) * 64 + nth_set64(ob1, x - n0);
                }
                owners &= owners - 1;
            }
            claimed += gtot;
        }
        if (claimed < take) {
            u32 more = sp.step(v) ? 1u : 0u;
            more = __shfl_sync(mask, more, __ffs(mask) - 1);
            if (!more) { if (lane == __ffs(mask) - 1) raise_err(v, OURO_ERR_TIMEOUT); break; }
        }
    }
    return page;
}

// ------------------------------------------------------------ allocators ----
// Page kind, class group `gm` (SPEC.md:258-262 + 335-339).
template <int FL>
__device__ __forceinline__ void pq_alloc(const ouro_heap_view& v, u32 k, u32 gm, u32 mask, u32 lane,
                                         void** res, int* st) {
    u32 todo = gm, attempt = 0;
    const u32 lt = lanemask_lt();
    const u32 gl0 = __ffs(gm) - 1;
    u64 retries = 0;
#if OURO_STORM_STATS
    const u64 tp0 = clock64();
    u64 tp1 = 0, tp2 = 0;
#endif
    while (todo) {
        const u32 rank = __popc(todo & lt);
        u32 h = NONE;
        // retry tries follow a poll that saw the queue non-empty: straight to the RMW
        const u32 got = q_dequeue<FL>(v, k, mask, lane, todo, 0, &h, false, false);
        const bool mine = ((todo >> lane) & 1u) && rank < got;
        bool ok = mine && h != NONE;
        u32 c = 0, p = 0;
        if (ok) {
            c = h >> v.page_bits;
            p = h & ((1u << v.page_bits) - 1u);
        }
        if (got) {
            // clear the page bits, one fetch-AND per distinct word
            u64* wp = bm_row(v, c) + (p >> 6);
            const u64 bit = ok ? (1ull << (p & 63)) : 0ull;
            const u32 grp = __match_any_sync(mask, ok ? (u64)wp : (~0ull - lane));
            const u32 lo = __reduce_or_sync(grp, (u32)bit), hi = __reduce_or_sync(grp, (u32)(bit >> 32));
            const u64 bits = ((u64)hi << 32) | lo;
            const u32 gl = __ffs(grp) - 1;
            if (ok && lane == gl) {  // mark the pages allocated
                if (v.checks) {
                    const u64 old = atomicOr(wp, bits);
                    if (old & bits) raise_err(v, OURO_ERR_CORRUPTION);
                } else {
                    atomicOr(wp, bits);  // result unused: RED
                }
            }
            // free_count -= pages taken, one add per distinct chunk
            const u32 cg = __match_any_sync(mask, ok ? (u64)c : (~0ull - lane));
            if (ok && lane == __ffs(cg) - 1) atomicAdd(v.meta + c, (u64)(-(i64)__popc(cg)));
            if (mine) {
                if (ok) { *res = v.base + ((u64)c << v.chunk_shift) + ((u64)p << (v.min_shift + k)); *st = OURO_OK; }
                else *st = OURO_ERR_TIMEOUT;
            }
        }
        todo &= ~__ballot_sync(mask, mine);
        if (!todo) break;
        // Failed try.  Further failed rounds run on the leader alone: backoff,
        // then the block-combined poll; the full reservation is retried only
        // when a poll says the queue is non-empty.  Round accounting is the
        // oracle's (one failed try per round, OOM after max_retries).
        const u32 leader = __ffs(todo) - 1, rem = __popc(todo);
        u32 a = attempt, oom = 0;
#if OURO_STORM_STATS
        if (!tp1) tp1 = clock64();
#endif
        if (lane == leader) oom = fail_rounds(v, v.q + k, nullptr, 0, &a) ? 1u : 0u;
#if OURO_STORM_STATS
        tp2 = clock64();
#endif
        a = __shfl_sync(mask, a, leader);
        oom = __shfl_sync(mask, oom, leader);
        retries += (u64)rem * (a - attempt);
        attempt = a;
        if (oom) {
            if (lane == gl0) atomicAdd(ctr_at(v, v.K + k), (u64)rem);
            if ((todo >> lane) & 1u) *st = OURO_ERR_OOM;
            break;
        }
    }
    if (retries && lane == gl0) atomicAdd(ctr_at(v, k), retries);  // one update per call, not per round
#if OURO_STORM_STATS
    if (lane == gl0 && tp1) {
        OURO_DBG(16, 1);
        OURO_DBG(17, tp1 - tp0);
        OURO_DBG(18, tp2 - tp1);
        OURO_DBG(19, clock64() - tp2);
    }
#endif
}

#ifndef OURO_CQ_SKIP_CLASS
#define OURO_CQ_SKIP_CLASS 1
#endif
// Chunk kind, class group `gm` (SPEC.md:261, 299, 206 + G4, 193-197).
template <int FL>
__device__ __forceinline__ void cq_alloc(const ouro_heap_view& v, u32 k, u32 gm, u32 mask, u32 lane,
                                         void** res, int* st) {
    u32 todo = gm, attempt = 0;
    const u32 lt = lanemask_lt();
    const u32 ppc = ppc_of(v, k);
    const u32 pool = v.K;
    const u32 gl0 = __ffs(gm) - 1;
    u64 retries = 0;
#if OURO_STORM_STATS
    // per-call timeline of the leader (tools/cq_stats.py)
    const long long tc0 = clock64();
    long long tc = tc0;
    auto lap = [&](int i) { const long long x = clock64(); if (lane == gl0) OURO_DBG(i, x - tc); tc = x; };
    if (lane == gl0) OURO_DBG(25, 1);
#else
    auto lap = [](int) {};
#endif
    // Set after this call found the class queue empty and then used up a whole pool
    // chunk (nothing enqueued): its next pages come from the pool without another
    // class-queue try (classes with fewer pages per chunk than lanes -- 8 KiB: 4
    // pool chunks per warp -- otherwise pay a class-queue observation per chunk).
    // A warp alone sees exactly what the try would have seen (an empty queue); a
    // dry pool sends it back to the class queue before any retry round.
    bool skip_class = false;
    while (todo) {
        const u32 n = __popc(todo), rank = __popc(todo & lt), leader = __ffs(todo) - 1;
        const bool intodo = (todo >> lane) & 1u;
        u32 e = NONE;
        u32 got = 0;
        if (!OURO_CQ_SKIP_CLASS || !skip_class) {
            // first try: straight to the RMW unless this block saw the queue empty (hinted)
            got = q_dequeue<FL>(v, k, mask, lane, 1u << leader, 0, &e, attempt > 0, attempt > 0, false);
            e = __shfl_sync(mask, e, leader);
        }
        lap(26);
        if (got && e != NONE) {
            const u32 c = e & v.cmask;
            const u32 glow = v.chunk_bits >= 32 ? 0u : (e >> v.chunk_bits);
            u32 take = 0, oldfree = 0;
            if (lane == leader) {
                u64 m = ld_rlx(v.meta + c);
                for (;;) {
                    if (m_state(m) != k + 1 || (m_gen(m) & v.gmask) != glow || m_free(m) == 0) break;
                    const u32 f = m_free(m);
                    const u32 t = min(n, f);
                    const u64 prev = atomicCAS(v.meta + c, m, m - t);
                    if (prev == m) { take = t; oldfree = f; break; }
                    m = prev;
                }
                if (!take) atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_STALE), 1ull);
            }
            take = __shfl_sync(mask, take, leader);
            oldfree = __shfl_sync(mask, oldfree, leader);
            lap(27);
            if (!take) continue;
            const u32 page = warp_claim(v, c, k, take, mask, lane, (intodo && rank < take) ? rank : NONE);
            lap(28);
            // in-transit rule: the holder puts its entry back.  It cannot
            // overflow the queue -- our own dequeue freed a ring position and its count
            // -- so the count update is a fire-and-forget add instead of a
            // capacity-checked RMW round trip.  (Putting it back before the claim, so
            // other warps can claim in the chunk meanwhile, measured ~2 % slower.)
            q_enqueue<FL>(v, k, mask, lane, (oldfree - take > 0) ? (1u << leader) : 0u, e, true);
            lap(29);
            if (intodo && rank < take) {
                if (page != NONE) {
                    *res = v.base + ((u64)c << v.chunk_shift) + ((u64)page << (v.min_shift + k));
                    *st = OURO_OK;
                } else {
                    *st = OURO_ERR_CORRUPTION;
                }
            }
            todo &= ~__ballot_sync(mask, intodo && rank < take);
            continue;
        }
        u32 c = NONE;
        got = arr_dequeue(v, v.q + pool, mask, lane, 1u << leader, v.floor_F, &c, attempt > 0, attempt > 0,
                          OURO_POOL_HINT_SKIP);
        c = __shfl_sync(mask, c, leader);
        if (got && c != NONE) {
#if OURO_STORM_STATS
            if (lane == gl0) OURO_DBG(30, 1);
#endif
            const u32 take = min(n, ppc);
            u64 m = 0;
            if (lane == leader) {
                atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_POOL_DEQ), 1ull);
                m = ld_rlx(v.meta + c);
            }
            m = shfl64(mask, m, leader);
            if (m_state(m) != ST_UNASSIGNED) {
                if (lane == leader) raise_err(v, OURO_ERR_CORRUPTION);
                continue;
            }
            const u32 gen = (m_gen(m) + 1u) & 0xFFFFFFu;
            // chunk_assign fused with taking pages 0..take-1.  A pool chunk's bitmap
            // is all-zero (all free), so one fetch-OR marks the taken pages; the
            // header is published with an exchange issued only after that RMW has
            // returned (control dependency: both performed at L2, in order), and the
            // entry is enqueued after the exchange returned -- no device fence.
            if (lane == leader) {
                const u64 tb = (take >= 64) ? ~0ull : ((1ull << take) - 1ull);
                if (atomicOr(bm_row(v, c), tb) & tb) raise_err(v, OURO_ERR_CORRUPTION);
                const u64 prev = atomicExch(v.meta + c, mk_meta(gen, k + 1, ppc - take));
                if (m_state(prev) != ST_UNASSIGNED) raise_err(v, OURO_ERR_CORRUPTION);
                atomicAdd(v.assigned + k, 1u);
            }
            __syncwarp(mask);
            q_enqueue<FL>(v, k, mask, lane, (ppc - take > 0) ? (1u << leader) : 0u, q_entry(v, c, gen));
            skip_class = ppc == take;
            if (intodo && rank < take) {
                *res = v.base + ((u64)c << v.chunk_shift) + ((u64)rank << (v.min_shift + k));
                *st = OURO_OK;
            }
            todo &= ~__ballot_sync(mask, intodo && rank < take);
            continue;
        }
        if (skip_class) {  // the pool ran dry: the class queue first, then the retry rounds
            skip_class = false;
            continue;
        }
        // both empty: failed rounds on the leader alone until a poll sees work
        u32 a = attempt, oom = 0;
        if (lane == leader) oom = fail_rounds(v, v.q + k, v.q + pool, v.floor_F, &a) ? 1u : 0u;
        a = __shfl_sync(mask, a, leader);
        oom = __shfl_sync(mask, oom, leader);
        retries += (u64)n * (a - attempt);
        attempt = a;
        if (oom) {
            if (lane == leader) atomicAdd(ctr_at(v, v.K + k), (u64)n);
            if (intodo) *st = OURO_ERR_OOM;
            break;
        }
    }
#if OURO_STORM_STATS
    if (lane == gl0) OURO_DBG(31, clock64() - tc0);
#endif
    if (retries && lane == gl0) atomicAdd(ctr_at(v, k), retries);
}

// malloc for the converged lanes of the calling warp.
// `mask_hint`: the lanes the caller knows are calling together (0 = use
// __activemask(), which only sees the lanes that happen to be converged).
template <int KIND, int FL>
__device__ __forceinline__ void* malloc_impl(const ouro_heap_view& v, u64 bytes, int* status, u32 mask_hint = 0) {
    const u32 mask = mask_hint ? mask_hint : __activemask();
    if (mask_hint) __syncwarp(mask);
    const u32 lane = lane_id();
    u32 k = 0;
    const bool valid = size_class(v, bytes, &k);
    void* res = nullptr;
    int st = valid ? OURO_ERR_OOM : OURO_ERR_TOO_LARGE;
    const u32 bad = __ballot_sync(mask, !valid);
    if (bad && lane == (u32)(__ffs(bad) - 1)) atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_BAD_SIZE), (u64)__popc(bad));
    u32 pending = __ballot_sync(mask, valid);
    while (pending) {
        const u32 leader = __ffs(pending) - 1;
        const u32 gk = __shfl_sync(mask, k, leader);
        const u32 gm = __ballot_sync(mask, valid && ((pending >> lane) & 1u) && k == gk);
        if (KIND == KIND_PAGE) pq_alloc<FL>(v, gk, gm, mask, lane, &res, &st);
        else cq_alloc<FL>(v, gk, gm, mask, lane, &res, &st);
        pending &= ~gm;
    }
    if (status) *status = st;
    return res;
}

// free for the converged lanes of the calling warp.
template <int KIND, int FL>
__device__ __forceinline__ int free_impl(const ouro_heap_view& v, void* ptr, u32 mask_hint = 0) {
    const u32 mask = mask_hint ? mask_hint : __activemask();
    if (mask_hint) __syncwarp(mask);
    if (!__ballot_sync(mask, ptr != nullptr)) return OURO_OK;  // free(NULL) for the whole group: no-op
    const u32 lane = lane_id();
    const u32 lt = lanemask_lt();
    int st = OURO_OK;
    bool valid = false;
    u32 c = 0, k = 0, pi = 0;
    u64 off = 0;
    if (ptr != nullptr) {
        off = (u64)((uint8_t*)ptr - v.base);
        if (off >= v.heap_bytes) {
            st = OURO_ERR_INVALID_HANDLE;
        } else {
            c = (u32)(off >> v.chunk_shift);
            u32 s8;
            if (KIND == KIND_PAGE) {
                // static partition: class and Reserved-ness are arithmetic (no meta load)
                const u32 kk = c < v.pq_n0 ? 0u : 1u + (c - v.pq_n0) / v.pq_q;
                const u32 start = kk == 0 ? 0u : v.pq_n0 + (kk - 1) * v.pq_q;
                s8 = (kk >= v.K) ? 0u : ((c - start < v.pq_s[kk]) ? ST_RESERVED : kk + 1);
            } else {
                s8 = m_state(ld_rlx(v.meta + c));
            }
            if (s8 == ST_UNASSIGNED || s8 == ST_RESERVED || s8 > v.K) {
                st = OURO_ERR_INVALID_HANDLE;
            } else {
                k = s8 - 1;
                const u64 in = off & (v.chunk_bytes - 1);
                if (in & ((1ull << (v.min_shift + k)) - 1)) st = OURO_ERR_INVALID_HANDLE;
                else { pi = (u32)(in >> (v.min_shift + k)); valid = true; }
            }
        }
    }
    // duplicates inside the group: all but the lowest lane are double frees
    {
        const u32 same = __match_any_sync(mask, valid ? off : (~0ull - lane));
        if (valid && (same & lt)) { valid = false; st = OURO_ERR_DOUBLE_FREE; }
    }
    // clear the allocated bits, one fetch-AND per distinct word (bit already clear => DoubleFree)
    {
        u64* wp = bm_row(v, c) + (pi >> 6);
        const u64 bit = valid ? (1ull << (pi & 63)) : 0ull;
        const u32 grp = __match_any_sync(mask, valid ? (u64)wp : (~0ull - lane));
        const u32 lo = __reduce_or_sync(grp, (u32)bit), hi = __reduce_or_sync(grp, (u32)(bit >> 32));
        const u32 gl = __ffs(grp) - 1;
        u64 old = 0;
        if (valid && lane == gl) old = atomicAnd(wp, ~(((u64)hi << 32) | lo));
        old = shfl64(mask, old, gl);
        if (valid && !(old & bit)) { valid = false; st = OURO_ERR_DOUBLE_FREE; }
    }
    {
        const u32 nd = __ballot_sync(mask, st == OURO_ERR_DOUBLE_FREE);
        const u32 ni = __ballot_sync(mask, st == OURO_ERR_INVALID_HANDLE);
        if (nd && lane == (u32)(__ffs(nd) - 1)) {
            atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_DOUBLE_FREE), (u64)__popc(nd));
            raise_err(v, OURO_ERR_DOUBLE_FREE);
        }
        if (ni && lane == (u32)(__ffs(ni) - 1)) {
            atomicAdd(ctr_at(v, 2 * v.K + OURO_CTR_INVALID_FREE), (u64)__popc(ni));
            raise_err(v, OURO_ERR_INVALID_HANDLE);
        }
    }
    // free_count += pages released, one add per distinct chunk
    const u32 cg = __match_any_sync(mask, valid ? (u64)c : (~0ull - lane));
    const u32 cgl = __ffs(cg) - 1;
    const bool cl = valid && lane == cgl;
    u64 oldm = 0;
    if (KIND == KIND_CHUNK) {
        if (cl) oldm = atomicAdd(v.meta + c, (u64)__popc(cg));
    } else {
        if (cl) atomicAdd(v.meta + c, (u64)__popc(cg));  // result unused: fire-and-forget RED
    }
    const u32 oldfree = m_free(oldm), newfree = oldfree + (u32)__popc(cg), gen = m_gen(oldm);
    if (KIND == KIND_CHUNK) {
        const u32 ppc = ppc_of(v, k);
        const bool closer = cl && newfree == ppc;
        // watermark (gap G3): per class, min(#closers, assigned-1) may close
        const u32 g2 = __match_any_sync(mask, closer ? (u64)k : (~0ull - lane));
        const u32 g2l = __ffs(g2) - 1, r2 = __popc(g2 & lt);
        u32 take = 0;
        if (closer && lane == g2l) {
            // take = min(want, assigned - 1) atomically: fetch-sub then give back
            // the excess (no CAS loop; equivalent, since a closer that over-asks
            // leaves exactly one chunk and concurrent closers could get none anyway)
            const u32 want = __popc(g2);
            const u32 old = atomicSub(v.assigned + k, want);
            take = old > 1 ? min(want, old - 1) : 0u;
            if (want - take) atomicAdd(v.assigned + k, want - take);
        }
        take = __shfl_sync(mask, take, g2l);
        bool closed = false;
        if (closer && r2 < take) {
            const u64 expect = mk_meta(gen, k + 1, ppc);
            if (atomicCAS(v.meta + c, expect, mk_meta(gen, ST_UNASSIGNED, 0)) == expect) closed = true;
            else atomicAdd(v.assigned + k, 1u);
        }
        // a fully free chunk's bitmap is already all-zero: return it to the pool
        // right after its close CAS returned
        const u32 cm = __ballot_sync(mask, closed);
        if (cm) arr_enqueue(v, v.q + v.K, mask, lane, cm, c, true);
        // 0 -> >0: the releaser re-enqueues the chunk
        q_enqueue_by_queue<FL>(v, mask, lane, cl && oldfree == 0 && !closed, k, q_entry(v, c, gen));
    } else {
        q_enqueue_by_queue<FL>(v, mask, lane, valid, k, (c << v.page_bits) | pi, true);
    }
    return st;
}

// all-or-nothing group allocation (alloc_coalesced)
template <int KIND, int FL>
__device__ __forceinline__ void* malloc_coalesced_impl(const ouro_heap_view& v, u64 bytes, int* status,
                                                       u32 mask_hint = 0) {
    const u32 mask = mask_hint ? mask_hint : __activemask();
    int st;
    void* p = malloc_impl<KIND, FL>(v, bytes, &st, mask);
    const u32 fails = __ballot_sync(mask, st != OURO_OK);
    if (fails) {
        const bool tl = __shfl_sync(mask, st, __ffs(mask) - 1) == OURO_ERR_TOO_LARGE;
        const u32 rb = __ballot_sync(mask, p != nullptr);
        if (p) free_impl<KIND, FL>(v, p, rb);  // roll back partial grants
        __syncwarp(mask);
        p = nullptr;
        st = tl ? OURO_ERR_TOO_LARGE : OURO_ERR_OOM;
    }
    if (status) *status = st;
    return p;
}

}  // namespace ouro_dev

// ---------------------------------------------------------------- public ----
// Block-level allocator state.  ouro_block_init(), called by EVERY thread of the
// block before any allocator call of the block, clears the block's retry-poll
// cache ("poll combining" above).  Optional -- entries are validated by queue
// tag and time -- but it keeps a block from reusing an observation another
// kernel left in shared memory.  The C-ABI launchers call it.
__device__ __forceinline__ void ouro_block_init() {
    const unsigned t = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const unsigned nt = blockDim.x * blockDim.y * blockDim.z;
    for (unsigned i = t; i < 3 * ouro_dev::kPollEntries; i += nt) ouro_dev::poll_cache()[i] = 0;
    __syncthreads();
}
// Same, and seed the block's hints from the latest observations other blocks on
// this SM published for heap `h` (one L2 load per hint entry, at block start).
__device__ __forceinline__ void ouro_block_init(const ouro_heap_view& h) {
    using namespace ouro_dev;
    const unsigned t = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const unsigned nt = blockDim.x * blockDim.y * blockDim.z;
    u64* cache = poll_cache();
    for (unsigned i = t; i < 3 * kPollEntries; i += nt) cache[i] = 0;
    __syncthreads();
    const u64* row = sm_hint_row(h);
    if (row) {
        // Chunk kind: only the pool's hint.  A chunk class queue is empty whenever
        // its few entries are in transit, so a seeded "empty" would
        // send served requests to the pool with an older observation.
        const u64 pool_tag = poll_tag(h.q + h.K);
        const u32 now = gtime32();
        for (unsigned i = t; i < 32; i += nt) {
            if (h.kind == KIND_CHUNK && i != pool_tag) continue;
            const u64 e = ld_rlx(row + i);
            // entry of queue tag i, recent: may go to the hint slot (tags i and i+16 share one)
            if (tag_is(e, i) && time_recent(now, e, 4 * kPollWindow)) cache[kPollEntries + (i & 15)] = e;
        }
    }
    __syncthreads();
}

// Compile-time variant entry points (fastest: no dispatch).
// `lanes`: optional mask of the lanes of this warp that make the call together
// (all of them must pass the same mask); 0 = whatever __activemask() reports.
template <int KIND, int FLAVOR>
__device__ __forceinline__ void* ouro_malloc_t(const ouro_heap_view& h, size_t bytes, int* status = nullptr,
                                               unsigned lanes = 0) {
    return ouro_dev::malloc_impl<KIND, FLAVOR>(h, (unsigned long long)bytes, status, lanes);
}
template <int KIND, int FLAVOR>
__device__ __forceinline__ int ouro_free_t(const ouro_heap_view& h, void* p, unsigned lanes = 0) {
    return ouro_dev::free_impl<KIND, FLAVOR>(h, p, lanes);
}
template <int KIND, int FLAVOR>
__device__ __forceinline__ void* ouro_malloc_coalesced_t(const ouro_heap_view& h, size_t bytes, int* status = nullptr,
                                                         unsigned lanes = 0) {
    return ouro_dev::malloc_coalesced_impl<KIND, FLAVOR>(h, (unsigned long long)bytes, status, lanes);
}

// Runtime-dispatched entry points (variant read from the view).
#define OURO_DISPATCH(h, CALL)                                                            \
    switch ((h).kind * 3 + (h).flavor) {                                                   \
    case 0: CALL(0, 0); case 1: CALL(0, 1); case 2: CALL(0, 2);                            \
    case 3: CALL(1, 0); case 4: CALL(1, 1); default: CALL(1, 2);                           \
    }

static __device__ __noinline__ void* ouro_malloc(const ouro_heap_view& h, size_t bytes) {
#define OURO_M(K, F) return ouro_malloc_t<K, F>(h, bytes)
    OURO_DISPATCH(h, OURO_M)
#undef OURO_M
}
static __device__ __noinline__ void ouro_free(const ouro_heap_view& h, void* p) {
#define OURO_F(K, F) ouro_free_t<K, F>(h, p); return
    OURO_DISPATCH(h, OURO_F)
#undef OURO_F
}
static __device__ __noinline__ void* ouro_malloc_coalesced(const ouro_heap_view& h, size_t bytes) {
#define OURO_C(K, F) return ouro_malloc_coalesced_t<K, F>(h, bytes)
    OURO_DISPATCH(h, OURO_C)
#undef OURO_C
}

#endif  // OURO_DEVICE_CUH
