// ouro_oracle.cpp -- CPU restatement of the reference allocator (TEST INFRASTRUCTURE).
//
// See ouro_oracle.hpp for scope, provenance and parity status.  Every protocol
// decision the SPEC leaves open (gaps G1..G8) is settled
// here once; DESIGN.md §3 states the same rules and the CUDA build follows them.
// Citations are /root/reference-relative.
#include "ouro_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

namespace {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

template <class T>
inline std::atomic_ref<T> A(T& x) { return std::atomic_ref<T>(x); }
constexpr auto RLX = std::memory_order_relaxed;
constexpr auto ACQ = std::memory_order_acquire;
constexpr auto REL = std::memory_order_release;
constexpr auto AR = std::memory_order_acq_rel;

constexpr u32 NONE = 0xFFFFFFFFu;
constexpr u64 NONE_LINK = ~0ull;
constexpr u32 ST_UNASSIGNED = 0;
constexpr u32 ST_RESERVED = 0xFF;  // page kind, virtual flavours: segment storage (gap G1)

// ---------------------------------------------------------------- config ----
// HeapConfig::validate, proj/src/config.cpp:16-42.  Same order, same messages.
bool pow2(u64 v) { return v != 0 && std::has_single_bit(v); }

ouro_status validate(const ouro_config* c, const char** why) {
    if (!pow2(c->heap_bytes) || !pow2(c->chunk_bytes) || !pow2(c->min_page_bytes) ||
        !pow2(c->max_page_bytes)) {
        *why = "heap, chunk and page-class sizes must be powers of two";
        return OURO_ERR_CONFIG;
    }
    if (c->min_page_bytes > c->max_page_bytes) { *why = "min_page_bytes exceeds max_page_bytes"; return OURO_ERR_CONFIG; }
    if (c->max_page_bytes > c->chunk_bytes) { *why = "max_page_bytes exceeds chunk_bytes"; return OURO_ERR_CONFIG; }
    if (c->chunk_bytes > c->heap_bytes) { *why = "chunk_bytes exceeds heap_bytes"; return OURO_ERR_CONFIG; }
    const u64 chunks = c->heap_bytes / c->chunk_bytes;
    if (chunks > (1ull << 24)) {
        *why = "more than 2^24 chunks; chunk index does not fit a packed handle";
        return OURO_ERR_CONFIG;
    }
    const int page_bits = std::countr_zero(c->chunk_bytes / c->min_page_bytes);
    const int chunk_bits = 64 - std::countl_zero(chunks - 1 ? chunks - 1 : 0);
    if (page_bits + chunk_bits > 32) { *why = "chunk/page split does not fit a 32-bit handle"; return OURO_ERR_CONFIG; }
    if (c->max_retries == 0) { *why = "max_retries must be at least 1"; return OURO_ERR_CONFIG; }
    *why = "";
    return OURO_OK;
}

struct Geo {
    u64 heap, chunk, minp, maxp;
    u32 N, K, page_bits, chunk_bits, chunk_shift, min_shift, Wmax, gen_bits;
    u32 gmask, cmask;
    u32 ppc(u32 k) const { return (u32)(chunk >> (min_shift + k)); }
    u32 words(u32 k) const { return (ppc(k) + 63) / 64; }
    u64 page_bytes(u32 k) const { return minp << k; }
};

// Extra limits of this build beyond validate(): <= 32 classes, and virtual
// flavours need room for a 2-word list header plus one slot (chunk >= 32 B).
ouro_status make_geo(const ouro_config* c, Geo* g) {
    const char* why;
    if (validate(c, &why) != OURO_OK) return OURO_ERR_CONFIG;
    if (c->queue_flavor > 2 || c->allocator_kind > 1 || c->backoff > 1) return OURO_ERR_CONFIG;
    g->heap = c->heap_bytes; g->chunk = c->chunk_bytes; g->minp = c->min_page_bytes; g->maxp = c->max_page_bytes;
    const u64 chunks = g->heap / g->chunk;
    g->N = (u32)chunks;
    g->K = (u32)std::countr_zero(g->maxp / g->minp) + 1;
    g->page_bits = (u32)std::countr_zero(g->chunk / g->minp);
    g->chunk_bits = (u32)(64 - std::countl_zero(chunks - 1 ? chunks - 1 : 0));
    g->chunk_shift = (u32)std::countr_zero(g->chunk);
    g->min_shift = (u32)std::countr_zero(g->minp);
    g->Wmax = (u32)((g->chunk / g->minp + 63) / 64);
    g->gen_bits = std::min<u32>(24, 32 - g->chunk_bits);
    g->gmask = g->gen_bits >= 32 ? 0xFFFFFFFFu : ((1u << g->gen_bits) - 1);
    g->cmask = g->chunk_bits == 0 ? 0 : (g->chunk_bits >= 32 ? 0xFFFFFFFFu : ((1u << g->chunk_bits) - 1));
    if (g->K > OURO_MAX_CLASSES) return OURO_ERR_CONFIG;
    if (c->queue_flavor != OURO_FLAVOR_ARRAY && g->chunk < 32) return OURO_ERR_CONFIG;
    return OURO_OK;
}

// size_class_of: smallest k with min<<k >= max(req, min).
// Request 0 is outside the precondition; gap G5 rejects it like TooLarge.
ouro_status size_class(const Geo& g, u64 req, u32* k) {
    if (req == 0 || req > g.maxp) return OURO_ERR_TOO_LARGE;
    const u32 lg = req <= 1 ? 0 : (u32)(64 - std::countl_zero(req - 1));
    *k = lg > g.min_shift ? lg - g.min_shift : 0;
    return OURO_OK;
}

u64 mix64(u64 x) {  // splitmix64 finaliser
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Pattern (gap G6): one mix per slot, then one
// multiply-xor per 8-byte word.
u64 pattern_base(u64 seed, u64 slot, u32 it) {
    return mix64(seed ^ (slot * 0xD1B54A32D192ED03ull) ^ ((u64)it * 0x8CB92BA72F3D8DD7ull));
}
u64 pattern_word(u64 base, u64 w) { return base ^ (w * 0x9E3779B97F4A7C15ull) ^ (w << 7); }

// backoff mapping.
u64 backoff_ns(u8 policy, u32 attempt, u32 base, u32 cap) {
    if (policy != OURO_BACKOFF_SLEEP) return 0;
    if (attempt >= 40) return cap;
    const u64 v = (u64)base << attempt;
    return v > cap ? cap : v;
}

// Bounded spin: every wait in the oracle gives up with TimeoutError instead of
// hanging (failure detection).
struct Spin {
    u64 n = 0;
    std::chrono::steady_clock::time_point t0;
    double limit_s;
    explicit Spin(double lim = 20.0) : limit_s(lim) {}
    bool ok() {
        ++n;
        if ((n & 63) == 0) std::this_thread::yield();
        if ((n & 4095) == 0) {
            if (n == 4096) t0 = std::chrono::steady_clock::now();
            else if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit_s) return false;
        }
        return true;
    }
};

// ---------------------------------------------------------------- queues ----
// IndexQueue: count reservation, then ticket, then slot turn.
struct Queue {
    u32 flavor = 0;
    u64 cap = 0;
    alignas(64) i64 count = 0;
    alignas(64) u64 head = 0;
    alignas(64) u64 tail = 0;
    // Array: power-of-two ring, slot = {tag:32, value:32}; ticket t uses slot
    // t & mask in round r = t >> shift; tag 2r = empty for round r, 2r+1 = full.
    u32 ring_shift = 0;
    u64 ring_mask = 0;
    std::vector<u64> slots;
    // VirtualArray: directory of D entries {seq:32, chunk:32}; dcnt = dequeues done per segment.
    u32 D = 0;
    std::vector<u64> dir;
    std::vector<u32> dcnt;
    // VirtualList: head / tail segment links {seq:32, chunk:32}.
    alignas(64) u64 vl_head = 0;
    alignas(64) u64 vl_tail = 0;
    int seg_src = -1;  // Array queue supplying segment chunks
    u64 seg_live = 0, seg_hwm = 0;
};

u64 next_pow2(u64 v) { return v <= 1 ? 1 : (1ull << (64 - std::countl_zero(v - 1))); }

struct Arena;  // forward: segments live in arena chunks

struct Errors {
    u32 first = 0, mask = 0;
    u64 stale_drops = 0, double_frees = 0, invalid_frees = 0, bad_sizes = 0, timeouts = 0, corruptions = 0;
    void raise(ouro_status s) {
        u32 z = 0;
        A(first).compare_exchange_strong(z, (u32)s, AR, RLX);
        A(mask).fetch_or(1u << (u32)s, RLX);
        if (s == OURO_ERR_TIMEOUT) A(timeouts).fetch_add(1, RLX);
        if (s == OURO_ERR_CORRUPTION) A(corruptions).fetch_add(1, RLX);
    }
};

// Memory that backs virtual segments: the heap itself.
struct Arena {
    u64 chunk_bytes = 0;
    u64 words_per_chunk = 0;
    u64* words = nullptr;  // heap bytes as 64-bit words (calloc: lazily committed)
    std::vector<Queue> q;
    u32 backoff = 0, base_ns = 100, cap_ns = 100000;
    Errors err;
    u64 queue_ops = 0;     // enqueue/dequeue calls (criterion 7 counters)

    u64* cw(u32 c) { return words + (u64)c * words_per_chunk; }
    u64 S_va() const { return words_per_chunk; }
    u64 S_vl() const { return words_per_chunk - 2; }

    void do_backoff(u32 attempt) {
        std::atomic_thread_fence(std::memory_order_seq_cst);
        const u64 ns = backoff_ns((u8)backoff, attempt, base_ns, cap_ns);
        if (ns) std::this_thread::sleep_for(std::chrono::nanoseconds(ns));
        else std::this_thread::yield();
    }

    // ---- count reservation ----
    u32 reserve_deq(Queue& Q, u32 n, i64 floor) {
        if (A(Q.count).load(ACQ) - floor <= 0) return 0;  // pre-check: no RMW when empty
        const i64 old = A(Q.count).fetch_sub(n, AR);
        i64 avail = old - floor;
        u32 got = avail <= 0 ? 0 : (avail >= (i64)n ? n : (u32)avail);
        if (got < n) A(Q.count).fetch_add((i64)(n - got), AR);
        return got;
    }
    bool reserve_enq(Queue& Q, u32 n) {
        if (A(Q.count).load(ACQ) + (i64)n > (i64)Q.cap) return false;
        const i64 old = A(Q.count).fetch_add(n, AR);
        if (old + (i64)n > (i64)Q.cap) { A(Q.count).fetch_sub(n, AR); return false; }
        return true;
    }

    static u64 tv(u32 tag, u32 v) { return ((u64)tag << 32) | v; }
    static u32 vtag(u64 t) { return ((u32)t & 0x7FFFFFFFu) | 0x80000000u; }

    // ---- segment supply (segments are arena chunks) ----
    bool seg_acquire(Queue& Q, u32* c) {
        Queue& P = q[Q.seg_src];
        Spin sp;
        for (u32 attempt = 1;; ++attempt) {
            u32 v;
            if (deq1(P, 0, &v)) { *c = v; return true; }
            if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
            do_backoff(attempt < 8 ? attempt : 8);
        }
    }
    void seg_release(Queue& Q, u32 c) {
        if (!enq1(q[Q.seg_src], c)) err.raise(OURO_ERR_CORRUPTION);
    }
    void seg_count(Queue& Q, int d) {
        if (d > 0) {
            u64 now = A(Q.seg_live).fetch_add(1, RLX) + 1;
            u64 h = A(Q.seg_hwm).load(RLX);
            while (now > h && !A(Q.seg_hwm).compare_exchange_weak(h, now, RLX, RLX)) {}
        } else {
            A(Q.seg_live).fetch_sub(1, RLX);
        }
    }
    void zero_chunk(u32 c) {
        u64* w = cw(c);
        for (u64 i = 0; i < words_per_chunk; ++i) A(w[i]).store(0, RLX);
    }

    // ---- VirtualArray ----
    bool va_create(Queue& Q, u64 s) {
        u64& e = Q.dir[s % Q.D];
        const u64 want = ((u64)(u32)s << 32) | NONE;
        Spin sp;
        while (A(e).load(ACQ) != want)
            if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
        u32 c;
        if (!seg_acquire(Q, &c)) return false;
        zero_chunk(c);
        A(Q.dcnt[s % Q.D]).store(0, RLX);
        A(e).store(((u64)(u32)s << 32) | c, REL);
        seg_count(Q, +1);
        return true;
    }
    bool va_find(Queue& Q, u64 s, u32* c) {
        u64& e = Q.dir[s % Q.D];
        Spin sp;
        for (;;) {
            const u64 v = A(e).load(ACQ);
            if ((u32)(v >> 32) == (u32)s && (u32)v != NONE) { *c = (u32)v; return true; }
            if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
        }
    }
    void va_consumed(Queue& Q, u64 s, u32 cnt) {
        const u32 n = A(Q.dcnt[s % Q.D]).fetch_add(cnt, AR) + cnt;
        if (n == (u32)Q_S(Q)) {
            u64& e = Q.dir[s % Q.D];
            const u32 c = (u32)A(e).load(ACQ);
            seg_release(Q, c);
            A(e).store(((u64)(u32)(s + Q.D) << 32) | NONE, REL);
            seg_count(Q, -1);
        }
    }
    u64 Q_S(const Queue& Q) const { return Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY ? S_va() : S_vl(); }

    // ---- VirtualList ----
    static u32 lseq(u64 l) { return (u32)(l >> 32); }
    static u32 lchunk(u64 l) { return (u32)l; }
    static u64 link(u64 s, u32 c) { return ((u64)(u32)s << 32) | c; }
    u32& vl_counter(u32 c) { return reinterpret_cast<u32*>(cw(c) + 1)[0]; }

    bool vl_locate(Queue& Q, u64 s, u32* out) {
        Spin sp;
        for (;;) {
            const u64 tl = A(Q.vl_tail).load(ACQ);
            if (lchunk(tl) != NONE && lseq(tl) == (u32)s) { *out = lchunk(tl); return true; }
            const u64 h = A(Q.vl_head).load(ACQ);
            if (lchunk(h) != NONE) {
                u32 i = lseq(h), cur = lchunk(h);
                if ((u32)((u32)s - i) >= 0x80000000u) { err.raise(OURO_ERR_CORRUPTION); return false; }
                bool ok = true;
                while (i != (u32)s) {
                    const u64 nx = A(cw(cur)[0]).load(ACQ);
                    if (A(Q.vl_head).load(ACQ) != h || nx == NONE_LINK) { ok = false; break; }
                    cur = lchunk(nx);
                    ++i;
                }
                if (ok) { *out = cur; return true; }
            }
            if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
        }
    }
    void vl_tail_max(Queue& Q, u64 l) {
        u64 cur = A(Q.vl_tail).load(ACQ);
        for (;;) {
            if (lchunk(cur) != NONE && (int32_t)(lseq(l) - lseq(cur)) <= 0) return;
            if (A(Q.vl_tail).compare_exchange_weak(cur, l, AR, ACQ)) return;
        }
    }
    void vl_try_advance(Queue& Q) {
        const u32 full = (u32)S_vl() + 1;
        for (;;) {
            u64 h = A(Q.vl_head).load(ACQ);
            const u32 ch = lchunk(h);
            if (ch == NONE) return;
            if (A(vl_counter(ch)).load(ACQ) != full) return;
            const u64 nx = A(cw(ch)[0]).load(ACQ);
            if (nx == NONE_LINK) return;
            if (A(Q.vl_head).compare_exchange_strong(h, nx, AR, ACQ)) {
                seg_release(Q, ch);
                seg_count(Q, -1);
            }
        }
    }
    void vl_add(Queue& Q, u32 segc, u32 cnt) {
        const u32 n = A(vl_counter(segc)).fetch_add(cnt, AR) + cnt;
        if (n == (u32)S_vl() + 1) vl_try_advance(Q);
    }
    bool vl_create(Queue& Q, u64 s) {
        u32 c;
        if (!seg_acquire(Q, &c)) return false;
        zero_chunk(c);
        A(cw(c)[0]).store(NONE_LINK, RLX);
        seg_count(Q, +1);
        if (s == 0) {
            A(Q.vl_head).store(link(0, c), REL);
            vl_tail_max(Q, link(0, c));
            return true;
        }
        u32 p;
        if (!vl_locate(Q, s - 1, &p)) return false;
        A(cw(p)[0]).store(link(s, c), REL);
        vl_tail_max(Q, link(s, c));
        vl_add(Q, p, 1);  // link event: part of the predecessor's retire count
        return true;
    }

    // ---- slot access by ticket ----
    bool first_of_segment(const Queue& Q, u64 t) const {
        if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) return (t % S_va()) == 0;
        if (Q.flavor == OURO_FLAVOR_VIRTUAL_LIST) return (t % S_vl()) == 0;
        return false;
    }
    bool create_for(Queue& Q, u64 t) {
        if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) return va_create(Q, t / S_va());
        return vl_create(Q, t / S_vl());
    }
    bool put(Queue& Q, u64 t, u32 v) {
        Spin sp;
        if (Q.flavor == OURO_FLAVOR_ARRAY) {
            u64& s = Q.slots[t & Q.ring_mask];
            const u32 r = (u32)(t >> Q.ring_shift);
            while ((u32)(A(s).load(ACQ) >> 32) != 2 * r)
                if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
            A(s).store(tv(2 * r + 1, v), REL);
            return true;
        }
        u32 c;
        u64 j;
        if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) {
            if (!va_find(Q, t / S_va(), &c)) return false;
            j = t % S_va();
        } else {
            if (!vl_locate(Q, t / S_vl(), &c)) return false;
            j = 2 + t % S_vl();
        }
        A(cw(c)[j]).store(tv(vtag(t) , v), REL);
        return true;
    }
    // take: read the value of ticket t; returns the segment chunk in *segc.
    bool take(Queue& Q, u64 t, u32* v, u32* segc) {
        Spin sp;
        if (Q.flavor == OURO_FLAVOR_ARRAY) {
            u64& s = Q.slots[t & Q.ring_mask];
            const u32 r = (u32)(t >> Q.ring_shift);
            u64 x;
            while ((u32)((x = A(s).load(ACQ)) >> 32) != 2 * r + 1)
                if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
            *v = (u32)x;
            A(s).store(tv(2 * r + 2, 0), REL);
            *segc = NONE;
            return true;
        }
        u32 c;
        u64 j;
        if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) {
            if (!va_find(Q, t / S_va(), &c)) return false;
            j = t % S_va();
        } else {
            if (!vl_locate(Q, t / S_vl(), &c)) return false;
            j = 2 + t % S_vl();
        }
        u64 x;
        while ((u32)((x = A(cw(c)[j]).load(ACQ)) >> 32) != vtag(t))
            if (!sp.ok()) { err.raise(OURO_ERR_TIMEOUT); return false; }
        *v = (u32)x;
        *segc = c;
        return true;
    }
    // Consumption bookkeeping after a group's reads, per segment in ticket order.
    void consumed(Queue& Q, u64 t0, u32 n, const u32* segc) {
        if (Q.flavor == OURO_FLAVOR_ARRAY || n == 0) return;
        const u64 S = Q_S(Q);
        u32 i = 0;
        while (i < n) {
            const u64 s = (t0 + i) / S;
            u32 j = i;
            while (j < n && (t0 + j) / S == s) ++j;
            if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) va_consumed(Q, s, j - i);
            else vl_add(Q, segc[i], j - i);
            i = j;
        }
    }

    // ---- group operations (what one warp leader does for n lanes) ----
    u32 deq_group(Queue& Q, u32 n, i64 floor, u32* out) {
        const u32 got = reserve_deq(Q, n, floor);
        if (!got) return 0;
        A(queue_ops).fetch_add(1, RLX);
        const u64 t0 = A(Q.head).fetch_add(got, AR);
        u32 segc[64];
        for (u32 r = 0; r < got; ++r)
            if (!take(Q, t0 + r, &out[r], &segc[r])) { out[r] = NONE; segc[r] = NONE; }
        consumed(Q, t0, got, segc);
        return got;
    }
    bool enq_group(Queue& Q, u32 n, const u32* vals) {
        if (!n) return true;
        if (!reserve_enq(Q, n)) return false;
        A(queue_ops).fetch_add(1, RLX);
        const u64 t0 = A(Q.tail).fetch_add(n, AR);
        for (u32 r = 0; r < n; ++r)
            if (first_of_segment(Q, t0 + r) && !create_for(Q, t0 + r)) return false;
        for (u32 r = 0; r < n; ++r)
            if (!put(Q, t0 + r, vals[r])) return false;
        return true;
    }
    bool deq1(Queue& Q, i64 floor, u32* v) { return deq_group(Q, 1, floor, v) == 1 && *v != NONE; }
    bool enq1(Queue& Q, u32 v) { return enq_group(Q, 1, &v); }

    // ---- construction ----
    void init_queue(Queue& Q, u32 flavor, u64 cap, int seg_src) {
        Q.flavor = flavor;
        Q.cap = cap;
        Q.count = 0; Q.head = 0; Q.tail = 0;
        Q.seg_src = seg_src;
        Q.seg_live = Q.seg_hwm = 0;
        if (flavor == OURO_FLAVOR_ARRAY) {
            const u64 R = next_pow2(std::max<u64>(cap, 1));
            Q.ring_shift = (u32)std::countr_zero(R);
            Q.ring_mask = R - 1;
            Q.slots.assign(R, 0);
        } else if (flavor == OURO_FLAVOR_VIRTUAL_ARRAY) {
            Q.D = (u32)((cap + S_va() - 1) / S_va() + 2);
            Q.dir.resize(Q.D);
            Q.dcnt.assign(Q.D, 0);
            for (u32 i = 0; i < Q.D; ++i) Q.dir[i] = ((u64)i << 32) | NONE;
        } else {
            Q.vl_head = Q.vl_tail = link(0, NONE);
        }
    }
    // Single-threaded prefill of `n` values (construction only).
    // Virtual flavours take their initial segments from segs[] in order.
    void prefill(Queue& Q, u64 n, u32 (*val)(void*, u64), void* ctx, const u32* segs, u32 nsegs) {
        Q.count = (i64)n; Q.head = 0; Q.tail = n;
        if (Q.flavor == OURO_FLAVOR_ARRAY) {
            for (u64 t = 0; t < n; ++t) Q.slots[t] = tv(1, val(ctx, t));
            return;
        }
        const u64 S = Q_S(Q);
        const u64 m = (n + S - 1) / S;
        if (m > nsegs) { err.raise(OURO_ERR_CORRUPTION); return; }
        for (u64 i = 0; i < m; ++i) zero_chunk(segs[i]);
        for (u64 t = 0; t < n; ++t) {
            const u32 c = segs[t / S];
            const u64 j = (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY ? 0 : 2) + t % S;
            cw(c)[j] = tv(vtag(t), val(ctx, t));
        }
        Q.seg_live = Q.seg_hwm = m;
        if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) {
            for (u64 i = 0; i < m; ++i) Q.dir[i % Q.D] = ((u64)i << 32) | segs[i];
        } else if (m > 0) {
            for (u64 i = 0; i < m; ++i) {
                cw(segs[i])[0] = (i + 1 < m) ? link(i + 1, segs[i + 1]) : NONE_LINK;
                vl_counter(segs[i]) = (i + 1 < m) ? 1 : 0;
            }
            Q.vl_head = link(0, segs[0]);
            Q.vl_tail = link(m - 1, segs[m - 1]);
        }
    }
};

// ------------------------------------------------------------- allocator ----
struct Lane {
    u32 k;
    u64 off;
    int32_t st;
};

}  // namespace

struct orc_heap {
    ouro_config cfg;
    Geo g;
    Arena ar;
    u32 kind = 0, flavor = 0;
    // ChunkHeader side table: meta = {free:32, state:8, gen:24}.
    std::vector<u64> meta;
    // N * Wmax words, 1 = ALLOCATED (an unassigned or fully free chunk is all-zero, so
    // assigning needs no bitmap init and returning to the pool needs no clear)
    std::vector<u64> bitmap;
    std::vector<u32> assigned;  // chunk kind: chunks assigned per class (gap G3 watermark)
    // page-kind partition (gap G1)
    std::vector<u32> pq_start, pq_n, pq_s;
    i64 floor_F = 0;  // chunk kind, virtual: pool chunks kept for segments
    std::vector<u64> retries, ooms;
    u64 pool_dequeues = 0;

    static u32 m_free(u64 m) { return (u32)m; }
    static u32 m_state(u64 m) { return (u32)(m >> 32) & 0xFF; }
    static u32 m_gen(u64 m) { return (u32)(m >> 40); }
    static u64 mk(u32 gen, u32 state, u32 fr) { return ((u64)(gen & 0xFFFFFF) << 40) | ((u64)state << 32) | fr; }
    u64* bm(u32 c) { return bitmap.data() + (u64)c * g.Wmax; }
    u32 pool_idx() const { return g.K; }
    u32 priv_idx(u32 k) const { return g.K + 1 + k; }
    u32 entry(u32 c, u32 gen) const { return g.chunk_bits >= 32 ? c : (c | ((gen & g.gmask) << g.chunk_bits)); }
    u64 offset_of(u32 c, u32 k, u32 p) const { return ((u64)c << g.chunk_shift) + ((u64)p << (g.min_shift + k)); }
    u32 handle_of(u32 c, u32 p) const { return (c << g.page_bits) | p; }

    void build();
    // chunk bitmap primitives
    u32 claim_lowest(u32 c, u32 k, u32 take, u32* pages);
    u64 claim_collisions = 0;  // bitmap picks lost to a concurrent holder (retried)
    // allocation
    void alloc_class(u32 k, Lane** lanes, u32 n);
    void alloc_page(u32 k, Lane** lanes, u32 n);
    void alloc_chunk(u32 k, Lane** lanes, u32 n);
    void alloc_group(Lane* lanes, u32 n);
    void free_group(Lane* lanes, u32 n);
};

namespace {

u32 pq_handle_val(void* ctx, u64 t);
struct PrefillCtx { orc_heap* h; u32 k; };

u32 pq_handle_val(void* ctx, u64 t) {
    auto* p = static_cast<PrefillCtx*>(ctx);
    const u32 k = p->k;
    const u32 ppc = p->h->g.ppc(k);
    const u32 c = p->h->pq_start[k] + p->h->pq_s[k] + (u32)(t / ppc);
    return p->h->handle_of(c, (u32)(t % ppc));
}
u32 pool_val(void*, u64 t) { return (u32)t; }

}  // namespace

// Construction.
void orc_heap::build() {
    const u32 N = g.N, K = g.K;
    meta.assign(N, 0);
    bitmap.assign((u64)N * g.Wmax, 0);
    assigned.assign(K, 0);
    retries.assign(K, 0);
    ooms.assign(K, 0);
    ar.q.clear();
    ar.q.resize(2 * K + 1);
    if (kind == OURO_KIND_PAGE) {
        // Static equal partition by chunk count, remainder to class 0.
        pq_start.assign(K, 0); pq_n.assign(K, 0); pq_s.assign(K, 0);
        u32 at = 0;
        for (u32 k = 0; k < K; ++k) {
            pq_n[k] = N / K + (k == 0 ? N % K : 0);
            pq_start[k] = at;
            at += pq_n[k];
        }
        for (u32 k = 0; k < K; ++k) {
            const u64 ppc = g.ppc(k);
            // Gap G1: virtual flavours self-host their segments in the class's
            // first s_k chunks: the smallest s with ceil(cap(s)/S)+2 <= s.
            u32 s = 0;
            if (flavor != OURO_FLAVOR_ARRAY) {
                const u64 S = flavor == OURO_FLAVOR_VIRTUAL_ARRAY ? ar.S_va() : ar.S_vl();
                for (s = 0; s <= pq_n[k]; ++s) {
                    const u64 cap = (u64)(pq_n[k] - s) * ppc;
                    const u64 need = cap == 0 ? 0 : (cap + S - 1) / S + 2;
                    if (need <= s) break;
                }
            }
            pq_s[k] = s;
            const u64 cap = (u64)(pq_n[k] - s) * ppc;
            for (u32 i = 0; i < pq_n[k]; ++i) {
                const u32 c = pq_start[k] + i;
                if (i < s) {
                    meta[c] = mk(0, ST_RESERVED, 0);
                } else {
                    meta[c] = mk(1, k + 1, (u32)ppc);
                }
            }
            Queue& Q = ar.q[k];
            if (flavor == OURO_FLAVOR_ARRAY) {
                ar.init_queue(Q, OURO_FLAVOR_ARRAY, cap, -1);
                PrefillCtx ctx{this, k};
                ar.prefill(Q, cap, pq_handle_val, &ctx, nullptr, 0);
            } else {
                Queue& P = ar.q[priv_idx(k)];
                ar.init_queue(P, OURO_FLAVOR_ARRAY, std::max<u32>(s, 1), -1);
                ar.init_queue(Q, flavor, cap, (int)priv_idx(k));
                const u64 S = flavor == OURO_FLAVOR_VIRTUAL_ARRAY ? ar.S_va() : ar.S_vl();
                const u32 m = (u32)((cap + S - 1) / S);
                std::vector<u32> segs(s);
                for (u32 i = 0; i < s; ++i) segs[i] = pq_start[k] + i;
                PrefillCtx ctx{this, k};
                ar.prefill(Q, cap, pq_handle_val, &ctx, segs.data(), m);
                for (u32 i = m; i < s; ++i) {
                    P.slots[(i - m) & P.ring_mask] = Arena::tv(1, segs[i]);
                }
                P.count = (i64)(s - m); P.head = 0; P.tail = s - m;
            }
        }
        // unused class queues beyond K stay empty
        ar.init_queue(ar.q[pool_idx()], OURO_FLAVOR_ARRAY, 1, -1);
    } else {
        // Chunk kind: all chunks Unassigned in the pool (Array, gap G2), class
        // queues empty; class-queue capacity 2N absorbs stale entries (gap G3).
        Queue& P = ar.q[pool_idx()];
        ar.init_queue(P, OURO_FLAVOR_ARRAY, N, -1);
        ar.prefill(P, N, pool_val, nullptr, nullptr, 0);
        for (u32 k = 0; k < K; ++k) ar.init_queue(ar.q[k], flavor, 2ull * N, (int)pool_idx());
        floor_F = flavor == OURO_FLAVOR_ARRAY ? 0 : (i64)std::min<u32>(K, N / 8);
    }
}

// Claim the `take` lowest free pages (lowest free word
// first; free = clear bit below ppc, claimed with fetch-OR).  Returns pages claimed.
u32 orc_heap::claim_lowest(u32 c, u32 k, u32 take, u32* pages) {
    u32 got = 0;
    Spin sp;
    while (got < take) {
        for (u32 w = 0; w < g.words(k) && got < take; ++w) {
            const u32 ppc = g.ppc(k);
            const u64 valid = (ppc - w * 64 >= 64) ? ~0ull : ((1ull << (ppc - w * 64)) - 1);
            u64 snap = ~A(bm(c)[w]).load(ACQ) & valid;
            u64 pick = 0;
            while (snap && got + (u32)std::popcount(pick) < take) {
                pick |= snap & (~snap + 1);
                snap &= snap - 1;
            }
            if (!pick) continue;
            const u64 old = A(bm(c)[w]).fetch_or(pick, AR);
            // Bits another holder took between our snapshot and the fetch-OR are
            // contention, not corruption ("retry on contention"): every
            // holder reserved its pages on free_count first, so the rescan finds ours.
            u64 mine = ~old & pick;
            if (mine != pick) A(claim_collisions).fetch_add(1, RLX);
            while (mine) {
                pages[got++] = w * 64 + (u32)std::countr_zero(mine);
                mine &= mine - 1;
            }
        }
        if (got < take && !sp.ok()) { ar.err.raise(OURO_ERR_TIMEOUT); break; }
    }
    std::sort(pages, pages + got);
    return got;
}

// Page kind, one class group of n lanes (SPEC.md:258-262 + coalesce 335-339):
// reserve up to n, take consecutive tickets, lanes read in rank order; the
// remainder backs off and retries; OOM after max_retries failed tries.
void orc_heap::alloc_page(u32 k, Lane** L, u32 n) {
    Queue& Q = ar.q[k];
    u32 served = 0, attempt = 0;
    std::vector<u32> vals(n);
    while (served < n) {
        const u32 need = n - served;
        const u32 got = ar.deq_group(Q, need, 0, vals.data());
        for (u32 r = 0; r < got; ++r) {
            Lane* l = L[served + r];
            const u32 h = vals[r];
            if (h == NONE) { l->st = OURO_ERR_TIMEOUT; l->off = ~0ull; continue; }
            const u32 c = h >> g.page_bits, p = h & ((1u << g.page_bits) - 1);
            const u64 bit = 1ull << (p & 63);
            const u64 old = A(bm(c)[p >> 6]).fetch_or(bit, AR);
            if (old & bit) ar.err.raise(OURO_ERR_CORRUPTION);
            A(meta[c]).fetch_sub(1, AR);
            l->st = OURO_OK;
            l->off = offset_of(c, k, p);
        }
        served += got;
        if (served == n) break;
        A(retries[k]).fetch_add(n - served, RLX);
        if (++attempt >= cfg.max_retries) {
            for (u32 r = served; r < n; ++r) { L[r]->st = OURO_ERR_OOM; L[r]->off = ~0ull; }
            A(ooms[k]).fetch_add(n - served, RLX);
            return;
        }
        ar.do_backoff(attempt);
    }
}

// Chunk kind, one class group of n lanes (in-transit rule 299;
// ChunkFull/stale re-dequeue 206 + gap G4; fresh chunk from the pool 193-197).
void orc_heap::alloc_chunk(u32 k, Lane** L, u32 n) {
    Queue& CQ = ar.q[k];
    Queue& P = ar.q[pool_idx()];
    const u32 ppc = g.ppc(k);
    u32 served = 0, attempt = 0;
    u32 pages[64];
    Spin sp;
    while (served < n) {
        const u32 need = n - served;
        u32 e;
        if (ar.deq1(CQ, 0, &e)) {
            const u32 c = e & g.cmask;
            const u32 glow = g.chunk_bits >= 32 ? 0 : (e >> g.chunk_bits);
            // reserve pages: CAS on {gen, state, free} (free_count)
            u64 m = A(meta[c]).load(ACQ);
            u32 take = 0, oldfree = 0;
            for (;;) {
                if (m_state(m) != k + 1 || (m_gen(m) & g.gmask) != glow || m_free(m) == 0) break;
                oldfree = m_free(m);
                const u32 t = std::min(need, oldfree);
                if (A(meta[c]).compare_exchange_weak(m, m - t, AR, ACQ)) { take = t; break; }
            }
            if (!take) { A(ar.err.stale_drops).fetch_add(1, RLX); continue; }
            const u32 got = claim_lowest(c, k, take, pages);
            if (oldfree - take > 0) {  // in-transit rule: the holder re-enqueues
                Spin s2;
                while (!ar.enq1(CQ, e)) { if (!s2.ok()) { ar.err.raise(OURO_ERR_TIMEOUT); break; } ar.do_backoff(1); }
            }
            for (u32 r = 0; r < take; ++r) {
                Lane* l = L[served + r];
                if (r < got) { l->st = OURO_OK; l->off = offset_of(c, k, pages[r]); }
                else { l->st = OURO_ERR_CORRUPTION; l->off = ~0ull; }
            }
            served += take;
            continue;
        }
        u32 c;
        if (ar.deq1(P, floor_F, &c)) {
            A(pool_dequeues).fetch_add(1, RLX);
            const u32 take = std::min(need, ppc);
            const u64 m = A(meta[c]).load(ACQ);
            if (m_state(m) != ST_UNASSIGNED) { ar.err.raise(OURO_ERR_CORRUPTION); continue; }
            const u32 gen = (m_gen(m) + 1) & 0xFFFFFF;
            // chunk_assign fused with taking pages 0..take-1:
            // the bitmap of a pool chunk is all-zero (all free), so only the taken
            // bits are set (take <= group size <= 64: one word)
            const u64 tb = take >= 64 ? ~0ull : ((1ull << take) - 1);
            if (A(bm(c)[0]).fetch_or(tb, AR) & tb) ar.err.raise(OURO_ERR_CORRUPTION);
            A(meta[c]).exchange(mk(gen, k + 1, ppc - take), AR);
            A(assigned[k]).fetch_add(1, AR);
            if (ppc - take > 0) {
                Spin s2;
                while (!ar.enq1(CQ, entry(c, gen))) { if (!s2.ok()) { ar.err.raise(OURO_ERR_TIMEOUT); break; } ar.do_backoff(1); }
            }
            for (u32 r = 0; r < take; ++r) {
                Lane* l = L[served + r];
                l->st = OURO_OK;
                l->off = offset_of(c, k, r);
            }
            served += take;
            continue;
        }
        A(retries[k]).fetch_add(need, RLX);
        if (++attempt >= cfg.max_retries) {
            for (u32 r = served; r < n; ++r) { L[r]->st = OURO_ERR_OOM; L[r]->off = ~0ull; }
            A(ooms[k]).fetch_add(need, RLX);
            return;
        }
        ar.do_backoff(attempt);
    }
}

void orc_heap::alloc_class(u32 k, Lane** L, u32 n) {
    if (kind == OURO_KIND_PAGE) alloc_page(k, L, n);
    else alloc_chunk(k, L, n);
}

// One warp's malloc call: lanes grouped by size class, groups served in order
// of their lowest lane; ranks within a group follow lane order.
void orc_heap::alloc_group(Lane* lanes, u32 n) {
    std::vector<bool> done(n, false);
    for (u32 i = 0; i < n; ++i) {
        u32 k;
        if (size_class(g, lanes[i].off, &k) != OURO_OK) {
            lanes[i].st = OURO_ERR_TOO_LARGE;
            lanes[i].off = ~0ull;
            done[i] = true;
            A(ar.err.bad_sizes).fetch_add(1, RLX);
        } else {
            lanes[i].k = k;
        }
    }
    for (u32 i = 0; i < n; ++i) {
        if (done[i]) continue;
        std::vector<Lane*> grp;
        for (u32 j = i; j < n; ++j)
            if (!done[j] && lanes[j].k == lanes[i].k) { grp.push_back(&lanes[j]); done[j] = true; }
        alloc_class(lanes[i].k, grp.data(), (u32)grp.size());
    }
}

// One warp's free call.  Steps, in order:
// decode + in-group duplicates, bitmap fetch-AND (clear the allocated bit),
// per-chunk free_count add,
// chunk kind: watermark-limited closes (return to pool), class enqueues.
void orc_heap::free_group(Lane* L, u32 n) {
    struct V { u32 c, k, p; bool ok; };
    std::vector<V> v(n);
    for (u32 i = 0; i < n; ++i) {
        v[i].ok = false;
        const u64 off = L[i].off;
        L[i].st = OURO_OK;
        if (off >= g.heap) { L[i].st = OURO_ERR_INVALID_HANDLE; continue; }
        const u32 c = (u32)(off >> g.chunk_shift);
        const u64 m = A(meta[c]).load(ACQ);
        const u32 st = m_state(m);
        if (st == ST_UNASSIGNED || st == ST_RESERVED || st > g.K) { L[i].st = OURO_ERR_INVALID_HANDLE; continue; }
        const u32 k = st - 1;
        const u64 in = off & (g.chunk - 1);
        if (in & (g.page_bytes(k) - 1)) { L[i].st = OURO_ERR_INVALID_HANDLE; continue; }
        v[i] = {c, k, (u32)(in >> (g.min_shift + k)), true};
        for (u32 j = 0; j < i; ++j)
            if (v[j].ok && L[j].off == off) { L[i].st = OURO_ERR_DOUBLE_FREE; v[i].ok = false; break; }
    }
    for (u32 i = 0; i < n; ++i) {
        if (!v[i].ok) continue;
        const u64 bit = 1ull << (v[i].p & 63);
        const u64 old = A(bm(v[i].c)[v[i].p >> 6]).fetch_and(~bit, AR);
        if (!(old & bit)) { L[i].st = OURO_ERR_DOUBLE_FREE; v[i].ok = false; }
    }
    for (u32 i = 0; i < n; ++i) {
        if (L[i].st == OURO_ERR_DOUBLE_FREE) { A(ar.err.double_frees).fetch_add(1, RLX); ar.err.raise(OURO_ERR_DOUBLE_FREE); }
        if (L[i].st == OURO_ERR_INVALID_HANDLE) { A(ar.err.invalid_frees).fetch_add(1, RLX); ar.err.raise(OURO_ERR_INVALID_HANDLE); }
    }
    // per chunk, in order of the chunk's lowest valid lane
    struct CG { u32 c, k, cnt, oldfree, newfree, gen; bool closed; };
    std::vector<CG> cg;
    for (u32 i = 0; i < n; ++i) {
        if (!v[i].ok) continue;
        bool seen = false;
        for (auto& x : cg) if (x.c == v[i].c) { ++x.cnt; seen = true; break; }
        if (!seen) cg.push_back({v[i].c, v[i].k, 1, 0, 0, 0, false});
    }
    for (auto& x : cg) {
        const u64 old = A(meta[x.c]).fetch_add(x.cnt, AR);
        x.oldfree = m_free(old);
        x.newfree = x.oldfree + x.cnt;
        x.gen = m_gen(old);
    }
    if (kind == OURO_KIND_CHUNK) {
        // Watermark (gap G3): per class, closes allowed = min(#fully free, assigned-1),
        // lowest chunk-leader lanes first; then each close CASes the header.
        std::vector<u32> order;
        for (u32 i = 0; i < cg.size(); ++i)
            if (cg[i].newfree == g.ppc(cg[i].k)) order.push_back(i);
        std::vector<bool> allowed(cg.size(), false);
        std::vector<bool> handled(cg.size(), false);
        for (u32 a = 0; a < order.size(); ++a) {
            const u32 k = cg[order[a]].k;
            if (handled[order[a]]) continue;
            u32 want = 0;
            for (u32 b = a; b < order.size(); ++b) if (cg[order[b]].k == k) ++want;
            // take = min(want, assigned - 1): fetch-sub, give back the excess
            const u32 old = A(assigned[k]).fetch_sub(want, AR);
            const u32 take = old > 1 ? std::min(want, old - 1) : 0;
            if (want - take) A(assigned[k]).fetch_add(want - take, AR);
            u32 given = 0;
            for (u32 b = a; b < order.size(); ++b) {
                if (cg[order[b]].k != k) continue;
                handled[order[b]] = true;
                if (given < take) { allowed[order[b]] = true; ++given; }
            }
        }
        std::vector<u32> to_pool;
        for (u32 idx : order) {
            if (!allowed[idx]) continue;
            CG& x = cg[idx];
            const u32 ppc = g.ppc(x.k);
            u64 expect = mk(x.gen, x.k + 1, ppc);
            if (A(meta[x.c]).compare_exchange_strong(expect, mk(x.gen, ST_UNASSIGNED, 0), AR, ACQ)) {
                x.closed = true;  // fully free => bitmap already all-zero
                to_pool.push_back(x.c);
            } else {
                A(assigned[x.k]).fetch_add(1, AR);
            }
        }
        if (!to_pool.empty() && !ar.enq_group(ar.q[pool_idx()], (u32)to_pool.size(), to_pool.data()))
            ar.err.raise(OURO_ERR_CORRUPTION);
        // 0 -> >0 transitions re-enqueue the chunk, grouped by class.
        std::vector<bool> doneq(cg.size(), false);
        for (u32 a = 0; a < cg.size(); ++a) {
            if (doneq[a] || cg[a].closed || cg[a].oldfree != 0) continue;
            std::vector<u32> vals;
            for (u32 b = a; b < cg.size(); ++b) {
                if (doneq[b] || cg[b].closed || cg[b].oldfree != 0 || cg[b].k != cg[a].k) continue;
                doneq[b] = true;
                vals.push_back(entry(cg[b].c, cg[b].gen));
            }
            Spin s2;
            while (!ar.enq_group(ar.q[cg[a].k], (u32)vals.size(), vals.data())) {
                if (!s2.ok()) { ar.err.raise(OURO_ERR_TIMEOUT); break; }
                ar.do_backoff(1);
            }
        }
    } else {
        // Page kind: every freed handle goes back to its class queue.
        std::vector<bool> doneq(n, false);
        for (u32 i = 0; i < n; ++i) {
            if (!v[i].ok || doneq[i]) continue;
            std::vector<u32> vals;
            for (u32 j = i; j < n; ++j) {
                if (!v[j].ok || doneq[j] || v[j].k != v[i].k) continue;
                doneq[j] = true;
                vals.push_back(handle_of(v[j].c, v[j].p));
            }
            if (!ar.enq_group(ar.q[v[i].k], (u32)vals.size(), vals.data())) ar.err.raise(OURO_ERR_CORRUPTION);
        }
    }
}

// ================================================================= C ABI ====
extern "C" {

ouro_status orc_config_validate(const ouro_config* cfg, char* msg, size_t msg_len) {
    const char* why;
    const ouro_status s = validate(cfg, &why);
    if (msg && msg_len) { std::snprintf(msg, msg_len, "%s", why); }
    return s;
}

ouro_status orc_config_geometry(const ouro_config* cfg, ouro_geometry* out) {
    Geo g;
    const ouro_status s = make_geo(cfg, &g);
    if (s != OURO_OK) return s;
    out->num_chunks = g.N;
    out->max_pages_per_chunk = (u32)(g.chunk / g.minp);
    out->num_classes = g.K;
    out->page_bits = g.page_bits;
    out->chunk_bits = g.chunk_bits;
    out->gen_bits = g.gen_bits;
    out->bitmap_words = g.Wmax;
    out->reserved0 = 0;
    return OURO_OK;
}

// variant_name / variant_from_name, config.cpp:44-59, kAllVariants config.hpp:62-69.
const char* orc_variant_name(uint8_t kind, uint8_t flavor) {
    const bool page = kind == OURO_KIND_PAGE;
    if (kind > 1) return "?";
    switch (flavor) {
    case OURO_FLAVOR_ARRAY: return page ? "page" : "chunk";
    case OURO_FLAVOR_VIRTUAL_ARRAY: return page ? "va-page" : "va-chunk";
    case OURO_FLAVOR_VIRTUAL_LIST: return page ? "vl-page" : "vl-chunk";
    }
    return "?";
}

int orc_variant_from_name(const char* name, uint8_t* kind, uint8_t* flavor) {
    static const u8 order[6][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}, {0, 2}, {1, 2}};
    if (!name) return 0;
    for (auto& v : order) {
        if (std::strcmp(orc_variant_name(v[0], v[1]), name) == 0) {
            if (kind) *kind = v[0];
            if (flavor) *flavor = v[1];
            return 1;
        }
    }
    return 0;
}

ouro_status orc_size_class(const ouro_config* cfg, uint64_t bytes, uint32_t* cls) {
    Geo g;
    if (make_geo(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    return size_class(g, bytes, cls);
}

// encode/decode_handle: RangeError outside the grid.
ouro_status orc_handle_encode(const ouro_config* cfg, uint32_t c, uint32_t p, uint32_t* h) {
    Geo g;
    if (make_geo(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    if (c >= g.N || p >= (u32)(g.chunk / g.minp)) return OURO_ERR_RANGE;
    *h = (c << g.page_bits) | p;
    return OURO_OK;
}

ouro_status orc_handle_decode(const ouro_config* cfg, uint32_t h, uint32_t* c, uint32_t* p) {
    Geo g;
    if (make_geo(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    const u64 cc = (u64)h >> g.page_bits;
    if (cc >= g.N) return OURO_ERR_RANGE;
    *c = (u32)cc;
    *p = h & ((1u << g.page_bits) - 1);
    return OURO_OK;
}

uint64_t orc_backoff_ns(uint8_t policy, uint32_t attempt, uint32_t base_ns, uint32_t cap_ns) {
    return backoff_ns(policy, attempt, base_ns, cap_ns);
}
uint64_t orc_mix64(uint64_t x) { return mix64(x); }
uint64_t orc_pattern_word(uint64_t seed, uint64_t slot, uint32_t iteration, uint64_t word) {
    return pattern_word(pattern_base(seed, slot, iteration), word);
}

ouro_status orc_heap_create(const ouro_config* cfg, orc_heap** out) {
    Geo g;
    if (make_geo(cfg, &g) != OURO_OK) return OURO_ERR_CONFIG;
    auto* h = new (std::nothrow) orc_heap();
    if (!h) return OURO_ERR_OOM;
    h->cfg = *cfg;
    h->g = g;
    h->kind = cfg->allocator_kind;
    h->flavor = cfg->queue_flavor;
    h->ar.chunk_bytes = g.chunk;
    h->ar.words_per_chunk = g.chunk / 8;
    h->ar.backoff = cfg->backoff;
    h->ar.base_ns = cfg->sleep_base_ns;
    h->ar.cap_ns = cfg->sleep_cap_ns;
    h->ar.words = static_cast<u64*>(std::calloc(g.heap / 8, 8));
    if (!h->ar.words) { delete h; return OURO_ERR_OOM; }
    h->build();
    *out = h;
    return OURO_OK;
}

void orc_heap_destroy(orc_heap* h) {
    if (!h) return;
    std::free(h->ar.words);
    delete h;
}

ouro_status orc_alloc_group(orc_heap* h, uint32_t n, const uint64_t* sizes, uint64_t* out_off,
                            int32_t* out_status) {
    if (n == 0 || n > 64) return OURO_ERR_USAGE;
    std::vector<Lane> L(n);
    for (u32 i = 0; i < n; ++i) { L[i].off = sizes[i]; L[i].k = 0; L[i].st = 0; }
    h->alloc_group(L.data(), n);
    for (u32 i = 0; i < n; ++i) { out_off[i] = L[i].off; out_status[i] = L[i].st; }
    return OURO_OK;
}

ouro_status orc_free_group(orc_heap* h, uint32_t n, const uint64_t* offs, int32_t* out_status) {
    if (n == 0 || n > 64) return OURO_ERR_USAGE;
    std::vector<Lane> L(n);
    for (u32 i = 0; i < n; ++i) { L[i].off = offs[i]; L[i].st = 0; }
    h->free_group(L.data(), n);
    for (u32 i = 0; i < n; ++i) out_status[i] = L[i].st;
    return OURO_OK;
}

// alloc_coalesced: one class for all lanes; all-or-nothing.
ouro_status orc_alloc_coalesced(orc_heap* h, uint32_t n, uint64_t bytes, uint64_t* out_off,
                                int32_t* out_status) {
    if (n == 0 || n > 64) return OURO_ERR_USAGE;
    std::vector<Lane> L(n);
    for (u32 i = 0; i < n; ++i) { L[i].off = bytes; L[i].st = 0; }
    h->alloc_group(L.data(), n);
    bool all = true;
    for (u32 i = 0; i < n; ++i) all = all && L[i].st == OURO_OK;
    if (!all) {
        std::vector<Lane> R;
        for (u32 i = 0; i < n; ++i)
            if (L[i].st == OURO_OK) R.push_back(L[i]);
        if (!R.empty()) h->free_group(R.data(), (u32)R.size());
        const int32_t st = L[0].st == OURO_ERR_TOO_LARGE ? OURO_ERR_TOO_LARGE : OURO_ERR_OOM;
        for (u32 i = 0; i < n; ++i) { out_off[i] = ~0ull; out_status[i] = st; }
        return OURO_OK;
    }
    for (u32 i = 0; i < n; ++i) { out_off[i] = L[i].off; out_status[i] = OURO_OK; }
    return OURO_OK;
}

ouro_status orc_run_script(orc_heap* h, const ouro_script_step* steps, uint32_t nsteps,
                           uint64_t* out_offset, int32_t* out_status) {
    for (u32 s = 0; s < nsteps; ++s) {
        const ouro_script_step& st = steps[s];
        std::vector<Lane> L;
        std::vector<u32> lane;
        for (u32 i = 0; i < 32; ++i) {
            out_offset[s * 32 + i] = ~0ull;
            out_status[s * 32 + i] = -1;
            if (!(st.lane_mask >> i & 1)) continue;
            Lane l{};
            if (st.op != 1) {
                l.off = st.arg[i];
            } else {
                const u64 a = st.arg[i];
                if (a >> 63) l.off = a & ~(1ull << 63);
                else l.off = a < (u64)s * 32 ? out_offset[a] : ~0ull;
                if (l.off == ~0ull) l.off = ~1ull;  // freeing a failed alloc: invalid handle
            }
            L.push_back(l);
            lane.push_back(i);
        }
        if (L.empty()) continue;
        if (st.op == 0 || st.op == 2) h->alloc_group(L.data(), (u32)L.size());
        else h->free_group(L.data(), (u32)L.size());
        if (st.op == 2) {  // alloc_coalesced: all-or-nothing
            bool all = true;
            for (auto& l : L) all = all && l.st == OURO_OK;
            if (!all) {
                std::vector<Lane> R;
                for (auto& l : L) if (l.st == OURO_OK) R.push_back(l);
                if (!R.empty()) h->free_group(R.data(), (u32)R.size());
                const int32_t code = L[0].st == OURO_ERR_TOO_LARGE ? OURO_ERR_TOO_LARGE : OURO_ERR_OOM;
                for (auto& l : L) { l.st = code; l.off = ~0ull; }
            }
        }
        for (u32 j = 0; j < L.size(); ++j) {
            if (st.op != 1) out_offset[s * 32 + lane[j]] = L[j].off;
            out_status[s * 32 + lane[j]] = L[j].st;
        }
    }
    return OURO_OK;
}

// page_region.
ouro_status orc_page_region(orc_heap* h, uint32_t handle, uint64_t* off, uint64_t* len) {
    const Geo& g = h->g;
    const u64 c = (u64)handle >> g.page_bits;
    const u32 p = handle & ((1u << g.page_bits) - 1);
    if (c >= g.N) return OURO_ERR_RANGE;
    const u64 m = A(h->meta[c]).load(ACQ);
    const u32 st = orc_heap::m_state(m);
    if (st == ST_UNASSIGNED || st == ST_RESERVED || st > g.K) return OURO_ERR_INVALID_HANDLE;
    const u32 k = st - 1;
    if (p >= g.ppc(k)) return OURO_ERR_INVALID_HANDLE;
    *off = h->offset_of((u32)c, k, p);
    *len = g.page_bytes(k);
    return OURO_OK;
}

}  // extern "C"

namespace {
// Walk a quiescent queue's live tickets [head, tail).
template <class F>
void for_each_queued(orc_heap* h, Queue& Q, F f) {
    Arena& ar = h->ar;
    // VirtualList: one walk along the list as the tickets advance (segment order)
    u32 cur = (u32)Q.vl_head, i = (u32)(Q.vl_head >> 32);
    for (u64 t = Q.head; t < Q.tail; ++t) {
        u64 x;
        if (Q.flavor == OURO_FLAVOR_ARRAY) {
            x = Q.slots[t & Q.ring_mask];
        } else if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) {
            const u64 s = t / ar.S_va();
            const u64 e = Q.dir[s % Q.D];
            if ((u32)e == NONE) continue;
            x = ar.cw((u32)e)[t % ar.S_va()];
        } else {
            const u64 s = t / ar.S_vl();
            while (cur != NONE && i != (u32)s) {
                const u64 nx = ar.cw(cur)[0];
                cur = nx == NONE_LINK ? NONE : (u32)nx;
                ++i;
            }
            if (cur == NONE) continue;
            x = ar.cw(cur)[2 + t % ar.S_vl()];
        }
        f((u32)x);
    }
}
template <class F>
void for_each_segment(orc_heap* h, Queue& Q, F f) {
    Arena& ar = h->ar;
    if (Q.flavor == OURO_FLAVOR_VIRTUAL_ARRAY) {
        for (u32 i = 0; i < Q.D; ++i) if ((u32)Q.dir[i] != NONE) f((u32)Q.dir[i]);
    } else if (Q.flavor == OURO_FLAVOR_VIRTUAL_LIST) {
        u32 cur = (u32)Q.vl_head;
        u32 guard = 0;
        while (cur != NONE && guard++ < (1u << 26)) {
            f(cur);
            const u64 nx = ar.cw(cur)[0];
            cur = nx == NONE_LINK ? NONE : (u32)nx;
        }
    }
}
u64 hmix(u64 a, u64 b) { return mix64(a * 0x9E3779B97F4A7C15ull + mix64(b)); }
}  // namespace

extern "C" {

ouro_status orc_stats(orc_heap* h, ouro_stats* out) {
    std::memset(out, 0, sizeof(*out));
    const Geo& g = h->g;
    out->num_classes = g.K;
    out->num_chunks = g.N;
    out->sticky_first = h->ar.err.first;
    out->sticky_mask = h->ar.err.mask;
    out->stale_drops = h->ar.err.stale_drops;
    out->double_frees = h->ar.err.double_frees;
    out->invalid_frees = h->ar.err.invalid_frees;
    out->bad_sizes = h->ar.err.bad_sizes;
    out->timeouts = h->ar.err.timeouts;
    out->corruptions = h->ar.err.corruptions;
    if (h->kind == OURO_KIND_CHUNK) out->pool_len = (u64)h->ar.q[h->pool_idx()].count;
    for (u32 k = 0; k < g.K; ++k) {
        ouro_class_stats& cs = out->cls[k];
        cs.page_bytes = g.page_bytes(k);
        cs.pages_per_chunk = g.ppc(k);
        cs.retries = h->retries[k];
        cs.ooms = h->ooms[k];
        Queue& Q = h->ar.q[k];
        cs.queue_len = (u64)Q.count;
        cs.seg_live = Q.seg_live;
        cs.seg_hwm = Q.seg_hwm;
    }
    for (u32 c = 0; c < g.N; ++c) {
        const u64 m = h->meta[c];
        const u32 st = orc_heap::m_state(m);
        if (st == ST_UNASSIGNED || st == ST_RESERVED || st > g.K) continue;
        const u32 k = st - 1;
        out->cls[k].chunks += 1;
        out->cls[k].live_pages += g.ppc(k) - orc_heap::m_free(m);
    }
    for (u32 k = 0; k < g.K; ++k) {
        Queue& Q = h->ar.q[k];
        u64 live = 0;
        for_each_queued(h, Q, [&](u32 v) {
            if (h->kind == OURO_KIND_PAGE) { ++live; return; }
            const u32 c = v & g.cmask;
            const u32 glow = g.chunk_bits >= 32 ? 0 : v >> g.chunk_bits;
            const u64 m = h->meta[c];
            if (orc_heap::m_state(m) == k + 1 && (orc_heap::m_gen(m) & g.gmask) == glow) ++live;
        });
        out->cls[k].queued_live = live;
    }
    return OURO_OK;
}

// Canonical digest.  Quiescent only.
ouro_status orc_digest(orc_heap* h, ouro_digest* d) {
    std::memset(d, 0, sizeof(*d));
    const Geo& g = h->g;
    d->num_chunks = g.N;
    d->num_classes = g.K;
    d->sticky_mask = h->ar.err.mask;
    std::vector<u32> where(g.N, 0);
    bool ok = true;
    u64 assigned_total = 0;
    for (u32 c = 0; c < g.N; ++c) {
        const u64 m = h->meta[c];
        const u32 st = orc_heap::m_state(m);
        const u64* b = h->bm(c);
        u64 bh = 0;
        for (u32 w = 0; w < g.Wmax; ++w) bh = hmix(bh ^ w, b[w]);
        if (h->kind == OURO_KIND_PAGE) {
            d->header_hash += hmix(hmix(c, m), bh);
        } else {
            d->header_hash += hmix(m & 0xFFFFFFFFFFull, bh);  // generation excluded
        }
        if (st == ST_RESERVED) continue;
        if (st == ST_UNASSIGNED) {
            if (orc_heap::m_free(m) != 0) ok = false;
            for (u32 w = 0; w < g.Wmax; ++w) if (b[w]) ok = false;
            continue;
        }
        if (st > g.K) { ok = false; continue; }
        const u32 k = st - 1;
        ++where[c];
        ++assigned_total;
        d->class_chunks[k] += 1;
        const u64 live = g.ppc(k) - orc_heap::m_free(m);
        d->class_live_pages[k] += live;
        d->live_pages += live;
        u64 pc = 0;
        for (u32 w = 0; w < g.Wmax; ++w) pc += (u64)std::popcount(b[w]);
        if (g.ppc(k) - pc != orc_heap::m_free(m)) ok = false;  // allocated bits = live pages
    }
    if (h->kind == OURO_KIND_CHUNK) {
        for_each_queued(h, h->ar.q[h->pool_idx()], [&](u32 c) { if (c < g.N) ++where[c]; else ok = false; });
        std::vector<u32> entries(g.N, 0);
        for (u32 k = 0; k < g.K; ++k) {
            Queue& Q = h->ar.q[k];
            for_each_segment(h, Q, [&](u32 c) { if (c < g.N) ++where[c]; else ok = false; });
            for_each_queued(h, Q, [&](u32 v) {
                const u32 c = v & g.cmask;
                const u32 glow = g.chunk_bits >= 32 ? 0 : v >> g.chunk_bits;
                const u64 m = h->meta[c];
                if (orc_heap::m_state(m) == k + 1 && (orc_heap::m_gen(m) & g.gmask) == glow) {
                    ++entries[c];
                    d->class_queued_live[k] += 1;
                }
            });
        }
        for (u32 c = 0; c < g.N; ++c) {
            const u64 m = h->meta[c];
            const u32 st = orc_heap::m_state(m);
            const bool has_free = st >= 1 && st <= g.K && orc_heap::m_free(m) > 0;
            if (entries[c] != (has_free ? 1u : 0u)) ok = false;
        }
        d->queue_hash = 0;
    } else {
        for (u32 k = 0; k < g.K; ++k) {
            Queue& Q = h->ar.q[k];
            if (h->flavor != OURO_FLAVOR_ARRAY) {
                for_each_segment(h, Q, [&](u32 c) { if (c < g.N) ++where[c]; else ok = false; });
                for_each_queued(h, h->ar.q[h->priv_idx(k)], [&](u32 c) { if (c < g.N) ++where[c]; else ok = false; });
            }
            for_each_queued(h, Q, [&](u32 hd) {
                d->queue_hash += hmix(k + 1, hd);
                d->class_queued_live[k] += 1;
            });
        }
    }
    for (u32 c = 0; c < g.N; ++c) {
        const u32 st = orc_heap::m_state(h->meta[c]);
        if (h->kind == OURO_KIND_CHUNK || st != ST_RESERVED || h->flavor != OURO_FLAVOR_ARRAY) {
            if (where[c] != 1) ok = false;
        }
    }
    d->unassigned_chunks = g.N - assigned_total;
    d->partition_ok = ok ? 1 : 0;
    return OURO_OK;
}

uint64_t orc_queue_ops(orc_heap* h) { return h->ar.queue_ops; }
uint64_t orc_pool_dequeues(orc_heap* h) { return h->pool_dequeues; }

// ---- chunk module ops, single-page forms ----
ouro_status orc_chunk_assign(orc_heap* h, uint32_t c, uint32_t cls, uint32_t* gen) {
    if (c >= h->g.N || cls >= h->g.K) return OURO_ERR_RANGE;
    const u64 m = h->meta[c];
    if (orc_heap::m_state(m) != ST_UNASSIGNED) return OURO_ERR_ALREADY_ASSIGNED;
    const u32 ppc = h->g.ppc(cls);
    const u32 ng = (orc_heap::m_gen(m) + 1) & 0xFFFFFF;
    h->meta[c] = orc_heap::mk(ng, cls + 1, ppc);  // bitmap already all-zero (all free)
    h->assigned[cls] += 1;
    if (gen) *gen = ng;
    return OURO_OK;
}
ouro_status orc_chunk_acquire(orc_heap* h, uint32_t c, uint32_t* page) {
    if (c >= h->g.N) return OURO_ERR_RANGE;
    u64 m = A(h->meta[c]).load(ACQ);
    for (;;) {
        const u32 st = orc_heap::m_state(m);
        if (st == ST_UNASSIGNED || st > h->g.K) return OURO_ERR_INVALID_HANDLE;
        if (orc_heap::m_free(m) == 0) return OURO_ERR_CHUNK_FULL;
        if (A(h->meta[c]).compare_exchange_weak(m, m - 1, AR, ACQ)) break;
    }
    u32 p;
    if (h->claim_lowest(c, orc_heap::m_state(m) - 1, 1, &p) != 1) return OURO_ERR_CORRUPTION;
    *page = p;
    return OURO_OK;
}
ouro_status orc_chunk_release(orc_heap* h, uint32_t c, uint32_t page, uint32_t* occ_after) {
    if (c >= h->g.N) return OURO_ERR_RANGE;
    const u64 m0 = A(h->meta[c]).load(ACQ);
    const u32 st = orc_heap::m_state(m0);
    if (st == ST_UNASSIGNED || st > h->g.K || page >= h->g.ppc(st - 1)) return OURO_ERR_INVALID_HANDLE;
    const u64 bit = 1ull << (page & 63);
    const u64 old = A(h->bm(c)[page >> 6]).fetch_and(~bit, AR);
    if (!(old & bit)) return OURO_ERR_DOUBLE_FREE;
    const u64 m = A(h->meta[c]).fetch_add(1, AR);
    *occ_after = orc_heap::m_free(m) + 1;
    return OURO_OK;
}
ouro_status orc_chunk_unassign(orc_heap* h, uint32_t c) {
    if (c >= h->g.N) return OURO_ERR_RANGE;
    const u64 m = h->meta[c];
    const u32 st = orc_heap::m_state(m);
    if (st == ST_UNASSIGNED || st > h->g.K) return OURO_ERR_INVALID_HANDLE;
    if (orc_heap::m_free(m) != h->g.ppc(st - 1)) return OURO_ERR_USAGE;
    h->meta[c] = orc_heap::mk(orc_heap::m_gen(m), ST_UNASSIGNED, 0);  // bitmap already zero
    h->assigned[st - 1] -= 1;
    return OURO_OK;
}
ouro_status orc_chunk_state(orc_heap* h, uint32_t c, uint32_t* state, uint32_t* free_count,
                            uint32_t* gen, uint64_t* bitmap_popcount) {
    if (c >= h->g.N) return OURO_ERR_RANGE;
    const u64 m = h->meta[c];
    *state = orc_heap::m_state(m);
    *free_count = orc_heap::m_free(m);
    *gen = orc_heap::m_gen(m);
    u64 pc = 0;
    for (u32 w = 0; w < h->g.Wmax; ++w) pc += (u64)std::popcount(h->bm(c)[w]);
    const u32 st = orc_heap::m_state(m);
    *bitmap_popcount = (st >= 1 && st <= h->g.K) ? h->g.ppc(st - 1) - pc : 0;  // free pages
    return OURO_OK;
}

// ---- standalone queue ----
}  // extern "C"

struct orc_qt {
    Arena ar;
    u64 cap;
};

extern "C" {

ouro_status orc_qt_new(uint8_t flavor, uint64_t capacity, uint32_t pool_chunks,
                       uint64_t chunk_bytes, orc_qt** out) {
    // queue_new: capacity 0 -> ConfigError; virtual needs a pool.
    if (capacity == 0 || flavor > 2) return OURO_ERR_CONFIG;
    if (flavor != OURO_FLAVOR_ARRAY && (pool_chunks == 0 || chunk_bytes < 32 || !pow2(chunk_bytes)))
        return OURO_ERR_CONFIG;
    auto* q = new orc_qt();
    q->cap = capacity;
    q->ar.chunk_bytes = chunk_bytes ? chunk_bytes : 64;
    q->ar.words_per_chunk = q->ar.chunk_bytes / 8;
    const u32 pc = std::max<u32>(pool_chunks, 1);
    q->ar.words = static_cast<u64*>(std::calloc((size_t)pc * q->ar.words_per_chunk, 8));
    q->ar.q.resize(2);
    q->ar.init_queue(q->ar.q[1], OURO_FLAVOR_ARRAY, pc, -1);
    q->ar.prefill(q->ar.q[1], pool_chunks, pool_val, nullptr, nullptr, 0);
    q->ar.init_queue(q->ar.q[0], flavor, capacity, 1);
    *out = q;
    return OURO_OK;
}
void orc_qt_destroy(orc_qt* q) {
    if (!q) return;
    std::free(q->ar.words);
    delete q;
}
ouro_status orc_qt_enqueue(orc_qt* q, uint32_t v) {
    return q->ar.enq1(q->ar.q[0], v) ? OURO_OK : OURO_ERR_FULL;
}
ouro_status orc_qt_dequeue(orc_qt* q, uint32_t* v) {
    return q->ar.deq1(q->ar.q[0], 0, v) ? OURO_OK : OURO_ERR_EMPTY;
}
uint64_t orc_qt_len(orc_qt* q) { return (u64)A(q->ar.q[0].count).load(ACQ); }
uint64_t orc_qt_pool_len(orc_qt* q) { return (u64)A(q->ar.q[1].count).load(ACQ); }
uint64_t orc_qt_seg_live(orc_qt* q) { return A(q->ar.q[0].seg_live).load(ACQ); }

ouro_status orc_qt_mt_churn(orc_qt* q, uint32_t producers, uint32_t consumers, uint32_t per,
                            uint32_t* hist, double timeout_s) {
    const u64 total = (u64)producers * per;
    std::atomic<u64> delivered{0};
    std::atomic<bool> fail{false};
    const auto t0 = std::chrono::steady_clock::now();
    auto late = [&] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s;
    };
    std::vector<std::thread> th;
    for (u32 p = 0; p < producers; ++p)
        th.emplace_back([&, p] {
            for (u32 i = 0; i < per && !fail; ++i) {
                const u32 v = p * per + i;
                while (orc_qt_enqueue(q, v) != OURO_OK) {
                    if (late()) { fail = true; return; }
                    std::this_thread::yield();
                }
            }
        });
    for (u32 c = 0; c < consumers; ++c)
        th.emplace_back([&] {
            while (delivered.load() < total && !fail) {
                u32 v;
                if (orc_qt_dequeue(q, &v) == OURO_OK) {
                    if (v < total) std::atomic_ref<u32>(hist[v]).fetch_add(1);
                    delivered.fetch_add(1);
                } else {
                    if (late()) { fail = true; return; }
                    std::this_thread::yield();
                }
            }
        });
    for (auto& t : th) t.join();
    return fail ? OURO_ERR_TIMEOUT : OURO_OK;
}

// ---- coalesce: LaneGroup with a generation-counted barrier + timeout
ouro_status orc_active_mask(uint32_t width, const int32_t* active, uint32_t timeout_ms,
                            uint64_t* mask_out) {
    if (width == 0 || width > 64) return OURO_ERR_USAGE;
    std::mutex mu;
    std::condition_variable cv;
    u32 arrived = 0;
    u64 acc = 0;
    bool timed_out = false;
    std::vector<u64> got(width, 0);
    std::vector<std::thread> th;
    for (u32 i = 0; i < width; ++i) {
        if (active[i] < 0) continue;  // never arrives (the paper's deadlock)
        th.emplace_back([&, i] {
            std::unique_lock<std::mutex> lk(mu);
            acc |= active[i] ? (1ull << i) : 0;  // contribute 1<<lane or 0
            ++arrived;
            if (arrived == width) cv.notify_all();
            if (!cv.wait_for(lk, std::chrono::milliseconds(timeout_ms), [&] { return arrived == width; }))
                timed_out = true;
            got[i] = acc;
        });
    }
    for (auto& t : th) t.join();
    if (timed_out) return OURO_ERR_TIMEOUT;
    for (u32 i = 0; i < width; ++i)
        if (got[i] != acc) return OURO_ERR_CORRUPTION;
    *mask_out = acc;
    return OURO_OK;
}

// ---- bench on CPU threads behind a start barrier ----
}  // extern "C"
namespace {
struct Barrier {
    std::mutex m;
    std::condition_variable cv;
    u32 n, waiting = 0;
    u64 gen = 0;
    explicit Barrier(u32 n_) : n(n_) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m);
        const u64 g = gen;
        if (++waiting == n) { waiting = 0; ++gen; cv.notify_all(); return; }
        cv.wait(lk, [&] { return gen != g; });
    }
};
}  // namespace
extern "C" {

ouro_status orc_bench_trial(orc_heap* h, uint64_t n, uint64_t bytes, const uint32_t* sizes,
                            uint32_t iterations, uint32_t threads, uint64_t seed,
                            orc_trial_out* out) {
    if (iterations < 1 || iterations > 64 || threads == 0) return OURO_ERR_USAGE;
    std::memset(out, 0, sizeof(*out));
    out->threads = threads;
    std::vector<u64> offs(n, ~0ull);
    std::atomic<u64> ok{0}, bad{0}, mism{0};
    Barrier bar(threads + 1);
    std::atomic<int> phase{0};
    std::atomic<u32> it_now{0};
    u8* base = reinterpret_cast<u8*>(h->ar.words);
    auto work = [&](u32 tid) {
        for (;;) {
            bar.wait();
            const int ph = phase.load();
            if (ph < 0) return;
            const u32 it = it_now.load();
            for (u64 i = tid; i < n; i += threads) {
                if (ph == 1) {
                    Lane l{};
                    l.off = sizes ? sizes[i] : bytes;
                    h->alloc_group(&l, 1);
                    offs[i] = l.st == OURO_OK ? l.off : ~0ull;
                    (l.st == OURO_OK ? ok : bad).fetch_add(1, RLX);
                } else if (ph == 2) {
                    if (offs[i] == ~0ull) continue;
                    u64 len; u64 off;
                    const u32 c = (u32)(offs[i] >> h->g.chunk_shift);
                    const u32 k = orc_heap::m_state(h->meta[c]) - 1;
                    len = h->g.page_bytes(k); off = offs[i];
                    const u64 b = pattern_base(seed, i, it);
                    u64* w = reinterpret_cast<u64*>(base + off);
                    for (u64 j = 0; j < len / 8; ++j) w[j] = pattern_word(b, j);
                } else if (ph == 3) {
                    if (offs[i] == ~0ull) continue;
                    const u32 c = (u32)(offs[i] >> h->g.chunk_shift);
                    const u32 k = orc_heap::m_state(h->meta[c]) - 1;
                    const u64 len = h->g.page_bytes(k);
                    const u64 b = pattern_base(seed, i, it);
                    const u64* w = reinterpret_cast<const u64*>(base + offs[i]);
                    u64 bad_words = 0;
                    for (u64 j = 0; j < len / 8; ++j) bad_words += w[j] != pattern_word(b, j);
                    if (bad_words) mism.fetch_add(bad_words, RLX);
                } else if (ph == 4) {
                    if (offs[i] == ~0ull) continue;
                    Lane l{};
                    l.off = offs[i];
                    h->free_group(&l, 1);
                    offs[i] = ~0ull;
                }
            }
            bar.wait();
        }
    };
    std::vector<std::thread> th;
    for (u32 t = 0; t < threads; ++t) th.emplace_back(work, t);
    auto run_phase = [&](int ph) {
        phase = ph;
        const auto t0 = std::chrono::steady_clock::now();
        bar.wait();  // start barrier
        bar.wait();  // join
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    for (u32 it = 0; it < iterations; ++it) {
        it_now = it;
        out->alloc_ms[it] = run_phase(1);
        run_phase(2);
        run_phase(3);
        out->free_ms[it] = run_phase(4);
    }
    phase = -1;
    bar.wait();
    for (auto& t : th) t.join();
    out->ok_allocs = ok;
    out->failed_allocs = bad;
    out->verified = mism.load() == 0 ? 1 : 0;
    return OURO_OK;
}

// Mixed churn (BASELINE configs[3]).  Slot semantics: occupied & h&1 -> free;
// empty -> malloc(8 + (h>>1) % 4089) and stamp the first word; occupied & !(h&1)
// -> check the stamp.
ouro_status orc_churn(orc_heap* h, uint64_t n, uint32_t round_begin, uint32_t rounds,
                      uint64_t seed, uint32_t threads, uint64_t* slots, ouro_churn_result* out,
                      double* ms) {
    std::memset(out, 0, sizeof(*out));
    std::atomic<u64> mok{0}, mbad{0}, fr{0}, chk{0};
    u8* base = reinterpret_cast<u8*>(h->ar.words);
    const auto t0 = std::chrono::steady_clock::now();
    for (u32 r = round_begin; r < round_begin + rounds; ++r) {
        std::vector<std::thread> th;
        for (u32 tid = 0; tid < threads; ++tid)
            th.emplace_back([&, tid] {
                for (u64 t = tid; t < n; t += threads) {
                    const u64 hh = mix64(seed ^ (t << 32) ^ r);
                    u64& s = slots[t];
                    if (s != ~0ull && (hh & 1)) {
                        Lane l{};
                        l.off = s;
                        h->free_group(&l, 1);
                        s = ~0ull;
                        fr.fetch_add(1, RLX);
                    } else if (s == ~0ull) {
                        Lane l{};
                        l.off = 8 + (hh >> 1) % 4089;
                        h->alloc_group(&l, 1);
                        if (l.st == OURO_OK) {
                            s = l.off;
                            *reinterpret_cast<u64*>(base + s) = mix64(t ^ seed);
                            mok.fetch_add(1, RLX);
                        } else {
                            mbad.fetch_add(1, RLX);
                        }
                    } else {
                        if (*reinterpret_cast<u64*>(base + s) != mix64(t ^ seed)) chk.fetch_add(1, RLX);
                    }
                }
            });
        for (auto& x : th) x.join();
    }
    if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    out->mallocs_ok = mok;
    out->mallocs_failed = mbad;
    out->frees = fr;
    out->check_failures = chk;
    return OURO_OK;
}

// The GPU driver phases' demand on the oracle: n slots in warp groups of `group`
// lanes, slot order, one thread (deterministic).  Slot i requests sizes[i] (or
// `bytes`); out[i] = heap offset or ~0 on failure.  Returns the success count.
ouro_status orc_alloc_slots(orc_heap* h, uint64_t n, uint64_t bytes, const uint32_t* sizes, uint32_t group,
                            uint64_t* out, uint64_t* ok) {
    if (group == 0 || group > 64) return OURO_ERR_USAGE;
    std::vector<Lane> L(group);
    u64 good = 0;
    for (u64 i = 0; i < n; i += group) {
        const u32 m = (u32)std::min<u64>(group, n - i);
        for (u32 j = 0; j < m; ++j) { L[j] = Lane{}; L[j].off = sizes ? sizes[i + j] : bytes; }
        h->alloc_group(L.data(), m);
        for (u32 j = 0; j < m; ++j) {
            out[i + j] = L[j].st == OURO_OK ? L[j].off : ~0ull;
            good += L[j].st == OURO_OK;
        }
    }
    if (ok) *ok = good;
    return OURO_OK;
}
// Free the non-~0 offsets of n slots in warp groups of `group` lanes (slot order).
ouro_status orc_free_slots(orc_heap* h, uint64_t n, const uint64_t* offs, uint32_t group) {
    if (group == 0 || group > 64) return OURO_ERR_USAGE;
    std::vector<Lane> L(group);
    for (u64 i = 0; i < n; i += group) {
        u32 m = 0;
        for (u64 j = i; j < std::min<u64>(i + group, n); ++j)
            if (offs[j] != ~0ull) { L[m] = Lane{}; L[m].off = offs[j]; ++m; }
        if (m) h->free_group(L.data(), m);
    }
    return OURO_OK;
}

ouro_status orc_free_all(orc_heap* h, uint64_t n, uint64_t* slots) {
    for (u64 i = 0; i < n; ++i) {
        if (slots[i] == ~0ull) continue;
        Lane l{};
        l.off = slots[i];
        h->free_group(&l, 1);
        slots[i] = ~0ull;
    }
    return OURO_OK;
}

}  // extern "C"
