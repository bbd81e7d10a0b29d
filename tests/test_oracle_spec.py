"""The SPEC's known-answer examples and acceptance criteria, run against the
oracle (CPU only).  Each test cites the SPEC line it pins.
The same behaviours are checked on the GPU through parity with this oracle
(tests/test_gpu_*.py)."""
import ctypes as C
import json
import os
import random
import time

import pytest

from helpers import NAMES, VARIANTS, cfg
from oracle_lib import OHeap, TrialOut, oracle

OK, INVALID, DOUBLE, RANGE, TIMEOUT, CORRUPT, OOM, TOO_LARGE = 0, 2, 3, 4, 5, 6, 7, 8
FULL, EMPTY, CHUNK_FULL, ALREADY = 10, 11, 12, 13
KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_kats.json")))


# ------------------------------------------------------------------ queues
class Q:
    def __init__(self, flavor, cap, pool=64, chunk=256):
        self.L = oracle()
        h = C.c_void_p()
        self.st = self.L.orc_qt_new(flavor, cap, pool, chunk, C.byref(h))
        self.h = h

    def enq(self, v):
        return self.L.orc_qt_enqueue(self.h, v)

    def deq(self):
        v = C.c_uint32()
        st = self.L.orc_qt_dequeue(self.h, C.byref(v))
        return st, v.value

    def __len__(self):
        return self.L.orc_qt_len(self.h)

    def close(self):
        self.L.orc_qt_destroy(self.h)


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_queue_examples(flavor):
    q = Q(flavor, 8)
    assert q.st == OK and len(q) == 0                       # SPEC.md:133, 157 (fresh -> 0)
    assert q.deq()[0] == EMPTY
    assert q.enq(7) == OK and q.deq() == (OK, 7)
    for v in (1, 2, 3):
        assert q.enq(v) == OK
    assert len(q) == 3
    assert [q.deq()[1] for _ in range(3)] == [1, 2, 3]      # SPEC.md:151 FIFO
    q.close()
    q = Q(flavor, 1)
    assert q.enq(1) == OK and q.enq(2) == FULL
    q.close()


def test_queue_new_errors():
    assert Q(2, 0).st == 1                                  # SPEC.md:135 capacity 0 -> ConfigError
    assert Q(1, 16, pool=0).st == 1                         # SPEC.md:131 virtual without pool
    q = Q(1, 4096)                                          # lazy, 0 segments
    assert q.st == OK and q.L.orc_qt_seg_live(q.h) == 0
    q.close()


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_queue_flavour_equivalence(flavor):
    """identical outputs across flavours for a random sequence."""
    rng = random.Random(42)
    ops = [(rng.random() < 0.55, rng.randrange(1 << 20)) for _ in range(5000)]
    outs = {}
    for fl in (0, 1, 2):
        q = Q(fl, 300, pool=64, chunk=256)
        outs[fl] = [q.enq(v) if e else q.deq() for e, v in ops]
        q.close()
    assert outs[0] == outs[1] == outs[2]


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_queue_multiset_union(flavor):
    """N producers enqueue disjoint sets; drain -> exact union."""
    q = Q(flavor, 8 * 1000, pool=256, chunk=256)
    L = q.L
    hist = (C.c_uint32 * 8000)()
    assert L.orc_qt_mt_churn(q.h, 8, 1, 1000, hist, 60.0) == OK
    assert all(h == 1 for h in hist)
    q.close()


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_queue_mpmc_churn(flavor):
    """8P/8C churn, every element delivered exactly once
    (10^5 elements per flavour keeps the CPU suite fast)."""
    q = Q(flavor, 4096, pool=512, chunk=512)
    hist = (C.c_uint32 * 100000)()
    assert q.L.orc_qt_mt_churn(q.h, 8, 8, 12500, hist, 120.0) == OK
    assert all(h == 1 for h in hist)
    assert len(q) == 0
    q.close()


# ------------------------------------------------------------------- chunk
def _chunk_heap():
    return OHeap(cfg(1, 0, 1 << 20))


def test_chunk_examples():
    h = _chunk_heap()
    L = h.L
    gen = C.c_uint32()
    st, fc, g, pc = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
    assert L.orc_chunk_assign(h.h, 0, 6, C.byref(gen)) == OK          # class 1024
    L.orc_chunk_state(h.h, 0, C.byref(st), C.byref(fc), C.byref(g), C.byref(pc))
    assert fc.value == 64 and pc.value == 64
    assert L.orc_chunk_assign(h.h, 0, 6, C.byref(gen)) == ALREADY
    pages = []
    for _ in range(64):
        p = C.c_uint32()
        assert L.orc_chunk_acquire(h.h, 0, C.byref(p)) == OK
        pages.append(p.value)
    assert sorted(pages) == list(range(64))                           # SPEC.md:208 distinct
    p = C.c_uint32()
    assert L.orc_chunk_acquire(h.h, 0, C.byref(p)) == CHUNK_FULL      # 65th
    occ = C.c_uint32()
    assert L.orc_chunk_release(h.h, 0, 3, C.byref(occ)) == OK and occ.value == 1
    assert L.orc_chunk_release(h.h, 0, 3, C.byref(occ)) == DOUBLE
    for q in pages:
        if q != 3:
            assert L.orc_chunk_release(h.h, 0, q, C.byref(occ)) == OK
    assert occ.value == 64
    # drain, release-all, unassign, reassign to a different class
    assert L.orc_chunk_unassign(h.h, 0) == OK
    assert L.orc_chunk_assign(h.h, 0, 9, C.byref(gen)) == OK           # class 8192: 8 pages
    L.orc_chunk_state(h.h, 0, C.byref(st), C.byref(fc), C.byref(g), C.byref(pc))
    assert fc.value == 8 and pc.value == 8 and g.value == 2
    h.close()


def test_chunk_one_page():
    """a 1-page chunk (chunk = page = 8192)."""
    h = OHeap(cfg(1, 0, 1 << 16, 8192, 16, 8192))
    L = h.L
    gen, p = C.c_uint32(), C.c_uint32()
    assert L.orc_chunk_assign(h.h, 0, 9, C.byref(gen)) == OK
    assert L.orc_chunk_acquire(h.h, 0, C.byref(p)) == OK and p.value == 0
    assert L.orc_chunk_acquire(h.h, 0, C.byref(p)) == CHUNK_FULL
    h.close()


def test_chunk_trace_vs_bitset():
    """random acquire/release interleave vs a reference bitset."""
    h = _chunk_heap()
    L = h.L
    gen = C.c_uint32()
    L.orc_chunk_assign(h.h, 1, 2, C.byref(gen))  # class 64 B: 1024 pages
    rng = random.Random(5)
    held = set()
    free = set(range(1024))
    for _ in range(20000):
        if held and (rng.random() < 0.5 or not free):
            q = rng.choice(sorted(held))
            occ = C.c_uint32()
            assert L.orc_chunk_release(h.h, 1, q, C.byref(occ)) == OK
            held.discard(q)
            free.add(q)
            assert occ.value == len(free)
        else:
            p = C.c_uint32()
            st = L.orc_chunk_acquire(h.h, 1, C.byref(p))
            if not free:
                assert st == CHUNK_FULL
                continue
            assert st == OK and p.value == min(free)  # lowest-free-bit scan
            free.discard(p.value)
            held.add(p.value)
    h.close()


# ------------------------------------------------------------- page_region
def test_page_region_examples():
    h = _chunk_heap()
    L = h.L
    gen = C.c_uint32()
    assert h.page_region(0)[0] == INVALID                             # SPEC.md:76 unassigned
    L.orc_chunk_assign(h.h, 0, 6, C.byref(gen))
    L.orc_chunk_assign(h.h, 1, 6, C.byref(gen))
    for row in KATS["page_region"]:
        handle = (row["chunk"] << 12) | row["page"]
        assert h.page_region(handle) == (OK, row["offset"], row["len"])
    assert h.page_region((0 << 12) | 64)[0] == INVALID                # page >= ppc
    assert h.page_region(16 << 12)[0] == RANGE                        # chunk out of grid
    h.close()


# -------------------------------------------------------------- allocators
def test_first_touch_chunk_stats():
    """fresh 16-chunk chunk allocator, alloc(1000)."""
    h = _chunk_heap()
    off, st = h.alloc([1000])
    assert st == [OK]
    s = h.stats()
    assert s.cls[6].chunks == 1 and s.cls[6].live_pages == 1 and s.pool_len == 15
    h.close()


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_page_capacity_64(flavor):
    """a Page class with exactly 64 pages -> 65th OOM, free one, next OK.
    (Virtual flavours self-host their segments in the class's chunks, gap G1, so
    they need a larger heap for the class to keep any pages.)"""
    h = OHeap(cfg(0, flavor, 1 << 20 if flavor == 0 else 8 << 20, retries=2))
    cap = h.stats().cls[6].queue_len
    offs = []
    for _ in range(cap):
        o, st = h.alloc([1000])
        assert st == [OK]
        offs.append(o[0])
    if flavor == 0:
        assert cap == 64
    assert h.alloc([1000])[1] == [OOM]
    assert h.free([offs[17]]) == [OK]
    assert h.alloc([1000]) == ([offs[17]], [OK])
    h.close()


@pytest.mark.parametrize("variant", VARIANTS, ids=[NAMES[v] for v in VARIANTS])
def test_double_free_and_invalid(variant):
    h = OHeap(cfg(*variant, 8 << 20))
    o, st = h.alloc([100])
    assert st == [OK]
    assert h.free(o) == [OK]
    assert h.free(o) == [DOUBLE]
    assert h.free([o[0] + 8]) == [INVALID]                           # misaligned
    assert h.free([1 << 40]) == [INVALID]                            # outside the heap
    assert h.free([o[0], o[0]])[1] in (DOUBLE, INVALID)              # duplicate inside one group
    assert h.alloc([0])[1] == [TOO_LARGE] and h.alloc([8193])[1] == [TOO_LARGE]  # SPEC.md:58, G5
    h.close()


@pytest.mark.parametrize("variant", VARIANTS, ids=[NAMES[v] for v in VARIANTS])
def test_rounds_restore_state(variant):
    """alloc-all/free-all x10 rounds -> final state equals the state
    after the first round (canonical digest)."""
    h = OHeap(cfg(*variant, 1 << 22))
    digests = []
    for r in range(10):
        offs = []
        for i in range(0, 1024, 32):
            o, st = h.alloc([1000] * 32)
            offs += [x for x, s in zip(o, st) if s == OK]
        for i in range(0, len(offs), 32):
            assert all(s == OK for s in h.free(offs[i:i + 32]))
        digests.append(h.digest().as_dict())
    assert all(d == digests[0] for d in digests)
    assert digests[0]["partition_ok"] == 1 and digests[0]["live_pages"] == 0
    h.close()


def test_page_rounds_restore_fresh():
    h = OHeap(cfg(0, 0, 1 << 20))
    fresh = h.digest().as_dict()
    offs, _ = h.alloc([16] * 32)
    h.free(offs)
    assert h.digest().as_dict() == fresh
    h.close()


# ---------------------------------------------------------------- coalesce
def test_active_mask_examples():
    L = oracle()
    for row in KATS["active_mask"]:
        w = row["width"]
        act = (C.c_int32 * w)(*[1 if (row["active"] == "all" or i in row["active"]) else 0 for i in range(w)])
        m = C.c_uint64()
        assert L.orc_active_mask(w, act, 2000, C.byref(m)) == OK
        assert m.value == row["mask"]


def test_active_mask_bruteforce():
    """SPEC.md:477 / criterion 7: all 2^8 activity patterns at width 8."""
    L = oracle()
    for pat in range(256):
        act = (C.c_int32 * 8)(*[(pat >> i) & 1 for i in range(8)])
        m = C.c_uint64()
        assert L.orc_active_mask(8, act, 2000, C.byref(m)) == OK
        assert m.value == pat


def test_active_mask_non_arriving_lane_times_out():
    """a lane that never arrives -> Timeout, not a hang (< 2 s)."""
    L = oracle()
    act = (C.c_int32 * 8)(1, 1, -1, 1, 0, 1, 1, 1)
    m = C.c_uint64()
    t0 = time.time()
    assert L.orc_active_mask(8, act, 300, C.byref(m)) == TIMEOUT
    assert time.time() - t0 < 2.0


def test_coalesced_examples():
    h = _chunk_heap()
    o1, s1 = h.alloc_coalesced(1, 1000)                               # 1 lane == alloc
    h2 = _chunk_heap()
    assert (o1, s1) == h2.alloc([1000])
    h2.close()
    q0, p0 = h.queue_ops(), h.pool_dequeues()
    offs, st = h.alloc_coalesced(32, 1000)
    assert st == [OK] * 32 and len(set(offs)) == 32
    assert all((o % 65536) % 1024 == 0 for o in offs)
    assert h.pool_dequeues() - p0 <= 1                                # <= 1 pool acquisition
    assert h.queue_ops() - q0 < 32                                    # criterion 7: fewer queue ops
    h.close()


def test_coalesced_all_or_nothing():
    """16 pages left, 32 lanes -> OOM for all, zero pages leaked."""
    h = OHeap(cfg(0, 0, 1 << 20, retries=2))                          # page kind: class 8192 = 8 pages
    before = h.digest().as_dict()
    offs, st = h.alloc_coalesced(32, 8192)
    assert st == [OOM] * 32 and all(o == 2 ** 64 - 1 for o in offs)
    after = h.digest().as_dict()
    assert after["live_pages"] == 0 and after["class_queued_live"] == before["class_queued_live"]
    h.close()


# ------------------------------------------------------------------- bench
def _trial(h, n, nbytes, iters, threads=4):
    out = TrialOut()
    assert oracle().orc_bench_trial(h.h, n, nbytes, None, iters, threads, 3, C.byref(out)) == OK
    return out


@pytest.mark.parametrize("variant", VARIANTS, ids=[NAMES[v] for v in VARIANTS])
@pytest.mark.parametrize("size", [16, 1000, 1024, 8192])
def test_acceptance_integrity(variant, size):
    """Criterion 1: 1024 allocations x {16,1000,1024,8192} B x 10
    iterations verify byte-exact and leave zero leaked pages."""
    # "arena sized to fit cfg demand with >= 2x headroom"; the page
    # kind gives each class 1/10 of the heap
    h = OHeap(cfg(*variant, (16 << 20) if size <= 1024 else (256 << 20)))
    out = _trial(h, 1024, size, 10)
    assert out.verified == 1 and out.failed_allocs == 0 and out.ok_allocs == 10240
    d = h.digest()
    assert d.live_pages == 0 and d.partition_ok == 1 and d.sticky_mask == 0
    h.close()


def test_trial_minimal_and_oom_resilience():
    h = OHeap(cfg(0, 0, 1 << 20, retries=2))
    out = _trial(h, 1, 16, 2)
    assert out.verified == 1 and out.ok_allocs == 2
    out = _trial(h, 200, 8192, 2)                                     # SPEC.md:387 / criterion 8
    assert out.failed_allocs > 0 and out.verified == 1
    out = _trial(h, 1024, 1000, 2)
    assert out.failed_allocs > 0 or out.ok_allocs > 0
    out = _trial(h, 8, 8192, 2)                                       # the heap is still usable
    assert out.failed_allocs == 0 and out.verified == 1


@pytest.mark.parametrize("variant", VARIANTS, ids=[NAMES[v] for v in VARIANTS])
def test_concurrency_churn_no_duplicates(variant):
    """Criterion 4, scaled: 8 threads x churn with random sizes;
    no duplicate grants (every live region verified by its stamp), no false
    DoubleFree, full drain restores the canonical state."""
    h = OHeap(cfg(*variant, 64 << 20))
    n = 8192
    slots = (C.c_uint64 * n)(*([2 ** 64 - 1] * n))
    from paper_2504_18211_b200._abi import ChurnResult
    res = ChurnResult()
    ms = C.c_double()
    assert oracle().orc_churn(h.h, n, 0, 12, 99, 8, slots, C.byref(res), C.byref(ms)) == OK
    assert res.check_failures == 0 and res.mallocs_ok > 0 and res.frees > 0
    s = h.stats()
    assert s.double_frees == 0 and s.invalid_frees == 0 and s.timeouts == 0 and s.corruptions == 0
    oracle().orc_free_all(h.h, n, slots)
    d = h.digest()
    assert d.live_pages == 0 and d.partition_ok == 1
    h.close()


def test_alloc_slots_page_capacities():
    """orc_alloc_slots (the oracle side of tests/test_gpu_baseline.py): on the BASELINE
    configs[1] heap the page kind serves min(n, capacity) of 2^20 requests, capacity =
    1638 chunks x pages per chunk above the 64 B class, and a free-all
    restores the initial digest."""
    h = OHeap(cfg(0, 0, 1 << 30, retries=4))
    d0 = h.digest().as_dict()
    n = 1 << 20
    for size, want in ((16, n), (128, 1638 * 512), (8192, 1638 * 8)):
        offs, ok = h.alloc_slots(n, size)
        assert ok == want
        assert sum(1 for x in offs if x != 2 ** 64 - 1) == ok
        h.free_slots(offs)
        assert h.digest().as_dict() == d0
    h.close()


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_churn_digest_independent_of_threads(flavor):
    """The chunk kind's free-all state after churn does not depend on the interleaving
    (one thread vs eight): the property the GPU churn parity test relies on."""
    digests, counts = [], []
    for threads in (1, 8):
        h = OHeap(cfg(1, flavor, 64 << 20))
        slots, res = h.churn(8192, 0, 10, 5, threads=threads)
        assert res.mallocs_failed == 0 and res.check_failures == 0
        counts.append((res.mallocs_ok, res.frees))
        h.free_all(slots)
        digests.append(h.digest().as_dict())
        h.close()
    assert counts[0] == counts[1]
    assert digests[0] == digests[1]
