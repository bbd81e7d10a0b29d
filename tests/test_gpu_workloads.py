"""GPU workloads through the C-ABI beyond op-script parity: the paper's driver
(run_trial), mixed churn (BASELINE configs[3]), OOM resilience, error paths at
scale, virtual-queue segment stress, and the BASELINE-sized heaps."""
import pytest

import paper_2504_18211_b200 as ob
from helpers import NAMES, VARIANTS
from oracle_lib import OHeap

pytestmark = pytest.mark.gpu
IDS = [NAMES[v] for v in VARIANTS]


def _hc(kind, flavor, heap, chunk=64 << 10, maxp=8192, retries=64, backoff=0):
    return ob.HeapConfig(heap, chunk, 16, maxp, ob.QueueFlavor(flavor), ob.AllocatorKind(kind),
                         ob.BackoffPolicy(backoff), retries)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_run_trial_paper_driver(cuda, variant):
    """SPEC.md:385 (PAPER): 1024 allocations x 1000 B x 10 iterations -> Pass,
    mean_subsequent over iterations 2..10."""
    with ob.Heap(_hc(*variant, 64 << 20)) as h:
        r = h.run_trial(1024, 1000, iterations=10, seed=3)
        assert r.verified == 1 and r.ok_allocs == 10240 and r.failed_allocs == 0
        assert r.mean_subsequent_ms == pytest.approx(sum(r.alloc_ms[1:10]) / 9)
        assert r.mean_all_ms == pytest.approx(sum(r.alloc_ms[:10]) / 10)
        assert h.last_error()[0] == 0
        d = h.digest()
        assert d.live_pages == 0 and d.partition_ok == 1


def test_run_trial_with_host_sizes(cuda):
    with ob.Heap(_hc(1, 0, 256 << 20)) as h:
        sizes = [(i * 37) % 4000 + 1 for i in range(20000)]
        r = h.run_trial(len(sizes), sizes=sizes, iterations=3)
        assert r.verified == 1 and r.ok_allocs == 3 * len(sizes) and r.h2d_bytes == 4 * len(sizes)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_oom_resilience(cuda, variant):
    """Criterion 8: a trial demanding more than capacity fails
    without aborting, and a normal trial afterwards passes."""
    torch = cuda
    kind, flavor = variant
    with ob.Heap(_hc(kind, flavor, 16 << 20, retries=8)) as h:
        n = 1 << 16
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=4096)          # 256 MiB demand into a 16 MiB heap
        h.launch_count(n, ptrs, cnt)
        torch.cuda.synchronize()
        ok = int(cnt)
        assert 0 < ok < n
        a = h.audit(n, ptrs)
        assert a.live == ok and a.overlaps == 0 and a.out_of_heap == 0 and a.misaligned == 0
        s = h.stats()
        assert sum(s.cls[k].ooms for k in range(s.num_classes)) == n - ok
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        r = h.run_trial(1024, 100, iterations=2)
        assert r.verified == 1 and r.failed_allocs == 0
        assert h.last_error()[0] == 0


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_double_free_at_scale(cuda, variant):
    """DoubleFree is surfaced, never silently ignored (errors.hpp:22-27): free
    every pointer twice from 65 536 threads."""
    torch = cuda
    with ob.Heap(_hc(*variant, 64 << 20)) as h:
        n = 1 << 16
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=48)
        h.launch_free(n, ptrs)
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        s = h.stats()
        first, mask = h.last_error(clear=True)
        if variant[0] == 0:
            assert s.double_frees == n and s.invalid_frees == 0
            assert first == ob._abi.ERR_DOUBLE_FREE and mask == 1 << ob._abi.ERR_DOUBLE_FREE
        else:
            # chunk kind: fully freed chunks went back to the pool, so a
            # second free into them is an InvalidHandle; pages of retained chunks are DoubleFree
            assert s.double_frees + s.invalid_frees == n and s.double_frees > 0
            assert mask & ~((1 << ob._abi.ERR_DOUBLE_FREE) | (1 << ob._abi.ERR_INVALID_HANDLE)) == 0
        d = h.digest()
        assert d.live_pages == 0 and d.partition_ok == 1


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_invalid_frees_at_scale(cuda, variant):
    torch = cuda
    with ob.Heap(_hc(*variant, 64 << 20)) as h:
        n = 1 << 15
        base = h.base
        bogus = torch.arange(n, dtype=torch.int64, device="cuda") * 64 + base + 8   # misaligned
        h.launch_free(n, bogus)
        out = torch.full((n,), base + (64 << 20) + 4096, dtype=torch.int64, device="cuda")  # outside
        h.launch_free(n, out)
        torch.cuda.synchronize()
        s = h.stats()
        assert s.invalid_frees == 2 * n and s.double_frees == 0
        h.last_error(clear=True)
        d = h.digest()
        assert d.live_pages == 0 and d.partition_ok == 1


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_churn(cuda, variant):
    """BASELINE configs[3] shape (scaled): mixed sizes 8 B-4 KiB, interleaved
    alloc/free rounds in one kernel per round; stamps checked every round;
    free-all restores the canonical state the oracle reaches."""
    torch = cuda
    kind, flavor = variant
    heap = 1 << 30
    n = 1 << 18
    with ob.Heap(_hc(kind, flavor, heap)) as h:
        slots = torch.zeros(n, dtype=torch.int64, device="cuda")
        res = torch.zeros(5, dtype=torch.int64, device="cuda")
        h.launch_churn(n, 0, 20, 1, slots, res)
        torch.cuda.synchronize()
        ok, failed, frees, reused, bad = [int(x) for x in res]
        assert bad == 0 and ok > 0 and frees > 0 and reused > 0
        a = h.audit(n, slots)
        assert a.overlaps == 0 and a.out_of_heap == 0 and a.misaligned == 0 and a.not_marked == 0
        h.launch_free(n, slots)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0
        d = h.digest().as_dict()
        assert d["live_pages"] == 0 and d["partition_ok"] == 1
        if kind == 0:
            oh = OHeap(_hc(kind, flavor, heap).to_c())
            assert d == oh.digest().as_dict()     # page kind: back to the exact initial state
            oh.close()
        else:
            # chunk kind: exactly one retained chunk per class ever used (8 B-4 KiB -> classes 0..8)
            assert d["class_chunks"][:9] == [1] * 9 and d["class_chunks"][9] == 0


@pytest.mark.parametrize("flavor", [1, 2])
@pytest.mark.parametrize("kind", [0, 1])
def test_virtual_segment_stress(cuda, kind, flavor):
    """Tiny chunks (1 KiB -> 128 / 126-slot segments): 2^18 threads create and
    retire thousands of segments concurrently; audit + digest must stay exact."""
    torch = cuda
    hc = _hc(kind, flavor, 64 << 20, chunk=1024, maxp=1024)
    want = None
    n = 1 << 18
    with ob.Heap(hc) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        for it in range(3):
            cnt.zero_()
            h.launch_alloc(n, ptrs, size=64)
            h.launch_count(n, ptrs, cnt)
            torch.cuda.synchronize()
            a = h.audit(n, ptrs)
            assert a.live == int(cnt) and a.overlaps == 0 and a.not_marked == 0
            if want is None:
                want = int(cnt)
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
        assert h.last_error()[0] == 0
        s = h.stats()
        assert s.timeouts == 0 and s.corruptions == 0
        # page queues hold every free page, so they span many segments; chunk
        # queues only hold chunks with free pages (segments churn, hwm stays small)
        assert max(s.cls[k].seg_hwm for k in range(s.num_classes)) > (10 if kind == 0 else 0)
        d = h.digest()
        assert d.partition_ok == 1 and d.live_pages == 0


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_sleep_backoff(cuda, variant):
    """SleepRetry: nanosleep(min(base*2^a, cap)) between rounds."""
    torch = cuda
    with ob.Heap(_hc(*variant, 16 << 20, retries=6, backoff=1)) as h:
        n = 1 << 15
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=8192)
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0
        assert h.digest().live_pages == 0


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_baseline_heaps_1m_threads(cuda, variant):
    """BASELINE configs[1]/[2] sizes: 2^20 threads on a 1 GiB (Array) / 8 GiB
    (virtual) heap, 16 B and 512 B; audit + verify + canonical free-all."""
    torch = cuda
    kind, flavor = variant
    heap = (1 << 30) if flavor == 0 else (8 << 30)
    n = 1 << 20
    with ob.Heap(_hc(kind, flavor, heap)) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        for size in (16, 512):
            res = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device="cuda")
            h.launch_alloc(n, ptrs, size=size)
            h.launch_count(n, ptrs, res[2:3])
            h.launch_write(n, ptrs, 5, size)
            h.launch_verify(n, ptrs, 5, size, res)
            torch.cuda.synchronize()
            ok = int(res[2])
            if flavor != 0 or size == 16 or kind == 1:
                assert ok == n, (size, ok)
            assert int(res[0]) == 0
            a = h.audit(n, ptrs)
            assert a.live == ok and a.overlaps == 0 and a.not_marked == 0
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
        assert h.last_error()[0] == 0
        d = h.digest()
        assert d.live_pages == 0 and d.partition_ok == 1


def _spearman(xs, ys):
    def ranks(v):
        order = sorted(range(len(v)), key=lambda i: v[i])
        r = [0.0] * len(v)
        for pos, i in enumerate(order):
            r[i] = float(pos)
        return r
    rx, ry = ranks(xs), ranks(ys)
    n = len(xs)
    mx, my = sum(rx) / n, sum(ry) / n
    cov = sum((a - mx) * (b - my) for a, b in zip(rx, ry))
    return cov / (sum((a - mx) ** 2 for a in rx) * sum((b - my) ** 2 for b in ry)) ** 0.5


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_acceptance_5_chunk_shape_not_reproduced(cuda, flavor):
    """Acceptance criterion 5 asks the chunk allocator's mean_subsequent
    alloc time at 1024 allocations to RISE with the size class (Spearman >= 0.5) -- the
    paper's Fig. 2 effect of "having to walk through this link list as the chunk size
    increases".  This design claims pages from the chunk bitmap cooperatively per warp
    (and so does the CPU oracle), so there is no list walk and the curve is flat: at
    1024 allocations every size sits at the ~13 us launch floor, at 65 536 at ~23 us.
    Recorded as a deviation in DESIGN.md; this test pins the flat shape (max/min <= 3x,
    criterion 6's bound) so a regression that made big classes slow would show."""
    sizes = [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]
    with ob.Heap(_hc(1, flavor, 1 << 30)) as h:
        for n in (1024, 1 << 16):
            t = [min(h.run_trial(n, s, iterations=5, seed=s).mean_subsequent_ms for _ in range(2))
                 for s in sizes]
            assert max(t) / min(t) <= 3.0, (n, _spearman(sizes, t), t)


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_acceptance_6_page_flat(cuda, flavor):
    """Acceptance criterion 6: page allocator, 1024 allocations,
    max/min of mean_subsequent across {1000..8000} <= 3x."""
    # run_trial's precondition: the arena fits the demand with 2x headroom;
    # the page kind gives each class 1/10 of the heap, so 1024 x 8 KiB needs 256 MiB
    with ob.Heap(_hc(0, flavor, 256 << 20)) as h:
        t = [h.run_trial(1024, s, iterations=10, seed=s).mean_subsequent_ms for s in range(1000, 8001, 1000)]
        assert max(t) / min(t) <= 3.0, t


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_alloc_u16_sizes_match_u32(cuda, variant):
    """ouro_launch_alloc_u16: 16-bit request sizes give exactly the 32-bit launcher's
    results (success pattern, classes, TooLarge for 0 and > 8 KiB)."""
    torch = cuda
    n = 1 << 14
    g = torch.Generator().manual_seed(5)
    sz = torch.randint(0, 9000, (n,), generator=g, dtype=torch.int32)
    sz[::97] = 65535
    sz[::89] = 0
    res = {}
    for dt in (torch.int32, torch.int16):
        # 1 GiB: no class runs out (the page kind's 8 KiB class holds ~100 MiB), so the
        # success pattern is interleaving-independent
        with ob.Heap(_hc(*variant, 1 << 30)) as h:
            ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
            d = sz.to(dt).cuda() if dt == torch.int32 else sz.to(torch.int32).to(torch.int16).cuda()
            h.launch_alloc(n, ptrs, sizes=d)
            torch.cuda.synchronize()
            live = (ptrs != 0).cpu()
            s = h.stats()
            res[dt] = (live, s.bad_sizes if hasattr(s, "bad_sizes") else None,
                       [s.cls[k].live_pages for k in range(s.num_classes)])
            a = h.audit(n, ptrs)
            assert a.overlaps == 0 and a.misaligned == 0 and a.live == int(live.sum())
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
            assert h.last_error()[0] == 0
    assert torch.equal(res[torch.int32][0], res[torch.int16][0])
    assert res[torch.int32][2] == res[torch.int16][2]
    bad = (sz == 0) | (sz > 8192)
    assert not res[torch.int16][0][bad].any()


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_no_spurious_oom_while_queue_refills(cuda, flavor):
    """Regression: chunk kind, 2^16 x malloc(48) on a 64 MiB heap (3 MiB of demand).
    At kernel start the class queue is empty, thousands of warps take fresh chunks and
    the rest fail their first try while those chunks are being enqueued.  Every retry
    round must make its own observation (OutOfMemory only after
    max_retries rounds with no page obtainable), so all requests are served; a round
    that re-used one cached "empty" observation returned spurious OOMs here."""
    torch = cuda
    n = 1 << 16
    for rep in range(5):
        with ob.Heap(_hc(1, flavor, 64 << 20)) as h:
            ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
            h.launch_alloc(n, ptrs, size=48)
            torch.cuda.synchronize()
            ok = int((ptrs != 0).sum())
            assert ok == n, (rep, n - ok, h.stats().cls[2].ooms)
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
            assert h.last_error()[0] == 0


@pytest.mark.parametrize("kind", [0, 1])
def test_virtual_list_retirement_under_load(cuda, kind):
    """Regression: VirtualList segment retirement at 2^20 threads (8 GiB heap,
    8190-slot segments, ~128 segments retired and created per phase).  A head
    advance whose CAS won could miss a segment completed concurrently by a warp
    that saw the old head and lost its own CAS; the head then stalled, segment
    creation starved (TimeoutError) and the free-all partition broke in about a
    third of the runs.  Six alloc/free rounds, canonical digest after each."""
    torch = cuda
    n = 1 << 20
    with ob.Heap(_hc(kind, 2, 8 << 30)) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        for rep in range(6):
            size = 16 if rep % 2 == 0 else 512
            h.launch_alloc(n, ptrs, size=size)
            torch.cuda.synchronize()
            assert int((ptrs != 0).sum()) == n, rep
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
            assert h.last_error()[0] == 0, (rep, h.last_error(), h.stats().timeouts)
            d = h.digest()
            assert d.live_pages == 0 and d.partition_ok == 1, rep


@pytest.mark.parametrize("flavor", [1, 2])
@pytest.mark.parametrize("kind", [0, 1])
def test_virtual_churn_small_segments(cuda, kind, flavor):
    """Mixed alloc/free rounds in one kernel on 4 KiB chunks (510 / 512-slot
    segments): segment creation, linking and retirement interleave with
    enqueues and dequeues of the same queue inside each launch.  Stamps every
    round, audit, then free-all to an exact partition with no device error."""
    torch = cuda
    n = 1 << 16
    with ob.Heap(_hc(kind, flavor, 64 << 20, chunk=4096, maxp=4096)) as h:
        slots = torch.zeros(n, dtype=torch.int64, device="cuda")
        res = torch.zeros(5, dtype=torch.int64, device="cuda")
        h.launch_churn(n, 0, 30, 7, slots, res)
        torch.cuda.synchronize()
        ok, failed, frees, reused, bad = [int(x) for x in res]
        assert bad == 0 and ok > 0 and frees > 0
        a = h.audit(n, slots)
        assert a.overlaps == 0 and a.out_of_heap == 0 and a.misaligned == 0 and a.not_marked == 0
        h.launch_free(n, slots)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0, (h.last_error(), h.stats().timeouts)
        d = h.digest()
        assert d.live_pages == 0 and d.partition_ok == 1


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("size", [16, 64, 512, 1000, 2048, 4096, 8192])
def test_pattern_passes_cover_every_live_region(cuda, size, kind):
    """The write/verify passes must touch every byte of every live region (the
    passes map slots to lanes in strided runs; the verifier batches four 512 B
    steps of a region per pass): write seed 1, verify seed 2 -> every 8-byte word
    of every live region mismatches; verify seed 1 -> none.  Both kinds: the page
    kind's region length is partition arithmetic, the chunk kind's the header."""
    torch = cuda
    n = (1 << 18) + 77  # not a multiple of any run width
    with ob.Heap(_hc(kind, 0, 256 << 20)) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=size)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        h.launch_count(n, ptrs, cnt)
        h.launch_write(n, ptrs, 1, 0)
        good = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device="cuda")
        h.launch_verify(n, ptrs, 1, 0, good)
        other = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device="cuda")
        h.launch_verify(n, ptrs, 2, 0, other)
        torch.cuda.synchronize()
        live = int(cnt)
        page = max(16, 1 << (size - 1).bit_length())
        assert live > 0
        assert int(good[0]) == 0
        assert int(other[0]) == live * (page // 8)
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0


@pytest.mark.parametrize("size,word", [(8192, 3 * 64 + 5), (8192, 1023), (1024, 70), (512, 0), (16, 1)])
def test_verify_reports_corrupted_words(cuda, size, word):
    """A word flipped anywhere in a region (any 512 B step of the verifier's batch)
    is counted once and the lowest corrupted slot is reported."""
    torch = cuda
    n = 2048
    with ob.Heap(_hc(0, 0, 256 << 20)) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=size)
        h.launch_write(n, ptrs, 7, 1)
        torch.cuda.synchronize()
        words = max(16, size) // 8
        for slot in (1234, 100):
            p = int(ptrs[slot])
            assert p != 0

            class Region:
                __cuda_array_interface__ = {"shape": (words,), "typestr": "<i8", "data": (p, False), "version": 3}
            r = torch.as_tensor(Region(), device="cuda")
            r[word] ^= 1
        res = torch.tensor([0, -1], dtype=torch.int64, device="cuda")
        h.launch_verify(n, ptrs, 7, 1, res)
        torch.cuda.synchronize()
        assert int(res[0]) == 2 and int(res[1]) == 100
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
