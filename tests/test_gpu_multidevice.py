"""Multi-heap / multi-device host orchestration (BASELINE configs[4]).

Only one GPU is available to the test runs, so N devices are exercised as N heaps
on device 0 driven by N host threads -- the same code path (one host thread per
heap, a host barrier per step, per-device CUDA events, no collective).  Host API
calls bind the heap's device and restore the caller's (construction
single-threaded per heap, operations thread-safe)."""
import threading

import pytest

import paper_2504_18211_b200 as ob

pytestmark = pytest.mark.gpu


def _pq(heap=64 << 20):
    return ob.HeapConfig(heap, allocator_kind=ob.AllocatorKind.Page)


def test_multi_sweep_two_heaps_one_device(cuda):
    """ouro_multi_sweep with devices [0, 0]: two host threads, two independent heaps."""
    n, steps = 65536, 2
    cap_1k = (1024 // 10) * 64   # 64 MiB page heap: 102 chunks x 64 pages in the 1 KiB class
    r = ob.multi_sweep(_pq(), [0, 0], n, [16, 1024], warmup=1, steps=steps)
    assert r.ndev == 2 and r.verified == 1
    per_dev = steps * (n + cap_1k)
    assert [r.dev_pairs[0], r.dev_pairs[1]] == [per_dev, per_dev]
    assert r.pairs_total == 2 * per_dev
    assert r.max_ms == max(r.dev_ms[0], r.dev_ms[1]) > 0
    assert r.pairs_per_s == pytest.approx(r.pairs_total / (r.max_ms / 1e3))


@pytest.mark.parametrize("variant", [(0, 0), (1, 0), (1, 2)])
def test_multi_sweep_variants_four_heaps(cuda, variant):
    kind, flavor = variant
    hc = ob.HeapConfig(256 << 20, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
    r = ob.multi_sweep(hc, [0, 0, 0, 0], 1 << 16, [16, 256], warmup=1, steps=1)
    assert r.ndev == 4 and r.verified == 1
    assert len({r.dev_pairs[d] for d in range(4)}) == 1 and r.dev_pairs[0] == 2 * (1 << 16)


def test_two_host_threads_drive_two_heaps_concurrently(cuda):
    """Two Python threads (the C-ABI releases the GIL), each with its own heap on
    device 0, run the paper's driver at the same time; both verify clean and end in
    their canonical state."""
    results, errors = {}, []

    def work(tag, kind):
        try:
            hc = ob.HeapConfig(256 << 20, allocator_kind=ob.AllocatorKind(kind))
            with ob.Heap(hc, 0) as h:
                r = h.run_trial(1 << 16, 100, iterations=4, seed=tag)
                d = h.digest()
                results[tag] = (r.verified, r.failed_allocs, h.last_error()[0], d.live_pages, d.partition_ok)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(t, t % 2)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errors, errors
    assert results == {0: (1, 0, 0, 0, 1), 1: (1, 0, 0, 0, 1)}


def test_create_on_missing_device_fails_and_keeps_current_device(cuda):
    torch = cuda
    torch.cuda.set_device(0)
    bad = torch.cuda.device_count()
    with pytest.raises(ob.OuroError):
        ob.Heap(_pq(), bad)
    assert torch.cuda.current_device() == 0
    with ob.Heap(_pq(), 0) as h:
        h.last_error()
        assert torch.cuda.current_device() == 0


def test_launch_shape_is_per_heap(cuda):
    torch = cuda
    n = 1 << 16
    counts = []
    with ob.Heap(_pq()) as a, ob.Heap(_pq()) as b:
        a.set_launch_shape(64, 0)
        b.set_launch_shape(256, 2)   # persistent grid on b only
        for h in (a, b):
            ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            h.launch_alloc(n, ptrs, size=48)
            h.launch_count(n, ptrs, cnt)
            torch.cuda.synchronize()
            counts.append(int(cnt))
            assert h.audit(n, ptrs).overlaps == 0
            h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        assert a.last_error()[0] == 0 and b.last_error()[0] == 0
    assert counts == [n, n]


def test_launcher_arguments_are_checked(cuda):
    """ADVICE: an int64 `sizes` tensor or a short output buffer used to reach the
    kernels unchecked (misread sizes, out-of-bounds writes)."""
    torch = cuda
    n = 4096
    with ob.Heap(_pq()) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        with pytest.raises(ValueError):
            h.launch_alloc(n, ptrs, sizes=torch.full((n,), 16, dtype=torch.int64, device="cuda"))
        with pytest.raises(ValueError):
            h.launch_alloc(n, ptrs[: n // 2], size=16)
        with pytest.raises(ValueError):
            h.launch_alloc(n, torch.zeros(n, dtype=torch.int32, device="cuda"), size=16)
        with pytest.raises(ValueError):
            h.launch_free(n, ptrs.cpu())
        h.launch_alloc(n, ptrs, sizes=torch.full((n,), 16, dtype=torch.int32, device="cuda"))
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0
