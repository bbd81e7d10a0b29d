"""GPU parity with the oracle, through the C-ABI (libouro_b200.so).

* single-warp op scripts: every op's status and heap offset must equal the
  oracle's bit-for-bit (one warp => deterministic), then the canonical digest
  must be identical;
* concurrent phased workloads (thousands of warps): audit (in-heap, aligned,
  pairwise disjoint, bitmap-marked), pattern write/verify, free-all, and the
  interleaving-independent digest must equal the oracle's for the same demand.
"""
import ctypes as C

import pytest

import paper_2504_18211_b200 as ob
from helpers import NAMES, VARIANTS, cfg, random_script
from oracle_lib import OHeap

pytestmark = pytest.mark.gpu

IDS = [NAMES[v] for v in VARIANTS]


def _heap(c, checks=True):
    hc = ob.HeapConfig(c.heap_bytes, c.chunk_bytes, c.min_page_bytes, c.max_page_bytes,
                       ob.QueueFlavor(c.queue_flavor), ob.AllocatorKind(c.allocator_kind),
                       ob.BackoffPolicy(c.backoff), c.max_retries)
    h = ob.Heap(hc, 0)
    h.set_checks(checks)
    return h


def _script_parity(c, steps):
    h = _heap(c)
    goff, gst = h.run_script(steps)
    oh = OHeap(c)
    ooff, ost = oh.run_script(steps)
    for i in range(len(gst)):
        if gst[i] != ost[i] or goff[i] != ooff[i]:
            s = i // 32
            op, mask, args = steps[s]
            lanes = [j for j in range(32) if mask >> j & 1]
            detail = [(j, args[j], gst[s * 32 + j], ost[s * 32 + j], goff[s * 32 + j], ooff[s * 32 + j])
                      for j in lanes]
            raise AssertionError(f"first mismatch at step {s} lane {i % 32} op {op}: "
                                 f"(lane, arg, gpu st, oracle st, gpu off, oracle off) = {detail}")
    gd, od = h.digest().as_dict(), oh.digest().as_dict()
    assert gd == od
    gs, os_ = h.stats(), oh.stats()
    for k in range(gs.num_classes):
        for f in ("chunks", "live_pages", "queue_len", "queued_live", "seg_live", "seg_hwm", "ooms", "retries"):
            assert getattr(gs.cls[k], f) == getattr(os_.cls[k], f), (k, f)
    assert (gs.double_frees, gs.invalid_frees, gs.bad_sizes, gs.stale_drops) == \
        (os_.double_frees, os_.invalid_frees, os_.bad_sizes, os_.stale_drops)
    assert gs.timeouts == 0 and gs.corruptions == 0
    h.close()
    oh.close()
    return gst


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_single_lane_script_parity(cuda, variant):
    kind, flavor = variant
    steps = random_script(2024 + kind * 10 + flavor, 3000, p_free=0.4, bad=True)
    st = _script_parity(cfg(kind, flavor, 1 << 20, retries=3), steps)
    assert 7 in st or kind == 1  # OOM exercised (page kind always; chunk kind usually)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_single_lane_small_segments(cuda, variant):
    """512 B chunks: virtual segments of 64 / 62 slots are created and retired constantly."""
    kind, flavor = variant
    steps = random_script(99 + kind * 10 + flavor, 2500, sizes=[1, 16, 40, 100, 256], p_free=0.45)
    _script_parity(cfg(kind, flavor, 1 << 16, 512, 16, 256, retries=2), steps)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_warp_script_parity(cuda, variant):
    kind, flavor = variant
    steps = random_script(555 + kind * 10 + flavor, 1200, warp=True, p_free=0.45, bad=True)
    _script_parity(cfg(kind, flavor, 4 << 20, retries=3), steps)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_warp_script_small_chunks(cuda, variant):
    kind, flavor = variant
    steps = random_script(777 + kind * 10 + flavor, 1000, warp=True, sizes=[8, 16, 32, 64, 128, 256],
                          p_free=0.5)
    _script_parity(cfg(kind, flavor, 1 << 18, 1024, 16, 256, retries=2), steps)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_coalesced_script_parity(cuda, variant):
    kind, flavor = variant
    steps = random_script(31 + kind * 10 + flavor, 600, warp=True, sizes=[16, 1000, 8192], coalesced=True,
                          p_free=0.4)
    _script_parity(cfg(kind, flavor, 1 << 20, retries=2), steps)


def _oracle_run(c, sizes):
    """The oracle on the same demand (warps of 32 lanes in slot order): number
    of successful allocations, and the canonical digest after freeing them."""
    oh = OHeap(c)
    offs = []
    ok = 0
    for i in range(0, len(sizes), 32):
        o, s = oh.alloc(sizes[i:i + 32])
        offs += [x for x, st in zip(o, s) if st == 0]
        ok += sum(1 for st in s if st == 0)
    for i in range(0, len(offs), 32):
        assert all(x == 0 for x in oh.free(offs[i:i + 32]))
    d = oh.digest().as_dict()
    oh.close()
    return ok, d


def _heap_bytes(kind):
    # page kind: exact static partition (capacity identical on GPU and oracle);
    # chunk kind: room for warp herding (each warp's group may open a chunk)
    return (64 << 20) if kind == 0 else (256 << 20)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
@pytest.mark.parametrize("size", [16, 1000, 8192])
def test_concurrent_phased(cuda, variant, size):
    """BASELINE configs[0] shape: 65 536 threads, alloc/audit/write/verify/free x3."""
    torch = cuda
    kind, flavor = variant
    c = cfg(kind, flavor, _heap_bytes(kind), retries=64)
    n = 65536 if size <= 1000 else 8192
    want_ok, want_digest = _oracle_run(c, [size] * n)
    h = _heap(c, checks=(size != 1000))  # size 1000 runs the production (unchecked) path
    ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
    for it in range(3):
        res = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=size)
        h.launch_count(n, ptrs, res[2:3])
        torch.cuda.synchronize()
        assert int(res[2]) == want_ok, "success count differs from the oracle"
        a = h.audit(n, ptrs)
        assert (a.live, a.out_of_heap, a.misaligned, a.overlaps, a.not_marked) == (want_ok, 0, 0, 0, 0)
        h.launch_write(n, ptrs, 1234, it)
        h.launch_verify(n, ptrs, 1234, it, res)
        torch.cuda.synchronize()
        assert int(res[0]) == 0, "pattern verification failed"
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
    first, mask = h.last_error()
    assert first == 0, f"sticky device error {first} mask {mask:#x}"
    assert h.digest().as_dict() == want_digest
    h.close()


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_concurrent_mixed_sizes(cuda, variant):
    torch = cuda
    kind, flavor = variant
    c = cfg(kind, flavor, _heap_bytes(kind), retries=64)
    n = 65536
    g = torch.Generator().manual_seed(5)
    sizes = torch.randint(1, 513, (n,), generator=g, dtype=torch.int32)
    want_ok, want_digest = _oracle_run(c, sizes.tolist())
    h = _heap(c)
    ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
    dsz = sizes.cuda()
    res = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device="cuda")
    h.launch_alloc(n, ptrs, sizes=dsz)
    h.launch_count(n, ptrs, res[2:3])
    torch.cuda.synchronize()
    assert int(res[2]) == want_ok
    a = h.audit(n, ptrs)
    assert (a.live, a.out_of_heap, a.misaligned, a.overlaps, a.not_marked) == (want_ok, 0, 0, 0, 0)
    h.launch_write(n, ptrs, 9, 0)
    h.launch_verify(n, ptrs, 9, 0, res)
    h.launch_free(n, ptrs)
    torch.cuda.synchronize()
    assert int(res[0]) == 0
    assert h.last_error()[0] == 0
    assert h.digest().as_dict() == want_digest
    h.close()
