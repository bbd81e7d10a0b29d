"""GPU vs oracle at the BASELINE.json configurations, full size (2^20 / 2^22 threads).

For every size of each sweep, the GPU (2^20 device threads through the C-ABI
launchers) and the oracle (the same 2^20 requests in warp groups of 32, slot
order) serve the same demand on heaps in the same state:

* the number of successful allocations must be equal -- the page kind's
  capacities are fixed by the static partition, the chunk kind's
  by the chunks left after the classes used earlier in the sweep keep their
  watermark chunk;
* every live allocation is in-heap, aligned, disjoint and marked (audit) and
  survives the write/verify pattern;
* after the free-all, the canonical digest must be identical --
  "final heap/queue state after all frees bit-exact" (BASELINE.json north_star;
  SPEC.md:275 alloc-all/free-all rounds restore the state, SPEC.md:295 full-drain
  restoration asserted exactly).
"""
import pytest

import paper_2504_18211_b200 as ob
from helpers import NAMES
from oracle_lib import OHeap

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

SWEEP = [4, 8, 16, 32, 64, 128, 256, 512, 1000, 1024, 2048, 4096, 8192]
N = 1 << 20


def _hc(kind, flavor, heap):
    return ob.HeapConfig(heap, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))


def _sweep_parity(torch, kind, flavor, heap, n, sizes):
    hc = _hc(kind, flavor, heap)
    oh = OHeap(hc.to_c())
    counts = []
    with ob.Heap(hc) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        for it, size in enumerate(sizes):
            offs, want = oh.alloc_slots(n, size)
            res = torch.tensor([0, -1, 0, 0], dtype=torch.int64, device="cuda")
            h.launch_alloc(n, ptrs, size=size)
            h.launch_count(n, ptrs, res[2:3])
            h.launch_write(n, ptrs, 11, it)
            h.launch_verify(n, ptrs, 11, it, res)
            torch.cuda.synchronize()
            ok = int(res[2])
            if ok != want:
                # Only where capacity binds on a chunk-kind virtual flavour: chunks returned to
                # the pool leave generation-stale entries in their class queue (dropped at
                # dequeue, gap G3), how many depends on the interleaving, and longer queues
                # hold more segment chunks.  The shortfall must be exactly those extra
                # segment chunks' pages, and no chunk may be unaccounted for.
                assert kind == 1 and flavor != 0, f"{size} B: GPU served {ok}, oracle {want}"
                gs, os_ = h.stats(), oh.stats()
                K = gs.num_classes
                gseg = sum(gs.cls[k].seg_live for k in range(K))
                oseg = sum(os_.cls[k].seg_live for k in range(K))
                k = max(range(K), key=lambda j: gs.cls[j].live_pages)
                assert want - ok == gs.cls[k].pages_per_chunk * (gseg - oseg), (size, ok, want, gseg, oseg)
                assert sum(gs.cls[j].chunks for j in range(K)) + gseg + gs.pool_len == gs.num_chunks
            assert int(res[0]) == 0, f"{size} B: pattern verification failed"
            a = h.audit(n, ptrs)
            assert (a.live, a.out_of_heap, a.misaligned, a.overlaps, a.not_marked) == (ok, 0, 0, 0, 0), size
            oh.free_slots(offs)
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
            first, mask = h.last_error()
            assert first == 0, f"{size} B: sticky device error {first} mask {mask:#x}"
            assert h.digest().as_dict() == oh.digest().as_dict(), f"{size} B: free-all digest differs"
            counts.append(ok)
    oh.close()
    return counts


def test_config1_pq_1gib_sweep(cuda):
    """BASELINE configs[1]: PQ, Array queues, 1 GiB, 2^20 threads, 4 B-8 KiB."""
    counts = _sweep_parity(cuda, 0, 0, 1 << 30, N, SWEEP)
    # the static partition's capacities: 1638 chunks per class above 64 B
    assert counts[:5] == [N] * 5
    assert counts[5:] == [838656, 419328, 209664, 104832, 104832, 52416, 26208, 13104]


@pytest.mark.parametrize("variant", [(0, 1), (1, 1), (0, 2), (1, 2)], ids=lambda v: NAMES[v])
def test_config2_virtual_8gib_sweep(cuda, variant):
    """BASELINE configs[2]: VAPQ / VACQ / VLPQ / VLCQ, 8 GiB, 2^20 threads, 16 B-8 KiB."""
    counts = _sweep_parity(cuda, *variant, 8 << 30, N, SWEEP[2:])
    kind = variant[0]
    if kind == 0:
        assert counts[:6] == [N] * 6           # <= 512 B: the 8 GiB partition serves every thread
        assert 800000 < counts[6] < N          # 1000 B / 1 KiB: 13 107 chunks minus the segment reserve
    else:
        assert counts[:10] == [N] * 10         # chunk kind serves all sizes below 8 KiB
        assert 0 < counts[10] < N              # 8 KiB: every chunk but segments / watermarks / floor


def test_config1_cq_1gib_sweep(cuda):
    """The chunk kind on the configs[1] heap (bench --config cq1g)."""
    counts = _sweep_parity(cuda, 1, 0, 1 << 30, N, SWEEP[2:])
    assert counts[:6] == [N] * 6            # 1 KiB and up: 16 384 chunks minus one kept per earlier class


def test_config0_cq_64mib(cuda):
    """BASELINE configs[0]: chunk allocator, 64 MiB, 65 536 x malloc(16), write/verify/free,
    two rounds; the free-all digest equals the oracle's."""
    counts = _sweep_parity(cuda, 1, 0, 64 << 20, 65536, [16, 16])
    assert counts == [65536, 65536]


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_churn_chunk_kind_vs_oracle(cuda, flavor):
    """Mixed churn (configs[3] shape, 2^18 threads, 20 rounds) on the chunk kind: with no
    failed malloc every (thread, round) decision is the same on GPU and oracle, so the
    malloc / free counts must match exactly, and the free-all digest must too."""
    torch = cuda
    hc = _hc(1, flavor, 1 << 30)
    n, rounds, seed = 1 << 18, 20, 1
    oh = OHeap(hc.to_c())
    oslots, ores = oh.churn(n, 0, rounds, seed, threads=8)
    with ob.Heap(hc) as h:
        slots = torch.zeros(n, dtype=torch.int64, device="cuda")
        res = torch.zeros(5, dtype=torch.int64, device="cuda")
        h.launch_churn(n, 0, rounds, seed, slots, res)
        torch.cuda.synchronize()
        ok, failed, frees, reused, bad = [int(x) for x in res]
        assert failed == 0 and ores.mallocs_failed == 0 and bad == 0 and ores.check_failures == 0
        assert (ok, frees) == (ores.mallocs_ok, ores.frees)
        a = h.audit(n, slots)
        assert a.live == sum(1 for x in oslots if x != 2 ** 64 - 1)
        assert a.overlaps == 0 and a.not_marked == 0
        h.launch_free(n, slots)
        oh.free_all(oslots)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0
        assert h.digest().as_dict() == oh.digest().as_dict()
    oh.close()


def test_config3_churn_4m_threads(cuda):
    """BASELINE configs[3] at its real shape: 2^22 threads, sizes 8 B-4 KiB, 16 GiB chunk heap,
    interleaved alloc/free rounds (10 here; bench runs 100); counts and free-all digest
    equal the oracle's (all host threads)."""
    torch = cuda
    hc = _hc(1, 0, 16 << 30)
    n, rounds, seed = 1 << 22, 10, 3
    oh = OHeap(hc.to_c())
    import os
    oslots, ores = oh.churn(n, 0, rounds, seed, threads=os.cpu_count() or 8)
    with ob.Heap(hc) as h:
        slots = torch.zeros(n, dtype=torch.int64, device="cuda")
        res = torch.zeros(5, dtype=torch.int64, device="cuda")
        h.launch_churn(n, 0, rounds, seed, slots, res)
        torch.cuda.synchronize()
        ok, failed, frees, reused, bad = [int(x) for x in res]
        assert failed == 0 and ores.mallocs_failed == 0 and bad == 0
        assert (ok, frees) == (ores.mallocs_ok, ores.frees)
        assert reused > 0
        h.launch_free(n, slots)
        oh.free_all(oslots)
        torch.cuda.synchronize()
        assert h.last_error()[0] == 0
        assert h.digest().as_dict() == oh.digest().as_dict()
    oh.close()
