"""C-ABI entry points against the oracle on live device state: page_region
(SPEC.md:72-80), the pattern words of write/verify (gap G6),
and the bounded-wait watchdog (TimeoutError, errors.hpp:35-39)."""
import pytest

import paper_2504_18211_b200 as ob
from helpers import NAMES, VARIANTS, cfg, random_script
from oracle_lib import OHeap, oracle

pytestmark = pytest.mark.gpu
IDS = [NAMES[v] for v in VARIANTS]


def _heap(c):
    hc = ob.HeapConfig(c.heap_bytes, c.chunk_bytes, c.min_page_bytes, c.max_page_bytes,
                       ob.QueueFlavor(c.queue_flavor), ob.AllocatorKind(c.allocator_kind),
                       ob.BackoffPolicy(c.backoff), c.max_retries)
    return ob.Heap(hc, 0)


@pytest.mark.parametrize("variant", VARIANTS, ids=IDS)
def test_page_region_matches_oracle_on_live_state(cuda, variant):
    """After the same warp op script (identical offsets on both, checked), every
    handle (chunk, page) of the heap resolves identically on GPU and oracle: the
    same status (OK / InvalidHandle for unassigned or segment chunks and pages past
    the class's pages per chunk / Range past the last chunk) and the same region."""
    kind, flavor = variant
    c = cfg(kind, flavor, 1 << 20, retries=2)
    steps = random_script(4242 + kind * 10 + flavor, 400, warp=True, p_free=0.35)
    with _heap(c) as h:
        goff, gst = h.run_script(steps)
        oh = OHeap(c)
        ooff, ost = oh.run_script(steps)
        assert (goff, gst) == (ooff, ost)
        g = h.geometry
        pages = 1 << g.page_bits
        checked = mismatched = ok = 0
        for ch in range(g.num_chunks + 1):
            for p in list(range(0, 64)) + [pages // 2, pages - 1]:
                handle = (ch << g.page_bits) | p
                o_st, o_off, o_len = oh.page_region(handle)
                try:
                    r = (0,) + h.page_region(handle)
                except ob.OuroError as e:
                    r = (e.status, 0, 0)
                want = (o_st, o_off, o_len) if o_st == 0 else (o_st, 0, 0)
                checked += 1
                ok += o_st == 0
                mismatched += r != want
        oh.close()
    assert mismatched == 0
    assert ok > 0 and checked > ok


@pytest.mark.parametrize("size", [16, 48, 1000, 4096])
def test_pattern_words_equal_oracle(cuda, size):
    """Every word the GPU writer puts in a live region is orc_pattern_word(seed, slot,
    iteration, word) -- the same function the oracle's bench writes and verifies."""
    torch = cuda
    n, seed, it = 96, 0xC0FFEE, 3
    with ob.Heap(ob.HeapConfig(64 << 20)) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=size)
        h.launch_write(n, ptrs, seed, it)
        torch.cuda.synchronize()
        page = max(16, 1 << (size - 1).bit_length())
        words = page // 8
        L = oracle()
        for slot in range(0, n, 7):
            p = int(ptrs[slot])
            assert p != 0

            class Region:
                __cuda_array_interface__ = {"shape": (words,), "typestr": "<u8", "data": (p, False), "version": 3}
            got = torch.as_tensor(Region(), device="cuda").cpu().tolist()
            want = [L.orc_pattern_word(seed, slot, it, w) for w in range(words)]
            assert got == want, (slot, size)
        res = torch.tensor([0, -1], dtype=torch.int64, device="cuda")
        h.launch_verify(n, ptrs, seed, it, res)
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        assert int(res[0]) == 0


@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_watchdog_chunk_kind_missing_entry(cuda, flavor):
    """A class-queue count that promises an entry no slot will ever hold: the
    dequeuer's wait is bounded by spin_limit, raises the sticky TimeoutError and the
    call still completes (here from the pool) -- no hung GPU."""
    torch = cuda
    hc = ob.HeapConfig(16 << 20, allocator_kind=ob.AllocatorKind.Chunk, queue_flavor=ob.QueueFlavor(flavor))
    with ob.Heap(hc) as h:
        h.set_spin_limit(2000)
        h.debug_add_count(0, 1)               # class 0 (16 B) queue: count 1, no entry
        ptrs = torch.zeros(32, dtype=torch.int64, device="cuda")
        h.launch_alloc(32, ptrs, size=16)
        torch.cuda.synchronize()
        first, mask = h.last_error()
        assert first == ob._abi.ERR_TIMEOUT and mask & (1 << ob._abi.ERR_TIMEOUT)
        assert h.stats().timeouts >= 1
        assert int((ptrs != 0).sum()) == 32   # served from the pool after the bounded wait


def test_watchdog_page_kind_status(cuda):
    """Page kind: the lane whose ticket has no entry gets OURO_ERR_TIMEOUT as its
    own status, the others are served; the sticky word records TimeoutError."""
    c = cfg(0, 0, 1 << 20, retries=2)          # 16 chunks: class 9 (8 KiB) owns 1 chunk = 8 pages
    with _heap(c) as h:
        h.set_spin_limit(2000)
        h.debug_add_count(9, 1)
        off, st = h.run_script([(0, (1 << 9) - 1, [8192] * 32)])
        lanes = st[:9]
        assert sorted(lanes) == [0] * 8 + [ob._abi.ERR_TIMEOUT]
        assert h.last_error()[0] == ob._abi.ERR_TIMEOUT
