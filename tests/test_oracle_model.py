"""Acceptance criterion 3: a 10^4-op randomized single-threaded
alloc/free sequence per variant; the C oracle must match the free-list/bitset
model (tests/model.py) on every op's success/failure AND offset, and all live
regions must be pairwise disjoint.  CPU only."""
import random

import pytest

from helpers import NAMES, VARIANTS, cfg, random_script, single_lane_ops
from model import Model
from oracle_lib import OHeap

GEOMS = [
    # heap, chunk, min, max
    (1 << 20, 64 << 10, 16, 8192),      # SPEC.md:51 arena
    (1 << 18, 4 << 10, 16, 1024),       # many small chunks, tiny segments
    (1 << 16, 512, 16, 256),            # S_va = 64 slots: virtual segments churn constantly
]


def _check_disjoint(live):
    iv = sorted(live.values())
    for (a, la), (b, _) in zip(iv, iv[1:]):
        assert a + la <= b, "overlapping live regions"


@pytest.mark.parametrize("variant", VARIANTS, ids=[NAMES[v] for v in VARIANTS])
@pytest.mark.parametrize("geom", range(len(GEOMS)))
def test_oracle_matches_model(variant, geom):
    kind, flavor = variant
    heap, chunk, mn, mx = GEOMS[geom]
    n_ops = 10_000 if geom == 0 else 4_000
    sizes = [s for s in (1, 8, 16, 17, 32, 100, 128, 255, 256, 500, 1000, 1024, 2000, 4096, 8000, 8192) if s <= mx]
    steps = random_script(1000 + geom * 7 + kind * 3 + flavor, n_ops, sizes=sizes, p_free=0.4,
                          bad=True)
    c = cfg(kind, flavor, heap, chunk, mn, mx, retries=3)
    oh = OHeap(c)
    off, st = oh.run_script(steps)
    m = Model(heap, chunk, mn, mx, kind, flavor, max_retries=3)
    results = {}
    live = {}
    for s, (op, lane, arg) in enumerate(single_lane_ops(steps)):
        idx = s * 32 + lane
        if op == 0:
            o, code = m.alloc(arg)
            assert st[idx] == code, (s, arg)
            if code == 0:
                assert off[idx] == o, (s, arg)
                k = m.size_class(arg)
                live[idx] = (o, m.page_bytes(k))
            results[idx] = o
        else:
            if arg >> 63:
                target = arg & ~(1 << 63)
            else:
                target = results.get(arg)
                if target is None:
                    target = (1 << 64) - 2
            code = m.dealloc(target)
            assert st[idx] == code, (s, arg, target)
            if code == 0:
                for key, (o, _) in list(live.items()):
                    if o == target:
                        del live[key]
        if s % 500 == 0:
            _check_disjoint(live)
    _check_disjoint(live)
    # quiescent consistency of the oracle itself
    d = oh.digest()
    assert d.partition_ok == 1
    oh.close()


def test_warp_groups_equal_sequential_for_page_kind():
    """Page kind: a group of n lanes gets exactly what n sequential single-lane
    allocs would (consecutive FIFO tickets)."""
    a = OHeap(cfg(0, 0, 1 << 20))
    b = OHeap(cfg(0, 0, 1 << 20))
    rng = random.Random(3)
    for _ in range(200):
        sizes = [rng.choice([16, 1000]) for _ in range(rng.randint(1, 32))]
        first = sizes[0]
        sizes.sort(key=lambda s: s != first)  # group order = first-lane order
        oa, sa = a.alloc(sizes)
        seq = [b.alloc([s]) for s in sizes]
        assert oa == [x[0][0] for x in seq] and sa == [x[1][0] for x in seq]
