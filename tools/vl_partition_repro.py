"""test_baseline_heaps_1m_threads[vl-page] in a loop: 2^20 threads, 8 GiB VLPQ heap,
malloc(16) / malloc(512), verify, free; canonical digest after each round.
OURO_DIGEST_DEBUG=1 prints the chunks that break the partition."""
import os
import sys

sys.path.insert(0, os.environ.get("OURO_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 0
flavor = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
n = 1 << 20
fails = 0
for rep in range(reps):
    hc = ob.HeapConfig(8 << 30, queue_flavor=ob.QueueFlavor(flavor), allocator_kind=ob.AllocatorKind(kind))
    with ob.Heap(hc) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        for size in (16, 512):
            h.launch_alloc(n, ptrs, size=size)
            torch.cuda.synchronize()
            ok = int((ptrs != 0).sum())
            h.launch_free(n, ptrs)
            torch.cuda.synchronize()
            d = h.digest()
            s = h.stats()
            bad = not (d.live_pages == 0 and d.partition_ok == 1)
            fails += bad
            print(f"rep {rep} size {size}: ok {ok} live {d.live_pages} partition_ok {d.partition_ok} "
                  f"err {h.last_error()[0]} timeouts {s.timeouts}", flush=True)
print("FAILS", fails)
