"""test_virtual_segment_stress in a loop with timings (tiny 1 KiB chunks -> 126-slot
VirtualList segments).  Run under `timeout`."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18211_b200 as ob
kind = int(sys.argv[1]) if len(sys.argv) > 1 else 0
flavor = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 1 << 18
hc = ob.HeapConfig(64 << 20, 1024, 16, 1024, ob.QueueFlavor(flavor), ob.AllocatorKind(kind), ob.BackoffPolicy(0), 64)
with ob.Heap(hc) as h:
    ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
    for it in range(3):
        t0 = time.time()
        h.launch_alloc(n, ptrs, size=64)
        torch.cuda.synchronize()
        t1 = time.time()
        ok = int((ptrs != 0).sum())
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        t2 = time.time()
        s = h.stats()
        print(f"kind {kind} flavor {flavor} it {it}: alloc {1e3*(t1-t0):.1f} ms free {1e3*(t2-t1):.1f} ms ok {ok} "
              f"timeouts {s.timeouts} err {h.last_error()[0]} seg_live {s.cls[2].seg_live} hwm {s.cls[2].seg_hwm}", flush=True)
