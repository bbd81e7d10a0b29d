"""One 2^20-thread malloc(8192) on the PQ 1 GiB heap with max_retries=1 (first try only,
~99% OOM): the fixed cost of an OOM storm.  Run under ncu -k k_alloc -s 2 -c 1."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18211_b200 as ob
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
with ob.Heap(ob.HeapConfig(1 << 30, max_retries=1)) as h:
    for it in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_alloc(n, ptrs, size=8192); b.record(); b.synchronize()
        print(f"alloc_us={a.elapsed_time(b) * 1000:.1f}")
        h.launch_free(n, ptrs); torch.cuda.synchronize()
