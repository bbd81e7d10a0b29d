"""Cost of a failed retry round: time a 2^20-thread malloc(8192) on the PQ 1 GiB heap
(~99% OOM) for several max_retries; the slope is the per-round cost."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18211_b200 as ob
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
for backoff in (0, 1):
    for r in (1, 2, 8, 32, 64):
        hc = ob.HeapConfig(1 << 30, max_retries=r, backoff=ob.BackoffPolicy(backoff), sleep_base_ns=100)
        with ob.Heap(hc) as h:
            ts = []
            for it in range(4):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); h.launch_alloc(n, ptrs, size=8192); b.record(); b.synchronize()
                ts.append(a.elapsed_time(b) * 1000)
                h.launch_free(n, ptrs); torch.cuda.synchronize()
            print(f"backoff={backoff} max_retries={r:3d} alloc_us={min(ts[1:]):8.1f}")
