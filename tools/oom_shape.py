"""OOM-storm alloc (2^20 x malloc(8192) on the PQ 1 GiB heap, ~99% OOM) for
max_retries 1 / 2 / 64 under the one-thread-per-request and persistent launch shapes:
separates the first-try storm from the retry rounds."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18211_b200 as ob
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
for waves in (0, 1):
    ob.check(ob.lib().ouro_set_launch_shape(256, waves), "shape")
    for r in (1, 2, 64):
        with ob.Heap(ob.HeapConfig(1 << 30, max_retries=r)) as h:
            ts = []
            for it in range(4):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); h.launch_alloc(n, ptrs, size=8192); b.record(); b.synchronize()
                ts.append(a.elapsed_time(b) * 1000)
                h.launch_free(n, ptrs); torch.cuda.synchronize()
            print(f"waves={waves} max_retries={r:3d} alloc_us={min(ts[1:]):8.1f}")
