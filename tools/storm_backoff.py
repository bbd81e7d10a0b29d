"""OOM-storm alloc time (PQ 1 GiB, 2^20 x malloc(8192)) under each backoff policy:
FenceRetry (default: fence.sc.cta per round) vs SleepRetry with tiny sleeps -- the
cost the per-round fence adds to the retry rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
for name, kw in (("fence", dict()),
                 ("sleep 1..32 ns", dict(backoff=ob.BackoffPolicy(1), sleep_base_ns=1, sleep_cap_ns=32)),
                 ("sleep 100 ns..100 us (SPEC default)", dict(backoff=ob.BackoffPolicy(1)))):
    with ob.Heap(ob.HeapConfig(1 << 30, **kw)) as h:
        ts = []
        for it in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); h.launch_alloc(n, ptrs, size=8192); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
            h.launch_free(n, ptrs); torch.cuda.synchronize()
        print(f"{name:40s} alloc_us={min(ts[1:]):8.1f}")
