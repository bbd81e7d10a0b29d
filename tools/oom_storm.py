"""One 2^20-thread malloc(SIZE) on the PQ (or CQ) 1 GiB heap: an OOM storm with the
default max_retries.  For ncu: ncu -k regex:k_alloc -s 2 -c 1 python tools/oom_storm.py [size] [kind]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

size = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
with ob.Heap(ob.HeapConfig(1 << 30, allocator_kind=ob.AllocatorKind(kind))) as h:
    for it in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_alloc(n, ptrs, size=size); b.record(); b.synchronize()
        print(f"alloc_us={a.elapsed_time(b) * 1000:.1f}")
        h.launch_free(n, ptrs); torch.cuda.synchronize()
