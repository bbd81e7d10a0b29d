"""2^20-thread malloc(SIZE) / free cycles on an 8 GiB heap of a virtual flavour, for ncu:
ncu -k regex:k_alloc -s 2 -c 1 python tools/va_storm.py [size] [kind] [flavor]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

size = int(sys.argv[1]) if len(sys.argv) > 1 else 16
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
flavor = int(sys.argv[3]) if len(sys.argv) > 3 else 1
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
hc = ob.HeapConfig(8 << 30, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
with ob.Heap(hc) as h:
    for it in range(4):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(); h.launch_alloc(n, ptrs, size=size); b.record()
        h.launch_free(n, ptrs); c.record(); c.synchronize()
        print(f"alloc_us={a.elapsed_time(b) * 1000:.1f} free_us={b.elapsed_time(c) * 1000:.1f}")
